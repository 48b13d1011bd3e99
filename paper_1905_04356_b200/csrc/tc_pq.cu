// tc_pq.cu -- int8 tensor-core per-point products for small matrices
// (m <= 32: BASELINE cfg2 32x32x32, cfg3 16x16x16 per CRT prime) on the
// point-quad eval layout X[t/4][entry][t%4] that the blocked NTT kernels write
// with full-speed 16-byte stores (ntt.cuh eval_piece, pblk_log = 2).
// Replaces the per-point `_dense.mat_mul(a, b, p)` loop of `_pm_mul_ntt`
// (polmat.py:300; _dense.py:39-74).
//
// Arithmetic (tc_pointwise.cu): with s_q = 2^(8q) B mod p,
//   C = sum_r 2^(8r) D_r,  D_r[i][j] = sum_{l,q} byte_q(A[i][l]) byte_r(s_q[l][j]),
// one u8 x u8 -> s32 UMMA with K' = 4k (raw bytes of A) and N' = 4n.
//
// Grouping (tc_grouped.cu): mp = 16 or 32 (next power of two >= m),
// G = 128/mp points share one M = 128 tile (rows g*mp + i); point g is
// multiplied by its own B operand into its own TMEM accumulator, and only
// its lanes are read back.
//
// Layout work happens in shared memory, so every global access is a
// contiguous TMA box or a coalesced 16-byte store:
//   * TMA loads raw A [quad][i][l][4 pts] and raw B [quad][l][j][4 pts]
//     ((l, pt) and (j, pt) merged: 512-byte box rows, contiguous per quad);
//   * 2 "A warps" transpose raw A into the K-major SWIZZLE_128B UMMA tile;
//   * 8 "B warps" build each point's B operand (3 lazy Shoup scalings and a
//     4x4 byte transpose per element);
//   * 4 epilogue warps (one per TMEM lane quadrant) reduce the accumulators,
//     regroup the 4 points of each output entry through a swizzled staging
//     tile and store 16-byte point-quad pieces, fully coalesced.
// Warp 0 issues TMA, warp 1 owns TMEM and issues the MMAs.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "tc_common.cuh"
#include "tc_pointwise.cuh"

namespace fpm {
namespace {

constexpr int kEpiWarp0 = 2, kEpiWarps = 8;  // two per TMEM lane quadrant
constexpr int kBWarp0 = kEpiWarp0 + kEpiWarps, kBWarps = 8, kBThreads = kBWarps * 32;
constexpr int kAWarp0 = kBWarp0 + kBWarps, kAWarps = 2, kAThreads = kAWarps * 32;
constexpr int kThreads = (kAWarp0 + kAWarps) * 32;  // 20 warps (5 per SMSP, <= 102 regs)
constexpr int NSA = 3, NSB = 2;             // raw A / raw B load stages
constexpr uint32_t kRawA = 16384, kRawB = 16384;
constexpr int NA = 2;                       // A tile ring
constexpr uint32_t kTileA = 16384;          // 128 rows x 128 B, SWIZZLE_128B
constexpr uint32_t kStaging = 16384;        // one item's C values
constexpr int NSTG = 1;                     // staging buffers
constexpr uint32_t kSboB = 1040;            // B tile: 8 N' rows x 128 B + 16 B pad
constexpr uint32_t kRing = 80 * kSboB;      // B tile ring (83200 B)
constexpr uint32_t kOffA = 0;                               // 1 KB aligned
constexpr uint32_t kOffRawA = kOffA + NA * kTileA;
constexpr uint32_t kOffRawB = kOffRawA + NSA * kRawA;
constexpr uint32_t kOffStg = kOffRawB + NSB * kRawB;
constexpr uint32_t kOffRing = kOffStg + NSTG * kStaging;
constexpr size_t kSmem = kOffRing + kRing + 1024;
constexpr int kMaxRing = 24, kMaxAcc = 16;
constexpr int kPf = 3;                      // L2 prefetch distance (items)

struct QArgs {
  uint32_t* C;
  int m, k, n, npts, nz;
  long long c_ps;   // per-prime stride of C (words)
  int mp, G, nblk, ngroups, nch;
  int nring, nacc;
  int dbg;          // profiling only (FPM_TCPQ_DBG): skip stages, results invalid
  unsigned long long* trace;  // profiling only: per-item timestamps of CTA 0
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// trace slot: item (local index < 64) x event (< 8)
#define TRACE(ev, li)                                                       \
  if (a.trace && blockIdx.x == 0 && (li) < 64) a.trace[(li) * 8 + (ev)] = gtime();

struct RingPos {
  int idx;
  uint32_t ph;
  __device__ __forceinline__ void next(int n) {
    if (++idx == n) {
      idx = 0;
      ph ^= 1u;
    }
  }
};

__device__ __forceinline__ void decode(const QArgs& a, int it, int& z, int& gi, int& jb) {
  const int per_z = a.ngroups * a.nblk;
  z = it / per_z;
  const int rem = it - z * per_z;
  gi = rem / a.nblk;
  jb = rem - gi * a.nblk;
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t x, uint32_t y, uint32_t z,
                                             uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(x), "r"(y), "r"(z),
               "r"(w)
               : "memory");
}
__device__ __forceinline__ void st_shared_u32(uint32_t addr, uint32_t x) {
  asm volatile("st.shared.b32 [%0], %1;\n" ::"r"(addr), "r"(x) : "memory");
}
__device__ __forceinline__ uint4 ld_shared_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_shared_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];\n" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void epi_bar() {
  asm volatile("bar.sync 1, %0;\n" ::"n"(kEpiWarps * 32) : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const void* tmap, uint32_t mbar, int c0,
                                            int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5, %6}], [%2];\n" ::"r"(dst),
      "l"(tmap), "r"(mbar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_4d(const void* tmap, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.prefetch.tensor.4d.L2.global [%0, {%1, %2, %3, %4}];\n" ::"l"(tmap),
      "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void expect_tx(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mbar),
               "r"(bytes)
               : "memory");
}

template <int NB>
__global__ void __launch_bounds__(kThreads, 1)
    tc_pq_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ QArgs a, const __grid_constant__ PrimeSet ps) {
  constexpr uint32_t kTileB = (NB / 2) * kSboB;  // 4 NB rows of 128 B (+ pad)
  constexpr int kChunks = NB / 4;                // 16-byte chunks per staging row
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t fullA[NSA], emptyA[NSA], fullB[NSB], emptyB[NSB], afull[NA], aempty[NA];
  __shared__ uint64_t bfull[kMaxRing], bempty[kMaxRing], tfull[kMaxAcc], tempty[kMaxAcc];
  __shared__ uint32_t tmem_base;
  const uint32_t sraw = tc::smem_u32(smem_raw);
  const uint32_t sbase = (sraw + 1023u) & ~1023u;
  const uint32_t b_fullA = tc::smem_u32(fullA), b_emptyA = tc::smem_u32(emptyA);
  const uint32_t b_fullB = tc::smem_u32(fullB), b_emptyB = tc::smem_u32(emptyB);
  const uint32_t b_afull = tc::smem_u32(afull), b_aempty = tc::smem_u32(aempty);
  const uint32_t b_bfull = tc::smem_u32(bfull), b_bempty = tc::smem_u32(bempty);
  const uint32_t b_tfull = tc::smem_u32(tfull), b_tempty = tc::smem_u32(tempty);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = a.G, nch = a.nch, nring = a.nring, nacc = a.nacc, m = a.m, mp = a.mp;
  const int items = a.nz * a.ngroups * a.nblk;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmB);
    for (int s = 0; s < NSA; ++s) {
      tc::mbar_init(&fullA[s], 1);
      tc::mbar_init(&emptyA[s], kAWarps);
    }
    for (int s = 0; s < NSB; ++s) {
      tc::mbar_init(&fullB[s], 1);
      tc::mbar_init(&emptyB[s], kBWarps);
    }
    for (int s = 0; s < NA; ++s) {
      tc::mbar_init(&afull[s], kAWarps);
      tc::mbar_init(&aempty[s], 1);
    }
    for (int e = 0; e < nring; ++e) {
      tc::mbar_init(&bfull[e], kBWarps);
      tc::mbar_init(&bempty[e], 1);
    }
    for (int c = 0; c < nacc; ++c) {
      tc::mbar_init(&tfull[c], 1);
      tc::mbar_init(&tempty[c], 2);  // mp <= 32: the two warps of one quadrant
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(&tmem_base, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  pdl_wait();  // operands come from the forward transforms
  pdl_trigger();
  const uint32_t tmem = tmem_base;
  const int nq = G / 4;  // point quads per item

  if (warp == 0) {
    // ------------------------------ TMA producer ------------------------------
    if (lane == 0) {
      const uint32_t bytesA = (uint32_t)(nq * m * 32 * 16), bytesB = (uint32_t)(nq * 32 * NB * 16);
      RingPos sa{0, 0}, sb{0, 0};
      for (int it = blockIdx.x; it < items; it += gridDim.x) {
        int z, gi, jb;
        decode(a, it, z, gi, jb);
        // warm L2 with the item kPf steps ahead: the TMA loads below then see
        // L2 latency instead of DRAM latency under load
        {
          const int itp = it + kPf * (int)gridDim.x;
          if (itp < items) {
            int zp, gp, jp;
            decode(a, itp, zp, gp, jp);
            for (int ch = 0; ch < nch; ++ch) {
              tma_prefetch_4d(&tmA, ch * 128, 0, gp * nq, zp);
              tma_prefetch_4d(&tmB, jp * NB * 4, ch * 32, gp * nq, zp);
            }
          }
        }
        for (int ch = 0; ch < nch; ++ch, sa.next(NSA), sb.next(NSB)) {
          tc::mbar_wait_a(b_emptyA + 8 * sa.idx, sa.ph ^ 1u);
          expect_tx(b_fullA + 8 * sa.idx, bytesA);
          tma_load_4d(sbase + kOffRawA + sa.idx * kRawA, &tmA, b_fullA + 8 * sa.idx, ch * 128, 0,
                      gi * nq, z);
          tc::mbar_wait_a(b_emptyB + 8 * sb.idx, sb.ph ^ 1u);
          expect_tx(b_fullB + 8 * sb.idx, bytesB);
          tma_load_4d(sbase + kOffRawB + sb.idx * kRawB, &tmB, b_fullB + 8 * sb.idx, jb * NB * 4,
                      ch * 32, gi * nq, z);
          TRACE(0, (it - (int)blockIdx.x) / (int)gridDim.x);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------- MMA issuer -------------------------------
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_u8(128, 4 * NB);
      RingPos at{0, 0}, br{0, 0}, ac{0, 0};
      for (int it = blockIdx.x; it < items; it += gridDim.x) {
        for (int ch = 0; ch < nch; ++ch, at.next(NA)) {
          tc::mbar_wait_a(b_afull + 8 * at.idx, at.ph);
          tc::fence_after_sync();
          const uint32_t tA = sbase + kOffA + at.idx * kTileA;
          RingPos acc = ac;
          for (int g = 0; g < G; ++g, br.next(nring), acc.next(nacc)) {
            tc::mbar_wait_a(b_bfull + 8 * br.idx, br.ph);
            if (ch == 0) tc::mbar_wait_a(b_tempty + 8 * acc.idx, acc.ph ^ 1u);
            tc::fence_after_sync();
            const uint32_t tB = sbase + kOffRing + br.idx * kTileB;
            const uint32_t d = tmem + acc.idx * 4 * NB;
#pragma unroll
            for (int ks = 0; ks < ((a.dbg & 8) ? 0 : 4); ++ks)
              tc::mma_u8(d, tc::make_desc_sw128(tA + ks * 32),
                         tc::make_desc(tB + ks * 256, 128, kSboB), idesc,
                         (ch > 0 || ks > 0) ? 1u : 0u);
            tc::commit_a(b_bempty + 8 * br.idx);
            if (ch == nch - 1) tc::commit_a(b_tfull + 8 * acc.idx);
          }
          tc::commit_a(b_aempty + 8 * at.idx);
          TRACE(5, (it - (int)blockIdx.x) / (int)gridDim.x);
        }
        for (int g = 0; g < G; ++g) ac.next(nacc);
      }
    }
  } else if (warp < kBWarp0) {
    // -------------------------------- epilogue --------------------------------
    // warp pair (q, half): TMEM lane quadrant q, half of the accumulator
    // columns; both TMEM loads are issued before the slot is released, so the
    // MMAs of the next item overlap the reduction below
    const int q = warp & 3, half = (warp - kEpiWarp0) >> 2;
    constexpr int kLoads = NB / 8;                     // x32 loads per accumulator row
    constexpr int kMine = kLoads >= 2 ? kLoads / 2 : 1;  // per warp (<= 2)
    const bool active = kLoads >= 2 || half == 0;
    // points of this quadrant: one (mp = 32) or two (mp = 16, lanes 0-15 / 16-31)
    const int g_lo = (32 * q) / mp, g_hi = (32 * q + 31) / mp;
    const int sub = nacc / G;
    RingPos sp0{0, 0}, sp1{0, 0};
    int parity = 0;
    for (int it = blockIdx.x; it < items; it += gridDim.x, parity ^= 1) {
      int z, gi, jb;
      decode(a, it, z, gi, jb);
      const uint32_t p = ps.pr[z].p, m58 = ps.pr[z].m58;
      const uint32_t stg = sbase + kOffStg + (NSTG == 2 ? parity : 0) * kStaging;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int g = g_lo + u;
        if (g > g_hi) break;
        RingPos& r = u ? sp1 : sp0;
        const int slot = r.idx * G + g;
        tc::mbar_wait_a(b_tfull + 8 * slot, r.ph);
        if (lane == 0 && q == 0 && half == 0) TRACE(6, (it - (int)blockIdx.x) / (int)gridDim.x);
        tc::fence_after_sync();
        const int i = 32 * q + lane - g * mp;  // row of point g held by this lane
        const bool ok = i >= 0 && i < m;
        uint32_t v[2][32];
        if (active && !(a.dbg & 2)) {
#pragma unroll
          for (int c2 = 0; c2 < kMine; ++c2)
            tc::tmem_ld32_nw(tmem + ((uint32_t)(32 * q) << 16) + slot * 4 * NB +
                                 32 * (half * kMine + c2),
                             v[c2]);
          tc::tmem_wait_ld();
        }
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_a(b_tempty + 8 * slot);
        r.next(sub);
        if (active && !(a.dbg & 2)) {
#pragma unroll
          for (int c2 = 0; c2 < kMine; ++c2) {
            const int cc = half * kMine + c2;
            uint32_t o[8];
#pragma unroll
            for (int x = 0; x < 8; ++x) {
              uint64_t s = (uint64_t)v[c2][4 * x];
              s += (uint64_t)v[c2][4 * x + 1] << 8;
              s += (uint64_t)v[c2][4 * x + 2] << 16;
              s += (uint64_t)v[c2][4 * x + 3] << 24;
              o[x] = d_red56(s, p, m58);
            }
            if (ok) {
              // staging S[(i * G + g) * NB + 4 * (chunk ^ swz(i)) + w]
              const uint32_t row = stg + (uint32_t)((i * G + g) * NB) * 4;
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int c = 2 * cc + h;
                st_shared_v4(row + 16 * (c ^ (i & (kChunks - 1))), o[4 * h], o[4 * h + 1],
                             o[4 * h + 2], o[4 * h + 3]);
              }
            }
          }
        }
      }
      epi_bar();  // the item's staging tile is complete
      // 16-byte point-quad pieces C[quad][i*n + j][0..3], consecutive threads ->
      // consecutive j: fully coalesced
      const int j0 = jb * NB;
      const int ec = m * a.n;
      uint32_t* Cz = a.C + z * a.c_ps;
      const int ew = warp - kEpiWarp0;  // 0..7
      for (int qq = 0; qq < ((a.dbg & 16) ? 0 : nq); ++qq) {
        const int tq = gi * nq + qq;
        if (4 * tq >= a.npts) break;
        for (int i = ew; i < m; i += kEpiWarps) {
          for (int j = lane; j < NB; j += 32) {
            const int gj = j0 + j;
            if (gj >= a.n) break;
            const uint32_t base =
                stg + 4 * ((i * G + 4 * qq) * NB + 4 * ((j >> 2) ^ (i & (kChunks - 1))) + (j & 3));
            uint32_t w[4];
#pragma unroll
            for (int g4 = 0; g4 < 4; ++g4) w[g4] = ld_shared_u32(base + 4 * g4 * NB);
            *reinterpret_cast<uint4*>(Cz + ((long long)tq * ec + (long long)i * a.n + gj) * 4) =
                make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      }
      if (NSTG == 1) epi_bar();  // staging drained before the next item's writes
      if (lane == 0 && q == 0) TRACE(7, (it - (int)blockIdx.x) / (int)gridDim.x);
    }
  } else if (warp < kAWarp0) {
    // -------------------------------- B builders -------------------------------
    const int ct = tid - kBWarp0 * 32;
    RingPos st{0, 0}, br{0, 0};
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
      int z, gi, jb;
      decode(a, it, z, gi, jb);
      const PrimeConst& pc = ps.pr[z];
      const uint32_t p = pc.p;
      const uint32_t w1 = pc.sc[1].x, w1p = pc.sc[1].y, w2 = pc.sc[2].x, w2p = pc.sc[2].y;
      const uint32_t w3 = pc.sc[3].x, w3p = pc.sc[3].y;
      for (int ch = 0; ch < nch; ++ch, st.next(NSB)) {
        // every builder thread owns at most one task per (item, chunk): it
        // copies its raw values to registers and frees the stage at once
        const int base_tasks = nq * 8 * NB;
        const int split = base_tasks >= kBThreads ? 1 : (2 * base_tasks >= kBThreads ? 2 : 4);
        const int ppt = 4 / split;
        const int task = ct;
        const bool has = task < base_tasks * split && !(a.dbg & 1);
        const int part = task / base_tasks, t0 = task - part * base_tasks;
        const int j = t0 % NB, rest = t0 / NB;
        const int lq = rest % 8, qq = rest / 8;
        const int g_lo = part * ppt, g_hi = g_lo + ppt;
        uint4 raw[4];
        tc::mbar_wait_a(b_fullB + 8 * st.idx, st.ph);
        if (ct == 0) TRACE(3, (it - (int)blockIdx.x) / (int)gridDim.x);
        if (has) {
          const uint32_t rawB = sbase + kOffRawB + st.idx * kRawB;
#pragma unroll
          for (int uu = 0; uu < 4; ++uu)
            raw[uu] = ld_shared_v4(rawB + (uint32_t)(((qq * 32 + 4 * lq + uu) * NB + j) * 16));
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_a(b_emptyB + 8 * st.idx);
        {
          RingPos r = br;
          for (int u = 0; u < G; ++u, r.next(nring))
            tc::mbar_wait_a(b_bempty + 8 * r.idx, r.ph ^ 1u);
        }
        if (has) {
#pragma unroll
          for (int g4 = 0; g4 < 4; ++g4) {
            if (g4 < g_lo || g4 >= g_hi) continue;
            uint32_t w[4][4];  // [r][u]
#pragma unroll
            for (int uu = 0; uu < 4; ++uu) {
              const uint32_t b = g4 == 0 ? raw[uu].x : g4 == 1 ? raw[uu].y : g4 == 2 ? raw[uu].z
                                                                                    : raw[uu].w;
              const uint32_t s1 = d_shoup(b, w1, w1p, p);
              const uint32_t s2 = d_shoup(b, w2, w2p, p);
              const uint32_t s3 = d_shoup(b, w3, w3p, p);
              const uint32_t lo0 = __byte_perm(b, s1, 0x5140);
              const uint32_t hi0 = __byte_perm(b, s1, 0x7362);
              const uint32_t lo1 = __byte_perm(s2, s3, 0x5140);
              const uint32_t hi1 = __byte_perm(s2, s3, 0x7362);
              w[0][uu] = __byte_perm(lo0, lo1, 0x5410);
              w[1][uu] = __byte_perm(lo0, lo1, 0x7632);
              w[2][uu] = __byte_perm(hi0, hi1, 0x5410);
              w[3][uu] = __byte_perm(hi0, hi1, 0x7632);
            }
            int e = br.idx + 4 * qq + g4;
            if (e >= nring) e -= nring;
            const uint32_t tB = sbase + kOffRing + e * kTileB + lq * 128 + (j >> 1) * kSboB +
                                (j & 1) * 64;
#pragma unroll
            for (int r = 0; r < 4; ++r)
              st_shared_v4(tB + r * 16, w[r][0], w[r][1], w[r][2], w[r][3]);
          }
        }
        tc::fence_proxy_async();
        __syncwarp();
        for (int u = 0; u < G; ++u, br.next(nring))
          if (lane == 0) tc::mbar_arrive_a(b_bfull + 8 * br.idx);
        if (ct == 0) TRACE(4, (it - (int)blockIdx.x) / (int)gridDim.x);
      }
    }
  } else {
    // -------------------------------- A builders -------------------------------
    // raw [quad][i][l][4 pts] -> UMMA rows g*mp + i, 128 B of l, SWIZZLE_128B
    RingPos st{0, 0}, at{0, 0};
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
      for (int ch = 0; ch < nch; ++ch, st.next(NSA), at.next(NA)) {
        // claim the A tile first, so a raw stage is never held while waiting
        tc::mbar_wait_a(b_aempty + 8 * at.idx, at.ph ^ 1u);
        tc::mbar_wait_a(b_fullA + 8 * st.idx, st.ph);
        const uint32_t rawA = sbase + kOffRawA + st.idx * kRawA;
        if (lane == 0 && warp == kAWarp0) TRACE(1, (it - (int)blockIdx.x) / (int)gridDim.x);
        const uint32_t tA = sbase + kOffA + at.idx * kTileA;
        // one (quad, row) per warp iteration, lane = l: LDS.128 of 4 points,
        // four STS.32 into the rows of those points (conflict-free both ways)
        const int aw = warp - kAWarp0;
        for (int qq = 0; qq < nq; ++qq) {
          for (int i = aw; i < ((a.dbg & 4) ? 0 : m); i += kAWarps) {
            const uint4 v = ld_shared_v4(rawA + (uint32_t)(((qq * m + i) * 32 + lane) * 16));
#pragma unroll
            for (int g4 = 0; g4 < 4; ++g4) {
              const int r = (4 * qq + g4) * mp + i;
              const uint32_t val = g4 == 0 ? v.x : g4 == 1 ? v.y : g4 == 2 ? v.z : v.w;
              st_shared_u32(tA + r * 128 + ((((lane >> 2) ^ (r & 7)) << 4) | ((lane & 3) << 2)),
                            val);
            }
          }
        }
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          tc::mbar_arrive_a(b_afull + 8 * at.idx);
          if (warp == kAWarp0) TRACE(2, (it - (int)blockIdx.x) / (int)gridDim.x);
          tc::mbar_arrive_a(b_emptyA + 8 * st.idx);
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

int make_map4(CUtensorMap* map, const uint32_t* base, const uint64_t dims[4],
              const uint64_t strides[3], const uint32_t box[4]) {
  auto fn = encode_fn();
  if (!fn) {
    set_last_error("cuTensorMapEncodeTiled unavailable");
    return kCudaError;
  }
  const cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, const_cast<uint32_t*>(base), dims,
                  strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_last_error("cuTensorMapEncodeTiled (4-D) failed (%d)", (int)r);
    return kCudaError;
  }
  return kOk;
}

template <int NB>
int launch_nb(const CUtensorMap& mA, const CUtensorMap& mB, const QArgs& a, const PrimeSet& ps,
              unsigned grid, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    FPM_CUDA_TRY(cudaFuncSetAttribute(tc_pq_kernel<NB>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
    attr = true;
  }
  const cudaError_t lerr = launch_pdl(tc_pq_kernel<NB>, dim3(grid), dim3(kThreads), kSmem, st, mA, mB, a, ps);
  const cudaError_t err = lerr != cudaSuccess ? lerr : cudaGetLastError();
  if (err != cudaSuccess) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, tc_pq_kernel<NB>);
    set_last_error("tc_pq launch (%s): regs %d maxThreads %d static smem %zu max dyn %d req %zu",
                   cudaGetErrorString(err), fa.numRegs, fa.maxThreadsPerBlock,
                   fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes, kSmem);
    return kCudaError;
  }
  ++g_launch_count;
  return kOk;
}

unsigned long long* trace = nullptr;  // FPM_TCPQ_DBG & 32: per-item timestamps

}  // namespace

bool tc_pq_applicable(int m, int k, int n, int npts, uint32_t p) {
  // k <= 8192: see tc_grouped_applicable (accumulator bound D_r < 2^31)
  return p < (1u << 31) && p >= (1u << 30) && m >= 1 && m <= 32 && k >= 1 && k <= kTcMaxK &&
         n >= 1 && (npts % 8) == 0;
}

int launch_tc_pq(const TcArgs& t, const PrimeSet& ps, cudaStream_t st) {
  if (t.npts <= 0 || t.m <= 0 || t.n <= 0) return kOk;
  for (int i = 0; i < ps.count; ++i)
    if (!tc_pq_applicable(t.m, t.k, t.n, t.npts, ps.pr[i].p)) {
      set_last_error("tc_pq: unsupported shape %dx%dx%d", t.m, t.k, t.n);
      return kInvalidArgument;
    }
  QArgs a{};
  a.C = t.C; a.m = t.m; a.k = t.k; a.n = t.n; a.npts = t.npts; a.nz = ps.count;
  a.c_ps = t.c_ps;
#ifdef FPM_TRACE
  // profiling build only (tools/tcpq_trace.py): per-item phase clocks
  static const int dbg = std::getenv("FPM_TCPQ_DBG") ? std::atoi(std::getenv("FPM_TCPQ_DBG")) : 0;
  a.dbg = dbg;
  if ((dbg & 32) && !trace) {
    cudaMalloc(&trace, 64 * 8 * sizeof(unsigned long long));
    cudaMemset(trace, 0, 64 * 8 * sizeof(unsigned long long));
  }
  a.trace = (dbg & 32) ? trace : nullptr;
#else
  a.dbg = 0;
  a.trace = nullptr;
#endif
  a.mp = t.m <= 16 ? 16 : 32;
  a.G = 128 / a.mp;
  // NB: power of two, G accumulators of 4 NB columns fit the 512 TMEM columns
  // NB <= mp/2 when FPM_TCPQ_HALF: TMEM holds two items' accumulators
  int nb = 8;
  while (nb < t.n && nb < a.mp) nb <<= 1;
  a.nblk = (t.n + nb - 1) / nb;
  a.ngroups = (t.npts + a.G - 1) / a.G;
  a.nch = (t.k + 31) / 32;
  const uint32_t tileB = (uint32_t)(nb / 2) * kSboB;
  a.nring = (int)(kRing / tileB);
  if (a.nring > kMaxRing) a.nring = kMaxRing;
  a.nacc = 512 / (4 * nb);
  if (a.nacc > kMaxAcc) a.nacc = kMaxAcc;
  const long long items = (long long)ps.count * a.ngroups * a.nblk;
  if (items >= (1LL << 31)) {
    set_last_error("tc_pq: too many work items");
    return kUnsupported;
  }
  const uint64_t nz = (uint64_t)ps.count, nquad = (uint64_t)t.npts / 4;
  // (l, point) and (j, point) are contiguous inside a quad, so the boxes have
  // 512-byte inner rows (one TMA request per row, not per 16-byte piece)
  CUtensorMap mA, mB;
  {
    // A: [z][quad][i][(l, 4)]
    const uint64_t dims[4] = {(uint64_t)t.k * 4, (uint64_t)t.m, nquad, nz};
    const uint64_t ps_b = (uint64_t)(t.a_ps ? t.a_ps : (long long)t.npts * t.m * t.k) * 4;
    const uint64_t strides[3] = {(uint64_t)t.k * 16, (uint64_t)t.m * t.k * 16, ps_b};
    const uint32_t box[4] = {128, (uint32_t)t.m, (uint32_t)(a.G / 4), 1};
    FPM_TRY(make_map4(&mA, t.A, dims, strides, box));
  }
  {
    // B: [z][quad][l][(j, 4)]
    const uint64_t dims[4] = {(uint64_t)t.n * 4, (uint64_t)t.k, nquad, nz};
    const uint64_t ps_b = (uint64_t)(t.b_ps ? t.b_ps : (long long)t.npts * t.k * t.n) * 4;
    const uint64_t strides[3] = {(uint64_t)t.n * 16, (uint64_t)t.k * t.n * 16, ps_b};
    const uint32_t box[4] = {(uint32_t)(4 * nb), 32, (uint32_t)(a.G / 4), 1};
    FPM_TRY(make_map4(&mB, t.B, dims, strides, box));
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const unsigned grid = (unsigned)(items < sms ? items : sms);
  switch (nb) {
    case 8: return launch_nb<8>(mA, mB, a, ps, grid, st);
    case 16: return launch_nb<16>(mA, mB, a, ps, grid, st);
    default: return launch_nb<32>(mA, mB, a, ps, grid, st);
  }
}

}  // namespace fpm

// profiling only: timestamps recorded by CTA 0 under FPM_TCPQ_DBG & 32
#ifdef FPM_TRACE
extern "C" int fpm_debug_tcpq_trace(unsigned long long* host) {
  if (!fpm::trace) return 1;
  cudaDeviceSynchronize();
  cudaMemcpy(host, fpm::trace, 64 * 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  return 0;
}
#endif
