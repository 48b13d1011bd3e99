// tc_pq2.cu -- int8 tensor-core per-point products for m, n <= 32 on the
// point-quad eval layout X[t/4][entry][t%4] (BASELINE cfg2: 32x32x32 per
// point), limbs on the M side.  Replaces the per-point
// `_dense.mat_mul(a, b, p)` loop of `_pm_mul_ntt` (polmat.py:300;
// _dense.py:39-74).
//
// Arithmetic.  With b_q the raw little-endian bytes of B and
// s_q = 2^(8q) A mod p,
//   C[i][j] = sum_{l,q} s_q[i][l] b_q[l][j] = sum_r 2^(8r) D_r[i][j],
//   D_r[i][j] = sum_{l,q} byte_r(s_q[i][l]) * b_q[l][j],
// so per point ONE u8 x u8 -> s32 UMMA with M = 4m rows (4i + r), N = n
// columns and K' = 4k (the raw bytes of B^T) gives every D_r; D_r < 4k 255^2
// and sum_r 2^(8r) D_r < 2^56 (d_red56).
//
// Compared with tc_pq.cu (limbs on N, four points per M tile) a point needs
// only n = 32 TMEM columns (16 points in flight instead of 4) and the tensor
// core does no padding work; the limb sum moves into the epilogue as a
// two-step shuffle reduce-scatter inside each group of 4 lanes.
//
// Warp roles (persistent, one CTA per SM, 20 warps), one item = one quad of
// points (4), one K chunk = 32 l:
//   warp 0      TMA producer: raw A [i][l][4 pts], raw B [l][j][4 pts]
//   warp 1      TMEM owner, single-thread MMA issuer (M128 N32 K32, 4 per chunk)
//   warps 2-9   epilogue (TMEM lane quadrant q = rows i of 8q..8q+7; two
//               warps per quadrant take alternate points): tcgen05.ld, limb
//               reduce-scatter, d_red56, quad regrouping in a staging tile,
//               coalesced 16-byte stores
//   warps 10-17 A builders: 3 lazy Shoup scalings + 4x4 byte transpose per
//               element into per-point K-major tiles (LBO 144 B: the stores of
//               8 consecutive K chunks hit 8 different bank groups)
//   warps 18-19 B^T builders: u32 transpose of raw B into K-major tiles
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "tc_common.cuh"
#include "tc_pointwise.cuh"

namespace fpm {
namespace {

constexpr int kEpiWarp0 = 2, kEpiWarps = 8;  // two per TMEM lane quadrant
constexpr int kAWarp0 = 10, kAWarps = 8, kAThreads = kAWarps * 32;
constexpr int kBWarp0 = 18, kBWarps = 2, kBThreads = kBWarps * 32;
constexpr int kThreads = 20 * 32;             // 5 warps per SMSP: <= 102 registers
constexpr int NSA = 2, NSB = 2;             // raw load stages
constexpr uint32_t kRaw = 16384;            // one quad block (4 pts x 32 x 32 x 4 B)
constexpr uint32_t kLboA = 144, kSboA = 8 * kLboA;   // A'' tile: 16 row groups
constexpr uint32_t kTileA = 16 * kSboA;               // 18432 B
constexpr uint32_t kTileB = 4 * 1024;                 // B^T tile: 32 rows x 128 B
constexpr int kRingA = 5, kRingB = 8;
constexpr uint32_t kStaging = 16384;
constexpr uint32_t kOffRawA = 0;
constexpr uint32_t kOffRawB = kOffRawA + NSA * kRaw;
constexpr uint32_t kOffA = kOffRawB + NSB * kRaw;
constexpr uint32_t kOffB = kOffA + kRingA * kTileA;
constexpr uint32_t kOffStg = kOffB + kRingB * kTileB;
constexpr size_t kSmem = kOffStg + kStaging + 1024;
constexpr int kAcc = 16;                    // TMEM slots of 32 columns

struct Q2Args {
  uint32_t* C;
  int m, k, n, npts, nz, nquads, nch;
  long long c_ps;
  unsigned long long* trace;  // profiling only (FPM_TCPQ2_TRACE): CTA 0 timestamps
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
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

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t x, uint32_t y, uint32_t z,
                                             uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(x), "r"(y), "r"(z),
               "r"(w)
               : "memory");
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
__device__ __forceinline__ void expect_tx(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mbar),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ uint32_t pick(const uint4& v, int g) {
  return g == 0 ? v.x : g == 1 ? v.y : g == 2 ? v.z : v.w;
}

__global__ void __launch_bounds__(kThreads, 1)
    tc_pq2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  const __grid_constant__ Q2Args a, const __grid_constant__ PrimeSet ps) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t fullA[NSA], emptyA[NSA], fullB[NSB], emptyB[NSB];
  __shared__ uint64_t afull[kRingA], aempty[kRingA], bfull[kRingB], bempty[kRingB];
  __shared__ uint64_t tfull[kAcc], tempty[kAcc];
  __shared__ uint32_t tmem_base;
  const uint32_t sraw = tc::smem_u32(smem_raw);
  const uint32_t sbase = (sraw + 1023u) & ~1023u;
  const uint32_t b_fullA = tc::smem_u32(fullA), b_emptyA = tc::smem_u32(emptyA);
  const uint32_t b_fullB = tc::smem_u32(fullB), b_emptyB = tc::smem_u32(emptyB);
  const uint32_t b_afull = tc::smem_u32(afull), b_aempty = tc::smem_u32(aempty);
  const uint32_t b_bfull = tc::smem_u32(bfull), b_bempty = tc::smem_u32(bempty);
  const uint32_t b_tfull = tc::smem_u32(tfull), b_tempty = tc::smem_u32(tempty);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m = a.m, n = a.n, nch = a.nch;
  const int items = a.nz * a.nquads;

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
    for (int e = 0; e < kRingA; ++e) {
      tc::mbar_init(&afull[e], kAWarps);
      tc::mbar_init(&aempty[e], 1);
    }
    for (int e = 0; e < kRingB; ++e) {
      tc::mbar_init(&bfull[e], kBWarps);
      tc::mbar_init(&bempty[e], 1);
    }
    for (int c = 0; c < kAcc; ++c) {
      tc::mbar_init(&tfull[c], 1);
      tc::mbar_init(&tempty[c], 4);  // the four quadrant warps of one half
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(&tmem_base, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    // ------------------------------ TMA producer ------------------------------
    if (lane == 0) {
      const uint32_t bytesA = (uint32_t)(m * 32 * 16), bytesB = (uint32_t)(32 * n * 16);
      RingPos sa{0, 0}, sb{0, 0};
      for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const int z = it / a.nquads, tq = it - z * a.nquads;
        for (int ch = 0; ch < nch; ++ch, sa.next(NSA), sb.next(NSB)) {
          tc::mbar_wait_a(b_emptyA + 8 * sa.idx, sa.ph ^ 1u);
          expect_tx(b_fullA + 8 * sa.idx, bytesA);
          tma_load_4d(sbase + kOffRawA + sa.idx * kRaw, &tmA, b_fullA + 8 * sa.idx, ch * 128, 0,
                      tq, z);
          tc::mbar_wait_a(b_emptyB + 8 * sb.idx, sb.ph ^ 1u);
          expect_tx(b_fullB + 8 * sb.idx, bytesB);
          tma_load_4d(sbase + kOffRawB + sb.idx * kRaw, &tmB, b_fullB + 8 * sb.idx, 0, ch * 32,
                      tq, z);
          TRACE(0, (it - (int)blockIdx.x) / (int)gridDim.x);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------- MMA issuer -------------------------------
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_u8(128, 32);
      RingPos ra{0, 0}, rb{0, 0}, ac{0, 0};
      for (int it = blockIdx.x; it < items; it += gridDim.x) {
        for (int ch = 0; ch < nch; ++ch) {
          RingPos acc = ac;
          for (int g = 0; g < 4; ++g, ra.next(kRingA), rb.next(kRingB), acc.next(kAcc)) {
            tc::mbar_wait_a(b_afull + 8 * ra.idx, ra.ph);
            tc::mbar_wait_a(b_bfull + 8 * rb.idx, rb.ph);
            if (ch == 0) tc::mbar_wait_a(b_tempty + 8 * acc.idx, acc.ph ^ 1u);
            tc::fence_after_sync();
            const uint32_t tA = sbase + kOffA + ra.idx * kTileA;
            const uint32_t tB = sbase + kOffB + rb.idx * kTileB;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              tc::mma_u8(tmem + acc.idx * 32, tc::make_desc(tA + ks * 2 * kLboA, kLboA, kSboA),
                         tc::make_desc(tB + ks * 256, 128, 1024), idesc,
                         (ch > 0 || ks > 0) ? 1u : 0u);
            tc::commit_a(b_aempty + 8 * ra.idx);
            tc::commit_a(b_bempty + 8 * rb.idx);
            if (ch == nch - 1) tc::commit_a(b_tfull + 8 * acc.idx);
          }
        }
        TRACE(4, (it - (int)blockIdx.x) / (int)gridDim.x);
        for (int g = 0; g < 4; ++g) ac.next(kAcc);
      }
    }
  } else if (warp < kAWarp0) {

    // -------------------------------- epilogue --------------------------------
    // lane L of quadrant q holds D row 4i' + r (i = 8q + i', r = L & 3); after
    // the reduce-scatter, lane r of each group of 4 owns columns 8r .. 8r+7
    // half hw of the epilogue warps takes the points g with g % 2 == hw
    const int q = warp & 3, ip = lane >> 2, r = lane & 3, hw = (warp - kEpiWarp0) >> 2;
    const int i = 8 * q + ip;
    const uint32_t stg = sbase + kOffStg;
    RingPos ac{0, 0};
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
      const int z = it / a.nquads, tq = it - z * a.nquads;
      const uint32_t p = ps.pr[z].p, m58 = ps.pr[z].m58;
      for (int g = 0; g < 4; ++g, ac.next(kAcc)) {
        if ((g & 1) != hw) continue;
        tc::mbar_wait_a(b_tfull + 8 * ac.idx, ac.ph);
        if (g == 0 && q == 0 && lane == 0) TRACE(5, (it - (int)blockIdx.x) / (int)gridDim.x);
        tc::fence_after_sync();
        uint32_t v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + ac.idx * 32, v);
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_a(b_tempty + 8 * ac.idx);
        // step 1 (partner r ^ 2): keep columns [16 h, 16 h + 16), h = r >> 1
        const int h = r >> 1;
        uint64_t s16[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const uint32_t mine = h ? v[16 + c] : v[c];
          const uint32_t send = h ? v[c] : v[16 + c];
          const uint32_t recv = __shfl_xor_sync(0xffffffffu, send, 2);
          s16[c] = ((uint64_t)mine << (8 * r)) + ((uint64_t)recv << (8 * (r ^ 2)));
        }
        // step 2 (partner r ^ 1): keep [8 (r & 1), +8) of the 16
        const int h2 = r & 1;
        uint32_t o[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint64_t mine = h2 ? s16[8 + c] : s16[c];
          const uint64_t send = h2 ? s16[c] : s16[8 + c];
          const uint32_t lo = __shfl_xor_sync(0xffffffffu, (uint32_t)send, 1);
          const uint32_t hi = __shfl_xor_sync(0xffffffffu, (uint32_t)(send >> 32), 1);
          o[c] = d_red56(mine + (((uint64_t)hi << 32) | lo), p, m58);
        }
        // staging S[(i * 4 + g) * 32 + 8 r + c], 16-byte chunks XOR-swizzled by i
        if (i < m) {
          const uint32_t row = stg + (uint32_t)((i * 4 + g) * 32) * 4;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int ch16 = (2 * r + hh) ^ (i & 7);
            st_shared_v4(row + 16 * ch16, o[4 * hh], o[4 * hh + 1], o[4 * hh + 2],
                         o[4 * hh + 3]);
          }
        }
      }
      epi_bar();  // the quad's staging tile is complete
      if (q == 0 && hw == 0 && lane == 0) TRACE(6, (it - (int)blockIdx.x) / (int)gridDim.x);
      // C[quad][i*n + j][0..3], consecutive threads -> consecutive j (coalesced)
      uint32_t* Cz = a.C + z * a.c_ps;
      const int ec = m * n;
      const int ew = warp - kEpiWarp0;
      for (int ii = ew; ii < m; ii += kEpiWarps) {
        const int j = lane;
        if (j < n) {
          uint32_t w[4];
#pragma unroll
          for (int g4 = 0; g4 < 4; ++g4) {
            const int ch16 = (j >> 2) ^ (ii & 7);
            w[g4] = ld_shared_u32(stg + 4 * ((ii * 4 + g4) * 32 + 4 * ch16 + (j & 3)));
          }
          *reinterpret_cast<uint4*>(Cz + ((long long)tq * ec + (long long)ii * n + j) * 4) =
              make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
      epi_bar();  // staging drained before the next quad's writes
      if (q == 0 && hw == 0 && lane == 0) TRACE(7, (it - (int)blockIdx.x) / (int)gridDim.x);
    }
  } else if (warp < kBWarp0) {
    // -------------------------------- A builders -------------------------------
    // task (i, lq): 4 LDS.128 = 4 l x 4 points; per point 4 rows 4i + r of 16 B
    const int ct = tid - kAWarp0 * 32;
    const int i = ct >> 3, lq = ct & 7;
    RingPos st{0, 0}, ra{0, 0};
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
      const int z = it / a.nquads;
      const PrimeConst& pc = ps.pr[z];
      const uint32_t p = pc.p;
      const uint32_t w1 = pc.sc[1].x, w1p = pc.sc[1].y, w2 = pc.sc[2].x, w2p = pc.sc[2].y;
      const uint32_t w3 = pc.sc[3].x, w3p = pc.sc[3].y;
      for (int ch = 0; ch < nch; ++ch, st.next(NSA)) {
        uint4 raw[4];
        tc::mbar_wait_a(b_fullA + 8 * st.idx, st.ph);
        if (ct == 0) TRACE(1, (it - (int)blockIdx.x) / (int)gridDim.x);
        if (i < m) {
          const uint32_t rawA = sbase + kOffRawA + st.idx * kRaw;
#pragma unroll
          for (int uu = 0; uu < 4; ++uu)
            raw[uu] = ld_shared_v4(rawA + (uint32_t)((i * 32 + 4 * lq + uu) * 16));
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_a(b_emptyA + 8 * st.idx);
        {
          RingPos rr = ra;
          for (int u = 0; u < 4; ++u, rr.next(kRingA))
            tc::mbar_wait_a(b_aempty + 8 * rr.idx, rr.ph ^ 1u);
        }
        if (i < m) {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            uint32_t w[4][4];  // [r][u]
#pragma unroll
            for (int uu = 0; uu < 4; ++uu) {
              const uint32_t x = pick(raw[uu], g);
              const uint32_t s1 = d_shoup(x, w1, w1p, p);
              const uint32_t s2 = d_shoup(x, w2, w2p, p);
              const uint32_t s3 = d_shoup(x, w3, w3p, p);
              const uint32_t lo0 = __byte_perm(x, s1, 0x5140);
              const uint32_t hi0 = __byte_perm(x, s1, 0x7362);
              const uint32_t lo1 = __byte_perm(s2, s3, 0x5140);
              const uint32_t hi1 = __byte_perm(s2, s3, 0x7362);
              w[0][uu] = __byte_perm(lo0, lo1, 0x5410);
              w[1][uu] = __byte_perm(lo0, lo1, 0x7632);
              w[2][uu] = __byte_perm(hi0, hi1, 0x5410);
              w[3][uu] = __byte_perm(hi0, hi1, 0x7632);
            }
            int e = ra.idx + g;
            if (e >= kRingA) e -= kRingA;
            const uint32_t tA = sbase + kOffA + e * kTileA + lq * kLboA;
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) {
              const int R = 4 * i + rr;
              st_shared_v4(tA + (R >> 3) * kSboA + (R & 7) * 16, w[rr][0], w[rr][1], w[rr][2],
                           w[rr][3]);
            }
          }
        }
        tc::fence_proxy_async();
        __syncwarp();
        for (int u = 0; u < 4; ++u, ra.next(kRingA))
          if (lane == 0) tc::mbar_arrive_a(b_afull + 8 * ra.idx);
        if (ct == 0) TRACE(2, (it - (int)blockIdx.x) / (int)gridDim.x);
      }
    }
  } else {
    // ------------------------------- B^T builders ------------------------------
    // raw [l][j][4 pts] -> per point K-major rows j, bytes 4l .. 4l+3 = B[l][j]
    const int ct = tid - kBWarp0 * 32;
    RingPos st{0, 0}, rb{0, 0};
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
      for (int ch = 0; ch < nch; ++ch, st.next(NSB)) {
        tc::mbar_wait_a(b_fullB + 8 * st.idx, st.ph);
        {
          RingPos rr = rb;
          for (int u = 0; u < 4; ++u, rr.next(kRingB))
            tc::mbar_wait_a(b_bempty + 8 * rr.idx, rr.ph ^ 1u);
        }
        const uint32_t rawB = sbase + kOffRawB + st.idx * kRaw;
        for (int task = ct; task < 32 * 8; task += kBThreads) {
          const int j = task & 31, lq = task >> 5;
          uint4 raw[4];
#pragma unroll
          for (int uu = 0; uu < 4; ++uu)
            raw[uu] = j < n ? ld_shared_v4(rawB + (uint32_t)(((4 * lq + uu) * n + j) * 16))
                            : make_uint4(0, 0, 0, 0);
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            int e = rb.idx + g;
            if (e >= kRingB) e -= kRingB;
            st_shared_v4(sbase + kOffB + e * kTileB + (j >> 3) * 1024 + lq * 128 + (j & 7) * 16,
                         pick(raw[0], g), pick(raw[1], g), pick(raw[2], g), pick(raw[3], g));
          }
        }
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_a(b_emptyB + 8 * st.idx);
        for (int u = 0; u < 4; ++u, rb.next(kRingB))
          if (lane == 0) tc::mbar_arrive_a(b_bfull + 8 * rb.idx);
        if (ct == 0) TRACE(3, (it - (int)blockIdx.x) / (int)gridDim.x);
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

unsigned long long* g_trace2 = nullptr;

}  // namespace

bool tc_pq2_applicable(int m, int k, int n, int npts, uint32_t p) {
  return p < (1u << 31) && p >= (1u << 30) && m >= 1 && m <= 32 && n >= 1 && n <= 32 &&
         k >= 1 && (npts % 4) == 0;
}

int launch_tc_pq2(const TcArgs& t, const PrimeSet& ps, cudaStream_t st) {
  if (t.npts <= 0 || t.m <= 0 || t.n <= 0) return kOk;
  for (int i = 0; i < ps.count; ++i)
    if (!tc_pq2_applicable(t.m, t.k, t.n, t.npts, ps.pr[i].p)) {
      set_last_error("tc_pq2: unsupported shape %dx%dx%d", t.m, t.k, t.n);
      return kInvalidArgument;
    }
  Q2Args a{};
  a.C = t.C; a.m = t.m; a.k = t.k; a.n = t.n; a.npts = t.npts; a.nz = ps.count;
  a.nquads = t.npts / 4;
  a.nch = (t.k + 31) / 32;
  a.c_ps = t.c_ps;
  if (std::getenv("FPM_TCPQ2_TRACE")) {
    if (!g_trace2) cudaMalloc(&g_trace2, 64 * 8 * sizeof(unsigned long long));
    a.trace = g_trace2;
  }
  const long long items = (long long)ps.count * a.nquads;
  if (items >= (1LL << 31)) {
    set_last_error("tc_pq2: too many work items");
    return kUnsupported;
  }
  const uint64_t nz = (uint64_t)ps.count, nquad = (uint64_t)a.nquads;
  CUtensorMap mA, mB;
  {
    // A: [z][quad][i][(l, 4)]
    const uint64_t dims[4] = {(uint64_t)t.k * 4, (uint64_t)t.m, nquad, nz};
    const uint64_t ps_b = (uint64_t)(t.a_ps ? t.a_ps : (long long)t.npts * t.m * t.k) * 4;
    const uint64_t strides[3] = {(uint64_t)t.k * 16, (uint64_t)t.m * t.k * 16, ps_b};
    const uint32_t box[4] = {128, (uint32_t)t.m, 1, 1};
    FPM_TRY(make_map4(&mA, t.A, dims, strides, box));
  }
  {
    // B: [z][quad][l][(j, 4)]
    const uint64_t dims[4] = {(uint64_t)t.n * 4, (uint64_t)t.k, nquad, nz};
    const uint64_t ps_b = (uint64_t)(t.b_ps ? t.b_ps : (long long)t.npts * t.k * t.n) * 4;
    const uint64_t strides[3] = {(uint64_t)t.n * 16, (uint64_t)t.k * t.n * 16, ps_b};
    const uint32_t box[4] = {(uint32_t)(4 * t.n), 32, 1, 1};
    FPM_TRY(make_map4(&mB, t.B, dims, strides, box));
  }
  static bool attr = false;
  if (!attr) {
    FPM_CUDA_TRY(cudaFuncSetAttribute(tc_pq2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kSmem));
    attr = true;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const unsigned grid = (unsigned)(items < sms ? items : sms);
  tc_pq2_kernel<<<grid, kThreads, kSmem, st>>>(mA, mB, a, ps);
  FPM_LAUNCH_CHECK();
  return kOk;
}

}  // namespace fpm

// profiling only: per-item timestamps of CTA 0 (FPM_TCPQ2_TRACE)
extern "C" int fpm_debug_tcpq2_trace(unsigned long long* host) {
  if (!fpm::g_trace2) return 1;
  cudaDeviceSynchronize();
  cudaMemcpy(host, fpm::g_trace2, 64 * 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  return 0;
}
