// tc_pair.cu -- int8 tensor-core per-point products for 128 < m <= 256
// (BASELINE cfg5: 256x256 . 256x256 at 4096 points).  Replaces the per-point
// `_dense.mat_mul(a, b, p)` loop of `_pm_mul_ntt` (polmat.py:300-303,
// _dense.py:39-74) for the large shapes.
//
// Same limb identity as tc_grouped.cu: A's raw little-endian bytes on K'
// (K' = 4k), B pre-scaled s_q = 2^(8q) B mod p and split into byte planes on
// N' (N' = 4n), C = sum_r 2^(8r) D_r reduced by d_red56.
//
// Work item = (point, 32-column block of C).  Both 128-row M tiles of the
// point are multiplied by the SAME B tile: one build of each B element
// (3 Shoup scalings + a 4x4 byte transpose) instead of one per M tile, which
// is what bounds tc_grouped at m = 256 (its CUDA cores, not its tensor
// cores).  TMEM: two accumulator slots of 2 x 128 columns, so the epilogue
// of item i overlaps the MMAs of item i + 1.
//
// Warp roles (persistent, one CTA per SM, 18 warps):
//   warp 0      TMA producer: both A tiles (128 rows x 128 B, SWIZZLE_128B)
//               and the raw 32 x 32 u32 B block of a K chunk, NS stages
//   warp 1      TMEM allocator and single-thread MMA issuer (M128 N128 K32,
//               4 per M tile per K chunk)
//   warps 2-9   epilogue: lane quarter warp % 4, M tile (warp - 2) / 4
//   warps 10-17 B builders: one (quad of l, column) task per thread per chunk
#include <cuda.h>
#include <cudaTypedefs.h>

#include "tc_common.cuh"
#include "tc_pointwise.cuh"

namespace fpm {
namespace {

constexpr int kNB = 32;                            // C columns per item
constexpr int kNS = 4;                             // load stages
constexpr int kNR = 4;                             // built B tiles in flight
constexpr uint32_t kTileA = 16384;                 // 128 rows x 128 B
constexpr uint32_t kRawB = 32 * kNB * 4;           // 32 l x 32 j words
constexpr uint32_t kStage = 2 * kTileA + kRawB;    // 36 KB (1 KB multiple)
constexpr uint32_t kSbo = 1040;                    // 8 N' rows x 128 B + 16 B pad
constexpr uint32_t kTileB = 16 * kSbo;             // N' = 4 kNB = 128 rows
constexpr uint32_t kOffRing = kNS * kStage;
constexpr size_t kSmem = kOffRing + kNR * kTileB + 1024;  // + 1 KB alignment slack
constexpr int kEpiWarp0 = 2, kEpiWarps = 8;
constexpr int kBldWarp0 = kEpiWarp0 + kEpiWarps, kBldWarps = 8;
constexpr int kThreads = (kBldWarp0 + kBldWarps) * 32;

struct PArgs {
  uint32_t* C;
  int m, k, n, npts, nz;
  long long c_ps;
  int nblk, nch;
  long long items;
};

struct Ring {
  int idx;
  uint32_t ph;
  __device__ __forceinline__ void next(int n) {
    if (++idx == n) {
      idx = 0;
      ph ^= 1u;
    }
  }
};

__device__ __forceinline__ void decode(const PArgs& a, long long it, int& z, int& t, int& jb) {
  const long long per_z = (long long)a.npts * a.nblk;
  z = (int)(it / per_z);
  const long long rem = it - (long long)z * per_z;
  t = (int)(rem / a.nblk);
  jb = (int)(rem - (long long)t * a.nblk);
}

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t x, uint32_t y, uint32_t z,
                                       uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(x), "r"(y), "r"(z),
               "r"(w)
               : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    tc_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ PArgs a, const __grid_constant__ PrimeSet ps) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t full[kNS], empty[kNS], bfull[kNR], bempty[kNR], afull[2], aempty[2];
  __shared__ uint32_t tmem_base;
  const uint32_t sraw = tc::smem_u32(smem_raw);
  const uint32_t sbase = (sraw + 1023u) & ~1023u;  // SWIZZLE_128B tiles: 1 KB aligned
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmB);
    for (int s = 0; s < kNS; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1 + kBldWarps);  // MMA commit (A) + builders (raw B)
    }
    for (int r = 0; r < kNR; ++r) {
      tc::mbar_init(&bfull[r], kBldWarps);
      tc::mbar_init(&bempty[r], 1);
    }
    for (int c = 0; c < 2; ++c) {
      tc::mbar_init(&afull[c], 1);
      tc::mbar_init(&aempty[c], kEpiWarps);
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(&tmem_base, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  pdl_wait();  // operands come from the forward transforms
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    // ------------------------------ TMA producer ------------------------------
    if (lane == 0) {
      Ring st{0, 0};
      for (long long it = blockIdx.x; it < a.items; it += gridDim.x) {
        int z, t, jb;
        decode(a, it, z, t, jb);
        for (int ch = 0; ch < a.nch; ++ch, st.next(kNS)) {
          tc::mbar_wait_a(tc::smem_u32(&empty[st.idx]), st.ph ^ 1u);
          tc::mbar_expect_tx(&full[st.idx], kStage);
          const uint32_t s0 = sbase + st.idx * kStage;
          tc::tma_load_4d(s0, &tmA, &full[st.idx], ch * 32, 0, t, z);
          tc::tma_load_4d(s0 + kTileA, &tmA, &full[st.idx], ch * 32, 128, t, z);
          tc::tma_load_4d(s0 + 2 * kTileA, &tmB, &full[st.idx], jb * kNB, ch * 32, t, z);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------- MMA issuer -------------------------------
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_u8(128, 4 * kNB);
      Ring st{0, 0}, br{0, 0}, ac{0, 0};
      for (long long it = blockIdx.x; it < a.items; it += gridDim.x, ac.next(2)) {
        tc::mbar_wait_spin(tc::smem_u32(&aempty[ac.idx]), ac.ph ^ 1u);
        for (int ch = 0; ch < a.nch; ++ch, st.next(kNS), br.next(kNR)) {
          tc::mbar_wait_spin(tc::smem_u32(&full[st.idx]), st.ph);
          tc::mbar_wait_spin(tc::smem_u32(&bfull[br.idx]), br.ph);
          tc::fence_after_sync();
          const uint32_t tA = sbase + st.idx * kStage;
          const uint32_t tB = sbase + kOffRing + br.idx * kTileB;
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            const uint32_t d = tmem + ac.idx * 256 + mt * 128;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              tc::mma_u8(d, tc::make_desc_sw128(tA + mt * kTileA + ks * 32),
                         tc::make_desc(tB + ks * 256, 128, kSbo), idesc,
                         (ch > 0 || ks > 0) ? 1u : 0u);
          }
          tc::commit(&bempty[br.idx]);
          tc::commit(&empty[st.idx]);
        }
        tc::commit(&afull[ac.idx]);
      }
    }
  } else if (warp < kBldWarp0) {
    // -------------------------------- epilogue --------------------------------
    const int q = warp & 3;                    // TMEM lane quarter this warp may access
    const int mt = (warp - kEpiWarp0) >> 2;    // M tile
    const int il = mt * 128 + 32 * q + lane;   // row of C within the point
    const bool row_ok = il < a.m;
    Ring ac{0, 0};
    for (long long it = blockIdx.x; it < a.items; it += gridDim.x, ac.next(2)) {
      int z, t, jb;
      decode(a, it, z, t, jb);
      const uint32_t p = ps.pr[z].p, m58 = ps.pr[z].m58;
      tc::mbar_wait_sleep_a(tc::smem_u32(&afull[ac.idx]), ac.ph);
      tc::fence_after_sync();
      uint32_t* Crow = a.C + z * a.c_ps + ((long long)t * a.m + (row_ok ? il : 0)) * a.n;
#pragma unroll 1
      for (int cc = 0; cc < kNB / 8; ++cc) {
        uint32_t v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + ac.idx * 256 + mt * 128 + 32 * cc, v);
        if (row_ok) {
          uint32_t o[8];
#pragma unroll
          for (int x = 0; x < 8; ++x) {
            // D_r < 4k 255^2 <= 2^31, so the limb sum is < 2^56
            uint64_t acc = (uint64_t)v[4 * x];
            acc += (uint64_t)v[4 * x + 1] << 8;
            acc += (uint64_t)v[4 * x + 2] << 16;
            acc += (uint64_t)v[4 * x + 3] << 24;
            o[x] = d_red56(acc, p, m58);
          }
          const int j = jb * kNB + 8 * cc;
          if (j + 8 <= a.n) {
            *reinterpret_cast<uint4*>(Crow + j) = make_uint4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<uint4*>(Crow + j + 4) = make_uint4(o[4], o[5], o[6], o[7]);
          } else {
#pragma unroll
            for (int x = 0; x < 8; ++x)
              if (j + x < a.n) Crow[j + x] = o[x];
          }
        }
      }
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&aempty[ac.idx]);
    }
  } else {
    // -------------------------------- B builders -------------------------------
    // task = (quad lq of the 32 l values, column j): the 4 elements B[4lq+u][j]
    // become 16 bytes (b, s1, s2, s3 byte planes) in 4 B-operand rows 4j + r
    const int ct = tid - kBldWarp0 * 32;       // 0 .. 255
    const int lq = ct >> 5, j = ct & 31;
    Ring st{0, 0}, br{0, 0};
    for (long long it = blockIdx.x; it < a.items; it += gridDim.x) {
      int z, t, jb;
      decode(a, it, z, t, jb);
      const PrimeConst& pc = ps.pr[z];
      const uint32_t p = pc.p;
      const uint32_t w1 = pc.sc[1].x, w1p = pc.sc[1].y, w2 = pc.sc[2].x, w2p = pc.sc[2].y;
      const uint32_t w3 = pc.sc[3].x, w3p = pc.sc[3].y;
      for (int ch = 0; ch < a.nch; ++ch, st.next(kNS), br.next(kNR)) {
        tc::mbar_wait_sleep_a(tc::smem_u32(&full[st.idx]), st.ph);
        tc::mbar_wait_sleep_a(tc::smem_u32(&bempty[br.idx]), br.ph ^ 1u);
        const uint32_t* raw =
            reinterpret_cast<const uint32_t*>(smem_raw + (sbase - sraw) + st.idx * kStage + 2 * kTileA);
        const uint32_t* src = raw + (4 * lq) * kNB + j;
        uint32_t w[4][4];  // [r][u]: bytes (b_r, s1_r, s2_r, s3_r) of element l = 4lq+u
#pragma unroll
        for (int uu = 0; uu < 4; ++uu) {
          const uint32_t b = src[uu * kNB];
          // lazy Shoup: any value < 2^32 congruent to 2^(8q) b is exact here
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
        // rows c = 4j + r: (c >> 3) = j >> 1, (c & 7) = 4 (j & 1) + r
        const uint32_t tB = sbase + kOffRing + br.idx * kTileB + lq * 128 + (j >> 1) * kSbo +
                            (j & 1) * 64;
#pragma unroll
        for (int r = 0; r < 4; ++r) sts128(tB + r * 16, w[r][0], w[r][1], w[r][2], w[r][3]);
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          tc::mbar_arrive(&bfull[br.idx]);
          tc::mbar_arrive(&empty[st.idx]);
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// ---- CTA-pair variant (cta_group::2) -------------------------------------------
// One MMA instruction covers both M tiles (M = 256) across the two SMs of a
// cluster: each CTA loads only ITS 128 A rows and builds only ITS half of the
// B columns (N' = 256 = 2 x 128), so per SM the loaded bytes per MMA work
// halve (A re-read 4x instead of 8x per point for n = 256) and every B
// element is still built once.  Each CTA's TMEM holds its 128 rows x 256
// columns.  The leader (rank 0) issues the MMAs; commits multicast to both
// CTAs; the follower's builders and epilogue arrive on the leader's
// barriers through shared::cluster addresses.
constexpr int kNB2 = 64;                           // C columns per pair item (32 per CTA)
constexpr int kNS2 = 6;
constexpr int kNR2 = 4;
constexpr uint32_t kRawB2 = 32 * 32 * 4;           // 32 l x this CTA's 32 columns
constexpr uint32_t kStage2 = kTileA + kRawB2;      // 20 KB
constexpr uint32_t kOffRing2 = kNS2 * kStage2;
constexpr size_t kSmem2 = kOffRing2 + kNR2 * kTileB + 1024;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t peer_addr(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void arrive_cluster(uint32_t cluster_addr) {
  // default semantics (as CUTLASS's ClusterBarrier::arrive): an explicit
  // .release.cluster costs a cluster-wide MEMBAR per arrival (measured 30 %
  // of the stall samples); the writer's fence.proxy.async orders the data
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}
// wait with cluster-scope acquire (arrivals come from the peer CTA too)
__device__ __forceinline__ void wait_cluster(uint32_t addr, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mma_u8_cg2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// MMA completion -> the barrier at this offset in both CTAs
__device__ __forceinline__ void commit_both(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\t"
      "mov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], m;\n\t}\n" ::"r"(bar)
      : "memory");
}
// 2-SM TMA load: lands in this CTA's smem, completes bytes on the leader's barrier
__device__ __forceinline__ void tma_load_4d_cg2(uint32_t dst, const void* tmap, uint32_t mbar,
                                                int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5, %6}], [%2];\n" ::"r"(dst),
      "l"(tmap), "r"(mbar & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d_local(uint32_t dst, const void* tmap, uint32_t mbar,
                                                  int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5, %6}], [%2];\n" ::"r"(dst),
      "l"(tmap), "r"(mbar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void expect_tx_a(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mbar), "r"(bytes)
               : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    tc_pair2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ PArgs a, const __grid_constant__ PrimeSet ps) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t full[kNS2], rawfull[kNS2], empty[kNS2], bfull[kNR2], bempty[kNR2];
  __shared__ uint64_t afull[2], aempty[2];
  __shared__ uint32_t tmem_base;
  const uint32_t sraw = tc::smem_u32(smem_raw);
  const uint32_t sbase = (sraw + 1023u) & ~1023u;  // SWIZZLE_128B tiles: 1 KB aligned
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const long long pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  auto A = [](const uint64_t* b) { return tc::smem_u32(b); };

  if (tid == 0) {
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmB);
    for (int s = 0; s < kNS2; ++s) {
      tc::mbar_init(&full[s], 1);                 // leader: both CTAs' A bytes
      tc::mbar_init(&rawfull[s], 1);              // this CTA's raw B bytes
      tc::mbar_init(&empty[s], 1 + kBldWarps);    // MMA commit + local builders
    }
    for (int r = 0; r < kNR2; ++r) {
      tc::mbar_init(&bfull[r], 2 * kBldWarps);    // leader: builders of both CTAs
      tc::mbar_init(&bempty[r], 1);
    }
    for (int c = 0; c < 2; ++c) {
      tc::mbar_init(&afull[c], 1);
      tc::mbar_init(&aempty[c], 2 * kEpiWarps);   // leader: epilogues of both CTAs
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        tc::smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  tc::fence_before_sync();
  cluster_sync();
  tc::fence_after_sync();
  pdl_wait();  // operands come from the forward transforms
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    // ------------------------------ TMA producer ------------------------------
    if (lane == 0) {
      Ring st{0, 0};
      for (long long it = pair; it < a.items; it += npairs) {
        int z, t, jb;
        decode(a, it, z, t, jb);
        for (int ch = 0; ch < a.nch; ++ch, st.next(kNS2)) {
          tc::mbar_wait_a(A(&empty[st.idx]), st.ph ^ 1u);
          if (leader) expect_tx_a(A(&full[st.idx]), 2 * kTileA);
          expect_tx_a(A(&rawfull[st.idx]), kRawB2);
          const uint32_t s0 = sbase + st.idx * kStage2;
          tma_load_4d_cg2(s0, &tmA, A(&full[st.idx]), ch * 32, 128 * (int)rank, t, z);
          tma_load_4d_local(s0 + kTileA, &tmB, A(&rawfull[st.idx]), jb * kNB2 + 32 * (int)rank,
                            ch * 32, t, z);
        }
      }
    }
  } else if (warp == 1) {
    // ----------------------- MMA issuer (leader CTA only) -----------------------
    if (leader && lane == 0) {
      const uint32_t idesc = tc::idesc_u8(256, 256);
      Ring st{0, 0}, br{0, 0}, ac{0, 0};
      for (long long it = pair; it < a.items; it += npairs, ac.next(2)) {
        wait_cluster(A(&aempty[ac.idx]), ac.ph ^ 1u);
        for (int ch = 0; ch < a.nch; ++ch, st.next(kNS2), br.next(kNR2)) {
          tc::mbar_wait_spin(A(&full[st.idx]), st.ph);
          wait_cluster(A(&bfull[br.idx]), br.ph);
          tc::fence_after_sync();
          const uint32_t tA = sbase + st.idx * kStage2;
          const uint32_t tB = sbase + kOffRing2 + br.idx * kTileB;
          const uint32_t d = tmem + ac.idx * 256;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            mma_u8_cg2(d, tc::make_desc_sw128(tA + ks * 32), tc::make_desc(tB + ks * 256, 128, kSbo),
                       idesc, (ch > 0 || ks > 0) ? 1u : 0u);
          commit_both(A(&bempty[br.idx]));
          commit_both(A(&empty[st.idx]));
        }
        commit_both(A(&afull[ac.idx]));
      }
    }
  } else if (warp < kBldWarp0) {
    // -------------------------------- epilogue --------------------------------
    const int q = warp & 3;                    // TMEM lane quarter this warp may access
    const int hc = (warp - kEpiWarp0) >> 2;    // column half: 32 of the 64 outputs
    const int il = 128 * (int)rank + 32 * q + lane;
    const bool row_ok = il < a.m;
    const uint32_t aempty_l = peer_addr(A(&aempty[0]), 0);
    Ring ac{0, 0};
    for (long long it = pair; it < a.items; it += npairs, ac.next(2)) {
      int z, t, jb;
      decode(a, it, z, t, jb);
      const uint32_t p = ps.pr[z].p, m58 = ps.pr[z].m58;
      tc::mbar_wait_sleep_a(A(&afull[ac.idx]), ac.ph);
      tc::fence_after_sync();
      uint32_t* Crow = a.C + z * a.c_ps + ((long long)t * a.m + (row_ok ? il : 0)) * a.n;
#pragma unroll 1
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + ac.idx * 256 + hc * 128 + 32 * cc, v);
        if (row_ok) {
          uint32_t o[8];
#pragma unroll
          for (int x = 0; x < 8; ++x) {
            uint64_t acc = (uint64_t)v[4 * x];
            acc += (uint64_t)v[4 * x + 1] << 8;
            acc += (uint64_t)v[4 * x + 2] << 16;
            acc += (uint64_t)v[4 * x + 3] << 24;
            o[x] = d_red56(acc, p, m58);
          }
          const int j = jb * kNB2 + 32 * hc + 8 * cc;
          if (j + 8 <= a.n) {
            *reinterpret_cast<uint4*>(Crow + j) = make_uint4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<uint4*>(Crow + j + 4) = make_uint4(o[4], o[5], o[6], o[7]);
          } else {
#pragma unroll
            for (int x = 0; x < 8; ++x)
              if (j + x < a.n) Crow[j + x] = o[x];
          }
        }
      }
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) arrive_cluster(aempty_l + 8u * ac.idx);
    }
  } else {
    // -------------------------------- B builders -------------------------------
    const int ct = tid - kBldWarp0 * 32;       // 0 .. 255
    const int lq = ct >> 5, j = ct & 31;
    const uint32_t bfull_l = peer_addr(A(&bfull[0]), 0);
    Ring st{0, 0}, br{0, 0};
    for (long long it = pair; it < a.items; it += npairs) {
      int z, t, jb;
      decode(a, it, z, t, jb);
      const PrimeConst& pc = ps.pr[z];
      const uint32_t p = pc.p;
      const uint32_t w1 = pc.sc[1].x, w1p = pc.sc[1].y, w2 = pc.sc[2].x, w2p = pc.sc[2].y;
      const uint32_t w3 = pc.sc[3].x, w3p = pc.sc[3].y;
      for (int ch = 0; ch < a.nch; ++ch, st.next(kNS2), br.next(kNR2)) {
        tc::mbar_wait_sleep_a(A(&rawfull[st.idx]), st.ph);
        tc::mbar_wait_sleep_a(A(&bempty[br.idx]), br.ph ^ 1u);
        const uint32_t* raw = reinterpret_cast<const uint32_t*>(smem_raw + (sbase - sraw) +
                                                                st.idx * kStage2 + kTileA);
        const uint32_t* src = raw + (4 * lq) * 32 + j;
        uint32_t w[4][4];
#pragma unroll
        for (int uu = 0; uu < 4; ++uu) {
          const uint32_t b = src[uu * 32];
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
        const uint32_t tB = sbase + kOffRing2 + br.idx * kTileB + lq * 128 + (j >> 1) * kSbo +
                            (j & 1) * 64;
#pragma unroll
        for (int r = 0; r < 4; ++r) sts128(tB + r * 16, w[r][0], w[r][1], w[r][2], w[r][3]);
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          arrive_cluster(bfull_l + 8u * br.idx);
          tc::mbar_arrive(&empty[st.idx]);
        }
      }
    }
  }
  tc::fence_before_sync();
  cluster_sync();
  if (warp == 1) {
    tc::fence_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 pair_encode_fn() {
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

int pair_map(CUtensorMap* m, const uint32_t* base, const cuuint64_t dims[4],
             const cuuint64_t strides[3], const cuuint32_t box[4], bool swz128) {
  auto fn = pair_encode_fn();
  if (!fn) {
    set_last_error("cuTensorMapEncodeTiled unavailable");
    return kCudaError;
  }
  const cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, const_cast<uint32_t*>(base), dims,
                  strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swz128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_last_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return kCudaError;
  }
  return kOk;
}

}  // namespace

bool tc_pair_applicable(int m, int k, int n, uint32_t p) {
  return m > 128 && m <= 256 && tc_grouped_applicable(m, k, n, p);
}

int launch_tc_pair(const TcArgs& t, const PrimeSet& ps, cudaStream_t st) {
  if (t.npts <= 0 || t.m <= 0 || t.n <= 0) return kOk;
  for (int i = 0; i < ps.count; ++i)
    if (!tc_pair_applicable(t.m, t.k, t.n, ps.pr[i].p)) {
      set_last_error("tc_pair: unsupported shape %dx%dx%d", t.m, t.k, t.n);
      return kInvalidArgument;
    }
  PArgs a{};
  a.C = t.C; a.m = t.m; a.k = t.k; a.n = t.n; a.npts = t.npts; a.nz = ps.count;
  a.c_ps = t.c_ps;
  a.nblk = (t.n + kNB - 1) / kNB;
  a.nch = (t.k + 31) / 32;
  a.items = (long long)ps.count * t.npts * a.nblk;
  const cuuint64_t nz = (cuuint64_t)ps.count;
  CUtensorMap mA, mB;
  {
    const cuuint64_t dims[4] = {(cuuint64_t)t.k, (cuuint64_t)t.m, (cuuint64_t)t.npts, nz};
    const cuuint64_t pstride = (cuuint64_t)(t.a_ps ? t.a_ps : (long long)t.npts * t.m * t.k) * 4;
    const cuuint64_t strides[3] = {(cuuint64_t)t.k * 4, (cuuint64_t)t.m * t.k * 4, pstride};
    const cuuint32_t box[4] = {32, 128, 1, 1};
    FPM_TRY(pair_map(&mA, t.A, dims, strides, box, true));
  }
  {
    const cuuint64_t dims[4] = {(cuuint64_t)t.n, (cuuint64_t)t.k, (cuuint64_t)t.npts, nz};
    const cuuint64_t pstride = (cuuint64_t)(t.b_ps ? t.b_ps : (long long)t.npts * t.k * t.n) * 4;
    const cuuint64_t strides[3] = {(cuuint64_t)t.n * 4, (cuuint64_t)t.k * t.n * 4, pstride};
    const cuuint32_t box[4] = {(cuuint32_t)kNB, 32, 1, 1};
    FPM_TRY(pair_map(&mB, t.B, dims, strides, box, false));
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (option(kOptTcPair1) == 0) {
    // CTA pairs: items of 64 columns, an even grid of clusters (2, 1, 1)
    a.nblk = (t.n + kNB2 - 1) / kNB2;
    a.items = (long long)ps.count * t.npts * a.nblk;
    CUtensorMap mB2;
    {
      const cuuint64_t dims[4] = {(cuuint64_t)t.n, (cuuint64_t)t.k, (cuuint64_t)t.npts, nz};
      const cuuint64_t pstride = (cuuint64_t)(t.b_ps ? t.b_ps : (long long)t.npts * t.k * t.n) * 4;
      const cuuint64_t strides[3] = {(cuuint64_t)t.n * 4, (cuuint64_t)t.k * t.n * 4, pstride};
      const cuuint32_t box[4] = {32, 32, 1, 1};
      FPM_TRY(pair_map(&mB2, t.B, dims, strides, box, false));
    }
    static bool attr2 = false;
    if (!attr2) {
      FPM_CUDA_TRY(cudaFuncSetAttribute(tc_pair2_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem2));
      attr2 = true;
    }
    long long pairs = a.items < sms / 2 ? a.items : sms / 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * pairs));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmem2;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    FPM_CUDA_TRY(cudaLaunchKernelEx(&cfg, tc_pair2_kernel, mA, mB2, a, ps));
    FPM_LAUNCH_CHECK();
    return kOk;
  }
  static bool attr = false;
  if (!attr) {
    FPM_CUDA_TRY(cudaFuncSetAttribute(tc_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kSmem));
    attr = true;
  }
  const unsigned grid = (unsigned)(a.items < sms ? a.items : sms);
  FPM_CUDA_TRY(launch_pdl(tc_pair_kernel, dim3(grid), dim3(kThreads), kSmem, st, mA, mB, a, ps));
  FPM_LAUNCH_CHECK();
  return kOk;
}

}  // namespace fpm
