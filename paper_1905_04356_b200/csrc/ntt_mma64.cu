// ntt_mma64.cu -- batched forward N = 4096 NTTs on the int8 tensor cores in
// TWO radix-64 passes (sm_100a).
//
// Same job and same output as ntt_mma.cu (modring.ntt_forward as used by
// polmat._pm_mul_ntt, modring.py:253-269, polmat.py:298-300, point-major
// evaluations in the DIF placement), but 4096 = 64 x 64 instead of 16^3: the
// CUDA-core epilogue (limb fold + twiddle per value and pass) bounds the
// radix-16 kernel, and two passes fold each value twice and twiddle it once
// instead of three folds and two twiddles; the extra MMA work (64-point DFTs
// as K' = 256 GEMMs) lands on the otherwise idle tensor pipe.
//
// Decomposition (n = a + 64 b, k = k0 + 64 k1, w = w_4096, w64 = w^64):
//   P1  Y[a, k0] = sum_b x[a + 64 b] w64^(b k0),   Y' = Y w^(a k0)
//   P2  X[k0 + 64 k1] = sum_a Y'[a, k0] w64^(a k1)
// Point k leaves at position brev12(k) = brev6(k1) + 64 brev6(k0).
//
// One tile = 8 transforms.  A pass is 4 chunks, each ONE accumulator of
// M = 128 rows x N' = 256 columns (8 or 4 MMAs M128 N256 K32):
//   P1 chunk s: rows (a & 15, t) of the a with a >> 4 = s, K' = 4 bytes of
//               the 64 (or 32, len <= 2048) inputs b;
//   P2 chunk s: rows (k0 >> 2, t) of the k0 with k0 & 3 = s, K' over a.
// Column 4 j + r of either pass is byte plane r of DFT output K(j) =
// brev6(pl(j)), pl(16 h + 8 g + i) = 32 g + 8 h + i (worker column part h,
// half g, value i): in P2 pl is the low position digit, and the values of one
// half of a chunk are one TMA box of 8 entries x 512 positions.  Both passes
// share one 64 KB B operand: s_q = 2^(8q) w64^(n K(j)) mod p split in byte
// planes; D_r <= 256 * 255^2 < 2^24 (D_3 < 2^23: the top byte of s_q < 2^7).
//
// In place: the tile's 128 KB of operands are 4 slices of 32 KB.  P1's A of
// chunk s is slice s ("slice-major"); the P1 epilogue of chunk s -- one
// 4-byte store per value, a warp store = one 128-byte core matrix -- writes
// the K chunks 4 s .. 4 s + 3 (a >> 2) of ALL four P2 operands into slice s
// ("chunk-major"), which only the finished MMAs of chunk s have read.
//
// Shared memory: 128 KB data + 64 KB B + two 16 KB output staging buffers
// (one TMA box each: workers fill one while the TMA engine reads the other).
// The 16 KB of twiddles (Montgomery form, 4 bytes each) do not fit beside
// them: a worker warp needs only 4 rows x 16 columns per chunk, 256 words per
// tile, kept as 8 registers per lane and fetched by warp shuffles.  TMEM: two
// 256-column accumulators.  Roles as in ntt_mma.cu:
// warp 0 MMA issuer, warps 1..16 workers (TMEM lane quarter warp % 4, column
// quarter (warp - 1) / 4), warp 17 TMA stores + L2 prefetch of the next
// tile's rows, warps 18..19 input loaders.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <vector>

#include "ntt.cuh"
#include "runtime.cuh"
#include "tc_common.cuh"

namespace fpm {

namespace {
inline int h_brev6(int x) {
  int r = 0;
  for (int i = 0; i < 6; ++i) r |= ((x >> i) & 1) << (5 - i);
  return r;
}
// DFT output index of accumulator column group j
inline int h_kof(int j) {
  const int h = j >> 4, g = (j >> 3) & 1, i = j & 7;
  return h_brev6(32 * g + 8 * h + i);
}
}  // namespace

// ---- host tables (appended to Plan::mma at kMma64TabOff) -----------------------
//   [0, 64K)     B operand, K-major SWIZZLE_NONE, LBO 128 (K), SBO 2048 (rows):
//                row 4 j + r, K byte 4 n + q = byte r of 2^(8q) w64^(n K(j))
//   [64K, 80K)   twiddles, u32 tw[a][j] = w^(a K(j)) 2^32 mod p
void mma64_ntt_tables(uint32_t p, uint32_t omega, std::vector<uint8_t>* out) {
  const size_t base = out->size();
  out->resize(base + kMma64TabBytes, 0);
  uint8_t* t = out->data() + base;
  const uint64_t w64 = h_powmod(omega, 64, p);
  for (int j = 0; j < 64; ++j) {
    const int k = h_kof(j);
    for (int n = 0; n < 64; ++n) {
      const uint64_t b0 = h_powmod(w64, (uint64_t)n * k, p);
      for (int q = 0; q < 4; ++q) {
        const uint32_t s = (uint32_t)h_mulmod(b0, ((uint64_t)1 << (8 * q)) % p, p);
        for (int r = 0; r < 4; ++r) {
          const int row = 4 * j + r, kb = 4 * n + q;
          t[(row >> 3) * 2048 + (kb >> 4) * 128 + (row & 7) * 16 + (kb & 15)] =
              (uint8_t)(s >> (8 * r));
        }
      }
    }
  }
  uint32_t* tw = reinterpret_cast<uint32_t*>(t + 65536);
  const uint64_t R = (((uint64_t)1) << 32) % p;
  for (int a = 0; a < 64; ++a)
    for (int j = 0; j < 64; ++j)
      tw[a * 64 + j] = (uint32_t)h_mulmod(h_powmod(omega, (uint64_t)a * h_kof(j), p), R, p);
}

namespace {

#ifndef FPM_M64_VARIANT
#define FPM_M64_VARIANT 15  // measured on cfg5: 0 -> 3.28 ms per product, 14 / 15 -> 3.205
#endif
constexpr bool kP1MH = (FPM_M64_VARIANT & 1) != 0, kP1ML = (FPM_M64_VARIANT & 2) != 0;
constexpr bool kP2MH = (FPM_M64_VARIANT & 4) != 0, kP2ML = (FPM_M64_VARIANT & 8) != 0;
constexpr int kWorkers = 16;                     // worker warps (warps 1 .. 16)
constexpr int kLoaders = 2;                      // input warps (after the store warp)
constexpr int kThreads = 32 * (2 + kWorkers + kLoaders);
constexpr int kLT = 32 * kLoaders;               // loader threads
constexpr uint32_t kData = 131072;               // 8 transforms x 4096 words
constexpr uint32_t kOffB = kData;                // B operand (64 KB)
constexpr uint32_t kOffStage = kOffB + 65536;    // output staging: two TMA boxes of 16 KB
constexpr uint32_t kOffBar = kOffStage + 32768;
constexpr size_t kSmem = kOffBar + 256;
static_assert(kSmem <= 232448, "shared memory per CTA");

struct Mma64Args {
  const uint32_t* in1;
  const uint32_t* in2;
  long long in1_stride, in2_stride;  // words between entries' coefficient rows
  uint32_t* out1;
  uint32_t* out2;
  int n1, n2;                        // entries of the two batches
  int len;                           // coefficients per entry
  int kc1;                           // 16-byte K chunks of P1 (8: len <= 2048, else 16)
  int vec;                           // 16-byte aligned rows: vector loads
  long long tiles1, tiles;
  uint32_t p, w16s, pinv;            // w16s = floor(2^48 / p), pinv = p^-1 mod 2^32
  uint32_t negp, zero;               // 2^32 - p; 0 (opaque: keeps 3-input adds on the ALU pipe)
  uint32_t c256;                     // 256 (opaque: keeps d * 256 + e one IMAD)
  const uint8_t* tab;
  int tma_out;                       // point-major output by TMA stores
  int dbg;                           // timing experiments (option ntt_mma_dbg): 1 = no input loads
};

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t x, uint32_t y, uint32_t z,
                                       uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(x), "r"(y), "r"(z),
               "r"(w)
               : "memory");
}
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t x) {
  asm volatile("st.shared.b32 [%0], %1;\n" ::"r"(addr), "r"(x) : "memory");
}
// 4-D TMA tensor store shared -> global (bulk group)
__device__ __forceinline__ void tma_store_4d(const void* tmap, uint32_t src, int c0, int c1, int c2,
                                             int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];\n" ::"l"(
          tmap),
      "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
// 32 lanes x 16 columns of 32-bit, no wait
__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
// byte permute with a zero second operand (ALU pipe, not an IMAD shift)
__device__ __forceinline__ uint32_t prmt0(uint32_t a, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(0u), "r"(sel));
  return r;
}

// V = sum_r 2^(8r) d[r] (d0..d2 <= 256 * 255^2, d3 < 2^23) -> a congruent word
// < 2p + 2^16 with ONE multiply-high: L = d0 + 2^8 d1 <= 257 * 256 * 255^2 <
// 2^32 and H = d2 + 2^8 d3 < 2^24 + 2^31 are exact, V = L + 2^16 H = 2^16 Hs +
// (L mod 2^16) with Hs = H + floor(L / 2^16) < 2^32; q = hi(Hs floor(2^48 / p))
// is the Shoup quotient of Hs 2^16, so 0 <= 2^16 Hs - q p < 2p and
// V - q p = L + (H << 16) - q p (mod 2^32) < 2p + 2^16 < 2^32.
// MH / ML: form H / L with one IMAD by c256 (= 256, opaque so that it stays a
// multiply on the FMA pipe) instead of a byte permute and a 3-input add (z = 0,
// opaque: a 2-input add would be issued as IMAD.IADD) on the ALU pipe.
template <bool MH, bool ML>
__device__ __forceinline__ uint32_t fold4w(uint32_t d0, uint32_t d1, uint32_t d2, uint32_t d3,
                                           uint32_t negp, uint32_t w16s, uint32_t z,
                                           uint32_t c256) {
  const uint32_t H = MH ? d3 * c256 + d2 : d2 + prmt0(d3, 0x2104) + z;  // d2 + (d3 << 8)
  const uint32_t L = ML ? d1 * c256 + d0 : d0 + prmt0(d1, 0x2104) + z;  // d0 + (d1 << 8)
  const uint32_t q = __umulhi(H + (L >> 16), w16s);
  return (L + (H << 16)) + q * negp;
}
// Montgomery product y W 2^-32 mod p (y < 2^32, W < p) in (0, 2p)
__device__ __forceinline__ uint32_t mont(uint32_t y, uint32_t W, uint32_t p, uint32_t pinv) {
  const uint64_t t = (uint64_t)y * W;
  const uint32_t m = (uint32_t)t * pinv;
  return (uint32_t)(t >> 32) - __umulhi(m, p) + p;
}

struct TileSrc {
  const uint32_t* in;
  long long stride;
  int ne;
  long long e0;
};
__device__ __forceinline__ TileSrc tile_src(const Mma64Args& a, long long tile) {
  TileSrc s;
  if (tile < a.tiles1) {
    s.in = a.in1; s.stride = a.in1_stride; s.ne = a.n1; s.e0 = tile * 8;
  } else {
    s.in = a.in2; s.stride = a.in2_stride; s.ne = a.n2; s.e0 = (tile - a.tiles1) * 8;
  }
  return s;
}

// ---- input of one slice (P1 operand of chunk s) --------------------------------
// item = (transform t, a-quad aq, K chunk kc): four 16-byte loads
// x[16 s + 4 aq .. + 3 + 64 b], b = 4 kc .. 4 kc + 3, transposed into the
// 16-byte K chunks of rows (4 aq + c, t).  32 kc1 items per slice.
constexpr int kLoadItems = 4;
struct LoadBuf {
  uint4 g[kLoadItems][4];
};
__device__ __forceinline__ void slice_load(const Mma64Args& a, const TileSrc& s, int sl, int i0,
                                           LoadBuf& lb) {
#pragma unroll
  for (int r = 0; r < kLoadItems; ++r) {
    const int it = i0 + kLT * r;
    const int t = it & 7, aq = (it >> 3) & 3, kc = it >> 5;
    const long long e = s.e0 + t;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int n = 16 * sl + 4 * aq + 64 * (4 * kc + i);
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      if (e < s.ne) {
        const uint32_t* src = s.in + e * s.stride + n;
        if (a.vec && n + 3 < a.len) {
          v = __ldg(reinterpret_cast<const uint4*>(src));
        } else {
          if (n < a.len) v.x = __ldg(src);
          if (n + 1 < a.len) v.y = __ldg(src + 1);
          if (n + 2 < a.len) v.z = __ldg(src + 2);
          if (n + 3 < a.len) v.w = __ldg(src + 3);
        }
      }
      lb.g[r][i] = v;
    }
  }
}
__device__ __forceinline__ void slice_store(uint32_t sdata, int sl, int i0, const LoadBuf& lb) {
#pragma unroll
  for (int r = 0; r < kLoadItems; ++r) {
    const int it = i0 + kLT * r;
    const int t = it & 7, aq = (it >> 3) & 3, kc = it >> 5;
    const uint4* g = lb.g[r];
    const uint32_t b = sdata + (uint32_t)(sl * 32768 + kc * 2048 + (4 * aq) * 128 + t * 16);
    sts128(b, g[0].x, g[1].x, g[2].x, g[3].x);
    sts128(b + 128, g[0].y, g[1].y, g[2].y, g[3].y);
    sts128(b + 256, g[0].z, g[1].z, g[2].z, g[3].z);
    sts128(b + 384, g[0].w, g[1].w, g[2].w, g[3].w);
  }
}

__device__ __forceinline__ int brev2(int x) { return ((x & 1) << 1) | ((x >> 1) & 1); }
__host__ __device__ constexpr int brev3c(int x) {
  return ((x & 1) << 2) | (x & 2) | ((x >> 2) & 1);
}

__global__ void __launch_bounds__(kThreads, 1)
    ntt_mma64_kernel(const __grid_constant__ Mma64Args a, const __grid_constant__ CUtensorMap om1,
                     const __grid_constant__ CUtensorMap om2) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = tc::smem_u32(smem);
  const uint32_t sdata = sbase, sB = sbase + kOffB, sStage = sbase + kOffStage;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  // full[2], empty[2], slice ready[4], P1 done, P2 MMAs done, staged[2], stage free[2];
  // TMEM base
  uint64_t *full = bars, *empty = bars + 2, *ready = bars + 4, *pdone = bars + 16;  // pdone[3]
  uint64_t* pd3 = bars + 20;  // pd3[4]: slice 3's part of P2 operand s' (8 warps, one half each)
  uint64_t *p2done = bars + 9, *staged = bars + 10, *stfree = bars + 12;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // the B operand (read once per CTA)
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.tab);
    uint4* dst = reinterpret_cast<uint4*>(smem + kOffB);
    for (int i = tid; i < 65536 / 16; i += kThreads) dst[i] = __ldg(src + i);
  }
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&full[b], 1);
      tc::mbar_init(&empty[b], kWorkers);
      tc::mbar_init(&staged[b], kWorkers);
      tc::mbar_init(&stfree[b], 1);
    }
    for (int j = 0; j < 4; ++j) {
      tc::mbar_init(&ready[j], kLoaders);
      tc::mbar_init(&pdone[j], kWorkers);
      tc::mbar_init(&pd3[j], kWorkers / 2);
    }
    tc::mbar_init(p2done, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_proxy_async();  // B operand: generic stores -> tensor-core reads
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // inputs may come from the previous kernel

  if (warp == 0) {
    // ------------------------------- MMA issuer -------------------------------
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_u8(128, 256);
      // an operand offset adds (offset >> 4) to the 14-bit start-address field
      // (all addresses < 256 KB: no carry out)
      const uint64_t dA = tc::make_desc(sdata, 2048, 128);
      const uint64_t dB = tc::make_desc(sB, 128, 2048);
      const int ks1 = a.kc1 >> 1;  // K32 steps of P1
      int it = 0;
      for (long long tile = blockIdx.x; tile < a.tiles; tile += gridDim.x, ++it) {
        // P1: chunk s reads slice s
#pragma unroll 1
        for (int s = 0; s < 4; ++s) {
          const int buf = s & 1;
          tc::mbar_wait_spin(tc::smem_u32(&empty[buf]), ((s >> 1) & 1) ^ 1);
          if (!(a.dbg & 2)) tc::mbar_wait_spin(tc::smem_u32(&ready[s]), it & 1);
          tc::fence_after_sync();
          const uint32_t d = tmem + buf * 256;
          for (int i = 0; i < ks1; ++i)
            tc::mma_u8(d, dA + ((uint32_t)(s * 32768 + i * 4096) >> 4),
                       dB + ((uint32_t)(i * 256) >> 4), idesc, i > 0 ? 1u : 0u);
          tc::commit(&full[buf]);
        }
        // P2: chunk s reads its 8 KB of every slice; the K steps of slice sl
        // (chunk 0) start as soon as the P1 epilogue of chunk sl has written it,
        // those of slice 3 as soon as the 8 warps that write operand s have
#pragma unroll 1
        for (int s = 0; s < 4; ++s) {
          const int buf = s & 1;
          tc::mbar_wait_spin(tc::smem_u32(&empty[buf]), ((s >> 1) & 1) ^ 1);
          tc::fence_after_sync();
          const uint32_t d = tmem + buf * 256;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (s == 0 && i < 6 && (i & 1) == 0) {
              tc::mbar_wait_spin(tc::smem_u32(&pdone[i >> 1]), it & 1);
              tc::fence_after_sync();
            }
            if (i == 6) {
              // operand s of slice 3: the half s & 1 of the warps h >> 1 = s >> 1
              tc::mbar_wait_spin(tc::smem_u32(&pd3[s]), it & 1);
              tc::fence_after_sync();
            }
            tc::mma_u8(d, dA + ((uint32_t)((i >> 1) * 32768 + s * 8192 + (i & 1) * 4096) >> 4),
                       dB + ((uint32_t)(i * 256) >> 4), idesc, i > 0 ? 1u : 0u);
          }
          tc::commit(&full[buf]);
        }
        tc::commit(p2done);  // the data region may be refilled
      }
    }
  } else if (warp == kWorkers + 1) {
    // ------------------------- output store warp (TMA) -------------------------
    if (a.tma_out && lane == 0) {
      tc::prefetch_tmap(&om1);
      tc::prefetch_tmap(&om2);
      long long nbox = 0;
      for (long long tile = blockIdx.x; tile < a.tiles; tile += gridDim.x) {
        const bool second = tile >= a.tiles1;
        const int e0 = (int)((second ? tile - a.tiles1 : tile) * 8);
        // the next tile's input rows into L2 a tile ahead
        if (a.vec && tile + gridDim.x < a.tiles) {
          const TileSrc ns = tile_src(a, tile + gridDim.x);
          const uint32_t bytes = (uint32_t)((a.len * 4 + 15) & ~15);
          for (int t = 0; t < 8 && ns.e0 + t < ns.ne; ++t)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(
                             ns.in + (ns.e0 + t) * ns.stride),
                         "r"(bytes)
                         : "memory");
        }
        // box bx = (chunk s, half g) from staging buffer g; a buffer is free
        // once the store issued before the latest one has read it
        for (int bx = 0; bx < 8; ++bx) {
          const int s = bx >> 1, g = bx & 1;
          tc::mbar_wait(&staged[g], s & 1);
          tma_store_4d(second ? &om2 : &om1, sStage + g * 16384, e0, 4 * brev2(s), 32 * g, 0);
          tc::bulk_commit();
          asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
          if (nbox > 0) tc::mbar_arrive(&stfree[g ^ 1]);
          ++nbox;
        }
      }
      tc::bulk_wait0();
    }
  } else if (warp > kWorkers + 1) {
    // ------------------------------ input warps -------------------------------
    // the slices of tile `it` once the P2 MMAs of tile it - 1 are done; the
    // loads of the first round are in flight while waiting
    const int i0 = (warp - kWorkers - 2) * 32 + lane;
    const uint32_t p2a = tc::smem_u32(p2done);
    // a thread's items of a round: (t, aq) fixed, kc = kcb + 2 r (+ 8 part)
    const int lt = i0 & 7, aq = (i0 >> 3) & 3, kcb = i0 >> 5;
    const uint32_t dst0 = sdata + (uint32_t)(kcb * 2048 + (4 * aq) * 128 + lt * 16);
    // rows of whole 64-word blocks, 16-byte aligned: every load is one
    // predicated LDG.128 at a constant offset from the tile's row pointer
    const bool fast = a.vec && (a.len & 63) == 0;
    int it = 0;
    for (long long tile = blockIdx.x; tile < a.tiles; tile += gridDim.x, ++it) {
      const TileSrc s = tile_src(a, tile);
      if (fast) {
        const bool valid = s.e0 + lt < s.ne && !(a.dbg & 1);
        const uint4* src =
            reinterpret_cast<const uint4*>(s.in + (s.e0 + lt) * s.stride + 4 * aq) + 64 * kcb;
#pragma unroll
        for (int sl = 0; sl < 4; ++sl) {
#pragma unroll 1
          for (int part = 0; part < a.kc1 / 8; ++part) {
            const int lim = (a.len >> 6) - 4 * kcb - 32 * part;  // valid b: 8 r + i < lim
            const uint4* sp = src + 512 * part + 4 * sl;
            uint4 g[4][4];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
              for (int i = 0; i < 4; ++i)
                g[r][i] = (valid && 8 * r + i < lim) ? __ldg(sp + 128 * r + 16 * i)
                                                     : make_uint4(0u, 0u, 0u, 0u);
            if (sl == 0 && part == 0 && it > 0) tc::mbar_wait_sleep_a(p2a, (it - 1) & 1);
            const uint32_t d = dst0 + (uint32_t)(sl * 32768 + part * 16384);
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              sts128(d + r * 4096, g[r][0].x, g[r][1].x, g[r][2].x, g[r][3].x);
              sts128(d + r * 4096 + 128, g[r][0].y, g[r][1].y, g[r][2].y, g[r][3].y);
              sts128(d + r * 4096 + 256, g[r][0].z, g[r][1].z, g[r][2].z, g[r][3].z);
              sts128(d + r * 4096 + 384, g[r][0].w, g[r][1].w, g[r][2].w, g[r][3].w);
            }
          }
          tc::fence_proxy_async();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&ready[sl]);
        }
        continue;
      }
#pragma unroll 1
      for (int sl = 0; sl < 4; ++sl) {
#pragma unroll 1
        for (int part = 0; part < a.kc1 / 8; ++part) {
          LoadBuf lb;
          slice_load(a, s, sl, i0 + part * kLT * kLoadItems, lb);
          if (sl == 0 && part == 0 && it > 0) tc::mbar_wait_sleep_a(p2a, (it - 1) & 1);
          slice_store(sdata, sl, i0 + part * kLT * kLoadItems, lb);
        }
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&ready[sl]);
      }
    }
  } else {
    // --------------------------------- workers --------------------------------
    const int wk = warp - 1;          // 0 .. kWorkers - 1
    const int q = warp & 3;           // TMEM lane quarter this warp may access
    const int h = wk >> 2;            // column quarter: 16 of the 64 outputs
    const int R = 32 * q + lane;      // operand row = TMEM lane
    const int t = R & 7, lq = lane >> 3;  // transform of the tile; row digit = 4 q + lq
    const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(64 * h);
    const uint32_t p = a.p, w16s = a.w16s, negp = a.negp, pinv = a.pinv, z = a.zero;
    const uint32_t c256 = a.c256;
    // P1 -> P2 operand: value (a = 16 s + 4 q + lq, column j = 16 h + 8 g + i)
    // -> slice s, operand K(j) & 3 = g + 2 (h >> 1), row group K(j) >> 2 =
    // (h & 1) + 2 brev3(i), K chunk q, word lq
    const uint32_t sNext = sdata + (uint32_t)((h >> 1) * 16384 + q * 2048 + (h & 1) * 128 + t * 16 +
                                              lq * 4);
    // twiddles of this warp: tw[16 s + 4 q + lq][16 h + i], value v = 16 s + i
    // in register v >> 3 of lane 8 lq + (v & 7)
    uint32_t twr[8];
    {
      const uint32_t* tw = reinterpret_cast<const uint32_t*>(a.tab + 65536);
#pragma unroll
      for (int r = 0; r < 8; ++r)
        twr[r] = __ldg(tw + (16 * (r >> 1) + 4 * q + lq) * 64 + 16 * h + 8 * (r & 1) + t);
    }
    // staging word t + 8 m1 + 32 (8 h + i) + 1024 m0, m1 = brev2(lq), m0 = brev2(q)
    const uint32_t sSt = sStage + 4u * (uint32_t)(t + 8 * brev2(lq) + 256 * h + 1024 * brev2(q));
    for (long long tile = blockIdx.x; tile < a.tiles; tile += gridDim.x) {
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const int buf = s & 1;
          tc::mbar_wait(&full[buf], (s >> 1) & 1);
          tc::fence_after_sync();
          // the chunk's 64 columns in quarters of 4 values through two register
          // buffers: the next quarter's TMEM load is in flight while one is folded
          const uint32_t tb = tl + buf * 256;
          uint32_t va[16], vb[16], y[8];
          tmem_ld16_nw(tb, va);
          tmem_ld16_nw(tb + 16, vb);
          tc::tmem_wait_ld();
#pragma unroll
          for (int g = 0; g < 2; ++g) {
#pragma unroll
            for (int hq = 0; hq < 2; ++hq) {
              const uint32_t(&v)[16] = hq == 0 ? va : vb;
#pragma unroll
              for (int i = 0; i < 4; ++i)
                y[4 * hq + i] =
                    pass == 0 ? fold4w<kP1MH, kP1ML>(v[4 * i], v[4 * i + 1], v[4 * i + 2],
                                                     v[4 * i + 3], negp, w16s, z, c256)
                              : fold4w<kP2MH, kP2ML>(v[4 * i], v[4 * i + 1], v[4 * i + 2],
                                                     v[4 * i + 3], negp, w16s, z, c256);
              if (g == 0) {
                // refill this buffer with the matching quarter of the second half
                if (hq == 0) {
                  tmem_ld16_nw(tb + 32, va);
                } else {
                  tc::tmem_wait_ld();  // va (third quarter) has landed
                  tmem_ld16_nw(tb + 48, vb);
                }
              } else if (hq == 0) {
                tc::tmem_wait_ld();    // vb: the accumulator is read out
                tc::fence_before_sync();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&empty[buf]);
              }
            }
            if (pass == 0) {
              const uint32_t nb = sNext + (uint32_t)(s * 32768 + g * 8192);
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const uint32_t W = __shfl_sync(0xffffffffu, twr[2 * s + g], (lane & 24) | i);
                sts32(nb + (uint32_t)(2 * brev3c(i)) * 128u, mont(y[i], W, p, pinv));
              }
              if (s == 3) {
                // this half completes the P2 operand g + 2 (h >> 1)
                tc::fence_proxy_async();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&pd3[g + 2 * (h >> 1)]);
              }
            } else if (a.tma_out) {
              // buffer g, its s-th use of the tile (4 per tile)
              tc::mbar_wait(&stfree[g], (s & 1) ^ 1);
#pragma unroll
              for (int i = 0; i < 8; ++i)
                sts32(sSt + (uint32_t)(g * 16384 + 32 * i * 4), y[i]);
              tc::fence_proxy_async();
              __syncwarp();
              if (lane == 0) tc::mbar_arrive(&staged[g]);
            } else {
              // position pl + 64 m0 + 256 m1 + 1024 brev2(s), pl = 32 g + 8 h + i
              const bool second = tile >= a.tiles1;
              const long long ne = second ? a.n2 : a.n1;
              const long long e = (second ? tile - a.tiles1 : tile) * 8 + t;
              if (e < ne) {
                uint32_t* pj = (second ? a.out2 : a.out1) + e +
                               (long long)(32 * g + 8 * h + 64 * brev2(q) + 256 * brev2(lq) +
                                           1024 * brev2(s)) * ne;
#pragma unroll
                for (int i = 0; i < 8; ++i) pj[i * ne] = y[i];
              }
            }
          }
          if (pass == 0 && s < 3) {
            // slice s now holds its part of the P2 operands
            tc::fence_proxy_async();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&pdone[s]);
          }
        }
      }
    }
    pdl_trigger();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
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

// point-major output E[pl + 64 m0 + 256 m1'][entry] viewed as (entry, m1', pl,
// m0) with boxes of 8 entries x 4 m1' x 32 pl x 4 m0 (the staging order)
bool out_map(CUtensorMap* m, uint32_t* base, long long ne) {
  auto fn = encode_fn();
  if (!fn || !base || ((uintptr_t)base & 15) || (ne & 3) || ne <= 0) return false;
  const cuuint64_t dims[4] = {(cuuint64_t)ne, 16, 64, 4};
  const cuuint64_t strides[3] = {(cuuint64_t)ne * 1024, (cuuint64_t)ne * 4, (cuuint64_t)ne * 256};
  const cuuint32_t box[4] = {8, 4, 32, 4};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, base, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool aligned16(const void* ptr) { return ((uintptr_t)ptr & 15) == 0; }

}  // namespace

int launch_ntt_fwd_mma64(const NttFwdArgs& f, const PrimeSet& ps, cudaStream_t st) {
  Mma64Args a{};
  a.in1 = (const uint32_t*)f.in; a.in1_stride = f.in_stride; a.out1 = f.out; a.n1 = f.n_entries;
  a.in2 = (const uint32_t*)f.in2; a.in2_stride = f.in2_stride; a.out2 = f.out2;
  a.n2 = f.n_entries2 > 0 ? f.n_entries2 : 0;
  a.len = f.len;
  a.kc1 = f.len <= 2048 ? 8 : 16;
  a.vec = (f.in_stride % 4 == 0) && aligned16(f.in) &&
          (a.n2 == 0 || ((f.in2_stride % 4 == 0) && aligned16(f.in2)));
  a.tiles1 = (a.n1 + 7) / 8;
  a.tiles = a.tiles1 + (a.n2 + 7) / 8;
  if (a.tiles == 0) return kOk;
  a.p = ps.pr[0].p;
  a.w16s = (uint32_t)((((uint64_t)1) << 48) / a.p);
  uint32_t inv = a.p;  // Newton: p^-1 mod 2^32 (p odd: 3 correct bits, doubled 4 times)
  for (int i = 0; i < 5; ++i) inv *= 2u - a.p * inv;
  a.pinv = inv;
  a.negp = 0u - a.p;
  a.zero = 0;
  a.c256 = 256;
  a.dbg = (int)option(kOptNttMmaDbg);
  a.tab = ps.pr[0].mma + kMma64TabOff;
  static bool attr = false;
  if (!attr) {
    FPM_CUDA_TRY(cudaFuncSetAttribute(ntt_mma64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kSmem));
    attr = true;
  }
  CUtensorMap om1{}, om2{};
  if (option(kOptNttPmLsu) == 0 && out_map(&om1, a.out1, a.n1) &&
      (a.n2 == 0 || out_map(&om2, a.out2, a.n2)))
    a.tma_out = 1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long grid = a.tiles < sms ? a.tiles : sms;
  FPM_CUDA_TRY(launch_pdl(ntt_mma64_kernel, dim3((unsigned)grid), dim3(kThreads), kSmem, st, a,
                          om1, om2));
  FPM_LAUNCH_CHECK();
  return kOk;
}

}  // namespace fpm
