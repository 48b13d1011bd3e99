// ntt_mma.cu -- batched forward N = 4096 NTTs on the int8 tensor cores (sm_100a).
//
// Replaces modring.ntt_forward as used by polmat._pm_mul_ntt (modring.py:253-
// 269, polmat.py:298-300) for the point-major product path (cfg5: 256x256x256,
// deg < 2048) -- the evaluation of every entry of A and B at the 4096 points.
// The word-size Shoup NTT (ntt_persist.cu) is bound by the integer multiply
// pipe (IMAD.HI at quarter rate, ~21 K modmuls per transform); here the
// radix-16 DFTs run as u8 x u8 -> s32 GEMMs on tcgen05 and the CUDA cores
// fold limbs, apply one scalar twiddle per point per pass boundary and move
// data.
//
// Decomposition (n = a + 16 b + 256 c, k = k0 + 16 k1 + 256 k2, w = w_4096,
// w16 = w^256):
//   P1  Y1[a,b,k0] = sum_c x[a,b,c] w16^(c k0),   Y1' = Y1 w^((a + 16 b) k0)
//   P2  Y2[a,k0,k1] = sum_b Y1' w16^(b k1),       Y2' = Y2 w^(16 a k1)
//   P3  X[k0 + 16 k1 + 256 k2] = sum_a Y2' w16^(a k2)
// Point k leaves at position brev12(k) = brev4(k2) + 16 brev4(k1) + 256
// brev4(k0): the bit-reversed (DIF) placement of the Shoup kernels, so the
// inverse transforms (ntt_persist.cu / ntt_tma.cu) and the pointwise kernels
// consume these evaluations unchanged.  The reversal costs nothing: P2 writes
// k1 into row group brev4(k1) and k0 into matrix brev4(k0) of P3's operand,
// and P3's DFT matrix has bit-reversed output columns.
//
// Each pass is 16 MMAs M = 128, N' = 64, K' = 64 (K' = 32 for P1 when the
// input has <= 2048 coefficients): the 128 rows are (digit u, transform t)
// = u * 8 + t for a tile of 8 transforms, the per-MMA fixed digit selects
// the A matrix, K' = 16 values x 4 raw little-endian bytes, N' = 16 outputs
// x 4 byte planes of the pre-scaled DFT matrix s_q = 2^(8q) w16^(nk) mod p
// (tc_grouped.cu's limb identity): D_r = sum byte_q(x) byte_r(s_q) < 2^22 and
// sum_r 2^(8r) D_r == DFT (mod p).
//
// The epilogue folds the 4 planes to a word < 2^32 (Shoup by 2^16, one
// IMAD.HI), applies the pass's twiddle (Shoup, from a swizzled 32 KB smem
// table), and writes the value straight into the NEXT pass's K-major A
// operand: the next pass's K digit is this pass's MMA digit, so a thread
// holding 4 consecutive MMAs of a chunk emits one 16-byte K chunk per
// output column (conflict-free: the 8 lanes of a quarter warp are the 8
// transforms of one row group).  Any residue < 2^32 is a valid operand, and
// the evaluations feed only the int8 tensor-core products, which take any
// 32-bit residue: nothing is reduced below p.
//
// Shared memory (one persistent CTA per SM): a 128 KB data region holding
// the tile's operands in place -- alternately "slice-major" (matrix m in
// slice m/4) and "chunk-major" (K chunk kc of every matrix in slice kc), so
// that chunk j of a pass only overwrites what the MMAs of chunk j have read
// -- the B matrices, the twiddle table and a 32 KB output staging tile.
// TMEM: two 256-column buffers (4 MMAs x 64 columns each), so the MMAs of
// chunk j+1 overlap the epilogue of chunk j.  Roles: warp 0 issues the MMAs
// (one thread); warps 1..16 are the workers (TMEM lane quarter warp % 4,
// column quarter (warp-1) / 4); warp 17 issues the TMA stores of the outputs
// (one box of 8 entries x 1024 positions, 32-byte point rows, per chunk of
// the last pass) and prefetches the next tile's input rows into L2; warps
// 18..19 load the next tile's input (L2 hits) and store slice j as soon as
// the last pass's MMAs of chunk j are done.
//
// Measured on cfg5 (timeline of clock64 stamps per chunk, profiles/r02):
// P1 / P2 chunks ~1.1-1.5 K cycles, P3 chunks bound by the TMA store of the
// 32-byte point rows (~1.5-2 K cycles per 32 KB box); the L2 prefetch of the
// next tile's input took the kernel 1.58 -> 1.38 ms, the input warps 1.38 ->
// 1.33 ms.  Rejected (slower): two 8-warp worker groups on alternating
// chunks (1.47), per-MMA TMEM-slot release (1.73), out-of-order MMA issue per
// group (2.12), staging in the freed data slices (1.46), half-chunk ping-pong
// staging (1.34-1.37: the TMA store rate, not the wait, bounds P3).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <vector>

#include "ntt.cuh"
#include "runtime.cuh"
#include "tc_common.cuh"

namespace fpm {

// ---- host tables --------------------------------------------------------------
// layout of Plan::mma (bytes):
//   [0, 4K)      DFT16 B operand (K-major SWIZZLE_NONE, LBO 128, SBO 512)
//   [4K, 8K)     the same with bit-reversed output columns (pass 3)
//   [8K, 40K)    twiddles: row m < 256, column j < 16: w^(m j)
// twiddle rows hold 16 (w, floor(w 2^32 / p)) pairs = 128 bytes; the 16-byte
// chunk c of row m is stored at chunk c ^ (m & 7) (conflict-free row reads).
constexpr uint32_t kMmaTabB = 0, kMmaTabBr = 4096, kMmaTabTw = 8192;
constexpr uint32_t kMmaTabBytes = 8192 + 32768;

void mma_ntt_tables(uint32_t p, uint32_t omega, std::vector<uint8_t>* out) {
  out->assign(kMmaTabBytes, 0);
  uint8_t* t = out->data();
  const uint64_t w16 = h_powmod(omega, 256, p);
  // row 4 c + r of the B operand: byte r of 2^(8q) w16^(n k), k = col(c), n =
  // the K slot's input digit
  auto bmat = [&](uint8_t* dst, bool rev) {
    for (int c = 0; c < 16; ++c) {
      const int k = rev ? ((c & 1) << 3) | ((c & 2) << 1) | ((c & 4) >> 1) | ((c & 8) >> 3) : c;
      for (int n = 0; n < 16; ++n) {
        const uint64_t base = h_powmod(w16, (uint64_t)n * k, p);
        for (int q = 0; q < 4; ++q) {
          const uint32_t s = (uint32_t)h_mulmod(base, ((uint64_t)1 << (8 * q)) % p, p);
          for (int r = 0; r < 4; ++r) {
            const int row = 4 * c + r, kb = 4 * n + q;
            dst[(row >> 3) * 512 + (kb >> 4) * 128 + (row & 7) * 16 + (kb & 15)] =
                (uint8_t)(s >> (8 * r));
          }
        }
      }
    }
  };
  bmat(t + kMmaTabB, false);
  bmat(t + kMmaTabBr, true);
  for (int m = 0; m < 256; ++m)
    for (int j = 0; j < 16; ++j) {
      const uint64_t w = h_powmod(omega, (uint64_t)m * j, p);
      const uint32_t pr[2] = {(uint32_t)w, h_shoup((uint32_t)w, p)};
      memcpy(t + kMmaTabTw + m * 128 + (((j >> 1) ^ (m & 7)) << 4) + (j & 1) * 8, pr, 8);
    }
}

namespace {

constexpr int kWorkers = 16;                     // worker warps (warps 1 .. 16)
constexpr int kLoaders = 2;                      // input warps (after the store warp)
constexpr int kVpm = 4;                          // outputs of one MMA per worker thread
constexpr int kThreads = 32 * (2 + kWorkers + kLoaders);
constexpr int kLT = 32 * kLoaders;               // loader threads
constexpr uint32_t kData = 131072;               // 8 transforms x 4096 words
constexpr uint32_t kOffB = kData;                // B matrices (natural, reversed columns)
constexpr uint32_t kOffTw = kOffB + 8192;
constexpr uint32_t kOffStage = kOffTw + 32768;   // output staging (one TMA box)
constexpr uint32_t kOffBar = kOffStage + 32768;
constexpr size_t kSmem = kOffBar + 256;

struct MmaArgs {
  const uint32_t* in1;
  const uint32_t* in2;
  long long in1_stride, in2_stride;  // words between entries' coefficient rows
  uint32_t* out1;
  uint32_t* out2;
  int n1, n2;                        // entries of the two batches
  int len;                           // coefficients per entry
  int kc1;                           // K chunks of P1 (2: len <= 2048, else 4)
  int vec;                           // 16-byte aligned rows: vector loads
  long long tiles1, tiles;
  uint32_t p, w16s;                  // w16s = floor(2^48 / p): Shoup companion of 2^16
  const uint8_t* tab;
  int tma_out;                       // point-major output by TMA stores
};

// data region offsets: slice-major (matrix m in slice m / 4) and chunk-major
// (K chunk kc of every matrix in slice kc); R = row = u * 8 + t
__device__ __forceinline__ uint32_t off_s(int m, int kc, int R) {
  return (uint32_t)((m >> 2) * 32768 + kc * 8192 + (m & 3) * 2048 + (R >> 3) * 128 + (R & 7) * 16);
}
__device__ __forceinline__ uint32_t off_k(int m, int kc, int R) {
  return (uint32_t)(kc * 32768 + m * 2048 + (R >> 3) * 128 + (R & 7) * 16);
}

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
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr));
  return v;
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

// byte permute with a zero second operand (ALU pipe; ptxas would turn a
// shift-add into IMAD on the multiply pipe, which the epilogue saturates)
__device__ __forceinline__ uint32_t prmt0(uint32_t a, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(0u), "r"(sel));
  return r;
}

// sum_r 2^(8r) d[r] (d[r] < 2^22) -> a congruent word < 2^31 + p:
// H = d2 + 2^8 d3 < 2^31, H 2^16 mod p by Shoup (q = hi(H w16s)), then
// d0 + 2^8 d1 + (H 2^16 mod p).  negp = 2^32 - p.
__device__ __forceinline__ uint32_t fold4(uint32_t d0, uint32_t d1, uint32_t d2, uint32_t d3,
                                          uint32_t p, uint32_t negp, uint32_t w16s) {
  const uint32_t H = d2 + prmt0(d3, 0x2104);            // d2 + (d3 << 8)
  const uint32_t q = __umulhi(H, w16s);
  uint32_t r = prmt0(H, 0x1044) + q * negp;             // (H << 16) - q p, in [0, 2p)
  r = min(r, r - p);
  return d0 + prmt0(d1, 0x2104) + r;                    // d0 + (d1 << 8) + r
}
// Shoup multiply with the negated modulus: a w - hi(a w') p, in [0, 2p)
__device__ __forceinline__ uint32_t shoup_n(uint32_t a, uint32_t w, uint32_t ws, uint32_t negp) {
  return a * w + __umulhi(a, ws) * negp;
}

// which batch a tile belongs to
struct TileSrc {
  const uint32_t* in;
  long long stride;
  int ne;
  long long e0;
};
__device__ __forceinline__ TileSrc tile_src(const MmaArgs& a, long long tile) {
  TileSrc s;
  if (tile < a.tiles1) {
    s.in = a.in1; s.stride = a.in1_stride; s.ne = a.n1; s.e0 = tile * 8;
  } else {
    s.in = a.in2; s.stride = a.in2_stride; s.ne = a.n2; s.e0 = (tile - a.tiles1) * 8;
  }
  return s;
}

// ---- input of one slice (P1 operand, slice-major) -----------------------------
// item = (transform t, a-quad aq, matrix b = 4j + sm, K chunk kc): four
// 16-byte loads x[4aq .. 4aq+3 + 16 b + 256 c], c = 4 kc .. 4 kc + 3,
// transposed into four 16-byte K chunks of rows (a, t).  128 kc1 items per
// slice, kLT * kLoadItems per round.
constexpr int kLoadItems = 4;
struct LoadBuf {
  uint4 g[kLoadItems][4];
};
__device__ __forceinline__ void slice_load(const MmaArgs& a, const TileSrc& s, int j, int i0,
                                           LoadBuf& lb) {
#pragma unroll
  for (int r = 0; r < kLoadItems; ++r) {
    const int it = i0 + kLT * r;
    const int t = it & 7, aq = (it >> 3) & 3, sm = (it >> 5) & 3, kc = it >> 7;
    const long long e = s.e0 + t;
    const int b = 4 * j + sm;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int n = 4 * aq + 16 * b + 256 * (4 * kc + i);
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
__device__ __forceinline__ void slice_store(uint32_t sdata, int j, int i0, const LoadBuf& lb) {
#pragma unroll
  for (int r = 0; r < kLoadItems; ++r) {
    const int it = i0 + kLT * r;
    const int t = it & 7, aq = (it >> 3) & 3, sm = (it >> 5) & 3, kc = it >> 7;
    const int b = 4 * j + sm;
    const uint4* g = lb.g[r];
    sts128(sdata + off_s(b, kc, (4 * aq + 0) * 8 + t), g[0].x, g[1].x, g[2].x, g[3].x);
    sts128(sdata + off_s(b, kc, (4 * aq + 1) * 8 + t), g[0].y, g[1].y, g[2].y, g[3].y);
    sts128(sdata + off_s(b, kc, (4 * aq + 2) * 8 + t), g[0].z, g[1].z, g[2].z, g[3].z);
    sts128(sdata + off_s(b, kc, (4 * aq + 3) * 8 + t), g[0].w, g[1].w, g[2].w, g[3].w);
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    ntt_mma_kernel(const __grid_constant__ MmaArgs a, const __grid_constant__ CUtensorMap om1,
                   const __grid_constant__ CUtensorMap om2) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = tc::smem_u32(smem);
  const uint32_t sdata = sbase, sB = sbase + kOffB, sTw = sbase + kOffTw, sStage = sbase + kOffStage;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  // full[2], empty[2], slice ready[4], last-pass chunk done[4], pass done[2],
  // staged, stage free; TMEM base
  uint64_t *full = bars, *empty = bars + 2, *ready = bars + 4, *p3done = bars + 8;
  uint64_t *pdone = bars + 12, *staged = bars + 14, *stfree = bars + 15;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // constant tables: the two B matrices and the twiddles (read once per CTA)
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.tab);
    uint4* dst = reinterpret_cast<uint4*>(smem + kOffB);  // B, B rev, twiddles: contiguous
    for (int i = tid; i < (int)(kMmaTabBytes / 16); i += kThreads) dst[i] = __ldg(src + i);
  }
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&full[b], 1);
      tc::mbar_init(&empty[b], kWorkers);
      tc::mbar_init(&pdone[b], kWorkers);
    }
    for (int j = 0; j < 4; ++j) {
      tc::mbar_init(&ready[j], kLoaders);
      tc::mbar_init(&p3done[j], 1);
    }
    tc::mbar_init(staged, kWorkers);
    tc::mbar_init(stfree, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_proxy_async();  // B matrices: generic stores -> tensor-core reads
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // inputs may come from the previous kernel

  if (warp == 0) {
    // ------------------------------- MMA issuer -------------------------------
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_u8(128, 64);
      // descriptors built once; an operand offset adds (offset >> 4) to the
      // 14-bit start-address field (all addresses < 256 KB: no carry out)
      const uint64_t dS = tc::make_desc(sdata, 8192, 128), dK = tc::make_desc(sdata, 32768, 128);
      const uint64_t dB = tc::make_desc(sB, 128, 512);
      int it = 0;
      for (long long tile = blockIdx.x; tile < a.tiles; tile += gridDim.x, ++it) {
#pragma unroll
        for (int pass = 0; pass < 3; ++pass) {
          const bool lay_k = pass == 1;
          const int ksteps = pass == 0 ? a.kc1 / 2 : 2;
          const uint64_t db = dB + (pass == 2 ? (uint64_t)(4096u >> 4) : 0u);  // reversed columns
          const uint64_t da = lay_k ? dK : dS;
          const uint32_t lbo = lay_k ? 32768u : 8192u;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            // buffer j & 1, its (j >> 1)-th use in this pass; the MMA thread
            // polls (test_wait): it must react at once
            const int buf = j & 1;
            tc::mbar_wait_spin(tc::smem_u32(&empty[buf]), ((j >> 1) & 1) ^ 1);
            if (pass == 0)
              tc::mbar_wait_spin(tc::smem_u32(&ready[j]), it & 1);
            else if (j == 0)
              tc::mbar_wait_spin(tc::smem_u32(&pdone[pass - 1]), it & 1);
            tc::fence_after_sync();
#pragma unroll
            for (int s = 0; s < 4; ++s) {
              const int m = 4 * j + s;
              const uint32_t a0 = lay_k ? (uint32_t)m * 2048u : (uint32_t)(m >> 2) * 32768u + (m & 3) * 2048u;
              const uint32_t d = tmem + buf * 256 + s * 64;
              tc::mma_u8(d, da + (a0 >> 4), db, idesc, 0u);
              if (ksteps == 2)
                tc::mma_u8(d, da + ((a0 + 2 * lbo) >> 4), db + (256 >> 4), idesc, 1u);
            }
            tc::commit(&full[buf]);
            if (pass == 2) tc::commit(&p3done[j]);  // slice j may be refilled
          }
        }
      }
    }
  } else if (warp == kWorkers + 1) {
    // ------------------------- output store warp (TMA) -------------------------
    if (a.tma_out && lane == 0) {
      tc::prefetch_tmap(&om1);
      tc::prefetch_tmap(&om2);
      for (long long tile = blockIdx.x; tile < a.tiles; tile += gridDim.x) {
        const bool second = tile >= a.tiles1;
        const int e0 = (int)((second ? tile - a.tiles1 : tile) * 8);
        // the next tile's input rows into L2 a tile ahead, so that the input
        // warps see L2 latency, not DRAM's (-12 % kernel time on cfg5)
        if (a.vec && tile + gridDim.x < a.tiles) {
          const TileSrc ns = tile_src(a, tile + gridDim.x);
          const uint32_t bytes = (uint32_t)((a.len * 4 + 15) & ~15);
          for (int t = 0; t < 8 && ns.e0 + t < ns.ne; ++t)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(
                             ns.in + (ns.e0 + t) * ns.stride),
                         "r"(bytes)
                         : "memory");
        }
        for (int j = 0; j < 4; ++j) {
          tc::mbar_wait(staged, j & 1);
          tma_store_4d(second ? &om2 : &om1, sStage, e0, 0, 0, 4 * j);
          tc::bulk_commit();
          tc::bulk_wait_read0();
          tc::mbar_arrive(stfree);
        }
      }
      tc::bulk_wait0();
    }
  } else if (warp > kWorkers + 1) {
    // ------------------------------ input warps -------------------------------
    // slice j of tile `it` once the last pass of tile it - 1 has read it; the
    // loads of the next slice are in flight while waiting
    const int i0 = (warp - kWorkers - 2) * 32 + lane;
    const uint32_t p3a = tc::smem_u32(p3done);
    int it = 0;
    for (long long tile = blockIdx.x; tile < a.tiles; tile += gridDim.x, ++it) {
      const TileSrc s = tile_src(a, tile);
#pragma unroll 1
      for (int j = 0; j < 4; ++j) {
#pragma unroll 1
        for (int part = 0; part < a.kc1 / 2; ++part) {
          LoadBuf lb;
          slice_load(a, s, j, i0 + part * kLT * kLoadItems, lb);
          if (part == 0 && it > 0) tc::mbar_wait_sleep_a(p3a + 8 * j, (it - 1) & 1);
          slice_store(sdata, j, i0 + part * kLT * kLoadItems, lb);
        }
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&ready[j]);
      }
    }
  } else {
    // --------------------------------- workers --------------------------------
    const int wk = warp - 1;          // 0 .. kWorkers - 1
    const int q = warp & 3;           // TMEM lane quarter this warp may access
    const int h = wk >> 2;            // column part: kVpm of the 16 outputs of each MMA
    const int R = 32 * q + lane;      // operand row = TMEM lane
    const int u = R >> 3, t = R & 7;  // row digit, transform of the tile
    const int c0 = kVpm * h;          // first output column of this thread
    const int ur = (int)(__brev((unsigned)u) >> 28);  // brev4(u)
    const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(4 * c0);
    const uint32_t p = a.p, w16s = a.w16s, negp = 0u - a.p;
    // per-thread bases: next-operand rows (P1 -> P2: column c0 + i -> row
    // group c0 + i; P2 -> P3: row group brev4(c0 + i)), staging slot
    const uint32_t sRow = sdata + (uint32_t)(c0 * 8 + t) * 16u;
    const uint32_t sRowR = sdata + (uint32_t)t * 16u;
    const uint32_t sSt = sStage + (uint32_t)(c0 * 128 + u * 8 + t) * 4u;  // [s][c][u][t]
    for (long long tile = blockIdx.x; tile < a.tiles; tile += gridDim.x) {
#pragma unroll
      for (int pass = 0; pass < 3; ++pass) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int buf = j & 1;
          tc::mbar_wait(&full[buf], (j >> 1) & 1);
          tc::fence_after_sync();
          uint32_t y[4][kVpm];
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            // two MMAs at a time (register budget: 20 warps -> 96 per thread)
            uint32_t v[2][4 * kVpm];
            tmem_ld16_nw(tl + buf * 256 + (2 * hf) * 64, v[0]);
            tmem_ld16_nw(tl + buf * 256 + (2 * hf + 1) * 64, v[1]);
            tc::tmem_wait_ld();
            if (hf == 1) {
              tc::fence_before_sync();
              __syncwarp();
              if (lane == 0) tc::mbar_arrive(&empty[buf]);
            }
#pragma unroll
            for (int ss = 0; ss < 2; ++ss)
#pragma unroll
              for (int i = 0; i < kVpm; ++i)
                y[2 * hf + ss][i] = fold4(v[ss][4 * i], v[ss][4 * i + 1], v[ss][4 * i + 2],
                                          v[ss][4 * i + 3], p, negp, w16s);
          }
          if (pass < 2) {
            // w^((u + 16 m) col) in P1 (row digit a = u, MMA digit b),
            // w^(16 m col) in P2 (MMA digit a)
#pragma unroll
            for (int s = 0; s < 4; ++s) {
              const int m = 16 * (4 * j + s) + (pass == 0 ? u : 0);  // m & 7 == (pass ? 0 : u & 7)
              const uint32_t rb = sTw + (uint32_t)m * 128u;
              const int sw = pass == 0 ? (u & 7) : 0;
#pragma unroll
              for (int i = 0; i < kVpm; i += 2) {
                const uint4 c = lds128(rb + ((uint32_t)(((c0 + i) >> 1) ^ sw) << 4));
                y[s][i] = shoup_n(y[s][i], c.x, c.y, negp);
                y[s][i + 1] = shoup_n(y[s][i + 1], c.z, c.w, negp);
              }
            }
            if (pass == 0) {
              // P2 operand: matrix u (= a), row (k0 = c0 + i, t), K chunk j
              const uint32_t mb = off_k(u, j, 0);
#pragma unroll
              for (int i = 0; i < kVpm; ++i)
                sts128(sRow + mb + (uint32_t)i * 128u, y[0][i], y[1][i], y[2][i], y[3][i]);
            } else {
              // P3 operand: matrix brev4(u) (u = k0), row (brev4(k1), t), K chunk j
              const uint32_t mb = off_s(ur, j, 0);
#pragma unroll
              for (int i = 0; i < kVpm; ++i) {
                const uint32_t rg = __brev((unsigned)(c0 + i)) >> 28;
                sts128(sRowR + mb + rg * 128u, y[0][i], y[1][i], y[2][i], y[3][i]);
              }
            }
          } else if (a.tma_out) {
            // position c + 16 u + 256 (4 j + s) (= brev12 of the point index);
            // staging [s][c][u][t]: one TMA box (8 entries x 1024 positions)
            tc::mbar_wait(stfree, (j & 1) ^ 1);
#pragma unroll
            for (int s = 0; s < 4; ++s)
#pragma unroll
              for (int i = 0; i < kVpm; ++i)
                sts32(sSt + (uint32_t)(s * 2048 + i * 128) * 4u, y[s][i]);
            tc::fence_proxy_async();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(staged);
          } else {
            // each warp store writes 4 full 32-byte sectors
            const bool second = tile >= a.tiles1;
            const long long ne = second ? a.n2 : a.n1;
            const long long e = (second ? tile - a.tiles1 : tile) * 8 + t;
            if (e < ne) {
              uint32_t* pj = (second ? a.out2 : a.out1) + e + (16 * u + c0 + 1024 * j) * ne;
#pragma unroll
              for (int s = 0; s < 4; ++s) {
                uint32_t* ps = pj + 256 * s * ne;
#pragma unroll
                for (int i = 0; i < kVpm; ++i) ps[i * ne] = y[s][i];
              }
            }
          }
        }
        if (pass < 2) {
          tc::fence_proxy_async();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&pdone[pass]);
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

PFN_cuTensorMapEncodeTiled_v12000 mma_encode_fn() {
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

// point-major output E[c + 16 u + 256 v][entry] viewed as (entry, u, c, v)
// with boxes of 8 entries x 16 u x 16 c x 4 v (the staging order)
bool out_map(CUtensorMap* m, uint32_t* base, long long ne) {
  auto fn = mma_encode_fn();
  if (!fn || !base || ((uintptr_t)base & 15) || (ne & 3) || ne <= 0) return false;
  const cuuint64_t dims[4] = {(cuuint64_t)ne, 16, 16, 16};
  const cuuint64_t strides[3] = {(cuuint64_t)ne * 64, (cuuint64_t)ne * 4, (cuuint64_t)ne * 1024};
  const cuuint32_t box[4] = {8, 16, 16, 4};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, base, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool aligned16(const void* ptr) { return ((uintptr_t)ptr & 15) == 0; }

}  // namespace

bool ntt_mma_fwd_ok(int logn, const NttFwdArgs& a, const PrimeSet& ps) {
  if (logn != 12 || option(kOptNttNoMma) != 0) return false;
  if (ps.count != 1 || ps.pr[0].mma == nullptr) return false;
  if (a.len2 > 0 && a.len2 != a.len) return false;  // one length for both batches
  if (ps.pr[0].p <= (1u << 30) || ps.pr[0].p >= (1u << 31)) return false;
  // 32-bit point offsets: 4096 * entries < 2^32
  return a.pm && !a.natural && !a.fold && !a.in64 && !a.reduce && a.len > 0 && a.len <= 4096 &&
         a.n_entries <= (1 << 20) && a.n_entries2 <= (1 << 20);
}

int launch_ntt_fwd_mma(const NttFwdArgs& f, const PrimeSet& ps, cudaStream_t st) {
  MmaArgs a{};
  a.in1 = (const uint32_t*)f.in; a.in1_stride = f.in_stride; a.out1 = f.out; a.n1 = f.n_entries;
  a.in2 = (const uint32_t*)f.in2; a.in2_stride = f.in2_stride; a.out2 = f.out2;
  a.n2 = f.n_entries2 > 0 ? f.n_entries2 : 0;
  a.len = f.len;
  a.kc1 = f.len <= 2048 ? 2 : 4;
  a.vec = (f.in_stride % 4 == 0) && aligned16(f.in) &&
          (a.n2 == 0 || ((f.in2_stride % 4 == 0) && aligned16(f.in2)));
  a.tiles1 = (a.n1 + 7) / 8;
  a.tiles = a.tiles1 + (a.n2 + 7) / 8;
  if (a.tiles == 0) return kOk;
  a.p = ps.pr[0].p;
  a.w16s = (uint32_t)((((uint64_t)1) << 48) / a.p);
  a.tab = ps.pr[0].mma;
  static bool attr = false;
  if (!attr) {
    FPM_CUDA_TRY(cudaFuncSetAttribute(ntt_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
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
  FPM_CUDA_TRY(launch_pdl(ntt_mma_kernel, dim3((unsigned)grid), dim3(kThreads), kSmem, st, a, om1,
                          om2));
  FPM_LAUNCH_CHECK();
  return kOk;
}

}  // namespace fpm
