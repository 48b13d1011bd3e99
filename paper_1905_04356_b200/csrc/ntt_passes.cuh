// ntt_passes.cuh -- register/shared-memory building blocks of the NTT kernels
// (ntt.cu generic kernels, ntt_persist.cu persistent kernels).  See ntt.cu
// for the four-step radix-32 formulation.
#pragma once
#include "common.cuh"

namespace fpm {
namespace nttp {

// PM (point-major output) launches use TPCX >= 2 transforms per CTA so each
// evaluation point receives a >= 8-byte contiguous row segment.
// TPCX == kPaired: two transforms per CTA on interleaved lanes (tr = lane & 1),
// so the two values of one point meet in a lane pair (shuffle, no smem).
constexpr int kPaired = 102;

template <int LOGN, int TPCX = 0>
struct Geo {
  static constexpr int N = 1 << LOGN;
  static constexpr int TPT = N / 32;                       // threads per transform
  static constexpr bool PAIRED = TPCX == kPaired;
  static constexpr int TPC = PAIRED ? 2 : (TPCX ? TPCX : (N >= 8192 ? 1 : 8192 / N));
  static constexpr int THREADS = TPT * TPC;                // 256 (N<=8192), 512, 1024
  static constexpr int NPASS = (LOGN + 4) / 5;             // 1, 2 or 3 passes
  static constexpr int LAST_R = LOGN - 5 * (NPASS - 1);    // bits of the last pass
  // padded smem words / transform (+16 when paired: the two transforms of a
  // warp then sit in opposite bank halves)
  static constexpr int STRIDE = N + N / 32 + (PAIRED ? 16 : 0);
  static constexpr int SMEM_BYTES = TPC * STRIDE * 4;
};

// Pass maps: thread-local element i (0..31) of local thread lt -> index x.
enum { MAP_TOP = 0, MAP_MID = 1, MAP_LAST = 2 };

template <int LOGN, int MAP>
__device__ __forceinline__ int xmap(int lt, int i) {
  if (MAP == MAP_TOP) return lt + (i << (LOGN - 5));
  if (MAP == MAP_MID) {
    constexpr int lo = LOGN - 10;
    return ((lt >> lo) << (LOGN - 5)) | (i << lo) | (lt & ((1 << lo) - 1));
  }
  return (lt << 5) | i;
}

__device__ __forceinline__ int pad(int x) { return x + (x >> 5); }

__host__ __device__ constexpr int brev5(int i) {
  return ((i & 1) << 4) | ((i & 2) << 2) | (i & 4) | ((i & 8) >> 2) | ((i & 16) >> 4);
}

// radix-2^R DIF over the low R bits of the register array (natural ->
// bit-reversed within each 2^R block); twiddles w_{2h}^j = w32^(j*16/h)
template <int R>
__device__ __forceinline__ void dif_small(uint32_t (&v)[32], const uint2* w, uint32_t p,
                                          bool upper_zero) {
#pragma unroll
  for (int hb = R - 1; hb >= 0; --hb) {
    const int h = 1 << hb;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (i & h) continue;
      const int e = (i & (h - 1)) * (16 / h);
      const uint32_t u = v[i];
      if (R == 5 && hb == 4 && upper_zero) {
        // first stage of a zero-padded input: (u, 0) -> (u, u*w)
        v[i + h] = e ? d_red(d_shoup(u, w[e].x, w[e].y, p), p) : u;
        continue;
      }
      const uint32_t b = v[i + h];
      const uint32_t s = d_red(u + b, p);
      uint32_t d = u - b + p;  // [1, 2p)
      if (e) d = d_shoup(d, w[e].x, w[e].y, p);
      v[i] = s;
      v[i + h] = d_red(d, p);
    }
  }
}

// radix-2^R DIT over the low R bits (bit-reversed -> natural), inverse roots
template <int R>
__device__ __forceinline__ void dit_small(uint32_t (&v)[32], const uint2* w, uint32_t p) {
#pragma unroll
  for (int hb = 0; hb < R; ++hb) {
    const int h = 1 << hb;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (i & h) continue;
      const int e = (i & (h - 1)) * (16 / h);
      const uint32_t u = v[i];
      uint32_t t = v[i + h];
      if (e) t = d_red(d_shoup(t, w[e].x, w[e].y, p), p);
      v[i] = d_red(u + t, p);
      v[i + h] = d_red(u - t + p, p);
    }
  }
}

template <int R>
__host__ __device__ constexpr int brev_r(int i) {
  int r = 0;
  for (int b = 0; b < R; ++b)
    if (i & (1 << b)) r |= 1 << (R - 1 - b);
  return r;
}
// register index of DIT-space index i: identity, or the low-R-bit reversal
template <int R, bool ALIAS>
__host__ __device__ constexpr int dit_ix(int i) {
  return ALIAS ? ((i & ~((1 << R) - 1)) | brev_r<R>(i & ((1 << R) - 1))) : i;
}

// radix-2^R DIT over the low R bits with lazy reductions (ntt_tma.cu).
//  * ALIAS = false: bit-reversed -> natural (inverse passes).
//  * ALIAS = true: the same butterflies on registers renamed by the R-bit
//    reversal compute the DFT of naturally ordered values and leave X[k] in
//    register brev(k) -- exactly the DIF placement -- so forward passes use it
//    too (the network and the results are the DIF ones).
//  * A value that the next stage only multiplies (a b-operand with a nonzero
//    twiddle) skips its reduction: the Shoup multiply accepts any input
//    < 2^32 and the sums / differences stay < 2p < 2^32.  LAZY_OUT extends
//    this to the last stage when a row-twiddle multiply follows every value.
//  * HALF_ZERO (forward, R = 5): the upper 16 natural inputs are zero, so the
//    first stage is a copy (u, 0) -> (u, u).
// Inputs must be < p.
template <int R, bool ALIAS, bool LAZY_OUT, bool HALF_ZERO = false>
__device__ __forceinline__ void dit_lazy(uint32_t (&v)[32], const uint2* w, uint32_t p) {
#pragma unroll
  for (int hb = 0; hb < R; ++hb) {
    const int h = 1 << hb;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (i & h) continue;
      const int a = dit_ix<R, ALIAS>(i), b = dit_ix<R, ALIAS>(i + h);
      if (HALF_ZERO && hb == 0) {
        v[b] = v[a];
        continue;
      }
      const int e = (i & (h - 1)) * (16 / h);
      bool lazy_a = LAZY_OUT, lazy_b = LAZY_OUT;
      if (hb < R - 1) {
        const int h2 = 2 * h;
        lazy_a = (i & h2) && (i & (h2 - 1));
        lazy_b = ((i + h) & h2) && ((i + h) & (h2 - 1));
      }
      uint32_t t = v[b];
      if (e) t = d_red(d_shoup(t, w[e].x, w[e].y, p), p);
      const uint32_t u = v[a];
      const uint32_t s = u + t, d = u - t + p;
      v[a] = lazy_a ? s : d_red(s, p);
      v[b] = lazy_b ? d : d_red(d, p);
    }
  }
}

// split load / apply so a row's 16-byte loads are issued a whole radix-32
// DFT (or smem exchange) ahead of their use
struct Row {
  uint4 t[16];
};
__device__ __forceinline__ void row_load(Row& r, const uint2* __restrict__ row) {
  const uint4* r4 = reinterpret_cast<const uint4*>(row);
#pragma unroll
  for (int q = 0; q < 16; ++q) r.t[q] = __ldg(r4 + q);
}
__device__ __forceinline__ void row_apply(uint32_t (&v)[32], const Row& r, uint32_t p) {
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const uint4 t = r.t[q];
    const int k0 = 2 * q, k1 = 2 * q + 1;
    if (k0) {
      const int i0 = brev5(k0);
      v[i0] = d_red(d_shoup(v[i0], t.x, t.y, p), p);
    }
    const int i1 = brev5(k1);
    v[i1] = d_red(d_shoup(v[i1], t.z, t.w, p), p);
  }
}

template <int LOGN, int MAP>
__device__ __forceinline__ void to_smem(uint32_t* smt, const uint32_t (&v)[32], int lt) {
#pragma unroll
  for (int i = 0; i < 32; ++i) smt[pad(xmap<LOGN, MAP>(lt, i))] = v[i];
}
template <int LOGN, int MAP>
__device__ __forceinline__ void from_smem(const uint32_t* smt, uint32_t (&v)[32], int lt) {
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = smt[pad(xmap<LOGN, MAP>(lt, i))];
}


}  // namespace nttp
}  // namespace fpm
