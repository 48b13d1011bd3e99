// mbasis_fast.cu -- M-Basis leaf as two kernels (31-bit primes).
//
// The reference M-Basis (appint.py:143-180) interleaves three things per
// order-1 step: the residual R_k = coeff_k(P F), the canonical step
// (appint.py:24-60) and P <- Q_k P plus s <- rdeg_s(P).  Two facts split the
// work into a short sequential chain and a wide parallel product:
//   * s <- rdeg_s(P) equals s + delta (delta = 1 on the step's pivot rows):
//     P stays s-ordered weak Popov, hence s-reduced, and the predictable
//     degree property gives rdeg(Q_k P) = rdeg_{rdeg(P)}(Q_k) = s + delta
//     (checked against the reference on 3595 steps incl. degenerate inputs);
//   * so the chain needs only the residual list G = P F mod x^T, updated by
//     each step (the reference's update_list variant, appint.py:173-178).
// Kernel A runs the T steps in one CTA with G in shared memory and records
// every step (pivot order + kernel-row coefficients).  Kernel B rebuilds
// P = Q_{T-1} ... Q_0 from the records, one CTA per column of P (the update
// P <- Q P never mixes columns).
//
// Canonical step, exactly as the reference: rows ranked by (s_i, i); the
// pivot rows are the rows outside the span of their predecessors, found by
// column elimination that always picks the lowest-ranked remaining row (the
// pivot SET is the greedy basis, independent of elimination order); kernel
// row i of the basis is e_i - sum_j c_ij e_j over pivot rows j (unique).
// The elimination is division free: row_i <- (a*row_i - b*row_r) * 2^-32
// (one Montgomery reduction; a nonzero row factor is harmless), with a
// transform matrix X tracking each row; at the end c_ij = -X_ij / X_ii.
// One barrier per column: while updating, the owner of column c+1 of each
// row already reduces the next pivot key.
#include <climits>
#include <cstdlib>
#include "pmbasis.cuh"
#include "tc_common.cuh"

namespace fpm {
namespace {

struct F31 {
  uint32_t p, pinv;  // pinv = -p^-1 mod 2^32
  uint64_t mu;       // floor(2^64 / p)
  uint32_t c32;      // 2^32 mod p
  uint32_t r2;       // 2^64 mod p (into the Montgomery domain)
  uint32_t m58;      // floor(2^58 / p): d_red56 of the residual-list sums
  uint32_t w24s;     // floor(2^56 / p): Shoup companion of 2^24 (byte-plane scalings)
};

// release / acquire of a step-done flag at GPU scope (the build kernel runs
// beside the steps kernel and follows it step by step)
__device__ __forceinline__ void flag_release(uint32_t* f, uint32_t v) {
  // after a CTA barrier: the release is cumulative over the other threads' writes
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(f), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t flag_acquire(const uint32_t* f) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(f) : "memory");
  return v;
}

// (a*w + (p-b)*y) * 2^-32 mod p, all inputs < p, result < p
__device__ __forceinline__ uint32_t redc_axby(uint32_t a, uint32_t w, uint32_t b, uint32_t y,
                                              const F31& f) {
  const uint64_t acc = (uint64_t)a * w + (uint64_t)(f.p - b) * y;  // < 2p^2 < 2^63
  const uint32_t m = (uint32_t)acc * f.pinv;
  const uint32_t t = (uint32_t)((acc + (uint64_t)m * f.p) >> 32);  // < 2p
  return min(t, t - f.p);
}

__device__ __forceinline__ uint32_t mulmod(uint32_t a, uint32_t b, const F31& f) {
  return d_red64((uint64_t)a * b, f.p, f.mu);
}

// Montgomery product a b 2^-32 mod p (a, b < p)
__device__ __forceinline__ uint32_t redc_mul(uint32_t a, uint32_t b, const F31& f) {
  const uint64_t acc = (uint64_t)a * b;
  const uint32_t m = (uint32_t)acc * f.pinv;
  const uint32_t t = (uint32_t)((acc + (uint64_t)m * f.p) >> 32);
  return min(t, t - f.p);
}

// a^(p-2) by square-and-multiply in the Montgomery domain (cheaper products
// than Barrett; x -> x 2^32 on entry via r2 = 2^64 mod p, 2^-32 on exit)
// (r2 precomputed on the host: a 128-bit modulo here costs thousands of cycles)
__device__ uint32_t invmod(uint32_t a, const F31& f) {
  uint32_t b = redc_mul(a, f.r2, f);         // a R
  uint32_t r = redc_mul(1u, f.r2, f);        // R
  const uint32_t e = f.p - 2;                // < 2^31: 31 right-to-left steps
#pragma unroll
  for (int i = 0; i < 31; ++i) {
    const uint32_t rb = redc_mul(r, b, f);   // independent of the squaring chain
    r = (e >> i) & 1u ? rb : r;
    b = redc_mul(b, b, f);
  }
  return redc_mul(r, 1u, f);                 // out of the Montgomery domain
}

__device__ __forceinline__ uint64_t fold(uint64_t acc, uint32_t c32) {
  return (uint64_t)(uint32_t)(acc >> 32) * c32 + (uint32_t)acc;
}

// (d*v - al*x - be*y) * 2^-32 mod p, all inputs < p, result < p
__device__ __forceinline__ uint32_t redc3(uint32_t d, uint32_t v, uint32_t al, uint32_t x,
                                          uint32_t be, uint32_t y, const F31& f) {
  uint64_t acc = (uint64_t)d * v + (uint64_t)(f.p - al) * x + (uint64_t)(f.p - be) * y;  // < 3p^2
  acc = fold(acc, f.c32);                                 // < 2^63, same residue
  const uint32_t m = (uint32_t)acc * f.pinv;
  const uint32_t t = (uint32_t)((acc + (uint64_t)m * f.p) >> 32);  // < 2p
  return min(t, t - f.p);
}

// Generic canonical step for n = NC pivot columns, m <= 64 rows, 512 threads:
// Gauss-Jordan on [R_P^T | R_K^T] (NC x m; R_P = the NC lowest-ranked rows
// of the residual, R_K = the others in index order), TWO columns per barrier.
// For the 2 x 2 pivot block [[a, b], [d, e]] (rows c, c+1) and any other row
// with entries (x, y) in those columns,
//    row <- D row - (x e - y d) row_c - (y a - x b) row_{c+1},  D = a e - b d,
//    row_c <- e row_c - b row_{c+1},  row_{c+1} <- a row_{c+1} - d row_c
// clear both columns (every row picks up a nonzero factor, harmless).  With
// a != 0 and D != 0 at every block all leading principal minors of R_P are
// nonzero, so the reference's column elimination (appint.py:41-58) takes
// exactly the rows in rank order as pivots and the kernel coefficients are the
// unique C = R_K R_P^-1; the left block ends diagonal (d_q) and the right
// block is D C^T, so Ct[q][kr] = -right[q][kr] / d_q with no product phase.
// Thread (gi, gs) holds row gi, columns gs + 16u.  W is R_k with row stride
// NC + 1 (conflict-free column reads).  Returns false (uniformly) on a zero
// leading minor; the shared step state is then untouched.
//
// No CTA barrier per block: rows c, c+1 live in warp c / 2, which publishes
// them in the block's OWN buffer (NC / 2 buffers of 128 words) when it gets to
// block c -- it has applied every earlier block by then -- and arrives on the
// block's mbarrier bars[c / 2] (phase parity par of this call); the other
// warps wait on it, suspended, and each runs ahead as far as its data allows
// (a barrier per block cost as much as the block's arithmetic).
template <int NC>
__device__ bool solve_pairs(const uint32_t* W, int m, const int* ord, const int* klist,
                            uint32_t* pbuf, const F31& f, uint32_t* Ct, uint32_t* recC,
                            unsigned long long* trace, uint32_t* sig, uint32_t epoch,
                            uint64_t* bars, uint32_t par) {
  static_assert(NC == 32, "16 threads x 4 columns per row, 64 columns");
  const int tid = threadIdx.x, gi = tid >> 4, gs = tid & 15;
  const int nk = m - NC;
  uint32_t v[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int col = gs + 16 * u;
    v[u] = col < NC ? W[ord[col] * (NC + 1) + gi]
                    : (col < m ? W[klist[col - NC] * (NC + 1) + gi] : 0u);
  }
  // once c >= 16, columns 0..15 (u = 0) of every row are final zeros except
  // the diagonals of rows < 16, which each block only rescales by D 2^-32:
  // u = 0 is skipped and the product of those factors kept in S (Montgomery
  // form) for the final diagonal
  uint32_t S = f.c32;
#pragma unroll
  for (int c = 0; c < NC; c += 2) {
    constexpr int kSkip = 16;
    const int u0 = c >= kSkip ? 1 : 0;
    uint32_t* pb = pbuf + (c >> 1) * 128;
    if ((tid >> 5) == (c >> 1)) {  // the warp of rows c, c + 1
#pragma unroll
      for (int u = 0; u < 4; ++u) pb[(gi - c) * 64 + gs + 16 * u] = v[u];
      __syncwarp();
      if ((tid & 31) == 0) tc::mbar_arrive(&bars[c >> 1]);
    }
    tc::mbar_wait(&bars[c >> 1], par);
    const uint32_t a = pb[c], b = pb[c + 1], d = pb[64 + c], e = pb[64 + c + 1];
    const uint32_t dl = redc_axby(a, e, b, d, f);
    if (a == 0 || dl == 0) return false;  // every thread read the same block
    if (trace && c == 0 && tid == 0) trace[7] = clock64();
    const uint32_t x = __shfl_sync(0xffffffffu, v[c >> 4], c & 15, 16);
    const uint32_t y = __shfl_sync(0xffffffffu, v[(c + 1) >> 4], (c + 1) & 15, 16);
    // the row factors al = x e - y d (even lanes), be = y a - x b (odd lanes),
    // once per lane pair instead of both in every lane
    const bool odd = gs & 1;
    const uint32_t ab = redc_axby(odd ? y : x, odd ? a : e, odd ? x : y, odd ? b : d, f);
    const uint32_t al = __shfl_sync(0xffffffffu, ab, 0, 16);
    const uint32_t be = __shfl_sync(0xffffffffu, ab, 1, 16);
    if (c >= kSkip) S = redc_mul(S, dl, f);
    uint32_t rc[4], rd[4];
#pragma unroll
    for (int u = u0; u < 4; ++u) {
      rc[u] = pb[gs + 16 * u];
      rd[u] = pb[64 + gs + 16 * u];
    }
    if (gi == c) {
#pragma unroll
      for (int u = u0; u < 4; ++u) v[u] = redc_axby(e, rc[u], b, rd[u], f);
    } else if (gi == c + 1) {
#pragma unroll
      for (int u = u0; u < 4; ++u) v[u] = redc_axby(a, rd[u], d, rc[u], f);
    } else {
#pragma unroll
      for (int u = u0; u < 4; ++u) v[u] = redc3(dl, v[u], al, rc[u], be, rd[u], f);
    }
  }
  if (trace && tid == 0) trace[6] = clock64();
  // d_q = M[q][q] (row q: lane q & 15, register q >> 4) is published in
  // block 0's pivot buffer (every warp is past it: each waited for the last
  // block, whose rows were published by a warp that had read all the others'
  // -- but a warp may still be reading the LAST block's buffer, hence the CTA
  // barrier first); one warp inverts all NC of them (16 lanes per row
  // inverting the same value cost 4x the issue slots)
  __syncthreads();
  if (gs == (gi & 15)) pbuf[gi] = (gi >> 4) ? v[1] : v[0];
  __syncthreads();
  if (tid < NC) {
    uint32_t dq = pbuf[tid];
    if (NC > 16 && tid < 16) dq = redc_mul(dq, S, f);  // the skipped rescalings
    pbuf[64 + tid] = invmod(dq, f);
  } else if (sig && tid == (int)blockDim.x - 1) {
    // the previous step's done flag: its GPU-scope release (~0.7 us) hides
    // behind the inversions instead of delaying a barrier
    flag_release(sig, epoch);
  }
  __syncthreads();
  const uint32_t iq = pbuf[64 + gi];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int col = gs + 16 * u;
    if (col >= NC && col < m) {
      const uint32_t c = mulmod(v[u], iq, f);
      const uint32_t val = c ? f.p - c : 0u;
      Ct[gi * nk + col - NC] = val;
      recC[gi * nk + col - NC] = val;
    }
  }
  return true;
}

// Residual-list update on R x 4 tiles (aligned shapes, folds every 4
// products): G[t][klist[kr]][j] += sum_q Ct[q][kr] G[t][plist[q]][j] for the
// kernel rows kr of one R-row block and 4 columns j.  Smaller R spreads a
// short list (few t) over all threads instead of leaving most of them idle.
template <int R>
__device__ __forceinline__ void residual_tiles(uint32_t* G, const uint32_t* Ct,
                                               const long long* krow, const long long* prow,
                                               int n, int nk, int np, int k, int nt, size_t mn,
                                               const F31& f) {
  const int rb_n = nk / R, cb_n = n >> 2;
  const int blocks = rb_n * cb_n * nt;
  for (int b = threadIdx.x; b < blocks; b += blockDim.x) {
    const int t = k + 1 + b / (rb_n * cb_n);
    const int rem = b - (b / (rb_n * cb_n)) * (rb_n * cb_n);
    const int rb = rem / cb_n, cb = rem - (rem / cb_n) * cb_n;
    uint32_t* Gt = G + (size_t)t * mn;
    long long rows[R];
    uint64_t acc[R][4];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      rows[r] = krow[rb * R + r];
      const uint4 g = *reinterpret_cast<const uint4*>(Gt + rows[r] + cb * 4);
      acc[r][0] = g.x; acc[r][1] = g.y; acc[r][2] = g.z; acc[r][3] = g.w;
    }
#pragma unroll 4
    for (int q = 0; q < np; ++q) {
      const uint4 g4 = *reinterpret_cast<const uint4*>(Gt + prow[q] + cb * 4);
      const uint32_t gv[4] = {g4.x, g4.y, g4.z, g4.w};
      uint32_t cv[R];
      if constexpr (R == 4) {
        const uint4 c4 = *reinterpret_cast<const uint4*>(Ct + q * nk + rb * 4);
        cv[0] = c4.x; cv[1] = c4.y; cv[2] = c4.z; cv[3] = c4.w;
      } else if constexpr (R == 2) {
        const uint2 c2 = *reinterpret_cast<const uint2*>(Ct + q * nk + rb * 2);
        cv[0] = c2.x; cv[1] = c2.y;
      } else {
        cv[0] = Ct[q * nk + rb];
      }
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) acc[r][cc] += (uint64_t)cv[r] * gv[cc];
      if ((q & 3) == 3) {
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) acc[r][cc] = fold(acc[r][cc], f.c32);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
      *reinterpret_cast<uint4*>(Gt + rows[r] + cb * 4) =
          make_uint4(d_red64(acc[r][0], f.p, f.mu), d_red64(acc[r][1], f.p, f.mu),
                     d_red64(acc[r][2], f.p, f.mu), d_red64(acc[r][3], f.p, f.mu));
  }
}

// Residual-list update of the pair path (m = 64, n = np = nk = 32) on the
// int8 tensor cores with register-level mma.sync (m16n8k32, u8 x u8 -> s32,
// 8 cycles per warp-mma per SMSP measured, tools/micro/imma.cu):
// G_t[klist[kr]][j] += sum_q Ct[q][kr] G_t[plist[q]][j] for every t > k,
// computed transposed (M = j, N = kr).  With K' = (q, b) (b = byte of G) and
// S_b = 2^(8b) Ct mod p split into bytes r, the sum is sum_r 2^(8r) D_r,
// D_r[j][kr] = sum_K' byte_b(G_t[plist[q]][j]) byte_r(S_b[q][kr]): the A
// fragments are the raw residual words themselves, the B fragments (one kr
// tile per warp, all four planes, 32 registers) are built once per step in
// Apk (4 planes x 32 x 32 words, XOR-swizzled rows) and stay in registers.
// D_r < 128 * 255^2 < 2^23, so sum_r 2^(8r) D_r + G < 2^49 is one d_red56.
__device__ __forceinline__ int apk_idx(int r, int row, int q) {
  return (r * 32 + row) * 32 + (q ^ ((row & 7) << 2));
}
__device__ __forceinline__ void mma_u8_16832(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                             uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};\n"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ void residual_mma(uint32_t* G, const uint32_t* Ct, uint32_t* Apk,
                             const long long* krow, const long long* prow, int k, int nt,
                             size_t mn, const F31& f) {
  const bool big = f.p >= (1u << 30);  // d_red56 / the shared Shoup quotient need p >= 2^30
  {
    // 2^(8b) c mod p for b = 1, 2, 3 from ONE multiply-high (p >= 2^30, c < p):
    // q3 = hi(c floor(2^56 / p)) is the Shoup quotient of c 2^24 (error < 2),
    // and q3 >> 8, q3 >> 16 are those of c 2^16, c 2^8 with error < 1.01, so
    // every c 2^(8b) - q p lies in [0, 2p) -- any such residue is a valid operand
    for (int idx = threadIdx.x; idx < 32 * 32; idx += blockDim.x) {
      const int kr = idx >> 5, q = idx & 31;
      const uint32_t c = Ct[q * 32 + kr];
      uint32_t sb[4] = {c, 0u, 0u, 0u};
      if (big) {
        const uint32_t q3 = __umulhi(c, f.w24s);
        sb[1] = (c << 8) - (q3 >> 16) * f.p;
        sb[2] = (c << 16) - (q3 >> 8) * f.p;
        sb[3] = (c << 24) - q3 * f.p;
      } else {
        sb[1] = mulmod(c, 256u % f.p, f);
        sb[2] = mulmod(c, (uint32_t)(65536ull % f.p), f);
        sb[3] = mulmod(c, (uint32_t)((1ull << 24) % f.p), f);
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {  // byte r of sb[0..3] (PRMT)
        const uint32_t lo = __byte_perm(sb[0], sb[1], r | ((4 + r) << 4));
        const uint32_t hi = __byte_perm(sb[2], sb[3], r | ((4 + r) << 4));
        Apk[apk_idx(r, kr, q)] = __byte_perm(lo, hi, 0x5410);
      }
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
  const int nw = blockDim.x >> 5;          // 16: 4 kr tiles x 4 tile streams
  const int nbk = warp & 3, sub = warp >> 2, nsub = nw >> 2;
  const int kr_b = nbk * 8 + g;            // B fragment column n = g
  uint32_t bf[4][4][2];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      bf[r][kk][0] = Apk[apk_idx(r, kr_b, kk * 8 + tig)];
      bf[r][kk][1] = Apk[apk_idx(r, kr_b, kk * 8 + tig + 4)];
    }
  const int tiles = 2 * nt;  // (t, 16 columns j) per kr tile
  for (int tile = sub; tile < tiles; tile += nsub) {
    const int t = k + 1 + (tile >> 1), j0 = (tile & 1) * 16;
    uint32_t* Gt = G + (size_t)t * mn;
    int d[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int e = 0; e < 4; ++e) d[r][e] = 0;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const uint32_t* g0 = Gt + prow[kk * 8 + tig] + j0 + g;
      const uint32_t* g1 = Gt + prow[kk * 8 + tig + 4] + j0 + g;
      const uint32_t a0 = g0[0], a1 = g0[8], a2 = g1[0], a3 = g1[8];
#pragma unroll
      for (int r = 0; r < 4; ++r) mma_u8_16832(d[r], a0, a1, a2, a3, bf[r][kk][0], bf[r][kk][1]);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int j = j0 + g + (e >> 1) * 8, kr = nbk * 8 + tig * 2 + (e & 1);
      uint32_t* dst = Gt + krow[kr] + j;
      const uint64_t acc = (uint64_t)(uint32_t)d[0][e] + ((uint64_t)(uint32_t)d[1][e] << 8) +
                           ((uint64_t)(uint32_t)d[2][e] << 16) +
                           ((uint64_t)(uint32_t)d[3][e] << 24) + *dst;
      *dst = big ? d_red56(acc, f.p, f.m58) : d_red64(acc, f.p, f.mu);
    }
  }
}

struct StepArgs {
  const uint32_t* F;
  long long fs;
  long long ts;           // F[e * fs + t * ts]: coefficient (or point) t of entry e
  const uint32_t* alpha;  // interpolant points (m_intbasis), nullptr for approximants
  int lf, m, n, T;
  const int64_t* s;   // device shift (m)
  int* rec_np;        // [T] number of pivots
  int* rec_plist;     // [T][m] pivot rows in discovery order
  uint32_t* rec_Ct;   // [T][m*m] compact: Ct[q*nk + kr] = -c_{klist[kr], plist[q]}
  int64_t* sft_out;   // final shift (m)
  int fold_k;         // products between folds (pointwise.cu fold_period)
  F31 f;
  unsigned long long* trace;  // profiling only (FPM_MBASIS_TRACE): [T][6] clocks
  uint32_t* flags;    // [T + 1]: flags[k] = epoch once step k's record is written
  uint32_t epoch;     //          flags[T] = epoch once every output is written
};

constexpr int kStepThreads = 512;

#define STEP_TRACE(ev) \
  if (a.trace && tid == 0) a.trace[k * 8 + (ev)] = clock64();

__global__ void __launch_bounds__(kStepThreads, 1) mbasis_steps_kernel(const __grid_constant__ StepArgs a) {
  pdl_wait();
  pdl_trigger();  // the build kernel starts now and waits on the step flags
  extern __shared__ __align__(16) unsigned char smraw[];
  const int m = a.m, n = a.n, T = a.T;
  const int tid = threadIdx.x;
  if (a.trace && tid == 0) a.trace[63 * 8] = clock64();  // kernel start (after the dependency wait)
  const F31 f = a.f;
  const uint32_t p = f.p;
  const size_t mn = (size_t)m * n;
  int64_t* sft = (int64_t*)smraw;                 // m
  uint32_t* G = (uint32_t*)(sft + m);             // [T][m][n]
  uint32_t* W = G + (size_t)T * mn;               // [m][n]  (later: compact Ct)
  uint32_t* X = W + mn;                           // [m][m]
  uint32_t* inv = X + (size_t)m * m;              // m
  int* rank = (int*)(inv + m);                    // m
  int* ord = rank + m;                            // m
  int* piv = ord + m;                             // m
  int* plist = piv + m;                           // m
  int* klist = plist + m;                         // m
  // Per-row coefficient offsets: multiplying pivot row i by x shifts its
  // residual coefficients (G[t][i] <- G[t-1][i]); instead of moving data the
  // row's offset grows, coefficient t of row i living in slot t - off[i].
  // rowoff[i] = i*n - off[i]*mn, so G[t][i] starts at G + t*mn + rowoff[i].
  int* off = klist + m;                           // m
  long long* rowoff = (long long*)(((uintptr_t)(off + m) + 7) & ~(uintptr_t)7);  // m
  long long* prow = rowoff + m;                   // m: rowoff[plist[q]] of the step
  long long* krow = prow + m;                     // m: rowoff[klist[kr]] of the step
  __shared__ int s_key[2];
  __shared__ int s_nk;
  // block solves: pivot rows (+ column); solve_pairs: one 128-word buffer and
  // one mbarrier per 2 x 2 block
  __shared__ uint32_t sbuf[16 * 128];
  __shared__ uint64_t sbar[16];
  uint32_t spar = 0;  // phase parity of sbar for the next solve_pairs call
  if (threadIdx.x == 0) {
    for (int b = 0; b < 16; ++b) tc::mbar_init(&sbar[b], 1);
    tc::fence_mbar_init();
  }

  const int hw = tid >> 4, l16 = tid & 15;  // half-warp per row
  constexpr int kRowsPerPass = kStepThreads / 16;

  // the residual list G = F mod x^T: every load of two entries is issued before
  // the first store.  (The whole prologue -- this load, the barrier setup and
  // the first ranking -- is 9.3 K cycles of a 228 K-cycle leaf, tools/mbasis_trace.py.)
  for (int e0 = tid; e0 < (int)mn; e0 += 2 * kStepThreads) {
    for (int t0 = 0; t0 < T; t0 += 8) {
      uint32_t v[2][8];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int e = e0 + j * kStepThreads;
        const uint32_t* fe = a.F + (long long)e * a.fs;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int t = t0 + u;
          v[j][u] = (e < (int)mn && t < T && t < a.lf) ? __ldg(fe + (long long)t * a.ts) : 0u;
        }
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int e = e0 + j * kStepThreads;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (e < (int)mn && t0 + u < T) G[(size_t)(t0 + u) * mn + e] = v[j][u];
      }
    }
  }
  for (int i = tid; i < m; i += kStepThreads) {
    sft[i] = a.s[i];
    off[i] = 0;
    rowoff[i] = (long long)i * n;
  }
  __syncthreads();

  int pending = -1;  // step whose done flag is not released yet
  for (int k = 0; k < T; ++k) {
    const uint32_t* Gk = G + (size_t)k * mn;  // + rowoff[i] - i*n per row
    auto gk = [&](int idx) {
      const int i = idx / n;
      return Gk[rowoff[i] + (idx - i * n)];
    };
    const bool pairs_shape = n == 32 && m > n && m <= 64;  // solve_pairs
    if (pairs_shape) {
      // the pair solve reads R_k column-wise: a copy with row stride n + 1
      // (in X, unused on that path) makes those reads bank-conflict free
      for (int idx = tid; idx < (int)mn; idx += kStepThreads)
        X[(idx / n) * (n + 1) + (idx - (idx / n) * n)] = gk(idx);
    } else {
      for (int idx = tid; idx < (int)mn; idx += kStepThreads) W[idx] = gk(idx);
    }
    const bool try_fast = !pairs_shape && m > n && n <= 32 && 2 * n * n + n * (m - n + 1) <= m * m;
    if (!try_fast && !pairs_shape)
      for (int idx = tid; idx < m * m; idx += kStepThreads)
        X[idx] = (idx / m == idx - (idx / m) * m) ? 1u : 0u;
    // rank of row i by (s_i, i): 8 threads per row, shuffle-reduced
    for (int i0 = 0; i0 < m; i0 += kStepThreads / 8) {
      const int i = i0 + (tid >> 3), part = tid & 7;
      int r = 0;
      if (i < m) {
        const int64_t si = sft[i];
        for (int j = part; j < m; j += 8) r += (sft[j] < si) || (sft[j] == si && j < i);
      }
      r += __shfl_xor_sync(0xffffffffu, r, 1);
      r += __shfl_xor_sync(0xffffffffu, r, 2);
      r += __shfl_xor_sync(0xffffffffu, r, 4);
      if (i < m && part == 0) {
        rank[i] = r;
        ord[r] = i;
        piv[i] = 0;
      }
    }
    if (tid < 2) s_key[tid] = INT_MAX;
    __syncthreads();
    STEP_TRACE(0);

    // ---- generic residual: block solve ----------------------------------------
    // When every leading principal minor of R_P (the n lowest-ranked rows,
    // columns 0..n-1) is nonzero, the column elimination below would pick
    // exactly those rows as pivots in rank order, and the kernel-row
    // coefficients are C = R_K R_P^-1 (unique).  Gauss-Jordan on [R_P | I]
    // with the rows in registers (16 threads x 4 columns per row; one
    // barrier per column, pivot row / column broadcast through double-
    // buffered shared memory) plus one dense product give C; a zero leading
    // minor (degenerate residual) falls back to the general elimination.
    bool fast_done = false, pairs_done = false;
    if (n == 32 && m > n && m <= 64) {
      // pivots = the n lowest-ranked rows; kernel rows in index order
      for (int i = tid; i < m; i += kStepThreads) piv[i] = rank[i] < n ? 1 : 0;
      for (int q = tid; q < n; q += kStepThreads) plist[q] = ord[q];
      if (tid < 32) {  // warp 0: klist by ballot / popc prefix over the m rows
        int base = 0;
        for (int i0 = 0; i0 < m; i0 += 32) {
          const int i = i0 + tid;
          const bool kr = i < m && rank[i] >= n;
          const unsigned bal = __ballot_sync(0xffffffffu, kr);
          if (kr) klist[base + __popc(bal & ((1u << tid) - 1u))] = i;
          base += __popc(bal);
        }
        if (tid == 0) s_nk = base;
      }
      __syncthreads();
      if (solve_pairs<32>(X, m, ord, klist, sbuf, f, W, a.rec_Ct + (size_t)k * m * m,
                          a.trace ? a.trace + k * 8 : nullptr,
                          pending >= 0 ? a.flags + pending : nullptr, a.epoch, sbar, spar)) {
        fast_done = pairs_done = true;
        pending = -1;
        spar ^= 1u;
      } else {
        // degenerate residual: the general elimination on W = R_k from X = I
        __syncthreads();
        if (tid == 0) {  // only the blocks before the zero minor completed a phase
          for (int b = 0; b < 16; ++b) tc::mbar_init(&sbar[b], 1);
          tc::fence_mbar_init();
        }
        spar = 0;
        for (int idx = tid; idx < (int)mn; idx += kStepThreads) W[idx] = gk(idx);
        for (int i = tid; i < m; i += kStepThreads) piv[i] = 0;
        for (int idx = tid; idx < m * m; idx += kStepThreads)
          X[idx] = (idx / m == idx - (idx / m) * m) ? 1u : 0u;
      }
      __syncthreads();
      STEP_TRACE(5);
    }
    const int n2 = 2 * n;
    uint32_t* A = X;                          // [n][2n] after the solve
    uint32_t* Cs = X + (size_t)n * n2;        // Ct [n][m-n+1] (padded rows)
    if (try_fast) {
      const int gi = tid >> 4, gs = tid & 15;  // row gi, columns gs + 16u
      uint32_t av4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = gs + 16 * u;
        av4[u] = (gi < n && j < n2)
                     ? (j < n ? W[(size_t)ord[gi] * n + j] : (j - n == gi ? 1u : 0u))
                     : 0u;
      }
      bool ok = true;
      for (int c = 0; c < n; ++c) {
        uint32_t* pb = sbuf + (c & 1) * 96;   // pivot row (64) + pivot column (32)
        if (gi == c) {
#pragma unroll
          for (int u = 0; u < 4; ++u) pb[gs + 16 * u] = av4[u];
        }
        if (gi < n && gs == (c & 15)) pb[64 + gi] = av4[c >> 4];
        __syncthreads();
        const uint32_t av = pb[c];
        if (av == 0) {
          ok = false;  // uniform: every thread read the same pivot
          break;
        }
        const uint32_t bv = gi < n ? pb[64 + gi] : 0u;
        if (gi < n && gi != c && bv != 0) {
#pragma unroll
          for (int u = 0; u < 4; ++u) av4[u] = redc_axby(av, av4[u], bv, pb[gs + 16 * u], f);
        }
      }
      STEP_TRACE(5);
      if (ok) {
        if (gi < n) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (gs + 16 * u < n2) A[gi * n2 + gs + 16 * u] = av4[u];
        }
        __syncthreads();
        // R_P^-1 = D^-1 Y: row l of Y scaled by 1 / d_l
        for (int l = tid; l < n; l += kStepThreads) inv[l] = invmod(A[l * n2 + l], f);
        // pivots = the n lowest-ranked rows; kernel rows in index order
        for (int i = tid; i < m; i += kStepThreads) piv[i] = rank[i] < n ? 1 : 0;
        for (int q = tid; q < n; q += kStepThreads) plist[q] = ord[q];
        if (tid < 32) {  // warp 0: klist by ballot / popc prefix over the m rows
          int base = 0;
          for (int i0 = 0; i0 < m; i0 += 32) {
            const int i = i0 + tid;
            const bool kr = i < m && rank[i] >= n;
            const unsigned bal = __ballot_sync(0xffffffffu, kr);
            if (kr) klist[base + __popc(bal & ((1u << tid) - 1u))] = i;
            base += __popc(bal);
          }
          if (tid == 0) s_nk = base;
        }
        __syncthreads();
        for (int idx = tid; idx < n * n; idx += kStepThreads) {
          const int l = idx / n, q = idx - (idx / n) * n;
          A[l * n2 + n + q] = mulmod(A[l * n2 + n + q], inv[l], f);
        }
        __syncthreads();
        STEP_TRACE(6);
        // Ct[q][kr] = -(R_K Y')[kr][q]; four independent partial sums (ILP)
        const int nk = s_nk;
        // lanes run over q: Y' reads are consecutive, the R_K row is a broadcast
        for (int idx = tid; idx < n * nk; idx += kStepThreads) {
          const int kr = idx / n, q = idx - (idx / n) * n;
          const uint32_t* rk = W + (size_t)klist[kr] * n;
          uint64_t acc[4] = {0, 0, 0, 0};
          int cnt = 0;
          for (int l = 0; l < n; l += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (l + u < n) acc[u] += (uint64_t)rk[l + u] * A[(l + u) * n2 + n + q];
            if (++cnt == a.fold_k) {
              cnt = 0;
#pragma unroll
              for (int u = 0; u < 4; ++u) acc[u] = fold(acc[u], f.c32);
            }
          }
          uint64_t tot = 0;
#pragma unroll
          for (int u = 0; u < 4; ++u) tot += d_red64(acc[u], p, f.mu);
          const uint32_t v = d_red64(tot, p, f.mu);
          Cs[q * (nk + 1) + kr] = v ? p - v : 0u;  // padded rows: conflict-free stores
        }
        fast_done = true;
      } else {
        // fallback: the general elimination starts from X = I
        for (int idx = tid; idx < m * m; idx += kStepThreads)
          X[idx] = (idx / m == idx - (idx / m) * m) ? 1u : 0u;
      }
      __syncthreads();
    }

    // ---- column elimination, lowest-rank pivot per column --------------------
    // Fast mode: while the pivots so far are exactly ranks 0..np-1, the pivot
    // of column c is the rank-np row if its entry is nonzero (it is then the
    // lowest-ranked candidate) -- no search.  Otherwise (rare: degenerate
    // residuals) switch to the general search for the rest of the step.
    int np = fast_done ? n : 0;
    bool fastm = true;
    for (int c = 0; c < (fast_done ? 0 : n); ++c) {
      int r = -1;
      if (fastm && np < m) {
        const int rr = ord[np];
        if (W[(size_t)rr * n + c] != 0) r = rr;
      }
      if (r < 0) {
        fastm = false;
        // general: lowest rank among non-pivot rows with a nonzero in column c
        const int slot = c & 1;
        for (int i = hw; i < m; i += kRowsPerPass)
          if (l16 == 0 && !piv[i] && W[(size_t)i * n + c] != 0) atomicMin(&s_key[slot], rank[i]);
        __syncthreads();
        const int key = s_key[slot];
        if (tid == 0) s_key[slot ^ 1] = INT_MAX;
        if (key == INT_MAX) {
          __syncthreads();
          continue;  // uniform: empty column
        }
        r = ord[key];
      }
      const uint32_t av = W[(size_t)r * n + c];
      for (int i = hw; i < m; i += kRowsPerPass) {
        if (piv[i] || i == r) continue;
        uint32_t* Wi = W + (size_t)i * n;
        const uint32_t bv = Wi[c];
        if (bv == 0) continue;
        const uint32_t* Wr = W + (size_t)r * n;
        uint32_t* Xi = X + (size_t)i * m;
        const uint32_t* Xr = X + (size_t)r * m;
#pragma unroll 4
        for (int j = c + 1 + l16; j < n; j += 16) Wi[j] = redc_axby(av, Wi[j], bv, Wr[j], f);
        // X: columns of earlier pivots, the new pivot r, and the diagonal
#pragma unroll 4
        for (int q = l16; q < np + 2; q += 16) {
          const int l = q < np ? plist[q] : (q == np ? r : i);
          Xi[l] = redc_axby(av, Xi[l], bv, Xr[l], f);
        }
      }
      if (tid == 0) {
        piv[r] = 1;
        plist[np] = r;
      }
      ++np;
      __syncthreads();
    }

    STEP_TRACE(1);
    // ---- record the step; normalise kernel rows: Ct = X_il / X_ii ------------
    if (tid == 0) {
      if (!fast_done) {
        int nk = 0;
        for (int i = 0; i < m; ++i)
          if (!piv[i]) klist[nk++] = i;
        s_nk = nk;
      }
      a.rec_np[k] = np;
    }
    for (int q = tid; q < np; q += kStepThreads) a.rec_plist[(size_t)k * m + q] = plist[q];
    __syncthreads();
    const int nk = s_nk;
    if (np == 0) {  // R = 0: nothing changes (appint.py:171)
      if (tid == 0) {
        if (pending >= 0) flag_release(a.flags + pending, a.epoch);
        flag_release(a.flags + k, a.epoch);
      }
      pending = -1;
      continue;
    }
    uint32_t* Ct = W;  // compact [np][nk]
    uint32_t* recC = a.rec_Ct + (size_t)k * m * m;
    if (pairs_done) {
      // solve_pairs wrote Ct (here, in W) and the record
    } else if (fast_done) {
      for (int idx = tid; idx < np * nk; idx += kStepThreads) {
        const int q = idx / nk, kr = idx - (idx / nk) * nk;
        const uint32_t v = Cs[q * (nk + 1) + kr];
        Ct[idx] = v;
        recC[idx] = v;
      }
    } else {
      for (int kr = tid; kr < nk; kr += kStepThreads) {
        const int i = klist[kr];
        inv[kr] = invmod(X[(size_t)i * m + i], f);
      }
      __syncthreads();
      for (int idx = tid; idx < np * nk; idx += kStepThreads) {
        const int q = idx / nk, kr = idx - (idx / nk) * nk;
        const uint32_t v = mulmod(X[(size_t)klist[kr] * m + plist[q]], inv[kr], f);
        Ct[idx] = v;
        recC[idx] = v;
      }
    }
    __syncthreads();
    STEP_TRACE(2);
    // step k's record is complete.  A GPU-scope release costs ~0.7 us on the
    // thread that issues it, so the flag of every step but the last is left
    // pending and released from an idle thread inside the next step's solve
    // (the build kernel only needs to keep up, not to be early)
    if (pending >= 0 && tid == 0) flag_release(a.flags + pending, a.epoch);
    pending = k;
    if (k == T - 1) {
      if (tid == 0) flag_release(a.flags + k, a.epoch);
      pending = -1;
    }

    // ---- residual list: kernel rows G[t][i] += sum_q Ct G[t][plist[q]], t > k -
    for (int q = tid; q < np; q += kStepThreads) prow[q] = rowoff[plist[q]];
    for (int kr = tid; kr < nk; kr += kStepThreads) krow[kr] = rowoff[klist[kr]];
    __syncthreads();
    if (pairs_done && m == 64 && nk == 32 && np == 32) {
      // X (the stride-(n+1) copy of R_k, 64 x 64 words) is free after the solve
      if (T - k - 1 > 0) residual_mma(G, Ct, X, krow, prow, k, T - k - 1, mn, f);
    } else if (((n | nk) & 3) == 0 && a.fold_k == 4) {
      const int nt = T - k - 1;
      if (nt <= 2)
        residual_tiles<1>(G, Ct, krow, prow, n, nk, np, k, nt, mn, f);
      else if (nt <= 4)
        residual_tiles<2>(G, Ct, krow, prow, n, nk, np, k, nt, mn, f);
      else
        residual_tiles<4>(G, Ct, krow, prow, n, nk, np, k, nt, mn, f);
    } else {
      const int rb_n = (nk + 3) >> 2, cb_n = (n + 3) >> 2, nt = T - k - 1;
      const int blocks = rb_n * cb_n * nt;
      const int K = a.fold_k;
      for (int b = tid; b < blocks; b += kStepThreads) {
        const int t = k + 1 + b / (rb_n * cb_n);
        const int rem = b - (b / (rb_n * cb_n)) * (rb_n * cb_n);
        const int rb = rem / cb_n, cb = rem - (rem / cb_n) * cb_n;
        uint32_t* Gt = G + (size_t)t * mn;
        int rows[4];
        uint64_t acc[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int kr = rb * 4 + r;
          rows[r] = kr < nk ? klist[kr] : -1;
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const int j = cb * 4 + cc;
            acc[r][cc] = (rows[r] >= 0 && j < n) ? Gt[krow[rb * 4 + r] + j] : 0;
          }
        }
        if (((n | nk) & 3) == 0 && K == 4) {
          // aligned fast path: 16-byte shared loads, folds at fixed positions
#pragma unroll 4
          for (int q = 0; q < np; ++q) {
            const uint4 g4 = *reinterpret_cast<const uint4*>(Gt + prow[q] + cb * 4);
            const uint4 c4 = *reinterpret_cast<const uint4*>(Ct + q * nk + rb * 4);
            const uint32_t gv[4] = {g4.x, g4.y, g4.z, g4.w}, cv[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
              for (int cc = 0; cc < 4; ++cc) acc[r][cc] += (uint64_t)cv[r] * gv[cc];
            if ((q & 3) == 3) {
#pragma unroll
              for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) acc[r][cc] = fold(acc[r][cc], f.c32);
            }
          }
        } else {
          int cnt = 0;
          for (int q = 0; q < np; ++q) {
            const uint32_t* gl = Gt + prow[q] + cb * 4;
            uint32_t gv[4], cv[4];
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) gv[cc] = (cb * 4 + cc < n) ? gl[cc] : 0u;
#pragma unroll
            for (int r = 0; r < 4; ++r) cv[r] = (rb * 4 + r < nk) ? Ct[q * nk + rb * 4 + r] : 0u;
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
              for (int cc = 0; cc < 4; ++cc) acc[r][cc] += (uint64_t)cv[r] * gv[cc];
            if (++cnt == K) {
              cnt = 0;
#pragma unroll
              for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) acc[r][cc] = fold(acc[r][cc], f.c32);
            }
          }
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (rows[r] < 0) continue;
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const int j = cb * 4 + cc;
            if (j < n) Gt[krow[rb * 4 + r] + j] = d_red64(acc[r][cc], p, f.mu);
          }
        }
      }
    }
    __syncthreads();
    STEP_TRACE(3);
    if (a.alpha) {
      // ---- interpolants: pivot rows times (x - alpha_k), so their residual
      // at point t (> k) is scaled by alpha_t - alpha_k (appint.py:79-117) ----
      const uint32_t ak = a.alpha[k];
      for (int idx = tid; idx < np * n * (T - k - 1); idx += kStepThreads) {
        const int t = k + 1 + idx / (np * n), r = idx - (idx / (np * n)) * (np * n);
        const int i = plist[r / n], j = r - (r / n) * n;
        const uint32_t d = a.alpha[t] >= ak ? a.alpha[t] - ak : a.alpha[t] + p - ak;
        uint32_t* g = G + (size_t)t * mn + rowoff[i] + j;
        *g = mulmod(*g, d, f);
      }
    } else {
      // ---- pivot rows: G_i <- x G_i (coefficient t takes t-1; k+1 takes R_k):
      // the row's offset grows, no data moves ----
      for (int q = tid; q < np; q += kStepThreads) {
        const int i = plist[q];
        off[i] += 1;
        rowoff[i] -= (long long)mn;
      }
    }
    for (int i = tid; i < m; i += kStepThreads) sft[i] += piv[i];
    __syncthreads();
    STEP_TRACE(4);
  }
  for (int i = tid; i < m; i += kStepThreads) a.sft_out[i] = sft[i];
  __syncthreads();
  if (tid == 0) flag_release(a.flags + T, a.epoch);
  if (a.trace && tid == 0) a.trace[63 * 8 + 1] = clock64();  // kernel end
}

struct BuildArgs {
  const int* rec_np;
  const int* rec_plist;
  const uint32_t* rec_Ct;
  int m, T;
  uint32_t* P;  // entry-major output, stride ps
  long long ps;
  int fold_k;
  F31 f;
  const uint32_t* alpha;  // interpolants: pivot rows times (x - alpha_k)
  const uint32_t* flags;  // step-done flags of the steps kernel (see StepArgs)
  uint32_t epoch;
};

// one CTA per column j of P: apply Q_0 .. Q_{T-1} to e_j.  Step k's record
// (pivot list, compact Ct) is staged into shared memory when its flag is set;
// the step then gathers the pivot rows' coefficients (and shifts them by x)
// and computes the kernel rows P1[t][klist[kr]] = P0[t][klist[kr]]
// + sum_q Ct[q][kr] P0[t][plist[q]] with independent shared loads.
__global__ void __launch_bounds__(256) mbasis_build_kernel(BuildArgs a) {
  // no pdl_wait: launched as the programmatic dependent of the steps kernel
  // (which triggers right after its own wait), this kernel runs BESIDE it and
  // applies step k as soon as flags[k] says its record is written; only the
  // last step's update is left when the steps kernel ends.  Records are read
  // with ld.global.cg: the buffers are reused leaf after leaf, and L1 may
  // hold an earlier leaf's lines.
  extern __shared__ __align__(16) uint32_t bsm[];
  const int m = a.m, T = a.T, j = blockIdx.x;
  const int tid = threadIdx.x, NT = blockDim.x;
  const int L1 = T + 1;
  const int cmax = (m / 2) * ((m + 1) / 2);  // np * nk <= m^2 / 4
  uint32_t* P0 = bsm;                                     // [L1][m]
  uint32_t* P1 = P0 + (size_t)L1 * m;                     // [L1][m]
  uint32_t* Pp = P1 + (size_t)L1 * m;                     // [L1][m] gathered pivot rows
  uint32_t* Cs = Pp + (size_t)L1 * m;                     // [cmax] compact Ct of the step
  short* pl = (short*)(Cs + cmax);                        // [m] pivot rows
  short* kl = pl + m;                                     // [m] kernel rows in index order
  short* isp = kl + m;                                    // [m] pivot flag
  for (int idx = tid; idx < L1 * m; idx += NT) P0[idx] = (idx == j) ? 1u : 0u;
  const bool k4 = a.fold_k >= 4;
  int L = 1;
  for (int k = 0; k < T; ++k) {
    if (tid == 0)
      while (flag_acquire(a.flags + k) != a.epoch) __nanosleep(64);
    __syncthreads();  // also: the previous step's reads of Cs / pl / kl are done
    const int np = __ldcg(a.rec_np + k);
    if (np == 0) continue;  // R = 0: the reference leaves P unchanged
    const int nk = m - np;
    for (int i = tid; i < m; i += NT) isp[i] = 0;
    for (int c = tid; c < np * nk; c += NT) Cs[c] = __ldcg(a.rec_Ct + (size_t)k * m * m + c);
    __syncthreads();
    for (int q = tid; q < np; q += NT) {
      const int i = __ldcg(a.rec_plist + (size_t)k * m + q);
      pl[q] = (short)i;
      isp[i] = 1;
    }
    __syncthreads();
    if (tid < 32) {  // kernel rows in index order: ballot prefix
      int base = 0;
      for (int i0 = 0; i0 < m; i0 += 32) {
        const int i = i0 + tid;
        const bool kr = i < m && !isp[i];
        const unsigned bal = __ballot_sync(0xffffffffu, kr);
        if (kr) kl[base + __popc(bal & ((1u << tid) - 1u))] = (short)i;
        base += __popc(bal);
      }
    }
    const uint32_t* Ct = Cs;
    // pivot rows: gather (t < L) and shift by x into P1 (t = 0 .. L)
    for (int idx = tid; idx < (L + 1) * np; idx += NT) {
      const int t = idx / np, q = idx - (idx / np) * np;
      const int i = pl[q];
      const uint32_t cur = t < L ? P0[(size_t)t * m + i] : 0u;
      if (t < L) Pp[t * m + q] = cur;
      uint32_t v = t >= 1 ? P0[(size_t)(t - 1) * m + i] : 0u;
      if (a.alpha) {  // x P - alpha_k P
        const uint32_t ac = mulmod(cur, a.alpha[k], a.f);
        v = v >= ac ? v - ac : v + a.f.p - ac;
      }
      P1[(size_t)t * m + i] = v;
    }
    __syncthreads();
    for (int idx = tid; idx < (L + 1) * nk; idx += NT) {
      const int t = idx / nk, kr = idx - (idx / nk) * nk;
      const int i = kl[kr];
      uint32_t v = 0;
      if (t < L) {
        const uint32_t* pp = Pp + t * m;
        uint64_t acc0 = P0[(size_t)t * m + i], acc1 = 0;
        int q = 0;
        if (k4) {
          for (; q + 4 <= np; q += 4) {
            acc0 += (uint64_t)Ct[(size_t)q * nk + kr] * pp[q];
            acc1 += (uint64_t)Ct[(size_t)(q + 1) * nk + kr] * pp[q + 1];
            acc0 += (uint64_t)Ct[(size_t)(q + 2) * nk + kr] * pp[q + 2];
            acc1 += (uint64_t)Ct[(size_t)(q + 3) * nk + kr] * pp[q + 3];
            acc0 = fold(acc0, a.f.c32);
            acc1 = fold(acc1, a.f.c32);
          }
        }
        for (; q < np; ++q) {
          acc0 += (uint64_t)Ct[(size_t)q * nk + kr] * pp[q];
          acc0 = fold(acc0, a.f.c32);
        }
        v = d_red(d_red64(acc0, a.f.p, a.f.mu) + d_red64(acc1, a.f.p, a.f.mu), a.f.p);
      }
      P1[(size_t)t * m + i] = v;
    }
    __syncthreads();
    uint32_t* tmp = P0; P0 = P1; P1 = tmp;
    ++L;
  }
  // every output of the steps kernel (the final shift) is written: this
  // kernel's completion then orders the whole leaf before its successors
  if (tid == 0)
    while (flag_acquire(a.flags + T) != a.epoch) __nanosleep(64);
  __syncthreads();
  // column j of P, entry-major: P[(i*m + j)*ps + t]
  const int ps = (int)a.ps;
  for (int idx = tid; idx < m * ps; idx += NT) {
    const int i = idx / ps, t = idx - (idx / ps) * ps;
    a.P[((long long)i * m + j) * ps + t] = t < L ? P0[(size_t)t * m + i] : 0u;
  }
}

unsigned long long* g_step_trace = nullptr;  // FPM_MBASIS_TRACE

F31 make_f31(uint32_t p) {
  F31 f;
  f.p = p;
  uint32_t inv = p;
  for (int i = 0; i < 5; ++i) inv *= 2 - p * inv;
  f.pinv = 0u - inv;
  f.mu = (uint64_t)((((u128)1) << 64) / p);
  f.c32 = (uint32_t)(((uint64_t)1 << 32) % p);
  f.r2 = (uint32_t)((((u128)1) << 64) % p);
  f.m58 = p >= (1u << 30) ? (uint32_t)((((uint64_t)1) << 58) / p) : 0u;
  f.w24s = p >= (1u << 30) ? (uint32_t)((((uint64_t)1) << 56) / p) : 0u;
  return f;
}

size_t steps_smem(int m, int n, int T) {
  return 8 * (size_t)m + 4 * ((size_t)T * m * n + (size_t)m * n + (size_t)m * m + m) +
         4 * 6 * (size_t)m + 8 + 8 * 3 * (size_t)m;
}

}  // namespace

int fold_period(uint32_t p);  // pointwise.cu

// mbasis_build_kernel: three P buffers, one step's compact record and row maps
size_t build_smem(int m, int order) {
  const size_t cmax = (size_t)(m / 2) * ((m + 1) / 2);
  return 3 * (size_t)(order + 1) * m * 4 + cmax * 4 + (size_t)m * 6 + 16;
}

int mbasis_fast_max_order(int m, int n) {
  // largest leaf order whose residual list fits in shared memory
  const size_t cap = 200 * 1024;
  if (2 * (size_t)2 * m * 4 > cap) return 0;
  int T = 0;
  while (T < 64 && steps_smem(m, n, T + 1) <= cap && build_smem(m, T + 1) <= cap) ++T;
  return T;
}

int mbasis_fast(Context& cx, uint32_t p, const void* F, int m, int n, long long fs, int lf,
                int order, const int64_t* s_dev, void* P, long long ps, int64_t* sft_dev,
                const uint32_t* alpha_dev, long long ts) {
  if (order < 1 || order > mbasis_fast_max_order(m, n)) {
    set_last_error("mbasis_fast: shape m=%d n=%d order=%d exceeds shared memory", m, n, order);
    return kUnsupported;
  }
  const size_t smem = steps_smem(m, n, order);
  Workspace ws(cx);
  int* rec_np;
  int* rec_plist;
  uint32_t* rec_Ct;
  FPM_TRY(ws.get((size_t)order, &rec_np));
  FPM_TRY(ws.get((size_t)order * m, &rec_plist));
  FPM_TRY(ws.get((size_t)order * m * m, &rec_Ct));
  const F31 f = make_f31(p);
  const int K = fold_period(p);
  StepArgs sa{};
  sa.F = (const uint32_t*)F; sa.fs = fs; sa.lf = lf < order ? lf : order;
  sa.ts = ts; sa.alpha = alpha_dev;
  sa.m = m; sa.n = n; sa.T = order; sa.s = s_dev;
  sa.rec_np = rec_np; sa.rec_plist = rec_plist; sa.rec_Ct = rec_Ct;
  sa.sft_out = sft_dev; sa.fold_k = K; sa.f = f;
  FPM_TRY(cx.leaf_flags(&sa.flags, &sa.epoch));
#ifdef FPM_TRACE
  // profiling build only (tools/mbasis_trace.py)
  if (std::getenv("FPM_MBASIS_TRACE")) {
    if (!g_step_trace) cudaMalloc(&g_step_trace, 64 * 8 * sizeof(unsigned long long));
    sa.trace = g_step_trace;
  }
#endif
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    FPM_CUDA_TRY(cudaFuncSetAttribute(mbasis_steps_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  {
    StageTimer t_(cx, "mbasis_steps");
    FPM_CUDA_TRY(launch_pdl(mbasis_steps_kernel, dim3(1), dim3(kStepThreads), smem, cx.stream(), sa));
    FPM_LAUNCH_CHECK();
  }
  BuildArgs ba{};
  ba.rec_np = rec_np; ba.rec_plist = rec_plist; ba.rec_Ct = rec_Ct; ba.m = m; ba.T = order;
  ba.alpha = alpha_dev;
  ba.P = (uint32_t*)P; ba.ps = ps; ba.fold_k = K; ba.f = f;
  ba.flags = sa.flags; ba.epoch = sa.epoch;
  const size_t bsmem = build_smem(m, order);
  static size_t battr = 0;
  if (bsmem > 48 * 1024 && bsmem > battr) {
    FPM_CUDA_TRY(cudaFuncSetAttribute(mbasis_build_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem));
    battr = bsmem;
  }
  {
    StageTimer t_(cx, "mbasis_build");
    FPM_CUDA_TRY(launch_pdl(mbasis_build_kernel, dim3(m), dim3(256), bsmem, cx.stream(), ba));
    FPM_LAUNCH_CHECK();
  }
  return kOk;
}

}  // namespace fpm

#ifdef FPM_TRACE
// profiling only: per-step phase clocks of the last leaf (FPM_MBASIS_TRACE)
extern "C" int fpm_debug_mbasis_trace(unsigned long long* host) {
  if (!fpm::g_step_trace) return 1;
  cudaDeviceSynchronize();
  cudaMemcpy(host, fpm::g_step_trace, 64 * 8 * sizeof(unsigned long long),
             cudaMemcpyDeviceToHost);
  return 0;
}
#endif
