// pointwise.cuh -- per-evaluation-point constant-matrix products mod p.
//
// Replaces `[_dense.mat_mul(a, b, p) for a, b in zip(va, vb)]`
// (polmat.py:300, :514; _dense.py:39-74): for every evaluation point t,
// C_t = A_t * B_t mod p with A_t (m x k), B_t (k x n).
//
// Operands are in the NTT eval layout E[t/32][entry][t%32] (ntt.cuh), so a
// warp owns one 32-point block: lane = point, and the warp walks an RT x CT
// tile of C for its 32 points.  Loads are 128-byte coalesced lines; products
// accumulate in 64-bit with one IMAD.WIDE per multiply-add and a fold
// acc = hi*(2^32 mod p) + lo every K products (K chosen per prime so the sum
// cannot overflow 2^64), then one Barrett reduction per output.
#pragma once
#include "common.cuh"

namespace fpm {

struct PointwiseArgs {
  const uint32_t* A;   // E_A[nblk][m*k][32]
  const uint32_t* B;   // E_B[nblk][k*n][32]
  uint32_t* C;         // E_C[nblk][m*n][32]
  int m, k, n;
  int nblk;            // N / 32
  long long a_prime_stride, b_prime_stride, c_prime_stride;
};

// fold period K (products between folds) that is overflow-safe for p
int fold_period(uint32_t p);
int launch_pointwise(const PointwiseArgs& a, const PrimeSet& ps, cudaStream_t st);

}  // namespace fpm
