// tc_pointwise.cuh -- int8 tensor-core (tcgen05) per-point products mod p.
#pragma once
#include "common.cuh"

namespace fpm {

// point-major operands: A_t = A + z*a_ps + t*m*k (row-major m x k), etc.
struct TcArgs {
  const uint32_t* A;
  const uint32_t* B;
  uint32_t* C;
  int m, k, n, npts;
  long long a_ps, b_ps, c_ps;  // per-prime strides (elements)
};

// Largest contraction the int8 kernels take: each limb-diagonal accumulator
// sums 4k byte products (< 255^2), all K chunks into one s32 TMEM column, so
// D_r < 4k*255^2 <= 2^31 needs k <= 8192.  Larger k runs on the CUDA cores.
constexpr int kTcMaxK = 8192;

bool tc_pointwise_applicable(int m, int k, int n, uint32_t p);
int launch_tc_pointwise(const TcArgs& a, const PrimeSet& ps, cudaStream_t st);

// small matrices (m <= 128): G = 128/mp points per UMMA tile, TMA-fed,
// warp-specialised (tc_grouped.cu)
bool tc_grouped_applicable(int m, int k, int n, uint32_t p);
int launch_tc_grouped(const TcArgs& a, const PrimeSet& ps, cudaStream_t st);

// 128 < m <= 256: both M tiles of a point share one built B tile (tc_pair.cu)
bool tc_pair_applicable(int m, int k, int n, uint32_t p);
int launch_tc_pair(const TcArgs& a, const PrimeSet& ps, cudaStream_t st);

// m <= 32 on the point-quad eval layout X[t/4][entry][t%4] (tc_pq.cu)
bool tc_pq_applicable(int m, int k, int n, int npts, uint32_t p);
int launch_tc_pq(const TcArgs& a, const PrimeSet& ps, cudaStream_t st);

}  // namespace fpm
