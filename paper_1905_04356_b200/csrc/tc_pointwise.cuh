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

bool tc_pointwise_applicable(int m, int k, int n, uint32_t p);
int launch_tc_pointwise(const TcArgs& a, const PrimeSet& ps, cudaStream_t st);

}  // namespace fpm
