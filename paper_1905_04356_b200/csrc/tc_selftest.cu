// tc_selftest.cu -- single-CTA tcgen05 kind::i8 GEMM used to validate the
// descriptor / TMEM plumbing of tc_common.cuh against torch on the device.
// D (M x N, s32) = A (M x K, u8, row-major) * B^T (B: N x K, u8, row-major)
#include "common.cuh"
#include "tc_common.cuh"
#include "../../include/fpmat_b200.h"

namespace fpm {
namespace {

__global__ void __launch_bounds__(128, 1)
    tc_gemm_test_kernel(const uint8_t* A, const uint8_t* B, int32_t* D, int M, int N, int K) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sA = sm;                       // M x K  (128 x K)
  uint8_t* sB = sm + (size_t)M * K;       // N x K
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int idx = tid; idx < M * K; idx += blockDim.x) {
    const int r = idx / K, k = idx - r * K;
    sA[tc::kmajor_off(r, k, K)] = A[idx];
  }
  for (int idx = tid; idx < N * K; idx += blockDim.x) {
    const int r = idx / K, k = idx - r * K;
    sB[tc::kmajor_off(r, k, K)] = B[idx];
  }
  tc::fence_proxy_async();
  if (warp == 0) tc::tmem_alloc(&tmem_base, 256);
  if (tid == 0) tc::mbar_init(&mbar, 1);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tb = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = tc::idesc_u8(M, N);
    for (int ks = 0; ks < K / 32; ++ks) {
      const uint64_t ad = tc::make_desc(tc::smem_u32(sA) + ks * 256, 128, K * 8);
      const uint64_t bd = tc::make_desc(tc::smem_u32(sB) + ks * 256, 128, K * 8);
      tc::mma_u8(tb, ad, bd, idesc, ks > 0 ? 1u : 0u);
    }
    tc::commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after_sync();
  // epilogue: warp w reads lanes 32w..32w+31 (rows), 32 columns at a time
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t v[32];
    tc::tmem_ld32(tb + ((uint32_t)(32 * warp) << 16) + c0, v);
    const int row = 32 * warp + lane;
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (c0 + j < N) D[(size_t)row * N + c0 + j] = (int32_t)v[j];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tb, 256);
}

}  // namespace
}  // namespace fpm

extern "C" int fpm_selftest_tc_gemm(const void* A, const void* B, void* D, int M, int N, int K) {
  using namespace fpm;
  if (M != 128 || N < 16 || N > 256 || N % 16 || K < 32 || K > 256 || K % 32) {
    set_last_error("selftest shape: M=128, N in [16,256] step 16, K in [32,256] step 32");
    return kInvalidArgument;
  }
  const size_t smem = (size_t)(M + N) * K;
  FPM_CUDA_TRY(cudaFuncSetAttribute(tc_gemm_test_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  tc_gemm_test_kernel<<<1, 128, smem>>>((const uint8_t*)A, (const uint8_t*)B, (int32_t*)D, M, N,
                                        K);
  FPM_LAUNCH_CHECK();
  FPM_CUDA_TRY(cudaDeviceSynchronize());
  return kOk;
}

#include "runtime.cuh"
#include "tc_pointwise.cuh"

// point-major tensor-core product for tests: C_t = A_t B_t mod p, t < npts
extern "C" int fpm_selftest_tc_pointwise(fpm_context* ctx, uint32_t p, const void* A,
                                         const void* B, void* C, int m, int k, int n,
                                         int npts);

struct fpm_context {
  fpm::Context* cx;
  int pmbasis_T;
};

extern "C" int fpm_selftest_tc_pointwise(fpm_context* ctx, uint32_t p, const void* A,
                                         const void* B, void* C, int m, int k, int n,
                                         int npts) {
  using namespace fpm;
  if (!ctx || !tc_pointwise_applicable(m, k, n, p)) {
    set_last_error("tc_pointwise not applicable to m=%d k=%d n=%d", m, k, n);
    return kInvalidArgument;
  }
  PrimeSet ps;
  ps.count = 1;
  FPM_TRY(ctx->cx->prime_const(p, 5, &ps.pr[0]));
  TcArgs a{};
  a.A = (const uint32_t*)A; a.B = (const uint32_t*)B; a.C = (uint32_t*)C;
  a.m = m; a.k = k; a.n = n; a.npts = npts;
  FPM_TRY(launch_tc_pointwise(a, ps, ctx->cx->stream()));
  FPM_CUDA_TRY(cudaStreamSynchronize(ctx->cx->stream()));
  return kOk;
}

// grouped small-matrix kernel for tests: for prime z < nprimes and t < npts,
// C[z][t] = A[z][t] B[z][t] mod primes[z] (point-major, primes stacked)
extern "C" int fpm_selftest_tc_grouped(fpm_context* ctx, const uint32_t* primes, int nprimes,
                                       const void* A, const void* B, void* C, int m, int k,
                                       int n, int npts) {
  using namespace fpm;
  if (!ctx || nprimes < 1 || nprimes > 8) {
    set_last_error("tc_grouped selftest: bad arguments");
    return kInvalidArgument;
  }
  PrimeSet ps;
  ps.count = nprimes;
  for (int i = 0; i < nprimes; ++i) {
    if (!tc_grouped_applicable(m, k, n, primes[i])) {
      set_last_error("tc_grouped not applicable to m=%d k=%d n=%d", m, k, n);
      return kInvalidArgument;
    }
    FPM_TRY(ctx->cx->prime_const(primes[i], 5, &ps.pr[i]));
  }
  TcArgs a{};
  a.A = (const uint32_t*)A; a.B = (const uint32_t*)B; a.C = (uint32_t*)C;
  a.m = m; a.k = k; a.n = n; a.npts = npts;
  a.a_ps = (long long)npts * m * k; a.b_ps = (long long)npts * k * n;
  a.c_ps = (long long)npts * m * n;
  FPM_TRY(launch_tc_grouped(a, ps, ctx->cx->stream()));
  FPM_CUDA_TRY(cudaStreamSynchronize(ctx->cx->stream()));
  return kOk;
}

// point-quad kernel for tests: operands in the eval layout X[z][t/4][entry][t%4]
extern "C" int fpm_selftest_tc_pq(fpm_context* ctx, const uint32_t* primes, int nprimes,
                                  const void* A, const void* B, void* C, int m, int k, int n,
                                  int npts) {
  using namespace fpm;
  if (!ctx || nprimes < 1 || nprimes > 8) {
    set_last_error("tc_pq selftest: bad arguments");
    return kInvalidArgument;
  }
  PrimeSet ps;
  ps.count = nprimes;
  for (int i = 0; i < nprimes; ++i) FPM_TRY(ctx->cx->prime_const(primes[i], 5, &ps.pr[i]));
  TcArgs a{};
  a.A = (const uint32_t*)A; a.B = (const uint32_t*)B; a.C = (uint32_t*)C;
  a.m = m; a.k = k; a.n = n; a.npts = npts;
  a.a_ps = (long long)npts * m * k; a.b_ps = (long long)npts * k * n;
  a.c_ps = (long long)npts * m * n;
  FPM_TRY(launch_tc_pq(a, ps, ctx->cx->stream()));
  FPM_CUDA_TRY(cudaStreamSynchronize(ctx->cx->stream()));
  return kOk;
}
