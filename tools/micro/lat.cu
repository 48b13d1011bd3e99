// Latency micro-benchmarks (clock64 in one CTA): dependent chains of the
// integer ops the M-Basis leaf uses, and __syncthreads at 512 threads.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t redc_mul(uint32_t a, uint32_t b, uint32_t p, uint32_t pinv) {
  const uint64_t acc = (uint64_t)a * b;
  const uint32_t m = (uint32_t)acc * pinv;
  const uint32_t t = (uint32_t)((acc + (uint64_t)m * p) >> 32);
  return min(t, t - p);
}
__device__ __forceinline__ uint32_t shoup(uint32_t a, uint32_t w, uint32_t wp, uint32_t p) {
  uint32_t q = __umulhi(a, wp);
  uint32_t r = a * w - q * p;
  return min(r, r - p);
}
__global__ void k(uint32_t* out, long long* cyc, uint32_t x0, uint32_t p, uint32_t pinv, int iters) {
  __shared__ uint32_t sh[1024];
  uint32_t x = x0 + threadIdx.x;
  sh[threadIdx.x] = x;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = redc_mul(x, x, p, pinv);
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) x = shoup(x, 12345u, 67890u, p);
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) { x = (uint32_t)(((uint64_t)x * x) >> 17); }
  long long t3 = clock64();
  for (int i = 0; i < iters; ++i) { __syncthreads(); x += 1; }
  long long t4 = clock64();
  for (int i = 0; i < iters; ++i) { x = sh[(x + i) & 1023]; }
  long long t5 = clock64();
  for (int i = 0; i < iters; ++i) { x = __umulhi(x, x) + 1; }
  long long t6 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
  }
}
int main() {
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, 1 << 20); cudaMallocManaged(&cyc, 64);
  const uint32_t p = 2013265921u;
  uint32_t inv = p; for (int i = 0; i < 5; ++i) inv *= 2 - p * inv;
  const int iters = 1000;
  for (int nt : {32, 512}) {
    k<<<1, nt>>>(out, cyc, 7, p, 0u - inv, iters);
    cudaDeviceSynchronize();
    printf("threads %d per-op cycles: redc_mul %.1f shoup %.1f mul64>>17 %.1f syncthreads %.1f lds-chain %.1f umulhi+1 %.1f\n", nt,
           cyc[0] / (double)iters, cyc[1] / (double)iters, cyc[2] / (double)iters, cyc[3] / (double)iters,
           cyc[4] / (double)iters, cyc[5] / (double)iters);
  }
  return 0;
}
