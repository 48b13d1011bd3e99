// Legacy mma.sync m16n8k32 u8 on sm_100a: cycles per warp-mma per SMSP with
// CH independent accumulator chains per warp (throughput) and with one chain
// (latency), 16 warps per SM, 148 CTAs.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void mma(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                    uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};\n"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
template <int CH>
__global__ void k(int* out, long long* cyc, uint32_t s, int iters) {
  int d[CH][4];
  for (int c = 0; c < CH; ++c)
    for (int e = 0; e < 4; ++e) d[c][e] = 0;
  const uint32_t a = s * threadIdx.x, b = s + threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) mma(d[c], a, a + 1, a + 2, a + 3, b, b + c);
  }
  __syncthreads();
  long long t1 = clock64();
  int r = 0;
  for (int c = 0; c < CH; ++c)
    for (int e = 0; e < 4; ++e) r += d[c][e];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[CH] = t1 - t0;
}
int main() {
  int* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 24);
  cudaMallocManaged(&cyc, 64 * 8);
  const int iters = 1000;
  for (int w : {1, 4, 16}) {
    k<1><<<148, 32 * w>>>(out, cyc, 3, iters);
    k<8><<<148, 32 * w>>>(out, cyc, 3, iters);
    cudaDeviceSynchronize();
    const double warps_per_smsp = w / 4.0 < 1 ? 1 : w / 4.0;
    printf("warps/SM %2d: 1 chain %.1f cycles per mma (latency per warp); 8 chains %.2f cycles "
           "per warp-mma per SMSP\n",
           w, (double)cyc[1] / iters, (double)cyc[8] / (iters * 8.0) / warps_per_smsp);
  }
  return 0;
}
