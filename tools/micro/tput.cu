// Issue throughput of integer ops (inline PTX, 8 independent chains per
// thread, 16 warps per SM, 148 CTAs): cycles per warp-instruction per SMSP.
#include <cstdio>
#include <cstdint>
template <int MODE>
__global__ void k(uint32_t* out, long long* cyc, uint32_t s, int iters) {
  uint32_t b[8], c[8];
  for (int j = 0; j < 8; ++j) { b[j] = s + threadIdx.x * 8 + j; c[j] = b[j] * 7u + 1u; }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0) asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(b[j]) : "r"(c[j]));
      if (MODE == 1) asm volatile("mad.hi.u32 %0, %0, %1, %0;" : "+r"(b[j]) : "r"(c[j]));
      if (MODE == 2) {
        uint64_t w;
        asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(w) : "r"(b[j]), "r"(c[j]), "l"((uint64_t)c[j]));
        b[j] = (uint32_t)(w >> 32) ^ (uint32_t)w;
      }
      if (MODE == 3) asm volatile("{.reg .u32 t; add.u32 t, %0, %1; min.u32 %0, t, %0;}" : "+r"(b[j]) : "r"(c[j]));
      if (MODE == 4) asm volatile("add.u32 %0, %0, %1;" : "+r"(b[j]) : "r"(c[j]));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t r = 0;
  for (int j = 0; j < 8; ++j) r += b[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[MODE] = t1 - t0;
}
int main() {
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, 1 << 24); cudaMallocManaged(&cyc, 64);
  const int iters = 2000, threads = 512;
  k<0><<<148, threads>>>(out, cyc, 3, iters);
  k<1><<<148, threads>>>(out, cyc, 3, iters);
  k<2><<<148, threads>>>(out, cyc, 3, iters);
  k<3><<<148, threads>>>(out, cyc, 3, iters);
  k<4><<<148, threads>>>(out, cyc, 3, iters);
  cudaDeviceSynchronize();
  const double winstr = (double)iters * 8 * (threads / 32) / 4;  // warp-ops per SMSP
  printf("cycles per warp-op per SMSP: mad.lo %.2f  mad.hi %.2f  mad.wide(+xor,shift) %.2f  add+min %.2f  add %.2f\n",
         cyc[0] / winstr, cyc[1] / winstr, cyc[2] / winstr, cyc[3] / winstr, cyc[4] / winstr);
  return 0;
}
