// pointwise.cu -- CUDA-core mod-p matrix products per evaluation point.
#include "pointwise.cuh"

namespace fpm {
namespace {

constexpr int kWarps = 8;

template <int RT, int CT, int K>
__global__ void __launch_bounds__(kWarps * 32)
    pointwise_cc_kernel(PointwiseArgs a, PrimeSet ps) {
  const PrimeConst& pc = ps.pr[blockIdx.z];
  const uint32_t p = pc.p, c32 = pc.c32;
  const uint64_t mu = pc.mu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int m = a.m, k = a.k, n = a.n;
  const long long tb = blockIdx.x;
  const uint32_t* Ab = a.A + blockIdx.z * a.a_prime_stride + tb * (long long)(m * k) * 32 + lane;
  const uint32_t* Bb = a.B + blockIdx.z * a.b_prime_stride + tb * (long long)(k * n) * 32 + lane;
  uint32_t* Cb = a.C + blockIdx.z * a.c_prime_stride + tb * (long long)(m * n) * 32 + lane;
  const int ntn = (n + CT - 1) / CT;
  const int ntiles = ((m + RT - 1) / RT) * ntn;
  for (int tile = blockIdx.y * kWarps + warp; tile < ntiles; tile += gridDim.y * kWarps) {
    const int i0 = (tile / ntn) * RT, j0 = (tile % ntn) * CT;
    const uint32_t* ap[RT];
    const uint32_t* bp[CT];
#pragma unroll
    for (int r = 0; r < RT; ++r) ap[r] = Ab + (long long)(min(i0 + r, m - 1) * k) * 32;
#pragma unroll
    for (int c = 0; c < CT; ++c) bp[c] = Bb + (long long)min(j0 + c, n - 1) * 32;
    uint64_t acc[RT][CT];
#pragma unroll
    for (int r = 0; r < RT; ++r)
#pragma unroll
      for (int c = 0; c < CT; ++c) acc[r][c] = 0;
    int l = 0;
    for (; l + K <= k; l += K) {
#pragma unroll
      for (int u = 0; u < K; ++u) {
        uint32_t av[RT], bv[CT];
#pragma unroll
        for (int r = 0; r < RT; ++r) av[r] = __ldg(ap[r] + (long long)(l + u) * 32);
#pragma unroll
        for (int c = 0; c < CT; ++c) bv[c] = __ldg(bp[c] + (long long)(l + u) * n * 32);
#pragma unroll
        for (int r = 0; r < RT; ++r)
#pragma unroll
          for (int c = 0; c < CT; ++c) acc[r][c] += (uint64_t)av[r] * bv[c];
      }
#pragma unroll
      for (int r = 0; r < RT; ++r)
#pragma unroll
        for (int c = 0; c < CT; ++c)
          acc[r][c] = (uint64_t)(uint32_t)(acc[r][c] >> 32) * c32 + (uint32_t)acc[r][c];
    }
    for (; l < k; ++l) {
      uint32_t av[RT], bv[CT];
#pragma unroll
      for (int r = 0; r < RT; ++r) av[r] = __ldg(ap[r] + (long long)l * 32);
#pragma unroll
      for (int c = 0; c < CT; ++c) bv[c] = __ldg(bp[c] + (long long)l * n * 32);
#pragma unroll
      for (int r = 0; r < RT; ++r)
#pragma unroll
        for (int c = 0; c < CT; ++c) {
          acc[r][c] += (uint64_t)av[r] * bv[c];
          acc[r][c] = (uint64_t)(uint32_t)(acc[r][c] >> 32) * c32 + (uint32_t)acc[r][c];
        }
    }
#pragma unroll
    for (int r = 0; r < RT; ++r) {
      if (i0 + r >= m) break;
#pragma unroll
      for (int c = 0; c < CT; ++c) {
        if (j0 + c >= n) break;
        Cb[(long long)((i0 + r) * n + j0 + c) * 32] = d_red64(acc[r][c], p, mu);
      }
    }
  }
}

template <int K>
int launch_k(const PointwiseArgs& a, const PrimeSet& ps, cudaStream_t st) {
  constexpr int RT = 4, CT = 4;
  const int ntiles = ((a.m + RT - 1) / RT) * ((a.n + CT - 1) / CT);
  const int per_cta = (ntiles + kWarps - 1) / kWarps;
  // enough CTAs to cover ~4 waves of 148 SMs when the point count is small
  long long want = 4LL * 148 / ((long long)a.nblk * ps.count) + 1;
  int gy = (int)(want < per_cta ? want : per_cta);
  if (gy < 1) gy = 1;
  dim3 grid((unsigned)a.nblk, (unsigned)gy, (unsigned)ps.count);
  pointwise_cc_kernel<RT, CT, K><<<grid, kWarps * 32, 0, st>>>(a, ps);
  FPM_LAUNCH_CHECK();
  return kOk;
}

}  // namespace

int fold_period(uint32_t p) {
  const u128 two64 = (u128)1 << 64;
  const u128 c32 = ((u128)1 << 32) % p;
  const u128 fold_max = (((u128)1 << 32) - 1) * c32 + (((u128)1 << 32) - 1);
  const u128 sq = (u128)(p - 1) * (p - 1);
  int K = 1;
  while (K < 4 && fold_max + (u128)(K + 1) * sq < two64) ++K;
  return K;
}

int launch_pointwise(const PointwiseArgs& a, const PrimeSet& ps, cudaStream_t st) {
  if (a.nblk <= 0 || a.m <= 0 || a.n <= 0) return kOk;
  int K = 4;
  for (int i = 0; i < ps.count; ++i) {
    int k = fold_period(ps.pr[i].p);
    if (k < K) K = k;
  }
  switch (K) {
    case 4: return launch_k<4>(a, ps, st);
    case 3: return launch_k<3>(a, ps, st);
    case 2: return launch_k<2>(a, ps, st);
    default: return launch_k<1>(a, ps, st);
  }
}

}  // namespace fpm
