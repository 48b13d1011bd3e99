// intbasis.cu -- interpolant bases on the GPU:
// appint.m_intbasis / pm_intbasis and appint.eval_polmat_points
// (ref appint.py:208-319).
//
// Same structure as the PM-Basis driver (pmbasis.cu): the basis is the
// product of the canonical order-1 steps (appint.py:24-60), now with pivot
// rows multiplied by (x - alpha_k) instead of x, so the output is independent
// of the leaf size and equals the reference's for any threshold.
//   * leaves: the shared-memory M-Basis kernels in interpolant mode
//     (mbasis_fast.cu: the residual list holds P(alpha_t) E_t and pivot rows
//     are rescaled by alpha_t - alpha_k instead of shifted);
//   * internal nodes: P1 is evaluated at the tail points (Horner, each thread
//     one entry at 8 points, `eval_points_kernel`), the residuals
//     R_t = P1(alpha_t) E_t are per-point products (`point_product_kernel`),
//     then P = P2 * P1 on the NTT product path;
//   * shifts stay on the device (s <- s + delta through the leaves), lengths
//     use deg P <= order: no host synchronisation inside the recursion.
// Points are arbitrary distinct field elements (the reference's geometric
// chirp evaluation is an optimisation of the same values).
#include <algorithm>
#include <vector>

#include "ops.cuh"
#include "pmbasis.cuh"
#include "runtime.cuh"
#include "tc_pointwise.cuh"

namespace fpm {
int mbasis_fast_max_order(int m, int n);
int mbasis_fast(Context& cx, uint32_t p, const void* F, int m, int n, long long fs, int lf,
                int order, const int64_t* s_dev, void* P, long long ps, int64_t* sft_dev,
                const uint32_t* alpha_dev, long long ts);
int fold_period(uint32_t p);  // pointwise.cu

namespace {

constexpr int kPts = 8;  // points per thread in the evaluation kernel

// EV[t][e] = sum_c P[e*ps + c] alpha_t^c for e < E (entries), t < npts
__global__ void __launch_bounds__(128) eval_points_kernel(const uint32_t* __restrict__ P,
                                                          long long ps, int L, long long E,
                                                          const uint32_t* __restrict__ alpha,
                                                          int npts, uint32_t p,
                                                          uint32_t* __restrict__ EV) {
  pdl_wait();
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int t0 = blockIdx.y * kPts;
  uint32_t w[kPts], wp[kPts], acc[kPts];
#pragma unroll
  for (int u = 0; u < kPts; ++u) {
    const int t = t0 + u;
    w[u] = t < npts ? alpha[t] : 0u;
    wp[u] = (uint32_t)(((uint64_t)w[u] << 32) / p);
    acc[u] = 0u;
  }
  if (e >= E) return;
  const uint32_t* pe = P + e * ps;
  for (int c = L - 1; c >= 0; --c) {
    const uint32_t v = __ldg(pe + c);
#pragma unroll
    for (int u = 0; u < kPts; ++u) acc[u] = d_red(d_red(d_shoup(acc[u], w[u], wp[u], p), p) + v, p);
  }
#pragma unroll
  for (int u = 0; u < kPts; ++u)
    if (t0 + u < npts) EV[(long long)(t0 + u) * E + e] = acc[u];
}

// R[t] = A[t] (m x k) * B[t] (k x n) mod p, point-major operands; one CTA per
// point, operands staged in shared memory, 64-bit accumulation with folds
__global__ void __launch_bounds__(256) point_product_kernel(const uint32_t* __restrict__ A,
                                                            const uint32_t* __restrict__ B,
                                                            uint32_t* __restrict__ R, int m,
                                                            int k, int n, uint32_t p,
                                                            uint32_t c32, uint64_t mu, int K) {
  pdl_wait();
  extern __shared__ uint32_t sh[];
  uint32_t* As = sh;
  uint32_t* Bs = sh + (size_t)m * k;
  const long long t = blockIdx.x;
  const uint32_t* At = A + t * m * k;
  const uint32_t* Bt = B + t * k * n;
  for (int i = threadIdx.x; i < m * k; i += blockDim.x) As[i] = At[i];
  for (int i = threadIdx.x; i < k * n; i += blockDim.x) Bs[i] = Bt[i];
  __syncthreads();
  for (int o = threadIdx.x; o < m * n; o += blockDim.x) {
    const int i = o / n, j = o - (o / n) * n;
    uint64_t acc = 0;
    int cnt = 0;
    for (int l = 0; l < k; ++l) {
      acc += (uint64_t)As[i * k + l] * Bs[l * n + j];
      if (++cnt == K) {
        cnt = 0;
        acc = (uint64_t)(uint32_t)(acc >> 32) * c32 + (uint32_t)acc;
      }
    }
    R[t * m * n + o] = d_red64(acc, p, mu);
  }
}

int eval_points(Context& cx, uint32_t p, const uint32_t* P, long long ps, int L, long long E,
                const uint32_t* alpha, int npts, uint32_t* EV) {
  if (E <= 0 || npts <= 0) return kOk;
  if (L <= 0) {
    FPM_CUDA_TRY(cudaMemsetAsync(EV, 0, sizeof(uint32_t) * (size_t)E * npts, cx.stream()));
    return kOk;
  }
  dim3 grid((unsigned)((E + 127) / 128), (unsigned)((npts + kPts - 1) / kPts));
  FPM_CUDA_TRY(launch_pdl(eval_points_kernel, grid, dim3(128), 0, cx.stream(), P, ps, L, E,
                          alpha, npts, p, EV));
  FPM_LAUNCH_CHECK();
  return kOk;
}

int point_product(Context& cx, uint32_t p, const uint32_t* A, const uint32_t* B, uint32_t* R,
                  int m, int k, int n, int npts) {
  if (npts <= 0 || m <= 0 || n <= 0) return kOk;
  // larger residual products on the int8 tensor cores: the operands are
  // already point-major, the layout tc_grouped_kernel reads (as ops.cu, m > 32)
  if (m > 32 && tc_grouped_applicable(m, k, n, p)) {
    PrimeSet ps;
    ps.count = 1;
    FPM_TRY(cx.prime_const(p, 5, &ps.pr[0]));
    TcArgs ta{};
    ta.A = A; ta.B = B; ta.C = R; ta.m = m; ta.k = k; ta.n = n; ta.npts = npts;
    ta.a_ps = (long long)npts * m * k; ta.b_ps = (long long)npts * k * n;
    ta.c_ps = (long long)npts * m * n;
    return launch_tc_grouped(ta, ps, cx.stream());
  }
  const size_t smem = sizeof(uint32_t) * ((size_t)m * k + (size_t)k * n);
  if (smem > 200 * 1024) {
    set_last_error("interpolant residual: %d x %d x %d per point exceeds shared memory", m, k, n);
    return kUnsupported;
  }
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    FPM_CUDA_TRY(cudaFuncSetAttribute(point_product_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  const uint32_t c32 = (uint32_t)(((uint64_t)1 << 32) % p);
  const uint64_t mu = (uint64_t)((((u128)1) << 64) / p);
  FPM_CUDA_TRY(launch_pdl(point_product_kernel, dim3((unsigned)npts), dim3(256), smem,
                          cx.stream(), A, B, R, m, k, n, p, c32, mu, fold_period(p)));
  FPM_LAUNCH_CHECK();
  return kOk;
}

// E: [order][m][n] point-major, alpha: [order] device
int intbasis_rec_dev(Context& cx, uint32_t p, const uint32_t* E, const uint32_t* alpha, int m,
                     int n, int order, const int64_t* s_dev, int T, uint32_t* P, long long ps,
                     int64_t* sft_dev) {
  if (order <= T)
    return mbasis_fast(cx, p, E, m, n, 1, order, order, s_dev, P, ps, sft_dev, alpha,
                       (long long)m * n);
  const int o1 = (order + 1) / 2, o2 = order - o1;
  Workspace ws(cx);
  uint32_t *P1, *EV, *R, *P2;
  int64_t* s1;
  FPM_TRY(ws.get((size_t)m * m * (o1 + 1), &P1));
  FPM_TRY(ws.get((size_t)m, &s1));
  FPM_TRY(intbasis_rec_dev(cx, p, E, alpha, m, n, o1, s_dev, T, P1, o1 + 1, s1));
  // residuals of the tail points: R_t = P1(alpha_t) E_t (appint.py:300-312)
  FPM_TRY(ws.get((size_t)o2 * m * m, &EV));
  FPM_TRY(ws.get((size_t)o2 * m * n, &R));
  FPM_TRY(eval_points(cx, p, P1, o1 + 1, o1 + 1, (long long)m * m, alpha + o1, o2, EV));
  FPM_TRY(point_product(cx, p, EV, E + (size_t)o1 * m * n, R, m, m, n, o2));
  FPM_TRY(ws.get((size_t)m * m * (o2 + 1), &P2));
  FPM_TRY(intbasis_rec_dev(cx, p, R, alpha + o1, m, n, o2, s1, T, P2, o2 + 1, sft_dev));
  MatRef A2{P2, 0, o2 + 1, o2 + 1};
  MatRef B2{P1, 0, o1 + 1, o1 + 1};
  OutRef Co{P, 0, ps, (int)ps};
  return polmat_mul(cx, p, m, m, m, A2, B2, Co);
}

}  // namespace

int intbasis_run(Context& cx, uint64_t p, const void* E, int m, int n, int order,
                 const uint64_t* alpha_host, const int64_t* shift, int T, void* P, long long ps,
                 int* lp, int64_t* rdeg_out) {
  if (p >= (1ull << 31)) {
    set_last_error("interpolant bases run on the 31-bit prime path (p = %llu)",
                   (unsigned long long)p);
    return kUnsupported;
  }
  // appint._check_points: pairwise distinct points (as field elements)
  std::vector<uint32_t> pts(order);
  for (int t = 0; t < order; ++t) pts[t] = (uint32_t)(alpha_host[t] % p);
  {
    std::vector<uint32_t> srt(pts);
    std::sort(srt.begin(), srt.end());
    if (std::adjacent_find(srt.begin(), srt.end()) != srt.end()) {
      set_last_error("interpolation points must be pairwise distinct");
      return kDuplicatePoints;
    }
  }
  if (T < 1) T = 1;
  const int tf = mbasis_fast_max_order(m, n);
  if (tf < 1) {
    set_last_error("interpolant basis: m=%d n=%d exceeds the shared-memory leaf", m, n);
    return kUnsupported;
  }
  if (T > tf) T = tf;
  if (T > 8) T = 8;  // as pmbasis_run: leaf order 8 balances leaf and tree
  Workspace ws(cx);
  int64_t *s_dev, *sft_dev;
  uint32_t* a_dev;
  FPM_TRY(ws.get((size_t)m, &s_dev));
  FPM_TRY(ws.get((size_t)m, &sft_dev));
  FPM_TRY(ws.get((size_t)(order > 0 ? order : 1), &a_dev));
  FPM_CUDA_TRY(cudaMemcpyAsync(s_dev, shift, sizeof(int64_t) * m, cudaMemcpyHostToDevice,
                               cx.stream()));
  if (order > 0)
    FPM_CUDA_TRY(cudaMemcpyAsync(a_dev, pts.data(), sizeof(uint32_t) * order,
                                 cudaMemcpyHostToDevice, cx.stream()));
  if (order == 0) {
    // identity basis, shift unchanged (m_intbasis with no points)
    FPM_CUDA_TRY(cudaMemsetAsync(P, 0, sizeof(uint32_t) * (size_t)m * m * ps, cx.stream()));
    std::vector<uint32_t> one(1, 1u);
    for (int i = 0; i < m; ++i)
      FPM_CUDA_TRY(cudaMemcpyAsync((uint32_t*)P + ((size_t)i * m + i) * ps, one.data(), 4,
                                   cudaMemcpyHostToDevice, cx.stream()));
    FPM_CUDA_TRY(cudaStreamSynchronize(cx.stream()));
    *lp = 1;
    if (rdeg_out) std::copy(shift, shift + m, rdeg_out);
    return kOk;
  }
  FPM_TRY(intbasis_rec_dev(cx, (uint32_t)p, (const uint32_t*)E, a_dev, m, n, order, s_dev, T,
                           (uint32_t*)P, ps, sft_dev));
  int deg = -1;
  FPM_TRY(matrix_degree(cx, P, 0, (long long)m * m, (int)ps, &deg));  // synchronizes
  *lp = deg + 1;
  if (rdeg_out)
    FPM_CUDA_TRY(cudaMemcpy(rdeg_out, sft_dev, sizeof(int64_t) * m, cudaMemcpyDeviceToHost));
  return kOk;
}

int eval_points_run(Context& cx, uint64_t p, const void* P, int m, int n, int L,
                    const uint64_t* pts_host, int npts, void* out) {
  if (p >= (1ull << 31)) {
    set_last_error("point evaluation runs on the 31-bit prime path (p = %llu)",
                   (unsigned long long)p);
    return kUnsupported;
  }
  if (npts <= 0 || (long long)m * n == 0) return kOk;
  std::vector<uint32_t> pts(npts);
  for (int t = 0; t < npts; ++t) pts[t] = (uint32_t)(pts_host[t] % p);
  Workspace ws(cx);
  uint32_t* a_dev;
  FPM_TRY(ws.get((size_t)npts, &a_dev));
  FPM_CUDA_TRY(cudaMemcpyAsync(a_dev, pts.data(), sizeof(uint32_t) * npts,
                               cudaMemcpyHostToDevice, cx.stream()));
  return eval_points(cx, (uint32_t)p, (const uint32_t*)P, L, L, (long long)m * n, a_dev, npts,
                     (uint32_t*)out);
}

}  // namespace fpm
