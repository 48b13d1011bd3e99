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
//   * internal nodes: P1 is evaluated at the tail points -- by a chirp
//     middle product on the NTT path when the points form a geometric
//     progression (as the reference does), else by Horner (each thread one
//     entry at 8 points, `eval_points_kernel`) -- the residuals
//     R_t = P1(alpha_t) E_t are per-point products (int8 tensor cores via
//     tc_grouped_kernel, or `point_product_kernel`), then P = P2 * P1 on the
//     NTT product path;
//   * shifts stay on the device (s <- s + delta through the leaves), lengths
//     use deg P <= order: no host synchronisation inside the recursion.
// Points are arbitrary distinct field elements.
#include <algorithm>
#include <cstdlib>
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

// ---- geometric points: chirp (Bluestein) evaluation on the NTT path -------
// With alpha_t = a0 r^t and C(u) = u(u-1)/2, r^(i j) = r^C(i+j) r^-C(i) r^-C(j),
// so f(a0 r^j) = r^-C(j) sum_i (c_i a0^i r^-C(i)) r^C(i+j): one middle
// product of the scaled coefficients with the chirp r^C(u) per entry
// (ref upoly._eval_geometric_raw, upoly.py:455-472, used by
// appint.eval_polmat_points for geometric points, appint.py:268-282).
struct GeoPts {
  bool on;
  uint32_t r, rinv;
};

__device__ __forceinline__ uint32_t powmod_dev(uint32_t a, uint64_t e, uint32_t p, uint64_t mu) {
  uint32_t r = 1u;
  while (e) {
    if (e & 1) r = d_red64((uint64_t)r * a, p, mu);
    a = d_red64((uint64_t)a * a, p, mu);
    e >>= 1;
  }
  return r;
}

// w[j] = a0^j r^-C(j) (j < la), tri[u] = r^C(u) (u < la + npts - 1),
// tinv[j] = r^-C(j) (j < npts); a0 read on the device (no host round trip)
__global__ void chirp_tables_kernel(const uint32_t* __restrict__ a0p, uint32_t r, uint32_t rinv,
                                    int la, int npts, uint32_t p, uint64_t mu,
                                    uint32_t* __restrict__ w, uint32_t* __restrict__ tri,
                                    uint32_t* __restrict__ tinv) {
  pdl_wait();
  const uint32_t a0 = *a0p;
  const int total = la + npts - 1;
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < total; u += gridDim.x * blockDim.x) {
    const uint64_t cu = ((uint64_t)u * (uint64_t)(u > 0 ? u - 1 : 0) / 2) % (p - 1);
    tri[u] = powmod_dev(r, cu, p, mu);
    if (u < la || u < npts) {
      const uint32_t ri = powmod_dev(rinv, cu, p, mu);
      if (u < npts) tinv[u] = ri;
      if (u < la) w[u] = d_red64((uint64_t)powmod_dev(a0, (uint64_t)u, p, mu) * ri, p, mu);
    }
  }
}

// U[e][j] = P[e*ps + la-1-j] w[la-1-j]: scaled and reversed (the correlation
// sum_i U_i r^C(i+j) becomes the product coefficient la-1+j)
__global__ void scale_rows_kernel(const uint32_t* __restrict__ P, long long ps, int la, long long E,
                                  const uint32_t* __restrict__ w, uint32_t p, uint64_t mu,
                                  uint32_t* __restrict__ U) {
  pdl_wait();
  const long long total = E * la;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long e = i / la;
    const int j = la - 1 - (int)(i - e * la);
    U[i] = d_red64((uint64_t)P[e * ps + j] * w[j], p, mu);
  }
}

// EV[t][e] = M[e][t] tinv[t]: 32 x 32 tiles through shared memory
__global__ void transpose_scale_kernel(const uint32_t* __restrict__ M, long long E, int npts,
                                       const uint32_t* __restrict__ tinv, uint32_t p, uint64_t mu,
                                       uint32_t* __restrict__ EV) {
  pdl_wait();
  __shared__ uint32_t tile[32][33];
  const long long e0 = (long long)blockIdx.x * 32;
  const int t0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const long long e = e0 + r;
    const int t = t0 + threadIdx.x;
    tile[r][threadIdx.x] = (e < E && t < npts) ? M[e * npts + t] : 0u;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int t = t0 + r;
    const long long e = e0 + threadIdx.x;
    if (t < npts && e < E) EV[(long long)t * E + e] = d_red64((uint64_t)tile[threadIdx.x][r] * tinv[t], p, mu);
  }
}

int eval_points_geo(Context& cx, uint32_t p, const uint32_t* P, long long ps, int la, long long E,
                    const uint32_t* a0_dev, int npts, const GeoPts& g, uint32_t* EV) {
  const uint64_t mu = (uint64_t)((((u128)1) << 64) / p);
  const int lt = la + npts - 1;
  Workspace ws(cx);
  uint32_t *w, *tri, *tinv, *U, *Mv;
  FPM_TRY(ws.get((size_t)la, &w));
  FPM_TRY(ws.get((size_t)lt, &tri));
  FPM_TRY(ws.get((size_t)npts, &tinv));
  FPM_TRY(ws.get((size_t)E * la, &U));
  FPM_TRY(ws.get((size_t)E * npts, &Mv));
  const cudaStream_t st = cx.stream();
  FPM_CUDA_TRY(launch_pdl(chirp_tables_kernel, dim3((unsigned)((lt + 255) / 256)), dim3(256), 0, st,
                          a0_dev, g.r, g.rinv, la, npts, p, mu, w, tri, tinv));
  FPM_LAUNCH_CHECK();
  const long long tot = E * la;
  FPM_CUDA_TRY(launch_pdl(scale_rows_kernel, dim3((unsigned)std::min<long long>((tot + 255) / 256, 148 * 16)),
                          dim3(256), 0, st, P, ps, la, E, w, p, mu, U));
  FPM_LAUNCH_CHECK();
  MatRef A{U, 0, la, la};
  MatRef B{tri, 0, lt, lt};
  OutRef C{Mv, 0, npts, npts};
  FPM_TRY(polmat_middle(cx, p, (int)E, 1, 1, A, B, la - 1, lt - 1, la - 1, npts, 1, C));
  dim3 grid((unsigned)((E + 31) / 32), (unsigned)((npts + 31) / 32));
  FPM_CUDA_TRY(launch_pdl(transpose_scale_kernel, grid, dim3(32, 8), 0, st, Mv, E, npts, tinv, p,
                          mu, EV));
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
                     int64_t* sft_dev, const GeoPts& geo) {
  if (order <= T)
    return mbasis_fast(cx, p, E, m, n, 1, order, order, s_dev, P, ps, sft_dev, alpha,
                       (long long)m * n);
  const int o1 = (order + 1) / 2, o2 = order - o1;
  Workspace ws(cx);
  uint32_t *P1, *EV, *R, *P2;
  int64_t* s1;
  FPM_TRY(ws.get((size_t)m * m * (o1 + 1), &P1));
  FPM_TRY(ws.get((size_t)m, &s1));
  FPM_TRY(intbasis_rec_dev(cx, p, E, alpha, m, n, o1, s_dev, T, P1, o1 + 1, s1, geo));
  // residuals of the tail points: R_t = P1(alpha_t) E_t (appint.py:300-312)
  FPM_TRY(ws.get((size_t)o2 * m * m, &EV));
  FPM_TRY(ws.get((size_t)o2 * m * n, &R));
  // geometric tail points of a long P1: chirp evaluation (NTT path),
  // otherwise Horner (the reference switches at degree 16, appint.py:268)
  if (geo.on && o1 + 1 >= 64 && o2 >= 64)
    FPM_TRY(eval_points_geo(cx, p, P1, o1 + 1, o1 + 1, (long long)m * m, alpha + o1, o2, geo, EV));
  else
    FPM_TRY(eval_points(cx, p, P1, o1 + 1, o1 + 1, (long long)m * m, alpha + o1, o2, EV));
  FPM_TRY(point_product(cx, p, EV, E + (size_t)o1 * m * n, R, m, m, n, o2));
  FPM_TRY(ws.get((size_t)m * m * (o2 + 1), &P2));
  FPM_TRY(intbasis_rec_dev(cx, p, R, alpha + o1, m, n, o2, s1, T, P2, o2 + 1, sft_dev, geo));
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
  // appint._check_points (appint.py:203-205) compares the integers as given,
  // not their residues: [1, 1 + p] is accepted and runs with a repeated point
  std::vector<uint32_t> pts(order);
  for (int t = 0; t < order; ++t) pts[t] = (uint32_t)(alpha_host[t] % p);
  {
    std::vector<uint64_t> srt(alpha_host, alpha_host + order);
    std::sort(srt.begin(), srt.end());
    if (std::adjacent_find(srt.begin(), srt.end()) != srt.end()) {
      set_last_error("interpolation points must be pairwise distinct");
      return kDuplicatePoints;
    }
  }
  // geometric progression (appint._is_geometric, appint.py:248-259): every
  // contiguous range of the points is then one as well, with the same ratio
  GeoPts geo{false, 1u, 1u};
  if (order >= 3 && pts[0] != 0 && pts[1] != 0) {
    const uint64_t r = h_mulmod(pts[1], h_invmod(pts[0], p), p);
    bool ok = true;
    uint64_t cur = pts[1];
    for (int t = 2; t < order && ok; ++t) {
      cur = h_mulmod(cur, r, p);
      ok = cur == pts[t];
    }
    const bool off = option(kOptNoChirp) != 0;
    if (ok && !off) geo = GeoPts{true, (uint32_t)r, (uint32_t)h_invmod(r, p)};
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
                           (uint32_t*)P, ps, sft_dev, geo));
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
  // geometric points and degree >= 16: the chirp route (appint.py:268-282)
  if (npts >= 3 && L >= 17 && pts[0] != 0 && pts[1] != 0) {
    const uint64_t r = h_mulmod(pts[1], h_invmod(pts[0], p), p);
    bool ok = r != 1;
    uint64_t cur = pts[1];
    for (int t = 2; t < npts && ok; ++t) {
      cur = h_mulmod(cur, r, p);
      ok = cur == pts[t];
    }
    const bool off = option(kOptNoChirp) != 0;
    if (ok && !off)
      return eval_points_geo(cx, (uint32_t)p, (const uint32_t*)P, L, L, (long long)m * n, a_dev,
                             npts, GeoPts{true, (uint32_t)r, (uint32_t)h_invmod(r, p)},
                             (uint32_t*)out);
  }
  return eval_points(cx, (uint32_t)p, (const uint32_t*)P, L, L, (long long)m * n, a_dev, npts,
                     (uint32_t*)out);
}

}  // namespace fpm
