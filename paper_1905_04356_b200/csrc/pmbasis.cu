// pmbasis.cu -- M-Basis leaf kernel and the PM-Basis recursion driver.
//
// The basis is the product of canonical order-1 steps (appint.py:24-60),
// so the output is independent of the base threshold and of the product
// algorithms; this file reproduces the step exactly:
//   * rows are ranked by (s_i, i) (appint.py:34);
//   * the pivot rows are the rows not in the span of their predecessors --
//     computed by column elimination that always picks the lowest-ranked
//     non-pivot row with a nonzero entry (equivalent);
//   * kernel rows get the unique combination over the pivot rows, tracked
//     in an m x m transform matrix X (basis row i = X[i]);
//   * P <- Q P with pivot rows shifted by x (appint.py:79-117), trailing
//     zero coefficient matrices popped, s <- rdeg_s(P) (appint.py:179).
#include <cstdlib>

#include "pmbasis.cuh"
#include <algorithm>
#include <climits>
#include <vector>
#include "crt.cuh"

namespace fpm {
int mbasis_fast_max_order(int m, int n);
int mbasis_fast(Context& cx, uint32_t p, const void* F, int m, int n, long long fs, int lf,
                int order, const int64_t* s_dev, void* P, long long ps, int64_t* sft_dev,
                const uint32_t* alpha_dev = nullptr, long long ts = 1);
}  // namespace fpm

namespace fpm {

namespace {

template <typename T>
struct Arith;

template <>
struct Arith<uint32_t> {
  uint32_t p;
  uint64_t mu;
  __device__ __forceinline__ uint32_t mul(uint32_t a, uint32_t b) const {
    return d_red64((uint64_t)a * b, p, mu);
  }
  __device__ __forceinline__ uint32_t add(uint32_t a, uint32_t b) const { return d_red(a + b, p); }
  __device__ __forceinline__ uint32_t sub(uint32_t a, uint32_t b) const {
    return d_red(a - b + p, p);
  }
};

template <>
struct Arith<uint64_t> {
  uint64_t p, pni, r2;
  __device__ __forceinline__ uint64_t mont(uint64_t a, uint64_t b) const {
    const uint64_t lo = a * b, hi = __umul64hi(a, b);
    const uint64_t m = lo * pni;
    uint64_t r = hi + __umul64hi(m, p) + (lo != 0);
    return r >= p ? r - p : r;
  }
  __device__ __forceinline__ uint64_t mul(uint64_t a, uint64_t b) const {
    return mont(mont(a, r2), b);
  }
  __device__ __forceinline__ uint64_t add(uint64_t a, uint64_t b) const {
    const uint64_t s = a + b;
    return s >= p ? s - p : s;
  }
  __device__ __forceinline__ uint64_t sub(uint64_t a, uint64_t b) const {
    return a >= b ? a - b : a + p - b;
  }
};

template <typename T>
__device__ T d_inv(const Arith<T>& ar, T a) {
  // Fermat: a^(p-2)
  T r = 1, b = a;
  uint64_t e = (uint64_t)ar.p - 2;
  while (e) {
    if (e & 1) r = ar.mul(r, b);
    b = ar.mul(b, b);
    e >>= 1;
  }
  return r;
}

template <typename T>
struct LeafArgs {
  const T* F;
  long long fs;
  int lf;
  int m, n, order;
  const int64_t* s;  // device
  T* Pa;
  T* Pb;             // coefficient-major buffers [(order+2)][m][m]
  T* Pout;
  long long ps;
  int* lp_out;
  int64_t* sft_out;
  Arith<T> ar;
};

constexpr int kLeafThreads = 1024;

template <typename T>
__global__ void __launch_bounds__(kLeafThreads) mbasis_leaf_kernel(LeafArgs<T> a) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smraw[];
  const int m = a.m, n = a.n;
  const int tid = threadIdx.x, NT = blockDim.x;
  const Arith<T>& ar = a.ar;
  // carve: sft (int64, m) | W (m*n) | X (m*m) | fac (m) | rank | ord | piv
  int64_t* sft = (int64_t*)smraw;
  T* W = (T*)(sft + m);
  T* X = W + (size_t)m * n;
  T* fac = X + (size_t)m * m;
  int* rank = (int*)(fac + m);
  int* ord = rank + m;
  int* piv = ord + m;
  __shared__ int s_key[3];
  __shared__ int s_maxt;
  __shared__ T s_inv;
  __shared__ int64_t s_smin;

  const size_t mm = (size_t)m * m;
  T* Pc = a.Pa;
  T* Pn = a.Pb;
  for (size_t idx = tid; idx < mm; idx += NT) Pc[idx] = (idx / m == idx % m) ? T(1) : T(0);
  for (int i = tid; i < m; i += NT) sft[i] = a.s[i];
  if (tid == 0) {
    long long mn = LLONG_MAX;
    for (int i = 0; i < m; ++i) mn = min(mn, (long long)a.s[i]);
    s_smin = mn;
  }
  int L = 1;
  __syncthreads();

  for (int k = 0; k < a.order; ++k) {
    // ---- residual R_k = sum_t P_t F_{k-t} (appint.py:157-169) -------------
    const int tmax = min(L - 1, k);
    for (int idx = tid; idx < m * n; idx += NT) {
      const int i = idx / n, j = idx - (idx / n) * n;
      T acc = 0;
      for (int t = 0; t <= tmax; ++t) {
        const int fk = k - t;
        if (fk >= a.lf) continue;
        const T* prow = Pc + ((size_t)t * m + i) * m;
        for (int l = 0; l < m; ++l) {
          const T pv = prow[l];
          if (pv) acc = ar.add(acc, ar.mul(pv, a.F[((long long)l * n + j) * a.fs + fk]));
        }
      }
      W[idx] = acc;
    }
    // ---- ranks by (s_i, i) and transform X = I ----------------------------
    for (int i = tid; i < m; i += NT) {
      int r = 0;
      const int64_t si = sft[i];
      for (int j = 0; j < m; ++j) r += (sft[j] < si) || (sft[j] == si && j < i);
      rank[i] = r;
      ord[r] = i;
      piv[i] = 0;
    }
    for (size_t idx = tid; idx < mm; idx += NT) X[idx] = (idx / m == idx % m) ? T(1) : T(0);
    if (tid == 0) { s_key[0] = INT_MAX; s_key[1] = INT_MAX; s_key[2] = INT_MAX; }
    __syncthreads();

    // ---- column elimination with lowest-rank pivots (appint.py:38-58) -------
    int npiv = 0;
    for (int c = 0; c < n; ++c) {
      // three rotating slots: slot (c+1)%3 was last read in iteration c-2,
      // before the barrier of iteration c-1, so resetting it here is safe
      const int slot = c % 3;
      int key = INT_MAX;
      for (int i = tid; i < m; i += NT)
        if (!piv[i] && W[(size_t)i * n + c] != 0) key = min(key, rank[i]);
      key = __reduce_min_sync(0xffffffffu, key);
      if ((tid & 31) == 0 && key != INT_MAX) atomicMin(&s_key[slot], key);
      if (tid == 0) s_key[(c + 1) % 3] = INT_MAX;
      __syncthreads();
      key = s_key[slot];
      if (key == INT_MAX) continue;  // uniform: column already zero
      const int r = ord[key];
      if (tid == 0) {
        piv[r] = 1;
        s_inv = d_inv(ar, W[(size_t)r * n + c]);
      }
      __syncthreads();
      const T inv = s_inv;
      for (int i = tid; i < m; i += NT) {
        const T w = W[(size_t)i * n + c];
        fac[i] = (!piv[i] && w != 0) ? ar.mul(w, inv) : T(0);
      }
      __syncthreads();
      const int wd = n - c + m;
      for (int idx = tid; idx < m * wd; idx += NT) {
        const int i = idx / wd, col = idx - (idx / wd) * wd;
        const T f = fac[i];
        if (f == 0) continue;
        if (col < n - c) {
          const size_t o = (size_t)i * n + c + col;
          W[o] = ar.sub(W[o], ar.mul(f, W[(size_t)r * n + c + col]));
        } else {
          const int cc = col - (n - c);
          const size_t o = (size_t)i * m + cc;
          X[o] = ar.sub(X[o], ar.mul(f, X[(size_t)r * m + cc]));
        }
      }
      __syncthreads();
      ++npiv;
    }

    // ---- P <- Q P (appint.py:79-117), trim, shift update --------------------
    if (npiv > 0) {
      if (tid == 0) s_maxt = -1;
      __syncthreads();
      int lmax = -1;
      const size_t tot = (size_t)(L + 1) * mm;
      for (size_t idx = tid; idx < tot; idx += NT) {
        const int t = (int)(idx / mm);
        const size_t rem = idx - (size_t)t * mm;
        const int i = (int)(rem / m), col = (int)(rem - (size_t)(rem / m) * m);
        T v = 0;
        if (piv[i]) {
          if (t >= 1) v = Pc[((size_t)(t - 1) * m + i) * m + col];
        } else if (t < L) {
          const T* xr = X + (size_t)i * m;
          const T* pt = Pc + (size_t)t * mm + col;
          for (int j = 0; j < m; ++j) {
            const T xv = xr[j];
            if (xv) v = ar.add(v, ar.mul(xv, pt[(size_t)j * m]));
          }
        }
        Pn[idx] = v;
        if (v != 0) lmax = max(lmax, t);
      }
      lmax = __reduce_max_sync(0xffffffffu, lmax);
      if ((tid & 31) == 0 && lmax >= 0) atomicMax(&s_maxt, lmax);
      __syncthreads();
      L = s_maxt + 1;
      for (int i = tid; i < m; i += NT) {
        long long best = LLONG_MIN;
        for (int t = 0; t < L; ++t) {
          const T* row = Pn + ((size_t)t * m + i) * m;
          for (int j = 0; j < m; ++j)
            if (row[j] != 0) best = max((long long)best, (long long)(t + a.s[j]));
        }
        sft[i] = best == LLONG_MIN ? s_smin : best;
      }
      T* tmp = Pc; Pc = Pn; Pn = tmp;
      __syncthreads();
    }
  }

  // ---- PolMat.from_matpoly: entry-major output ------------------------------
  const long long ps = a.ps;
  for (long long idx = tid; idx < (long long)mm * ps; idx += NT) {
    const long long e = idx / ps;
    const int t = (int)(idx - e * ps);
    a.Pout[idx] = t < L ? Pc[(size_t)t * mm + e] : T(0);
  }
  if (tid == 0) *a.lp_out = L;
  for (int i = tid; i < m; i += NT) a.sft_out[i] = sft[i];
}

size_t leaf_smem_bytes(int m, int n, size_t esz) {
  return 8 * (size_t)m + esz * ((size_t)m * n + (size_t)m * m + m) + 4 * 3 * (size_t)m;
}

template <typename T>
int launch_leaf(Context& cx, uint64_t p, const void* F, int m, int n, long long fs, int lf,
                int order, const int64_t* s_dev, void* P, long long ps, int* lp_dev,
                int64_t* sft_dev) {
  Workspace ws(cx);
  const size_t mm = (size_t)m * m;
  T* Pa;
  T* Pb;
  FPM_TRY(ws.get((size_t)(order + 2) * mm, &Pa));
  FPM_TRY(ws.get((size_t)(order + 2) * mm, &Pb));
  LeafArgs<T> la{};
  la.F = (const T*)F; la.fs = fs; la.lf = lf; la.m = m; la.n = n; la.order = order;
  la.s = s_dev; la.Pa = Pa; la.Pb = Pb; la.Pout = (T*)P; la.ps = ps;
  la.lp_out = lp_dev; la.sft_out = sft_dev;
  if constexpr (sizeof(T) == 4) {
    la.ar.p = (uint32_t)p;
    la.ar.mu = (uint64_t)((((u128)1) << 64) / p);
  } else {
    CrtArgs tmp{};
    const uint32_t q1 = 2013265921u;
    crt_prepare(tmp, &q1, 1, p);
    la.ar.p = p;
    la.ar.pni = tmp.Pni;
    const u128 R = ((u128)1 << 64) % p;
    la.ar.r2 = (uint64_t)(R * R % p);
  }
  const size_t smem = leaf_smem_bytes(m, n, sizeof(T));
  if (smem > 200 * 1024) {
    set_last_error("mbasis leaf: m=%d n=%d needs %zu bytes of shared memory", m, n, smem);
    return kUnsupported;
  }
  if (smem > 48 * 1024)
    FPM_CUDA_TRY(cudaFuncSetAttribute(mbasis_leaf_kernel<T>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  FPM_CUDA_TRY(launch_pdl(mbasis_leaf_kernel<T>, dim3(1), dim3(kLeafThreads), smem, cx.stream(), la));
  FPM_LAUNCH_CHECK();
  // the pooled Pa/Pb return to the pool; stream order keeps reuse safe
  return kOk;
}

int leaf(Context& cx, uint64_t p, int is64, const void* F, int m, int n, long long fs, int lf,
         int order, const std::vector<int64_t>& s, void* P, long long ps, int* lp,
         std::vector<int64_t>* sft_out) {
  Workspace ws(cx);
  int64_t* s_dev;
  int64_t* sft_dev;
  int* lp_dev;
  FPM_TRY(ws.get(m > 0 ? m : 1, &s_dev));
  FPM_TRY(ws.get(m > 0 ? m : 1, &sft_dev));
  FPM_TRY(ws.get(1, &lp_dev));
  if (m > 0)
    FPM_CUDA_TRY(cudaMemcpyAsync(s_dev, s.data(), sizeof(int64_t) * m, cudaMemcpyHostToDevice,
                                 cx.stream()));
  const bool fast = !is64 && p < (1ull << 31) && order >= 1 && order <= mbasis_fast_max_order(m, n);
  if (fast) {
    FPM_TRY(mbasis_fast(cx, (uint32_t)p, F, m, n, fs, lf, order, s_dev, P, ps, sft_dev));
    FPM_TRY(launch_max_len(P, 0, (long long)m * m, (int)ps, lp_dev, cx.stream()));
  } else if (is64) {
    FPM_TRY(launch_leaf<uint64_t>(cx, p, F, m, n, fs, lf, order, s_dev, P, ps, lp_dev, sft_dev));
  } else {
    FPM_TRY(launch_leaf<uint32_t>(cx, p, F, m, n, fs, lf, order, s_dev, P, ps, lp_dev, sft_dev));
  }
  FPM_CUDA_TRY(cudaMemcpyAsync(lp, lp_dev, sizeof(int), cudaMemcpyDeviceToHost, cx.stream()));
  if (sft_out) {
    sft_out->resize(m);
    if (m > 0)
      FPM_CUDA_TRY(cudaMemcpyAsync(sft_out->data(), sft_dev, sizeof(int64_t) * m,
                                   cudaMemcpyDeviceToHost, cx.stream()));
  }
  FPM_CUDA_TRY(cudaStreamSynchronize(cx.stream()));
  return kOk;
}

// rdeg_s(P) with _finish_shift (appint.py:134-136, forms.py:47-51)
int rdeg_host(Context& cx, int is64, const void* P, int m, long long ps,
              const std::vector<int64_t>& s, std::vector<int64_t>& out) {
  Workspace ws(cx);
  int64_t* s_dev;
  int64_t* o_dev;
  FPM_TRY(ws.get(m, &s_dev));
  FPM_TRY(ws.get(m, &o_dev));
  FPM_CUDA_TRY(cudaMemcpyAsync(s_dev, s.data(), sizeof(int64_t) * m, cudaMemcpyHostToDevice,
                               cx.stream()));
  FPM_TRY(launch_rdeg(P, is64, m, m, (int)ps, s_dev, o_dev, cx.stream()));
  out.resize(m);
  FPM_CUDA_TRY(cudaMemcpyAsync(out.data(), o_dev, sizeof(int64_t) * m, cudaMemcpyDeviceToHost,
                               cx.stream()));
  FPM_CUDA_TRY(cudaStreamSynchronize(cx.stream()));
  return kOk;
}

int pmbasis_rec(Context& cx, uint64_t p, int is64, const void* F, int m, int n, long long fs,
                int lf, int order, const std::vector<int64_t>& s, int T, void* P, long long ps,
                int* lp) {
  const int lt = lf < order ? lf : order;
  if (order <= T) return leaf(cx, p, is64, F, m, n, fs, lt, order, s, P, ps, lp, nullptr);
  const size_t esz = is64 ? 8 : 4;
  const int o1 = (order + 1) / 2, o2 = order - o1;
  Workspace ws(cx);
  void* P1;
  FPM_TRY(ws.get(esz * (size_t)m * m * (o1 + 1), (unsigned char**)&P1));
  int lp1 = 0;
  FPM_TRY(pmbasis_rec(cx, p, is64, F, m, n, fs, lf < o1 ? lf : o1, o1, s, T, P1, o1 + 1, &lp1));
  // R = _pm_middle(P1, F.truncate(order), o1, o2)   (appint.py:191)
  void* R;
  FPM_TRY(ws.get(esz * (size_t)m * n * (o2 > 0 ? o2 : 1), (unsigned char**)&R));
  MatRef A{P1, is64, o1 + 1, lp1};
  MatRef B{F, is64, fs, lt};
  OutRef Ro{R, is64, o2, o2};
  FPM_TRY(polmat_middle(cx, p, m, m, n, A, B, lp1 - 1, lt - 1, o1, o2, 0, Ro));
  // s1 = _finish_shift(rdeg(P1, s), s)   (appint.py:192-194)
  std::vector<int64_t> s1;
  FPM_TRY(rdeg_host(cx, is64, P1, m, o1 + 1, s, s1));
  void* P2;
  FPM_TRY(ws.get(esz * (size_t)m * m * (o2 + 1), (unsigned char**)&P2));
  int lp2 = 0;
  FPM_TRY(pmbasis_rec(cx, p, is64, R, m, n, o2, o2, o2, s1, T, P2, o2 + 1, &lp2));
  // P = pm_mul(P2, P1)   (appint.py:196)
  MatRef A2{P2, is64, o2 + 1, lp2};
  MatRef B2{P1, is64, o1 + 1, lp1};
  const int lc = lp2 + lp1 - 1;
  if (lc > ps) {
    set_last_error("internal: product length %d exceeds output capacity %lld", lc, ps);
    return kInvalidArgument;
  }
  OutRef Co{P, is64, ps, (int)ps};
  FPM_TRY(polmat_mul(cx, p, m, m, m, A2, B2, Co));
  int deg = -1;
  FPM_TRY(matrix_degree(cx, P, is64, (long long)m * m, (int)ps, &deg));
  *lp = deg + 1;
  return kOk;
}

// nodes of this order and above size their products from P1's / P2's actual
// degrees (two host synchronisations per node: 7 nodes at cfg4's sigma 4096)
constexpr int kSizedNode = 1024;

// Sync-free recursion for 31-bit primes with shared-memory leaves: the
// shift stays on the device (each leaf turns s into s + delta, which equals
// rdeg_s of its basis, and composing leaves composes the shifts), and all
// lengths use the a-priori bound deg P <= order, so no node waits for the
// host.  Inside PM-Basis P1 F = 0 mod x^o1, so the reference's _pm_middle
// equals the true slice (exact = 1) whatever the cyclic length.
int pmbasis_rec_dev(Context& cx, uint32_t p, const void* F, int m, int n, long long fs, int lf,
                    int order, const int64_t* s_dev, int T, void* P, long long ps,
                    int64_t* sft_dev) {
  const int lt = lf < order ? lf : order;
  if (order <= T) return mbasis_fast(cx, p, F, m, n, fs, lt, order, s_dev, P, ps, sft_dev);
  const int o1 = (order + 1) / 2, o2 = order - o1;
  Workspace ws(cx);
  uint32_t *P1, *R, *P2;
  int64_t* s1;
  FPM_TRY(ws.get((size_t)m * m * (o1 + 1), &P1));
  FPM_TRY(ws.get((size_t)m, &s1));
  FPM_TRY(pmbasis_rec_dev(cx, p, F, m, n, fs, lf < o1 ? lf : o1, o1, s_dev, T, P1, o1 + 1, s1));
  // large nodes read the actual degree of P1 back (one host synchronisation):
  // generic bases have degree ~ order n / m, and the product below then runs
  // at half the transform length of the a-priori bound deg P <= order
  const bool sized = order >= kSizedNode;
  int lp1 = o1 + 1;
  if (sized) {
    int dg = -1;
    FPM_TRY(matrix_degree(cx, P1, 0, (long long)m * m, o1 + 1, &dg));
    lp1 = dg + 1 > 0 ? dg + 1 : 1;
  }
  FPM_TRY(ws.get((size_t)m * n * (o2 > 0 ? o2 : 1), &R));
  {
    MatRef A{P1, 0, o1 + 1, lp1};
    MatRef B{F, 0, fs, lt};
    OutRef Ro{R, 0, o2, o2};
    FPM_TRY(polmat_middle(cx, p, m, m, n, A, B, lp1 - 1, lt - 1, o1, o2, 1, Ro));
  }
  FPM_TRY(ws.get((size_t)m * m * (o2 + 1), &P2));
  FPM_TRY(pmbasis_rec_dev(cx, p, R, m, n, o2, o2, o2, s1, T, P2, o2 + 1, sft_dev));
  int lp2 = o2 + 1;
  if (sized) {
    int dg = -1;
    FPM_TRY(matrix_degree(cx, P2, 0, (long long)m * m, o2 + 1, &dg));
    lp2 = dg + 1 > 0 ? dg + 1 : 1;
  }
  MatRef A2{P2, 0, o2 + 1, lp2};
  MatRef B2{P1, 0, o1 + 1, lp1};
  OutRef Co{P, 0, ps, (int)ps};
  return polmat_mul(cx, p, m, m, m, A2, B2, Co);
}

}  // namespace

int mbasis_run(Context& cx, uint64_t p, int is64, const void* F, int m, int n, long long fs,
               int lf, int order, const int64_t* shift, void* P, long long ps, int* lp,
               int64_t* rdeg_out) {
  std::vector<int64_t> s(shift, shift + m);
  std::vector<int64_t> sft;
  const int lt = lf < order ? lf : order;
  FPM_TRY(leaf(cx, p, is64, F, m, n, fs, lt, order, s, P, ps, lp, rdeg_out ? &sft : nullptr));
  if (rdeg_out) {
    std::vector<int64_t> rd;
    FPM_TRY(rdeg_host(cx, is64, P, m, ps, s, rd));
    std::copy(rd.begin(), rd.end(), rdeg_out);
  }
  return kOk;
}

int pmbasis_run(Context& cx, uint64_t p, int is64, const void* F, int m, int n, long long fs,
                int lf, int order, const int64_t* shift, int T, void* P, long long ps, int* lp,
                int64_t* rdeg_out) {
  if (T < 1) T = 1;
  // the output does not depend on T (product of canonical steps): cap it so
  // leaves run on the shared-memory M-Basis kernels when they apply
  if (!is64 && p < (1ull << 31)) {
    // shared-memory leaves; order 8 balances the per-step residual-list
    // update (grows with the leaf order) against the tree's products
    // (cfg4 with the tensor-core residual update, tools/pmb_T.py: T = 32
    // 95.7 ms, 16 95.6, 12 93.7, 8 93.7)
    const int tf = mbasis_fast_max_order(m, n);
    const int tmax = (int)option(kOptPmbasisLeaf);
    const int tcap = tf < tmax ? tf : tmax;
    if (tf >= 1 && T > tcap) T = tcap;
  }
  std::vector<int64_t> s(shift, shift + m);
  const bool dev_off = option(kOptPmbasisHostSync) != 0;
  if (!dev_off && !is64 && p < (1ull << 31) && m > 0 && order >= 1 && T >= 1 &&
      T <= mbasis_fast_max_order(m, n) && ps >= order + 1) {
    Workspace ws(cx);
    int64_t *s_dev, *sft_dev;
    FPM_TRY(ws.get((size_t)m, &s_dev));
    FPM_TRY(ws.get((size_t)m, &sft_dev));
    FPM_CUDA_TRY(cudaMemcpyAsync(s_dev, s.data(), sizeof(int64_t) * m, cudaMemcpyHostToDevice,
                                 cx.stream()));
    FPM_TRY(pmbasis_rec_dev(cx, (uint32_t)p, F, m, n, fs, lf, order, s_dev, T, P, ps, sft_dev));
    int deg = -1;
    FPM_TRY(matrix_degree(cx, P, 0, (long long)m * m, (int)ps, &deg));  // synchronizes
    *lp = deg + 1;
    if (rdeg_out)
      FPM_CUDA_TRY(cudaMemcpy(rdeg_out, sft_dev, sizeof(int64_t) * m, cudaMemcpyDeviceToHost));
    return kOk;
  }
  FPM_TRY(pmbasis_rec(cx, p, is64, F, m, n, fs, lf, order, s, T, P, ps, lp));
  if (rdeg_out) {
    std::vector<int64_t> rd;
    FPM_TRY(rdeg_host(cx, is64, P, m, ps, s, rd));
    std::copy(rd.begin(), rd.end(), rdeg_out);
  }
  return kOk;
}

}  // namespace fpm
