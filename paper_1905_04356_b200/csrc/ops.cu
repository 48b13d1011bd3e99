// ops.cu -- evaluation/interpolation product engine (direct and multi-prime).
#include "ops.cuh"
#include <cmath>
#include "crt.cuh"
#include "ntt.cuh"
#include "pointwise.cuh"
#include "tc_pointwise.cuh"

namespace fpm {

// NTT primes for the multi-prime path: 31-bit, two-adicity >= 24, largest first
static const uint32_t kCrtPrimes[] = {2130706433u, 2113929217u, 2013265921u, 1811939329u,
                                      1711276033u, 1224736769u, 1107296257u};
static const int kNumCrtPrimes = 7;

int ceil_log2_min1(long long need) {
  int b = 0;
  long long x = need - 1;
  while (x > 0) { ++b; x >>= 1; }
  return b < 1 ? 1 : b;
}

namespace {

// the element kernels index with I = uint32_t when the index space fits (a
// 64-bit division per element is a long software sequence)
template <typename I>
__global__ void widen_kernel(const uint32_t* in, long long in_stride, uint64_t* out,
                             long long out_stride, long long entries, int len) {
  pdl_wait();
  const I total = (I)entries * (I)len, l = (I)len;
  for (I i = blockIdx.x * (I)blockDim.x + threadIdx.x; i < total; i += (I)gridDim.x * blockDim.x) {
    const I e = i / l;
    const int t = (int)(i - e * l);
    out[(long long)e * out_stride + t] = in[(long long)e * in_stride + t];
  }
}

// out[z][e][t] = in[e][t] mod prime z (u32), t < len: lets wide or unreduced
// inputs use the persistent u32 NTT (one cheap streaming pass; each input
// word is read once and reduced into every prime's plane)
template <typename I>
__global__ void split_reduce_kernel(const void* in, int in64, int reduce, long long stride,
                                    long long entries, int len, const __grid_constant__ PrimeSet ps,
                                    uint32_t* out) {
  pdl_wait();
  const I total = (I)entries * (I)len, l = (I)len;
  for (I i = blockIdx.x * (I)blockDim.x + threadIdx.x; i < total; i += (I)gridDim.x * blockDim.x) {
    const I e = i / l;
    const long long src = (long long)e * stride + (long long)(i - e * l);
    const uint64_t raw = in64 ? ((const unsigned long long*)in)[src]
                              : (uint64_t)((const uint32_t*)in)[src];
#pragma unroll
    for (int z = 0; z < kMaxPrimes; ++z) {
      if (z >= ps.count) break;
      out[(long long)z * (long long)total + i] =
          reduce ? d_red64(raw, ps.pr[z].p, ps.pr[z].mu) : (uint32_t)raw;
    }
  }
}

template <typename I>
__global__ void zero_tail_kernel(void* out, int is64, long long stride, long long entries,
                                 int from, int to) {
  pdl_wait();
  const I w = (I)(to - from);
  const I total = (I)entries * w;
  for (I i = blockIdx.x * (I)blockDim.x + threadIdx.x; i < total; i += (I)gridDim.x * blockDim.x) {
    const I e = i / w;
    const int t = from + (int)(i - e * w);
    if (is64)
      ((uint64_t*)out)[(long long)e * stride + t] = 0;
    else
      ((uint32_t*)out)[(long long)e * stride + t] = 0;
  }
}

// 32-bit indices when every index a grid-stride loop forms stays below 2^32
bool idx32(long long total, unsigned grid) { return total + (long long)grid * 256 < (1LL << 32); }

unsigned grid_for(long long total) {
  long long b = (total + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  if (b < 1) b = 1;
  return (unsigned)b;
}

int zero_out(OutRef C, long long entries, int from, int to, cudaStream_t st) {
  if (to <= from || entries <= 0) return kOk;
  const unsigned g = grid_for(entries * (to - from));
  if (idx32(entries * (to - from), g))
    FPM_CUDA_TRY(launch_pdl(zero_tail_kernel<uint32_t>, dim3(g), dim3(256), 0, st, C.ptr, C.is64,
                            C.stride, entries, from, to));
  else
    FPM_CUDA_TRY(launch_pdl(zero_tail_kernel<unsigned long long>, dim3(g), dim3(256), 0, st,
                            C.ptr, C.is64, C.stride, entries, from, to));
  FPM_LAUNCH_CHECK();
  return kOk;
}

bool direct_ok(uint64_t p, int logn) {
  return p < (1ull << 31) && p > 2 && h_two_adicity(p) >= logn;
}

}  // namespace

int matrix_degree(Context& cx, const void* M, int is64, long long entries, int L, int* deg) {
  return matrix_degrees(cx, M, is64, entries, L, nullptr, 0, 0, deg, nullptr);
}

int matrix_degrees(Context& cx, const void* M1, int is64, long long e1, int L1, const void* M2,
                   long long e2, int L2, int* deg1, int* deg2) {
  const bool two = deg2 != nullptr;
  const bool any1 = e1 > 0 && L1 > 0, any2 = two && e2 > 0 && L2 > 0;
  *deg1 = -1;
  if (two) *deg2 = -1;
  if (!any1 && !any2) return kOk;
  Workspace ws(cx);
  int* d = nullptr;
  FPM_TRY(ws.get(2, &d));
  if (any1) FPM_TRY(launch_max_len(M1, is64, e1, L1, d, cx.stream()));
  if (any2) FPM_TRY(launch_max_len(M2, is64, e2, L2, d + 1, cx.stream()));
  int h[2] = {0, 0};
  FPM_CUDA_TRY(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, cx.stream()));
  // the one host synchronisation of the degree-dependent entry points
  FPM_CUDA_TRY(cudaStreamSynchronize(cx.stream()));
  *deg1 = h[0] - 1;
  if (two) *deg2 = h[1] - 1;
  return kOk;
}

int select_primes(uint64_t p, int k, long long la, long long lb, int logn, uint32_t* primes,
                  int* count) {
  int r = 0;
  if (direct_ok(p, logn)) {
    primes[r++] = (uint32_t)p;
    *count = r;
    return kOk;
  }
  // exact integer cyclic convolution needs prod(q) > bound
  const long long N = 1LL << logn;
  const bool fold = lb > N;
  const double nfold = fold ? std::ceil((double)lb / (double)N) : 1.0;
  double terms = (double)la;
  if (!fold && lb < terms) terms = (double)lb;
  if (terms > (double)N) terms = (double)N;
  const double lg = std::log2((double)(k > 0 ? k : 1)) + std::log2(terms) + std::log2(nfold) +
                    2.0 * std::log2((double)(p - 1)) + 2.0;
  double have = 0.0;
  for (int i = 0; i < kNumCrtPrimes && have <= lg; ++i) {
    if (h_two_adicity(kCrtPrimes[i]) < logn) continue;
    primes[r++] = kCrtPrimes[i];
    have += std::log2((double)kCrtPrimes[i]);
  }
  if (have <= lg) {
    set_last_error("coefficient bound 2^%.1f exceeds the multi-prime capacity", lg);
    return kUnsupported;
  }
  *count = r;
  return kOk;
}

int cyclic_product(Context& cx, uint64_t p, int m, int k, int n, MatRef A, MatRef B,
                   int logn, long long off, OutRef C, EvalCache* cache, EvalCache* cache_b) {
  cudaStream_t st = cx.stream();
  const long long ec = (long long)m * n;
  if (ec == 0 || C.len <= 0) return kOk;
  if (k == 0 || A.len <= 0 || B.len <= 0) return zero_out(C, ec, 0, C.len, st);
  if (logn < kMinLogN) logn = kMinLogN;  // a larger cyclic length is exact as well
  // beyond one CTA (2^15): multi-pass transforms over HBM (ntt_big.cu)
  const bool big = logn > kMaxLogN;
  if (big && !ntt_big_ok(logn)) {
    set_last_error("transform length 2^%d beyond the supported 2^30", logn);
    return kUnsupported;
  }
  const long long N = 1LL << logn;
  const int fold = B.len > N ? 1 : 0;
  if (A.len > N) {
    set_last_error("left operand longer than the cyclic length");
    return kInvalidArgument;
  }
  const int wlen = C.len < N ? C.len : (int)N;  // coefficients carrying data
  off %= N;

  // ---- prime selection -----------------------------------------------------
  uint32_t primes[kMaxPrimes];
  int r = 0;
  const bool direct = direct_ok(p, logn);
  FPM_TRY(select_primes(p, k, A.len, B.len, logn, primes, &r));
  PrimeSet ps;
  ps.count = r;
  for (int i = 0; i < r; ++i) FPM_TRY(cx.prime_const(primes[i], logn, &ps.pr[i]));

  // ---- workspaces ------------------------------------------------------------
  Workspace ws(cx);
  const long long ea = (long long)m * k, eb = (long long)k * n;
  uint32_t *EA = nullptr, *EB = nullptr, *EC;
  if (!cache) FPM_TRY(ws.get(r * N * ea, &EA));
  if (!cache_b || fold) FPM_TRY(ws.get(r * N * eb, &EB));
  FPM_TRY(ws.get(r * N * ec, &EC));
  uint32_t* scratch = nullptr;  // long transforms: entry-major intermediate
  if (big) {
    long long most = ea > eb ? ea : eb;
    if (ec > most) most = ec;
    FPM_TRY(ws.get((size_t)r * N * most, &scratch));
  }

  const int reduce_needed = direct ? 0 : (p > primes[r - 1] ? 1 : 0);
  // pointwise engine: int8 tensor cores where the contraction is a real dense
  // product, CUDA cores otherwise (m <= 16: cfg3 35 vs 75 us on the TC path)
  // - point-quad kernel (tc_pq.cu) for 16 < m <= 32 (cfg2: 0.205 vs 0.225 ms)
  // - grouped / M-tiled point-major kernel (tc_grouped.cu) for m > 32
  // - tc_pointwise.cu for shapes neither takes (p < 2^30)
  bool pq = logn <= 13 && m > 16 && (long long)m * k * n >= 4096;
  for (int i = 0; i < r && pq; ++i) pq = tc_pq_applicable(m, k, n, (int)N, primes[i]);
  bool grouped = !pq && logn <= 13 && m > 32 && (long long)m * k * n >= 4096;
  for (int i = 0; i < r && grouped; ++i) grouped = tc_grouped_applicable(m, k, n, primes[i]);
  bool use_tc = logn <= 13;
  for (int i = 0; i < r && use_tc; ++i) use_tc = tc_pointwise_applicable(m, k, n, primes[i]);
  use_tc = !pq && (use_tc || grouped);
  // forward transforms (all primes in one launch: blockIdx.z = prime)
  NttFwdArgs fa{};
  fa.in = A.ptr; fa.in64 = A.is64; fa.in_stride = A.stride; fa.in_prime_stride = 0;
  fa.len = A.len; fa.fold = 0; fa.reduce = reduce_needed || (!direct && A.is64);
  fa.natural = 0; fa.pm = use_tc; fa.pblk_log = pq ? 2 : 5;
  fa.n_entries = (int)ea; fa.out = EA; fa.out_prime_stride = N * ea;
  if (direct && A.is64) fa.reduce = 0;
  NttFwdArgs fb = fa;
  fb.in = B.ptr; fb.in64 = B.is64; fb.in_stride = B.stride; fb.len = B.len; fb.fold = fold;
  fb.reduce = reduce_needed || (!direct && B.is64);
  if (direct && B.is64) fb.reduce = 0;
  fb.n_entries = (int)eb; fb.out = EB; fb.out_prime_stride = N * eb;
  // u64 / unreduced operands: one split-reduce pass, then the persistent
  // u32 transform (all primes at once) instead of the generic kernel
  auto to_u32 = [&](NttFwdArgs& f, long long entries) -> int {
    if (!(f.in64 || f.reduce) || f.fold || f.len <= 0 || logn > 13) return kOk;
    uint32_t* buf;
    FPM_TRY(ws.get((size_t)r * entries * f.len, &buf));
    dim3 g((unsigned)grid_for(entries * f.len), 1u);
    if (idx32(entries * f.len, g.x))
      FPM_CUDA_TRY(launch_pdl(split_reduce_kernel<uint32_t>, dim3(g), dim3(256), 0, st, f.in,
                              f.in64, f.reduce, f.in_stride, entries, f.len, ps, buf));
    else
      FPM_CUDA_TRY(launch_pdl(split_reduce_kernel<unsigned long long>, dim3(g), dim3(256), 0, st,
                              f.in, f.in64, f.reduce, f.in_stride, entries, f.len, ps, buf));
    FPM_LAUNCH_CHECK();
    f.in = buf; f.in64 = 0; f.reduce = 0; f.in_stride = f.len;
    f.in_prime_stride = entries * f.len;
    return kOk;
  };
  // cached evaluations (Multiplier; blocked host pipeline): an operand whose
  // transforms are already in its cache for this exact plan is not transformed
  auto bind = [&](EvalCache* c, int rows, int cols, int len, long long entries, uint32_t** E,
                  bool* hit) -> int {
    const int pm_now = use_tc ? 1 : 0, pl_now = pq ? 2 : 5;
    bool match = c->valid && c->p == p && c->m == rows && c->k == cols && c->a_len == len &&
                 c->logn == logn && c->r == r && c->pm == pm_now && c->pblk_log == pl_now;
    for (int i = 0; i < r && match; ++i) match = c->primes[i] == primes[i];
    const size_t words = (size_t)r * N * entries;
    if (!match) {
      if (c->EA && c->words < words) {
        cx.release(c->EA);
        c->EA = nullptr;
      }
      if (!c->EA) {
        void* ptr = nullptr;
        FPM_TRY(cx.alloc(words * 4, &ptr));
        c->EA = (uint32_t*)ptr;
        c->words = words;
      }
      c->valid = false;
      c->p = p; c->m = rows; c->k = cols; c->a_len = len; c->logn = logn;
      c->r = r; c->pm = pm_now; c->pblk_log = pl_now;
      for (int i = 0; i < r; ++i) c->primes[i] = primes[i];
    }
    *E = c->EA;
    *hit = match;
    return kOk;
  };
  bool a_cached = false, b_cached = false;
  if (cache) {
    FPM_TRY(bind(cache, m, k, A.len, ea, &EA, &a_cached));
    fa.out = EA;
  }
  if (cache_b && !fold) {
    FPM_TRY(bind(cache_b, k, n, B.len, eb, &EB, &b_cached));
    fb.out = EB;
  }
  if (!b_cached) FPM_TRY(to_u32(fb, eb));
  // both operands in one launch when their transforms are alike (persistent
  // grid: one tail wave instead of two)
  if (!a_cached) FPM_TRY(to_u32(fa, ea));
  if (big) {
    if (!a_cached) {
      StageTimer t_(cx, "ntt_fwd_A");
      FPM_TRY(launch_ntt_fwd_big(cx, logn, fa, ps, scratch, st));
    }
    if (!b_cached) {
      StageTimer t_(cx, "ntt_fwd_B");
      FPM_TRY(launch_ntt_fwd_big(cx, logn, fb, ps, scratch, st));
    }
  } else if (a_cached && b_cached) {
    // both evaluations reused
  } else if (a_cached) {
    StageTimer t_(cx, "ntt_fwd_B");
    FPM_TRY(launch_ntt_fwd(logn, fb, ps, st));
  } else if (b_cached) {
    StageTimer t_(cx, "ntt_fwd_A");
    FPM_TRY(launch_ntt_fwd(logn, fa, ps, st));
  } else if (fa.in64 == fb.in64 && fa.fold == fb.fold && fa.reduce == fb.reduce &&
             ntt_persist_fwd_ok(logn, fa) &&
             (fa.len == fb.len || logn <= 10)) {
    // short transforms are latency-bound: operands of different lengths (a
    // middle product) share the launch as well
    NttFwdArgs fab = fa;
    fab.len2 = fb.len;
    fab.in2 = fb.in; fab.in2_stride = fb.in_stride; fab.in2_prime_stride = fb.in_prime_stride;
    fab.n_entries2 = fb.n_entries; fab.out2 = fb.out; fab.out2_prime_stride = fb.out_prime_stride;
    StageTimer t_(cx, "ntt_fwd_AB");
    FPM_TRY(launch_ntt_fwd(logn, fab, ps, st));
  } else {
    {
      StageTimer t_(cx, "ntt_fwd_A");
      FPM_TRY(launch_ntt_fwd(logn, fa, ps, st));
    }
    StageTimer t_(cx, "ntt_fwd_B");
    FPM_TRY(launch_ntt_fwd(logn, fb, ps, st));
  }

  if (cache_b && !fold) cache_b->valid = true;
  if (cache) cache->valid = true;  // A's evaluations are in place (stream order)

  if (pq) {
    TcArgs ta{};
    ta.A = EA; ta.B = EB; ta.C = EC; ta.m = m; ta.k = k; ta.n = n; ta.npts = (int)N;
    ta.a_ps = N * ea; ta.b_ps = N * eb; ta.c_ps = N * ec;
    StageTimer t_(cx, "pointwise_tc");
    FPM_TRY(launch_tc_pq(ta, ps, st));
  } else if (use_tc) {
    TcArgs ta{};
    ta.A = EA; ta.B = EB; ta.C = EC; ta.m = m; ta.k = k; ta.n = n; ta.npts = (int)N;
    ta.a_ps = N * ea; ta.b_ps = N * eb; ta.c_ps = N * ec;
    StageTimer t_(cx, "pointwise_tc");
    bool pair = grouped && option(kOptTcNoPair) == 0;
    for (int i = 0; i < r && pair; ++i) pair = tc_pair_applicable(m, k, n, primes[i]);
    if (pair)
      FPM_TRY(launch_tc_pair(ta, ps, st));
    else if (grouped)
      FPM_TRY(launch_tc_grouped(ta, ps, st));
    else
      FPM_TRY(launch_tc_pointwise(ta, ps, st));
  } else {
    PointwiseArgs pa{};
    pa.A = EA; pa.B = EB; pa.C = EC; pa.m = m; pa.k = k; pa.n = n; pa.nblk = (int)(N / 32);
    pa.a_prime_stride = N * ea; pa.b_prime_stride = N * eb; pa.c_prime_stride = N * ec;
    StageTimer t_(cx, "pointwise");
    FPM_TRY(launch_pointwise(pa, ps, st));
  }

  NttInvArgs ia{};
  ia.in = EC; ia.in_prime_stride = N * ec; ia.natural = 0; ia.pm = use_tc; ia.n_entries = (int)ec;
  ia.pblk_log = pq ? 2 : 5;
  ia.out_len = wlen; ia.off = (int)off; ia.scale = 1;
  auto inverse = [&]() -> int {
    return big ? launch_ntt_inv_big(cx, logn, ia, ps, scratch, st)
               : launch_ntt_inv(logn, ia, ps, st);
  };
  if (direct && !C.is64) {
    ia.out = (uint32_t*)C.ptr; ia.out_stride = C.stride; ia.out_prime_stride = 0;
    StageTimer t_(cx, "ntt_inv");
    FPM_TRY(inverse());
  } else {
    uint32_t* R;
    FPM_TRY(ws.get((long long)r * ec * wlen, &R));
    ia.out = R; ia.out_stride = wlen; ia.out_prime_stride = ec * wlen;
    {
      StageTimer t_(cx, "ntt_inv");
      FPM_TRY(inverse());
    }
    StageTimer t2_(cx, direct ? "widen" : "crt");
    if (direct) {
      const unsigned g = grid_for(ec * wlen);
      if (idx32(ec * wlen, g))
        FPM_CUDA_TRY(launch_pdl(widen_kernel<uint32_t>, dim3(g), dim3(256), 0, st, R, wlen,
                                (uint64_t*)C.ptr, C.stride, ec, wlen));
      else
        FPM_CUDA_TRY(launch_pdl(widen_kernel<unsigned long long>, dim3(g), dim3(256), 0, st, R,
                                wlen, (uint64_t*)C.ptr, C.stride, ec, wlen));
      FPM_LAUNCH_CHECK();
    } else {
      CrtArgs ca{};
      crt_prepare(ca, primes, r, p);
      ca.res = R; ca.res_prime_stride = ec * wlen; ca.res_stride = wlen;
      ca.n_entries = (int)ec; ca.len = wlen;
      ca.out = C.ptr; ca.out64 = C.is64; ca.out_stride = C.stride;
      FPM_TRY(launch_crt(ca, st));
    }
  }
  return zero_out(C, ec, wlen, C.len, st);
}

int polmat_mul(Context& cx, uint64_t p, int m, int k, int n, MatRef A, MatRef B, OutRef C) {
  return polmat_mul_cached(cx, p, m, k, n, A, B, C, nullptr, nullptr);
}

int polmat_mul_cached(Context& cx, uint64_t p, int m, int k, int n, MatRef A, MatRef B,
                      OutRef C, EvalCache* ca, EvalCache* cb) {
  if (A.len <= 0 || B.len <= 0 || k == 0)
    return zero_out(C, (long long)m * n, 0, C.len, cx.stream());
  const long long need = (long long)A.len + B.len - 1;
  const int logn = ceil_log2_min1(need);
  return cyclic_product(cx, p, m, k, n, A, B, logn, 0, C, ca, cb);
}

int polmat_middle(Context& cx, uint64_t p, int m, int k, int n, MatRef A, MatRef B,
                  int da, int db, long long c, int d, int exact, OutRef C) {
  cudaStream_t st = cx.stream();
  const long long ec = (long long)m * n;
  if (da < 0 || db < 0 || d <= 0) return zero_out(C, ec, 0, C.len, st);
  A.len = da + 1;
  B.len = db + 1;
  if (exact) {
    // true slice: a cyclic length N with c + w <= N (the window fits) and
    // plen - N <= c (product coefficients >= N alias below c, never into the
    // window); A must fit (da < N), B longer than N is folded.  At the PM-Basis
    // nodes (da ~ c, db ~ 2c) this is half the full-product length.
    if (c > da + db) return zero_out(C, ec, 0, C.len, st);
    const long long plen = (long long)da + db + 1;
    OutRef C2 = C;
    long long w = d < C.len ? d : C.len;
    if (w > plen - c) w = plen - c;  // positions past the product are zero
    long long need = c + w;
    if (plen - c > need) need = plen - c;
    if (da + 1 > need) need = da + 1;
    const int logn = ceil_log2_min1(need);
    C2.len = (int)w;
    FPM_TRY(cyclic_product(cx, p, m, k, n, A, B, logn, c, C2));
    return zero_out(C, ec, C2.len, C.len, st);
  }
  // reference dispatch (polmat.py:490-497)
  const long long need = (long long)da + d + 1;
  const int log_len = ceil_log2_min1(need);
  const long long Nn = 1LL << (log_len < 62 ? log_len : 62);
  const bool wrap_ok = c + Nn > (long long)da + db;
  const int two = h_two_adicity(p);
  if (need >= 64 && log_len <= two && wrap_ok) {
    // matrix cyclic path: B folded mod x^N, window at (c + t) mod N
    OutRef C2 = C;
    C2.len = d < C.len ? d : C.len;
    if (log_len < kMinLogN) {
      // cannot happen (need >= 64) -- kept for clarity
      set_last_error("internal: cyclic length below minimum");
      return kInvalidArgument;
    }
    FPM_TRY(cyclic_product(cx, p, m, k, n, A, B, log_len, c, C2));
    return zero_out(C, ec, C2.len, C.len, st);
  }
  if (need < 64) {
    // every entry pair takes the schoolbook branch of upoly._middle
    // (la*d <= need^2/4 < 1024): the result is the exact slice
    return polmat_middle(cx, p, m, k, n, A, B, da, db, c, d, 1, C);
  }
  // generic entrywise semantics (small two-adicity primes): direct kernel
  MiddleEntryArgs ma{};
  ma.A = A.ptr; ma.B = B.ptr; ma.out = C.ptr;
  ma.in64 = A.is64; ma.out64 = C.is64;
  // the kernel trims every entry within its stride (a basis P1 has room for
  // order+1 coefficients but length deg P1 + 1), so only C must be dense
  if (A.is64 != B.is64 || A.is64 != C.is64 || C.stride != d || C.len != d) {
    set_last_error("entrywise middle product needs operands of one element width");
    return kInvalidArgument;
  }
  ma.m = m; ma.k = k; ma.n = n; ma.la = (int)A.stride; ma.lb = (int)B.stride;
  ma.c = c; ma.d = d;
  CrtArgs tmp{};
  crt_prepare(tmp, kCrtPrimes, 1, p);
  ma.P = p; ma.Pni = tmp.Pni;
  {
    const u128 R = ((u128)1 << 64) % p;
    ma.R2 = (uint64_t)(R * R % p);
  }
  ma.two_adicity = two;
  return launch_middle_entrywise(ma, st);
}

}  // namespace fpm
