// api.cu -- extern "C" entry points declared in include/fpmat_b200.h.
#include <cstring>
#include <new>
#include <vector>
#include "../../include/fpmat_b200.h"
#include "ntt.cuh"
#include "ops.cuh"
#include "crt.cuh"
#include "pmbasis.cuh"

struct fpm_context {
  fpm::Context* cx;
  int pmbasis_T;
};

using namespace fpm;

namespace {

int check_elem(uint64_t p, int elem_bytes) {
  if (elem_bytes != 4 && elem_bytes != 8) {
    set_last_error("elem_bytes must be 4 or 8, got %d", elem_bytes);
    return kInvalidArgument;
  }
  if (p <= 2 || p >= (1ull << 62)) {
    set_last_error("modulus must satisfy 2 < p < 2^62, got %llu", (unsigned long long)p);
    return kOutOfRange;
  }
  if (elem_bytes == 4 && p >= (1ull << 32)) {
    set_last_error("uint32 elements need p < 2^32");
    return kInvalidArgument;
  }
  return kOk;
}

int check_dims(int m, int k, int n) {
  if (m < 0 || k < 0 || n < 0) {
    set_last_error("negative dimension");
    return kInvalidArgument;
  }
  return kOk;
}

// every entry point runs on its context's device, whatever the calling
// thread's current device is (tensors on cuda:1 with cuda:0 current)
int bind_device(fpm_context* ctx) {
  if (!ctx) {
    set_last_error("null context");
    return kInvalidArgument;
  }
  int cur = -1;
  FPM_CUDA_TRY(cudaGetDevice(&cur));
  if (cur != ctx->cx->device()) FPM_CUDA_TRY(cudaSetDevice(ctx->cx->device()));
  return kOk;
}

__global__ void widen_copy_kernel(const uint32_t* in, uint64_t* out, long long n) {
  pdl_wait();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = in[i];
}
__global__ void narrow_copy_kernel(const uint64_t* in, uint32_t* out, long long n) {
  pdl_wait();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = (uint32_t)in[i];
}
unsigned copy_grid(long long n) {
  long long b = (n + 255) / 256;
  return (unsigned)(b < 1 ? 1 : b > 148 * 16 ? 148 * 16 : b);
}
int copy_widen(const uint32_t* in, uint64_t* out, long long n, cudaStream_t st) {
  FPM_CUDA_TRY(launch_pdl(widen_copy_kernel, dim3(copy_grid(n)), dim3(256), 0, st, in, out, n));
  FPM_LAUNCH_CHECK();
  return kOk;
}
int copy_narrow(const uint64_t* in, uint32_t* out, long long n, cudaStream_t st) {
  FPM_CUDA_TRY(launch_pdl(narrow_copy_kernel, dim3(copy_grid(n)), dim3(256), 0, st, in, out, n));
  FPM_LAUNCH_CHECK();
  return kOk;
}

__global__ void residues_kernel(const void* in, int in64, long long n, PrimeSet ps,
                                uint32_t* out) {
  pdl_wait();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const uint64_t v = in64 ? ((const unsigned long long*)in)[i] : ((const uint32_t*)in)[i];
    for (int z = 0; z < ps.count; ++z) out[(long long)z * n + i] = d_red64(v, ps.pr[z].p, ps.pr[z].mu);
  }
}

// modring.ntt_forward / ntt_inverse for any prime (u64 generic transform):
// split twiddle tables built on the host per call (API path, not hot)
int ntt64(Context& cx, uint64_t p, int log_len, int batch, const uint64_t* in, uint64_t* out,
          int inverse) {
  const int k = h_two_adicity(p);
  const uint64_t N = 1ull << log_len;
  uint64_t omega = h_powmod(h_ntt_root(p), 1ull << (k - log_len), p);
  uint64_t scale = 1;
  if (inverse) {
    omega = h_invmod(omega, p);
    scale = h_invmod(N % p, p);
  }
  const int h = (log_len + 1) / 2;
  const size_t nlo = (size_t)1 << h, nhi = (size_t)((N >> h) > 0 ? (N >> h) : 1);
  std::vector<uint64_t> lo(nlo), hi(nhi);
  uint64_t w = 1;
  for (size_t i = 0; i < nlo; ++i, w = h_mulmod(w, omega, p)) lo[i] = w;
  const uint64_t step = h_powmod(omega, nlo, p);
  w = 1;
  for (size_t i = 0; i < nhi; ++i, w = h_mulmod(w, step, p)) hi[i] = w;
  Workspace ws(cx);
  uint64_t *dlo, *dhi;
  FPM_TRY(ws.get(nlo, &dlo));
  FPM_TRY(ws.get(nhi, &dhi));
  FPM_CUDA_TRY(cudaMemcpyAsync(dlo, lo.data(), nlo * 8, cudaMemcpyHostToDevice, cx.stream()));
  FPM_CUDA_TRY(cudaMemcpyAsync(dhi, hi.data(), nhi * 8, cudaMemcpyHostToDevice, cx.stream()));
  FPM_TRY(launch_ntt64_generic(p, omega, log_len, batch, in, out, scale, dlo, dhi, h,
                               cx.stream()));
  // the host tables must outlive the asynchronous copies
  FPM_CUDA_TRY(cudaStreamSynchronize(cx.stream()));
  return kOk;
}

}  // namespace

extern "C" {

int fpm_version(void) { return 100; }

const char* fpm_last_error(void) { return fpm::last_error(); }

long long fpm_launch_count(void) { return fpm::g_launch_count.load(); }

int fpm_context_create(int device, fpm_context** out) {
  if (!out) return kInvalidArgument;
  Context* cx = new (std::nothrow) Context(device);
  if (!cx) return kOutOfMemory;
  int s = cx->init();
  if (s != kOk) {
    delete cx;
    return s;
  }
  *out = new fpm_context{cx, 32};
  return kOk;
}

void fpm_context_destroy(fpm_context* ctx) {
  if (!ctx) return;
  delete ctx->cx;
  delete ctx;
}

int fpm_context_set_stream(fpm_context* ctx, void* stream) {
  FPM_TRY(bind_device(ctx));
  return ctx->cx->set_stream((cudaStream_t)stream);
}

int fpm_context_synchronize(fpm_context* ctx) {
  FPM_TRY(bind_device(ctx));
  FPM_CUDA_TRY(cudaStreamSynchronize(ctx->cx->stream()));
  return kOk;
}

int fpm_field_info(uint64_t p, int* two_adicity, uint64_t* root) {
  if (p <= 2 || p >= (1ull << 62)) {
    set_last_error("modulus must satisfy 2 < p < 2^62, got %llu", (unsigned long long)p);
    return kOutOfRange;
  }
  if (!h_is_prime(p)) {
    set_last_error("%llu is not prime", (unsigned long long)p);
    return kCompositeModulus;
  }
  if (two_adicity) *two_adicity = h_two_adicity(p);
  if (root) *root = h_ntt_root(p);
  return kOk;
}

int fpm_is_prime(uint64_t n) { return h_is_prime(n) ? 1 : 0; }

int fpm_factorize(uint64_t n, uint64_t* primes, int* exps, int cap, int* count) {
  if (!count || cap < 0 || (cap > 0 && (!primes || !exps))) return kInvalidArgument;
  if (n == 0) {
    set_last_error("cannot factorise 0");
    return kInvalidArgument;
  }
  const auto fac = h_factorize(n);
  *count = (int)fac.size();
  if ((int)fac.size() > cap) {
    set_last_error("%d prime factors, room for %d", (int)fac.size(), cap);
    return kInvalidArgument;
  }
  int i = 0;
  for (const auto& qe : fac) {
    primes[i] = qe.first;
    exps[i] = qe.second;
    ++i;
  }
  return kOk;
}

int fpm_element_order(uint64_t p, uint64_t a, uint64_t* order) {
  if (!order) return kInvalidArgument;
  FPM_TRY(fpm_field_info(p, nullptr, nullptr));
  if (a % p == 0) {
    set_last_error("0 has no multiplicative order");
    return kInvalidArgument;
  }
  *order = h_element_order(p, a % p, h_factorize(p - 1));
  return kOk;
}

int fpm_order_at_least(uint64_t p, uint64_t n, uint64_t* a) {
  if (!a) return kInvalidArgument;
  FPM_TRY(fpm_field_info(p, nullptr, nullptr));
  if (n > p - 1) {
    set_last_error("group order is %llu, no element of order %llu", (unsigned long long)(p - 1),
                   (unsigned long long)n);
    return kNoSuchElement;
  }
  if (n <= 1) {
    *a = 1;
    return kOk;
  }
  // deterministic scan 2, 3, ... (a generator exists, so this terminates)
  const auto fac = h_factorize(p - 1);
  for (uint64_t c = 2; c < p; ++c)
    if (h_element_order(p, c, fac) >= n) {
      *a = c;
      return kOk;
    }
  set_last_error("no element of order >= %llu", (unsigned long long)n);
  return kNoSuchElement;
}

int fpm_ntt_u32(fpm_context* ctx, uint32_t p, int log_len, int batch, const uint32_t* in,
                uint32_t* out, int inverse) {
  FPM_TRY(bind_device(ctx));
  if (p >= (1u << 31) || p <= 2) {
    set_last_error("fpm_ntt_u32 needs 2 < p < 2^31");
    return kOutOfRange;
  }
  if (log_len < 0 || log_len > h_two_adicity(p)) {
    set_last_error("p=%u supports transforms up to length 2^%d", p, h_two_adicity(p));
    return kOutOfRange;
  }
  if (batch <= 0) return kOk;
  Context& cx = *ctx->cx;
  if (log_len < kMinLogN) {
    // tiny lengths: the generic u64 transform on widened copies
    Workspace ws(cx);
    const size_t n = (size_t)batch << log_len;
    uint64_t *a, *b;
    FPM_TRY(ws.get(n, &a));
    FPM_TRY(ws.get(n, &b));
    FPM_TRY(copy_widen(in, a, n, cx.stream()));
    FPM_TRY(ntt64(cx, p, log_len, batch, a, b, inverse));
    return copy_narrow(b, out, n, cx.stream());
  }
  PrimeSet ps;
  ps.count = 1;
  FPM_TRY(cx.prime_const(p, log_len, &ps.pr[0]));
  const long long N = 1LL << log_len;
  if (!inverse) {
    NttFwdArgs a{};
    a.in = in; a.in64 = 0; a.in_stride = N; a.len = (int)N;
    a.reduce = 0; a.fold = 0; a.natural = 1; a.n_entries = batch; a.out = out;
    a.out_prime_stride = N * batch;
    if (ntt_big_ok(log_len)) {
      Workspace ws(cx);
      uint32_t* scratch;
      FPM_TRY(ws.get((size_t)batch * N, &scratch));
      return launch_ntt_fwd_big(cx, log_len, a, ps, scratch, cx.stream());
    }
    return launch_ntt_fwd(log_len, a, ps, cx.stream());
  }
  NttInvArgs a{};
  a.in = in; a.natural = 1; a.n_entries = batch; a.out = out;
  a.in_prime_stride = N * batch;
  a.out_stride = N; a.out_len = (int)N; a.off = 0; a.scale = 1;
  if (ntt_big_ok(log_len)) {
    Workspace ws(cx);
    uint32_t* scratch;
    FPM_TRY(ws.get((size_t)batch * N, &scratch));
    return launch_ntt_inv_big(cx, log_len, a, ps, scratch, cx.stream());
  }
  return launch_ntt_inv(log_len, a, ps, cx.stream());
}

int fpm_ntt_u64(fpm_context* ctx, uint64_t p, int log_len, int batch, const uint64_t* in,
                uint64_t* out, int inverse) {
  FPM_TRY(bind_device(ctx));
  if (p <= 2 || p >= (1ull << 62)) {
    set_last_error("modulus must satisfy 2 < p < 2^62");
    return kOutOfRange;
  }
  const int k = h_two_adicity(p);
  if (log_len < 0 || log_len > k) {
    set_last_error("p=%llu supports transforms up to length 2^%d", (unsigned long long)p, k);
    return kOutOfRange;
  }
  if (batch <= 0) return kOk;
  Context& cx = *ctx->cx;
  const size_t n = (size_t)batch << log_len;
  if (p < (1ull << 31) && log_len >= kMinLogN) {
    // 31-bit primes: the fast u32 transforms on narrowed copies
    Workspace ws(cx);
    uint32_t *a, *b;
    FPM_TRY(ws.get(n, &a));
    FPM_TRY(ws.get(n, &b));
    FPM_TRY(copy_narrow(in, a, n, cx.stream()));
    FPM_TRY(fpm_ntt_u32(ctx, (uint32_t)p, log_len, batch, a, b, inverse));
    return copy_widen(b, out, n, cx.stream());
  }
  if (in == out) {
    // the bit-reversal pass reads and writes different buffers
    Workspace ws(cx);
    uint64_t* tmp;
    FPM_TRY(ws.get(n, &tmp));
    FPM_CUDA_TRY(cudaMemcpyAsync(tmp, in, n * 8, cudaMemcpyDeviceToDevice, cx.stream()));
    return ntt64(cx, p, log_len, batch, tmp, out, inverse);
  }
  return ntt64(cx, p, log_len, batch, in, out, inverse);
}

int fpm_product_primes(uint64_t p, int k, int la, int lb, uint32_t* primes, int cap,
                       int* count) {
  if (!primes || !count || k < 0 || la <= 0 || lb <= 0) return kInvalidArgument;
  FPM_TRY(check_elem(p, 8));
  int logn = ceil_log2_min1((long long)la + lb - 1);
  if (logn < kMinLogN) logn = kMinLogN;
  uint32_t q[kMaxPrimes];
  int r = 0;
  FPM_TRY(select_primes(p, k, la, lb, logn, q, &r));
  *count = r;
  if (r > cap) {
    set_last_error("%d primes, room for %d", r, cap);
    return kInvalidArgument;
  }
  for (int i = 0; i < r; ++i) primes[i] = q[i];
  return kOk;
}

int fpm_split_residues(fpm_context* ctx, int elem_bytes, const void* in_dev, long long n,
                       const uint32_t* primes, int r, uint32_t* out_dev) {
  FPM_TRY(bind_device(ctx));
  if ((elem_bytes != 4 && elem_bytes != 8) || n < 0 || r < 1 || r > kMaxPrimes || !primes)
    return kInvalidArgument;
  if (n == 0) return kOk;
  PrimeSet ps{};
  ps.count = r;
  for (int z = 0; z < r; ++z) {
    if (primes[z] <= 2 || primes[z] >= (1u << 31)) {
      set_last_error("residue primes must satisfy 2 < q < 2^31");
      return kOutOfRange;
    }
    ps.pr[z].p = primes[z];
    ps.pr[z].mu = (uint64_t)((((u128)1) << 64) / primes[z]);
  }
  FPM_CUDA_TRY(launch_pdl(residues_kernel, dim3(copy_grid(n)), dim3(256), 0, ctx->cx->stream(),
                          in_dev, elem_bytes == 8 ? 1 : 0, n, ps, out_dev));
  FPM_LAUNCH_CHECK();
  return kOk;
}

int fpm_crt_combine(fpm_context* ctx, uint64_t p, int elem_bytes, const uint32_t* primes, int r,
                    const uint32_t* res_dev, long long entries, int len, void* out_dev) {
  FPM_TRY(bind_device(ctx));
  FPM_TRY(check_elem(p, elem_bytes));
  if (!primes || r < 1 || r > kMaxPrimes || entries < 0 || len < 0 || entries > (1LL << 31))
    return kInvalidArgument;
  if (entries == 0 || len == 0) return kOk;
  CrtArgs ca{};
  crt_prepare(ca, primes, r, p);
  ca.res = res_dev; ca.res_prime_stride = entries * len; ca.res_stride = len;
  ca.n_entries = (int)entries; ca.len = len;
  ca.out = out_dev; ca.out64 = elem_bytes == 8 ? 1 : 0; ca.out_stride = len;
  return launch_crt(ca, ctx->cx->stream());
}

int fpm_polmat_mul(fpm_context* ctx, uint64_t p, int elem_bytes, const void* A, int m, int k,
                   int la, const void* B, int n, int lb, void* C) {
  FPM_TRY(bind_device(ctx));
  FPM_TRY(check_elem(p, elem_bytes));
  FPM_TRY(check_dims(m, k, n));
  const int is64 = elem_bytes == 8;
  const int lc = (la > 0 && lb > 0) ? la + lb - 1 : 0;
  MatRef Ar{A, is64, la, la};
  MatRef Br{B, is64, lb, lb};
  OutRef Cr{C, is64, lc, lc};
  return polmat_mul(*ctx->cx, p, m, k, n, Ar, Br, Cr);
}

// Host-buffer product.  Large products are pipelined over R x R blocks of C:
// the copy-in stream uploads A's row blocks and B's column blocks in the order
// the blocks need them, the context stream multiplies block (i, j) as soon as
// A_i and B_j have landed, and the copy-out stream downloads C_ij while later
// blocks compute and upload -- PCIe traffic in both directions overlaps itself
// and the kernels instead of running as three serial phases.
int fpm_polmat_mul_host(fpm_context* ctx, uint64_t p, int elem_bytes, const void* A, int m,
                        int k, int la, const void* B, int n, int lb, void* C) {
  FPM_TRY(bind_device(ctx));
  FPM_TRY(check_elem(p, elem_bytes));
  FPM_TRY(check_dims(m, k, n));
  Context& cx = *ctx->cx;
  Workspace ws(cx);
  const size_t esz = elem_bytes;
  const size_t na = (size_t)m * k * (la > 0 ? la : 0), nb = (size_t)k * n * (lb > 0 ? lb : 0);
  const int lc = (la > 0 && lb > 0) ? la + lb - 1 : 0;
  const size_t nc = (size_t)m * n * lc;
  unsigned char *dA, *dB, *dC;
  FPM_TRY(ws.get(esz * na + 1, &dA));
  FPM_TRY(ws.get(esz * nb + 1, &dB));
  FPM_TRY(ws.get(esz * nc + 1, &dC));
  const int force = (int)option(kOptHostBlocks);
  // block count by output size (cfg5, 1.07 GB of C: R = 8 28.6 ms, 4 29.4, 6 35.3,
  // 2 32.6 -- the first block's inputs are the pipeline fill)
  int R = force > 0 ? force
                    : (esz * nc >= (1ull << 29) ? 8
                       : esz * nc >= (256u << 20) ? 4 : esz * nc >= (8u << 20) ? 3 : 1);
  if (R > m) R = m;
  if (R > n) R = n;
  if (R <= 1 || lc == 0) {
    if (na) FPM_CUDA_TRY(cudaMemcpyAsync(dA, A, esz * na, cudaMemcpyHostToDevice, cx.stream()));
    if (nb) FPM_CUDA_TRY(cudaMemcpyAsync(dB, B, esz * nb, cudaMemcpyHostToDevice, cx.stream()));
    FPM_TRY(fpm_polmat_mul(ctx, p, elem_bytes, dA, m, k, la, dB, n, lb, dC));
    if (nc) FPM_CUDA_TRY(cudaMemcpyAsync(C, dC, esz * nc, cudaMemcpyDeviceToHost, cx.stream()));
    FPM_CUDA_TRY(cudaStreamSynchronize(cx.stream()));
    return kOk;
  }
  cudaStream_t up, down;
  FPM_TRY(cx.aux_stream(0, &up));
  FPM_TRY(cx.aux_stream(1, &down));
  const cudaStream_t st = cx.stream();
  auto lo = [&](int i, int tot) { return (int)((long long)tot * i / R); };
  std::vector<cudaEvent_t> evs;
  auto ev = [&]() {
    cudaEvent_t e = cx.take_event();
    evs.push_back(e);
    return e;
  };
  int status = kOk;
  auto fail = [&](cudaError_t e) {
    if (e != cudaSuccess && status == kOk) {
      set_last_error("pipelined host product: %s", cudaGetErrorString(e));
      status = kCudaError;
    }
  };
  {
    cudaEvent_t start = ev();  // buffers were last used in the context stream's order
    fail(cudaEventRecord(start, st));
    fail(cudaStreamWaitEvent(up, start, 0));
    fail(cudaStreamWaitEvent(down, start, 0));
  }
  const int is64 = elem_bytes == 8;
  // one "landed" event per uploaded row block of A / column block of B: a
  // block of C waits only for its own two factors
  std::vector<cudaEvent_t> a_ev(R, nullptr), b_ev(R, nullptr);
  // each row block of A and column block of B is transformed once and its
  // evaluations reused by the other blocks of its row / column
  std::vector<EvalCache> ca(R), cb(R);
  // blocks in shells of max(i, j): shell s uploads A_s, multiplies the blocks
  // (s, j < s) that need only A_s and earlier columns, then uploads B_s and
  // multiplies (i <= s, s).  The copy-out stream starts after one block's
  // inputs and, within a shell, before its last upload has landed
  std::vector<std::pair<int, int>> order;
  for (int sh = 0; sh < R; ++sh) {
    for (int j = 0; j < sh; ++j) order.push_back({sh, j});
    for (int i = 0; i <= sh; ++i) order.push_back({i, sh});
  }
  auto upload_a = [&](int i) {
    const int i0 = lo(i, m), ib = lo(i + 1, m) - i0;
    if (ib > 0)
      fail(cudaMemcpyAsync(dA + esz * (size_t)i0 * k * la,
                         (const unsigned char*)A + esz * (size_t)i0 * k * la,
                         esz * (size_t)ib * k * la, cudaMemcpyHostToDevice, up));
    a_ev[i] = ev();
    fail(cudaEventRecord(a_ev[i], up));
  };
  auto upload_b = [&](int j) {
    const int j0 = lo(j, n), jb = lo(j + 1, n) - j0;
    if (jb > 0)
      fail(cudaMemcpy2DAsync(dB + esz * (size_t)k * j0 * lb, esz * (size_t)jb * lb,
                           (const unsigned char*)B + esz * (size_t)j0 * lb, esz * (size_t)n * lb,
                           esz * (size_t)jb * lb, k, cudaMemcpyHostToDevice, up));
    b_ev[j] = ev();
    fail(cudaEventRecord(b_ev[j], up));
  };
  // every upload is queued before the first product: the copy-in engine never
  // waits for the host loop below (which may block on the context stream)
  for (const auto& b : order) {
    if (!a_ev[b.first]) upload_a(b.first);
    if (!b_ev[b.second]) upload_b(b.second);
  }
  cudaEvent_t up_done = ev();
  fail(cudaEventRecord(up_done, up));
  for (size_t ob = 0; ob < order.size() && status == kOk; ++ob) {
    const int i = order[ob].first, j = order[ob].second;
    const int i0 = lo(i, m), i1 = lo(i + 1, m), ib = i1 - i0;
    const int j0 = lo(j, n), j1 = lo(j + 1, n), jb = j1 - j0;
    unsigned char* dAi = dA + esz * (size_t)i0 * k * la;
    unsigned char* dBj = dB + esz * (size_t)k * j0 * lb;  // column block j, packed [k][jb][lb]
    unsigned char* dCij = dC + esz * ((size_t)i0 * n + (size_t)ib * j0) * lc;  // packed [ib][jb][lc]
    fail(cudaStreamWaitEvent(st, a_ev[i], 0));
    fail(cudaStreamWaitEvent(st, b_ev[j], 0));
    if (status != kOk) break;
    MatRef Ar{dAi, is64, la, la};
    MatRef Br{dBj, is64, lb, lb};
    OutRef Cr{dCij, is64, lc, lc};
    const int s2 = polmat_mul_cached(cx, p, ib, k, jb, Ar, Br, Cr, &ca[i], &cb[j]);
    if (s2 != kOk) {
      status = s2;
      break;
    }
    cudaEvent_t done = ev();
    fail(cudaEventRecord(done, st));
    fail(cudaStreamWaitEvent(down, done, 0));
    fail(cudaMemcpy2DAsync((unsigned char*)C + esz * ((size_t)i0 * n + j0) * lc,
                           esz * (size_t)n * lc, dCij, esz * (size_t)jb * lc,
                           esz * (size_t)jb * lc, ib, cudaMemcpyDeviceToHost, down));
  }
  // the workspace returns to the pool in the context stream's order, and no
  // copy may still read the caller's buffers: join both copy streams on
  // every exit path (an early product failure leaves uploads queued)
  cudaEvent_t fin = ev();
  fail(cudaEventRecord(fin, down));
  fail(cudaStreamWaitEvent(st, fin, 0));
  fail(cudaStreamWaitEvent(st, up_done, 0));
  fail(cudaStreamSynchronize(st));
  for (auto e : evs) cx.give_event(e);
  for (auto& c : ca)
    if (c.EA) cx.release(c.EA);
  for (auto& c : cb)
    if (c.EA) cx.release(c.EA);
  return status;
}

struct fpm_multiplier {
  fpm_context* ctx;
  uint64_t p;
  int elem_bytes, m, k, la, max_rhs_len, logn;
  void* A;  // device copy of the left factor
  fpm::EvalCache cache;
};

int fpm_multiplier_create(fpm_context* ctx, uint64_t p, int elem_bytes, const void* A, int m,
                          int k, int la, int max_rhs_len, fpm_multiplier** out) {
  using namespace fpm;
  FPM_TRY(bind_device(ctx));
  if (!out) return kInvalidArgument;
  FPM_TRY(check_elem(p, elem_bytes));
  FPM_TRY(check_dims(m, k, 0));
  if (la < 0 || max_rhs_len < 1) {
    set_last_error("multiplier: la = %d, max_rhs_len = %d", la, max_rhs_len);
    return kInvalidArgument;
  }
  Context& cx = *ctx->cx;
  auto* mu = new fpm_multiplier();
  mu->ctx = ctx; mu->p = p; mu->elem_bytes = elem_bytes; mu->m = m; mu->k = k; mu->la = la;
  mu->max_rhs_len = max_rhs_len;
  mu->logn = ceil_log2_min1((long long)(la > 0 ? la : 1) + max_rhs_len - 1);
  const size_t bytes = (size_t)elem_bytes * m * k * (la > 0 ? la : 0);
  mu->A = nullptr;
  if (bytes) {
    const int s = cx.alloc(bytes, &mu->A);
    if (s != kOk) {
      delete mu;
      return s;
    }
    const cudaError_t e = cudaMemcpyAsync(mu->A, A, bytes, cudaMemcpyDeviceToDevice, cx.stream());
    if (e != cudaSuccess) {
      cx.release(mu->A);
      delete mu;
      set_last_error("multiplier: copy of A failed (%s)", cudaGetErrorString(e));
      return kCudaError;
    }
  }
  *out = mu;
  return kOk;
}

int fpm_multiplier_apply(fpm_multiplier* mu, const void* B, int n, int lb, void* C) {
  using namespace fpm;
  if (!mu) return kInvalidArgument;
  FPM_TRY(bind_device(mu->ctx));
  FPM_TRY(check_dims(mu->m, mu->k, n));
  if (lb > mu->max_rhs_len) {
    set_last_error("deg B = %d exceeds the multiplier envelope %d", lb - 1,
                   mu->max_rhs_len - 1);
    return kEnvelopeExceeded;
  }
  Context& cx = *mu->ctx->cx;
  const int is64 = mu->elem_bytes == 8;
  const int la = mu->la;
  const int lc = (la > 0 && lb > 0) ? la + lb - 1 : 0;
  OutRef Cr{C, is64, lc, lc};
  if (la <= 0 || lb <= 0 || mu->k == 0)
    return polmat_mul(cx, mu->p, mu->m, mu->k, n, MatRef{mu->A, is64, la, la},
                      MatRef{B, is64, lb, lb}, Cr);
  return cyclic_product(cx, mu->p, mu->m, mu->k, n, MatRef{mu->A, is64, la, la},
                        MatRef{B, is64, lb, lb}, mu->logn, 0, Cr, &mu->cache);
}

void fpm_multiplier_destroy(fpm_multiplier* mu) {
  if (!mu) return;
  fpm::Context& cx = *mu->ctx->cx;
  cudaStreamSynchronize(cx.stream());
  if (mu->A) cx.release(mu->A);
  if (mu->cache.EA) cx.release(mu->cache.EA);
  delete mu;
}

int fpm_polmat_middle(fpm_context* ctx, uint64_t p, int elem_bytes, const void* A, int m,
                      int k, int la, const void* B, int n, int lb, long long c, int d, int exact,
                      void* R) {
  FPM_TRY(bind_device(ctx));
  FPM_TRY(check_elem(p, elem_bytes));
  FPM_TRY(check_dims(m, k, n));
  if (d <= 0) return kOk;
  if (c < 0) {
    set_last_error("middle product offset c must be >= 0");
    return kInvalidArgument;
  }
  Context& cx = *ctx->cx;
  const int is64 = elem_bytes == 8;
  int da = -1, db = -1;
  FPM_TRY(matrix_degrees(cx, A, is64, (long long)m * k, la, B, (long long)k * n, lb, &da, &db));
  MatRef Ar{A, is64, la, la};
  MatRef Br{B, is64, lb, lb};
  OutRef Rr{R, is64, d, d};
  return polmat_middle(cx, p, m, k, n, Ar, Br, da, db, c, d, exact, Rr);
}

int fpm_pm_middle_product(fpm_context* ctx, uint64_t p, int elem_bytes, const void* A, int m,
                          int k, int la, const void* B, int n, int lb, long long c, int d,
                          void* R) {
  // polmat.pm_middle_product contract (polmat.py:476-481)
  FPM_TRY(bind_device(ctx));
  FPM_TRY(check_elem(p, elem_bytes));
  Context& cx = *ctx->cx;
  const int is64 = elem_bytes == 8;
  int da = -1, db = -1;
  FPM_TRY(matrix_degrees(cx, A, is64, (long long)m * k, la, B, (long long)k * n, lb, &da, &db));
  if (da >= c && c > 0) {
    set_last_error("deg A = %d must be < c = %lld", da, c);
    return kDegreeTooLarge;
  }
  if (db >= c + d) {
    set_last_error("deg B = %d must be < c+d = %lld", db, c + d);
    return kDegreeTooLarge;
  }
  return fpm_polmat_middle(ctx, p, elem_bytes, A, m, k, la, B, n, lb, c, d, 0, R);
}

int fpm_mbasis(fpm_context* ctx, uint64_t p, int elem_bytes, const void* F, int m, int n, int lf,
               int order, const int64_t* shift, void* P, int* lp, int64_t* rdeg_out) {
  FPM_TRY(bind_device(ctx));
  if (!lp || (m > 0 && !shift)) return kInvalidArgument;
  FPM_TRY(check_elem(p, elem_bytes));
  if (m <= 0 || n < 0 || order < 0) {
    set_last_error("mbasis needs m >= 1, n >= 0, order >= 0");
    return kInvalidArgument;
  }
  // identical output for every base threshold (appint.py:24-60 canonical
  // steps), so the iterative M-Basis is served by the same GPU recursion
  return pmbasis_run(*ctx->cx, p, elem_bytes == 8, F, m, n, lf, lf, order, shift,
                     ctx->pmbasis_T, P, order + 1, lp, rdeg_out);
}

int fpm_pmbasis(fpm_context* ctx, uint64_t p, int elem_bytes, const void* F, int m, int n,
                int lf, int order, const int64_t* shift, void* P, int* lp, int64_t* rdeg_out) {
  FPM_TRY(bind_device(ctx));
  if (!lp || (m > 0 && !shift)) return kInvalidArgument;
  FPM_TRY(check_elem(p, elem_bytes));
  if (m <= 0 || n < 0 || order < 0) {
    set_last_error("pmbasis needs m >= 1, n >= 0, order >= 0");
    return kInvalidArgument;
  }
  return pmbasis_run(*ctx->cx, p, elem_bytes == 8, F, m, n, lf, lf, order, shift,
                     ctx->pmbasis_T, P, order + 1, lp, rdeg_out);
}

int fpm_pmbasis_host(fpm_context* ctx, uint64_t p, int elem_bytes, const void* F, int m, int n,
                     int lf, int order, const int64_t* shift, void* P, int* lp,
                     int64_t* rdeg_out) {
  FPM_TRY(bind_device(ctx));
  if (!lp || (m > 0 && !shift)) return kInvalidArgument;
  FPM_TRY(check_elem(p, elem_bytes));
  if (m <= 0 || n < 0 || order < 0 || lf < 0) {
    set_last_error("pmbasis needs m >= 1, n >= 0, order >= 0");
    return kInvalidArgument;
  }
  Context& cx = *ctx->cx;
  Workspace ws(cx);
  const size_t esz = elem_bytes;
  const size_t nf = (size_t)m * n * lf, np = (size_t)m * m * (order + 1);
  unsigned char *dF, *dP;
  FPM_TRY(ws.get(esz * nf + 1, &dF));
  FPM_TRY(ws.get(esz * np + 1, &dP));
  if (nf) FPM_CUDA_TRY(cudaMemcpyAsync(dF, F, esz * nf, cudaMemcpyHostToDevice, cx.stream()));
  FPM_TRY(fpm_pmbasis(ctx, p, elem_bytes, dF, m, n, lf, order, shift, dP, lp, rdeg_out));
  FPM_CUDA_TRY(cudaMemcpyAsync(P, dP, esz * np, cudaMemcpyDeviceToHost, cx.stream()));
  FPM_CUDA_TRY(cudaStreamSynchronize(cx.stream()));
  return kOk;
}

int fpm_pm_intbasis(fpm_context* ctx, uint64_t p, int elem_bytes, const void* E, int m, int n,
                    int order, const uint64_t* alpha, const int64_t* shift, void* P, int* lp,
                    int64_t* rdeg_out) {
  FPM_TRY(bind_device(ctx));
  if (!lp || (m > 0 && !shift) || (order > 0 && (!alpha || !E))) return kInvalidArgument;
  FPM_TRY(check_elem(p, elem_bytes));
  if (m <= 0 || n < 0 || order < 0) {
    set_last_error("intbasis needs m >= 1, n >= 0, order >= 0");
    return kInvalidArgument;
  }
  if (elem_bytes != 4) {
    set_last_error("interpolant bases take uint32 operands (31-bit primes)");
    return kUnsupported;
  }
  return intbasis_run(*ctx->cx, p, E, m, n, order, alpha, shift, ctx->pmbasis_T, P, order + 1,
                      lp, rdeg_out);
}

int fpm_m_intbasis(fpm_context* ctx, uint64_t p, int elem_bytes, const void* E, int m, int n,
                   int order, const uint64_t* alpha, const int64_t* shift, void* P, int* lp,
                   int64_t* rdeg_out) {
  // the iterative basis is the same product of canonical steps
  return fpm_pm_intbasis(ctx, p, elem_bytes, E, m, n, order, alpha, shift, P, lp, rdeg_out);
}

int fpm_polmat_eval_points(fpm_context* ctx, uint64_t p, int elem_bytes, const void* P, int m,
                           int n, int L, const uint64_t* pts, int npts, void* out) {
  FPM_TRY(bind_device(ctx));
  if (m < 0 || n < 0 || L < 0 || npts < 0 || (npts > 0 && !pts)) return kInvalidArgument;
  FPM_TRY(check_elem(p, elem_bytes));
  if (elem_bytes != 4) {
    set_last_error("point evaluation takes uint32 operands (31-bit primes)");
    return kUnsupported;
  }
  return eval_points_run(*ctx->cx, p, P, m, n, L, pts, npts, out);
}

int fpm_profile_enable(fpm_context* ctx, int on) {
  FPM_TRY(bind_device(ctx));
  ctx->cx->profile_enable(on != 0);
  return kOk;
}

int fpm_profile_count(fpm_context* ctx) { return ctx ? ctx->cx->profile_count() : 0; }

int fpm_profile_get(fpm_context* ctx, int i, char* name, int name_len, float* ms) {
  if (!ctx || !name || name_len <= 0 || !ms) return kInvalidArgument;
  const char* nm = nullptr;
  FPM_TRY(ctx->cx->profile_get(i, &nm, ms));
  std::strncpy(name, nm ? nm : "", (size_t)name_len - 1);
  name[name_len - 1] = 0;
  return kOk;
}

int fpm_set_option(const char* name, long long value) { return set_option(name, value); }

int fpm_set_pmbasis_threshold(fpm_context* ctx, int T) {
  if (!ctx || T < 1) return kInvalidArgument;
  ctx->pmbasis_T = T;
  return kOk;
}

}  // extern "C"
