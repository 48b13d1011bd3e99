// runtime.cu -- context, allocator, plan cache, error string, host number theory.
#include "runtime.cuh"
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>

namespace fpm {

std::atomic<long long> g_launch_count{0};

static thread_local char g_err[1024] = "";

void set_last_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
const char* last_error() { return g_err; }

// ---- number theory (host) ---------------------------------------------------
bool h_is_prime(uint64_t n) {
  // deterministic Miller-Rabin for n < 2^64 (same witness set as modring.py:20)
  if (n < 2) return false;
  static const uint64_t W[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  for (uint64_t q : W)
    if (n % q == 0) return n == q;
  uint64_t d = n - 1;
  int r = 0;
  while ((d & 1) == 0) { d >>= 1; ++r; }
  for (uint64_t a : W) {
    uint64_t x = h_powmod(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int i = 0; i < r - 1; ++i) {
      x = h_mulmod(x, x, n);
      if (x == n - 1) { comp = false; break; }
    }
    if (comp) return false;
  }
  return true;
}
int h_two_adicity(uint64_t p) {
  uint64_t m = p - 1;
  int k = 0;
  while (m && (m & 1) == 0) { m >>= 1; ++k; }
  return k;
}
// ---- factorisation of n < 2^64 (host): small primes by division, the
// cofactor split by Pollard's rho with Brent's cycle search and batched gcds
namespace {
uint64_t gcd_u64(uint64_t a, uint64_t b) {
  while (b) {
    const uint64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}
uint64_t rho_split(uint64_t n) {
  if ((n & 1) == 0) return 2;
  for (uint64_t c = 1;; ++c) {
    auto f = [&](uint64_t x) { return (uint64_t)(((u128)x * x + c) % n); };
    uint64_t y = 2, x = 2, g = 1, q = 1, ys = 2;
    const uint64_t batch = 64;
    for (uint64_t r = 1; g == 1; r <<= 1) {
      x = y;
      for (uint64_t i = 0; i < r; ++i) y = f(y);
      for (uint64_t k = 0; k < r && g == 1; k += batch) {
        ys = y;
        const uint64_t lim = (r - k) < batch ? (r - k) : batch;
        for (uint64_t i = 0; i < lim; ++i) {
          y = f(y);
          q = h_mulmod(q, x > y ? x - y : y - x, n);
        }
        g = gcd_u64(q, n);
      }
    }
    if (g == n) {
      // the batch overshot: step one at a time from its start
      do {
        ys = f(ys);
        g = gcd_u64(x > ys ? x - ys : ys - x, n);
      } while (g == 1);
    }
    if (g != n) return g;
  }
}
void factor_rec(uint64_t n, std::map<uint64_t, int>& out) {
  if (n == 1) return;
  if (h_is_prime(n)) {
    ++out[n];
    return;
  }
  const uint64_t d = rho_split(n);
  factor_rec(d, out);
  factor_rec(n / d, out);
}
}  // namespace

std::map<uint64_t, int> h_factorize(uint64_t n) {
  std::map<uint64_t, int> out;
  if (n < 2) return out;
  for (uint64_t q = 2; q < 1024 && q * q <= n; q += (q == 2 ? 1 : 2))
    while (n % q == 0) {
      ++out[q];
      n /= q;
    }
  factor_rec(n, out);
  return out;
}

uint64_t h_element_order(uint64_t p, uint64_t a, const std::map<uint64_t, int>& fac) {
  // smallest divisor d of p - 1 with a^d = 1: strip each prime factor while
  // the power stays 1
  uint64_t ord = p - 1;
  for (const auto& qe : fac)
    for (int e = 0; e < qe.second; ++e) {
      if (h_powmod(a, ord / qe.first, p) != 1) break;
      ord /= qe.first;
    }
  return ord;
}

uint64_t h_ntt_root(uint64_t p) {
  const int k = h_two_adicity(p);
  uint64_t a = 2;
  while (h_powmod(a, (p - 1) / 2, p) == 1) ++a;
  return h_powmod(a, (p - 1) >> k, p);
}

// ---- context ----------------------------------------------------------------
Context::Context(int device) : device_(device) {}

int Context::init() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    set_last_error("no CUDA device available");
    return kNoDevice;
  }
  if (device_ < 0 || device_ >= n) {
    set_last_error("device %d out of range (%d devices)", device_, n);
    return kInvalidArgument;
  }
  FPM_CUDA_TRY(cudaSetDevice(device_));
  cudaDeviceProp prop;
  FPM_CUDA_TRY(cudaGetDeviceProperties(&prop, device_));
  if (prop.major < 10) {
    set_last_error("device %d is sm_%d%d; this library is built for sm_100a", device_,
                   prop.major, prop.minor);
    return kNoDevice;
  }
  FPM_CUDA_TRY(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  own_stream_ = true;
  return kOk;
}

Context::~Context() {
  cudaSetDevice(device_);
  if (stream_) cudaStreamSynchronize(stream_);
  for (auto& kv : free_) cudaFree(kv.second);
  for (auto& kv : used_) cudaFree(kv.first);
  for (auto& kv : plans_) {
    cudaFree(kv.second.tw);
    cudaFree(kv.second.itw);
    cudaFree(kv.second.itw_s);
  }
  for (auto& kv : big_plans_) {
    for (uint2* t : {kv.second.lo, kv.second.hi, kv.second.ilo, kv.second.ihi, kv.second.r1k,
                     kv.second.ir1k})
      cudaFree(t);
  }
  if (pinned_) cudaFreeHost(pinned_);
  if (leaf_flags_) cudaFree(leaf_flags_);
  for (auto& a : aux_)
    if (a) cudaStreamDestroy(a);
  for (auto e : ev_pool_) cudaEventDestroy(e);
  if (own_stream_ && stream_) cudaStreamDestroy(stream_);
}

int Context::leaf_flags(uint32_t** flags, uint32_t* epoch) {
  std::lock_guard<std::mutex> lk(mu_);
  if (!leaf_flags_) {
    FPM_CUDA_TRY(cudaMalloc(&leaf_flags_, 128 * sizeof(uint32_t)));
    FPM_CUDA_TRY(cudaMemset(leaf_flags_, 0, 128 * sizeof(uint32_t)));
  }
  if (++leaf_epoch_ == 0) ++leaf_epoch_;  // 0 is the cleared state
  *flags = leaf_flags_;
  *epoch = leaf_epoch_;
  return kOk;
}

int Context::set_stream(cudaStream_t s) {
  std::lock_guard<std::mutex> lk(mu_);
  if (s == stream_) return kOk;
  // pooled blocks were last used in the old stream's order: drain it first
  if (stream_) FPM_CUDA_TRY(cudaStreamSynchronize(stream_));
  if (own_stream_ && stream_) cudaStreamDestroy(stream_);
  own_stream_ = false;
  stream_ = s;
  return kOk;
}

int Context::alloc(size_t bytes, void** out) {
  std::lock_guard<std::mutex> lk(mu_);
  bytes = (bytes + 255) & ~(size_t)255;
  auto it = free_.lower_bound(bytes);
  if (it != free_.end() && it->first <= 2 * bytes + (1 << 20)) {
    *out = it->second;
    used_[it->second] = it->first;
    free_.erase(it);
    return kOk;
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    // release cached blocks and retry once
    cudaStreamSynchronize(stream_);
    for (auto& kv : free_) cudaFree(kv.second);
    free_.clear();
    e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      set_last_error("cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
      return kOutOfMemory;
    }
  }
  used_[p] = bytes;
  *out = p;
  return kOk;
}

void Context::release(void* ptr) {
  std::lock_guard<std::mutex> lk(mu_);
  auto it = used_.find(ptr);
  if (it == used_.end()) return;
  free_.emplace(it->second, ptr);
  used_.erase(it);
}

int Context::pinned(size_t bytes, void** out) {
  std::lock_guard<std::mutex> lk(mu_);
  if (pinned_bytes_ < bytes) {
    if (pinned_) {
      FPM_CUDA_TRY(cudaStreamSynchronize(stream_));
      cudaFreeHost(pinned_);
      pinned_ = nullptr;
    }
    FPM_CUDA_TRY(cudaMallocHost(&pinned_, bytes));
    pinned_bytes_ = bytes;
  }
  *out = pinned_;
  return kOk;
}

int Context::plan(uint32_t p, int logn, const Plan** out) {
  std::lock_guard<std::mutex> lk(mu_);
  auto key = std::make_pair(p, logn);
  auto it = plans_.find(key);
  if (it != plans_.end()) {
    *out = &it->second;
    return kOk;
  }
  const int k = h_two_adicity(p);
  if (logn > k) {
    set_last_error("p=%u supports transforms up to length 2^%d, not 2^%d", p, k, logn);
    return kOrderTooSmall;
  }
  const size_t N = (size_t)1 << logn;
  // omega = root^(2^(k - logn)) (modring.py:233)
  const uint64_t omega = h_powmod(h_ntt_root(p), (uint64_t)1 << (k - logn), p);
  const uint64_t iomega = h_invmod(omega, p);
  // twiddle rows: tw[r*32 + c] = omega^(r*c), r < N/32, c < 32 (4-step
  // inter-pass twiddles; ntt.cu), same for omega^-1
  std::vector<uint2> tw(N), itw(N);
  const size_t rows = N / 32;
  for (size_t r = 0; r < rows; ++r) {
    const uint64_t wr = h_powmod(omega, r, p), iwr = h_powmod(iomega, r, p);
    uint64_t w = 1, iw = 1;
    for (size_t c = 0; c < 32; ++c) {
      tw[r * 32 + c] = make_uint2((uint32_t)w, h_shoup((uint32_t)w, p));
      itw[r * 32 + c] = make_uint2((uint32_t)iw, h_shoup((uint32_t)iw, p));
      w = h_mulmod(w, wr, p);
      iw = h_mulmod(iw, iwr, p);
    }
  }
  Plan pl;
  pl.p = p;
  pl.logn = logn;
  FPM_CUDA_TRY(cudaMalloc(&pl.tw, N * sizeof(uint2)));
  FPM_CUDA_TRY(cudaMalloc(&pl.itw, N * sizeof(uint2)));
  FPM_CUDA_TRY(cudaMemcpy(pl.tw, tw.data(), N * sizeof(uint2), cudaMemcpyHostToDevice));
  FPM_CUDA_TRY(cudaMemcpy(pl.itw, itw.data(), N * sizeof(uint2), cudaMemcpyHostToDevice));
  {
    // inverse rows pre-multiplied by N^-1: the last inverse pass applies its
    // row twiddles to all 32 values (k = 0 included), which also scales
    const uint64_t ni = h_invmod(N % p, p);
    std::vector<uint2> its(N);
    for (size_t i = 0; i < N; ++i) {
      const uint32_t w = (uint32_t)h_mulmod(itw[i].x, ni, p);
      its[i] = make_uint2(w, h_shoup(w, p));
    }
    FPM_CUDA_TRY(cudaMalloc(&pl.itw_s, N * sizeof(uint2)));
    FPM_CUDA_TRY(cudaMemcpy(pl.itw_s, its.data(), N * sizeof(uint2), cudaMemcpyHostToDevice));
  }
  // radix-32 inner roots w32 = omega^(N/32) (logn >= 5 in every kernel)
  const uint64_t w32 = h_powmod(omega, N >= 32 ? N / 32 : 1, p), iw32 = h_invmod(w32, p);
  uint64_t a = 1, b = 1;
  for (int e = 0; e < 16; ++e) {
    pl.w32[e] = make_uint2((uint32_t)a, h_shoup((uint32_t)a, p));
    pl.iw32[e] = make_uint2((uint32_t)b, h_shoup((uint32_t)b, p));
    a = h_mulmod(a, w32, p);
    b = h_mulmod(b, iw32, p);
  }
  pl.ninv = (uint32_t)h_invmod(N % p, p);
  pl.ninv_sh = h_shoup(pl.ninv, p);
  if (logn == 12 && p > (1u << 30) && p < (1u << 31)) {
    std::vector<uint8_t> tab;
    mma_ntt_tables(p, (uint32_t)omega, &tab);
    mma64_ntt_tables(p, (uint32_t)omega, &tab);  // appended at kMma64TabOff
    FPM_CUDA_TRY(cudaMalloc(&pl.mma, tab.size()));
    FPM_CUDA_TRY(cudaMemcpy(pl.mma, tab.data(), tab.size(), cudaMemcpyHostToDevice));
  }
  auto res = plans_.emplace(key, pl);
  *out = &res.first->second;
  return kOk;
}

cudaEvent_t Context::get_event() {
  if (!ev_free_.empty()) {
    cudaEvent_t e = ev_free_.back();
    ev_free_.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

void Context::profile_enable(bool on) {
  for (auto& s : stages_) {
    ev_free_.push_back(s.a);
    ev_free_.push_back(s.b);
  }
  stages_.clear();
  profiling_ = on;
}

int Context::stage_mark(const char* name, bool begin) {
  if (begin) {
    StageRec r{name, get_event(), get_event()};
    FPM_CUDA_TRY(cudaEventRecord(r.a, stream_));
    stages_.push_back(r);
  } else {
    for (auto it = stages_.rbegin(); it != stages_.rend(); ++it) {
      // close the innermost open stage (b not yet recorded is marked by name)
      if (it->name) {
        FPM_CUDA_TRY(cudaEventRecord(it->b, stream_));
        break;
      }
    }
  }
  return kOk;
}

int Context::profile_get(int i, const char** name, float* ms) {
  if (i < 0 || i >= (int)stages_.size()) return kInvalidArgument;
  FPM_CUDA_TRY(cudaEventSynchronize(stages_[i].b));
  FPM_CUDA_TRY(cudaEventElapsedTime(ms, stages_[i].a, stages_[i].b));
  *name = stages_[i].name;
  return kOk;
}

int Context::aux_stream(int i, cudaStream_t* out) {
  std::lock_guard<std::mutex> lk(mu_);
  if (!aux_[i]) FPM_CUDA_TRY(cudaStreamCreateWithFlags(&aux_[i], cudaStreamNonBlocking));
  *out = aux_[i];
  return kOk;
}

cudaEvent_t Context::take_event() {
  std::lock_guard<std::mutex> lk(mu_);
  if (!ev_pool_.empty()) {
    cudaEvent_t e = ev_pool_.back();
    ev_pool_.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  return e;
}

void Context::give_event(cudaEvent_t e) {
  std::lock_guard<std::mutex> lk(mu_);
  ev_pool_.push_back(e);
}

namespace {
struct OptDef {
  const char* name;
  long long dflt;
};
const OptDef kOptDefs[kOptCount] = {
    {"no_pdl", 0},      {"host_blocks", 0},   {"no_chirp", 0},     {"ntt_generic", 0},
    {"ntt_no_tma", 0},  {"ntt_no_small", 0},  {"ntt_pm_lsu", 0},   {"ntt_pm_scatter", 0},
    {"pmbasis_leaf", 8}, {"pmbasis_host_sync", 0}, {"ntt_no_mma", 0}, {"tc_no_pair", 0}, {"tc_pair1", 0},
    {"ntt_mma_r16", 0}, {"ntt_mma_dbg", 0}, {"tc_narrow", 8},
};
std::atomic<long long> g_opt[kOptCount] = {};
std::atomic<bool> g_opt_init{false};
std::mutex g_opt_mu;
void opt_init() {
  if (g_opt_init.load(std::memory_order_acquire)) return;
  std::lock_guard<std::mutex> lk(g_opt_mu);
  if (g_opt_init.load(std::memory_order_relaxed)) return;
  for (int i = 0; i < kOptCount; ++i) g_opt[i].store(kOptDefs[i].dflt);
  g_opt_init.store(true, std::memory_order_release);
}
}  // namespace

long long option(Option o) {
  opt_init();
  return g_opt[o].load(std::memory_order_relaxed);
}

int set_option(const char* name, long long value) {
  opt_init();
  if (!name) {
    // reset every option to its default
    for (int i = 0; i < kOptCount; ++i) g_opt[i].store(kOptDefs[i].dflt);
    return kOk;
  }
  for (int i = 0; i < kOptCount; ++i)
    if (std::strcmp(name, kOptDefs[i].name) == 0) {
      g_opt[i].store(value);
      return kOk;
    }
  set_last_error("unknown option '%s'", name);
  return kInvalidArgument;
}

bool pdl_enabled() { return option(kOptNoPdl) == 0; }

int Context::prime_const(uint32_t p, int logn, PrimeConst* out) {
  const Plan* pl = nullptr;
  if (logn > 15) {
    // long transforms keep their own split tables (big_plan, ntt_big.cu):
    // no N-entry row table here, only the scalars
    if (logn > h_two_adicity(p)) {
      set_last_error("p=%u supports transforms up to length 2^%d, not 2^%d", p,
                     h_two_adicity(p), logn);
      return kOrderTooSmall;
    }
    *out = PrimeConst{};
    out->p = p;
    out->c32 = (uint32_t)(((uint64_t)1 << 32) % p);
    out->mu = (uint64_t)((((u128)1) << 64) / p);
    out->m58 = (uint32_t)((((u128)1) << 58) / p);
    out->ninv = (uint32_t)h_invmod((1ull << logn) % p, p);
    out->ninv_sh = h_shoup(out->ninv, p);
    return kOk;
  }
  FPM_TRY(plan(p, logn, &pl));
  out->p = p;
  out->c32 = (uint32_t)(((uint64_t)1 << 32) % p);
  out->mu = (uint64_t)((((u128)1) << 64) / p);
  out->m58 = (uint32_t)((((u128)1) << 58) / p);
  out->ninv = pl->ninv;
  out->ninv_sh = pl->ninv_sh;
  for (int q = 0; q < 4; ++q) {
    const uint32_t v = (uint32_t)(((uint64_t)1 << (8 * q)) % p);
    out->sc[q] = make_uint2(v, h_shoup(v, p));
  }
  out->tw = pl->tw;
  out->itw = pl->itw;
  out->itw_s = pl->itw_s;
  out->mma = pl->mma;
  for (int e = 0; e < 16; ++e) {
    out->w32[e] = pl->w32[e];
    out->iw32[e] = pl->iw32[e];
  }
  return kOk;
}

}  // namespace fpm
