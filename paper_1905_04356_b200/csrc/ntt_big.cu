// ntt_big.cu -- transforms longer than one CTA holds: N = 2^16 .. 2^27.
//
// The reference runs _pm_mul_ntt up to N = 2^two_adicity (polmat.py:290-296,
// NttPlan accepts any log_len <= two_adicity, modring.py:212-250); the
// single-CTA kernels stop at 2^15.  Here a length-N transform is a sequence
// of P = ceil(log N / 10) passes over HBM (four-step / six-step
// decomposition), each pass a batch of R-point DFTs (R = 2^b <= 1024) on
// columns of the entry viewed as blocks:
//
//   pass j: block size M_j = N / (R_1 ... R_{j-1}), stride S_j = M_j / R_j.
//   Column (blk, x), x < S: elements a[blk M + x + S j'], j' < R.
//   forward:  Y = DFT_R over j' (natural in, natural out), then
//             Y[k1] *= w_M^(x k1), stored back at blk M + x + S k1;
//   inverse:  the transposed network, passes in reverse order: twiddle
//             w_M^-(x k1) first, then the inverse DFT_R, N^-1 on the last.
//
// X[k1 + R_1 k'] then sits at position S_1 k1 + pos'(k') (digit-reversed
// order, the single-CTA kernels' bit reversal generalised); the product path
// is order agnostic and the public natural-order API permutes once.
//
// A CTA owns X columns of one entry (X R <= 8192 words in shared memory):
// loads are coalesced (consecutive columns for S >= X, consecutive rows for
// the last pass where S = 1), the R-point DFT runs as radix-2 DIT stages in
// shared memory on bit-reversed placement, and the column twiddle w_N^E,
// E = x k1 N / M < N, is two Shoup products with a split table (w_N^(E & mask)
// times w_N^(E >> h) h = ceil(logN / 2): 2 x 2^14 entries at N = 2^27).
// Bound: HBM, 8 bytes per element per pass (P = 2 for N <= 2^20, 3 above).
#include <vector>
#include "ntt.cuh"
#include "runtime.cuh"

namespace fpm {
namespace {

constexpr int kBigThreads = 256;
constexpr int kTileWords = 8192;  // R * X

struct BigPrime {
  uint32_t p;
  uint64_t mu;
  const uint2* lo;   // w_N^i, i < 2^h
  const uint2* hi;   // w_N^(i 2^h), i < N / 2^h
  const uint2* r1k;  // w_1024^i, i < 512 (inner R-point DFT roots)
  uint32_t ninv, ninv_sh;
};

struct BigArgs {
  int logn, b, X, h;     // R = 2^b, columns per CTA, split-table shift
  long long M, S;        // block size and stride of this pass
  int inverse;
  // input role: 0 = entry-major scratch, 1 = coefficients (first forward
  // pass), 2 = blocked eval layout E[N/32][entry][32] (first inverse pass)
  int in_kind;
  // output role: 0 = entry-major scratch, 1 = coefficient window (last
  // inverse pass), 2 = blocked eval layout (last forward pass)
  int out_kind;
  int n_entries;
  const uint32_t* src;   // scratch / blocked input (per prime: + z * src_ps)
  long long src_ps;
  uint32_t* dst;         // scratch / blocked output
  long long dst_ps;
  // coefficient input (in_kind 1)
  const void* in;
  long long in_stride, in_prime_stride;
  int in64, len, fold, reduce;
  // coefficient output (out_kind 1)
  uint32_t* out;
  long long out_stride, out_prime_stride;
  int out_len, off, scale;
  BigPrime pr[kMaxPrimes];
};

__device__ __forceinline__ uint32_t bmul(uint32_t a, uint2 w, uint32_t p) {
  return d_red(d_shoup(a, w.x, w.y, p), p);
}

__device__ __forceinline__ long long blocked_ix(long long pos, long long e, long long ne) {
  return (((pos >> 5) * ne + e) << 5) + (pos & 31);
}

__device__ __forceinline__ uint32_t coef_in(const BigArgs& a, const BigPrime& bp, int z,
                                            long long e, long long n, long long N) {
  const long long base = e * a.in_stride + (long long)z * a.in_prime_stride;
  uint32_t acc = 0;
  for (long long t = n; t < a.len; t += N) {
    const uint64_t raw = a.in64 ? __ldg((const unsigned long long*)a.in + base + t)
                                : (uint64_t)__ldg((const uint32_t*)a.in + base + t);
    const uint32_t r = a.reduce ? d_red64(raw, bp.p, bp.mu) : (uint32_t)raw;
    acc = d_red(acc + r, bp.p);
    if (!a.fold) break;
  }
  return acc;
}

__global__ void __launch_bounds__(kBigThreads) big_pass_kernel(const __grid_constant__ BigArgs a) {
  pdl_wait();
  extern __shared__ uint32_t tile[];  // [R][X + 1]
  uint2* roots = reinterpret_cast<uint2*>(tile + kTileWords + kTileWords / 8 + 64);
  const int z = blockIdx.z;
  const BigPrime& bp = a.pr[z];
  const uint32_t p = bp.p;
  const int R = 1 << a.b, X = a.X, pitch = X + 1;
  const long long N = 1LL << a.logn;
  const long long e = blockIdx.y;
  const long long c0 = (long long)blockIdx.x * X;
  const long long M = a.M, S = a.S;
  const int tid = threadIdx.x;
  // inner DFT roots (w_1024^i, forward or inverse table)
  for (int i = tid; i < 512; i += kBigThreads) roots[i] = __ldg(bp.r1k + i);
  const bool rowmajor = S >= X;  // consecutive columns contiguous in memory
  const long long ebase = (e + (long long)z * a.n_entries) * N;  // scratch
  auto addr = [&](int r, int xi) -> long long {
    const long long c = c0 + xi;
    return (c / S) * M + (c % S) + S * r;
  };
  const long long mask = (1LL << a.h) - 1;
  auto twiddle = [&](uint32_t v, int r, int xi) -> uint32_t {
    const long long x = (c0 + xi) % S;
    if (x == 0 || r == 0) return v;
    const long long E = ((x * r) * (N / M)) & (N - 1);
    v = bmul(v, __ldg(bp.lo + (E & mask)), p);
    return bmul(v, __ldg(bp.hi + (E >> a.h)), p);
  };
  // ---- load (bit-reversed row placement) --------------------------------
  const int total = R * X;
  for (int idx = tid; idx < total; idx += kBigThreads) {
    int r, xi;
    if (rowmajor) { r = idx / X; xi = idx % X; } else { xi = idx / R; r = idx % R; }
    const long long pos = addr(r, xi);
    uint32_t v;
    if (a.in_kind == 1)
      v = coef_in(a, bp, z, e, pos, N);
    else if (a.in_kind == 2)
      v = __ldg(a.src + z * a.src_ps + blocked_ix(pos, e, a.n_entries));
    else
      v = a.src[ebase + pos];
    if (a.inverse) v = twiddle(v, r, xi);
    const int rr = (int)(__brev((unsigned)r) >> (32 - a.b));
    tile[rr * pitch + xi] = v;
  }
  __syncthreads();
  // ---- R-point DIT stages (natural output order) ------------------------
  const int half = (R / 2) * X;
  for (int hb = 0; hb < a.b; ++hb) {
    const int hh = 1 << hb;
    for (int q = tid; q < half; q += kBigThreads) {
      const int xi = q % X, bi = q / X;
      const int i = bi & (hh - 1), g = bi >> hb;
      const int u = g * 2 * hh + i, v = u + hh;
      uint32_t t = tile[v * pitch + xi];
      if (i) t = bmul(t, roots[i << (9 - hb)], p);
      const uint32_t s = tile[u * pitch + xi];
      tile[u * pitch + xi] = d_red(s + t, p);
      tile[v * pitch + xi] = d_red(s - t + p, p);
    }
    __syncthreads();
  }
  // ---- store ------------------------------------------------------------
  for (int idx = tid; idx < total; idx += kBigThreads) {
    int r, xi;
    if (rowmajor) { r = idx / X; xi = idx % X; } else { xi = idx / R; r = idx % R; }
    uint32_t v = tile[r * pitch + xi];
    const long long pos = addr(r, xi);
    if (!a.inverse) v = twiddle(v, r, xi);
    if (a.out_kind == 1) {
      long long i = (pos - a.off) & (N - 1);
      if (i < a.out_len) {
        if (a.scale) v = d_red(d_shoup(v, bp.ninv, bp.ninv_sh, p), p);
        a.out[e * a.out_stride + (long long)z * a.out_prime_stride + i] = v;
      }
    } else if (a.out_kind == 2) {
      a.dst[z * a.dst_ps + blocked_ix(pos, e, a.n_entries)] = v;
    } else {
      a.dst[ebase + pos] = v;
    }
  }
}

// natural order <-> digit-reversed positions (public NTT API)
struct PermArgs {
  const uint32_t* src;
  uint32_t* dst;
  long long N;
  int np;           // passes
  int bits[4];      // b_j
  int to_natural;   // 1: dst[k] = src[pos(k)], 0: dst[pos(k)] = src[k]
  long long entries;
};

__global__ void big_perm_kernel(const __grid_constant__ PermArgs a) {
  pdl_wait();
  const long long total = a.entries * a.N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long e = i / a.N, k = i - e * a.N;
    // k = sum_j k_j prod_{i<j} R_i ; pos = sum_j k_j prod_{i>j} R_i
    long long rest = k, pos = 0, sfx = a.N;
    for (int j = 0; j < a.np; ++j) {
      const long long R = 1LL << a.bits[j];
      sfx /= R;
      pos += (rest & (R - 1)) * sfx;
      rest >>= a.bits[j];
    }
    if (a.to_natural)
      a.dst[e * a.N + k] = a.src[e * a.N + pos];
    else
      a.dst[e * a.N + pos] = a.src[e * a.N + k];
  }
}

void split_bits(int logn, int* np, int bits[4]) {
  *np = (logn + 9) / 10;
  int left = logn;
  for (int j = 0; j < *np; ++j) {
    bits[j] = left / (*np - j);
    left -= bits[j];
  }
}

size_t big_smem() { return (kTileWords + kTileWords / 8 + 64) * 4 + 512 * sizeof(uint2); }

int fill_primes(Context& cx, int logn, const PrimeSet& ps, bool inverse, BigArgs& a) {
  for (int z = 0; z < ps.count; ++z) {
    const BigPlan* bp = nullptr;
    FPM_TRY(cx.big_plan(ps.pr[z].p, logn, &bp));
    a.pr[z].p = bp->p;
    a.pr[z].mu = ps.pr[z].mu;
    a.pr[z].lo = inverse ? bp->ilo : bp->lo;
    a.pr[z].hi = inverse ? bp->ihi : bp->hi;
    a.pr[z].r1k = inverse ? bp->ir1k : bp->r1k;
    a.pr[z].ninv = bp->ninv;
    a.pr[z].ninv_sh = bp->ninv_sh;
    a.h = bp->h;
  }
  return kOk;
}

int run_pass(BigArgs& a, int j, int np, const int bits[4], int nprimes, cudaStream_t st) {
  long long M = 1LL << a.logn;
  for (int i = 0; i < j; ++i) M >>= bits[i];
  a.b = bits[j];
  a.M = M;
  a.S = M >> bits[j];
  int X = kTileWords >> a.b;
  if (X > 32) X = 32;
  a.X = X;
  const long long cols = (1LL << a.logn) >> a.b;
  static bool attr = false;
  if (!attr) {
    FPM_CUDA_TRY(cudaFuncSetAttribute(big_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)big_smem()));
    attr = true;
  }
  dim3 grid((unsigned)(cols / X), (unsigned)a.n_entries, (unsigned)nprimes);
  FPM_CUDA_TRY(launch_pdl(big_pass_kernel, grid, dim3(kBigThreads), big_smem(), st, a));
  FPM_LAUNCH_CHECK();
  (void)np;
  return kOk;
}

}  // namespace

bool ntt_big_ok(int logn) { return logn > kMaxLogN && logn <= 30; }

int launch_ntt_fwd_big(Context& cx, int logn, const NttFwdArgs& f, const PrimeSet& ps,
                       uint32_t* scratch, cudaStream_t st) {
  int np, bits[4];
  split_bits(logn, &np, bits);
  auto one = [&](const void* in, long long in_stride, long long in_ps, int n_entries,
                 uint32_t* out, long long out_ps) -> int {
    if (n_entries <= 0) return kOk;
    if (n_entries > 65535) {
      set_last_error("long transforms: %d entries exceed one grid dimension", n_entries);
      return kUnsupported;
    }
    BigArgs a{};
    a.logn = logn;
    a.inverse = 0;
    a.n_entries = n_entries;
    FPM_TRY(fill_primes(cx, logn, ps, false, a));
    a.in = in; a.in_stride = in_stride; a.in_prime_stride = in_ps;
    a.in64 = f.in64; a.len = f.len; a.fold = f.fold; a.reduce = f.reduce;
    const long long N = 1LL << logn;
    for (int j = 0; j < np; ++j) {
      a.in_kind = j == 0 ? 1 : 0;
      a.src = scratch; a.src_ps = (long long)n_entries * N;
      const bool last = j == np - 1;
      // natural-order API: the last pass leaves digit-reversed data in scratch
      a.out_kind = last && !f.natural && !f.pm ? 2 : 0;
      a.dst = a.out_kind == 2 ? out : scratch;
      a.dst_ps = a.out_kind == 2 ? out_ps : (long long)n_entries * N;
      FPM_TRY(run_pass(a, j, np, bits, ps.count, st));
    }
    if (f.natural) {
      for (int z = 0; z < ps.count; ++z) {
        PermArgs pa{};
        pa.src = scratch + z * (long long)n_entries * N;
        pa.dst = out + z * out_ps;
        pa.N = N; pa.np = np; pa.to_natural = 1; pa.entries = n_entries;
        for (int j = 0; j < np; ++j) pa.bits[j] = bits[j];
        FPM_CUDA_TRY(launch_pdl(big_perm_kernel, dim3(148 * 8), dim3(256), 0, st, pa));
        FPM_LAUNCH_CHECK();
      }
    }
    return kOk;
  };
  if (f.pm) {
    set_last_error("long transforms produce the blocked layout only");
    return kUnsupported;
  }
  FPM_TRY(one(f.in, f.in_stride, f.in_prime_stride, f.n_entries, f.out, f.out_prime_stride));
  if (f.n_entries2 > 0)
    FPM_TRY(one(f.in2, f.in2_stride, f.in2_prime_stride, f.n_entries2, f.out2,
                f.out2_prime_stride));
  return kOk;
}

int launch_ntt_inv_big(Context& cx, int logn, const NttInvArgs& v, const PrimeSet& ps,
                       uint32_t* scratch, cudaStream_t st) {
  if (v.n_entries <= 0) return kOk;
  if (v.pm) {
    set_last_error("long transforms take the blocked layout only");
    return kUnsupported;
  }
  if (v.n_entries > 65535) {
    set_last_error("long transforms: %d entries exceed one grid dimension", v.n_entries);
    return kUnsupported;
  }
  int np, bits[4];
  split_bits(logn, &np, bits);
  const long long N = 1LL << logn;
  const long long sps = (long long)v.n_entries * N;
  BigArgs a{};
  a.logn = logn;
  a.inverse = 1;
  a.n_entries = v.n_entries;
  FPM_TRY(fill_primes(cx, logn, ps, true, a));
  if (v.natural) {
    for (int z = 0; z < ps.count; ++z) {
      PermArgs pa{};
      pa.src = v.in + z * v.in_prime_stride;
      pa.dst = scratch + z * sps;
      pa.N = N; pa.np = np; pa.to_natural = 0; pa.entries = v.n_entries;
      for (int j = 0; j < np; ++j) pa.bits[j] = bits[j];
      FPM_CUDA_TRY(launch_pdl(big_perm_kernel, dim3(148 * 8), dim3(256), 0, st, pa));
      FPM_LAUNCH_CHECK();
    }
  }
  a.out = v.out; a.out_stride = v.out_stride; a.out_prime_stride = v.out_prime_stride;
  a.out_len = v.out_len; a.off = v.off; a.scale = v.scale;
  for (int j = np - 1; j >= 0; --j) {
    const bool first = j == np - 1, last = j == 0;
    a.in_kind = first && !v.natural ? 2 : 0;
    a.src = a.in_kind == 2 ? v.in : scratch;
    a.src_ps = a.in_kind == 2 ? v.in_prime_stride : sps;
    a.out_kind = last ? 1 : 0;
    a.dst = scratch;
    a.dst_ps = sps;
    FPM_TRY(run_pass(a, j, np, bits, ps.count, st));
  }
  return kOk;
}

// ---- plan: split twiddle tables and the inner 1024-point roots ----------
int Context::big_plan(uint32_t p, int logn, const BigPlan** out) {
  std::lock_guard<std::mutex> lk(mu_);
  auto key = std::make_pair(p, logn);
  auto it = big_plans_.find(key);
  if (it != big_plans_.end()) {
    *out = &it->second;
    return kOk;
  }
  const int k = h_two_adicity(p);
  if (logn > k || logn < 10) {
    set_last_error("p=%u: no long transform of length 2^%d", p, logn);
    return kOrderTooSmall;
  }
  const uint64_t N = 1ull << logn;
  const uint64_t omega = h_powmod(h_ntt_root(p), 1ull << (k - logn), p);
  const uint64_t iomega = h_invmod(omega, p);
  BigPlan bp;
  bp.p = p;
  bp.h = (logn + 1) / 2;
  const size_t nlo = (size_t)1 << bp.h, nhi = (size_t)(N >> bp.h);
  auto table = [&](uint64_t base, size_t cnt, uint2** dst) -> int {
    std::vector<uint2> t(cnt);
    uint64_t w = 1;
    for (size_t i = 0; i < cnt; ++i) {
      t[i] = make_uint2((uint32_t)w, h_shoup((uint32_t)w, p));
      w = h_mulmod(w, base, p);
    }
    FPM_CUDA_TRY(cudaMalloc(dst, cnt * sizeof(uint2)));
    FPM_CUDA_TRY(cudaMemcpy(*dst, t.data(), cnt * sizeof(uint2), cudaMemcpyHostToDevice));
    return kOk;
  };
  FPM_TRY(table(omega, nlo, &bp.lo));
  FPM_TRY(table(h_powmod(omega, nlo, p), nhi, &bp.hi));
  FPM_TRY(table(iomega, nlo, &bp.ilo));
  FPM_TRY(table(h_powmod(iomega, nlo, p), nhi, &bp.ihi));
  FPM_TRY(table(h_powmod(omega, N / 1024, p), 512, &bp.r1k));
  FPM_TRY(table(h_powmod(iomega, N / 1024, p), 512, &bp.ir1k));
  bp.ninv = (uint32_t)h_invmod(N % p, p);
  bp.ninv_sh = h_shoup(bp.ninv, p);
  auto res = big_plans_.emplace(key, bp);
  *out = &res.first->second;
  return kOk;
}

}  // namespace fpm
