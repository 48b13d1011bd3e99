// crt.cu -- Garner CRT, generic-modulus middle product, degree helpers.
#include "crt.cuh"
#include <algorithm>
#include <climits>

namespace fpm {

__device__ __forceinline__ uint64_t d_montmul(uint64_t a, uint64_t b, uint64_t P, uint64_t Pni) {
  // (a*b + m*P) / 2^64 with m = -a*b*P^-1 mod 2^64; a*b < 2^64 * P required
  const uint64_t lo = a * b, hi = __umul64hi(a, b);
  const uint64_t m = lo * Pni;
  const uint64_t mh = __umul64hi(m, P);
  uint64_t r = hi + mh + (lo != 0);
  r = r >= P ? r - P : r;
  return r >= P ? r - P : r;
}
__device__ __forceinline__ uint64_t d_mulmod_any(uint64_t a, uint64_t b, uint64_t P,
                                                 uint64_t Pni, uint64_t R2) {
  return d_montmul(d_montmul(a, R2, P, Pni), b, P, Pni);
}
__device__ __forceinline__ uint64_t d_addmod64(uint64_t a, uint64_t b, uint64_t P) {
  const uint64_t s = a + b;  // P < 2^62
  return s >= P ? s - P : s;
}

namespace {

// Garner over R primes, then X mod P = REDC(sum_i v_i Mmont_i): the 32 x 64
// products are summed as one 128-bit value (< 8 * 2^31 * P < P 2^64) and
// reduced once (Mmont_i = (prod_{j<i} q_j mod P) 2^64 mod P), instead of a
// 64-bit Montgomery product per prime
template <int R, typename I>
__global__ void __launch_bounds__(256) crt_kernel(CrtArgs a) {
  pdl_wait();
  // I = uint32_t when the index space fits: a 64-bit division per output
  // is a long software sequence
  const I total = (I)a.n_entries * (I)a.len, len = (I)a.len;
  for (I idx = blockIdx.x * (I)blockDim.x + threadIdx.x; idx < total;
       idx += (I)gridDim.x * blockDim.x) {
    const I e = idx / len;
    const int t = (int)(idx - e * len);
    const uint32_t* src = a.res + e * a.res_stride + t;
    uint32_t x0[R];
#pragma unroll
    for (int i = 0; i < R; ++i) x0[i] = src[i * a.res_prime_stride];  // loads first
    uint32_t v[R];
    uint64_t lo = 0, hi = 0;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const uint32_t qi = a.q[i];
      uint32_t x = x0[i];
#pragma unroll
      for (int j = 0; j < i; ++j) {
        const uint32_t vj = v[j] >= qi ? v[j] - qi : v[j];
        x = x - vj + qi;  // [1, 2 qi)
        x = d_red(d_shoup(x, a.g[j][i], a.gsh[j][i], qi), qi);
      }
      v[i] = x;
      const uint64_t M = a.Mmont[i];
      const uint64_t p0 = (uint64_t)x * (uint32_t)M;
      const uint64_t p1 = (uint64_t)x * (uint32_t)(M >> 32);
      lo += p0;
      hi += lo < p0;
      const uint64_t s1 = p1 << 32;
      lo += s1;
      hi += (lo < s1) + (p1 >> 32);
    }
    const uint64_t mq = lo * a.Pni;
    uint64_t s = hi + __umul64hi(mq, a.P) + (lo != 0);
    s = s >= a.P ? s - a.P : s;
    if (a.out64)
      ((uint64_t*)a.out)[e * a.out_stride + t] = s;
    else
      ((uint32_t*)a.out)[e * a.out_stride + t] = (uint32_t)s;
  }
}

template <typename T>
__device__ __forceinline__ int trimmed_len(const T* e, int L) {
  while (L > 0 && e[L - 1] == 0) --L;
  return L;
}

template <typename Tin, typename Tout>
__global__ void middle_entrywise_kernel(MiddleEntryArgs a) {
  pdl_wait();
  const Tin* A = (const Tin*)a.A;
  const Tin* B = (const Tin*)a.B;
  Tout* out = (Tout*)a.out;
  const long long total = (long long)a.m * a.n * a.d;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long ij = idx / a.d;
    const int tt = (int)(idx - ij * a.d);
    const int i = (int)(ij / a.n), j = (int)(ij - (long long)i * a.n);
    const long long t = a.c + tt;
    uint64_t acc = 0;
    for (int l = 0; l < a.k; ++l) {
      const Tin* ae = A + ((long long)i * a.k + l) * a.la;
      const Tin* be = B + ((long long)l * a.n + j) * a.lb;
      const int la = trimmed_len(ae, a.la), lb = trimmed_len(be, a.lb);
      if (la == 0 || lb == 0) continue;
      const long long lad = (long long)la * a.d;
      bool cyclic = false;
      long long Ne = 0;
      if (!(lad <= 64 * 64 / 4 && lad <= 16384)) {
        const long long need = (long long)la + a.d;
        int lg = 0;
        while ((1LL << lg) < need) ++lg;  // max(1, (need-1).bit_length())
        if (lg < 1) lg = 1;
        if (lg <= a.two_adicity) { cyclic = true; Ne = 1LL << lg; }
      }
      if (!cyclic) {
        // exact coefficient t of a*b (schoolbook or full-product slice)
        long long lo = t - lb + 1 > 0 ? t - lb + 1 : 0;
        long long hi = la - 1 < t ? la - 1 : t;
        for (long long u = lo; u <= hi; ++u)
          acc = d_addmod64(acc, d_mulmod_any((uint64_t)ae[u], (uint64_t)be[t - u], a.P, a.Pni, a.R2), a.P);
      } else {
        // cyclic fold mod x^Ne - 1 (upoly.py:366-374): sum a_u b_w, u+w = t mod Ne
        const long long tm = t % Ne;
        for (int u = 0; u < la; ++u) {
          long long w0 = tm - u;
          w0 %= Ne;
          if (w0 < 0) w0 += Ne;
          for (long long w = w0; w < lb; w += Ne)
            acc = d_addmod64(acc, d_mulmod_any((uint64_t)ae[u], (uint64_t)be[w], a.P, a.Pni, a.R2), a.P);
        }
      }
    }
    out[ij * a.d + tt] = (Tout)acc;
  }
}

// max over entries of the trimmed length: one warp per entry scans 128-value
// chunks from the end (coalesced, 4 loads in flight) and stops at the first
// chunk holding a nonzero coefficient
template <typename T>
__global__ void max_len_kernel(const T* M, long long entries, int L, int* out) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  int best = 0;
  for (long long e = w0; e < entries; e += nw) {
    const T* row = M + e * L;
    for (int hi = L; hi > best; hi -= 128) {
      T v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int t = hi - 128 + 32 * q + lane;
        v[q] = t >= 0 && t < hi ? row[t] : (T)0;
      }
      int found = 0;
#pragma unroll
      for (int q = 3; q >= 0; --q) {
        const unsigned bal = __ballot_sync(0xffffffffu, v[q] != 0);
        if (!found && bal) found = hi - 128 + 32 * q + 32 - __clz(bal);
      }
      if (found) {
        best = max(best, found);
        break;
      }
    }
  }
  if (lane == 0 && best > 0) atomicMax(out, best);
}

template <typename T>
__global__ void rdeg_kernel(const T* M, int rows, int cols, int L, const int64_t* s, int64_t* out) {
  pdl_wait();
  // one warp per row
  const int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  long long best = LLONG_MIN, smin = LLONG_MAX;
  for (int j = lane; j < cols; j += 32) {
    smin = min(smin, (long long)s[j]);
    const int l = trimmed_len(M + ((long long)row * cols + j) * L, L);
    if (l > 0) best = max(best, (long long)(l - 1) + (long long)s[j]);
  }
  for (int o = 16; o; o >>= 1) {
    best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    smin = min(smin, __shfl_xor_sync(0xffffffffu, smin, o));
  }
  if (lane == 0) out[row] = best == LLONG_MIN ? smin : best;
}

// generic radix-2 NTT over any odd p < 2^62 (u64, Montgomery products):
// bit-reversal copy, then log N global passes of DIT butterflies; twiddle
// w^e = lo[e & mask] * hi[e >> h] (split table, normal form)
__global__ void ntt64_bitrev_kernel(const uint64_t* in, uint64_t* out, int logn, long long batch) {
  pdl_wait();
  const long long N = 1LL << logn, total = batch * N;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long b = idx >> logn, j = idx & (N - 1);
    const long long r = logn ? (long long)(__brevll((unsigned long long)j) >> (64 - logn)) : 0;
    out[(b << logn) + r] = in[idx];
  }
}

__global__ void ntt64_stage_kernel(uint64_t* x, int logn, int hb, long long batch, uint64_t P,
                                   uint64_t Pni, uint64_t R2, const uint64_t* lo,
                                   const uint64_t* hi, int h, uint64_t scale, int last) {
  pdl_wait();
  const long long N = 1LL << logn, half = N >> 1, total = batch * half;
  const long long hh = 1LL << hb;
  const long long mask = (1LL << h) - 1;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long b = idx / half, q = idx - b * half;
    const long long i = q & (hh - 1), g = q >> hb;
    const long long u = (b << logn) + g * 2 * hh + i, v = u + hh;
    const long long e = i << (logn - 1 - hb);  // w_{2hh}^i = w_N^(i N / 2hh)
    uint64_t t = x[v];
    if (e) {
      const uint64_t w = d_mulmod_any(lo[e & mask], hi[e >> h], P, Pni, R2);
      t = d_mulmod_any(t, w, P, Pni, R2);
    }
    const uint64_t s = x[u];
    uint64_t a0 = d_addmod64(s, t, P), a1 = d_addmod64(s, P - t, P);
    if (last && scale != 1) {
      a0 = d_mulmod_any(a0, scale, P, Pni, R2);
      a1 = d_mulmod_any(a1, scale, P, Pni, R2);
    }
    x[u] = a0;
    x[v] = a1;
  }
}

}  // namespace

int launch_ntt64_generic(uint64_t p, uint64_t omega, int logn, int batch, const uint64_t* in,
                         uint64_t* out, uint64_t scale, const uint64_t* lo, const uint64_t* hi,
                         int h, cudaStream_t st) {
  const long long N = 1LL << logn, total = (long long)batch * N;
  if (total <= 0) return kOk;
  CrtArgs tmp{};
  const uint32_t q1 = 2013265921u;
  crt_prepare(tmp, &q1, 1, p);
  const u128 R = ((u128)1 << 64) % p;
  const uint64_t R2 = (uint64_t)(R * R % p);
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  FPM_CUDA_TRY(launch_pdl(ntt64_bitrev_kernel, dim3((unsigned)blocks), dim3(256), 0, st, in, out,
                          logn, (long long)batch));
  FPM_LAUNCH_CHECK();
  if (logn == 0 && scale != 1) {
    set_last_error("internal: length-1 inverse");  // N^-1 = 1: never reached
    return kInvalidArgument;
  }
  for (int hb = 0; hb < logn; ++hb) {
    FPM_CUDA_TRY(launch_pdl(ntt64_stage_kernel, dim3((unsigned)blocks), dim3(256), 0, st, out,
                            logn, hb, (long long)batch, p, tmp.Pni, R2, lo, hi, h, scale,
                            hb == logn - 1 ? 1 : 0));
    FPM_LAUNCH_CHECK();
  }
  (void)omega;
  return kOk;
}

void crt_prepare(CrtArgs& a, const uint32_t* q, int r, uint64_t P) {
  // the constants depend on (q, P) only: the last set is reused (per thread)
  thread_local CrtArgs last{};
  thread_local bool have = false;
  if (have && last.r == r && last.P == P && std::equal(q, q + r, last.q)) {
    a.r = r;
    a.P = P;
    a.Pni = last.Pni;
    std::copy(last.q, last.q + kMaxPrimes, a.q);
    std::copy(&last.g[0][0], &last.g[0][0] + kMaxPrimes * kMaxPrimes, &a.g[0][0]);
    std::copy(&last.gsh[0][0], &last.gsh[0][0] + kMaxPrimes * kMaxPrimes, &a.gsh[0][0]);
    std::copy(last.Mmont, last.Mmont + kMaxPrimes, a.Mmont);
    return;
  }
  a.r = r;
  for (int i = 0; i < r; ++i) a.q[i] = q[i];
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < i; ++j) {
      const uint32_t inv = (uint32_t)h_invmod(q[j] % q[i], q[i]);
      a.g[j][i] = inv;
      a.gsh[j][i] = h_shoup(inv, q[i]);
    }
  a.P = P;
  // -P^-1 mod 2^64 by Newton iteration
  uint64_t inv = P;  // correct to 3 bits for odd P
  for (int it = 0; it < 6; ++it) inv *= 2 - P * inv;
  a.Pni = (uint64_t)0 - inv;
  uint64_t prod = 1 % P;
  const u128 R = ((u128)1 << 64) % P;
  for (int i = 0; i < r; ++i) {
    a.Mmont[i] = (uint64_t)((u128)prod * R % P);
    prod = h_mulmod(prod, q[i] % P, P);
  }
  last = a;
  have = true;
}

template <int R>
int launch_crt_r(const CrtArgs& a, long long total, cudaStream_t st) {
  // one resident wave (grid-stride loop): no partial last wave
  static int per_sm = 0, sms = 0;
  if (!per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, crt_kernel<R, uint32_t>, 256, 0);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    if (per_sm < 1) per_sm = 1;
    if (sms < 1) sms = 148;
  }
  long long blocks = (total + 255) / 256;
  if (blocks > (long long)per_sm * sms) blocks = (long long)per_sm * sms;
  if (total + (long long)blocks * 256 < (1LL << 32))
    FPM_CUDA_TRY(launch_pdl(crt_kernel<R, uint32_t>, dim3((unsigned)blocks), dim3(256), 0, st, a));
  else
    FPM_CUDA_TRY(launch_pdl(crt_kernel<R, unsigned long long>, dim3((unsigned)blocks), dim3(256), 0, st, a));
  FPM_LAUNCH_CHECK();
  return kOk;
}

int launch_crt(const CrtArgs& a, cudaStream_t st) {
  const long long total = (long long)a.n_entries * a.len;
  if (total <= 0) return kOk;
  static_assert(kMaxPrimes == 8, "crt_kernel instantiations");
  switch (a.r) {
    case 1: return launch_crt_r<1>(a, total, st);
    case 2: return launch_crt_r<2>(a, total, st);
    case 3: return launch_crt_r<3>(a, total, st);
    case 4: return launch_crt_r<4>(a, total, st);
    case 5: return launch_crt_r<5>(a, total, st);
    case 6: return launch_crt_r<6>(a, total, st);
    case 7: return launch_crt_r<7>(a, total, st);
    case 8: return launch_crt_r<8>(a, total, st);
  }
  set_last_error("CRT over %d primes (1..%d supported)", a.r, kMaxPrimes);
  return kInvalidArgument;
}

int launch_middle_entrywise(const MiddleEntryArgs& a, cudaStream_t st) {
  const long long total = (long long)a.m * a.n * a.d;
  if (total <= 0) return kOk;
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (a.in64 && a.out64)
    FPM_CUDA_TRY(launch_pdl(middle_entrywise_kernel<uint64_t, uint64_t>, dim3((unsigned)blocks), dim3(256), 0, st, a));
  else if (!a.in64 && !a.out64)
    FPM_CUDA_TRY(launch_pdl(middle_entrywise_kernel<uint32_t, uint32_t>, dim3((unsigned)blocks), dim3(256), 0, st, a));
  else {
    set_last_error("middle_entrywise: mixed element widths unsupported");
    return kInvalidArgument;
  }
  FPM_LAUNCH_CHECK();
  return kOk;
}

int launch_max_len(const void* M, int in64, long long entries, int L, int* out, cudaStream_t st) {
  FPM_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(int), st));
  if (entries <= 0 || L <= 0) return kOk;
  long long blocks = (entries * 32 + 255) / 256;  // one warp per entry
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (in64)
    FPM_CUDA_TRY(launch_pdl(max_len_kernel<uint64_t>, dim3((unsigned)blocks), dim3(256), 0, st, (const uint64_t*)M, entries, L, out));
  else
    FPM_CUDA_TRY(launch_pdl(max_len_kernel<uint32_t>, dim3((unsigned)blocks), dim3(256), 0, st, (const uint32_t*)M, entries, L, out));
  FPM_LAUNCH_CHECK();
  return kOk;
}

int launch_rdeg(const void* M, int in64, int rows, int cols, int L, const int64_t* s,
                int64_t* out, cudaStream_t st) {
  if (rows <= 0) return kOk;
  const int wpb = 8;
  const unsigned blocks = (unsigned)((rows + wpb - 1) / wpb);
  if (in64)
    FPM_CUDA_TRY(launch_pdl(rdeg_kernel<uint64_t>, dim3(blocks), dim3(wpb * 32), 0, st, (const uint64_t*)M, rows, cols, L, s, out));
  else
    FPM_CUDA_TRY(launch_pdl(rdeg_kernel<uint32_t>, dim3(blocks), dim3(wpb * 32), 0, st, (const uint32_t*)M, rows, cols, L, s, out));
  FPM_LAUNCH_CHECK();
  return kOk;
}

}  // namespace fpm
