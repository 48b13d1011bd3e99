// ntt.cu -- batched NTT kernels; see ntt.cuh for the design summary.
#include "ntt.cuh"

namespace fpm {
namespace {

template <int LOGN>
struct Geo {
  static constexpr int N = 1 << LOGN;
  static constexpr int TPT = N / 32;                       // threads per transform
  static constexpr int TPC = N >= 8192 ? 1 : 8192 / N;     // transforms per CTA
  static constexpr int THREADS = TPT * TPC;                // 256 (N<=8192), 512, 1024
  static constexpr int NPASS = (LOGN + 4) / 5;             // 1, 2 or 3 passes
  static constexpr int LAST_R = LOGN - 5 * (NPASS - 1);    // bits of the last pass
  static constexpr int STRIDE = N + N / 32;                // padded smem words / transform
  static constexpr int SMEM_BYTES = TPC * STRIDE * 4;
};

// Pass maps: thread-local element i (0..31) of local thread lt -> index x.
enum { MAP_TOP = 0, MAP_MID = 1, MAP_LAST = 2 };

template <int LOGN, int MAP>
__device__ __forceinline__ int xmap(int lt, int i) {
  if (MAP == MAP_TOP) return lt + (i << (LOGN - 5));
  if (MAP == MAP_MID) {
    constexpr int lo = LOGN - 10;
    return ((lt >> lo) << (LOGN - 5)) | (i << lo) | (lt & ((1 << lo) - 1));
  }
  return (lt << 5) | i;
}
template <int LOGN, int MAP>
struct PassBits {
  static constexpr int BB = MAP == MAP_TOP ? LOGN - 5 : (MAP == MAP_MID ? LOGN - 10 : 0);
  static constexpr int R = MAP == MAP_LAST ? Geo<LOGN>::LAST_R : 5;
};
// runtime part of the twiddle exponent (x mod 2^b) << (LOGN-1-b) for stage bit b
template <int LOGN, int MAP>
__device__ __forceinline__ int tw_base(int lt, int b) {
  const int sh = LOGN - 1 - b;
  if (MAP == MAP_TOP) return lt << sh;
  if (MAP == MAP_MID) {
    constexpr int lo = LOGN - 10;
    return (lt & ((1 << lo) - 1)) << sh;
  }
  return 0;
}

__device__ __forceinline__ int pad(int x) { return x + (x >> 5); }

// Gentleman-Sande pass over the pass's active bits, high to low.
template <int LOGN, int MAP>
__device__ __forceinline__ void dif_pass(uint32_t (&v)[32], int lt,
                                         const uint2* __restrict__ tw, uint32_t p) {
  constexpr int BB = PassBits<LOGN, MAP>::BB, R = PassBits<LOGN, MAP>::R;
#pragma unroll
  for (int ib = R - 1; ib >= 0; --ib) {
    const int b = BB + ib;
    const uint2* twb = tw + tw_base<LOGN, MAP>(lt, b);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (i & (1 << ib)) continue;
      const int j = i | (1 << ib);
      const uint32_t u = v[i], w = v[j];
      const uint32_t s = d_red(u + w, p);
      uint32_t d = u - w + p;  // [1, 2p)
      if (b != 0) {
        const uint2 t = __ldg(twb + ((i & ((1 << ib) - 1)) << (LOGN - 1 - ib)));
        d = d_shoup(d, t.x, t.y, p);
      }
      v[i] = s;
      v[j] = d_red(d, p);
    }
  }
}

// Cooley-Tukey pass over the pass's active bits, low to high (inverse table).
template <int LOGN, int MAP>
__device__ __forceinline__ void dit_pass(uint32_t (&v)[32], int lt,
                                         const uint2* __restrict__ itw, uint32_t p) {
  constexpr int BB = PassBits<LOGN, MAP>::BB, R = PassBits<LOGN, MAP>::R;
#pragma unroll
  for (int ib = 0; ib < R; ++ib) {
    const int b = BB + ib;
    const uint2* twb = itw + tw_base<LOGN, MAP>(lt, b);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (i & (1 << ib)) continue;
      const int j = i | (1 << ib);
      const uint32_t u = v[i];
      uint32_t t = v[j];
      if (b != 0) {
        const uint2 w = __ldg(twb + ((i & ((1 << ib) - 1)) << (LOGN - 1 - ib)));
        t = d_red(d_shoup(t, w.x, w.y, p), p);
      }
      v[i] = d_red(u + t, p);
      v[j] = d_red(u - t + p, p);
    }
  }
}

template <int LOGN, int MAP>
__device__ __forceinline__ void to_smem(uint32_t* smt, const uint32_t (&v)[32], int lt) {
#pragma unroll
  for (int i = 0; i < 32; ++i) smt[pad(xmap<LOGN, MAP>(lt, i))] = v[i];
}
template <int LOGN, int MAP>
__device__ __forceinline__ void from_smem(const uint32_t* smt, uint32_t (&v)[32], int lt) {
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = smt[pad(xmap<LOGN, MAP>(lt, i))];
}

__device__ __forceinline__ uint32_t reduce_in(uint64_t raw, bool reduce, const PrimeConst& pc) {
  if (!reduce) return (uint32_t)raw;
  return d_red64(raw, pc.p, pc.mu);
}

// coefficient x of entry e (zero padded, optionally folded / reduced)
__device__ __forceinline__ uint32_t load_coef(const NttFwdArgs& a, const PrimeConst& pc,
                                              long long ebase, int x, int N) {
  if (!a.fold) {
    if (x >= a.len) return 0;
    uint64_t raw = a.in64 ? __ldg((const unsigned long long*)a.in + ebase + x)
                          : (uint64_t)__ldg((const uint32_t*)a.in + ebase + x);
    return reduce_in(raw, a.reduce, pc);
  }
  uint32_t acc = 0;
  for (int t = x; t < a.len; t += N) {
    uint64_t raw = a.in64 ? __ldg((const unsigned long long*)a.in + ebase + t)
                          : (uint64_t)__ldg((const uint32_t*)a.in + ebase + t);
    uint32_t r = a.reduce ? reduce_in(raw, true, pc) : (uint32_t)raw;
    acc = d_red(acc + r, pc.p);
  }
  return acc;
}

template <int LOGN>
__global__ void __launch_bounds__(Geo<LOGN>::THREADS)
    ntt_fwd_kernel(NttFwdArgs a, PrimeSet ps) {
  using G = Geo<LOGN>;
  extern __shared__ uint32_t sm[];
  const PrimeConst& pc = ps.pr[blockIdx.z];
  const uint32_t p = pc.p;
  const int tid = threadIdx.x;
  const int tr = tid / G::TPT, lt = tid % G::TPT;
  const long long e0 = (long long)blockIdx.x * G::TPC;
  const long long e = e0 + tr;
  const bool valid = e < a.n_entries;
  uint32_t* smt = sm + tr * G::STRIDE;
  const long long pin = (long long)blockIdx.z * a.in_prime_stride;
  uint32_t v[32];

  constexpr int FIRST = G::NPASS == 1 ? MAP_LAST : MAP_TOP;
  if (G::TPT >= 32) {
    // direct coalesced load: consecutive lanes read consecutive coefficients
    const long long eb = pin + e * a.in_stride;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      v[i] = valid ? load_coef(a, pc, eb, xmap<LOGN, FIRST>(lt, i), G::N) : 0u;
  } else {
    // small N: cooperative coalesced load of TPC transforms through smem
    for (int idx = tid; idx < G::TPC * G::N; idx += G::THREADS) {
      const int t2 = idx >> LOGN, x = idx & (G::N - 1);
      const long long e2 = e0 + t2;
      uint32_t val = e2 < a.n_entries ? load_coef(a, pc, pin + e2 * a.in_stride, x, G::N) : 0u;
      sm[t2 * G::STRIDE + pad(x)] = val;
    }
    __syncthreads();
    from_smem<LOGN, FIRST>(smt, v, lt);
  }

  if (G::NPASS == 1) {
    dif_pass<LOGN, MAP_LAST>(v, lt, pc.tw, p);
  } else if (G::NPASS == 2) {
    dif_pass<LOGN, MAP_TOP>(v, lt, pc.tw, p);
    __syncthreads();
    to_smem<LOGN, MAP_TOP>(smt, v, lt);
    __syncthreads();
    from_smem<LOGN, MAP_LAST>(smt, v, lt);
    dif_pass<LOGN, MAP_LAST>(v, lt, pc.tw, p);
  } else {
    dif_pass<LOGN, MAP_TOP>(v, lt, pc.tw, p);
    __syncthreads();
    to_smem<LOGN, MAP_TOP>(smt, v, lt);
    __syncthreads();
    from_smem<LOGN, MAP_MID>(smt, v, lt);
    dif_pass<LOGN, MAP_MID>(v, lt, pc.tw, p);
    __syncthreads();
    to_smem<LOGN, MAP_MID>(smt, v, lt);
    __syncthreads();
    from_smem<LOGN, MAP_LAST>(smt, v, lt);
    dif_pass<LOGN, MAP_LAST>(v, lt, pc.tw, p);
  }
  if (!valid) return;
  uint32_t* out = a.out + (long long)blockIdx.z * a.out_prime_stride;
  if (a.natural) {
    // public ntt_forward order: out[k] = F(w^k), k = bitrev(x)
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int x = xmap<LOGN, MAP_LAST>(lt, i);
      const int k = __brev(x) >> (32 - LOGN);
      out[e * G::N + k] = v[i];
    }
  } else {
    // eval layout: this thread owns point block lt (x = 32*lt + i)
    uint4* dst = reinterpret_cast<uint4*>(out + ((long long)lt * a.n_entries + e) * 32);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      dst[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  }
}

template <int LOGN>
__global__ void __launch_bounds__(Geo<LOGN>::THREADS)
    ntt_inv_kernel(NttInvArgs a, PrimeSet ps) {
  using G = Geo<LOGN>;
  extern __shared__ uint32_t sm[];
  const PrimeConst& pc = ps.pr[blockIdx.z];
  const uint32_t p = pc.p;
  const int tid = threadIdx.x;
  const int tr = tid / G::TPT, lt = tid % G::TPT;
  const long long e0 = (long long)blockIdx.x * G::TPC;
  const long long e = e0 + tr;
  const bool valid = e < a.n_entries;
  uint32_t* smt = sm + tr * G::STRIDE;
  const uint32_t* in = a.in + (long long)blockIdx.z * a.in_prime_stride;
  uint32_t v[32];

  if (a.natural) {
    // public ntt_inverse: value at DIT position x is input[bitrev(x)]
    for (int idx = tid; idx < G::TPC * G::N; idx += G::THREADS) {
      const int t2 = idx >> LOGN, k = idx & (G::N - 1);
      const long long e2 = e0 + t2;
      const int x = __brev(k) >> (32 - LOGN);
      sm[t2 * G::STRIDE + pad(x)] = e2 < a.n_entries ? in[e2 * G::N + k] : 0u;
    }
    __syncthreads();
    from_smem<LOGN, MAP_LAST>(smt, v, lt);
  } else if (valid) {
    const uint4* src = reinterpret_cast<const uint4*>(in + ((long long)lt * a.n_entries + e) * 32);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint4 t = __ldg(src + q);
      v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = 0;
  }

  constexpr int FINAL = G::NPASS == 1 ? MAP_LAST : MAP_TOP;
  if (G::NPASS == 1) {
    dit_pass<LOGN, MAP_LAST>(v, lt, pc.itw, p);
  } else if (G::NPASS == 2) {
    dit_pass<LOGN, MAP_LAST>(v, lt, pc.itw, p);
    __syncthreads();
    to_smem<LOGN, MAP_LAST>(smt, v, lt);
    __syncthreads();
    from_smem<LOGN, MAP_TOP>(smt, v, lt);
    dit_pass<LOGN, MAP_TOP>(v, lt, pc.itw, p);
  } else {
    dit_pass<LOGN, MAP_LAST>(v, lt, pc.itw, p);
    __syncthreads();
    to_smem<LOGN, MAP_LAST>(smt, v, lt);
    __syncthreads();
    from_smem<LOGN, MAP_MID>(smt, v, lt);
    dit_pass<LOGN, MAP_MID>(v, lt, pc.itw, p);
    __syncthreads();
    to_smem<LOGN, MAP_MID>(smt, v, lt);
    __syncthreads();
    from_smem<LOGN, MAP_TOP>(smt, v, lt);
    dit_pass<LOGN, MAP_TOP>(v, lt, pc.itw, p);
  }
  if (a.scale) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = d_red(d_shoup(v[i], pc.ninv, pc.ninv_sh, p), p);
  }
  uint32_t* out = a.out + (long long)blockIdx.z * a.out_prime_stride;
  if (a.natural) {
    if (!valid) return;
#pragma unroll
    for (int i = 0; i < 32; ++i) out[e * G::N + xmap<LOGN, FINAL>(lt, i)] = v[i];
    return;
  }
  if (G::TPT >= 32) {
    if (!valid) return;
    uint32_t* oe = out + e * a.out_stride;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int t = (xmap<LOGN, FINAL>(lt, i) - a.off) & (G::N - 1);
      if (t < a.out_len) oe[t] = v[i];
    }
  } else {
    // small N: stage through smem, then a coalesced cooperative store
    __syncthreads();
    to_smem<LOGN, FINAL>(smt, v, lt);
    __syncthreads();
    const int ol = a.out_len < G::N ? a.out_len : G::N;
    for (int idx = tid; idx < G::TPC * ol; idx += G::THREADS) {
      const int t2 = idx / ol, t = idx - t2 * ol;
      const long long e2 = e0 + t2;
      if (e2 < a.n_entries) {
        const int x = (t + a.off) & (G::N - 1);
        out[e2 * a.out_stride + t] = sm[t2 * G::STRIDE + pad(x)];
      }
    }
  }
}

template <int LOGN>
int fwd_impl(const NttFwdArgs& a, const PrimeSet& ps, cudaStream_t st) {
  using G = Geo<LOGN>;
  if (G::SMEM_BYTES > 48 * 1024) {
    static bool once = false;
    if (!once) {
      FPM_CUDA_TRY(cudaFuncSetAttribute(ntt_fwd_kernel<LOGN>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        G::SMEM_BYTES));
      once = true;
    }
  }
  dim3 grid((unsigned)((a.n_entries + G::TPC - 1) / G::TPC), 1, (unsigned)ps.count);
  ntt_fwd_kernel<LOGN><<<grid, G::THREADS, G::SMEM_BYTES, st>>>(a, ps);
  FPM_LAUNCH_CHECK();
  return kOk;
}

template <int LOGN>
int inv_impl(const NttInvArgs& a, const PrimeSet& ps, cudaStream_t st) {
  using G = Geo<LOGN>;
  if (G::SMEM_BYTES > 48 * 1024) {
    static bool once = false;
    if (!once) {
      FPM_CUDA_TRY(cudaFuncSetAttribute(ntt_inv_kernel<LOGN>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        G::SMEM_BYTES));
      once = true;
    }
  }
  dim3 grid((unsigned)((a.n_entries + G::TPC - 1) / G::TPC), 1, (unsigned)ps.count);
  ntt_inv_kernel<LOGN><<<grid, G::THREADS, G::SMEM_BYTES, st>>>(a, ps);
  FPM_LAUNCH_CHECK();
  return kOk;
}

}  // namespace

int launch_ntt_fwd(int logn, const NttFwdArgs& a, const PrimeSet& ps, cudaStream_t st) {
  if (a.n_entries <= 0) return kOk;
  switch (logn) {
    case 5: return fwd_impl<5>(a, ps, st);
    case 6: return fwd_impl<6>(a, ps, st);
    case 7: return fwd_impl<7>(a, ps, st);
    case 8: return fwd_impl<8>(a, ps, st);
    case 9: return fwd_impl<9>(a, ps, st);
    case 10: return fwd_impl<10>(a, ps, st);
    case 11: return fwd_impl<11>(a, ps, st);
    case 12: return fwd_impl<12>(a, ps, st);
    case 13: return fwd_impl<13>(a, ps, st);
    case 14: return fwd_impl<14>(a, ps, st);
    case 15: return fwd_impl<15>(a, ps, st);
  }
  set_last_error("NTT length 2^%d outside the supported range [2^5, 2^15]", logn);
  return kUnsupported;
}

int launch_ntt_inv(int logn, const NttInvArgs& a, const PrimeSet& ps, cudaStream_t st) {
  if (a.n_entries <= 0) return kOk;
  switch (logn) {
    case 5: return inv_impl<5>(a, ps, st);
    case 6: return inv_impl<6>(a, ps, st);
    case 7: return inv_impl<7>(a, ps, st);
    case 8: return inv_impl<8>(a, ps, st);
    case 9: return inv_impl<9>(a, ps, st);
    case 10: return inv_impl<10>(a, ps, st);
    case 11: return inv_impl<11>(a, ps, st);
    case 12: return inv_impl<12>(a, ps, st);
    case 13: return inv_impl<13>(a, ps, st);
    case 14: return inv_impl<14>(a, ps, st);
    case 15: return inv_impl<15>(a, ps, st);
  }
  set_last_error("NTT length 2^%d outside the supported range [2^5, 2^15]", logn);
  return kUnsupported;
}

}  // namespace fpm
