// ntt.cu -- batched NTT kernels; see ntt.cuh for the design summary.
//
// Four-step radix-32 formulation.  A length-N DIF transform is split into
// passes over 5-bit digits of the index (top, middle, last).  In each pass a
// thread owns one 32-element sub-sequence and runs a radix-32 DFT in
// registers whose twiddles are the 32nd roots w32^e -- identical for every
// thread, read from kernel-parameter (constant-bank) space.  Between passes
// every element is multiplied by one "twiddle row" value w^(r*kappa), r the
// thread's row, kappa the DFT output index; each thread reads its 32 row
// entries as 16 contiguous 16-byte loads.  Output order is the standard DIF
// bit-reversed order, consumed unchanged by the pointwise stage and by the
// inverse (the exact transposed network: twiddle rows, then radix-32 DIT).
#include "ntt.cuh"
#include "ntt_passes.cuh"
#include <cstdlib>

namespace fpm {
namespace {
using namespace nttp;

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

// SINGLE: one prime -> every PrimeConst field is a constant-bank operand
// (no LDC); otherwise blockIdx.z selects the prime of a multi-prime batch.
template <int LOGN, bool SINGLE, int TPCX>
__global__ void __launch_bounds__(Geo<LOGN, TPCX>::THREADS)
    ntt_fwd_kernel(const __grid_constant__ NttFwdArgs a, const __grid_constant__ PrimeSet ps) {
  pdl_wait();
  using G = Geo<LOGN, TPCX>;
  extern __shared__ uint32_t sm[];
  const PrimeConst& pc = ps.pr[SINGLE ? 0 : blockIdx.z];
  const uint32_t p = pc.p;
  const int tid = threadIdx.x;
  const int tr = tid / G::TPT, lt = tid % G::TPT;
  const long long e0 = (long long)blockIdx.x * G::TPC;
  const long long e = e0 + tr;
  const bool valid = e < a.n_entries;
  uint32_t* smt = sm + tr * G::STRIDE;
  const long long pin = (long long)blockIdx.z * a.in_prime_stride;
  // the upper half of a zero-padded input is zero: skip its loads and adds
  const bool upper_zero = G::NPASS > 1 && !a.fold && a.len <= G::N / 2;
  uint32_t v[32];

  constexpr int FIRST = G::NPASS == 1 ? MAP_LAST : MAP_TOP;
  if (G::TPT >= 32) {
    // direct coalesced load: consecutive lanes read consecutive coefficients
    const long long eb = pin + e * a.in_stride;
    if (!a.fold && !a.in64 && !a.reduce) {
      // common case: branch-free predicated loads, all issued before use
      const uint32_t* src = (const uint32_t*)a.in + eb;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int x = xmap<LOGN, FIRST>(lt, i);
        const bool ld = valid && x < a.len && !(upper_zero && i >= 16);
        v[i] = ld ? __ldg(src + x) : 0u;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        if (upper_zero && i >= 16) {
          v[i] = 0;
          continue;
        }
        v[i] = valid ? load_coef(a, pc, eb, xmap<LOGN, FIRST>(lt, i), G::N) : 0u;
      }
    }
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
    dif_small<5>(v, pc.w32, p, false);
  } else {
    {
      Row r1;
      row_load(r1, pc.tw + lt * 32);  // w^(lt * kappa)
      dif_small<5>(v, pc.w32, p, upper_zero);
      row_apply(v, r1, p);
    }
    __syncthreads();
    to_smem<LOGN, MAP_TOP>(smt, v, lt);
    if (G::NPASS == 3) {
      constexpr int lo = LOGN - 10;
      Row r2;
      row_load(r2, pc.tw + (lt & ((1 << lo) - 1)) * 32 * 32);  // w^(32 lt' kappa')
      __syncthreads();
      from_smem<LOGN, MAP_MID>(smt, v, lt);
      dif_small<5>(v, pc.w32, p, false);
      row_apply(v, r2, p);
      __syncthreads();
      to_smem<LOGN, MAP_MID>(smt, v, lt);
    }
    __syncthreads();
    from_smem<LOGN, MAP_LAST>(smt, v, lt);
    dif_small<G::LAST_R>(v, pc.w32, p, false);
  }
  uint32_t* out = a.out + (long long)blockIdx.z * a.out_prime_stride;
  if (a.pm) {
    // point-major: out[x * n_entries + e], a CTA writes TPC consecutive
    // entries of every point as 16-byte pieces (staged through smem)
    __syncthreads();
    to_smem<LOGN, MAP_LAST>(smt, v, lt);
    __syncthreads();
    constexpr int PW = G::TPC < 4 ? G::TPC : 4;  // values per row piece
    constexpr int GQ = G::TPC / PW;
    const bool vec = (a.n_entries % PW) == 0;
    for (int idx = tid; idx < G::N * GQ; idx += G::THREADS) {
      const int x = idx / GQ, gq = idx - (idx / GQ) * GQ;
      const long long eb = e0 + PW * gq;
      uint32_t w[PW];
#pragma unroll
      for (int q = 0; q < PW; ++q) w[q] = sm[(PW * gq + q) * G::STRIDE + pad(x)];
      uint32_t* dst = out + (long long)x * a.n_entries + eb;
      if (vec && eb + PW - 1 < a.n_entries) {
        if constexpr (PW == 4)
          *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
        else
          *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[PW - 1]);
      } else {
#pragma unroll
        for (int q = 0; q < PW; ++q)
          if (eb + q < a.n_entries) dst[q] = w[q];
      }
    }
    return;
  }
  if (!valid) return;
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
    const int pl = a.pblk_log ? a.pblk_log : 5;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      *reinterpret_cast<uint4*>(out + eval_piece(lt * 32 + 4 * q, e, a.n_entries, pl)) =
          make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  }
}

template <int LOGN, bool SINGLE, int TPCX>
__global__ void __launch_bounds__(Geo<LOGN, TPCX>::THREADS)
    ntt_inv_kernel(const __grid_constant__ NttInvArgs a, const __grid_constant__ PrimeSet ps) {
  pdl_wait();
  using G = Geo<LOGN, TPCX>;
  extern __shared__ uint32_t sm[];
  const PrimeConst& pc = ps.pr[SINGLE ? 0 : blockIdx.z];
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
  } else if (a.pm) {
    constexpr int PW = G::TPC < 4 ? G::TPC : 4;  // values per row piece
    constexpr int GQ = G::TPC / PW;
    const bool vec = (a.n_entries % PW) == 0;
    for (int idx = tid; idx < G::N * GQ; idx += G::THREADS) {
      const int x = idx / GQ, gq = idx - (idx / GQ) * GQ;
      const long long eb = e0 + PW * gq;
      const uint32_t* src = in + (long long)x * a.n_entries + eb;
      uint32_t w[PW];
      if (vec && eb + PW - 1 < a.n_entries) {
        if constexpr (PW == 4) {
          const uint4 t = __ldg(reinterpret_cast<const uint4*>(src));
          w[0] = t.x; w[1] = t.y; w[2] = t.z; w[3] = t.w;
        } else {
          const uint2 t = __ldg(reinterpret_cast<const uint2*>(src));
          w[0] = t.x; w[PW - 1] = t.y;
        }
      } else {
#pragma unroll
        for (int q = 0; q < PW; ++q) w[q] = eb + q < a.n_entries ? src[q] : 0u;
      }
#pragma unroll
      for (int q = 0; q < PW; ++q) sm[(PW * gq + q) * G::STRIDE + pad(x)] = w[q];
    }
    __syncthreads();
    from_smem<LOGN, MAP_LAST>(smt, v, lt);
  } else if (valid) {
    const int pl = a.pblk_log ? a.pblk_log : 5;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint4 t = __ldg(
          reinterpret_cast<const uint4*>(in + eval_piece(lt * 32 + 4 * q, e, a.n_entries, pl)));
      v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = 0;
  }

  constexpr int FINAL = G::NPASS == 1 ? MAP_LAST : MAP_TOP;
  if (G::NPASS == 1) {
    dit_small<5>(v, pc.iw32, p);
  } else {
    if (G::NPASS == 3) {
      constexpr int lo = LOGN - 10;
      Row r2;
      row_load(r2, pc.itw + (lt & ((1 << lo) - 1)) * 32 * 32);
      dit_small<G::LAST_R>(v, pc.iw32, p);
      __syncthreads();
      to_smem<LOGN, MAP_LAST>(smt, v, lt);
      __syncthreads();
      from_smem<LOGN, MAP_MID>(smt, v, lt);
      row_apply(v, r2, p);
      Row r1;
      row_load(r1, pc.itw + lt * 32);
      dit_small<5>(v, pc.iw32, p);
      __syncthreads();
      to_smem<LOGN, MAP_MID>(smt, v, lt);
      __syncthreads();
      from_smem<LOGN, MAP_TOP>(smt, v, lt);
      row_apply(v, r1, p);
    } else {
      Row r1;
      row_load(r1, pc.itw + lt * 32);
      dit_small<G::LAST_R>(v, pc.iw32, p);
      __syncthreads();
      to_smem<LOGN, MAP_LAST>(smt, v, lt);
      __syncthreads();
      from_smem<LOGN, MAP_TOP>(smt, v, lt);
      row_apply(v, r1, p);
    }
    dit_small<5>(v, pc.iw32, p);
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

template <int LOGN, bool SINGLE, int TPCX>
int fwd_launch(const NttFwdArgs& a, const PrimeSet& ps, cudaStream_t st) {
  using G = Geo<LOGN, TPCX>;
  if (G::SMEM_BYTES > 48 * 1024) {
    static bool once = false;
    if (!once) {
      FPM_CUDA_TRY(cudaFuncSetAttribute(ntt_fwd_kernel<LOGN, SINGLE, TPCX>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        G::SMEM_BYTES));
      once = true;
    }
  }
  dim3 grid((unsigned)((a.n_entries + G::TPC - 1) / G::TPC), 1, (unsigned)ps.count);
  FPM_CUDA_TRY(launch_pdl(ntt_fwd_kernel<LOGN, SINGLE, TPCX>, dim3(grid), dim3(G::THREADS), G::SMEM_BYTES, st, a, ps));
  FPM_LAUNCH_CHECK();
  return kOk;
}

// point-major launches: 512 threads per CTA (2048: 8, 4096: 4, 8192: 2
// transforms -> 32/16/8-byte row pieces); N <= 1024 keeps the default TPC >= 8
template <int LOGN>
constexpr int pm_tpc() {
  return (1 << LOGN) <= 1024 ? 0 : (LOGN >= 14 ? 1 : (1 << (14 - LOGN)));
}

template <int LOGN>
int fwd_impl(const NttFwdArgs& a, const PrimeSet& ps, cudaStream_t st) {
  if (a.pm) {
    if constexpr (pm_tpc<LOGN>() >= 2 || pm_tpc<LOGN>() == 0) {
      return ps.count == 1 ? fwd_launch<LOGN, true, pm_tpc<LOGN>()>(a, ps, st)
                           : fwd_launch<LOGN, false, pm_tpc<LOGN>()>(a, ps, st);
    } else {
      set_last_error("point-major NTT layout needs N <= 2^13");
      return kUnsupported;
    }
  }
  return ps.count == 1 ? fwd_launch<LOGN, true, 0>(a, ps, st) : fwd_launch<LOGN, false, 0>(a, ps, st);
}

template <int LOGN, bool SINGLE, int TPCX>
int inv_launch(const NttInvArgs& a, const PrimeSet& ps, cudaStream_t st) {
  using G = Geo<LOGN, TPCX>;
  if (G::SMEM_BYTES > 48 * 1024) {
    static bool once = false;
    if (!once) {
      FPM_CUDA_TRY(cudaFuncSetAttribute(ntt_inv_kernel<LOGN, SINGLE, TPCX>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        G::SMEM_BYTES));
      once = true;
    }
  }
  dim3 grid((unsigned)((a.n_entries + G::TPC - 1) / G::TPC), 1, (unsigned)ps.count);
  FPM_CUDA_TRY(launch_pdl(ntt_inv_kernel<LOGN, SINGLE, TPCX>, dim3(grid), dim3(G::THREADS), G::SMEM_BYTES, st, a, ps));
  FPM_LAUNCH_CHECK();
  return kOk;
}

template <int LOGN>
int inv_impl(const NttInvArgs& a, const PrimeSet& ps, cudaStream_t st) {
  if (a.pm) {
    if constexpr (pm_tpc<LOGN>() >= 2 || pm_tpc<LOGN>() == 0) {
      return ps.count == 1 ? inv_launch<LOGN, true, pm_tpc<LOGN>()>(a, ps, st)
                           : inv_launch<LOGN, false, pm_tpc<LOGN>()>(a, ps, st);
    } else {
      set_last_error("point-major NTT layout needs N <= 2^13");
      return kUnsupported;
    }
  }
  return ps.count == 1 ? inv_launch<LOGN, true, 0>(a, ps, st) : inv_launch<LOGN, false, 0>(a, ps, st);
}

}  // namespace

int launch_ntt_fwd(int logn, const NttFwdArgs& a_in, const PrimeSet& ps, cudaStream_t st) {
  // tensor-core transforms (same DIF point order as the kernels below)
  if (ntt_mma_fwd_ok(logn, a_in, ps))
    return option(kOptNttMmaR16) != 0 ? launch_ntt_fwd_mma(a_in, ps, st)
                                      : launch_ntt_fwd_mma64(a_in, ps, st);
  const bool no_persist = option(kOptNttGeneric) != 0;
  if (!no_persist && ntt_tma_fwd_ok(logn, a_in)) return launch_ntt_fwd_tma(logn, a_in, ps, st);
  if (a_in.n_entries2 > 0) {
    if (!no_persist && ntt_persist_fwd_ok(logn, a_in) && a_in.n_entries > 0)
      return launch_ntt_fwd_persist(logn, a_in, ps, st);
    // generic kernels take one batch at a time
    NttFwdArgs b1 = a_in, b2 = a_in;
    b1.n_entries2 = 0; b1.len2 = 0;
    b2.in = a_in.in2; b2.in_stride = a_in.in2_stride; b2.in_prime_stride = a_in.in2_prime_stride;
    b2.n_entries = a_in.n_entries2; b2.out = a_in.out2; b2.out_prime_stride = a_in.out2_prime_stride;
    b2.n_entries2 = 0; b2.len2 = 0;
    if (a_in.len2 > 0) b2.len = a_in.len2;
    FPM_TRY(launch_ntt_fwd(logn, b1, ps, st));
    return launch_ntt_fwd(logn, b2, ps, st);
  }
  const NttFwdArgs& a = a_in;
  if (a.n_entries <= 0) return kOk;
  if (!no_persist && ntt_persist_fwd_ok(logn, a)) return launch_ntt_fwd_persist(logn, a, ps, st);
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
  const bool no_persist = option(kOptNttGeneric) != 0;
  if (!no_persist && ntt_tma_inv_ok(logn, a)) return launch_ntt_inv_tma(logn, a, ps, st);
  if (!no_persist && ntt_persist_inv_ok(logn, a)) return launch_ntt_inv_persist(logn, a, ps, st);
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
