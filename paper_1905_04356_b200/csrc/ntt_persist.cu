// ntt_persist.cu -- persistent batched NTT kernels (N <= 8192, 31-bit primes).
//
// Same four-step radix-32 network as ntt.cu, organised for latency hiding:
//   * each CTA stays resident and loops over groups of TPC transforms;
//   * the (row, kappa) twiddle table is staged ONCE per CTA in shared memory
//     (XOR-swizzled by row so 16-byte row reads are bank-conflict free) --
//     no global twiddle loads inside the passes;
//   * the next group's input is prefetched into 32 registers per thread
//     while the current group runs its passes, so HBM latency overlaps
//     butterfly work instead of stalling it.
// Forward: u32 input (no fold / no reduction), blocked-eval or point-major
// output.  Inverse: blocked-eval or point-major input.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdlib>
#include <mutex>

#include "ntt.cuh"
#include "ntt_passes.cuh"
#include "tc_common.cuh"

namespace fpm {
namespace {
using namespace nttp;

// pair q (entries 2q, 2q+1) of twiddle row r is stored at pair q ^ sw(r)
__device__ __forceinline__ int sw_row(int r) { return (r ^ (r >> 5)) & 7; }

// v[i] *= row r [brev5(i)], pairs read from the swizzled smem table just in
// time; every value (row[0] = 1 also reduces the lazy outputs of dit_lazy)
__device__ __forceinline__ void row_apply_s(uint32_t (&v)[32], const uint2* tws, int r,
                                            uint32_t p) {
  const uint4* base = reinterpret_cast<const uint4*>(tws + (size_t)r * 32);
  const int s = sw_row(r);
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const uint4 t = base[q ^ s];
    const int k0 = 2 * q, k1 = 2 * q + 1;
    {
      const int i0 = brev5(k0);
      v[i0] = d_red(d_shoup(v[i0], t.x, t.y, p), p);
    }
    const int i1 = brev5(k1);
    v[i1] = d_red(d_shoup(v[i1], t.z, t.w, p), p);
  }
}

// asynchronous copy of the twiddle table into shared memory (cp.async: all
// pieces in flight at once, no register round trip); the caller's
// __syncthreads() after cp_async_wait_all() publishes it
template <int LOGN>
__device__ __forceinline__ void stage_table(uint2* tws, const uint2* __restrict__ tw) {
  constexpr int N = 1 << LOGN;
  // N entries = N/32 rows x 16 pairs
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(tws);
  for (int idx = threadIdx.x; idx < N / 2; idx += blockDim.x) {
    const int r = idx >> 4, q = idx & 15;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                     base + 16u * (uint32_t)(r * 16 + (q ^ sw_row(r)))),
                 "l"(reinterpret_cast<const uint4*>(tw) + idx));
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

template <int LOGN, int TPCX>
__device__ __forceinline__ void fwd_passes(uint32_t (&v)[32], uint32_t* smt, const uint2* tws,
                                           const PrimeConst& pc, int lt, bool upper_zero) {
  using G = Geo<LOGN, TPCX>;
  const uint32_t p = pc.p;
  // radix passes as DIT on bit-reverse-aliased registers with lazy
  // reductions (ntt_passes.cuh dit_lazy): the DIF network and placement
  if (G::NPASS == 1) {
    dit_lazy<5, true, false>(v, pc.w32, p);
    return;
  }
  if (upper_zero)
    dit_lazy<5, true, true, true>(v, pc.w32, p);
  else
    dit_lazy<5, true, true>(v, pc.w32, p);
  row_apply_s(v, tws, lt, p);
  __syncthreads();
  to_smem<LOGN, MAP_TOP>(smt, v, lt);
  if (G::NPASS == 3) {
    constexpr int lo = LOGN - 10;
    __syncthreads();
    from_smem<LOGN, MAP_MID>(smt, v, lt);
    dit_lazy<5, true, true>(v, pc.w32, p);
    row_apply_s(v, tws, (lt & ((1 << lo) - 1)) * 32, p);
    __syncthreads();
    to_smem<LOGN, MAP_MID>(smt, v, lt);
  }
  __syncthreads();
  from_smem<LOGN, MAP_LAST>(smt, v, lt);
  dit_lazy<G::LAST_R, true, false>(v, pc.w32, p);
}

template <int LOGN, int TPCX>
__device__ __forceinline__ void inv_passes(uint32_t (&v)[32], uint32_t* smt, const uint2* tws,
                                           const PrimeConst& pc, int lt) {
  using G = Geo<LOGN, TPCX>;
  const uint32_t p = pc.p;
  if (G::NPASS == 1) {
    dit_lazy<5, false, false>(v, pc.iw32, p);
    return;
  }
  dit_lazy<G::LAST_R, false, true>(v, pc.iw32, p);  // the next pass multiplies every value
  __syncthreads();
  to_smem<LOGN, MAP_LAST>(smt, v, lt);
  __syncthreads();
  if (G::NPASS == 3) {
    constexpr int lo = LOGN - 10;
    from_smem<LOGN, MAP_MID>(smt, v, lt);
    row_apply_s(v, tws, (lt & ((1 << lo) - 1)) * 32, p);
    dit_lazy<5, false, true>(v, pc.iw32, p);
    __syncthreads();
    to_smem<LOGN, MAP_MID>(smt, v, lt);
    __syncthreads();
  }
  from_smem<LOGN, MAP_TOP>(smt, v, lt);
  row_apply_s(v, tws, lt, p);
  dit_lazy<5, false, false>(v, pc.iw32, p);
}

template <int THREADS>
constexpr int min_blocks() {
  return THREADS <= 256 ? 2 : 1;  // <= 128 registers per thread
}

template <int LOGN, bool SINGLE, int TPCX>
__global__ void __launch_bounds__(Geo<LOGN, TPCX>::THREADS, min_blocks<Geo<LOGN, TPCX>::THREADS>())
    ntt_fwd_persist(const __grid_constant__ NttFwdArgs a, const __grid_constant__ PrimeSet ps,
                    const __grid_constant__ CUtensorMap om1, const __grid_constant__ CUtensorMap om2) {
  using G = Geo<LOGN, TPCX>;
  extern __shared__ __align__(16) uint32_t sm[];
  uint2* tws = reinterpret_cast<uint2*>(sm + ((G::TPC * G::STRIDE + 3) & ~3));
  // point-major output of the TPC >= 4 transforms of a CTA by TMA: dense
  // [N][TPC] staging after the twiddle table (TPC * N = 8192 words); the
  // elected thread stores boxes of TPC entries x BP points
  constexpr bool kTmaPm = G::TPC == 4 && !G::PAIRED;  // N = 2048, 4096 (measured: smaller N lose)
  constexpr int BP = G::N < 256 ? G::N : 256;
  uint4* stage = reinterpret_cast<uint4*>(tws + G::N);
  const int z = SINGLE ? 0 : blockIdx.z;
  const PrimeConst& pc = ps.pr[z];
  const int tid = threadIdx.x;
  const int tr = G::PAIRED ? (tid & 1) : tid / G::TPT;
  const int lt = G::PAIRED ? (tid >> 1) : tid % G::TPT;
  uint32_t* smt = sm + tr * G::STRIDE;
  const long long groups1 = (a.n_entries + G::TPC - 1) / G::TPC;
  const long long groups = groups1 + (a.n_entries2 + G::TPC - 1) / G::TPC;
  const uint32_t* in1 = (const uint32_t*)a.in + (long long)z * a.in_prime_stride;
  uint32_t* out1 = a.out + (long long)z * a.out_prime_stride;
  const uint32_t* in2 =
      a.n_entries2 ? (const uint32_t*)a.in2 + (long long)z * a.in2_prime_stride : in1;
  uint32_t* out2 = a.n_entries2 ? a.out2 + (long long)z * a.out2_prime_stride : out1;
  // the two batches may differ in length (A and B of a middle product)
  const int len1 = a.len, len2 = a.len2 > 0 ? a.len2 : a.len;
  constexpr int FIRST = G::NPASS == 1 ? MAP_LAST : MAP_TOP;

  stage_table<LOGN>(tws, pc.tw);
  pdl_wait();  // constant tables above; data below may come from the previous kernel
  // (no early launch_dependents: a dependent made resident beside these short
  // kernels measured slower -- cfg4 81.4 vs 80.7 ms, cfg1 / 2 / 3 / 5 unchanged)

  uint32_t pre[32];
  auto load_group = [&](long long grp) {
    const bool second = grp >= groups1;
    const uint32_t* in = second ? in2 : in1;
    const long long jn = second ? a.n_entries2 : a.n_entries;
    const long long jstride = second ? a.in2_stride : a.in_stride;
    const int len = second ? len2 : len1;
    const bool upper_zero = G::NPASS > 1 && len <= G::N / 2;
    if (second) grp -= groups1;
    if (G::TPT >= 32) {
      const long long e = grp * G::TPC + tr;
      const bool valid = e < jn;
      const uint32_t* src = in + e * jstride;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int x = xmap<LOGN, FIRST>(lt, i);
        pre[i] = (valid && x < len && !(upper_zero && i >= 16)) ? __ldg(src + x) : 0u;
      }
    } else {
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        const int idx = tid + u * G::THREADS;
        const int t2 = idx >> LOGN, x = idx & (G::N - 1);
        const long long e = grp * G::TPC + t2;
        pre[u] = (e < jn && x < len) ? __ldg(in + e * jstride + x) : 0u;
      }
    }
  };

  long long grp = blockIdx.x;
  if (grp < groups) load_group(grp);
  cp_async_wait_all();
  __syncthreads();  // table staged
  for (; grp < groups; grp += gridDim.x) {
    uint32_t v[32];
    if (G::TPT >= 32) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = pre[i];
    } else {
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        const int idx = tid + u * G::THREADS;
        sm[(idx >> LOGN) * G::STRIDE + pad(idx & (G::N - 1))] = pre[u];
      }
      __syncthreads();
      from_smem<LOGN, FIRST>(smt, v, lt);
    }
    const long long nxt = grp + gridDim.x;
    constexpr bool kPrefetch = G::THREADS <= 512;  // 32 extra registers
    if (kPrefetch && nxt < groups) load_group(nxt);  // in flight during the passes
    const bool second = grp >= groups1;
    fwd_passes<LOGN, TPCX>(v, smt, tws, pc, lt,
                           G::NPASS > 1 && (second ? len2 : len1) <= G::N / 2);
    uint32_t* out = second ? out2 : out1;
    const long long jn = second ? a.n_entries2 : a.n_entries;
    const long long e0 = (second ? grp - groups1 : grp) * G::TPC, e = e0 + tr;
    if (G::PAIRED && a.pm) {
      // lane pair (tr = 0, 1) holds the two transforms of the same 32 points:
      // exchange half of them so each lane writes (T0[x], T1[x]) as 8 bytes
      const bool vec = (jn & 1) == 0 && e0 + 1 < jn;
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const uint32_t send = tr ? v[i] : v[i + 1];
        const uint32_t recv = __shfl_xor_sync(0xffffffffu, send, 1);
        const int x = xmap<LOGN, MAP_LAST>(lt, i + tr);
        const uint32_t lo = tr ? recv : v[i], hi = tr ? v[i + 1] : recv;
        uint32_t* dst = out + (long long)x * jn + e0;
        if (vec) {
          *reinterpret_cast<uint2*>(dst) = make_uint2(lo, hi);
        } else {
          if (e0 < jn) dst[0] = lo;
          if (e0 + 1 < jn) dst[1] = hi;
        }
      }
    } else if (G::TPC == 1 && a.pm) {
      // point-major scatter straight from registers (4-byte pieces; the
      // other entries of each 32-byte sector come from neighbouring CTAs)
      if (e < jn) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          out[(long long)xmap<LOGN, MAP_LAST>(lt, i) * jn + e] = v[i];
      }
    } else if (kTmaPm && a.pm && a.tma_pm) {
      // 16-byte row pieces (4 entries of one point) leave through the TMA
      // unit: the LSU would issue one 16-byte store per point and stall on
      // its queue (ncu: long-scoreboard on the store address registers)
      __syncthreads();
      to_smem<LOGN, MAP_LAST>(smt, v, lt);
      if (tid == 0) tc::bulk_wait_read0();  // previous group's stores have read the staging
      __syncthreads();
      constexpr int Q4 = G::TPC / 4;  // 16-byte chunks per point
      for (int idx = tid; idx < G::N * Q4; idx += G::THREADS) {
        const int x = idx / Q4, c = idx - (idx / Q4) * Q4;
        stage[idx] = make_uint4(sm[(4 * c) * G::STRIDE + pad(x)], sm[(4 * c + 1) * G::STRIDE + pad(x)],
                                sm[(4 * c + 2) * G::STRIDE + pad(x)],
                                sm[(4 * c + 3) * G::STRIDE + pad(x)]);
      }
      tc::fence_proxy_async();
      __syncthreads();
      if (tid == 0) {
        const CUtensorMap* om = second ? &om2 : &om1;
        const uint32_t sbase = tc::smem_u32(stage);
#pragma unroll 1
        for (int j = 0; j < G::N / BP; ++j)
          tc::tma_store_3d(om, sbase + (uint32_t)(BP * G::TPC * 4) * j, (int)e0, BP * j, z);
        tc::bulk_commit();
      }
    } else if (a.pm) {
      __syncthreads();
      to_smem<LOGN, MAP_LAST>(smt, v, lt);
      __syncthreads();
      constexpr int PW = G::TPC < 4 ? G::TPC : 4;  // values per row piece
      constexpr int GQ = G::TPC / PW;
      const bool vec = (jn % PW) == 0;
#pragma unroll 8
      for (int idx = tid; idx < G::N * GQ; idx += G::THREADS) {
        const int x = idx / GQ, gq = idx - (idx / GQ) * GQ;
        const long long eb = e0 + PW * gq;
        uint32_t w[PW];
#pragma unroll
        for (int q = 0; q < PW; ++q) w[q] = sm[(PW * gq + q) * G::STRIDE + pad(x)];
        uint32_t* dst = out + (long long)x * jn + eb;
        if (vec && eb + PW - 1 < jn) {
          if constexpr (PW == 4)
            *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
          else
            *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[PW - 1]);
        } else {
#pragma unroll
          for (int q = 0; q < PW; ++q)
            if (eb + q < jn) dst[q] = w[q];
        }
      }
    } else if (e < jn) {
      const int pl = a.pblk_log ? a.pblk_log : 5;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<uint4*>(out + eval_piece(lt * 32 + 4 * q, e, jn, pl)) =
            make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
    __syncthreads();  // smem exchange buffer reused by the next group
    if (!kPrefetch && nxt < groups) load_group(nxt);
  }
  if (kTmaPm && a.tma_pm && tid == 0) tc::bulk_wait0();
}

template <int LOGN, bool SINGLE, int TPCX>
__global__ void __launch_bounds__(Geo<LOGN, TPCX>::THREADS, min_blocks<Geo<LOGN, TPCX>::THREADS>())
    ntt_inv_persist(const __grid_constant__ NttInvArgs a, const __grid_constant__ PrimeSet ps,
                    const __grid_constant__ CUtensorMap im) {
  using G = Geo<LOGN, TPCX>;
  extern __shared__ __align__(16) uint32_t sm[];
  uint2* tws = reinterpret_cast<uint2*>(sm + ((G::TPC * G::STRIDE + 3) & ~3));
  // point-major input of the TPC >= 4 transforms of a CTA by TMA: boxes of
  // TPC entries x BP points land in a dense [N][TPC] staging tile a group
  // ahead (mbarrier)
  constexpr bool kTmaPm = G::TPC == 4 && !G::PAIRED;  // N = 2048, 4096 (measured: smaller N lose)
  constexpr int BP = G::N < 256 ? G::N : 256;
  const bool tma_in = kTmaPm && a.pm && a.tma_pm;
  uint4* stage = reinterpret_cast<uint4*>(tws + G::N);
  uint64_t* mb = reinterpret_cast<uint64_t*>(stage + (kTmaPm ? G::N * G::TPC / 4 : 0));
  const int z = SINGLE ? 0 : blockIdx.z;
  const PrimeConst& pc = ps.pr[z];
  const uint32_t p = pc.p;
  const int tid = threadIdx.x;
  const int tr = G::PAIRED ? (tid & 1) : tid / G::TPT;
  const int lt = G::PAIRED ? (tid >> 1) : tid % G::TPT;
  uint32_t* smt = sm + tr * G::STRIDE;
  const long long groups = (a.n_entries + G::TPC - 1) / G::TPC;
  const uint32_t* in = a.in + (long long)z * a.in_prime_stride;
  uint32_t* out = a.out + (long long)z * a.out_prime_stride;
  constexpr int FINAL = G::NPASS == 1 ? MAP_LAST : MAP_TOP;
  constexpr int PW = G::TPC < 4 ? G::TPC : 4;  // point-major row piece (values)
  constexpr int GQ = G::TPC / PW;

  stage_table<LOGN>(tws, pc.itw);
  if (tma_in && tid == 0) {
    tc::mbar_init(mb, 1);
    tc::fence_mbar_init();
    tc::prefetch_tmap(&im);
  }
  pdl_wait();
  auto tma_group = [&](long long g) {  // elected thread
    tc::mbar_expect_tx(mb, (uint32_t)G::N * G::TPC * 4u);
    const uint32_t sbase = tc::smem_u32(stage);
#pragma unroll 1
    for (int j = 0; j < G::N / BP; ++j)
      tc::tma_load_3d(sbase + (uint32_t)(BP * G::TPC * 4) * j, &im, mb, (int)(g * G::TPC), BP * j, z);
  };
  uint32_t phase = 0;

  uint32_t pre[32];
  auto load_group = [&](long long grp) {
    const long long e0 = grp * G::TPC;
    if (G::PAIRED && a.pm) {
      // raw (T0[x], T1[x]) pairs for x = point of element i + tr; swapped
      // into place when the group is consumed
      const bool vec = (a.n_entries & 1) == 0 && e0 + 1 < a.n_entries;
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const int x = xmap<LOGN, MAP_LAST>(lt, i + tr);
        const uint32_t* src = in + (long long)x * a.n_entries + e0;
        if (vec) {
          const uint2 t = __ldg(reinterpret_cast<const uint2*>(src));
          pre[i] = t.x; pre[i + 1] = t.y;
        } else {
          pre[i] = e0 < a.n_entries ? src[0] : 0u;
          pre[i + 1] = e0 + 1 < a.n_entries ? src[1] : 0u;
        }
      }
    } else if (G::TPC == 1 && a.pm) {
      const long long e = e0 + tr;
#pragma unroll
      for (int i = 0; i < 32; ++i)
        pre[i] = e < a.n_entries
                     ? __ldg(in + (long long)xmap<LOGN, MAP_LAST>(lt, i) * a.n_entries + e)
                     : 0u;
    } else if (a.pm) {
      // this thread's share of the group's point-major input: PW-value pieces
      const bool vec = (a.n_entries % PW) == 0;
#pragma unroll
      for (int u = 0; u < 32 / PW; ++u) {
        const int idx = tid + u * G::THREADS;
        const int x = idx / GQ, gq = idx - (idx / GQ) * GQ;
        const long long eb = e0 + PW * gq;
        const uint32_t* src = in + (long long)x * a.n_entries + eb;
        if (vec && eb + PW - 1 < a.n_entries) {
          if constexpr (PW == 4) {
            const uint4 t = __ldg(reinterpret_cast<const uint4*>(src));
            pre[4 * u] = t.x; pre[4 * u + 1] = t.y; pre[4 * u + 2] = t.z; pre[4 * u + 3] = t.w;
          } else {
            const uint2 t = __ldg(reinterpret_cast<const uint2*>(src));
            pre[PW * u] = t.x; pre[PW * u + PW - 1] = t.y;
          }
        } else {
#pragma unroll
          for (int q = 0; q < PW; ++q) pre[PW * u + q] = eb + q < a.n_entries ? src[q] : 0u;
        }
      }
    } else {
      const long long e = e0 + tr;
      if (e < a.n_entries) {
        const int pl = a.pblk_log ? a.pblk_log : 5;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint4 t = __ldg(reinterpret_cast<const uint4*>(
              in + eval_piece(lt * 32 + 4 * q, e, a.n_entries, pl)));
          pre[4 * q] = t.x; pre[4 * q + 1] = t.y; pre[4 * q + 2] = t.z; pre[4 * q + 3] = t.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) pre[i] = 0;
      }
    }
  };

  long long grp = blockIdx.x;
  if (grp < groups) {
    if (tma_in) {
      __syncthreads();  // barrier initialised
      if (tid == 0) tma_group(grp);
    } else {
      load_group(grp);
    }
  }
  cp_async_wait_all();
  __syncthreads();  // table staged
  for (; grp < groups; grp += gridDim.x) {
    uint32_t v[32];
    if (tma_in) {
      tc::mbar_wait(mb, phase);
      phase ^= 1u;
      constexpr int Q4 = G::TPC / 4;
      for (int idx = tid; idx < G::N * Q4; idx += G::THREADS) {
        const int x = idx / Q4, c = idx - (idx / Q4) * Q4;
        const uint4 t = stage[idx];
        sm[(4 * c) * G::STRIDE + pad(x)] = t.x;
        sm[(4 * c + 1) * G::STRIDE + pad(x)] = t.y;
        sm[(4 * c + 2) * G::STRIDE + pad(x)] = t.z;
        sm[(4 * c + 3) * G::STRIDE + pad(x)] = t.w;
      }
      __syncthreads();  // staging consumed: the next group may land
      if (tid == 0 && grp + gridDim.x < groups) tma_group(grp + gridDim.x);
      from_smem<LOGN, MAP_LAST>(smt, v, lt);
    } else if (G::PAIRED && a.pm) {
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        // pre[i..i+1] = (T0, T1) at point i + tr; this lane wants T_tr at i, i+1
        const uint32_t send = tr ? pre[i] : pre[i + 1];
        const uint32_t recv = __shfl_xor_sync(0xffffffffu, send, 1);
        v[i] = tr ? recv : pre[i];
        v[i + 1] = tr ? pre[i + 1] : recv;
      }
    } else if (a.pm && G::TPC > 1) {
#pragma unroll
      for (int u = 0; u < 32 / PW; ++u) {
        const int idx = tid + u * G::THREADS;
        const int x = idx / GQ, gq = idx - (idx / GQ) * GQ;
#pragma unroll
        for (int q = 0; q < PW; ++q) sm[(PW * gq + q) * G::STRIDE + pad(x)] = pre[PW * u + q];
      }
      __syncthreads();
      from_smem<LOGN, MAP_LAST>(smt, v, lt);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = pre[i];
    }
    const long long nxt = grp + gridDim.x;
    constexpr bool kPrefetch = G::THREADS <= 512;
    if (!tma_in && kPrefetch && nxt < groups) load_group(nxt);
    inv_passes<LOGN, TPCX>(v, smt, tws, pc, lt);
    if (a.scale) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = d_red(d_shoup(v[i], pc.ninv, pc.ninv_sh, p), p);
    }
    const long long e0 = grp * G::TPC, e = e0 + tr;
    if (G::TPT >= 32) {
      if (e < a.n_entries) {
        uint32_t* oe = out + e * a.out_stride;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int t = (xmap<LOGN, FINAL>(lt, i) - a.off) & (G::N - 1);
          if (t < a.out_len) oe[t] = v[i];
        }
      }
    } else {
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
    __syncthreads();
    if (!tma_in && !kPrefetch && nxt < groups) load_group(nxt);
  }
}

// point-major: 4 transforms per CTA (16-byte row pieces) for N = 4096, 2
// (8-byte pieces) for N = 8192 so a CTA stays at 512 threads / 128 registers
template <int LOGN>
constexpr int pm_tpc2() {
  return (1 << LOGN) <= 2048 ? 0 : ((1 << LOGN) <= 4096 ? 4 : kPaired);
}

PFN_cuTensorMapEncodeTiled_v12000 pm_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

// point-major evaluations E[z][t][entry]: boxes of 4 entries x 256 points
bool pm_map(CUtensorMap* m, uint32_t* base, long long entries, int N, long long prime_stride,
            int primes, int tpc) {
  auto fn = pm_encode_fn();
  if (!fn || !base || ((uintptr_t)base & 15) || (entries & 3) || (prime_stride & 3) ||
      (tpc & 3))
    return false;
  const cuuint64_t dims[3] = {(cuuint64_t)entries, (cuuint64_t)N, (cuuint64_t)primes};
  const cuuint64_t strides[2] = {(cuuint64_t)entries * 4,
                                 (cuuint64_t)(primes > 1 ? prime_stride : (long long)N * entries) * 4};
  const cuuint32_t box[3] = {(cuuint32_t)tpc, (cuuint32_t)(N < 256 ? N : 256), 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, base, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int LOGN, bool SINGLE, int TPCX, bool FWD, typename Args>
int persist_launch(const Args& a_in, const PrimeSet& ps, cudaStream_t st) {
  using G = Geo<LOGN, TPCX>;
  Args a = a_in;
  CUtensorMap om1{}, om2{};
  constexpr bool kTmaPm = G::TPC == 4 && !G::PAIRED;  // N = 2048, 4096 (measured: smaller N lose)
  if constexpr (kTmaPm && !FWD) {
    const bool off = option(kOptNttPmLsu) != 0;
    a.tma_pm = (!off && a.pm &&
                pm_map(&om1, const_cast<uint32_t*>(a.in), a.n_entries, G::N, a.in_prime_stride,
                       ps.count, G::TPC)) ? 1 : 0;
  }
  if constexpr (kTmaPm && FWD) {
    const bool off = option(kOptNttPmLsu) != 0;
    a.tma_pm = 0;
    if (!off && a.pm &&
        pm_map(&om1, a.out, a.n_entries, G::N, a.out_prime_stride, ps.count, G::TPC)) {
      a.tma_pm = 1;
      if (a.n_entries2 > 0)
        a.tma_pm =
            pm_map(&om2, a.out2, a.n_entries2, G::N, a.out2_prime_stride, ps.count, G::TPC) ? 1 : 0;
      else
        om2 = om1;
    }
  }
  const size_t smem = (size_t)((G::TPC * G::STRIDE + 3) & ~3) * 4 + (size_t)G::N * 8 +
                      (kTmaPm ? (size_t)G::N * G::TPC * 4 + 16 : 0);
  const void* kern;
  if constexpr (FWD)
    kern = (const void*)ntt_fwd_persist<LOGN, SINGLE, TPCX>;
  else
    kern = (const void*)ntt_inv_persist<LOGN, SINGLE, TPCX>;
  static int blocks_per_sm = 0;
  if (!blocks_per_sm) {
    FPM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
    FPM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern,
                                                               G::THREADS, smem));
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long groups = (a.n_entries + G::TPC - 1) / G::TPC;
  if constexpr (FWD) groups += (a.n_entries2 + G::TPC - 1) / G::TPC;
  long long grid = (long long)blocks_per_sm * sms / ps.count;
  if (grid < 1) grid = 1;
  if (grid > groups) grid = groups;
  dim3 g3((unsigned)grid, 1, (unsigned)ps.count);
  if constexpr (FWD)
    FPM_CUDA_TRY(launch_pdl(ntt_fwd_persist<LOGN, SINGLE, TPCX>, dim3(g3), dim3(G::THREADS), smem, st, a, ps,
                            om1, om2));
  else
    FPM_CUDA_TRY(launch_pdl(ntt_inv_persist<LOGN, SINGLE, TPCX>, dim3(g3), dim3(G::THREADS), smem, st, a, ps,
                            om1));
  FPM_LAUNCH_CHECK();
  return kOk;
}

template <int LOGN, bool FWD, typename Args>
int persist_impl(const Args& a, const PrimeSet& ps, cudaStream_t st) {
  const bool pm_scatter = option(kOptNttPmScatter) != 0;
  if (a.pm && pm_scatter && (1 << LOGN) >= 256) {
    return ps.count == 1 ? persist_launch<LOGN, true, 1, FWD>(a, ps, st)
                         : persist_launch<LOGN, false, 1, FWD>(a, ps, st);
  }
  if constexpr (LOGN <= 7) {
    // a short batch of short transforms (the PM-Basis nodes of order 16 ... 64)
    // fills a fraction of the SMs at the default 8192 / N transforms per CTA
    // and is all latency: a quarter of that per CTA spreads it over 4x the SMs
    constexpr int kSmallTpc = 2048 >> LOGN;
    long long tr = a.n_entries;
    if constexpr (FWD) tr += a.n_entries2;
    if (option(kOptNttNoSmall) == 0 && tr * 2 <= 148LL * (8192 >> LOGN))
      return ps.count == 1 ? persist_launch<LOGN, true, kSmallTpc, FWD>(a, ps, st)
                           : persist_launch<LOGN, false, kSmallTpc, FWD>(a, ps, st);
  }
  if (a.pm) {
    return ps.count == 1 ? persist_launch<LOGN, true, pm_tpc2<LOGN>(), FWD>(a, ps, st)
                         : persist_launch<LOGN, false, pm_tpc2<LOGN>(), FWD>(a, ps, st);
  }
  return ps.count == 1 ? persist_launch<LOGN, true, 0, FWD>(a, ps, st)
                       : persist_launch<LOGN, false, 0, FWD>(a, ps, st);
}

}  // namespace

bool ntt_persist_fwd_ok(int logn, const NttFwdArgs& a) {
  return logn >= 5 && logn <= 13 && !a.fold && !a.in64 && !a.reduce && !a.natural;
}
bool ntt_persist_inv_ok(int logn, const NttInvArgs& a) {
  return logn >= 5 && logn <= 13 && !a.natural;
}

int launch_ntt_fwd_persist(int logn, const NttFwdArgs& a, const PrimeSet& ps, cudaStream_t st) {
  switch (logn) {
    case 5: return persist_impl<5, true>(a, ps, st);
    case 6: return persist_impl<6, true>(a, ps, st);
    case 7: return persist_impl<7, true>(a, ps, st);
    case 8: return persist_impl<8, true>(a, ps, st);
    case 9: return persist_impl<9, true>(a, ps, st);
    case 10: return persist_impl<10, true>(a, ps, st);
    case 11: return persist_impl<11, true>(a, ps, st);
    case 12: return persist_impl<12, true>(a, ps, st);
    case 13: return persist_impl<13, true>(a, ps, st);
  }
  return kUnsupported;
}

int launch_ntt_inv_persist(int logn, const NttInvArgs& a, const PrimeSet& ps, cudaStream_t st) {
  switch (logn) {
    case 5: return persist_impl<5, false>(a, ps, st);
    case 6: return persist_impl<6, false>(a, ps, st);
    case 7: return persist_impl<7, false>(a, ps, st);
    case 8: return persist_impl<8, false>(a, ps, st);
    case 9: return persist_impl<9, false>(a, ps, st);
    case 10: return persist_impl<10, false>(a, ps, st);
    case 11: return persist_impl<11, false>(a, ps, st);
    case 12: return persist_impl<12, false>(a, ps, st);
    case 13: return persist_impl<13, false>(a, ps, st);
  }
  return kUnsupported;
}

}  // namespace fpm
