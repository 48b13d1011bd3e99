// ntt_tma.cu -- grouped persistent NTT with TMA input/output (N = 2^11 .. 2^13,
// 31-bit primes): the product path's forward transforms (u32 coefficients ->
// blocked / point-quad evaluations) and inverse transforms (evaluations ->
// natural-order coefficients times N^-1).
//
// Replaces, for those layouts, the per-entry evaluation / interpolation of
// polmat._pm_mul_ntt (ref polmat.py:275-307) like ntt_persist.cu, with the
// same four-step radix-32 network (ntt_passes.cuh) and the same results; what
// changes is how the work is fed:
//   * a CTA holds G independent transform GROUPS (N/32 threads each) that
//     synchronise with their own named barrier (bar.sync 1+g), so while one
//     group waits for memory or a barrier the others keep the integer pipes
//     busy (the single-transform CTAs of ntt_persist.cu stall in lock step);
//   * forward input: one cp.async.bulk of the entry's coefficients per
//     transform into the group's input buffer, issued a transform ahead and
//     completed on an mbarrier (no prefetch registers, no predicated loads);
//   * forward output: the last pass writes its rows (32 consecutive points
//     per thread) into a dense SWIZZLE_128B staging tile and ONE elected
//     thread stores it with TMA tensor stores (the direct 16-byte stores of
//     ntt_persist.cu scatter 32 lines per warp instruction and stall on the
//     store queue);
//   * inverse input: TMA tensor loads of the blocked / point-quad evaluations
//     straight into the staging tile, issued while the previous transform is
//     in its last pass;
//   * inverse scaling by N^-1 is folded into the last pass's row twiddles
//     (Plan::itw_s), one Shoup multiply per value instead of two;
//   * twiddle rows sit in shared memory with a 16-byte pad per row (272 B):
//     the 16-byte row reads of 32 lanes on 32 rows are conflict free with
//     immediate offsets (no per-read swizzle arithmetic).
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
using tc::smem_u32;

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

constexpr int kRowBytes = 272;  // 32 (w, w') pairs + 16 B pad

template <int LOGN, int G>
struct TG {
  static_assert(LOGN >= 11 && LOGN <= 13, "three-pass geometry");
  static constexpr int N = 1 << LOGN;
  static constexpr int TPT = N / 32;  // threads per transform group
  static constexpr int THREADS = TPT * G;
  static constexpr int LO = LOGN - 10;  // middle-pass row bits (ntt_passes.cuh MAP_MID)
  static constexpr int LAST_R = LOGN - 10;
  static constexpr int TOP_ROWS = N / 32;
  static constexpr int MID_ROWS = 1 << LO;
  static constexpr int TAB_BYTES = ((TOP_ROWS + MID_ROWS) * kRowBytes + 1023) & ~1023;
  static constexpr int TILE_BYTES = ((N + N / 32) * 4 + 1023) & ~1023;
};

struct TmaFwdArgs {
  const uint32_t* in1;
  long long in1_stride, in1_ps;
  long long n1;
  const uint32_t* in2;
  long long in2_stride, in2_ps;
  long long n2;
  int len;       // coefficients per entry (multiple of 4)
  int in_words;  // input buffer words: N/2 (upper half zero) or N
  int pl;        // eval block log: 5 (E[N/32][e][32]) or 2 (E[N/4][e][4])
};

struct TmaInvArgs {
  uint32_t* out;
  long long out_stride, out_ps;
  long long n;
  int out_len, off;
  int pl;
};

__device__ __forceinline__ void gsync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes,
                                          uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void expect_tx(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mbar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_store_4d(const void* tmap, uint32_t src, int c0, int c1, int c2,
                                             int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];\n" ::"l"(
          tmap),
      "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_store_5d(const void* tmap, uint32_t src, int c0, int c1, int c2,
                                             int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];\n" ::"l"(
          tmap),
      "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void tma_load_5d(uint32_t dst, const void* tmap, uint32_t mbar, int c0,
                                            int c1, int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5, %6, %7}], [%2];\n" ::"r"(dst),
      "l"(tmap), "r"(mbar), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// v[i] *= row[brev5(i)]: 16-byte pieces of one padded smem row; ALL also
// multiplies element 0 (the scaled inverse rows have row[0] = N^-1)
template <bool ALL>
__device__ __forceinline__ void row_apply_t(uint32_t (&v)[32], const uint8_t* row, uint32_t p) {
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const uint4 t = *reinterpret_cast<const uint4*>(row + 16 * q);
    const int i0 = brev5(2 * q), i1 = brev5(2 * q + 1);
    if (ALL || q) v[i0] = d_red(d_shoup(v[i0], t.x, t.y, p), p);
    v[i1] = d_red(d_shoup(v[i1], t.z, t.w, p), p);
  }
}

// top rows r < N/32 of `top` and middle rows 32 j (j < 2^LO) of `mid` into
// padded smem rows (cp.async, 16-byte pieces)
template <int LOGN, int G>
__device__ __forceinline__ void stage_tables(uint8_t* tab, const uint2* __restrict__ top,
                                             const uint2* __restrict__ mid) {
  using T = TG<LOGN, G>;
  const uint32_t base = smem_u32(tab);
  constexpr int PIECES = (T::TOP_ROWS + T::MID_ROWS) * 16;
  for (int idx = threadIdx.x; idx < PIECES; idx += T::THREADS) {
    const int r = idx >> 4, q = idx & 15;
    const uint2* src = r < T::TOP_ROWS ? top + (size_t)r * 32 + 2 * q
                                       : mid + (size_t)(r - T::TOP_ROWS) * 32 * 32 + 2 * q;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(base + r * kRowBytes + 16 * q),
                 "l"(src));
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// byte offset in the staging tile of the 16-byte chunk c (points 32 lt + 4c ..
// 32 lt + 4c + 3) of thread lt.  PL = 5: SWIZZLE_128B rows of 128 B (one TMA
// box {32, 1, N/32}); PL = 2: eight regions of N/32 chunks, region c holding
// every thread's chunk c (TMA boxes {4, 1, 1, N/32} over the quad layout viewed
// as [N/32][8][entry][4]); both conflict free for 16-byte accesses
template <int LOGN, int PL>
__device__ __forceinline__ int chunk_off(int lt, int c) {
  if constexpr (PL == 5)
    return lt * 128 + ((c ^ (lt & 7)) << 4);
  else
    return c * ((1 << LOGN) / 2) + lt * 16;
}

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  const uint32_t s = smem_u32(p);
  return p + (((s + 1023u) & ~1023u) - s);
}

// ---------------------------------------------------------------------------
template <int LOGN, int G, int PL>
__global__ void __launch_bounds__(TG<LOGN, G>::THREADS, 1)
    ntt_fwd_tma(const __grid_constant__ CUtensorMap om1, const __grid_constant__ CUtensorMap om2,
                const __grid_constant__ TmaFwdArgs a, const __grid_constant__ PrimeSet ps) {
  using T = TG<LOGN, G>;
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = align1024(smraw);
  const int z = blockIdx.z;
  const PrimeConst& pc = ps.pr[z];
  const uint32_t p = pc.p;
  const int g = threadIdx.x / T::TPT, lt = threadIdx.x % T::TPT;
  const bool leader = lt == 0;
  const int bar = 1 + g;
  uint8_t* tab = sm;
  uint8_t* tile8 = sm + T::TAB_BYTES + g * T::TILE_BYTES;
  uint32_t* tile = reinterpret_cast<uint32_t*>(tile8);
  uint32_t* inb =
      reinterpret_cast<uint32_t*>(sm + T::TAB_BYTES + G * T::TILE_BYTES) + (size_t)g * a.in_words;
  uint64_t* mb = reinterpret_cast<uint64_t*>(sm + T::TAB_BYTES + G * T::TILE_BYTES +
                                             (size_t)G * a.in_words * 4) + g;
  const uint32_t mbar = smem_u32(mb), inb_s = smem_u32(inb), tile_s = smem_u32(tile8);

  stage_tables<LOGN, G>(tab, pc.tw, pc.tw);
  for (int w = a.len + lt; w < a.in_words; w += T::TPT) inb[w] = 0u;  // zero padding, once
  tc::fence_proxy_async();
  if (leader) {
    tc::mbar_init(mb, 1);
    tc::fence_mbar_init();
    tc::prefetch_tmap(&om1);
    tc::prefetch_tmap(&om2);
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  pdl_wait();  // inputs / outputs may belong to the previous kernel
  pdl_trigger();

  const long long items = a.n1 + a.n2;
  // point quads: groups take items round-robin across the whole grid, so
  // the eight entries sharing a 128-byte quad line are stored close in time;
  // blocked rows own their lines: a contiguous range per CTA (every SM gets
  // floor or ceil of items / CTAs)
  const long long total = items;
  const bool rr = PL == 2;
  const long long hi = rr ? total : total * (blockIdx.x + 1) / gridDim.x;
  const long long step = rr ? (long long)gridDim.x * G : G;
  long long item = rr ? (long long)blockIdx.x * G + g : total * blockIdx.x / gridDim.x + g;
  const uint32_t bytes = (uint32_t)a.len * 4u;
  auto src_of = [&](long long it) -> const uint32_t* {
    return it < a.n1 ? a.in1 + z * a.in1_ps + it * a.in1_stride
                     : a.in2 + z * a.in2_ps + (it - a.n1) * a.in2_stride;
  };
  if (leader && item < hi) {
    expect_tx(mbar, bytes);
    bulk_load(inb_s, src_of(item), bytes, mbar);
  }
  const bool upper_zero = a.in_words == T::N / 2;
  const uint8_t* top_row = tab + lt * kRowBytes;
  const uint8_t* mid_row = tab + (T::TOP_ROWS + (lt & (T::MID_ROWS - 1))) * kRowBytes;
  uint32_t phase = 0;
  for (; item < hi; item += step) {
    tc::mbar_wait_a(mbar, phase);
    phase ^= 1u;
    uint32_t v[32];
    // pass 1: radix-32 over stride N/32, then the row-lt twiddles (every
    // value: row[0] = 1 reduces the lazy outputs too)
    if (upper_zero) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = i < 16 ? inb[lt + (i << (LOGN - 5))] : 0u;
      dit_lazy<5, true, true, true>(v, pc.w32, p);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = inb[lt + (i << (LOGN - 5))];
      dit_lazy<5, true, true, false>(v, pc.w32, p);
    }
    row_apply_t<true>(v, top_row, p);
    if (leader) bulk_wait_read0();  // the previous output store has read the tile
    gsync(bar, T::TPT);             // input reads done, tile free
    if (leader && item + step < hi) {
      expect_tx(mbar, bytes);
      bulk_load(inb_s, src_of(item + step), bytes, mbar);
    }
    to_smem<LOGN, MAP_TOP>(tile, v, lt);
    gsync(bar, T::TPT);
    // pass 2
    from_smem<LOGN, MAP_MID>(tile, v, lt);
    dit_lazy<5, true, true>(v, pc.w32, p);
    row_apply_t<true>(v, mid_row, p);
    to_smem<LOGN, MAP_MID>(tile, v, lt);  // the positions this thread read: no barrier
    gsync(bar, T::TPT);
    // pass 3: thread lt ends with points 32 lt .. 32 lt + 31
    from_smem<LOGN, MAP_LAST>(tile, v, lt);
    dit_lazy<T::LAST_R, true, false>(v, pc.w32, p);
    // (the 16-byte quad pieces could also leave through the LSU: measured
    // slower than the TMA unit alone, so every chunk is staged)
    const bool second = item >= a.n1;
    gsync(bar, T::TPT);  // every padded read done before dense rows overwrite the tile
#pragma unroll
    for (int c = 0; c < 8; ++c)
      *reinterpret_cast<uint4*>(tile8 + chunk_off<LOGN, PL>(lt, c)) =
          make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
    tc::fence_proxy_async();
    gsync(bar, T::TPT);
    if (leader) {
      const CUtensorMap* om = second ? &om2 : &om1;
      const int e = (int)(second ? item - a.n1 : item);
      if constexpr (PL == 5) {
        tma_store_4d(om, tile_s, 0, e, 0, z);
      } else {
#pragma unroll
        for (int c = 0; c < 8; ++c) tma_store_5d(om, tile_s + c * (T::N / 2), 0, e, c, 0, z);
      }
      bulk_commit();
    }
  }
  if (leader) bulk_wait0();
}

// ---------------------------------------------------------------------------
template <int LOGN, int G, int PL>
__global__ void __launch_bounds__(TG<LOGN, G>::THREADS, 1)
    ntt_inv_tma(const __grid_constant__ CUtensorMap im, const __grid_constant__ TmaInvArgs a,
                const __grid_constant__ PrimeSet ps) {
  using T = TG<LOGN, G>;
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = align1024(smraw);
  const int z = blockIdx.z;
  const PrimeConst& pc = ps.pr[z];
  const uint32_t p = pc.p;
  const int g = threadIdx.x / T::TPT, lt = threadIdx.x % T::TPT;
  const bool leader = lt == 0;
  const int bar = 1 + g;
  uint8_t* tab = sm;
  uint8_t* tile8 = sm + T::TAB_BYTES + g * T::TILE_BYTES;
  uint32_t* tile = reinterpret_cast<uint32_t*>(tile8);
  // evaluations land in a separate buffer, a whole transform ahead
  uint8_t* inb8 = sm + T::TAB_BYTES + G * T::TILE_BYTES + g * T::N * 4;
  uint64_t* mb = reinterpret_cast<uint64_t*>(sm + T::TAB_BYTES + G * (T::TILE_BYTES + T::N * 4)) + g;
  const uint32_t mbar = smem_u32(mb), inb_s = smem_u32(inb8);

  stage_tables<LOGN, G>(tab, pc.itw_s, pc.itw);
  if (leader) {
    tc::mbar_init(mb, 1);
    tc::fence_mbar_init();
    tc::prefetch_tmap(&im);
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  pdl_wait();
  pdl_trigger();

  // contiguous item range per CTA (its groups interleave inside it): every
  // SM gets floor or ceil of items / CTAs, not whole rounds of G
  const long long total = a.n;
  const long long hi = total * (blockIdx.x + 1) / gridDim.x;
  const long long step = G;
  long long item = total * blockIdx.x / gridDim.x + g;
  auto load = [&](long long it) {
    expect_tx(mbar, (uint32_t)T::N * 4u);
    if constexpr (PL == 5) {
      tc::tma_load_4d(inb_s, &im, mb, 0, (int)it, 0, z);
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c) tma_load_5d(inb_s + c * (T::N / 2), &im, mbar, 0, (int)it, c, 0, z);
    }
  };
  if (leader && item < hi) load(item);
  const uint8_t* top_row = tab + lt * kRowBytes;
  const uint8_t* mid_row = tab + (T::TOP_ROWS + (lt & (T::MID_ROWS - 1))) * kRowBytes;
  uint32_t phase = 0;
  for (; item < hi; item += step) {
    tc::mbar_wait_a(mbar, phase);
    phase ^= 1u;
    uint32_t v[32];
    // row lt (points 32 lt .. 32 lt + 31) of the landed evaluations
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint4 t = *reinterpret_cast<const uint4*>(inb8 + chunk_off<LOGN, PL>(lt, c));
      v[4 * c] = t.x; v[4 * c + 1] = t.y; v[4 * c + 2] = t.z; v[4 * c + 3] = t.w;
    }
    dit_lazy<T::LAST_R, false, true>(v, pc.iw32, p);
    // input buffer read by every thread (the next transform may land), and the
    // previous transform's last tile reads are done (tile free)
    gsync(bar, T::TPT);
    if (leader && item + step < hi) load(item + step);
    to_smem<LOGN, MAP_LAST>(tile, v, lt);
    gsync(bar, T::TPT);
    from_smem<LOGN, MAP_MID>(tile, v, lt);
    row_apply_t<true>(v, mid_row, p);  // row[0] = 1 reduces the lazy values
    dit_lazy<5, false, true>(v, pc.iw32, p);
    to_smem<LOGN, MAP_MID>(tile, v, lt);  // own positions
    gsync(bar, T::TPT);
    from_smem<LOGN, MAP_TOP>(tile, v, lt);
    row_apply_t<true>(v, top_row, p);  // twiddles times N^-1
    dit_lazy<5, false, false>(v, pc.iw32, p);
    uint32_t* oe = a.out + z * a.out_ps + item * a.out_stride;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int t = ((lt + (i << (LOGN - 5))) - a.off) & (T::N - 1);
      if (t < a.out_len) oe[t] = v[i];
    }
  }
}

// ---------------------------------------------------------------------------
int encode_eval_map(CUtensorMap* m, const uint32_t* base, long long n_entries, int N, int pl,
                    long long prime_stride, int primes) {
  auto fn = encode_fn();
  if (!fn) {
    set_last_error("cuTensorMapEncodeTiled unavailable");
    return kCudaError;
  }
  const cuuint64_t ps = (cuuint64_t)(primes > 1 ? prime_stride : (long long)N * n_entries) * 4;
  const cuuint64_t ne = (cuuint64_t)n_entries;
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r;
  if (pl == 5) {
    // E[N/32][entry][32]: {32, entries, N/32, primes}, box = one entry's N points
    const cuuint64_t dims[4] = {32, ne, (cuuint64_t)(N / 32), (cuuint64_t)primes};
    const cuuint64_t strides[3] = {128, ne * 128, ps};
    const cuuint32_t box[4] = {32, 1, (cuuint32_t)(N / 32), 1};
    r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, const_cast<uint32_t*>(base), dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    // E[N/4][entry][4] viewed as [N/32][8][entry][4]: {4, entries, 8, N/32, primes},
    // box = chunk c of every 32-point segment of one entry
    const cuuint64_t dims[5] = {4, ne, 8, (cuuint64_t)(N / 32), (cuuint64_t)primes};
    const cuuint64_t strides[4] = {16, ne * 16, ne * 128, ps};
    const cuuint32_t box[5] = {4, 1, 1, (cuuint32_t)(N / 32), 1};
    r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 5, const_cast<uint32_t*>(base), dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) {
    set_last_error("cuTensorMapEncodeTiled (NTT eval layout) failed (%d)", (int)r);
    return kCudaError;
  }
  return kOk;
}

// the driver's encoder costs microseconds per map, which a launch on an idle
// stream would expose: keep the recently used maps (keyed by every input)
int make_eval_map(CUtensorMap* m, const uint32_t* base, long long n_entries, int N, int pl,
                  long long prime_stride, int primes) {
  struct Key {
    const uint32_t* base;
    long long n, ps;
    int N, pl, primes;
    bool operator==(const Key& o) const {
      return base == o.base && n == o.n && ps == o.ps && N == o.N && pl == o.pl &&
             primes == o.primes;
    }
  };
  struct Slot {
    Key k;
    CUtensorMap m;
  };
  constexpr int kSlots = 16;
  static Slot slots[kSlots];
  static int used = 0, next = 0;
  static std::mutex mu;
  const Key k{base, n_entries, primes > 1 ? prime_stride : 0, N, pl, primes};
  std::lock_guard<std::mutex> lk(mu);
  for (int i = 0; i < used; ++i)
    if (slots[i].k == k) {
      *m = slots[i].m;
      return kOk;
    }
  FPM_TRY(encode_eval_map(m, base, n_entries, N, pl, prime_stride, primes));
  slots[next].k = k;
  slots[next].m = *m;
  next = (next + 1) % kSlots;
  if (used < kSlots) ++used;
  return kOk;
}

int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// raise the kernel's dynamic shared-memory limit when a launch needs more
// than any earlier one (`set` is the launcher's own static)
int prepare(const void* kern, size_t smem, size_t* set) {
  if (smem > *set) {
    FPM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    *set = smem;
  }
  return kOk;
}

constexpr size_t kMaxSmem = 227 * 1024;

template <int LOGN, int G>
size_t fwd_smem(int len) {
  using T = TG<LOGN, G>;
  const int in_words = len <= T::N / 2 ? T::N / 2 : T::N;
  return 1024 + T::TAB_BYTES + (size_t)G * T::TILE_BYTES + (size_t)G * in_words * 4 + 8 * G;
}
template <int LOGN, int G>
size_t inv_smem() {
  using T = TG<LOGN, G>;
  return 1024 + T::TAB_BYTES + (size_t)G * (T::TILE_BYTES + T::N * 4) + 8 * G;
}

long long grid_x(long long items, int G, int primes) {
  long long gx = (long long)sm_count() / primes;
  if (gx < 1) gx = 1;
  const long long need = (items + G - 1) / G;
  return gx < need ? gx : need;
}

template <int LOGN, int G, int PL>
int fwd_launch(const NttFwdArgs& f, const PrimeSet& ps, cudaStream_t st) {
  using T = TG<LOGN, G>;
  TmaFwdArgs a{};
  a.in1 = (const uint32_t*)f.in; a.in1_stride = f.in_stride; a.in1_ps = f.in_prime_stride;
  a.n1 = f.n_entries;
  const bool two = f.n_entries2 > 0;
  a.in2 = two ? (const uint32_t*)f.in2 : a.in1;
  a.in2_stride = two ? f.in2_stride : 0; a.in2_ps = two ? f.in2_prime_stride : 0;
  a.n2 = two ? f.n_entries2 : 0;
  a.len = f.len;
  a.in_words = f.len <= T::N / 2 ? T::N / 2 : T::N;
  a.pl = f.pblk_log ? f.pblk_log : 5;
  CUtensorMap m1, m2;
  FPM_TRY(make_eval_map(&m1, f.out, f.n_entries, T::N, a.pl, f.out_prime_stride, ps.count));
  if (two)
    FPM_TRY(make_eval_map(&m2, f.out2, f.n_entries2, T::N, a.pl, f.out2_prime_stride, ps.count));
  else
    m2 = m1;
  const size_t smem = fwd_smem<LOGN, G>(f.len);
  static size_t set = 0;
  FPM_TRY(prepare((const void*)ntt_fwd_tma<LOGN, G, PL>, smem, &set));
  dim3 grid((unsigned)grid_x(a.n1 + a.n2, G, ps.count), 1, (unsigned)ps.count);
  FPM_CUDA_TRY(launch_pdl(ntt_fwd_tma<LOGN, G, PL>, grid, dim3(T::THREADS), smem, st, m1, m2, a, ps));
  FPM_LAUNCH_CHECK();
  return kOk;
}

template <int LOGN, int G, int PL>
int inv_launch(const NttInvArgs& f, const PrimeSet& ps, cudaStream_t st) {
  using T = TG<LOGN, G>;
  TmaInvArgs a{};
  a.out = f.out; a.out_stride = f.out_stride; a.out_ps = f.out_prime_stride;
  a.n = f.n_entries; a.out_len = f.out_len; a.off = f.off;
  a.pl = f.pblk_log ? f.pblk_log : 5;
  CUtensorMap m;
  FPM_TRY(make_eval_map(&m, f.in, f.n_entries, T::N, a.pl, f.in_prime_stride, ps.count));
  const size_t smem = inv_smem<LOGN, G>();
  static size_t set = 0;
  FPM_TRY(prepare((const void*)ntt_inv_tma<LOGN, G, PL>, smem, &set));
  dim3 grid((unsigned)grid_x(a.n, G, ps.count), 1, (unsigned)ps.count);
  FPM_CUDA_TRY(launch_pdl(ntt_inv_tma<LOGN, G, PL>, grid, dim3(T::THREADS), smem, st, m, a, ps));
  FPM_LAUNCH_CHECK();
  return kOk;
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// variant 0: 512 threads per CTA (768 measured slower: spills);
// 2: one group per CTA, for batches too small to give every SM two groups
// (cfg1: latency, not throughput)
template <int PL>
int fwd_pl(int logn, int var, const NttFwdArgs& a, const PrimeSet& ps, cudaStream_t st) {
  switch (logn) {
    case 11:
      return var == 2 ? fwd_launch<11, 1, PL>(a, ps, st) : fwd_launch<11, 8, PL>(a, ps, st);
    case 12:
      return var == 2 ? fwd_launch<12, 1, PL>(a, ps, st) : fwd_launch<12, 4, PL>(a, ps, st);
    case 13:
      return var == 2 ? fwd_launch<13, 1, PL>(a, ps, st) : fwd_launch<13, 2, PL>(a, ps, st);
  }
  return kUnsupported;
}
template <int PL>
int inv_pl(int logn, int var, const NttInvArgs& a, const PrimeSet& ps, cudaStream_t st) {
  switch (logn) {
    case 11:
      return var == 2 ? inv_launch<11, 1, PL>(a, ps, st) : inv_launch<11, 8, PL>(a, ps, st);
    case 12:
      return var == 2 ? inv_launch<12, 1, PL>(a, ps, st) : inv_launch<12, 4, PL>(a, ps, st);
    case 13:
      return var == 2 ? inv_launch<13, 1, PL>(a, ps, st) : inv_launch<13, 2, PL>(a, ps, st);
  }
  return kUnsupported;
}

int small_batch(long long items, int primes) {
  const bool off = option(kOptNttNoSmall) != 0;
  return !off && items * primes <= 2LL * sm_count();
}

}  // namespace

bool ntt_tma_fwd_ok(int logn, const NttFwdArgs& a) {
  const bool off = option(kOptNttNoTma) != 0;
  if (off || logn < 11 || logn > 13) return false;
  if (a.len2 > 0 && a.len2 != a.len) return false;  // one length for both batches
  if (a.fold || a.in64 || a.reduce || a.natural || a.pm) return false;
  const int pl = a.pblk_log ? a.pblk_log : 5;
  if (pl != 5 && pl != 2) return false;
  if (a.len <= 0 || a.len > (1 << logn) || (a.len & 3) || a.n_entries <= 0) return false;
  if (logn == 13 && fwd_smem<13, 2>(a.len) > kMaxSmem) return false;
  if ((a.in_stride & 3) || (a.in_prime_stride & 3) || !aligned16(a.in) || !aligned16(a.out) ||
      (a.out_prime_stride & 3))
    return false;
  if (a.n_entries2 > 0 && ((a.in2_stride & 3) || (a.in2_prime_stride & 3) || !aligned16(a.in2) ||
                           !aligned16(a.out2) || (a.out2_prime_stride & 3)))
    return false;
  return true;
}

bool ntt_tma_inv_ok(int logn, const NttInvArgs& a) {
  const bool off = option(kOptNttNoTma) != 0;
  if (off || logn < 11 || logn > 13) return false;
  if (a.natural || a.pm || !a.scale || a.n_entries <= 0) return false;
  const int pl = a.pblk_log ? a.pblk_log : 5;
  if (pl != 5 && pl != 2) return false;
  return aligned16(a.in) && (a.in_prime_stride & 3) == 0;
}

int launch_ntt_fwd_tma(int logn, const NttFwdArgs& a, const PrimeSet& ps, cudaStream_t st) {
  int var = 0;
  if (small_batch((long long)a.n_entries + (a.n_entries2 > 0 ? a.n_entries2 : 0), ps.count)) var = 2;
  return (a.pblk_log == 2) ? fwd_pl<2>(logn, var, a, ps, st) : fwd_pl<5>(logn, var, a, ps, st);
}

int launch_ntt_inv_tma(int logn, const NttInvArgs& a, const PrimeSet& ps, cudaStream_t st) {
  int var = 0;
  if (small_batch(a.n_entries, ps.count)) var = 2;
  return (a.pblk_log == 2) ? inv_pl<2>(logn, var, a, ps, st) : inv_pl<5>(logn, var, a, ps, st);
}

}  // namespace fpm
