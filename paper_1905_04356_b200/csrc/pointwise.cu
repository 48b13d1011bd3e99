// pointwise.cu -- CUDA-core mod-p matrix products per evaluation point.
//
// One CTA owns a 32-point block (lane = point) and an MT x NT tile of C.
// k is walked in chunks of KC: A[MT][KC] and B[KC][NT] (32 points each) are
// staged into shared memory with 16-byte cp.async, double buffered, so the
// next chunk's global/L2 reads overlap the current chunk's multiply-adds.
// Each warp owns a 4 x 8 register tile of C (RT x CT) for its 32 points:
// per k step it reads 12 conflict-free words from shared memory and issues
// 32 IMAD.WIDE multiply-adds into 64-bit accumulators, folded every K steps
// (acc = hi * (2^32 mod p) + lo) and Barrett-reduced once at the end.
#include "pointwise.cuh"

namespace fpm {
namespace {

constexpr int RT = 4, CT = 8, KC = 8;

__device__ __forceinline__ void cp_async16(uint32_t* smem_dst, const uint32_t* gsrc, bool ok) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  const int src_bytes = ok ? 16 : 0;  // 0 -> zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gsrc),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int K, int WR, int WC>
__global__ void __launch_bounds__(WR * WC * 32, 1)
    pointwise_cc_kernel(const __grid_constant__ PointwiseArgs a,
                        const __grid_constant__ PrimeSet ps, int tiles_n) {
  pdl_wait();
  constexpr int wr = WR, wc = WC, nthreads = WR * WC * 32;
  extern __shared__ __align__(16) uint32_t sm[];
  const PrimeConst& pc = ps.pr[blockIdx.z];
  const uint32_t p = pc.p, c32 = pc.c32;
  constexpr int MT = wr * RT, NT = wc * CT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int m = a.m, k = a.k, n = a.n;
  const long long tb = blockIdx.x;
  const int i0 = (blockIdx.y / tiles_n) * MT, j0 = (blockIdx.y % tiles_n) * NT;
  const uint32_t* Ab = a.A + blockIdx.z * a.a_prime_stride + tb * (long long)(m * k) * 32;
  const uint32_t* Bb = a.B + blockIdx.z * a.b_prime_stride + tb * (long long)(k * n) * 32;
  uint32_t* Cb = a.C + blockIdx.z * a.c_prime_stride + tb * (long long)(m * n) * 32 + lane;

  constexpr int stageA = MT * KC * 32, stageB = KC * NT * 32;
  // buffer b: A at sm + b*(stageA+stageB), B right after it

  auto stage = [&](int chunk, int buf) {
    const int l0 = chunk * KC;
    // A: MT rows x KC cols, 8 16-byte pieces per (row, col) entry block
    constexpr int pa = MT * KC * 8;
    for (int q = threadIdx.x; q < pa; q += nthreads) {
      const int r = q / (KC * 8), rem = q - r * (KC * 8);
      const int l = rem >> 3, piece = rem & 7;
      const int gi = i0 + r, gl = l0 + l;
      const bool ok = gi < m && gl < k;
      const uint32_t* src = Ab + ((long long)(ok ? gi : 0) * k + (ok ? gl : 0)) * 32 + piece * 4;
      cp_async16(sm + buf * (stageA + stageB) + (r * KC + l) * 32 + piece * 4, src, ok);
    }
    constexpr int pb = KC * NT * 8;
    for (int q = threadIdx.x; q < pb; q += nthreads) {
      const int l = q / (NT * 8), rem = q - l * (NT * 8);
      const int c = rem >> 3, piece = rem & 7;
      const int gl = l0 + l, gj = j0 + c;
      const bool ok = gl < k && gj < n;
      const uint32_t* src = Bb + ((long long)(ok ? gl : 0) * n + (ok ? gj : 0)) * 32 + piece * 4;
      cp_async16(sm + buf * (stageA + stageB) + stageA + (l * NT + c) * 32 + piece * 4, src, ok);
    }
    cp_async_commit();
  };

  const int wi = warp / wc, wj = warp % wc;  // this warp's RT x CT tile
  uint64_t acc[RT][CT];
#pragma unroll
  for (int r = 0; r < RT; ++r)
#pragma unroll
    for (int c = 0; c < CT; ++c) acc[r][c] = 0;

  const int nchunks = (k + KC - 1) / KC;
  if (nchunks > 0) stage(0, 0);
  for (int ch = 0; ch < nchunks; ++ch) {
    const int buf = ch & 1;
    if (ch + 1 < nchunks) {
      stage(ch + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const uint32_t* A_s = sm + buf * (stageA + stageB) + (wi * RT) * KC * 32 + lane;
    const uint32_t* B_s = sm + buf * (stageA + stageB) + stageA + (wj * CT) * 32 + lane;
#pragma unroll
    for (int l = 0; l < KC; ++l) {
      uint32_t av[RT], bv[CT];
#pragma unroll
      for (int r = 0; r < RT; ++r) av[r] = A_s[(r * KC + l) * 32];
#pragma unroll
      for (int c = 0; c < CT; ++c) bv[c] = B_s[(l * NT + c) * 32];
#pragma unroll
      for (int r = 0; r < RT; ++r)
#pragma unroll
        for (int c = 0; c < CT; ++c) acc[r][c] += (uint64_t)av[r] * bv[c];
      if ((l + 1) % K == 0) {  // KC % K == 0: folds at fixed chunk positions
#pragma unroll
        for (int r = 0; r < RT; ++r)
#pragma unroll
          for (int c = 0; c < CT; ++c)
            acc[r][c] = (uint64_t)(uint32_t)(acc[r][c] >> 32) * c32 + (uint32_t)acc[r][c];
      }
    }
    __syncthreads();  // buffer `buf` is refilled by stage(ch + 2)
  }
  // zero-padded k (chunk tail) contributed zeros; reduce and store
#pragma unroll
  for (int r = 0; r < RT; ++r) {
    const int gi = i0 + wi * RT + r;
    if (gi >= m) break;
#pragma unroll
    for (int c = 0; c < CT; ++c) {
      const int gj = j0 + wj * CT + c;
      if (gj >= n) break;
      Cb[(long long)(gi * n + gj) * 32] = d_red64(acc[r][c], p, pc.mu);
    }
  }
}

template <int K, int WR, int WC>
int launch_t(const PointwiseArgs& a, const PrimeSet& ps, cudaStream_t st) {
  constexpr int MT = WR * RT, NT = WC * CT;
  const int tiles_m = (a.m + MT - 1) / MT, tiles_n = (a.n + NT - 1) / NT;
  constexpr size_t smem = 2 * (size_t)(MT * KC * 32 + KC * NT * 32) * 4;
  static bool attr = false;
  if (!attr && smem > 48 * 1024) {
    FPM_CUDA_TRY(cudaFuncSetAttribute(pointwise_cc_kernel<K, WR, WC>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  dim3 grid((unsigned)a.nblk, (unsigned)(tiles_m * tiles_n), (unsigned)ps.count);
  FPM_CUDA_TRY(launch_pdl(pointwise_cc_kernel<K, WR, WC>, dim3(grid), dim3(WR * WC * 32), smem, st, a, ps, tiles_n));
  FPM_LAUNCH_CHECK();
  return kOk;
}

template <int K>
int launch_k(const PointwiseArgs& a, const PrimeSet& ps, cudaStream_t st) {
  // compile-time tilings: rows 4*WR (WR in 1,2,4,8), cols 8*WC (WC in 1,2)
  const int wr = a.m > 16 ? 8 : a.m > 8 ? 4 : a.m > 4 ? 2 : 1;
  const int wc = a.n > 8 ? 2 : 1;
  switch (wr * 10 + wc) {
    case 82: return launch_t<K, 8, 2>(a, ps, st);
    case 81: return launch_t<K, 8, 1>(a, ps, st);
    case 42: return launch_t<K, 4, 2>(a, ps, st);
    case 41: return launch_t<K, 4, 1>(a, ps, st);
    case 22: return launch_t<K, 2, 2>(a, ps, st);
    case 21: return launch_t<K, 2, 1>(a, ps, st);
    case 12: return launch_t<K, 1, 2>(a, ps, st);
    default: return launch_t<K, 1, 1>(a, ps, st);
  }
}

}  // namespace

int fold_period(uint32_t p) {
  const u128 two64 = (u128)1 << 64;
  const u128 c32 = ((u128)1 << 32) % p;
  const u128 fold_max = (((u128)1 << 32) - 1) * c32 + (((u128)1 << 32) - 1);
  const u128 sq = (u128)(p - 1) * (p - 1);
  int K = 1;
  while (K < 4 && fold_max + (u128)(K + 1) * sq < two64) ++K;
  return K;
}

int launch_pointwise(const PointwiseArgs& a, const PrimeSet& ps, cudaStream_t st) {
  if (a.nblk <= 0 || a.m <= 0 || a.n <= 0) return kOk;
  int K = 4;
  for (int i = 0; i < ps.count; ++i) {
    int kk = fold_period(ps.pr[i].p);
    if (kk < K) K = kk;
  }
  switch (K) {
    case 4: return launch_k<4>(a, ps, st);
    case 3:  // KC % 3 != 0: fold every 2
    case 2: return launch_k<2>(a, ps, st);
    default: return launch_k<1>(a, ps, st);
  }
}

}  // namespace fpm
