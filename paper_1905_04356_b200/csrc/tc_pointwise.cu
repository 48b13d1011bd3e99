// tc_pointwise.cu -- per-point mod-p matrix products on the int8 tensor cores
// (tcgen05.mma kind::i8, accumulators in TMEM).  Replaces
// `[_dense.mat_mul(a, b, p) for a, b in zip(va, vb)]` (polmat.py:300, :514;
// _dense.py:39-74) when the contraction is large (BASELINE cfg5: 4096 points
// of 256 x 256 x 256).
//
// Exact limb arithmetic.  For p < 2^31 write a = sum_q 2^(8q) a_q (bytes).
//   C[i][j] = sum_l A[i][l] B[l][j]
//           = sum_l sum_q a_q(A[i][l]) * (2^(8q) B[l][j] mod p)      (mod p)
//           = sum_r 2^(8r) sum_{l,q} a_q(A[i][l]) * r-th byte of s_q(l,j)
// with s_q = 2^(8q) B mod p.  So one u8 x u8 GEMM with K' = 4k (interleaved
// K' = 4l + q: the A operand is just the raw little-endian bytes of A) and
// N' = 4n (column 4j + r) gives D[i][4j + r]; every D < 4k * 255^2 < 2^31
// (k <= 8192) and C[i][j] = D0 + 2^8 D1 + 2^16 D2 + 2^24 D3 mod p (< 2^51).
//
// Work item = (prime, point t, 256-row group, 64-column block).  Per K-chunk
// of 32 l's: the A tile (256 x 128 B) is copied raw with cp.async, the B tile
// (256 N' rows x 128 B) is built from the u32 B block (3 Shoup scalings + a
// 4x4 byte transpose per element), then one thread issues 2 x 4 UMMA
// (128 x 256 x 32).  Three smem stages: building chunk c+1 overlaps the
// tensor core on chunk c.  The epilogue reads TMEM (tcgen05.ld 32x32b),
// combines the four limb columns and Barrett-reduces.
//
// Operands are in the point-major layout X[t][row][col] (ntt.cu PM layout).
#include "tc_pointwise.cuh"
#include "tc_common.cuh"

namespace fpm {
namespace {

constexpr int kThreads = 256;
constexpr int KL = 32;                  // l per chunk (128 bytes of K')
constexpr int NB = 64;                  // output columns per work item
constexpr int MG = 256;                 // rows per work item (2 UMMA M tiles)
constexpr uint32_t SBO_A = 1024;        // 8 rows x 128 B
constexpr uint32_t SBO_B = 1040;        // +16 B: conflict-free B tile stores
constexpr uint32_t TILE_A = (MG / 8) * SBO_A;        // 32768
constexpr uint32_t TILE_B = (4 * NB / 8) * SBO_B;    // 33280
constexpr uint32_t STAGE = TILE_A + TILE_B;
constexpr int NSTAGE = 3;
constexpr uint32_t B32 = KL * NB * 4;               // raw u32 B block (8 KB)
constexpr size_t kSmem = (size_t)NSTAGE * STAGE + 2 * B32 + 1024;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
               "r"(ok ? 16 : 0));
}

__global__ void __launch_bounds__(kThreads, 1)
    tc_pointwise_kernel(const __grid_constant__ TcArgs a, const __grid_constant__ PrimeSet ps) {
  pdl_wait();
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar[NSTAGE];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m = a.m, k = a.k, n = a.n;
  const int mgroups = (m + MG - 1) / MG, nblocks = (n + NB - 1) / NB;
  const long long per_prime = (long long)a.npts * mgroups * nblocks;
  const long long items = per_prime * ps.count;
  const int nch = (k + KL - 1) / KL;
  const uint32_t sbase = tc::smem_u32(smem);

  if (warp == 0) tc::tmem_alloc(&tmem_base, 512);
  if (tid < NSTAGE) tc::mbar_init(&mbar[tid], 1);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = tc::idesc_u8(128, 4 * NB);

  long long g = 0;  // global chunk counter (stage / mbarrier phase bookkeeping)
  for (long long it = blockIdx.x; it < items; it += gridDim.x) {
    const int z = (int)(it / per_prime);
    long long rem = it - (long long)z * per_prime;
    const long long t = rem / ((long long)mgroups * nblocks);
    rem -= t * mgroups * nblocks;
    const int mg = (int)(rem / nblocks), jb = (int)(rem - (long long)mg * nblocks);
    const PrimeConst& pc = ps.pr[z];
    const uint32_t p = pc.p;
    const uint32_t* At = a.A + z * a.a_ps + t * (long long)m * k;
    const uint32_t* Bt = a.B + z * a.b_ps + t * (long long)k * n;
    const int i0 = mg * MG, j0 = jb * NB;

    // Pipeline per chunk g: loads of chunk g+1 (raw A bytes straight into its
    // UMMA tile, the u32 B block into a staging buffer) are in flight while
    // chunk g's B tile is built from smem and while the tensor core runs
    // chunk g-1.
    auto issue_loads = [&](int ch, long long gg) {
      const int s = (int)(gg % NSTAGE);
      const uint32_t tA = sbase + s * STAGE;
      const uint32_t tS = sbase + NSTAGE * STAGE + (uint32_t)(gg & 1) * B32;
      const int l0 = ch * KL;
#pragma unroll
      for (int u = 0; u < (MG * 8) / kThreads; ++u) {
        const int q = tid + u * kThreads;
        const int r = q >> 3, kc = q & 7;
        const int gi = i0 + r, gl = l0 + 4 * kc;
        const bool ok = gi < m && gl < k;
        const uint32_t* src = At + (ok ? (long long)gi * k + gl : 0);
        cp_async16(tA + (r >> 3) * SBO_A + kc * 128 + (r & 7) * 16, src, ok);
      }
      // B block rows l0..l0+31, columns j0..j0+63 (16-byte pieces when aligned)
      if ((n & 3) == 0) {
#pragma unroll
        for (int u = 0; u < (KL * NB / 4) / kThreads; ++u) {
          const int q = tid + u * kThreads;
          const int ll = q >> 4, jq = q & 15;
          const int gl = l0 + ll, gj = j0 + 4 * jq;
          const bool ok = gl < k && gj < n;
          const uint32_t* src = Bt + (ok ? (long long)gl * n + gj : 0);
          cp_async16(tS + (ll * NB + 4 * jq) * 4, src, ok);
        }
      } else {
        uint32_t* dS = reinterpret_cast<uint32_t*>(smem + NSTAGE * STAGE + (gg & 1) * B32);
        for (int q = tid; q < KL * NB; q += kThreads) {
          const int ll = q / NB, jj = q - (q / NB) * NB;
          const int gl = l0 + ll, gj = j0 + jj;
          dS[q] = (gl < k && gj < n) ? __ldg(Bt + (long long)gl * n + gj) : 0u;
        }
      }
      asm volatile("cp.async.commit_group;\n");
    };

    const long long g0 = g;
    if (g0 >= NSTAGE) tc::mbar_wait(&mbar[g0 % NSTAGE], (uint32_t)(((g0 / NSTAGE) - 1) & 1));
    issue_loads(0, g0);
    for (int ch = 0; ch < nch; ++ch, ++g) {
      const int s = (int)(g % NSTAGE);
      if (ch + 1 < nch) {
        const long long gn = g + 1;
        // stage of chunk g+1 was last read by the MMAs of chunk g+1-NSTAGE
        if (gn >= NSTAGE) tc::mbar_wait(&mbar[gn % NSTAGE], (uint32_t)(((gn / NSTAGE) - 1) & 1));
        issue_loads(ch + 1, gn);
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      }
      __syncthreads();  // chunk g's raw A tile and B block are visible
      const uint32_t tA = sbase + s * STAGE, tB = tA + TILE_A;
      uint8_t* pB = smem + s * STAGE + TILE_A;
      const uint32_t* sBr =
          reinterpret_cast<const uint32_t*>(smem + NSTAGE * STAGE + (g & 1) * B32);
      // ---- B tile: rows c = 4jj + r, bytes 4(l - l0) + q = byte r of s_q ----
      {
        const int jj = 8 * warp + (lane >> 2);
#pragma unroll 4
        for (int u = 0; u < KL / 4; ++u) {
          const int ll = 4 * u + (lane & 3);
          const uint32_t b = sBr[ll * NB + jj];
          const uint32_t s1 = d_red(d_shoup(b, pc.sc[1].x, pc.sc[1].y, p), p);
          const uint32_t s2 = d_red(d_shoup(b, pc.sc[2].x, pc.sc[2].y, p), p);
          const uint32_t s3 = d_red(d_shoup(b, pc.sc[3].x, pc.sc[3].y, p), p);
          // 4x4 byte transpose: w_r = (byte r of b, s1, s2, s3)
          const uint32_t lo0 = __byte_perm(b, s1, 0x5140);   // b0 s1_0 b1 s1_1
          const uint32_t hi0 = __byte_perm(b, s1, 0x7362);   // b2 s1_2 b3 s1_3
          const uint32_t lo1 = __byte_perm(s2, s3, 0x5140);
          const uint32_t hi1 = __byte_perm(s2, s3, 0x7362);
          const uint32_t w0 = __byte_perm(lo0, lo1, 0x5410);  // b0 s1_0 s2_0 s3_0
          const uint32_t w1 = __byte_perm(lo0, lo1, 0x7632);  // b1 s1_1 s2_1 s3_1
          const uint32_t w2 = __byte_perm(hi0, hi1, 0x5410);
          const uint32_t w3 = __byte_perm(hi0, hi1, 0x7632);
          const uint32_t base = (jj >> 1) * SBO_B + u * 128 + 4 * (lane & 3);
          const uint32_t rb = 4 * (jj & 1);
          *reinterpret_cast<uint32_t*>(pB + base + (rb + 0) * 16) = w0;
          *reinterpret_cast<uint32_t*>(pB + base + (rb + 1) * 16) = w1;
          *reinterpret_cast<uint32_t*>(pB + base + (rb + 2) * 16) = w2;
          *reinterpret_cast<uint32_t*>(pB + base + (rb + 3) * 16) = w3;
        }
      }
      tc::fence_proxy_async();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after_sync();
#pragma unroll
        for (int ks = 0; ks < KL * 4 / 32; ++ks) {
          const uint64_t bd = tc::make_desc(tB + ks * 256, 128, SBO_B);
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            const uint64_t ad = tc::make_desc(tA + mt * 16 * SBO_A + ks * 256, 128, SBO_A);
            tc::mma_u8(tmem + mt * 256, ad, bd, idesc, (ch > 0 || ks > 0) ? 1u : 0u);
          }
        }
        tc::commit(&mbar[s]);
      }
    }
    // ---- epilogue: wait for the last chunk's MMAs, combine limbs, reduce ----
    {
      const long long gl = g - 1;
      tc::mbar_wait(&mbar[gl % NSTAGE], (uint32_t)((gl / NSTAGE) & 1));
      tc::fence_after_sync();
      const int quad = warp & 3, mt = warp >> 2;
      const int gi = i0 + mt * 128 + 32 * quad + lane;
      uint32_t* Crow = a.C + z * a.c_ps + t * (long long)m * n + (long long)gi * n;
#pragma unroll 1
      for (int cc = 0; cc < 4 * NB / 32; ++cc) {
        uint32_t v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(32 * quad) << 16) + mt * 256 + 32 * cc, v);
        if (gi < m) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int gj = j0 + 8 * cc + q;
            const uint64_t x = (uint64_t)v[4 * q] + ((uint64_t)v[4 * q + 1] << 8) +
                               ((uint64_t)v[4 * q + 2] << 16) + ((uint64_t)v[4 * q + 3] << 24);
            if (gj < n) Crow[gj] = d_red64(x, p, pc.mu);
          }
        }
      }
      tc::fence_before_sync();
      __syncthreads();  // TMEM drained before the next item's first MMA
    }
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

}  // namespace

bool tc_pointwise_applicable(int m, int k, int n, uint32_t p) {
  return p < (1u << 31) && (k % 4) == 0 && k >= 64 && k <= kTcMaxK && m >= 64 && n >= 32;
}

int launch_tc_pointwise(const TcArgs& a, const PrimeSet& ps, cudaStream_t st) {
  if (a.npts <= 0 || a.m <= 0 || a.n <= 0) return kOk;
  static bool attr = false;
  if (!attr) {
    FPM_CUDA_TRY(cudaFuncSetAttribute(tc_pointwise_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
    attr = true;
  }
  const long long items = (long long)ps.count * a.npts * ((a.m + MG - 1) / MG) *
                          ((a.n + NB - 1) / NB);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long grid = items < sms ? items : sms;
  FPM_CUDA_TRY(launch_pdl(tc_pointwise_kernel, dim3((unsigned)grid), dim3(kThreads), kSmem, st, a, ps));
  FPM_LAUNCH_CHECK();
  return kOk;
}

}  // namespace fpm
