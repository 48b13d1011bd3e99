// tc_grouped.cu -- int8 tensor-core per-point products for SMALL matrices
// (m <= 128: BASELINE cfg2 32x32x32, cfg3 16x16x16 per CRT prime, the cfg4
// PM-Basis nodes 64x64x32).  Replaces the per-point `_dense.mat_mul(a, b, p)`
// loop of `_pm_mul_ntt` / `_pm_middle` (polmat.py:300, :514; _dense.py:39-74).
//
// Limb identity (as tc_pointwise.cu): with s_q = 2^(8q) B mod p,
//   C = sum_r 2^(8r) D_r,  D_r[i][j] = sum_{l,q} byte_q(A[i][l]) * byte_r(s_q[l][j])
// so one u8 x u8 -> s32 GEMM with K' = 4k (A's raw little-endian bytes) and
// N' = 4n (row 4j + r of the B operand) gives every D_r exactly.
//
// Grouping.  A UMMA tile has M = 128 rows; a point has only m rows.  Let
// mp = next power of two >= m (16..128) and G = 128 / mp: one TMA box loads
// the A blocks of G consecutive points as the 128 rows of one tile (rows
// g*mp + i, OOB rows zero).  For point g the MMA multiplies the WHOLE tile by
// point g's B operand into its own TMEM accumulator; only lanes g*mp .. +m-1
// of that accumulator are read back (the other lanes hold products of other
// points' A with B_g and are ignored).  The tensor core does G x the useful
// work, which it has to spare; the CUDA cores only build B operands and run
// the epilogue (about 20 instructions per element instead of 4 per MAC).
//
// Warp roles (persistent, one CTA per SM, 18 warps):
//   warp 0      TMA producer: A tile (128 B rows, SWIZZLE_128B) + raw u32 B
//               block of the G points, one mbarrier per stage (NS = 3)
//   warp 1      TMEM allocator and single-thread MMA issuer
//   warps 2-5   epilogue (one per TMEM lane quadrant):
//               tcgen05.ld -> combine limbs -> reduce -> global
//   warps 6-17  B builders: 3 lazy Shoup scalings + 4x4 byte transpose per
//               element into a ring of SWIZZLE_NONE K-major B tiles
// Accumulators rotate through 512 TMEM columns (4nb columns each), so the
// epilogue of point g overlaps the MMAs of later points.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "tc_common.cuh"
#include "tc_pointwise.cuh"

namespace fpm {
namespace {

constexpr int kEpiWarp0 = 2, kEpiWarps = 4;            // one warp per TMEM lane quadrant
constexpr int kConvWarp0 = kEpiWarp0 + kEpiWarps, kConvWarps = 12;
constexpr int kConvThreads = kConvWarps * 32;
constexpr int kThreads = (kConvWarp0 + kConvWarps) * 32;  // 18 warps
constexpr int NS = 3;                       // load stages
constexpr uint32_t kTileA = 16384;          // 128 rows x 128 B
constexpr uint32_t kRawB = 16384;           // G * 32 * NB u32 <= 16 KB
constexpr uint32_t kSboB = 1040;            // 8 N' rows x 128 B + 16 B pad
constexpr uint32_t kRing = 96 * kSboB;      // B tile ring (99840 B)
constexpr uint32_t kOffRaw = NS * kTileA;
constexpr uint32_t kOffRing = kOffRaw + NS * kRawB;
constexpr size_t kSmem = kOffRing + kRing + 1024;  // + 1024-B alignment slack
constexpr int kMaxRing = 24, kMaxAcc = 16;

struct GArgs {
  uint32_t* C;
  int m, k, n, npts, nz;
  long long c_ps;
  int mp, G, nblk, ngroups, nch;
  int nring, nacc;
  int mtiles;       // 128-row M tiles per point (m > 128: G = 1)
};

// position in a ring of mbarrier-guarded buffers (index + phase bit)
struct RingPos {
  int idx;
  uint32_t ph;
  __device__ __forceinline__ void next(int n) {
    if (++idx == n) {
      idx = 0;
      ph ^= 1u;
    }
  }
};

__device__ __forceinline__ void decode(const GArgs& a, int it, int& z, int& gi, int& mt,
                                       int& jb) {
  const int per_z = a.ngroups * a.mtiles * a.nblk;
  z = it / per_z;
  const int rem = it - z * per_z;
  const int gm = rem / a.nblk;
  jb = rem - gm * a.nblk;
  gi = gm / a.mtiles;
  mt = gm - gi * a.mtiles;
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t x, uint32_t y, uint32_t z,
                                             uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(x), "r"(y), "r"(z),
               "r"(w)
               : "memory");
}

template <int NB>
__global__ void __launch_bounds__(kThreads, 1)
    tc_grouped_kernel(const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmB, const __grid_constant__ GArgs a,
                      const __grid_constant__ PrimeSet ps) {
  constexpr uint32_t kTileB = (NB / 2) * kSboB;  // 4 NB rows of 128 B (+ pad)
  constexpr int kTasks = NB * 8;                 // (column, quad of l) per B tile
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t full[NS], empty[NS];
  __shared__ uint64_t bfull[kMaxRing], bempty[kMaxRing];
  __shared__ uint64_t afull[kMaxAcc], aempty[kMaxAcc];
  __shared__ uint32_t tmem_base;
  const uint32_t sraw = tc::smem_u32(smem_raw);
  const uint32_t sbase = (sraw + 1023u) & ~1023u;  // SWIZZLE_128B tiles: 1 KB aligned
  const uint32_t a_full = tc::smem_u32(full), a_empty = tc::smem_u32(empty);
  const uint32_t a_bfull = tc::smem_u32(bfull), a_bempty = tc::smem_u32(bempty);
  const uint32_t a_afull = tc::smem_u32(afull), a_aempty = tc::smem_u32(aempty);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = a.G, nch = a.nch, nring = a.nring, nacc = a.nacc;
  const int items = a.nz * a.ngroups * a.mtiles * a.nblk;  // < 2^31 (host-checked)

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmB);
    for (int s = 0; s < NS; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1 + kConvWarps);
    }
    for (int e = 0; e < nring; ++e) {
      tc::mbar_init(&bfull[e], kConvWarps);
      tc::mbar_init(&bempty[e], 1);
    }
    // accumulator slot c always holds point c % G (G divides nacc); it is
    // drained by the warps of the lane quadrants that point covers
    const int quads = a.mp >= 32 ? a.mp / 32 : 1;
    for (int c = 0; c < nacc; ++c) {
      tc::mbar_init(&afull[c], 1);
      tc::mbar_init(&aempty[c], quads);
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(&tmem_base, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  pdl_wait();  // operands come from the forward transforms
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    // ------------------------------ TMA producer ------------------------------
    if (lane == 0) {
      const uint32_t bytes = kTileA + (uint32_t)(128 * NB * G);
      RingPos st{0, 0};
      for (int it = blockIdx.x; it < items; it += gridDim.x) {
        int z, gi, mt, jb;
        decode(a, it, z, gi, mt, jb);
        for (int ch = 0; ch < nch; ++ch, st.next(NS)) {
          const int s = st.idx;
          tc::mbar_wait_a(a_empty + 8 * s, st.ph ^ 1u);
          tc::mbar_expect_tx(&full[s], bytes);
          tc::tma_load_4d(sbase + s * kTileA, &tmA, &full[s], ch * 32, mt * 128, gi * G, z);
          tc::tma_load_4d(sbase + kOffRaw + s * kRawB, &tmB, &full[s], jb * NB, ch * 32, gi * G,
                          z);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------- MMA issuer -------------------------------
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_u8(128, 4 * NB);
      RingPos st{0, 0}, br{0, 0}, ac{0, 0};
      for (int it = blockIdx.x; it < items; it += gridDim.x) {
        for (int ch = 0; ch < nch; ++ch, st.next(NS)) {
          tc::mbar_wait_a(a_full + 8 * st.idx, st.ph);
          tc::fence_after_sync();
          const uint32_t tA = sbase + st.idx * kTileA;
          RingPos acc = ac;
          for (int g = 0; g < G; ++g, br.next(nring), acc.next(nacc)) {
            tc::mbar_wait_a(a_bfull + 8 * br.idx, br.ph);
            if (ch == 0) tc::mbar_wait_a(a_aempty + 8 * acc.idx, acc.ph ^ 1u);
            tc::fence_after_sync();
            const uint32_t tB = sbase + kOffRing + br.idx * kTileB;
            const uint32_t d = tmem + acc.idx * 4 * NB;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
              tc::mma_u8(d, tc::make_desc_sw128(tA + ks * 32),
                         tc::make_desc(tB + ks * 256, 128, kSboB), idesc,
                         (ch > 0 || ks > 0) ? 1u : 0u);
            }
            tc::commit_a(a_bempty + 8 * br.idx);
            if (ch == nch - 1) tc::commit_a(a_afull + 8 * acc.idx);
          }
          tc::commit_a(a_empty + 8 * st.idx);
        }
        for (int g = 0; g < G; ++g) ac.next(nacc);
      }
    }
  } else if (warp < kConvWarp0) {
    // -------------------------------- epilogue --------------------------------
    const int q = warp & 3;                       // TMEM lane quadrant this warp may access
    constexpr int kLoads = NB / 8;                // tcgen05.ld x32 per accumulator row
    {
      // the points whose rows lie in this quadrant: one (mp >= 32) or two (mp = 16)
      const int g_lo = (32 * q) / a.mp, g_hi = (32 * q + 31) / a.mp;
      const int sub = nacc / G;                   // slots per point
      RingPos sp0{0, 0}, sp1{0, 0};
      for (int it = blockIdx.x; it < items; it += gridDim.x) {
        int z, gi, mt, jb;
        decode(a, it, z, gi, mt, jb);
        const uint32_t p = ps.pr[z].p;
        const uint32_t m58 = ps.pr[z].m58;
        const int j0 = jb * NB;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int g = g_lo + u;
          if (g > g_hi) break;
          RingPos& r = u ? sp1 : sp0;
          const int slot = r.idx * G + g;
          tc::mbar_wait_sleep_a(a_afull + 8 * slot, r.ph);
          tc::fence_after_sync();
          const int il = 32 * q + lane - g * a.mp;  // row within the point's tile
          const int i = mt * 128 + il;
          const int t = gi * G + g;
          const bool ok = il >= 0 && il < a.mp && i < a.m && t < a.npts;
          uint32_t* Crow = a.C + z * a.c_ps + ((long long)t * a.m + (ok ? i : 0)) * a.n;
#pragma unroll 1
          for (int cc = 0; cc < kLoads; ++cc) {
            uint32_t v[32];
            tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + slot * 4 * NB + 32 * cc, v);
            if (ok) {
              uint32_t o[8];
#pragma unroll
              for (int x = 0; x < 8; ++x) {
                // D_r < 4k 255^2 <= 2^31, so the limb sum is < 2^56
                uint64_t acc = (uint64_t)v[4 * x];
                acc += (uint64_t)v[4 * x + 1] << 8;
                acc += (uint64_t)v[4 * x + 2] << 16;
                acc += (uint64_t)v[4 * x + 3] << 24;
                o[x] = d_red56(acc, p, m58);
              }
              const int j = j0 + 8 * cc;
              if (j + 8 <= a.n) {
                *reinterpret_cast<uint4*>(Crow + j) = make_uint4(o[0], o[1], o[2], o[3]);
                *reinterpret_cast<uint4*>(Crow + j + 4) = make_uint4(o[4], o[5], o[6], o[7]);
              } else {
#pragma unroll
                for (int x = 0; x < 8; ++x)
                  if (j + x < a.n) Crow[j + x] = o[x];
              }
            }
          }
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive_a(a_aempty + 8 * slot);
          r.next(sub);
        }
      }
    }
  } else {
    // -------------------------------- B builders -------------------------------
    // all G points' B tiles of a stage are built in one flat task loop
    // (task = point, quad of l, column), then released to the MMA together
    const int ct = tid - kConvWarp0 * 32;
    const uint8_t* smem = smem_raw + (sbase - sraw);
    RingPos st{0, 0}, br{0, 0};
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
      int z, gi, mt, jb;
      decode(a, it, z, gi, mt, jb);
      const PrimeConst& pc = ps.pr[z];
      const uint32_t p = pc.p;
      const uint32_t w1 = pc.sc[1].x, w1p = pc.sc[1].y, w2 = pc.sc[2].x, w2p = pc.sc[2].y;
      const uint32_t w3 = pc.sc[3].x, w3p = pc.sc[3].y;
      for (int ch = 0; ch < nch; ++ch, st.next(NS)) {
        tc::mbar_wait_sleep_a(a_full + 8 * st.idx, st.ph);
        const uint32_t* raw = reinterpret_cast<const uint32_t*>(smem + kOffRaw + st.idx * kRawB);
        {
          RingPos r = br;
          for (int u = 0; u < G; ++u, r.next(nring)) tc::mbar_wait_sleep_a(a_bempty + 8 * r.idx, r.ph ^ 1u);
        }
        for (int task = ct; task < G * kTasks; task += kConvThreads) {
          const int gg = task / kTasks, tt = task - gg * kTasks;
          const int lq = tt / NB, j = tt - lq * NB;
          int e = br.idx + gg;
          if (e >= nring) e -= nring;
          const uint32_t* src = raw + (gg * 32 + 4 * lq) * NB + j;
          uint32_t w[4][4];  // [r][u]: bytes (b_r, s1_r, s2_r, s3_r) of element l = 4lq+u
#pragma unroll
          for (int uu = 0; uu < 4; ++uu) {
            const uint32_t b = src[uu * NB];
            // lazy Shoup: any value < 2^32 congruent to 2^(8q) b is exact here
            const uint32_t s1 = d_shoup(b, w1, w1p, p);
            const uint32_t s2 = d_shoup(b, w2, w2p, p);
            const uint32_t s3 = d_shoup(b, w3, w3p, p);
            const uint32_t lo0 = __byte_perm(b, s1, 0x5140);
            const uint32_t hi0 = __byte_perm(b, s1, 0x7362);
            const uint32_t lo1 = __byte_perm(s2, s3, 0x5140);
            const uint32_t hi1 = __byte_perm(s2, s3, 0x7362);
            w[0][uu] = __byte_perm(lo0, lo1, 0x5410);
            w[1][uu] = __byte_perm(lo0, lo1, 0x7632);
            w[2][uu] = __byte_perm(hi0, hi1, 0x5410);
            w[3][uu] = __byte_perm(hi0, hi1, 0x7632);
          }
          // rows c = 4j + r: (c >> 3) = j >> 1, (c & 7) = 4 (j & 1) + r
          const uint32_t tB = sbase + kOffRing + e * kTileB + lq * 128 + (j >> 1) * kSboB +
                              (j & 1) * 64;
#pragma unroll
          for (int r = 0; r < 4; ++r)
            st_shared_v4(tB + r * 16, w[r][0], w[r][1], w[r][2], w[r][3]);
        }
        tc::fence_proxy_async();
        __syncwarp();
        for (int u = 0; u < G; ++u, br.next(nring))
          if (lane == 0) tc::mbar_arrive_a(a_bfull + 8 * br.idx);
        if (lane == 0) tc::mbar_arrive_a(a_empty + 8 * st.idx);
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

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

// 4-D u32 tensor map: dims (d0 contiguous, d1, d2, d3), byte strides of d1..d3
int make_map(CUtensorMap* m, const uint32_t* base, const uint64_t dims[4],
             const uint64_t strides[3], const uint32_t box[4], bool swz128) {
  auto fn = encode_fn();
  if (!fn) {
    set_last_error("cuTensorMapEncodeTiled unavailable");
    return kCudaError;
  }
  const cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, const_cast<uint32_t*>(base), dims,
                  strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swz128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_last_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return kCudaError;
  }
  return kOk;
}

template <int NB>
int launch_nb(const CUtensorMap& mA, const CUtensorMap& mB, const GArgs& a, const PrimeSet& ps,
              unsigned grid, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    FPM_CUDA_TRY(cudaFuncSetAttribute(tc_grouped_kernel<NB>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
    attr = true;
  }
  FPM_CUDA_TRY(launch_pdl(tc_grouped_kernel<NB>, dim3(grid), dim3(kThreads), kSmem, st, mA, mB, a, ps));
  FPM_LAUNCH_CHECK();
  return kOk;
}

}  // namespace

bool tc_grouped_applicable(int m, int k, int n, uint32_t p) {
  // k <= 8192: one s32 TMEM accumulator per limb diagonal takes every K
  // chunk, and the epilogue's bound D_r < 4k*255^2 <= 2^31 needs it
  return p < (1u << 31) && p >= (1u << 30) && m >= 1 && k >= 1 && k <= kTcMaxK && (k % 4) == 0 &&
         n >= 1 && (n % 4) == 0;
}

int launch_tc_grouped(const TcArgs& t, const PrimeSet& ps, cudaStream_t st) {
  if (t.npts <= 0 || t.m <= 0 || t.n <= 0) return kOk;
  if (!tc_grouped_applicable(t.m, t.k, t.n, ps.pr[0].p)) {
    set_last_error("tc_grouped: unsupported shape %dx%dx%d", t.m, t.k, t.n);
    return kInvalidArgument;
  }
  GArgs a{};
  a.C = t.C; a.m = t.m; a.k = t.k; a.n = t.n; a.npts = t.npts; a.nz = ps.count;
  a.c_ps = t.c_ps;
  a.mp = 16;
  while (a.mp < t.m && a.mp < 128) a.mp <<= 1;
  a.G = 128 / a.mp;
  // NB: power of two in [8, 64], <= mp so G accumulators of 4 NB columns fit TMEM
  int nb = 8;
  while (nb < t.n && nb < 64) nb <<= 1;
  if (nb > a.mp) nb = a.mp;
  a.ngroups = (t.npts + a.G - 1) / a.G;
  a.mtiles = (t.m + 127) / 128;
  {
    // few evaluation points (the PM-Basis nodes of order 16 ... 128): one item
    // per CTA is all latency (B build, MMAs and epilogue of the whole column
    // block in sequence), so narrower column blocks spread it over more SMs
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int narrow = (int)option(kOptTcNarrow);
    while (narrow && nb > narrow &&
           (long long)ps.count * a.ngroups * a.mtiles * ((t.n + nb - 1) / nb) * 2 <= sms)
      nb >>= 1;
  }
  a.nblk = (t.n + nb - 1) / nb;
  a.nch = (t.k + 31) / 32;
  const uint32_t tileB = (uint32_t)(nb / 2) * kSboB;
  a.nring = (int)(kRing / tileB);
  if (a.nring > kMaxRing) a.nring = kMaxRing;
  a.nacc = 512 / (4 * nb);
  if (a.nacc > kMaxAcc) a.nacc = kMaxAcc;

  const uint64_t nz = (uint64_t)ps.count;
  CUtensorMap mA, mB;
  {
    const uint64_t dims[4] = {(uint64_t)t.k, (uint64_t)t.m, (uint64_t)t.npts, nz};
    const uint64_t pstride = (uint64_t)(t.a_ps ? t.a_ps : (long long)t.npts * t.m * t.k) * 4;
    const uint64_t strides[3] = {(uint64_t)t.k * 4, (uint64_t)t.m * t.k * 4, pstride};
    const uint32_t box[4] = {32, (uint32_t)a.mp, (uint32_t)a.G, 1};  // mp <= 128 rows
    FPM_TRY(make_map(&mA, t.A, dims, strides, box, true));
  }
  {
    const uint64_t dims[4] = {(uint64_t)t.n, (uint64_t)t.k, (uint64_t)t.npts, nz};
    const uint64_t pstride = (uint64_t)(t.b_ps ? t.b_ps : (long long)t.npts * t.k * t.n) * 4;
    const uint64_t strides[3] = {(uint64_t)t.n * 4, (uint64_t)t.k * t.n * 4, pstride};
    const uint32_t box[4] = {(uint32_t)nb, 32, (uint32_t)a.G, 1};
    FPM_TRY(make_map(&mB, t.B, dims, strides, box, false));
  }
  const long long items = (long long)ps.count * a.ngroups * a.mtiles * a.nblk;
  if (items >= (1LL << 31)) {
    set_last_error("tc_grouped: too many work items");
    return kUnsupported;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const unsigned grid = (unsigned)(items < sms ? items : sms);
  switch (nb) {
    case 8: return launch_nb<8>(mA, mB, a, ps, grid, st);
    case 16: return launch_nb<16>(mA, mB, a, ps, grid, st);
    case 32: return launch_nb<32>(mA, mB, a, ps, grid, st);
    default: return launch_nb<64>(mA, mB, a, ps, grid, st);
  }
}

}  // namespace fpm
