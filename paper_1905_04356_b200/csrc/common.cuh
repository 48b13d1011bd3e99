// common.cuh -- shared types, modular arithmetic and error plumbing for the
// B200 F_p polynomial-matrix library (libfpm_b200.so).
//
// Word-size arithmetic conventions (all kernels):
//   * NTT primes are < 2^31, so 2p < 2^32 and every value lives in [0, p)
//     between butterflies; DIF butterflies feed the unreduced difference
//     (< 2p) straight into a Shoup multiply (Harvey's trick restricted to the
//     one place 2^32 > 2p allows it).
//   * Twiddles are stored as (w, w') with w' = floor(w * 2^32 / p) (Shoup).
//   * Pointwise accumulation is 64-bit with a periodic fold
//     acc = hi(acc) * (2^32 mod p) + lo(acc); see pointwise.cu.
#pragma once
#include <cstdint>
#include <cstddef>
#include <cuda_runtime.h>
#include <atomic>

namespace fpm {

// ---- status codes (mirror include/fpmat_b200.h) ---------------------------
enum Status : int {
  kOk = 0,
  kDimMismatch = 1,
  kCtxMismatch = 2,
  kOrderTooSmall = 3,
  kFieldTooSmall = 4,
  kDegreeTooLarge = 5,
  kEnvelopeExceeded = 6,
  kLengthMismatch = 7,
  kOutOfRange = 8,
  kCompositeModulus = 9,
  kDuplicatePoints = 10,
  kNoSuchElement = 11,
  kInvalidArgument = 20,
  kUnsupported = 21,
  kCudaError = 30,
  kNoDevice = 31,
  kOutOfMemory = 32,
};

extern std::atomic<long long> g_launch_count;  // kernels launched (all contexts)
void set_last_error(const char* fmt, ...);
const char* last_error();

#define FPM_CUDA_TRY(expr)                                                     \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) {                                                   \
      ::fpm::set_last_error("%s:%d: %s -> %s", __FILE__, __LINE__, #expr,      \
                            cudaGetErrorString(_e));                           \
      return ::fpm::kCudaError;                                                \
    }                                                                          \
  } while (0)

#define FPM_TRY(expr)                                                          \
  do {                                                                         \
    int _s = (expr);                                                           \
    if (_s != ::fpm::kOk) return _s;                                           \
  } while (0)

#define FPM_LAUNCH_CHECK()                                                     \
  do {                                                                         \
    ::fpm::g_launch_count.fetch_add(1, std::memory_order_relaxed);             \
    cudaError_t _e = cudaGetLastError();                                       \
    if (_e != cudaSuccess) {                                                   \
      ::fpm::set_last_error("%s:%d: kernel launch -> %s", __FILE__, __LINE__,  \
                            cudaGetErrorString(_e));                           \
      return ::fpm::kCudaError;                                                \
    }                                                                          \
  } while (0)

// ---- host-side exact arithmetic ---------------------------------------------
typedef unsigned __int128 u128;

static inline uint64_t h_mulmod(uint64_t a, uint64_t b, uint64_t p) {
  return (uint64_t)((u128)a * b % p);
}
static inline uint64_t h_powmod(uint64_t a, uint64_t e, uint64_t p) {
  uint64_t r = 1 % p;
  a %= p;
  while (e) {
    if (e & 1) r = h_mulmod(r, a, p);
    a = h_mulmod(a, a, p);
    e >>= 1;
  }
  return r;
}
static inline uint64_t h_invmod(uint64_t a, uint64_t p) { return h_powmod(a, p - 2, p); }
static inline uint32_t h_shoup(uint32_t w, uint32_t p) {
  return (uint32_t)(((uint64_t)w << 32) / p);
}
bool h_is_prime(uint64_t n);          // deterministic Miller-Rabin (modring.py:25-47)
int h_two_adicity(uint64_t p);        // modring.py:161-165
uint64_t h_ntt_root(uint64_t p);      // smallest QNR ^ ((p-1) >> k), modring.py:166-170
}  // namespace fpm
#include <map>
namespace fpm {
std::map<uint64_t, int> h_factorize(uint64_t n);  // {prime: exponent}, modring.py:74-105
// multiplicative order of a mod p given the factorisation of p - 1
uint64_t h_element_order(uint64_t p, uint64_t a, const std::map<uint64_t, int>& fac);

// ---- device helpers ---------------------------------------------------------
__device__ __forceinline__ uint32_t d_red(uint32_t x, uint32_t p) {
  // x in [0, 2p) -> [0, p); unsigned min trick (x - p wraps when x < p)
  return min(x, x - p);
}
// Shoup multiply: any a < 2^32, w < p, wp = floor(w 2^32 / p) -> [0, 2p)
__device__ __forceinline__ uint32_t d_shoup(uint32_t a, uint32_t w, uint32_t wp,
                                            uint32_t p) {
  uint32_t q = __umulhi(a, wp);
  return a * w - q * p;
}
// full reduction of a 64-bit value: x mod p for p < 2^31
// mu = floor(2^64 / p) (needs p not a power of two; p odd prime > 2)
__device__ __forceinline__ uint32_t d_red64(uint64_t x, uint32_t p, uint64_t mu) {
  uint64_t q = __umul64hi(x, mu);
  uint64_t r = x - q * (uint64_t)p;  // < 2p (Barrett error <= 1)
  uint32_t r32 = (uint32_t)r;
  return r >= p ? r32 - p : r32;
}

// x mod p for x < 2^56 and 2^30 <= p < 2^31, with m58 = floor(2^58 / p):
// q = floor((x >> 26) m58 / 2^32) is floor(x/p) or one less (the dropped low
// 26 bits and the truncation of m58 cost < 0.32), so x - q p lies in [0, 2p)
// and its low 32 bits are exact.
__device__ __forceinline__ uint32_t d_red56(uint64_t x, uint32_t p, uint32_t m58) {
  const uint32_t q = __umulhi((uint32_t)(x >> 26), m58);
  const uint32_t r = (uint32_t)x - q * p;
  return min(r, r - p);
}

// ---- programmatic dependent launch (PDL) ------------------------------------
// A kernel launched with launch_pdl() may start while the previous kernel in
// the stream drains: its prologue (tables, barriers, TMEM, descriptors)
// overlaps that kernel's tail and the launch latency.  Every such kernel
// calls pdl_wait() before touching global data another kernel may write; it
// is a no-op for an ordinary launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
// Tuning / A-B switches (fpm_set_option, include/fpmat_b200.h).  The
// defaults are the product configuration; nothing reads the environment.
enum Option : int {
  kOptNoPdl = 0,          // "no_pdl": plain launches instead of PDL
  kOptHostBlocks,         // "host_blocks": force R x R blocks in fpm_polmat_mul_host
  kOptNoChirp,            // "no_chirp": Horner instead of chirp evaluation (intbasis)
  kOptNttGeneric,         // "ntt_generic": generic single-CTA NTT kernels only
  kOptNttNoTma,           // "ntt_no_tma": skip the grouped TMA NTT
  kOptNttNoSmall,         // "ntt_no_small": no one-group-per-CTA variant
  kOptNttPmLsu,           // "ntt_pm_lsu": point-major pieces by LSU stores, not TMA
  kOptNttPmScatter,       // "ntt_pm_scatter": one transform per CTA in PM layout
  kOptPmbasisLeaf,        // "pmbasis_leaf": cap of the device leaf order (default 8)
  kOptPmbasisHostSync,    // "pmbasis_host_sync": host-synchronised recursion
  kOptNttNoMma,           // "ntt_no_mma": no tensor-core NTT (ntt_mma.cu)
  kOptTcNoPair,           // "tc_no_pair": tc_grouped instead of tc_pair for 128 < m <= 256
  kOptTcPair1,            // "tc_pair1": one-SM tc_pair instead of the CTA-pair kernel
  kOptNttMmaR16,          // "ntt_mma_r16": three radix-16 passes (ntt_mma.cu), not two radix-64
  kOptNttMmaDbg,          // "ntt_mma_dbg": timing experiments of ntt_mma64.cu (WRONG results)
  kOptTcNarrow,           // "tc_narrow": narrowest column block tc_grouped may pick to fill the SMs (0: off)
  kOptCount
};
long long option(Option o);
int set_option(const char* name, long long value);
bool pdl_enabled();  // option no_pdl

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, ((KArgs)args)...);
}

// Per-prime constants handed to kernels by value (kernel-parameter space, so
// the radix-32 root constants are constant-bank operands, not loads).
struct PrimeConst {
  uint32_t p;
  uint32_t c32;      // 2^32 mod p (pointwise fold)
  uint64_t mu;       // floor(2^64 / p) (Barrett)
  uint32_t ninv;     // N^-1 mod p for the transform length in use
  uint32_t ninv_sh;  // Shoup companion of ninv
  const uint2* tw;   // forward twiddle rows: tw[r*32 + k] = w^(r*k), N entries
  const uint2* itw;  // inverse rows: w^-(r*k), N entries
  const uint2* itw_s;  // inverse rows times N^-1 (ntt_tma.cu last pass)
  uint2 w32[16];     // (w32^e, Shoup) e < 16, w32 = w^(N/32): inner radix-32 DFTs
  uint2 iw32[16];    // inverse roots
  uint2 sc[4];       // (2^(8q) mod p, Shoup), q = 0..3: limb scaling (tc_pointwise.cu)
  uint32_t m58;      // floor(2^58 / p): reduction of < 2^56 limb sums (d_red56)
  const uint8_t* mma;  // tensor-core NTT tables (N = 4096, 2^30 < p < 2^31; ntt_mma.cu)
};

constexpr int kMaxPrimes = 8;
struct PrimeSet {
  int count;
  PrimeConst pr[kMaxPrimes];
};

}  // namespace fpm
