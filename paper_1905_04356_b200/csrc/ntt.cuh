// ntt.cuh -- batched forward/inverse NTT over 31-bit primes (sm_100a).
//
// Replaces modring.ntt_forward / ntt_inverse (modring.py:253-286) and the
// per-entry evaluation / interpolation loops of polmat._pm_mul_ntt
// (polmat.py:275-307) and polmat._pm_middle (polmat.py:498-521).
//
// Design (DESIGN.md section "NTT"):
//  * one transform of N = 2^LOGN (32 <= N <= 32768) is held by N/32 threads,
//    32 values each in registers; the LOGN DIF stages are split in passes of
//    <= 5 bits (radix-32 register butterflies), passes exchange through a
//    padded shared-memory tile (index x + x/32 => bank-conflict free);
//  * forward = Gentleman-Sande DIF (natural -> bit-reversed order), inverse =
//    Cooley-Tukey DIT (bit-reversed -> natural), so the product path never
//    permutes: evaluation points stay in DIF order between the transforms and
//    the pointwise stage, which is order agnostic;
//  * evaluations are written in the blocked point-major "eval layout"
//        E[t / 32][entry][t % 32]
//    so each thread stores one full 128-byte line per entry and the pointwise
//    kernel reads all entries of a 32-point block contiguously;
//  * twiddles come from a per-(p, N) table of (w, floor(w 2^32 / p)) pairs;
//    per-thread table offsets are hoisted so the inner loop is one LDG.64
//    with an immediate offset per butterfly (L1 resident, shared by all CTAs).
#pragma once
#include "common.cuh"

namespace fpm {

struct NttFwdArgs {
  const void* in;            // coefficients, entry e at in + e * in_stride
  long long in_stride;       // elements between consecutive entries
  long long in_prime_stride; // elements between per-prime input copies (0 = shared)
  int in64;                  // 1: uint64 elements, 0: uint32
  int len;                   // coefficients to read per entry (zero-padded to N)
  int fold;                  // len > N: fold cyclically mod x^N - 1
  int reduce;                // inputs may be >= p: reduce on load
  int natural;               // 1: natural-order output out[e*N + k] (public API)
  int pm;                    // 1: point-major output out[x*n_entries + e]
  int pblk_log;              // eval layout block: 0/5 -> E[N/32][E][32], 2 -> E[N/4][E][4]
  int n_entries;
  uint32_t* out;             // eval layout E[N/32][n_entries][32] (or natural / PM)
  long long out_prime_stride;
  // optional second batch with the same N, len and flags (persistent kernel
  // only): one launch for both product operands, no second tail wave
  const void* in2;
  long long in2_stride, in2_prime_stride;
  int n_entries2;            // 0: none
  int len2;                  // coefficients per entry of the second batch (0: len)
  uint32_t* out2;
  long long out2_prime_stride;
  int tma_pm;                // set by the persistent launcher: PM output by TMA stores
};

struct NttInvArgs {
  const uint32_t* in;        // eval layout (or natural when natural != 0)
  long long in_prime_stride;
  int natural;               // 1: natural-order input in[e*N + k] (public API)
  int pm;                    // 1: point-major input in[x*n_entries + e]
  int pblk_log;              // eval layout block (as NttFwdArgs)
  int n_entries;
  uint32_t* out;             // out[e * out_stride + t] = coeff[(off + t) mod N]
  long long out_stride;
  long long out_prime_stride;
  int out_len;
  int off;
  int scale;                 // multiply by N^-1 (1 for the product path)
  int tma_pm;                // set by the persistent launcher: PM input by TMA loads
};

// host launchers (ntt.cu); LOGN in [5, 15]
int launch_ntt_fwd(int logn, const NttFwdArgs& a, const PrimeSet& ps, cudaStream_t st);
int launch_ntt_inv(int logn, const NttInvArgs& a, const PrimeSet& ps, cudaStream_t st);

// persistent kernels (ntt_persist.cu) for the common cases, N <= 8192
bool ntt_persist_fwd_ok(int logn, const NttFwdArgs& a);
bool ntt_persist_inv_ok(int logn, const NttInvArgs& a);
int launch_ntt_fwd_persist(int logn, const NttFwdArgs& a, const PrimeSet& ps, cudaStream_t st);
int launch_ntt_inv_persist(int logn, const NttInvArgs& a, const PrimeSet& ps, cudaStream_t st);

// grouped TMA-fed kernels (ntt_tma.cu) for N = 2^11..2^13, blocked / quad layouts
bool ntt_tma_fwd_ok(int logn, const NttFwdArgs& a);
bool ntt_tma_inv_ok(int logn, const NttInvArgs& a);
int launch_ntt_fwd_tma(int logn, const NttFwdArgs& a, const PrimeSet& ps, cudaStream_t st);
int launch_ntt_inv_tma(int logn, const NttInvArgs& a, const PrimeSet& ps, cudaStream_t st);

// forward transforms on the int8 tensor cores (ntt_mma.cu): N = 4096, one
// prime 2^30 < p < 2^31, point-major output in the same DIF point order as
// the kernels above (launch_ntt_fwd picks it when it applies)
bool ntt_mma_fwd_ok(int logn, const NttFwdArgs& a, const PrimeSet& ps);
int launch_ntt_fwd_mma(const NttFwdArgs& a, const PrimeSet& ps, cudaStream_t st);
// the same transforms in two radix-64 passes (ntt_mma64.cu); the default
int launch_ntt_fwd_mma64(const NttFwdArgs& a, const PrimeSet& ps, cudaStream_t st);

// word offset of the 16-byte piece holding points x0 .. x0+3 (x0 % 4 == 0)
// of entry e in the blocked eval layout E[N / 2^pl][n_entries][2^pl]
__host__ __device__ __forceinline__ long long eval_piece(int x0, long long e, long long n_entries,
                                                        int pl) {
  return (((long long)(x0 >> pl) * n_entries + e) << pl) + (x0 & ((1 << pl) - 1));
}

constexpr int kMinLogN = 5;
constexpr int kMaxLogN = 15;  // single-CTA kernels; longer transforms: ntt_big.cu

// transforms of 2^16 .. 2^30 points as passes over HBM (ntt_big.cu): blocked
// eval layout (pblk_log 5) or natural order, any number of primes.  scratch:
// n_entries * N * primes words (entry-major intermediate).
class Context;
bool ntt_big_ok(int logn);
int launch_ntt_fwd_big(Context& cx, int logn, const NttFwdArgs& a, const PrimeSet& ps,
                       uint32_t* scratch, cudaStream_t st);
int launch_ntt_inv_big(Context& cx, int logn, const NttInvArgs& a, const PrimeSet& ps,
                       uint32_t* scratch, cudaStream_t st);

}  // namespace fpm
