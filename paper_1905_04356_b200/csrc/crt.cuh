// crt.cuh -- multi-prime recombination and generic-modulus helpers.
//
// For moduli the direct 31-bit NTT cannot serve (p >= 2^31 such as the
// 60-bit prime of cfg3, or primes whose two-adicity is below log2 N) the
// product is computed exactly over Z through r word-size NTT primes and
// recombined here (Garner mixed radix, then reduction mod p with 64-bit
// Montgomery arithmetic).  The reference computes the same unique product by
// geometric evaluation/interpolation (polmat.py:318-346) or Kronecker lifting
// (upoly.py:127-137); S:244 makes every strategy's output identical.
#pragma once
#include "common.cuh"

namespace fpm {

struct CrtArgs {
  const uint32_t* res;        // residues, prime z at res + z*res_prime_stride
  long long res_prime_stride;
  long long res_stride;       // elements between entries
  int n_entries, len;
  void* out;                  // u32 (out64 == 0) or u64 entries
  int out64;
  long long out_stride;
  int r;                      // number of primes
  uint32_t q[kMaxPrimes];
  uint32_t g[kMaxPrimes][kMaxPrimes];     // q_j^-1 mod q_i (j < i)
  uint32_t gsh[kMaxPrimes][kMaxPrimes];   // Shoup companions
  uint64_t P;                 // target modulus (odd, < 2^62)
  uint64_t Pni;               // -P^-1 mod 2^64
  uint64_t Mmont[kMaxPrimes]; // (prod_{j<i} q_j mod P) * 2^64 mod P
};
int launch_crt(const CrtArgs& a, cudaStream_t st);
// host: fill the Garner / Montgomery constants for primes q[0..r) and P
void crt_prepare(CrtArgs& a, const uint32_t* q, int r, uint64_t P);

// Reference `_pm_middle` entrywise semantics (polmat.py:523-536 ->
// upoly._middle, upoly.py:347-377), generic modulus, element type u32/u64.
struct MiddleEntryArgs {
  const void* A; const void* B; void* out;
  int in64, out64;
  int m, k, n, la, lb;        // dense lengths
  long long c; int d;
  uint64_t P, Pni, R2;        // Montgomery constants (R2 = 2^128 mod P)
  int two_adicity;
};
int launch_middle_entrywise(const MiddleEntryArgs& a, cudaStream_t st);

// radix-2 NTT over any odd p < 2^62 (u64 elements), natural order in and
// out: out[j] = sum_t in[t] w^(j t); scale multiplies the last stage (N^-1
// for the inverse).  lo / hi: split twiddle tables w^i (i < 2^h) and
// w^(i 2^h) (i < N / 2^h), device, normal form.  The public NTT entry point
// for moduli >= 2^31 (log N global passes; not a product-path kernel).
int launch_ntt64_generic(uint64_t p, uint64_t omega, int logn, int batch, const uint64_t* in,
                         uint64_t* out, uint64_t scale, const uint64_t* lo, const uint64_t* hi,
                         int h, cudaStream_t st);

// max trimmed entry length over a dense (rows*cols, L) matrix, written to
// *out (device int); used for degree bookkeeping (polmat.py:95-104).
int launch_max_len(const void* M, int in64, long long entries, int L, int* out,
                   cudaStream_t st);
// per-row shifted degree rdeg_s (forms.py:20-51 / appint.py:120-136):
// out[i] = max_{j, M[i][j] != 0} (len(M[i][j]) - 1 + s[j]), zero rows -> min(s)
int launch_rdeg(const void* M, int in64, int rows, int cols, int L, const int64_t* s,
                int64_t* out, cudaStream_t st);

}  // namespace fpm
