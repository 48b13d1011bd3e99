// ops.cuh -- polynomial-matrix products built from the kernels:
//   eval (forward NTT) -> pointwise mod-p matrix products -> interpolate
//   (inverse NTT) [-> CRT for moduli outside the direct 31-bit NTT range].
//
// Reference counterparts: polmat._pm_mul_ntt (polmat.py:290-308) and the
// cyclic branch of polmat._pm_middle (polmat.py:493-522); the dispatch
// wrappers mirror pm_mul (polmat.py:447-467) and _pm_middle (:484-536).
#pragma once
#include "runtime.cuh"

namespace fpm {

// dense polynomial matrix operand: entry e's coefficients at
// ptr + e*stride (elements), `len` coefficients used (rest implied zero)
struct MatRef {
  const void* ptr;
  int is64;
  long long stride;
  int len;
};

struct OutRef {
  void* ptr;
  int is64;
  long long stride;
  int len;  // coefficients written per entry
};

// cached evaluations of a fixed left factor (Multiplier, polmat.py:550-610):
// valid for one (p, m, k, len(A), N, prime set, eval layout); refreshed in
// place when a product needs another layout
struct EvalCache {
  bool valid = false;
  uint64_t p = 0;
  int m = 0, k = 0, a_len = 0, logn = 0, r = 0, pm = 0, pblk_log = 0;
  uint32_t primes[kMaxPrimes] = {};
  uint32_t* EA = nullptr;  // context allocation, r * N * m * k words
  size_t words = 0;
};

// C = window of (A * fold_N(B)) mod (x^N - 1) over F_p:
//   C[e][t] = cyc[(off + t) mod N], t < out.len, N = 2^logn.
// With N >= len(A) + len(B) - 1 and no fold this is the plain product.
// With `cache` (`cache_b`), A's (B's) forward transforms are taken from /
// stored into it.
int cyclic_product(Context& cx, uint64_t p, int m, int k, int n, MatRef A, MatRef B,
                   int logn, long long off, OutRef C, EvalCache* cache = nullptr,
                   EvalCache* cache_b = nullptr);

// product with optional evaluation caches for either factor (host pipeline)
int polmat_mul_cached(Context& cx, uint64_t p, int m, int k, int n, MatRef A, MatRef B,
                      OutRef C, EvalCache* ca, EvalCache* cb);

// full product A*B (length la + lb - 1, truncated/padded to C.len)
int polmat_mul(Context& cx, uint64_t p, int m, int k, int n, MatRef A, MatRef B, OutRef C);

// reference `_pm_middle(A, B, c, d)` semantics (incl. its cyclic fold) when
// exact == 0; the true coefficient slice [c, c+d) of A*B when exact == 1.
// da/db: matrix degrees of A and B (-1 for zero matrices).
int polmat_middle(Context& cx, uint64_t p, int m, int k, int n, MatRef A, MatRef B,
                  int da, int db, long long c, int d, int exact, OutRef C);

// smallest logn with 2^logn >= need, at least 1 (polmat.py:294)
int ceil_log2_min1(long long need);

// device-side degree of a dense matrix (max trimmed length - 1), synchronous
// deg = max entry degree (-1 for zero); synchronizes the context stream once
// (the reference's dispatch depends on the degrees, polmat.py:477-497)
// the word primes a product A (m x k, length la) * B (k x n, length lb) at
// cyclic length 2^logn runs over: {p} when p is a 31-bit NTT prime of
// two-adicity >= logn, else the CRT set whose product bounds the integer
// convolution (kCrtPrimes order)
int select_primes(uint64_t p, int k, long long la, long long lb, int logn, uint32_t* primes,
                  int* count);
int matrix_degree(Context& cx, const void* M, int is64, long long entries, int L, int* deg);
int matrix_degrees(Context& cx, const void* M1, int is64, long long e1, int L1, const void* M2,
                   long long e2, int L2, int* deg1, int* deg2);

}  // namespace fpm
