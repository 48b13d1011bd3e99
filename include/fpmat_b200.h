/*
 * fpmat_b200.h -- C ABI of libfpm_b200.so, the B200 (sm_100a) drop-in for the
 * F_p polynomial-matrix multiply and PM-Basis path of the reference `fpmat`
 * package (/root/reference/pkg/src/fpmat, arXiv:1905.04356 / PML).
 *
 * The reference has no FFI of its own: its boundary is the set of Python
 * callables below.  Every entry point here replaces
 * exactly one of them; INTEGRATION.md shows the ctypes binding a maintainer
 * adds to fpmat to route those callables through this library.
 *
 * Conventions
 *   - Plain pointers and sizes only.  "dev" buffers are device pointers on
 *     the context's device, ordered on the context stream; "host" buffers
 *     are host pointers (pinned or pageable), copied synchronously.
 *   - Polynomial matrices are dense, entry-major: coefficient t of entry
 *     (i, j) of an r x c matrix with length L sits at [(i*c + j)*L + t]
 *     (low degree first, trailing zeros allowed; the reference trims,
 *     upoly.py:34-37, and compares trimmed lists, polmat.py:184-189).
 *   - elem_bytes = 4: uint32 elements (requires p < 2^32);
 *     elem_bytes = 8: uint64 elements (any prime 2 < p < 2^62).
 *     All inputs must already be reduced into [0, p).
 *   - Every function returns 0 on success or an FPM_ERR_* code; the message
 *     is available from fpm_last_error() (thread-local).  Error codes map
 *     1:1 onto the reference exception classes (fpmat/errors.py).
 *   - Calls are deterministic: no result depends on atomics ordering.
 *   - Device entry points are stream-ordered and return without waiting,
 *     except where the reference's own dispatch needs a device value on the
 *     host: fpm_polmat_middle / fpm_pm_middle_product read deg A and deg B
 *     (one synchronisation, polmat.py:477-497) and fpm_mbasis / fpm_pmbasis
 *     return *lp = deg P + 1 (one synchronisation at exit; fpm_pmbasis also
 *     reads back the degrees of the two child bases at every node of order
 *     >= 1024 to size that node's product).  *_host entry points return
 *     after their results are in host memory.
 */
#ifndef FPMAT_B200_H
#define FPMAT_B200_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes -> reference exceptions (errors.py) */
#define FPM_OK 0
#define FPM_ERR_DIM_MISMATCH 1        /* errors.DimMismatch     (polmat.py:250-253) */
#define FPM_ERR_CTX_MISMATCH 2        /* errors.CtxMismatch     (polmat.py:241-243) */
#define FPM_ERR_ORDER_TOO_SMALL 3     /* errors.OrderTooSmall   (polmat.py:295-296) */
#define FPM_ERR_FIELD_TOO_SMALL 4     /* errors.FieldTooSmall   (polmat.py:397-398) */
#define FPM_ERR_DEGREE_TOO_LARGE 5    /* errors.DegreeTooLarge  (polmat.py:477-480) */
#define FPM_ERR_ENVELOPE_EXCEEDED 6   /* errors.EnvelopeExceeded (polmat.py:583-586) */
#define FPM_ERR_LENGTH_MISMATCH 7     /* errors.LengthMismatch  (modring.py:274-275) */
#define FPM_ERR_OUT_OF_RANGE 8        /* errors.OutOfRange      (modring.py:157-158) */
#define FPM_ERR_COMPOSITE_MODULUS 9   /* errors.CompositeModulus (modring.py:159-160) */
#define FPM_ERR_DUPLICATE_POINTS 10   /* errors.DuplicatePoints (appint.py:203-205) */
#define FPM_ERR_NO_SUCH_ELEMENT 11    /* errors.NoSuchElement   (modring.py:195-196) */
#define FPM_ERR_INVALID_ARGUMENT 20   /* ValueError */
#define FPM_ERR_UNSUPPORTED 21        /* size outside the implemented kernels */
#define FPM_ERR_CUDA 30
#define FPM_ERR_NO_DEVICE 31
#define FPM_ERR_OUT_OF_MEMORY 32

typedef struct fpm_context fpm_context;

/* ---- runtime ---------------------------------------------------------- */
int fpm_version(void);
const char* fpm_last_error(void);
/* number of kernels this library has launched (all contexts) */
long long fpm_launch_count(void);
int fpm_context_create(int device, fpm_context** out);
void fpm_context_destroy(fpm_context* ctx);
/* use a caller-owned cudaStream_t (e.g. torch.cuda.current_stream()) */
int fpm_context_set_stream(fpm_context* ctx, void* cuda_stream);
int fpm_context_synchronize(fpm_context* ctx);

/* ---- field (modring.field_new, modring.py:151-171) ----------------------
 * two_adicity and the 2^k-order root (smallest QNR ^ ((p-1) >> k)).
 * FPM_ERR_OUT_OF_RANGE unless 2 < p < 2^62; FPM_ERR_COMPOSITE_MODULUS. */
int fpm_field_info(uint64_t p, int* two_adicity, uint64_t* ntt_root);
/* modring.is_prime (modring.py:25-47): 1 if n is prime (any n < 2^64) */
int fpm_is_prime(uint64_t n);
/* modring.factorize (modring.py:74-105): distinct primes ascending with
 * exponents; *count = number of primes (FPM_ERR_INVALID_ARGUMENT if > cap) */
int fpm_factorize(uint64_t n, uint64_t* primes, int* exps, int cap, int* count);
/* FieldCtx.element_order (modring.py:131-148): order of a mod p, a != 0 */
int fpm_element_order(uint64_t p, uint64_t a, uint64_t* order);
/* modring.order_at_least (modring.py:186-201): the smallest a >= 2 of
 * multiplicative order >= n (1 for n <= 1); FPM_ERR_NO_SUCH_ELEMENT when
 * n > p - 1 */
int fpm_order_at_least(uint64_t p, uint64_t n, uint64_t* a);

/* ---- NTT (modring.ntt_forward / ntt_inverse, modring.py:272-286) --------
 * batch transforms of length 2^log_len, natural order in and out:
 * forward out[j] = F(w^j) with the reference root w (modring.py:233);
 * inverse applies w^-1 and scales by N^-1.  dev buffers, batch*N elements.
 * Any 0 <= log_len <= two_adicity(p) (modring.py:220-224, FPM_ERR_OUT_OF_RANGE
 * beyond): single-CTA kernels up to 2^15, multi-pass transforms over HBM
 * above (2^16 .. 2^27 for p = 2013265921).
 * fpm_ntt_u32: 2 < p < 2^31.  fpm_ntt_u64: any prime 2 < p < 2^62 (31-bit
 * primes take the u32 kernels, larger ones a radix-2 Montgomery transform). */
int fpm_ntt_u32(fpm_context* ctx, uint32_t p, int log_len, int batch,
                const uint32_t* in_dev, uint32_t* out_dev, int inverse);
int fpm_ntt_u64(fpm_context* ctx, uint64_t p, int log_len, int batch,
                const uint64_t* in_dev, uint64_t* out_dev, int inverse);

/* ---- pm_mul (polmat.pm_mul, polmat.py:447-467) ---------------------------
 * C (m x n, length la+lb-1) = A (m x k, length la) * B (k x n, length lb).
 * Exact product; identical to every reference strategy.
 * 31-bit NTT primes run a direct transform; every other prime runs an exact
 * multi-prime product with CRT reconstruction. */
int fpm_polmat_mul(fpm_context* ctx, uint64_t p, int elem_bytes,
                   const void* A_dev, int m, int k, int la,
                   const void* B_dev, int n, int lb, void* C_dev);
int fpm_polmat_mul_host(fpm_context* ctx, uint64_t p, int elem_bytes,
                        const void* A_host, int m, int k, int la,
                        const void* B_host, int n, int lb, void* C_host);

/* ---- multi-prime pieces (for splitting a product over GPUs by prime,
 *      SURVEY.md 8e) -------------------------------------------------------
 * fpm_product_primes: the word primes fpm_polmat_mul runs a product of
 * A (m x k, length la) by B (k x n, length lb) over -- {p} for a 31-bit NTT
 * prime of enough two-adicity, else the CRT set (the reference computes the
 * same unique product geometrically, polmat.py:311-346).
 * fpm_split_residues: out[z][i] = in[i] mod primes[z] (device, n elements).
 * fpm_crt_combine: residues [r][entries][len] (device) -> out mod p, the
 * Garner recombination fpm_polmat_mul applies (elem_bytes 4 or 8). */
int fpm_product_primes(uint64_t p, int k, int la, int lb, uint32_t* primes, int cap,
                       int* count);
int fpm_split_residues(fpm_context* ctx, int elem_bytes, const void* in_dev, long long n,
                       const uint32_t* primes, int r, uint32_t* out_dev);
int fpm_crt_combine(fpm_context* ctx, uint64_t p, int elem_bytes, const uint32_t* primes, int r,
                    const uint32_t* res_dev, long long entries, int len, void* out_dev);

/* ---- Multiplier (polmat.Multiplier / multiplier_precompute /
 *      multiplier_apply, polmat.py:550-610) ------------------------------------
 * A fixed left factor A (m x k, length la; copied on create) whose forward
 * transforms stay cached on the device: each apply transforms only B.
 * max_rhs_len = max_rhs_degree + 1 fixes the cyclic length; an apply with
 * lb > max_rhs_len returns FPM_ERR_ENVELOPE_EXCEEDED (polmat.py:583-586).
 * C_dev receives m x n with length la + lb - 1. */
typedef struct fpm_multiplier fpm_multiplier;
int fpm_multiplier_create(fpm_context* ctx, uint64_t p, int elem_bytes, const void* A_dev,
                          int m, int k, int la, int max_rhs_len, fpm_multiplier** out);
int fpm_multiplier_apply(fpm_multiplier* mult, const void* B_dev, int n, int lb, void* C_dev);
void fpm_multiplier_destroy(fpm_multiplier* mult);

/* ---- middle product (polmat._pm_middle / pm_middle_product,
 *      polmat.py:470-536) ----------------------------------------------------
 * R (m x n, length d): exact == 0 reproduces the reference `_pm_middle`
 * bit for bit (including its cyclic fold); exact == 1 returns
 * the true slice [c, c+d) of A*B (the SPEC S:219 contract).  The checked
 * public variant raises FPM_ERR_DEGREE_TOO_LARGE like pm_middle_product. */
int fpm_polmat_middle(fpm_context* ctx, uint64_t p, int elem_bytes,
                      const void* A_dev, int m, int k, int la,
                      const void* B_dev, int n, int lb,
                      long long c, int d, int exact, void* R_dev);
int fpm_pm_middle_product(fpm_context* ctx, uint64_t p, int elem_bytes,
                          const void* A_dev, int m, int k, int la,
                          const void* B_dev, int n, int lb,
                          long long c, int d, void* R_dev);

/* ---- approximant bases (appint.mbasis / pmbasis, appint.py:143-196) -----
 * F (m x n, length lf) device; shift: m int64 (host).  P_dev receives the
 * m x m basis with room for order+1 coefficients; *lp = deg(P)+1.
 * Output identical to the reference for every base threshold (the result
 * is the product of the canonical order-1 steps, appint.py:24-60).
 * rdeg_out (host, optional, m int64): rdeg_s(P) after _finish_shift. */
int fpm_mbasis(fpm_context* ctx, uint64_t p, int elem_bytes,
               const void* F_dev, int m, int n, int lf, int order,
               const int64_t* shift, void* P_dev, int* lp, int64_t* rdeg_out);
int fpm_pmbasis(fpm_context* ctx, uint64_t p, int elem_bytes,
                const void* F_dev, int m, int n, int lf, int order,
                const int64_t* shift, void* P_dev, int* lp, int64_t* rdeg_out);
int fpm_pmbasis_host(fpm_context* ctx, uint64_t p, int elem_bytes,
                     const void* F_host, int m, int n, int lf, int order,
                     const int64_t* shift, void* P_host, int* lp, int64_t* rdeg_out);
/* ---- interpolant bases (appint.m_intbasis / pm_intbasis,
 *      appint.py:208-319) --------------------------------------------------
 * E_dev: order constant matrices m x n, point-major [order][m][n]; alpha:
 * order host points as uint64 integers, pairwise distinct as integers like
 * appint._check_points (appint.py:203-205; else FPM_ERR_DUPLICATE_POINTS),
 * reduced mod p inside (1 and 1 + p are distinct points with one residue);
 * shift: m int64 (host).  P_dev receives the
 * m x m s-ordered weak Popov interpolant basis with room for order+1
 * coefficients; *lp = deg(P)+1; rdeg_out (host, optional) = rdeg_s(P).
 * Pivot rows are multiplied by (x - alpha_k) (appint.py:79-117); the output
 * is the reference's for every base threshold.  31-bit primes only
 * (FPM_ERR_UNSUPPORTED otherwise), elem_bytes = 4. */
int fpm_pm_intbasis(fpm_context* ctx, uint64_t p, int elem_bytes, const void* E_dev, int m,
                    int n, int order, const uint64_t* alpha, const int64_t* shift,
                    void* P_dev, int* lp, int64_t* rdeg_out);
int fpm_m_intbasis(fpm_context* ctx, uint64_t p, int elem_bytes, const void* E_dev, int m,
                   int n, int order, const uint64_t* alpha, const int64_t* shift,
                   void* P_dev, int* lp, int64_t* rdeg_out);
/* eval_polmat_points (appint.py:262-287): out_dev[t][i][j] = P_ij(pts[t]),
 * P_dev m x n of length L; npts host points; 31-bit primes, elem_bytes 4. */
int fpm_polmat_eval_points(fpm_context* ctx, uint64_t p, int elem_bytes, const void* P_dev,
                           int m, int n, int L, const uint64_t* pts, int npts, void* out_dev);

/* Tuning / A-B switches of the kernel selection (no environment variable
 * is read).  Defaults are the product configuration; name NULL resets all.
 * Names: no_pdl, host_blocks, no_chirp, ntt_generic, ntt_no_tma,
 * ntt_no_small, ntt_pm_lsu, ntt_pm_scatter, pmbasis_leaf, pmbasis_host_sync,
 * ntt_no_mma, tc_no_pair, tc_pair1, ntt_mma_r16, tc_narrow.
 * FPM_ERR_INVALID_ARGUMENT for an unknown name. */
int fpm_set_option(const char* name, long long value);

/* base-case threshold used by fpm_pmbasis (default 32, config.py:18) */
int fpm_set_pmbasis_threshold(fpm_context* ctx, int T);

/* ---- interchange formats (polmat.polmat_to_text / polmat_from_text,
 *      polmat.py:617-647) -- host code, all host threads --------------------
 * Text is the reference's CLI format byte for byte: header "p m n", one line
 * per entry (row-major), trimmed coefficients low degree first separated by
 * one space, empty line for the zero polynomial, final newline.  M is a dense
 * host matrix m x n x L (elem_bytes 4 or 8, entries trimmed on output).
 * Reading follows polmat_from_text: str.splitlines() / str.split()
 * semantics, integer tokens of any size reduced with Python's `% p`, missing
 * lines are zero entries; FPM_ERR_INVALID_ARGUMENT (ValueError) for an empty
 * text, a header that is not three integers or a non-integer token. */
int fpm_polmat_text_size(uint64_t p, int elem_bytes, const void* M_host, int m, int n, int L,
                         size_t* bytes);
int fpm_polmat_to_text(uint64_t p, int elem_bytes, const void* M_host, int m, int n, int L,
                       char* out, size_t cap, size_t* written);
/* header and the longest entry after reduction and trimming */
int fpm_polmat_text_dims(const char* text, size_t len, long long* p, int* m, int* n,
                         int* max_len);
/* dense m x n x L host output, zero-padded */
int fpm_polmat_from_text(const char* text, size_t len, int elem_bytes, void* M_host, int L);

/* ---- tracing: per-stage device time (CUDA events on the context stream) --
 * enable (clears previous records), run calls, then read stage i's name and
 * milliseconds (synchronizes on that stage). */
int fpm_profile_enable(fpm_context* ctx, int on);
int fpm_profile_count(fpm_context* ctx);
int fpm_profile_get(fpm_context* ctx, int i, char* name, int name_len, float* ms);

#ifdef __cplusplus
}
#endif
#endif /* FPMAT_B200_H */
