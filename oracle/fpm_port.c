/*
 * fpm_port.c -- multi-threaded CPU port of the reference product path
 * polmat._pm_mul_ntt (/root/reference/pkg/src/fpmat/polmat.py:290-308) for
 * 31-bit NTT primes, used ONLY as the CPU baseline / reference arm of
 * bench.py (cpu_baseline, --impl reference).  TEST INFRASTRUCTURE, never
 * linked into the product library.
 *
 * Same algorithm as the reference, organised for host cores:
 *   1. forward NTT of every entry of A and B, zero-padded to N = 2^ceil(log2
 *      (la + lb - 1)) (polmat.py:293-294; modring.ntt_forward,
 *      modring.py:253-276), as radix-2 DIF with per-stage Shoup twiddle
 *      tables (evaluations left in bit-reversed point order, the inverse
 *      below consumes that order);
 *   2. per evaluation point the m x k times k x n product mod p
 *      (_dense.mat_mul, _dense.py:39-74): B's values split into 16-bit
 *      halves so every partial sum a * b_half < 2^47 accumulates exactly in
 *      64 bits over k <= 2^16 terms, one reduction per output;
 *   3. inverse NTT (DIT, w^-1, times N^-1; modring.py:279-286) of every
 *      output entry, truncated to la + lb - 1 coefficients (polmat.py:306).
 * Results equal fpo_pm_mul (oracle/fpm_oracle.c) and the reference on the
 * same inputs (tests/test_oracle_golden.py checks it).
 * Threads: OpenMP over entry blocks and evaluation points (all host cores).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

typedef unsigned __int128 u128;

static uint64_t pw(uint64_t a, uint64_t e, uint64_t p) {
    uint64_t r = 1;
    a %= p;
    while (e) {
        if (e & 1) r = (uint64_t)((u128)r * a % p);
        a = (uint64_t)((u128)a * a % p);
        e >>= 1;
    }
    return r;
}

static int adicity(uint64_t p) {
    int k = 0;
    uint64_t m = p - 1;
    while (!(m & 1)) { m >>= 1; ++k; }
    return k;
}

/* the reference root: smallest QNR ^ ((p-1) >> k) (modring.py:166-170) */
static uint64_t root2k(uint64_t p) {
    uint64_t a = 2;
    while (pw(a, (p - 1) / 2, p) == 1) ++a;
    return pw(a, (p - 1) >> adicity(p), p);
}

/* per-stage twiddle tables: stage with half-length h holds w_{2h}^j, j < h,
 * at offset h - 1 (total N - 1 entries), value and Shoup quotient */
typedef struct {
    uint32_t *w, *ws;
} Tw;

static void make_tw(Tw *t, uint32_t p, uint64_t omega, int logn) {
    const size_t N = (size_t)1 << logn;
    t->w = (uint32_t *)malloc(sizeof(uint32_t) * N);
    t->ws = (uint32_t *)malloc(sizeof(uint32_t) * N);
    for (size_t h = 1; h < N; h <<= 1) {
        const uint64_t step = pw(omega, N / (2 * h), p);
        uint64_t cur = 1;
        for (size_t j = 0; j < h; ++j) {
            t->w[h - 1 + j] = (uint32_t)cur;
            t->ws[h - 1 + j] = (uint32_t)(((uint64_t)cur << 32) / p);
            cur = cur * step % p;
        }
    }
}

static inline uint32_t shoup(uint32_t a, uint32_t w, uint32_t ws, uint32_t p) {
    const uint32_t q = (uint32_t)(((uint64_t)a * ws) >> 32);
    const uint32_t r = a * w - q * p; /* [0, 2p) */
    return r >= p ? r - p : r;
}

#define EB 16 /* entries transformed together, interleaved: x[t * EB + c] */

/* EB interleaved transforms (lane c = entry c), natural order in,
 * bit-reversed out (DIF): every butterfly is one EB-lane vector operation */
__attribute__((target_clones("avx512f", "avx2", "default")))
static void dif16(uint32_t *x, int logn, const Tw *t, uint32_t p) {
    const size_t N = (size_t)1 << logn;
    for (size_t h = N >> 1; h >= 1; h >>= 1) {
        const uint32_t *w = t->w + h - 1, *ws = t->ws + h - 1;
        for (size_t s = 0; s < N; s += 2 * h)
            for (size_t j = 0; j < h; ++j) {
                uint32_t *a = x + (s + j) * EB, *b = x + (s + j + h) * EB;
                const uint32_t wj = w[j], wsj = ws[j];
                for (int c = 0; c < EB; ++c) {
                    const uint32_t u = a[c], v = b[c];
                    const uint32_t sum = u + v;
                    a[c] = sum >= p ? sum - p : sum;
                    const uint32_t d = u + p - v;
                    const uint32_t q = (uint32_t)(((uint64_t)d * wsj) >> 32);
                    const uint32_t r = d * wj - q * p;
                    b[c] = r >= p ? r - p : r;
                }
            }
        if (h == 1) break;
    }
}

/* EB interleaved inverse transforms: bit-reversed in, natural out (DIT) */
__attribute__((target_clones("avx512f", "avx2", "default")))
static void dit16(uint32_t *x, int logn, const Tw *t, uint32_t p) {
    const size_t N = (size_t)1 << logn;
    for (size_t h = 1; h < N; h <<= 1) {
        const uint32_t *w = t->w + h - 1, *ws = t->ws + h - 1;
        for (size_t s = 0; s < N; s += 2 * h)
            for (size_t j = 0; j < h; ++j) {
                uint32_t *a = x + (s + j) * EB, *b = x + (s + j + h) * EB;
                const uint32_t wj = w[j], wsj = ws[j];
                for (int c = 0; c < EB; ++c) {
                    const uint32_t bv = b[c];
                    const uint32_t q = (uint32_t)(((uint64_t)bv * wsj) >> 32);
                    uint32_t v = bv * wj - q * p;
                    v = v >= p ? v - p : v;
                    const uint32_t u = a[c];
                    const uint32_t sum = u + v;
                    a[c] = sum >= p ? sum - p : sum;
                    const uint32_t d = u + p - v;
                    b[c] = d >= p ? d - p : d;
                }
            }
    }
}

/* C_t = A_t B_t mod p for one point: A_t m x k, B_t k x n (row-major).
 * Register tiles of 4 rows x 16 columns, two 64-bit accumulators (the 16-bit
 * halves of B) per output: a * b_half < 2^47, exact over 2^16 terms.  The
 * AVX-512 tile keeps its 16 accumulator vectors in registers (vpmuludq);
 * other hosts run the portable tile. */
#include <immintrin.h>

__attribute__((target("avx512f")))
static void tile_avx512(const uint32_t *At, int lda, int k, int ri, const uint32_t *blo,
                        const uint32_t *bhi, int np, uint64_t lo[4][16], uint64_t hi[4][16]) {
    __m512i L[4][2], H[4][2];
    for (int r = 0; r < 4; ++r)
        for (int h = 0; h < 2; ++h) L[r][h] = H[r][h] = _mm512_setzero_si512();
    for (int l = 0; l < k; ++l) {
        const __m512i bl0 = _mm512_cvtepu32_epi64(_mm256_loadu_si256((const __m256i *)(blo + (size_t)l * np)));
        const __m512i bl1 = _mm512_cvtepu32_epi64(_mm256_loadu_si256((const __m256i *)(blo + (size_t)l * np + 8)));
        const __m512i bh0 = _mm512_cvtepu32_epi64(_mm256_loadu_si256((const __m256i *)(bhi + (size_t)l * np)));
        const __m512i bh1 = _mm512_cvtepu32_epi64(_mm256_loadu_si256((const __m256i *)(bhi + (size_t)l * np + 8)));
        for (int r = 0; r < 4; ++r) {
            const __m512i a = _mm512_set1_epi64(r < ri ? (long long)At[(size_t)r * lda + l] : 0);
            L[r][0] = _mm512_add_epi64(L[r][0], _mm512_mul_epu32(a, bl0));
            L[r][1] = _mm512_add_epi64(L[r][1], _mm512_mul_epu32(a, bl1));
            H[r][0] = _mm512_add_epi64(H[r][0], _mm512_mul_epu32(a, bh0));
            H[r][1] = _mm512_add_epi64(H[r][1], _mm512_mul_epu32(a, bh1));
        }
    }
    for (int r = 0; r < 4; ++r) {
        _mm512_storeu_si512((void *)lo[r], L[r][0]);
        _mm512_storeu_si512((void *)(lo[r] + 8), L[r][1]);
        _mm512_storeu_si512((void *)hi[r], H[r][0]);
        _mm512_storeu_si512((void *)(hi[r] + 8), H[r][1]);
    }
}

static void tile_generic(const uint32_t *At, int lda, int k, int ri, const uint32_t *blo,
                         const uint32_t *bhi, int np, uint64_t lo[4][16], uint64_t hi[4][16]) {
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 16; ++c) lo[r][c] = hi[r][c] = 0;
    for (int l = 0; l < k; ++l) {
        const uint32_t *bl = blo + (size_t)l * np, *bh = bhi + (size_t)l * np;
        for (int r = 0; r < ri; ++r) {
            const uint64_t a = At[(size_t)r * lda + l];
            for (int c = 0; c < 16; ++c) {
                lo[r][c] += a * bl[c];
                hi[r][c] += a * bh[c];
            }
        }
    }
}

static void point_product(const uint32_t *At, const uint32_t *Bt, uint32_t *Ct, int m, int k,
                          int n, uint32_t p, uint32_t *blo, uint32_t *bhi, int avx512) {
    const int np = (n + 15) & ~15;
    for (int l = 0; l < k; ++l)
        for (int j = 0; j < np; ++j) {
            const uint32_t b = j < n ? Bt[(size_t)l * n + j] : 0;
            blo[(size_t)l * np + j] = b & 0xffffu;
            bhi[(size_t)l * np + j] = b >> 16;
        }
    uint64_t lo[4][16], hi[4][16];
    for (int i0 = 0; i0 < m; i0 += 4) {
        const int ri = m - i0 < 4 ? m - i0 : 4;
        for (int j0 = 0; j0 < np; j0 += 16) {
            /* 2^16-term slabs keep every 64-bit partial sum exact */
            uint64_t slo[4][16] = {{0}}, shi[4][16] = {{0}};
            for (int l0 = 0; l0 < k; l0 += 65536) {
                const int kk = k - l0 < 65536 ? k - l0 : 65536;
                if (avx512)
                    tile_avx512(At + (size_t)i0 * k + l0, k, kk, ri, blo + (size_t)l0 * np + j0,
                                bhi + (size_t)l0 * np + j0, np, lo, hi);
                else
                    tile_generic(At + (size_t)i0 * k + l0, k, kk, ri, blo + (size_t)l0 * np + j0,
                                 bhi + (size_t)l0 * np + j0, np, lo, hi);
                for (int r = 0; r < 4; ++r)
                    for (int c = 0; c < 16; ++c) {
                        slo[r][c] = (slo[r][c] + lo[r][c] % p) % p;
                        shi[r][c] = (shi[r][c] + hi[r][c] % p) % p;
                    }
            }
            for (int r = 0; r < ri; ++r)
                for (int c = 0; c < 16 && j0 + c < n; ++c)
                    Ct[(size_t)(i0 + r) * n + j0 + c] = (uint32_t)((slo[r][c] + (shi[r][c] << 16)) % p);
        }
    }
}

/* C (m x n, length la+lb-1) = A (m x k, la) * B (k x n, lb), u32 values in
 * [0, p).  Requires p < 2^31 prime with two-adicity >= log2 N.  Returns 0,
 * -1 for an unsupported prime, -2 on allocation failure. */
int fpo_port_mul31(uint32_t p, const uint32_t *A, int m, int k, int la, const uint32_t *B, int n,
                   int lb, uint32_t *C, int threads) {
    if (la <= 0 || lb <= 0 || m <= 0 || n <= 0) return 0;
    const int lc = la + lb - 1;
    if (k == 0) {
        memset(C, 0, sizeof(uint32_t) * (size_t)m * n * lc);
        return 0;
    }
    int logn = 1;
    while ((1L << logn) < lc) ++logn;
    if (p >= (1u << 31) || adicity(p) < logn) return -1;
    const size_t N = (size_t)1 << logn;
    const uint64_t om = pw(root2k(p), (uint64_t)1 << (adicity(p) - logn), p);
    Tw tf, ti;
    make_tw(&tf, p, om, logn);
    make_tw(&ti, p, pw(om, p - 2, p), logn);
    const uint64_t ninv = pw(N % p, p - 2, p);
    const uint32_t ninv_s = (uint32_t)((ninv << 32) / p);
    /* evaluation buffers persist across calls (repeated bench steps do not
     * page-fault gigabytes of fresh memory each time); one caller at a time */
    static uint32_t *ws_buf = NULL;
    static size_t ws_words = 0;
    const size_t need = N * ((size_t)m * k + (size_t)k * n + (size_t)m * n);
    if (need > ws_words) {
        free(ws_buf);
        ws_buf = (uint32_t *)malloc(sizeof(uint32_t) * need);
        ws_words = ws_buf ? need : 0;
    }
    if (!ws_buf) {
        free(tf.w); free(tf.ws); free(ti.w); free(ti.ws);
        return -2;
    }
    uint32_t *EA = ws_buf, *EBv = EA + N * m * k, *EC = EBv + N * k * n;
    if (threads < 1) threads = omp_get_max_threads();
    /* 1. forward transforms, scattered to point-major E[t][row][col] */
    for (int which = 0; which < 2; ++which) {
        const uint32_t *src = which ? B : A;
        uint32_t *dst = which ? EBv : EA;
        const int rows = which ? k : m, cols = which ? n : k, len = which ? lb : la;
        const int cb = (cols + EB - 1) / EB;
#pragma omp parallel num_threads(threads)
        {
            uint32_t *buf = (uint32_t *)malloc(sizeof(uint32_t) * N * EB);
#pragma omp for schedule(dynamic)
            for (long task = 0; task < (long)rows * cb; ++task) {
                const int r = (int)(task / cb), c0 = (int)(task % cb) * EB;
                const int w = cols - c0 < EB ? cols - c0 : EB;
                memset(buf, 0, sizeof(uint32_t) * N * EB);
                for (int c = 0; c < w; ++c) {
                    const uint32_t *e = src + ((size_t)r * cols + c0 + c) * len;
                    for (int t = 0; t < len; ++t) buf[(size_t)t * EB + c] = e[t];
                }
                dif16(buf, logn, &tf, p);
                for (size_t t = 0; t < N; ++t)
                    memcpy(dst + (t * rows + r) * cols + c0, buf + t * EB, sizeof(uint32_t) * w);
            }
            free(buf);
        }
    }
    /* 2. per-point products */
#pragma omp parallel num_threads(threads)
    {
        const size_t np = (size_t)((n + 15) & ~15);
        uint32_t *blo = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)k * np);
        uint32_t *bhi = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)k * np);
        const int avx512 = __builtin_cpu_supports("avx512f");
#pragma omp for schedule(static)
        for (long t = 0; t < (long)N; ++t)
            point_product(EA + (size_t)t * m * k, EBv + (size_t)t * k * n, EC + (size_t)t * m * n,
                          m, k, n, p, blo, bhi, avx512);
        free(blo); free(bhi);
    }
    /* 3. inverse transforms of the output entries */
    const int cb = (n + EB - 1) / EB;
#pragma omp parallel num_threads(threads)
    {
        uint32_t *buf = (uint32_t *)malloc(sizeof(uint32_t) * N * EB);
#pragma omp for schedule(dynamic)
        for (long task = 0; task < (long)m * cb; ++task) {
            const int i = (int)(task / cb), j0 = (int)(task % cb) * EB;
            const int w = n - j0 < EB ? n - j0 : EB;
            for (size_t t = 0; t < N; ++t)
                memcpy(buf + t * EB, EC + (t * m + i) * n + j0, sizeof(uint32_t) * w);
            dit16(buf, logn, &ti, p);
            for (int c = 0; c < w; ++c) {
                uint32_t *o = C + ((size_t)i * n + j0 + c) * lc;
                for (int t = 0; t < lc; ++t)
                    o[t] = shoup(buf[(size_t)t * EB + c], (uint32_t)ninv, ninv_s, p);
            }
        }
        free(buf);
    }
    free(tf.w); free(tf.ws); free(ti.w); free(ti.ws);
    return 0;
}
