/*
 * fpm_oracle.c -- CPU restatement of the reference `fpmat` hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path and the CPU baseline ("kind": "port") timed by bench.py.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it.  The product library (libfpm_b200.so) never
 * links or calls it.
 *
 * Parity pinning: tests/test_oracle_golden.py checks every function below
 * against fixtures produced by running the reference itself in the build
 * container (tests/golden/make_golden.py, tests/golden/make_golden_big.py).
 *
 * Element type is uint64_t throughout (the reference accepts 2 < p < 2^62,
 * modring.py:157).  Polynomial matrices are dense, entry-major:
 * M[(i*ncols + j)*len + t] = coefficient t of entry (i, j); trailing zeros
 * are allowed (the reference trims, upoly.py:34-37; equality is on trimmed
 * lists, polmat.py:184-189, so dense+trim is equivalent).
 *
 * Reference anchors (paths relative to /root/reference/pkg/src/fpmat/):
 *   field / root convention ...... modring.py:151-171
 *   NTT (radix-2 DIT, natural) ... modring.py:204-286
 *   pm_mul ....................... polmat.py:447-467 (+ _pm_mul_ntt :290-308,
 *                                  _pm_mul_naive :256-272; all strategies
 *                                  return the same unique product)
 *   _pm_middle ................... polmat.py:484-536, upoly._middle :347-377
 *   _mbasis1_struct .............. appint.py:24-60
 *   _apply_step .................. appint.py:79-117
 *   _rdeg_from_coeffs/_finish .... appint.py:120-136
 *   mbasis ....................... appint.py:143-180
 *   pmbasis ...................... appint.py:183-196
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

static int g_threads = 1;
void fpo_set_threads(int n) { g_threads = n > 0 ? n : 1; }
int fpo_get_threads(void) { return g_threads; }

static inline uint64_t mulmod(uint64_t a, uint64_t b, uint64_t p) {
    return (uint64_t)((u128)a * b % p);
}
static inline uint64_t addmod(uint64_t a, uint64_t b, uint64_t p) {
    uint64_t s = a + b;  /* p < 2^62: no overflow */
    return s >= p ? s - p : s;
}
static inline uint64_t submod(uint64_t a, uint64_t b, uint64_t p) {
    return a >= b ? a - b : a + p - b;
}
static uint64_t powmod(uint64_t a, uint64_t e, uint64_t p) {
    uint64_t r = 1 % p;
    a %= p;
    while (e) {
        if (e & 1) r = mulmod(r, a, p);
        a = mulmod(a, a, p);
        e >>= 1;
    }
    return r;
}
static uint64_t invmod(uint64_t a, uint64_t p) { return powmod(a, p - 2, p); }

/* ---- field (modring.py:151-171) ---------------------------------------- */
int fpo_two_adicity(uint64_t p) {
    uint64_t m = p - 1;
    int k = 0;
    while ((m & 1) == 0) { m >>= 1; k++; }
    return k;
}
/* smallest quadratic non-residue q, root = q^((p-1) >> k) (modring.py:166-170) */
uint64_t fpo_ntt_root(uint64_t p) {
    int k = fpo_two_adicity(p);
    uint64_t a = 2;
    while (powmod(a, (p - 1) / 2, p) == 1) a++;
    return powmod(a, (p - 1) >> k, p);
}

/* ---- NTT (modring.py:204-286) ------------------------------------------ */
/* omega = root^(2^(k - log_len)) (modring.py:233); forward natural order
 * out[j] = F(omega^j); inverse uses omega^-1 then scales by N^-1. */
int fpo_ntt(uint64_t p, int log_len, uint64_t *v, int inverse) {
    int k = fpo_two_adicity(p);
    if (log_len > k || log_len < 0) return -1;
    size_t n = (size_t)1 << log_len;
    uint64_t omega = powmod(fpo_ntt_root(p), (uint64_t)1 << (k - log_len), p);
    if (inverse) omega = invmod(omega, p);
    /* bit-reversal (modring.py:204-209, :255) */
    for (size_t i = 1, j = 0; i < n; i++) {
        size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) { uint64_t t = v[i]; v[i] = v[j]; v[j] = t; }
    }
    uint64_t *tw = (uint64_t *)malloc(sizeof(uint64_t) * (n / 2 + 1));
    for (int s = 0; s < log_len; s++) {
        size_t half = (size_t)1 << s, span = half * 2;
        uint64_t w = powmod(omega, n / span, p);
        tw[0] = 1;
        for (size_t i = 1; i < half; i++) tw[i] = mulmod(tw[i - 1], w, p);
        for (size_t start = 0; start < n; start += span)
            for (size_t i = 0; i < half; i++) {
                uint64_t t = mulmod(v[start + i + half], tw[i], p);
                uint64_t u = v[start + i];
                v[start + i] = addmod(u, t, p);
                v[start + i + half] = submod(u, t, p);
            }
    }
    free(tw);
    if (inverse) {
        uint64_t s = invmod(n % p, p);
        for (size_t i = 0; i < n; i++) v[i] = mulmod(v[i], s, p);
    }
    return 0;
}

/* ---- helpers ------------------------------------------------------------ */
static int entry_len(const uint64_t *e, int L) {
    while (L > 0 && e[L - 1] == 0) L--;
    return L;
}
/* matrix degree (polmat.py:95-104): max trimmed entry length - 1 */
static int mat_degree(const uint64_t *M, int rows, int cols, int L) {
    int d = -1;
    for (long e = 0; e < (long)rows * cols; e++) {
        int l = entry_len(M + e * (long)L, L);
        if (l - 1 > d) d = l - 1;
    }
    return d;
}
static int ceil_log2_min1(long need) {
    /* max(1, (need - 1).bit_length()) as in polmat.py:294 */
    int b = 0;
    long x = need - 1;
    while (x > 0) { b++; x >>= 1; }
    return b < 1 ? 1 : b;
}

/* ---- pm_mul ------------------------------------------------------------- */
/* C must hold m*n*(la+lb-1) entries; returns 0. The product is unique, so
 * this equals every reference strategy. NTT path when the reference's
 * _pm_mul_ntt applies (polmat.py:293-296), schoolbook otherwise
 * (_pm_mul_naive, polmat.py:256-272). */
int fpo_pm_mul(uint64_t p, const uint64_t *A, int m, int k, int la,
               const uint64_t *B, int n, int lb, uint64_t *C) {
    int lc = la + lb - 1;
    if (la <= 0 || lb <= 0) return 0;
    memset(C, 0, sizeof(uint64_t) * (size_t)m * n * lc);
    int da = mat_degree(A, m, k, la), db = mat_degree(B, k, n, lb);
    if (da < 0 || db < 0 || m == 0 || n == 0 || k == 0) return 0;
    long need = (long)da + db + 1;
    int log_len = ceil_log2_min1(need);
    int two = fpo_two_adicity(p);
    if (log_len <= two) {
        size_t N = (size_t)1 << log_len;
        uint64_t *va = (uint64_t *)calloc((size_t)m * k * N, sizeof(uint64_t));
        uint64_t *vb = (uint64_t *)calloc((size_t)k * n * N, sizeof(uint64_t));
        uint64_t *vc = (uint64_t *)calloc((size_t)m * n * N, sizeof(uint64_t));
        int ea = m * k, eb = k * n;
#pragma omp parallel for schedule(dynamic) num_threads(g_threads)
        for (int e = 0; e < ea + eb; e++) {
            uint64_t *dst = e < ea ? va + (size_t)e * N : vb + (size_t)(e - ea) * N;
            const uint64_t *src = e < ea ? A + (size_t)e * la : B + (size_t)(e - ea) * lb;
            int l = e < ea ? la : lb;
            int cl = l < (int)N ? l : (int)N;
            for (int t = 0; t < cl; t++) dst[t] = src[t] % p;
            fpo_ntt(p, log_len, dst, 0);
        }
        /* pointwise: for each point t, C_t = A_t B_t (_dense.mat_mul) */
#pragma omp parallel for schedule(static) num_threads(g_threads)
        for (long t = 0; t < (long)N; t++) {
            for (int i = 0; i < m; i++)
                for (int j = 0; j < n; j++) {
                    u128 acc = 0;
                    int cnt = 0;
                    for (int l = 0; l < k; l++) {
                        acc += (u128)va[((size_t)i * k + l) * N + t] * vb[((size_t)l * n + j) * N + t];
                        if (++cnt == 16) { acc %= p; cnt = 0; }  /* 16*(2^62)^2 < 2^128 */
                    }
                    vc[((size_t)i * n + j) * N + t] = (uint64_t)(acc % p);
                }
        }
#pragma omp parallel for schedule(dynamic) num_threads(g_threads)
        for (int e = 0; e < m * n; e++) {
            uint64_t *col = vc + (size_t)e * N;
            fpo_ntt(p, log_len, col, 1);
            int cl = lc < (int)N ? lc : (int)N;
            memcpy(C + (size_t)e * lc, col, sizeof(uint64_t) * cl);
        }
        free(va); free(vb); free(vc);
        return 0;
    }
    /* schoolbook over Z with 128-bit accumulation per output coefficient */
#pragma omp parallel for schedule(dynamic) num_threads(g_threads)
    for (int e = 0; e < m * n; e++) {
        int i = e / n, j = e % n;
        uint64_t *out = C + (size_t)e * lc;
        for (int t = 0; t < lc; t++) {
            uint64_t acc = 0;
            for (int l = 0; l < k; l++) {
                const uint64_t *a = A + ((size_t)i * k + l) * la;
                const uint64_t *b = B + ((size_t)l * n + j) * lb;
                int lo = t - lb + 1 > 0 ? t - lb + 1 : 0;
                int hi = t < la - 1 ? t : la - 1;
                u128 s = 0;
                int cnt = 0;
                for (int u = lo; u <= hi; u++) {
                    s += (u128)a[u] * b[t - u];
                    if (++cnt == 16) { s %= p; cnt = 0; }  /* 16*(2^62)^2 < 2^128 */
                }
                acc = addmod(acc, (uint64_t)(s % p), p);
            }
            out[t] = acc;
        }
    }
    return 0;
}

/* cyclic convolution of a (len la <= N) and b folded mod x^N - 1 (len lb),
 * accumulated into out[N] (mod p).  Via the reference NTT when available. */
static void cyclic_acc(uint64_t p, int log_len, const uint64_t *a, int la,
                       const uint64_t *b, int lb, uint64_t *out) {
    size_t N = (size_t)1 << log_len;
    uint64_t *fa = (uint64_t *)calloc(N, sizeof(uint64_t));
    uint64_t *fb = (uint64_t *)calloc(N, sizeof(uint64_t));
    for (int t = 0; t < la; t++) fa[t % N] = addmod(fa[t % N], a[t] % p, p);
    for (int t = 0; t < lb; t++) fb[t % N] = addmod(fb[t % N], b[t] % p, p);
    fpo_ntt(p, log_len, fa, 0);
    fpo_ntt(p, log_len, fb, 0);
    for (size_t t = 0; t < N; t++) fa[t] = mulmod(fa[t], fb[t], p);
    fpo_ntt(p, log_len, fa, 1);
    for (size_t t = 0; t < N; t++) out[t] = addmod(out[t], fa[t], p);
    free(fa); free(fb);
}

/* upoly._middle (upoly.py:347-377) for one entry pair, accumulated into out[d] */
static void middle_entry(uint64_t p, const uint64_t *a, int la, const uint64_t *b,
                         int lb, long c, int d, uint64_t *out) {
    la = entry_len(a, la);
    lb = entry_len(b, lb);
    if (la == 0 || lb == 0 || d <= 0) return;
    long lad = (long)la * d;
    if (lad <= 64 * 64 / 4 && lad <= 16384) {
        for (int tt = 0; tt < d; tt++) {
            long t = c + tt;
            long lo = t - lb + 1 > 0 ? t - lb + 1 : 0;
            long hi = la - 1 < t ? la - 1 : t;
            u128 s = 0;
            int cnt = 0;
            for (long j = lo; j <= hi; j++) {
                s += (u128)a[j] * b[t - j];
                if (++cnt == 16) { s %= p; cnt = 0; }
            }
            out[tt] = addmod(out[tt], (uint64_t)(s % p), p);
        }
        return;
    }
    long need = (long)la + d;
    int log_len = ceil_log2_min1(need);
    if (log_len <= fpo_two_adicity(p)) {
        size_t N = (size_t)1 << log_len;
        uint64_t *cyc = (uint64_t *)calloc(N, sizeof(uint64_t));
        cyclic_acc(p, log_len, a, la, b, lb, cyc);
        for (int tt = 0; tt < d; tt++) out[tt] = addmod(out[tt], cyc[(c + tt) % N], p);
        free(cyc);
        return;
    }
    /* full product slice */
    for (int tt = 0; tt < d; tt++) {
        long t = c + tt;
        long lo = t - lb + 1 > 0 ? t - lb + 1 : 0;
        long hi = la - 1 < t ? la - 1 : t;
        u128 s = 0;
        int cnt = 0;
        for (long j = lo; j <= hi; j++) {
            s += (u128)a[j] * b[t - j];
            if (++cnt == 16) { s %= p; cnt = 0; }
        }
        out[tt] = addmod(out[tt], (uint64_t)(s % p), p);
    }
}

/* _pm_middle with the reference's exact dispatch (polmat.py:484-536),
 * including its cyclic fold.  out: m*n*d. */
int fpo_pm_middle(uint64_t p, const uint64_t *A, int m, int k, int la,
                  const uint64_t *B, int n, int lb, long c, int d, uint64_t *out) {
    if (d <= 0) return 0;
    memset(out, 0, sizeof(uint64_t) * (size_t)m * n * d);
    int da = mat_degree(A, m, k, la), db = mat_degree(B, k, n, lb);
    if (da < 0 || db < 0) return 0;
    long need = (long)da + d + 1;
    int log_len = ceil_log2_min1(need);
    long N = 1L << log_len;
    int wrap_ok = c + N > (long)da + db;
    if (need >= 64 && log_len <= fpo_two_adicity(p) && wrap_ok) {
#pragma omp parallel for schedule(dynamic) num_threads(g_threads)
        for (int e = 0; e < m * n; e++) {
            int i = e / n, j = e % n;
            uint64_t *cyc = (uint64_t *)calloc((size_t)N, sizeof(uint64_t));
            for (int l = 0; l < k; l++)
                cyclic_acc(p, log_len, A + ((size_t)i * k + l) * la, la,
                           B + ((size_t)l * n + j) * lb, lb, cyc);
            for (int tt = 0; tt < d; tt++) out[(size_t)e * d + tt] = cyc[(c + tt) % N];
            free(cyc);
        }
        return 0;
    }
#pragma omp parallel for schedule(dynamic) num_threads(g_threads)
    for (int e = 0; e < m * n; e++) {
        int i = e / n, j = e % n;
        for (int l = 0; l < k; l++)
            middle_entry(p, A + ((size_t)i * k + l) * la, la,
                         B + ((size_t)l * n + j) * lb, lb, c, d, out + (size_t)e * d);
    }
    return 0;
}

/* ---- M-Basis (appint.py:24-180) ----------------------------------------- */
/* _mbasis1_struct: R is m x n (row-major).  Outputs is_pivot[m] and
 * kern[m*m] with kern[i*m+j] = c such that basis row i = e_i - sum c e_j. */
static void mbasis1_struct(uint64_t p, const uint64_t *R, int m, int n,
                           const int64_t *s, int *is_pivot, uint64_t *kern) {
    int *order = (int *)malloc(sizeof(int) * m);
    for (int i = 0; i < m; i++) order[i] = i;
    /* sorted(range(m), key=(s_i, i)) -- stable insertion sort */
    for (int a = 1; a < m; a++) {
        int x = order[a], b = a - 1;
        while (b >= 0 && (s[order[b]] > s[x] || (s[order[b]] == s[x] && order[b] > x))) {
            order[b + 1] = order[b];
            b--;
        }
        order[b + 1] = x;
    }
    uint64_t *red_w = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)m * n);
    uint64_t *red_x = (uint64_t *)calloc((size_t)m * m, sizeof(uint64_t));
    int *red_col = (int *)malloc(sizeof(int) * m);
    int nred = 0;
    uint64_t *v = (uint64_t *)malloc(sizeof(uint64_t) * n);
    uint64_t *expr = (uint64_t *)malloc(sizeof(uint64_t) * m);
    memset(kern, 0, sizeof(uint64_t) * (size_t)m * m);
    for (int oi = 0; oi < m; oi++) {
        int i = order[oi];
        for (int j = 0; j < n; j++) v[j] = R[(size_t)i * n + j] % p;
        memset(expr, 0, sizeof(uint64_t) * m);
        for (int r = 0; r < nred; r++) {
            uint64_t c = v[red_col[r]];
            if (c) {
                const uint64_t *w = red_w + (size_t)r * n;
                for (int j = 0; j < n; j++) v[j] = submod(v[j], mulmod(c, w[j], p), p);
                const uint64_t *wx = red_x + (size_t)r * m;
                for (int j = 0; j < m; j++)
                    if (wx[j]) expr[j] = addmod(expr[j], mulmod(c, wx[j], p), p);
            }
        }
        int nz = -1;
        for (int j = 0; j < n; j++) if (v[j]) { nz = j; break; }
        if (nz < 0) {
            is_pivot[i] = 0;
            for (int j = 0; j < m; j++) kern[(size_t)i * m + j] = expr[j];
        } else {
            uint64_t inv = invmod(v[nz], p);
            uint64_t *w = red_w + (size_t)nred * n;
            for (int j = 0; j < n; j++) w[j] = mulmod(v[j], inv, p);
            uint64_t *wx = red_x + (size_t)nred * m;
            for (int j = 0; j < m; j++) wx[j] = expr[j] ? mulmod(p - expr[j], inv, p) : 0;
            wx[i] = inv;
            red_col[nred++] = nz;
            is_pivot[i] = 1;
        }
    }
    free(order); free(red_w); free(red_x); free(red_col); free(v); free(expr);
}

/* exported for tests: mbasis1 structure */
void fpo_mbasis1_struct(uint64_t p, const uint64_t *R, int m, int n,
                        const int64_t *s, int *is_pivot, uint64_t *kern) {
    mbasis1_struct(p, R, m, n, s, is_pivot, kern);
}

/* mbasis (appint.py:143-180).  F: m x n x lf (coefficients beyond lf are 0,
 * i.e. F.truncate(order) is taken by the caller contract).  P out: m x m x
 * (order+1) dense; *lp = number of coefficient matrices (len(P) list).
 * shift_out (optional): final sft. */
int fpo_mbasis(uint64_t p, const uint64_t *F, int m, int n, int lf, int order,
               const int64_t *s, uint64_t *P_out, int *lp, int64_t *shift_out) {
    size_t mm = (size_t)m * m;
    int cap = order + 2;
    uint64_t *P = (uint64_t *)calloc(mm * cap, sizeof(uint64_t)); /* P[t][i][j] */
    uint64_t *Pn = (uint64_t *)calloc(mm * cap, sizeof(uint64_t));
    int L = 1;
    for (int i = 0; i < m; i++) P[(size_t)i * m + i] = 1;
    int64_t *sft = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
    for (int i = 0; i < m; i++) sft[i] = s[i];
    uint64_t *R = (uint64_t *)malloc(sizeof(uint64_t) * ((size_t)m * n + 1));
    int *isp = (int *)malloc(sizeof(int) * (size_t)(m > 0 ? m : 1));
    uint64_t *kern = (uint64_t *)malloc(sizeof(uint64_t) * (mm + 1));
    int64_t smin = 0;
    for (int i = 0; i < m; i++) if (i == 0 || s[i] < smin) smin = s[i];
    for (int k = 0; k < order; k++) {
        /* R = sum_t P_t F_{k-t} (appint.py:157-169) */
        for (size_t e = 0; e < (size_t)m * n; e++) R[e] = 0;
        int tmax = L - 1 < k ? L - 1 : k;
        for (int i = 0; i < m; i++)
            for (int j = 0; j < n; j++) {
                u128 acc = 0;
                int cnt = 0;
                for (int t = 0; t <= tmax; t++) {
                    int fk = k - t;
                    if (fk >= lf) continue;
                    const uint64_t *Pt = P + (size_t)t * mm + (size_t)i * m;
                    for (int l = 0; l < m; l++) {
                        if (!Pt[l]) continue;
                        acc += (u128)Pt[l] * F[((size_t)l * n + j) * lf + fk];
                        if (++cnt == 16) { acc %= p; cnt = 0; }
                    }
                }
                R[(size_t)i * n + j] = (uint64_t)(acc % p);
            }
        mbasis1_struct(p, R, m, n, sft, isp, kern);
        int nk = 0;
        for (int i = 0; i < m; i++) nk += !isp[i];
        if (nk < m) {
            /* _apply_step (appint.py:79-117) */
            memset(Pn, 0, sizeof(uint64_t) * mm * (L + 1));
            for (int t = 0; t <= L; t++) {
                for (int i = 0; i < m; i++) {
                    uint64_t *row = Pn + (size_t)t * mm + (size_t)i * m;
                    if (isp[i]) {
                        if (t >= 1) memcpy(row, P + (size_t)(t - 1) * mm + (size_t)i * m, sizeof(uint64_t) * m);
                    } else if (t < L) {
                        const uint64_t *cur = P + (size_t)t * mm;
                        for (int j = 0; j < m; j++) row[j] = cur[(size_t)i * m + j];
                        for (int jj = 0; jj < m; jj++) {
                            uint64_t c = kern[(size_t)i * m + jj];
                            if (!c) continue;
                            for (int j = 0; j < m; j++)
                                row[j] = submod(row[j], mulmod(c, cur[(size_t)jj * m + j], p), p);
                        }
                    }
                }
            }
            int Ln = L + 1;
            while (Ln > 0) {
                const uint64_t *last = Pn + (size_t)(Ln - 1) * mm;
                size_t z;
                for (z = 0; z < mm; z++) if (last[z]) break;
                if (z < mm) break;
                Ln--;
            }
            uint64_t *tmp = P; P = Pn; Pn = tmp;
            L = Ln;
            /* sft = _finish_shift(_rdeg_from_coeffs(P, s, m), s) */
            for (int i = 0; i < m; i++) {
                int have = 0;
                int64_t best = 0;
                for (int t = 0; t < L; t++)
                    for (int j = 0; j < m; j++)
                        if (P[(size_t)t * mm + (size_t)i * m + j]) {
                            int64_t v = t + s[j];
                            if (!have || v > best) { best = v; have = 1; }
                        }
                sft[i] = have ? best : smin;
            }
        }
    }
    /* PolMat.from_matpoly(ctx, P): dense output, cap order+1 coefficients */
    memset(P_out, 0, sizeof(uint64_t) * mm * (order + 1));
    for (int t = 0; t < L && t <= order; t++)
        for (size_t e = 0; e < mm; e++) P_out[e * (order + 1) + t] = P[(size_t)t * mm + e];
    *lp = L;
    if (shift_out) for (int i = 0; i < m; i++) shift_out[i] = sft[i];
    free(P); free(Pn); free(sft); free(R); free(isp); free(kern);
    return 0;
}

/* rdeg(P, s) of a dense m x m x lp matrix; zero rows -> min(s) via
 * _finish_shift (appint.py:134-136, forms.py:20-51). */
static void rdeg_finish(const uint64_t *P, int m, int lp, const int64_t *s, int64_t *out) {
    int64_t smin = 0;
    for (int i = 0; i < m; i++) if (i == 0 || s[i] < smin) smin = s[i];
    for (int i = 0; i < m; i++) {
        int have = 0;
        int64_t best = 0;
        for (int j = 0; j < m; j++) {
            int l = entry_len(P + ((size_t)i * m + j) * lp, lp);
            if (l) {
                int64_t v = l - 1 + s[j];
                if (!have || v > best) { best = v; have = 1; }
            }
        }
        out[i] = have ? best : smin;
    }
}

/* pmbasis (appint.py:183-196) with base threshold T (config.py:18 default 32).
 * F: m x n x lf.  P out: m x m x (order+1).  *lp = degree(P)+1. */
int fpo_pmbasis(uint64_t p, const uint64_t *F, int m, int n, int lf, int order,
                const int64_t *s, int T, uint64_t *P_out, int *lp) {
    size_t mm = (size_t)m * m;
    int lt = lf < order ? lf : order;
    if (order <= T) {
        /* mbasis(F.truncate(order), order, s) */
        uint64_t *Ft = (uint64_t *)calloc((size_t)m * n * (lt > 0 ? lt : 1), sizeof(uint64_t));
        for (size_t e = 0; e < (size_t)m * n; e++)
            for (int t = 0; t < lt; t++) Ft[e * lt + t] = F[e * lf + t];
        int L;
        fpo_mbasis(p, Ft, m, n, lt > 0 ? lt : 1, order, s, P_out, &L, NULL);
        free(Ft);
        *lp = L;
        return 0;
    }
    int o1 = (order + 1) / 2, o2 = order - o1;
    uint64_t *P1 = (uint64_t *)calloc(mm * (o1 + 1), sizeof(uint64_t));
    int lp1;
    fpo_pmbasis(p, F, m, n, lf, o1, s, T, P1, &lp1);
    /* R = _pm_middle(P1, F.truncate(order), o1, o2) */
    uint64_t *Ftr = (uint64_t *)calloc((size_t)m * n * (lt > 0 ? lt : 1), sizeof(uint64_t));
    for (size_t e = 0; e < (size_t)m * n; e++)
        for (int t = 0; t < lt; t++) Ftr[e * lt + t] = F[e * lf + t];
    uint64_t *P1c = (uint64_t *)calloc(mm * (lp1 > 0 ? lp1 : 1), sizeof(uint64_t));
    for (size_t e = 0; e < mm; e++)
        for (int t = 0; t < lp1; t++) P1c[e * lp1 + t] = P1[e * (o1 + 1) + t];
    uint64_t *R = (uint64_t *)calloc((size_t)m * n * (o2 > 0 ? o2 : 1), sizeof(uint64_t));
    fpo_pm_middle(p, P1c, m, m, lp1 > 0 ? lp1 : 1, Ftr, n, lt > 0 ? lt : 1, o1, o2, R);
    int64_t *s1 = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
    rdeg_finish(P1c, m, lp1 > 0 ? lp1 : 1, s, s1);
    uint64_t *P2 = (uint64_t *)calloc(mm * (o2 + 1), sizeof(uint64_t));
    int lp2;
    fpo_pmbasis(p, R, m, n, o2 > 0 ? o2 : 1, o2, s1, T, P2, &lp2);
    uint64_t *P2c = (uint64_t *)calloc(mm * (lp2 > 0 ? lp2 : 1), sizeof(uint64_t));
    for (size_t e = 0; e < mm; e++)
        for (int t = 0; t < lp2; t++) P2c[e * lp2 + t] = P2[e * (o2 + 1) + t];
    /* pm_mul(P2, P1) */
    int a2 = lp2 > 0 ? lp2 : 1, a1 = lp1 > 0 ? lp1 : 1;
    int lc = a2 + a1 - 1;
    uint64_t *Pc = (uint64_t *)calloc(mm * lc, sizeof(uint64_t));
    fpo_pm_mul(p, P2c, m, m, a2, P1c, m, a1, Pc);
    memset(P_out, 0, sizeof(uint64_t) * mm * (order + 1));
    int d = mat_degree(Pc, m, m, lc);
    for (size_t e = 0; e < mm; e++)
        for (int t = 0; t <= d && t <= order; t++) P_out[e * (order + 1) + t] = Pc[e * lc + t];
    *lp = d + 1;
    free(P1); free(Ftr); free(P1c); free(R); free(s1); free(P2); free(P2c); free(Pc);
    return 0;
}
