/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle of Algorithm 1
 * ("FTM", arXiv 1509.04863).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or constant with the CUDA path in
 * paper_1509_04863_b200/csrc, and it never calls it.
 *
 * Every function follows one passage of the paper, step by step, with the
 * loop order of the paper's formula; no blocking, no fusion, no FFT.
 *   - integer data (int8 samples) is accumulated exactly in int64;
 *   - real data (float32 samples) is accumulated in fp64.
 * Readings where the paper is silent or garbled are the ones listed in
 * DESIGN.md section "Readings" (C1..C20 of SURVEY.md 8(c.1)).
 *
 * Parity pins: every exported function is pinned in tests/test_oracle.py
 * against brute force, a dense-matrix construction, closed forms or the
 * paper's printed values.  No function here is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

void or_thm1_That_y_i64(const int64_t *y, int64_t M, const int8_t *t, int64_t K, int64_t *out);

/* ------------------------------------------------------------------ */
/* helpers                                                              */
/* ------------------------------------------------------------------ */

/* ceil(a / b) for a >= 0, b > 0 -- the paper's \lceil N/M \rceil. */
int64_t or_ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

/* (i mod N) in [0, N): the paper's index convention (x)_i = (x)_{i mod N}
 * (section 2). */
static int64_t or_mod(int64_t i, int64_t N) {
    int64_t r = i % N;
    return r < 0 ? r + N : r;
}

/* ------------------------------------------------------------------ */
/* O1  Alg. 1 step 2: pick co-prime M1, M2 with M1*M2 > N,        */
/*     M1 >= K, M2 >= K.  The paper's rule is M1 = K, M2 = K+1 (P:299,    */
/*     P:320); M (if nonzero) overrides M1, and M2 = M1 + 1 (consecutive  */
/*     integers are co-prime).  Returns 0 on success, -1 if invalid.      */
/* ------------------------------------------------------------------ */
int or_moduli(int64_t N, int64_t K, int64_t M, int64_t *M1, int64_t *M2) {
    int64_t m1 = (M != 0) ? M : K;
    int64_t m2 = m1 + 1;
    if (N < 1 || K < 1 || m1 < K) return -1;
    /* M1*M2 > N.  Use 128-bit so that no overflow hides a failure. */
    if ((__int128)m1 * (__int128)m2 <= (__int128)N) return -1;
    *M1 = m1;
    *M2 = m2;
    return 0;
}

/* ------------------------------------------------------------------ */
/* O2  Downsampling, Eq. (2) / Alg. 1 step 3:      */
/*       y_k = sum_{i=0}^{ceil(N/M)-1} x_{(k + i M) mod N},              */
/*       k = 0 .. M+K-1   (strategy 1, D_{M+K}).              */
/* Literal loop order: for every i, for every k.                         */
/* Partial variant: only positions p in [lo, lo+len) contribute          */
/* (0 <= lo, lo+len <= N).  lo = 0, len = N is the paper's fold.         */
/* ------------------------------------------------------------------ */
void or_fold_i8(const int8_t *x, int64_t N, int64_t M, int64_t K,
                int64_t lo, int64_t len, int64_t *y) {
    int64_t q = or_ceil_div(N, M);
    for (int64_t k = 0; k < M + K; ++k) y[k] = 0;
    for (int64_t i = 0; i < q; ++i) {
        for (int64_t k = 0; k < M + K; ++k) {
            int64_t p = or_mod(k + i * M, N);
            if (p >= lo && p < lo + len) y[k] += (int64_t)x[p];
        }
    }
}

/* One entry of Eq. (2): y_k = sum_{i<ceil(N/M)} x_{(k+iM) mod N} -- the fold
 * evaluated bin by bin, for sampled checks at sizes where the whole fold is
 * too slow for the oracle (N = 2^31).  Same formula, same order as or_fold. */
void or_fold_bins_i8(const int8_t *x, int64_t N, int64_t M, const int64_t *bins, int64_t nb,
                     int64_t *out) {
    int64_t q = or_ceil_div(N, M);
    for (int64_t b = 0; b < nb; ++b) {
        int64_t s = 0;
        for (int64_t i = 0; i < q; ++i) s += (int64_t)x[or_mod(bins[b] + i * M, N)];
        out[b] = s;
    }
}

void or_fold_f32(const float *x, int64_t N, int64_t M, int64_t K,
                 int64_t lo, int64_t len, double *y) {
    int64_t q = or_ceil_div(N, M);
    for (int64_t k = 0; k < M + K; ++k) y[k] = 0.0;
    for (int64_t i = 0; i < q; ++i) {
        for (int64_t k = 0; k < M + K; ++k) {
            int64_t p = or_mod(k + i * M, N);
            if (p >= lo && p < lo + len) y[k] += (double)x[p];
        }
    }
}

/* ------------------------------------------------------------------ */
/* O3  Low-dimensional correlation, Alg. 1 steps 4-6, read as  */
/*     the cross-correlation of section 3 -- reading C3: the plain */
/*     product t~ .* y~ of step 6 is a convolution; the method needs      */
/*       r_k = sum_{i=0}^{K-1} t_i y_{k+i},   k = 0 .. M-1                */
/*     (t_M = [t 0] zero-padded, step 4, so no term wraps: k+i <= M+K-2). */
/*     Direct sum, i ascending.  No FFT.                                  */
/* ------------------------------------------------------------------ */
void or_correlate_i64(const int64_t *y, int64_t M, int64_t K,
                      const int8_t *t, int64_t *r) {
    for (int64_t k = 0; k < M; ++k) {
        int64_t s = 0;
        for (int64_t i = 0; i < K; ++i) s += (int64_t)t[i] * y[k + i];
        r[k] = s;
    }
}

/* Selected entries of O3, one output at a time: r_k for k = ks[0..nk) with the
 * same formula and order as or_correlate_i64 (sampled checks where the whole
 * correlation is too slow for the oracle: K = 2^18, 2^19 at N = 2^31). */
void or_correlate_at_i64(const int64_t *y, int64_t K, const int8_t *t,
                         const int64_t *ks, int64_t nk, int64_t *r) {
    for (int64_t j = 0; j < nk; ++j) {
        int64_t s = 0;
        for (int64_t i = 0; i < K; ++i) s += (int64_t)t[i] * y[ks[j] + i];
        r[j] = s;
    }
}

void or_correlate_f64(const double *y, int64_t M, int64_t K,
                      const float *t, double *r) {
    for (int64_t k = 0; k < M; ++k) {
        double s = 0.0;
        for (int64_t i = 0; i < K; ++i) s += (double)t[i] * y[k + i];
        r[k] = s;
    }
}

/* ------------------------------------------------------------------ */
/* O4  Alg. 1 step 7: m~ = argmax_{i} r_i over i in [0, M)       */
/*     (reading C6: "i <= M" would alias residue 0), ties to the lowest   */
/*     index (reading C7).                                                */
/* ------------------------------------------------------------------ */
int64_t or_argmax_i64(const int64_t *r, int64_t M) {
    int64_t best = 0;
    for (int64_t k = 1; k < M; ++k)
        if (r[k] > r[best]) best = k;
    return best;
}

int64_t or_argmax_f64(const double *r, int64_t M) {
    int64_t best = 0;
    for (int64_t k = 1; k < M; ++k)
        if (r[k] > r[best]) best = k;
    return best;
}

/* ------------------------------------------------------------------ */
/* O5  Theorem 4, CRT: the unique z in [0, M1*M2) with        */
/*     z = m1 (mod M1) and z = m2 (mod M2), by the extended Euclidean     */
/*     algorithm.  Returns -1 if gcd(M1, M2) != 1.                        */
/* ------------------------------------------------------------------ */
int64_t or_crt(int64_t m1, int64_t M1, int64_t m2, int64_t M2) {
    /* extended Euclid on (M1, M2): g = a*M1 + b*M2 */
    __int128 old_r = M1, r = M2, old_s = 1, s = 0;
    while (r != 0) {
        __int128 qq = old_r / r, tmp;
        tmp = r;  r = old_r - qq * r;  old_r = tmp;
        tmp = s;  s = old_s - qq * s;  old_s = tmp;
    }
    if (old_r != 1) return -1;
    /* inv = M1^{-1} mod M2 */
    __int128 inv = old_s % M2;
    if (inv < 0) inv += M2;
    /* z = m1 + M1 * ((m2 - m1) * inv mod M2) */
    __int128 d = ((__int128)m2 - (__int128)m1) % M2;
    if (d < 0) d += M2;
    __int128 u = (d * inv) % M2;
    return (int64_t)((__int128)m1 + (__int128)M1 * u);
}

/* ------------------------------------------------------------------ */
/* O5' Alg. 1 steps 8-9 literally:                           */
/*     S_Mj = { m~j + i*Mj : i = 0 .. ceil(N/Mj)-1 },  m^ = S_M1 ∩ S_M2. */
/*     Returns the single common element, -1 if the intersection is empty */
/*     (reading C9: NO_MATCH), -2 if it had more than one element.        */
/*     O(|S_M1| * |S_M2|) -- small N only (tests).                        */
/* ------------------------------------------------------------------ */
int64_t or_crt_sets(int64_t m1, int64_t M1, int64_t m2, int64_t M2, int64_t N) {
    int64_t q1 = or_ceil_div(N, M1), q2 = or_ceil_div(N, M2);
    int64_t found = -1, count = 0;
    for (int64_t i = 0; i < q1; ++i) {
        int64_t a = m1 + i * M1;
        for (int64_t j = 0; j < q2; ++j) {
            if (a == m2 + j * M2) {
                if (count == 0) found = a;
                ++count;
            }
        }
    }
    if (count > 1) return -2;
    return found;
}

/* ------------------------------------------------------------------ */
/* O5'' Alg. 1 steps 8-9 with the candidate sets taken modulo N (the      */
/*     paper's index convention (x)_i = (x)_{i mod N}): reading C10's */
/*     alias repair (opt-in).                             */
/*       S_Mj mod N = { (m~j + i Mj) mod N : i = 0 .. ceil(N/Mj)-1 }       */
/*     Returns the single common element, -1 if empty, -2 if several.      */
/*     S_M2 mod N is sorted once and every element of S_M1 mod N is looked */
/*     up by bisection: O(q log q), usable at every BASELINE size.        */
/* ------------------------------------------------------------------ */
static int or_cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

int64_t or_crt_sets_modN(int64_t m1, int64_t M1, int64_t m2, int64_t M2, int64_t N) {
    int64_t q1 = or_ceil_div(N, M1), q2 = or_ceil_div(N, M2);
    int64_t *s2 = (int64_t *)malloc(sizeof(int64_t) * q2);
    for (int64_t j = 0; j < q2; ++j) s2[j] = or_mod(m2 + j * M2, N);
    qsort(s2, (size_t)q2, sizeof(int64_t), or_cmp_i64);
    int64_t found = -1, count = 0;
    for (int64_t i = 0; i < q1; ++i) {
        int64_t a = or_mod(m1 + i * M1, N);
        int64_t lo = 0, hi = q2;  /* first index with s2[idx] >= a */
        while (lo < hi) {
            int64_t mid = (lo + hi) / 2;
            if (s2[mid] < a) lo = mid + 1; else hi = mid;
        }
        if (lo < q2 && s2[lo] == a) {  /* a common element; count distinct values */
            if (count == 0) { found = a; count = 1; }
            else if (a != found) count = 2;
        }
    }
    free(s2);
    if (count > 1) return -2;
    return found;
}

/* Steps 8-9 resolution used by FTM(): the literal unreduced sets (reading C9,
   computed by Theorem 4: k = z if z < N, else NO_MATCH), or, with repair, the
   mod-N sets above (NO_MATCH if they do not meet in exactly one element). */
int64_t or_resolve(int64_t m1, int64_t M1, int64_t m2, int64_t M2, int64_t N, int repair) {
    int64_t z = or_crt(m1, M1, m2, M2);
    if (z >= 0 && z < N) return z;
    if (!repair) return -1;
    int64_t v = or_crt_sets_modN(m1, M1, m2, M2, N);
    return v >= 0 ? v : -1;
}

/* ------------------------------------------------------------------ */
/* O6  Algorithm 1, FTM(), end to end.                        */
/*     k^ = z if z < N else -1 (NO_MATCH, reading C9); repair != 0: the   */
/*     mod-N reading of steps 8-9 (or_resolve).                           */
/*     Optional outputs (NULL to skip): residues[2], y1[M1+K], y2[M2+K],  */
/*     r1[M1], r2[M2].  Returns k^, or -3 on invalid arguments.           */
/* ------------------------------------------------------------------ */
int64_t or_ftm_i8(const int8_t *x, int64_t N, const int8_t *t, int64_t K, int64_t M, int repair,
                  int64_t *residues, int64_t *y1o, int64_t *y2o,
                  int64_t *r1o, int64_t *r2o) {
    int64_t M1, M2;
    if (or_moduli(N, K, M, &M1, &M2) != 0) return -3;               /* step 2 */
    int64_t *y1 = (int64_t *)malloc(sizeof(int64_t) * (M1 + K));
    int64_t *y2 = (int64_t *)malloc(sizeof(int64_t) * (M2 + K));
    int64_t *r1 = (int64_t *)malloc(sizeof(int64_t) * M1);
    int64_t *r2 = (int64_t *)malloc(sizeof(int64_t) * M2);
    or_fold_i8(x, N, M1, K, 0, N, y1);                               /* step 3 */
    or_fold_i8(x, N, M2, K, 0, N, y2);
    or_correlate_i64(y1, M1, K, t, r1);                              /* steps 4-6 */
    or_correlate_i64(y2, M2, K, t, r2);
    int64_t m1 = or_argmax_i64(r1, M1);                              /* step 7 */
    int64_t m2 = or_argmax_i64(r2, M2);
    int64_t k = or_resolve(m1, M1, m2, M2, N, repair);               /* steps 8-9 */
    if (residues) { residues[0] = m1; residues[1] = m2; }
    if (y1o) memcpy(y1o, y1, sizeof(int64_t) * (M1 + K));
    if (y2o) memcpy(y2o, y2, sizeof(int64_t) * (M2 + K));
    if (r1o) memcpy(r1o, r1, sizeof(int64_t) * M1);
    if (r2o) memcpy(r2o, r2, sizeof(int64_t) * M2);
    free(y1); free(y2); free(r1); free(r2);
    return k;
}

int64_t or_ftm_f32(const float *x, int64_t N, const float *t, int64_t K, int64_t M, int repair,
                   int64_t *residues, double *y1o, double *y2o,
                   double *r1o, double *r2o) {
    int64_t M1, M2;
    if (or_moduli(N, K, M, &M1, &M2) != 0) return -3;
    double *y1 = (double *)malloc(sizeof(double) * (M1 + K));
    double *y2 = (double *)malloc(sizeof(double) * (M2 + K));
    double *r1 = (double *)malloc(sizeof(double) * M1);
    double *r2 = (double *)malloc(sizeof(double) * M2);
    or_fold_f32(x, N, M1, K, 0, N, y1);
    or_fold_f32(x, N, M2, K, 0, N, y2);
    or_correlate_f64(y1, M1, K, t, r1);
    or_correlate_f64(y2, M2, K, t, r2);
    int64_t m1 = or_argmax_f64(r1, M1);
    int64_t m2 = or_argmax_f64(r2, M2);
    int64_t k = or_resolve(m1, M1, m2, M2, N, repair);
    if (residues) { residues[0] = m1; residues[1] = m2; }
    if (y1o) memcpy(y1o, y1, sizeof(double) * (M1 + K));
    if (y2o) memcpy(y2o, y2, sizeof(double) * (M2 + K));
    if (r1o) memcpy(r1o, r1, sizeof(double) * M1);
    if (r2o) memcpy(r2o, r2, sizeof(double) * M2);
    free(y1); free(y2); free(r1); free(r2);
    return k;
}

/* ------------------------------------------------------------------ */
/* Theorem 4 with alpha moduli: "any integer m is uniquely     */
/* specified mod N by its remainders modulo alpha relatively prime         */
/* integers M_1 .. M_alpha as long as prod M_i >= N" (Alg. 1 uses alpha =  */
/* 2).  The unique z in [0, prod M_i) with       */
/* z = m_i (mod M_i), by folding the congruences in one at a time with the */
/* two-modulus rule of or_crt (extended Euclid).  Returns -1 if two moduli */
/* share a factor, INT64_MAX if z does not fit (prod M_i beyond 2^63).     */
/* ------------------------------------------------------------------ */
int64_t or_crt_multi(const int64_t *m, const int64_t *M, int alpha) {
    __int128 z = m[0], P = M[0];
    for (int j = 1; j < alpha; ++j) {
        /* extended Euclid on (P mod M_j, M_j) -> inverse of P modulo M_j */
        __int128 old_r = P % M[j], r = M[j], old_s = 1, s = 0;
        while (r != 0) {
            __int128 qq = old_r / r, tmp;
            tmp = r;  r = old_r - qq * r;  old_r = tmp;
            tmp = s;  s = old_s - qq * s;  old_s = tmp;
        }
        if (old_r != 1) return -1;
        __int128 inv = old_s % M[j];
        if (inv < 0) inv += M[j];
        __int128 d = ((__int128)m[j] - z) % M[j];
        if (d < 0) d += M[j];
        z += P * ((d * inv) % M[j]);   /* z = m_i (mod M_i) for every i <= j */
        P *= M[j];
        if (P > ((__int128)1 << 100)) return INT64_MAX;
    }
    return z > (__int128)INT64_MAX ? INT64_MAX : (int64_t)z;
}

/* Steps 8-9 literally for alpha sets: the elements common to   */
/* every S_Mj = { m_j + i M_j : i < ceil(N / M_j) }.  Returns the single     */
/* common element, -1 if none, -2 if several.  Small N only (tests).        */
int64_t or_crt_sets_multi(const int64_t *m, const int64_t *M, int alpha, int64_t N) {
    int64_t found = -1, count = 0;
    for (int64_t i = 0; i < or_ceil_div(N, M[0]); ++i) {
        int64_t a = m[0] + i * M[0];
        int in_all = 1;
        for (int j = 1; j < alpha && in_all; ++j) {
            in_all = 0;
            for (int64_t u = 0; u < or_ceil_div(N, M[j]); ++u)
                if (m[j] + u * M[j] == a) { in_all = 1; break; }
        }
        if (in_all) { if (count == 0) found = a; ++count; }
    }
    return count > 1 ? -2 : found;
}

/* FTM() with alpha moduli: for each M_j the Eq. 2 fold (strategy 1, M_j + K */
/* entries), the correlation and the argmax of Alg. 1 steps 3-7; then z =    */
/* or_crt_multi and k = z if z < N else -1 (reading C9).  Requires K <= M_j, */
/* pairwise co-prime moduli and prod M_j > N (else returns -3).  Outputs:    */
/* residues[alpha] (may be NULL).                                            */
int64_t or_ftm_multi_i8(const int8_t *x, int64_t N, const int8_t *t, int64_t K, const int64_t *M, int alpha,
                        int64_t *residues) {
    __int128 P = 1;
    for (int j = 0; j < alpha; ++j) {
        if (M[j] < K) return -3;
        for (int i = 0; i < j; ++i) {
            int64_t a = M[i], b = M[j];
            while (b) { int64_t r = a % b; a = b; b = r; }
            if (a != 1) return -3;
        }
        P *= M[j];
        if (P > ((__int128)1 << 100)) P = ((__int128)1 << 100);
    }
    if (P <= N) return -3;
    int64_t m[16];
    for (int j = 0; j < alpha; ++j) {
        int64_t *y = (int64_t *)malloc(sizeof(int64_t) * (M[j] + K));
        int64_t *r = (int64_t *)malloc(sizeof(int64_t) * M[j]);
        or_fold_i8(x, N, M[j], K, 0, N, y);                          /* step 3 */
        or_correlate_i64(y, M[j], K, t, r);                          /* steps 4-6 */
        m[j] = or_argmax_i64(r, M[j]);                               /* step 7 */
        free(y); free(r);
    }
    if (residues) for (int j = 0; j < alpha; ++j) residues[j] = m[j];
    int64_t z = or_crt_multi(m, M, alpha);                           /* steps 8-9 */
    return (z >= 0 && z < N) ? z : -1;
}

/* The same for float32 data: Eq. 2 folds and correlations in fp64. */
int64_t or_ftm_multi_f32(const float *x, int64_t N, const float *t, int64_t K, const int64_t *M, int alpha,
                         int64_t *residues) {
    __int128 P = 1;
    for (int j = 0; j < alpha; ++j) {
        if (M[j] < K) return -3;
        for (int i = 0; i < j; ++i) {
            int64_t a = M[i], b = M[j];
            while (b) { int64_t r = a % b; a = b; b = r; }
            if (a != 1) return -3;
        }
        P *= M[j];
        if (P > ((__int128)1 << 100)) P = ((__int128)1 << 100);
    }
    if (P <= N) return -3;
    int64_t m[16];
    for (int j = 0; j < alpha; ++j) {
        double *y = (double *)malloc(sizeof(double) * (M[j] + K));
        double *r = (double *)malloc(sizeof(double) * M[j]);
        or_fold_f32(x, N, M[j], K, 0, N, y);
        or_correlate_f64(y, M[j], K, t, r);
        m[j] = or_argmax_f64(r, M[j]);
        free(y); free(r);
    }
    if (residues) for (int j = 0; j < alpha; ++j) residues[j] = m[j];
    int64_t z = or_crt_multi(m, M, alpha);
    return (z >= 0 && z < N) ? z : -1;
}

/* ------------------------------------------------------------------ */
/* Strategy 2 (Theorem 2): the Block sampling       */
/* matrix Phi = [Phi_M Phi_M ... Phi_M] (ceil(N/M) blocks), Phi_M an M x M */
/* circulant, applied to x zero-padded to ceil(N/M)*M samples ("we can    */
/* pad zeros into the tail of x until M divides N"):               */
/*     y_j = sum_{c < N} Phi_M[j][c mod M] x_c,   j = 0 .. M-1,            */
/*     Phi_M = circ(phi): Phi_M[j][l] = phi[(l - j) mod M].      */
/* phi == NULL is Eq. (3)'s sampling vector r restricted to one block      */
/* (r_k = 1 iff k mod M == 0), i.e. Phi_M = I, and the literal      */
/* sum becomes y_j = sum_{i : j + iM < N} x_{j + iM} (i ascending).        */
/* A non-null phi (a seeded circulant) is the general Theorem 2 operator;  */
/* it serves the dense Theorem 2 pin only (it scrambles the peak of Eq. 5, */
/* which needs Phi_M = I -- reading C21).                                  */
/* ------------------------------------------------------------------ */
void or_block_fold_i8(const int8_t *x, int64_t N, int64_t M, const int8_t *phi, int64_t *y) {
    for (int64_t j = 0; j < M; ++j) {
        int64_t s = 0;
        if (!phi) {
            for (int64_t p = j; p < N; p += M) s += (int64_t)x[p];
        } else {
            for (int64_t c = 0; c < N; ++c) s += (int64_t)phi[or_mod(c % M - j, M)] * (int64_t)x[c];
        }
        y[j] = s;
    }
}

void or_block_fold_f32(const float *x, int64_t N, int64_t M, const float *phi, double *y) {
    for (int64_t j = 0; j < M; ++j) {
        double s = 0.0;
        if (!phi) {
            for (int64_t p = j; p < N; p += M) s += (double)x[p];
        } else {
            for (int64_t c = 0; c < N; ++c) s += (double)phi[or_mod(c % M - j, M)] * (double)x[c];
        }
        y[j] = s;
    }
}

/* Theorem 2's T^ = circ(t) with t zero-padded to M:        */
/*     (T^ y)_i = sum_{u=0}^{K-1} t_u y_{(i+u) mod M},  i = 0 .. M-1.       */
void or_block_correlate_f64(const double *y, int64_t M, const float *t, int64_t K, double *out) {
    for (int64_t i = 0; i < M; ++i) {
        double acc = 0.0;
        for (int64_t u = 0; u < K; ++u) acc += (double)t[u] * y[or_mod(i + u, M)];
        out[i] = acc;
    }
}

/* FTM() with strategy 2 (Phi_M = I): steps 2, 3 (Block fold), 4-6 (T^ y,  */
/* cyclic), 7, 8-9 (or_resolve).  Outputs as or_ftm_*; y has M entries.    */
int64_t or_ftm_block_i8(const int8_t *x, int64_t N, const int8_t *t, int64_t K, int64_t M,
                        int64_t *residues, int64_t *y1o, int64_t *y2o, int64_t *r1o, int64_t *r2o) {
    int64_t M1, M2;
    if (or_moduli(N, K, M, &M1, &M2) != 0) return -3;
    int64_t *y1 = (int64_t *)malloc(sizeof(int64_t) * M1), *y2 = (int64_t *)malloc(sizeof(int64_t) * M2);
    int64_t *r1 = (int64_t *)malloc(sizeof(int64_t) * M1), *r2 = (int64_t *)malloc(sizeof(int64_t) * M2);
    or_block_fold_i8(x, N, M1, NULL, y1);
    or_block_fold_i8(x, N, M2, NULL, y2);
    or_thm1_That_y_i64(y1, M1, t, K, r1);
    or_thm1_That_y_i64(y2, M2, t, K, r2);
    int64_t m1 = or_argmax_i64(r1, M1), m2 = or_argmax_i64(r2, M2);
    int64_t k = or_resolve(m1, M1, m2, M2, N, 0);
    if (residues) { residues[0] = m1; residues[1] = m2; }
    if (y1o) memcpy(y1o, y1, sizeof(int64_t) * M1);
    if (y2o) memcpy(y2o, y2, sizeof(int64_t) * M2);
    if (r1o) memcpy(r1o, r1, sizeof(int64_t) * M1);
    if (r2o) memcpy(r2o, r2, sizeof(int64_t) * M2);
    free(y1); free(y2); free(r1); free(r2);
    return k;
}

int64_t or_ftm_block_f32(const float *x, int64_t N, const float *t, int64_t K, int64_t M,
                         int64_t *residues, double *y1o, double *y2o, double *r1o, double *r2o) {
    int64_t M1, M2;
    if (or_moduli(N, K, M, &M1, &M2) != 0) return -3;
    double *y1 = (double *)malloc(sizeof(double) * M1), *y2 = (double *)malloc(sizeof(double) * M2);
    double *r1 = (double *)malloc(sizeof(double) * M1), *r2 = (double *)malloc(sizeof(double) * M2);
    or_block_fold_f32(x, N, M1, NULL, y1);
    or_block_fold_f32(x, N, M2, NULL, y2);
    or_block_correlate_f64(y1, M1, t, K, r1);
    or_block_correlate_f64(y2, M2, t, K, r2);
    int64_t m1 = or_argmax_f64(r1, M1), m2 = or_argmax_f64(r2, M2);
    int64_t k = or_resolve(m1, M1, m2, M2, N, 0);
    if (residues) { residues[0] = m1; residues[1] = m2; }
    if (y1o) memcpy(y1o, y1, sizeof(double) * M1);
    if (y2o) memcpy(y2o, y2, sizeof(double) * M2);
    if (r1o) memcpy(r1o, r1, sizeof(double) * M1);
    if (r2o) memcpy(r2o, r2, sizeof(double) * M2);
    free(y1); free(y2); free(r1); free(r2);
    return k;
}

/* ------------------------------------------------------------------ */
/* Aux: the full-resolution score of section 3:                   */
/*     (Tx)_k = sum_{i=0}^{K-1} t_i x_{(k+i) mod N},  k = 0 .. N-1.       */
/*     N*K work: the Eq. (1) brute-force full search (tiny N only).       */
/* ------------------------------------------------------------------ */
void or_full_corr_i8(const int8_t *x, int64_t N, const int8_t *t, int64_t K, int64_t *s) {
    for (int64_t k = 0; k < N; ++k) {
        int64_t acc = 0;
        for (int64_t i = 0; i < K; ++i) acc += (int64_t)t[i] * (int64_t)x[or_mod(k + i, N)];
        s[k] = acc;
    }
}

void or_full_corr_f32(const float *x, int64_t N, const float *t, int64_t K, double *s) {
    for (int64_t k = 0; k < N; ++k) {
        double acc = 0.0;
        for (int64_t i = 0; i < K; ++i) acc += (double)t[i] * (double)x[or_mod(k + i, N)];
        s[k] = acc;
    }
}

/* ------------------------------------------------------------------ */
/* Aux: Eq. (3) as a dense matrix, rows = M+K (strategy 1):  */
/*     Phi = D_rows(circ(r)),  r_k = 1 iff k mod M == 0 (0 <= k < N),     */
/*     circ(v) row j = v right-shifted j times:                 */
/*     Phi[j][c] = r[(c - j) mod N].   Output: int8 [rows][N].            */
/* ------------------------------------------------------------------ */
void or_phi_dense(int64_t N, int64_t M, int64_t rows, int8_t *Phi) {
    for (int64_t j = 0; j < rows; ++j)
        for (int64_t c = 0; c < N; ++c)
            Phi[j * N + c] = (or_mod(c - j, N) % M == 0) ? 1 : 0;
}

/* ------------------------------------------------------------------ */
/* Aux: Theorem 1's T^ = circ([t 0_{M-K}]) applied to y[0..M):   */
/*     (T^ y)_i = sum_{u=0}^{K-1} t_u y_{(i+u) mod M},  i = 0 .. M-1.     */
/* ------------------------------------------------------------------ */
void or_thm1_That_y_i64(const int64_t *y, int64_t M, const int8_t *t, int64_t K, int64_t *out) {
    for (int64_t i = 0; i < M; ++i) {
        int64_t acc = 0;
        for (int64_t u = 0; u < K; ++u) acc += (int64_t)t[u] * y[or_mod(i + u, M)];
        out[i] = acc;
    }
}
