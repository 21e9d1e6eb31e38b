/*
 * cq_oracle.c -- CPU ORACLE. TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference quantiser's hot path
 * (arXiv 1101.0395 artifact, /root/reference/proj), used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the checker.
 * Nothing in the product (paper_1101_0395_b200/) links, imports or calls this
 * file; the product path fails loudly when its CUDA library is missing.
 *
 * Parity pin: tests/test_oracle_golden.py checks this oracle against the
 * reference's golden sweep rows (proj/tmp_acceptance/sweep_a.csv:2-13, via the
 * committed fixtures in tests/golden/) and, where oracle/_ref/libquantref.so
 * exists (compiled from the reference's own sources by oracle/Makefile),
 * against the reference itself on seeded inputs.
 *
 * Two update rules are provided for the Lloyd loop:
 *   CQO_UPDATE_REFERENCE  -- the reference's sequential FP64 sums
 *                            (kmeans.cpp:228-245) and sequential SSE
 *                            (kmeans.cpp:107-114): bit-faithful to the reference.
 *   CQO_UPDATE_EXACT      -- exact integer moments (n, S, Q per cluster), centre
 *                            = S/n in FP64, SSE from the moments with an
 *                            int128 numerator: the device's contract, which is
 *                            bit-identical to the reference for power-of-two
 *                            pixel counts.
 * Assignment (the FP64 walk) is the reference's in both modes.
 *
 * Must be compiled with -ffp-contract=off (the reference Release build has no
 * FMA in these objects: SURVEY.md §0 finding 3).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define CQO_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------------ */
/* mt19937_64 + portable draws (reference: include/quant/rng.hpp:17-54)     */
/* ------------------------------------------------------------------------ */

#define MT_N 312
#define MT_M 156

typedef struct {
    uint64_t s[MT_N];
    int i;
} cqo_rng;

CQO_API void cqo_rng_seed(cqo_rng *r, uint64_t seed) {
    r->s[0] = seed;
    for (int k = 1; k < MT_N; ++k)
        r->s[k] = 6364136223846793005ULL * (r->s[k - 1] ^ (r->s[k - 1] >> 62)) + (uint64_t)k;
    r->i = MT_N;
}

static void mt_refill(cqo_rng *r) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    const uint64_t mat = 0xB5026F5AA96619E9ULL;
    for (int k = 0; k < MT_N; ++k) {
        uint64_t y = (r->s[k] & upper) | (r->s[(k + 1) % MT_N] & lower);
        uint64_t v = r->s[(k + MT_M) % MT_N] ^ (y >> 1);
        if (y & 1ULL) v ^= mat;
        r->s[k] = v;
    }
    r->i = 0;
}

CQO_API uint64_t cqo_rng_u64(cqo_rng *r) {
    if (r->i >= MT_N) mt_refill(r);
    uint64_t x = r->s[r->i++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

/* rng.hpp:25-33: rejection sampling, no modulo bias */
CQO_API uint64_t cqo_rng_below(cqo_rng *r, uint64_t n) {
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t x;
    do { x = cqo_rng_u64(r); } while (x >= limit);
    return x % n;
}

/* rng.hpp:36 */
CQO_API double cqo_rng_unit(cqo_rng *r) { return (double)(cqo_rng_u64(r) >> 11) * 0x1.0p-53; }

CQO_API int cqo_rng_size(void) { return (int)sizeof(cqo_rng); }

/* rng.hpp:43-54: sequential prefix draw. Returns -1 if total mass <= 0. */
static int64_t weighted_draw(const double *mass, uint64_t n, cqo_rng *r) {
    double total = 0.0;
    for (uint64_t i = 0; i < n; ++i) total += mass[i];
    if (!(total > 0.0)) return -1;
    const double u = cqo_rng_unit(r) * total;
    double acc = 0.0;
    for (uint64_t i = 0; i + 1 < n; ++i) {
        acc += mass[i];
        if (u < acc) return (int64_t)i;
    }
    return (int64_t)n - 1;
}

/* ------------------------------------------------------------------------ */
/* colour helpers (reference: include/quant/color.hpp:47-72)                */
/* ------------------------------------------------------------------------ */

static inline double d2pt(const double *a, const double *b) {
    const double dr = a[0] - b[0], dg = a[1] - b[1], db = a[2] - b[2];
    return dr * dr + dg * dg + db * db; /* ((dr*dr)+(dg*dg))+(db*db), no FMA */
}

static inline void unpack(uint32_t c, double *x) {
    x[0] = (double)((c >> 16) & 255u);
    x[1] = (double)((c >> 8) & 255u);
    x[2] = (double)(c & 255u);
}

/* color.hpp:63-68: round half up, clamp */
CQO_API uint8_t cqo_channel_to_u8(double v) {
    double r = floor(v + 0.5);
    if (r < 0.0) r = 0.0;
    if (r > 255.0) r = 255.0;
    return (uint8_t)r;
}

/* correctly rounded unsigned __int128 -> double (shared contract with the device) */
static double u128_to_double(unsigned __int128 x) {
    const uint64_t hi = (uint64_t)(x >> 64);
    if (hi == 0) return (double)(uint64_t)x;
    const int s = 64 - __builtin_clzll(hi);
    uint64_t v = (uint64_t)(x >> s);
    const unsigned __int128 lostmask = (((unsigned __int128)1) << s) - 1;
    if ((x & lostmask) != 0) v |= 1ULL;
    return ldexp((double)v, s);
}

/* ------------------------------------------------------------------------ */
/* histogram in first-occurrence order (reference: src/histogram.cpp:69-104) */
/* The reference dedups through a seeded chained hash; the output contract   */
/* (distinct colours in order of first sight, raw counts, weights =          */
/* count*(1/P)) does not depend on the hash, so a direct 2^24 table states   */
/* the same function.                                                        */
/* ------------------------------------------------------------------------ */

CQO_API int64_t cqo_histogram(const uint8_t *rgb, uint64_t P, uint32_t *colors, uint32_t *counts,
                              uint32_t *first) {
    if (P == 0) return -1;
    int32_t *slot = (int32_t *)malloc(sizeof(int32_t) << 24);
    if (!slot) return -2;
    memset(slot, 0xFF, sizeof(int32_t) << 24);
    int64_t n = 0;
    for (uint64_t p = 0; p < P; ++p) {
        const uint32_t c = ((uint32_t)rgb[3 * p] << 16) | ((uint32_t)rgb[3 * p + 1] << 8) | rgb[3 * p + 2];
        int32_t s = slot[c];
        if (s >= 0) {
            counts[s]++;
        } else {
            slot[c] = (int32_t)n;
            colors[n] = c;
            counts[n] = 1;
            if (first) first[n] = (uint32_t)p;
            ++n;
        }
    }
    free(slot);
    return n;
}

/* histogram.cpp:99-102 */
CQO_API void cqo_weights(const uint32_t *counts, uint64_t n, uint64_t P, double *w) {
    const double inv = 1.0 / (double)P;
    for (uint64_t i = 0; i < n; ++i) w[i] = (double)counts[i] * inv;
}

/* ------------------------------------------------------------------------ */
/* centre distance table (reference: src/kmeans.cpp:14-38)                  */
/* ------------------------------------------------------------------------ */

typedef struct {
    double d;
    uint32_t j;
} dj_t;

static int cmp_dj(const void *a, const void *b) {
    const dj_t *x = (const dj_t *)a, *y = (const dj_t *)b;
    if (x->d != y->d) return x->d < y->d ? -1 : 1;
    return x->j < y->j ? -1 : (x->j > y->j);
}

CQO_API void cqo_center_table(const double *c, int K, double *d2, uint32_t *order) {
    dj_t *row = (dj_t *)malloc(sizeof(dj_t) * (size_t)K);
    for (int i = 0; i < K; ++i)
        for (int j = 0; j < K; ++j) d2[(size_t)i * K + j] = d2pt(c + 3 * i, c + 3 * j);
    for (int i = 0; i < K; ++i) {
        for (int j = 0; j < K; ++j) row[j] = (dj_t){d2[(size_t)i * K + j], (uint32_t)j};
        qsort(row, (size_t)K, sizeof(dj_t), cmp_dj);
        /* self first (kmeans.cpp:32-35): rotate i to the front */
        int at = 0;
        while (row[at].j != (uint32_t)i) ++at;
        dj_t self = row[at];
        memmove(row + 1, row, sizeof(dj_t) * (size_t)at);
        row[0] = self;
        for (int j = 0; j < K; ++j) order[(size_t)i * K + j] = row[j].j;
    }
    free(row);
}

/* kmeans.cpp:40-54 */
CQO_API uint32_t cqo_nearest_full(const double *x, const double *c, int K, uint64_t *ndc) {
    uint32_t best = 0;
    double bd = d2pt(x, c);
    ++*ndc;
    for (int j = 1; j < K; ++j) {
        const double d = d2pt(x, c + 3 * j);
        ++*ndc;
        if (d < bd) { bd = d; best = (uint32_t)j; }
    }
    return best;
}

/* kmeans.cpp:56-79 */
CQO_API uint32_t cqo_assign_sortmeans(const double *x, uint32_t prev, const double *d2,
                                      const uint32_t *order, const double *c, int K,
                                      uint64_t *ndc) {
    const double *drow = d2 + (size_t)prev * K;
    const uint32_t *orow = order + (size_t)prev * K;
    const double pd = d2pt(x, c + 3 * prev);
    ++*ndc;
    const double cutoff = 4.0 * pd;
    double bd = pd;
    uint32_t best = prev;
    for (int j = 1; j < K; ++j) {
        const uint32_t t = orow[j];
        if (drow[t] >= cutoff) break;
        const double d = d2pt(x, c + 3 * t);
        ++*ndc;
        if (d < bd) { bd = d; best = t; }
    }
    return best;
}

/* kmeans.cpp:81-105 */
CQO_API uint32_t cqo_nearest_lowest(const double *x, uint32_t hint, const double *d2,
                                    const uint32_t *order, const double *c, int K,
                                    uint64_t *ndc) {
    const double *drow = d2 + (size_t)hint * K;
    const uint32_t *orow = order + (size_t)hint * K;
    const double pd = d2pt(x, c + 3 * hint);
    ++*ndc;
    const double cutoff = 4.0 * pd;
    double bd = pd;
    uint32_t best = hint;
    for (int j = 1; j < K; ++j) {
        const uint32_t t = orow[j];
        if (drow[t] > cutoff) break;
        const double d = d2pt(x, c + 3 * t);
        ++*ndc;
        if (d < bd || (d == bd && t < best)) { bd = d; best = t; }
    }
    return best;
}

/* ------------------------------------------------------------------------ */
/* empty-cluster repair (reference: src/kmeans.cpp:124-169)                  */
/* ------------------------------------------------------------------------ */

static int repair_empty(const double *pts, const double *w, uint64_t n, double *c, int K,
                        uint32_t *m) {
    uint64_t *size = (uint64_t *)calloc((size_t)K, sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) size[m[i]]++;
    int repairs = 0;
    for (int e = 0; e < K;) {
        if (size[e] != 0) { ++e; continue; }
        uint64_t donor = n;
        double best = -1.0;
        for (uint64_t i = 0; i < n; ++i) {
            const double v = w[i] * d2pt(pts + 3 * i, c + 3 * m[i]);
            if (v > best) { best = v; donor = i; }
        }
        if (best <= 0.0) {
            donor = n;
            for (uint64_t i = 0; i < n; ++i)
                if (size[m[i]] >= 2) { donor = i; break; }
            if (donor == n) { free(size); return -1; }
        }
        size[m[donor]]--;
        m[donor] = (uint32_t)e;
        memcpy(c + 3 * e, pts + 3 * donor, 3 * sizeof(double));
        size[e]++;
        ++repairs;
        e = 0;
    }
    free(size);
    return repairs;
}

/* ------------------------------------------------------------------------ */
/* weighted sort-means (reference: src/kmeans.cpp:173-277, run_lloyd + wsm)  */
/* ------------------------------------------------------------------------ */

enum { CQO_UPDATE_REFERENCE = 0, CQO_UPDATE_EXACT = 1 };

/* error codes mirror the reference's exception sites */
enum {
    CQO_OK = 0,
    CQO_E_NO_CENTERS = -10,   /* kmeans.cpp:176 */
    CQO_E_NO_POINTS = -11,    /* kmeans.cpp:177 */
    CQO_E_K_GT_N = -12,       /* kmeans.cpp:178-181 */
    CQO_E_EPS = -13,          /* kmeans.cpp:185 */
    CQO_E_MAXIT = -14,        /* kmeans.cpp:186 */
    CQO_E_FIXED = -15,        /* kmeans.cpp:187-188 */
    CQO_E_REPAIR = -16,       /* kmeans.cpp:159 */
    CQO_E_INIT_K = -20,       /* init.cpp:15-19 */
    CQO_E_MASS = -21,         /* rng.hpp:47 */
};

/* The exact-moment SSE's summation order over clusters: pairwise on a complete
 * binary tree over the next power of two >= K (zero padding), left + right at
 * every node, in place. The device sums the same tree level by level in
 * parallel (tree_sum_block, lloyd.cu). The reference sums points sequentially
 * (kmeans.cpp:107-114); every order is within its recursive-sum error bound. */
static double tree_sum(double *a, int K) {
    for (int st = 1; st < K; st <<= 1)
        for (int i = 0; i + st < K; i += 2 * st) a[i] = a[i] + a[i + st];
    return K > 0 ? a[0] : 0.0;
}

/* SSE of one cluster from exact moments: (n*Q - |S|^2)/n, numerator in int128 */
static double cluster_sse_exact(uint64_t n, const int64_t *S, uint64_t Q) {
    const unsigned __int128 nq = (unsigned __int128)n * Q;
    const unsigned __int128 ss = (unsigned __int128)((__int128)S[0] * S[0]) +
                                 (unsigned __int128)((__int128)S[1] * S[1]) +
                                 (unsigned __int128)((__int128)S[2] * S[2]);
    return u128_to_double(nq - ss) / (double)n;
}

CQO_API int cqo_wsm(const uint32_t *colors, const uint32_t *counts, uint64_t n, uint64_t P,
                    const double *init, int K, double eps, int max_it, int fixed_it, int mode,
                    double *centers_out, uint32_t *labels_out, double *sse_trace, int *iters_out,
                    uint64_t *ndc_out, int *repairs_out, uint32_t *hist_labels,
                    double *hist_centers) {
    /* validate_run (kmeans.cpp:173-188) and wsm weights check (:275) */
    if (K <= 0) return CQO_E_NO_CENTERS;
    if (n == 0) return CQO_E_NO_POINTS;
    if ((uint64_t)K > n) return CQO_E_K_GT_N;
    if (eps < 0.0) return CQO_E_EPS;
    if (max_it <= 0) return CQO_E_MAXIT;
    if (fixed_it < 0) return CQO_E_FIXED;
    const int limit = fixed_it > 0 ? fixed_it : max_it;

    double *pts = (double *)malloc(sizeof(double) * 3 * n);
    double *w = (double *)malloc(sizeof(double) * n);
    for (uint64_t i = 0; i < n; ++i) unpack(colors[i], pts + 3 * i);
    cqo_weights(counts, n, P, w);

    double *c = centers_out;
    memcpy(c, init, sizeof(double) * 3 * (size_t)K);
    uint32_t *m = labels_out;
    memset(m, 0, sizeof(uint32_t) * n);
    double *tab = (double *)malloc(sizeof(double) * (size_t)K * K);
    uint32_t *ord = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)K * K);
    double *sum = (double *)malloc(sizeof(double) * 4 * (size_t)K);
    uint64_t *mn = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)K);
    int64_t *mS = (int64_t *)malloc(sizeof(int64_t) * 3 * (size_t)K);
    uint64_t *mQ = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)K);
    double *sterm = (double *)malloc(sizeof(double) * (size_t)K);

    uint64_t ndc = 0;
    int repairs = 0, iter, rc = CQO_OK;
    for (iter = 1;; ++iter) {
        if (iter > 1) {
            cqo_center_table(c, K, tab, ord);
            for (uint64_t i = 0; i < n; ++i)
                m[i] = cqo_assign_sortmeans(pts + 3 * i, m[i], tab, ord, c, K, &ndc);
        } else {
            for (uint64_t i = 0; i < n; ++i) m[i] = cqo_nearest_full(pts + 3 * i, c, K, &ndc);
        }
        if (hist_labels) memcpy(hist_labels + (size_t)(iter - 1) * n, m, sizeof(uint32_t) * n);
        if (hist_centers)
            memcpy(hist_centers + (size_t)(iter - 1) * 3 * K, c, sizeof(double) * 3 * (size_t)K);

        const int rep = repair_empty(pts, w, n, c, K, m);
        if (rep < 0) { rc = CQO_E_REPAIR; break; }
        repairs += rep;

        double sse = 0.0;
        if (mode == CQO_UPDATE_REFERENCE) {
            memset(sum, 0, sizeof(double) * 4 * (size_t)K);
            for (uint64_t i = 0; i < n; ++i) {
                double *s = sum + 4 * m[i];
                s[0] += w[i] * pts[3 * i];
                s[1] += w[i] * pts[3 * i + 1];
                s[2] += w[i] * pts[3 * i + 2];
                s[3] += w[i];
            }
            for (int k = 0; k < K; ++k) {
                const double *s = sum + 4 * k;
                if (s[3] > 0.0) {
                    c[3 * k] = s[0] / s[3];
                    c[3 * k + 1] = s[1] / s[3];
                    c[3 * k + 2] = s[2] / s[3];
                }
            }
            for (uint64_t i = 0; i < n; ++i) sse += w[i] * d2pt(pts + 3 * i, c + 3 * m[i]);
        } else {
            memset(mn, 0, sizeof(uint64_t) * (size_t)K);
            memset(mS, 0, sizeof(int64_t) * 3 * (size_t)K);
            memset(mQ, 0, sizeof(uint64_t) * (size_t)K);
            for (uint64_t i = 0; i < n; ++i) {
                const uint32_t k = m[i], q = counts[i];
                const int64_t r = (colors[i] >> 16) & 255, g = (colors[i] >> 8) & 255, b = colors[i] & 255;
                mn[k] += q;
                mS[3 * k] += (int64_t)q * r;
                mS[3 * k + 1] += (int64_t)q * g;
                mS[3 * k + 2] += (int64_t)q * b;
                mQ[k] += (uint64_t)q * (uint64_t)(r * r + g * g + b * b);
            }
            for (int k = 0; k < K; ++k) {
                sterm[k] = 0.0;
                if (mn[k] == 0) continue;
                const double nd = (double)mn[k];
                c[3 * k] = (double)mS[3 * k] / nd;
                c[3 * k + 1] = (double)mS[3 * k + 1] / nd;
                c[3 * k + 2] = (double)mS[3 * k + 2] / nd;
                sterm[k] = cluster_sse_exact(mn[k], mS + 3 * k, mQ[k]);
            }
            sse = tree_sum(sterm, K) / (double)P;
        }
        sse_trace[iter - 1] = sse;

        /* termination (kmeans.cpp:249-257) */
        if (fixed_it > 0) {
            if (iter >= limit) break;
        } else {
            if (sse == 0.0) break;
            if (iter >= 2 && (sse_trace[iter - 2] - sse) / sse <= eps) break;
            if (iter >= limit) break;
        }
    }
    *iters_out = iter;
    *ndc_out = ndc;
    *repairs_out = repairs;
    free(pts); free(w); free(tab); free(ord); free(sum); free(mn); free(mS); free(mQ); free(sterm);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* initialisers (reference: src/init.cpp:37-52, 127-138, 295-314)            */
/* ------------------------------------------------------------------------ */

CQO_API int cqo_init_maximin(const uint32_t *colors, const uint32_t *counts, uint64_t n, uint64_t P,
                             int K, uint64_t seed, int weighted_first, double *centers) {
    if (K < 1 || (uint64_t)K > n) return CQO_E_INIT_K;
    cqo_rng rng;
    cqo_rng_seed(&rng, seed);
    double *w = (double *)malloc(sizeof(double) * n);
    cqo_weights(counts, n, P, w);
    int64_t first = weighted_first ? weighted_draw(w, n, &rng) : (int64_t)cqo_rng_below(&rng, n);
    free(w);
    if (first < 0) return CQO_E_MASS;
    double *pts = (double *)malloc(sizeof(double) * 3 * n);
    double *md = (double *)malloc(sizeof(double) * n);
    for (uint64_t i = 0; i < n; ++i) unpack(colors[i], pts + 3 * i);
    memcpy(centers, pts + 3 * first, 3 * sizeof(double));
    for (uint64_t i = 0; i < n; ++i) md[i] = d2pt(pts + 3 * i, centers);
    for (int k = 1; k < K; ++k) {
        uint64_t best = 0;
        for (uint64_t p = 1; p < n; ++p)
            if (md[p] > md[best]) best = p;
        memcpy(centers + 3 * k, pts + 3 * best, 3 * sizeof(double));
        for (uint64_t p = 0; p < n; ++p) {
            const double d = d2pt(pts + 3 * p, centers + 3 * k);
            if (d < md[p]) md[p] = d;
        }
    }
    free(pts); free(md);
    return CQO_OK;
}

CQO_API int cqo_init_kmeanspp(const uint32_t *colors, const uint32_t *counts, uint64_t n, uint64_t P,
                              int K, uint64_t seed, double *centers) {
    if (K < 1 || (uint64_t)K > n) return CQO_E_INIT_K;
    cqo_rng rng;
    cqo_rng_seed(&rng, seed);
    double *w = (double *)malloc(sizeof(double) * n);
    double *pts = (double *)malloc(sizeof(double) * 3 * n);
    double *md = (double *)malloc(sizeof(double) * n);
    double *mass = (double *)malloc(sizeof(double) * n);
    cqo_weights(counts, n, P, w);
    for (uint64_t i = 0; i < n; ++i) unpack(colors[i], pts + 3 * i);
    int rc = CQO_OK;
    int64_t pick = weighted_draw(w, n, &rng);
    if (pick < 0) { rc = CQO_E_MASS; goto out; }
    memcpy(centers, pts + 3 * pick, 3 * sizeof(double));
    for (uint64_t i = 0; i < n; ++i) md[i] = d2pt(pts + 3 * i, centers);
    for (int k = 1; k < K; ++k) {
        for (uint64_t i = 0; i < n; ++i) mass[i] = w[i] * md[i];
        pick = weighted_draw(mass, n, &rng);
        if (pick < 0) { rc = CQO_E_MASS; goto out; }
        memcpy(centers + 3 * k, pts + 3 * pick, 3 * sizeof(double));
        for (uint64_t i = 0; i < n; ++i) {
            const double d = d2pt(pts + 3 * i, centers + 3 * k);
            if (d < md[i]) md[i] = d;
        }
    }
out:
    free(w); free(pts); free(md); free(mass);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* pixel mapping + MSE (reference: src/metrics.cpp:15-55)                    */
/* mode REFERENCE: the reference's sequential hint walk and FP64 total.      */
/* mode EXACT: the same lookup (lowest-index exact argmin, kmeans.hpp:88-96; */
/* ndc = MappingResult::ndc) and MSE from exact per-cluster pixel moments:   */
/*   sum_k [ (n Q - |S|^2)/n + n*|c - S/n|^2 ] / P, k ascending.             */
/* ------------------------------------------------------------------------ */

CQO_API int cqo_map_pixels(const uint8_t *rgb, uint64_t P, const double *pal, int K, int mode,
                           uint32_t *indices, uint8_t *quant, double *mse_out, uint64_t *ndc_out) {
    if (K < 1) return -30;
    if (P == 0) return -31;
    uint8_t *pal8 = (uint8_t *)malloc(3 * (size_t)K);
    for (int k = 0; k < 3 * K; ++k) pal8[k] = cqo_channel_to_u8(pal[k]);
    double *tab = (double *)malloc(sizeof(double) * (size_t)K * K);
    uint32_t *ord = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)K * K);
    cqo_center_table(pal, K, tab, ord);
    int32_t *cache = (int32_t *)malloc(sizeof(int32_t) << 24);
    memset(cache, 0xFF, sizeof(int32_t) << 24);
    uint64_t ndc = 0;
    if (mode == CQO_UPDATE_REFERENCE) {
        double total = 0.0;
        uint32_t hint = 0;
        for (uint64_t p = 0; p < P; ++p) {
            const uint32_t key = ((uint32_t)rgb[3 * p] << 16) | ((uint32_t)rgb[3 * p + 1] << 8) | rgb[3 * p + 2];
            double x[3];
            unpack(key, x);
            uint32_t idx;
            if (cache[key] >= 0) {
                idx = (uint32_t)cache[key];
            } else {
                idx = cqo_nearest_lowest(x, hint, tab, ord, pal, K, &ndc);
                cache[key] = (int32_t)idx;
                hint = idx;
            }
            indices[p] = idx;
            memcpy(quant + 3 * p, pal8 + 3 * idx, 3);
            total += d2pt(pal + 3 * idx, x);
        }
        *mse_out = total / (double)P;
    } else {
        uint64_t *mn = (uint64_t *)calloc((size_t)K, sizeof(uint64_t));
        int64_t *mS = (int64_t *)calloc(3 * (size_t)K, sizeof(int64_t));
        uint64_t *mQ = (uint64_t *)calloc((size_t)K, sizeof(uint64_t));
        uint32_t hint = 0;
        for (uint64_t p = 0; p < P; ++p) {
            const uint32_t key = ((uint32_t)rgb[3 * p] << 16) | ((uint32_t)rgb[3 * p + 1] << 8) | rgb[3 * p + 2];
            uint32_t idx;
            if (cache[key] >= 0) {
                idx = (uint32_t)cache[key];
            } else {
                /* the same hint-seeded pruned lookup as the reference (so ndc is
                 * MappingResult::ndc): its result is the exact lowest-index argmin */
                double x[3];
                unpack(key, x);
                idx = cqo_nearest_lowest(x, hint, tab, ord, pal, K, &ndc);
                cache[key] = (int32_t)idx;
                hint = idx;
            }
            indices[p] = idx;
            memcpy(quant + 3 * p, pal8 + 3 * idx, 3);
            const int64_t r = rgb[3 * p], g = rgb[3 * p + 1], b = rgb[3 * p + 2];
            mn[idx] += 1;
            mS[3 * idx] += r;
            mS[3 * idx + 1] += g;
            mS[3 * idx + 2] += b;
            mQ[idx] += (uint64_t)(r * r + g * g + b * b);
        }
        double total = 0.0;
        for (int k = 0; k < K; ++k) {
            if (mn[k] == 0) continue;
            const double nd = (double)mn[k];
            const double a = cluster_sse_exact(mn[k], mS + 3 * k, mQ[k]);
            const double dr = pal[3 * k] - (double)mS[3 * k] / nd;
            const double dg = pal[3 * k + 1] - (double)mS[3 * k + 1] / nd;
            const double db = pal[3 * k + 2] - (double)mS[3 * k + 2] / nd;
            total += a + nd * (dr * dr + dg * dg + db * db);
        }
        *mse_out = total / (double)P;
        free(mn); free(mS); free(mQ);
    }
    if (ndc_out) *ndc_out = ndc;
    free(pal8); free(tab); free(ord); free(cache);
    return 0;
}

/* psnr (metrics.cpp:71-75) */
CQO_API double cqo_psnr(double mse) {
    if (mse == 0.0) return INFINITY;
    return 20.0 * log10(255.0 / sqrt(mse));
}

/* coarse 32x32x32 histogram (precluster.cpp:13-47; bin_index/bin_of,
 * precluster.hpp:26-29): per bin (r>>3, g>>3, b>>3), r-major, the count and
 * the sums of r, g, b and r^2+g^2+b^2 over the original values, weighted by
 * each distinct colour's pixel count (the weighted overload; the pixel
 * overload is the same with every pixel counted once).
 * out: 5 x 32768 int64 -- count | sum_r | sum_g | sum_b | sum_sq. */
CQO_API void cqo_coarse_histogram(const uint32_t *colors, const uint32_t *counts, uint64_t n, int64_t *out) {
    const size_t B = 32768;
    memset(out, 0, sizeof(int64_t) * 5 * B);
    for (uint64_t i = 0; i < n; ++i) {
        const int64_t r = (colors[i] >> 16) & 255, g = (colors[i] >> 8) & 255, b = colors[i] & 255;
        const int64_t c = counts[i];
        const size_t bin = ((size_t)(r >> 3) * 32 + (size_t)(g >> 3)) * 32 + (size_t)(b >> 3);
        out[bin] += c;
        out[B + bin] += c * r;
        out[2 * B + bin] += c * g;
        out[3 * B + bin] += c * b;
        out[4 * B + bin] += c * (r * r + g * g + b * b);
    }
}
