/*
 * semd_oracle.c -- TEST INFRASTRUCTURE ONLY (see semd_oracle.h).
 *
 * A line-by-line restatement, in plain C, of the reference algorithm for the
 * serial-EMD hot path. Every floating-point expression keeps the reference's
 * operation order so that, compiled with -ffp-contract=off and no FMA, the
 * results are bit-identical to /root/reference/proj/src/emd.cpp and
 * serialize.cpp. Citations are relative to /root/reference/proj/.
 */
#include "semd_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* so_last_error(void) { return g_err; }
void so_free(void* p) { free(p); }

void so_decomp_free(so_decomp* d) {
    if (!d) return;
    free(d->imfs);
    free(d->residue);
    free(d->sift_counts);
    memset(d, 0, sizeof *d);
}

static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* Order-sensitive list hash: sum over ranks j of mix64(side | j<<32 ^ idx).
 * Integer addition commutes, so the GPU computes it with a parallel reduction. */
uint64_t so_trace_hash(const size_t* max_idx, size_t n_max, const size_t* min_idx, size_t n_min) {
    uint64_t h = 0;
    for (size_t j = 0; j < n_max; ++j) h += mix64(((uint64_t)j << 32) ^ (uint64_t)max_idx[j]);
    for (size_t j = 0; j < n_min; ++j)
        h += mix64(0x8000000000000000ULL ^ ((uint64_t)j << 32) ^ (uint64_t)min_idx[j]);
    return h;
}

static void trace_push(so_trace* tr, int task, int m, int k, int iter, size_t nmax, size_t nmin, uint64_t h) {
    if (!tr) return;
    if (tr->count < tr->cap) {
        so_trace_rec* r = &tr->rec[tr->count];
        r->task = task; r->m = m; r->k = k; r->iter = iter;
        r->n_max = (uint32_t)nmax; r->n_min = (uint32_t)nmin; r->hash = h;
    }
    tr->count++;
}

/* Trace context threaded through the sifting calls. */
typedef struct { so_trace* tr; int task, m, k; } tctx;

/* ---------------------------------------------------------------- extrema */

/* emd.cpp:10-35: runs of exactly equal samples; an interior run is a max if
 * strictly above both neighbours, a min if strictly below; reported at the
 * floor midpoint; runs touching index 0 or n-1 are never extrema. */
int so_find_extrema(const double* x, size_t n, size_t* max_idx, double* max_val, size_t* n_max,
                    size_t* min_idx, double* min_val, size_t* n_min) {
    if (n < 3) return fail(SO_INVALID, "find_extrema: signal too short (need at least 3 samples)");
    size_t nM = 0, nm = 0, run_start = 0;
    for (size_t i = 1; i <= n; ++i) {
        if (i < n && x[i] == x[run_start]) continue;
        const size_t run_end = i - 1;
        if (run_start > 0 && run_end < n - 1) {
            const double v = x[run_start];
            const double left = x[run_start - 1];
            const double right = x[run_end + 1];
            const size_t mid = (run_start + run_end) / 2;
            if (v > left && v > right) {
                max_idx[nM] = mid; max_val[nM] = v; ++nM;
            } else if (v < left && v < right) {
                min_idx[nm] = mid; min_val[nm] = v; ++nm;
            }
        }
        run_start = i;
    }
    *n_max = nM;
    *n_min = nm;
    return SO_OK;
}

/* --------------------------------------------------------------- envelope */

/* emd.cpp:41-87: natural cubic spline through (xs, ys) sampled at 0..length-1. */
static int spline_sample(const double* xs, const double* ys, size_t n, size_t length, double* out) {
    if (n == 2) { /* :46-51 */
        const double slope = (ys[1] - ys[0]) / (xs[1] - xs[0]);
        for (size_t t = 0; t < length; ++t) out[t] = ys[0] + slope * ((double)t - xs[0]);
        return SO_OK;
    }
    double* m = calloc(n, sizeof(double));
    double* diag = calloc(n, sizeof(double));
    double* rhs = calloc(n, sizeof(double));
    double* upper = calloc(n, sizeof(double));
    if (!m || !diag || !rhs || !upper) {
        free(m); free(diag); free(rhs); free(upper);
        return fail(SO_NOMEM, "out of memory");
    }
    for (size_t i = 1; i + 1 < n; ++i) { /* :57-63 */
        const double h0 = xs[i] - xs[i - 1];
        const double h1 = xs[i + 1] - xs[i];
        diag[i] = 2.0 * (h0 + h1);
        upper[i] = h1;
        rhs[i] = 6.0 * ((ys[i + 1] - ys[i]) / h1 - (ys[i] - ys[i - 1]) / h0);
    }
    for (size_t i = 2; i + 1 < n; ++i) { /* :64-69 Thomas forward sweep */
        const double h0 = xs[i] - xs[i - 1];
        const double w = h0 / diag[i - 1];
        diag[i] -= w * upper[i - 1];
        rhs[i] -= w * rhs[i - 1];
    }
    for (size_t i = n - 2; i >= 1; --i) { /* :70-73 back substitution */
        m[i] = (rhs[i] - upper[i] * m[i + 1]) / diag[i];
        if (i == 1) break;
    }
    size_t seg = 0; /* :76-85 segment march */
    for (size_t t = 0; t < length; ++t) {
        const double tt = (double)t;
        while (seg + 2 < n && tt > xs[seg + 1]) ++seg;
        const double h = xs[seg + 1] - xs[seg];
        const double a = (xs[seg + 1] - tt) / h;
        const double b = (tt - xs[seg]) / h;
        out[t] = a * ys[seg] + b * ys[seg + 1] +
                 ((a * a * a - a) * m[seg] + (b * b * b - b) * m[seg + 1]) * (h * h) / 6.0;
    }
    free(m); free(diag); free(rhs); free(upper);
    return SO_OK;
}

/* emd.cpp:91-125: mirror the two outermost extrema across each end unless an
 * extremum sits on that end, then fit the natural spline. */
int so_envelope(const size_t* idx, const double* val, size_t n, size_t length, double* out) {
    if (n < 2) return fail(SO_INSUFFICIENT, "envelope: need at least 2 extrema, got %zu", n);
    const double end = (double)(length - 1);
    double* xs = malloc((n + 4) * sizeof(double));
    double* ys = malloc((n + 4) * sizeof(double));
    if (!xs || !ys) { free(xs); free(ys); return fail(SO_NOMEM, "out of memory"); }
    size_t N = 0;
    if (idx[0] != 0) { /* :107-112 descending source order */
        for (size_t k = (n < 2 ? n : 2); k-- > 0;) {
            xs[N] = -(double)idx[k];
            ys[N] = val[k];
            ++N;
        }
    }
    for (size_t k = 0; k < n; ++k) { xs[N] = (double)idx[k]; ys[N] = val[k]; ++N; }
    if (idx[n - 1] != length - 1) { /* :117-122 (emits the non-monotone last knot) */
        for (size_t k = (n >= 2 ? n - 2 : 0); k < n; ++k) {
            xs[N] = 2.0 * end - (double)idx[k];
            ys[N] = val[k];
            ++N;
        }
    }
    int rc = spline_sample(xs, ys, N, length, out);
    free(xs); free(ys);
    return rc;
}

/* ------------------------------------------------------------ extract_imf */

typedef struct {
    size_t *max_idx, *min_idx;
    double *max_val, *min_val, *upper, *lower;
} scratch;

static int scratch_init(scratch* s, size_t n) {
    s->max_idx = malloc(n * sizeof(size_t));
    s->min_idx = malloc(n * sizeof(size_t));
    s->max_val = malloc(n * sizeof(double));
    s->min_val = malloc(n * sizeof(double));
    s->upper = malloc(n * sizeof(double));
    s->lower = malloc(n * sizeof(double));
    if (!s->max_idx || !s->min_idx || !s->max_val || !s->min_val || !s->upper || !s->lower)
        return fail(SO_NOMEM, "out of memory");
    return SO_OK;
}

static void scratch_free(scratch* s) {
    free(s->max_idx); free(s->min_idx); free(s->max_val); free(s->min_val); free(s->upper); free(s->lower);
}

/* Test hook: num/den of every sift of the next extract_imf (so_sd_ratios). */
static double* g_ratio_out = NULL;
static size_t g_ratio_cap = 0, g_ratio_n = 0;

/* emd.cpp:127-153 */
static int extract_imf_t(const double* x, size_t n, const so_sift_cfg* cfg, double* cur, int32_t* count,
                         const tctx* tc) {
    memcpy(cur, x, n * sizeof(double));
    *count = 0;
    if (cfg->max_sift_iters <= 0) return SO_OK;
    scratch s;
    int rc = scratch_init(&s, n);
    if (rc) { scratch_free(&s); return rc; }
    for (int iter = 0; iter < cfg->max_sift_iters; ++iter) {
        size_t nM, nm;
        rc = so_find_extrema(cur, n, s.max_idx, s.max_val, &nM, s.min_idx, s.min_val, &nm);
        if (rc) break;
        if (tc) trace_push(tc->tr, tc->task, tc->m, tc->k, iter, nM, nm,
                           so_trace_hash(s.max_idx, nM, s.min_idx, nm));
        rc = so_envelope(s.max_idx, s.max_val, nM, n, s.upper);
        if (rc == SO_OK) rc = so_envelope(s.min_idx, s.min_val, nm, n, s.lower);
        if (rc == SO_INSUFFICIENT) {
            rc = (*count == 0) ? SO_INSUFFICIENT : SO_OK; /* :137-139 */
            break;
        }
        if (rc) break;
        double num = 0.0, den = 0.0; /* :142-148 */
        for (size_t i = 0; i < n; ++i) {
            const double mean = 0.5 * (s.upper[i] + s.lower[i]);
            num += mean * mean;
            den += cur[i] * cur[i];
            cur[i] -= mean;
        }
        ++*count;
        if (g_ratio_out && g_ratio_n < g_ratio_cap) g_ratio_out[g_ratio_n++] = num / den;
        if (den == 0.0 || num / den < cfg->sd_threshold) break; /* :150 */
    }
    scratch_free(&s);
    return rc;
}

int so_extract_imf(const double* x, size_t n, const so_sift_cfg* cfg, double* imf, int32_t* sift_count,
                   so_trace* tr) {
    tctx tc = {tr, 0, 0, 0};
    return extract_imf_t(x, n, cfg, imf, sift_count, &tc);
}

/* extract_imf (emd.cpp:127-153) recording the reference's SD ratio num/den of every sift
 * (emd.cpp:150, sequential sums) -- the adversarial-threshold tests of the GPU's certified stop test. */
int so_sd_ratios(const double* x, size_t n, const so_sift_cfg* cfg, double* imf, int32_t* sift_count, double* ratios,
                 size_t cap, size_t* count) {
    g_ratio_out = ratios;
    g_ratio_cap = cap;
    g_ratio_n = 0;
    const int rc = extract_imf_t(x, n, cfg, imf, sift_count, NULL);
    *count = g_ratio_n;
    g_ratio_out = NULL;
    return rc;
}

/* -------------------------------------------------------------------- emd */

typedef struct {
    double* data;
    int32_t* counts;
    size_t K, cap, n;
} imf_list;

static int list_push(imf_list* l, const double* v, int32_t count) {
    if (l->K == l->cap) {
        size_t nc = l->cap ? 2 * l->cap : 8;
        double* nd = realloc(l->data, nc * l->n * sizeof(double));
        if (!nd) return fail(SO_NOMEM, "out of memory");
        l->data = nd;
        int32_t* ncn = realloc(l->counts, nc * sizeof(int32_t));
        if (!ncn) return fail(SO_NOMEM, "out of memory");
        l->counts = ncn;
        l->cap = nc;
    }
    if (v) memcpy(l->data + l->K * l->n, v, l->n * sizeof(double));
    else memset(l->data + l->K * l->n, 0, l->n * sizeof(double));
    l->counts[l->K] = count;
    l->K++;
    return SO_OK;
}

static void to_decomp(imf_list* l, double* residue, so_decomp* out) {
    out->K = l->K;
    out->n = l->n;
    out->imfs = l->data ? l->data : malloc(1);
    out->sift_counts = l->counts ? l->counts : malloc(sizeof(int32_t));
    out->residue = residue;
}

/* emd.cpp:155-172 */
static int emd_t(const double* x, size_t n, const so_sift_cfg* cfg, so_decomp* out, so_trace* tr, int m) {
    if (n < 4) return fail(SO_INVALID, "emd: signal too short (need at least 4 samples)");
    imf_list l = {0};
    l.n = n;
    double* residue = malloc(n * sizeof(double));
    double* imf = malloc(n * sizeof(double));
    if (!residue || !imf) { free(residue); free(imf); return fail(SO_NOMEM, "out of memory"); }
    memcpy(residue, x, n * sizeof(double));
    int rc = SO_OK;
    while (cfg->max_imfs == 0 || l.K < (size_t)cfg->max_imfs) {
        int32_t count = 0;
        tctx tc = {tr, 0, m, (int)l.K};
        rc = extract_imf_t(residue, n, cfg, imf, &count, &tc);
        if (rc == SO_INSUFFICIENT) { rc = SO_OK; break; }
        if (rc) break;
        for (size_t i = 0; i < n; ++i) residue[i] -= imf[i];
        rc = list_push(&l, imf, count);
        if (rc) break;
    }
    free(imf);
    if (rc) { free(residue); free(l.data); free(l.counts); return rc; }
    to_decomp(&l, residue, out);
    return SO_OK;
}

int so_emd(const double* x, size_t n, const so_sift_cfg* cfg, so_decomp* out, so_trace* tr) {
    return emd_t(x, n, cfg, out, tr, 0);
}

/* ------------------------------------------------------------------ noise */

/* emd.cpp:174-179 (splitmix64 finaliser of base + golden-ratio * (index+1)) */
uint64_t so_derive_seed(uint64_t base, uint64_t index) {
    uint64_t z = base + 0x9E3779B97F4A7C15ULL * (index + 1);
    return mix64(z);
}

/* std::mt19937_64 as specified by [rand.eng.mers] / [rand.predef]:
 * w=64 n=312 m=156 r=31 a=0xB5026F5AA96619E9 u=29 d=0x5555555555555555
 * s=17 b=0x71D67FFFEDA60000 t=37 c=0xFFF7EEE000000000 l=43 f=6364136223846793005 */
typedef struct { uint64_t mt[312]; int idx; } mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i) g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

void so_mt19937_64(uint64_t seed, size_t n, uint64_t* out) {
    mt64 g;
    mt64_seed(&g, seed);
    for (size_t i = 0; i < n; ++i) out[i] = mt64_next(&g);
}

/* emd.cpp:181-200: Box-Muller over ((draw >> 11) + 1) * 2^-53 in (0, 1]. */
int so_white_noise(size_t n, uint64_t seed, double std, double* out) {
    if (std < 0.0) return fail(SO_INVALID, "white_noise: std must be non-negative");
    if (std == 0.0) { memset(out, 0, n * sizeof(double)); return SO_OK; }
    mt64 g;
    mt64_seed(&g, seed);
    const double two_pi = 6.283185307179586476925286766559;
    for (size_t i = 0; i < n; i += 2) {
        const double u1 = (double)((mt64_next(&g) >> 11) + 1) * 0x1.0p-53;
        const double r = std * sqrt(-2.0 * log(u1));
        const double u2 = (double)((mt64_next(&g) >> 11) + 1) * 0x1.0p-53;
        const double theta = two_pi * u2;
        out[i] = r * cos(theta);
        if (i + 1 < n) out[i + 1] = r * sin(theta);
    }
    return SO_OK;
}

/* emd.cpp:202-207 */
int so_noise_mode(const double* w, size_t n, size_t i, const so_sift_cfg* cfg, double* out) {
    if (i == 0) return fail(SO_INVALID, "noise_mode: mode index is 1-based");
    so_decomp d = {0};
    int rc = so_emd(w, n, cfg, &d, NULL);
    if (rc) return rc;
    if (i - 1 < d.K) memcpy(out, d.imfs + (i - 1) * n, n * sizeof(double));
    else memset(out, 0, n * sizeof(double));
    so_decomp_free(&d);
    return SO_OK;
}

/* emd.cpp:209-217: two-pass population std with sequential sums. */
double so_signal_std(const double* x, size_t n) {
    if (n == 0) return 0.0;
    double mean = 0.0;
    for (size_t i = 0; i < n; ++i) mean += x[i];
    mean /= (double)n;
    double acc = 0.0;
    for (size_t i = 0; i < n; ++i) acc += (x[i] - mean) * (x[i] - mean);
    return sqrt(acc / (double)n);
}

static int validate_ensemble(const so_ens_cfg* e) { /* emd.cpp:221-224 */
    if (e->nr < 1) return fail(SO_INVALID, "ensemble: nr must be at least 1");
    if (e->nstd < 0.0) return fail(SO_INVALID, "ensemble: nstd must be non-negative");
    return SO_OK;
}

/* ------------------------------------------------------------------- eemd */

/* emd.cpp:237-251, streamed: realization m's IMF k is added to sums[k] in
 * realization order, exactly the reference's accumulation order (:249-251),
 * without holding all NR decompositions. Sums are left unscaled. */
int so_eemd_partial(const double* x, size_t n, const so_sift_cfg* cfg, const so_ens_cfg* ens,
                    int32_t m_begin, int32_t m_end, so_decomp* sums, so_trace* tr) {
    int rc = validate_ensemble(ens);
    if (rc) return rc;
    const double beta = ens->nstd * so_signal_std(x, n); /* :233 */
    imf_list l = {0};
    l.n = n;
    double* w = malloc((n ? n : 1) * sizeof(double));
    double* xm = malloc((n ? n : 1) * sizeof(double));
    if (!w || !xm) { free(w); free(xm); return fail(SO_NOMEM, "out of memory"); }
    for (int32_t m = m_begin; m < m_end && rc == SO_OK; ++m) {
        so_white_noise(n, so_derive_seed(ens->base_seed, (uint64_t)m), 1.0, w); /* :238 */
        for (size_t i = 0; i < n; ++i) xm[i] = x[i] + beta * w[i];              /* :240 */
        so_decomp d = {0};
        rc = emd_t(xm, n, cfg, &d, tr, m); /* :241 */
        if (rc) break;
        while (l.K < d.K && rc == SO_OK) rc = list_push(&l, NULL, 0);
        for (size_t k = 0; k < d.K; ++k) {
            double* o = l.data + k * n;
            const double* v = d.imfs + k * n;
            for (size_t i = 0; i < n; ++i) o[i] += v[i];
        }
        so_decomp_free(&d);
    }
    free(w); free(xm);
    if (rc) { free(l.data); free(l.counts); return rc; }
    double* residue = calloc(n ? n : 1, sizeof(double));
    to_decomp(&l, residue, sums);
    return SO_OK;
}

int so_eemd(const double* x, size_t n, const so_sift_cfg* cfg, const so_ens_cfg* ens, so_decomp* out,
            so_trace* tr) {
    int rc = validate_ensemble(ens);
    if (rc) return rc;
    if (ens->nstd == 0.0) return emd_t(x, n, cfg, out, tr, 0); /* :230 */
    rc = so_eemd_partial(x, n, cfg, ens, 0, ens->nr, out, tr);
    if (rc) return rc;
    const double inv = 1.0 / (double)ens->nr; /* :252-254 */
    for (size_t q = 0; q < out->K * n; ++q) out->imfs[q] *= inv;
    memcpy(out->residue, x, n * sizeof(double)); /* :258-260 */
    for (size_t k = 0; k < out->K; ++k)
        for (size_t i = 0; i < n; ++i) out->residue[i] -= out->imfs[k * n + i];
    memset(out->sift_counts, 0, (out->K ? out->K : 1) * sizeof(int32_t));
    return SO_OK;
}

/* ---------------------------------------------------------------- ceemdan */

/* emd.cpp:280-286: first mode of s, or zeros when s cannot be sifted. */
static int first_mode(const double* s, size_t n, const so_sift_cfg* cfg, double* out, const tctx* tc) {
    int32_t c;
    int rc = extract_imf_t(s, n, cfg, out, &c, tc);
    if (rc == SO_INSUFFICIENT) { memset(out, 0, n * sizeof(double)); return SO_OK; }
    return rc;
}

/* emd.cpp:264-344 */
int so_ceemdan(const double* x, size_t n, const so_sift_cfg* cfg, const so_ens_cfg* ens, so_decomp* out,
               so_trace* tr) {
    int rc = validate_ensemble(ens);
    if (rc) return rc;
    if (ens->nstd == 0.0) return emd_t(x, n, cfg, out, tr, 0); /* :266 */
    if (n < 4) return fail(SO_INVALID, "ceemdan: signal too short (need at least 4 samples)");
    const size_t nr = (size_t)ens->nr;
    double* noise_res = malloc(nr * n * sizeof(double));
    unsigned char* alive = malloc(nr);
    double* residue = malloc(n * sizeof(double));
    double* mode = malloc(n * sizeof(double));
    double* sm = malloc(n * sizeof(double));
    double* ei = malloc(n * sizeof(double));
    double* e1 = malloc(n * sizeof(double));
    scratch s;
    int src = scratch_init(&s, n);
    imf_list l = {0};
    l.n = n;
    if (!noise_res || !alive || !residue || !mode || !sm || !ei || !e1 || src) {
        rc = fail(SO_NOMEM, "out of memory");
        goto done;
    }
    for (size_t m = 0; m < nr; ++m) { /* :276-277 */
        so_white_noise(n, so_derive_seed(ens->base_seed, m), 1.0, noise_res + m * n);
        alive[m] = 1;
    }
    memcpy(residue, x, n * sizeof(double));
    { /* mode 1, :292-307 */
        const double beta0 = ens->nstd * so_signal_std(x, n);
        memset(mode, 0, n * sizeof(double));
        for (size_t m = 0; m < nr; ++m) {
            const double* w = noise_res + m * n;
            for (size_t i = 0; i < n; ++i) sm[i] = x[i] + beta0 * w[i];
            tctx tc = {tr, 2, (int)m, 0};
            rc = first_mode(sm, n, cfg, e1, &tc);
            if (rc) goto done;
            for (size_t i = 0; i < n; ++i) mode[i] += e1[i];
        }
        const double inv = 1.0 / (double)nr;
        for (size_t i = 0; i < n; ++i) {
            mode[i] *= inv;
            residue[i] -= mode[i];
        }
        rc = list_push(&l, mode, 0);
        if (rc) goto done;
    }
    while (cfg->max_imfs == 0 || l.K < (size_t)cfg->max_imfs) { /* :310 */
        size_t nM, nm;
        so_find_extrema(residue, n, s.max_idx, s.max_val, &nM, s.min_idx, s.min_val, &nm);
        trace_push(tr, 3, -1, (int)l.K, 0, nM, nm, so_trace_hash(s.max_idx, nM, s.min_idx, nm));
        if (nM + nm < 3) break; /* :311 */
        const double beta_i = ens->nstd * so_signal_std(residue, n);
        memset(mode, 0, n * sizeof(double));
        for (size_t m = 0; m < nr; ++m) {
            memset(ei, 0, n * sizeof(double));
            double* nres = noise_res + m * n;
            if (alive[m]) { /* :317-325 */
                int32_t c;
                tctx tc = {tr, 1, (int)m, (int)l.K};
                rc = extract_imf_t(nres, n, cfg, ei, &c, &tc);
                if (rc == SO_OK) {
                    for (size_t i = 0; i < n; ++i) nres[i] -= ei[i];
                } else if (rc == SO_INSUFFICIENT) {
                    rc = SO_OK;
                    memset(ei, 0, n * sizeof(double));
                    alive[m] = 0;
                } else {
                    goto done;
                }
            }
            for (size_t i = 0; i < n; ++i) sm[i] = residue[i] + beta_i * ei[i]; /* :326-327 */
            tctx tc = {tr, 2, (int)m, (int)l.K};
            rc = first_mode(sm, n, cfg, e1, &tc);
            if (rc) goto done;
            for (size_t i = 0; i < n; ++i) mode[i] += e1[i];
        }
        const double inv = 1.0 / (double)nr; /* :331-337 */
        int all_zero = 1;
        for (size_t i = 0; i < n; ++i) {
            mode[i] *= inv;
            if (mode[i] != 0.0) all_zero = 0;
        }
        if (all_zero) break;
        for (size_t i = 0; i < n; ++i) residue[i] -= mode[i]; /* :338 */
        rc = list_push(&l, mode, 0);
        if (rc) goto done;
    }
done:
    free(noise_res); free(alive); free(mode); free(sm); free(ei); free(e1);
    scratch_free(&s);
    if (rc) { free(residue); free(l.data); free(l.counts); return rc; }
    to_decomp(&l, residue, out);
    memset(out->sift_counts, 0, (out->K ? out->K : 1) * sizeof(int32_t));
    return SO_OK;
}

int so_decompose(const double* x, size_t n, int algo, const so_sift_cfg* cfg, const so_ens_cfg* ens,
                 so_decomp* out, so_trace* tr) {
    switch (algo) { /* emd.cpp:365-373 */
        case 0: return so_emd(x, n, cfg, out, tr);
        case 1: return so_eemd(x, n, cfg, ens, out, tr);
        case 2: return so_ceemdan(x, n, cfg, ens, out, tr);
    }
    return fail(SO_INVALID, "unknown algorithm value");
}

/* ------------------------------------------------------------- serializer */

int so_transition_weights(size_t d, double* out) { /* serialize.cpp:7-13 */
    if (d < 1) return fail(SO_INVALID, "transition_weights: D must be at least 1");
    for (size_t i = 0; i < d; ++i) out[i] = (double)(i + 1) / (double)(d + 1);
    return SO_OK;
}

size_t so_default_transition_length(size_t rows) { /* serialize.cpp:15-18 */
    long long d = llround(0.2 * (double)rows);
    size_t v = d < 1 ? 1 : (size_t)d;
    return v < rows ? v : rows;
}

static int validate_ser(size_t M, size_t N, size_t D) { /* serialize.cpp:22-26 */
    if (M == 0 || N == 0) return fail(SO_INVALID, "concatenate: empty input");
    if (D < 1) return fail(SO_INVALID, "concatenate: D must be at least 1");
    if (D > M) return fail(SO_INVALID, "concatenate: transition longer than channel");
    return SO_OK;
}

/* serialize.cpp:30-50 */
int so_concatenate(const double* x, size_t M, size_t N, size_t D, double* out) {
    int rc = validate_ser(M, N, D);
    if (rc) return rc;
    double* a = malloc(D * sizeof(double));
    if (!a) return fail(SO_NOMEM, "out of memory");
    so_transition_weights(D, a);
    size_t o = 0;
    for (size_t j = 0; j < N; ++j) {
        const double* ch = x + j * M;
        memcpy(out + o, ch, M * sizeof(double));
        o += M;
        if (j + 1 == N) break;
        const double* next = x + (j + 1) * M;
        for (size_t t = 0; t < D; ++t) out[o++] = next[D - 1 - t] * a[t] + ch[M - 1 - t] * a[D - 1 - t];
    }
    free(a);
    return SO_OK;
}

/* serialize.cpp:52-71 */
int so_concatenate_naive(const double* x, size_t M, size_t N, size_t D, double* out) {
    int rc = validate_ser(M, N, D);
    if (rc) return rc;
    size_t o = 0;
    for (size_t j = 0; j < N; ++j) {
        for (size_t i = 0; i < M; ++i) out[o++] = x[j * M + i];
        if (j + 1 == N) break;
        for (size_t i = 1; i <= D; ++i) {
            const double wg = (double)i / (double)(D + 1);
            const double wf = (double)(D + 1 - i) / (double)(D + 1);
            out[o++] = wg * x[(j + 1) * M + (D - i)] + wf * x[j * M + (M - i)];
        }
    }
    return SO_OK;
}

/* serialize.cpp:73-95 */
int so_deconcatenate(const double* modes, size_t K, size_t L, size_t M, size_t N, size_t D, double* out) {
    if (K == 0) return fail(SO_INVALID, "deconcatenate: no modes given");
    if (M == 0 || N == 0) return fail(SO_INVALID, "deconcatenate: empty target shape");
    const size_t expect = M * N + D * (N - 1);
    if (L != expect)
        return fail(SO_INVALID, "deconcatenate: mode length %zu does not match M*N + D*(N-1) = %zu", L, expect);
    const size_t stride = M + D;
    for (size_t k = 0; k < K; ++k)
        for (size_t j = 0; j < N; ++j) {
            const double* src = modes + k * L + j * stride;
            double* dst = out + (k * N + j) * M;
            for (size_t i = 0; i < M; ++i) dst[i] = src[i];
        }
    return SO_OK;
}

/* serialize.cpp:97-105 */
int so_serial_decompose(const double* x, size_t M, size_t N, size_t D, int algo, const so_sift_cfg* cfg,
                        const so_ens_cfg* ens, double** tensor_out, size_t* modes_out, so_trace* tr) {
    int rc = validate_ser(M, N, D);
    if (rc) return rc;
    const size_t L = M * N + D * (N - 1);
    double* s = malloc(L * sizeof(double));
    if (!s) return fail(SO_NOMEM, "out of memory");
    so_concatenate(x, M, N, D, s);
    so_decomp d = {0};
    rc = so_decompose(s, L, algo, cfg, ens, &d, tr);
    free(s);
    if (rc) return rc;
    const size_t K1 = d.K + 1;
    double* modes = malloc(K1 * L * sizeof(double));
    double* t = malloc(K1 * M * N * sizeof(double));
    if (!modes || !t) { free(modes); free(t); so_decomp_free(&d); return fail(SO_NOMEM, "out of memory"); }
    memcpy(modes, d.imfs, d.K * L * sizeof(double));
    memcpy(modes + d.K * L, d.residue, L * sizeof(double));
    so_decomp_free(&d);
    rc = so_deconcatenate(modes, K1, L, M, N, D, t);
    free(modes);
    if (rc) { free(t); return rc; }
    *tensor_out = t;
    *modes_out = K1;
    return SO_OK;
}

/* synth.cpp:9-45 with the standard pick-up mask */
int so_multivariate_sinusoids(size_t n_samples, double fs, double* out) {
    static const int mask[4][6] = {{1, 1, 0, 1, 0, 0}, {1, 1, 1, 0, 1, 0}, {1, 1, 1, 1, 1, 1}, {1, 0, 1, 1, 0, 1}};
    static const double freqs[4] = {32.0, 16.0, 8.0, 2.0};
    if (fs <= 2.0 * 32.0)
        return fail(SO_INVALID, "multivariate_sinusoids: fs must exceed twice the highest tone (aliasing)");
    if (n_samples < 2) return fail(SO_INVALID, "multivariate_sinusoids: need at least 2 samples");
    const double two_pi = 6.283185307179586476925286766559;
    memset(out, 0, n_samples * 6 * sizeof(double));
    for (size_t j = 0; j < 6; ++j) {
        double* ch = out + j * n_samples;
        for (size_t i = 0; i < 4; ++i) {
            if (!mask[i][j]) continue;
            const double f = freqs[i];
            for (size_t k = 0; k < n_samples; ++k) ch[k] += sin(two_pi * f * (double)k / fs);
        }
    }
    return SO_OK;
}
