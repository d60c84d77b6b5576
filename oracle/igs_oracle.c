/*
 * igs_oracle.c -- plain-C restatement of the reference hot path.
 * TEST INFRASTRUCTURE ONLY (see igs_oracle.h).  Build: oracle/Makefile
 * (gcc -O2 -ffp-contract=off, x86-64 baseline: no FMA, like the reference).
 *
 * Citations are /root/reference/proj/<file>:<line>.
 */
#define _GNU_SOURCE
#include "igs_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define KPI 3.141592653589793 /* std::numbers::pi */
#define NORM_EPS 1e-8         /* renderer.hpp:14 kNormEps */
#define SCALE_MIN 1e-4        /* gaussian.hpp:12 */
#define SCALE_MAX 2.0         /* gaussian.hpp:13 */

/* ======================================================================= */
/* RNG: std::mt19937_64 (C++ [rand.eng.mers] parameters) + rng.hpp:15-24   */
/* ======================================================================= */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL

void orc_rng_seed(orc_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = MT_N;
}

static void mt_twist(orc_rng* r) {
    for (int i = 0; i < MT_N; ++i) {
        const uint64_t y = (r->mt[i] & MT_UPPER) | (r->mt[(i + 1) % MT_N] & MT_LOWER);
        uint64_t nv = r->mt[(i + MT_M) % MT_N] ^ (y >> 1);
        if (y & 1ULL) nv ^= 0xB5026F5AA96619E9ULL;
        r->mt[i] = nv;
    }
    r->idx = 0;
}

uint64_t orc_rng_u64(orc_rng* r) {
    if (r->idx >= MT_N) mt_twist(r);
    uint64_t x = r->mt[r->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

/* rng.hpp:18 next_double = (u64 >> 11) * 2^-53 */
double orc_rng_double(orc_rng* r) { return (double)(orc_rng_u64(r) >> 11) * 0x1.0p-53; }
/* rng.hpp:21 next_index = u64 % n */
uint64_t orc_rng_index(orc_rng* r, uint64_t n) { return orc_rng_u64(r) % n; }
/* rng.hpp:24 next_range = lo + (hi - lo) * next_double */
double orc_rng_range(orc_rng* r, double lo, double hi) { return lo + (hi - lo) * orc_rng_double(r); }

void orc_rng_stream(uint64_t seed, uint64_t skip, uint32_t count, uint64_t* out) {
    orc_rng r;
    orc_rng_seed(&r, seed);
    for (uint64_t i = 0; i < skip; ++i) (void)orc_rng_u64(&r);
    for (uint32_t i = 0; i < count; ++i) out[i] = orc_rng_u64(&r);
}

/* ======================================================================= */
/* Synthetic inputs: tests/test_support.hpp                                */
/* ======================================================================= */
static void set_px(float* img, int W, int h, int w, double r, double g, double b) {
    float* p = img + ((size_t)h * W + w) * 3;
    p[0] = (float)r;
    p[1] = (float)g;
    p[2] = (float)b;
}

/* test_support.hpp:15-30; draw order mu.x, mu.y, theta, s1, s2, r, g, b */
void orc_random_set(uint32_t n, uint64_t seed, double smin, double smax, double* out8) {
    orc_rng r;
    orc_rng_seed(&r, seed);
    for (uint32_t i = 0; i < n; ++i) {
        double* g = out8 + (size_t)i * 8;
        g[0] = orc_rng_double(&r);
        g[1] = orc_rng_double(&r);
        g[2] = orc_rng_range(&r, 0.0, 3.141592653589793);
        g[3] = orc_rng_range(&r, smin, smax);
        g[4] = orc_rng_range(&r, smin, smax);
        g[5] = orc_rng_double(&r);
        g[6] = orc_rng_double(&r);
        g[7] = orc_rng_double(&r);
    }
}

/* test_support.hpp:32-39 */
void orc_random_image(int W, int H, uint64_t seed, float* out) {
    orc_rng r;
    orc_rng_seed(&r, seed);
    for (int h = 0; h < H; ++h)
        for (int w = 0; w < W; ++w) {
            const double a = orc_rng_double(&r), b = orc_rng_double(&r), c = orc_rng_double(&r);
            set_px(out, W, h, w, a, b, c);
        }
}

/* test_support.hpp:42-65: 12 blobs over a ramp */
void orc_photo_like_image(int W, int H, uint64_t seed, float* out) {
    orc_rng r;
    orc_rng_seed(&r, seed);
    double bl[12][6];
    for (int i = 0; i < 12; ++i) {
        bl[i][0] = orc_rng_double(&r);
        bl[i][1] = orc_rng_double(&r);
        bl[i][2] = orc_rng_range(&r, 0.05, 0.3);
        bl[i][3] = orc_rng_double(&r);
        bl[i][4] = orc_rng_double(&r);
        bl[i][5] = orc_rng_double(&r);
    }
    for (int h = 0; h < H; ++h)
        for (int w = 0; w < W; ++w) {
            const double u = (w + 0.5) / W, v = (h + 0.5) / H;
            double cr = 0.2 + 0.6 * u, cg = 0.3 + 0.4 * v, cb = 0.5;
            for (int i = 0; i < 12; ++i) {
                const double d2 = (u - bl[i][0]) * (u - bl[i][0]) + (v - bl[i][1]) * (v - bl[i][1]);
                const double wgt = exp(-d2 / (2.0 * bl[i][2] * bl[i][2]));
                const double om = 1.0 - wgt;
                cr = cr * om + bl[i][3] * wgt;
                cg = cg * om + bl[i][4] * wgt;
                cb = cb * om + bl[i][5] * wgt;
            }
            set_px(out, W, h, w, cr, cg, cb);
        }
}

/* test_support.hpp:68-90: 10 hard discs */
void orc_vector_like_image(int W, int H, uint64_t seed, float* out) {
    orc_rng r;
    orc_rng_seed(&r, seed);
    double d[10][6];
    for (int i = 0; i < 10; ++i) {
        d[i][0] = orc_rng_double(&r);
        d[i][1] = orc_rng_double(&r);
        d[i][2] = orc_rng_range(&r, 0.05, 0.25);
        d[i][3] = orc_rng_double(&r);
        d[i][4] = orc_rng_double(&r);
        d[i][5] = orc_rng_double(&r);
    }
    for (int h = 0; h < H; ++h)
        for (int w = 0; w < W; ++w) {
            const double u = (w + 0.5) / W, v = (h + 0.5) / H;
            double c[3];
            if (u < 0.5) {
                c[0] = 0.95; c[1] = 0.95; c[2] = 0.9;
            } else {
                c[0] = 0.1; c[1] = 0.2; c[2] = 0.4;
            }
            for (int i = 0; i < 10; ++i) {
                const double d2 = (u - d[i][0]) * (u - d[i][0]) + (v - d[i][1]) * (v - d[i][1]);
                if (d2 < d[i][2] * d[i][2]) {
                    c[0] = d[i][3]; c[1] = d[i][4]; c[2] = d[i][5];
                }
            }
            set_px(out, W, h, w, c[0], c[1], c[2]);
        }
}

/* test_support.hpp:93-106: sinusoids */
void orc_texture_like_image(int W, int H, uint64_t seed, float* out) {
    orc_rng r;
    orc_rng_seed(&r, seed);
    const double p1 = orc_rng_range(&r, 15.0, 25.0);
    const double p2 = orc_rng_range(&r, 25.0, 40.0);
    const double ph1 = orc_rng_range(&r, 0.0, 6.28);
    const double ph2 = orc_rng_range(&r, 0.0, 6.28);
    for (int h = 0; h < H; ++h)
        for (int w = 0; w < W; ++w) {
            const double u = (w + 0.5) / W, v = (h + 0.5) / H;
            const double a = 0.5 + 0.5 * sin(p1 * u + ph1) * cos(p2 * v + ph2);
            const double b = 0.5 + 0.5 * sin(p2 * (u + v) + ph2);
            set_px(out, W, h, w, a, b, 0.5 + 0.25 * (a - b));
        }
}

/* ======================================================================= */
/* Gaussian math: gaussian.cpp                                              */
/* ======================================================================= */
static double clamp01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }
static double clamp_scale(double v) { return v < SCALE_MIN ? SCALE_MIN : (v > SCALE_MAX ? SCALE_MAX : v); }

/* gaussian.cpp:74-90 constrain */
static int constrain_one(double* g) {
    for (int p = 0; p < 8; ++p)
        if (!isfinite(g[p])) return ORC_E_INVALID_PARAMETER;
    g[0] = clamp01(g[0]);
    g[1] = clamp01(g[1]);
    double th = fmod(g[2], KPI);
    if (th < 0.0) th += KPI;
    if (th >= KPI) th = 0.0;
    g[2] = th;
    g[3] = clamp_scale(g[3]);
    g[4] = clamp_scale(g[4]);
    g[5] = clamp01(g[5]);
    g[6] = clamp01(g[6]);
    g[7] = clamp01(g[7]);
    return ORC_OK;
}

int orc_constrain(double* p8, uint32_t n) {
    for (uint32_t i = 0; i < n; ++i) {
        const int e = constrain_one(p8 + (size_t)i * 8);
        if (e) return e;
    }
    return ORC_OK;
}

/* gaussian.cpp:38-48 density */
double orc_density(const double* g, double u, double v) {
    const double c = cos(g[2]), s = sin(g[2]);
    const double dx = u - g[0], dy = v - g[1];
    const double e1 = c * dx + s * dy;
    const double e2 = -s * dx + c * dy;
    const double q = e1 * e1 / (g[3] * g[3]) + e2 * e2 / (g[4] * g[4]);
    return exp(-0.5 * q);
}

/* ======================================================================= */
/* Renderer: renderer.cpp                                                   */
/* ======================================================================= */

/* PreparedGaussian (renderer.hpp:20-27), built at renderer.cpp:32-51 */
typedef struct {
    double mu_x, mu_y, cos_t, sin_t, inv_a, inv_b, inv_s1, inv_s2, r, g, b;
} prep_t;

static prep_t* prepare(const double* p8, uint32_t n) {
    prep_t* ps = (prep_t*)malloc(sizeof(prep_t) * (n ? n : 1));
    for (uint32_t i = 0; i < n; ++i) {
        const double* g = p8 + (size_t)i * 8;
        prep_t* q = ps + i;
        q->mu_x = g[0];
        q->mu_y = g[1];
        q->cos_t = cos(g[2]);
        q->sin_t = sin(g[2]);
        q->inv_s1 = 1.0 / g[3];
        q->inv_s2 = 1.0 / g[4];
        q->inv_a = q->inv_s1 * q->inv_s1;
        q->inv_b = q->inv_s2 * q->inv_s2;
        q->r = g[5];
        q->g = g[6];
        q->b = g[7];
    }
    return ps;
}

void orc_prepare_scan(const double* p8, uint32_t n, double* scan6) {
    prep_t* ps = prepare(p8, n);
    for (uint32_t i = 0; i < n; ++i) {
        double* o = scan6 + (size_t)i * 6;
        o[0] = ps[i].mu_x; o[1] = ps[i].mu_y; o[2] = ps[i].cos_t; o[3] = ps[i].sin_t;
        o[4] = ps[i].inv_a; o[5] = ps[i].inv_b;
    }
    free(ps);
}

/* renderer.cpp:17-23 mahalanobis_sq: no FMA, left-to-right. */
static inline double maha(const prep_t* g, double x, double y) {
    const double dx = x - g->mu_x;
    const double dy = y - g->mu_y;
    const double e1 = g->cos_t * dx + g->sin_t * dy;
    const double e2 = -g->sin_t * dx + g->cos_t * dy;
    return e1 * e1 * g->inv_a + e2 * e2 * g->inv_b;
}

typedef struct {
    double q;
    uint32_t idx;
} entry_t;

/* renderer.cpp:53-74 select_top_k_entries: out sorted ascending by (q, idx). */
static int select_topk(const prep_t* ps, const uint32_t* cands, size_t ncand, double x, double y, int k,
                       entry_t* out) {
    int n = 0;
    for (size_t c = 0; c < ncand; ++c) {
        const uint32_t idx = cands ? cands[c] : (uint32_t)c;
        const double q = maha(ps + idx, x, y);
        if (n == k) {
            const entry_t* worst = &out[n - 1];
            if (q > worst->q || (q == worst->q && idx > worst->idx)) continue;
            --n;
        }
        int pos = n;
        while (pos > 0 && (q < out[pos - 1].q || (q == out[pos - 1].q && idx < out[pos - 1].idx))) {
            out[pos] = out[pos - 1];
            --pos;
        }
        out[pos].q = q;
        out[pos].idx = idx;
        ++n;
    }
    return n;
}

/* renderer.cpp:76-89 blend_entries; returns total, color in c[3]. */
static double blend(const prep_t* ps, const entry_t* e, int n, double* c) {
    double total = 0.0, ar = 0.0, ag = 0.0, ab = 0.0;
    for (int i = 0; i < n; ++i) {
        const double w = exp(-0.5 * e[i].q);
        const prep_t* g = ps + e[i].idx;
        total += w;
        ar += w * g->r;
        ag += w * g->g;
        ab += w * g->b;
    }
    const double inv = 1.0 / (NORM_EPS + total);
    c[0] = ar * inv;
    c[1] = ag * inv;
    c[2] = ab * inv;
    return total;
}

/* renderer.cpp:91-122 sample_gradients: d[8] per entry. */
static void sample_grads(const prep_t* ps, double x, double y, const entry_t* e, int n, const double* up,
                         const double* blended, double total, double* d /* n x 8 */) {
    const double inv_denom = 1.0 / (NORM_EPS + total);
    for (int i = 0; i < n; ++i) {
        const prep_t* g = ps + e[i].idx;
        const double w = exp(-0.5 * e[i].q);
        const double dL_dw =
            (up[0] * (g->r - blended[0]) + up[1] * (g->g - blended[1]) + up[2] * (g->b - blended[2])) * inv_denom;
        const double wc = w * inv_denom;
        const double dx = x - g->mu_x;
        const double dy = y - g->mu_y;
        const double e1 = g->cos_t * dx + g->sin_t * dy;
        const double e2 = -g->sin_t * dx + g->cos_t * dy;
        const double v1 = e1 * g->inv_a;
        const double v2 = e2 * g->inv_b;
        double* o = d + (size_t)i * 8;
        o[0] = dL_dw * w * (g->cos_t * v1 - g->sin_t * v2);
        o[1] = dL_dw * w * (g->sin_t * v1 + g->cos_t * v2);
        o[2] = dL_dw * -w * e1 * e2 * (g->inv_a - g->inv_b);
        o[3] = dL_dw * w * e1 * e1 * g->inv_a * g->inv_s1;
        o[4] = dL_dw * w * e2 * e2 * g->inv_b * g->inv_s2;
        o[5] = up[0] * wc;
        o[6] = up[1] * wc;
        o[7] = up[2] * wc;
    }
}

static float clampf_out(double v) { return (float)clamp01(v); }

/* renderer.cpp:161-191 render_image_impl (serial == parallel bit-for-bit). */
int orc_render_image(const double* p8, uint32_t n, int W, int H, int k, float* out, uint32_t* topk_idx) {
    if (n == 0) return ORC_E_EMPTY_SET;
    if (W < 1 || H < 1) return ORC_E_INVALID_PARAMETER;
    if (k < 1) return ORC_E_INVALID_PARAMETER;
    prep_t* ps = prepare(p8, n);
    const int kk = (int)((uint32_t)k < n ? (uint32_t)k : n);
    entry_t* e = (entry_t*)malloc(sizeof(entry_t) * kk);
    for (int h = 0; h < H; ++h)
        for (int w = 0; w < W; ++w) {
            const double u = (w + 0.5) / W, v = (h + 0.5) / H; /* image.hpp:18-20 */
            const int cnt = select_topk(ps, NULL, n, u, v, kk, e);
            double c[3];
            blend(ps, e, cnt, c);
            float* px = out + ((size_t)h * W + w) * 3;
            px[0] = clampf_out(c[0]);
            px[1] = clampf_out(c[1]);
            px[2] = clampf_out(c[2]);
            if (topk_idx) {
                uint32_t* t = topk_idx + ((size_t)h * W + w) * kk;
                for (int j = 0; j < kk; ++j) t[j] = j < cnt ? e[j].idx : 0xFFFFFFFFu;
            }
        }
    free(e);
    free(ps);
    return ORC_OK;
}

/* renderer.cpp:134-148 select_top_k */
int orc_select_top_k(const double* p8, uint32_t n, double u, double v, int k, uint32_t* idx, double* w,
                     int* count) {
    if (n == 0) return ORC_E_EMPTY_SET;
    if (k < 1) return ORC_E_INVALID_PARAMETER;
    prep_t* ps = prepare(p8, n);
    const int kk = (int)((uint32_t)k < n ? (uint32_t)k : n);
    entry_t* e = (entry_t*)malloc(sizeof(entry_t) * kk);
    const int cnt = select_topk(ps, NULL, n, u, v, kk, e);
    for (int i = 0; i < cnt; ++i) {
        idx[i] = e[i].idx;
        w[i] = exp(-0.5 * e[i].q);
    }
    *count = cnt;
    free(e);
    free(ps);
    return ORC_OK;
}

/* renderer.cpp:150-157 render_topk (one PreparedSet for all points; the
 * reference rebuilds it per call, which is value-identical). */
int orc_render_topk(const double* p8, uint32_t n, const double* uv, uint32_t npts, int k, double* rgb) {
    if (n == 0) return ORC_E_EMPTY_SET;
    if (k < 1) return ORC_E_INVALID_PARAMETER;
    prep_t* ps = prepare(p8, n);
    const int kk = (int)((uint32_t)k < n ? (uint32_t)k : n);
    entry_t* e = (entry_t*)malloc(sizeof(entry_t) * kk);
    for (uint32_t i = 0; i < npts; ++i) {
        const int cnt = select_topk(ps, NULL, n, uv[2 * i], uv[2 * i + 1], kk, e);
        blend(ps, e, cnt, rgb + 3 * (size_t)i);
    }
    free(e);
    free(ps);
    return ORC_OK;
}

/* renderer.cpp:124-132 render_naive (density() per Gaussian, in index order) */
int orc_render_naive(const double* p8, uint32_t n, const double* uv, uint32_t npts, double* rgb) {
    if (n == 0) return ORC_E_EMPTY_SET;
    for (uint32_t i = 0; i < npts; ++i) {
        double r = 0, g = 0, b = 0;
        for (uint32_t j = 0; j < n; ++j) {
            const double* G = p8 + (size_t)j * 8;
            const double w = orc_density(G, uv[2 * i], uv[2 * i + 1]);
            r = r + G[5] * w;
            g = g + G[6] * w;
            b = b + G[7] * w;
        }
        rgb[3 * i] = r;
        rgb[3 * i + 1] = g;
        rgb[3 * i + 2] = b;
    }
    return ORC_OK;
}

/* renderer.cpp:193-205 accumulate_contribs */
static void accumulate(const entry_t* e, const double* d, int cnt, double* grads8) {
    for (int j = 0; j < cnt; ++j) {
        double* gg = grads8 + (size_t)e[j].idx * 8;
        for (int p = 0; p < 8; ++p) gg[p] += d[(size_t)j * 8 + p];
    }
}

/* renderer.cpp:262-280 backward_serial (== backward bit-for-bit: the
 * parallel version reduces in the same sample order, :249-251). */
int orc_backward(const double* p8, uint32_t n, const double* s5, uint32_t ns, int k, double* grads8) {
    if (n == 0) return ORC_E_EMPTY_SET;
    if (k < 1) return ORC_E_INVALID_PARAMETER;
    for (uint32_t i = 0; i < ns; ++i) /* renderer.cpp:224-226 validate first */
        for (int c = 2; c < 5; ++c)
            if (!isfinite(s5[(size_t)i * 5 + c])) return ORC_E_INVALID_PARAMETER;
    prep_t* ps = prepare(p8, n);
    const int kk = (int)((uint32_t)k < n ? (uint32_t)k : n);
    entry_t* e = (entry_t*)malloc(sizeof(entry_t) * kk);
    double* d = (double*)malloc(sizeof(double) * 8 * kk);
    memset(grads8, 0, sizeof(double) * 8 * n);
    for (uint32_t i = 0; i < ns; ++i) {
        const double* s = s5 + (size_t)i * 5;
        const int cnt = select_topk(ps, NULL, n, s[0], s[1], kk, e);
        double c[3];
        const double total = blend(ps, e, cnt, c);
        sample_grads(ps, s[0], s[1], e, cnt, s + 2, c, total, d);
        accumulate(e, d, cnt, grads8);
    }
    free(d);
    free(e);
    free(ps);
    return ORC_OK;
}

static double sign_of(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); } /* fit.cpp:39 */

/* fit.cpp:51-106 train_step_gradients: loss = (1/ns) sum_i |c_r - c_t|_1 with
 * both reductions in sample order. */
int orc_train_step(const double* p8, uint32_t n, const float* target, int W, int H, const uint32_t* sidx,
                   uint32_t ns, int k, double* loss_out, double* grads8) {
    if (n == 0) return ORC_E_EMPTY_SET;
    if (k < 1) return ORC_E_INVALID_PARAMETER;
    prep_t* ps = prepare(p8, n);
    const int kk = (int)((uint32_t)k < n ? (uint32_t)k : n);
    const double inv_n = 1.0 / (double)ns;
    entry_t* e = (entry_t*)malloc(sizeof(entry_t) * kk);
    double* d = (double*)malloc(sizeof(double) * 8 * kk);
    memset(grads8, 0, sizeof(double) * 8 * n);
    double loss = 0.0;
    for (uint32_t i = 0; i < ns; ++i) {
        const int h = (int)sidx[i] / W;
        const int w = (int)sidx[i] % W;
        const double x = (w + 0.5) / W, y = (h + 0.5) / H;
        const float* t = target + ((size_t)h * W + w) * 3;
        const int cnt = select_topk(ps, NULL, n, x, y, kk, e);
        double c[3];
        const double total = blend(ps, e, cnt, c);
        const double dr = c[0] - (double)t[0], dg = c[1] - (double)t[1], db = c[2] - (double)t[2];
        loss += fabs(dr) + fabs(dg) + fabs(db);
        const double up[3] = {sign_of(dr) * inv_n, sign_of(dg) * inv_n, sign_of(db) * inv_n};
        sample_grads(ps, x, y, e, cnt, up, c, total, d);
        accumulate(e, d, cnt, grads8);
    }
    *loss_out = loss * inv_n;
    free(d);
    free(e);
    free(ps);
    return ORC_OK;
}

/* The map half of train_step_gradients (fit.cpp:65-84) for a block of
 * samples, with a caller-given 1/NS (the multi-rank decomposition: a rank
 * owns a contiguous block of the iteration's samples): per-sample loss,
 * and per slot (sample, entry) the Gaussian index (n for an empty slot) and
 * the 8 gradient partials.  The ordered reduction is the caller's. */
int orc_train_contribs(const double* p8, uint32_t n, const float* target, int W, int H, const uint32_t* sidx,
                       uint32_t ns, int k, double inv_n, double* losses, uint32_t* keys, double* contrib) {
    if (n == 0) return ORC_E_EMPTY_SET;
    if (k < 1) return ORC_E_INVALID_PARAMETER;
    prep_t* ps = prepare(p8, n);
    const int kk = (int)((uint32_t)k < n ? (uint32_t)k : n);
    entry_t* e = (entry_t*)malloc(sizeof(entry_t) * kk);
    for (uint32_t i = 0; i < ns; ++i) {
        const int h = (int)sidx[i] / W;
        const int w = (int)sidx[i] % W;
        const double x = (w + 0.5) / W, y = (h + 0.5) / H;
        const float* t = target + ((size_t)h * W + w) * 3;
        const int cnt = select_topk(ps, NULL, n, x, y, kk, e);
        double c[3];
        const double total = blend(ps, e, cnt, c);
        const double dr = c[0] - (double)t[0], dg = c[1] - (double)t[1], db = c[2] - (double)t[2];
        losses[i] = fabs(dr) + fabs(dg) + fabs(db);
        const double up[3] = {sign_of(dr) * inv_n, sign_of(dg) * inv_n, sign_of(db) * inv_n};
        double* d = contrib + (size_t)i * kk * 8;
        memset(d, 0, sizeof(double) * 8 * kk);
        sample_grads(ps, x, y, e, cnt, up, c, total, d);
        for (int j = 0; j < kk; ++j) keys[(size_t)i * kk + j] = j < cnt ? e[j].idx : n;
    }
    free(e);
    free(ps);
    return ORC_OK;
}

/* ======================================================================= */
/* Adam: adam.cpp:10-52                                                     */
/* ======================================================================= */
int orc_adam_step(double* p8, const double* g8, double* m, double* v, uint32_t n, const double* lr4, long long t,
                  int64_t* bad) {
    if (t < 1) return ORC_E_INVALID_PARAMETER;
    const double b1 = 0.9, b2 = 0.999, eps = 1e-8; /* adam.hpp:33-35 */
    const double bc1 = 1.0 - pow(b1, (double)t);
    const double bc2 = 1.0 - pow(b2, (double)t);
    /* (mu, mu, theta, scale, scale, color, color, color); lr4 = mu,color,scale,theta */
    const double lr8[8] = {lr4[0], lr4[0], lr4[3], lr4[2], lr4[2], lr4[1], lr4[1], lr4[1]};
    for (uint32_t i = 0; i < n; ++i) {
        double upd[8];
        for (int p = 0; p < 8; ++p) {
            const double g = g8[(size_t)i * 8 + p];
            if (!isfinite(g)) {
                if (bad) *bad = (int64_t)i * 8 + p;
                return ORC_E_INVALID_PARAMETER;
            }
            double* mm = m + (size_t)i * 8 + p;
            double* vv = v + (size_t)i * 8 + p;
            *mm = b1 * *mm + (1.0 - b1) * g;
            *vv = b2 * *vv + (1.0 - b2) * g * g;
            const double m_hat = *mm / bc1;
            const double v_hat = *vv / bc2;
            upd[p] = lr8[p] * m_hat / (sqrt(v_hat) + eps);
        }
        double* G = p8 + (size_t)i * 8;
        for (int p = 0; p < 8; ++p) G[p] -= upd[p];
        const int e = constrain_one(G);
        if (e) return e;
    }
    return ORC_OK;
}

/* ======================================================================= */
/* Sampling: sampling.cpp                                                   */
/* ======================================================================= */

/* sampling.cpp:14-23 */
double orc_kahan_sum(const double* v, size_t n) {
    double sum = 0.0, comp = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double y = v[i] - comp;
        const double t = sum + y;
        comp = (t - sum) - y;
        sum = t;
    }
    return sum;
}

static int clampi(int v, int hi) { return v < 0 ? 0 : (v > hi ? hi : v); }

/* sampling.cpp:44-67 Sobel L2 over six responses, replicate padding */
void orc_image_gradient_magnitude(const float* img, int W, int H, double* mag) {
#define AT(hh, ww, cc) ((double)img[((size_t)(hh) * W + (ww)) * 3 + (cc)])
    for (int h = 0; h < H; ++h)
        for (int w = 0; w < W; ++w) {
            const int hm = clampi(h - 1, H - 1), hp = clampi(h + 1, H - 1);
            const int wm = clampi(w - 1, W - 1), wp = clampi(w + 1, W - 1);
            double acc = 0.0;
            for (int c = 0; c < 3; ++c) {
                const double tl = AT(hm, wm, c), tc = AT(hm, w, c), tr = AT(hm, wp, c);
                const double ml = AT(h, wm, c), mr = AT(h, wp, c);
                const double bl = AT(hp, wm, c), bc = AT(hp, w, c), br = AT(hp, wp, c);
                const double gx = (tr + 2.0 * mr + br) - (tl + 2.0 * ml + bl);
                const double gy = (bl + 2.0 * bc + br) - (tl + 2.0 * tc + tr);
                acc += gx * gx + gy * gy;
            }
            mag[(size_t)h * W + w] = sqrt(acc);
        }
#undef AT
}

/* sampling.cpp:25-40 gradient_mixture (init_distribution / opt_distribution) */
int orc_gradient_mixture(const float* img, int W, int H, double lambda, double* p) {
    if (lambda < 0.0 || lambda > 1.0) return ORC_E_INVALID_PARAMETER;
    const size_t n = (size_t)W * H;
    orc_image_gradient_magnitude(img, W, H, p);
    const double total = orc_kahan_sum(p, n);
    const double uniform = 1.0 / (double)n;
    if (total > 0.0) {
        const double scale = (1.0 - lambda) / total;
        for (size_t i = 0; i < n; ++i) p[i] = p[i] * scale + lambda * uniform;
    } else {
        for (size_t i = 0; i < n; ++i) p[i] = uniform;
    }
    return ORC_OK;
}

/* sampling.cpp:77-94 add_distribution (Eq. 8 L1 error map) */
int orc_add_distribution(const float* rendered, const float* target, int W, int H, double* p) {
    const size_t n = (size_t)W * H;
    for (size_t i = 0; i < n; ++i) {
        const double dr = (double)rendered[3 * i] - (double)target[3 * i];
        const double dg = (double)rendered[3 * i + 1] - (double)target[3 * i + 1];
        const double db = (double)rendered[3 * i + 2] - (double)target[3 * i + 2];
        p[i] = fabs(dr) + fabs(dg) + fabs(db);
    }
    const double total = orc_kahan_sum(p, n);
    if (total > 0.0) {
        const double inv = 1.0 / total;
        for (size_t i = 0; i < n; ++i) p[i] *= inv;
    } else {
        for (size_t i = 0; i < n; ++i) p[i] = 1.0 / (double)n;
    }
    return ORC_OK;
}

/* sampling.cpp:96-128 Walker/Vose construction */
int orc_alias_build(const double* weights, size_t n, double* prob, uint32_t* alias) {
    if (n == 0) return ORC_E_INVALID_PARAMETER;
    const double total = orc_kahan_sum(weights, n);
    if (!(total > 0.0)) return ORC_E_INVALID_PARAMETER;
    double* scaled = (double*)malloc(sizeof(double) * n);
    uint32_t* small = (uint32_t*)malloc(sizeof(uint32_t) * n);
    uint32_t* large = (uint32_t*)malloc(sizeof(uint32_t) * n);
    size_t ns = 0, nl = 0;
    for (size_t i = 0; i < n; ++i) {
        if (weights[i] < 0.0) {
            free(scaled); free(small); free(large);
            return ORC_E_INVALID_PARAMETER;
        }
        scaled[i] = weights[i] * (double)n / total;
        prob[i] = 0.0;
        alias[i] = 0;
    }
    for (size_t i = 0; i < n; ++i) {
        if (scaled[i] < 1.0) small[ns++] = (uint32_t)i;
        else large[nl++] = (uint32_t)i;
    }
    while (ns > 0 && nl > 0) {
        const uint32_t s = small[--ns];
        const uint32_t l = large[--nl];
        prob[s] = scaled[s];
        alias[s] = l;
        scaled[l] = (scaled[l] + scaled[s]) - 1.0;
        if (scaled[l] < 1.0) small[ns++] = l;
        else large[nl++] = l;
    }
    for (size_t i = 0; i < nl; ++i) prob[large[i]] = 1.0;
    for (size_t i = 0; i < ns; ++i) prob[small[i]] = 1.0;
    free(scaled); free(small); free(large);
    return ORC_OK;
}

/* sampling.cpp:130-133: index draw first, then the coin */
uint32_t orc_alias_sample(const double* prob, const uint32_t* alias, size_t n, orc_rng* r) {
    const size_t i = (size_t)orc_rng_index(r, n);
    return orc_rng_double(r) < prob[i] ? (uint32_t)i : alias[i];
}

/* sampling.cpp:154-174 initialize_set */
int orc_initialize_set(const float* img, int W, int H, int count, double lambda, uint64_t seed, double* out8) {
    if (count < 1) return ORC_E_INVALID_PARAMETER;
    const size_t n = (size_t)W * H;
    double* p = (double*)malloc(sizeof(double) * n);
    int e = orc_gradient_mixture(img, W, H, lambda, p);
    if (e) { free(p); return e; }
    double* prob = (double*)malloc(sizeof(double) * n);
    uint32_t* alias = (uint32_t*)malloc(sizeof(uint32_t) * n);
    e = orc_alias_build(p, n, prob, alias);
    if (e) { free(p); free(prob); free(alias); return e; }
    orc_rng r;
    orc_rng_seed(&r, seed);
    const double s0 = 2.0 / (double)(W > H ? W : H);
    for (int i = 0; i < count; ++i) {
        const uint32_t flat = orc_alias_sample(prob, alias, n, &r);
        const int h = (int)flat / W, w = (int)flat % W;
        double* g = out8 + (size_t)i * 8;
        g[0] = (w + 0.5) / W;
        g[1] = (h + 0.5) / H;
        g[2] = 0.0;
        g[3] = s0;
        g[4] = s0;
        g[5] = (double)img[((size_t)h * W + w) * 3];
        g[6] = (double)img[((size_t)h * W + w) * 3 + 1];
        g[7] = (double)img[((size_t)h * W + w) * 3 + 2];
    }
    free(p); free(prob); free(alias);
    return ORC_OK;
}

/* ======================================================================= */
/* Metrics: metrics.cpp:12-27                                               */
/* ======================================================================= */
double orc_psnr(const float* a, const float* b, size_t count) {
    double se = 0.0, comp = 0.0;
    for (size_t i = 0; i < count; ++i) {
        const double d = (double)a[i] - (double)b[i];
        const double y = d * d - comp;
        const double t = se + y;
        comp = (t - se) - y;
        se = t;
    }
    if (se == 0.0) return INFINITY;
    const double mse = se / (double)count;
    return 10.0 * log10(1.0 / mse);
}

/* ======================================================================= */
/* BSP: bsp.cpp                                                             */
/* ======================================================================= */
typedef struct { double x1, y1, x2, y2; } rect_t;

typedef struct {
    int axis;
    double line;
    int32_t low, high, block;
    rect_t bbox;
} node_t;

typedef struct { uint32_t* v; size_t n, cap; } vec_u32;
static void vpush(vec_u32* a, uint32_t x) {
    if (a->n == a->cap) {
        a->cap = a->cap ? a->cap * 2 : 8;
        a->v = (uint32_t*)realloc(a->v, sizeof(uint32_t) * a->cap);
    }
    a->v[a->n++] = x;
}

struct orc_partition {
    uint32_t nb, source_size;
    int n_max;
    rect_t* blocks;
    rect_t* shells;
    vec_u32* block_members;
    vec_u32* shell_members;
    node_t* nodes;
    size_t n_nodes, cap_nodes;
    int32_t root;
    size_t cap_blocks;
    int grid_dim;
    vec_u32* grid_cells;
};

/* bsp.cpp:14-23 shell_of: 1/4 extent per side, clipped to [0,1]^2 */
static rect_t shell_of(rect_t b) {
    const double ex = (b.x2 - b.x1) * 0.25;
    const double ey = (b.y2 - b.y1) * 0.25;
    rect_t s = {b.x1 - ex, b.y1 - ey, b.x2 + ex, b.y2 + ey};
    s.x1 = s.x1 > 0.0 ? s.x1 : 0.0;
    s.y1 = s.y1 > 0.0 ? s.y1 : 0.0;
    s.x2 = s.x2 < 1.0 ? s.x2 : 1.0;
    s.y2 = s.y2 < 1.0 ? s.y2 : 1.0;
    return s;
}

static int contains_closed(rect_t r, double x, double y) { return x >= r.x1 && x <= r.x2 && y >= r.y1 && y <= r.y2; }
static int contains_half_open(rect_t r, double x, double y) {
    const int ix = x >= r.x1 && (x < r.x2 || (r.x2 >= 1.0 && x <= r.x2));
    const int iy = y >= r.y1 && (y < r.y2 || (r.y2 >= 1.0 && y <= r.y2));
    return ix && iy;
}
static int intersects_closed(rect_t a, rect_t o) { return a.x1 <= o.x2 && o.x1 <= a.x2 && a.y1 <= o.y2 && o.y1 <= a.y2; }

typedef struct {
    const double* p8;
    int axis;
} sort_ctx;

static double coord_of(const double* p8, uint32_t i, int axis) { return p8[(size_t)i * 8 + axis]; }

/* bsp.cpp:47-50: strict total order (coord, idx) */
static int cmp_coord(const void* a, const void* b, void* c) {
    const sort_ctx* s = (const sort_ctx*)c;
    const uint32_t ia = *(const uint32_t*)a, ib = *(const uint32_t*)b;
    const double ca = coord_of(s->p8, ia, s->axis), cb = coord_of(s->p8, ib, s->axis);
    if (ca < cb || (ca == cb && ia < ib)) return -1;
    if (cb < ca || (ca == cb && ib < ia)) return 1;
    return 0;
}
static int cmp_u32(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

static int32_t new_node(orc_partition* p) {
    if (p->n_nodes == p->cap_nodes) {
        p->cap_nodes = p->cap_nodes ? p->cap_nodes * 2 : 64;
        p->nodes = (node_t*)realloc(p->nodes, sizeof(node_t) * p->cap_nodes);
    }
    node_t* nd = &p->nodes[p->n_nodes];
    nd->axis = 0;
    nd->line = 0.0;
    nd->low = nd->high = nd->block = -1;
    return (int32_t)p->n_nodes++;
}

/* bsp.cpp:120-129 point_bbox */
static rect_t point_bbox(const double* p8, const uint32_t* m, size_t n) {
    rect_t b = {1.0, 1.0, 0.0, 0.0};
    for (size_t j = 0; j < n; ++j) {
        const double x = p8[(size_t)m[j] * 8], y = p8[(size_t)m[j] * 8 + 1];
        b.x1 = x < b.x1 ? x : b.x1;
        b.y1 = y < b.y1 ? y : b.y1;
        b.x2 = b.x2 < x ? x : b.x2;
        b.y2 = b.y2 < y ? y : b.y2;
    }
    return b;
}

/* bsp.cpp:32-118 Builder::build: alternating-axis median split with the
 * tie-aware split position; leaves numbered in DFS (low-first) order.
 * `m` is owned (freed) by this call. */
static int32_t bsp_build(orc_partition* p, const double* p8, rect_t rect, uint32_t* m, size_t n, int depth) {
    const int32_t id = new_node(p);
    p->nodes[id].bbox = point_bbox(p8, m, n);
    if ((long long)n <= (long long)p->n_max) {
        qsort(m, n, sizeof(uint32_t), cmp_u32);
        if (p->nb == p->cap_blocks) {
            p->cap_blocks = p->cap_blocks ? p->cap_blocks * 2 : 16;
            p->blocks = (rect_t*)realloc(p->blocks, sizeof(rect_t) * p->cap_blocks);
            p->block_members = (vec_u32*)realloc(p->block_members, sizeof(vec_u32) * p->cap_blocks);
        }
        p->nodes[id].block = (int32_t)p->nb;
        p->blocks[p->nb] = rect;
        p->block_members[p->nb].v = m;
        p->block_members[p->nb].n = n;
        p->block_members[p->nb].cap = n;
        p->nb++;
        return id;
    }
    const int axis = depth % 2;
    sort_ctx sc = {p8, axis};
    qsort_r(m, n, sizeof(uint32_t), cmp_coord, &sc);
#define C(j) coord_of(p8, m[j], axis)
    const size_t half = n / 2;
    size_t pos = 0;
    double line = 0.0;
    int forced = 0;
    if (C(half - 1) < C(half)) {
        pos = half;
    } else {
        size_t lo = 0, hi = 0;
        int has_lo = 0, has_hi = 0;
        for (size_t j = half; j-- > 1;)
            if (C(j - 1) < C(j)) { lo = j; has_lo = 1; break; }
        for (size_t j = half + 1; j < n; ++j)
            if (C(j - 1) < C(j)) { hi = j; has_hi = 1; break; }
        if (has_lo && (!has_hi || half - lo <= hi - half)) pos = lo;
        else if (has_hi) pos = hi;
        else forced = 1;
    }
    if (forced) {
        pos = half;
        line = C(0);
    } else {
        const double lo_c = C(pos - 1), hi_c = C(pos);
        line = 0.5 * (lo_c + hi_c);
        if (!(line > lo_c)) line = hi_c;
    }
#undef C
    uint32_t* lower = (uint32_t*)malloc(sizeof(uint32_t) * pos);
    uint32_t* upper = (uint32_t*)malloc(sizeof(uint32_t) * (n - pos));
    memcpy(lower, m, sizeof(uint32_t) * pos);
    memcpy(upper, m + pos, sizeof(uint32_t) * (n - pos));
    free(m);
    rect_t lr = rect, hr = rect;
    if (axis == 0) { lr.x2 = line; hr.x1 = line; }
    else { lr.y2 = line; hr.y1 = line; }
    p->nodes[id].axis = axis;
    p->nodes[id].line = line;
    const int32_t l = bsp_build(p, p8, lr, lower, pos, depth + 1);
    p->nodes[id].low = l;
    const int32_t h = bsp_build(p, p8, hr, upper, n - pos, depth + 1);
    p->nodes[id].high = h;
    return id;
}

/* bsp.cpp:132-143 collect_shell_members */
static void collect_shell(const orc_partition* p, const double* p8, int32_t nid, rect_t shell, vec_u32* out) {
    const node_t* nd = &p->nodes[nid];
    if (!intersects_closed(shell, nd->bbox)) return;
    if (nd->block >= 0) {
        const vec_u32* bm = &p->block_members[nd->block];
        for (size_t j = 0; j < bm->n; ++j) {
            const uint32_t i = bm->v[j];
            if (contains_closed(shell, p8[(size_t)i * 8], p8[(size_t)i * 8 + 1])) vpush(out, i);
        }
        return;
    }
    collect_shell(p, p8, nd->low, shell, out);
    collect_shell(p, p8, nd->high, shell, out);
}

/* bsp.cpp:153-176 build_partition */
orc_partition* orc_partition_build(const double* p8, uint32_t n, int n_max, int* err) {
    if (n == 0) { *err = ORC_E_EMPTY_SET; return NULL; }
    if (n_max < 1) { *err = ORC_E_INVALID_PARAMETER; return NULL; }
    orc_partition* p = (orc_partition*)calloc(1, sizeof(orc_partition));
    p->n_max = n_max;
    p->source_size = n;
    uint32_t* all = (uint32_t*)malloc(sizeof(uint32_t) * n);
    for (uint32_t i = 0; i < n; ++i) all[i] = i;
    rect_t unit = {0.0, 0.0, 1.0, 1.0};
    p->root = bsp_build(p, p8, unit, all, n, 0);
    p->shells = (rect_t*)malloc(sizeof(rect_t) * p->nb);
    p->shell_members = (vec_u32*)calloc(p->nb, sizeof(vec_u32));
    for (uint32_t b = 0; b < p->nb; ++b) p->shells[b] = shell_of(p->blocks[b]);
    for (uint32_t b = 0; b < p->nb; ++b) {
        collect_shell(p, p8, p->root, p->shells[b], &p->shell_members[b]);
        qsort(p->shell_members[b].v, p->shell_members[b].n, sizeof(uint32_t), cmp_u32);
    }
    *err = ORC_OK;
    return p;
}

/* bsp.cpp:178-195 build_grid_locator */
static void cell_range(int gd, double lo, double hi, int* c0, int* c1) {
    int a = (int)floor(lo * gd), b = (int)ceil(hi * gd) - 1;
    a = a < 0 ? 0 : (a > gd - 1 ? gd - 1 : a);
    b = b < 0 ? 0 : (b > gd - 1 ? gd - 1 : b);
    if (b < a) b = a;
    *c0 = a;
    *c1 = b;
}

static void build_grid(orc_partition* p) {
    const int nb = (int)p->nb;
    int gd = (int)ceil(sqrt((double)nb));
    if (gd < 1) gd = 1;
    p->grid_dim = gd;
    p->grid_cells = (vec_u32*)calloc((size_t)gd * gd, sizeof(vec_u32));
    for (int b = 0; b < nb; ++b) {
        int cx0, cx1, cy0, cy1;
        cell_range(gd, p->blocks[b].x1, p->blocks[b].x2, &cx0, &cx1);
        cell_range(gd, p->blocks[b].y1, p->blocks[b].y2, &cy0, &cy1);
        for (int cy = cy0; cy <= cy1; ++cy)
            for (int cx = cx0; cx <= cx1; ++cx) vpush(&p->grid_cells[(size_t)cy * gd + cx], (uint32_t)b);
    }
}

/* bsp.cpp:197-218 rebuild_partition */
orc_partition* orc_partition_rebuild(const double* rects4, uint32_t nb, const double* p8, uint32_t n, int* err) {
    if (nb == 0) { *err = ORC_E_INVALID_PARAMETER; return NULL; }
    orc_partition* p = (orc_partition*)calloc(1, sizeof(orc_partition));
    p->nb = nb;
    p->source_size = n;
    p->root = -1;
    p->blocks = (rect_t*)malloc(sizeof(rect_t) * nb);
    p->shells = (rect_t*)malloc(sizeof(rect_t) * nb);
    memcpy(p->blocks, rects4, sizeof(rect_t) * nb);
    for (uint32_t b = 0; b < nb; ++b) p->shells[b] = shell_of(p->blocks[b]);
    build_grid(p);
    p->block_members = (vec_u32*)calloc(nb, sizeof(vec_u32));
    p->shell_members = (vec_u32*)calloc(nb, sizeof(vec_u32));
    for (uint32_t i = 0; i < n; ++i) {
        const int b = orc_locate_block(p, p8[(size_t)i * 8], p8[(size_t)i * 8 + 1]);
        vpush(&p->block_members[b], i);
    }
    for (uint32_t b = 0; b < nb; ++b)
        for (uint32_t i = 0; i < n; ++i)
            if (contains_closed(p->shells[b], p8[(size_t)i * 8], p8[(size_t)i * 8 + 1])) vpush(&p->shell_members[b], i);
    *err = ORC_OK;
    return p;
}

void orc_partition_free(orc_partition* p) {
    if (!p) return;
    for (uint32_t b = 0; b < p->nb; ++b) {
        free(p->block_members[b].v);
        free(p->shell_members[b].v);
    }
    if (p->grid_cells)
        for (int c = 0; c < p->grid_dim * p->grid_dim; ++c) free(p->grid_cells[c].v);
    free(p->grid_cells);
    free(p->block_members);
    free(p->shell_members);
    free(p->blocks);
    free(p->shells);
    free(p->nodes);
    free(p);
}

uint32_t orc_partition_nblocks(const orc_partition* p) { return p->nb; }
uint64_t orc_partition_shell_total(const orc_partition* p) {
    uint64_t t = 0;
    for (uint32_t b = 0; b < p->nb; ++b) t += p->shell_members[b].n;
    return t;
}
void orc_partition_rects(const orc_partition* p, double* blocks4, double* shells4) {
    if (blocks4) memcpy(blocks4, p->blocks, sizeof(rect_t) * p->nb);
    if (shells4) memcpy(shells4, p->shells, sizeof(rect_t) * p->nb);
}
static void csr(const vec_u32* v, uint32_t nb, uint32_t* off, uint32_t* mem) {
    uint32_t o = 0;
    for (uint32_t b = 0; b < nb; ++b) {
        off[b] = o;
        memcpy(mem + o, v[b].v, sizeof(uint32_t) * v[b].n);
        o += (uint32_t)v[b].n;
    }
    off[nb] = o;
}
void orc_partition_shell_members(const orc_partition* p, uint32_t* off, uint32_t* mem) { csr(p->shell_members, p->nb, off, mem); }
void orc_partition_block_members(const orc_partition* p, uint32_t* off, uint32_t* mem) { csr(p->block_members, p->nb, off, mem); }

/* bsp.cpp:220-264 locate_block: tree descent, else grid + nearest fallback */
int orc_locate_block(const orc_partition* p, double u, double v) {
    if (p->n_nodes > 0) {
        int32_t id = p->root;
        while (p->nodes[id].block < 0) {
            const node_t* nd = &p->nodes[id];
            const double c = nd->axis == 0 ? u : v;
            id = c < nd->line ? nd->low : nd->high;
        }
        return p->nodes[id].block;
    }
    const int gd = p->grid_dim;
    int cx = (int)(u * gd), cy = (int)(v * gd);
    cx = cx < 0 ? 0 : (cx > gd - 1 ? gd - 1 : cx);
    cy = cy < 0 ? 0 : (cy > gd - 1 ? gd - 1 : cy);
    const vec_u32* cands = &p->grid_cells[(size_t)cy * gd + cx];
    int best = -1;
    double best_d = INFINITY;
    for (size_t j = 0; j < cands->n; ++j) {
        const rect_t r = p->blocks[cands->v[j]];
        if (contains_half_open(r, u, v)) return (int)cands->v[j];
        double dx = r.x1 - u;
        if (u - r.x2 > dx) dx = u - r.x2;
        if (0.0 > dx) dx = 0.0;
        double dy = r.y1 - v;
        if (v - r.y2 > dy) dy = v - r.y2;
        if (0.0 > dy) dy = 0.0;
        const double d = dx > dy ? dx : dy;
        if (d < best_d) { best_d = d; best = (int)cands->v[j]; }
    }
    if (best >= 0) return best;
    for (uint32_t b = 0; b < p->nb; ++b) {
        const rect_t r = p->blocks[b];
        if (contains_half_open(r, u, v)) return (int)b;
        double dx = r.x1 - u;
        if (u - r.x2 > dx) dx = u - r.x2;
        if (0.0 > dx) dx = 0.0;
        double dy = r.y1 - v;
        if (v - r.y2 > dy) dy = v - r.y2;
        if (0.0 > dy) dy = 0.0;
        const double d = dx > dy ? dx : dy;
        if (d < best_d) { best_d = d; best = (int)b; }
    }
    return best;
}

/* bsp.cpp:268-276 blocked_pixel */
static void blocked_pixel(const prep_t* ps, uint32_t n, const orc_partition* part, double x, double y, int k,
                          entry_t* e, double* c) {
    const int b = orc_locate_block(part, x, y);
    const vec_u32* mem = &part->shell_members[b];
    const int kk = (int)((uint32_t)k < n ? (uint32_t)k : n);
    const int cnt = select_topk(ps, mem->v, mem->n, x, y, kk, e);
    blend(ps, e, cnt, c);
}

/* bsp.cpp:278-282 check_partition */
static int check_part(const orc_partition* part, uint32_t n) {
    if (part->nb == 0) return ORC_E_INVALID_PARAMETER;
    if (part->source_size != n) return ORC_E_INVALID_PARAMETER;
    return ORC_OK;
}

/* bsp.cpp:289-317 render_image_blocked_impl */
int orc_render_image_blocked(const double* p8, uint32_t n, const orc_partition* part, int W, int H, int k,
                             float* out) {
    if (n == 0) return ORC_E_EMPTY_SET;
    if (W < 1 || H < 1 || k < 1) return ORC_E_INVALID_PARAMETER;
    const int e0 = check_part(part, n);
    if (e0) return e0;
    prep_t* ps = prepare(p8, n);
    const int kk = (int)((uint32_t)k < n ? (uint32_t)k : n);
    entry_t* e = (entry_t*)malloc(sizeof(entry_t) * kk);
    for (int h = 0; h < H; ++h)
        for (int w = 0; w < W; ++w) {
            const double u = (w + 0.5) / W, v = (h + 0.5) / H;
            double c[3];
            blocked_pixel(ps, n, part, u, v, k, e, c);
            float* px = out + ((size_t)h * W + w) * 3;
            px[0] = clampf_out(c[0]);
            px[1] = clampf_out(c[1]);
            px[2] = clampf_out(c[2]);
        }
    free(e);
    free(ps);
    return ORC_OK;
}

/* bsp.cpp:321-332 render_topk_blocked at many points (unclamped) */
int orc_render_points_blocked(const double* p8, uint32_t n, const orc_partition* part, const double* uv,
                              uint32_t npts, int k, double* rgb) {
    if (n == 0) return ORC_E_EMPTY_SET;
    if (k < 1) return ORC_E_INVALID_PARAMETER;
    const int e0 = check_part(part, n);
    if (e0) return e0;
    prep_t* ps = prepare(p8, n);
    const int kk = (int)((uint32_t)k < n ? (uint32_t)k : n);
    entry_t* e = (entry_t*)malloc(sizeof(entry_t) * kk);
    for (uint32_t i = 0; i < npts; ++i) blocked_pixel(ps, n, part, uv[2 * i], uv[2 * i + 1], k, e, rgb + 3 * (size_t)i);
    free(e);
    free(ps);
    return ORC_OK;
}

/* ======================================================================= */
/* Certified tile culling: restatement of the B200 build's predicate        */
/* (paper_2407_01866_b200/csrc/cull_math.cuh, cull.cu), op for op, so the    */
/* device's tile lists can be compared bit-exactly.  Not a reference         */
/* algorithm: the reference has no culling (renderer.cpp:168-176 ranks all   */
/* N); the predicate's soundness is what tests/test_cull.py checks against   */
/* the reference's own top-K.  Input: prepared records                       */
/* (mu_x, mu_y, cos, sin, inv_a, inv_b) as the device computed them.        */
/* ======================================================================= */
typedef struct { double mx, my, c, s, ia, ib, A, B, C; } cg_t;
#define CULL_ERRU (64.0 * 1.1102230246251565e-16)
#define CULL_UP (1.0 + 9.313225746154785e-10)
#define CULL_DN (1.0 - 9.313225746154785e-10)

static double cq_at(const cg_t* g, double x, double y) {
    const double dx = x - g->mx, dy = y - g->my;
    const double e1 = g->c * dx + g->s * dy;
    const double e2 = -g->s * dx + g->c * dy;
    return e1 * e1 * g->ia + e2 * e2 * g->ib;
}
static double c_err(const cg_t* g, double x0, double x1, double y0, double y1) {
    const double ax = fmax(fabs(x0 - g->mx), fabs(x1 - g->mx));
    const double ay = fmax(fabs(y0 - g->my), fabs(y1 - g->my));
    const double l = ax + ay;
    return CULL_ERRU * (g->ia + g->ib) * l * l;
}
static double c_qmax(const cg_t* g, double x0, double x1, double y0, double y1) {
    const double a = cq_at(g, x0, y0), b = cq_at(g, x1, y0), c = cq_at(g, x0, y1), d = cq_at(g, x1, y1);
    const double m = fmax(fmax(a, b), fmax(c, d));
    return m * CULL_UP + 2.0 * c_err(g, x0, x1, y0, y1);
}
static double c_qmin(const cg_t* g, double x0, double x1, double y0, double y1) {
    const int in_x = g->mx >= x0 && g->mx <= x1, in_y = g->my >= y0 && g->my <= y1;
    if (in_x && in_y) return 0.0;
    double best = INFINITY;
    const double det = g->ia * g->ib;
    if (!in_x) {
        const double xe = g->mx < x0 ? x0 : x1, dx = xe - g->mx;
        double v = (det * (dx * dx)) / g->C;
        const double ys = g->my - (g->B * dx) / g->C;
        if (ys < y0) v = fmax(v, cq_at(g, xe, y0) * CULL_DN);
        else if (ys > y1) v = fmax(v, cq_at(g, xe, y1) * CULL_DN);
        best = fmin(best, v);
    }
    if (!in_y) {
        const double ye = g->my < y0 ? y0 : y1, dy = ye - g->my;
        double v = (det * (dy * dy)) / g->A;
        const double xs = g->mx - (g->B * dy) / g->A;
        if (xs < x0) v = fmax(v, cq_at(g, x0, ye) * CULL_DN);
        else if (xs > x1) v = fmax(v, cq_at(g, x1, ye) * CULL_DN);
        best = fmin(best, v);
    }
    const double lb = best * CULL_DN - 2.0 * c_err(g, x0, x1, y0, y1);
    return lb > 0.0 ? lb : 0.0;
}
static double ccenter(int i, int n) { return ((double)i + 0.5) / (double)n; }
static int cmp_dbl(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* Returns the total list length; offsets[ntiles+1], tau[ntiles] and
 * members (ascending per tile; nullable on a sizing call). */
uint64_t orc_cull_lists(const double* scan6, uint32_t n, int W, int H, int k, int T, uint32_t* offsets,
                        uint32_t* members, double* tau) {
    const int TX = (W + T - 1) / T, TY = (H + T - 1) / T, nt = TX * TY;
    const int kk = (int)((uint32_t)k < n ? (uint32_t)k : n);
    cg_t* g = (cg_t*)malloc(sizeof(cg_t) * (n ? n : 1));
    int* bin = (int*)malloc(sizeof(int) * (n ? n : 1));
    uint32_t* bcnt = (uint32_t*)calloc(nt, sizeof(uint32_t));
    for (uint32_t i = 0; i < n; ++i) {
        const double* r = scan6 + (size_t)i * 6;
        g[i].mx = r[0]; g[i].my = r[1]; g[i].c = r[2]; g[i].s = r[3]; g[i].ia = r[4]; g[i].ib = r[5];
        const double c2 = g[i].c * g[i].c, s2 = g[i].s * g[i].s, cs = g[i].c * g[i].s;
        g[i].A = c2 * g[i].ia + s2 * g[i].ib;
        g[i].B = cs * (g[i].ia - g[i].ib);
        g[i].C = s2 * g[i].ia + c2 * g[i].ib;
        const double fx = floor(g[i].mx * (double)W), fy = floor(g[i].my * (double)H);
        const int cx = isfinite(fx) ? (int)fmin(fmax(fx, 0.0), (double)(W - 1)) : 0;
        const int cy = isfinite(fy) ? (int)fmin(fmax(fy, 0.0), (double)(H - 1)) : 0;
        bin[i] = (cy / T) * TX + cx / T;
        bcnt[bin[i]]++;
    }
    double* vals = (double*)malloc(sizeof(double) * (n ? n : 1));
    uint64_t total = 0;
    for (int t = 0; t < nt; ++t) {
        const int tx = t % TX, ty = t / TX;
        const double x0 = ccenter(tx * T, W), x1 = ccenter((W < (tx + 1) * T ? W : (tx + 1) * T) - 1, W);
        const double y0 = ccenter(ty * T, H), y1 = ccenter((H < (ty + 1) * T ? H : (ty + 1) * T) - 1, H);
        int r = 1, ax, bx, ay, by;
        for (;; ++r) {
            ax = tx - r > 0 ? tx - r : 0; bx = tx + r < TX - 1 ? tx + r : TX - 1;
            ay = ty - r > 0 ? ty - r : 0; by = ty + r < TY - 1 ? ty + r : TY - 1;
            uint64_t c = 0;
            for (int yy = ay; yy <= by; ++yy)
                for (int xx = ax; xx <= bx; ++xx) c += bcnt[yy * TX + xx];
            if (c >= (uint64_t)kk || (ax == 0 && ay == 0 && bx == TX - 1 && by == TY - 1)) break;
        }
        size_t nv = 0;
        for (uint32_t i = 0; i < n; ++i) {
            const int bt = bin[i], bxx = bt % TX, byy = bt / TX;
            if (bxx >= ax && bxx <= bx && byy >= ay && byy <= by) vals[nv++] = c_qmax(&g[i], x0, x1, y0, y1);
        }
        qsort(vals, nv, sizeof(double), cmp_dbl);
        const double tt = vals[kk - 1];
        if (tau) tau[t] = tt;
        if (offsets) offsets[t] = (uint32_t)total;
        for (uint32_t i = 0; i < n; ++i)
            if (c_qmin(&g[i], x0, x1, y0, y1) <= tt) {
                if (members) members[total] = i;
                ++total;
            }
    }
    if (offsets) offsets[nt] = (uint32_t)total;
    free(vals); free(bcnt); free(bin); free(g);
    return total;
}
