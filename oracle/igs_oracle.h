/*
 * igs_oracle.h -- CPU restatement of the Image-GS reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is part of the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it, and only as the checker or the CPU
 * baseline.  The product path (paper_2407_01866_b200/) never links it.
 *
 * Every function restates one reference function (file:line under
 * /root/reference/proj) in plain C99, compiled without FMA contraction so
 * each double operation rounds exactly like the reference's SSE2 build.
 * The restatement is pinned against the reference itself compiled from its
 * own sources (oracle/_ref, see oracle/Makefile): tests/test_oracle_pin.py
 * requires bit-identical results on every shared entry point.
 *
 * Layouts (zero-copy with the reference's structs):
 *   Gaussian record  : double[8] = mu_u, mu_v, theta, s1, s2, r, g, b
 *                      (gaussian.hpp:19-24, same order as GaussianGrad and
 *                      the Adam slots, adam.hpp:20-31)
 *   PixelSample      : double[5] = u, v, up_r, up_g, up_b (renderer.hpp:102-105)
 *   Image            : float[H][W][3] row-major (image.hpp:24-59)
 *   Rect             : double[4] = x1, y1, x2, y2 (bsp.hpp:14)
 *   Learning rates   : double[4] = mu, color, scale, theta (adam.hpp:11-16)
 *
 * Return codes: 0 = ok, otherwise 1 + igs::ErrorKind (error.hpp:8-17).
 */
#ifndef IGS_ORACLE_H
#define IGS_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_OK 0
#define ORC_E_INVALID_PARAMETER 1
#define ORC_E_DIMENSION_MISMATCH 2
#define ORC_E_EMPTY_SET 6

/* ---- RNG: std::mt19937_64 + the draw helpers of rng.hpp:11-28 ---------- */
typedef struct {
    uint64_t mt[312];
    int idx;
} orc_rng;

void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_u64(orc_rng* r);
double orc_rng_double(orc_rng* r);
uint64_t orc_rng_index(orc_rng* r, uint64_t n);
double orc_rng_range(orc_rng* r, double lo, double hi);
/* Convenience: first `count` raw outputs of mt19937_64(seed). */
void orc_rng_stream(uint64_t seed, uint64_t skip, uint32_t count, uint64_t* out);

/* ---- synthetic inputs (tests/test_support.hpp:15-106) ------------------- */
void orc_random_set(uint32_t n, uint64_t seed, double smin, double smax, double* out8);
void orc_random_image(int W, int H, uint64_t seed, float* out);
void orc_photo_like_image(int W, int H, uint64_t seed, float* out);
void orc_vector_like_image(int W, int H, uint64_t seed, float* out);
void orc_texture_like_image(int W, int H, uint64_t seed, float* out);

/* ---- Gaussian math (gaussian.cpp) --------------------------------------- */
int orc_constrain(double* p8, uint32_t n);
double orc_density(const double* g8, double u, double v);

/* ---- renderer (renderer.cpp) --------------------------------------------- */
/* Global top-K raster; topk_idx (nullable) receives H*W*kk indices, kk =
 * min(k, n), unused slots 0xFFFFFFFF. */
int orc_render_image(const double* p8, uint32_t n, int W, int H, int k, float* out, uint32_t* topk_idx);
/* select_top_k at one point: idx/w sized min(k,n); returns the count in *count. */
int orc_select_top_k(const double* p8, uint32_t n, double u, double v, int k, uint32_t* idx, double* w,
                     int* count);
/* render_topk (unclamped) at npts points uv[2*i]. */
int orc_render_topk(const double* p8, uint32_t n, const double* uv, uint32_t npts, int k, double* rgb);
int orc_render_naive(const double* p8, uint32_t n, const double* uv, uint32_t npts, double* rgb);
int orc_backward(const double* p8, uint32_t n, const double* samples5, uint32_t ns, int k, double* grads8);
/* fit.cpp:51-106 train_step_gradients (+ the sign/loss logic). */
/* fit.cpp:65-84 map half for a sample block with a given 1/NS (multi-rank) */
int orc_train_contribs(const double* p8, uint32_t n, const float* target, int W, int H, const uint32_t* sidx,
                       uint32_t ns, int k, double inv_n, double* losses, uint32_t* keys, double* contrib);
int orc_train_step(const double* p8, uint32_t n, const float* target, int W, int H, const uint32_t* sample_idx,
                   uint32_t ns, int k, double* loss, double* grads8);

/* ---- Adam (adam.cpp:10-52) ------------------------------------------------ */
/* On a non-finite gradient returns ORC_E_INVALID_PARAMETER with *bad =
 * i*8+p (first offending slot in record order). */
int orc_adam_step(double* p8, const double* g8, double* m, double* v, uint32_t n, const double* lr4, long long t,
                  int64_t* bad);

/* ---- sampling (sampling.cpp) ---------------------------------------------- */
double orc_kahan_sum(const double* v, size_t n);
void orc_image_gradient_magnitude(const float* img, int W, int H, double* mag);
int orc_gradient_mixture(const float* img, int W, int H, double lambda, double* p);
int orc_add_distribution(const float* rendered, const float* target, int W, int H, double* p);
/* Walker/Vose table; prob/alias sized n. */
int orc_alias_build(const double* weights, size_t n, double* prob, uint32_t* alias);
uint32_t orc_alias_sample(const double* prob, const uint32_t* alias, size_t n, orc_rng* r);
/* initialize_set (sampling.cpp:154-174) with a fresh Rng(seed). */
int orc_initialize_set(const float* img, int W, int H, int count, double lambda, uint64_t seed, double* out8);

/* ---- metrics (metrics.cpp:12-27) ----------------------------------------- */
double orc_psnr(const float* a, const float* b, size_t count);

/* ---- BSP (bsp.cpp) -------------------------------------------------------- */
typedef struct orc_partition orc_partition;
orc_partition* orc_partition_build(const double* p8, uint32_t n, int n_max, int* err);
orc_partition* orc_partition_rebuild(const double* rects4, uint32_t nb, const double* p8, uint32_t n, int* err);
void orc_partition_free(orc_partition* p);
uint32_t orc_partition_nblocks(const orc_partition* p);
uint64_t orc_partition_shell_total(const orc_partition* p);
void orc_partition_rects(const orc_partition* p, double* blocks4, double* shells4);
/* CSR: offsets[nb+1], members[shell_total]. */
void orc_partition_shell_members(const orc_partition* p, uint32_t* offsets, uint32_t* members);
void orc_partition_block_members(const orc_partition* p, uint32_t* offsets, uint32_t* members);
int orc_locate_block(const orc_partition* p, double u, double v);
int orc_render_image_blocked(const double* p8, uint32_t n, const orc_partition* part, int W, int H, int k,
                             float* out);
int orc_render_points_blocked(const double* p8, uint32_t n, const orc_partition* part, const double* uv,
                              uint32_t npts, int k, double* rgb);

/* ---- certified tile culling (restates the B200 build's predicate) ------- */
/* scan6: prepared records (mu_x, mu_y, cos, sin, inv_a, inv_b).  Returns the
 * total list length; offsets[ntiles+1], tau[ntiles], members nullable. */
uint64_t orc_cull_lists(const double* scan6, uint32_t n, int W, int H, int k, int T, uint32_t* offsets,
                        uint32_t* members, double* tau);
/* PreparedSet scan records (renderer.cpp:32-51) with glibc sin/cos. */
void orc_prepare_scan(const double* p8, uint32_t n, double* scan6);

#ifdef __cplusplus
}
#endif
#endif
