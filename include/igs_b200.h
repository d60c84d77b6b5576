/*
 * igs_b200.h -- C-ABI of the B200-native Image-GS hot path.
 *
 * The reference (/root/reference/proj) exposes its hot path as a C++ header
 * API in namespace igs (the headers proj/include/igs/NAME.hpp); it has no FFI of its own.
 * This header is the thin C boundary a maintainer binds to replace that
 * path: plain pointers and sizes, no C++ or torch types.
 * shows the C++ shim (same igs:: signatures) and the Python ctypes binding.
 *
 * Layouts are zero-copy with the reference's structs:
 *   Gaussian record  double[8] = mu_u, mu_v, theta, s1, s2, r, g, b
 *                    (gaussian.hpp:19-24 Gaussian2D; GaussianGrad
 *                    renderer.hpp:95-100 and the Adam slots adam.hpp:20-31
 *                    use the same order)
 *   PixelSample      double[5] = u, v, up_r, up_g, up_b (renderer.hpp:102-105)
 *   Image            float32[H][W][3] row-major (image.hpp:24-59)
 *   Rect             double[4] = x1, y1, x2, y2 (bsp.hpp:14-16)
 *   LearningRates    double[4] = mu, color, scale, theta (adam.hpp:11-16)
 *
 * Every host pointer argument may be NULL where marked "nullable"; a NULL
 * output keeps the result device-resident in the context (used by the
 * device-resident benchmark and by fused multi-step calls).
 *
 * Errors: every call returns 0 or 1 + igs::ErrorKind (error.hpp:8-17);
 * IGS_E_CUDA for device failures.  igs_last_error() returns the message of
 * the last failing call on that context (text matches the reference where
 * its tests inspect it, e.g. "non-finite gradient for Gaussian 1
 * parameter s2", adam.cpp:29-31).  Validation happens before any launch, as
 * in the reference (renderer.cpp:224-226).
 *
 * Threading: a context is externally synchronized (one host thread at a
 * time), like the reference's fit().  One context per GPU.
 */
#ifndef IGS_B200_H
#define IGS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IGS_OK 0
#define IGS_E_INVALID_PARAMETER 1 /* ErrorKind::invalid_parameter  */
#define IGS_E_DIMENSION_MISMATCH 2 /* ErrorKind::dimension_mismatch */
#define IGS_E_BAD_MAGIC 3
#define IGS_E_BAD_VERSION 4
#define IGS_E_TRUNCATED 5
#define IGS_E_EMPTY_SET 6 /* ErrorKind::empty_set */
#define IGS_E_IO 7
#define IGS_E_UNSUPPORTED_FORMAT 8
#define IGS_E_CUDA 100 /* device / driver failure (no reference analogue) */

typedef struct igs_ctx igs_ctx;

/* ---- context ------------------------------------------------------------ */
int igs_ctx_create(int device, igs_ctx** out);
void igs_ctx_destroy(igs_ctx* ctx);
const char* igs_last_error(const igs_ctx* ctx);
/* Waits for all work queued on the context's stream. */
int igs_sync(igs_ctx* ctx);
/* Number of kernels this context launched since creation (diagnostics). */
uint64_t igs_kernel_launches(const igs_ctx* ctx);

/* Options (igs_set_option):                                                  */
#define IGS_OPT_CULL 1          /* 1 = certified tile culling for global top-K (default), 0 = brute force */
#define IGS_OPT_DETERMINISTIC 2 /* 1 = sample-ordered gradient reduction, bit-exact (default); 0 = fp64 atomics */
#define IGS_OPT_TILE 3          /* tile edge in pixels for culling (default 16) */
#define IGS_OPT_RASTER 4        /* culled global render: 0 = loose-quadtree patch search (default, k <= 32),
                                   1 = certified per-tile candidate lists */
#define IGS_OPT_SHARD_ADAM 5    /* multi-rank fused iterations: 1 = each rank reduces + updates its 1/R slice of
                                   the set and the parameters are all-gathered (default); 0 = every rank
                                   updates the whole set (replicated).  Bit-identical either way. */
int igs_set_option(igs_ctx* ctx, int option, int64_t value);
int64_t igs_get_option(const igs_ctx* ctx, int option);

/* ---- Gaussian set (GaussianSet, gaussian.hpp:27-33) ------------------------ */
/* Uploads n records and re-derives the per-Gaussian cache (PreparedSet,
 * renderer.cpp:32-51).  Resets Adam moments.  A resident partition is kept
 * (like a caller-held BspPartition); blocked renders reject it once the
 * Gaussian count differs from the one it was built for. */
int igs_set_params(igs_ctx* ctx, const double* params8, uint32_t n);
/* Appends n records (densification, fit.cpp:185-199): indices stay stable,
 * new Adam moments are zero (AdamState::resize, adam.hpp:26-29). */
int igs_append_params(igs_ctx* ctx, const double* params8, uint32_t n);
int igs_get_params(igs_ctx* ctx, double* params8 /* n*8 */, uint32_t n);
uint32_t igs_num_gaussians(const igs_ctx* ctx);
/* Device pointer of the resident params (double[n][8]) for zero-copy use. */
const double* igs_device_params(const igs_ctx* ctx);

/* ---- renderer (renderer.hpp:107-138) --------------------------------------- */
/* render_image (renderer.cpp:209): global normalized top-K blend at every
 * pixel center, clamped to [0,1], float32.  out_rgb nullable (keeps the
 * image on device); topk_idx nullable: H*W*min(k,n) indices, sorted
 * best-first, unused slots 0xFFFFFFFF (debug / parity). */
int igs_render_image(igs_ctx* ctx, int width, int height, int k, float* out_rgb, uint32_t* topk_idx);
/* Rows [row0, row1) of the same raster (tile-row sharding across GPUs);
 * out_rgb receives (row1-row0)*W*3 floats. */
int igs_render_image_rows(igs_ctx* ctx, int width, int height, int k, int row0, int row1, float* out_rgb);
/* Device pointer of the last rendered image (float32 H*W*3). */
const float* igs_device_image(const igs_ctx* ctx);

/* select_top_k at npts points (renderer.cpp:134-148): idx/weights are
 * npts*min(k,n), best-first; counts (nullable) per point. */
int igs_select_top_k(igs_ctx* ctx, const double* uv, uint32_t npts, int k, uint32_t* idx, double* weights,
                     int32_t* counts);
/* render_topk at npts points (renderer.cpp:150-157): unclamped double RGB. */
int igs_render_points(igs_ctx* ctx, const double* uv, uint32_t npts, int k, double* rgb);

/* backward (renderer.cpp:254-260): loss gradients for arbitrary samples,
 * reduced per Gaussian in sample order.  grads8 nullable (device-resident). */
int igs_backward(igs_ctx* ctx, const double* samples5, uint32_t ns, int k, double* grads8);

/* ---- training (fit.cpp:51-106, 149-157) --------------------------------- */
/* Uploads the target image once (float32 H*W*3). */
int igs_set_target(igs_ctx* ctx, const float* rgb, int width, int height);
/* train_step_gradients: forward + L1 loss + backward at the sampled pixel
 * centers (flat indices h*W+w into the target).  loss/grads8 nullable. */
int igs_train_step(igs_ctx* ctx, const uint32_t* sample_idx, uint32_t ns, int k, double* loss, double* grads8);
/* adam_step (adam.cpp:10-52) on the resident gradients; lr4 = mu, color,
 * scale, theta; t = 1-based step (bias correction 1 - beta^t uses the
 * host's libm pow exactly like the reference). */
int igs_adam_step(igs_ctx* ctx, const double* lr4, long long t);
/* Fused iteration: train_step + adam_step.  With a communicator attached
 * the contributions of every rank's sample block are all-gathered between
 * them (and, with IGS_OPT_SHARD_ADAM, each rank updates its slice of the set
 * and the parameters are all-gathered); bit-identical to one GPU. */
int igs_train_iteration(igs_ctx* ctx, const uint32_t* sample_idx, uint32_t ns, int k, const double* lr4,
                        long long t, double* loss);
/* Asynchronous form for pipelined drivers: enqueues the iteration (the
 * sample indices are staged through pinned memory; returns immediately) --
 * igs_train_wait() then waits for the oldest outstanding iteration, checks
 * its status and reports its loss.  At most two iterations may be
 * outstanding: enqueueing t+1 before waiting on t overlaps the host's
 * enqueue with the device's work (the iterations still run in order). */
int igs_train_iteration_async(igs_ctx* ctx, const uint32_t* sample_idx, uint32_t ns, int k, const double* lr4,
                              long long t);
int igs_train_wait(igs_ctx* ctx, double* loss);
/* Uploads per-step sample indices to a device buffer of `steps` x ns
 * entries so igs_train_iterations can run fully device-resident. */
int igs_upload_samples(igs_ctx* ctx, const uint32_t* sample_idx, uint32_t ns, uint32_t steps);
/* Runs `steps` fused iterations t = t0..t0+steps-1; step t uses uploaded
 * sample slot (t-1) mod steps_uploaded.  losses (nullable): one per step. */
int igs_train_iterations(igs_ctx* ctx, uint32_t steps, int k, const double* lr4, long long t0, double* losses);
/* Resident gradient buffer (double[n][8]). */
const double* igs_device_grads(const igs_ctx* ctx);
int igs_get_grads(igs_ctx* ctx, double* grads8, uint32_t n);
/* Sets the resident gradients (adam_step's `grads` argument, adam.hpp:40). */
int igs_set_grads(igs_ctx* ctx, const double* grads8, uint32_t n);
/* Adam moments in record order (AdamState m/v). */
int igs_get_adam_state(igs_ctx* ctx, double* m, double* v, uint32_t n);
int igs_set_adam_state(igs_ctx* ctx, const double* m, const double* v, uint32_t n);

/* ---- error map & metrics (sampling.cpp:77-94, metrics.cpp:12-27) -------- */
/* add_distribution(rendered, target): per-pixel L1 error normalized to a
 * distribution (uniform when zero).  rendered nullable = last device image. */
int igs_add_distribution(igs_ctx* ctx, const float* rendered, int width, int height, double* p);
/* psnr(rendered, target); rendered nullable = last device image. */
int igs_psnr(igs_ctx* ctx, const float* rendered, int width, int height, double* out);

/* image_gradient_magnitude(img) (sampling.cpp:44-67) on the device: per-pixel
 * L2 norm of the six Sobel responses, replicate padding; img nullable = the
 * resident target; mag = H*W doubles (nullable: stays on the device). */
int igs_image_gradient_magnitude(igs_ctx* ctx, const float* img, int width, int height, double* mag);
/* init_distribution / opt_distribution (sampling.cpp:25-40): (1-lambda) *
 * |grad| / Kahan-sum|grad| + lambda / (H*W), uniform when the gradient field
 * is zero.  img nullable = the target; p = H*W doubles. */
int igs_gradient_mixture(igs_ctx* ctx, const float* img, int width, int height, double lambda, double* p);

/* initialize_set(img, count, lambda, rng) (sampling.cpp:154-174): count
 * Gaussians at init_distribution draws (pixel centres, the pixel's colour,
 * s = 2/max(W,H), theta = 0).  raw2: the 2*count raw mt19937_64 outputs the
 * reference's draws consume (next_index, then next_double, per Gaussian),
 * taken from the caller's Rng (Rng::next_u64) -- so the caller's engine
 * advances exactly as the reference's would.  out8: count records. */
int igs_initialize_set(igs_ctx* ctx, const float* img, int width, int height, int count, double lambda,
                       const uint64_t* raw2, double* out8);

/* ssim(rendered, target) (metrics.cpp:33-112); rendered nullable = last image. */
int igs_ssim(igs_ctx* ctx, const float* rendered, int width, int height, double* out);

/* ---- encoder (fit.hpp:19-64) -------------------------------------------------- */
typedef struct {
    int budget;          /* target Gaussian count (final = budget/2 + 4*(budget/8)) */
    int k;               /* top-K */
    double lambda_init, lambda_opt;
    int iterations, samples_per_iter;
    double lr[4];        /* mu, color, scale, theta */
    int eval_interval, plateau_patience;
    double lr_decay;     /* multiplier, applied at most once */
    int warmup_iters, densify_interval;
    uint64_t seed;
    int compute_ssim;    /* 1 = evaluate SSIM like the reference, 0 = skip (logged as 0) */
} igs_fit_config;
typedef struct {
    int iteration, count;
    double loss, psnr, ssim, best_psnr;
} igs_eval_record;
/* LoD checkpoint (fit.hpp:56-58): stage, iteration, id "lod<s>_iter<i>_n<c>", the set. */
typedef void (*igs_checkpoint_fn)(void* user, int stage, int iteration, const char* id, const double* params8,
                                  uint32_t n);
/* FitConfig defaults (fit.hpp:19-33). */
void igs_fit_config_default(igs_fit_config* cfg);
/* fit() (fit.cpp:116-207): content-adaptive init, importance-sampled L1
 * optimisation with Adam, periodic BSP-render evaluation with one-shot LR
 * decay, error-guided densification, LoD checkpoints.  RNG draws (mt19937_64,
 * Walker alias tables) run on the host in the reference's order; every
 * render, train step, Adam step and metric runs on the device.  The final
 * set stays resident (igs_get_params).  evals (nullable) receives up to
 * max_evals records; log (nullable) receives FitReport::write's text
 * (fit.cpp:209-231), NUL-terminated, truncated to log_cap. */
int igs_fit(igs_ctx* ctx, const float* target, int width, int height, const igs_fit_config* cfg,
            igs_checkpoint_fn cb, void* user, igs_eval_record* evals, int max_evals, int* n_evals,
            int* lr_decay_iteration, int* final_count, char* log, size_t log_cap);

/* ---- BSP acceleration (bsp.hpp:70-106) ------------------------------------ */
/* build_partition(set, n_max) over the resident set. */
int igs_partition_build(igs_ctx* ctx, int n_max);
/* rebuild_partition(blocks, set): shells and memberships re-derived from
 * bare block corners (decode path, bsp.cpp:197-218). */
int igs_partition_rebuild(igs_ctx* ctx, const double* rects4, uint32_t n_blocks);
int igs_partition_info(igs_ctx* ctx, uint32_t* n_blocks, uint64_t* shell_total);
int igs_partition_get(igs_ctx* ctx, double* blocks4, double* shells4, uint32_t* shell_offsets /* nb+1 */,
                      uint32_t* shell_members);
/* The rest of a BspPartition (bsp.hpp:44-66), for handing the resident
 * partition to the reference's own struct: n_max, source_size, and either
 * the split tree (root, n_nodes; nodes as axis, low, high, block + lines) or
 * the grid locator (grid_dim, cell CSR).  Block members: the builder's leaf
 * lists (built) or locate_block of each centre (rebuilt), ascending. */
int igs_partition_export(igs_ctx* ctx, int* n_max, uint32_t* source_size, int32_t* root, uint32_t* n_nodes,
                         int* grid_dim, uint32_t* grid_total);
int igs_partition_get_tree(igs_ctx* ctx, int32_t* nodes4, double* lines);
int igs_partition_get_grid(igs_ctx* ctx, uint32_t* cell_offsets /* grid_dim^2 + 1 */, uint32_t* cell_blocks);
int igs_partition_block_members(igs_ctx* ctx, uint32_t* offsets /* nb + 1 */, uint32_t* members);
/* Installs a caller-held partition (e.g. an igs::BspPartition): blocks, and
 * the split tree when n_nodes > 0 (else the grid locator is derived); shells
 * and shell members are re-derived from the resident set; source_size is
 * kept for the stale-partition check (bsp.cpp:278-282). */
int igs_partition_set(igs_ctx* ctx, const double* blocks4, uint32_t n_blocks, const int32_t* nodes4,
                      const double* lines, uint32_t n_nodes, int32_t root, int n_max, uint32_t source_size);
/* locate_block at npts points. */
int igs_locate_blocks(igs_ctx* ctx, const double* uv, uint32_t npts, int32_t* blocks);
/* render_image_blocked (bsp.cpp:334) through the resident partition. */
int igs_render_image_blocked(igs_ctx* ctx, int width, int height, int k, float* out_rgb);
/* Rows [row0, row1) of the blocked render (tile-row sharding of the decode /
 * evaluation render); out_rgb receives (row1-row0)*W*3 floats (nullable). */
int igs_render_image_blocked_rows(igs_ctx* ctx, int width, int height, int k, int row0, int row1, float* out_rgb);
/* render_topk_blocked at npts points (random-access decode queries). */
int igs_render_points_blocked(igs_ctx* ctx, const double* uv, uint32_t npts, int k, double* rgb);

/* bench_render (bsp.hpp:89-106, bsp.cpp:343-406): `pixels` random points
 * from Rng(seed); rows[0] = the unpartitioned global top-K baseline
 * (n_max 0, n_b 0, candidates = N), rows[1 + i] = n_max_values[i]:
 * build_partition, then blocked queries.  Times are device time per trial
 * (CUDA events), in ms per 10k points, mean and population std over
 * `trials` after `warmup`; mean_candidates is the reference's count.  The
 * last partition stays resident. */
typedef struct {
    int n_max, n_b;
    double mean_ms_per_10k, std_ms, mean_candidates;
} igs_bench_row;
int igs_bench_render(igs_ctx* ctx, int pixels, const int* n_max_values, int n_values, uint64_t seed, int trials,
                     int warmup, igs_bench_row* rows /* n_values + 1 */);

/* The device's prepared scan records (mu_x, mu_y, cos, sin, 1/s1^2, 1/s2^2)
 * per Gaussian (PreparedSet::scan, renderer.hpp:31-34): n*6 doubles. */
int igs_get_prepared(igs_ctx* ctx, double* scan6, uint32_t n);

/* ---- culling introspection (tile lists for parity tests) ------------------ */
/* Builds the certified candidate lists for a W x H raster at k and returns
 * the CSR (offsets ntiles+1, members ascending within each tile).  Pass
 * NULL arrays to query sizes via ntiles/total. */
int igs_tile_lists(igs_ctx* ctx, int width, int height, int k, uint32_t* ntiles, uint64_t* total,
                   uint32_t* offsets, uint32_t* members, double* tau);

/* ---- IGS2 container (codec.hpp:46-57, codec.cpp:141-224) ------------------- */
/* encode(set, partition?, width, height, k): the resident set (and, with
 * with_partition, the resident partition's blocks) as IGS2 bytes -- binary16
 * packing on the device.  out == NULL or cap too small: *size only. */
int igs_encode(igs_ctx* ctx, int with_partition, uint32_t width, uint32_t height, int k, uint8_t* out, size_t cap,
               size_t* size);
/* decode(bytes): validates like the reference, unpacks + constrains the set on
 * the device (it becomes the resident set), and rebuilds the partition from
 * the stored block corners when there are any (rebuild_partition). */
int igs_decode(igs_ctx* ctx, const uint8_t* bytes, size_t size, uint32_t* width, uint32_t* height, int* k,
               uint32_t* n_blocks);
/* quantize_set (codec.cpp:69-81) in place: every parameter through binary16, re-constrained. */
int igs_quantize_set(igs_ctx* ctx);

/* ---- benchmark support (device timing on the context's stream) ----------- */
int igs_timer_begin(igs_ctx* ctx);
/* Records the stop event (unless igs_train_iterations already recorded it
 * right after its last kernel), waits for it, returns elapsed ms. */
int igs_timer_end(igs_ctx* ctx, float* ms);
/* Numbered timing marks for pipelined loops: records event `idx` on the
 * stream without waiting; igs_timer_between waits for mark b and returns the
 * elapsed ms from mark a to mark b. */
int igs_timer_mark(igs_ctx* ctx, uint32_t idx);
int igs_timer_between(igs_ctx* ctx, uint32_t a, uint32_t b, float* ms);
/* Overwrites a scratch buffer of `bytes` (choose > 126 MB L2) on the stream. */
int igs_flush_l2(igs_ctx* ctx, size_t bytes);
/* Microbenchmarks the FP64 add/mul pipe (independent DADD/DMUL chains,
 * every SM): returns operations per second. */
int igs_fp64_peak(igs_ctx* ctx, double* ops_per_s);
/* glibc-exact exp(x) and sincos(x) (csrc/glibc_math.cuh) evaluated on the
 * device: out3[3i..3i+2] = exp, sin, cos of x[i] (parity diagnostics). */
int igs_libm_eval(igs_ctx* ctx, const double* x, uint32_t n, double* out3);
/* The hand-written device primitives of kernel 2 on host arrays (tests):
 * exclusive scan of n u32, and the stable LSD radix sort of (key, value)
 * pairs by the low `bits` key bits. */
int igs_debug_scan(igs_ctx* ctx, const uint32_t* in, uint32_t n, uint32_t* out);
int igs_debug_sort_pairs(igs_ctx* ctx, const uint64_t* keys, const uint32_t* vals, uint32_t n, int bits,
                         uint64_t* keys_out, uint32_t* vals_out);
/* Per-kernel-family CUDA-event profiling of the launches the context issues. */
#define IGS_PROF_SCAN 0    /* top-K candidate scans (raster, point/sample scans) */
#define IGS_PROF_FINISH 1  /* per-sample blend + loss + contributions */
#define IGS_PROF_REDUCE 2  /* sample-ordered gradient reduction (sort + segment sum) */
#define IGS_PROF_ADAM 3    /* fused Adam + constrain + prepare */
#define IGS_PROF_CULL 4    /* certified tile-list construction */
#define IGS_PROF_BLOCKED 5 /* BSP shell binning + blocked raster */
#define IGS_PROF_KNN_HARD 6 /* work = points resolved by the full-scan fallback */
#define IGS_PROF_FAMILIES 8
int igs_profile_enable(igs_ctx* ctx, int on);
/* total ms, launch count and algorithmic work (pairs for scans, bytes for
 * Adam) accumulated since igs_profile_enable(ctx, 1). */
int igs_profile_read(igs_ctx* ctx, int family, double* ms, uint64_t* launches, double* work);

/* ---- multi-GPU (one context per GPU, one process or thread each) --------- */
/* Training splits each iteration's samples into contiguous equal rank blocks;
 * every rank searches its block, an in-place all-gather completes the
 * per-sample contribution / key / loss arrays in global sample order, and
 * the sample-ordered reduction + Adam follow (bit-identical to one GPU).
 * The fp64-atomics mode (IGS_OPT_DETERMINISTIC 0) all-reduces the gradients
 * instead.  Rendering needs no communication (igs_render_image_rows). */
int igs_comm_unique_id(uint8_t id[128]);
/* NCCL communicator over NVLink (one rank per context). */
int igs_comm_init(igs_ctx* ctx, const uint8_t id[128], int nranks, int rank);
/* In-process loopback group of nranks contexts (any devices, including one
 * device for all ranks): the same collectives as cudaMemcpyAsync between the
 * contexts' buffers, ordered by events; each rank must then be driven by
 * its own host thread, as with NCCL.  For testing the R-rank exchange on
 * one GPU (NCCL rejects two ranks on one device). */
int igs_comm_init_loopback(igs_ctx** ctxs, int nranks);
int igs_comm_destroy(igs_ctx* ctx);
/* With IGS_OPT_SHARD_ADAM each rank keeps only its slice of the Adam
 * moments current; this (collective: every rank calls it) all-gathers them,
 * e.g. before igs_get_adam_state.  Calls that change the set (set_params,
 * append_params, decode, adam_step) must be made on every rank alike. */
int igs_comm_gather_moments(igs_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
