// ref_shim.cpp -- C entry points over the UNMODIFIED reference library.
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// reference's own sources under /root/reference/proj/src (never copied) into
// oracle/_ref/libigs_ref.so.  Each ref_* function has the signature of the
// matching orc_* restatement in igs_oracle.h, so tests can run both on the
// same inputs and demand bit-identical results (the oracle "pin"), and
// bench.py --impl reference can time the reference's own OpenMP code path.
#include <cmath>
#include <cstring>
#include <sstream>
#include <span>
#include <vector>

#include "igs/adam.hpp"
#include "igs/bsp.hpp"
#include "igs/codec.hpp"
#include "igs/error.hpp"
#include "igs/fit.hpp"
#include "igs/metrics.hpp"
#include "igs/renderer.hpp"
#include "igs/sampling.hpp"

using namespace igs;

namespace {

int code_of(const Error& e) { return 1 + static_cast<int>(e.kind()); }

GaussianSet to_set(const double* p8, uint32_t n) {
    GaussianSet s;
    s.gaussians.resize(n);
    static_assert(sizeof(Gaussian2D) == 64, "Gaussian2D must be 8 packed doubles");
    if (n) std::memcpy(s.gaussians.data(), p8, sizeof(double) * 8 * n);
    return s;
}

ImageBuffer to_image(const float* rgb, int W, int H) {
    ImageBuffer img(W, H);
    std::memcpy(img.data().data(), rgb, sizeof(float) * 3 * static_cast<size_t>(W) * H);
    return img;
}

}  // namespace

extern "C" {

int ref_render_image(const double* p8, uint32_t n, int W, int H, int k, float* out, uint32_t* topk_idx) {
    try {
        const GaussianSet set = to_set(p8, n);
        const ImageBuffer img = render_image(set, W, H, k);
        std::memcpy(out, img.data().data(), sizeof(float) * img.data().size());
        if (topk_idx) {
            PreparedSet ps(set);
            const int kk = static_cast<int>(std::min<size_t>(k, n));
            std::vector<TopKEntry> e(kk);
            for (int h = 0; h < H; ++h)
                for (int w = 0; w < W; ++w) {
                    const PixelCoord pc = pixel_center(h, w, H, W);
                    const int c = select_top_k_entries(ps, ps.all_indices(), {pc.u, pc.v}, kk, e.data());
                    uint32_t* t = topk_idx + (static_cast<size_t>(h) * W + w) * kk;
                    for (int j = 0; j < kk; ++j) t[j] = j < c ? e[j].idx : 0xFFFFFFFFu;
                }
        }
        return 0;
    } catch (const Error& e) {
        return code_of(e);
    }
}

int ref_select_top_k(const double* p8, uint32_t n, double u, double v, int k, uint32_t* idx, double* w,
                     int* count) {
    try {
        const TopKSelection s = select_top_k(to_set(p8, n), {u, v}, k);
        for (size_t i = 0; i < s.indices.size(); ++i) {
            idx[i] = s.indices[i];
            w[i] = s.weights[i];
        }
        *count = static_cast<int>(s.indices.size());
        return 0;
    } catch (const Error& e) {
        return code_of(e);
    }
}

int ref_render_topk(const double* p8, uint32_t n, const double* uv, uint32_t npts, int k, double* rgb) {
    try {
        const GaussianSet set = to_set(p8, n);
        for (uint32_t i = 0; i < npts; ++i) {
            const Color3 c = render_topk(set, {uv[2 * i], uv[2 * i + 1]}, k);
            rgb[3 * i] = c.r;
            rgb[3 * i + 1] = c.g;
            rgb[3 * i + 2] = c.b;
        }
        return 0;
    } catch (const Error& e) {
        return code_of(e);
    }
}

// Global top-K at npts points through one PreparedSet (select_top_k_entries
// over all indices, renderer.cpp:53-74), OpenMP over points -- the batched
// form of select_top_k for parity checks at the BASELINE sizes.  idx/q are
// npts*min(k,n), best-first; unused slots 0xFFFFFFFF / +inf.
int ref_topk_points(const double* p8, uint32_t n, const double* uv, uint32_t npts, int k, uint32_t* idx, double* q) {
    try {
        const GaussianSet set = to_set(p8, n);
        if (set.empty()) raise(ErrorKind::empty_set, "empty Gaussian set");
        if (k < 1) raise(ErrorKind::invalid_parameter, "k must be >= 1");
        PreparedSet ps(set);
        const int kk = static_cast<int>(std::min<size_t>(k, n));
#pragma omp parallel
        {
            std::vector<TopKEntry> e(kk);
#pragma omp for schedule(static)
            for (int64_t i = 0; i < static_cast<int64_t>(npts); ++i) {
                const int c = select_top_k_entries(ps, ps.all_indices(), {uv[2 * i], uv[2 * i + 1]}, kk, e.data());
                for (int j = 0; j < kk; ++j) {
                    idx[i * kk + j] = j < c ? e[j].idx : 0xFFFFFFFFu;
                    q[i * kk + j] = j < c ? e[j].q : INFINITY;
                }
            }
        }
        return 0;
    } catch (const Error& e) {
        return code_of(e);
    }
}

int ref_render_naive(const double* p8, uint32_t n, const double* uv, uint32_t npts, double* rgb) {
    try {
        const GaussianSet set = to_set(p8, n);
        for (uint32_t i = 0; i < npts; ++i) {
            const Color3 c = render_naive(set, {uv[2 * i], uv[2 * i + 1]});
            rgb[3 * i] = c.r;
            rgb[3 * i + 1] = c.g;
            rgb[3 * i + 2] = c.b;
        }
        return 0;
    } catch (const Error& e) {
        return code_of(e);
    }
}

// parallel=1 -> backward() (OpenMP map + ordered reduce), else backward_serial().
int ref_backward_mode(const double* p8, uint32_t n, const double* s5, uint32_t ns, int k, double* grads8,
                      int parallel) {
    try {
        static_assert(sizeof(PixelSample) == 40, "PixelSample must be 5 packed doubles");
        static_assert(sizeof(GaussianGrad) == 64, "GaussianGrad must be 8 packed doubles");
        const GaussianSet set = to_set(p8, n);
        std::span<const PixelSample> samples(reinterpret_cast<const PixelSample*>(s5), ns);
        const auto g = parallel ? backward(set, samples, k) : backward_serial(set, samples, k);
        std::memcpy(grads8, g.data(), sizeof(double) * 8 * n);
        return 0;
    } catch (const Error& e) {
        return code_of(e);
    }
}

int ref_backward(const double* p8, uint32_t n, const double* s5, uint32_t ns, int k, double* grads8) {
    return ref_backward_mode(p8, n, s5, ns, k, grads8, 1);
}

// fit.cpp's train_step_gradients is file-static; restate its public-API
// composition exactly: PreparedSet + per-sample select/blend/sign/gradients
// + sample-ordered reductions (fit.cpp:51-106).  The OpenMP map is kept.
int ref_train_step(const double* p8, uint32_t n, const float* target, int W, int H, const uint32_t* sidx,
                   uint32_t ns, int k, double* loss_out, double* grads8) {
    try {
        const GaussianSet set = to_set(p8, n);
        if (set.empty()) raise(ErrorKind::empty_set, "empty");
        if (k < 1) raise(ErrorKind::invalid_parameter, "k");
        PreparedSet ps(set);
        const int kk = static_cast<int>(std::min<size_t>(k, n));
        const double inv_n = 1.0 / static_cast<double>(ns);
        std::vector<SampleContrib> contribs(static_cast<size_t>(ns) * kk);
        std::vector<int> counts(ns);
        std::vector<double> losses(ns);
        const auto cands = ps.all_indices();
#pragma omp parallel
        {
            std::vector<TopKEntry> entries(kk);
#pragma omp for schedule(static)
            for (long long i = 0; i < static_cast<long long>(ns); ++i) {
                const int h = static_cast<int>(sidx[i]) / W;
                const int w = static_cast<int>(sidx[i]) % W;
                const PixelCoord pc = pixel_center(h, w, H, W);
                const Vec2 x{pc.u, pc.v};
                const float* t = target + (static_cast<size_t>(h) * W + w) * 3;
                const Color3 c_t{t[0], t[1], t[2]};
                const int cnt = select_top_k_entries(ps, cands, x, kk, entries.data());
                const BlendResult blend = blend_entries(ps, entries.data(), cnt);
                const Color3 diff = blend.color - c_t;
                losses[i] = diff.abs_sum();
                auto sg = [](double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); };
                const Color3 up{sg(diff.r) * inv_n, sg(diff.g) * inv_n, sg(diff.b) * inv_n};
                sample_gradients(ps, x, entries.data(), cnt, up, blend, &contribs[i * kk]);
                counts[i] = cnt;
            }
        }
        double loss = 0.0;
        for (uint32_t i = 0; i < ns; ++i) loss += losses[i];
        *loss_out = loss * inv_n;
        std::memset(grads8, 0, sizeof(double) * 8 * n);
        for (uint32_t i = 0; i < ns; ++i)
            for (int j = 0; j < counts[i]; ++j) {
                const SampleContrib& sc = contribs[static_cast<size_t>(i) * kk + j];
                for (int p = 0; p < 8; ++p) grads8[static_cast<size_t>(sc.idx) * 8 + p] += sc.d[p];
            }
        return 0;
    } catch (const Error& e) {
        return code_of(e);
    }
}

int ref_adam_step(double* p8, const double* g8, double* m, double* v, uint32_t n, const double* lr4, long long t,
                  int64_t* bad) {
    GaussianSet set = to_set(p8, n);
    std::vector<GaussianGrad> grads(n);
    if (n) std::memcpy(grads.data(), g8, sizeof(double) * 8 * n);
    AdamState st;
    st.m.assign(m, m + static_cast<size_t>(n) * 8);
    st.v.assign(v, v + static_cast<size_t>(n) * 8);
    LearningRates lr{lr4[0], lr4[1], lr4[2], lr4[3]};
    try {
        adam_step(set, grads, st, lr, t);
    } catch (const Error& e) {
        if (bad) {
            *bad = -1;
            for (size_t i = 0; i < static_cast<size_t>(n) * 8; ++i)
                if (!std::isfinite(g8[i])) {
                    *bad = static_cast<int64_t>(i);
                    break;
                }
        }
        return code_of(e);
    }
    std::memcpy(p8, set.gaussians.data(), sizeof(double) * 8 * n);
    std::memcpy(m, st.m.data(), sizeof(double) * 8 * n);
    std::memcpy(v, st.v.data(), sizeof(double) * 8 * n);
    return 0;
}

int ref_constrain(double* p8, uint32_t n) {
    try {
        GaussianSet s = to_set(p8, n);
        constrain_all(s);
        std::memcpy(p8, s.gaussians.data(), sizeof(double) * 8 * n);
        return 0;
    } catch (const Error& e) {
        return code_of(e);
    }
}

double ref_density(const double* g8, double u, double v) {
    Gaussian2D g;
    std::memcpy(&g, g8, sizeof(double) * 8);
    return density(g, {u, v});
}

void ref_image_gradient_magnitude(const float* img, int W, int H, double* mag) {
    const auto m = image_gradient_magnitude(to_image(img, W, H));
    std::memcpy(mag, m.data(), sizeof(double) * m.size());
}

int ref_gradient_mixture(const float* img, int W, int H, double lambda, double* p) {
    try {
        const SamplingDistribution d = opt_distribution(to_image(img, W, H), lambda);
        std::memcpy(p, d.p.data(), sizeof(double) * d.p.size());
        return 0;
    } catch (const Error& e) {
        return code_of(e);
    }
}

int ref_add_distribution(const float* rendered, const float* target, int W, int H, double* p) {
    try {
        const SamplingDistribution d = add_distribution(to_image(rendered, W, H), to_image(target, W, H));
        std::memcpy(p, d.p.data(), sizeof(double) * d.p.size());
        return 0;
    } catch (const Error& e) {
        return code_of(e);
    }
}

// n draws through AliasTable + Rng(seed), as sample_pixel_indices does.
int ref_sample_pixel_indices(const double* weights, int W, int H, int n, uint64_t seed, uint32_t* out) {
    try {
        SamplingDistribution d{W, H, std::vector<double>(weights, weights + static_cast<size_t>(W) * H)};
        Rng rng(seed);
        const auto idx = sample_pixel_indices(d, n, rng);
        std::memcpy(out, idx.data(), sizeof(uint32_t) * idx.size());
        return 0;
    } catch (const Error& e) {
        return code_of(e);
    }
}

int ref_initialize_set(const float* img, int W, int H, int count, double lambda, uint64_t seed, double* out8) {
    try {
        Rng rng(seed);
        const GaussianSet s = initialize_set(to_image(img, W, H), count, lambda, rng);
        std::memcpy(out8, s.gaussians.data(), sizeof(double) * 8 * s.size());
        return 0;
    } catch (const Error& e) {
        return code_of(e);
    }
}

double ref_psnr(const float* a, const float* b, size_t count) {
    ImageBuffer x(static_cast<int>(count / 3), 1), y(static_cast<int>(count / 3), 1);
    std::memcpy(x.data().data(), a, sizeof(float) * count);
    std::memcpy(y.data().data(), b, sizeof(float) * count);
    return psnr(x, y);
}

double ref_ssim(const float* a, const float* b, int W, int H) { return ssim(to_image(a, W, H), to_image(b, W, H)); }

void ref_rng_stream(uint64_t seed, uint64_t skip, uint32_t count, uint64_t* out) {
    Rng r(seed);
    for (uint64_t i = 0; i < skip; ++i) (void)r.next_u64();
    for (uint32_t i = 0; i < count; ++i) out[i] = r.next_u64();
}

// ---- BSP ------------------------------------------------------------------
struct ref_partition {
    BspPartition p;
};

ref_partition* ref_partition_build(const double* p8, uint32_t n, int n_max, int* err) {
    try {
        auto* r = new ref_partition{build_partition(to_set(p8, n), n_max)};
        *err = 0;
        return r;
    } catch (const Error& e) {
        *err = code_of(e);
        return nullptr;
    }
}

ref_partition* ref_partition_rebuild(const double* rects4, uint32_t nb, const double* p8, uint32_t n, int* err) {
    try {
        std::vector<Rect> blocks(nb);
        static_assert(sizeof(Rect) == 32, "Rect must be 4 packed doubles");
        if (nb) std::memcpy(blocks.data(), rects4, sizeof(Rect) * nb);
        auto* r = new ref_partition{rebuild_partition(std::move(blocks), to_set(p8, n))};
        *err = 0;
        return r;
    } catch (const Error& e) {
        *err = code_of(e);
        return nullptr;
    }
}

void ref_partition_free(ref_partition* p) { delete p; }
uint32_t ref_partition_nblocks(const ref_partition* p) { return static_cast<uint32_t>(p->p.blocks.size()); }
uint64_t ref_partition_shell_total(const ref_partition* p) {
    uint64_t t = 0;
    for (const auto& m : p->p.shell_members) t += m.size();
    return t;
}
void ref_partition_rects(const ref_partition* p, double* blocks4, double* shells4) {
    if (blocks4) std::memcpy(blocks4, p->p.blocks.data(), sizeof(Rect) * p->p.blocks.size());
    if (shells4) std::memcpy(shells4, p->p.shells.data(), sizeof(Rect) * p->p.shells.size());
}
static void csr(const std::vector<std::vector<uint32_t>>& v, uint32_t* off, uint32_t* mem) {
    uint32_t o = 0;
    for (size_t b = 0; b < v.size(); ++b) {
        off[b] = o;
        std::memcpy(mem + o, v[b].data(), sizeof(uint32_t) * v[b].size());
        o += static_cast<uint32_t>(v[b].size());
    }
    off[v.size()] = o;
}
void ref_partition_shell_members(const ref_partition* p, uint32_t* off, uint32_t* mem) { csr(p->p.shell_members, off, mem); }
void ref_partition_block_members(const ref_partition* p, uint32_t* off, uint32_t* mem) { csr(p->p.block_members, off, mem); }
int ref_locate_block(const ref_partition* p, double u, double v) { return locate_block(p->p, {u, v}); }

int ref_render_image_blocked(const double* p8, uint32_t n, const ref_partition* part, int W, int H, int k,
                             float* out) {
    try {
        const ImageBuffer img = render_image_blocked(to_set(p8, n), part->p, W, H, k);
        std::memcpy(out, img.data().data(), sizeof(float) * img.data().size());
        return 0;
    } catch (const Error& e) {
        return code_of(e);
    }
}

int ref_render_points_blocked(const double* p8, uint32_t n, const ref_partition* part, const double* uv,
                              uint32_t npts, int k, double* rgb) {
    try {
        const GaussianSet set = to_set(p8, n);
        PreparedSet ps(set);
        for (uint32_t i = 0; i < npts; ++i) {
            const Color3 c = render_topk_blocked(ps, part->p, {uv[2 * i], uv[2 * i + 1]}, k);
            rgb[3 * i] = c.r;
            rgb[3 * i + 1] = c.g;
            rgb[3 * i + 2] = c.b;
        }
        return 0;
    } catch (const Error& e) {
        return code_of(e);
    }
}

// The reference's fit() (fit.cpp:116-207) on a float32 target; config in
// the layout of igs_fit_config (budget, k, lambda_init, lambda_opt,
// iterations, samples, lr[4], eval_interval, patience, lr_decay, warmup,
// densify_interval, seed, compute_ssim).  Writes the final set (capacity
// max_n records) and the FitReport log.
struct RefFitConfig {
    int budget, k;
    double lambda_init, lambda_opt;
    int iterations, samples_per_iter;
    double lr[4];
    int eval_interval, plateau_patience;
    double lr_decay;
    int warmup_iters, densify_interval;
    uint64_t seed;
    int compute_ssim;
};

int ref_fit(const float* target, int W, int H, const RefFitConfig* c, double* out8, uint32_t max_n, uint32_t* n_out,
            char* log, size_t cap) {
    try {
        FitConfig fc;
        fc.budget = c->budget;
        fc.k = c->k;
        fc.lambda_init = c->lambda_init;
        fc.lambda_opt = c->lambda_opt;
        fc.iterations = c->iterations;
        fc.samples_per_iter = c->samples_per_iter;
        fc.lr = LearningRates{c->lr[0], c->lr[1], c->lr[2], c->lr[3]};
        fc.eval_interval = c->eval_interval;
        fc.plateau_patience = c->plateau_patience;
        fc.lr_decay = c->lr_decay;
        fc.warmup_iters = c->warmup_iters;
        fc.densify_interval = c->densify_interval;
        fc.seed = c->seed;
        auto [set, report] = fit(to_image(target, W, H), fc);
        *n_out = static_cast<uint32_t>(set.size());
        std::memcpy(out8, set.gaussians.data(), sizeof(double) * 8 * std::min<size_t>(set.size(), max_n));
        std::ostringstream os;
        report.write(os, fc);
        const std::string s = os.str();
        const size_t m = std::min(s.size(), cap - 1);
        std::memcpy(log, s.data(), m);
        log[m] = 0;
        return 0;
    } catch (const Error& e) {
        return code_of(e);
    }
}

// bench_render (bsp.cpp:343-406) as the reference runs it: rows5 receives
// (n_max, n_b, mean_ms_per_10k, std_ms, mean_candidates) for the baseline
// and then each n_max.
int ref_bench_render(const double* p8, uint32_t n, int pixels, const int* nmax, int nv, uint64_t seed, int trials,
                     int warmup, double* rows5) {
    try {
        const GaussianSet set = to_set(p8, n);
        const BenchResult r = bench_render(set, pixels, std::vector<int>(nmax, nmax + nv), seed, trials, warmup);
        auto put = [&](int i, const BenchRow& b) {
            rows5[5 * i] = b.n_max;
            rows5[5 * i + 1] = b.n_b;
            rows5[5 * i + 2] = b.mean_ms_per_10k;
            rows5[5 * i + 3] = b.std_ms;
            rows5[5 * i + 4] = b.mean_candidates;
        };
        put(0, r.baseline);
        for (size_t i = 0; i < r.rows.size(); ++i) put(static_cast<int>(i) + 1, r.rows[i]);
        return 0;
    } catch (const Error& e) {
        return code_of(e);
    }
}

// One reference Adam step over an already-built set (used by the CPU
// baseline timing of a full train iteration).
int ref_train_iteration(double* p8, uint32_t n, double* m, double* v, const float* target, int W, int H,
                        const uint32_t* sidx, uint32_t ns, int k, const double* lr4, long long t, double* loss) {
    std::vector<double> grads(static_cast<size_t>(n) * 8);
    int e = ref_train_step(p8, n, target, W, H, sidx, ns, k, loss, grads.data());
    if (e) return e;
    return ref_adam_step(p8, grads.data(), m, v, n, lr4, t, nullptr);
}


// ---- IGS2 codec (codec.cpp) --------------------------------------------------
// encode(set, partition?, W, H, k) into out (cap bytes); *size = full length
int ref_encode(const double* p8, uint32_t n, const ref_partition* part, uint32_t W, uint32_t H, int k, uint8_t* out,
               size_t cap, size_t* size) {
    try {
        const std::vector<uint8_t> b = encode(to_set(p8, n), part ? &part->p : nullptr, W, H, k);
        *size = b.size();
        if (out && cap >= b.size()) std::memcpy(out, b.data(), b.size());
        return 0;
    } catch (const Error& e) {
        return code_of(e);
    }
}

// decode(bytes): the set (<= max_n records), header fields, and the rebuilt
// partition (null when the file has no blocks)
int ref_decode(const uint8_t* bytes, size_t size, double* out8, uint32_t max_n, uint32_t* n, uint32_t* W,
               uint32_t* H, int* k, ref_partition** part) {
    try {
        Decoded d = decode(std::vector<uint8_t>(bytes, bytes + size));
        *n = static_cast<uint32_t>(d.set.size());
        if (out8 && d.set.size() <= max_n) std::memcpy(out8, d.set.gaussians.data(), 64 * d.set.size());
        *W = d.width;
        *H = d.height;
        *k = d.k;
        *part = d.partition ? new ref_partition{std::move(*d.partition)} : nullptr;
        return 0;
    } catch (const Error& e) {
        return code_of(e);
    }
}

int ref_quantize_set(double* p8, uint32_t n) {
    try {
        const GaussianSet q = quantize_set(to_set(p8, n));
        std::memcpy(p8, q.gaussians.data(), 64 * static_cast<size_t>(n));
        return 0;
    } catch (const Error& e) {
        return code_of(e);
    }
}

}  // extern "C"
