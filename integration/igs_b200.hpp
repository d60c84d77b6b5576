// igs_b200.hpp -- header-only C++ drop-in over the B200 C-ABI, using the
// reference's own types (include/igs/*.hpp) and signatures.
//
// A reference user switches a call site from igs::render_image(...) to
// igs_b200::render_image(...) (or adds `namespace igs = igs_b200;` in a
// translation unit that only uses the hot-path API).  The types --
// GaussianSet, ImageBuffer, PixelSample, GaussianGrad, AdamState,
// LearningRates, BspPartition, SamplingDistribution, FitConfig/FitReport,
// Decoded, igs::Error -- are the reference's; only the implementation moves
// to the GPU.  Errors come back as igs::Error with the reference's
// ErrorKind and message.
//
// Covered (reference header:line): renderer.hpp:110-138 (select_top_k,
// render_topk, render_image, backward), adam.hpp:40-41 (adam_step),
// bsp.hpp:70-93 (build_partition, rebuild_partition, locate_block,
// render_topk_blocked, render_image_blocked), sampling.hpp:36-59
// (init/opt/add_distribution, initialize_set), metrics.hpp:9-14 (psnr,
// ssim), codec.hpp:24,52-57 (quantize_set, encode, decode) and fit.hpp:63-64
// (fit with CheckpointFn -> {GaussianSet, FitReport}).
//
// Calls are pure like the reference's: each uploads what it needs (the set,
// a partition) to the device context and reads the result back.  Keep a
// Device and call the C-ABI directly to stay device-resident across calls.
//
// Link: -ligs_b200 (paper_2407_01866_b200/libigs_b200.so); needs only the
// reference's headers, not its library.
#pragma once

#include <algorithm>
#include <cstring>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "igs/adam.hpp"
#include "igs/bsp.hpp"
#include "igs/codec.hpp"
#include "igs/error.hpp"
#include "igs/fit.hpp"
#include "igs/gaussian.hpp"
#include "igs/image.hpp"
#include "igs/renderer.hpp"
#include "igs/rng.hpp"
#include "igs/sampling.hpp"
#include "igs_b200.h"

namespace igs_b200 {

static_assert(sizeof(igs::Gaussian2D) == 64, "Gaussian2D must be 8 packed doubles");
static_assert(sizeof(igs::GaussianGrad) == 64, "GaussianGrad must be 8 packed doubles");
static_assert(sizeof(igs::PixelSample) == 40, "PixelSample must be 5 packed doubles");
static_assert(sizeof(igs::Rect) == 32, "Rect must be 4 packed doubles");

// igs_ctx RAII holder; one per GPU.  The free functions below use a
// process-wide device-0 context unless one is passed explicitly.
class Device {
public:
    explicit Device(int device = 0) {
        if (igs_ctx_create(device, &ctx_) != IGS_OK) throw std::runtime_error("igs_b200: no CUDA device");
    }
    ~Device() { igs_ctx_destroy(ctx_); }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    igs_ctx* get() const { return ctx_; }

    // Maps an ABI status to the reference's exception (error.hpp:8-28).
    void check(int code) const {
        if (code == IGS_OK) return;
        const std::string msg = igs_last_error(ctx_);
        if (code >= 1 && code <= 8) throw igs::Error(static_cast<igs::ErrorKind>(code - 1), msg);
        throw std::runtime_error("igs_b200: " + msg);
    }
    void upload(const igs::GaussianSet& set) const {
        check(igs_set_params(ctx_, reinterpret_cast<const double*>(set.gaussians.data()),
                             static_cast<uint32_t>(set.size())));
    }

private:
    igs_ctx* ctx_ = nullptr;
};

inline Device& default_device() {
    static Device d(0);
    return d;
}

namespace detail {

inline void require_nonempty(const igs::GaussianSet& set, const char* what) {
    if (set.empty()) throw igs::Error(igs::ErrorKind::empty_set, std::string(what) + " requires a non-empty GaussianSet");
}

inline const float* pixels(const igs::ImageBuffer& img) { return img.data().data(); }

// the resident partition as the reference's struct
inline igs::BspPartition download_partition(Device& dev) {
    uint32_t nb = 0;
    uint64_t shell_total = 0;
    dev.check(igs_partition_info(dev.get(), &nb, &shell_total));
    int n_max = 0, grid_dim = 0;
    uint32_t source = 0, n_nodes = 0, grid_total = 0;
    int32_t root = -1;
    dev.check(igs_partition_export(dev.get(), &n_max, &source, &root, &n_nodes, &grid_dim, &grid_total));
    igs::BspPartition p;
    p.blocks.resize(nb);
    p.shells.resize(nb);
    std::vector<uint32_t> soff(nb + 1), smem(shell_total);
    dev.check(igs_partition_get(dev.get(), reinterpret_cast<double*>(p.blocks.data()),
                                reinterpret_cast<double*>(p.shells.data()), soff.data(), smem.data()));
    p.shell_members.resize(nb);
    for (uint32_t b = 0; b < nb; ++b) p.shell_members[b].assign(smem.begin() + soff[b], smem.begin() + soff[b + 1]);
    std::vector<uint32_t> boff(nb + 1), bmem(source);
    dev.check(igs_partition_block_members(dev.get(), boff.data(), bmem.data()));
    p.block_members.resize(nb);
    for (uint32_t b = 0; b < nb; ++b) p.block_members[b].assign(bmem.begin() + boff[b], bmem.begin() + boff[b + 1]);
    p.n_max = n_max;
    p.source_size = source;
    p.root = root;
    if (n_nodes) {
        std::vector<int32_t> nodes4(4 * (size_t)n_nodes);
        std::vector<double> lines(n_nodes);
        dev.check(igs_partition_get_tree(dev.get(), nodes4.data(), lines.data()));
        p.nodes.resize(n_nodes);
        for (uint32_t i = 0; i < n_nodes; ++i) {
            p.nodes[i].axis = nodes4[4 * i];
            p.nodes[i].line = lines[i];
            p.nodes[i].low = nodes4[4 * i + 1];
            p.nodes[i].high = nodes4[4 * i + 2];
            p.nodes[i].block = nodes4[4 * i + 3];
        }
    }
    p.grid_dim = grid_dim;
    if (grid_dim > 0) {
        std::vector<uint32_t> goff((size_t)grid_dim * grid_dim + 1), gblk(grid_total);
        dev.check(igs_partition_get_grid(dev.get(), goff.data(), gblk.data()));
        p.grid_cells.resize((size_t)grid_dim * grid_dim);
        for (size_t c = 0; c < p.grid_cells.size(); ++c)
            p.grid_cells[c].assign(gblk.begin() + goff[c], gblk.begin() + goff[c + 1]);
    }
    return p;
}

// fills BspNode::point_bbox (bsp.cpp:120-130: bbox of the subtree's member
// positions; {1, 1, 0, 0} when empty) bottom-up from the block members
inline void fill_point_bboxes(igs::BspPartition& p, const igs::GaussianSet& set) {
    if (p.nodes.empty()) return;
    std::vector<int32_t> order;  // preorder, so children follow their parent
    std::vector<int32_t> stack{p.root};
    while (!stack.empty()) {
        const int32_t id = stack.back();
        stack.pop_back();
        order.push_back(id);
        if (p.nodes[id].block < 0) {
            stack.push_back(p.nodes[id].high);
            stack.push_back(p.nodes[id].low);
        }
    }
    for (auto it = order.rbegin(); it != order.rend(); ++it) {
        igs::BspNode& nd = p.nodes[*it];
        igs::Rect b{1.0, 1.0, 0.0, 0.0};
        if (nd.block >= 0) {
            for (uint32_t i : p.block_members[nd.block]) {
                b.x1 = std::min(b.x1, set[i].mu.x);
                b.y1 = std::min(b.y1, set[i].mu.y);
                b.x2 = std::max(b.x2, set[i].mu.x);
                b.y2 = std::max(b.y2, set[i].mu.y);
            }
        } else {
            const igs::Rect& l = p.nodes[nd.low].point_bbox;
            const igs::Rect& h = p.nodes[nd.high].point_bbox;
            b = {std::min(l.x1, h.x1), std::min(l.y1, h.y1), std::max(l.x2, h.x2), std::max(l.y2, h.y2)};
        }
        nd.point_bbox = b;
    }
}

// a caller-held partition onto the device (tree or grid locator)
inline void upload_partition(Device& dev, const igs::BspPartition& p) {
    std::vector<int32_t> nodes4(4 * p.nodes.size());
    std::vector<double> lines(p.nodes.size());
    for (size_t i = 0; i < p.nodes.size(); ++i) {
        nodes4[4 * i] = p.nodes[i].axis;
        nodes4[4 * i + 1] = p.nodes[i].low;
        nodes4[4 * i + 2] = p.nodes[i].high;
        nodes4[4 * i + 3] = p.nodes[i].block;
        lines[i] = p.nodes[i].line;
    }
    dev.check(igs_partition_set(dev.get(), reinterpret_cast<const double*>(p.blocks.data()),
                                static_cast<uint32_t>(p.blocks.size()), nodes4.data(), lines.data(),
                                static_cast<uint32_t>(p.nodes.size()), p.root, p.n_max, p.source_size));
}

inline igs::SamplingDistribution to_dist(int w, int h, std::vector<double> p) {
    igs::SamplingDistribution d;
    d.width = w;
    d.height = h;
    d.p = std::move(p);
    return d;
}

}  // namespace detail

// ---- renderer.hpp ---------------------------------------------------------
// renderer.hpp:117 render_image
inline igs::ImageBuffer render_image(const igs::GaussianSet& set, int width, int height, int k,
                                     Device& dev = default_device()) {
    dev.upload(set);
    if (width < 1 || height < 1) dev.check(igs_render_image(dev.get(), width, height, k, nullptr, nullptr));
    igs::ImageBuffer img(width, height);
    dev.check(igs_render_image(dev.get(), width, height, k, img.data().data(), nullptr));
    return img;
}

// renderer.hpp:110 select_top_k
inline igs::TopKSelection select_top_k(const igs::GaussianSet& set, igs::PixelCoord x, int k,
                                       Device& dev = default_device()) {
    dev.upload(set);
    const size_t kk = std::max<size_t>(1, std::min<size_t>(k < 1 ? 1 : k, set.size()));
    std::vector<uint32_t> idx(kk);
    std::vector<double> w(kk);
    int32_t cnt = 0;
    const double uv[2] = {x.u, x.v};
    dev.check(igs_select_top_k(dev.get(), uv, 1, k, idx.data(), w.data(), &cnt));
    igs::TopKSelection s;
    s.indices.assign(idx.begin(), idx.begin() + cnt);
    s.weights.assign(w.begin(), w.begin() + cnt);
    return s;
}

// renderer.hpp:113 render_topk
inline igs::Color3 render_topk(const igs::GaussianSet& set, igs::PixelCoord x, int k,
                               Device& dev = default_device()) {
    dev.upload(set);
    const double uv[2] = {x.u, x.v};
    double rgb[3];
    dev.check(igs_render_points(dev.get(), uv, 1, k, rgb));
    return {rgb[0], rgb[1], rgb[2]};
}

// renderer.hpp:125 backward
inline std::vector<igs::GaussianGrad> backward(const igs::GaussianSet& set, std::span<const igs::PixelSample> samples,
                                               int k, Device& dev = default_device()) {
    dev.upload(set);
    std::vector<igs::GaussianGrad> g(set.size());
    dev.check(igs_backward(dev.get(), reinterpret_cast<const double*>(samples.data()),
                           static_cast<uint32_t>(samples.size()), k, reinterpret_cast<double*>(g.data())));
    return g;
}

// ---- adam.hpp -------------------------------------------------------------
// adam.hpp:40-41 adam_step: the moments travel with the call like AdamState.
inline void adam_step(igs::GaussianSet& set, const std::vector<igs::GaussianGrad>& grads, igs::AdamState& state,
                      const igs::LearningRates& lr, long long t, Device& dev = default_device()) {
    if (grads.size() != set.size())
        throw igs::Error(igs::ErrorKind::dimension_mismatch, "gradient count != Gaussian count");
    state.resize(set.size());
    dev.upload(set);
    const uint32_t n = static_cast<uint32_t>(set.size());
    dev.check(igs_set_adam_state(dev.get(), state.m.data(), state.v.data(), n));
    dev.check(igs_set_grads(dev.get(), reinterpret_cast<const double*>(grads.data()), n));
    const double lr4[4] = {lr.mu, lr.color, lr.scale, lr.theta};
    dev.check(igs_adam_step(dev.get(), lr4, t));
    dev.check(igs_get_params(dev.get(), reinterpret_cast<double*>(set.gaussians.data()), n));
    dev.check(igs_get_adam_state(dev.get(), state.m.data(), state.v.data(), n));
}

// ---- bsp.hpp --------------------------------------------------------------
// bsp.hpp:70 build_partition: built on the device, returned as the
// reference's struct (blocks, shells, members, split tree with point boxes)
inline igs::BspPartition build_partition(const igs::GaussianSet& set, int n_max, Device& dev = default_device()) {
    detail::require_nonempty(set, "build_partition");
    dev.upload(set);
    dev.check(igs_partition_build(dev.get(), n_max));
    igs::BspPartition p = detail::download_partition(dev);
    detail::fill_point_bboxes(p, set);
    return p;
}

// bsp.hpp:74 rebuild_partition (the decode path): grid locator, memberships
inline igs::BspPartition rebuild_partition(std::vector<igs::Rect> blocks, const igs::GaussianSet& set,
                                           Device& dev = default_device()) {
    dev.upload(set);
    dev.check(igs_partition_rebuild(dev.get(), reinterpret_cast<const double*>(blocks.data()),
                                    static_cast<uint32_t>(blocks.size())));
    return detail::download_partition(dev);
}

// bsp.hpp:78 locate_block
inline int locate_block(const igs::BspPartition& p, igs::PixelCoord x, Device& dev = default_device()) {
    detail::upload_partition(dev, p);
    const double uv[2] = {x.u, x.v};
    int32_t b = -1;
    dev.check(igs_locate_blocks(dev.get(), uv, 1, &b));
    return b;
}

// bsp.hpp:82 render_topk_blocked
inline igs::Color3 render_topk_blocked(const igs::GaussianSet& set, const igs::BspPartition& p, igs::PixelCoord x,
                                       int k, Device& dev = default_device()) {
    dev.upload(set);
    detail::upload_partition(dev, p);
    const double uv[2] = {x.u, x.v};
    double rgb[3];
    dev.check(igs_render_points_blocked(dev.get(), uv, 1, k, rgb));
    return {rgb[0], rgb[1], rgb[2]};
}

// bsp.hpp:86 render_image_blocked
inline igs::ImageBuffer render_image_blocked(const igs::GaussianSet& set, const igs::BspPartition& p, int width,
                                             int height, int k, Device& dev = default_device()) {
    dev.upload(set);
    detail::upload_partition(dev, p);
    igs::ImageBuffer img(width, height);
    dev.check(igs_render_image_blocked(dev.get(), width, height, k, img.data().data()));
    return img;
}

// ---- sampling.hpp ---------------------------------------------------------
// sampling.hpp:28-35 init_distribution / opt_distribution (the gradient mixture)
inline igs::SamplingDistribution init_distribution(const igs::ImageBuffer& img, double lambda,
                                                   Device& dev = default_device()) {
    std::vector<double> p(img.pixel_count());
    dev.check(igs_gradient_mixture(dev.get(), detail::pixels(img), img.width(), img.height(), lambda, p.data()));
    return detail::to_dist(img.width(), img.height(), std::move(p));
}
inline igs::SamplingDistribution opt_distribution(const igs::ImageBuffer& img, double lambda,
                                                  Device& dev = default_device()) {
    return init_distribution(img, lambda, dev);
}

// sampling.hpp:24 image_gradient_magnitude
inline std::vector<double> image_gradient_magnitude(const igs::ImageBuffer& img, Device& dev = default_device()) {
    std::vector<double> m(img.pixel_count());
    dev.check(igs_image_gradient_magnitude(dev.get(), detail::pixels(img), img.width(), img.height(), m.data()));
    return m;
}

// sampling.hpp:59 initialize_set(img, count, lambda, rng): the caller's Rng
// advances by exactly the draws the reference makes (two per Gaussian)
inline igs::GaussianSet initialize_set(const igs::ImageBuffer& img, int count, double lambda, igs::Rng& rng,
                                       Device& dev = default_device()) {
    if (count < 1) throw igs::Error(igs::ErrorKind::invalid_parameter, "initialization count must be >= 1");
    std::vector<uint64_t> raw(2 * static_cast<size_t>(count));
    for (auto& r : raw) r = rng.next_u64();
    igs::GaussianSet set;
    set.gaussians.resize(static_cast<size_t>(count));
    dev.check(igs_initialize_set(dev.get(), detail::pixels(img), img.width(), img.height(), count, lambda, raw.data(),
                                 reinterpret_cast<double*>(set.gaussians.data())));
    return set;
}

// sampling.hpp:39 add_distribution(rendered, target)
inline igs::SamplingDistribution add_distribution(const igs::ImageBuffer& rendered, const igs::ImageBuffer& target,
                                                  Device& dev = default_device()) {
    if (!rendered.same_shape(target))
        throw igs::Error(igs::ErrorKind::dimension_mismatch, "rendered/target dimensions differ");
    dev.check(igs_set_target(dev.get(), detail::pixels(target), target.width(), target.height()));
    std::vector<double> p(target.pixel_count());
    dev.check(igs_add_distribution(dev.get(), detail::pixels(rendered), target.width(), target.height(), p.data()));
    return detail::to_dist(target.width(), target.height(), std::move(p));
}

// ---- metrics.hpp ----------------------------------------------------------
inline double psnr(const igs::ImageBuffer& a, const igs::ImageBuffer& b, Device& dev = default_device()) {
    if (!a.same_shape(b)) throw igs::Error(igs::ErrorKind::dimension_mismatch, "psnr: image dimensions differ");
    dev.check(igs_set_target(dev.get(), detail::pixels(b), b.width(), b.height()));
    double out = 0.0;
    dev.check(igs_psnr(dev.get(), detail::pixels(a), a.width(), a.height(), &out));
    return out;
}

inline double ssim(const igs::ImageBuffer& a, const igs::ImageBuffer& b, Device& dev = default_device()) {
    if (!a.same_shape(b)) throw igs::Error(igs::ErrorKind::dimension_mismatch, "ssim: image dimensions differ");
    dev.check(igs_set_target(dev.get(), detail::pixels(b), b.width(), b.height()));
    double out = 0.0;
    dev.check(igs_ssim(dev.get(), detail::pixels(a), a.width(), a.height(), &out));
    return out;
}

// ---- codec.hpp ------------------------------------------------------------
// codec.hpp:24 quantize_set
inline igs::GaussianSet quantize_set(const igs::GaussianSet& set, Device& dev = default_device()) {
    dev.upload(set);
    dev.check(igs_quantize_set(dev.get()));
    igs::GaussianSet out = set;
    dev.check(igs_get_params(dev.get(), reinterpret_cast<double*>(out.gaussians.data()),
                             static_cast<uint32_t>(out.size())));
    return out;
}

// codec.hpp:52-53 encode(set, partition*, width, height, k)
inline std::vector<uint8_t> encode(const igs::GaussianSet& set, const igs::BspPartition* partition, uint32_t width,
                                   uint32_t height, int k, Device& dev = default_device()) {
    dev.upload(set);
    if (partition) detail::upload_partition(dev, *partition);
    size_t size = 0;
    dev.check(igs_encode(dev.get(), partition ? 1 : 0, width, height, k, nullptr, 0, &size));
    std::vector<uint8_t> out(size);
    dev.check(igs_encode(dev.get(), partition ? 1 : 0, width, height, k, out.data(), out.size(), &size));
    return out;
}

// codec.hpp:57 decode(bytes): the set, the header, and the partition rebuilt
// from the stored corners when the file carries any
inline igs::Decoded decode(const std::vector<uint8_t>& bytes, Device& dev = default_device()) {
    uint32_t w = 0, h = 0, nb = 0;
    int k = 0;
    dev.check(igs_decode(dev.get(), bytes.data(), bytes.size(), &w, &h, &k, &nb));
    igs::Decoded d;
    const uint32_t n = igs_num_gaussians(dev.get());
    d.set.gaussians.resize(n);
    dev.check(igs_get_params(dev.get(), reinterpret_cast<double*>(d.set.gaussians.data()), n));
    d.width = w;
    d.height = h;
    d.k = k;
    if (nb) d.partition = detail::download_partition(dev);
    return d;
}

// ---- fit.hpp --------------------------------------------------------------
namespace detail {
struct FitCallback {
    const igs::CheckpointFn* fn;
    std::vector<std::string>* ids;
};
inline void on_checkpoint(void* user, int stage, int iteration, const char* id, const double* params8, uint32_t n) {
    auto* cb = static_cast<FitCallback*>(user);
    cb->ids->push_back(id);
    if (cb->fn && *cb->fn) {
        igs::GaussianSet s;
        s.gaussians.resize(n);
        std::memcpy(s.gaussians.data(), params8, sizeof(double) * 8 * n);
        (*cb->fn)(stage, iteration, std::string(id), s);
    }
}
}  // namespace detail

// fit.hpp:63-64 fit(target, config, on_checkpoint) -> {final set, FitReport}
inline std::pair<igs::GaussianSet, igs::FitReport> fit(const igs::ImageBuffer& target, const igs::FitConfig& c,
                                                       const igs::CheckpointFn& on_checkpoint = {},
                                                       Device& dev = default_device()) {
    igs_fit_config cfg;
    igs_fit_config_default(&cfg);
    cfg.budget = c.budget;
    cfg.k = c.k;
    cfg.lambda_init = c.lambda_init;
    cfg.lambda_opt = c.lambda_opt;
    cfg.iterations = c.iterations;
    cfg.samples_per_iter = c.samples_per_iter;
    cfg.lr[0] = c.lr.mu;
    cfg.lr[1] = c.lr.color;
    cfg.lr[2] = c.lr.scale;
    cfg.lr[3] = c.lr.theta;
    cfg.eval_interval = c.eval_interval;
    cfg.plateau_patience = c.plateau_patience;
    cfg.lr_decay = c.lr_decay;
    cfg.warmup_iters = c.warmup_iters;
    cfg.densify_interval = c.densify_interval;
    cfg.seed = c.seed;
    igs::FitReport report;
    detail::FitCallback cb{&on_checkpoint, &report.checkpoints};
    const int max_evals = c.iterations / std::max(1, c.eval_interval) + 2;
    std::vector<igs_eval_record> evals(static_cast<size_t>(max_evals));
    int n_evals = 0, decay = -1, final_count = 0;
    dev.check(igs_fit(dev.get(), detail::pixels(target), target.width(), target.height(), &cfg,
                      detail::on_checkpoint, &cb, evals.data(), max_evals, &n_evals, &decay, &final_count, nullptr, 0));
    for (int i = 0; i < n_evals; ++i) {
        const igs_eval_record& e = evals[static_cast<size_t>(i)];
        report.evals.push_back({e.iteration, e.count, e.loss, e.psnr, e.ssim, e.best_psnr});
    }
    report.lr_decay_iteration = decay;
    report.final_count = final_count;
    igs::GaussianSet set;
    set.gaussians.resize(static_cast<size_t>(final_count));
    dev.check(igs_get_params(dev.get(), reinterpret_cast<double*>(set.gaussians.data()),
                             static_cast<uint32_t>(final_count)));
    return {std::move(set), std::move(report)};
}

}  // namespace igs_b200
