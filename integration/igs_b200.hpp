// igs_b200.hpp -- header-only C++ drop-in over the B200 C-ABI, using the
// reference's own types (include/igs/*.hpp) and signatures.
//
// A reference user switches a call site from igs::render_image(...) to
// igs_b200::render_image(...) (or adds `namespace igs = igs_b200;` in a
// translation unit that only uses the hot-path API).  The types --
// GaussianSet, ImageBuffer, PixelSample, GaussianGrad, AdamState,
// LearningRates, BspPartition-like handles, igs::Error -- are the
// reference's; only the implementation moves to the GPU.  Errors come back
// as igs::Error with the reference's ErrorKind and message.
//
// Link: -ligs_b200 (paper_2407_01866_b200/libigs_b200.so); needs only the
// reference's headers, not its library.
#pragma once

#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "igs/adam.hpp"
#include "igs/error.hpp"
#include "igs/fit.hpp"
#include "igs/gaussian.hpp"
#include "igs/image.hpp"
#include "igs/renderer.hpp"
#include "igs_b200.h"

namespace igs_b200 {

static_assert(sizeof(igs::Gaussian2D) == 64, "Gaussian2D must be 8 packed doubles");
static_assert(sizeof(igs::GaussianGrad) == 64, "GaussianGrad must be 8 packed doubles");
static_assert(sizeof(igs::PixelSample) == 40, "PixelSample must be 5 packed doubles");

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

// bsp.hpp:80-88 render_image_blocked through a partition built with
// build_partition(set, n_max) on the device (the partition stays resident).
inline igs::ImageBuffer render_image_blocked(const igs::GaussianSet& set, int n_max, int width, int height, int k,
                                             Device& dev = default_device()) {
    dev.upload(set);
    dev.check(igs_partition_build(dev.get(), n_max));
    igs::ImageBuffer img(width, height);
    dev.check(igs_render_image_blocked(dev.get(), width, height, k, img.data().data()));
    return img;
}

// fit.hpp:63-64 fit(target, config, on_checkpoint)
inline std::pair<igs::GaussianSet, std::string> fit(const igs::ImageBuffer& target, const igs::FitConfig& c,
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
    std::string log(1 << 20, '\0');
    int n_evals = 0, decay = -1, final_count = 0;
    dev.check(igs_fit(dev.get(), target.data().data(), target.width(), target.height(), &cfg, nullptr, nullptr,
                      nullptr, 0, &n_evals, &decay, &final_count, log.data(), log.size()));
    log.resize(std::strlen(log.c_str()));
    igs::GaussianSet set;
    set.gaussians.resize(static_cast<size_t>(final_count));
    dev.check(igs_get_params(dev.get(), reinterpret_cast<double*>(set.gaussians.data()),
                             static_cast<uint32_t>(final_count)));
    return {std::move(set), std::move(log)};
}

}  // namespace igs_b200
