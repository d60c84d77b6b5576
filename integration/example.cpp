// example.cpp -- the reference's own C++ API next to the drop-in wrapper on
// identical inputs.  igs::* resolves to the unmodified reference library
// (oracle/_ref/libigs_ref.so), igs_b200::* to the B200 library.  Exits 0
// when every comparison holds; prints one line per check.
#include <cmath>
#include <cstdio>
#include <vector>

#include "igs/bsp.hpp"
#include "igs/renderer.hpp"
#include "igs/rng.hpp"
#include "igs_b200.hpp"

static igs::GaussianSet random_set(size_t n, uint64_t seed, double smin, double smax) {
    igs::Rng rng(seed);
    igs::GaussianSet s;
    for (size_t i = 0; i < n; ++i) {
        igs::Gaussian2D g;
        g.mu = {rng.next_double(), rng.next_double()};
        g.theta = rng.next_range(0.0, 3.141592653589793);
        g.scale = {rng.next_range(smin, smax), rng.next_range(smin, smax)};
        g.color = {rng.next_double(), rng.next_double(), rng.next_double()};
        s.gaussians.push_back(g);
    }
    return s;
}

static int failures = 0;
static void report(const char* what, bool ok, double err) {
    std::printf("%-44s %s (max err %.3g)\n", what, ok ? "ok" : "FAIL", err);
    failures += ok ? 0 : 1;
}

int main() {
    const igs::GaussianSet set = random_set(3000, 42, 0.005, 0.06);
    // render_image
    const igs::ImageBuffer a = igs::render_image(set, 160, 120, 10);
    const igs::ImageBuffer b = igs_b200::render_image(set, 160, 120, 10);
    double err = 0;
    for (size_t i = 0; i < a.data().size(); ++i) err = std::max(err, (double)std::fabs(a.data()[i] - b.data()[i]));
    report("render_image (global exact top-K)", err <= 1e-4, err);
    // select_top_k
    bool same = true;
    igs::Rng rng(7);
    for (int t = 0; t < 200; ++t) {
        const igs::PixelCoord x{rng.next_double(), rng.next_double()};
        same = same && igs::select_top_k(set, x, 10).indices == igs_b200::select_top_k(set, x, 10).indices;
    }
    report("select_top_k indices (200 points)", same, same ? 0.0 : 1.0);
    // backward
    std::vector<igs::PixelSample> samples(4000);
    for (auto& s : samples)
        s = {{rng.next_double(), rng.next_double()},
             {rng.next_range(-1, 1), rng.next_range(-1, 1), rng.next_range(-1, 1)}};
    const auto ga = igs::backward(set, samples, 10);
    const auto gb = igs_b200::backward(set, samples, 10);
    err = 0;
    for (size_t i = 0; i < ga.size(); ++i) {
        const double* x = &ga[i].d_mu.x;
        const double* y = &gb[i].d_mu.x;
        for (int p = 0; p < 8; ++p) err = std::max(err, std::fabs(x[p] - y[p]) / std::max(1e-9, std::fabs(x[p])));
    }
    report("backward (relative, 8 parameters)", err <= 1e-9, err);
    // adam_step on identical gradients
    igs::GaussianSet sa = set, sb = set;
    igs::AdamState ma, mb;
    igs::adam_step(sa, ga, ma, igs::LearningRates{}, 1);
    igs_b200::adam_step(sb, ga, mb, igs::LearningRates{}, 1);
    same = std::memcmp(sa.gaussians.data(), sb.gaussians.data(), 64 * sa.size()) == 0 && ma.m == mb.m && ma.v == mb.v;
    report("adam_step (bit-exact)", same, same ? 0.0 : 1.0);
    // blocked render through a partition
    const igs::BspPartition part = igs::build_partition(set, 64);
    const igs::ImageBuffer c = igs::render_image_blocked(set, part, 160, 120, 10);
    const igs::ImageBuffer d = igs_b200::render_image_blocked(set, 64, 160, 120, 10);
    err = 0;
    for (size_t i = 0; i < c.data().size(); ++i) err = std::max(err, (double)std::fabs(c.data()[i] - d.data()[i]));
    report("render_image_blocked (n_max 64)", err <= 1e-4, err);
    // errors keep the reference's kind
    try {
        igs_b200::render_image(igs::GaussianSet{}, 8, 8, 10);
        report("empty set raises igs::Error(empty_set)", false, 1);
    } catch (const igs::Error& e) {
        report("empty set raises igs::Error(empty_set)", e.kind() == igs::ErrorKind::empty_set, 0);
    }
    return failures;
}
