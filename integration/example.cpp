// example.cpp -- the reference's own C++ API next to the drop-in wrapper on
// identical inputs.  igs::* resolves to the unmodified reference library
// (oracle/_ref/libigs_ref.so), igs_b200::* to the B200 library.  Exits 0
// when every comparison holds; prints one line per check.  Every check is
// bit-for-bit (the device reproduces the reference's arithmetic, libm
// included).
#include <cmath>
#include <cstdio>
#include <sstream>
#include <vector>

#include "igs/bsp.hpp"
#include "igs/codec.hpp"
#include "igs/metrics.hpp"
#include "igs/renderer.hpp"
#include "igs/rng.hpp"
#include "igs/sampling.hpp"
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

// photo-like: a ramp plus soft blobs (test_support.hpp's spirit)
static igs::ImageBuffer photo(int W, int H, uint64_t seed) {
    igs::Rng rng(seed);
    igs::ImageBuffer img(W, H);
    double cx[6], cy[6], r[6], col[6][3];
    for (int b = 0; b < 6; ++b) {
        cx[b] = rng.next_double();
        cy[b] = rng.next_double();
        r[b] = rng.next_range(0.05, 0.3);
        for (int c = 0; c < 3; ++c) col[b][c] = rng.next_double();
    }
    for (int h = 0; h < H; ++h)
        for (int w = 0; w < W; ++w) {
            const double u = (w + 0.5) / W, v = (h + 0.5) / H;
            igs::Color3 c{0.2 + 0.5 * u, 0.3 + 0.4 * v, 0.5};
            for (int b = 0; b < 6; ++b) {
                const double d2 = ((u - cx[b]) * (u - cx[b]) + (v - cy[b]) * (v - cy[b])) / (r[b] * r[b]);
                const double a = std::exp(-d2);
                c.r = c.r * (1 - a) + col[b][0] * a;
                c.g = c.g * (1 - a) + col[b][1] * a;
                c.b = c.b * (1 - a) + col[b][2] * a;
            }
            img.set_pixel(h, w, c);
        }
    return img;
}

static int failures = 0;
static void report(const char* what, bool ok) {
    std::printf("%-58s %s\n", what, ok ? "ok" : "FAIL");
    failures += ok ? 0 : 1;
}

static bool same_image(const igs::ImageBuffer& a, const igs::ImageBuffer& b) {
    return a.same_shape(b) && a.data() == b.data();
}

static bool same_set(const igs::GaussianSet& a, const igs::GaussianSet& b) {
    return a.size() == b.size() && std::memcmp(a.gaussians.data(), b.gaussians.data(), 64 * a.size()) == 0;
}

static bool same_rects(const std::vector<igs::Rect>& a, const std::vector<igs::Rect>& b) {
    return a.size() == b.size() && std::memcmp(a.data(), b.data(), sizeof(igs::Rect) * a.size()) == 0;
}

static bool same_partition(const igs::BspPartition& a, const igs::BspPartition& b) {
    bool ok = same_rects(a.blocks, b.blocks) && same_rects(a.shells, b.shells) &&
              a.block_members == b.block_members && a.shell_members == b.shell_members && a.n_max == b.n_max &&
              a.source_size == b.source_size && a.root == b.root && a.nodes.size() == b.nodes.size() &&
              a.grid_dim == b.grid_dim && a.grid_cells == b.grid_cells;
    for (size_t i = 0; ok && i < a.nodes.size(); ++i) {
        const igs::BspNode &x = a.nodes[i], &y = b.nodes[i];
        ok = x.axis == y.axis && x.line == y.line && x.low == y.low && x.high == y.high && x.block == y.block &&
             std::memcmp(&x.point_bbox, &y.point_bbox, sizeof(igs::Rect)) == 0;
    }
    return ok;
}

int main() {
    const igs::GaussianSet set = random_set(3000, 42, 0.005, 0.06);
    // ---- renderer.hpp
    report("render_image (global exact top-K)", same_image(igs::render_image(set, 160, 120, 10),
                                                            igs_b200::render_image(set, 160, 120, 10)));
    bool same = true;
    igs::Rng rng(7);
    for (int t = 0; t < 200; ++t) {
        const igs::PixelCoord x{rng.next_double(), rng.next_double()};
        const auto a = igs::select_top_k(set, x, 10), b = igs_b200::select_top_k(set, x, 10);
        same = same && a.indices == b.indices && a.weights == b.weights;
        const igs::Color3 ca = igs::render_topk(set, x, 10), cb = igs_b200::render_topk(set, x, 10);
        same = same && ca.r == cb.r && ca.g == cb.g && ca.b == cb.b;
    }
    report("select_top_k + render_topk (200 points)", same);
    std::vector<igs::PixelSample> samples(4000);
    for (auto& s : samples)
        s = {{rng.next_double(), rng.next_double()},
             {rng.next_range(-1, 1), rng.next_range(-1, 1), rng.next_range(-1, 1)}};
    const auto ga = igs::backward(set, samples, 10);
    const auto gb = igs_b200::backward(set, samples, 10);
    report("backward (8 parameters, bit-exact)", std::memcmp(ga.data(), gb.data(), 64 * ga.size()) == 0);
    // ---- adam.hpp
    igs::GaussianSet sa = set, sb = set;
    igs::AdamState ma, mb;
    igs::adam_step(sa, ga, ma, igs::LearningRates{}, 1);
    igs_b200::adam_step(sb, ga, mb, igs::LearningRates{}, 1);
    report("adam_step (bit-exact)", same_set(sa, sb) && ma.m == mb.m && ma.v == mb.v);
    // ---- bsp.hpp
    const igs::BspPartition pa = igs::build_partition(set, 64);
    const igs::BspPartition pb = igs_b200::build_partition(set, 64);
    report("build_partition (blocks, shells, members, tree, boxes)", same_partition(pa, pb));
    same = true;
    for (int t = 0; t < 100; ++t) {
        const igs::PixelCoord x{rng.next_double(), rng.next_double()};
        same = same && igs::locate_block(pa, x) == igs_b200::locate_block(pa, x);
        const igs::Color3 ca = igs::render_topk_blocked(set, pa, x, 10);
        const igs::Color3 cb = igs_b200::render_topk_blocked(set, pa, x, 10);
        same = same && ca.r == cb.r && ca.g == cb.g && ca.b == cb.b;
    }
    report("locate_block + render_topk_blocked (100 points)", same);
    report("render_image_blocked(set, partition, ...)", same_image(igs::render_image_blocked(set, pa, 160, 120, 10),
                                                                   igs_b200::render_image_blocked(set, pa, 160, 120,
                                                                                                  10)));
    const igs::BspPartition ra = igs::rebuild_partition(pa.blocks, set);
    const igs::BspPartition rb = igs_b200::rebuild_partition(pa.blocks, set);
    report("rebuild_partition (grid locator, members)", same_partition(ra, rb));
    // ---- sampling.hpp / metrics.hpp
    const igs::ImageBuffer target = photo(96, 72, 11);
    const igs::ImageBuffer rendered = igs::render_image(set, 96, 72, 10);
    report("init_distribution", igs::init_distribution(target, 0.3).p == igs_b200::init_distribution(target, 0.3).p);
    report("add_distribution", igs::add_distribution(rendered, target).p ==
                                   igs_b200::add_distribution(rendered, target).p);
    igs::Rng r1(99), r2(99);
    const igs::GaussianSet ia = igs::initialize_set(target, 500, 0.3, r1);
    const igs::GaussianSet ib = igs_b200::initialize_set(target, 500, 0.3, r2);
    report("initialize_set (and the caller's Rng advances alike)", same_set(ia, ib) && r1.next_u64() == r2.next_u64());
    report("psnr", igs::psnr(rendered, target) == igs_b200::psnr(rendered, target));
    report("ssim", igs::ssim(rendered, target) == igs_b200::ssim(rendered, target));
    // ---- codec.hpp
    report("quantize_set", same_set(igs::quantize_set(set), igs_b200::quantize_set(set)));
    const std::vector<uint8_t> fa = igs::encode(set, &pa, 160, 120, 10);
    report("encode (IGS2 bytes, with partition)", fa == igs_b200::encode(set, &pa, 160, 120, 10));
    const igs::Decoded da = igs::decode(fa), db = igs_b200::decode(fa);
    report("decode (set, header, rebuilt partition)",
           same_set(da.set, db.set) && da.width == db.width && da.height == db.height && da.k == db.k &&
               da.partition.has_value() == db.partition.has_value() && same_partition(*da.partition, *db.partition));
    // ---- fit.hpp
    igs::FitConfig cfg;
    cfg.budget = 96;
    cfg.iterations = 200;
    cfg.samples_per_iter = 2000;
    cfg.eval_interval = 40;
    cfg.warmup_iters = 60;
    cfg.densify_interval = 40;
    cfg.seed = 3;
    cfg.plateau_patience = 2;
    std::vector<std::string> ids_a, ids_b;
    std::vector<size_t> sizes_a, sizes_b;
    const auto [fs_a, rep_a] = igs::fit(target, cfg, [&](int, int, const std::string& id, const igs::GaussianSet& s) {
        ids_a.push_back(id);
        sizes_a.push_back(s.size());
    });
    const auto [fs_b, rep_b] = igs_b200::fit(target, cfg, [&](int, int, const std::string& id,
                                                              const igs::GaussianSet& s) {
        ids_b.push_back(id);
        sizes_b.push_back(s.size());
    });
    std::ostringstream la, lb;
    rep_a.write(la, cfg);
    rep_b.write(lb, cfg);
    report("fit (final set, FitReport log, CheckpointFn calls)",
           same_set(fs_a, fs_b) && la.str() == lb.str() && ids_a == ids_b && sizes_a == sizes_b &&
               rep_a.final_count == rep_b.final_count && rep_a.lr_decay_iteration == rep_b.lr_decay_iteration);
    // ---- errors keep the reference's kind
    try {
        igs_b200::render_image(igs::GaussianSet{}, 8, 8, 10);
        report("empty set raises igs::Error(empty_set)", false);
    } catch (const igs::Error& e) {
        report("empty set raises igs::Error(empty_set)", e.kind() == igs::ErrorKind::empty_set);
    }
    try {
        igs::GaussianSet stale = set;
        stale.gaussians.pop_back();
        igs_b200::render_image_blocked(stale, pa, 16, 16, 10);
        report("stale partition raises igs::Error(invalid_parameter)", false);
    } catch (const igs::Error& e) {
        report("stale partition raises igs::Error(invalid_parameter)", e.kind() == igs::ErrorKind::invalid_parameter);
    }
    return failures;
}
