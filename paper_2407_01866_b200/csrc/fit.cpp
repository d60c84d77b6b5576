// fit.cpp -- the encoder loop (fit.cpp:116-207 of the reference) as native
// host code driving the device through the C-ABI.
//
// Host side (exactly the reference's arithmetic and RNG order, compiled with
// -ffp-contract=off): std::mt19937_64 with rng.hpp's draw helpers, the Sobel
// / mixture init distribution (sampling.cpp:14-75), Walker/Vose alias tables
// (sampling.cpp:96-133), initialize_set (:154-174), the schedule, plateau
// LR decay, densification appends and the log format.
// Device side: every train iteration (exact top-K + loss + backward + Adam),
// the evaluation renders (BSP partition with n_max = 64 + blocked raster,
// fit.cpp:34-37), PSNR, SSIM and the Eq. 8 error map.
//
// Pipelining: iteration t's sample indices are drawn before it is launched;
// while the device runs iteration t the host draws iteration t+1's samples
// -- unless iteration t evaluates or densifies, in which case the host waits,
// does that work first and then draws (the reference's RNG order: samples_t,
// densification draws at t, samples_{t+1}).
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "igs_b200.h"

// ctx.cu: records the message returned by igs_last_error
extern "C" int igs_internal_fail(igs_ctx* ctx, int code, const char* msg);
extern "C" int igs_internal_set_sampler(igs_ctx* ctx, const double* prob, const uint32_t* alias, uint64_t n);
extern "C" void igs_internal_ranks(const igs_ctx* ctx, int* rank, int* nranks);
extern "C" int igs_internal_eval_render(igs_ctx* ctx, int W, int H, int k);
extern "C" int igs_internal_train_iteration_async_raw(igs_ctx* ctx, const unsigned long long* raw2, uint32_t ns,
                                                      int k, const double* lr4, long long t);

namespace {

// rng.hpp:11-28
struct Rng {
    std::mt19937_64 e;
    explicit Rng(uint64_t seed) : e(seed) {}
    double next_double() { return (e() >> 11) * 0x1.0p-53; }
    uint64_t next_index(uint64_t n) { return e() % n; }
};

// sampling.cpp:14-23
template <class V>
double kahan_sum(const V& v) {
    double sum = 0.0, comp = 0.0;
    for (double x : v) {
        const double y = x - comp;
        const double t = sum + y;
        comp = (t - sum) - y;
        sum = t;
    }
    return sum;
}

// Runs f(begin, end) over [0, n) on the host's cores (per-element work with
// no cross-element arithmetic, so the split does not change any result).
// A vector whose resize leaves new elements uninitialised (they are
// written by the caller, in parallel -- which also spreads the first-touch
// page faults of a fresh 32 MB table over the host's cores).
template <class T>
struct NoInit : std::allocator<T> {
    template <class U>
    struct rebind {
        using other = NoInit<U>;
    };
    NoInit() = default;
    template <class U>
    NoInit(const NoInit<U>&) {}
    template <class U>
    void construct(U* p) noexcept {
        ::new (static_cast<void*>(p)) U;
    }
    template <class U, class... A>
    void construct(U* p, A&&... a) {
        ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
    }
};
template <class T>
using fast_vector = std::vector<T, NoInit<T>>;

size_t parallel_parts(size_t n) {
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    return std::min<size_t>(hw, std::max<size_t>(1, n / 65536));
}

// f(part, begin, end) over parallel_parts(n) contiguous parts of [0, n)
template <class F>
void parallel_parts_for(size_t n, F f) {
    const size_t parts = parallel_parts(n);
    const size_t step = (n + parts - 1) / parts;
    if (parts <= 1) {
        f((size_t)0, (size_t)0, n);
        return;
    }
    std::vector<std::thread> th;
    for (size_t p = 1; p < parts; ++p) th.emplace_back(f, p, std::min(n, p * step), std::min(n, (p + 1) * step));
    f((size_t)0, (size_t)0, std::min(n, step));
    for (auto& t : th) t.join();
}

template <class F>
void parallel_for(size_t n, F f) {
    parallel_parts_for(n, [&](size_t, size_t b, size_t e) { f(b, e); });
}

}  // namespace

// sampling.cpp:84-93 add_distribution's normalisation: Kahan total in index
// order, then v *= 1/total (elementwise, any split), uniform when zero.
extern "C" void igs_internal_kahan_normalize(double* p, size_t n) {
    double sum = 0.0, comp = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double y = p[i] - comp;
        const double t = sum + y;
        comp = (t - sum) - y;
        sum = t;
    }
    if (sum > 0.0) {
        const double inv = 1.0 / sum;
        parallel_for(n, [&](size_t b, size_t e) {
            for (size_t i = b; i < e; ++i) p[i] *= inv;
        });
    } else {
        const double u = 1.0 / (double)n;
        for (size_t i = 0; i < n; ++i) p[i] = u;
    }
}

namespace {
template <class V>
fast_vector<double> gradient_mixture(const V& mag, double total, double lambda);
}  // namespace

// sampling.cpp:25-40 gradient_mixture from a magnitude table (in place
// allowed): Kahan total in index order, then the elementwise mixture.
extern "C" void igs_internal_gradient_mixture(const double* mag, size_t n, double lambda, double* p) {
    std::vector<double> m(mag, mag + n);
    const fast_vector<double> q = gradient_mixture(m, kahan_sum(m), lambda);
    std::memcpy(p, q.data(), n * sizeof(double));
}

namespace {

// sampling.cpp:25-40 gradient_mixture (init_distribution / opt_distribution)
// from a precomputed gradient magnitude and its Kahan total: the init and
// optimisation distributions share both (only lambda differs), so the
// Sobel pass and the sum run once.
template <class V>
fast_vector<double> gradient_mixture(const V& mag, double total, double lambda) {
    fast_vector<double> q(mag.size());
    const double uniform = 1.0 / (double)q.size();
    const double scale = total > 0.0 ? (1.0 - lambda) / total : 0.0;
    parallel_for(q.size(), [&](size_t b, size_t e) {  // (elementwise: any split)
        for (size_t i = b; i < e; ++i) q[i] = total > 0.0 ? mag[i] * scale + lambda * uniform : uniform;
    });
    return q;
}

// sampling.cpp:96-133 Walker/Vose table; draw = index, then coin.  The
// scratch (scaled weights, the two stacks) and the table's own vectors are
// reused from build to build: at 4M entries a fresh ~110 MB costs more in
// first-touch page faults than the table itself.
struct AliasScratch {
    fast_vector<double> scaled;
    fast_vector<uint32_t> small, large;
    std::vector<size_t> part_small;  // per part: small entries (then their offsets)
};

struct Alias {
    fast_vector<double> prob;
    fast_vector<uint32_t> alias;
    bool ok = false;

    Alias() = default;
    template <class V>
    explicit Alias(const V& w) {
        AliasScratch S;
        build(w.data(), w.size(), S);
    }
    template <class V>
    void build(const V& w, AliasScratch& S) {
        build(w.data(), w.size(), S);
    }
    void build(const double* w, size_t n, AliasScratch& S) {
        ok = false;
        if (n == 0) return;
        // the Kahan total in index order (and, in the same pass, the
        // reference's check for negative weights -- which fails either way)
        double total = 0.0, comp = 0.0;
        bool neg = false;
        for (size_t i = 0; i < n; ++i) {
            const double x = w[i];
            neg |= x < 0.0;
            const double y = x - comp;
            const double t = total + y;
            comp = (t - total) - y;
            total = t;
        }
        if (!(total > 0.0) || neg) return;
        // (every prob entry is written below; alias stays 0 where prob = 1)
        prob.resize(n);
        alias.resize(n);
        S.scaled.resize(n);
        S.small.resize(n);
        S.large.resize(n);
        parallel_for(n, [&](size_t b, size_t e) {
            std::memset(alias.data() + b, 0, (e - b) * sizeof(uint32_t));
            std::memset(prob.data() + b, 0, (e - b) * sizeof(double));
        });
        // scaled weights and the small / large stacks in index order: a
        // stable partition (per-part counts, offsets, then each part writes
        // its own range -- the order of a sequential pass)
        const size_t parts = parallel_parts(n);
        S.part_small.assign(parts + 1, 0);
        parallel_parts_for(n, [&](size_t p, size_t b, size_t e) {
            size_t k = 0;
            for (size_t i = b; i < e; ++i) {
                S.scaled[i] = w[i] * n / total;
                k += S.scaled[i] < 1.0;
            }
            S.part_small[p + 1] = k;
        });
        for (size_t p = 0; p < parts; ++p) S.part_small[p + 1] += S.part_small[p];
        parallel_parts_for(n, [&](size_t p, size_t b, size_t e) {
            size_t ks = S.part_small[p], kl = b - S.part_small[p];
            for (size_t i = b; i < e; ++i) {
                if (S.scaled[i] < 1.0)
                    S.small[ks++] = (uint32_t)i;
                else
                    S.large[kl++] = (uint32_t)i;
            }
        });
        size_t ns = S.part_small[parts], nl = n - ns;
        // Vose's loop, the reference's stack order: pop s and l; l takes
        // s's deficit and goes back on top of the small or large stack.
        // The large item stays in a register while it remains large (it
        // would be popped again at once).
        double* scaled = S.scaled.data();
        uint32_t* small = S.small.data();
        uint32_t* large = S.large.data();
        while (ns > 0 && nl > 0) {
            uint32_t l = large[--nl];
            double sl = scaled[l];
            for (;;) {
                const uint32_t s = small[--ns];
                prob[s] = scaled[s];
                alias[s] = l;
                sl = (sl + scaled[s]) - 1.0;
                if (sl < 1.0) {
                    scaled[l] = sl;
                    small[ns++] = l;  // l is the next s
                    break;
                }
                if (ns == 0) {  // l stays large, the loop ends
                    scaled[l] = sl;
                    large[nl++] = l;
                    break;
                }
            }
        }
        for (size_t j = 0; j < nl; ++j) prob[large[j]] = 1.0;
        for (size_t j = 0; j < ns; ++j) prob[small[j]] = 1.0;
        ok = true;
    }
    uint32_t sample(Rng& r) const {
        const size_t i = (size_t)r.next_index(prob.size());
        return r.next_double() < prob[i] ? (uint32_t)i : alias[i];
    }
};

void add_gaussian(std::vector<double>& out, const float* img, int W, int H, uint32_t flat, double s0) {
    const int h = (int)flat / W, w = (int)flat % W;
    out.push_back((w + 0.5) / W);  // pixel_center (image.hpp:18-20)
    out.push_back((h + 0.5) / H);
    out.push_back(0.0);
    out.push_back(s0);
    out.push_back(s0);
    out.push_back((double)img[((size_t)h * W + w) * 3]);
    out.push_back((double)img[((size_t)h * W + w) * 3 + 1]);
    out.push_back((double)img[((size_t)h * W + w) * 3 + 2]);
}

struct Fail {
    int code;
};

}  // namespace

extern "C" {

// sampling.cpp:154-174 initialize_set(img, count, lambda, rng): the init
// distribution (device Sobel, the Kahan total and mixture here), the Vose
// table, and `count` draws that consume raw2[2j] (next_index) and
// raw2[2j + 1] (next_double) -- the caller's engine outputs, in order.
int igs_initialize_set(igs_ctx* ctx, const float* img, int W, int H, int count, double lambda,
                       const uint64_t* raw2, double* out8) {
    if (!ctx || !img || (count > 0 && (!raw2 || !out8))) return IGS_E_INVALID_PARAMETER;
    if (count < 1) return igs_internal_fail(ctx, IGS_E_INVALID_PARAMETER, "initialization count must be >= 1");
    std::vector<double> p((size_t)W * H);
    int e;
    if ((e = igs_gradient_mixture(ctx, img, W, H, lambda, p.data()))) return e;
    const Alias table(p);
    if (!table.ok) return igs_internal_fail(ctx, IGS_E_INVALID_PARAMETER, "alias table weights must have positive sum");
    std::vector<double> set;
    set.reserve((size_t)count * 8);
    const double s0 = 2.0 / std::max(W, H);
    for (int j = 0; j < count; ++j) {
        const size_t i = (size_t)(raw2[2 * (size_t)j] % table.prob.size());
        const double coin = (double)(raw2[2 * (size_t)j + 1] >> 11) * 0x1.0p-53;
        add_gaussian(set, img, W, H, coin < table.prob[i] ? (uint32_t)i : table.alias[i], s0);
    }
    std::memcpy(out8, set.data(), set.size() * sizeof(double));
    return IGS_OK;
}

void igs_fit_config_default(igs_fit_config* c) {
    c->budget = 0;
    c->k = 10;
    c->lambda_init = 0.3;
    c->lambda_opt = 0.8;
    c->iterations = 50000;
    c->samples_per_iter = 10000;
    c->lr[0] = 2e-4;  // mu
    c->lr[1] = 2e-3;  // color
    c->lr[2] = 1e-3;  // scale
    c->lr[3] = 1e-3;  // theta
    c->eval_interval = 1000;
    c->plateau_patience = 3;
    c->lr_decay = 0.1;
    c->warmup_iters = 10000;
    c->densify_interval = 5000;
    c->seed = 0;
    c->compute_ssim = 1;
}

int igs_fit(igs_ctx* ctx, const float* target, int W, int H, const igs_fit_config* cfg, igs_checkpoint_fn cb,
            void* user, igs_eval_record* evals, int max_evals, int* n_evals, int* lr_decay_iteration,
            int* final_count, char* log, size_t log_cap) {
    if (!ctx || !cfg || !target) return IGS_E_INVALID_PARAMETER;
    const igs_fit_config& c = *cfg;
    // fit.cpp:19-29 validate (messages are the reference's; see igs_last_error)
    auto bad = [&](const char* msg) { return igs_internal_fail(ctx, IGS_E_INVALID_PARAMETER, msg); };
    if (c.budget < 8) return bad("budget must be >= 8");
    if (c.k < 1) return bad("k must be >= 1");
    if (c.lambda_init < 0.0 || c.lambda_init > 1.0 || c.lambda_opt < 0.0 || c.lambda_opt > 1.0)
        return bad("lambda values must lie in [0,1]");
    if (c.iterations < 1 || c.samples_per_iter < 1 || c.eval_interval < 1 || c.plateau_patience < 1 ||
        c.warmup_iters < 1 || c.densify_interval < 1)
        return bad("schedule counts must be >= 1");
    if (c.lr[0] <= 0.0 || c.lr[1] <= 0.0 || c.lr[2] <= 0.0 || c.lr[3] <= 0.0 || c.lr_decay <= 0.0)
        return bad("rates must be positive");
    if (W < 1 || H < 1) return bad("image dimensions must be positive");
    // multi-rank (a communicator attached): every rank runs this same driver
    // with the same config and target; rank r trains on samples
    // [r ns/R, (r+1) ns/R) of every iteration's draw, renders its band of the
    // evaluation image, and all host-side decisions are replicated
    int rank = 0, nranks = 1;
    igs_internal_ranks(ctx, &rank, &nranks);
    if (c.samples_per_iter % nranks) return bad("samples_per_iter must divide evenly over the ranks");

    int e;
    std::string text;
    char line[512];
    std::snprintf(line, sizeof(line),
                  "config budget=%d k=%d lambda_init=%.6g lambda_opt=%.6g iterations=%d samples=%d "
                  "lr_mu=%.6g lr_color=%.6g lr_scale=%.6g lr_theta=%.6g eval_interval=%d patience=%d "
                  "lr_decay=%.6g warmup=%d densify_interval=%d seed=%llu\n",
                  c.budget, c.k, c.lambda_init, c.lambda_opt, c.iterations, c.samples_per_iter, c.lr[0], c.lr[1],
                  c.lr[2], c.lr[3], c.eval_interval, c.plateau_patience, c.lr_decay, c.warmup_iters,
                  c.densify_interval, (unsigned long long)c.seed);
    text += line;

    // IGS_FIT_TRACE=1: wall time per phase on stderr (init, iterations,
    // evaluation renders, densification)
    const bool trace = std::getenv("IGS_FIT_TRACE") != nullptr;
    using clk = std::chrono::steady_clock;
    double t_init = 0, t_eval = 0, t_densify = 0, t_render = 0, t_metric = 0;
    const auto t_start = clk::now();
    auto since = [](clk::time_point a) { return std::chrono::duration<double, std::milli>(clk::now() - a).count(); };
    Rng rng(c.seed);
    // initialize_set(target, budget/2, lambda_init, rng) (sampling.cpp:154-174)
    const int init_count = c.budget / 2;
    std::vector<double> set;
    // image_gradient_magnitude on the device (sobel_kernel, bit-identical),
    // its Kahan total and the mixtures here
    auto mark = [&](const char* what, clk::time_point& t) {
        if (trace) std::fprintf(stderr, "igs_fit:   %s %.2f ms\n", what, since(t));
        t = clk::now();
    };
    AliasScratch alias_ws;  // shared by every table of the fit (see Alias)
    Alias add;              // the densification tables, one at a time
    auto tm = clk::now();
    if ((e = igs_set_target(ctx, target, W, H))) return e;
    fast_vector<double> mag((size_t)W * H);  // (written by igs_image_gradient_magnitude)
    if ((e = igs_image_gradient_magnitude(ctx, nullptr, W, H, mag.data()))) return e;
    mark("target + gradient magnitude", tm);
    const double mag_total = kahan_sum(mag);
    mark("kahan total", tm);
    // the optimisation table needs no engine output, so it is built on a
    // second host thread while the init table is built and drawn from
    Alias opt;
    AliasScratch opt_ws;
    std::thread opt_builder([&] { opt.build(gradient_mixture(mag, mag_total, c.lambda_opt), opt_ws); });
    struct Joiner {
        std::thread& t;
        ~Joiner() {
            if (t.joinable()) t.join();
        }
    } join_opt{opt_builder};
    {
        const fast_vector<double> mix = gradient_mixture(mag, mag_total, c.lambda_init);
        mark("init mixture", tm);
        Alias init;
        init.build(mix, alias_ws);
        mark("init alias table", tm);
        if (!init.ok) return bad("alias table weights must have positive sum");
        const double s0 = 2.0 / std::max(W, H);
        set.reserve((size_t)init_count * 8);
        for (int i = 0; i < init_count; ++i) add_gaussian(set, target, W, H, init.sample(rng), s0);
        mark("init draws", tm);
    }
    opt_builder.join();
    mark("opt mixture + alias table (join)", tm);
    if (!opt.ok) return bad("alias table weights must have positive sum");
    if ((e = igs_set_params(ctx, set.data(), (uint32_t)init_count))) return e;
    // the per-iteration draws from `opt` happen on the device (the host only
    // advances the engine): the table goes up once
    if ((e = igs_internal_set_sampler(ctx, opt.prob.data(), opt.alias.data(), opt.prob.size()))) return e;
    mark("set_params + sampler upload", tm);
    t_init = since(t_start);

    double lr[4] = {c.lr[0], c.lr[1], c.lr[2], c.lr[3]};
    bool decayed = false;
    int decay_iter = -1;
    double best_psnr = -std::numeric_limits<double>::infinity();
    int streak = 0;
    const double default_scale = 2.0 / std::max(W, H);
    const int add_count = c.budget / 8;
    int stage = 0;
    std::vector<igs_eval_record> recs;
    std::vector<std::string> checkpoints;
    fast_vector<double> dist((size_t)W * H);  // (written by igs_add_distribution)
    // one sample = opt.sample(rng) = next_index (one engine output) then
    // next_double (one more): the raw outputs, in that order
    std::vector<unsigned long long> cur(2 * (size_t)c.samples_per_iter), next(2 * (size_t)c.samples_per_iter);
    auto draw = [&](std::vector<unsigned long long>& s) {
        for (auto& v : s) v = rng.e();
    };
    const uint32_t ns = (uint32_t)(c.samples_per_iter / nranks);  // this rank's block
    const size_t raw0 = 2 * (size_t)rank * ns;                      // its first raw output
    auto emit_checkpoint = [&](int iteration) -> int {
        const uint32_t n = igs_num_gaussians(ctx);
        char id[64];
        std::snprintf(id, sizeof(id), "lod%d_iter%d_n%u", stage, iteration, n);
        checkpoints.push_back(id);
        if (cb) {
            std::vector<double> p((size_t)n * 8);
            int ee = igs_get_params(ctx, p.data(), n);
            if (ee) return ee;
            cb(user, stage, iteration, id, p.data(), n);
        }
        return IGS_OK;
    };
    // fit.cpp:34-37 render_current: build_partition(set, 64) + render_image_blocked
    // (band per rank + all-gather when there are several)
    auto render_current = [&]() -> int { return igs_internal_eval_render(ctx, W, H, c.k); };

    // drains an enqueued iteration after a failure, keeping the first error
    auto drain = [&](int code) {
        const std::string keep = igs_last_error(ctx);
        igs_train_wait(ctx, nullptr);
        return igs_internal_fail(ctx, code, keep.c_str());
    };
    // Iterations are pipelined two deep: while the device runs iteration t,
    // the host draws t+1's samples and enqueues it (unless t evaluates or
    // densifies, which needs the set after t), then waits on t.
    draw(cur);
    if (c.iterations >= 1 && (e = igs_internal_train_iteration_async_raw(ctx, cur.data() + raw0, ns, c.k, lr, 1))) return e;
    for (int iter = 1; iter <= c.iterations; ++iter) {
        const bool do_eval = iter % c.eval_interval == 0 || iter == c.iterations;
        const bool do_densify = stage < 4 && iter == c.warmup_iters + stage * c.densify_interval;
        double loss = 0.0;
        if (!do_eval && !do_densify) {
            if (iter < c.iterations) {
                draw(next);  // overlaps the device step
                if ((e = igs_internal_train_iteration_async_raw(ctx, next.data() + raw0, ns, c.k, lr, iter + 1)))
                    return drain(e);  // t is still outstanding
            }
            if ((e = igs_train_wait(ctx, &loss))) return iter < c.iterations ? drain(e) : e;  // t+1 outstanding
            std::swap(cur, next);
            continue;
        }
        if ((e = igs_train_wait(ctx, &loss))) return e;
        bool have_render = false;
        const auto t_post = clk::now();
        if (do_eval) {
            const auto t_r = clk::now();
            if ((e = render_current())) return e;
            igs_sync(ctx);
            t_render += since(t_r);
            if (trace) std::fprintf(stderr, "igs_fit: eval render at %d: %.2f ms\n", iter, since(t_r));
            const auto t_m = clk::now();
            have_render = true;
            double p = 0.0, s = 0.0;
            if ((e = igs_psnr(ctx, nullptr, W, H, &p))) return e;
            if (c.compute_ssim && (e = igs_ssim(ctx, nullptr, W, H, &s))) return e;
            t_metric += since(t_m);
            if (p >= best_psnr + 0.01) {
                best_psnr = p;
                streak = 0;
            } else {
                best_psnr = std::max(best_psnr, p);
                ++streak;
                if (!decayed && streak >= c.plateau_patience) {
                    for (double& v : lr) v *= c.lr_decay;  // LearningRates::scaled
                    decayed = true;
                    decay_iter = iter;
                }
            }
            recs.push_back({iter, (int)igs_num_gaussians(ctx), loss, p, s, best_psnr});
        }
        t_eval += since(t_post);
        const auto t_dens = clk::now();
        if (do_densify) {
            auto td = clk::now();
            if ((e = emit_checkpoint(iter))) return e;
            if (!have_render && (e = render_current())) return e;
            mark("densify: checkpoint + render", td);
            // add_distribution(rendered, target) on the device, Vose + draws here
            if ((e = igs_add_distribution(ctx, nullptr, W, H, dist.data()))) return e;
            mark("densify: add_distribution", td);
            add.build(dist, alias_ws);
            mark("densify: alias table", td);
            if (!add.ok) return bad("alias table weights must have positive sum");
            std::vector<double> fresh;
            fresh.reserve((size_t)add_count * 8);
            for (int a = 0; a < add_count; ++a) add_gaussian(fresh, target, W, H, add.sample(rng), default_scale);
            if (add_count > 0 && (e = igs_append_params(ctx, fresh.data(), (uint32_t)add_count))) return e;
            mark("densify: draws + append", td);
            ++stage;
        }
        t_densify += since(t_dens);
        if (iter < c.iterations) {
            draw(next);
            std::swap(cur, next);
            if ((e = igs_internal_train_iteration_async_raw(ctx, cur.data() + raw0, ns, c.k, lr, iter + 1))) return e;
        }
    }
    if ((e = emit_checkpoint(c.iterations))) return e;
    if (trace) {
        const double total = since(t_start);
        std::fprintf(stderr, "igs_fit: %.1f ms total: init %.1f, evaluation %.1f (render %.1f, metrics %.1f), "
                     "densification %.1f, iterations %.1f (%d)\n", total, t_init, t_eval, t_render, t_metric,
                     t_densify, total - t_init - t_eval - t_densify, c.iterations);
    }

    // FitReport::write (fit.cpp:209-231)
    for (const auto& r : recs) {
        std::snprintf(line, sizeof(line), "eval iter=%d n=%d loss=%.9e psnr=%.6f ssim=%.8f best=%.6f\n", r.iteration,
                      r.count, r.loss, r.psnr, r.ssim, r.best_psnr);
        text += line;
    }
    if (decay_iter >= 0) {
        std::snprintf(line, sizeof(line), "event lr_decay iter=%d\n", decay_iter);
        text += line;
    }
    for (const auto& id : checkpoints) text += "checkpoint id=" + id + "\n";
    const int fc = (int)igs_num_gaussians(ctx);
    text += "final n=" + std::to_string(fc) + "\n";

    if (evals) std::memcpy(evals, recs.data(), sizeof(igs_eval_record) * std::min<size_t>(recs.size(), max_evals));
    if (n_evals) *n_evals = (int)recs.size();
    if (lr_decay_iteration) *lr_decay_iteration = decay_iter;
    if (final_count) *final_count = fc;
    if (log && log_cap) {
        const size_t m = std::min(text.size(), log_cap - 1);
        std::memcpy(log, text.data(), m);
        log[m] = 0;
    }
    return IGS_OK;
}

}  // extern "C"
