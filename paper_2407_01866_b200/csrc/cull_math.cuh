// cull_math.cuh -- the certified tile-culling predicate (kernel 2), shared by
// the device kernels (cull.cu) and restated op-for-op by the CPU oracle
// (the test-only C checker, orc_cull_lists) so tile lists compare
// bit-exactly.  Device-only; compiled with -fmad=false.
//
// The reference ranks ALL Gaussians at every pixel (renderer.cpp:168-176);
// there is no cutoff radius, so a plain 3-sigma screen is not exact.  Here a
// Gaussian g is a candidate of tile T iff qmin_lb(g, T) <= tau_T where
//   * tau_T   = the kk-th smallest qmax_ub(g', T) over any set of Gaussians
//               (the "seeds": centres in the 3x3, 5x5, ... tile neighbourhood)
//               -- for every pixel p of T those kk Gaussians have q <= tau_T,
//               so p's kk-th best q is <= tau_T;
//   * qmin_lb = a lower bound of the computed q(g, p) over every pixel centre
//               p of T: if it exceeds tau_T, g is strictly worse than p's
//               kk-th best at every p, hence in no pixel's top-K (no tie can
//               involve it).
// Both bounds are on the FLOATING-POINT q the scan computes (maha()), not on
// real-number q: E bounds |fl(q) - q| for points of the box (forward error
// analysis of renderer.cpp:17-23 gives 9u(ia+ib)L1^2; we use 64u), and a
// 2^-30 relative slack absorbs the rounding of the bound formulas.
#pragma once
#include <math.h>

#ifndef IGS_CULL_HD
#define IGS_CULL_HD __device__ __forceinline__
#endif

namespace igs_cull {

constexpr double kErrU = 64.0 * 1.1102230246251565e-16;   // 64 * 2^-53
constexpr double kSlackUp = 1.0 + 9.313225746154785e-10;  // 1 + 2^-30
constexpr double kSlackDn = 1.0 - 9.313225746154785e-10;  // 1 - 2^-30
constexpr double kPrune = 1.0 - 9.5367431640625e-07;      // 1 - 2^-20 (pyramid nodes)

struct G {
    double mx, my, c, s, ia, ib;  // ScanRec fields
    double A, B, C;               // conic Sigma^-1 = [[A, B], [B, C]]
};

// q exactly as the scan computes it (renderer.cpp:17-23, no FMA).
IGS_CULL_HD double q_at(const G& g, double x, double y) {
    const double dx = x - g.mx;
    const double dy = y - g.my;
    const double e1 = g.c * dx + g.s * dy;
    const double e2 = -g.s * dx + g.c * dy;
    return e1 * e1 * g.ia + e2 * e2 * g.ib;
}

IGS_CULL_HD void conic(G& g) {
    const double c2 = g.c * g.c, s2 = g.s * g.s, cs = g.c * g.s;
    g.A = c2 * g.ia + s2 * g.ib;
    g.B = cs * (g.ia - g.ib);
    g.C = s2 * g.ia + c2 * g.ib;
}

// Forward-error bound of fl(q) over the box: 64u (ia+ib) L1max^2.
IGS_CULL_HD double err_bound(const G& g, double x0, double x1, double y0, double y1) {
    const double ax = fmax(fabs(x0 - g.mx), fabs(x1 - g.mx));
    const double ay = fmax(fabs(y0 - g.my), fabs(y1 - g.my));
    const double l = ax + ay;
    return kErrU * (g.ia + g.ib) * l * l;
}

// Upper bound of fl(q) at every point of the box (convex: max at a corner).
IGS_CULL_HD double qmax_ub(const G& g, double x0, double x1, double y0, double y1) {
    const double a = q_at(g, x0, y0), b = q_at(g, x1, y0), c = q_at(g, x0, y1), d = q_at(g, x1, y1);
    const double m = fmax(fmax(a, b), fmax(c, d));
    return m * kSlackUp + 2.0 * err_bound(g, x0, x1, y0, y1);
}

// Lower bound of fl(q) at every point of the box.  If the centre is outside,
// the minimum lies on an edge facing it; on the edge x = xe the minimum over
// the whole line is ia*ib*dx^2 / C (det Sigma^-1 = ia*ib, no cancellation),
// and when the line optimum falls outside the segment the nearer corner
// gives a tighter value.
IGS_CULL_HD double qmin_lb(const G& g, double x0, double x1, double y0, double y1) {
    const bool in_x = g.mx >= x0 && g.mx <= x1;
    const bool in_y = g.my >= y0 && g.my <= y1;
    if (in_x && in_y) return 0.0;
    double best = __longlong_as_double(0x7ff0000000000000LL);
    const double det = g.ia * g.ib;
    if (!in_x) {
        const double xe = g.mx < x0 ? x0 : x1;
        const double dx = xe - g.mx;
        double v = (det * (dx * dx)) / g.C;
        const double ys = g.my - (g.B * dx) / g.C;
        if (ys < y0) v = fmax(v, q_at(g, xe, y0) * kSlackDn);
        else if (ys > y1) v = fmax(v, q_at(g, xe, y1) * kSlackDn);
        best = fmin(best, v);
    }
    if (!in_y) {
        const double ye = g.my < y0 ? y0 : y1;
        const double dy = ye - g.my;
        double v = (det * (dy * dy)) / g.A;
        const double xs = g.mx - (g.B * dy) / g.A;
        if (xs < x0) v = fmax(v, q_at(g, x0, ye) * kSlackDn);
        else if (xs > x1) v = fmax(v, q_at(g, x1, ye) * kSlackDn);
        best = fmin(best, v);
    }
    const double lb = best * kSlackDn - 2.0 * err_bound(g, x0, x1, y0, y1);
    return lb > 0.0 ? lb : 0.0;
}

}  // namespace igs_cull
