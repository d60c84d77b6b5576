// igs_math.cuh -- correctly-rounded double sin/cos for the prepare step.
//
// The reference caches cos(theta), sin(theta) per Gaussian with glibc libm
// (renderer.cpp:41-42, gcc merges them into one sincos call).  Every
// squared Mahalanobis distance q -- and therefore every top-K ranking -- is
// built from those two doubles, so the device must reproduce them bit for
// bit.  CUDA's sin/cos carry up to 2 ulp of error; glibc 2.39's are within
// ~0.55 ulp and almost always correctly rounded.  We therefore evaluate
// sin/cos in double-double arithmetic (Cody-Waite reduction by pi/2 with a
// 3-part constant, degree-27 Taylor series in double-double) and round once,
// which is correctly rounded except on astronomically rare hard cases.
// tests/test_math_host.py checks this exact code (compiled for the host)
// against glibc on millions of angles.
//
// Host+device so the same source is testable on the CPU.  Must be compiled
// without FMA contraction (nvcc -fmad=false, gcc -ffp-contract=off): every
// fused op below is an explicit fma().
#pragma once
#include <math.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define IGS_HD __host__ __device__ __forceinline__
#else
#define IGS_HD static inline
#endif

namespace igs_math {

struct dd {
    double hi, lo;
};

IGS_HD dd two_sum(double a, double b) {
    const double s = a + b;
    const double bb = s - a;
    const double e = (a - (s - bb)) + (b - bb);
    return {s, e};
}
IGS_HD dd quick_two_sum(double a, double b) {
    const double s = a + b;
    return {s, b - (s - a)};
}
IGS_HD dd two_prod(double a, double b) {
    const double p = a * b;
    return {p, fma(a, b, -p)};
}
IGS_HD dd dd_add(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi);
    dd t = two_sum(a.lo, b.lo);
    s.lo += t.hi;
    s = quick_two_sum(s.hi, s.lo);
    s.lo += t.lo;
    return quick_two_sum(s.hi, s.lo);
}
IGS_HD dd dd_mul(dd a, dd b) {
    dd p = two_prod(a.hi, b.hi);
    p.lo += a.hi * b.lo + a.lo * b.hi;
    return quick_two_sum(p.hi, p.lo);
}
IGS_HD dd dd_mul_d(dd a, double b) {
    dd p = two_prod(a.hi, b);
    p.lo += a.lo * b;
    return quick_two_sum(p.hi, p.lo);
}

// Inverse factorials 1/n! as double-double (hi, lo), n = 0..27.
// Generated with exact rational arithmetic (tests/test_math_host.py
// regenerates and compares them).
#define IGS_INV_FACT_TABLE \
    {1.0, 0.0}, \
    {1.0, 0.0}, \
    {0.5, 0.0}, \
    {0.16666666666666666, 9.25185853854297e-18}, \
    {0.041666666666666664, 2.3129646346357427e-18}, \
    {0.008333333333333333, 1.1564823173178714e-19}, \
    {0.001388888888888889, -5.300543954373577e-20}, \
    {0.0001984126984126984, 1.7209558293420705e-22}, \
    {2.48015873015873e-05, 2.1511947866775882e-23}, \
    {2.7557319223985893e-06, -1.858393274046472e-22}, \
    {2.755731922398589e-07, 2.3767714622250297e-23}, \
    {2.505210838544172e-08, -1.448814070935912e-24}, \
    {2.08767569878681e-09, -1.20734505911326e-25}, \
    {1.6059043836821613e-10, 1.2585294588752098e-26}, \
    {1.1470745597729725e-11, 2.0655512752830745e-28}, \
    {7.647163731819816e-13, 7.03872877733453e-30}, \
    {4.779477332387385e-14, 4.399205485834081e-31}, \
    {2.8114572543455206e-15, 1.6508842730861433e-31}, \
    {1.5619206968586225e-16, 1.1910679660273754e-32}, \
    {8.22063524662433e-18, 2.2141894119604265e-34}, \
    {4.110317623312165e-19, 1.4412973378659527e-36}, \
    {1.9572941063391263e-20, -1.3643503830087908e-36}, \
    {8.896791392450574e-22, -7.911402614872376e-38}, \
    {3.868170170630684e-23, -8.843177655482344e-40}, \
    {1.6117375710961184e-24, -3.6846573564509766e-41}, \
    {6.446950284384474e-26, -1.9330404233703465e-42}, \
    {2.4795962632247976e-27, -1.2953730964765229e-43}, \
    {9.183689863795546e-29, 1.4303150396787322e-45}

// pi/2 split: P1 has 33 significant bits so k*P1 is exact for |k| < 2^20;
// P2 and P3 carry the next bits (fdlibm's pio2_1/pio2_1t style).
#define IGS_PIO2_1 1.57079632673412561417e+00
#define IGS_PIO2_2 6.07710050630396597660e-11
#define IGS_PIO2_3 2.02226624879595063154e-21
#define IGS_2_OVER_PI 6.36619772367581382433e-01

// Reduce x to r = x - k*pi/2 in double-double.  Valid for |x| < 2^19.
IGS_HD dd reduce_pio2(double x, int* quadrant) {
    const double kd = rint(x * IGS_2_OVER_PI);
    // k*P1 exact; x - k*P1 exact by Sterbenz for the reduced range.
    const double r1 = x - kd * IGS_PIO2_1;
    dd t = two_prod(kd, IGS_PIO2_2);
    dd r = two_sum(r1, -t.hi);
    r.lo -= t.lo;
    dd t3 = two_prod(kd, IGS_PIO2_3);
    r.lo -= t3.hi;
    r = quick_two_sum(r.hi, r.lo);
    *quadrant = ((int)(long long)kd) & 3;
    return r;
}

// sin(r), cos(r) for |r| <= ~pi/4 in double-double (Taylor, Horner).
IGS_HD void dd_sincos_reduced(dd r, dd* s, dd* c) {
    const dd inv_fact[28] = {IGS_INV_FACT_TABLE};
    const dd r2 = dd_mul(r, r);
    // sin: r * sum_{j=0..13} (-1)^j r^{2j} / (2j+1)!
    dd ps = inv_fact[27];
    for (int j = 12; j >= 0; --j) {
        ps = dd_mul(ps, r2);
        ps = {-ps.hi, -ps.lo};
        ps = dd_add(ps, inv_fact[2 * j + 1]);
    }
    *s = dd_mul(ps, r);
    // cos: sum_{j=0..13} (-1)^j r^{2j} / (2j)!
    dd pc = inv_fact[26];
    for (int j = 12; j >= 0; --j) {
        pc = dd_mul(pc, r2);
        pc = {-pc.hi, -pc.lo};
        pc = dd_add(pc, inv_fact[2 * j]);
    }
    *c = pc;
}

// dd + dd where |a| >= |b| is known (Horner steps c_k + z*S with the
// coefficient dominating): cheaper than the general dd_add.
IGS_HD dd dd_add_big(dd a, dd b) {
    const double s = a.hi + b.hi;
    const double e = ((a.hi - s) + b.hi) + (a.lo + b.lo);
    return quick_two_sum(s, e);
}

// Fast path (Ziv): sin(r), cos(r) for the reduced r with the three leading
// Taylor coefficients in double-double and the tail -- below 2^-14 (sin) /
// 2^-18 (cos) of the result -- in double.  The evaluation error is below
// 2^-66 relative (largest seen against the full series over 2M angles:
// 2^-70 for cos, 2^-73 for sin); the doubles are accepted only when
// rounding is the same at both ends of a 2^-65 relative interval,
// otherwise (about 1 in 2^11 values) the caller runs the full series.
IGS_HD bool fast_sincos_reduced(dd r, double* sh_out, double* ch_out) {
    const dd z = dd_mul(r, r);
    const double zd = z.hi;
    // sin(r) = r (1 + z P),  P = -1/3! + z/5! - z^2/7! + z^3 Ts
    double ts = -3.868170170630684e-23;  // -1/23!
    ts = ts * zd + 1.9572941063391263e-20;   // 1/21!
    ts = ts * zd - 8.22063524662433e-18;     // -1/19!
    ts = ts * zd + 2.8114572543455206e-15;   // 1/17!
    ts = ts * zd - 7.647163731819816e-13;    // -1/15!
    ts = ts * zd + 1.6059043836821613e-10;   // 1/13!
    ts = ts * zd - 2.505210838544172e-08;    // -1/11!
    ts = ts * zd + 2.7557319223985893e-06;   // 1/9!
    dd ps = dd_add_big(dd{-0.0001984126984126984, -1.7209558293420705e-22}, two_prod(zd, ts));  // -1/7!
    ps = dd_add_big(dd{0.008333333333333333, 1.1564823173178714e-19}, dd_mul(z, ps));          // 1/5!
    ps = dd_add_big(dd{-0.16666666666666666, -9.25185853854297e-18}, dd_mul(z, ps));           // -1/3!
    const dd s = dd_add(r, dd_mul(r, dd_mul(z, ps)));
    // cos(r) = 1 + z Q,  Q = -1/2! + z/4! - z^2/6! + z^3 Tc
    double tc = 1.6117375710961184e-24;      // 1/24!
    tc = tc * zd - 8.896791392450574e-22;    // -1/22!
    tc = tc * zd + 4.110317623312165e-19;    // 1/20!
    tc = tc * zd - 1.5619206968586225e-16;   // -1/18!
    tc = tc * zd + 4.779477332387385e-14;    // 1/16!
    tc = tc * zd - 1.1470745597729725e-11;   // -1/14!
    tc = tc * zd + 2.08767569878681e-09;     // 1/12!
    tc = tc * zd - 2.755731922398589e-07;    // -1/10!
    tc = tc * zd + 2.48015873015873e-05;     // 1/8!
    dd pc = dd_add_big(dd{-0.001388888888888889, 5.300543954373577e-20}, two_prod(zd, tc));    // -1/6!
    pc = dd_add_big(dd{0.041666666666666664, 2.3129646346357427e-18}, dd_mul(z, pc));         // 1/4!
    pc = dd_add_big(dd{-0.5, 0.0}, dd_mul(z, pc));                                            // -1/2!
    const dd c = dd_add_big(dd{1.0, 0.0}, dd_mul(z, pc));
    // rounding test at +-2^-65 relative
    const double es = fabs(s.hi) * 0x1p-65, ec = fabs(c.hi) * 0x1p-65;
    const double s0 = s.hi + (s.lo - es), s1 = s.hi + (s.lo + es);
    const double c0 = c.hi + (c.lo - ec), c1 = c.hi + (c.lo + ec);
    *sh_out = s0;
    *ch_out = c0;
    return s0 == s1 && c0 == c1;
}

// Correctly rounded (except on hard cases) sin and cos of x.
IGS_HD void cr_sincos(double x, double* sin_out, double* cos_out) {
    if (!(fabs(x) < 524288.0)) {  // huge or non-finite: libm semantics
        *sin_out = sin(x);
        *cos_out = cos(x);
        return;
    }
    if (x == 0.0) {  // keeps sin(-0) = -0
        *sin_out = x;
        *cos_out = 1.0;
        return;
    }
    int q;
    const dd r = reduce_pio2(x, &q);
    double sh, ch;
    if (!fast_sincos_reduced(r, &sh, &ch)) {
        dd s, c;
        dd_sincos_reduced(r, &s, &c);
        sh = s.hi + s.lo;
        ch = c.hi + c.lo;
    }
    switch (q) {
        case 0: *sin_out = sh; *cos_out = ch; break;
        case 1: *sin_out = ch; *cos_out = -sh; break;
        case 2: *sin_out = -sh; *cos_out = -ch; break;
        default: *sin_out = -ch; *cos_out = sh; break;
    }
}

// The full series only (tests compare the fast path against it).
IGS_HD void cr_sincos_full(double x, double* sin_out, double* cos_out) {
    if (!(fabs(x) < 524288.0) || x == 0.0) {
        cr_sincos(x, sin_out, cos_out);
        return;
    }
    int q;
    const dd r = reduce_pio2(x, &q);
    dd s, c;
    dd_sincos_reduced(r, &s, &c);
    const double sh = s.hi + s.lo, ch = c.hi + c.lo;
    switch (q) {
        case 0: *sin_out = sh; *cos_out = ch; break;
        case 1: *sin_out = ch; *cos_out = -sh; break;
        case 2: *sin_out = -sh; *cos_out = -ch; break;
        default: *sin_out = -ch; *cos_out = sh; break;
    }
}

// a / b correctly rounded, from y = RN(1/b) computed once for many a (the
// Adam bias corrections are per-step constants): q0 = a*y is within 1.5 ulp
// of a/b; one Markstein correction q + (a - b q) y brings it within 1 ulp,
// and a second one -- Markstein's theorem: y = RN(1/b) and q within 1 ulp
// => RN(q + r y) = RN(a/b) -- rounds correctly.  Requires normal operands
// away from the exponent limits (the caller checks 2^-960 <= |a| <= 2^1000,
// 2^-20 <= b <= 2^20); tests/test_math_host.py checks it against IEEE
// division on random, per-step and near-midpoint operands.
IGS_HD double div_by_recip(double a, double b, double y) {
    double q = a * y;
    double r = fma(-b, q, a);
    q = fma(r, y, q);
    r = fma(-b, q, a);
    return fma(r, y, q);
}

}  // namespace igs_math
