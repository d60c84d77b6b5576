// glibc_math.cuh -- the reference's exp() and sincos(), bit for bit, on the device.
//
// The reference computes every blend weight and gradient weight with
// std::exp (renderer.cpp:80,98,145; gaussian.cpp:47,60) and caches
// cos(theta)/sin(theta) with std::cos/std::sin, which gcc merges into one
// sincos() call (renderer.cpp:40-41; the built library imports
// sincos@GLIBC_2.2.5 and exp@GLIBC_2.29).  On an x86-64 host with FMA and
// AVX2, glibc 2.39 binds both through IFUNC to FMA-compiled variants
// (__exp_fma, __sincos_fma) whose results differ from CUDA's exp/sincos --
// and from the correctly rounded value -- in the last ulp for some inputs.
// Any such ulp feeds q, the top-K ranking, the blend and the gradients, and
// over a 5,000-iteration fit it grows into a different trajectory.
//
// This header restates those two routines operation for operation,
// including which multiply-adds the FMA build fuses (read from the
// disassembly of libm.so.6, Ubuntu GLIBC 2.39-0ubuntu8.5: __exp_fma at
// 0x79b60, __sincos_fma at 0x7c2c0).  Algorithms (glibc, public):
//   exp    -- sysdeps/ieee754/dbl-64/e_exp.c (ARM optimized-routines):
//             x = k ln2/128 + r, 2^(k/128) from a 128-entry table,
//             degree-5 polynomial, specialcase() near over/underflow;
//   sincos -- sysdeps/ieee754/dbl-64/s_sincos.c + s_sin.c (IBM Accurate
//             Mathematical Library): |x| < 2^-27 -> (x, 1); |x| < 0.855469
//             -> do_sin/do_cos(x, 0); |x| < 2.426265 -> the pi/2 - |x|
//             split; |x| < 105414350 -> reduce_sincos (Cody-Waite by pi/2
//             in four parts) + do_sincos; table __sincostab of
//             sin/cos(i/128) as double-double pairs.
// The numeric constants are in glibc_math_data.h (tools/gen_glibc_math.c
// reads and checks them out of libm).  Beyond |x| >= 105414350 glibc uses
// a multi-precision reduction (__branred); there we fall back to the
// correctly rounded igs_math::cr_sincos (constrain() keeps theta in [0, pi),
// so no set the reference produces reaches it).
//
// Host + device, compiled WITHOUT contraction (nvcc -fmad=false, gcc
// -ffp-contract=off): every fused operation is an explicit fma().
// tests/test_glibc_math.py runs this exact code on the host against the
// system libm on tens of millions of arguments.
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "glibc_math_data.h"
#include "igs_math.cuh"

namespace glibc_math {

#if defined(__CUDACC__)
static __device__ const uint64_t k_exp_tab[256] = GLIBC_EXP_TAB_INIT;
static __device__ const uint64_t k_sincostab[440] = GLIBC_SINCOSTAB_INIT;
#endif
static const uint64_t k_exp_tab_h[256] = GLIBC_EXP_TAB_INIT;
static const uint64_t k_sincostab_h[440] = GLIBC_SINCOSTAB_INIT;

IGS_HD uint64_t as_u64(double d) {
#if defined(__CUDA_ARCH__)
    return static_cast<uint64_t>(__double_as_longlong(d));
#else
    uint64_t u;
    memcpy(&u, &d, 8);
    return u;
#endif
}
IGS_HD double as_f64(uint64_t u) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double(static_cast<long long>(u));
#else
    double d;
    memcpy(&d, &u, 8);
    return d;
#endif
}
IGS_HD uint64_t exp_tab(int i) {
#if defined(__CUDA_ARCH__)
    return __ldg(reinterpret_cast<const unsigned long long*>(k_exp_tab) + i);
#else
    return k_exp_tab_h[i];
#endif
}
IGS_HD double sc_tab(int i) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double(__ldg(reinterpret_cast<const long long*>(k_sincostab) + i));
#else
    return as_f64(k_sincostab_h[i]);
#endif
}

IGS_HD double copysign_of(double mag, double sgn) {
    return as_f64((as_u64(mag) & 0x7fffffffffffffffull) | (as_u64(sgn) & 0x8000000000000000ull));
}

// ---------------------------------------------------------------- exp
// e_exp.c specialcase(): |x| in [512, 1024) where 2^(k/N) over/underflows.
IGS_HD double exp_specialcase(double tmp, uint64_t sbits, uint64_t ki) {
    if ((ki & 0x80000000ull) == 0) {
        sbits -= 1009ull << 52;
        const double scale = as_f64(sbits);
        return 0x1p1009 * fma(scale, tmp, scale);
    }
    sbits += 1022ull << 52;
    const double scale = as_f64(sbits);
    const double st = tmp * scale;  // not fused in the FMA build (reused below)
    double y = scale + st;
    if (1.0 > y) {
        const double hi = y + 1.0;
        double lo = (scale - y) + st;
        lo = ((1.0 - hi) + y) + lo;
        y = (lo + hi) - 1.0;
        if (y == 0.0) y = 0.0;  // no -0.0
    }
    return 0x1p-1022 * y;
}

IGS_HD double exp(double x) {
    const uint64_t ix = as_u64(x);
    uint32_t abstop = static_cast<uint32_t>(ix >> 52) & 0x7ff;
    if (abstop - 0x3c9u > 0x3eu) {          // |x| < 2^-54 or |x| >= 512 (or inf/nan)
        if (static_cast<int32_t>(abstop - 0x3c9u) < 0) return 1.0 + x;  // tiny
        if (abstop >= 0x409) {                // |x| >= 1024
            if (ix == 0xfff0000000000000ull) return 0.0;
            if (abstop == 0x7ff) return 1.0 + x;
            return (ix >> 63) ? 0.0 : INFINITY;  // __math_uflow / __math_oflow
        }
        abstop = 0;  // large |x|: handled by specialcase
    }
    double kd = fma(x, GLIBC_EXP_INVLN2N, GLIBC_EXP_SHIFT);
    const uint64_t ki = as_u64(kd);
    kd = kd - GLIBC_EXP_SHIFT;
    double r = fma(kd, GLIBC_EXP_NEGLN2HIN, x);
    r = fma(kd, GLIBC_EXP_NEGLN2LON, r);
    const int idx = 2 * static_cast<int>(ki & 127);
    const uint64_t top = ki << 45;
    const double tail = as_f64(exp_tab(idx));
    const uint64_t sbits = exp_tab(idx + 1) + top;
    const double p23 = fma(r, GLIBC_EXP_C3, GLIBC_EXP_C2);
    const double p45 = fma(r, GLIBC_EXP_C5, GLIBC_EXP_C4);
    const double r2 = r * r;
    double tmp = fma(p23, r2, r + tail);
    tmp = fma(r2 * r2, p45, tmp);
    if (abstop == 0) return exp_specialcase(tmp, sbits, ki);
    const double scale = as_f64(sbits);
    return fma(scale, tmp, scale);
}

// ---------------------------------------------------------------- sincos
struct Row {
    double sn, ssn, cs, ccs;
};

// u = big + |x| puts round(|x| * 128) in the low word (s_sin.c SINCOS_TABLE_LOOKUP).
IGS_HD Row sc_row(double absx, double* xs) {
    const double u = GLIBC_SC_BIG + absx;
    *xs = absx - (u - GLIBC_SC_BIG);
    const int i = static_cast<int>(static_cast<uint32_t>(as_u64(u)) << 2);
    return {sc_tab(i), sc_tab(i + 1), sc_tab(i + 2), sc_tab(i + 3)};
}

// TAYLOR_SIN(xx, a, da) for |a| < 0.126
IGS_HD double taylor_sin(double a, double da) {
    const double xx = a * a;
    double p = fma(xx, GLIBC_SC_S5, GLIBC_SC_S4);
    p = fma(xx, p, GLIBC_SC_S3);
    p = fma(xx, p, GLIBC_SC_S2);
    p = fma(xx, p, GLIBC_SC_S1);
    const double t = fma(p, a, -(da * GLIBC_SC_CS2));  // POLYNOMIAL(xx)*a - 0.5*da (cs2 == 0.5)
    return (fma(xx, t, da)) + a;
}

// do_sin(x, dx) for |x| >= 0.126 (non-Taylor part); xs, row from sc_row(|x|).
IGS_HD double do_sin_tab(double x, double dx, double xs, const Row& t) {
    if (x <= 0) dx = -dx;
    const double xx = xs * xs;
    const double s = fma(xx * xs, fma(xx, GLIBC_SC_SN5, GLIBC_SC_SN3), dx) + xs;
    const double c = fma(dx, xs, xx * fma(fma(xx, GLIBC_SC_CS6, GLIBC_SC_CS4), xx, GLIBC_SC_CS2));
    double cor = fma(s, t.ccs, t.ssn);
    cor = fma(-c, t.sn, cor);
    cor = fma(s, t.cs, cor);
    return copysign_of(cor + t.sn, x);
}

// do_cos(x, dx); xs, row from sc_row(|x|).
IGS_HD double do_cos_tab(double x, double dx, double xs, const Row& t) {
    if (x < 0) dx = -dx;
    const double y = xs + dx;
    const double xx = y * y;
    const double s = fma(y * xx, fma(xx, GLIBC_SC_SN5, GLIBC_SC_SN3), y);
    const double c = xx * fma(fma(xx, GLIBC_SC_CS6, GLIBC_SC_CS4), xx, GLIBC_SC_CS2);
    double cor = fma(-s, t.ssn, t.ccs);
    cor = fma(-t.cs, c, cor);
    cor = fma(-s, t.sn, cor);
    return cor + t.cs;
}

IGS_HD void sincos(double x, double* sin_out, double* cos_out) {
    const uint64_t ix = as_u64(x);
    const uint32_t k = static_cast<uint32_t>(ix >> 32) & 0x7fffffffu;
    const double ax = fabs(x);
    if (k < 0x400368fdu) {
        if (k < 0x3e400000u) {  // |x| < 2^-27
            *sin_out = x;
            *cos_out = 1.0;
            return;
        }
        if (k < 0x3feb6000u) {  // |x| < 0.855469
            double xs;
            const Row t = sc_row(ax, &xs);
            *sin_out = ax < GLIBC_SC_TAYLOR_MAX ? taylor_sin(x, 0.0) : do_sin_tab(x, 0.0, xs, t);
            *cos_out = do_cos_tab(x, 0.0, xs, t);
            return;
        }
        // |x| < 2.426265: pi/2 - |x| = a + da
        const double y = GLIBC_SC_HP0 - ax;
        const double a = y + GLIBC_SC_HP1;
        const double da = (y - a) + GLIBC_SC_HP1;
        double xs;
        const Row t = sc_row(fabs(a), &xs);
        *sin_out = copysign_of(do_cos_tab(a, da, xs, t), x);
        *cos_out = fabs(a) < GLIBC_SC_TAYLOR_MAX ? taylor_sin(a, da) : do_sin_tab(a, da, xs, t);
        return;
    }
    if (k >= 0x7ff00000u) {  // inf / nan
        *sin_out = *cos_out = x - x + NAN;
        return;
    }
    if (k >= 0x419921fbu) {  // glibc: __branred (multi-precision); see header
        igs_math::cr_sincos_full(x, sin_out, cos_out);
        return;
    }
    // reduce_sincos: x = n pi/2 + (a + da)
    const double tt = fma(x, GLIBC_SC_HPINV, GLIBC_SC_TOINT);
    const double xn = tt - GLIBC_SC_TOINT;
    const int n = static_cast<int>(as_u64(tt) & 3);
    double yy = fma(-xn, GLIBC_SC_MP1, x);
    yy = fma(-xn, GLIBC_SC_MP2, yy);
    const double t2 = fma(-xn, GLIBC_SC_PP3, yy);
    double db = fma(-xn, GLIBC_SC_PP3, yy - t2);
    const double b = fma(-xn, GLIBC_SC_PP4, t2);
    db = db + fma(-xn, GLIBC_SC_PP4, t2 - b);
    // do_sincos(a, da, n) for sin and n + 1 for cos, as the FMA build
    // arranges it: (a, da) negated for n in {1, 2}, then
    // sin-part = do_sin(a', da'), cos-part = do_cos(a', da'), assigned by n.
    double a = b, da = db;
    if (n == 1 || n == 2) {
        a = -a;
        da = -da;
    }
    double xs;
    const Row t = sc_row(fabs(a), &xs);
    const double sp = fabs(a) < GLIBC_SC_TAYLOR_MAX ? taylor_sin(a, da) : do_sin_tab(a, da, xs, t);
    double cp = do_cos_tab(a, da, xs, t);
    if (n & 2) cp = -cp;
    if (n & 1) {
        *cos_out = sp;
        *sin_out = cp;
    } else {
        *sin_out = sp;
        *cos_out = cp;
    }
}

}  // namespace glibc_math
