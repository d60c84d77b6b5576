// Host check of csrc/glibc_math.cuh against the system libm (the library the
// reference binds): compiled by tests/test_glibc_math.py with
// g++ -O2 -mfma -ffp-contract=off, loaded with ctypes.  Each entry point
// draws `count` arguments from a family and returns the number whose result
// differs from libm's in any bit (first offender in *bad).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>

#include "glibc_math.cuh"

namespace {

uint64_t bits(double d) {
    uint64_t u;
    std::memcpy(&u, &d, 8);
    return u;
}

double draw(std::mt19937_64& g, int family) {
    std::uniform_real_distribution<double> u01(0.0, 1.0);
    switch (family) {
        case 0: return u01(g) * M_PI;                        // theta after constrain(): [0, pi)
        case 1: return (u01(g) * 2 - 1) * 8.0;               // all sincos branches up to 8
        case 2: return std::ldexp(u01(g) * 2 - 1, static_cast<int>(g() % 60) - 33);  // 2^-33 .. 2^26
        case 3: {                                            // raw bit patterns below 105414350
            double d;
            uint64_t b = g() & 0x7fffffffffffffffull;
            b = b % 0x4199000000000000ull;
            std::memcpy(&d, &b, 8);
            return (g() & 1) ? -d : d;
        }
        case 4: return -0.5 * (u01(g) * 200.0);              // exp(-q/2), q in [0, 200)
        case 5: return -0.5 * std::ldexp(u01(g), static_cast<int>(g() % 80) - 60);  // tiny..large q
        case 6: return (u01(g) * 2 - 1) * 760.0;             // exp specialcase + over/underflow
        case 7: return (u01(g) * 2 - 1) * 1e-15;             // exp tiny
        case 8: {                                            // near multiples of pi/2 (hard reduction)
            const double m = static_cast<double>(g() % 64);
            return std::nextafter(m * M_PI_2, 0.0) + (static_cast<double>(g() % 5) - 2) * 4e-16 * (m + 1);
        }
        default: return 0.0;
    }
}

}  // namespace

extern "C" {

long long check_sincos(long long count, uint64_t seed, int family, double* bad) {
    std::mt19937_64 g(seed);
    long long n = 0;
    for (long long i = 0; i < count; ++i) {
        const double x = draw(g, family);
        double s0, c0, s1, c1;
        sincos(x, &s0, &c0);
        glibc_math::sincos(x, &s1, &c1);
        if (bits(s0) != bits(s1) || bits(c0) != bits(c1)) {
            if (n == 0 && bad) *bad = x;
            ++n;
        }
    }
    return n;
}

long long check_exp(long long count, uint64_t seed, int family, double* bad) {
    std::mt19937_64 g(seed);
    long long n = 0;
    for (long long i = 0; i < count; ++i) {
        const double x = draw(g, family);
        const double e0 = std::exp(x), e1 = glibc_math::exp(x);
        if (bits(e0) != bits(e1)) {
            if (n == 0 && bad) *bad = x;
            ++n;
        }
    }
    return n;
}

int check_special(double* bad) {
    const double xs[] = {0.0, -0.0, 1e-300, -1e-300, 4.9e-324, INFINITY, -INFINITY, NAN, 1.0, -1.0,
                         M_PI, -M_PI, M_PI_2, 0.855469, 0.126, 2.426265, 105414349.0, 2e8, 1e300,
                         -708.0, -745.0, -745.2, -1000.0, -1100.0, 709.0, 710.0, 1100.0, -512.0, 512.0};
    int n = 0;
    for (double x : xs) {
        double s0, c0, s1, c1;
        sincos(x, &s0, &c0);
        glibc_math::sincos(x, &s1, &c1);
        const double e0 = std::exp(x), e1 = glibc_math::exp(x);
        const bool nan_ok = std::isnan(x);
        const bool ok = nan_ok ? (std::isnan(s1) && std::isnan(c1) && std::isnan(e1))
                               : (bits(s0) == bits(s1) && bits(c0) == bits(c1) && bits(e0) == bits(e1));
        if (!ok) {
            if (n == 0 && bad) *bad = x;
            ++n;
        }
    }
    return n;
}
}
