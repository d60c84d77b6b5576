// codec.cu -- the IGS2 container (codec.cpp) with the per-parameter binary16
// packing and unpacking on the device.
//
// Layout (codec.hpp:46-50): "IGS2" | version u8 | flags u8 | k u16 |
// width u16 | height u16 | n_g u32 | n_b u32, little-endian (20 bytes), then
// n_g records of 8 float16 (mu_u, mu_v, theta, s1, s2, r, g, b) and n_b
// records of 4 float16 (x1, y1, x2, y2).
//
// float16 conversions restate codec.cpp:12-66 bit for bit (double -> float
// by IEEE rounding, then the reference's round-to-nearest-even packing,
// including its subnormal and overflow handling); decode and quantize_set
// re-constrain (gaussian.cpp:74-90) like the reference.  The header and the
// block table (a few thousand corners) are handled on the host with the
// same conversion functions.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>

#include "igs_internal.cuh"

using namespace igs_dev;

#define IGS_CODEC_HD __host__ __device__ __forceinline__

namespace igs_codec {

// codec.cpp:12-40 float_to_half
IGS_CODEC_HD uint16_t float_to_half(float f) {
    uint32_t x;
    memcpy(&x, &f, 4);
    const uint32_t sign = (x >> 16) & 0x8000u;
    uint32_t mant = x & 0x007fffffu;
    const int32_t exp = (int32_t)((x >> 23) & 0xffu);
    if (exp == 0xff) return (uint16_t)(sign | 0x7c00u | (mant ? (0x200u | (mant >> 13)) : 0u));
    const int32_t e = exp - 127 + 15;
    if (e >= 0x1f) return (uint16_t)(sign | 0x7c00u);
    if (e <= 0) {
        const int32_t shift = 14 - e;
        if (shift > 24 || exp == 0) return (uint16_t)sign;
        mant |= 0x00800000u;
        uint32_t kept = mant >> shift;
        const uint32_t rem = mant & ((1u << shift) - 1u);
        const uint32_t half_point = 1u << (shift - 1);
        if (rem > half_point || (rem == half_point && (kept & 1u))) ++kept;
        return (uint16_t)(sign | kept);
    }
    uint32_t h = sign | ((uint32_t)e << 10) | (mant >> 13);
    const uint32_t rem = mant & 0x1fffu;
    if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ++h;
    return (uint16_t)h;
}

// codec.cpp:42-66 half_to_float
IGS_CODEC_HD float half_to_float(uint16_t h) {
    const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
    const uint32_t exp = (h >> 10) & 0x1fu;
    uint32_t mant = h & 0x3ffu;
    uint32_t x;
    if (exp == 0) {
        if (mant == 0) {
            x = sign;
        } else {
            int e = -1;
            do {
                mant <<= 1;
                ++e;
            } while (!(mant & 0x400u));
            mant &= 0x3ffu;
            x = sign | ((uint32_t)(127 - 15 - e) << 23) | (mant << 13);
        }
    } else if (exp == 0x1f) {
        x = sign | 0x7f800000u | (mant << 13);
    } else {
        x = sign | ((exp - 15 + 127) << 23) | (mant << 13);
    }
    float f;
    memcpy(&f, &x, 4);
    return f;
}

IGS_CODEC_HD uint16_t double_to_half(double d) { return float_to_half((float)d); }
IGS_CODEC_HD double half_to_double(uint16_t h) { return (double)half_to_float(h); }

// codec.cpp:136-139 check_encodable
IGS_CODEC_HD bool encodable(double v) { return isfinite(v) && fabs(v) <= 65504.0; }

}  // namespace igs_codec

namespace {

__device__ __forceinline__ double clamp01c(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

// gaussian.cpp:74-90 constrain, parameter p of a record
__device__ __forceinline__ double constrain_p(int p, double v) {
    if (p == 2) {
        double th = fmod(v, kPi);
        if (th < 0.0) th = __dadd_rn(th, kPi);
        if (th >= kPi) th = 0.0;
        return th;
    }
    if (p == 3 || p == 4) return v < kScaleMin ? kScaleMin : (v > kScaleMax ? kScaleMax : v);
    return clamp01c(v);
}

// encode: one thread per parameter; status[1] <- first unencodable slot
__global__ void pack_kernel(const double* __restrict__ params, size_t count, uint16_t* __restrict__ out,
                            long long* __restrict__ status) {
    const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= count) return;
    const double v = params[e];
    if (!igs_codec::encodable(v)) atomicMin(status + 1, (long long)e);
    out[e] = igs_codec::double_to_half(v);
}

// decode / quantize_set: binary16 -> double, re-constrained (codec.cpp:200-211,
// codec.cpp:69-81); a record with a non-finite value raises in constrain, so
// status[1] <- first such Gaussian
__global__ void unpack_kernel(const uint16_t* __restrict__ in, const double* __restrict__ src, size_t count,
                              double* __restrict__ params, long long* __restrict__ status) {
    const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= count) return;
    const uint16_t h = in ? in[e] : igs_codec::double_to_half(src[e]);
    const double v = igs_codec::half_to_double(h);
    if (!isfinite(v)) atomicMin(status + 1, (long long)(e / 8));
    params[e] = constrain_p((int)(e % 8), v);
}

}  // namespace

int igs_codec_pack(igs_ctx* ctx, uint16_t* dev_out) {
    const size_t count = (size_t)ctx->n * 8;
    pack_kernel<<<(unsigned)((count + 255) / 256), 256, 0, ctx->stream>>>(ctx->params, count, dev_out, ctx->status);
    IGS_LAUNCHED(ctx);
    return IGS_OK;
}

// binary16 -> double + constrain into dev_out (n records): from packed
// halves (dev_in, decode) or by rounding doubles through binary16 (dev_src,
// quantize_set).  status[1] <- first record with a non-finite value; the
// caller commits dev_out only when it is clear.
int igs_codec_unpack(igs_ctx* ctx, const uint16_t* dev_in, const double* dev_src, uint32_t n, double* dev_out) {
    const size_t count = (size_t)n * 8;
    unpack_kernel<<<(unsigned)((count + 255) / 256), 256, 0, ctx->stream>>>(dev_in, dev_src, count, dev_out,
                                                                           ctx->status);
    IGS_LAUNCHED(ctx);
    return IGS_OK;
}

uint16_t igs_host_double_to_half(double d) { return igs_codec::double_to_half(d); }
double igs_host_half_to_double(uint16_t h) { return igs_codec::half_to_double(h); }
bool igs_host_encodable(double v) { return igs_codec::encodable(v); }
