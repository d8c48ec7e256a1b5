// dpd_math.cuh -- device-side scalar numerics for the B200 DPD engine.
//
// Two families:
//  * bit-exact fp64 restatements of the reference's fastmath / RNG
//    (inc/fastmath.hpp:26-151, inc/rng.hpp:16-91) using explicit
//    __dmul_rn/__dadd_rn/__fma_rn so nvcc cannot contract differently from
//    the (-ffp-contract=off) CPU build.  Used by the RNG-stream parity entry
//    points and the signature kernel.
//  * the fp32 hot-path Gaussian used inside the pair-force kernel: same
//    TEA-4 uniforms (bit-exact), Box-Muller radial term through an fp32
//    z = (x-1)/(x+1) log core whose x-1 is formed exactly in integers, phase
//    through MUFU sin.  Agrees with the fp64 gaussian to ~1e-6 absolute.
#pragma once
#include <cstdint>

namespace dpdb {

// ---------------------------------------------------------------- TEA / rng
__host__ __device__ __forceinline__ void tea_rounds(int rounds, uint32_t& v0, uint32_t& v1) {
    uint32_t acc = 0;
    for (int r = 0; r < rounds; ++r) {
        acc += 0x9E3779B9u;
        v0 += ((v1 << 4) + 0xA341316Cu) ^ ((v1 >> 5) + 0xC8013EA4u) ^ (v1 + acc);
        v1 += ((v0 << 4) + 0xAD90777Du) ^ ((v0 >> 5) + 0x7E95761Eu) ^ (v0 + acc);
    }
}

// compile-time unrolled 4-round TEA for the pair stream (inc/rng.hpp:77-83)
__device__ __forceinline__ void tea4(uint32_t& v0, uint32_t& v1) {
#pragma unroll
    for (int r = 1; r <= 4; ++r) {
        const uint32_t acc = 0x9E3779B9u * (uint32_t)r;
        v0 += ((v1 << 4) + 0xA341316Cu) ^ ((v1 >> 5) + 0xC8013EA4u) ^ (v1 + acc);
        v1 += ((v0 << 4) + 0xAD90777Du) ^ ((v0 >> 5) + 0x7E95761Eu) ^ (v0 + acc);
    }
}

__host__ __device__ __forceinline__ uint32_t step_mix_of(uint32_t seed, uint32_t step) {
    uint32_t a = seed, b = step;
    tea_rounds(4, a, b);
    return b;
}

// Spread the low 11 bits of m so bit k lands on bit 3k (bit 10 -> 30, so it
// fits 32 bits: 32-bit masks, checked against the bit-by-bit definition for
// all 2048 inputs; the 64-bit formulation cost twice the instructions in the
// fused force epilogue, which signs every particle every step).
__device__ __forceinline__ uint32_t spread3_11(uint32_t m) {
    uint32_t x = m & 0x7FFu;
    x = (x | (x << 16)) & 0x070000FFu;
    x = (x | (x << 8)) & 0x0700F00Fu;
    x = (x | (x << 4)) & 0x430C30C3u;
    x = (x | (x << 2)) & 0x49249249u;
    return x;
}

// inc/rng.hpp:43-62: per-particle signature from the fp64 velocity bits
__device__ __forceinline__ uint32_t make_signature(uint32_t tag, double vx, double vy, double vz) {
    const uint32_t mx = (uint32_t)((uint64_t)__double_as_longlong(vx) >> 41) & 0x7FFu;
    const uint32_t my = (uint32_t)((uint64_t)__double_as_longlong(vy) >> 41) & 0x7FFu;
    const uint32_t mz = (uint32_t)((uint64_t)__double_as_longlong(vz) >> 41) & 0x7FFu;
    const uint32_t w = spread3_11(mx) | (spread3_11(my) << 1) | (spread3_11(mz) << 2);
    uint32_t a = __brev(tag), b = w;
    tea_rounds(16, a, b);
    return a ^ b;
}

// --------------------------------------------------------- fp64 fastmath
// Frozen minimax tables: inc/fastmath.hpp:35-57 (data, must be identical).
#define DPDB_LNQ {0x1.555555555397ap-1, 0x1.999999a28e942p-2, 0x1.2492417a9975ap-2, \
                  0x1.c72276984c243p-3, 0x1.732c520e537b1p-3, 0x1.587592fb5a518p-3}
#define DPDB_LOG2Q {0x1.ec709dc3a0455p-1, 0x1.2776c50ee73bep-1, 0x1.a61762d1f5b51p-2, \
                    0x1.484afcfb984e8p-2, 0x1.0ca11d4fbc32dp-2, 0x1.c479f5cc9ee5ep-3, \
                    0x1.b52725f185dd3p-3}
#define DPDB_EXP2R {0x1.62e42fefa39f5p-1, 0x1.ebfbdff82c04bp-3, 0x1.c6b08d7065838p-5,   \
                    0x1.3b2ab6f73416fp-7, 0x1.5d87ff4d2262ap-10, 0x1.4308fa1dd16ddp-13, \
                    0x1.ffcfc6a9b62c8p-17, 0x1.628f3583fa66bp-20, 0x1.b85f42cc9ad9ap-24, \
                    0x1.c2c47913b09f9p-28, 0x1.58566e8b85bdfp-31}
#define DPDB_SINP {0x1.921fb5441e49dp+1, -0x1.4abbce4f1a2d1p+2, 0x1.466bbfc24f863p+1, \
                   -0x1.32d11201b18c4p-1, 0x1.500ff7f212ce7p-4, -0x1.cc345a6170d5cp-8}

template <int N>
__device__ __forceinline__ double horner_rn(const double (&c)[N], double x) {
    double p = c[N - 1];
#pragma unroll
    for (int k = N - 2; k >= 0; --k) p = __fma_rn(p, x, c[k]);
    return p;
}

__device__ __forceinline__ double power2_64(int n) {
    return __longlong_as_double((long long)((uint64_t)(1023 + n) << 52));
}

__device__ __forceinline__ void log2_frac_ext64(double x, double& rhi, double& rlo) {
    constexpr double q[7] = DPDB_LOG2Q;
    const double k2l = 0x1.71547652b82fep+1, k2lres = 0x1.777d0ffda0d24p-55;
    const bool big = x >= 1.4142135623730951;
    const double xr = big ? __dmul_rn(0.5, x) : x;
    const double z = __ddiv_rn(__dsub_rn(xr, 1.0), __dadd_rn(xr, 1.0));
    const double w = __dmul_rn(z, z);
    const double t = __dmul_rn(w, horner_rn(q, w));
    const double shi = __dadd_rn(k2l, t);
    const double slo = __dadd_rn(__dadd_rn(__dsub_rn(k2l, shi), t), k2lres);
    const double fhi = __dmul_rn(z, shi);
    const double flo = __dadd_rn(__fma_rn(z, shi, -fhi), __dmul_rn(z, slo));
    const double add = big ? 1.0 : 0.0;
    rhi = __dadd_rn(add, fhi);
    rlo = __dadd_rn(__dadd_rn(__dsub_rn(add, rhi), fhi), flo);
}

__device__ __forceinline__ double exp2_frac64(double x) {
    constexpr double r[11] = DPDB_EXP2R;
    return __fma_rn(x, horner_rn(r, x), 1.0);
}

__device__ __forceinline__ double log2_frac64(double x) {
    double h, l;
    log2_frac_ext64(x, h, l);
    return __dadd_rn(h, l);
}

// inc/fastmath.hpp:108-118
__device__ __forceinline__ double fastlog64(uint32_t v) {
    constexpr double q[6] = DPDB_LNQ;
    const int e = 31 - __clz(v);
    const double x0 = __dmul_rn((double)v, power2_64(-e));
    const bool big = x0 >= 1.4142135623730951;
    const double x = big ? __dmul_rn(0.5, x0) : x0;
    const double di = (double)(e + (int)big - 32);
    const double z = __ddiv_rn(__dsub_rn(x, 1.0), __dadd_rn(x, 1.0));
    const double w = __dmul_rn(z, z);
    const double lnx = __fma_rn(__dmul_rn(z, w), horner_rn(q, w), __dmul_rn(2.0, z));
    return __fma_rn(di, 0x1.62e42fef00000p-1, __fma_rn(di, 0x1.473de6af278edp-34, lnx));
}

// inc/fastmath.hpp:122-130
__device__ __forceinline__ double fastcos2pi64(uint32_t v) {
    constexpr double s[6] = DPDB_SINP;
    const uint32_t b = v >> 31;
    const double u = __dmul_rn((double)(v & 0x7FFFFFFFu), 0x1p-31);
    const double y = __dsub_rn(u, 0.5);
    const double r = __dmul_rn(y, horner_rn(s, __dmul_rn(y, y)));
    const unsigned long long flip = (unsigned long long)(b ^ 1u) << 63;
    return __longlong_as_double((long long)((unsigned long long)__double_as_longlong(r) ^ flip));
}

// inc/fastmath.hpp:135-151
__device__ __forceinline__ double fastpow64(double a, double b) {
    const uint64_t bits = (uint64_t)__double_as_longlong(a);
    const int ie = (int)(bits >> 52) - 1023;
    const double m = __longlong_as_double(
        (long long)((bits & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull));
    double fh, fl;
    log2_frac_ext64(m, fh, fl);
    const double di = (double)ie;
    const double y = __dmul_rn(b, __dadd_rn(di, fh));
    double ii = floor(y);
    if (ii > 1024.0) ii = 1024.0;
    if (ii < -1022.0) ii = -1022.0;
    double frac = __fma_rn(b, fh, __fma_rn(b, di, -ii));
    frac = __fma_rn(b, fl, frac);
    return __dmul_rn(power2_64((int)ii), exp2_frac64(frac));
}

// inc/rng.hpp:88-91
__device__ __forceinline__ double gaussian64(uint32_t ua, uint32_t ub) {
    ua |= (ua == 0u);
    return __dmul_rn(__dsqrt_rn(__dmul_rn(-2.0, fastlog64(ua))), fastcos2pi64(ub));
}

// ------------------------------------------------------- fp32 hot path
// ln(u * 2^-32) for u >= 1.  x = u/2^k in [sqrt2/2, sqrt2); x-1 is formed
// exactly in integer arithmetic so the relative error stays flat as u ->
// 2^32 (where ln -> 0), which is what keeps the Box-Muller radius accurate
// in the tail.  ~1 ulp fp32.
__device__ __forceinline__ float fastlog32(uint32_t u) {
    const int e = 31 - __clz(u);
    // big <=> u >= sqrt2 * 2^e; compare on the top 24 bits (monotone, exact enough
    // for choosing the reduction branch -- both branches are valid near the split)
    const uint32_t top = u << (31 - e);  // normalized: bit31 set
    const int big = top >= 0xB504F334u;  // sqrt(2) * 2^31
    const int k = e + big;               // 0..32
    const uint32_t pk = k >= 32 ? 0u : (1u << k);
    const int num = (int)(u - pk);  // exact: x-1 scaled by 2^k
    const float numf = (float)num;
    const float pkf = __int_as_float((127 + k) << 23);  // 2^k
    const float den = fmaf(2.0f, pkf, numf);             // (x+1)*2^k = u + 2^k, no cancellation
    const float z = __fdividef(numf, den);
    const float w = z * z;
    float p = fmaf(w, 0.2222222222f, 0.2857142857f);
    p = fmaf(w, p, 0.4f);
    p = fmaf(w, p, 0.6666666667f);
    const float lnx = fmaf(z * w, p, 2.0f * z);
    const float di = (float)(k - 32);
    return fmaf(di, 0.693147180559945f, lnx);
}

// Box-Muller on the TEA-4 pair words, fp32: sqrt(-2 ln ua) * cos(2 pi ub)
// cos(2 pi t) = -(-1)^b sin(pi y), y = low31(ub)/2^31 - 1/2 (inc/fastmath.hpp:122-130)
__device__ __forceinline__ float gaussian32(uint32_t ua, uint32_t ub) {
    ua = max(ua, 1u);
    const float rad = sqrtf(-2.0f * fastlog32(ua));
    const float y = (float)(int)((ub & 0x7FFFFFFFu) - 0x40000000u) * 0x1p-31f;
    float s = __sinf(3.14159265358979f * y);
    s = (ub >> 31) ? s : -s;
    return rad * s;
}

}  // namespace dpdb
