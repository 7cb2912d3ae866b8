// qpm_common.cuh -- device helpers shared by the HWSDA kernels (sm_100a).
//
// Everything here is exact integer or IEEE-754 binary64 arithmetic.  The
// library is compiled with -fmad=false so that no multiply/add pair is
// contracted into an FMA behind our back: the reference (numba without
// fastmath, numpy) rounds every product and sum separately.  Where a kernel
// wants an FMA (the fast fitness scan) it calls fma() explicitly.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace qpm {

// ---------------------------------------------------------------- RNG
// splitmix64 counter streams, rng.py:12-36 and _kernels.py:87-98.
constexpr uint64_t kGold = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kMix1 = 0xBF58476D1CE4E5B9ULL;
constexpr uint64_t kMix2 = 0x94D049BB133111EBULL;
constexpr double kTwoM53 = 1.1102230246251565404236316680908203125e-16;  // 2^-53
constexpr uint64_t kTwo53 = 1ULL << 53;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * kMix1;
    z = (z ^ (z >> 27)) * kMix2;
    return z ^ (z >> 31);
}

// rng.fold_key(seed, g, i)
__host__ __device__ __forceinline__ uint64_t fold_key3(uint64_t seed, uint64_t a, uint64_t b) {
    uint64_t h = mix64(seed);
    h = mix64(h + kGold + a);
    return mix64(h + kGold + b);
}

// the 53-bit integer m of draw `pos` (u = m * 2^-53)
__device__ __forceinline__ uint64_t draw53(uint64_t key, uint64_t pos) {
    return mix64(key + (pos + 1ULL) * kGold) >> 11;
}

__device__ __forceinline__ double draw_u(uint64_t key, uint64_t pos) {
    return (double)draw53(key, pos) * kTwoM53;
}

// CounterStream.randint: min(int(u * bound), bound - 1) with an FP64 product
__device__ __forceinline__ int64_t randint(uint64_t key, uint64_t pos, int64_t bound) {
    double u = draw_u(key, pos);
    int64_t r = (int64_t)(u * (double)bound);
    return r < bound - 1 ? r : bound - 1;
}

// u < p  <=>  m < ceil(p * 2^53)   (p in [0, 1], scaling by 2^53 is exact)
__host__ __device__ __forceinline__ uint64_t lt_threshold(double p) {
    if (!(p > 0.0)) return 0;
    if (p >= 1.0) return kTwo53 + 1;  // every m < 2^53 passes
    return (uint64_t)ceil(p * 9007199254740992.0);
}
// u <= p  <=>  m <= floor(p * 2^53)  <=>  m < floor(p * 2^53) + 1
__host__ __device__ __forceinline__ uint64_t le_threshold(double p) {
    if (p < 0.0) return 0;
    if (p >= 1.0) return kTwo53 + 1;
    return (uint64_t)floor(p * 9007199254740992.0) + 1;
}

// -------------------------------------------------------------- hypot
// glibc 2.39 hypot (Borges' correction, non-FMA build), which numba's
// abs(complex) calls on x86-64.  Verified bit-equal to libm on 2e6 random
// pairs in the build container; see DESIGN.md.
__device__ __forceinline__ double hypot_kernel(double ax, double ay) {
    double h = sqrt(ax * ax + ay * ay);
    double t1, t2;
    if (h <= 2.0 * ay) {
        double delta = h - ay;
        t1 = ax * (2.0 * delta - ax);
        t2 = (delta - 2.0 * (ax - ay)) * delta;
    } else {
        double delta = h - ax;
        t1 = 2.0 * delta * (ax - 2.0 * ay);
        t2 = (4.0 * delta - ay) * ay + delta * delta;
    }
    h -= (t1 + t2) / (2.0 * h);
    return h;
}

__device__ __forceinline__ double hypot_glibc(double x, double y) {
    if (!isfinite(x) || !isfinite(y)) {
        if (isinf(x) || isinf(y)) return __longlong_as_double(0x7FF0000000000000LL);
        return x + y;
    }
    x = fabs(x);
    y = fabs(y);
    double ax = x < y ? y : x;
    double ay = x < y ? x : y;
    const double kScale = 0x1p-600, kLarge = 0x1p+511, kTiny = 0x1p-511, kEps = 0x1p-54;
    if (ax > kLarge) {
        if (ay <= ax * kEps) return ax + ay;
        return hypot_kernel(ax * kScale, ay * kScale) / kScale;
    }
    if (ay < kTiny) {
        if (ax >= ay / kEps) return ax + ay;
        return hypot_kernel(ax / kScale, ay / kScale) * kScale;
    }
    if (ay <= ax * kEps) return ax + ay;
    return hypot_kernel(ax, ay);
}

// ------------------------------------------------------ numpy pairwise sum
// numpy/_core/src/umath/loops_utils.h.src pairwise_sum, the summation that
// np.sum / np.mean / np.std use on contiguous float64.  Sequential device
// version (one thread); used for short vectors (wavelength axis).
__device__ inline double pairwise_leaf(const double *a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; ++i) res += a[i];
        return res;
    }
    double r0 = a[0], r1 = a[1], r2 = a[2], r3 = a[3], r4 = a[4], r5 = a[5], r6 = a[6], r7 = a[7];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8) {
        r0 += a[i + 0];
        r1 += a[i + 1];
        r2 += a[i + 2];
        r3 += a[i + 3];
        r4 += a[i + 4];
        r5 += a[i + 5];
        r6 += a[i + 6];
        r7 += a[i + 7];
    }
    double res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
    for (; i < n; ++i) res += a[i];
    return res;
}

__device__ inline double pairwise_sum_seq(const double *a, int64_t n) {
    // explicit stack instead of recursion: post-order over the split tree
    struct Frame {
        int64_t off, n;
        int state;
        double left;
    };
    Frame st[48];
    int top = 0;
    st[0] = {0, n, 0, 0.0};
    double ret = 0.0;
    while (top >= 0) {
        Frame &f = st[top];
        if (f.n <= 128) {
            ret = pairwise_leaf(a + f.off, f.n);
            --top;
            continue;
        }
        int64_t n2 = f.n / 2;
        n2 -= n2 % 8;
        if (f.state == 0) {
            f.state = 1;
            st[top + 1] = {f.off, n2, 0, 0.0};
            ++top;
        } else if (f.state == 1) {
            f.left = ret;
            f.state = 2;
            st[top + 1] = {f.off + n2, f.n - n2, 0, 0.0};
            ++top;
        } else {
            ret = f.left + ret;
            --top;
        }
    }
    return ret;
}

// ------------------------------------------------------------ sign bits
// bit j of a row is 1 iff domain j is -1 (genome < 0; -0.0 projects to +1,
// optimizer.py:55 and tests/test_optimizer.py:49-52).
__device__ __forceinline__ uint64_t sign_mask64(uint32_t bit) { return (uint64_t)bit << 63; }

__device__ __forceinline__ double flip_if(double x, uint64_t mask) {
    return __longlong_as_double(__double_as_longlong(x) ^ (long long)mask);
}

}  // namespace qpm
