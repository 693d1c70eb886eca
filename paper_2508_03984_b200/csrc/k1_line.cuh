// K1 line finalize helpers shared by the stats kernels (k1_scale.cu) and the
// fused single-pass K1 kernels (k1_fused.cu): the fast-mode exponent of one
// row/column from its order-free max and sum of squares, and the exact
// sequential recompute of a line whose floor is too close to call
// (reference: scaling.cpp:45-99).
#pragma once

#include "ozk_device.cuh"

namespace ozk {
namespace {

// Guard band of the parallel sum against the reference's sequential one: both
// approximate S = sum (a 2^-g)^2 within (k+1) u S, so their budgets differ by
// at most 0.51 * 2 (k+1) u / ln 2 < 1.5 (k+1) u; log2/round-off adds < 1e-13.
__device__ __forceinline__ double guard_band(int64_t k) { return 4.0 * static_cast<double>(k + 2) * 0x1.0p-53 + 1e-11; }

__device__ __forceinline__ bool needs_exact(double y, double mx, int64_t k) {
    const double d = fmin(y - floor(y), ceil(y) - y);
    // |x| >= 2^500 could overflow sum x^2; tiny maxima could underflow it
    return d < guard_band(k) || mx >= 0x1.0p+500 || mx < 0x1.0p-400;
}

// max |x| over a line, tracked on the bit patterns: an unsigned max of the high
// words with the sign shifted out (IEEE order of |x| is the integer order of
// the pattern) is 2 integer ops per element, where fmax(double) costs a
// DSETP/FSEL/SEL/LOP3 sequence. It keeps the exponent and the top 19 mantissa
// bits of max |x| — all the line finalize reads from the maximum (the zero
// test, ilogb, the [2^-400, 2^500) range, Inf). A line whose nonzero elements
// all have zero high words (|x| < 2^-1042) comes out as the smallest
// subnormal, below 2^-400, so it takes the exact recompute, which takes its
// own maximum.
struct AbsMax {
    uint32_t key = 0;  // max over (high word << 1)
    uint32_t lo = 0;   // OR of the low words
    __device__ __forceinline__ void add(double x) {
        key = max(key, static_cast<uint32_t>(__double2hiint(x)) << 1);
        lo |= static_cast<uint32_t>(__double2loint(x));
    }
    __device__ __forceinline__ void merge(uint32_t k, uint32_t l) {
        key = max(key, k);
        lo |= l;
    }
    __device__ __forceinline__ void warp_reduce() {
#pragma unroll
        for (int o = 16; o; o >>= 1) merge(__shfl_xor_sync(0xffffffffu, key, o), __shfl_xor_sync(0xffffffffu, lo, o));
    }
    __device__ __forceinline__ double value() const {
        if (key == 0) return lo ? 0x1p-1074 : 0.0;
        return __hiloint2double(static_cast<int>(key >> 1), 0);
    }
};

// fast / accurate exponent of one line from its max and sum of squares (e);
// returns whether the line needs the exact sequential recompute
__device__ __forceinline__ bool line_exponent(const LineFinal& F, double mx, double s, int& e) {
    if (F.mode == OZK_FAST) {
        e = 0;  // zero line: sentinel mu = 1 (scaling.cpp:80, :88)
        if (mx == 0.0) return false;
        const int g = ilogb(mx);
        const double y = fast_budget(ldexp(s, -2 * g), F.k, F.pp_fast);
        e = fast_exponent_from_budget(y, g, F.prec, F.fix);
        return needs_exact(y, mx, F.k);
    }
    e = mx != 0.0 ? 5 - ilogb(mx) : INT32_MIN;
    return false;
}
// the same, written to exp_out (and, accurate mode, the line's bound maximum cleared)
__device__ __forceinline__ bool finalize_line(const LineFinal& F, int64_t line, double mx, double s) {
    int e;
    const bool flag = line_exponent(F, mx, s, e);
    F.exp_out[line] = e;
    if (F.mode != OZK_FAST && F.zero_out) F.zero_out[line] = 0;
    return flag;
}

// Warp-collective, reference order: s = 0; for h: nh = ldexp(x_h, -g); s += nh*nh (no FMA).
// Returns the fast-mode exponent on every lane.
__device__ int exact_line_exponent(const LineFinal& F, int64_t line, int lane) {
    const int64_t off = line * F.line_step;
    const int64_t k = F.k;
    double mx = 0.0;
    for (int64_t h = lane; h < k; h += 32) mx = fmax(mx, fabs(load_as_double(F.base, off + h * F.elem_step, F.is_f32)));
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const int g = ilogb(mx);
    double s = 0.0;
    for (int64_t h0 = 0; h0 < k; h0 += 32) {
        const int64_t h = h0 + lane;
        double sq = 0.0;
        if (h < k) {
            const double nh = ldexp(load_as_double(F.base, off + h * F.elem_step, F.is_f32), -g);
            sq = __dmul_rn(nh, nh);
        }
        const int cnt = k - h0 < 32 ? static_cast<int>(k - h0) : 32;
        for (int q = 0; q < cnt; ++q) s = __dadd_rn(s, __shfl_sync(0xffffffffu, sq, q));
    }
    // the floor from the host-built step table: the reference's glibc log2 decides
    // it even where y = pp - 0.51 log2(ub) is within an ulp of an integer
    return fast_exponent_from_floor(fast_floor_table(fast_ub(s, k), F.fast_floor), g, F.prec, F.fix);
}
__device__ void exact_line(const LineFinal& F, int64_t line, int lane) {
    const int e = exact_line_exponent(F, line, lane);
    if (lane == 0) F.exp_out[line] = e;
}

}  // namespace
}  // namespace ozk
