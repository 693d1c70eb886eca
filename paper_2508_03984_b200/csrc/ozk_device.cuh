// Device-side arithmetic shared by the kernels. Every FP operation that the
// reference performs as separately rounded ops is spelled with the explicit
// _rn intrinsics (the library is also compiled with --fmad=false), so no
// multiply-add pair is contracted behind our back (SURVEY §7 "hard parts").
#pragma once

#include <cstdint>

#include "ozk_internal.h"

namespace ozk {

// 2^e as a double for e in [-1022, 1023] (exact).
__device__ __forceinline__ double pow2d(int e) {
    return __longlong_as_double(static_cast<long long>(e + 1023) << 52);
}
// 2^e as a float for e in [-126, 127] (exact).
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((e + 127) << 23); }

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// truncate_scale element (residue.cpp:15,18): trunc(x * (T)scale), scale = 2^e.
__device__ __forceinline__ double trunc_scaled(double x, int e) { return trunc(__dmul_rn(x, pow2d(e))); }
__device__ __forceinline__ float trunc_scaled(float x, int e) { return truncf(__fmul_rn(x, pow2f(e))); }

// rmod_fast (residue.hpp:39-53) with the refinement thresholds of :17-20.
__device__ __forceinline__ int8_t rmod_fast(double x, int p, double pinv64, float pinv32, int n) {
    float y = __double2float_rn(__fma_rn(rint(__dmul_rn(x, pinv64)), -static_cast<double>(p), x));
    const float pf = static_cast<float>(p);
    if (n >= 13) y = __fmaf_rn(rintf(__fmul_rn(y, pinv32)), -pf, y);
    if (n >= 19) y = __fmaf_rn(rintf(__fmul_rn(y, pinv32)), -pf, y);
    return static_cast<int8_t>(__float2int_rz(y));
}
__device__ __forceinline__ int8_t rmod_fast(float x, int p, double /*pinv64*/, float pinv32, int n) {
    const float pf = static_cast<float>(p);
    float y = __fmaf_rn(rintf(__fmul_rn(x, pinv32)), -pf, x);
    if (n >= 5) y = __fmaf_rn(rintf(__fmul_rn(y, pinv32)), -pf, y);
    if (n >= 11) y = __fmaf_rn(rintf(__fmul_rn(y, pinv32)), -pf, y);
    return static_cast<int8_t>(__float2int_rz(y));
}

// ---- exact fast residues ---------------------------------------------------
// rmod_fast first forms q = rint(fl(x * fl(1/p))). Its total error against x/p
// is below |x/p| 2^-52, while an integer x sits at least 1/(2p) from a
// half-integer multiple of p (p odd; p = 256 is exact). So for |x| <= 2^50 the
// first step already yields the symmetric residue r in [-(p-1)/2, (p-1)/2]
// (p = 256: +-128 -> byte 0x80 either way), and the FP32 refinement passes of
// residue.hpp:42-43 leave it unchanged (|r * pinv32| < 1/2). The FP32 path
// (residue.hpp:47-53) gives the symmetric residue for |x| <= 2^21 at any N and
// for all representable |x| < 2^44 once one refinement runs (N >= 5).
// Inside that domain we compute the symmetric residue with one full-rate FP64
// FMA and one 32-bit IMAD, no conversion-class instructions (F2F/FRND/F2I run
// at 16/clk/SM on sm_100 and made the literal sequence conversion-bound):
//   qM = fma(x, pinv64, M) = M + q,  q = nearest(x/p)     (M = 1.5 * 2^52)
//   r  = lo32(x + M) - lo32(qM) * p   (mod 2^32; exact because |r| <= 128)
// since the low 32 bits of the encoding of M + v are v mod 2^32 for any
// integer |v| < 2^51. Outside the domain the literal reference sequence runs.
constexpr double kMagic52 = 6755399441055744.0;  // 1.5 * 2^52

__device__ __forceinline__ bool symmetric_residue_domain(double x, int prec, int n) {
    const double ax = fabs(x);
    if (prec == OZK_FP64) return ax <= 0x1.0p50;
    return ax <= 0x1.0p21 || (n >= 5 && ax <= 0x1.0p43);
}
// x integer-valued, |x| <= 2^50; xlo = lo32(x + kMagic52); neg_p = -p mod 2^32.
// Returns r mod 2^32 (the int8 plane byte is its low byte): one DFMA + one IMAD.
__device__ __forceinline__ uint32_t symmetric_residue(double x, uint32_t xlo, uint32_t neg_p, double pinv64) {
    const uint32_t qlo = static_cast<uint32_t>(__double2loint(__fma_rn(x, pinv64, kMagic52)));
    return xlo + qlo * neg_p;
}
// four residue words -> one packed word of their low bytes (3 PRMT)
__device__ __forceinline__ uint32_t pack_low_bytes(uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
    return __byte_perm(__byte_perm(r0, r1, 0x0040), __byte_perm(r2, r3, 0x0040), 0x5410);
}

template <typename T>
__device__ __forceinline__ uint32_t literal_byte(T x, const DevConsts& c, int t) {
    return static_cast<uint32_t>(static_cast<uint8_t>(rmod_fast(x, c.p[t], c.pinv64[t], c.pinv32[t], c.n)));
}

// 8-byte plane store, optionally with an L2 eviction-priority policy
template <bool kHint>
__device__ __forceinline__ void store_plane8(int8_t* p, uint2 w, uint64_t pol) {
    if constexpr (kHint)
        asm volatile("st.global.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;" ::"l"(p), "r"(w.x), "r"(w.y), "l"(pol)
                     : "memory");
    else
        *reinterpret_cast<uint2*>(p) = w;
}

// K1b core (residue.cpp:24-42): the N residue bytes of 8 consecutive
// truncated-scaled elements x of one column, one 8-byte word per plane at
// dst0 + t * plane_stride. fast (warp-uniform): every x of the warp lies in
// the symmetric-residue domain (one DFMA per element and modulus, one IMAD
// per element and modulus to pack the bytes); else the literal rmod_fast
// sequence.
// kMaxMod: the modulus count rounded up to a bucket (8/12/14/16/20): the
// modulus loop is unrolled, and only the moduli past the bucket below
// (kMinMod) test t < n.
__host__ __device__ constexpr int min_mod_of_bucket(int kMaxMod) {
    return kMaxMod <= 8 ? 1 : (kMaxMod <= 12 ? 9 : (kMaxMod <= 14 ? 13 : (kMaxMod <= 16 ? 15 : 17)));
}
template <typename T, int kMaxMod, bool kHint = false>
__device__ __forceinline__ void residue_planes8(const T (&x)[8], bool fast, int8_t* dst0, int64_t plane_stride,
                                                const DevConsts& c, uint64_t st_pol = 0) {
    constexpr int kBPerThread = 8;
    constexpr int kMinMod = min_mod_of_bucket(kMaxMod);
    uint32_t xlo[kBPerThread];
#pragma unroll
    for (int u = 0; u < kBPerThread; ++u)
        xlo[u] = static_cast<uint32_t>(__double2loint(__dadd_rn(static_cast<double>(x[u]), kMagic52)));
    // the fast/literal choice is warp-uniform: branch once, outside the modulus
    // loop (a table with 256 anywhere but first — never from select_moduli —
    // takes the literal sequence)
    if (fast && !c.p256_later) {
        // four residues r_u in one word without byte shuffles:
        // xlo_u + qlo_u (-p) = r_u (mod 2^32) with |r_u| <= 127 (p < 256), so
        // sum_u (xlo_u + 128 + qlo_u (-p)) 2^(8u) = sum_u (r_u + 128) 2^(8u)
        // exactly (no carries), and XOR 0x80 per byte leaves r_u mod 256. The
        // modulus-dependent half is (-p) * sum_u qlo_u 2^(8u) (mod 2^32): three
        // shift-adds and ONE multiply by the modulus' constant per word.
        uint32_t xb[2] = {0u, 0u};
#pragma unroll
        for (int u = 0; u < kBPerThread; ++u) xb[u >> 2] += (xlo[u] + 128u) << (8 * (u & 3));
        int8_t* dst = dst0;
        const bool first256 = c.p[0] == 256;  // the tables' first modulus (select_moduli)
#pragma unroll
        for (int t = 0; t < kMaxMod; ++t) {
            if (t >= kMinMod && t >= c.n) break;  // uniform
            uint2 word;
            // p = 256: the residue is the low byte of x (+-128 -> 0x80 either way)
            if (t == 0 && first256) {
                word = make_uint2(pack_low_bytes(xlo[0], xlo[1], xlo[2], xlo[3]),
                                  pack_low_bytes(xlo[4], xlo[5], xlo[6], xlo[7]));
            } else {
                const double pinv = c.pinv64[t];
                const uint32_t negp = c.negp[t];
                uint32_t w[2];
#pragma unroll
                for (int hlf = 0; hlf < 2; ++hlf) {
                    uint32_t q = 0;
#pragma unroll
                    for (int u = 3; u >= 0; --u) {
                        const uint32_t qlo = static_cast<uint32_t>(
                            __double2loint(__fma_rn(static_cast<double>(x[4 * hlf + u]), pinv, kMagic52)));
                        q = (q << 8) + qlo;
                    }
                    w[hlf] = (xb[hlf] + q * negp) ^ 0x80808080u;
                }
                word = make_uint2(w[0], w[1]);
            }
            store_plane8<kHint>(dst, word, st_pol);
            dst += plane_stride;
        }
    } else {
#pragma unroll 1
        for (int t = 0; t < c.n; ++t) {
            uint32_t v[kBPerThread];
#pragma unroll
            for (int u = 0; u < kBPerThread; ++u) v[u] = literal_byte(x[u], c, t);
            store_plane8<kHint>(dst0 + t * plane_stride,
                                make_uint2(pack_low_bytes(v[0], v[1], v[2], v[3]), pack_low_bytes(v[4], v[5], v[6], v[7])),
                                st_pol);
        }
    }
}

// mod_u8 (reconstruct.hpp:31-37): high-half multiply by floor(2^32/p - 1)
// then two one-sided corrections. The true y lies in (-p, 2p), so the 32-bit
// wrapping difference is exact.
__device__ __forceinline__ uint32_t mod_u8(int32_t x, int32_t p, int32_t pinv) {
    const int32_t hi = __mulhi(x, pinv);
    int32_t y = static_cast<int32_t>(static_cast<uint32_t>(x) - static_cast<uint32_t>(hi) * static_cast<uint32_t>(p));
    y = y >= p ? y - p : y;
    y = y < 0 ? y + p : y;
    return static_cast<uint32_t>(y);
}

// scaling.cpp:15,18
__device__ __forceinline__ int magnitude_cap(int prec) { return prec == OZK_FP64 ? 72 : 44; }
__device__ __forceinline__ int exponent_clamp(int prec) { return prec == OZK_FP64 ? 1021 : 125; }

// The fast-mode budget y = pp_fast - max(1, 0.51 log2 ub) of fast_exponent
// (scaling.cpp:50-52), ub = sum_upper_bound(s, k) (scaling.cpp:45-47).
__device__ __forceinline__ double fast_ub(double s, int64_t k) {
    const double factor = __dadd_rn(1.0, __dmul_rn(__dmul_rn(2.0, static_cast<double>(k + 2)), 0x1.0p-53));
    return __dmul_rn(s, factor);
}
__device__ __forceinline__ double fast_budget(double s, int64_t k, float pp_fast) {
    const double l = __dmul_rn(0.51, log2(fast_ub(s, k)));
    const double t = l > 1.0 ? l : 1.0;
    return __dsub_rn(static_cast<double>(pp_fast), t);
}
// floor(pp_fast - max(1, 0.51 log2 ub)) as the reference's host evaluates it
// (glibc log2), from the step table built on the host (FastFloorTable): exact
// for every ub, so no device log2 is involved where the floor is close
__device__ __forceinline__ int fast_floor_table(double ub, const FastFloorTable& T) {
    int f = T.floor0;
#pragma unroll 4
    for (int i = 0; i < T.n; ++i) f -= ub >= T.thr[i] ? 1 : 0;
    return f;
}
// fast_exponent tail (scaling.cpp:52-55); the reference omits the "- g" term
// and so do we, unless OZK_FLAG_FAST_EXPONENT_FIX asks for it.
__device__ __forceinline__ int fast_exponent_from_floor(int fl, int g, int prec, int fix = 0) {
    int e = fl - (fix ? g : 0);
    const int cap = magnitude_cap(prec) - 1 - g;
    e = e < cap ? e : cap;
    const int cl = exponent_clamp(prec);
    return clampi(e, -cl, cl);
}
__device__ __forceinline__ int fast_exponent_from_budget(double y, int g, int prec, int fix = 0) {
    int e = static_cast<int>(floor(y)) - (fix ? g : 0);
    const int cap = magnitude_cap(prec) - 1 - g;
    e = e < cap ? e : cap;
    const int cl = exponent_clamp(prec);
    return clampi(e, -cl, cl);
}

__device__ __forceinline__ double load_as_double(const void* p, int64_t idx, int is_f32) {
    return is_f32 ? static_cast<double>(static_cast<const float*>(p)[idx]) : static_cast<const double*>(p)[idx];
}

}  // namespace ozk
