// K1b — truncation + residue slicing (reference: residue.cpp:7-42,
// residue.hpp:39-53) and the accurate-mode Abar/Bbar operands
// (scaling.cpp:118-133), written straight into the K-major int8 planes the
// tensor-core GEMM consumes.
//
// Data layout in HBM: every plane keeps its operand's
// column-major layout, with the leading dimension padded to 16 bytes (a TMA
// stride rule): plane t of A is k columns x ld_a = round_up(m, 16) bytes (the
// GEMM reads A MN-major), plane t of B is n columns x ld_b = round_up(k, 16)
// bytes (read K-major). So both operands stream through the same kernel: each
// thread reads 8 consecutive elements of one column (64 B of FP64, a warp
// covers 2 KB contiguous) and writes 8 bytes per plane (256 B per warp) — no
// transpose, no shared-memory staging.
// Residues use the exact conversion-free symmetric-residue form where it
// provably equals rmod_fast (ozk_device.cuh), else the literal sequence.
// Each input element is read once and each plane byte written once: the pass
// is HBM-bound at (s + N) bytes per element.
#include <climits>

#include "ozk_device.cuh"

namespace ozk {
namespace {

constexpr int kBPerThread = 8;  // elements per thread (8 bytes per plane)

// Abar/Bbar entry (scaling.cpp:124-132): ceil(ldexp(|x|, e)) in [0, 64], with
// the power of two applied as one (correctly rounded) multiply when 2^e is a
// normal double and the ceiling as a round-up add against 2^52.
__device__ __forceinline__ uint32_t bound_entry(double x, int e) {
    if (e == INT32_MIN) return 0;
    const double v = (e >= -1022 && e <= 1023) ? __dmul_rn(fabs(x), pow2d(e)) : ldexp(fabs(x), e);
    return static_cast<uint32_t>(__double2loint(__dadd_ru(v, 0x1.0p52))) & 0xffu;
}

// 8 consecutive values from a 32-byte aligned address (read-only path)
__device__ __forceinline__ void load8(const double* p, double (&v)[8]) {
    asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
                 : "l"(p));
    asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(v[4]), "=d"(v[5]), "=d"(v[6]), "=d"(v[7])
                 : "l"(p + 4));
}
__device__ __forceinline__ void load8(const float* p, float (&v)[8]) {
    asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "l"(p));
}
__device__ __forceinline__ void load8(const int32_t* p, int (&v)[8]) {
    asm volatile("ld.global.nc.v8.s32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "l"(p));
}

// elements [i0, i0 + 8) of a line and (ROW_EXP) their exponents, zeros past len
template <typename T, bool ROW_EXP>
__device__ __forceinline__ void load8_guarded(const T* col, const int32_t* exps, int64_t i0, int64_t len, T (&v)[8],
                                           int (&ev)[8]) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const bool ok = i0 + u < len;
        v[u] = ok ? col[i0 + u] : T(0);
        ev[u] = ROW_EXP && ok ? exps[i0 + u] : 0;
    }
}

// Column-major rows x cols input -> N column-major int8 planes (ld bytes per
// column, plane_stride bytes apart). ROW_EXP: the scale exponent is per row
// (A: mu), else per column (B: nu). Each thread handles 8 consecutive rows of
// one column: 64 (FP64) contiguous bytes in, 8 bytes out per plane.
// kMaxMod: the modulus count rounded up to a bucket (8/12/14/16/20): the
// modulus loop is unrolled, so p_t and 1/p_t are constant-bank operands of the
// DFMA / IMAD and the plane address advances by one add per modulus.
template <typename T, int KIND, bool ROW_EXP, int kMaxMod>
__global__ void __launch_bounds__(128)
    planes_kernel(const T* __restrict__ b, int64_t k, int64_t n, int64_t ldb, const int32_t* __restrict__ exps,
                  const DevConsts c, int8_t* __restrict__ planes, int64_t ld, int64_t plane_stride, int64_t extent) {
    const int64_t j = blockIdx.x;
    const int64_t i0 = (static_cast<int64_t>(blockIdx.y) * blockDim.x + threadIdx.x) * kBPerThread;
    const bool active = i0 < extent;  // rows up to plane_ld(rows): the zero padding K2's 16-byte rows need
    const int e = ROW_EXP ? 0 : exps[j];
    const T* col = b + j * ldb;
    T x[kBPerThread];
    int ex[ROW_EXP ? kBPerThread : 1];
    bool fast = true;
    // whole, 32-byte aligned runs: 256-bit loads of the 8 elements (and of
    // their 8 row exponents) instead of 8 + 8 scalar ones
    T vin[kBPerThread];
    int ein[kBPerThread];
    const bool vec = active && i0 + kBPerThread <= k && (reinterpret_cast<uintptr_t>(col + i0) & 31) == 0 &&
                     (!ROW_EXP || (reinterpret_cast<uintptr_t>(exps + i0) & 31) == 0);
    if (vec) {
        load8(col + i0, vin);
        if constexpr (ROW_EXP) load8(exps + i0, ein);
    } else {
        // ragged / unaligned run (a real branch, not 16 predicated loads on the
        // common path: that cost ~8 instructions per element in every thread)
        load8_guarded<T, ROW_EXP>(col, exps, i0, active ? k : 0, vin, ein);
    }
#pragma unroll
    for (int u = 0; u < kBPerThread; ++u) {
        const T v = vin[u];
        const int eu = ROW_EXP ? ein[u] : e;
        if constexpr (ROW_EXP) ex[u] = eu;
        if constexpr (KIND == 0) {
            x[u] = trunc_scaled(v, eu);
            // the residue sequence follows the element type (residue.hpp:39-53 overloads
            // rmod_fast on T), the tables may be of either precision
            fast &= symmetric_residue_domain(static_cast<double>(x[u]), sizeof(T) == 4 ? OZK_FP32 : OZK_FP64, c.n);
        } else {
            x[u] = v;
        }
    }
    fast = __all_sync(0xffffffffu, fast);
    // extent is a multiple of 16, so a thread's 8 bytes are either all in [0, extent) or all past it
    if (!active) return;
    int8_t* dst0 = planes + j * ld + i0;
    if constexpr (KIND == 1) {
        uint32_t v[kBPerThread];
#pragma unroll
        for (int u = 0; u < kBPerThread; ++u) v[u] = bound_entry(static_cast<double>(x[u]), ROW_EXP ? ex[u] : e);
        *reinterpret_cast<uint2*>(dst0) = make_uint2(pack_low_bytes(v[0], v[1], v[2], v[3]),
                                                     pack_low_bytes(v[4], v[5], v[6], v[7]));
        return;
    }
    residue_planes8<T, kMaxMod>(x, fast, dst0, plane_stride, c);
}

__global__ void round_to_f32_kernel(const double* __restrict__ x, int64_t rows, int64_t cols, int64_t ld,
                                    float* __restrict__ out, int64_t ldo) {
    const int64_t total = rows * cols;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e % rows, j = e / rows;
        out[i + j * ldo] = __double2float_rn(x[i + j * ld]);
    }
}

template <int KIND, bool ROW_EXP>
void planes_dispatch(const void* x, int is_f32, int64_t rows, int64_t cols, int64_t ldx, const int32_t* exps,
                     const DevConsts& c, int8_t* planes, int64_t ld, int64_t stride, cudaStream_t s) {
    // only rows [0, plane_ld(rows)) are written: a column block of an MN-major
    // plane (ld > rows) must not touch its neighbours
    const int64_t extent = plane_ld(rows);
    dim3 grid(static_cast<unsigned>(cols),
              static_cast<unsigned>((extent + 128 * kBPerThread - 1) / (128 * kBPerThread)));
#define OZK_K1B(MAXN)                                                                                            \
    do {                                                                                                         \
        if (is_f32)                                                                                              \
            planes_kernel<float, KIND, ROW_EXP, MAXN><<<grid, 128, 0, s>>>(static_cast<const float*>(x), rows,   \
                                                                           cols, ldx, exps, c, planes, ld,       \
                                                                           stride, extent);                      \
        else                                                                                                     \
            planes_kernel<double, KIND, ROW_EXP, MAXN><<<grid, 128, 0, s>>>(static_cast<const double*>(x), rows, \
                                                                            cols, ldx, exps, c, planes, ld,      \
                                                                            stride, extent);                     \
    } while (0)
    if (KIND == 1 || c.n <= 8)  // the bound planes have no modulus loop
        OZK_K1B(8);
    else if (c.n <= 12)
        OZK_K1B(12);
    else if (c.n <= 14)
        OZK_K1B(14);
    else if (c.n <= 16)
        OZK_K1B(16);
    else
        OZK_K1B(OZK_MAX_MODULI);
#undef OZK_K1B
}

}  // namespace

// A planes are column-major like A (MN-major operand of the GEMM): ld = plane_ld(m)
void launch_a_planes(const void* a, int is_f32, int64_t m, int64_t k, int64_t lda, const int32_t* row_exp,
                     const DevConsts& c, int kind, int8_t* planes, int64_t ld, int64_t plane_stride, cudaStream_t s) {
    if (kind == 0)
        planes_dispatch<0, true>(a, is_f32, m, k, lda, row_exp, c, planes, ld, plane_stride, s);
    else
        planes_dispatch<1, true>(a, is_f32, m, k, lda, row_exp, c, planes, ld, plane_stride, s);
}

// B planes are column-major like B (K-major operand of the GEMM): ld = plane_ld(k)
void launch_b_planes(const void* b, int is_f32, int64_t k, int64_t n, int64_t ldb, const int32_t* col_exp,
                     const DevConsts& c, int kind, int8_t* planes, int64_t ld, int64_t plane_stride, cudaStream_t s) {
    if (kind == 0)
        planes_dispatch<0, false>(b, is_f32, k, n, ldb, col_exp, c, planes, ld, plane_stride, s);
    else
        planes_dispatch<1, false>(b, is_f32, k, n, ldb, col_exp, c, planes, ld, plane_stride, s);
}

void launch_round_to_f32(const double* x, int64_t rows, int64_t cols, int64_t ld, float* out, int64_t ldo,
                         cudaStream_t s) {
    round_to_f32_kernel<<<148 * 8, 256, 0, s>>>(x, rows, cols, ld, out, ldo);
}

}  // namespace ozk
