// K1b — truncation + residue slicing (reference: residue.cpp:7-42,
// residue.hpp:39-53) and the accurate-mode Abar/Bbar operands
// (scaling.cpp:118-133), written straight into the K-major int8 planes the
// tensor-core GEMM consumes.
//
// Data layout in HBM: plane t of A is m rows x ld bytes
// (row i holds a'_i. mod p_t along k, K-major); plane t of B is n rows x ld
// bytes (column j of B along k). ld = round_up(k, 16).
//   * A is column-major, so a 32-row x 128-k tile is read with 256-byte
//     coalesced column segments (one warp = 32 consecutive rows of one
//     column); each thread owns 4 consecutive k of a row, packs its 4 residue
//     bytes into one 32-bit shared-memory word (conflict-free: 33-word row
//     pitch), and the tile leaves as 128-byte row segments. The shared tile is
//     double-buffered so each plane costs one __syncthreads.
//   * B columns are already contiguous along k: each thread reads 4 consecutive
//     elements and writes one 32-bit word per plane (128 B per warp).
// Residues use the exact conversion-free symmetric-residue form where it
// provably equals rmod_fast (ozk_device.cuh), else the literal sequence.
// Each input element is read once and each plane byte written once: the pass
// is HBM-bound at (s + N) bytes per element.
#include <climits>

#include "ozk_device.cuh"

namespace ozk {
namespace {

constexpr int kTileRows = 32;
constexpr int kTileK = 128;
constexpr int kWords = kTileK / 4;            // 32 packed words per tile row
constexpr int kGroups = 256 / kTileRows;      // 8 column-quad groups
constexpr int kQuads = kWords / kGroups;      // 4 quads (16 elements) per thread
constexpr int kBPerThread = 8;                // B elements per thread (8 bytes per plane)

// Abar/Bbar entry (scaling.cpp:124-132): ceil(ldexp(|x|, e)) in [0, 64], with
// the power of two applied as one (correctly rounded) multiply when 2^e is a
// normal double and the ceiling as a round-up add against 2^52.
__device__ __forceinline__ uint32_t bound_entry(double x, int e) {
    if (e == INT32_MIN) return 0;
    const double v = (e >= -1022 && e <= 1023) ? __dmul_rn(fabs(x), pow2d(e)) : ldexp(fabs(x), e);
    return static_cast<uint32_t>(__double2loint(__dadd_ru(v, 0x1.0p52))) & 0xffu;
}

template <typename T>
__device__ __forceinline__ uint32_t literal_byte(T x, const DevConsts& c, int t) {
    return static_cast<uint32_t>(static_cast<uint8_t>(rmod_fast(x, c.p[t], c.pinv64[t], c.pinv32[t], c.n)));
}

template <typename T, int KIND>
__global__ void __launch_bounds__(256)
    a_planes_kernel(const T* __restrict__ a, int64_t m, int64_t k, int64_t lda, const int32_t* __restrict__ row_exp,
                    const DevConsts c, int8_t* __restrict__ planes, int64_t ld, int64_t plane_stride) {
    __shared__ uint32_t tile[2][kTileRows][kWords + 1];
    // per-modulus constants staged in shared memory: a rolled modulus loop keeps
    // the code small (a 20-way unroll thrashed the instruction cache) and
    // broadcast LDS avoids dynamically indexed constant-bank loads
    __shared__ double s_pinv[OZK_MAX_MODULI];
    __shared__ uint32_t s_p[OZK_MAX_MODULI];
    if (threadIdx.x < OZK_MAX_MODULI) {
        s_pinv[threadIdx.x] = c.pinv64[threadIdx.x];
        s_p[threadIdx.x] = static_cast<uint32_t>(c.p[threadIdx.x]);
    }
    const int r = threadIdx.x % kTileRows, g = threadIdx.x / kTileRows;
    const int64_t row = static_cast<int64_t>(blockIdx.y) * kTileRows + r;
    const int64_t k0 = static_cast<int64_t>(blockIdx.x) * kTileK;
    const bool row_ok = row < m;
    const int e = row_ok ? row_exp[row] : 0;

    T x[kQuads * 4];
    bool fast = true;
#pragma unroll
    for (int q = 0; q < kQuads; ++q)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t col = k0 + 4 * (g + kGroups * q) + u;
            const T v = (row_ok && col < k) ? a[row + col * lda] : T(0);
            if constexpr (KIND == 0) {
                x[4 * q + u] = trunc_scaled(v, e);
                fast &= symmetric_residue_domain(static_cast<double>(x[4 * q + u]), c.precision, c.n);
            } else {
                x[4 * q + u] = v;
            }
        }
    fast = __all_sync(0xffffffffu, fast);
    __syncthreads();  // s_p / s_pinv
    uint32_t xlo[KIND == 0 ? kQuads * 4 : 1];
    if constexpr (KIND == 0) {
#pragma unroll
        for (int i = 0; i < kQuads * 4; ++i)
            xlo[i] = static_cast<uint32_t>(__double2loint(__dadd_rn(static_cast<double>(x[i]), kMagic52)));
    }

    const int nplanes = KIND == 0 ? c.n : 1;
#pragma unroll 1
    for (int t = 0; t < nplanes; ++t) {
        uint32_t(*buf)[kWords + 1] = tile[t & 1];
        const uint32_t pt = s_p[t];
        const double pinvt = s_pinv[t];
#pragma unroll
        for (int q = 0; q < kQuads; ++q) {
            uint32_t v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = 4 * q + u;
                if constexpr (KIND == 0) {
                    if (fast && pt == 256)  // p = 256: the residue is the low byte of x
                        v[u] = xlo[i];
                    else
                        v[u] = fast ? symmetric_residue(static_cast<double>(x[i]), xlo[i], pt, pinvt)
                                    : literal_byte(x[i], c, t);
                } else {
                    v[u] = bound_entry(static_cast<double>(x[i]), e);
                }
            }
            buf[r][g + kGroups * q] = pack_low_bytes(v[0], v[1], v[2], v[3]);
        }
        __syncthreads();
        int8_t* dst = planes + t * plane_stride;
#pragma unroll
        for (int it = 0; it < (kTileRows * kWords) / 256; ++it) {
            const int idx = it * 256 + threadIdx.x;
            const int rr = idx / kWords, w = idx % kWords;
            const int64_t grow = static_cast<int64_t>(blockIdx.y) * kTileRows + rr;
            const int64_t gcol = k0 + 4 * w;
            if (grow < m && gcol < ld) *reinterpret_cast<uint32_t*>(dst + grow * ld + gcol) = buf[rr][w];
        }
        // the next plane writes the other buffer; its previous readers finished
        // before this iteration's barrier
    }
}

template <typename T, int KIND>
__global__ void __launch_bounds__(128)
    b_planes_kernel(const T* __restrict__ b, int64_t k, int64_t n, int64_t ldb, const int32_t* __restrict__ col_exp,
                    const DevConsts c, int8_t* __restrict__ planes, int64_t ld, int64_t plane_stride) {
    __shared__ double s_pinv[OZK_MAX_MODULI];
    __shared__ uint32_t s_p[OZK_MAX_MODULI];
    if (threadIdx.x < OZK_MAX_MODULI) {
        s_pinv[threadIdx.x] = c.pinv64[threadIdx.x];
        s_p[threadIdx.x] = static_cast<uint32_t>(c.p[threadIdx.x]);
    }
    const int64_t j = blockIdx.x;
    const int64_t i0 = (static_cast<int64_t>(blockIdx.y) * blockDim.x + threadIdx.x) * kBPerThread;
    const bool active = i0 < ld;
    const int e = col_exp[j];
    const T* col = b + j * ldb;
    T x[kBPerThread];
    bool fast = true;
#pragma unroll
    for (int u = 0; u < kBPerThread; ++u) {
        const int64_t i = i0 + u;
        const T v = (active && i < k) ? col[i] : T(0);
        if constexpr (KIND == 0) {
            x[u] = trunc_scaled(v, e);
            fast &= symmetric_residue_domain(static_cast<double>(x[u]), c.precision, c.n);
        } else {
            x[u] = v;
        }
    }
    fast = __all_sync(0xffffffffu, fast);
    __syncthreads();  // s_p / s_pinv
    // ld is a multiple of 16, so a thread's 8 bytes are either all in [0, ld) or all past it
    if (!active) return;
    int8_t* dst0 = planes + j * ld + i0;
    if constexpr (KIND == 1) {
        uint32_t v[kBPerThread];
#pragma unroll
        for (int u = 0; u < kBPerThread; ++u) v[u] = bound_entry(static_cast<double>(x[u]), e);
        *reinterpret_cast<uint2*>(dst0) = make_uint2(pack_low_bytes(v[0], v[1], v[2], v[3]),
                                                     pack_low_bytes(v[4], v[5], v[6], v[7]));
        return;
    }
    uint32_t xlo[kBPerThread];
#pragma unroll
    for (int u = 0; u < kBPerThread; ++u)
        xlo[u] = static_cast<uint32_t>(__double2loint(__dadd_rn(static_cast<double>(x[u]), kMagic52)));
#pragma unroll 1
    for (int t = 0; t < c.n; ++t) {
        const uint32_t pt = s_p[t];
        const double pinvt = s_pinv[t];
        uint32_t v[kBPerThread];
#pragma unroll
        for (int u = 0; u < kBPerThread; ++u) {
            if (fast && pt == 256)
                v[u] = xlo[u];
            else
                v[u] = fast ? symmetric_residue(static_cast<double>(x[u]), xlo[u], pt, pinvt) : literal_byte(x[u], c, t);
        }
        *reinterpret_cast<uint2*>(dst0 + t * plane_stride) =
            make_uint2(pack_low_bytes(v[0], v[1], v[2], v[3]), pack_low_bytes(v[4], v[5], v[6], v[7]));
    }
}

__global__ void round_to_f32_kernel(const double* __restrict__ x, int64_t rows, int64_t cols, int64_t ld,
                                    float* __restrict__ out) {
    const int64_t total = rows * cols;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e % rows, j = e / rows;
        out[e] = __double2float_rn(x[i + j * ld]);
    }
}

template <int KIND>
void a_planes_dispatch(const void* a, int is_f32, int64_t m, int64_t k, int64_t lda, const int32_t* row_exp,
                       const DevConsts& c, int8_t* planes, int64_t ld, cudaStream_t s) {
    dim3 grid(static_cast<unsigned>((k + kTileK - 1) / kTileK), static_cast<unsigned>((m + kTileRows - 1) / kTileRows));
    const int64_t stride = m * ld;
    if (is_f32)
        a_planes_kernel<float, KIND><<<grid, 256, 0, s>>>(static_cast<const float*>(a), m, k, lda, row_exp, c, planes,
                                                          ld, stride);
    else
        a_planes_kernel<double, KIND><<<grid, 256, 0, s>>>(static_cast<const double*>(a), m, k, lda, row_exp, c,
                                                           planes, ld, stride);
}

template <int KIND>
void b_planes_dispatch(const void* b, int is_f32, int64_t k, int64_t n, int64_t ldb, const int32_t* col_exp,
                       const DevConsts& c, int8_t* planes, int64_t ld, int64_t stride, cudaStream_t s) {
    dim3 grid(static_cast<unsigned>(n), static_cast<unsigned>((ld + 128 * kBPerThread - 1) / (128 * kBPerThread)));
    if (is_f32)
        b_planes_kernel<float, KIND><<<grid, 128, 0, s>>>(static_cast<const float*>(b), k, n, ldb, col_exp, c, planes,
                                                          ld, stride);
    else
        b_planes_kernel<double, KIND><<<grid, 128, 0, s>>>(static_cast<const double*>(b), k, n, ldb, col_exp, c,
                                                           planes, ld, stride);
}

}  // namespace

void launch_a_planes(const void* a, int is_f32, int64_t m, int64_t k, int64_t lda, const int32_t* row_exp,
                     const DevConsts& c, int kind, int8_t* planes, int64_t ld, cudaStream_t s) {
    if (kind == 0)
        a_planes_dispatch<0>(a, is_f32, m, k, lda, row_exp, c, planes, ld, s);
    else
        a_planes_dispatch<1>(a, is_f32, m, k, lda, row_exp, c, planes, ld, s);
}

void launch_b_planes(const void* b, int is_f32, int64_t k, int64_t n, int64_t ldb, const int32_t* col_exp,
                     const DevConsts& c, int kind, int8_t* planes, int64_t ld, int64_t plane_stride, cudaStream_t s) {
    if (kind == 0)
        b_planes_dispatch<0>(b, is_f32, k, n, ldb, col_exp, c, planes, ld, plane_stride, s);
    else
        b_planes_dispatch<1>(b, is_f32, k, n, ldb, col_exp, c, planes, ld, plane_stride, s);
}

void launch_round_to_f32(const double* x, int64_t rows, int64_t cols, int64_t ld, float* out, cudaStream_t s) {
    round_to_f32_kernel<<<148 * 8, 256, 0, s>>>(x, rows, cols, ld, out);
}

}  // namespace ozk
