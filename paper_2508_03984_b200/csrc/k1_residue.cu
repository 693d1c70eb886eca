// K1b — truncation + residue slicing (reference: residue.cpp:7-42,
// residue.hpp:39-53) and the accurate-mode Abar/Bbar operands
// (scaling.cpp:118-133), written straight into the K-major int8 planes the
// tensor-core GEMM consumes.
//
// Data layout in HBM: plane t of A is m rows x ld bytes
// (row i holds a'_i. mod p_t along k, K-major); plane t of B is n rows x ld
// bytes (column j of B along k). ld = round_up(k, 16).
//   * A is column-major, so a 64-row x 128-k tile is read with 256-byte
//     coalesced column segments, transposed through shared memory one plane at
//     a time, and written back as 128-byte row segments.
//   * B columns are already contiguous along k: each thread reads 4 consecutive
//     elements and writes one 32-bit word per plane (128 B per warp).
// Each input element is read once per call of this pass and every plane byte
// written once, so the pass is HBM-bound at (s + N) bytes per element.
#include <climits>

#include "ozk_device.cuh"

namespace ozk {
namespace {

constexpr int kTileRows = 64;
constexpr int kTileK = 128;
constexpr int kPerThread = kTileK / 4;  // 4 column groups x 32 columns

// Abar/Bbar entry (scaling.cpp:124-132): ceil(ldexp(|x|, e)) in [0, 64].
__device__ __forceinline__ int8_t bound_entry(double x, int e) {
    if (e == INT32_MIN) return 0;
    return static_cast<int8_t>(ceil(ldexp(fabs(x), e)));
}

template <typename T, int KIND>
__global__ void __launch_bounds__(256)
    a_planes_kernel(const T* __restrict__ a, int64_t m, int64_t k, int64_t lda, const int32_t* __restrict__ row_exp,
                    const DevConsts c, int8_t* __restrict__ planes, int64_t ld, int64_t plane_stride) {
    __shared__ uint32_t tile[kTileRows][kTileK / 4 + 1];  // +1 word: conflict-free byte column writes
    uint8_t* tb = reinterpret_cast<uint8_t*>(&tile[0][0]);
    constexpr int kRowBytes = (kTileK / 4 + 1) * 4;

    const int r = threadIdx.x % kTileRows, g = threadIdx.x / kTileRows;
    const int64_t row = static_cast<int64_t>(blockIdx.y) * kTileRows + r;
    const int64_t k0 = static_cast<int64_t>(blockIdx.x) * kTileK;
    const bool row_ok = row < m;
    const int e = row_ok ? row_exp[row] : 0;

    T x[kPerThread];
    int8_t bar[KIND == 1 ? kPerThread : 1];
#pragma unroll
    for (int q = 0; q < kPerThread; ++q) {
        const int64_t col = k0 + g + 4 * q;
        const bool ok = row_ok && col < k;
        const T v = ok ? a[row + col * lda] : T(0);
        if constexpr (KIND == 0)
            x[q] = trunc_scaled(v, e);
        else
            bar[q] = ok ? bound_entry(static_cast<double>(v), e) : int8_t(0);
    }
    const int nplanes = KIND == 0 ? c.n : 1;
    for (int t = 0; t < nplanes; ++t) {
#pragma unroll
        for (int q = 0; q < kPerThread; ++q) {
            int8_t v;
            if constexpr (KIND == 0)
                v = rmod_fast(x[q], c.p[t], c.pinv64[t], c.pinv32[t], c.n);
            else
                v = bar[q];
            tb[r * kRowBytes + g + 4 * q] = static_cast<uint8_t>(v);
        }
        __syncthreads();
        int8_t* dst = planes + t * plane_stride;
#pragma unroll
        for (int q = 0; q < (kTileRows * kTileK / 4) / 256; ++q) {
            const int idx = q * 256 + threadIdx.x;
            const int rr = idx / (kTileK / 4), w = idx % (kTileK / 4);
            const int64_t grow = static_cast<int64_t>(blockIdx.y) * kTileRows + rr;
            const int64_t gcol = k0 + 4 * w;
            if (grow < m && gcol < ld) *reinterpret_cast<uint32_t*>(dst + grow * ld + gcol) = tile[rr][w];
        }
        __syncthreads();
    }
}

template <typename T, int KIND>
__global__ void __launch_bounds__(128)
    b_planes_kernel(const T* __restrict__ b, int64_t k, int64_t n, int64_t ldb, const int32_t* __restrict__ col_exp,
                    const DevConsts c, int8_t* __restrict__ planes, int64_t ld, int64_t plane_stride) {
    const int64_t j = blockIdx.x;
    const int64_t i0 = (static_cast<int64_t>(blockIdx.y) * blockDim.x + threadIdx.x) * 4;
    if (i0 >= ld) return;
    const int e = col_exp[j];
    const T* col = b + j * ldb;
    T x[4];
    int8_t bar[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + u;
        const T v = i < k ? col[i] : T(0);
        if constexpr (KIND == 0)
            x[u] = trunc_scaled(v, e);
        else
            bar[u] = i < k ? bound_entry(static_cast<double>(v), e) : int8_t(0);
    }
    const int nplanes = KIND == 0 ? c.n : 1;
    for (int t = 0; t < nplanes; ++t) {
        uint32_t word = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            int8_t v;
            if constexpr (KIND == 0)
                v = rmod_fast(x[u], c.p[t], c.pinv64[t], c.pinv32[t], c.n);
            else
                v = bar[u];
            word |= static_cast<uint32_t>(static_cast<uint8_t>(v)) << (8 * u);
        }
        *reinterpret_cast<uint32_t*>(planes + t * plane_stride + j * ld + i0) = word;
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
                       const DevConsts& c, int8_t* planes, int64_t ld, cudaStream_t s) {
    dim3 grid(static_cast<unsigned>(n), static_cast<unsigned>((ld + 511) / 512));
    const int64_t stride = n * ld;
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
                     const DevConsts& c, int kind, int8_t* planes, int64_t ld, cudaStream_t s) {
    if (kind == 0)
        b_planes_dispatch<0>(b, is_f32, k, n, ldb, col_exp, c, planes, ld, s);
    else
        b_planes_dispatch<1>(b, is_f32, k, n, ldb, col_exp, c, planes, ld, s);
}

void launch_round_to_f32(const double* x, int64_t rows, int64_t cols, int64_t ld, float* out, cudaStream_t s) {
    round_to_f32_kernel<<<148 * 8, 256, 0, s>>>(x, rows, cols, ld, out);
}

}  // namespace ozk
