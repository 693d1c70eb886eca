// Element-wise device kernels behind the reference's public stage helpers
// (truncate_scale, to_residue_slices, reduce_products_u8, accumulate,
// crt_reduce, unscale — residue.hpp:31-62, reconstruct.hpp:43-59). The fused
// pipeline never calls these; they let a caller of the reference's stage-level
// API (its tests, SPEC.md's harness) run each stage on the GPU, bit-identically.
#include "ozk_device.cuh"

namespace ozk {
namespace {

constexpr int kThreads = 256;

unsigned blocks_for(int64_t count) {
    const int64_t b = (count + kThreads - 1) / kThreads;
    return static_cast<unsigned>(b < (int64_t(1) << 30) ? b : (int64_t(1) << 30));
}

template <typename T>
__global__ void truncate_kernel(const T* __restrict__ x, int64_t rows, int64_t cols, int64_t ldx,
                                const int32_t* __restrict__ se, int side, T* __restrict__ out, int64_t ldo) {
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < rows * cols;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e % rows, j = e / rows;
        out[i + j * ldo] = trunc_scaled(x[i + j * ldx], side == 0 ? se[i] : se[j]);
    }
}

// rmod_fast of every entry as given (residue.cpp:36-38): the literal reference
// sequence, so non-integer inputs behave exactly like the reference too
template <typename T>
__global__ void residues_kernel(const T* __restrict__ x, int64_t rows, int64_t cols, int64_t ldx, const DevConsts c,
                                int8_t* __restrict__ planes, int64_t ldp) {
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < rows * cols;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e % rows, j = e / rows;
        const T v = x[i + j * ldx];
        for (int t = 0; t < c.n; ++t)
            planes[t * cols * ldp + j * ldp + i] = rmod_fast(v, c.p[t], c.pinv64[t], c.pinv32[t], c.n);
    }
}

__global__ void mod_u8_kernel(const int32_t* __restrict__ x, int64_t count, int32_t p, int32_t pinv,
                              uint8_t* __restrict__ out) {
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < count;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[e] = static_cast<uint8_t>(mod_u8(x[e], p, pinv));
}

// accumulate (reconstruct.cpp:22-38): mul then add per term, index ascending
__global__ void accumulate_kernel(const uint8_t* __restrict__ u, int64_t count, const DevConsts c,
                                  double* __restrict__ c1, double* __restrict__ c2) {
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < count;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double a = 0.0, b = 0.0;
        for (int t = 0; t < c.n; ++t) {
            const double v = static_cast<double>(u[t * count + e]);
            a = __dadd_rn(a, __dmul_rn(c.s1[t], v));
            b = __dadd_rn(b, __dmul_rn(c.s2[t], v));
        }
        c1[e] = a;
        c2[e] = b;
    }
}

// crt_reduce_element (reconstruct.hpp:51-54)
__global__ void crt_reduce_kernel(const double* __restrict__ c1, const double* __restrict__ c2, int64_t count,
                                  const DevConsts c, double* __restrict__ out) {
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < count;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double q = rint(__dmul_rn(c.P_inv, c1[e]));
        out[e] = __fma_rn(-c.P2, q, __dadd_rn(__fma_rn(-c.P1, q, c1[e]), c2[e]));
    }
}

// unscale (reconstruct.cpp:49-69)
__global__ void unscale_kernel(const double* __restrict__ cpp, int64_t m, int64_t n, int64_t ldc,
                               const int32_t* __restrict__ mu, const int32_t* __restrict__ nu,
                               double* __restrict__ out, int64_t ldo) {
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < m * n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e % m, j = e / m;
        out[i + j * ldo] = ldexp(cpp[i + j * ldc], -(mu[i] + nu[j]));
    }
}

// int8_gemm_reference (int8_engine.cpp:66-80): the reference's plain triple
// loop, one thread per C entry on the CUDA cores, uint32 wrapping sum in
// index order. Deliberately independent of the tensor-core engine (K2), so a
// caller cross-checking int8_gemm against it compares two implementations.
__global__ void int8_gemm_simple_kernel(const int8_t* __restrict__ a, const int8_t* __restrict__ b, int64_t m,
                                        int64_t n, int64_t k, int64_t lda, int64_t ldb, int32_t* __restrict__ c,
                                        int64_t ldc) {
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < m * n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e % m, j = e / m;
        uint32_t s = 0;
        for (int64_t h = 0; h < k; ++h)
            s += static_cast<uint32_t>(static_cast<int32_t>(a[i + h * lda]) * static_cast<int32_t>(b[h + j * ldb]));
        c[i + j * ldc] = static_cast<int32_t>(s);
    }
}

// row / column maxima of the int64 bound product (k > 2^19): one block per column
__global__ void bound_max64_kernel(const long long* __restrict__ cbar, int64_t m, int64_t ld,
                                   unsigned long long* __restrict__ rowmax, unsigned long long* __restrict__ colmax) {
    const int64_t j = blockIdx.x;
    unsigned long long cm = 0;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
        const unsigned long long v = static_cast<unsigned long long>(cbar[i + j * ld]);  // >= 0
        cm = v > cm ? v : cm;
        atomicMax(rowmax + i, v);
    }
    for (int o = 16; o; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(0xffffffffu, cm, o);
        cm = x > cm ? x : cm;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(colmax + j, cm);
}

}  // namespace

void launch_bound_max64(const long long* cbar, int64_t m, int64_t n, int64_t ld, unsigned long long* rowmax,
                        unsigned long long* colmax, cudaStream_t s) {
    bound_max64_kernel<<<static_cast<unsigned>(n), kThreads, 0, s>>>(cbar, m, ld, rowmax, colmax);
}

void launch_int8_gemm_simple(const int8_t* a, const int8_t* b, int64_t m, int64_t n, int64_t k, int64_t lda,
                             int64_t ldb, int32_t* c, int64_t ldc, cudaStream_t s) {
    int8_gemm_simple_kernel<<<blocks_for(m * n), kThreads, 0, s>>>(a, b, m, n, k, lda, ldb, c, ldc);
}

void launch_truncate(int is_f32, const void* x, int64_t rows, int64_t cols, int64_t ldx, const int32_t* se, int side,
                     void* out, int64_t ldo, cudaStream_t s) {
    if (is_f32)
        truncate_kernel<float><<<blocks_for(rows * cols), kThreads, 0, s>>>(
            static_cast<const float*>(x), rows, cols, ldx, se, side, static_cast<float*>(out), ldo);
    else
        truncate_kernel<double><<<blocks_for(rows * cols), kThreads, 0, s>>>(
            static_cast<const double*>(x), rows, cols, ldx, se, side, static_cast<double*>(out), ldo);
}

void launch_residues_literal(int is_f32, const void* x, int64_t rows, int64_t cols, int64_t ldx, const DevConsts& c,
                             int8_t* planes, int64_t ldp, cudaStream_t s) {
    if (is_f32)
        residues_kernel<float><<<blocks_for(rows * cols), kThreads, 0, s>>>(static_cast<const float*>(x), rows, cols,
                                                                            ldx, c, planes, ldp);
    else
        residues_kernel<double><<<blocks_for(rows * cols), kThreads, 0, s>>>(static_cast<const double*>(x), rows,
                                                                             cols, ldx, c, planes, ldp);
}

void launch_mod_u8(const int32_t* x, int64_t count, int32_t p, int32_t pinv, uint8_t* out, cudaStream_t s) {
    mod_u8_kernel<<<blocks_for(count), kThreads, 0, s>>>(x, count, p, pinv, out);
}

void launch_accumulate(const uint8_t* u, int64_t count, const DevConsts& c, double* c1, double* c2, cudaStream_t s) {
    accumulate_kernel<<<blocks_for(count), kThreads, 0, s>>>(u, count, c, c1, c2);
}

void launch_crt_reduce(const double* c1, const double* c2, int64_t count, const DevConsts& c, double* out,
                       cudaStream_t s) {
    crt_reduce_kernel<<<blocks_for(count), kThreads, 0, s>>>(c1, c2, count, c, out);
}

void launch_unscale(const double* cpp, int64_t m, int64_t n, int64_t ldc, const int32_t* mu, const int32_t* nu,
                    double* out, int64_t ldo, cudaStream_t s) {
    unscale_kernel<<<blocks_for(m * n), kThreads, 0, s>>>(cpp, m, n, ldc, mu, nu, out, ldo);
}

}  // namespace ozk
