// K1a — scale exponents (reference: scaling.cpp:20-184).
//
// Memory-bound reductions over the FP64/FP32 inputs, one HBM read of A and of
// B per pass:
//   * row_stats  : per row of column-major A, max|a| and sum a^2 (partial per
//                  k-split), 64 rows x 8 B = 512 B coalesced per column;
//   * col_stats  : per column of B, one warp streams the contiguous column;
//   * finalize   : fast mode evaluates the budget of fast_exponent
//                  (scaling.cpp:50-56) from the order-free sum and FLAGS every
//                  line whose floor() argument lies within `guard` of an
//                  integer (or whose magnitude leaves the a^2-safe range);
//   * exact      : flagged lines are recomputed in the reference's sequential
//                  order (scaling.cpp:69-78 rows, :90-94 columns) — products in
//                  parallel across a warp, the additions strictly in index
//                  order on lane 0 — so mu/nu are bit-identical to the
//                  reference (the floor can only differ inside the guard band).
//   * accurate   : mu'/nu' = 2^(5 - ilogb max) (scaling.cpp:110-116) and, after
//                  the Abar*Bbar bound GEMM (K2 with the max epilogue), the
//                  budget of scaling.cpp:151-165.
#include <cfloat>
#include <climits>

#include "ozk_device.cuh"

namespace ozk {
namespace {

constexpr int kRowTile = 64;  // rows per block in row_stats
constexpr int kColGroups = 4; // column groups per block in row_stats

__global__ void __launch_bounds__(kRowTile* kColGroups)
    row_stats_kernel(const void* __restrict__ a, int is_f32, int64_t m, int64_t k, int64_t lda, int64_t k_per_split,
                     double* __restrict__ pmax, double* __restrict__ psum, int32_t* __restrict__ nonfinite) {
    __shared__ double smax[kColGroups][kRowTile];
    __shared__ double ssum[kColGroups][kRowTile];
    const int r = threadIdx.x % kRowTile, g = threadIdx.x / kRowTile;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * kRowTile + r;
    const int64_t j0 = static_cast<int64_t>(blockIdx.y) * k_per_split;
    const int64_t j1 = j0 + k_per_split < k ? j0 + k_per_split : k;
    double mx = 0.0, s0 = 0.0, s1 = 0.0;
    if (row < m) {
        int64_t j = j0 + g;
        if (is_f32) {
            const float* p = static_cast<const float*>(a) + row;
            for (; j + kColGroups < j1; j += 2 * kColGroups) {
                const double x0 = p[j * lda], x1 = p[(j + kColGroups) * lda];
                mx = fmax(mx, fmax(fabs(x0), fabs(x1)));
                s0 = __fma_rn(x0, x0, s0);
                s1 = __fma_rn(x1, x1, s1);
            }
            for (; j < j1; j += kColGroups) {
                const double x0 = p[j * lda];
                mx = fmax(mx, fabs(x0));
                s0 = __fma_rn(x0, x0, s0);
            }
        } else {
            const double* p = static_cast<const double*>(a) + row;
            for (; j + kColGroups < j1; j += 2 * kColGroups) {
                const double x0 = p[j * lda], x1 = p[(j + kColGroups) * lda];
                mx = fmax(mx, fmax(fabs(x0), fabs(x1)));
                s0 = __fma_rn(x0, x0, s0);
                s1 = __fma_rn(x1, x1, s1);
            }
            for (; j < j1; j += kColGroups) {
                const double x0 = p[j * lda];
                mx = fmax(mx, fabs(x0));
                s0 = __fma_rn(x0, x0, s0);
            }
        }
    }
    // non-finite inputs (emulator.cpp:19-22): +-Inf shows up in the max, NaN
    // (ignored by fmax) propagates into the sum of squares, which otherwise
    // only adds non-negative terms and so cannot turn NaN by itself
    if (__any_sync(0xffffffffu, isinf(mx) || isnan(s0 + s1)) && (threadIdx.x % 32) == 0) atomicOr(nonfinite, 1);
    smax[g][r] = mx;
    ssum[g][r] = s0 + s1;
    __syncthreads();
    if (g == 0 && row < m) {
        double M = smax[0][r], S = ssum[0][r];
        for (int q = 1; q < kColGroups; ++q) {
            M = fmax(M, smax[q][r]);
            S += ssum[q][r];
        }
        pmax[static_cast<int64_t>(blockIdx.y) * m + row] = M;
        psum[static_cast<int64_t>(blockIdx.y) * m + row] = S;
    }
}

// one warp per column of B (contiguous), 8 loads in flight per lane
__global__ void __launch_bounds__(256)
    col_stats_kernel(const void* __restrict__ b, int is_f32, int64_t k, int64_t n, int64_t ldb,
                     double* __restrict__ cmax, double* __restrict__ csum, int32_t* __restrict__ nonfinite) {
    const int lane = threadIdx.x % 32;
    const int64_t col = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
    if (col >= n) return;
    double mx = 0.0, s[4] = {0.0, 0.0, 0.0, 0.0};
    int64_t i = lane;
    if (is_f32) {
        const float* p = static_cast<const float*>(b) + col * ldb;
        for (; i + 96 < k; i += 128) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double x = p[i + 32 * u];
                mx = fmax(mx, fabs(x));
                s[u] = __fma_rn(x, x, s[u]);
            }
        }
        for (; i < k; i += 32) {
            const double x = p[i];
            mx = fmax(mx, fabs(x));
            s[0] = __fma_rn(x, x, s[0]);
        }
    } else {
        const double* p = static_cast<const double*>(b) + col * ldb;
        for (; i + 96 < k; i += 128) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double x = p[i + 32 * u];
                mx = fmax(mx, fabs(x));
                s[u] = __fma_rn(x, x, s[u]);
            }
        }
        for (; i < k; i += 32) {
            const double x = p[i];
            mx = fmax(mx, fabs(x));
            s[0] = __fma_rn(x, x, s[0]);
        }
    }
    double sum = (s[0] + s[1]) + (s[2] + s[3]);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
    }
    if (lane == 0) {
        cmax[col] = mx;
        csum[col] = sum;
        if (isinf(mx) || isnan(sum)) atomicOr(nonfinite, 1);
    }
}

// Guard band of the parallel sum against the reference's sequential one: both
// approximate S = sum (a 2^-g)^2 within (k+1) u S, so their budgets differ by
// at most 0.51 * 2 (k+1) u / ln 2 < 1.5 (k+1) u; log2/round-off adds < 1e-13.
__device__ __forceinline__ double guard_band(int64_t k) { return 4.0 * static_cast<double>(k + 2) * 0x1.0p-53 + 1e-11; }

__device__ __forceinline__ bool needs_exact(double y, double mx, int64_t k) {
    const double d = fmin(y - floor(y), ceil(y) - y);
    // |x| >= 2^500 could overflow sum x^2; tiny maxima could underflow it
    return d < guard_band(k) || mx >= 0x1.0p+500 || mx < 0x1.0p-400;
}

__global__ void fast_finalize_kernel(const double* __restrict__ pmax, const double* __restrict__ psum, int splits,
                                     const double* __restrict__ cmax, const double* __restrict__ csum, int64_t m,
                                     int64_t n, int64_t k, float pp_fast, int prec, int32_t* __restrict__ mu_exp,
                                     int32_t* __restrict__ nu_exp, int32_t* __restrict__ flag_count,
                                     int32_t* __restrict__ flag_rows, int32_t* __restrict__ flag_cols) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= m + n) return;
    const bool is_row = t < m;
    double mx, s;
    if (is_row) {
        mx = pmax[t];
        s = psum[t];
        for (int q = 1; q < splits; ++q) {
            mx = fmax(mx, pmax[q * m + t]);
            s += psum[q * m + t];
        }
    } else {
        mx = cmax[t - m];
        s = csum[t - m];
    }
    int e = 0;  // zero line: sentinel mu = 1 (scaling.cpp:80, :88)
    if (mx != 0.0) {
        const int g = ilogb(mx);
        const double y = fast_budget(ldexp(s, -2 * g), k, pp_fast);
        e = fast_exponent_from_budget(y, g, prec);
        if (needs_exact(y, mx, k)) {
            const int slot = atomicAdd(flag_count + (is_row ? 0 : 1), 1);
            (is_row ? flag_rows : flag_cols)[slot] = static_cast<int32_t>(is_row ? t : t - m);
        }
    }
    if (is_row)
        mu_exp[t] = e;
    else
        nu_exp[t - m] = e;
}

// One warp per flagged line: elements x[0..k) at base + h*stride.
// Reference order: s = 0; for h: nh = ldexp(x_h, -g); s += nh*nh (no FMA).
__global__ void fast_exact_kernel(const void* __restrict__ a, const void* __restrict__ b, int is_f32, int64_t m,
                                  int64_t n, int64_t k, int64_t lda, int64_t ldb, float pp_fast, int prec,
                                  const int32_t* __restrict__ flag_count, const int32_t* __restrict__ flag_rows,
                                  const int32_t* __restrict__ flag_cols, int32_t* __restrict__ mu_exp,
                                  int32_t* __restrict__ nu_exp) {
    const int lane = threadIdx.x % 32;
    const int warps = gridDim.x * (blockDim.x / 32);
    const int nrows = flag_count[0], ncols = flag_count[1];
    for (int w = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; w < nrows + ncols; w += warps) {
        const bool is_row = w < nrows;
        const int64_t line = is_row ? flag_rows[w] : flag_cols[w - nrows];
        const void* base = is_row ? a : b;
        const int64_t off = is_row ? line : line * ldb;
        const int64_t stride = is_row ? lda : 1;
        double mx = 0.0;
        for (int64_t h = lane; h < k; h += 32) mx = fmax(mx, fabs(load_as_double(base, off + h * stride, is_f32)));
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const int g = ilogb(mx);
        double s = 0.0;
        for (int64_t h0 = 0; h0 < k; h0 += 32) {
            const int64_t h = h0 + lane;
            double sq = 0.0;
            if (h < k) {
                const double nh = ldexp(load_as_double(base, off + h * stride, is_f32), -g);
                sq = __dmul_rn(nh, nh);
            }
            const int cnt = k - h0 < 32 ? static_cast<int>(k - h0) : 32;
            for (int q = 0; q < cnt; ++q) s = __dadd_rn(s, __shfl_sync(0xffffffffu, sq, q));
        }
        if (lane == 0) {
            const int e = fast_exponent_from_budget(fast_budget(s, k, pp_fast), g, prec);
            if (is_row)
                mu_exp[line] = e;
            else
                nu_exp[line] = e;
        }
    }
}

// mu' = 2^(5 - ilogb max|a_i.|) (scaling.cpp:112-116); INT32_MIN marks a zero line
__global__ void accurate_base_kernel(const double* __restrict__ pmax, int splits, const double* __restrict__ cmax,
                                     int64_t m, int64_t n, int32_t* __restrict__ ma, int32_t* __restrict__ nb) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= m + n) return;
    double mx;
    if (t < m) {
        mx = pmax[t];
        for (int q = 1; q < splits; ++q) mx = fmax(mx, pmax[q * m + t]);
    } else {
        mx = cmax[t - m];
    }
    const int32_t e = mx != 0.0 ? 5 - ilogb(mx) : INT32_MIN;
    if (t < m)
        ma[t] = e;
    else
        nb[t - m] = e;
}

// budget of scaling.cpp:151-165: e = min(floor(pp_accu - 0.51 log2 cmax), cap),
// mu = 2^clamp(mu' exponent + e); cmax == 0 keeps mu'; zero lines keep 1.
__global__ void accurate_budget_kernel(const int32_t* __restrict__ ma, const int32_t* __restrict__ nb,
                                       const int32_t* __restrict__ rowmax, const int32_t* __restrict__ colmax,
                                       int64_t m, int64_t n, float pp_accu, int prec, int32_t* __restrict__ mu_exp,
                                       int32_t* __restrict__ nu_exp) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= m + n) return;
    const int32_t base = t < m ? ma[t] : nb[t - m];
    const int32_t cmax = t < m ? rowmax[t] : colmax[t - m];
    int32_t out = 0;
    if (base != INT32_MIN) {
        int e = 0;
        if (cmax > 0) {
            e = static_cast<int>(
                floor(__dsub_rn(static_cast<double>(pp_accu), __dmul_rn(0.51, log2(static_cast<double>(cmax))))));
            const int cap = magnitude_cap(prec) - 6;
            e = e < cap ? e : cap;
        }
        const int cl = exponent_clamp(prec);
        out = clampi(base + e, -cl, cl);
    }
    if (t < m)
        mu_exp[t] = out;
    else
        nu_exp[t - m] = out;
}

}  // namespace

int row_stats_splits(int64_t m, int64_t k) {
    const int64_t row_blocks = (m + kRowTile - 1) / kRowTile;
    int64_t splits = (4 * 148 + row_blocks - 1) / row_blocks;  // ~4 waves of blocks
    const int64_t max_splits = (k + 255) / 256;                 // keep >= 256 columns per split
    if (splits > max_splits) splits = max_splits;
    if (splits < 1) splits = 1;
    if (splits > 64) splits = 64;
    return static_cast<int>(splits);
}

void launch_row_stats(const void* a, int is_f32, int64_t m, int64_t k, int64_t lda, const LineStats& st,
                      cudaStream_t s) {
    const int64_t kps = (k + st.splits - 1) / st.splits;
    dim3 grid(static_cast<unsigned>((m + kRowTile - 1) / kRowTile), static_cast<unsigned>(st.splits));
    row_stats_kernel<<<grid, kRowTile * kColGroups, 0, s>>>(a, is_f32, m, k, lda, kps, st.amax, st.asum, st.nonfinite);
}

void launch_col_stats(const void* b, int is_f32, int64_t k, int64_t n, int64_t ldb, const LineStats& st,
                      cudaStream_t s) {
    col_stats_kernel<<<static_cast<unsigned>((n + 7) / 8), 256, 0, s>>>(b, is_f32, k, n, ldb, st.bmax, st.bsum, st.nonfinite);
}

void launch_fast_finalize(const LineStats& st, int64_t m, int64_t n, int64_t k, const DevConsts& c, int32_t* mu_exp,
                          int32_t* nu_exp, int32_t* flag_count, int32_t* flag_rows, int32_t* flag_cols,
                          cudaStream_t s) {
    cudaMemsetAsync(flag_count, 0, 2 * sizeof(int32_t), s);
    const int64_t lines = m + n;
    fast_finalize_kernel<<<static_cast<unsigned>((lines + 255) / 256), 256, 0, s>>>(
        st.amax, st.asum, st.splits, st.bmax, st.bsum, m, n, k, c.pp_fast, c.precision, mu_exp, nu_exp, flag_count,
        flag_rows, flag_cols);
}

void launch_fast_exact(const void* a, const void* b, int is_f32, int64_t m, int64_t n, int64_t k, int64_t lda,
                       int64_t ldb, const DevConsts& c, const int32_t* flag_count, const int32_t* flag_rows,
                       const int32_t* flag_cols, int32_t* mu_exp, int32_t* nu_exp, cudaStream_t s) {
    // The flagged count lives on the device; a fixed grid strides over it, so
    // the common case (nothing flagged) costs one tiny launch and no host sync.
    fast_exact_kernel<<<148, 256, 0, s>>>(a, b, is_f32, m, n, k, lda, ldb, c.pp_fast, c.precision, flag_count,
                                          flag_rows, flag_cols, mu_exp, nu_exp);
}

void launch_accurate_base(const LineStats& st, int64_t m, int64_t n, int32_t* ma, int32_t* nb, cudaStream_t s) {
    const int64_t lines = m + n;
    accurate_base_kernel<<<static_cast<unsigned>((lines + 255) / 256), 256, 0, s>>>(st.amax, st.splits, st.bmax, m,
                                                                                    n, ma, nb);
}

void launch_accurate_budget(const int32_t* ma, const int32_t* nb, const int32_t* rowmax, const int32_t* colmax,
                            int64_t m, int64_t n, const DevConsts& c, int32_t* mu_exp, int32_t* nu_exp,
                            cudaStream_t s) {
    const int64_t lines = m + n;
    accurate_budget_kernel<<<static_cast<unsigned>((lines + 255) / 256), 256, 0, s>>>(
        ma, nb, rowmax, colmax, m, n, c.pp_accu, c.precision, mu_exp, nu_exp);
}

}  // namespace ozk
