// K1a — scale exponents (reference: scaling.cpp:20-184).
//
// Memory-bound reductions over the FP64/FP32 inputs, one HBM read of A and of
// B per pass, with the per-line exponent step fused in (no separate launches):
//   * row_stats  : per row of column-major A, max|a| and sum a^2 (partial per
//                  k-split); the last block of each 64-row group combines the
//                  splits and finalizes those rows;
//   * col_stats  : per column of B, one warp streams the contiguous column and
//                  finalizes it;
//   * finalize   : fast mode evaluates the budget of fast_exponent
//                  (scaling.cpp:50-56) from the order-free sum; a line whose
//                  floor() argument lies within `guard` of an integer (or whose
//                  magnitude leaves the a^2-safe range) is recomputed at once
//                  in the reference's sequential order (scaling.cpp:69-78 rows,
//                  :90-94 columns) — products in parallel across a warp, the
//                  additions strictly in index order — so mu/nu are
//                  bit-identical to the reference (the floor can only differ
//                  inside the guard band). Accurate mode: mu'/nu' =
//                  2^(5 - ilogb max) (scaling.cpp:110-116), the line's bound
//                  maximum cleared; after the Abar*Bbar bound GEMM (K2 with the
//                  max epilogue) the budget of scaling.cpp:151-165.
#include <cfloat>
#include <climits>

#include "k1_line.cuh"
#include "ozk_device.cuh"

namespace ozk {
namespace {

constexpr int kRowTile = 64;  // rows per block in row_stats
constexpr int kColGroups = 4; // column groups per block in row_stats

// The last block of a 64-row group (over its k-splits) combines the partials
// [split][lines] of its rows, finalizes them and recomputes flagged rows.
// Called by every block after writing its partials; returns at once unless last.
__device__ void row_group_finalize(const LineFinal& F, const double* pmax, const double* psum, int splits,
                                   int64_t lines, int32_t* counters) {
    __shared__ int s_last, s_nflag;
    __shared__ int s_flag[kRowTile];
    __syncthreads();  // this block's partials are written
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(counters + blockIdx.x, 1) == splits - 1;
        s_nflag = 0;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();  // the other splits' partials are visible
    if (threadIdx.x == 0) counters[blockIdx.x] = 0;  // ready for the next call
    const int64_t row = static_cast<int64_t>(blockIdx.x) * kRowTile + threadIdx.x;
    if (threadIdx.x < kRowTile && row < lines) {
        double mx = pmax[row], sm = psum[row];
        for (int q = 1; q < splits; ++q) {
            mx = fmax(mx, pmax[q * lines + row]);
            sm += psum[q * lines + row];
        }
        if (finalize_line(F, row, mx, sm)) s_flag[atomicAdd(&s_nflag, 1)] = threadIdx.x;
    }
    __syncthreads();
    const int nflag = s_nflag;
    for (int w = threadIdx.x / 32; w < nflag; w += blockDim.x / 32)
        exact_line(F, static_cast<int64_t>(blockIdx.x) * kRowTile + s_flag[w], threadIdx.x % 32);
}

__global__ void __launch_bounds__(kRowTile* kColGroups)
    row_stats_kernel(const void* __restrict__ a, int is_f32, int64_t m, int64_t k, int64_t lda, int64_t k_per_split,
                     double* __restrict__ pmax, double* __restrict__ psum, int32_t* __restrict__ nonfinite,
                     int32_t* __restrict__ counters, const LineFinal F) {
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
    row_group_finalize(F, pmax, psum, gridDim.y, m, counters);
}

// FP64 rows, vectorised: a block still owns 64 rows x one k-split, but each
// lane reads two adjacent rows (16 B) of a column and the 8 warps take every
// 8th column, 4 columns in flight per lane: a warp moves 512 B per column
// and a thread keeps 64 B of loads outstanding (the scalar kernel above has
// 16 B). Needs 16-byte aligned columns (even lda, aligned A) and full 64-row
// tiles; anything else takes row_stats_kernel. The sums run in a different
// order than the scalar kernel's, which the fast-mode guard band allows for
// (any order is within (k+1)u of the exact sum).
constexpr int kVecGroups = 8;
__global__ void __launch_bounds__(32 * kVecGroups)
    row_stats_vec_kernel(const double* __restrict__ a, int64_t m, int64_t k, int64_t lda, int64_t k_per_split,
                         double* __restrict__ pmax, double* __restrict__ psum, int32_t* __restrict__ nonfinite,
                         int32_t* __restrict__ counters, const LineFinal F) {
    __shared__ double smax[kVecGroups][kRowTile];
    __shared__ double ssum[kVecGroups][kRowTile];
    const int lane = threadIdx.x % 32, g = threadIdx.x / 32;
    const int64_t row0 = static_cast<int64_t>(blockIdx.x) * kRowTile + 2 * lane;
    const int64_t j0 = static_cast<int64_t>(blockIdx.y) * k_per_split;
    const int64_t j1 = j0 + k_per_split < k ? j0 + k_per_split : k;
    const double* p = a + row0;
    AbsMax am0, am1;
    double s0 = 0.0, s1 = 0.0, t0 = 0.0, t1 = 0.0;
    int64_t j = j0 + g;
    for (; j + 3 * kVecGroups < j1; j += 4 * kVecGroups) {
        double2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldg(reinterpret_cast<const double2*>(p + (j + u * kVecGroups) * lda));
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            am0.add(v[u].x);
            am1.add(v[u].y);
            if (u & 1) {
                t0 = __fma_rn(v[u].x, v[u].x, t0);
                t1 = __fma_rn(v[u].y, v[u].y, t1);
            } else {
                s0 = __fma_rn(v[u].x, v[u].x, s0);
                s1 = __fma_rn(v[u].y, v[u].y, s1);
            }
        }
    }
    for (; j < j1; j += kVecGroups) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(p + j * lda));
        am0.add(v.x);
        am1.add(v.y);
        s0 = __fma_rn(v.x, v.x, s0);
        s1 = __fma_rn(v.y, v.y, s1);
    }
    s0 += t0;
    s1 += t1;
    const double mx0 = am0.value(), mx1 = am1.value();
    if (__any_sync(0xffffffffu, isinf(mx0) || isinf(mx1) || isnan(s0 + s1)) && lane == 0) atomicOr(nonfinite, 1);
    smax[g][2 * lane] = mx0;
    smax[g][2 * lane + 1] = mx1;
    ssum[g][2 * lane] = s0;
    ssum[g][2 * lane + 1] = s1;
    __syncthreads();
    if (threadIdx.x < kRowTile) {
        const int r = threadIdx.x;
        double M = smax[0][r], S = ssum[0][r];
        for (int q = 1; q < kVecGroups; ++q) {
            M = fmax(M, smax[q][r]);
            S += ssum[q][r];
        }
        const int64_t row = static_cast<int64_t>(blockIdx.x) * kRowTile + r;
        pmax[static_cast<int64_t>(blockIdx.y) * m + row] = M;
        psum[static_cast<int64_t>(blockIdx.y) * m + row] = S;
    }
    row_group_finalize(F, pmax, psum, gridDim.y, m, counters);
}

// one warp per column of B (contiguous), 8 loads in flight per lane
__global__ void __launch_bounds__(256)
    col_stats_kernel(const void* __restrict__ b, int is_f32, int64_t k, int64_t n, int64_t ldb,
                     double* __restrict__ cmax, double* __restrict__ csum, int32_t* __restrict__ nonfinite,
                     const LineFinal F) {
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
        AbsMax am;
        for (; i + 96 < k; i += 128) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double x = p[i + 32 * u];
                am.add(x);
                s[u] = __fma_rn(x, x, s[u]);
            }
        }
        for (; i < k; i += 32) {
            const double x = p[i];
            am.add(x);
            s[0] = __fma_rn(x, x, s[0]);
        }
        mx = am.value();
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
    // every lane holds the reduced mx / sum: finalize on lane 0, recompute as a warp
    const bool flag = __shfl_sync(0xffffffffu, lane == 0 ? finalize_line(F, col, mx, sum) : false, 0);
    if (flag) exact_line(F, col, lane);
}

// budget of scaling.cpp:151-165: e = min(floor(pp_accu - 0.51 log2 cmax), cap),
// mu = 2^clamp(mu' exponent + e); cmax == 0 keeps mu'; zero lines keep 1.
// rows and columns in one launch: lines [0, lines) with (base, cmax_in,
// exp_out), then [lines, lines + lines2) with the second triple
template <typename CT>
__global__ void accurate_budget_kernel(const int32_t* __restrict__ base, const CT* __restrict__ cmax_in,
                                       int64_t lines, float pp_accu, int prec, int32_t* __restrict__ exp_out,
                                       const int32_t* __restrict__ base2, const CT* __restrict__ cmax2,
                                       int64_t lines2, int32_t* __restrict__ exp_out2) {
    int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= lines) {
        t -= lines;
        if (t >= lines2) return;
        base = base2;
        cmax_in = cmax2;
        exp_out = exp_out2;
    }
    const int32_t b0 = base[t];
    const CT cmax = cmax_in[t];
    int32_t out = 0;
    if (b0 != INT32_MIN) {
        int e = 0;
        if (cmax > 0) {
            e = static_cast<int>(
                floor(__dsub_rn(static_cast<double>(pp_accu), __dmul_rn(0.51, log2(static_cast<double>(cmax))))));
            const int cap = magnitude_cap(prec) - 6;
            e = e < cap ? e : cap;
        }
        const int cl = exponent_clamp(prec);
        out = clampi(b0 + e, -cl, cl);
    }
    exp_out[t] = out;
}

}  // namespace

int row_stats_splits(int64_t m, int64_t k) {
    const int64_t row_blocks = (m + kRowTile - 1) / kRowTile;
    int64_t splits = (4 * 148 + row_blocks - 1) / row_blocks;  // ~4 waves of blocks
    const int64_t max_splits = (k + 63) / 64;                   // keep >= 64 columns per split
    if (splits > max_splits) splits = max_splits;
    if (splits < 1) splits = 1;
    if (splits > 64) splits = 64;
    return static_cast<int>(splits);
}

int64_t row_stat_groups(int64_t m) { return (m + kRowTile - 1) / kRowTile; }

void launch_row_stats(const void* a, int is_f32, int64_t m, int64_t k, int64_t lda, int splits, double* pmax,
                      double* psum, int32_t* nonfinite, int32_t* counters, const LineFinal& fin, cudaStream_t s) {
    const int64_t kps = (k + splits - 1) / splits;
    if (!is_f32 && m % kRowTile == 0 && lda % 2 == 0 && reinterpret_cast<uintptr_t>(a) % 16 == 0) {
        dim3 grid(static_cast<unsigned>(m / kRowTile), static_cast<unsigned>(splits));
        row_stats_vec_kernel<<<grid, 32 * kVecGroups, 0, s>>>(static_cast<const double*>(a), m, k, lda, kps, pmax,
                                                              psum, nonfinite, counters, fin);
        return;
    }
    dim3 grid(static_cast<unsigned>(row_stat_groups(m)), static_cast<unsigned>(splits));
    row_stats_kernel<<<grid, kRowTile * kColGroups, 0, s>>>(a, is_f32, m, k, lda, kps, pmax, psum, nonfinite,
                                                            counters, fin);
}

void launch_col_stats(const void* b, int is_f32, int64_t k, int64_t n, int64_t ldb, double* pmax, double* psum,
                      int32_t* nonfinite, const LineFinal& fin, cudaStream_t s) {
    col_stats_kernel<<<static_cast<unsigned>((n + 7) / 8), 256, 0, s>>>(b, is_f32, k, n, ldb, pmax, psum, nonfinite,
                                                                        fin);
}

void launch_accurate_budget(const int32_t* base, const int32_t* cmax, int64_t lines, int32_t* exp_out,
                            const int32_t* base2, const int32_t* cmax2, int64_t lines2, int32_t* exp_out2,
                            const DevConsts& c, cudaStream_t s) {
    accurate_budget_kernel<int32_t><<<static_cast<unsigned>((lines + lines2 + 255) / 256), 256, 0, s>>>(
        base, cmax, lines, c.pp_accu, c.precision, exp_out, base2, cmax2, lines2, exp_out2);
}

void launch_accurate_budget64(const int32_t* base, const unsigned long long* cmax, int64_t lines, int32_t* exp_out,
                              const int32_t* base2, const unsigned long long* cmax2, int64_t lines2,
                              int32_t* exp_out2, const DevConsts& c, cudaStream_t s) {
    accurate_budget_kernel<unsigned long long><<<static_cast<unsigned>((lines + lines2 + 255) / 256), 256, 0, s>>>(
        base, cmax, lines, c.pp_accu, c.precision, exp_out, base2, cmax2, lines2, exp_out2);
}

}  // namespace ozk
