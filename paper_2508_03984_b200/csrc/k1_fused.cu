// K1 in one pass over each operand: the line statistics, the line exponent
// and the planes of the same data while it is still in L2 (reference:
// scaling.cpp:20-133 and residue.cpp:7-42, as in k1_scale.cu / k1_residue.cu).
//
// The two-kernel K1 (stats kernel, then planes kernel) reads every FP64 input
// twice from HBM: 16.1 GB per 16384^3 call against 11.8 GB of compulsory
// bytes. Here the second read of a line comes from L2, because the planes of
// a line are written right after its exponent is known:
//
//  * cols_fused_kernel — lines are contiguous columns (B, or A stored
//    transposed): one 512-thread block per column (two per SM), a block-wide
//    max / sum of squares, the exponent (exact sequential recompute of flagged
//    lines by warp 0, k1_line.cuh), then the column again (evict-first) into
//    its K-major planes. In flight: ~2 columns per SM, so a column is re-read
//    after ~300 other columns' bytes (38 MB at k = 16384), well inside L2.
//
//  * rows_fused_kernel — lines are rows of a column-major operand (A, or B
//    stored transposed): a row's statistics need all k columns, so the work
//    is cut into 64-row x 64-column slices handed out by ticket counters in
//    group-major order. Per block: a statistics role (8 warps) accumulates
//    slice statistics into per-row max / sum words (atomics; any summation
//    order lies inside the guard band of the fast exponent, and flagged rows
//    are recomputed exactly), the last slice of a 64-row group finalizes the
//    group's exponents and publishes them with a flag; a planes producer warp
//    claims slices from a second counter, waits for the slice's group and
//    stages the slice's 64 column runs into shared memory with bulk copies
//    (double-buffered, mbarrier completion: bytes in flight cost no
//    registers); 7 consumer warps write the planes from shared memory. The
//    statistics stay within `lag` (>= one group) slices of the planes
//    counter, so the staged runs are L2 hits, and — since a planes ticket that
//    far behind belongs to a group whose statistics slices are all claimed,
//    and a claimed statistics slice finishes without waiting — nothing
//    deadlocks whatever the residency. All state words clear themselves at
//    the end of the launch (CUDA graphs can replay it).
//
// Bit-exactness is unchanged: the exponents come from the same finalize code
// as the two-kernel path (guard band + exact recompute), and the plane bytes
// from the same residue_planes8 / bound entries.
//
// Measured (profiles/r02_k1_fused_ab.md): the column kernel runs
// at 5.6-5.9 TB/s with 0.03-0.13 GB of its second read missing L2 and is the
// default for columns of >= 4096 elements (>= 1024 of them); the row kernel
// reads only the compulsory bytes (2.22 of 2.15 GB) but takes 2.07 ms against
// 0.39 + 0.93 ms for row_stats + planes (its roles keep the SM issue only
// ~34 % busy), so it stays opt-in (OZK_K1_FUSED=3).
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "k1_line.cuh"
#include "ozk_device.cuh"

namespace ozk {
namespace {

__device__ __forceinline__ uint64_t pol_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t pol_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// 8 consecutive elements from a 32-byte aligned address, with an L2 policy
__device__ __forceinline__ void load8h(const double* p, double (&v)[8], uint64_t pol) {
    asm volatile("ld.global.nc.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
                 : "l"(p), "l"(pol));
    asm volatile("ld.global.nc.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
                 : "=d"(v[4]), "=d"(v[5]), "=d"(v[6]), "=d"(v[7])
                 : "l"(p + 4), "l"(pol));
}
__device__ __forceinline__ void load8h(const float* p, float (&v)[8], uint64_t pol) {
    asm volatile("ld.global.nc.L2::cache_hint.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8], %9;"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "l"(p), "l"(pol));
}
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

// elements [i, i + 8) of a line (zeros past `len`); vector loads when aligned
template <typename T>
__device__ __forceinline__ void line8(const T* p, int64_t i, int64_t len, bool vec, T (&v)[8], uint64_t pol) {
    if (vec && i + 8 <= len) {
        load8h(p + i, v, pol);
        return;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = i + u < len ? p[i + u] : T(0);
}
template <typename T>
__device__ __forceinline__ void line8_first(const T* p, int64_t i, int64_t len, bool vec, T (&v)[8], uint64_t pol) {
    if (vec && i + 8 <= len) {
        load8h(p + i, v, pol);
        return;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = i + u < len ? p[i + u] : T(0);
}

// Abar/Bbar entry (scaling.cpp:124-132), as in k1_residue.cu
__device__ __forceinline__ uint32_t bound_entry(double x, int e) {
    if (e == INT32_MIN) return 0;
    const double v = (e >= -1022 && e <= 1023) ? __dmul_rn(fabs(x), pow2d(e)) : ldexp(fabs(x), e);
    return static_cast<uint32_t>(__double2loint(__dadd_ru(v, 0x1.0p52))) & 0xffu;
}

// the planes (KIND 0: N residue planes; KIND 1: the bound plane) of 8
// consecutive elements sharing one exponent column-wise (ex: per element)
template <typename T, int KIND, int kMaxMod>
__device__ __forceinline__ void write_planes8(const T (&v)[8], const int (&ex)[8], bool active, int8_t* dst0,
                                              int64_t plane_stride, const DevConsts& c, uint64_t st_pol) {
    if constexpr (KIND == 1) {
        if (!active) return;
        uint32_t b[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) b[u] = bound_entry(static_cast<double>(v[u]), ex[u]);
        store_plane8<true>(dst0, make_uint2(pack_low_bytes(b[0], b[1], b[2], b[3]), pack_low_bytes(b[4], b[5], b[6], b[7])),
                           st_pol);
    } else {
        T x[8];
        bool fast = true;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            x[u] = trunc_scaled(v[u], ex[u]);
            fast &= symmetric_residue_domain(static_cast<double>(x[u]), sizeof(T) == 4 ? OZK_FP32 : OZK_FP64, c.n);
        }
        fast = __all_sync(0xffffffffu, fast);  // warp-uniform branch inside residue_planes8
        if (!active) return;
        residue_planes8<T, kMaxMod, true>(x, fast, dst0, plane_stride, c, st_pol);
    }
}

constexpr int kColThreads = 512;
constexpr int kColWarps = kColThreads / 32;

template <typename T, int KIND, int kMaxMod>
__global__ void __launch_bounds__(kColThreads, 2)
    cols_fused_kernel(const T* __restrict__ x, int64_t rows, int64_t cols, int64_t ldx, int vec,
                      int32_t* __restrict__ nonfinite, const LineFinal F, const DevConsts c,
                      int8_t* __restrict__ planes, int64_t ld, int64_t plane_stride) {
    __shared__ uint32_t s_key[kColWarps], s_lo[kColWarps];
    __shared__ double s_sm[kColWarps];
    __shared__ int s_e;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t extent = (rows + 15) / 16 * 16;  // plane_ld(rows)
    // L2 priorities: first read evict_last (the line must survive until its
    // planes pass), second read and the plane stores evict_first
    const uint64_t pol = pol_evict_first(), pol_keep = pol_evict_last();
    for (int64_t j = blockIdx.x; j < cols; j += gridDim.x) {
        const T* col = x + j * ldx;
        AbsMax am;
        double s0 = 0.0, s1 = 0.0;
        for (int64_t i = static_cast<int64_t>(tid) * 8; i < rows; i += 2 * 8 * kColThreads) {
            T v0[8], v1[8];
            line8(col, i, rows, vec, v0, pol_keep);
            line8(col, i + 8 * kColThreads, rows, vec, v1, pol_keep);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const double a = static_cast<double>(v0[u]), b = static_cast<double>(v1[u]);
                am.add(a);
                am.add(b);
                s0 = __fma_rn(a, a, s0);
                s1 = __fma_rn(b, b, s1);
            }
        }
        double sm = s0 + s1;
        am.warp_reduce();
#pragma unroll
        for (int o = 16; o; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
        if (lane == 0) {
            s_key[warp] = am.key;
            s_lo[warp] = am.lo;
            s_sm[warp] = sm;
        }
        __syncthreads();
        if (warp == 0) {
            AbsMax bm;
            if (lane < kColWarps) bm.merge(s_key[lane], s_lo[lane]);
            sm = lane < kColWarps ? s_sm[lane] : 0.0;
            bm.warp_reduce();
#pragma unroll
            for (int o = 16; o; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
            const double mx = bm.value();
            // non-finite inputs (emulator.cpp:19-22): Inf in the max, NaN in the sum
            if (lane == 0 && (isinf(mx) || isnan(sm))) atomicOr(nonfinite, 1);
            const bool flag = __shfl_sync(0xffffffffu, lane == 0 ? finalize_line(F, j, mx, sm) : false, 0);
            if (flag) exact_line(F, j, lane);
            if (lane == 0) s_e = F.exp_out[j];  // this thread wrote it (finalize / exact_line)
        }
        // the first planes chunk is loaded before the exponent is known: its
        // L2 latency overlaps warp 0's finalize instead of following it
        const int64_t i_first = static_cast<int64_t>(tid) * 8;
        T vn[8];
        line8_first(col, i_first < extent ? i_first : 0, i_first < extent ? rows : 0, vec, vn, pol);
        __syncthreads();
        const int e = s_e;
        int ex[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) ex[u] = e;
        // the planes, rows [0, extent): zero padding past `rows` (K2's 16-byte columns)
        for (int64_t i0 = 0; i0 < extent; i0 += 8 * kColThreads) {
            const int64_t i = i0 + static_cast<int64_t>(tid) * 8;
            const bool active = i < extent;
            T v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = vn[u];
            const int64_t inext = i + 8 * kColThreads;  // the next chunk in flight during this one's arithmetic
            if (i0 + 8 * kColThreads < extent)
                line8_first(col, inext < extent ? inext : 0, inext < extent ? rows : 0, vec, vn, pol);
            write_planes8<T, KIND, kMaxMod>(v, ex, active, planes + j * ld + i, plane_stride, c, pol);
        }
    }
}

// ---- rows ------------------------------------------------------------------
constexpr int kRowThreads = 512;
constexpr int kRowGroup = 64;  // rows per group (one exponent publication)
constexpr int kSliceCols = 64;  // columns per slice (ticket): 32 KB of FP64 per slice
constexpr int kPlaneBufs = 2;   // planes role: slices staged in shared memory (double buffer)
constexpr int kStatsWarps = 8;  // warps of the statistics role (the rest: planes producer + consumers)

struct RowsFusedState {
    double* acc_max;      // [rows] non-negative max |x| bits (atomicMax on the encoding); zero between calls
    double* acc_sum;      // [rows] sum x^2 (atomicAdd); zero between calls
    int32_t* grp_cnt;     // [groups] finished statistics slices; zero between calls
    uint32_t* grp_ready;  // [groups] 1: the group's exponents are published; zero between calls
    uint32_t* tickets;    // [0] statistics, [1] planes, [2] finished roles; zero between calls
};

__device__ __forceinline__ void role_sync(int id, int count = kRowThreads / 2) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// a contiguous run of global memory into shared memory by the bulk-copy
// engine (16-byte aligned, multiple of 16 bytes), completing on an mbarrier
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}

// Warp-specialised: warps 0-7 run statistics tickets, warps 8-15 planes
// tickets, each role with its own named barrier, so one role's
// synchronisation (reductions, atomics, the group finalize, the wait for a
// group's exponents) never stalls the other role's memory stream.
template <typename T, int KIND, int kMaxMod>
__global__ void __launch_bounds__(kRowThreads, 2)
    rows_fused_kernel(const T* __restrict__ x, int64_t rows, int64_t cols, int64_t ldx, int splits, int lag,
                      int32_t* __restrict__ nonfinite, const LineFinal F, const DevConsts c,
                      int8_t* __restrict__ planes, int64_t ld, int64_t plane_stride, const RowsFusedState S) {
    // statistics: kStatsWarps warps (they read each slice once, from HBM); planes:
    // one producer warp and the rest consumers (they convert and write N bytes
    // per element: the heavier half)
    constexpr int kRoleThreads = 32 * kStatsWarps, kRoleWarps = kStatsWarps;
    __shared__ double s_mx[kRoleWarps][kRowGroup];
    __shared__ double s_sm[kRoleWarps][kRowGroup];
    __shared__ int s_exp2[kPlaneBufs][kRowGroup];
    __shared__ int s_flag[kRowGroup];
    __shared__ int s_nflag, s_last;
    __shared__ uint32_t s_t;
    __shared__ uint32_t s_pslot[kPlaneBufs];
    __shared__ __align__(8) uint64_t s_full[kPlaneBufs], s_empty[kPlaneBufs];
    extern __shared__ __align__(128) uint8_t dyn_smem[];  // [kPlaneBufs][kSliceCols][kRowGroup] T
    const int tid = threadIdx.x, lane = tid & 31;
    const bool stats_role = tid < kRoleThreads;
    const int rt = stats_role ? tid : tid - kRoleThreads;  // thread index inside the role
    const int rw = rt >> 5;                                  // warp index inside the role
    const int64_t groups = (rows + kRowGroup - 1) / kRowGroup;
    const uint32_t total = static_cast<uint32_t>(groups * splits);
    const int64_t extent = (rows + 15) / 16 * 16;  // plane_ld(rows)
    const uint64_t pol = pol_evict_first(), pol_keep = pol_evict_last();
    if (tid == 0) {
        for (int b = 0; b < kPlaneBufs; ++b) {
            mbar_init(smem_addr(&s_full[b]), 1);
            mbar_init(smem_addr(&s_empty[b]), kRowThreads / 32 - kStatsWarps - 1);  // one arrival per consumer warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (stats_role) {
        for (;;) {
            if (rt == 0) {
                // stay within `lag` slices of the planes: the slices between a
                // statistics read and its planes re-read must fit in L2. No
                // deadlock for lag >= splits: a planes ticket below
                // (statistics counter - lag) belongs to a group whose statistics
                // slices are all claimed already, and claimed statistics slices
                // finish without waiting, so the planes counter keeps moving.
                const unsigned long long t0 = globaltimer_ns();
                while (ld_acquire(S.tickets) > ld_acquire(S.tickets + 1) + static_cast<uint32_t>(lag)) {
                    __nanosleep(256);
                    if (globaltimer_ns() - t0 > 4000000000ull) __trap();
                }
                s_t = atomicAdd(S.tickets, 1u);
            }
            role_sync(1, kRoleThreads);
            const uint32_t t = s_t;
            if (t >= total) break;
            // ---- statistics of slice t: rows [r0, r0 + 64), columns [h0, h1) ----
            const int64_t g = t / splits;
            const int64_t r0 = g * kRowGroup, h0 = static_cast<int64_t>(t % splits) * kSliceCols;
            const int64_t h1 = h0 + kSliceCols < cols ? h0 + kSliceCols : cols;
            const int64_t ra = r0 + 2 * lane;
            double mx0 = 0.0, mx1 = 0.0, sa = 0.0, sb = 0.0;
            if (ra + 1 < rows && (ldx & 1) == 0) {  // two adjacent rows per lane (8 / 16 B)
#pragma unroll 8
                for (int64_t h = h0 + rw; h < h1; h += kRoleWarps) {
                    double a, b;
                    if constexpr (sizeof(T) == 8) {
                        asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                                     : "=d"(a), "=d"(b)
                                     : "l"(x + ra + h * ldx), "l"(pol_keep));
                    } else {
                        float fa, fb;
                        asm volatile("ld.global.nc.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;"
                                     : "=f"(fa), "=f"(fb)
                                     : "l"(x + ra + h * ldx), "l"(pol_keep));
                        a = fa;
                        b = fb;
                    }
                    mx0 = fmax(mx0, fabs(a));
                    mx1 = fmax(mx1, fabs(b));
                    sa = __fma_rn(a, a, sa);
                    sb = __fma_rn(b, b, sb);
                }
            } else {
                for (int64_t h = h0 + rw; h < h1; h += kRoleWarps) {
                    const double a = ra < rows ? static_cast<double>(x[ra + h * ldx]) : 0.0;
                    const double b = ra + 1 < rows ? static_cast<double>(x[ra + 1 + h * ldx]) : 0.0;
                    mx0 = fmax(mx0, fabs(a));
                    mx1 = fmax(mx1, fabs(b));
                    sa = __fma_rn(a, a, sa);
                    sb = __fma_rn(b, b, sb);
                }
            }
            if (__any_sync(0xffffffffu, isinf(mx0) || isinf(mx1) || isnan(sa + sb)) && lane == 0)
                atomicOr(nonfinite, 1);
            s_mx[rw][2 * lane] = mx0;
            s_mx[rw][2 * lane + 1] = mx1;
            s_sm[rw][2 * lane] = sa;
            s_sm[rw][2 * lane + 1] = sb;
            role_sync(1, kRoleThreads);
            if (rt < kRowGroup && r0 + rt < rows) {
                double M = s_mx[0][rt], Sm = s_sm[0][rt];
#pragma unroll
                for (int q = 1; q < kRoleWarps; ++q) {
                    M = fmax(M, s_mx[q][rt]);
                    Sm += s_sm[q][rt];
                }
                atomicMax(reinterpret_cast<unsigned long long*>(S.acc_max + r0 + rt),
                          static_cast<unsigned long long>(__double_as_longlong(M)));
                atomicAdd(S.acc_sum + r0 + rt, Sm);
                __threadfence();
            }
            role_sync(1, kRoleThreads);
            if (rt == 0) {
                s_last = atomicAdd(S.grp_cnt + g, 1) == splits - 1;
                s_nflag = 0;
            }
            role_sync(1, kRoleThreads);
            if (s_last) {
                // ---- the group's last slice: finalize its exponents ----
                __threadfence();
                if (rt < kRowGroup && r0 + rt < rows) {
                    const int64_t row = r0 + rt;
                    const double M = __longlong_as_double(static_cast<long long>(
                        atomicExch(reinterpret_cast<unsigned long long*>(S.acc_max + row), 0ull)));
                    const double Sm = __longlong_as_double(static_cast<long long>(
                        atomicExch(reinterpret_cast<unsigned long long*>(S.acc_sum + row), 0ull)));
                    if (finalize_line(F, row, M, Sm)) s_flag[atomicAdd(&s_nflag, 1)] = rt;
                }
                role_sync(1, kRoleThreads);
                for (int w = rw; w < s_nflag; w += kRoleWarps) exact_line(F, r0 + s_flag[w], lane);
                __threadfence();
                role_sync(1, kRoleThreads);
                if (rt == 0) {
                    S.grp_cnt[g] = 0;  // ready for the next call
                    st_release(S.grp_ready + g, 1u);
                }
            }
            role_sync(1, kRoleThreads);  // s_t, s_last and the shared partials are reused
        }
    } else if (rw == 0) {
        // ---- planes producer (one warp): claims slices, waits for their group,
        // stages each slice's columns into shared memory with bulk copies (the
        // bytes in flight cost no registers) and its group's exponents ----
        for (int iter = 0;; ++iter) {
            const int bsl = iter % kPlaneBufs;
            const uint32_t ph = static_cast<uint32_t>(iter / kPlaneBufs) & 1u;
            uint32_t p = 0;
            if (lane == 0) p = atomicAdd(S.tickets + 1, 1u);
            p = __shfl_sync(0xffffffffu, p, 0);
            mbar_wait(smem_addr(&s_empty[bsl]), ph ^ 1u);  // the consumers released this buffer
            if (p >= total) {
                if (lane == 0) {
                    s_pslot[bsl] = p;  // the consumers' exit signal
                    mbar_arrive(smem_addr(&s_full[bsl]));
                }
                break;
            }
            const int64_t g = p / splits;
            const int64_t r0 = g * kRowGroup, h0 = static_cast<int64_t>(p % splits) * kSliceCols;
            const int64_t h1 = h0 + kSliceCols < cols ? h0 + kSliceCols : cols;
            const int64_t nr = rows - r0 < kRowGroup ? rows - r0 : kRowGroup;
            if (lane == 0) {
                // statistics never wait on the planes counter's progress except
                // through `lag`, which admits every statistics slice of this
                // group, so the group is published; bounded anyway (trap, not hang)
                const unsigned long long t0 = globaltimer_ns();
                while (ld_acquire(S.grp_ready + g) != 1u) {
                    __nanosleep(128);
                    if (globaltimer_ns() - t0 > 4000000000ull) __trap();
                }
            }
            __syncwarp();
            s_exp2[bsl][lane] = r0 + lane < rows ? __ldcg(F.exp_out + r0 + lane) : 0;
            s_exp2[bsl][lane + 32] = r0 + lane + 32 < rows ? __ldcg(F.exp_out + r0 + lane + 32) : 0;
            if (lane == 0) s_pslot[bsl] = p;
            __syncwarp();  // the exponents and the slot are written before the arrival
            const uint32_t bytes = static_cast<uint32_t>(nr * sizeof(T));
            const uint32_t full = smem_addr(&s_full[bsl]);
            if (lane == 0) mbar_expect_tx(full, bytes * static_cast<uint32_t>(h1 - h0));
            __syncwarp();
            T* buf = reinterpret_cast<T*>(dyn_smem) + static_cast<size_t>(bsl) * kSliceCols * kRowGroup;
            for (int64_t h = h0 + lane; h < h1; h += 32)
                bulk_g2s(smem_addr(buf + (h - h0) * kRowGroup), x + r0 + h * ldx, bytes, full, pol);
        }
    } else {
        // ---- planes consumers (7 warps): residue planes of the staged slice ----
        constexpr int kConsumers = kRowThreads - kRoleThreads - 32;
        const int ct = rt - 32;
        for (int iter = 0;; ++iter) {
            const int bsl = iter % kPlaneBufs;
            const uint32_t ph = static_cast<uint32_t>(iter / kPlaneBufs) & 1u;
            mbar_wait(smem_addr(&s_full[bsl]), ph);
            const uint32_t p = s_pslot[bsl];
            if (p >= total) break;
            const int64_t g = p / splits;
            const int64_t r0 = g * kRowGroup, h0 = static_cast<int64_t>(p % splits) * kSliceCols;
            const int64_t h1 = h0 + kSliceCols < cols ? h0 + kSliceCols : cols;
            const T* buf = reinterpret_cast<const T*>(dyn_smem) + static_cast<size_t>(bsl) * kSliceCols * kRowGroup;
            // 8 rows x 1 column per item: 8 items per column
#pragma unroll 1
            for (int it = ct; it < kSliceCols * (kRowGroup / 8); it += kConsumers) {
                const int cl = it / (kRowGroup / 8), rc = (it % (kRowGroup / 8)) * 8;
                const int64_t h = h0 + cl, rr = r0 + rc;
                const bool active = h < h1 && rr < extent;
                T v[8];
                const T* src = buf + cl * kRowGroup + rc;
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = active && rr + u < rows ? src[u] : T(0);
                int ex[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) ex[u] = s_exp2[bsl][rc + u];
                write_planes8<T, KIND, kMaxMod>(v, ex, active, planes + (active ? h : 0) * ld + (active ? rr : 0),
                                                plane_stride, c, pol);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_addr(&s_empty[bsl]));
        }
    }
    // each role of each block made exactly one failing claim and makes no more:
    // the last role out resets the counters for the next call
    // (with the group flags, so the state is all zero between calls and a
    // captured CUDA graph can replay the launch: nothing is baked in per call)
    if (rt == 0 && atomicAdd(S.tickets + 2, 1u) == 2u * gridDim.x - 1u) {  // stats rt 0 and the producer's lane 0
        const int64_t groups_all = (rows + kRowGroup - 1) / kRowGroup;
        for (int64_t g = 0; g < groups_all; ++g) S.grp_ready[g] = 0;
        S.tickets[0] = 0;
        S.tickets[1] = 0;
        S.tickets[2] = 0;
    }
}

template <typename T, int KIND>
void cols_dispatch(const T* x, int64_t rows, int64_t cols, int64_t ldx, int32_t* nonfinite, const LineFinal& F,
                   const DevConsts& c, int8_t* planes, int64_t ld, int64_t stride, int num_sms, cudaStream_t s) {
    const int vec = (reinterpret_cast<uintptr_t>(x) & 31) == 0 && (ldx * static_cast<int64_t>(sizeof(T))) % 32 == 0;
    const int64_t grid = std::min<int64_t>(cols, 2 * static_cast<int64_t>(num_sms));
#define OZK_K1F(MAXN)                                                                                        \
    cols_fused_kernel<T, KIND, MAXN><<<static_cast<unsigned>(grid), kColThreads, 0, s>>>(x, rows, cols, ldx, \
                                                                                         vec, nonfinite, F, c, \
                                                                                         planes, ld, stride)
    if (KIND == 1 || c.n <= 8)
        OZK_K1F(8);
    else if (c.n <= 12)
        OZK_K1F(12);
    else if (c.n <= 14)
        OZK_K1F(14);
    else if (c.n <= 16)
        OZK_K1F(16);
    else
        OZK_K1F(OZK_MAX_MODULI);
#undef OZK_K1F
}

template <typename T, int KIND>
void rows_dispatch(const T* x, int64_t rows, int64_t cols, int64_t ldx, int32_t* nonfinite,
                   const LineFinal& F, const DevConsts& c, int8_t* planes, int64_t ld, int64_t stride,
                   const RowsFusedState& S, int num_sms, cudaStream_t s) {
    const int splits = static_cast<int>((cols + kSliceCols - 1) / kSliceCols);
    const int64_t groups = (rows + kRowGroup - 1) / kRowGroup;
    const int64_t total = groups * splits;
    constexpr int smem = kPlaneBufs * kSliceCols * kRowGroup * static_cast<int>(sizeof(T));
    int per_sm = 0;
    cudaFuncSetAttribute(rows_fused_kernel<T, KIND, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rows_fused_kernel<T, KIND, 8>, kRowThreads, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t grid = std::min<int64_t>(total, static_cast<int64_t>(per_sm) * num_sms);
    // statistics may run this many slices ahead of the planes (>= one group;
    // OZK_K1_LAG overrides): one group plus half a grid of slices in flight
    int lag = splits + static_cast<int>(grid / 2);
    if (const char* e = std::getenv("OZK_K1_LAG")) lag = std::max(splits, std::atoi(e));
#define OZK_K1F(MAXN)                                                                                          \
    do {                                                                                                       \
        cudaFuncSetAttribute(rows_fused_kernel<T, KIND, MAXN>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                             smem);                                                                            \
        rows_fused_kernel<T, KIND, MAXN><<<static_cast<unsigned>(grid), kRowThreads, smem, s>>>(               \
            x, rows, cols, ldx, splits, lag, nonfinite, F, c, planes, ld, stride, S);                          \
    } while (0)
    if (KIND == 1 || c.n <= 8)
        OZK_K1F(8);
    else if (c.n <= 12)
        OZK_K1F(12);
    else if (c.n <= 14)
        OZK_K1F(14);
    else if (c.n <= 16)
        OZK_K1F(16);
    else
        OZK_K1F(OZK_MAX_MODULI);
#undef OZK_K1F
}

}  // namespace

size_t rows_fused_state_bytes(int64_t rows) {
    const int64_t groups = (rows + kRowGroup - 1) / kRowGroup;
    return sizeof(double) * 2 * static_cast<size_t>(rows) + sizeof(int32_t) * 2 * static_cast<size_t>(groups) + 64;
}

void launch_cols_fused(const void* x, int is_f32, int64_t rows, int64_t cols, int64_t ldx, int32_t* nonfinite,
                       const LineFinal& F, const DevConsts& c, int kind, int8_t* planes, int64_t ld, int64_t stride,
                       int num_sms, cudaStream_t s) {
    if (is_f32) {
        if (kind == 0)
            cols_dispatch<float, 0>(static_cast<const float*>(x), rows, cols, ldx, nonfinite, F, c, planes, ld, stride,
                                    num_sms, s);
        else
            cols_dispatch<float, 1>(static_cast<const float*>(x), rows, cols, ldx, nonfinite, F, c, planes, ld, stride,
                                    num_sms, s);
    } else {
        if (kind == 0)
            cols_dispatch<double, 0>(static_cast<const double*>(x), rows, cols, ldx, nonfinite, F, c, planes, ld,
                                     stride, num_sms, s);
        else
            cols_dispatch<double, 1>(static_cast<const double*>(x), rows, cols, ldx, nonfinite, F, c, planes, ld,
                                     stride, num_sms, s);
    }
}

void launch_rows_fused(const void* x, int is_f32, int64_t rows, int64_t cols, int64_t ldx,
                       void* state, int32_t* nonfinite, const LineFinal& F, const DevConsts& c, int kind,
                       int8_t* planes, int64_t ld, int64_t stride, int num_sms, cudaStream_t s) {
    const int64_t groups = (rows + kRowGroup - 1) / kRowGroup;
    RowsFusedState S;
    S.acc_max = static_cast<double*>(state);
    S.acc_sum = S.acc_max + rows;
    S.grp_cnt = reinterpret_cast<int32_t*>(S.acc_sum + rows);
    S.grp_ready = reinterpret_cast<uint32_t*>(S.grp_cnt + groups);
    S.tickets = S.grp_ready + groups;
    if (is_f32) {
        if (kind == 0)
            rows_dispatch<float, 0>(static_cast<const float*>(x), rows, cols, ldx, nonfinite, F, c, planes, ld,
                                    stride, S, num_sms, s);
        else
            rows_dispatch<float, 1>(static_cast<const float*>(x), rows, cols, ldx, nonfinite, F, c, planes, ld,
                                    stride, S, num_sms, s);
    } else {
        if (kind == 0)
            rows_dispatch<double, 0>(static_cast<const double*>(x), rows, cols, ldx, nonfinite, F, c, planes,
                                     ld, stride, S, num_sms, s);
        else
            rows_dispatch<double, 1>(static_cast<const double*>(x), rows, cols, ldx, nonfinite, F, c, planes,
                                     ld, stride, S, num_sms, s);
    }
}

}  // namespace ozk
