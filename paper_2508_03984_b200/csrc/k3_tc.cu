// K3 with the C1 sum on the tensor cores (FP64 tables; reference:
// emulator.cpp:49-53 weighted sums, reconstruct.hpp:51-54, reconstruct.cpp:49-69).
//
// With FP64 tables every s1_i is an integer multiple S_i of one power of two
// 2^E (the head of W_i on the common grid, crt_tables.cpp:165-169), S_i < 2^48,
// and sum_i S_i (p_i - 1) < 2^53: each product s1_i u and each partial sum of
// the reference's c1 += s1_i * u is exact, so c1 = 2^E * sum_i S_i u_i for any
// evaluation order. That integer dot product over the moduli is an int8 GEMM:
//   [128 rows x 32 moduli] (U tile, u8, MN-major) x [32 moduli x 16] (the
//   base-256 digits of S_i, u8, K-major) -> [128 x 16] s32 in TMEM,
// one tcgen05.mma.kind::i8 (M = 128, N = 16, K = 32) per 128-row group, column
// b holding sum_i D_ib u_i < 2^21 for digit b. The epilogue forms
//   c1 = fma(Z, 2^(E+32), fma(Y, 2^(E+16), X 2^E)),
//   X = P0 + 256 P1, Y = P2 + 256 P3, Z = P4 + 256 P5,
// exact (every partial sum is a multiple of 2^E below 2^53 * 2^E). This takes
// the C1 chain (DADD + DFMA per element and modulus) off the FP64 pipe; the C2
// chain keeps the reference's roundings (fl(s2 u) = fma(s2, 2^52 + u, -s2 2^52),
// then the rounded add), so K3 does 2 instead of 4 FP64 ops per element-modulus.
//
// Data movement: one TMA (cp.async.bulk.tensor, 128B swizzle) per 128-row
// group lands [P planes][128 rows] (P = 16 or 24; planes >= N zero-filled by
// TMA) — exactly the canonical MN-major SW128 operand of the MMA — into a
// two-slot ring. The C2 chain reads the same bytes (8 consecutive rows per
// thread, one 8-byte LDS per plane at the swizzled address); TMEM rows belong
// to warp (row / 32) % 4, so the exact c1 values cross to the row owners
// through a (bank-swizzled) shared buffer and one 128-thread named barrier.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "ozk_device.cuh"

namespace ozk {
namespace {

constexpr int kConsumers = 128;
constexpr int kThreads = kConsumers + 32;  // + one producer warp

struct TcParams {
    unsigned long long s_int[OZK_MAX_MODULI];  // S_i = s1_i / 2^E
    double sc0, sc0m52;                        // 2^E, -2^(52+E)
};

__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
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
// producer-side wait: a lane polling a ring slot with try_wait in a tight loop
// issued ~40 instructions per element of K3 (a quarter of the SM's issue
// slots, taken from the consumer warps); it has a full stage of slack, so it
// backs off with nanosleep between polls
__device__ __forceinline__ void mbar_wait_backoff(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    for (;;) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
        if (done) return;
        __nanosleep(256);
    }
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1, int c2,
                                       uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, "
        "%4, %5}], [%2], %6;" ::"r"(dst),
        "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory"); }

// 128B-swizzled shared-memory descriptor (sm_100 version 1), SBO = 1024 B
// (8 rows of 128 B); LBO = 16 B (K-major: unused within one atom column;
// MN-major with M = 128: one atom wide, unused)
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t a) {
    return static_cast<uint64_t>((a >> 4) & 0x3FFFu) | (static_cast<uint64_t>(1) << 16) |
           (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
           (static_cast<uint64_t>(2) << 61);
}
// u8 x u8 -> s32, A MN-major (bit 15), B K-major, N = 16, M = 128
constexpr uint32_t kIdesc = (2u << 4) | (0u << 7) | (0u << 10) | (1u << 15) | ((16u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void mma_u8(uint32_t d, uint64_t a, uint64_t b) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(kIdesc));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void ld_nc_v8(const int32_t* p, int* v) {
    asm volatile("ld.global.nc.v8.s32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "l"(p));
}
__device__ __forceinline__ void st_v4_f64(double* p, const double* v) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
                 : "memory");
}
__device__ __forceinline__ void st_v8_f32(float* p, const float* v) {
    asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(v[0]), "f"(v[1]),
                 "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}

__device__ __forceinline__ double scale_pow2(double x, int e) {
    if (e >= -1022 && e <= 1023) {
        const double r = __dmul_rn(x, pow2d(e));
        if (fabs(r) >= 0x1.0p-1022 && fabs(r) <= 0x1.fffffffffffffp+1023) return r;
        if (r == 0.0 && x == 0.0) return r;
    }
    return ldexp(x, e);
}
// ldexp by moving the exponent field when x and the result are normal
__device__ __forceinline__ double unscale_fast(double x, int e) {
    const int hi = __double2hiint(x);
    const int ex = (hi >> 20) & 0x7ff;
    if (ex != 0 && static_cast<unsigned>(ex + e - 1) < 2046u)
        return __hiloint2double(hi + static_cast<int>(static_cast<unsigned>(e) << 20), __double2loint(x));
    return scale_pow2(x, e);
}

template <int R>
struct RowWord;
template <>
struct RowWord<4> {
    static __device__ __forceinline__ uint2 lds(uint32_t a) {
        uint2 w;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w.x) : "r"(a));
        w.y = 0;
        return w;
    }
};
template <>
struct RowWord<8> {
    static __device__ __forceinline__ uint2 lds(uint32_t a) {
        uint2 w;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w.x), "=r"(w.y) : "r"(a));
        return w;
    }
};

// Tile = 128 R rows of one column (R MMA groups of 128 rows); each consumer
// thread owns R consecutive rows for the C2 chain and the output.
template <int R, int S, int P>
struct TcCfg {
    static constexpr int kRows = 128 * R;
    static constexpr int kGroupBytes = P * 128;
    static constexpr int kStageBytes = R * kGroupBytes;
    static constexpr int kTmemCols = 16 * R < 32 ? 32 : 16 * R;
    // [S][R groups][P planes][128 B] | B digits [16][128 B]. The K = 32 MMA
    // of a stage's last group reads (32 - P) planes past the stage: the next
    // stage or the digit block, inside the allocation (those bytes meet zero
    // digit rows). The c1 exchange reuses the consumed stage (kRows doubles).
    static constexpr int kSmem = 1024 /*align*/ + S * kStageBytes + 2048;
    static_assert((32 - P) * 128 <= 2048, "MMA over-read leaves the allocation");
    static_assert(kRows * 8 <= kStageBytes, "exchange does not fit the stage");
};

template <bool kF32Out, bool kPlain, int kMaxMod, int P, int R, int S>
__global__ void __launch_bounds__(kThreads, R == 4 ? 5 : 4)
    reconstruct_tc_kernel(const __grid_constant__ CUtensorMap umap, int64_t m, int64_t n, int64_t row_chunks,
                          const int32_t* __restrict__ mu_exp, const int32_t* __restrict__ nu_exp, const DevConsts c,
                          const TcParams tp, double alpha, double beta, void* __restrict__ C, int64_t ldc,
                          bool vec_ok, int probe) {
    using Cf = TcCfg<R, S, P>;
    constexpr int kRows = Cf::kRows, kGroupBytes = Cf::kGroupBytes, kStageBytes = Cf::kStageBytes;
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t full[S], empty[S], mma_bar;
    __shared__ uint32_t tmem_slot;
    uint8_t* sbuf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* bdig = sbuf + S * kStageBytes;

    const int tid = threadIdx.x;
    const int n_mod = c.n;
    if (tid == 0) {
        for (int st = 0; st < S; ++st) {
            mbar_init(saddr(&full[st]), 1);
            mbar_init(saddr(&empty[st]), kConsumers / 32);
        }
        mbar_init(saddr(&mma_bar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // B operand: row b (digit), K-major 128 B rows, byte k = digit b of S_k,
    // 16-byte chunk k / 16 XOR-swizzled by b % 8 (the TMA SW128 pattern);
    // rows 6..15 and moduli >= N are zero
    for (int i = tid; i < 16 * 32; i += kThreads) {
        const int b = i >> 5, k = i & 31;
        const uint32_t v =
            (b < 6 && k < n_mod) ? static_cast<uint32_t>((tp.s_int[k] >> (8 * b)) & 0xFFu) : 0u;
        bdig[b * 128 + ((((k >> 4) ^ (b & 7)) << 4) | (k & 15))] = static_cast<uint8_t>(v);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tmem_slot)),
                     "n"(Cf::kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_before();
    __syncthreads();
    tc_after();
    const uint32_t tbase = tmem_slot;

    const int64_t tiles = row_chunks * n;
    const int64_t dj = gridDim.x / row_chunks, dr = gridDim.x % row_chunks;
    int64_t j = blockIdx.x / row_chunks, chunk = blockIdx.x % row_chunks;
    auto advance = [&]() {
        chunk += dr;
        j += dj;
        if (chunk >= row_chunks) {
            chunk -= row_chunks;
            ++j;
        }
    };

    if (tid >= kConsumers) {  // producer warp: one lane issues the TMA boxes
        if (tid == kConsumers) {
            const uint64_t pol = evict_first();
            for (int64_t k = 0, tile = blockIdx.x; tile < tiles; ++k, tile += gridDim.x, advance()) {
                const int st = static_cast<int>(k % S);
                mbar_wait_backoff(saddr(&empty[st]), static_cast<uint32_t>(((k / S) & 1) ^ 1));
                const int64_t i0 = chunk * kRows;
                const int64_t rem = (m - i0 + 127) / 128;
                const int ng = rem < R ? static_cast<int>(rem) : R;
                const uint32_t fb = saddr(&full[st]);
                if (probe == 2) {  // compute-only probe: stale planes, no loads
                    mbar_arrive(fb);
                    continue;
                }
                mbar_expect_tx(fb, static_cast<uint32_t>(ng * kGroupBytes));
                const uint32_t dst = saddr(sbuf) + st * kStageBytes;
                for (int g = 0; g < ng; ++g)
                    tma_3d(dst + g * kGroupBytes, &umap, fb, static_cast<int>(i0 + 128 * g), 0, static_cast<int>(j),
                           pol);
            }
        }
        return;
    }

    const int warp = tid >> 5, lane = tid & 31;
    // C2-chain geometry: rows R tid .. R tid + R - 1 = group tid / (128 / R),
    // bytes o .. o + R - 1 of each 128-byte plane row, o = R (tid % (128 / R)),
    // at 16-byte chunk o / 16 XOR (plane % 8)
    constexpr int kPerGroup = 128 / R;
    const int grp = tid / kPerGroup, o = R * (tid % kPerGroup), chk = o >> 4;
    const uint32_t row_off = static_cast<uint32_t>(grp * kGroupBytes + (o & 15));
    // exchange (bytes): owner tid reads its R rows as R/2 16-byte chunks,
    // chunk jj at 16 ((R/2) tid + (jj ^ sw(tid))), sw(t) = (t >> log2(16/R)) % (R/2),
    // so 8 consecutive owners hit 8 bank groups; the writer of tile row
    // 128 g + 32 warp + lane (TMEM lane owner) uses the same map, which is
    // 1024 g bytes past its g = 0 slot
    constexpr int kHalf = R / 2, kSwShift = R == 8 ? 1 : 2;
    const int r0 = 32 * warp + lane, own0 = r0 / R;
    const uint32_t xw = 8u * static_cast<uint32_t>(R * own0 + 2 * (((r0 >> 1) & (kHalf - 1)) ^
                                                                  ((own0 >> kSwShift) & (kHalf - 1))) +
                                                   (r0 & 1));
    const uint32_t xr = 8u * R * static_cast<uint32_t>(tid), xr_x = static_cast<uint32_t>((tid >> kSwShift) & (kHalf - 1));
    const uint32_t bdesc_lo = saddr(bdig);
    for (int64_t k = 0, tile = blockIdx.x; tile < tiles; ++k, tile += gridDim.x, advance()) {
        const int st = static_cast<int>(k % S);
        const int64_t i0 = chunk * kRows + tid * R;
        const bool vec = vec_ok && i0 + R <= m;
        int me[R];
        if (vec) {
            if constexpr (R == 8)
                ld_nc_v8(mu_exp + i0, me);
            else
                asm volatile("ld.global.nc.v4.s32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(me[0]), "=r"(me[1]), "=r"(me[2]), "=r"(me[3])
                             : "l"(mu_exp + i0));
        } else {
#pragma unroll
            for (int q = 0; q < R; ++q) me[q] = i0 + q < m ? mu_exp[i0 + q] : 0;
        }
        const int ne = nu_exp[j];
        mbar_wait(saddr(&full[st]), static_cast<uint32_t>((k / S) & 1));
        if (probe == 1) {  // memory-only probe (tools/k3_time.py): planes in, zeros out
            __syncwarp();
            if (lane == 0) mbar_arrive(saddr(&empty[st]));
            if (vec) {
                double z[R] = {};
#pragma unroll
                for (int v = 0; v < R; v += 4) st_v4_f64(static_cast<double*>(C) + i0 + v + j * ldc, z + v);
            }
            continue;
        }
        const uint32_t stage = saddr(sbuf) + st * kStageBytes;
        if (tid == 0) {
            tc_after();
            const uint64_t bd = sdesc_sw128(bdesc_lo);
#pragma unroll
            for (int g = 0; g < R; ++g) mma_u8(tbase + g * 16, sdesc_sw128(stage + g * kGroupBytes), bd);
            mma_commit(saddr(&mma_bar));
        }
        // C2 = sum fl(s2_t u) in ascending t, from the swizzled plane rows
        double c2[R];
#pragma unroll
        for (int q = 0; q < R; ++q) c2[q] = 0.0;
        const uint32_t rowbase = stage + row_off;
#pragma unroll
        for (int t = 0; t < kMaxMod; ++t) {
            const uint2 w = RowWord<R>::lds(rowbase + t * 128 + ((chk ^ (t & 7)) << 4));
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const uint32_t ub = __byte_perm(q < 4 ? w.x : w.y, 0u, 0x4440u | (q & 3));
                const double V = __hiloint2double(0x43300000, static_cast<int>(ub));  // 2^52 + u
                c2[q] = __dadd_rn(c2[q], __fma_rn(c.s2[t], V, c.s2_m52[t]));
            }
        }
        mbar_wait(saddr(&mma_bar), static_cast<uint32_t>(k & 1));
        tc_after();
        // exact c1 of this warp's TMEM rows 128 g + 32 warp + lane, exchanged
        // through the consumed stage (every warp's LDS of it and the MMA are
        // done once all consumers pass the first barrier):
        // T = X + 2^16 Y + 2^32 Z < 2^52 as an integer pair, c1 = T 2^E by one
        // DFMA on 2^52 + T (exact: (2^52 + T) 2^E - 2^(52+E) is representable)
        double c1w[R];
        constexpr int kBatch = R < 4 ? R : 4;
#pragma unroll
        for (int h = 0; h < R / kBatch; ++h) {
            uint32_t v[kBatch][8];
#pragma unroll
            for (int g = 0; g < kBatch; ++g)
                tmem_ld8(tbase + (static_cast<uint32_t>(warp * 32) << 16) + (kBatch * h + g) * 16, v[g]);
            tmem_wait_ld();
#pragma unroll
            for (int g = 0; g < kBatch; ++g) {
                const uint32_t X = v[g][0] + (v[g][1] << 8), Y = v[g][2] + (v[g][3] << 8), Z = v[g][4] + (v[g][5] << 8);
                const uint64_t T =
                    static_cast<uint64_t>(X) + (static_cast<uint64_t>(Y) << 16) + (static_cast<uint64_t>(Z) << 32);
                const double V = __hiloint2double(static_cast<int>(static_cast<uint32_t>(T >> 32) | 0x43300000u),
                                                  static_cast<int>(static_cast<uint32_t>(T)));
                c1w[kBatch * h + g] = __fma_rn(V, tp.sc0, tp.sc0m52);
            }
        }
        tc_before();
        consumers_sync();
#pragma unroll
        for (int g = 0; g < R; ++g)
            asm volatile("st.shared.f64 [%0], %1;" ::"r"(stage + xw + g * 1024), "d"(c1w[g]) : "memory");
        consumers_sync();
        double c1[R];
#pragma unroll
        for (int jj = 0; jj < kHalf; ++jj)
            asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
                         : "=d"(c1[2 * jj]), "=d"(c1[2 * jj + 1])
                         : "r"(stage + xr + ((jj ^ xr_x) << 4))
                         : "memory");
        // slot st back to the producer: order this thread's generic accesses
        // before the TMA (async proxy) overwrite
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(saddr(&empty[st]));
        double r[R];
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const double qv = rint(__dmul_rn(c.P_inv, c1[q]));
            const double cpp = __fma_rn(-c.P2, qv, __dadd_rn(__fma_rn(-c.P1, qv, c1[q]), c2[q]));
            r[q] = unscale_fast(cpp, -(me[q] + ne));
        }
        if (!kPlain) {
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const int64_t i = i0 + q;
                const double old = (beta != 0.0 && i < m)
                                       ? (kF32Out ? static_cast<double>(static_cast<float*>(C)[i + j * ldc])
                                                  : static_cast<double*>(C)[i + j * ldc])
                                       : 0.0;
                r[q] = __dadd_rn(__dmul_rn(alpha, r[q]), __dmul_rn(beta, old));
            }
        }
        if (vec) {
            if constexpr (kF32Out && R == 8) {
                float f[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) f[q] = __double2float_rn(r[q]);
                st_v8_f32(static_cast<float*>(C) + i0 + j * ldc, f);
            } else if constexpr (kF32Out) {
                asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(static_cast<float*>(C) + i0 + j * ldc),
                             "f"(__double2float_rn(r[0])), "f"(__double2float_rn(r[1])), "f"(__double2float_rn(r[2])),
                             "f"(__double2float_rn(r[3]))
                             : "memory");
            } else {
#pragma unroll
                for (int v = 0; v < R; v += 4) st_v4_f64(static_cast<double*>(C) + i0 + v + j * ldc, r + v);
            }
        } else {
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const int64_t i = i0 + q;
                if (i < m) {
                    if (kF32Out)
                        static_cast<float*>(C)[i + j * ldc] = __double2float_rn(r[q]);
                    else
                        static_cast<double*>(C)[i + j * ldc] = r[q];
                }
            }
        }
    }
    tc_before();
    consumers_sync();
    if (warp == 0) {
        tc_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(Cf::kTmemCols));
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    }();
    return fn;
}

template <bool kF32Out, bool kPlain, int kMaxMod, int P, int R, int S>
bool launch_t(const CUtensorMap& map, int num_sms, cudaStream_t s, int64_t m, int64_t n, const int32_t* mu_exp,
              const int32_t* nu_exp, const DevConsts& c, const TcParams& tp, double alpha, double beta, void* C,
              int64_t ldc, bool vec_ok) {
    using Cf = TcCfg<R, S, P>;
    auto kern = reconstruct_tc_kernel<kF32Out, kPlain, kMaxMod, P, R, S>;
    constexpr int smem = Cf::kSmem;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        attr = true;
    }
    // blocks per SM from the resources (the occupancy API reports 1 for
    // kernels that allocate TMEM): shared memory, registers, TMEM columns
    static int per_sm = [&] {
        int dev = 0, smem_sm = 0, regs_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, kern);
        const int by_smem = smem_sm / (smem + static_cast<int>(fa.sharedSizeBytes) + 1024);
        const int regs_warp = (fa.numRegs * 32 + 255) / 256 * 256;
        const int by_regs = regs_sm / (regs_warp * (kThreads / 32));
        return std::min(std::min(by_smem, by_regs), 512 / Cf::kTmemCols);
    }();
    if (per_sm < 1) return false;
    const int64_t row_chunks = (m + Cf::kRows - 1) / Cf::kRows;
    const int64_t grid = std::min<int64_t>(row_chunks * n, static_cast<int64_t>(num_sms) * per_sm);
    static const int probe = std::getenv("OZK_K3_PROBE") ? std::atoi(std::getenv("OZK_K3_PROBE")) : 0;
    kern<<<static_cast<unsigned>(grid), kThreads, smem, s>>>(map, m, n, row_chunks, mu_exp, nu_exp, c, tp, alpha, beta,
                                                             C, ldc, vec_ok, kF32Out ? 0 : probe);
    return true;
}

int k3_tc_rows() {
    static const int r = [] {
        const char* e = std::getenv("OZK_K3_TC_ROWS");
        return e && std::atoi(e) == 4 ? 4 : 8;
    }();
    return r;
}

template <bool kF32Out, bool kPlain>
bool launch_variant(const CUtensorMap& map, int sms, cudaStream_t s, int64_t m, int64_t n, const int32_t* mu_exp,
                    const int32_t* nu_exp, const DevConsts& c, const TcParams& tp, double alpha, double beta, void* C,
                    int64_t ldc, bool vec_ok) {
#define OZK_K3T(MAXN, P)                                                                                     \
    (k3_tc_rows() == 8                                                                                           \
         ? launch_t<kF32Out, kPlain, MAXN, P, 8, P == 16 ? 3 : 2>(map, sms, s, m, n, mu_exp, nu_exp, c, tp, alpha, beta, C, ldc, \
                                                    vec_ok)                                                    \
         : launch_t<kF32Out, kPlain, MAXN, P, 4, 4>(map, sms, s, m, n, mu_exp, nu_exp, c, tp, alpha, beta, C, ldc, \
                                                    vec_ok))
    if (c.n <= 8) return OZK_K3T(8, 16);
    if (c.n <= 12) return OZK_K3T(12, 16);
    if (c.n <= 14) return OZK_K3T(14, 16);
    if (c.n <= 16) return OZK_K3T(16, 16);
    return OZK_K3T(OZK_MAX_MODULI, 24);
#undef OZK_K3T
}

// opt-in (OZK_K3_TC=1): measured slower than the all-FP64 bulk kernel at
// every N, so the production path does not take it
bool k3_tc_enabled() {
    static const bool b = [] {
        const char* e = std::getenv("OZK_K3_TC");
        return e && std::atoi(e) == 1;
    }();
    return b;
}

}  // namespace

// The tensor-core K3 for FP64 tables (see the header comment); returns false
// (nothing launched) when its preconditions do not hold, and the caller takes
// the all-FP64 kernel: FP32 tables (full-width s1, rounded products), an s1
// table that is not on a common grid below 2^48 / 2^53, a U layout TMA cannot
// describe, or OZK_K3_TC=0.
bool launch_reconstruct_tc(const uint8_t* u, int64_t ldu, int64_t stride, int64_t m, int64_t n, const int32_t* mu_exp,
                           const int32_t* nu_exp, const DevConsts& c, double alpha, double beta, void* C, int64_t ldc,
                           int c_is_f32, cudaStream_t s) {
    if (!k3_tc_enabled() || c.precision != OZK_FP64 || c.n < 1 || c.n > OZK_MAX_MODULI) return false;
    if (m < 1 || n < 1 || m > (int64_t(1) << 31) - 1024 || n > (int64_t(1) << 31) - 1) return false;
    if (reinterpret_cast<uintptr_t>(u) % 16 || ldu % 16 || stride % 16 || ldu < m) return false;
    // common grid 2^E of the s1 table and the exactness bound
    int E = 1 << 30;
    for (int t = 0; t < c.n; ++t) {
        const double v = c.s1[t];
        if (!(v >= 0.0) || std::isinf(v)) return false;
        if (v == 0.0) continue;
        int ex = 0;
        double fr = std::frexp(v, &ex);  // v = fr 2^ex, fr in [0.5, 1)
        unsigned long long mant = static_cast<unsigned long long>(std::ldexp(fr, 53));
        int lsb = ex - 53;
        while ((mant & 1ull) == 0) {
            mant >>= 1;
            ++lsb;
        }
        E = std::min(E, lsb);
    }
    if (E == (1 << 30)) E = 0;
    if (E < -1000 || E > 1023 - 52) return false;
    TcParams tp{};
    unsigned __int128 total = 0;
    for (int t = 0; t < c.n; ++t) {
        const double q = std::ldexp(c.s1[t], -E);
        if (q >= 0x1p48) return false;
        tp.s_int[t] = static_cast<unsigned long long>(q);
        if (static_cast<double>(tp.s_int[t]) != q) return false;
        total += static_cast<unsigned __int128>(tp.s_int[t]) * static_cast<unsigned>(c.p[t] - 1);
    }
    if (total >= (static_cast<unsigned __int128>(1) << 52)) return false;  // T < 2^52: one-DFMA conversion
    tp.sc0 = std::ldexp(1.0, E);
    tp.sc0m52 = -std::ldexp(1.0, E + 52);

    auto enc = encode_fn();
    if (!enc) return false;
    const int P = c.n <= 16 ? 16 : 24;
    CUtensorMap map;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(m), static_cast<cuuint64_t>(c.n), static_cast<cuuint64_t>(n)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(stride), static_cast<cuuint64_t>(ldu)};
    cuuint32_t box[3] = {128u, static_cast<cuuint32_t>(P), 1u};
    cuuint32_t estr[3] = {1, 1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(u), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;

    const int esz = c_is_f32 ? 4 : 8;
    const bool vec_ok = (reinterpret_cast<uintptr_t>(mu_exp) % 32 == 0) && (reinterpret_cast<uintptr_t>(C) % 32 == 0) &&
                        ((ldc * esz) % 32 == 0);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const bool plain = alpha == 1.0 && beta == 0.0;
    if (c_is_f32)
        return plain ? launch_variant<true, true>(map, sms, s, m, n, mu_exp, nu_exp, c, tp, alpha, beta, C, ldc, vec_ok)
                     : launch_variant<true, false>(map, sms, s, m, n, mu_exp, nu_exp, c, tp, alpha, beta, C, ldc,
                                                   vec_ok);
    return plain ? launch_variant<false, true>(map, sms, s, m, n, mu_exp, nu_exp, c, tp, alpha, beta, C, ldc, vec_ok)
                 : launch_variant<false, false>(map, sms, s, m, n, mu_exp, nu_exp, c, tp, alpha, beta, C, ldc, vec_ok);
}

}  // namespace ozk
