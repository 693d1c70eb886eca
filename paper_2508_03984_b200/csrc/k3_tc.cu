// K3 on the tensor cores with a verified C2 (FP64 tables; reference:
// emulator.cpp:49-53 weighted sums, reconstruct.hpp:51-54 crt_reduce_element,
// reconstruct.cpp:49-69 unscale).
//
// The reference forms, per output element, c1 = sum_i s1_i u_i and
// c2 = sum_i fl(s2_i u_i) (ascending i, every product and add rounded), then
// C'' = fma(-P2, Q, fl(fma(-P1, Q, c1) + c2)), Q = rint(P_inv c1).
// * c1 is exact: every s1_i is S1_i 2^E1 with sum_i S1_i (p_i - 1) < 2^52
//   (checked per call), so c1 = 2^E1 sum_i S1_i u_i, an integer dot product.
// * c2 carries roundings, but only its value near a rounding boundary of the
//   final result matters. s2_i = S2_i 2^E2 with S2_i < 2^64, so the exact sum
//   S = sum_i s2_i u_i is an integer dot product too, and the reference's
//   recursive sum of N rounded products satisfies |c2 - S| <= gamma_(N+1) S
//   (all terms are >= 0). With c2~ = fl(S) the interval
//   [c2~ - r, c2~ + r], r = (N + 3) 2^-53 c2~ (directed roundings) holds c2.
//   fl(X + y) and fma(-P2, Q, .) are monotone in y, so when both interval ends
//   give the same C'' bit pattern that IS the reference's C''. Otherwise (rare:
//   the interval is ~2^-48 c2 wide and c2 is ~2^-25 of X) the thread replays
//   the reference's sequential c2 from the planes still in shared memory.
// Both dot products are one tcgen05.mma.kind::i8 per 128-row group:
//   [128 rows x 32 moduli] (the U tile, u8, MN-major SW128, landed by one
//   TMA box {128 rows, P planes}) x [32 moduli x 16] (u8 digits, K-major:
//   columns 0-5 the base-256 digits of S1_i, 6-13 those of S2_i) -> s32 TMEM,
// each digit column sum_i D_ib u_i < 2^21. So the per-element FP64 chain of
// the all-FP64 kernel (4 FP64 ops per element and modulus) becomes a fixed
// 11 FP64 ops per element (c1 1, c2 2, Q 3, X 1, the interval ends 2 FMAs,
// C'' 1, unscale 1) in the column-tiled kernel, independent of N.
//
// Warp roles: warp 4 lane 0 issues the TMA boxes into an S-slot ring, lane 1
// the MMAs into a double-buffered TMEM accumulator (2 x 64
// columns: 4 groups x 16); warps 0-3 drain TMEM lanes 32w..32w+31 — the row
// 128 g + 32 w + lane of each group g — so every output row is finished by the
// thread that holds its digit sums (no exchange), and stores are coalesced.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "ozk_device.cuh"

namespace ozk {
namespace {

constexpr int kConsumers = 128;
constexpr int kThreads = kConsumers + 32;  // + one control warp (lane 0 TMA, lane 1 MMA)
constexpr int kGroups = 4;                 // 128-row MMA groups per tile
constexpr int kRows = 128 * kGroups;       // rows per tile (one column)
constexpr int kTmemCols = 2 * 16 * kGroups;  // two accumulator buffers

struct TcParams {
    unsigned long long s1_int[OZK_MAX_MODULI];  // S1_i = s1_i / 2^E1
    unsigned long long s2_int[OZK_MAX_MODULI];  // S2_i = s2_i / 2^E2
    double sc1, sc1m;                           // 2^E1, -2^(52+E1)
    double sc2h, sc2hm, sc2l, sc2lm;            // 2^(32+E2), -2^(84+E2), 2^E2, -2^(52+E2)
    double sc2b;                                // -(2^(84+E2) + 2^(52+E2))
    uint32_t l_hi;                              // high word of 2^(52+E2): (1075 + E2) << 20
    double rfac;                                // (N + 3) 2^-53
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
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, "
        "[%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }


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

template <int P, int S>
struct TcCfg {
    static constexpr int kGroupBytes = P * 128;
    static constexpr int kStageBytes = kGroups * kGroupBytes;
    // [S][4 groups][P planes][128 B] | B digits [16][128 B]. The K = 32 MMA
    // of a stage's last group reads (32 - P) planes past the stage: the next
    // stage or the digit block (those bytes meet zero digit rows).
    static constexpr int kSmem = 1024 /*align*/ + S * kStageBytes + 2048;
    static_assert((32 - P) * 128 <= 2048, "MMA over-read leaves the allocation");
};

// rint(y) for |y| < 2^51 by the round-to-nearest-even addition of 1.5 2^52
// (two DADDs on the FP64 pipe: FRND.F64 issues at ~1/4 of the DADD rate here,
// tools/micro/fp64_rate.cu): y + M is rounded to an integer, ties to even
// since M is even, and subtracting M is exact. Q = rint(P_inv c1) with
// 0 <= c1 < 2^52 2^E1 (checked per call) is far inside the range.
__device__ __forceinline__ double rint_small(double y) {
    constexpr double M = 6755399441055744.0;  // 1.5 * 2^52
    return __dadd_rn(__dadd_rn(y, M), -M);
}

// (2^52 + T) with T < 2^52 given as a 64-bit integer, as a double
__device__ __forceinline__ double pair52(uint64_t T) {
    return __hiloint2double(static_cast<int>(static_cast<uint32_t>(T >> 32) | 0x43300000u),
                            static_cast<int>(static_cast<uint32_t>(T)));
}
// (2^52 + x + 2^16 y) 2^e for x, y < 2^30 (x + 2^16 y < 2^52), with hi = the high
// word of 2^(52+e): the integer placed straight into the mantissa of a double
// of exponent 52 + e (no FP64 operation)
__device__ __forceinline__ double pair52_xy_hi(uint32_t x, uint32_t y, uint32_t hi_base) {
    uint32_t lo, hi;
    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, %5;"
        : "=r"(lo), "=r"(hi)
        : "r"(x), "r"(y << 16), "r"(y >> 16), "r"(hi_base));
    return __hiloint2double(static_cast<int>(hi), static_cast<int>(lo));
}
// 2^52 + x + 2^16 y (+ 2^32 z) for x, y, z < 2^30 without 64-bit arithmetic:
// low word x + (y << 16) with carry, high word 0x43300000 + (y >> 16) + z + carry
__device__ __forceinline__ double pair52_xyz(uint32_t x, uint32_t y, uint32_t z) {
    uint32_t lo, hi;
    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, %5;"
        : "=r"(lo), "=r"(hi)
        : "r"(x), "r"(y << 16), "r"(y >> 16), "r"(z + 0x43300000u));
    return __hiloint2double(static_cast<int>(hi), static_cast<int>(lo));
}

template <bool kF32Out, bool kPlain, bool kExact, int P, int S, int kTmemBatch = 2>
__global__ void __launch_bounds__(kThreads, 4)
    reconstruct_tc_kernel(const __grid_constant__ CUtensorMap umap, int64_t m, int64_t n, int64_t row_chunks,
                          const int32_t* __restrict__ mu_exp, const int32_t* __restrict__ nu_exp, const DevConsts c,
                          const TcParams tp, double alpha, double beta, void* __restrict__ C, int64_t ldc,
                          unsigned long long* __restrict__ replays) {
    using Cf = TcCfg<P, S>;
    constexpr int kGroupBytes = Cf::kGroupBytes, kStageBytes = Cf::kStageBytes;
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t full[S], empty[S], mma_full[2], tmem_empty[2];
    __shared__ uint32_t tmem_slot;
    uint8_t* sbuf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* bdig = sbuf + S * kStageBytes;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n_mod = c.n;
    if (tid == 0) {
        for (int st = 0; st < S; ++st) {
            mbar_init(saddr(&full[st]), 1);
            mbar_init(saddr(&empty[st]), kConsumers / 32);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(saddr(&mma_full[b]), 1);
            mbar_init(saddr(&tmem_empty[b]), kConsumers / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // B operand: digit row b (K-major, 128 B rows, 16-byte chunk k / 16
    // XOR-swizzled by b % 8 as TMA SW128 would): rows 0-5 the digits of S1_k,
    // rows 6-13 those of S2_k, rows 14-15 and moduli >= N zero
    for (int i = tid; i < 16 * 32; i += kThreads) {
        const int b = i >> 5, k = i & 31;
        uint32_t v = 0;
        if (k < n_mod && b < 6) v = static_cast<uint32_t>((tp.s1_int[k] >> (8 * b)) & 0xFFu);
        if (k < n_mod && b >= 6 && b < 14) v = static_cast<uint32_t>((tp.s2_int[k] >> (8 * (b - 6))) & 0xFFu);
        bdig[b * 128 + ((((k >> 4) ^ (b & 7)) << 4) | (k & 15))] = static_cast<uint8_t>(v);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tmem_slot)),
                     "n"(kTmemCols));
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

    if (warp == 4 && lane == 0) {  // TMA producer
        {
            const uint64_t pol = evict_first();
            for (int64_t k = 0, tile = blockIdx.x; tile < tiles; ++k, tile += gridDim.x, advance()) {
                const int st = static_cast<int>(k % S);
                mbar_wait_backoff(saddr(&empty[st]), static_cast<uint32_t>(((k / S) & 1) ^ 1));
                const int64_t i0 = chunk * kRows;
                const int64_t rem = (m - i0 + 127) / 128;
                const int ng = rem < kGroups ? static_cast<int>(rem) : kGroups;
                const uint32_t fb = saddr(&full[st]);
                mbar_expect_tx(fb, static_cast<uint32_t>(ng * kGroupBytes));
                const uint32_t dst = saddr(sbuf) + st * kStageBytes;
                for (int g = 0; g < ng; ++g)
                    tma_3d(dst + g * kGroupBytes, &umap, fb, static_cast<int>(i0 + 128 * g), 0, static_cast<int>(j),
                           pol);
            }
        }
        return;
    }
    if (warp == 4) {  // lane 1: MMA issuer
        if (lane == 1) {
            const uint64_t bd = sdesc_sw128(saddr(bdig));
            for (int64_t k = 0, tile = blockIdx.x; tile < tiles; ++k, tile += gridDim.x) {
                const int st = static_cast<int>(k % S), b = static_cast<int>(k & 1);
                mbar_wait(saddr(&full[st]), static_cast<uint32_t>((k / S) & 1));
                mbar_wait(saddr(&tmem_empty[b]), static_cast<uint32_t>(((k >> 1) & 1) ^ 1));
                tc_after();
                const uint32_t stage = saddr(sbuf) + st * kStageBytes;
#pragma unroll
                for (int g = 0; g < kGroups; ++g)
                    mma_u8(tbase + b * (16 * kGroups) + g * 16, sdesc_sw128(stage + g * kGroupBytes), bd);
                mma_commit(saddr(&mma_full[b]));
            }
        }
        return;
    }

    // consumers: row 128 g + 32 warp + lane of each group g
    const int rin = 32 * warp + lane;
    // swizzled byte of that row in plane t of group g: chunk rin / 16 XOR (t % 8)
    const uint32_t row_lo = static_cast<uint32_t>(rin & 15), row_chunk = static_cast<uint32_t>(rin >> 4);
    unsigned long long n_replay = 0;
    for (int64_t k = 0, tile = blockIdx.x; tile < tiles; ++k, tile += gridDim.x, advance()) {
        const int st = static_cast<int>(k % S), b = static_cast<int>(k & 1);
        const int64_t row0 = chunk * kRows;
        const int rows_left = m - row0 < kRows ? static_cast<int>(m - row0) : kRows;
        const int32_t* mu_t = mu_exp + row0 + rin;
        int me[kGroups];
#pragma unroll
        for (int g = 0; g < kGroups; ++g) me[g] = 128 * g + rin < rows_left ? __ldg(mu_t + 128 * g) : 0;
        const int ne = __ldg(nu_exp + j);
        mbar_wait(saddr(&mma_full[b]), static_cast<uint32_t>((k >> 1) & 1));
        tc_after();
        double c1[kGroups], c2[kGroups];
#pragma unroll
        for (int h = 0; h < kGroups / kTmemBatch; ++h) {
            uint32_t v[kTmemBatch][16];
            const uint32_t ta =
                tbase + (static_cast<uint32_t>(warp * 32) << 16) + b * (16 * kGroups) + h * (16 * kTmemBatch);
#pragma unroll
            for (int q = 0; q < kTmemBatch; ++q) tmem_ld16(ta + 16 * q, v[q]);
            tmem_wait_ld();
#pragma unroll
            for (int q = 0; q < kTmemBatch; ++q) {
                const uint32_t* w = v[q];
                // c1 = 2^E1 (X1 + 2^16 Y1 + 2^32 Z1) exactly: one DFMA on 2^52 + T1
                c1[kTmemBatch * h + q] = __fma_rn(
                    pair52_xyz(w[0] + (w[1] << 8), w[2] + (w[3] << 8), w[4] + (w[5] << 8)), tp.sc1, tp.sc1m);
                // S = 2^E2 (H 2^32 + L), H, L < 2^46: both parts exact, one rounding
                const double Lp = pair52_xyz(w[6] + (w[7] << 8), w[8] + (w[9] << 8), 0u);
                const double Hp = pair52_xyz(w[10] + (w[11] << 8), w[12] + (w[13] << 8), 0u);
                c2[kTmemBatch * h + q] = __dadd_rn(__fma_rn(Hp, tp.sc2h, tp.sc2hm), __fma_rn(Lp, tp.sc2l, tp.sc2lm));
            }
        }
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(saddr(&tmem_empty[b]));
        const uint32_t stage = saddr(sbuf) + st * kStageBytes;
        double* Cd = static_cast<double*>(C) + j * ldc + row0 + rin;
        float* Cf32 = static_cast<float*>(C) + j * ldc + row0 + rin;
#pragma unroll
        for (int g = 0; g < kGroups; ++g) {
            const bool live = 128 * g + rin < rows_left;
            const double qv = rint(__dmul_rn(c.P_inv, c1[g]));
            const double X = __fma_rn(-c.P1, qv, c1[g]);
            double cpp;
            bool decided = true;
            if constexpr (kExact) {  // c2 exact: no interval
                cpp = __fma_rn(-c.P2, qv, __dadd_rn(X, c2[g]));
            } else {
                const double rad = __dmul_ru(c2[g], tp.rfac);
                cpp = __fma_rn(-c.P2, qv, __dadd_rn(X, __dsub_rd(c2[g], rad)));
                const double zhi = __fma_rn(-c.P2, qv, __dadd_rn(X, __dadd_ru(c2[g], rad)));
                decided = __double_as_longlong(cpp) == __double_as_longlong(zhi) || !live;
            }
            // unscale by moving the exponent field (x and the result normal)
            const int e = -(me[g] + ne);
            const int hi = __double2hiint(cpp);
            const int ex = (hi >> 20) & 0x7ff;
            const bool normal = ex != 0 && static_cast<unsigned>(ex + e - 1) < 2046u;
            double r = __hiloint2double(hi + static_cast<int>(static_cast<unsigned>(e) << 20), __double2loint(cpp));
            // rare paths, taken warp-uniformly: the interval did not decide
            // (replay the reference's c2, emulator.cpp:53, from the planes) or
            // the unscale leaves the normal range (general ldexp)
            if (!__all_sync(0xffffffffu, decided && normal)) {
                if (!decided) {
                    const uint32_t line = stage + g * kGroupBytes + row_lo;
                    double c2r = 0.0;
#pragma unroll 1
                    for (int t = 0; t < n_mod; ++t) {
                        uint32_t ub;
                        asm volatile("ld.shared.u8 %0, [%1];"
                                     : "=r"(ub)
                                     : "r"(line + t * 128 + ((row_chunk ^ static_cast<uint32_t>(t & 7)) << 4)));
                        c2r = __dadd_rn(c2r, __fma_rn(c.s2[t], __hiloint2double(0x43300000, static_cast<int>(ub)),
                                                      c.s2_m52[t]));
                    }
                    cpp = __fma_rn(-c.P2, qv, __dadd_rn(X, c2r));
                    ++n_replay;
                }
                r = unscale_fast(cpp, e);
            }
            if (live) {
                if (!kPlain) {
                    const double old = beta != 0.0 ? (kF32Out ? static_cast<double>(Cf32[128 * g]) : Cd[128 * g]) : 0.0;
                    r = __dadd_rn(__dmul_rn(alpha, r), __dmul_rn(beta, old));
                }
                if (kF32Out)
                    Cf32[128 * g] = __double2float_rn(r);
                else
                    Cd[128 * g] = r;
            }
        }
        // slot st: the MMA has read it (mma_full) and any replay is done
        __syncwarp();
        if (lane == 0) mbar_arrive(saddr(&empty[st]));
    }
    if (replays && n_replay) atomicAdd(replays, n_replay);
    tc_before();
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
    if (warp == 0) {
        tc_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(kTmemCols));
    }
}

// ---------------------------------------------------------------------------
// Column-tiled variant (the default): a tile is 128 rows x 4 columns of C,
// landed by ONE TMA box {128 rows, P planes, 4 columns} (column q's planes at
// q * P * 128 B, the same MN-major SW128 operand layout per column), four MMAs
// (one per column) into a 64-column TMEM buffer. A consumer thread owns one
// row, so its mu and the row's unscale range check are loaded once per row
// chunk instead of per element, and the per-tile bookkeeping (barrier waits,
// TMEM addressing, exponent loads) is shared by 4 (kCW = 4) or 2 (kCW = 8)
// elements. kCW = 8: warps w and w + 4 drain the same TMEM lane quarter, two
// columns each (a warp may only read the lanes of its warp % 4 quarter).
// Per element: the digit combines, c1 (1 DFMA), c2~ (2 DFMA + DADD), Q (DMUL,
// FRND), X (DFMA), the interval ends as directed products c2~ (1 -+ rf)
// (2 DMUL) and sums (2 DADD), C'' (DFMA), and the unscale as one DMUL by 2^e:
// a correctly rounded product by a power of two IS ldexp's result (both round
// the exact value once, subnormal or overflowing results included), valid
// whenever 2^e is a normal double, which |mu|, |nu| <= 511 guarantees; other
// rows / columns, and undecided intervals, take the warp-uniform slow path.
constexpr int kTileCols = 4;

template <int P, int S, int kTC = kTileCols>
struct Tc4Cfg {
    static constexpr int kColBytes = P * 128;
    static constexpr int kStageBytes = kTC * kColBytes;
    static constexpr int kSmem = 1024 + S * kStageBytes + 2048;
    static_assert((32 - P) * 128 <= 2048, "MMA over-read leaves the allocation");
};

// wait with the hardware suspend hint: the thread sleeps in try_wait until the
// phase completes (or the hint expires) instead of re-issuing the poll, so
// waiting warps leave the issue slots to the warps that have work
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity), "r"(0x989680)
        : "memory");
}

// kFull: every row chunk and column group is complete and nu is 16-byte
// aligned (m % 128 == 0, n % kTC == 0: the bench shapes), so the per-tile bounds
// checks, the scalar exponent loads and the per-column store predicates drop out.
// kTC: columns per tile. kTC = 8 gives each consumer thread 8 columns per tile,
// reconstructed as two halves of 4 (the TMEM words of one half in registers at
// a time), so the per-tile work — ring waits, tile indices, exponent loads —
// is shared by 8 elements; its TMEM accumulator is single-buffered (8 x 16
// columns), which keeps 4 blocks per SM within the 512 TMEM columns.
template <bool kF32Out, bool kPlain, bool kExact, int P, int S, int kCW, bool kFull = false, int kTC = kTileCols>
__global__ void __launch_bounds__(32 * kCW + 32, kCW == 4 ? 4 : 3)
    reconstruct_tc4_kernel(const __grid_constant__ CUtensorMap umap, int m, int n, int row_chunks, int tiles,
                           const int32_t* __restrict__ mu_exp, const int32_t* __restrict__ nu_exp, int nu_vec,
                           const DevConsts c, const TcParams tp, double lo_fac, double hi_fac, double alpha,
                           double beta, void* __restrict__ C, int64_t ldc, unsigned long long* __restrict__ replays) {
    using Cf = Tc4Cfg<P, S, kTC>;
    using OutT = typename std::conditional<kF32Out, float, double>::type;
    constexpr int kColBytes = Cf::kColBytes, kStageBytes = Cf::kStageBytes;
    constexpr int kConsumersT = 32 * kCW;
    constexpr int kCPT = kTC * 4 / kCW;  // columns per consumer thread
    constexpr int kQ = kCPT < 4 ? kCPT : 4;  // columns per half (TMEM words of kQ columns live at once)
    constexpr int kHalves = kCPT / kQ;
    static_assert(!kFull || kCPT % 4 == 0, "the full-tile variant loads int4s of nu per thread");
    static_assert(kTC == kTileCols || (kFull && kCW == 4), "8-column tiles: full tiles, 4 consumer warps");
    constexpr int kNB = kTC == kTileCols ? 2 : 1;  // TMEM accumulator buffers
    constexpr uint32_t kBufCols = 16 * kTC;
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t full[S], empty[S], mma_full[2], tmem_empty[2];
    __shared__ uint32_t tmem_slot;
    uint8_t* sbuf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* bdig = sbuf + S * kStageBytes;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n_mod = c.n;
    if (tid == 0) {
        for (int st = 0; st < S; ++st) {
            mbar_init(saddr(&full[st]), 1);
            mbar_init(saddr(&empty[st]), kCW);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(saddr(&mma_full[b]), 1);
            mbar_init(saddr(&tmem_empty[b]), kCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < 16 * 32; i += blockDim.x) {  // B digits, as in reconstruct_tc_kernel
        const int b = i >> 5, k = i & 31;
        uint32_t v = 0;
        if (k < n_mod && b < 6) v = static_cast<uint32_t>((tp.s1_int[k] >> (8 * b)) & 0xFFu);
        if (k < n_mod && b >= 6 && b < 14) v = static_cast<uint32_t>((tp.s2_int[k] >> (8 * (b - 6))) & 0xFFu);
        bdig[b * 128 + ((((k >> 4) ^ (b & 7)) << 4) | (k & 15))] = static_cast<uint8_t>(v);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tmem_slot)),
                     "n"(kNB * kBufCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_before();
    __syncthreads();
    tc_after();
    const uint32_t tbase = tmem_slot;
    const uint32_t sb0 = saddr(sbuf);
    const uint32_t full0 = saddr(&full[0]), empty0 = saddr(&empty[0]);
    const uint32_t mfull0 = saddr(&mma_full[0]), tempty0 = saddr(&tmem_empty[0]);

    // tile t = chunk + row_chunks * cg: concurrently running blocks cover
    // neighbouring row chunks of the same columns
    const int dj = static_cast<int>(gridDim.x) / row_chunks, dr = static_cast<int>(gridDim.x) % row_chunks;
    int cg = static_cast<int>(blockIdx.x) / row_chunks, chunk = static_cast<int>(blockIdx.x) % row_chunks;
    const int step = gridDim.x;

    if (warp == kCW) {
        if (lane == 0) {  // TMA producer: one box per tile
            const uint64_t pol = evict_first();
            int st = 0;
            uint32_t ph = 1;
            for (int tile = blockIdx.x; tile < tiles; tile += step) {
                mbar_wait_backoff(empty0 + 8 * st, ph);
                const uint32_t fb = full0 + 8 * st;
                mbar_expect_tx(fb, static_cast<uint32_t>(kStageBytes));
                tma_3d(sb0 + st * kStageBytes, &umap, fb, chunk * 128, 0, cg * kTC, pol);
                chunk += dr;
                cg += dj;
                if (chunk >= row_chunks) {
                    chunk -= row_chunks;
                    ++cg;
                }
                if (++st == S) {
                    st = 0;
                    ph ^= 1u;
                }
            }
        } else if (lane == 1) {  // MMA issuer
            const uint64_t bd = sdesc_sw128(saddr(bdig));
            int st = 0, b = 0;
            uint32_t ph = 0, tph = 1;
            for (int tile = blockIdx.x; tile < tiles; tile += step) {
                mbar_wait_sleep(full0 + 8 * st, ph);
                mbar_wait_sleep(tempty0 + 8 * b, tph);
                tc_after();
                const uint32_t stage = sb0 + st * kStageBytes;
#pragma unroll
                for (int q = 0; q < kTC; ++q)
                    mma_u8(tbase + b * kBufCols + q * 16, sdesc_sw128(stage + q * kColBytes), bd);
                mma_commit(mfull0 + 8 * b);
                if (++st == S) {
                    st = 0;
                    ph ^= 1u;
                }
                if (++b == kNB) {
                    b = 0;
                    tph ^= 1u;
                }
            }
        }
        return;
    }

    // consumers: row 32 (warp % 4) + lane of the chunk, columns q0 .. q0 + kCPT - 1
    const int quarter = warp & 3;
    const int q0 = (warp >> 2) * kCPT;
    const int rin = 32 * quarter + lane;
    const uint32_t row_lo = static_cast<uint32_t>(rin & 15), row_chunk = static_cast<uint32_t>(rin >> 4);
    const uint32_t tq = tbase + (static_cast<uint32_t>(32 * quarter) << 16) + q0 * 16;
    unsigned long long n_replay = 0;
    // the exponents of tile k + 1 are loaded while tile k is reconstructed (the
    // loads take a full tile of time; issued right before their use they were
    // the kernel's largest stall); a full column group of an aligned nu is one
    // vector load
    auto load_exps = [&](int ch, int g, int& me_o, int (&ne_o)[kCPT]) {
        const int r = ch * 128 + rin;
        const int j = g * kTC + q0;
        if constexpr (kFull) {
            me_o = __ldg(mu_exp + r);
#pragma unroll
            for (int v4 = 0; v4 < kCPT / 4; ++v4) {
                const int4 v = __ldg(reinterpret_cast<const int4*>(nu_exp + j) + v4);
                ne_o[4 * v4] = v.x;
                ne_o[4 * v4 + 1] = v.y;
                ne_o[4 * v4 + 2] = v.z;
                ne_o[4 * v4 + 3] = v.w;
            }
            return;
        }
        me_o = r < m ? __ldg(mu_exp + r) : 0;
        if (nu_vec && j + kCPT <= n) {
            if constexpr (kCPT == 4) {
                const int4 v = __ldg(reinterpret_cast<const int4*>(nu_exp + j));
                ne_o[0] = v.x;
                ne_o[1] = v.y;
                ne_o[2] = v.z;
                ne_o[3] = v.w;
            } else {
                const int2 v = __ldg(reinterpret_cast<const int2*>(nu_exp + j));
                ne_o[0] = v.x;
                ne_o[1] = v.y;
            }
        } else {
#pragma unroll
            for (int q = 0; q < kCPT; ++q) ne_o[q] = j + q < n ? __ldg(nu_exp + j + q) : 0;
        }
    };
    int me_n, ne_n[kCPT];
    if (static_cast<int>(blockIdx.x) < tiles) load_exps(chunk, cg, me_n, ne_n);
    int st = 0, b = 0;
    uint32_t tph = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += step) {
        const int me = me_n;
        int ne[kCPT];
#pragma unroll
        for (int q = 0; q < kCPT; ++q) ne[q] = ne_n[q];
        const int row = chunk * 128 + rin;
        const int j0 = cg * kTC + q0;
        chunk += dr;
        cg += dj;
        if (chunk >= row_chunks) {
            chunk -= row_chunks;
            ++cg;
        }
        if (tile + step < tiles) load_exps(chunk, cg, me_n, ne_n);
        mbar_wait_sleep(mfull0 + 8 * b, tph);
        tc_after();
        const bool live_row = kFull || row < m;
        const uint32_t emp = empty0 + 8 * st;
#pragma unroll
        for (int h = 0; h < kHalves; ++h) {
            const int qb = h * kQ;  // this half's first column (of the thread's kCPT)
            double c1[kQ], cpp[kQ];
            uint32_t und = 0;  // bit q: the interval of column qb + q did not decide
            {
                uint32_t v[kQ][16];
#pragma unroll
                for (int q = 0; q < kQ; ++q) tmem_ld16(tq + b * kBufCols + 16 * (qb + q), v[q]);
                tmem_wait_ld();
                if (h == kHalves - 1) {  // the accumulator is free for the next tile's MMAs
                    tc_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(tempty0 + 8 * b);
                }
#pragma unroll
                for (int q = 0; q < kQ; ++q) {
                    const uint32_t* w = v[q];
                    c1[q] = __fma_rn(pair52_xyz(w[0] + (w[1] << 8), w[2] + (w[3] << 8), w[4] + (w[5] << 8)), tp.sc1,
                                     tp.sc1m);
                    // c2~ = fl(H 2^(32+E2) + L 2^E2) in two FP64 operations: Lb = (2^52 + L) 2^E2
                    // is built in the mantissa directly, fma(2^52 + H, 2^(32+E2),
                    // -(2^(84+E2) + 2^(52+E2))) = H 2^(32+E2) - 2^(52+E2) is exact (<= 46
                    // significant bits), and the one rounding is the final add
                    const double Lb = pair52_xy_hi(w[6] + (w[7] << 8), w[8] + (w[9] << 8), tp.l_hi);
                    const double Hp = pair52_xyz(w[10] + (w[11] << 8), w[12] + (w[13] << 8), 0u);
                    const double c2 = __dadd_rn(__fma_rn(Hp, tp.sc2h, tp.sc2b), Lb);
                    const double qv = rint_small(__dmul_rn(c.P_inv, c1[q]));
                    const double X = __fma_rn(-c.P1, qv, c1[q]);
                    if constexpr (kExact) {
                        cpp[q] = __fma_rn(-c.P2, qv, __dadd_rn(X, c2));
                    } else {
                        // c2 lies in [c2~ (1 - rf), c2~ (1 + rf)] (c2~ >= 0); fl(X + .) is
                        // monotone, so equal sums at both ends are fl(X + c2). The ends
                        // enter exactly (inside the FMA), one rounding each.
                        const double slo = __fma_rn(c2, lo_fac, X);
                        const double shi = __fma_rn(c2, hi_fac, X);
                        cpp[q] = __fma_rn(-c.P2, qv, slo);
                        und |= (__double_as_longlong(slo) != __double_as_longlong(shi) ? 1u : 0u) << q;
                    }
                }
            }
            const int cols = kFull ? kQ : min(n - (j0 + qb), kQ);  // live columns of this half (may be <= 0)
            bool ok = static_cast<unsigned>(me + 511) <= 1022u;
#pragma unroll
            for (int q = 0; q < kQ; ++q) ok = ok && static_cast<unsigned>(ne[qb + q] + 511) <= 1022u;
            OutT* cptr = static_cast<OutT*>(C) + static_cast<int64_t>(j0 + qb) * ldc + row;
            if (__all_sync(0xffffffffu, und == 0 && ok)) {
                if (h == kHalves - 1) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(emp);
                }
                if (live_row) {
                    const int pow_row = (1023 - me) << 20;
                    OutT* p = cptr;
#pragma unroll
                    for (int q = 0; q < kQ; ++q, p += ldc) {
                        if (q < cols) {
                            double r = __dmul_rn(cpp[q], __hiloint2double(pow_row - (ne[qb + q] << 20), 0));
                            if (!kPlain) {
                                const double old = beta != 0.0 ? static_cast<double>(*p) : 0.0;
                                r = __dadd_rn(__dmul_rn(alpha, r), __dmul_rn(beta, old));
                            }
                            *p = static_cast<OutT>(r);
                        }
                    }
                }
            } else {
                // rare, warp-uniform: an undecided interval (replay the reference's c2,
                // emulator.cpp:53, from the planes in shared memory) or an unscale
                // factor that is not a normal power of two (general ldexp)
                const uint32_t stage = sb0 + st * kStageBytes;
#pragma unroll
                for (int q = 0; q < kQ; ++q) {
                    double cq = cpp[q];
                    if (!kExact && ((und >> q) & 1u)) {
                        const double qv = rint_small(__dmul_rn(c.P_inv, c1[q]));
                        const double X = __fma_rn(-c.P1, qv, c1[q]);
                        const uint32_t line = stage + (q0 + qb + q) * kColBytes + row_lo;
                        double c2r = 0.0;
#pragma unroll 1
                        for (int t = 0; t < n_mod; ++t) {
                            uint32_t ub;
                            asm volatile("ld.shared.u8 %0, [%1];"
                                         : "=r"(ub)
                                         : "r"(line + t * 128 + ((row_chunk ^ static_cast<uint32_t>(t & 7)) << 4)));
                            c2r = __dadd_rn(c2r, __fma_rn(c.s2[t], __hiloint2double(0x43300000, static_cast<int>(ub)),
                                                          c.s2_m52[t]));
                        }
                        cq = __fma_rn(-c.P2, qv, __dadd_rn(X, c2r));
                        if (live_row && q < cols) ++n_replay;
                    }
                    if (live_row && q < cols) {
                        double r = unscale_fast(cq, -(me + ne[qb + q]));
                        if (!kPlain) {
                            const double old = beta != 0.0 ? static_cast<double>(cptr[q * ldc]) : 0.0;
                            r = __dadd_rn(__dmul_rn(alpha, r), __dmul_rn(beta, old));
                        }
                        cptr[q * ldc] = static_cast<OutT>(r);
                    }
                }
                if (h == kHalves - 1) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(emp);
                }
            }
        }
        if (++st == S) st = 0;
        if (++b == kNB) {
            b = 0;
            tph ^= 1u;
        }
    }
    if (replays && n_replay) atomicAdd(replays, n_replay);
    tc_before();
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumersT) : "memory");
    if (warp == 0) {
        tc_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(kNB * kBufCols));
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

template <bool kF32Out, bool kPlain, bool kExact, int P, int S>
bool launch_t(const CUtensorMap& map, int num_sms, cudaStream_t s, int64_t m, int64_t n, const int32_t* mu_exp,
              const int32_t* nu_exp, const DevConsts& c, const TcParams& tp, double alpha, double beta, void* C,
              int64_t ldc, unsigned long long* replays) {
    using Cf = TcCfg<P, S>;
    auto kern = reconstruct_tc_kernel<kF32Out, kPlain, kExact, P, S>;
    constexpr int smem = Cf::kSmem;
    static std::atomic<unsigned long long> attr{0};  // per instantiation and device
    static std::atomic<int> per_sm_dev[64];
    const int dev = current_device() & 63;
    if (needs_setup(attr)) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        mark_setup(attr);
    }
    // blocks per SM from the resources (the occupancy API reports 1 for
    // kernels that allocate TMEM): shared memory, registers, TMEM columns
    int per_sm = per_sm_dev[dev].load(std::memory_order_relaxed);
    if (!per_sm) per_sm = [&] {
        int smem_sm = 0, regs_sm = 0;
        cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, kern);
        const int by_smem = smem_sm / (smem + static_cast<int>(fa.sharedSizeBytes) + 1024);
        const int regs_warp = (fa.numRegs * 32 + 255) / 256 * 256;
        const int by_regs = regs_sm / (regs_warp * (kThreads / 32));
        const int v = std::min(std::min(by_smem, by_regs), 512 / kTmemCols);
        per_sm_dev[dev].store(v < 1 ? -1 : v, std::memory_order_relaxed);
        return v < 1 ? -1 : v;
    }();
    if (per_sm < 1) return false;
    const int64_t row_chunks = (m + kRows - 1) / kRows;
    const int64_t grid = std::min<int64_t>(row_chunks * n, static_cast<int64_t>(num_sms) * per_sm);
    kern<<<static_cast<unsigned>(grid), kThreads, smem, s>>>(map, m, n, row_chunks, mu_exp, nu_exp, c, tp, alpha, beta,
                                                             C, ldc, replays);
    return true;
}

// the column-tiled kernel (reconstruct_tc4_kernel): kCW consumer warps
template <bool kF32Out, bool kPlain, bool kExact, int P, int S, int kCW, bool kFull = false, int kTC = kTileCols>
bool launch_t4(const CUtensorMap& map, int num_sms, cudaStream_t s, int64_t m, int64_t n, const int32_t* mu_exp,
               const int32_t* nu_exp, const DevConsts& c, const TcParams& tp, double lo_fac, double hi_fac,
               double alpha, double beta, void* C, int64_t ldc, unsigned long long* replays) {
    using Cf = Tc4Cfg<P, S, kTC>;
    auto kern = reconstruct_tc4_kernel<kF32Out, kPlain, kExact, P, S, kCW, kFull, kTC>;
    constexpr int smem = Cf::kSmem;
    constexpr int threads = 32 * kCW + 32;
    constexpr int tmem_cols = (kTC == kTileCols ? 2 : 1) * 16 * kTC;
    static std::atomic<unsigned long long> attr{0};
    static std::atomic<int> per_sm_dev[64];
    const int dev = current_device() & 63;
    if (needs_setup(attr)) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        mark_setup(attr);
    }
    int per_sm = per_sm_dev[dev].load(std::memory_order_relaxed);
    if (!per_sm) per_sm = [&] {
        int smem_sm = 0, regs_sm = 0;
        cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, kern);
        const int by_smem = smem_sm / (smem + static_cast<int>(fa.sharedSizeBytes) + 1024);
        const int regs_warp = (fa.numRegs * 32 + 255) / 256 * 256;
        const int by_regs = regs_sm / (regs_warp * (threads / 32));
        const int v = std::min(std::min(by_smem, by_regs), 512 / tmem_cols);
        per_sm_dev[dev].store(v < 1 ? -1 : v, std::memory_order_relaxed);
        return v < 1 ? -1 : v;
    }();
    if (per_sm < 1) return false;
    const int64_t row_chunks = (m + 127) / 128;
    const int64_t tiles = row_chunks * ((n + kTC - 1) / kTC);
    const int64_t grid = std::min<int64_t>(tiles, static_cast<int64_t>(num_sms) * per_sm);
    if (tiles + grid >= (int64_t(1) << 31)) return false;  // 32-bit tile arithmetic
    constexpr int cpt = kTC * 4 / kCW;
    const int nu_vec = reinterpret_cast<uintptr_t>(nu_exp) % (4 * cpt) == 0;
    kern<<<static_cast<unsigned>(grid), threads, smem, s>>>(
        map, static_cast<int>(m), static_cast<int>(n), static_cast<int>(row_chunks), static_cast<int>(tiles), mu_exp,
        nu_exp, nu_vec, c, tp, lo_fac, hi_fac, alpha, beta, C, ldc, replays);
    return true;
}

// OZK_K3_TILE=1: the 512-row x 1-column kernel (reconstruct_tc_kernel, A/B timing); 8: the
// column-tiled kernel with 8-column tiles where the tiles are full (default 4);
// OZK_K3_CW: consumer warps of the column-tiled kernel (4 or 8, default 4)
int k3_tile_mode() {
    static const int v = [] {
        const char* e = std::getenv("OZK_K3_TILE");
        return e ? std::atoi(e) : 4;
    }();
    return v;
}
int k3_consumer_warps() {
    static const int v = [] {
        const char* e = std::getenv("OZK_K3_CW");
        return e && std::atoi(e) == 8 ? 8 : 4;
    }();
    return v;
}

// OZK_K3_FULL=0: never take the full-tile instantiation (A/B timing, tests)
int k3_full_tiles() {
    static const int v = [] {
        const char* e = std::getenv("OZK_K3_FULL");
        return e ? std::atoi(e) : 1;
    }();
    return v;
}

int k3_stages() {
    static const int v = [] {
        const char* e = std::getenv("OZK_K3_STAGES");
        const int x = e ? std::atoi(e) : 6;
        return x == 4 || x == 8 ? x : 6;
    }();
    return v;
}

template <bool kF32Out, bool kPlain, bool kExact, int P>
bool launch_t4_cw(const CUtensorMap& map, const CUtensorMap& map8, int sms, cudaStream_t s, int64_t m, int64_t n, const int32_t* mu_exp,
                  const int32_t* nu_exp, const DevConsts& c, const TcParams& tp, double lo_fac, double hi_fac,
                  double alpha, double beta, void* C, int64_t ldc, unsigned long long* replays) {
    if (k3_consumer_warps() == 8)
        return launch_t4<kF32Out, kPlain, kExact, P, 4, 8>(map, sms, s, m, n, mu_exp, nu_exp, c, tp, lo_fac, hi_fac,
                                                           alpha, beta, C, ldc, replays);
    if (k3_stages() == 8)
        return launch_t4<kF32Out, kPlain, kExact, P, 8, 4>(map, sms, s, m, n, mu_exp, nu_exp, c, tp, lo_fac, hi_fac,
                                                           alpha, beta, C, ldc, replays);
    const bool full = k3_full_tiles() && m % 128 == 0 && reinterpret_cast<uintptr_t>(nu_exp) % 16 == 0;
    if (full && k3_tile_mode() == 8 && n % 8 == 0)
        return launch_t4<kF32Out, kPlain, kExact, P, 3, 4, true, 8>(map8, sms, s, m, n, mu_exp, nu_exp, c, tp, lo_fac,
                                                                    hi_fac, alpha, beta, C, ldc, replays);
    if (k3_stages() == 6) {
        if (full && n % kTileCols == 0)
            return launch_t4<kF32Out, kPlain, kExact, P, 6, 4, true>(map, sms, s, m, n, mu_exp, nu_exp, c, tp, lo_fac,
                                                                     hi_fac, alpha, beta, C, ldc, replays);
        return launch_t4<kF32Out, kPlain, kExact, P, 6, 4>(map, sms, s, m, n, mu_exp, nu_exp, c, tp, lo_fac, hi_fac,
                                                           alpha, beta, C, ldc, replays);
    }
    return launch_t4<kF32Out, kPlain, kExact, P, 4, 4>(map, sms, s, m, n, mu_exp, nu_exp, c, tp, lo_fac, hi_fac, alpha,
                                                       beta, C, ldc, replays);
}

template <bool kF32Out, bool kPlain>
bool launch_variant(const CUtensorMap& map, const CUtensorMap& map4, const CUtensorMap& map8, int sms, cudaStream_t s, int64_t m, int64_t n,
                    const int32_t* mu_exp, const int32_t* nu_exp, const DevConsts& c, const TcParams& tp,
                    double lo_fac, double hi_fac, double alpha, double beta, void* C, int64_t ldc,
                    unsigned long long* replays) {
    if (k3_tile_mode() != 1) {
        bool ok;
        if (tp.rfac == 0.0)
            ok = launch_t4_cw<kF32Out, kPlain, true, 16>(map4, map8, sms, s, m, n, mu_exp, nu_exp, c, tp, lo_fac, hi_fac,
                                                        alpha, beta, C, ldc, replays);
        else if (c.n <= 16)
            ok = launch_t4_cw<kF32Out, kPlain, false, 16>(map4, map8, sms, s, m, n, mu_exp, nu_exp, c, tp, lo_fac, hi_fac,
                                                         alpha, beta, C, ldc, replays);
        else
            ok = launch_t4_cw<kF32Out, kPlain, false, 24>(map4, map8, sms, s, m, n, mu_exp, nu_exp, c, tp, lo_fac, hi_fac,
                                                         alpha, beta, C, ldc, replays);
        if (ok) return true;
    }
    if (tp.rfac == 0.0)  // c2 exact (N <= 10): no interval, never a replay
        return launch_t<kF32Out, kPlain, true, 16, 4>(map, sms, s, m, n, mu_exp, nu_exp, c, tp, alpha, beta, C, ldc,
                                                      replays);
    if (c.n <= 16)
        return launch_t<kF32Out, kPlain, false, 16, 4>(map, sms, s, m, n, mu_exp, nu_exp, c, tp, alpha, beta, C, ldc,
                                                       replays);
    return launch_t<kF32Out, kPlain, false, 24, 4>(map, sms, s, m, n, mu_exp, nu_exp, c, tp, alpha, beta, C, ldc,
                                                   replays);
}

// OZK_K3_TC=0 selects the all-FP64 bulk kernel (A/B timing)
bool k3_tc_enabled() {
    static const bool b = [] {
        const char* e = std::getenv("OZK_K3_TC");
        return !(e && std::atoi(e) == 0);
    }();
    return b;
}

// lowest set bit exponent of a positive finite double
int lsb_exponent(double v) {
    int ex = 0;
    const double fr = std::frexp(v, &ex);
    unsigned long long mant = static_cast<unsigned long long>(std::ldexp(fr, 53));
    int lsb = ex - 53;
    while ((mant & 1ull) == 0) {
        mant >>= 1;
        ++lsb;
    }
    return lsb;
}

// S_i = v_i / 2^E on the common grid of the table (E = the lowest set bit);
// false if a value is negative / non-finite or an integer exceeds `max_bits`
bool integer_table(const double* v, int n, int max_bits, int* E_out, unsigned long long* out) {
    int E = 1 << 30;
    for (int t = 0; t < n; ++t) {
        if (!(v[t] >= 0.0) || std::isinf(v[t])) return false;
        if (v[t] != 0.0) E = std::min(E, lsb_exponent(v[t]));
    }
    if (E == (1 << 30)) E = 0;
    for (int t = 0; t < n; ++t) {
        const double q = std::ldexp(v[t], -E);
        if (q >= std::ldexp(1.0, max_bits)) return false;
        out[t] = static_cast<unsigned long long>(q);
        if (static_cast<double>(out[t]) != q) return false;
    }
    *E_out = E;
    return true;
}

}  // namespace

// per-device counters of replayed elements (tests / tools read them through
// ozk_k3_replays); nullptr until first asked for on that device
namespace {
constexpr int kMaxDevices = 64;
unsigned long long* g_replays[kMaxDevices] = {};
}  // namespace
unsigned long long* k3_replay_counter(bool create) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return nullptr;
    if (!g_replays[dev] && create) {
        unsigned long long* p = nullptr;
        if (cudaMalloc(&p, sizeof(unsigned long long)) != cudaSuccess) return nullptr;
        cudaMemset(p, 0, sizeof(unsigned long long));
        g_replays[dev] = p;
    }
    return g_replays[dev];
}

// The tensor-core K3 for FP64 tables (see the header comment); returns false
// (nothing launched) when its preconditions do not hold and the caller takes
// the all-FP64 kernel: FP32 tables (full-width s1, rounded products), tables
// off the integer grids checked here, a U layout TMA cannot describe, or
// OZK_K3_TC=0.
bool launch_reconstruct_tc(const uint8_t* u, int64_t ldu, int64_t stride, int64_t m, int64_t n, const int32_t* mu_exp,
                           const int32_t* nu_exp, const DevConsts& c, double alpha, double beta, void* C, int64_t ldc,
                           int c_is_f32, cudaStream_t s) {
    if (!k3_tc_enabled() || c.precision != OZK_FP64 || c.n < 1 || c.n > OZK_MAX_MODULI) return false;
    if (m < 1 || n < 1 || m > (int64_t(1) << 31) - 1024 || n > (int64_t(1) << 31) - 1) return false;
    if (reinterpret_cast<uintptr_t>(u) % 16 || ldu % 16 || stride % 16 || ldu < m) return false;
    TcParams tp{};
    int E1 = 0, E2 = 0;
    if (!integer_table(c.s1, c.n, 48, &E1, tp.s1_int)) return false;
    if (!integer_table(c.s2, c.n, 64, &E2, tp.s2_int)) return false;
    unsigned __int128 total = 0;  // c1 exact and T1 < 2^52 (one-DFMA conversion)
    for (int t = 0; t < c.n; ++t) total += static_cast<unsigned __int128>(tp.s1_int[t]) * static_cast<unsigned>(c.p[t] - 1);
    if (total >= (static_cast<unsigned __int128>(1) << 52)) return false;
    // Q = rint_small(P_inv c1) needs P_inv c1 < 2^51: c1 < 2^(52 + E1)
    if (!(c.P_inv >= 0.0) || c.P_inv * std::ldexp(1.0, 52 + E1) >= std::ldexp(1.0, 50)) return false;
    if (E1 < -1000 || E1 > 1023 - 52 || E2 < -1000 || E2 > 1023 - 84) return false;
    tp.sc1 = std::ldexp(1.0, E1);
    tp.sc1m = -std::ldexp(1.0, E1 + 52);
    tp.sc2h = std::ldexp(1.0, E2 + 32);
    tp.sc2hm = -std::ldexp(1.0, E2 + 84);
    tp.sc2l = std::ldexp(1.0, E2);
    tp.sc2lm = -std::ldexp(1.0, E2 + 52);
    tp.sc2b = -(std::ldexp(1.0, E2 + 84) + std::ldexp(1.0, E2 + 52));
    tp.l_hi = static_cast<uint32_t>(1075 + E2) << 20;
    // with every s2_i u_i and every partial sum on the 2^E2 grid below 2^53
    // the reference's c2 is exact (= S), so the interval collapses
    unsigned __int128 total2 = 0;
    for (int t = 0; t < c.n; ++t)
        total2 += static_cast<unsigned __int128>(tp.s2_int[t]) * static_cast<unsigned>(c.p[t] - 1);
    tp.rfac = total2 < (static_cast<unsigned __int128>(1) << 53) ? 0.0 : (c.n + 3) * 0x1p-53;
    // test hook: a radius of c2 itself sends (almost) every element through
    // the replay of the reference's sequential c2
    static const bool replay_all = [] {
        const char* e = std::getenv("OZK_K3_REPLAY_ALL");
        return e && std::atoi(e) == 1;
    }();
    if (replay_all) tp.rfac = 1.0;

    // interval ends as directed products: c2~ (1 - rf) is exact-representable
    // scaled by a representable factor; 1 + rf rounded up to the 2^-52 grid
    const double lo_fac = 1.0 - tp.rfac;
    const double hi_fac = 1.0 + std::ceil(tp.rfac * 0x1p52) * 0x1p-52;

    auto enc = encode_fn();
    if (!enc) return false;
    const int P = c.n <= 16 ? 16 : 24;
    CUtensorMap map, map4, map8;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(m), static_cast<cuuint64_t>(c.n), static_cast<cuuint64_t>(n)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(stride), static_cast<cuuint64_t>(ldu)};
    cuuint32_t box[3] = {128u, static_cast<cuuint32_t>(P), 1u};
    cuuint32_t box4[3] = {128u, static_cast<cuuint32_t>(P), static_cast<cuuint32_t>(kTileCols)};
    cuuint32_t box8[3] = {128u, static_cast<cuuint32_t>(P), 8u};
    cuuint32_t estr[3] = {1, 1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(u), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    if (enc(&map4, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(u), dims, strides, box4, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    if (enc(&map8, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(u), dims, strides, box8, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;

    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    unsigned long long* replays = k3_replay_counter(false);
    const bool plain = alpha == 1.0 && beta == 0.0;
    if (c_is_f32)
        return plain ? launch_variant<true, true>(map, map4, map8, sms, s, m, n, mu_exp, nu_exp, c, tp, lo_fac, hi_fac,
                                                  alpha, beta, C, ldc, replays)
                     : launch_variant<true, false>(map, map4, map8, sms, s, m, n, mu_exp, nu_exp, c, tp, lo_fac, hi_fac,
                                                   alpha, beta, C, ldc, replays);
    return plain ? launch_variant<false, true>(map, map4, map8, sms, s, m, n, mu_exp, nu_exp, c, tp, lo_fac, hi_fac, alpha,
                                               beta, C, ldc, replays)
                 : launch_variant<false, false>(map, map4, map8, sms, s, m, n, mu_exp, nu_exp, c, tp, lo_fac, hi_fac, alpha,
                                                beta, C, ldc, replays);
}

}  // namespace ozk
