// K2 — the N residue GEMMs on the 5th-generation tensor cores
// (reference: int8_engine.cpp:15-64 + the fused mod of emulator.cpp:45-53 /
// reconstruct.hpp:31-37; accurate-mode bound product scaling.cpp:135-149).
//
// One persistent, warp-specialised kernel runs every (modulus, tile) work item:
//   warp 0      TMA producer: A/B K-major int8 tiles (128 B rows, 128B swizzle)
//               into a kStages-deep shared-memory ring (mbarrier full/empty);
//   warp 1      MMA issuer (one elected lane of the leader CTA):
//               tcgen05.mma.kind::i8, s32 accumulate in TMEM, no saturation,
//               so the single k = 2^17 overflow wraps exactly like the
//               reference's uint32 accumulator (int8_engine.cpp:12-38);
//   warp 2      TMEM allocator (two 256-column accumulators: the epilogue of
//               tile t overlaps the MMAs of tile t+1);
//   warps 4-11  epilogue (two per TMEM lane quarter, half the columns each):
//               tcgen05.ld 32 columns at a time, then
//               U8  : U_i = mod_u8(C'_i)  -> 1 byte per element to HBM,
//               I32 : raw C'_i (debug / parity export),
//               MAX : row/column maxima of Cbar via atomics (the reference
//                     materialises an m x n int64 Cbar; we never do).
// CG = 2 pairs the two SMs of a TPC (cta_group::2, UMMA 256 x 256 x 32): each
// CTA stages half of A's 256 rows and half of B's 256 columns, the leader
// issues, and both CTAs drain their 128 TMEM lanes. CG = 1 is the single-SM
// 128 x 256 variant (kept for small problems and as a bring-up fallback).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <string>

#include "ozk_device.cuh"

namespace ozk {
namespace {

constexpr int kBK = 128;  // bytes (= int8 elements) of K per stage: one 128B swizzle atom
constexpr int64_t kChunkK = OZK_ENGINE_MAX_K;  // longest exact int32 accumulation
constexpr int kAccCols = 256;
constexpr int kEpiWarp0 = 4;
constexpr int kEpiWarps = 8;  // two warps per TMEM lane quarter, each draining half the columns
constexpr int kThreads = 32 * (kEpiWarp0 + kEpiWarps);

template <int CG>
struct Cfg {
    static constexpr int kBM = 128;                 // A rows per CTA
    static constexpr int kTileM = 128 * CG;         // rows per work tile
    static constexpr int kTileN = 256;              // columns per work tile (UMMA N)
    static constexpr int kBRows = kTileN / CG;      // B rows staged per CTA
    static constexpr int kStageA = kBM * kBK;       // 16 KB
    static constexpr int kStageB = kBRows * kBK;    // 16 KB (CG 2) / 32 KB (CG 1)
    static constexpr int kStages = CG == 2 ? 6 : 4;
    static constexpr int kSmem = kStages * (kStageA + kStageB) + 1024 /*align*/ + 256 /*barriers*/;
    static constexpr uint32_t kTxBytes = static_cast<uint32_t>(CG * (kStageA + kStageB));
};

struct K2Params {
    int m, n, k;
    int n_mod;
    int tiles_m, tiles_n, num_kb;
    void* out;
    long long ldo;
    long long plane_out;
    int* rowmax;
    int* colmax;
    int acc_first;  // ACC64
    int p[OZK_MAX_MODULI];
    int pinv[OZK_MAX_MODULI];
    int group;             // tile rows per raster group
    int order;             // 1: moduli inner per wave of tiles (fused-K3 schedule prototype)
    int snake;             // odd groups sweep the columns right to left (B panels reused across the group edge)
    int hints;             // bit 0: A loads evict_last, bit 1: B loads evict_last, bit 3: B loads
                           // evict_first (bit 2, streaming U stores, measured no gain: removed)
    int sync_mode;         // 0 off; 1 tile lockstep (slack 1); 2 k-block lockstep
    int sync_window;       // mode 2: max k-blocks ahead of the slowest cluster
    int sync_every;        // mode 2: check every this many k-blocks
    unsigned int* done;    // mode 1: completed (cluster, tile) count
    unsigned int* progress;  // mode 2: issued k-blocks per cluster
    unsigned long long sync_timeout_ns;  // a lockstep wait longer than this abandons the lockstep
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
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
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_bar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
// relaxed: orders nothing but the arrival itself. The epilogue's TMEM reads are
// ordered by tcgen05.wait::ld + tcgen05.fence::before_thread_sync; its global
// stores need no ordering against the MMA warp, and a release at cluster scope
// compiles to a GPU-wide MEMBAR that waits for them (µs per tile at small k)
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t cluster_bar) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                            int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
        "[%2];" ::"r"(dst),
        "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
// 2-SM variant: the completion bytes land on the leader CTA's barrier.
__device__ __forceinline__ void tma_load_3d_2sm(uint32_t dst, const CUtensorMap* map, uint32_t leader_bar, int c0,
                                                int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
        "%4, %5}], [%2];" ::"r"(dst),
        "l"(map), "r"(leader_bar), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d_hint(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                                 int c2, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, "
        "%4, %5}], [%2], %6;" ::"r"(dst),
        "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d_2sm_hint(uint32_t dst, const CUtensorMap* map, uint32_t leader_bar, int c0,
                                                     int c1, int c2, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(dst),
        "l"(map), "r"(leader_bar), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void st_release(unsigned int* p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

template <int CG>
__device__ __forceinline__ void tmem_alloc(uint32_t slot_addr, uint32_t cols) {
    if constexpr (CG == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot_addr), "r"(cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot_addr), "r"(cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
}
template <int CG>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
    if constexpr (CG == 2)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols));
    else
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols));
}
template <int CG>
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    if constexpr (CG == 2)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
    else
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// tcgen05.commit: the barrier fires once all previously issued MMAs finish.
template <int CG>
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    if constexpr (CG == 2)
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                bar),
            "h"(static_cast<uint16_t>(3))
            : "memory");
    else
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                     : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptors (128B swizzle, Blackwell version 1). Both
// stage tiles are 128 rows of 128 B written by TMA, rows XOR-swizzled in
// groups of 8 (1024 B apart = SBO):
//  * B, K-major: a row is one n index with 128 k bytes; a k step of 32 moves
//    the start address 32 B inside the swizzle atom;
//  * A, MN-major: a row is one k index with 128 m bytes (one atom wide, so
//    LBO — the next-atom stride along M — is never used); a k step of 32 moves
//    32 rows = 4 atoms = 4096 B.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr, uint32_t lbo_bytes) {
    return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16) |
           (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
           (static_cast<uint64_t>(2) << 61);
}
// Instruction descriptor: s8 x s8 -> s32, operand majors (bit 15 A, bit 16 B;
// 1 = MN-major), no saturate.
template <int CG, bool A_MN, bool B_MN>
__host__ __device__ constexpr uint32_t idesc_i8() {
    return (2u << 4) | (1u << 7) | (1u << 10) | (A_MN ? (1u << 15) : 0u) | (B_MN ? (1u << 16) : 0u) |
           (static_cast<uint32_t>(Cfg<CG>::kTileN >> 3) << 17) | (static_cast<uint32_t>(Cfg<CG>::kTileM >> 4) << 24);
}

// work item t -> (modulus, tile row, tile column), grouped raster of G tile
// rows per modulus so the co-resident tiles share A/B panels in L2.
// order 1 (OZK_K2_ORDER=1, the schedule a K3 fused into K2's epilogue would
// need: every cluster runs all moduli of its tile back to back, so a tile's N
// residues meet on chip): waves of W = nclusters tiles, moduli inner — cluster
// c takes tile (wave * W + c) for modulus 0, 1, ..., N-1. Kept as a measured
// prototype of that schedule's DRAM cost ("Not fused").
__device__ __forceinline__ void decode_tile(int t, int tiles_m, int tiles_n, int G, int snake, int& mod, int& tm,
                                            int& tn, int order = 0, int n_mod = 1, int W = 1) {
    const int per_mod = tiles_m * tiles_n;
    int r;
    if (order == 1) {
        const int span = W * n_mod;
        const int wave = t / span;
        const int base = wave * W;
        const int rem = per_mod - base < W ? per_mod - base : W;
        const int idx = t - wave * span;
        mod = idx / rem;
        r = base + idx % rem;
    } else {
        mod = t / per_mod;
        r = t - mod * per_mod;
    }
    const int group = r / (G * tiles_n);
    const int first = group * G;
    const int gsize = tiles_m - first < G ? tiles_m - first : G;
    const int w = r - group * G * tiles_n;
    tm = first + w % gsize;
    tn = w / gsize;
    if (snake && (group & 1)) tn = tiles_n - 1 - tn;
}

// max over the 32 lanes of column `lane` of a 32 x 32 register tile
// (reduce-scatter butterfly: 31 shuffles instead of 32 x 5)
__device__ __forceinline__ int32_t column_max_scatter(uint32_t (&v)[32], int lane) {
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const bool upper = (lane & s) != 0;
#pragma unroll
        for (int j = 0; j < s; ++j) {
            const int32_t keep = static_cast<int32_t>(upper ? v[j + s] : v[j]);
            const int32_t send = static_cast<int32_t>(upper ? v[j] : v[j + s]);
            const int32_t recv = __shfl_xor_sync(0xffffffffu, send, s);
            v[j] = static_cast<uint32_t>(keep > recv ? keep : recv);
        }
    }
    return static_cast<int32_t>(v[0]);
}

// A_MN / B_MN: operand stored MN-major (A: column-major A; B: column-major B^T)
// or K-major (A: column-major A^T; B: column-major B). Both majors are native
// tcgen05 int8 operand forms, so the BLAS transposes cost nothing here.
template <int CG, int KIND, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(kThreads, 1)
    residue_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const K2Params P) {
    using C = Cfg<CG>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + C::kStages * C::kStageA;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::kStages * C::kStageB);
    uint64_t* empty = full + C::kStages;
    uint64_t* tfull = empty + C::kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
    const bool leader = rank == 0;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmB);
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull + a, 1);
            mbar_init(tempty + a, kEpiWarps * CG);  // one arrival per epilogue warp of every CTA
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<CG>(smem_u32(tmem_slot), 2 * kAccCols);
    tc_fence_before();
    if constexpr (CG == 2)
        cluster_sync();
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int total = P.n_mod * P.tiles_m * P.tiles_n;
    const int cluster_id = blockIdx.x / CG, nclusters = gridDim.x / CG;

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        // lane 0 issues; the whole warp joins the k-block lockstep checks
        int stage = 0;
        uint32_t phase = 0;
        const uint32_t full0_leader = CG == 2 ? mapa(smem_u32(full), 0) : smem_u32(full);
        const uint64_t pol_a = (P.hints & 1) ? policy_evict_last() : policy_evict_normal();
        const uint64_t pol_b = (P.hints & 2) ? policy_evict_last()
                                             : ((P.hints & 8) ? policy_evict_first() : policy_evict_normal());
        const bool kstep = P.sync_mode == 2 && leader;
        bool lockstep = P.sync_mode == 1 && leader;
        int lt = 0;
        for (int t = cluster_id; t < total; t += nclusters, ++lt) {
            if (lockstep && lt >= 1 && lane == 0) {
                // tile lockstep: every cluster's producer must have issued its tile
                // lt - 1. Counting producers (not MMA completion) lets this cluster
                // keep its ring full while it waits, so the MMA pipe does not drain.
                // The grid is capped at the co-resident cluster count, but other
                // work (another stream, NCCL, MPS limits) can still hold SMs a
                // cluster of this launch is waiting for: a wait longer than the
                // timeout (many tile durations) drops the lockstep for the rest
                // of this launch instead of deadlocking.
                const unsigned int need = static_cast<unsigned int>(min(total, lt * nclusters));
                const unsigned long long t0 = globaltimer_ns();
                while (ld_acquire(P.done) < need) {
                    __nanosleep(128);
                    if (globaltimer_ns() - t0 > P.sync_timeout_ns) {
                        lockstep = false;
                        break;
                    }
                }
            }
            __syncwarp();
            int mod, tm, tn;
            decode_tile(t, P.tiles_m, P.tiles_n, P.group, P.snake, mod, tm, tn, P.order, P.n_mod, nclusters);
            const int m0 = tm * C::kTileM + static_cast<int>(rank) * C::kBM;
            const int n0 = tn * C::kTileN + static_cast<int>(rank) * C::kBRows;
            for (int kb = 0; kb < P.num_kb; ++kb) {
                if (kstep && (kb % P.sync_every) == 0) {
                    // k-block lockstep: publish this cluster's issued k-blocks, then
                    // stay within `window` k-blocks of the slowest cluster
                    const unsigned int g = static_cast<unsigned int>(lt * P.num_kb + kb);
                    if (lane == 0) st_release(P.progress + cluster_id, g);
                    if (g > static_cast<unsigned int>(P.sync_window)) {
                        const unsigned int target = g - static_cast<unsigned int>(P.sync_window);
                        while (true) {
                            unsigned int lo = 0xffffffffu;
                            for (int cl = lane; cl < nclusters; cl += 32) lo = min(lo, ld_acquire(P.progress + cl));
#pragma unroll
                            for (int o = 16; o; o >>= 1) lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
                            if (lo >= target) break;
                            __nanosleep(128);
                        }
                    }
                }
                if (lane == 0) {
                    mbar_wait(smem_u32(empty + stage), phase ^ 1);
                    const uint32_t fb = smem_u32(full + stage);
                    if (leader) mbar_arrive_expect_tx(fb, C::kTxBytes);
                    const uint32_t dA = smem_u32(sA + stage * C::kStageA);
                    const uint32_t dB = smem_u32(sB + stage * C::kStageB);
                    // coordinates: MN-major maps are (mn, k), K-major maps (k, mn)
                    const int ac0 = A_MN ? m0 : kb * kBK, ac1 = A_MN ? kb * kBK : m0;
                    const int bc0 = B_MN ? n0 : kb * kBK, bc1 = B_MN ? kb * kBK : n0;
                    constexpr int kBBoxes = (B_MN && C::kBRows > 128) ? C::kBRows / 128 : 1;
                    if constexpr (CG == 2) {
                        const uint32_t lb = full0_leader + 8u * stage;
                        if (P.hints & 11) {
                            tma_load_3d_2sm_hint(dA, &tmA, lb, ac0, ac1, mod, pol_a);
                            tma_load_3d_2sm_hint(dB, &tmB, lb, bc0, bc1, mod, pol_b);
                        } else {
                            tma_load_3d_2sm(dA, &tmA, lb, ac0, ac1, mod);
                            tma_load_3d_2sm(dB, &tmB, lb, bc0, bc1, mod);
                        }
                    } else {
                        tma_load_3d(dA, &tmA, fb, ac0, ac1, mod);
#pragma unroll
                        for (int bx = 0; bx < kBBoxes; ++bx)  // MN atoms 16 KB apart (the descriptor's LBO)
                            tma_load_3d(dB + bx * 16384, &tmB, fb, bc0 + bx * 128, bc1, mod);
                    }
                }
                if (++stage == C::kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (P.sync_mode == 1 && leader && lane == 0) atomicAdd(P.done, 1u);  // tile lt fully issued
        }
        if (kstep && lane == 0) st_release(P.progress + cluster_id, 0xffffffffu);  // done: never the minimum
    } else if (warp == 1) {
        if (leader) {
            // ---------------- MMA issuer ----------------
            constexpr uint32_t idesc = idesc_i8<CG, A_MN, B_MN>();
            int stage = 0;
            uint32_t phase = 0;
            int lt = 0;
            for (int t = cluster_id; t < total; t += nclusters, ++lt) {
                const int acc = lt & 1;
                const uint32_t acc_phase = (lt >> 1) & 1;
                mbar_wait(smem_u32(tempty + acc), acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * kAccCols;
                for (int kb = 0; kb < P.num_kb; ++kb) {
                    mbar_wait(smem_u32(full + stage), phase);
                    tc_fence_after();
                    if (lane == 0) {
                        const uint32_t a0 = smem_u32(sA + stage * C::kStageA);
                        const uint32_t b0 = smem_u32(sB + stage * C::kStageB);
#pragma unroll
                        for (int kk = 0; kk < kBK / 32; ++kk) {
                            // MN-major: a 32-k step is 32 rows = 4 swizzle atoms (4096 B);
                            // atoms along MN are 16 KB apart (LBO). K-major: 32 B inside the atom.
                            const uint64_t da = A_MN ? sdesc_sw128(a0 + kk * 32 * kBK, 16384)
                                                     : sdesc_sw128(a0 + kk * 32, 16);
                            const uint64_t db = B_MN ? sdesc_sw128(b0 + kk * 32 * kBK, 16384)
                                                     : sdesc_sw128(b0 + kk * 32, 16);
                            mma_i8<CG>(d_tmem, da, db, idesc, (kb | kk) != 0);
                        }
                        mma_commit<CG>(smem_u32(empty + stage));
                    }
                    __syncwarp();
                    if (++stage == C::kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (lane == 0) mma_commit<CG>(smem_u32(tfull + acc));
                __syncwarp();
            }
        }
    } else if (warp >= kEpiWarp0) {
        // ---------------- epilogue ----------------
        const int q = (warp - kEpiWarp0) % 4;     // TMEM lane quarter (warp % 4: the lanes it may read)
        const int half = (warp - kEpiWarp0) / 4;  // which half of the tile's columns it drains
        const uint32_t tempty0_leader = CG == 2 ? mapa(smem_u32(tempty), 0) : smem_u32(tempty);
        int lt = 0;
        for (int t = cluster_id; t < total; t += nclusters, ++lt) {
            const int acc = lt & 1;
            const uint32_t acc_phase = (lt >> 1) & 1;
            int mod, tm, tn;
            decode_tile(t, P.tiles_m, P.tiles_n, P.group, P.snake, mod, tm, tn, P.order, P.n_mod, nclusters);
            mbar_wait(smem_u32(tfull + acc), acc_phase);
            tc_fence_after();
            const int row = tm * C::kTileM + static_cast<int>(rank) * C::kBM + q * 32 + lane;
            const bool row_ok = row < P.m;
            int32_t rmax = 0;
            constexpr int kChunks = C::kTileN / 32 / (kEpiWarps / 4);
            for (int cb = half * kChunks; cb < (half + 1) * kChunks; ++cb) {
                uint32_t v[32];
                tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * kAccCols + cb * 32, v);
                const int col0 = tn * C::kTileN + cb * 32;
                if constexpr (KIND == K2_U8 || KIND == K2_U8ACC) {
                    uint8_t* dst = static_cast<uint8_t*>(P.out) + static_cast<long long>(mod) * P.plane_out + row;
                    const int pm = P.p[mod], pinv = P.pinv[mod];
                    if (row_ok) {
                        uint8_t* q = dst + static_cast<long long>(col0) * P.ldo;
                        const long long ldo = P.ldo;
                        if constexpr (KIND == K2_U8) {
                            if (col0 + 32 <= P.n) {  // interior chunk: no per-column checks
#pragma unroll
                                for (int j = 0; j < 32; ++j) {
                                    *q = static_cast<uint8_t>(mod_u8(static_cast<int32_t>(v[j]), pm, pinv));
                                    q += ldo;
                                }
                                continue;
                            }
                        }
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            if (col0 + j < P.n) {
                                uint32_t u = mod_u8(static_cast<int32_t>(v[j]), pm, pinv);
                                if constexpr (KIND == K2_U8ACC) {
                                    // later k chunk (emulator.cpp:57-73): sum of per-block
                                    // residues, reduced again; u + old < 2p
                                    u += *q;
                                    u = u >= static_cast<uint32_t>(pm) ? u - pm : u;
                                }
                                *q = static_cast<uint8_t>(u);
                            }
                            q += ldo;
                        }
                    }
                } else if constexpr (KIND == K2_I32) {
                    int32_t* dst = static_cast<int32_t*>(P.out) + static_cast<long long>(mod) * P.plane_out + row;
                    if (row_ok) {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (col0 + j < P.n) dst[static_cast<long long>(col0 + j) * P.ldo] = static_cast<int32_t>(v[j]);
                    }
                } else if constexpr (KIND == K2_ACC64) {
                    // bound product over k > 2^19 (entries up to 64*64*k): int64 sum of
                    // 2^17-deep chunks, each exact in int32
                    long long* dst = static_cast<long long*>(P.out) + row;
                    if (row_ok) {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (col0 + j < P.n) {
                                long long* q = dst + static_cast<long long>(col0 + j) * P.ldo;
                                const long long x = static_cast<int32_t>(v[j]);
                                *q = P.acc_first ? x : *q + x;
                            }
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) rmax = max(rmax, static_cast<int32_t>(v[j]));
                    const int32_t cmax = column_max_scatter(v, lane);
                    if (col0 + lane < P.n) atomicMax(P.colmax + col0 + lane, cmax);
                }
            }
            if constexpr (KIND == K2_MAX) {
                if (row_ok) atomicMax(P.rowmax + row, rmax);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster_relaxed(tempty0_leader + 8u * acc);
        }
    }

    // ---------------- teardown ----------------
    __syncwarp();
    tc_fence_before();
    if constexpr (CG == 2)
        cluster_sync();
    else
        __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<CG>(tmem_base, 2 * kAccCols);
    }
    // the last cluster out resets the lockstep words for the next launch (no
    // per-launch memset; every other cluster is past all of its waits)
    if (P.sync_mode > 0 && leader && threadIdx.x == 0) {
        unsigned int* finished = P.done + 8;
        __threadfence();
        if (atomicAdd(finished, 1u) == static_cast<unsigned int>(nclusters - 1)) {
            *P.done = 0;
            if (P.sync_mode == 2)
                for (int cl = 0; cl < nclusters; ++cl) P.progress[cl] = 0;
            *finished = 0;
            __threadfence();
        }
    }
}

// ------------------------------------------------------------- host helpers
int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 3-D map over n_mod column-major planes (inner extent `inner` bytes within a
// column of `ld` bytes, `cols` columns, plane_stride bytes apart); box
// {128 inner bytes, box_cols columns, 1}
bool make_plane_map(CUtensorMap* map, const int8_t* base, int64_t inner, int64_t cols, int64_t ld, int64_t plane_stride,
                    int n_mod, int box_cols) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(n_mod)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld), static_cast<cuuint64_t>(plane_stride)};
    cuuint32_t box[3] = {128u, static_cast<cuuint32_t>(box_cols), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int CG, int KIND, bool A_MN, bool B_MN>
int launch_impl(const K2Launch& L, cudaStream_t s) {
    using C = Cfg<CG>;
    CUtensorMap ma, mb;
    // MN-major planes: mn inner, k columns, box 128 mn x 128 k; K-major planes:
    // k inner, mn columns, box 128 k x (128 | 256) mn. L.lda / L.ld are the
    // column pitches of the A / B planes in whichever major they are stored.
    const bool ok_a = A_MN ? make_plane_map(&ma, L.a_planes, L.m, L.k, L.lda, L.a_stride, L.n_mod, kBK)
                           : make_plane_map(&ma, L.a_planes, L.k, L.m, L.lda, L.a_stride, L.n_mod, C::kBM);
    const bool ok_b = B_MN ? make_plane_map(&mb, L.b_planes, L.n, L.k, L.ld, L.b_stride, L.n_mod, kBK)
                           : make_plane_map(&mb, L.b_planes, L.k, L.n, L.ld, L.b_stride, L.n_mod, C::kBRows);
    if (!ok_a || !ok_b) {
        set_error("cuTensorMapEncodeTiled failed");
        return OZK_CUDA_ERROR;
    }
    K2Params P{};
    P.m = static_cast<int>(L.m);
    P.n = static_cast<int>(L.n);
    P.k = static_cast<int>(L.k);
    P.n_mod = L.n_mod;
    P.tiles_m = static_cast<int>((L.m + C::kTileM - 1) / C::kTileM);
    P.tiles_n = static_cast<int>((L.n + C::kTileN - 1) / C::kTileN);
    P.num_kb = static_cast<int>((L.k + kBK - 1) / kBK);
    P.out = L.out;
    P.ldo = L.ldo;
    P.plane_out = L.out_stride;
    P.rowmax = L.rowmax;
    P.colmax = L.colmax;
    P.acc_first = L.acc_first ? 1 : 0;
    for (int i = 0; i < L.n_mod && L.c; ++i) {
        P.p[i] = L.c->p[i];
        P.pinv[i] = L.c->pinv_mulhi[i];
    }
    P.group = std::max(1, env_int("OZK_K2_GROUP", 8));
    P.snake = env_int("OZK_K2_SNAKE", 1);  // serpentine raster: -1.3 GB DRAM per launch, +0.5 % in the bench (DESIGN)
    P.order = env_int("OZK_K2_ORDER", 0);  // 1: moduli-inner waves (fused-K3 schedule prototype)
    P.hints = env_int("OZK_K2_HINTS", 9);  // A evict_last, B evict_first (profiles/r01_k2_hints_sweep.md)
    // Lockstep (default on): co-resident clusters that share A/B panels stay
    // within one tile of each other, so the panels they all stream are still in
    // L2 when the trailing cluster reads them. Measured at 16384^3, N=14: DRAM
    // reads 214 GB -> 57 GB per launch, and the power freed lifts the capped SM
    // clock 1.15 -> 1.48 GHz (profiles/). The counter is per handle.
    P.sync_mode = L.sync_counter ? env_int("OZK_K2_SYNC", 1) : 0;
    P.sync_window = env_int("OZK_K2_SYNC_WINDOW", 32);
    P.sync_every = env_int("OZK_K2_SYNC_EVERY", 8);
    if (P.sync_every < 1) P.sync_every = 1;
    P.sync_timeout_ns = 1000ull * static_cast<unsigned long long>(env_int("OZK_K2_SYNC_TIMEOUT_US", 20000));
    P.done = L.sync_counter;
    P.progress = L.sync_counter ? L.sync_counter + 16 : nullptr;
    // the lockstep words start at zero (the handle clears its flag buffer once)
    // and each launch's last cluster resets them
    const long long total = static_cast<long long>(L.n_mod) * P.tiles_m * P.tiles_n;
    long long clusters = L.num_sms / CG;
    if (clusters > total) clusters = total;
    if (clusters < 1) clusters = 1;

    auto kern = residue_gemm_kernel<CG, KIND, A_MN, B_MN>;
    static std::atomic<unsigned long long> attr_set{0};  // per instantiation and device
    static std::atomic<int> resident[64];                // co-resident clusters per device
    const int dev = current_device() & 63;
    if (needs_setup(attr_set)) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
        mark_setup(attr_set);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(clusters * CG));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // the persistent grid never exceeds the clusters the device can hold at once
    // (the lockstep waits on every cluster of the launch)
    int fit = resident[dev].load(std::memory_order_relaxed);
    if (!fit) {
        if (cudaOccupancyMaxActiveClusters(&fit, kern, &cfg) != cudaSuccess || fit < 1) {
            cudaGetLastError();
            fit = L.num_sms / CG;
        }
        resident[dev].store(fit, std::memory_order_relaxed);
    }
    if (clusters > fit) {
        clusters = fit;
        cfg.gridDim = dim3(static_cast<unsigned>(clusters * CG));
    }
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ma, mb, P);
    if (e != cudaSuccess) {
        set_error(std::string("residue_gemm launch: ") + cudaGetErrorString(e));
        return OZK_CUDA_ERROR;
    }
    return OZK_OK;
}

template <int CG, bool A_MN, bool B_MN>
int launch_kind(const K2Launch& L, cudaStream_t s) {
    switch (L.kind) {
        case K2_I32:
            return launch_impl<CG, K2_I32, A_MN, B_MN>(L, s);
        case K2_U8:
            return launch_impl<CG, K2_U8, A_MN, B_MN>(L, s);
        case K2_U8ACC:
            return launch_impl<CG, K2_U8ACC, A_MN, B_MN>(L, s);
        case K2_ACC64:
            return launch_impl<CG, K2_ACC64, A_MN, B_MN>(L, s);
        default:
            return launch_impl<CG, K2_MAX, A_MN, B_MN>(L, s);
    }
}

template <int CG>
int launch_layout(const K2Launch& L, cudaStream_t s) {
    if (L.a_mn) return L.b_mn ? launch_kind<CG, true, true>(L, s) : launch_kind<CG, true, false>(L, s);
    return L.b_mn ? launch_kind<CG, false, true>(L, s) : launch_kind<CG, false, false>(L, s);
}

}  // namespace

int k2_cta_group() {
    static int cg = 0;
    if (!cg) {
        const char* env = std::getenv("OZK_CTA_GROUP");
        cg = (env && env[0] == '1') ? 1 : 2;
    }
    return cg;
}

int launch_k2(const K2Launch& L, cudaStream_t s) {
    if (L.m > (1LL << 31) - 1 || L.n > (1LL << 31) - 1 || L.k > (1LL << 31) - 1) {
        set_error("residue_gemm: dimension exceeds 2^31");
        return OZK_INPUT_ERROR;
    }
    auto one = [&](const K2Launch& X) { return k2_cta_group() == 1 ? launch_layout<1>(X, s) : launch_layout<2>(X, s); };
    // One int32 accumulation stays exact for k <= 2^17 (only the benign
    // k = 2^17 wrap, int8_engine.hpp:19-22); U8 products over a longer k run in
    // chunks of 2^17, each chunk's residues added into U and reduced again —
    // the reference's blocked path (emulator.cpp:57-73), whose value does not
    // depend on where the blocks fall.
    if ((L.kind != K2_U8 && L.kind != K2_ACC64) || L.k <= kChunkK) return one(L);
    for (int64_t k0 = 0; k0 < L.k; k0 += kChunkK) {
        K2Launch X = L;
        X.k = L.k - k0 < kChunkK ? L.k - k0 : kChunkK;
        X.a_planes = L.a_planes + (L.a_mn ? k0 * L.lda : k0);  // MN-major: k columns; K-major: inside a column
        X.b_planes = L.b_planes + (L.b_mn ? k0 * L.ld : k0);
        if (L.kind == K2_U8)
            X.kind = k0 == 0 ? K2_U8 : K2_U8ACC;
        else
            X.acc_first = k0 == 0;
        const int st = one(X);
        if (st != OZK_OK) return st;
    }
    return OZK_OK;
}

}  // namespace ozk
