/* ozaki2_b200.h — C ABI of the B200-native Ozaki scheme II GEMM emulation.
 *
 * This is the drop-in boundary for the reference's public C++ entry points
 * (/root/reference/proj/include/crtgemm). Plain pointers and sizes only: no
 * torch, no C++ types. The C++ drop-in (include/crtgemm/emulator.hpp,
 * built into the same library) and the Python host mirror
 * (paper_2508_03984_b200/) both sit on top of these functions.
 *
 * Conventions (reference matrix.hpp:9-32): matrices are column-major; every
 * GEMM computes C = alpha * (A x B) + beta * C with A m x k, B k x n, C m x n.
 * The reference has no alpha/beta: alpha = 1, beta = 0
 * reproduces it bit-for-bit; other values are applied in FP64 after
 * reconstruction (extension named by BASELINE.json's north star).
 *
 * Status codes map the reference exception taxonomy (errors.hpp:8-27):
 *   OZK_CONFIG_ERROR <- crtgemm::ConfigError, OZK_INPUT_ERROR <- InputError,
 *   OZK_DOMAIN_ERROR <- std::domain_error (mod_inverse).
 * A CUDA failure returns OZK_CUDA_ERROR; ozk_last_error() has the message.
 * There is no CPU fallback: without a B200 every compute entry point fails
 * with OZK_CUDA_ERROR.
 */
#ifndef OZAKI2_B200_H
#define OZAKI2_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OZK_OK 0
#define OZK_CONFIG_ERROR 1
#define OZK_INPUT_ERROR 2
#define OZK_CUDA_ERROR 3
#define OZK_DOMAIN_ERROR 4
#define OZK_INTERNAL_ERROR 5

#define OZK_MAX_MODULI 20
#define OZK_ENGINE_MAX_K (1 << 17) /* int8_engine.hpp:12 kEngineMaxK */

/* Precision (crt_tables.hpp:11) and ScaleMode (scaling.hpp:12) */
#define OZK_FP64 0
#define OZK_FP32 1
#define OZK_FAST 0
#define OZK_ACCURATE 1

/* ozk_config.flags. OZK_FLAG_FAST_EXPONENT_FIX: fast-mode scaling subtracts
 * the row/column max exponent g = floor(log2 max|x|), which the reference
 * omits (scaling.cpp:50-56 vs PAPER.md:313-314); without it the
 * reference's fast mode breaks the CRT range for |x| >= 2 rows/columns. Off by
 * default: results then equal the reference bit for bit. */
#define OZK_FLAG_FAST_EXPONENT_FIX 1
/* BLAS transposes (extension; the reference takes op(X) = X only,
 * emulator.hpp:23-32). C = alpha * op(A) * op(B) + beta * C with op(A) m x k,
 * op(B) k x n. OZK_FLAG_TRANS_A: A is stored k x m (column-major, lda >= k) and
 * op(A) = A^T; OZK_FLAG_TRANS_B: B is stored n x k (ldb >= n), op(B) = B^T.
 * Results equal the reference's gemm_emulated(op(A), op(B)) bit for bit; no
 * transpose is materialised (the GEMM reads either operand major). The stage
 * API (ozk_stage_residues / ozk_stage_products) takes untransposed operands. */
#define OZK_FLAG_TRANS_A 2
#define OZK_FLAG_TRANS_B 4
/* Stream-ordered call (extension): device-pointer entry points (ozk_gemm,
 * ozk_dgemm_ex, strided batches, the shard APIs) return after enqueuing, with
 * no host synchronisation, so back-to-back calls pipeline and a call can be
 * captured into a CUDA graph (after one warm-up call has sized the workspace).
 * The non-finite-input check (emulator.cpp:19-22) is then deferred: its flag
 * accumulates on the device until ozk_sync, which returns OZK_INPUT_ERROR if
 * any call since the last ozk_sync saw NaN/Inf. Without the flag every call
 * synchronises and reports it, like the reference. */
#define OZK_FLAG_ASYNC 8

/* storage types of A/B/C buffers */
#define OZK_R64F 0
#define OZK_R32F 1

/* Stage-2 output kinds for ozk_stage_products (debug/parity export) */
#define OZK_PRODUCTS_I32 0 /* raw wrapping int32 C'_i (int8_engine.hpp:19-24) */
#define OZK_PRODUCTS_U8 1  /* U_i = mod(C'_i, p_i)      (reconstruct.hpp:28-37) */

/* The constant table of crt_tables.hpp:40-61 (CrtConstants) in plain C. The
 * arbitrary-precision P is exported as 6 little-endian 32-bit limbs. */
typedef struct {
    int32_t n_moduli;
    int32_t precision;
    int32_t moduli[OZK_MAX_MODULI];
    int64_t q[OZK_MAX_MODULI];
    int32_t beta[OZK_MAX_MODULI];
    double P1, P2, P_inv;
    float pp_fast, pp_accu;
    double s1[OZK_MAX_MODULI], s2[OZK_MAX_MODULI];
    double pinv64[OZK_MAX_MODULI];
    float pinv32[OZK_MAX_MODULI];
    int32_t pinv_mulhi[OZK_MAX_MODULI];
    int32_t P_bits;
    uint32_t P_limbs[6];
} ozk_constants;

/* EmuConfig (emulator.hpp:12-18) plus the buffer types of this call.
 * constants == NULL means build_constants(n_moduli, precision)
 * (emulator.cpp:102-108); a non-NULL table is used as given (the explicit-
 * constants overloads emulator.hpp:28-32, e.g. for fault injection).
 * With precision OZK_FP32 and R64F inputs, A and B are first rounded to FP32
 * (emulator.cpp:84-91). */
typedef struct {
    int32_t n_moduli;
    int32_t mode;      /* OZK_FAST | OZK_ACCURATE */
    int32_t precision; /* OZK_FP64 | OZK_FP32 */
    int32_t a_type;    /* OZK_R64F | OZK_R32F (also B's type) */
    int32_t c_type;    /* OZK_R64F | OZK_R32F */
    int32_t flags;     /* OZK_FLAG_* (0 = the reference's behaviour) */
    int64_t block_k; /* validated in [1, 2^17] like the reference; results do not depend on it */
    const ozk_constants* constants;
} ozk_config;

typedef struct ozk_context* ozk_handle;

/* ---- lifetime ----------------------------------------------------------- */
int ozk_create(ozk_handle* handle, int device);
int ozk_destroy(ozk_handle handle);
/* cudaStream_t as void*; NULL = legacy default stream */
int ozk_set_stream(ozk_handle handle, void* stream);
const char* ozk_last_error(void);
int ozk_version(void);
/* default config for (n_moduli, mode, precision): R64F buffers, block_k 2^17 */
ozk_config ozk_default_config(int n_moduli, int mode, int precision);

/* ---- constants (crt_tables.hpp:63-79) ---------------------------------- */
int ozk_select_moduli(int n_moduli, int32_t* moduli_out);      /* select_moduli      crt_tables.cpp:15 */
int64_t ozk_mod_inverse(int64_t a, int64_t m, int* status);    /* mod_inverse        crt_tables.cpp:32 */
int ozk_build_constants(int n_moduli, int precision, ozk_constants* out); /* build_constants crt_tables.cpp:186 */
int ozk_dump_tables_csv(const ozk_constants* c, char* buf, int64_t buflen); /* dump_tables_csv crt_tables.cpp:199 */

/* ---- the GEMM (gemm_emulated, emulator.hpp:20-32) ---------------------- */
/* Device pointers; runs on the handle's stream (asynchronous). */
int ozk_gemm(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, int64_t k, double alpha, const void* A,
             int64_t lda, const void* B, int64_t ldb, double beta, void* C, int64_t ldc);
/* Host pointers (pageable or pinned): H2D, ozk_gemm, D2H, synchronous. This
 * is the reference-facing call (Matrix<T> buffers live in host memory). */
int ozk_gemm_host(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, int64_t k, double alpha,
                  const void* A, int64_t lda, const void* B, int64_t ldb, double beta, void* C, int64_t ldc);
/* BLAS-style conveniences over ozk_gemm (device pointers) */
int ozk_dgemm(ozk_handle h, int n_moduli, int mode, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
              int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc);
int ozk_sgemm(ozk_handle h, int n_moduli, int mode, int64_t m, int64_t n, int64_t k, float alpha, const float* A,
              int64_t lda, const float* B, int64_t ldb, float beta, float* C, int64_t ldc);
/* cublasDgemm-shaped: transa/transb 'N' or 'T' ('C' == 'T' for real data) */
int ozk_dgemm_ex(ozk_handle h, int n_moduli, int mode, char transa, char transb, int64_t m, int64_t n, int64_t k,
                 double alpha, const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
                 int64_t ldc);
/* Strided batch (cublasGemmStridedBatched shape): problem b uses A + b*stride_a,
 * B + b*stride_b, C + b*stride_c (elements); each equals ozk_gemm on that
 * slice. Batch entries run back to back on the handle's stream. */
int ozk_gemm_strided_batched(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, int64_t k, double alpha,
                             const void* A, int64_t lda, int64_t stride_a, const void* B, int64_t ldb,
                             int64_t stride_b, double beta, void* C, int64_t ldc, int64_t stride_c, int64_t batch);

/* Synchronise the handle's stream and collect the deferred non-finite check of
 * the OZK_FLAG_ASYNC calls since the last ozk_sync (then cleared). */
int ozk_sync(ozk_handle h);

/* ---- column-sharded GEMM (multi-GPU) --------------------------
 * This process computes C[:, shard] = alpha * A * B[:, shard] + beta * C[:, shard]
 * with the full A (the same on every process). nu is column-local in both
 * modes and fast-mode mu depends on A only; accurate-mode mu depends on the
 * row maxima of the bound product Abar*Bbar over ALL columns
 * (scaling.cpp:143-163). So:
 *   ozk_shard_begin   K1a for A's rows and this shard's columns;
 *   ozk_shard_rowmax  accurate mode: device pointer to the m int32 partial row
 *                     maxima, which the caller MAX-all-reduces across the
 *                     shards (NCCL) on the handle's stream before _end;
 *   ozk_shard_end     the budget, K1b, K2 and K3 for the shard.
 * The concatenated shards are bit-identical to the single-process result. */
int ozk_shard_begin(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, int64_t k, const void* A,
                    int64_t lda, const void* B, int64_t ldb);
int32_t* ozk_shard_rowmax(ozk_handle h);
int ozk_shard_end(ozk_handle h, double alpha, double beta, void* C, int64_t ldc);

/* Row-streamed column shard (fast mode): A arrives in row blocks — e.g. one
 * NCCL broadcast per block on another stream — and each block's work starts as
 * soon as it lands, so the broadcast of A overlaps the residue GEMMs instead of
 * preceding them. Fast-mode mu_i depends on row i of A only
 * (scaling.cpp:65-82) and nu_j on column j of B (:84-97), so the blocks are
 * bit-identical to the whole-A result.
 *   ozk_shard_stream_begin  K1a + K1b for this shard's columns of B; C, alpha,
 *                           beta fixed for the call (C = alpha A B + beta C);
 *   ozk_shard_stream_rows   rows [r0, r0+mr) of A (r0 a multiple of 16) as an
 *                           mr x k column-major block at A_rows (leading
 *                           dimension lda_rows >= mr),
 *                           ordered on the handle's stream after whatever
 *                           produced it: K1a/K1b of those rows, then K2 + K3
 *                           of C[r0:r0+mr, shard];
 *   ozk_shard_stream_end    the non-finite check; the blocks must cover [0, m).
 * OZK_CONFIG_ERROR for accurate mode (mu needs every column first), transposed
 * operands or FP64 storage with FP32 precision: those use ozk_shard_begin. */
int ozk_shard_stream_begin(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, int64_t k, const void* B,
                           int64_t ldb, double alpha, double beta, void* C, int64_t ldc);
int ozk_shard_stream_rows(ozk_handle h, int64_t r0, int64_t mr, const void* A_rows, int64_t lda_rows);
int ozk_shard_stream_end(ozk_handle h);

/* ---- stage-level exports (device pointers; parity / debug) -------------- */
/* K1a: scale exponents mu_i = 2^mu_exp[i], nu_j = 2^nu_exp[j]
 *      (scale_fast / scale_accurate, scaling.hpp:28-36). */
int ozk_stage_scale(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
                    const void* B, int64_t ldb, int32_t* mu_exp, int32_t* nu_exp);
/* column pitch (bytes) of a residue plane whose columns hold `rows` entries */
int64_t ozk_plane_ld(int64_t rows);
/* K1b: truncate_scale + to_residue_slices (residue.hpp:31-62). Planes keep
 * the reference's column-major slice layout (residue.cpp:24-42) with a
 * 16-byte-padded leading dimension: a_planes[N][k][ozk_plane_ld(m)] (read
 * MN-major by the GEMM), b_planes[N][n][ozk_plane_ld(k)] (read K-major);
 * plane i holds rmod(trunc(scaled x), p_i). */
int ozk_stage_residues(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, int64_t k, const void* A,
                       int64_t lda, const void* B, int64_t ldb, const int32_t* mu_exp, const int32_t* nu_exp,
                       int8_t* a_planes, int8_t* b_planes);
/* K2: the N residue GEMMs. out[N][n][ldo] column-major, ldo >= m:
 * OZK_PRODUCTS_I32 -> int32 C'_i, OZK_PRODUCTS_U8 -> uint8 U_i. */
int ozk_stage_products(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, int64_t k, const int8_t* a_planes,
                       const int8_t* b_planes, int kind, void* out, int64_t ldo);
/* K3: accumulate + crt_reduce + unscale (+ alpha/beta), reconstruct.hpp:46-59.
 * U[N][n][ldu] uint8 as written by ozk_stage_products(OZK_PRODUCTS_U8);
 * ldu a multiple of 8 and U 8-byte aligned. */
int ozk_stage_reconstruct(ozk_handle h, const ozk_config* cfg, int64_t m, int64_t n, const uint8_t* U, int64_t ldu,
                          const int32_t* mu_exp, const int32_t* nu_exp, double alpha, double beta, void* C,
                          int64_t ldc);

/* ---- the reference's element-wise stage helpers, on device buffers ---------
 * (used by the C++ drop-in's stage functions; all synchronous) */
/* int8_gemm (int8_engine.hpp:23-24): C = A B, int8 column-major A (m x k, lda)
 * and B (k x n, ldb) with lda, ldb multiples of 16; int32 column-major C
 * (ldc); two's-complement wrapping accumulation; k <= 2^17. */
int ozk_int8_gemm(ozk_handle h, int64_t m, int64_t n, int64_t k, const int8_t* A, int64_t lda, const int8_t* B,
                  int64_t ldb, int32_t* C, int64_t ldc);
/* int8_gemm_reference (int8_engine.hpp:27, int8_engine.cpp:66-80): the same
 * product from a plain CUDA-core triple loop (one thread per entry, uint32
 * wrapping sum in index order), independent of the tensor-core engine; any
 * lda >= m, ldb >= k; k <= 2^17. For cross-checking ozk_int8_gemm. */
int ozk_int8_gemm_reference(ozk_handle h, int64_t m, int64_t n, int64_t k, const int8_t* A, int64_t lda,
                            const int8_t* B, int64_t ldb, int32_t* C, int64_t ldc);
/* truncate_scale (residue.cpp:7-22): out = trunc(x * 2^e), e = scale_exp[i]
 * (side 0, rows) or scale_exp[j] (side 1, columns); type OZK_R64F | OZK_R32F */
int ozk_truncate_scale(ozk_handle h, int type, int64_t rows, int64_t cols, const void* x, int64_t ldx,
                       const int32_t* scale_exp, int side, void* out, int64_t ldo);
/* to_residue_slices (residue.cpp:24-42): planes[N][cols][ldp] = rmod_fast(x) */
int ozk_residues(ozk_handle h, const ozk_config* cfg, int64_t rows, int64_t cols, const void* x, int64_t ldx,
                 int8_t* planes, int64_t ldp);
/* mod_u8 over an array (reduce_products_u8, reconstruct.cpp:7-20) */
int ozk_mod_u8_array(ozk_handle h, int64_t count, const int32_t* x, int32_t p, int32_t pinv_mulhi, uint8_t* out);
/* accumulate (reconstruct.cpp:22-38): N uint8 planes of `count` entries -> C1, C2 */
int ozk_accumulate(ozk_handle h, const ozk_config* cfg, int64_t count, const uint8_t* u, double* c1, double* c2);
/* crt_reduce (reconstruct.cpp:40-47) */
int ozk_crt_reduce(ozk_handle h, const ozk_config* cfg, int64_t count, const double* c1, const double* c2,
                   double* out);
/* unscale (reconstruct.cpp:49-69): out = ldexp(cpp, -(mu_exp[i] + nu_exp[j])) */
int ozk_unscale(ozk_handle h, int64_t m, int64_t n, const double* cpp, int64_t ldc, const int32_t* mu_exp,
                const int32_t* nu_exp, double* out, int64_t ldo);

/* number of this library's kernels launched on the handle since creation */
int64_t ozk_kernel_launches(ozk_handle h);

/* ---- stage timing ---------------------------------------------------------
 * With profiling enabled, ozk_gemm brackets each stage with CUDA events on
 * the handle's stream. ozk_profile_read synchronises on them and returns the
 * accumulated milliseconds and call counts per slot (arrays of
 * OZK_PROFILE_SLOTS), optionally resetting the accumulators. */
#define OZK_PROFILE_SCALE 0       /* K1a (+ the accurate-mode bound GEMM) */
#define OZK_PROFILE_RESIDUES 1    /* K1b */
#define OZK_PROFILE_PRODUCTS 2    /* K2  */
#define OZK_PROFILE_RECONSTRUCT 3 /* K3  */
#define OZK_PROFILE_TOTAL 4       /* scale .. reconstruct */
#define OZK_PROFILE_SLOTS 5
int ozk_profile(ozk_handle h, int enable);
int ozk_profile_read(ozk_handle h, double* ms, int64_t* calls, int reset);

/* K3 diagnostics (extension; no reference counterpart). The tensor-core K3
 * (FP64 tables) takes C2 from an exact integer dot product and replays the
 * reference's sequential C2 (emulator.cpp:53) only for elements whose final
 * rounding the C2 interval cannot decide. ozk_k3_replays counts per device
 * (the handle's): the first call enables counting there; each call
 * synchronises that device and returns the elements replayed on it since
 * then (by any handle on the device), optionally resetting the count. */
int ozk_k3_replays(ozk_handle h, unsigned long long* count, int reset);

/* ---- device workspace (extension; no reference counterpart) ---------------
 * The reference needs one modulus's int32 product live at a time
 * (emulator.cpp:42-48). Here a call holds N int8 residue planes of A and of B
 * and the N uint8 product residues U of C in handle-owned device buffers,
 * reused across calls. When that workspace (about N bytes per element of A, B
 * and C) exceeds the handle's limit, ozk_gemm / ozk_gemm_host run in panels:
 * row panels of A and C times column panels of B and C, each panel's planes
 * written into the same buffers, in the loop order (and panel shape) that
 * re-derives the fewest residues. Results do not depend on the panelling
 * (every stage after the O(m + n) exponents is row/column-local).
 *   ozk_set_workspace_limit  bytes; 0 = automatic: the free device memory plus
 *                            what the handle already holds, minus
 *                            max(1 GiB, 10 % of the device) (env
 *                            OZK_WORKSPACE_GB overrides the automatic value)
 *   ozk_workspace_bytes      device bytes the handle holds now
 *   ozk_release_workspace    frees the planes, U and staging buffers (the
 *                            next call allocates what its plan needs)
 *   ozk_last_plan            the last ozk_gemm / ozk_gemm_host plan: out[0] row
 *                            panel height, out[1] column panel width, out[2]
 *                            panels, out[3] operand residue passes beyond one
 *                            per operand */
/* fast-mode exponent floor (scaling.cpp:50-52): floor(pp_fast - max(1, 0.51
 * log2 ub)) evaluated like the reference (from_table 0: std::log2 on the host)
 * or from the step table the kernels use for lines whose budget is near an
 * integer (from_table 1). Diagnostic; the two agree for every ub >= 1. */
int ozk_fast_floor(float pp_fast, double ub, int from_table);

int ozk_set_workspace_limit(ozk_handle h, int64_t bytes);
int64_t ozk_workspace_bytes(ozk_handle h);
int ozk_release_workspace(ozk_handle h);
int ozk_last_plan(ozk_handle h, int64_t out[4]);

#ifdef __cplusplus
}
#endif

#endif
