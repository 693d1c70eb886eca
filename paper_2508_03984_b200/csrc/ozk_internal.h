// Internal declarations shared by the host orchestration (api.cu), the
// constant tables (constants.cpp) and the kernels (k1_*.cu, k2_gemm.cu,
// k3_reconstruct.cu). Not part of the public ABI.
#pragma once

#include <atomic>
#include <cstdint>
#include <string>

#include <cuda_runtime.h>

#include "ozaki2_b200.h"

namespace ozk {

void set_error(const std::string& msg);
const ozk_constants* cached_constants(int n, int precision);

// floor(pp_fast - max(1, 0.51 log2 ub)) of the fast exponent (scaling.cpp:50-52)
// as a step function of ub >= 1, evaluated on the host with the reference's
// own arithmetic (std::log2 = glibc): floor0 at ub = 1, one less from each
// threshold thr[i] up (ascending). Lines whose budget lies near an integer
// take their floor from here instead of from a device log2.
struct FastFloorTable {
    double thr[24];
    int n;
    int floor0;
};
FastFloorTable fast_floor_table(float pp_fast);
int fast_floor_host(float pp_fast, double ub);  // the reference's expression, on the host

// Per-call constants as a by-value kernel parameter (about 1 KB).
struct DevConsts {
    int n;
    int precision;
    int p[OZK_MAX_MODULI];
    int pinv_mulhi[OZK_MAX_MODULI];
    double pinv64[OZK_MAX_MODULI];
    float pinv32[OZK_MAX_MODULI];
    double s1[OZK_MAX_MODULI];
    double s2[OZK_MAX_MODULI];
    double P1, P2, P_inv;
    float pp_fast, pp_accu;
    double s2_m52[OZK_MAX_MODULI];
    double s1_m52[OZK_MAX_MODULI];  // -s1_i * 2^52: fl(s1*u) = fma(s1, 2^52 + u, -s1 * 2^52) (FP32 tables)
    int fast_fix;  // OZK_FLAG_FAST_EXPONENT_FIX  // -s2_i * 2^52 (for fl(s2*u) = fma(s2, 2^52 + u, -s2 * 2^52))
    uint32_t negp[OZK_MAX_MODULI];  // -p_i mod 2^32: K1b packs four residue bytes with one IMAD per modulus
    int p256_later;  // some modulus after the first is 256 (never for select_moduli tables): checked K1b loop
    FastFloorTable fast_floor;
};

DevConsts to_dev(const ozk_constants& c);

// Pinned staging of pageable host buffers for ozk_gemm_host (host_stage.cpp).
bool host_is_pageable(const void* p);
class HostStager {
  public:
    explicit HostStager(int device);
    ~HostStager();
    HostStager(const HostStager&) = delete;
    HostStager& operator=(const HostStager&) = delete;
    // start a call on these copy streams (allocates the pinned slots once)
    cudaError_t begin(cudaStream_t h2d, cudaStream_t d2h);
    // queue a pitched host -> device copy (width bytes x height columns);
    // `done` (may be null) is recorded on the H2D stream after it. Returns a
    // ticket for wait_issued.
    int64_t h2d(void* dev, size_t dpitch, const void* host, size_t hpitch, size_t width, size_t height,
                cudaEvent_t done);
    // block until the copy with this ticket is on the stream (its event recorded)
    cudaError_t wait_issued(int64_t ticket);
    // queue a pitched device -> host copy that starts after `ready`
    void d2h(void* host, size_t hpitch, const void* dev, size_t dpitch, size_t width, size_t height,
             cudaEvent_t ready);
    // wait until every queued copy has landed in host memory
    cudaError_t finish();

  private:
    struct Impl;
    Impl* impl_ = nullptr;
};

// Kernel attributes (dynamic shared memory opt-in, carveout) and launch
// geometry are per device: a process may drive several GPUs (one handle per
// device). `done` holds one bit per device ordinal; the attribute is set before
// the bit, so a racing thread at worst sets it twice.
inline int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}
inline bool needs_setup(const std::atomic<unsigned long long>& done) {
    return !(done.load(std::memory_order_acquire) & (1ull << (current_device() & 63)));
}
inline void mark_setup(std::atomic<unsigned long long>& done) {
    done.fetch_or(1ull << (current_device() & 63), std::memory_order_release);
}

// Column pitch of the int8 planes: a multiple of 16 bytes (TMA global strides
// must be 16-byte multiples). A planes use plane_ld(m), B planes plane_ld(k).
inline int64_t plane_ld(int64_t k) { return (k + 15) / 16 * 16; }
// Leading dimension of the uint8 U planes (16-byte aligned columns).
inline int64_t u_ld(int64_t m) { return (m + 15) / 16 * 16; }

// ---- K1 launchers (k1_scale.cu / k1_residue.cu) ----------------------------
// Per-line reductions (rows of A split over k into `splits` partials laid out
// [split][m]; columns of B one warp each): max |x| and sum x^2, plus the
// non-finite flag of emulator.cpp:19-22.
// The per-line exponent step fused into the reductions above (no separate
// finalize launches): fast mode writes mu/nu (lines whose budget lies within
// the guard band of an integer are recomputed in the reference's sequential
// order by one warp, element h of line l at base[l*line_step + h*elem_step]);
// accurate mode writes mu'/nu' (5 - ilogb max; INT32_MIN = zero line) and
// clears the line's bound-GEMM maximum (zero_out). Row reductions split over
// k finish in the last block of each 64-row group (counters: one int per
// group, zero between calls; the last block resets its own).
struct LineFinal {
    int mode;  // OZK_FAST / OZK_ACCURATE
    int prec, fix;
    float pp_fast;
    int64_t k;
    int32_t* exp_out;
    int32_t* zero_out;
    const void* base;
    int is_f32;
    int64_t line_step, elem_step;
    FastFloorTable fast_floor;
};
int row_stats_splits(int64_t m, int64_t k);
int64_t row_stat_groups(int64_t m);  // counters a launch_row_stats over m lines needs
void launch_row_stats(const void* a, int is_f32, int64_t m, int64_t k, int64_t lda, int splits, double* pmax,
                      double* psum, int32_t* nonfinite, int32_t* counters, const LineFinal& fin, cudaStream_t s);
void launch_col_stats(const void* b, int is_f32, int64_t k, int64_t n, int64_t ldb, double* pmax, double* psum,
                      int32_t* nonfinite, const LineFinal& fin, cudaStream_t s);
// accurate-mode budgets from the bound-GEMM maxima (scaling.cpp:151-165), rows
// and columns in one launch; k > 2^19: int64 bound product, uint64 maxima
void launch_accurate_budget(const int32_t* base, const int32_t* cmax, int64_t lines, int32_t* exp_out,
                            const int32_t* base2, const int32_t* cmax2, int64_t lines2, int32_t* exp_out2,
                            const DevConsts& c, cudaStream_t s);
void launch_accurate_budget64(const int32_t* base, const unsigned long long* cmax, int64_t lines, int32_t* exp_out,
                              const int32_t* base2, const unsigned long long* cmax2, int64_t lines2,
                              int32_t* exp_out2, const DevConsts& c, cudaStream_t s);
void launch_bound_max64(const long long* cbar, int64_t m, int64_t n, int64_t ld, unsigned long long* rowmax,
                        unsigned long long* colmax, cudaStream_t s);

// Plane writers. kind 0: residues of trunc(x * 2^exp) (N planes);
// kind 1: Abar/Bbar = ceil(|x| * 2^exp) (1 plane; exp INT32_MIN = zero line).
void launch_a_planes(const void* a, int is_f32, int64_t m, int64_t k, int64_t lda, const int32_t* row_exp,
                     const DevConsts& c, int kind, int8_t* planes, int64_t ld, int64_t plane_stride, cudaStream_t s);
void launch_b_planes(const void* b, int is_f32, int64_t k, int64_t n, int64_t ldb, const int32_t* col_exp,
                     const DevConsts& c, int kind, int8_t* planes, int64_t ld, int64_t plane_stride, cudaStream_t s);
// One-pass K1 (k1_fused.cu): statistics, exponent (LineFinal) and planes of
// kind 0 (residues) / 1 (bound plane) in a single read of the operand from HBM
// (the planes re-read each line from L2). cols: lines are the contiguous
// columns of a rows x cols operand, planes K-major (column j at j * ld).
// rows: lines are the rows, planes MN-major (column h at h * ld); `state`
// holds rows_fused_state_bytes(rows) zeroed bytes (self-resetting: all zero
// again when the launch ends, so CUDA graphs can replay it).
size_t rows_fused_state_bytes(int64_t rows);
void launch_cols_fused(const void* x, int is_f32, int64_t rows, int64_t cols, int64_t ldx, int32_t* nonfinite,
                       const LineFinal& F, const DevConsts& c, int kind, int8_t* planes, int64_t ld, int64_t stride,
                       int num_sms, cudaStream_t s);
void launch_rows_fused(const void* x, int is_f32, int64_t rows, int64_t cols, int64_t ldx,
                       void* state, int32_t* nonfinite, const LineFinal& F, const DevConsts& c, int kind,
                       int8_t* planes, int64_t ld, int64_t stride, int num_sms, cudaStream_t s);
// FP64 -> FP32 rounding of an input (emulator.cpp:84-91), column-major with ld
void launch_round_to_f32(const double* x, int64_t rows, int64_t cols, int64_t ld, float* out, int64_t ldo,
                         cudaStream_t s);

// ---- K2 (k2_gemm.cu) -------------------------------------------------------
// ACC64: int64 accumulation of the bound product over 2^17 k-chunks (accurate mode, k > 2^19)
enum K2Kind { K2_I32 = 0, K2_U8 = 1, K2_MAX = 2, K2_U8ACC = 3, K2_ACC64 = 4 };
struct K2Launch {
    // planes are column-major byte matrices with column pitch lda / ld:
    //   A MN-major (a_mn): k columns of m;  A K-major: m columns of k
    //   B K-major:          n columns of k;  B MN-major (b_mn): k columns of n
    const int8_t* a_planes;  // n_mod planes, plane stride a_stride
    const int8_t* b_planes;  // n_mod planes, plane stride b_stride
    int64_t m, n, k, ld, lda;
    bool a_mn = true, b_mn = false;
    int64_t a_stride, b_stride;  // bytes between planes
    int64_t out_stride;          // elements between output planes (I32 / U8)
    int n_mod;
    int kind;
    void* out;  // I32 / U8: [n_mod][n][ldo]; ACC64: int64 [n][ldo]
    int64_t ldo;
    bool acc_first = true;  // ACC64: this chunk initialises the sum
    int32_t* rowmax;  // MAX
    int32_t* colmax;
    const DevConsts* c;
    int num_sms;
    unsigned int* sync_counter;  // per-handle device word for the inter-cluster lockstep (nullptr: off)
};
int launch_k2(const K2Launch& L, cudaStream_t s);

// ---- K3 (k3_reconstruct.cu) -----------------------------------------------
void launch_reconstruct(const uint8_t* u, int64_t ldu, int64_t plane_stride, int64_t m, int64_t n, const int32_t* mu_exp,
                        const int32_t* nu_exp, const DevConsts& c, double alpha, double beta, void* C, int64_t ldc,
                        int c_is_f32, cudaStream_t s);

// ---- element-wise stage helpers (k_misc.cu) ---------------------------------
void launch_int8_gemm_simple(const int8_t* a, const int8_t* b, int64_t m, int64_t n, int64_t k, int64_t lda,
                             int64_t ldb, int32_t* c, int64_t ldc, cudaStream_t s);
void launch_truncate(int is_f32, const void* x, int64_t rows, int64_t cols, int64_t ldx, const int32_t* se, int side,
                     void* out, int64_t ldo, cudaStream_t s);
void launch_residues_literal(int is_f32, const void* x, int64_t rows, int64_t cols, int64_t ldx, const DevConsts& c,
                             int8_t* planes, int64_t ldp, cudaStream_t s);
void launch_mod_u8(const int32_t* x, int64_t count, int32_t p, int32_t pinv, uint8_t* out, cudaStream_t s);
void launch_accumulate(const uint8_t* u, int64_t count, const DevConsts& c, double* c1, double* c2, cudaStream_t s);
void launch_crt_reduce(const double* c1, const double* c2, int64_t count, const DevConsts& c, double* out,
                       cudaStream_t s);
void launch_unscale(const double* cpp, int64_t m, int64_t n, int64_t ldc, const int32_t* mu, const int32_t* nu,
                    double* out, int64_t ldo, cudaStream_t s);

}  // namespace ozk
