// K3, register-staged variant — CRT reconstruction (reference: emulator.cpp:49-53 weighted sum,
// reconstruct.hpp:51-54 crt_reduce_element, reconstruct.cpp:49-69 unscale).
//
// One pass over the N uint8 residue planes U_i (column-major, ld = ldu) per
// output element, in the reference's per-element order:
//   c1 += s1_i * u  (exact by the beta_i construction, crt_tables.cpp:165-169)
//   c2 += s2_i * u  (mul then add: two roundings, as in emulator.cpp:53)
//   Q  = rint(P_inv * c1);  C'' = fma(-P2, Q, fma(-P1, Q, c1) + c2)
//   C  = ldexp(C'', -(e_mu_i + e_nu_j))
// then the optional alpha/beta extension in FP64 and the FP32 down-cast of
// to_fp32 (emulator.cpp:110-115) when C is single precision. Each thread owns
// eight consecutive rows: one 64-bit load per plane, 64 B of C out, so a warp
// moves 256 B per plane and 2 KB of C — HBM-bound at N + 8 bytes per element.
#include <cstdlib>

#include "ozk_device.cuh"

namespace ozk {
namespace regs {
namespace {

// Rows per thread R: one R-byte load per plane, 8R bytes of C out. The plane
// words of all N moduli are loaded up front, so registers grow with R x kMaxMod:
// both are template parameters (kMaxMod = the modulus count rounded up to a
// bucket) to keep occupancy up.
template <int R>
struct PlaneWord;
template <>
struct PlaneWord<8> {
    using T = uint2;
    static __device__ __forceinline__ uint32_t part(const uint2& w, int q) { return q < 4 ? w.x : w.y; }
};
template <>
struct PlaneWord<4> {
    using T = uint32_t;
    static __device__ __forceinline__ uint32_t part(const uint32_t& w, int) { return w; }
};

// ldexp(x, e) as one multiply by 2^e when that is exact-and-correctly-rounded
// (2^e normal, result normal); CUDA's general ldexp otherwise (subnormal or
// overflowing results, huge |e|)
__device__ __forceinline__ double scale_pow2(double x, int e) {
    if (e >= -1022 && e <= 1023) {
        const double r = __dmul_rn(x, pow2d(e));
        if (fabs(r) >= 0x1.0p-1022 && fabs(r) <= 0x1.fffffffffffffp+1023) return r;
        if (r == 0.0 && x == 0.0) return r;
    }
    return ldexp(x, e);
}

// 32-byte vector accesses (sm_100: LDG/STG .256)
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

template <bool kF32Out, bool kPlain, bool kFp64Tables, int kRows, int kMaxMod>
__global__ void __launch_bounds__(128)
    reconstruct_kernel(const uint8_t* __restrict__ u, int64_t ldu, int64_t plane_stride, int64_t m, int64_t n,
                       const int32_t* __restrict__ mu_exp, const int32_t* __restrict__ nu_exp, const DevConsts c,
                       double alpha, double beta, void* __restrict__ C, int64_t ldc, bool vec_ok) {
    const int64_t j = blockIdx.x;
    const int64_t i0 = (static_cast<int64_t>(blockIdx.y) * blockDim.x + threadIdx.x) * kRows;
    if (i0 >= m) return;
    double c1[kRows], c2[kRows];
#pragma unroll
    for (int q = 0; q < kRows; ++q) c1[q] = c2[q] = 0.0;
    const uint8_t* src = u + j * ldu + i0;
    const int n_mod = c.n;
    // all plane loads first (predicated, compile-time indices: registers), so
    // a thread has its N loads in flight at once instead of one per FP chain step
    using W = PlaneWord<kRows>;
    typename W::T w[kMaxMod];
#pragma unroll
    for (int t = 0; t < kMaxMod; ++t)
        w[t] = t < n_mod ? __ldg(reinterpret_cast<const typename W::T*>(src + t * plane_stride)) : typename W::T{};
#pragma unroll
    for (int t = 0; t < kMaxMod; ++t) {  // compile-time bound: constants become immediates
        if (t < n_mod) {
#pragma unroll
            for (int q = 0; q < kRows; ++q) {
                const uint32_t word = W::part(w[t], q);
                const uint32_t ub = __byte_perm(word, 0u, 0x4440u | (q & 3));  // byte q, zero-extended
                // V = 2^52 + u exactly (no conversion instruction); v = u
                const double V = __hiloint2double(0x43300000, static_cast<int>(ub));
                const double v = __dsub_rn(V, 0x1.0p52);
                // FP64 tables: s1*u is exact and so is the running sum (beta_i
                // construction), so the fused form equals the reference's
                // mul-then-add bit for bit. FP32 tables carry the full-width s1
                // (crt_tables.cpp:160-163): keep the two roundings there.
                c1[q] = kFp64Tables ? __fma_rn(c.s1[t], v, c1[q]) : __dadd_rn(c1[q], __dmul_rn(c.s1[t], v));
                // fl(s2 u) = fma(s2, 2^52 + u, -s2 2^52): the reference's rounded
                // product (emulator.cpp:53), then its rounded sum
                c2[q] = __dadd_rn(c2[q], __fma_rn(c.s2[t], V, c.s2_m52[t]));
            }
        }
    }
    const int ne = nu_exp[j];
    // full 8-row groups with aligned mu / C use 32-byte vector accesses: a
    // warp's C stores then cover whole sectors instead of 8-byte pieces at a
    // 64-byte lane stride
    const bool vec = kRows == 8 && vec_ok && i0 + kRows <= m;
    int me[kRows];
    if (vec) {
        ld_nc_v8(mu_exp + i0, me);
    } else {
#pragma unroll
        for (int q = 0; q < kRows; ++q) me[q] = i0 + q < m ? mu_exp[i0 + q] : 0;
    }
    double r[kRows];
#pragma unroll
    for (int q = 0; q < kRows; ++q) {
        const double qv = rint(__dmul_rn(c.P_inv, c1[q]));
        const double cpp = __fma_rn(-c.P2, qv, __dadd_rn(__fma_rn(-c.P1, qv, c1[q]), c2[q]));
        r[q] = scale_pow2(cpp, -(me[q] + ne));
    }
    if (!kPlain) {
#pragma unroll
        for (int q = 0; q < kRows; ++q) {
            const int64_t i = i0 + q;
            const double old = (beta != 0.0 && i < m)
                                   ? (kF32Out ? static_cast<double>(static_cast<float*>(C)[i + j * ldc])
                                              : static_cast<double*>(C)[i + j * ldc])
                                   : 0.0;
            r[q] = __dadd_rn(__dmul_rn(alpha, r[q]), __dmul_rn(beta, old));
        }
    }
    if (vec) {
        if constexpr (kF32Out) {
            float f[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) f[q] = __double2float_rn(r[q]);
            st_v8_f32(static_cast<float*>(C) + i0 + j * ldc, f);
        } else {
            st_v4_f64(static_cast<double*>(C) + i0 + j * ldc, r);
            st_v4_f64(static_cast<double*>(C) + i0 + 4 + j * ldc, r + 4);
        }
        return;
    }
#pragma unroll
    for (int q = 0; q < kRows; ++q) {
        const int64_t i = i0 + q;
        if (i >= m) break;
        if (kF32Out)
            static_cast<float*>(C)[i + j * ldc] = __double2float_rn(r[q]);
        else
            static_cast<double*>(C)[i + j * ldc] = r[q];
    }
}

int k3_rows() {
    static const int r = [] {
        const char* e = std::getenv("OZK_K3_ROWS");
        return e && std::atoi(e) == 4 ? 4 : 8;
    }();
    return r;
}

template <bool kF32Out, bool kPlain, bool kFp64, int kRows>
void launch_rows(int n_mod, dim3 grid, cudaStream_t s, const uint8_t* u, int64_t ldu, int64_t stride, int64_t m,
                 int64_t n, const int32_t* mu_exp, const int32_t* nu_exp, const DevConsts& c, double alpha,
                 double beta, void* C, int64_t ldc) {
    // vector path: 32-byte aligned mu and C columns
    const int esz = kF32Out ? 4 : 8;
    const bool vec_ok = (reinterpret_cast<uintptr_t>(mu_exp) % 32 == 0) &&
                        (reinterpret_cast<uintptr_t>(C) % 32 == 0) && ((ldc * esz) % 32 == 0);
#define OZK_K3(MAXN)                                                                                       \
    reconstruct_kernel<kF32Out, kPlain, kFp64, kRows, MAXN>                                                \
        <<<grid, 128, 0, s>>>(u, ldu, stride, m, n, mu_exp, nu_exp, c, alpha, beta, C, ldc, vec_ok)
    if (n_mod <= 8)
        OZK_K3(8);
    else if (n_mod <= 12)
        OZK_K3(12);
    else if (n_mod <= 14)
        OZK_K3(14);
    else if (n_mod <= 16)
        OZK_K3(16);
    else
        OZK_K3(OZK_MAX_MODULI);
#undef OZK_K3
}

template <bool kF32Out, bool kPlain>
void launch_variant(const uint8_t* u, int64_t ldu, int64_t stride, int64_t m, int64_t n, const int32_t* mu_exp,
                    const int32_t* nu_exp, const DevConsts& c, double alpha, double beta, void* C, int64_t ldc,
                    cudaStream_t s) {
    // with more than 16 planes the 8-row variant's prefetched words no longer stay
    // in registers (ptxas sinks the loads into the FP64 chain): 4 rows there
    const int rows = c.n > 16 ? 4 : k3_rows();
    dim3 grid(static_cast<unsigned>(n), static_cast<unsigned>((m + 128 * rows - 1) / (128 * rows)));
    const bool fp64 = c.precision == OZK_FP64;
    if (rows == 8) {
        if (fp64)
            launch_rows<kF32Out, kPlain, true, 8>(c.n, grid, s, u, ldu, stride, m, n, mu_exp, nu_exp, c, alpha, beta,
                                                   C, ldc);
        else
            launch_rows<kF32Out, kPlain, false, 8>(c.n, grid, s, u, ldu, stride, m, n, mu_exp, nu_exp, c, alpha,
                                                    beta, C, ldc);
    } else {
        if (fp64)
            launch_rows<kF32Out, kPlain, true, 4>(c.n, grid, s, u, ldu, stride, m, n, mu_exp, nu_exp, c, alpha, beta,
                                                   C, ldc);
        else
            launch_rows<kF32Out, kPlain, false, 4>(c.n, grid, s, u, ldu, stride, m, n, mu_exp, nu_exp, c, alpha,
                                                    beta, C, ldc);
    }
}

}  // namespace

void launch_reconstruct_regs_impl(const uint8_t* u, int64_t ldu, int64_t stride, int64_t m, int64_t n, const int32_t* mu_exp,
                        const int32_t* nu_exp, const DevConsts& c, double alpha, double beta, void* C, int64_t ldc,
                        int c_is_f32, cudaStream_t s) {
    const bool plain = alpha == 1.0 && beta == 0.0;
    if (c_is_f32) {
        if (plain)
            launch_variant<true, true>(u, ldu, stride, m, n, mu_exp, nu_exp, c, alpha, beta, C, ldc, s);
        else
            launch_variant<true, false>(u, ldu, stride, m, n, mu_exp, nu_exp, c, alpha, beta, C, ldc, s);
    } else {
        if (plain)
            launch_variant<false, true>(u, ldu, stride, m, n, mu_exp, nu_exp, c, alpha, beta, C, ldc, s);
        else
            launch_variant<false, false>(u, ldu, stride, m, n, mu_exp, nu_exp, c, alpha, beta, C, ldc, s);
    }
}

}  // namespace regs
}  // namespace ozk

namespace ozk {
// the fallback behind launch_reconstruct (k3_reconstruct.cu) for U layouts the
// bulk copies cannot take (unaligned base, ldu or plane stride)
void launch_reconstruct_regs(const uint8_t* u, int64_t ldu, int64_t stride, int64_t m, int64_t n,
                             const int32_t* mu_exp, const int32_t* nu_exp, const DevConsts& c, double alpha,
                             double beta, void* C, int64_t ldc, int c_is_f32, cudaStream_t s) {
    regs::launch_reconstruct_regs_impl(u, ldu, stride, m, n, mu_exp, nu_exp, c, alpha, beta, C, ldc, c_is_f32, s);
}
}  // namespace ozk
