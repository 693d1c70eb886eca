// K3 — CRT reconstruction (reference: emulator.cpp:49-53 weighted sum,
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
#include "ozk_device.cuh"

namespace ozk {
namespace {

constexpr int kRows = 8;  // rows per thread: one 8-byte load per plane, 64 B of C out

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

template <bool kF32Out, bool kPlain, bool kFp64Tables>
__global__ void __launch_bounds__(128)
    reconstruct_kernel(const uint8_t* __restrict__ u, int64_t ldu, int64_t plane_stride, int64_t m, int64_t n,
                       const int32_t* __restrict__ mu_exp, const int32_t* __restrict__ nu_exp, const DevConsts c,
                       double alpha, double beta, void* __restrict__ C, int64_t ldc) {
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
    uint2 w[OZK_MAX_MODULI];
#pragma unroll
    for (int t = 0; t < OZK_MAX_MODULI; ++t)
        w[t] = t < n_mod ? __ldg(reinterpret_cast<const uint2*>(src + t * plane_stride)) : make_uint2(0u, 0u);
#pragma unroll
    for (int t = 0; t < OZK_MAX_MODULI; ++t) {  // compile-time bound: constants become immediates
        if (t < n_mod) {
#pragma unroll
            for (int q = 0; q < kRows; ++q) {
                const uint32_t word = q < 4 ? w[t].x : w[t].y;
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
#pragma unroll
    for (int q = 0; q < kRows; ++q) {
        const int64_t i = i0 + q;
        if (i >= m) break;
        const double qv = rint(__dmul_rn(c.P_inv, c1[q]));
        const double cpp = __fma_rn(-c.P2, qv, __dadd_rn(__fma_rn(-c.P1, qv, c1[q]), c2[q]));
        double r = scale_pow2(cpp, -(mu_exp[i] + ne));
        if (!kPlain) {
            const double old = beta != 0.0 ? (kF32Out ? static_cast<double>(static_cast<float*>(C)[i + j * ldc])
                                                      : static_cast<double*>(C)[i + j * ldc])
                                           : 0.0;
            r = __dadd_rn(__dmul_rn(alpha, r), __dmul_rn(beta, old));
        }
        if (kF32Out)
            static_cast<float*>(C)[i + j * ldc] = __double2float_rn(r);
        else
            static_cast<double*>(C)[i + j * ldc] = r;
    }
}

template <bool kF32Out, bool kPlain>
void launch_variant(dim3 grid, cudaStream_t s, const uint8_t* u, int64_t ldu, int64_t stride, int64_t m, int64_t n,
                    const int32_t* mu_exp, const int32_t* nu_exp, const DevConsts& c, double alpha, double beta,
                    void* C, int64_t ldc) {
    if (c.precision == OZK_FP64)
        reconstruct_kernel<kF32Out, kPlain, true>
            <<<grid, 128, 0, s>>>(u, ldu, stride, m, n, mu_exp, nu_exp, c, alpha, beta, C, ldc);
    else
        reconstruct_kernel<kF32Out, kPlain, false>
            <<<grid, 128, 0, s>>>(u, ldu, stride, m, n, mu_exp, nu_exp, c, alpha, beta, C, ldc);
}

}  // namespace

void launch_reconstruct(const uint8_t* u, int64_t ldu, int64_t stride, int64_t m, int64_t n, const int32_t* mu_exp,
                        const int32_t* nu_exp, const DevConsts& c, double alpha, double beta, void* C, int64_t ldc,
                        int c_is_f32, cudaStream_t s) {
    dim3 grid(static_cast<unsigned>(n), static_cast<unsigned>((m + 128 * kRows - 1) / (128 * kRows)));
    const bool plain = alpha == 1.0 && beta == 0.0;
    if (c_is_f32) {
        if (plain)
            launch_variant<true, true>(grid, s, u, ldu, stride, m, n, mu_exp, nu_exp, c, alpha, beta, C, ldc);
        else
            launch_variant<true, false>(grid, s, u, ldu, stride, m, n, mu_exp, nu_exp, c, alpha, beta, C, ldc);
    } else {
        if (plain)
            launch_variant<false, true>(grid, s, u, ldu, stride, m, n, mu_exp, nu_exp, c, alpha, beta, C, ldc);
        else
            launch_variant<false, false>(grid, s, u, ldu, stride, m, n, mu_exp, nu_exp, c, alpha, beta, C, ldc);
    }
}

}  // namespace ozk
