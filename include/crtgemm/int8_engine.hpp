// Drop-in for int8_engine.hpp:10-34: the INT8 engine is the B200 tensor core
// (tcgen05.mma kind::i8) instead of a CPU loop; same wrapping int32 contract.
#pragma once

#include <cstdint>
#include <vector>

#include "crtgemm/matrix.hpp"

namespace crtgemm {

inline constexpr std::int64_t kEngineMaxK = std::int64_t(1) << 17;

struct Int32ProductMatrix {
    Matrix<std::int32_t> data;
    std::int64_t k_used = 0;
};

// n_threads is accepted for signature compatibility and ignored (GPU engine).
Int32ProductMatrix int8_gemm(const Matrix<std::int8_t>& a, const Matrix<std::int8_t>& b, int n_threads = 1);
Int32ProductMatrix int8_gemm_reference(const Matrix<std::int8_t>& a, const Matrix<std::int8_t>& b);
std::vector<Int32ProductMatrix> blocked_int8_gemm(const Matrix<std::int8_t>& a, const Matrix<std::int8_t>& b,
                                                  std::int64_t block_k, int n_threads = 1);

}  // namespace crtgemm
