// End-to-end timing of the reference-facing C++ API (bench.py "e2e_dropin"):
// crtgemm::gemm_emulated on Matrix<double> operands (std::vector storage, i.e.
// pageable host memory) exactly as a caller of the reference
// (/root/reference/proj/include/crtgemm/emulator.hpp:23) would call it.
// Inputs follow the paper's generator (rand - 0.5) * exp(0.5 randn).
//
//   dropin_bench n moduli mode(0 fast, 1 accurate) reps   -> one JSON line
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <thread>
#include <vector>

#include "crtgemm/emulator.hpp"

using namespace crtgemm;

static void fill(Matrix<double>& m, unsigned seed) {
    // column blocks in parallel, one generator per block (any data will do)
    const unsigned nt = std::max(1u, std::thread::hardware_concurrency());
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            std::mt19937_64 g(seed * 1000003ull + t);
            std::uniform_real_distribution<double> u(0.0, 1.0);
            std::normal_distribution<double> nrm(0.0, 1.0);
            for (std::int64_t j = t; j < m.cols; j += nt)
                for (std::int64_t i = 0; i < m.rows; ++i) m(i, j) = ((1.0 - u(g)) - 0.5) * std::exp(0.5 * nrm(g));
        });
    for (auto& x : th) x.join();
}

int main(int argc, char** argv) {
    const std::int64_t n = argc > 1 ? std::atoll(argv[1]) : 16384;
    const int moduli = argc > 2 ? std::atoi(argv[2]) : 14;
    const int mode = argc > 3 ? std::atoi(argv[3]) : 0;
    const int reps = argc > 4 ? std::atoi(argv[4]) : 2;
    Matrix<double> a(n, n), b(n, n);
    fill(a, 1);
    fill(b, 2);
    EmuConfig cfg;
    cfg.n_moduli = moduli;
    cfg.mode = mode ? ScaleMode::Accurate : ScaleMode::Fast;
    cfg.precision = Precision::Fp64;
    EmulationResult r = gemm_emulated(a, b, cfg);  // warm-up: handle, tables, workspace
    double best = 1e30, sum = 0.0;
    for (int i = 0; i < reps; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        r = gemm_emulated(a, b, cfg);
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        best = std::min(best, s);
        sum += s;
    }
    const double mean = sum / reps;
    // what the API's result type alone costs: a fresh Matrix<double>(n, n)
    // (std::vector value-initialisation of 8 n^2 bytes of new pages) and its release
    double alloc = 0.0;
    for (int i = 0; i < reps; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        {
            Matrix<double> t(n, n);
            if (t.data[static_cast<std::size_t>(n) * n - 1] != 0.0) std::printf("?");
        }
        alloc += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    alloc /= reps;
    std::printf(
        "{\"value\": %.6g, \"unit\": \"TFLOPS\", \"ms_per_step\": %.6g, \"best_ms\": %.6g, "
        "\"h2d_bytes_per_step\": %lld, \"d2h_bytes_per_step\": %lld, "
        "\"path\": \"crtgemm::gemm_emulated(Matrix<double>, Matrix<double>, EmuConfig) -> EmulationResult "
        "(std::vector storage, result allocated per call)\", \"result_alloc_ms\": %.6g, \"c00\": %.17g}\n",
        2.0 * n * n * n / mean / 1e12, mean * 1e3, best * 1e3, static_cast<long long>(16 * n * n),
        static_cast<long long>(8 * n * n), alloc * 1e3, r.c(0, 0));
    return 0;
}
