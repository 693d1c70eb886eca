// Drop-in check: a caller written against the reference's C++ API
// (crtgemm/emulator.hpp, /root/reference/proj/include/crtgemm/emulator.hpp:20-35)
// compiled against this repo's include/ and linked to libozaki2_b200.so.
//
//   dropin_test <dir> : reads dir/{a,b}.bin (m, k, n header + column-major FP64),
//   runs gemm_emulated for each mode line in dir/cases.txt ("N mode prec"),
//   writes dir/c_<i>.bin, and exercises the reference's error contract.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <limits>
#include <stdexcept>
#include <string>

#include "crtgemm/emulator.hpp"
#include "crtgemm/errors.hpp"
#include "crtgemm/int8_engine.hpp"
#include "crtgemm/reconstruct.hpp"
#include "crtgemm/residue.hpp"
#include "crtgemm/scaling.hpp"

using namespace crtgemm;

static Matrix<double> read_matrix(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    std::int64_t rc[2];
    f.read(reinterpret_cast<char*>(rc), sizeof rc);
    Matrix<double> m(rc[0], rc[1]);
    f.read(reinterpret_cast<char*>(m.data.data()), static_cast<std::streamsize>(sizeof(double) * m.data.size()));
    return m;
}

static void write_matrix(const std::string& path, const Matrix<double>& m) {
    std::ofstream f(path, std::ios::binary);
    const std::int64_t rc[2] = {m.rows, m.cols};
    f.write(reinterpret_cast<const char*>(rc), sizeof rc);
    f.write(reinterpret_cast<const char*>(m.data.data()), static_cast<std::streamsize>(sizeof(double) * m.data.size()));
}

template <typename E, typename F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const std::string dir = argv[1];
    const Matrix<double> a = read_matrix(dir + "/a.bin"), b = read_matrix(dir + "/b.bin");
    std::ifstream cases(dir + "/cases.txt");
    int n_mod, mode, prec, idx = 0;
    while (cases >> n_mod >> mode >> prec) {
        EmuConfig cfg;
        cfg.n_moduli = n_mod;
        cfg.mode = mode ? ScaleMode::Accurate : ScaleMode::Fast;
        cfg.precision = prec ? Precision::Fp32 : Precision::Fp64;
        const EmulationResult r = gemm_emulated(a, b, cfg);
        if (r.n_moduli != n_mod || r.c.rows != a.rows || r.c.cols != b.cols) return 3;
        write_matrix(dir + "/c_" + std::to_string(idx++) + ".bin", r.c);
    }
    // error contract (errors.hpp / emulator.cpp:12-23, crt_tables.cpp:186-189)
    EmuConfig bad;
    bad.n_moduli = 21;
    if (!throws<ConfigError>([&] { gemm_emulated(a, b, bad); })) return 4;
    EmuConfig ok;
    ok.n_moduli = 8;
    Matrix<double> nan_a = a;
    nan_a.data[0] = std::numeric_limits<double>::quiet_NaN();
    if (!throws<InputError>([&] { gemm_emulated(nan_a, b, ok); })) return 5;
    if (!throws<InputError>([&] { gemm_emulated(a, Matrix<double>(a.cols + 1, 3), ok); })) return 6;
    ok.threads = 0;
    if (!throws<ConfigError>([&] { gemm_emulated(a, b, ok); })) return 7;
    // tables and helpers
    const CrtConstants& c14 = build_constants(14, Precision::Fp64);
    std::ofstream(dir + "/tables_14.csv") << dump_tables_csv(c14);
    if (select_moduli(5).moduli[4] != 247 || mod_inverse(3, 10) != 7) return 8;
    if (mod_u8(-1, 255, c14.pinv_mulhi[1]) != 254) return 9;
    const Matrix<float> f = to_fp32(read_matrix(dir + "/a.bin"));
    if (f.rows != a.rows) return 10;
    // the stage-level API composes to exactly gemm_emulated (emulator.cpp:25-78)
    for (int accurate = 0; accurate < 2; ++accurate) {
        const CrtConstants& c = build_constants(14, Precision::Fp64);
        const ScalePair s = accurate ? scale_accurate(a, b, c) : scale_fast(a, b, c);
        const Matrix<double> ap = truncate_scale(a, s.mu, Side::Row), bp = truncate_scale(b, s.nu, Side::Col);
        const ResidueSlices sa = to_residue_slices(ap, c), sb = to_residue_slices(bp, c);
        std::vector<Int32ProductMatrix> prods;
        for (int i = 0; i < c.n(); ++i) {
            prods.push_back(int8_gemm(sa.slices[static_cast<size_t>(i)], sb.slices[static_cast<size_t>(i)]));
            const auto ref = int8_gemm_reference(sa.slices[static_cast<size_t>(i)], sb.slices[static_cast<size_t>(i)]);
            if (!(ref.data == prods.back().data)) return 11;
        }
        const auto blocks = blocked_int8_gemm(sa.slices[1], sb.slices[1], 32);
        Matrix<std::int32_t> sum(a.rows, b.cols);
        for (const auto& blk : blocks)
            for (size_t e = 0; e < sum.data.size(); ++e) sum.data[e] += blk.data.data[e];
        if (!(sum == prods[1].data)) return 12;
        const ResidueProducts u = reduce_products_u8(prods, c);
        const auto c12 = accumulate(u, c);
        const EmulationResult r = unscale(crt_reduce(c12.first, c12.second, c), s, c);
        EmuConfig cfg;
        cfg.n_moduli = 14;
        cfg.mode = accurate ? ScaleMode::Accurate : ScaleMode::Fast;
        const EmulationResult direct = gemm_emulated(a, b, cfg);
        if (!(r.c == direct.c)) return 13;
        write_matrix(dir + "/stages_" + std::to_string(accurate) + ".bin", r.c);
    }
    std::printf("dropin ok: %d cases\n", idx);
    return 0;
}
