"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

The reference ships no tests or fixtures, so these vectors are
produced by oracle/_ref/libcrtgemm_ref.so — the reference sources compiled
as-is through the GMP header shim (oracle/Makefile) — and committed so the
oracle restatement and the CUDA path are pinned even where the reference
cannot be built (the GPU box has no /root/reference).

    make -C oracle ref && python tests/golden/make_golden.py

Outputs:
  constants.json     every CrtConstants table, N = 2..20 (fp64) / 2..18 (fp32),
                     floats as C99 hex strings
  tables_*.csv       dump_tables_csv for the Appendix A tables
  gemm_cases.npz     small gemm_emulated cases: inputs, mu/nu, C (bit patterns)
  stages_case.npz    one case dumped at every stage boundary
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from _oracle import RefLib  # noqa: E402

from paper_2508_03984_b200.gen import gen_int_matrix, gen_matrix  # noqa: E402

# (m, n, k, phi, N, mode, prec, block_k)
GEMM_CASES = [
    (24, 20, 40, 0.0, 14, 1, 0, 1 << 17),   # BASELINE config 1 in miniature (uniform, accurate, N=14)
    (24, 20, 40, 0.5, 14, 0, 0, 1 << 17),
    (31, 17, 65, 0.5, 12, 1, 0, 1 << 17),
    (16, 16, 300, 0.5, 16, 0, 0, 128),      # blocked k path (emulator.cpp:57-73)
    (16, 16, 300, 0.5, 16, 1, 0, 128),
    (20, 30, 50, 2.0, 17, 1, 0, 1 << 17),
    (20, 30, 50, 4.0, 20, 1, 0, 1 << 17),
    (20, 30, 50, 4.0, 20, 0, 0, 1 << 17),
    (12, 9, 33, 1.0, 2, 0, 0, 1 << 17),
    (12, 9, 33, 1.0, 5, 1, 0, 1 << 17),
    (25, 14, 45, 0.5, 8, 0, 1, 1 << 17),    # SGEMM emulation
    (25, 14, 45, 0.5, 8, 1, 1, 1 << 17),
    (25, 14, 45, 1.5, 6, 1, 1, 1 << 17),
    (25, 14, 45, 0.5, 18, 0, 1, 1 << 17),
]


def hexf(x) -> str:
    return float(x).hex()


def main():
    ref = RefLib()
    consts = {}
    for prec, maxn in ((0, 20), (1, 18)):
        for n in range(2, maxn + 1):
            c = ref.constants(n, prec)
            consts[f"{n}_{prec}"] = {
                "moduli": c["moduli"], "q": c["q"], "beta": c["beta"], "P_bits": c["P_bits"],
                "P1": hexf(c["P1"]), "P2": hexf(c["P2"]), "P_inv": hexf(c["P_inv"]),
                "pp_fast": hexf(c["pp_fast"]), "pp_accu": hexf(c["pp_accu"]),
                "s1": [hexf(x) for x in c["s1"]], "s2": [hexf(x) for x in c["s2"]],
                "pinv64": [hexf(x) for x in c["pinv64"]], "pinv32": [hexf(x) for x in c["pinv32"]],
                "pinv_mulhi": c["pinv_mulhi"],
            }
    with open(os.path.join(HERE, "constants.json"), "w") as f:
        json.dump(consts, f, indent=1, sort_keys=True)
    for n, prec in ((14, 0), (8, 1), (20, 0)):
        with open(os.path.join(HERE, f"tables_{n}_{'fp64' if prec == 0 else 'fp32'}.csv"), "w") as f:
            f.write(ref.tables_csv(n, prec))

    arrays = {}
    for idx, (m, n, k, phi, N, mode, prec, bk) in enumerate(GEMM_CASES):
        dt = np.float64 if prec == 0 else np.float32
        a = gen_matrix(m, k, phi, 100 + idx, dt)
        b = gen_matrix(k, n, phi, 200 + idx, dt)
        if idx == 1:
            a[3, :] = 0.0  # zero row sentinel
            b[:, 2] = 0.0
        mu, nu = ref.scale(a, b, N, mode, prec, bk)
        c = ref.gemm(a, b, N, mode, prec, bk)
        arrays[f"case{idx}_a"] = a
        arrays[f"case{idx}_b"] = b
        arrays[f"case{idx}_mu"] = mu
        arrays[f"case{idx}_nu"] = nu
        arrays[f"case{idx}_c"] = c
    arrays["cases"] = np.array(GEMM_CASES, dtype=np.float64)
    # exactness case (accurate mode)
    ai = gen_int_matrix(10, 10, 100, seed=9)
    arrays["int_a"] = ai
    arrays["int_c"] = ref.gemm(ai, np.asfortranarray(np.eye(10)), 15, 1)
    np.savez_compressed(os.path.join(HERE, "gemm_cases.npz"), **arrays)

    # stage dump: accurate, N = 14, phi = 1
    m, n, k, N = 18, 13, 70, 14
    a = gen_matrix(m, k, 1.0, 301)
    b = gen_matrix(k, n, 1.0, 302)
    mu, nu = ref.scale(a, b, N, 1)
    ta, pa = ref.residues(a, mu, 0, N)
    tb, pb = ref.residues(b, nu, 1, N)
    prods = np.stack([ref.int8_gemm(pa[i], pb[i]) for i in range(N)])
    np.savez_compressed(os.path.join(HERE, "stages_case.npz"), a=a, b=b, mu=mu, nu=nu, trunc_a=ta, trunc_b=tb,
                        planes_a=pa, planes_b=pb, products=prods, c=ref.gemm(a, b, N, 1))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
