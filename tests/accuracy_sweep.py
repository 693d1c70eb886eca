"""Accuracy-sweep harness (SPEC.md bench_cli
run_accuracy_sweep / run_exactness_suite). TEST INFRASTRUCTURE: the emulated
GEMMs run on the GPU through the product API (gemm_emulated -> ozk_gemm_host);
the errors are measured against the reference's exact GMP oracle
(oracle.cpp:39-157 via oracle/_ref, ``RefLib.exact_compare``).

CSV schema (fixed order, golden-tested in tests/test_accuracy_sweep.py):

    m,n,k,phi,N,mode,precision,seed,max_rel_err,median_rel_err,wall_time

one row per grid point, in grid order (sizes, phis, precisions, seeds, then
the plain-matmul baseline rows with N = 0 and mode "fp64"/"fp32", then the
moduli x modes). wall_time is the emulation's host-visible seconds (or the
baseline matmul's); every other column is deterministic.

    python tests/accuracy_sweep.py --sizes 64,128 --phi 0.5,4 --moduli 12,14,16 \
        --mode fast,accurate --precision fp64 --seeds 1,2 --out sweep.csv
    python tests/accuracy_sweep.py --trials 100 --seed 7      # exactness suite
"""
from __future__ import annotations

import argparse
import csv
import io
import os
import sys
import time
from dataclasses import dataclass, field

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

HEADER = ["m", "n", "k", "phi", "N", "mode", "precision", "seed", "max_rel_err", "median_rel_err", "wall_time"]
EXIT_OK, EXIT_CONFIG, EXIT_IO, EXIT_SUITE = 0, 2, 3, 4


@dataclass
class SweepSpec:
    """SPEC.md SweepSpec: the experiment grid of §5.1"""
    sizes: list = field(default_factory=lambda: [(64, 64, 64)])
    phis: list = field(default_factory=lambda: [0.5])
    moduli_counts: list = field(default_factory=lambda: [14])
    modes: list = field(default_factory=lambda: ["accurate"])
    precisions: list = field(default_factory=lambda: ["fp64"])
    seeds: list = field(default_factory=lambda: [1])
    block_k: int = 1 << 17
    fast_exponent_fix: bool = False

    def validate(self):
        from paper_2508_03984_b200 import ConfigError

        for N in self.moduli_counts:
            for p in self.precisions:
                hi = 20 if p == "fp64" else 18
                if not 2 <= N <= hi:
                    raise ConfigError(f"N = {N} outside [2, {hi}] for {p}")
        for s in self.sizes:
            if min(s) < 1:
                raise ConfigError(f"non-positive size {s}")
        for md in self.modes:
            if md not in ("fast", "accurate"):
                raise ConfigError(f"unknown mode {md}")
        for p in self.precisions:
            if p not in ("fp64", "fp32"):
                raise ConfigError(f"unknown precision {p}")


def _inputs(m, n, k, phi, seed, prec):
    from paper_2508_03984_b200 import gen_matrix

    a = gen_matrix(m, k, phi, 2 * seed)
    b = gen_matrix(k, n, phi, 2 * seed + 1)
    if prec == "fp32":
        a, b = a.astype(np.float32), b.astype(np.float32)
    return a, b


def run_accuracy_sweep(spec: SweepSpec, ref=None) -> list:
    """one row (list, HEADER order) per grid point"""
    from _oracle import RefLib

    from paper_2508_03984_b200 import EmuConfig, Precision, ScaleMode, gemm_emulated

    spec.validate()
    ref = ref or RefLib()
    rows = []
    for (m, n, k) in spec.sizes:
        for phi in spec.phis:
            for prec in spec.precisions:
                pc = 0 if prec == "fp64" else 1
                for seed in spec.seeds:
                    a, b = _inputs(m, n, k, phi, seed, prec)
                    t0 = time.perf_counter()
                    plain = ref.plain_gemm(a, b, pc).astype(np.float64)
                    t = time.perf_counter() - t0
                    rep = ref.exact_compare(a, b, plain, pc)
                    rows.append([m, n, k, phi, 0, prec, prec, seed, rep["max_rel_err"], rep["median_rel_err"], t])
                    for N in spec.moduli_counts:
                        for md in spec.modes:
                            cfg = EmuConfig(n_moduli=N, mode=ScaleMode.Fast if md == "fast" else ScaleMode.Accurate,
                                            precision=Precision.Fp64 if pc == 0 else Precision.Fp32,
                                            block_k=spec.block_k, fast_exponent_fix=spec.fast_exponent_fix)
                            t0 = time.perf_counter()
                            c = gemm_emulated(a, b, cfg).c
                            t = time.perf_counter() - t0
                            rep = ref.exact_compare(a, b, c, pc)
                            rows.append([m, n, k, phi, N, md, prec, seed, rep["max_rel_err"],
                                         rep["median_rel_err"], t])
    return rows


def to_csv(rows) -> str:
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(HEADER)
    for r in rows:
        w.writerow([f"{x:.6e}" if isinstance(x, float) and i >= 8 else (repr(x) if isinstance(x, float) else x)
                    for i, x in enumerate(r)])
    return buf.getvalue()


def run_exactness_suite(trials: int, seed: int, ref=None, moduli=(2, 5, 10, 15, 20), max_dim=128,
                        oracle=None) -> dict:
    """SPEC acceptance 1: random integer matrices sized so that 2 sum|a||b| < P,
    full GPU pipeline vs the exact oracle. Reports every mismatch with a
    reproducer (dims, seed, N). With ``oracle`` given, also requires the GPU
    result to equal the oracle restatement bit for bit (parity)."""
    from _oracle import RefLib

    from paper_2508_03984_b200 import EmuConfig, ScaleMode, build_constants, gemm_emulated

    ref = ref or RefLib()
    rng = np.random.default_rng(seed)
    out = {"trials": 0, "exact": 0, "mismatches": [], "parity_failures": []}
    for t in range(trials):
        N = int(moduli[t % len(moduli)])
        m, n, k = (int(x) for x in rng.integers(1, max_dim + 1, 3))
        # accurate mode keeps integer inputs exact when mu = 2^(5 - g + e) >= 1 with
        # e >= floor(pp_accu - 0.51 log2(64 * 64 * k)) (scaling.cpp:151-160); the
        # scheme itself then guarantees 2 sum|a'||b'| < P
        e = int(np.floor(build_constants(N).pp_accu - 0.51 * np.log2(4096.0 * k)))
        bound = int(min(2 ** 20, max(1, 2 ** (6 + e) - 1)))
        ts = int(rng.integers(0, 2 ** 31))
        r2 = np.random.default_rng(ts)
        a = np.asfortranarray(r2.integers(-bound, bound + 1, (m, k)).astype(np.float64))
        b = np.asfortranarray(r2.integers(-bound, bound + 1, (k, n)).astype(np.float64))
        mode = ScaleMode.Accurate
        c = gemm_emulated(a, b, EmuConfig(n_moduli=N, mode=mode)).c
        rep = ref.exact_compare(a, b, c, 0)
        out["trials"] += 1
        repro = {"m": m, "n": n, "k": k, "N": N, "mode": mode.name, "bound": bound, "seed": ts}
        if rep["exact_match"]:
            out["exact"] += 1
        else:
            out["mismatches"].append({**repro, "max_rel_err": rep["max_rel_err"]})
        if oracle is not None:
            want = oracle.gemm(a, b, N, int(mode))
            if not np.array_equal(c.view(np.int64), want.view(np.int64)):
                out["parity_failures"].append(repro)
    return out


def _parse_list(s, conv):
    return [conv(x) for x in s.split(",") if x.strip()] if s else []


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--sizes", default="64,128,256,512", help="m=n=k list, or mxnxk entries")
    ap.add_argument("--phi", default="0.5,1,2,4")
    ap.add_argument("--moduli", default="8,10,12,14,16,18,20")
    ap.add_argument("--mode", default="fast,accurate")
    ap.add_argument("--precision", default="fp64")
    ap.add_argument("--seeds", default="1")
    ap.add_argument("--block-k", type=int, default=1 << 17)
    ap.add_argument("--fast-exponent-fix", action="store_true")
    ap.add_argument("--out", default="-")
    ap.add_argument("--trials", type=int, default=None, help="run the exactness suite instead")
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args(argv)
    from paper_2508_03984_b200 import ConfigError

    if args.trials is not None:
        rep = run_exactness_suite(args.trials, args.seed)
        print(f"exactness: {rep['exact']}/{rep['trials']} exact")
        for mm in rep["mismatches"]:
            print("mismatch:", mm)
        return EXIT_OK if not rep["mismatches"] else EXIT_SUITE

    def size(s):
        parts = [int(x) for x in s.split("x")]
        return tuple(parts * 3) if len(parts) == 1 else tuple(parts)

    spec = SweepSpec(sizes=_parse_list(args.sizes, size), phis=_parse_list(args.phi, float),
                     moduli_counts=_parse_list(args.moduli, int), modes=_parse_list(args.mode, str),
                     precisions=_parse_list(args.precision, str), seeds=_parse_list(args.seeds, int),
                     block_k=args.block_k, fast_exponent_fix=args.fast_exponent_fix)
    try:
        text = to_csv(run_accuracy_sweep(spec))
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return EXIT_CONFIG
    if args.out == "-":
        sys.stdout.write(text)
        return EXIT_OK
    try:
        with open(args.out, "w") as f:
            f.write(text)
    except OSError as e:
        print(f"cannot write {args.out}: {e}", file=sys.stderr)
        return EXIT_IO
    return EXIT_OK


if __name__ == "__main__":
    sys.exit(main())
