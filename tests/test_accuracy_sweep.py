"""The accuracy-sweep harness (tests/accuracy_sweep.py; SPEC.md bench_cli and
acceptance criteria 1 and 10). CPU tests cover the schema and the CLI exit
codes; GPU tests run grid points through the product path."""
import numpy as np
import pytest

import accuracy_sweep as sw


def _ref_or_skip():
    from _oracle import RefLib

    if not RefLib.available():
        pytest.skip("oracle/_ref not built")


def test_empty_grid_is_header_only():
    _ref_or_skip()
    text = sw.to_csv(sw.run_accuracy_sweep(sw.SweepSpec(sizes=[])))
    assert text == "m,n,k,phi,N,mode,precision,seed,max_rel_err,median_rel_err,wall_time\n"


def test_cli_exit_codes(tmp_path):
    _ref_or_skip()
    assert sw.main(["--sizes", "64", "--moduli", "25", "--out", str(tmp_path / "x.csv")]) == sw.EXIT_CONFIG
    assert sw.main(["--sizes", "64", "--moduli", "19", "--precision", "fp32"]) == sw.EXIT_CONFIG
    assert sw.main(["--sizes", "", "--out", str(tmp_path / "no" / "such" / "dir.csv")]) == sw.EXIT_IO
    assert sw.main(["--sizes", "", "--out", str(tmp_path / "empty.csv")]) == sw.EXIT_OK
    assert (tmp_path / "empty.csv").read_text().startswith("m,n,k,")


@pytest.mark.gpu
def test_sweep_rows_and_paper_claims():
    """SPEC bench_cli examples: accurate N=15 within 4x of the FP64 row at
    64^3, phi=0.5; at phi=4 fast mode is worse than accurate (N=14..17)."""
    _ref_or_skip()
    rows = sw.run_accuracy_sweep(sw.SweepSpec(sizes=[(64, 64, 64)], phis=[0.5], moduli_counts=[15],
                                              modes=["accurate"]))
    assert len(rows) == 2 and rows[0][4] == 0 and rows[0][5] == "fp64"
    assert rows[1][8] <= 4 * rows[0][8]
    rows = sw.run_accuracy_sweep(sw.SweepSpec(sizes=[(64, 64, 64)], phis=[4.0], moduli_counts=[14, 15, 16, 17],
                                              modes=["fast", "accurate"]))
    by = {(r[4], r[5]): r[8] for r in rows}
    for N in (14, 15, 16, 17):
        assert by[(N, "fast")] > by[(N, "accurate")]


@pytest.mark.gpu
def test_sweep_is_deterministic():
    """SPEC acceptance 10: identical CSV (all deterministic columns) across runs"""
    _ref_or_skip()
    spec = sw.SweepSpec(sizes=[(64, 64, 64), (33, 17, 90)], phis=[0.5, 2.0], moduli_counts=[10, 14],
                        modes=["fast", "accurate"], precisions=["fp64", "fp32"], seeds=[1, 2])

    def strip(text):
        return [",".join(line.split(",")[:-1]) for line in text.splitlines()]

    t1, t2 = sw.to_csv(sw.run_accuracy_sweep(spec)), sw.to_csv(sw.run_accuracy_sweep(spec))
    assert strip(t1) == strip(t2)
    assert len(t1.splitlines()) == 1 + 2 * 2 * 2 * 2 * (1 + 4)


@pytest.mark.gpu
def test_exactness_suite(oracle):
    """SPEC acceptance 1 (reduced trial count): integer inputs inside the CRT
    range come back exact, and equal the oracle restatement bit for bit."""
    _ref_or_skip()
    rep = sw.run_exactness_suite(60, seed=11, oracle=oracle)
    assert rep["trials"] == 60
    assert rep["parity_failures"] == []
    assert rep["mismatches"] == [], rep["mismatches"][:3]
