"""The bench CSV contract (bench.hpp:184-199 run_benchmark, 221-252 emit_csv)
of scripts/bench_csv.py: CPU rows from the reference itself (oracle/_ref),
checked here without a GPU; the GPU rows of the same grid under -m gpu."""
import csv
import io
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import bench_csv  # noqa: E402


def _check_contract(text, sizes, procs, algos, impls):
    lines = text.splitlines()
    assert lines[0] == "algorithm,n,p,mean_seconds,speedup,predicted_speedup,verified,impl"
    rows = list(csv.DictReader(io.StringIO(text)))
    pos = 0
    for n in sizes:
        # SR4 baseline rows (p = 1) first for every n, one per impl
        for impl in impls:
            r = rows[pos]
            assert (r["algorithm"], int(r["n"]), int(r["p"]), r["impl"]) == ("sr4", n, 1, impl)
            pos += 1
        if "cpu" in impls:
            assert rows[pos - len(impls)]["speedup"] == "1.0"
        for algo in algos:
            for p in procs:
                if algo == "btn" and p & (p - 1):
                    continue  # bench.hpp:150-154
                for impl in impls:
                    r = rows[pos]
                    assert (r["algorithm"], int(r["n"]), int(r["p"]), r["impl"]) == (algo, n, p, impl)
                    pos += 1
    assert pos == len(rows)
    for r in rows:
        assert r["verified"] == "true"
        for k in ("mean_seconds", "speedup", "predicted_speedup"):
            float(r[k])
            assert any(c in r[k] for c in ".en")  # format_number keeps doubles visibly floating point
        assert float(r["mean_seconds"]) > 0
    return rows


def test_format_number_and_seed():
    from paper_1708_09495_b200 import costmodel as cm
    from oracle.pyoracle import Oracle

    assert cm.format_number(2.0) == "2.0" and cm.format_number(0.5) == "0.5"
    assert cm.format_number(1e-05) == "1e-05" and cm.format_number(1.5e20) == "1.5e+20"
    orc = Oracle()
    for seed, rep in ((1, 0), (1, 3), (77, 2)):
        assert bench_csv.derive_seed(seed, rep) == orc.derive_seed(seed, rep)
    assert bench_csv.parse_size("2^20") == 1 << 20 and bench_csv.parse_size("16M") == 16 * 10**6


def test_cpu_rows_from_the_reference():
    from oracle.pyoracle import maybe_reference

    ref = maybe_reference()
    if ref is None:
        pytest.skip("oracle/_ref/libbspref.so not built")
    sizes, procs, algos = [4096, 10000], [2, 3], ["pr4", "pr2", "btn", "oet"]
    rows = bench_csv.build_rows(sizes, procs, ["sr4"] + algos, 1, 1, {"cpu": bench_csv.CpuCells(ref)})
    text = bench_csv.emit_csv(rows)
    out = _check_contract(text, sizes, procs, algos, ["cpu"])
    pred = {(r["algorithm"], r["p"]): float(r["predicted_speedup"]) for r in out if r["n"] == "4096"}
    assert pred[("sr4", "1")] == 1.0 and pred[("pr4", "2")] > 1.0


@pytest.mark.gpu
def test_gpu_rows_beside_cpu_rows(cuda):
    from oracle.pyoracle import maybe_reference

    runners = {}
    ref = maybe_reference()
    impls = ["gpu"]
    if ref is not None:
        runners["cpu"] = bench_csv.CpuCells(ref)
        impls = ["cpu", "gpu"]
    runners["gpu"] = bench_csv.GpuCells()
    sizes, procs, algos = [1 << 16], [2, 4], ["pr4", "pr2", "btn", "oet"]
    text = bench_csv.emit_csv(bench_csv.build_rows(sizes, procs, ["sr4"] + algos, 2, 1, runners))
    _check_contract(text, sizes, procs, algos, impls)
