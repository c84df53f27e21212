"""The reference's bench CSV contract with the reference's own
CPU rows beside this repo's GPU rows.

Runs the grid of bench.hpp:184-198 (`run_benchmark`): for every n an SR4
baseline row (p = 1) first, then every other algorithm over the processor
counts; repetition r sorts generate_uniform_keys(n, derive_seed(seed, r))
(bench.hpp:162-166).  Each cell is measured by

  cpu -- the reference itself (oracle/_ref/libbspref.so, its unmodified
         headers), timed like bench.hpp:114-141 `run_once`: serial_radix_sort,
         run_parallel_radix and run_block_network with their default
         executors on this host's cores, input preparation outside the timer;
  gpu -- this repo's C ABI on device-resident keys (CUDA events around the
         sort call).

Columns are bench.hpp:221 `csv_header` plus a trailing `impl` column (cpu /
gpu), so a reader of the reference's seven columns still parses every line.
`speedup` is relative to the CPU SR4 row of the same n when CPU rows are
measured (the paper's speedup over the sequential CPU sort), else to the GPU
SR4 row; `predicted_speedup` is the cost model (costmodel.py, g/G = 5,
bench.hpp:38, restated because costmodel.hpp needs Boost); `verified` is the
sorted-permutation check of bench.hpp (equality with np.sort).  BTN cells for
non-power-of-two p are skipped like bench.hpp:150-154.

usage: python scripts/bench_csv.py [--sizes 2^20,2^24] [--procs 2,4,8]
           [--algorithms pr4,pr2,btn,oet] [--reps 3] [--impls cpu,gpu] [--out F]
       (sizes accept K/M/G decimal suffixes like bspsort_bench.cpp:36-52, or 2^k)
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1708_09495_b200 import costmodel as cm  # noqa: E402

CSV_HEADER = cm.CSV_HEADER + ",impl"
ALGOS = ("sr4", "pr4", "pr2", "btn", "oet")


def parse_size(s: str) -> int:
    s = s.strip()
    if s.startswith("2^"):
        return 1 << int(s[2:])
    mult = {"K": 10**3, "M": 10**6, "G": 10**9}
    if s[-1].upper() in mult:
        return int(s[:-1]) * mult[s[-1].upper()]
    return int(s)


def splitmix64(x: int) -> int:
    m = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & m
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & m
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & m
    return x ^ (x >> 31)


def derive_seed(seed: int, rep: int) -> int:
    """bench.hpp:84-86."""
    return splitmix64(seed ^ splitmix64(rep))


class CpuCells:
    """The reference's own code (oracle/_ref), timed like bench.hpp run_once."""

    def __init__(self, ref):
        self.ref = ref

    def keys(self, n, seed):
        return self.ref.generate_uniform_keys(n, seed)

    def run(self, algo, keys, p):
        if algo == "sr4":
            return self.ref.time_serial_radix_sort(keys, 256)
        if algo in ("pr4", "pr2"):
            return self.ref.time_parallel_radix(keys, p, 256 if algo == "pr4" else 65536)
        return self.ref.time_network_once(0 if algo == "btn" else 1, keys, p)


class GpuCells:
    """This repo's C ABI on device-resident keys (CUDA events)."""

    def __init__(self):
        import torch

        import paper_1708_09495_b200 as bsg
        from paper_1708_09495_b200 import _lib

        self.torch, self.bsg, self._lib = torch, bsg, _lib
        self.ctx = _lib.context(0)
        self.L = _lib.lib()

    def keys(self, n, seed):
        return self.bsg.generate_uniform_keys(n, seed)

    def _call(self, algo, p, src, dst, n, st):
        L, h, dev = self.L, self.ctx.handle, self._lib.MEM_DEVICE
        if algo == "sr4":
            rc = L.bsg_radix_sort_u32(h, src, dst, n, 8, dev, st)
        elif algo in ("pr4", "pr2"):
            rc = L.bsg_parallel_radix_sort_u32(h, src, dst, n, p, 8 if algo == "pr4" else 16, -1, None, dev, st)
        else:
            rc = L.bsg_block_network_batched_u32(h, 0 if algo == "btn" else 1, src, dst, 1, n, p, -1, None, dev, st)
        self._lib.check(rc)

    def run(self, algo, keys, p):
        torch = self.torch
        t = torch.from_numpy(keys.view(np.int32)).cuda()
        o = torch.empty_like(t)
        st = torch.cuda.current_stream().cuda_stream
        self._call(algo, p, t.data_ptr(), o.data_ptr(), keys.size, st)  # warm (workspace sizing)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        self._call(algo, p, t.data_ptr(), o.data_ptr(), keys.size, st)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3, o.cpu().numpy().view(np.uint32)


def cell(runner, algo, n, p, reps, seed):
    """bench.hpp:143-178 run_cell: (mean seconds, verified) or None (skipped)."""
    if algo == "btn" and (p & (p - 1)) != 0:
        return None
    secs, ok = [], True
    for rep in range(reps):
        keys = runner.keys(n, derive_seed(seed, rep))
        s, out = runner.run(algo, keys, p)
        secs.append(s)
        ok = ok and np.array_equal(out, np.sort(keys))
    return sum(secs) / len(secs), ok


def build_rows(sizes, procs, algos, reps, seed, runners):
    """Rows (dicts) in run_benchmark order: per n the SR4 baseline (p = 1)
    first, then algorithm x processor count; per cell one row per impl."""
    algos = [a for a in algos if a != "sr4"]
    rows = []
    for n in sizes:
        base = {}
        for impl, r in runners.items():
            mean, ok = cell(r, "sr4", n, 1, reps, seed)
            base[impl] = mean
            rows.append(dict(algorithm="sr4", n=n, p=1, mean=mean, ok=ok, impl=impl))
        ref_base = base.get("cpu", base.get("gpu"))
        for row in rows:
            if row["n"] == n:
                row["speedup"] = ref_base / row["mean"] if row["mean"] > 0 else 0.0
        for algo in algos:
            for p in procs:
                for impl, r in runners.items():
                    res = cell(r, algo, n, p, reps, seed)
                    if res is None:
                        continue
                    mean, ok = res
                    rows.append(dict(algorithm=algo, n=n, p=p, mean=mean, ok=ok, impl=impl,
                                     speedup=ref_base / mean if mean > 0 else 0.0))
    for row in rows:
        row["predicted"] = cm.predicted_for(row["algorithm"], row["n"], row["p"])
    return rows


def emit_csv(rows) -> str:
    """bench.hpp:223-252 emit_csv, plus the impl column."""
    lines = [CSV_HEADER]
    for r in rows:
        lines.append(cm.csv_row(r["algorithm"], r["n"], r["p"], r["mean"], r["speedup"], r["predicted"], r["ok"]) +
                     "," + r["impl"])
    return "\n".join(lines) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="2^20,2^24")
    ap.add_argument("--procs", default="2,4,8")
    ap.add_argument("--algorithms", default="pr4,pr2,btn,oet")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--impls", default="cpu,gpu")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    sizes = [parse_size(s) for s in args.sizes.split(",")]
    procs = [int(p) for p in args.procs.split(",")]
    algos = [a.strip().lower() for a in args.algorithms.split(",") if a.strip()]
    for a in algos:
        if a not in ALGOS:
            raise SystemExit(f"unknown algorithm {a!r}")
    runners = {}
    for impl in [s.strip() for s in args.impls.split(",") if s.strip()]:
        if impl == "cpu":
            from oracle.pyoracle import maybe_reference

            ref = maybe_reference()
            if ref is None:
                print("# cpu rows skipped: oracle/_ref/libbspref.so not built", file=sys.stderr)
                continue
            runners["cpu"] = CpuCells(ref)
        elif impl == "gpu":
            runners["gpu"] = GpuCells()
        else:
            raise SystemExit(f"unknown impl {impl!r}")
    text = emit_csv(build_rows(sizes, procs, algos, args.reps, args.seed, runners))
    sys.stdout.write(text)
    if args.out:
        with open(args.out, "w") as f:
            f.write(text)


if __name__ == "__main__":
    main()
