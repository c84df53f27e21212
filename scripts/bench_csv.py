"""GPU rows in the reference's bench CSV contract.

Runs the grid of bench.hpp:184-198 (`run_benchmark`): for every n an SR4
baseline row (p = 1), then every other algorithm over the processor-count
list; rep r sorts generate_uniform_keys(n, derive_seed(seed, r)) (bench.hpp:
162-166).  `mean_seconds` is the mean device time of the sort call on
device-resident keys (CUDA events; the reference's run_once likewise keeps
input preparation outside the timer), `speedup` is relative to the SR4 row
at the same n, `predicted_speedup` comes from the cost model
(paper_1708_09495_b200/costmodel.py, g/G = 5, bench.hpp:38), and `verified`
is an on-device sorted-permutation check.  BTN rows for non-power-of-two p
are skipped like bench.hpp:150-154.

usage: python scripts/bench_csv.py [--sizes 1M,16M] [--procs 2,4,8] [--reps 3]
       (sizes accept K/M/G decimal suffixes like bspsort_bench.cpp:36-52, or 2^k)
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib
from paper_1708_09495_b200 import costmodel as cm


def parse_size(s: str) -> int:
    s = s.strip()
    if s.startswith("2^"):
        return 1 << int(s[2:])
    mult = {"K": 10**3, "M": 10**6, "G": 10**9}
    if s[-1].upper() in mult:
        return int(s[:-1]) * mult[s[-1].upper()]
    return int(s)


def verified(inp: torch.Tensor, out: torch.Tensor) -> bool:
    a = inp.to(torch.int64) & 0xFFFFFFFF
    b = out.to(torch.int64) & 0xFFFFFFFF
    if b.numel() > 1 and not bool((b[1:] >= b[:-1]).all()):
        return False
    m = 1000003
    sq = lambda x: int(((x % m) * (x % m) % m).sum())  # noqa: E731
    return int(a.sum()) == int(b.sum()) and sq(a) == sq(b)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="2^20,2^24,2^26")
    ap.add_argument("--procs", default="2,4,8")
    ap.add_argument("--algorithms", default="pr4,pr2,btn,oet")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    sizes = [parse_size(s) for s in args.sizes.split(",")]
    procs = [int(p) for p in args.procs.split(",")]
    algos = [a.strip().lower() for a in args.algorithms.split(",") if a.strip().lower() != "sr4"]

    ctx = _lib.context(0)
    L = _lib.lib()
    st = torch.cuda.current_stream().cuda_stream
    dev = _lib.MEM_DEVICE if hasattr(_lib, "MEM_DEVICE") else 1

    def call(algo, p, src, dst, n):
        if algo == "sr4":
            rc = L.bsg_radix_sort_u32(ctx.handle, src, dst, n, 8, dev, st)
        elif algo in ("pr4", "pr2"):
            rc = L.bsg_parallel_radix_sort_u32(ctx.handle, src, dst, n, p, 8 if algo == "pr4" else 16, -1, None,
                                               dev, st)
        else:
            rc = L.bsg_block_network_batched_u32(ctx.handle, 0 if algo == "btn" else 1, src, dst, 1, n, p, -1, None,
                                                 dev, st)
        _lib.check(rc)

    def cell(algo, n, p):
        secs, ok = [], True
        for rep in range(args.reps):
            keys = bsg.generate_uniform_keys(n, bsg.derive_seed(args.seed, rep))
            t = torch.from_numpy(keys.view(np.int32)).cuda()
            o = torch.empty_like(t)
            call(algo, p, t.data_ptr(), o.data_ptr(), n)  # warm (workspace sizing)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            call(algo, p, t.data_ptr(), o.data_ptr(), n)
            e1.record()
            torch.cuda.synchronize()
            secs.append(e0.elapsed_time(e1) / 1e3)
            ok = ok and verified(t, o)
        return sum(secs) / len(secs), ok

    lines = [cm.CSV_HEADER]
    for n in sizes:
        base, ok = cell("sr4", n, 1)
        lines.append(cm.csv_row("sr4", n, 1, base, 1.0, cm.predicted_for("sr4", n, 1), ok))
        print(lines[-1], flush=True)
        for algo in algos:
            for p in procs:
                if algo == "btn" and (p & (p - 1)) != 0:
                    continue
                mean, ok = cell(algo, n, p)
                lines.append(cm.csv_row(algo, n, p, mean, base / mean if mean > 0 else 0.0,
                                        cm.predicted_for(algo, n, p), ok))
                print(lines[-1], flush=True)
    if args.out:
        with open(args.out, "w") as f:
            f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
