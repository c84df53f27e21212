#!/usr/bin/env python
"""Measures every BASELINE.json config that fits one GPU, with the reference
CPU path timed beside it on this box's host cores, and writes one JSON record
per row (stdout; --out FILE to save).  Development/measurement aid; the
driver's contract benchmark is bench.py.

Rows:
  C1  SR4 of 2^20 keys (latency; working set fits L2)
  C2  LSD sort of 2^28 keys at r=2^8 and r=2^16
  C3  2^28 skewed keys: narrow [0,2^16), Zipf(1.1), all-equal; r=2^8 and r=2^16
  C4  2^16 arrays x 4096 keys, BTN and OET at p=2,4,8 (+ len sweep 256..16384 at p=8)
  PR  PR4/PR2 with p logical workers on one GPU (2^26 keys, p=2,4,8)
GPU times: CUDA events on the launching stream, device-resident inputs,
median of reps after warm-up.  CPU: the reference's own headers
(oracle/_ref), timed like bench.hpp run_once, on bounded samples.
"""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1708_09495_b200 as bsg  # noqa: E402
from paper_1708_09495_b200 import _lib  # noqa: E402
from oracle.pyoracle import maybe_reference  # noqa: E402

def _peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback


PEAK = _peak()


def gpu_time(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--only", default="C1,C2,C4,PR,C5", help="comma-separated sections: C1,C2,C4,PR,C5")
    args = ap.parse_args()
    only = set(args.only.split(","))
    ref = maybe_reference()
    ctx = _lib.context(0)
    L = _lib.lib()
    st = torch.cuda.current_stream().cuda_stream
    rows = []

    def emit(row):
        rows.append(row)
        print(json.dumps(row), flush=True)

    def sort_dev(t, out, bits):
        _lib.check(L.bsg_radix_sort_u32(ctx.handle, t.data_ptr(), out.data_ptr(), t.numel(), bits, 1, st))

    if "C1" in only:
        c1(ref, sort_dev, emit)
    if "C2" in only:
        c2(args, ref, ctx, sort_dev, emit)
    if "C4" in only:
        c4(args, ref, ctx, L, st, emit)
    if "PR" in only:
        pr_rows(args, ref, L, ctx, st, emit)
    if "C5" in only and not args.quick:
        c5_rows(args, ref, L, ctx, st, emit)
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"host_threads": os.cpu_count(), "gpu": torch.cuda.get_device_name(0), "rows": rows,
                       "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}, f, indent=1)


def c1(ref, sort_dev, emit):
    n = 1 << 20
    keys = bsg.generate_uniform_keys(n, bsg.derive_seed(1, 0))
    t = torch.from_numpy(keys.view(np.int32)).cuda()
    out = torch.empty_like(t)
    ms = gpu_time(lambda: sort_dev(t, out, 8), reps=50, warm=5)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), np.sort(keys))
    row = {"row": "C1 SR4 2^20", "n": n, "gpu_ms": ms, "gpu_keys_per_s": n / ms * 1e3}
    if ref is not None:
        tc = statistics.median([ref.time_serial_radix_sort(keys, 256)[0] for _ in range(3)])
        row.update({"cpu_ref_ms": tc * 1e3, "cpu_cores": 1, "speedup": tc * 1e3 / ms})
    emit(row)


def c2(args, ref, ctx, sort_dev, emit):
    # ---- C2 / C3 ----------------------------------------------------------
    L_ = _lib.lib()
    st_ = torch.cuda.current_stream().cuda_stream
    n = 1 << 28
    inputs = [("uniform", bsg.generate_uniform_keys(n, bsg.derive_seed(1, 0)))]
    if not args.quick:
        inputs += [("narrow16", bsg.generate_skewed_keys(n, bsg.derive_seed(1, 0), 0)),
                   ("zipf1.1", bsg.generate_skewed_keys(n, bsg.derive_seed(1, 0), 1, 1.1)),
                   ("all_equal", bsg.generate_skewed_keys(n, bsg.derive_seed(1, 0), 2))]
    sample = 1 << 24
    for name, keys in inputs:
        t = torch.from_numpy(keys.view(np.int32)).cuda()
        out = torch.empty_like(t)
        for bits in (8, 16):
            ctx.set_timing(True)
            ms = gpu_time(lambda: sort_dev(t, out, bits))
            os_ms, os_n = ctx.kernel_time(_lib.K_ONESWEEP)
            ctx.set_timing(False)
            ok = bool(torch.equal(out.to(torch.int64) & 0xFFFFFFFF, torch.sort(t.to(torch.int64) & 0xFFFFFFFF).values))
            sorts = os_n / 4  # every sort launches the four 8-bit passes (identity ones exit at once)
            # identity passes (one digit value over all keys) are skipped: the
            # roofline is taken over the executed passes only
            skipped = [p for p in range(4) if int(((keys >> (8 * p)) & 255).min()) == int(((keys >> (8 * p)) & 255).max())]
            passes = 4 - len(skipped)
            row = {"row": f"{'C2' if name == 'uniform' else 'C3'} {name} r=2^{bits}", "n": n, "gpu_ms": ms,
                   "gpu_keys_per_s": n / ms * 1e3, "executed_passes_per_sort": passes,
                   "skipped_identity_passes": skipped, "verified": ok}
            if os_n and passes:
                per = os_ms / (sorts * passes)
                row.update({"onesweep_ms_per_pass": per, "pass_GBps": 8 * n / per / 1e6,
                            "pass_frac_of_measured_hbm": 8 * n / per / 1e6 / PEAK})
            if ref is not None:
                smp = n if name == "uniform" else sample
                tc, _ = ref.time_serial_radix_sort(keys[:smp], 1 << bits)
                row.update({"cpu_ref_keys_per_s_1core": smp / tc, "cpu_sample": smp,
                            "speedup_vs_1core": (n / ms * 1e3) / (smp / tc)})
            emit(row)
        # K4: one r = 2^16 count-sort round (radix.hpp:44-65 at r = 65536):
        # both byte histograms from one read + two stable byte passes; the
        # paper's traffic model for a round is one read + one write (8 B/key)
        for rnd in (0, 1):
            def run_round():
                _lib.check(L_.bsg_count_sort_round_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, rnd, 16, 1, st_))
            ms = gpu_time(run_round)
            row = {"row": f"{'C2' if name == 'uniform' else 'C3'} {name} count_sort_round r=2^16 round {rnd} (K4)",
                   "n": n, "gpu_ms": ms, "round_GBps_8B_per_key": 8 * n / ms / 1e6,
                   "round_frac_of_measured_hbm": 8 * n / ms / 1e6 / PEAK,
                   "bytes_moved_per_key": 20, "moved_GBps": 20 * n / ms / 1e6}
            emit(row)
        del t, out


def c4(args, ref, ctx, L, st, emit):
    # ---- C4 ---------------------------------------------------------------
    num, ln = 1 << 16, 4096
    keys = bsg.generate_uniform_keys(num * ln, bsg.derive_seed(1, 0))
    t = torch.from_numpy(keys.view(np.int32)).cuda()
    out = torch.empty_like(t)
    sample_arrays = 256
    for net, nm in ((0, "BTN"), (1, "OET")):
        for p in (2, 4, 8):
            def run():
                _lib.check(L.bsg_block_network_batched_u32(ctx.handle, net, t.data_ptr(), out.data_ptr(), num, ln, p,
                                                           -1, None, 1, st))
            ms = gpu_time(run)
            ok = all(bool(torch.equal(out.view(num, ln)[a:a + 4096].to(torch.int64) & 0xFFFFFFFF,
                                      torch.sort(t.view(num, ln)[a:a + 4096].to(torch.int64) & 0xFFFFFFFF,
                                                 dim=1).values)) for a in range(0, num, 4096))  # all 65536 arrays
            row = {"row": f"C4 {nm} p={p} 2^16x4096", "n": num * ln, "gpu_ms": ms, "gpu_keys_per_s": num * ln / ms * 1e3,
                   "hbm_frac": 8 * num * ln / (ms * 1e-3) / 1e9 / PEAK, "verified": ok}
            if ref is not None:
                arrs = keys[:sample_arrays * ln].reshape(sample_arrays, ln)
                tc, _ = ref.time_block_network(net, arrs, p)
                row.update({"cpu_ref_keys_per_s_1core_seq_executor": sample_arrays * ln / tc,
                            "cpu_sample_arrays": sample_arrays})
            emit(row)
    if not args.quick:
        for ln2 in (256, 1024, 16384):
            num2 = (1 << 28) // ln2
            t2 = t[: num2 * ln2]
            out2 = out[: num2 * ln2]
            for net, nm in ((0, "BTN"), (1, "OET")):
                def run2():
                    _lib.check(L.bsg_block_network_batched_u32(ctx.handle, net, t2.data_ptr(), out2.data_ptr(), num2,
                                                               ln2, 8, -1, None, 1, st))
                ms = gpu_time(run2)
                emit({"row": f"C4-sweep {nm} p=8 len={ln2}", "n": num2 * ln2, "gpu_ms": ms,
                      "gpu_keys_per_s": num2 * ln2 / ms * 1e3})
    del t, out


def pr_rows(args, ref, L, ctx, st, emit):
    # ---- PR with logical workers on one GPU ------------------------------
    n = 1 << 26
    keys = bsg.generate_uniform_keys(n, bsg.derive_seed(1, 0))
    t = torch.from_numpy(keys.view(np.int32)).cuda()
    out = torch.empty_like(t)
    for radix_log2, nm in ((8, "PR4"), (16, "PR2")):
        for p in (2, 4, 8):
            def runp():
                _lib.check(L.bsg_parallel_radix_sort_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, p, radix_log2, -1,
                                                         None, 1, st))
            ms = gpu_time(runp, reps=5, warm=2)
            ok = bool(torch.equal(out.to(torch.int64) & 0xFFFFFFFF, torch.sort(t.to(torch.int64) & 0xFFFFFFFF).values))
            row = {"row": f"{nm} p={p} logical workers, 1 GPU", "n": n, "gpu_ms": ms, "gpu_keys_per_s": n / ms * 1e3,
                   "verified": ok}
            if ref is not None and not args.quick:
                tc, _ = ref.time_parallel_radix(keys, p, 1 << radix_log2)
                row.update({"cpu_ref_ms": tc * 1e3, "cpu_threads": p, "speedup": tc * 1e3 / ms})
            emit(row)


def c5_rows(args, ref, L, ctx, st, emit):
    # ---- C5 at its full size on one GPU: p logical workers ---------------
    # n = 2^33 keys of generate_uniform_keys(n, derive_seed(1, 0)), generated
    # on the device (bit-identical stream); verified by sortedness + multiset
    # checksums (tests/test_pr_gpu.py::test_c5_full_size_in_process)
    n = 1 << 33
    free, _ = torch.cuda.mem_get_info()
    if free < 17 * n:
        emit({"row": "C5 2^33 in-process", "skipped": f"needs ~{17 * n >> 30} GiB free, have {free >> 30}"})
        return
    t = bsg.generate_uniform_keys_device(n, bsg.derive_seed(1, 0)).view(torch.int32)
    out = torch.empty_like(t)
    for p in (2, 4, 8):
        def runp():
            _lib.check(L.bsg_parallel_radix_sort_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, p, 8, -1, None, 1,
                                                     st))
        ms = gpu_time(runp, reps=3, warm=1)
        step = 1 << 27
        ok = True
        prev = -1
        s_in = s_out = 0
        for a in range(0, n, step):
            y = out[a:a + step].to(torch.int64) & 0xFFFFFFFF
            x = t[a:a + step].to(torch.int64) & 0xFFFFFFFF
            ok = ok and bool((y[1:] >= y[:-1]).all()) and int(y[0]) >= prev
            prev = int(y[-1])
            s_in += int(x.sum()); s_out += int(y.sum())
        emit({"row": f"C5 PR4 p={p} logical workers, 1 GPU, n=2^33", "n": n, "gpu_ms": ms,
              "gpu_keys_per_s": n / ms * 1e3, "verified": ok and s_in == s_out,
              "note": "one GPU stands in for the data flow only (no NVLink): blocks of n/p keys, every round a "
                      "local pass + routing to the owners' blocks"})
    del t, out
    torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
