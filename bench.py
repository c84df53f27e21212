#!/usr/bin/env python
"""bench.py -- sorted uint32 keys per second on B200 (arXiv 1708.09495 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N = 1 (default): config 2 of BASELINE.json -- single-GPU LSD radix sort (SR4:
radix 2^8, 4 stable count-sort rounds) of n = 2^28 uint32 keys drawn by the
reference generator (generate_uniform_keys, core.hpp:93-99, seed
derive_seed(1, 0), bench.hpp:86-88), device-resident; a step is one full sort.
N > 1 (torchrun, one rank per GPU): config 5, the paper's PR4 parallel radix
sort of n = 2^33 keys in total (strong scaling), block-distributed n/N per
GPU (rank w generates its Partition block of generate_uniform_keys(n,
derive_seed(1, 0)) on the device at its stream offset).  Default --pr-variant P:
each round is ONE one-sweep pass per rank that stores every key at its final
position in its owner's CUDA-IPC-mapped block over NVLink (counts all-gathered
with NCCL; a 1-element all-reduce closes the round); A = the same rounds with
NCCL all-to-all-v + rebuild; B = single NCCL exchange + local sort.

--impl reference: the reference's own CPU implementation (its unmodified
headers compiled into oracle/_ref/libbspref.so, else the oracle port) on
this box's host cores: PR4 with p = all host threads, timed like
bench::detail::run_once, on a bounded sample of the workload per step.
Prints one JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "uint32 keys sorted/sec"
UNIT = "keys/s"
N_PER_GPU = 1 << 28
N_TOTAL_C5 = 1 << 33  # config 5: 2^33 keys (32 GiB) over the N GPUs


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _first_pass_roofline(f_ms, f_cnt, alg_bytes, peak):
    """The first pass of a full sort (K3f: no order inside a digit run), same
    8 B/key, timed live like the stable pass."""
    if not f_cnt:
        return None
    per = f_ms / f_cnt
    ach = alg_bytes / (per / 1e3) / 1e9
    return {"kernel": "first_pass_kernel (pass 0 of a full sort)", "avg_launch_ms": per, "achieved": ach,
            "frac": ach / peak, "launches_per_sort": f_cnt / 3}


def _variant_roofline(ms, cnt, alg_bytes, peak):
    if not cnt:
        return None
    per = ms / cnt
    ach = alg_bytes / (per / 1e3) / 1e9
    return {"avg_launch_ms": per, "achieved": ach, "frac": ach / peak, "launches_per_sort": cnt / 3}


def _traffic(kernel: str, n: int):
    """dram__bytes_read+write per launch from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        e = tr.get(kernel)
        if e and int(e.get("n", -1)) == n:
            return float(e["dram_bytes_per_launch"]), e.get("source")
    except Exception:
        pass
    return None, None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.25)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
                self.lines = [l for l in out.splitlines() if l.strip()]
            except Exception:
                pass

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            parts = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def _sorted_permutation_checks(inp, out) -> bool:
    import torch

    a = inp.to(torch.int64) & 0xFFFFFFFF
    b = out.to(torch.int64) & 0xFFFFFFFF
    if b.numel() > 1 and not bool((b[1:] >= b[:-1]).all()):
        return False
    m = 1000003
    sq = lambda x: int(((x % m) * (x % m) % m).sum())  # noqa: E731
    cube = lambda x: int(((x % m) * (x % m) % m * (x % m) % m).sum())  # noqa: E731
    return int(a.sum()) == int(b.sum()) and sq(a) == sq(b) and cube(a) == cube(b)


def cpu_baseline_sample(keys: np.ndarray, reps: int = 1):
    """The reference's serial_radix_sort(., 256) on one host core (SR4, the
    paper's baseline row, bench.hpp:185-199) on the SAME config-2 keys (all
    2^28 of them), timed like run_once (bench.hpp:114-141)."""
    from oracle.pyoracle import Oracle, maybe_reference

    ref = maybe_reference()
    impl, kind = (ref, "reference") if ref is not None else (Oracle(), "port")
    ts = []
    for _ in range(reps):
        t, out = impl.time_serial_radix_sort(keys, 256)
        ts.append(t)
    assert np.array_equal(out[:: max(1, keys.size // 65536)], np.sort(keys)[:: max(1, keys.size // 65536)])
    t = statistics.median(ts)
    return {"value": keys.size / t, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"serial_radix_sort(.,256) (SR4) of the config-2 keys (n={keys.size}) on 1 host core, "
                      f"{'median of ' + str(reps) if reps > 1 else 'one run'}, timed like bench.hpp run_once; "
                      f"host {os.cpu_count()} threads, {_cpu_model()}"}


def run_reference(args, rank: int, world: int):
    """--impl reference: the reference's own CPU implementation of config 2.

    Only the reference's headers compiled unmodified (oracle/_ref/libbspref.so)
    run here -- the product package is never imported, so libbsg.so is not
    loaded in this process.  Keys come from the reference's own
    generate_uniform_keys (core.hpp:93-99) with derive_seed(1, 0)
    (bench.hpp:86-88).  A step is run_parallel_radix PR4 (radix.hpp:260-303,
    r=256: the same 4 stable count-sort rounds as config 2) with p = every
    host thread over ALL n = 2^28 keys, timed like bench::detail::run_once
    (bench.hpp:114-141: prepare outside, run inside the clock).  Under torchrun
    only rank 0 runs; the others exit without work."""
    if rank != 0:
        return
    from oracle.pyoracle import Oracle, maybe_reference

    n = args.ref_n if args.ref_n else N_PER_GPU
    ref = maybe_reference()
    p = os.cpu_count() or 1
    seed = Oracle().derive_seed(1, 0)
    if ref is not None:
        kind = "reference"
        keys = ref.generate_uniform_keys(n, seed)
        step = lambda: ref.time_parallel_radix(keys, p, 256)  # noqa: E731
        what = f"reference run_parallel_radix PR4 (r=256, 4 rounds) with p={p} worker threads"
    else:  # the oracle port is single-threaded (only when the reference could not be compiled)
        orc = Oracle()
        kind, p = "port", 1
        keys = orc.generate_uniform_keys(n, seed)
        step = lambda: orc.time_serial_radix_sort(keys, 256)  # noqa: E731
        what = "oracle port serial_radix_sort(.,256), 1 thread"
    for _ in range(args.warmup):
        step()
    ts = []
    for _ in range(args.steps):
        t, out = step()
        ts.append(t)
    verified = bool(np.array_equal(out, np.sort(keys)))
    t = sum(ts) / len(ts)
    value = n / t
    full = n == N_PER_GPU and world == 1
    sample = (f"{what} on n={n} keys per step "
              + ("(the full config-2 workload)" if full else f"(a bounded sample of the {world}-GPU workload)")
              + f", mean of {args.steps} steps, timed like bench.hpp run_once; host: {os.cpu_count()} threads, "
              + _cpu_model())
    cfg = _config(1) if world == 1 else _config(world, args.pr_variant)
    cfg = dict(cfg, n=n, algorithm="PR4" if kind == "reference" else "SR4")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak" if world == 1 else "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (reference generator, seeded)", "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": p, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "verified": verified,
    }
    print(json.dumps(line), flush=True)


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for l in f:
                if l.startswith("model name"):
                    return l.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown CPU"


def _config(world: int, variant=None, n_total: int = None):
    if world == 1 and variant is None:
        return {"workload": "config 2: single-GPU LSD radix sort (SR4: radix 2^8, 4 stable count-sort rounds) of "
                            "n=2^28 uint32 keys, generate_uniform_keys(n, derive_seed(1,0))",
                "n": N_PER_GPU, "radix": 256, "rounds": 4, "parallelism": "single GPU",
                "l2": "inputs (1 GiB) larger than L2 (126 MB); no flush needed"}
    if variant == "A":
        what = ("PR4 as run_parallel_radix: per round digit count + NCCL all-gather of counts + local stable pass + "
                "NCCL all-to-all-v of the contiguous slices + rebuild (4 exchanges; per-round states bit-identical "
                "to the reference)")
    elif variant == "P":
        what = ("PR4 as run_parallel_radix with the exchange fused into the pass: per round digit count + NCCL "
                "all-gather of counts + ONE one-sweep pass per rank whose write-out stores every key at its final "
                "position in its owner's IPC-mapped next-round block over NVLink + a 1-element all-reduce barrier "
                "(per-round states bit-identical to the reference)")
    else:
        what = ("variant B: top-digit histogram + NCCL all-gather of counts + one stable partition pass + ONE NCCL "
                "all-to-all-v + local LSD sort (same sorted concatenation; per-rank sizes cut on digit boundaries)")
    n_total = n_total or N_TOTAL_C5
    return {"workload": f"config 5: multi-GPU parallel radix sort of n={n_total} uint32 keys "
                        f"(generate_uniform_keys(n, derive_seed(1,0)), block-distributed n/p per GPU, generated on "
                        f"each GPU at its stream offset) over {world} GPUs: " + what,
            "variant": variant, "n": n_total, "n_per_gpu": n_total // world, "radix": 256, "rounds": 4,
            "parallelism": f"dp{world}", "l2": "inputs larger than L2; no flush needed"}


def run_single(args):
    import torch
    import paper_1708_09495_b200 as bsg
    from paper_1708_09495_b200 import _lib

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    n = args.n
    keys = bsg.generate_uniform_keys(n, bsg.derive_seed(1, 0))
    d_in = torch.from_numpy(keys.view(np.int32)).to(dev)
    d_out = torch.empty_like(d_in)
    ctx = _lib.context(0)
    ctx.reserve(n)
    L = _lib.lib()
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream

    def step():
        _lib.check(L.bsg_radix_sort_u32(ctx.handle, d_in.data_ptr(), d_out.data_ptr(), n, 8, _lib.MEM_DEVICE, sh))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    l0 = ctx.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    launches = ctx.launches - l0
    # correctness of what was timed (untimed): sorted + same multiset
    # (sum, sum of squares mod a prime, xor) -- no second sort is launched
    ok = _sorted_permutation_checks(d_in, d_out)

    # dominant kernel, timed live on the launching stream
    ctx.set_timing(True)
    for _ in range(3):
        step()
    os_ms, os_cnt = ctx.kernel_time(_lib.K_ONESWEEP)
    h_ms, h_cnt = ctx.kernel_time(_lib.K_HIST)
    f_ms, f_cnt = ctx.kernel_time(_lib.K_FIRST_PASS)
    r_ms, r_cnt = ctx.kernel_time(_lib.K_RELAXED_PASS)
    ctx.set_timing(False)
    # onesweep_kernel runs passes 1-3: strictly stable (K3) or, where the runs
    # of equal low bits are long, value-stable (K3r) -- one kernel template,
    # averaged over all its launches; both variants reported beside it
    strict_ms, strict_cnt = os_ms, os_cnt
    os_ms, os_cnt = os_ms + r_ms, os_cnt + r_cnt
    per_launch_s = os_ms / max(os_cnt, 1) / 1e3
    alg_bytes = 8.0 * n  # one read + one write of every key per pass
    achieved = alg_bytes / per_launch_s / 1e9
    peak, peak_src = _peaks()
    traffic, tsrc = _traffic("onesweep_pass", n)

    # end to end through the public C ABI with pinned host buffers
    h_in = torch.from_numpy(keys.view(np.int32)).pin_memory()
    h_out = torch.empty_like(h_in).pin_memory()

    def e2e_step():
        _lib.check(L.bsg_radix_sort_u32(ctx.handle, h_in.data_ptr(), h_out.data_ptr(), n, 8, _lib.MEM_HOST, sh))

    e2e_step()
    # steps per lane: the pipeline's fill and drain (one H2D and one D2H
    # without a copy in the other direction) are inside the timed region
    ke = max(1, min(args.steps, args.e2e_steps))
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(ke):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_serial_ms = e0.elapsed_time(e1) / ke
    ok_e2e = bool(np.array_equal(h_out.numpy().view(np.uint32)[:: max(1, n // 4096)],
                                 d_out.cpu().numpy().view(np.uint32)[:: max(1, n // 4096)]))

    # Two sorts in flight (a serving pattern): two host threads, each with its
    # own context + stream + pinned buffers, call the same public API; one
    # step's D2H overlaps the next step's H2D on the full-duplex PCIe link.
    # Every step still copies its own input in and its result out.
    import threading

    lanes = [(ctx, stream, h_in, h_out)]
    for _ in range(args.e2e_inflight - 1):
        lanes.append((_lib.Context(0), torch.cuda.Stream(), torch.from_numpy(keys.view(np.int32)).pin_memory(),
                      torch.empty_like(h_in).pin_memory()))

    def lane_step(c, st, hi, ho):
        _lib.check(L.bsg_radix_sort_u32(c.handle, hi.data_ptr(), ho.data_ptr(), n, 8, _lib.MEM_HOST, st.cuda_stream))

    for lane in lanes:  # warm both contexts (workspace + staging allocation)
        lane_step(*lane)
    torch.cuda.synchronize()
    nl = len(lanes)
    kp = nl * ke

    def e2e_run():
        start = torch.cuda.Event(enable_timing=True)
        ends = [torch.cuda.Event(enable_timing=True) for _ in lanes]
        start.record(stream)
        for _, st_, _, _ in lanes[1:]:
            st_.wait_event(start)

        def worker(i):
            c, st, hi, ho = lanes[i]
            for _ in range(kp // nl):
                lane_step(c, st, hi, ho)
            ends[i].record(st)

        ths = [threading.Thread(target=worker, args=(i,)) for i in range(nl)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        torch.cuda.synchronize()
        return max(start.elapsed_time(e) for e in ends) / kp

    # The hosts are shared VMs whose PCIe duplex rate moves from second to
    # second: the whole timed e2e run (fill and drain included)
    # is repeated and the MEDIAN run is reported, every run listed beside it.
    e2e_runs = [e2e_run() for _ in range(max(1, args.e2e_repeats))]
    e2e_ms = sorted(e2e_runs)[len(e2e_runs) // 2]
    ref_s = d_out.cpu().numpy().view(np.uint32)[:: max(1, n // 4096)]
    for _, _, _, ho in lanes[1:]:
        ok_e2e = ok_e2e and bool(np.array_equal(ho.numpy().view(np.uint32)[:: max(1, n // 4096)], ref_s))
    del lanes

    line = {
        "metric": METRIC, "value": n / (ms / 1e3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u32", "data": "synthetic (reference generator, seeded)", "config": _config(1),
        "e2e": {"value": n / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": 4 * n,
                "ms_per_step": e2e_ms, "in_flight": args.e2e_inflight, "steps": kp,
                "runs_ms_per_step": e2e_runs, "reported": "median of the runs",

                "path": "bsg_radix_sort_u32(BSG_MEM_HOST) from pinned host memory; host threads, each with "
                        "its own context/stream, so one step's D2H overlaps another step's H2D",
                "serial_value": n / (e2e_serial_ms / 1e3), "serial_ms_per_step": e2e_serial_ms},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": "onesweep_kernel (one stable 8-bit pass; passes 1-3 of the sort)",
                     "algorithmic_bytes_per_launch": alg_bytes, "avg_launch_ms": per_launch_s * 1e3,
                     "peak_source": peak_src, "frac_of_8TBps_nominal": achieved / 8000.0,
                     "traffic_source": tsrc,
                     "launches_per_sort": os_cnt / 3,
                     "variants": {
                         "strictly_stable_K3": _variant_roofline(strict_ms, strict_cnt, alg_bytes, peak),
                         "value_stable_K3r": _variant_roofline(r_ms, r_cnt, alg_bytes, peak)},
                     "first_pass": _first_pass_roofline(f_ms, f_cnt, alg_bytes, peak)},
        "kernels_ms_per_sort": {"onesweep": os_ms / 3, "onesweep_strict": strict_ms / 3,
                                "onesweep_value_stable": r_ms / 3, "first_pass": f_ms / 3, "hist": h_ms / 3},
        "clocks": clk.summary(),
        "verified": ok and ok_e2e,
    }
    if not args.no_other_configs:
        line["other_configs"] = other_configs(bsg, _lib, L, ctx, d_in, d_out, stream, n)
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sample(keys)
    print(json.dumps(line), flush=True)


def other_configs(bsg, _lib, L, ctx, d_in, d_out, stream, n):
    """The other BASELINE configs that fit one GPU, measured in the same run
    (device-resident inputs, CUDA events on the launching stream, median of
    a few reps after a warm-up, every output compared bit for bit with
    torch.sort of the same keys on the device): C1 latency, C2 at r = 2^16,
    C3's three skewed 2^28 inputs, C4's 2^16 x 4096 batches (BTN/OET, p = 8)
    and PR4/PR2 with 8 logical workers on the config-2 keys."""
    import torch

    sh = stream.cuda_stream
    res = {}

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    def u64(t):
        return t.view(torch.int32).to(torch.int64) & 0xFFFFFFFF

    def sort_row(t, o, radix_log2, reps, label):
        m = t.numel()
        ms = timed(lambda: _lib.check(L.bsg_radix_sort_u32(ctx.handle, t.data_ptr(), o.data_ptr(), m, radix_log2,
                                                           _lib.MEM_DEVICE, sh)), reps)
        ok = bool(torch.equal(u64(o), torch.sort(u64(t)).values))
        return {"workload": label, "n": m, "ms": ms, "keys_per_s": m / ms * 1e3, "verified": ok}

    # C1: 2^20 keys (latency; one fused cooperative launch)
    n1 = 1 << 20
    k1 = torch.from_numpy(bsg.generate_uniform_keys(n1, bsg.derive_seed(1, 0)).view(np.int32)).cuda()
    o1 = torch.empty_like(k1)
    res["C1"] = sort_row(k1, o1, 8, 50, "config 1: SR4 of 2^20 uniform keys")
    res["C1"]["us"] = res["C1"]["ms"] * 1e3
    # C2 at r = 2^16 (2 rounds, each two stable byte sub-passes from one histogram read)
    res["C2_r65536"] = sort_row(d_in, d_out, 16, 5, "config 2 at radix 2^16 (2 count-sort rounds)")
    # C3: skewed 2^28 inputs (narrow = the config-2 keys & 0xFFFF, bsg_generate_skewed kind 0)
    t = torch.empty_like(d_in)
    for name, make in (("narrow16", lambda: torch.bitwise_and(d_in, 0xFFFF, out=t)),
                       ("all_equal", lambda: t.fill_(int(np.uint32(0xABCD1234).view(np.int32)))),
                       ("zipf1.1", lambda: t.copy_(torch.from_numpy(
                           bsg.generate_skewed_keys(n, bsg.derive_seed(1, 0), 1, 1.1).view(np.int32))))):
        make()
        res["C3_" + name] = sort_row(t, d_out, 8, 5, f"config 3: SR4 of 2^28 keys, {name}")
    del t
    # C4: 2^16 arrays x 4096 keys (the config-2 keys), BTN and OET at p = 8
    num, ln = 1 << 16, 4096
    if n >= num * ln:
        ref = torch.sort(u64(d_in[:num * ln]).view(num, ln), dim=1).values
        for net, name in ((0, "BTN"), (1, "OET")):
            ms = timed(lambda: _lib.check(L.bsg_block_network_batched_u32(ctx.handle, net, d_in.data_ptr(),
                                                                          d_out.data_ptr(), num, ln, 8, -1, None,
                                                                          _lib.MEM_DEVICE, sh)), 5)
            ok = bool(torch.equal(u64(d_out[:num * ln]).view(num, ln), ref))
            res["C4_" + name + "_p8"] = {"workload": f"config 4: {name}, 2^16 arrays x 4096 keys, p = 8",
                                         "n": num * ln, "ms": ms, "keys_per_s": num * ln / ms * 1e3, "verified": ok}
        del ref
    # PR4 / PR2 with p = 8 logical workers on one GPU (the per-round BSP algorithm)
    ref = torch.sort(u64(d_in)).values
    for bits, name in ((8, "PR4"), (16, "PR2")):
        ms = timed(lambda: _lib.check(L.bsg_parallel_radix_sort_u32(ctx.handle, d_in.data_ptr(), d_out.data_ptr(), n,
                                                                    8, bits, -1, None, _lib.MEM_DEVICE, sh)), 5)
        res[name + "_p8"] = {"workload": f"{name} with 8 logical workers, 2^28 keys, one GPU", "n": n, "ms": ms,
                             "keys_per_s": n / ms * 1e3, "verified": bool(torch.equal(u64(d_out), ref))}
    return res


def run_multi(args, rank: int, world: int, local_rank: int):
    """Config 5: n = 2^33 keys in total, Partition(n, N) block w on GPU w
    (generated there at its offset of the generate_uniform_keys stream),
    PR4 over torch.distributed / NCCL, one process per GPU; strong scaling
    (total work fixed).  Timed with CUDA events, max over ranks."""
    import torch
    import torch.distributed as dist
    import paper_1708_09495_b200 as bsg
    from paper_1708_09495_b200 import _lib, distributed as D

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    n_total = args.n_total
    n_local = D.partition_size_of(n_total, world, rank)
    off = D.partition_offset_of(n_total, world, rank)
    seed = bsg.derive_seed(1, 0)
    d_in = bsg.generate_uniform_keys_device(n_local, seed, device=local_rank, offset=off).view(torch.int32)
    ctx = _lib.context(local_rank)

    peer = None
    if args.pr_variant == "P":
        # map every rank's next-round blocks (CUDA IPC); if any rank cannot,
        # all ranks agree to run variant A instead and say so in the JSON line
        try:
            peer = D.PeerBlocks(n_total, device=dev)
            okflag = 1
        except Exception as exc:  # noqa: BLE001
            print(f"rank {rank}: peer mapping failed ({exc}); falling back to variant A", file=sys.stderr)
            okflag = 0
        flag = torch.tensor([okflag], dtype=torch.int32, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0:
            args.fallback_from = "P"
            args.pr_variant = "A"
            peer = None

    def step(events=None, cevents=None, blk=None):
        blk = d_in if blk is None else blk
        if args.pr_variant == "A":
            return D.parallel_radix_sort(blk, n_total, radix=256, a2a_events=events, count_events=cevents)
        if args.pr_variant == "P":
            return D.parallel_radix_sort(blk, n_total, radix=256, a2a_events=events, exchange="peer", peer=peer,
                                         count_events=cevents)
        return D.parallel_radix_sort_single_exchange(blk, a2a_events=events)

    for _ in range(args.warmup):
        out = step()
    torch.cuda.synchronize()
    dist.barrier()
    l0 = ctx.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            out = step()
        e1.record()
        torch.cuda.synchronize()
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    launches = ctx.launches - l0
    # phase split (separate, untimed steps with events): count + count
    # all-gather, and the exchange -- A/B: the NCCL all-to-all-v; P: the fused
    # pass + round barrier, compared with the same one-sweep pass storing
    # locally (bsg_count_sort_round on the rank's block), whose difference is
    # the NVLink cost the fused pass adds
    ev, cev = [], []
    for _ in range(2):
        step(ev, cev)
    torch.cuda.synchronize()
    ksteps = 2
    a2a_ms = sum(a.elapsed_time(b) for a, b in ev) / ksteps
    cnt_ms = sum(a.elapsed_time(b) for a, b in cev) / ksteps
    local_pass_ms = 0.0
    if args.pr_variant == "P":
        # the same fused-round kernel over the same block, as a one-worker
        # round (p = 1): identical work, every store local
        ops = D.CudaStepOps(dev)
        tmp = torch.empty_like(d_in)
        cnts = [ops.count(d_in, rnd, 8) for rnd in range(4)]
        le0, le1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        le0.record()
        for _ in range(ksteps):
            for rnd in range(4):
                ops.fused_round(d_in, cnts[rnd], n_local, 1, 0, rnd, 8, [tmp.data_ptr()])
        le1.record()
        torch.cuda.synchronize()
        local_pass_ms = le0.elapsed_time(le1) / ksteps
        del tmp, cnts
    t = torch.tensor([ms, a2a_ms, cnt_ms, local_pass_ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, a2a_max, cnt_max, local_max = t.tolist()
    # verification (untimed): local sortedness, boundaries, global checksums
    # (chunked: no n-sized int64 temporaries at 2^32 keys per GPU)
    m = 1000003
    sums = [0, 0, 0, 0]
    local_ok = True
    prev = None
    step_c = 1 << 27
    for a in range(0, n_local, step_c):
        x = d_in[a:a + step_c].to(torch.int64) & 0xFFFFFFFF
        y = out[a:a + step_c].to(torch.int64) & 0xFFFFFFFF
        local_ok = local_ok and bool((y[1:] >= y[:-1]).all()) and (prev is None or int(y[0]) >= prev)
        prev = int(y[-1])
        sums[0] += int((x % m).sum()); sums[1] += int((y % m).sum())
        sums[2] += int(((x % m) * (x % m) % m).sum()); sums[3] += int(((y % m) * (y % m) % m).sum())
        del x, y
    first = int(out[0].view(torch.int32).item()) & 0xFFFFFFFF if n_local else -1
    ends = torch.tensor([first, prev if prev is not None else -1], dtype=torch.int64, device=dev)
    allends = [torch.empty_like(ends) for _ in range(world)]
    dist.all_gather(allends, ends)
    nonempty = [e for e in allends if e[0].item() >= 0]
    bounds_ok = all(nonempty[w][1].item() <= nonempty[w + 1][0].item() for w in range(len(nonempty) - 1))
    cs = torch.tensor([s_ % m for s_ in sums] + [int(local_ok)], dtype=torch.float64, device=dev)
    dist.all_reduce(cs)
    ok = bounds_ok and int(cs[0].item()) % m == int(cs[1].item()) % m and \
        int(cs[2].item()) % m == int(cs[3].item()) % m and int(cs[4].item()) == world

    # e2e: each rank's block from pinned host memory, sort, result back
    h_in = d_in.cpu().pin_memory()
    h_out = torch.empty_like(h_in).pin_memory()

    def e2e_step():
        blk = h_in.to(dev, non_blocking=True)
        res = step(blk=blk)
        h_out[: res.numel()].copy_(res, non_blocking=True)

    e2e_step()
    torch.cuda.synchronize()
    dist.barrier()
    ke = max(1, min(args.steps, 3))
    e0.record()
    for _ in range(ke):
        e2e_step()
    e1.record()
    torch.cuda.synchronize()
    te = torch.tensor([e0.elapsed_time(e1) / ke], dtype=torch.float64, device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = te.item()
    if rank == 0:
        remote = 4.0 * n_total * 4 * (world - 1) / world  # key bytes crossing GPUs per step (uniform keys: (N-1)/N per round)
        line = {
            "metric": METRIC, "value": n_total / (ms_max / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic (reference generator, seeded; each GPU generates "
                                                          "its block of the stream on the device)",
            "config": dict(_config(world, args.pr_variant, n_total),
                           **({"fallback_from": args.fallback_from} if getattr(args, "fallback_from", None) else {})),
            "e2e": {"value": n_total / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": 4 * n_total,
                    "d2h_bytes_per_step": 4 * n_total, "ms_per_step": e2e_ms},
            "gpu_launches": launches,
            "phases_ms_per_step": {"count_and_count_allgather": cnt_max,
                                   ("fused_pass_and_barrier" if args.pr_variant == "P" else "all_to_all_v"): a2a_max,
                                   **({"same_passes_local_stores_only": local_max} if args.pr_variant == "P" else {})},
            "nvlink_all_to_all_ms_per_step": (max(0.0, a2a_max - local_max) if args.pr_variant == "P" else a2a_max),
            "nvlink_share_of_step": (max(0.0, a2a_max - local_max) if args.pr_variant == "P" else a2a_max) / ms_max,
            "nvlink_share_how": ("fused pass + barrier minus the same fused-round kernel as a one-worker round "
                                 "(same block, all stores local)"
                                 if args.pr_variant == "P" else "CUDA events around the NCCL all-to-all-v"),
            "nvlink_bytes_per_step": remote,
            "clocks": clk.summary(), "verified": ok,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=N_PER_GPU, help="keys (single GPU)")
    ap.add_argument("--n-total", type=int, default=N_TOTAL_C5, help="config 5 keys over all GPUs (N > 1)")
    ap.add_argument("--ref-n", type=int, default=0, help="keys per reference step (default: config 2's 2^28)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true",
                    help="skip the C1/C3/C4/PR rows measured after the config-2 line")
    ap.add_argument("--e2e-inflight", type=int, default=4,
                    help="sorts in flight in the e2e measurement (host threads, one context/stream each)")
    ap.add_argument("--e2e-repeats", type=int, default=3,
                    help="repetitions of the whole timed e2e run; the median is reported")
    ap.add_argument("--e2e-steps", type=int, default=20,
                    help="e2e steps per lane (capped by --steps); total e2e steps = lanes x this")
    ap.add_argument("--pr-variant", choices=["A", "B", "P"], default="P",
                    help="multi-GPU algorithm: A = per-round PR4 (4 NCCL exchanges), B = single exchange, "
                         "P = per-round PR4 with the exchange + rebuild as one peer-store kernel over NVLink")
    ap.add_argument("--distributed", action="store_true",
                    help="run the NCCL PR path even with one rank (exercises the multi-GPU code on one GPU)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world == 1 and not args.distributed:
        run_single(args)
    else:
        run_multi(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
