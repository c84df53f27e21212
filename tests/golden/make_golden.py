"""Generates tests/golden/golden.npz from the REFERENCE ITSELF: the unmodified
hot-path headers under /root/reference/proj/include compiled into
oracle/_ref/libbspref.so (oracle/Makefile).  Run here (where /root/reference
exists); the committed .npz travels to the GPU box.

    python tests/golden/make_golden.py

Contents (key -> uint32/int64 array):
  draws/42/6                 generate_uniform_keys(6, 42)        (core_test.cpp:24-31)
  csr/<radix>/<round>/<case> count_sort_round outputs           (radix.hpp:44-65)
  srs/<radix>/<case>         serial_radix_sort outputs          (radix.hpp:69-90)
  pr/<radix>/<p>/<k>         run_parallel_radix with plan.rounds=k (radix.hpp:260-303)
  prstats/<radix>/<p>/<k>    its RunStats (supersteps, msgs, words x2)
  net/<btn|oet>/<p>/<s>      run_block_network with stages[:s]   (netsort.hpp:157-199)
  netstats/<btn|oet>/<p>/<s> its RunStats
  ms/<i>/a,b,low,high        merge_split                         (netsort.hpp:30-51)
  in/<case>                  the inputs
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.pyoracle import Reference  # noqa: E402


def stats_vec(st):
    return np.array([st["supersteps"], st["messages_sent"], st["messages_delivered"], st["words_sent"],
                     st["words_delivered"]], dtype=np.int64)


def main():
    ref = Reference()
    g = {}
    g["draws/42/6"] = ref.generate_uniform_keys(6, 42)
    cases = {
        "u1000": ref.generate_uniform_keys(1000, 2024),
        "dup": ref.generate_uniform_keys(777, 13) % 31,
        "tag": ((ref.generate_uniform_keys(1500, 7) % (1 << 18)).astype(np.uint64) << np.uint64(14) | np.arange(1500, dtype=np.uint64)).astype(np.uint32),
        "same": np.full(100, 0xABCD1234, np.uint32),
        "asc": (np.arange(300, dtype=np.uint64) * 3).astype(np.uint32),
        "desc": ((300 - np.arange(300, dtype=np.uint64)) * 3).astype(np.uint32),
        "one": np.array([7], np.uint32),
        "empty": np.array([], np.uint32),
    }
    for name, k in cases.items():
        g[f"in/{name}"] = k
        for radix in (2, 4, 16, 256, 65536):
            bits = radix.bit_length() - 1
            for rnd in range(32 // bits):
                if radix == 2 and rnd not in (0, 13, 31):
                    continue
                g[f"csr/{radix}/{rnd}/{name}"] = ref.count_sort_round(k, rnd, radix)
            g[f"srs/{radix}/{name}"] = ref.serial_radix_sort(k, radix)
    prin = ref.generate_uniform_keys(1003, 77) % 5000
    g["in/pr"] = prin
    for radix in (256, 65536):
        rounds = 32 // (radix.bit_length() - 1)
        for p in (1, 2, 3, 5, 8, 16):
            for k in range(rounds + 1):
                out, st = ref.parallel_radix(prin, p, radix, k)
                g[f"pr/{radix}/{p}/{k}"] = out
                g[f"prstats/{radix}/{p}/{k}"] = stats_vec(st)
    netin = ref.generate_uniform_keys(480, 99)
    g["in/net"] = netin
    for net, name, ps in ((0, "btn", (1, 2, 4, 8, 16)), (1, "oet", (1, 2, 3, 4, 5, 8))):
        for p in ps:
            S = ref.schedule(net, p)[0].shape[0]
            for s in range(S + 1):
                out, st = ref.block_network(net, netin, p, s)
                g[f"net/{name}/{p}/{s}"] = out
                g[f"netstats/{name}/{p}/{s}"] = stats_vec(st)
    rng = np.random.default_rng(5)
    for i in range(8):
        a = np.sort(rng.integers(0, 50, rng.integers(0, 40)).astype(np.uint32))
        b = np.sort(rng.integers(0, 50, rng.integers(0, 40)).astype(np.uint32))
        lo, hi = ref.merge_split(a, b)
        g[f"ms/{i}/a"], g[f"ms/{i}/b"], g[f"ms/{i}/low"], g[f"ms/{i}/high"] = a, b, lo, hi
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **g)
    print(f"wrote {len(g)} arrays")


if __name__ == "__main__":
    main()
