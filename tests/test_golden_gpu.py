"""GPU: the product reproduces every golden vector the reference produced
(tests/golden/golden.npz) -- per-round count-sort outputs, serial sorts,
per-round PR states + RunStats, per-stage BTN/OET states + RunStats,
merge_split."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


def test_product_reproduces_golden(cuda, bsg):
    g = np.load(GOLDEN)
    checked = 0
    for key in g.files:
        parts = key.split("/")
        if parts[0] == "csr":
            radix, rnd, case = int(parts[1]), int(parts[2]), parts[3]
            np.testing.assert_array_equal(bsg.radix.count_sort_round(g[f"in/{case}"], rnd, radix), g[key], key)
        elif parts[0] == "srs":
            radix, case = int(parts[1]), parts[2]
            np.testing.assert_array_equal(bsg.radix.serial_radix_sort(g[f"in/{case}"], radix), g[key], key)
        elif parts[0] == "pr":
            radix, p, k = map(int, parts[1:])
            prep = bsg.radix.prepare_parallel_radix(g["in/pr"], p, radix)
            prep.plan.rounds = k
            res = bsg.radix.run_parallel_radix(prep)
            np.testing.assert_array_equal(res.output, g[key], key)
            st = res.stats
            assert [st["supersteps"], st["messages_sent"], st["messages_delivered"], st["words_sent"],
                    st["words_delivered"]] == g[f"prstats/{radix}/{p}/{k}"].tolist(), key
        elif parts[0] == "net":
            net = 0 if parts[1] == "btn" else 1
            p, s = int(parts[2]), int(parts[3])
            inp = g["in/net"]
            out, st = bsg.netsort.block_network_batched(inp.reshape(1, -1), p, net, s)
            exp = g[key]
            np.testing.assert_array_equal(out.reshape(-1)[:exp.size], exp, key)
            assert [st["supersteps"], st["messages_sent"], st["messages_delivered"], st["words_sent"],
                    st["words_delivered"]] == g[f"netstats/{parts[1]}/{p}/{s}"].tolist(), key
        elif parts[0] == "ms" and parts[2] == "a":
            i = parts[1]
            lo, hi = bsg.netsort.merge_split(g[f"ms/{i}/a"], g[f"ms/{i}/b"])
            np.testing.assert_array_equal(lo, g[f"ms/{i}/low"])
            np.testing.assert_array_equal(hi, g[f"ms/{i}/high"])
        else:
            continue
        checked += 1
    assert checked > 400
