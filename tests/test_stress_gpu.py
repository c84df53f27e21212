"""Stress tests standing in for compute-sanitizer racecheck/synccheck, which
the GPU pool does not allow (the memory-order argument is in
DESIGN.md §5).  A race in the decoupled look-back (relaxed flag+count words),
the TMA/mbarrier double buffer, the fused small-n kernel's grid barriers or
the register network's shared-memory exchanges shows up as a wrong or
non-deterministic result somewhere in a sweep of seeds, sizes (tile counts,
ragged last tiles), every one-sweep configuration row, skewed inputs (the
rank-first branch) and repeated runs of the same input: every result here is
compared bit for bit with torch.sort of the same keys on the device."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dev_sort_ref(torch, t):
    return torch.sort(t.view(torch.int32).to(torch.int64) & 0xFFFFFFFF).values


def _sort(bsg, torch, t, radix_log2=8):
    L = bsg._lib.lib()
    ctx = bsg._lib.context(0)
    out = torch.empty_like(t)
    bsg._lib.check(L.bsg_radix_sort_u32(ctx.handle, t.data_ptr(), out.data_ptr(), t.numel(), radix_log2, 1,
                                        torch.cuda.current_stream().cuda_stream))
    return out


def _eq(torch, out, ref):
    return bool(torch.equal(out.view(torch.int32).to(torch.int64) & 0xFFFFFFFF, ref))


def test_onesweep_every_config_many_seeds(cuda, bsg):
    torch = cuda
    L = bsg._lib.lib()
    rng = np.random.default_rng(2024)
    prev_small = L.bsg_debug_set_small_sort(0)
    try:
        for cfg in (0, 1, 2, 3, 4, 5, 6, 7):
            prev = L.bsg_debug_set_onesweep_cfg(cfg)
            try:
                for _ in range(24):
                    n = int(rng.integers(1, 1 << 23))
                    t = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device="cuda",
                                      generator=torch.Generator("cuda").manual_seed(int(rng.integers(1 << 30))))
                    if rng.random() < 0.3:  # skewed: narrow high bytes -> identity / rank-first passes
                        t &= int(rng.choice([0xFF, 0xFFFF, 0x0F0F0F0F, 0x7]))
                    assert _eq(torch, _sort(bsg, torch, t), _dev_sort_ref(torch, t)), (cfg, n)
            finally:
                L.bsg_debug_set_onesweep_cfg(prev)
    finally:
        L.bsg_debug_set_small_sort(prev_small)


def test_repeated_runs_are_identical(cuda, bsg):
    """The same input sorted 100 times (full size, fused small-n and multi-CTA
    look-back chains): any race would make some run differ."""
    torch = cuda
    for n in ((1 << 24) + 17, (1 << 20) + 5, 99991):
        t = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device="cuda",
                          generator=torch.Generator("cuda").manual_seed(n))
        ref = _dev_sort_ref(torch, t)
        first = _sort(bsg, torch, t)
        assert _eq(torch, first, ref)
        for _ in range(100):
            assert torch.equal(_sort(bsg, torch, t), first)


def test_zipf_and_equal_keys_repeated(cuda, bsg):
    """Heavy digits drive the rank-first branch and long look-back waits."""
    torch = cuda
    rng = np.random.default_rng(7)
    z = np.minimum(rng.zipf(1.1, 1 << 22), 1 << 31).astype(np.uint32) * np.uint32(2654435761)
    for keys in (z, np.full(1 << 22, 123456789, np.uint32), np.zeros(3000001, np.uint32)):
        t = torch.from_numpy(keys.view(np.int32)).cuda()
        ref = _dev_sort_ref(torch, t)
        for _ in range(5):
            assert _eq(torch, _sort(bsg, torch, t), ref)
        assert _eq(torch, _sort(bsg, torch, t, 16), ref)


def test_parallel_radix_many_worker_counts(cuda, bsg):
    torch = cuda
    L = bsg._lib.lib()
    ctx = bsg._lib.context(0)
    rng = np.random.default_rng(99)
    for _ in range(40):
        n = int(rng.integers(1000, 1 << 22))
        p = int(rng.integers(1, 65))
        bits = int(rng.choice([8, 16]))
        t = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device="cuda",
                          generator=torch.Generator("cuda").manual_seed(n + p))
        out = torch.empty_like(t)
        bsg._lib.check(L.bsg_parallel_radix_sort_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, p, bits, -1, None,
                                                     1, torch.cuda.current_stream().cuda_stream))
        assert _eq(torch, out, _dev_sort_ref(torch, t)), (n, p, bits)


def test_register_networks_repeated(cuda, bsg):
    """Every power-of-two block length of the register network (in-thread,
    in-warp shuffle, layout-B transposes, cross-warp exchanges), repeated."""
    torch = cuda
    L = bsg._lib.lib()
    ctx = bsg._lib.context(0)
    st = torch.cuda.current_stream().cuda_stream
    for ln, p in ((256, 16), (512, 2), (1024, 2), (2048, 4), (4096, 8), (8192, 2), (16384, 2), (16384, 8)):
        num = max(16, (1 << 22) // ln)
        t = torch.randint(-2**31, 2**31 - 1, (num * ln,), dtype=torch.int32, device="cuda",
                          generator=torch.Generator("cuda").manual_seed(ln + p))
        ref = torch.sort(t.view(torch.int32).to(torch.int64).view(num, ln) & 0xFFFFFFFF, dim=1).values
        for net in (0, 1):
            first = None
            for _ in range(4):
                out = torch.empty_like(t)
                bsg._lib.check(L.bsg_block_network_batched_u32(ctx.handle, net, t.data_ptr(), out.data_ptr(), num,
                                                               ln, p, -1, None, 1, st))
                got = out.view(torch.int32).to(torch.int64).view(num, ln) & 0xFFFFFFFF
                assert torch.equal(got, ref), (ln, p, net)


def test_full_sort_routes_agree_on_random_inputs(cuda, bsg):
    """Every route a full sort may take -- strictly stable passes, K3f for pass
    0, value-stable passes, the hybrid MSD route (forced) -- over random sizes
    and key shapes that move the runs of equal low bits around (uniform, few
    distinct keys, few distinct low/high halves, long constant runs, sorted,
    byte-wise low entropy): all results equal torch.sort of the same keys."""
    torch = cuda
    L = bsg._lib.lib()
    rng = np.random.default_rng(77)
    g = torch.Generator(device="cuda").manual_seed(5)
    prev = (L.bsg_debug_set_small_sort(0), L.bsg_debug_set_first_pass(-1), L.bsg_debug_set_relaxed_passes(-1),
            L.bsg_debug_set_msd(-1))

    def make(kind, n):
        u = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device="cuda", generator=g)
        if kind == 0:
            return u
        if kind == 1:  # few distinct keys
            return u[torch.randint(0, max(1, min(n, 37)), (n,), device="cuda", generator=g)]
        if kind == 2:  # few distinct low halves
            return (u & -65536) | (u & 0x0003)
        if kind == 3:  # few distinct high halves, random low bits
            return (u & 0xFFFF) | ((u >> 30) << 16)
        if kind == 4:  # long constant runs
            return torch.repeat_interleave(u[: max(1, n // 1000)], 1000)[:n].contiguous() if n >= 1000 else u
        if kind == 5:  # already sorted
            return torch.sort(u)[0]
        return u & 0x03030303  # byte-wise low entropy

    try:
        sizes = [int(x) for x in rng.integers(1, 1 << 25, 10)] + [(1 << 24) + 1, (1 << 25) + 4097]
        for i, n in enumerate(sizes):
            t = make(i % 7, n)
            n = t.numel()
            ref = _dev_sort_ref(torch, t)
            for first, relaxed, msd in ((0, 0, 1), (1, 0, 1), (1, 1, 1), (1, 1, 2)):
                L.bsg_debug_set_first_pass(first)
                L.bsg_debug_set_relaxed_passes(relaxed)
                L.bsg_debug_set_msd(msd)
                assert _eq(torch, _sort(bsg, torch, t), ref), (n, i % 7, first, relaxed, msd)
            del t, ref
    finally:
        L.bsg_debug_set_small_sort(prev[0])
        L.bsg_debug_set_first_pass(prev[1])
        L.bsg_debug_set_relaxed_passes(prev[2])
        L.bsg_debug_set_msd(prev[3])
