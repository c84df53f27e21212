"""Multi-GPU parallel radix sort (PR4 at r = 2^8, PR2 at r = 2^16): one
process per GPU, the reference's BSP supersteps re-expressed over NCCL.

Reference: run_parallel_radix (radix.hpp:260-303).  Per round, on every rank:

  superstep 2k     count_digits(block) (radix.hpp:127-132)          -> kernel
                   send the r counts to every worker (radix.hpp:275-277)
                                                  -> NCCL all_gather (p x r)
  superstep 2k+1   sort_and_scatter (radix.hpp:151-179): local stable pass
                   -> kernel; the routing plan from the count matrix
                   -> kernel; contiguous slices to their owners
                                                  -> NCCL all_to_all_v
  superstep 2k+2   gather_slices (radix.hpp:184-222) -> rebuild kernel

The block a rank holds after round k is bit-identical to worker `rank`'s
block in run_parallel_radix with plan.rounds = k.  The only host round trip
per round is the 2p split sizes NCCL's all-to-all-v needs on the host.

With ``exchange="peer"`` the all-to-all-v and the rebuild
are one kernel: every rank maps the next-round blocks of all ranks into its
address space (CUDA IPC, NVLink) and stores each key of its sorted block
straight at its final position in the owner's block; a barrier (a 1-element
NCCL all-reduce) closes the round.  No send/receive buffers, no host round
trip for split sizes.

`parallel_radix_sort_single_exchange` is variant B of SURVEY §8(e) (the
BASELINE config-5 formulation: one exchange, then a local sort).

The step operations are injectable (``ops``) so the host orchestration can
be exercised on CPU under gloo in tests; the product default is
:class:`CudaStepOps`, which fails loudly without libbsg.so / a GPU.
"""
from __future__ import annotations

import ctypes
from typing import List, Optional, Tuple

import torch
import torch.distributed as dist

from . import _lib
from .radix import checked_digit_bits


def partition_size_of(n: int, p: int, w: int) -> int:
    return int(_lib.lib().bsg_partition_size_of(n, p, w))


def partition_offset_of(n: int, p: int, w: int) -> int:
    return int(_lib.lib().bsg_partition_offset_of(n, p, w))


class CudaStepOps:
    """The per-worker PR steps as sm_100a kernels (C ABI, device memory)."""

    def __init__(self, device: torch.device):
        self.device = device
        self.ctx = _lib.context(device.index or 0)
        self.L = _lib.lib()

    def _stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def keys(self, n: int) -> torch.Tensor:
        return torch.empty(n, dtype=torch.int32, device=self.device)

    def count(self, block: torch.Tensor, rnd: int, bits: int) -> torch.Tensor:
        counts = torch.empty(1 << bits, dtype=torch.int64, device=self.device)
        _lib.check(self.L.bsg_pr_count_digits(self.ctx.handle, block.data_ptr(), block.numel(), rnd, bits,
                                              counts.data_ptr(), self._stream()), "pr count_digits")
        return counts

    def local_sort(self, block: torch.Tensor, rnd: int, bits: int) -> torch.Tensor:
        out = torch.empty_like(block)
        _lib.check(self.L.bsg_pr_local_sort(self.ctx.handle, block.data_ptr(), out.data_ptr(), block.numel(), rnd,
                                            bits, self._stream()), "pr local sort")
        return out

    def plan(self, counts_all: torch.Tensor, n: int, p: int, me: int, rnd: int, bits: int):
        sr = torch.empty(2 * p, dtype=torch.int64, device=self.device)
        delta = torch.empty(p << bits, dtype=torch.int64, device=self.device)
        _lib.check(self.L.bsg_pr_plan(self.ctx.handle, counts_all.data_ptr(), n, p, me, rnd, bits, sr.data_ptr(),
                                      sr[p:].data_ptr(), delta.data_ptr(), self._stream()), "pr plan")
        host = sr.cpu().tolist()  # the one host round trip per round: split sizes
        return host[:p], host[p:], sr[p:], delta

    def sort(self, keys: torch.Tensor) -> torch.Tensor:
        """Full LSD sort (serial_radix_sort) of a device block."""
        out = torch.empty_like(keys)
        _lib.check(self.L.bsg_radix_sort_u32(self.ctx.handle, keys.data_ptr(), out.data_ptr(), keys.numel(), 8,
                                             _lib.MEM_DEVICE, self._stream()), "local sort")
        return out

    def peer_scatter(self, sorted_: torch.Tensor, counts_all: torch.Tensor, n: int, p: int, me: int, rnd: int,
                     bits: int, peer_ptrs) -> None:
        arr = (ctypes.c_void_p * p)(*peer_ptrs)
        _lib.check(self.L.bsg_pr_peer_scatter(self.ctx.handle, sorted_.data_ptr(), sorted_.numel(),
                                              counts_all.data_ptr(), n, p, me, rnd, bits, arr, self._stream()),
                   "pr peer scatter")

    def fused_round(self, block: torch.Tensor, counts_all: torch.Tensor, n: int, p: int, me: int, rnd: int,
                    bits: int, peer_ptrs) -> None:
        """Local stable pass + exchange + rebuild as one pass (r <= 2^8)."""
        arr = (ctypes.c_void_p * p)(*peer_ptrs)
        _lib.check(self.L.bsg_pr_fused_round(self.ctx.handle, block.data_ptr(), block.numel(), counts_all.data_ptr(),
                                             n, p, me, rnd, bits, arr, self._stream()), "pr fused round")

    def rebuild(self, recv: torch.Tensor, recv_counts_dev: torch.Tensor, p: int, rnd: int, bits: int,
                delta: torch.Tensor, out_len: int) -> torch.Tensor:
        block = torch.empty(out_len, dtype=torch.int32, device=self.device)
        _lib.check(self.L.bsg_pr_rebuild(self.ctx.handle, recv.data_ptr(), recv.numel(), recv_counts_dev.data_ptr(),
                                         p, rnd, bits, delta.data_ptr(), block.data_ptr(), self._stream()),
                   "pr rebuild")
        return block


class PeerBlocks:
    """Two ping-pong next-round blocks per rank, mapped into every rank
    (CUDA IPC handles exchanged with all_gather_object; torch's own
    reduce_tensor/rebuild carries the allocation offset).  Round k's peer
    scatter writes buffer k % 2 of every owner; the owner last read that
    buffer in round k - 1, which the previous round's barrier closed."""

    def __init__(self, n_total: int, group=None, device: Optional[torch.device] = None):
        from torch.multiprocessing.reductions import reduce_tensor

        self.p = dist.get_world_size(group)
        self.me = dist.get_rank(group)
        self.n_total = n_total
        self.group = group
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        size = partition_size_of(n_total, self.p, self.me)
        self.size = size
        self.local = [torch.empty(max(size, 1), dtype=torch.int32, device=self.device) for _ in range(2)]
        gathered: List = [None] * self.p
        if self.p > 1:
            # kernels on this device store into blocks that live on the other
            # ranks' devices: enable peer access (NVLink) from this device
            ctx = _lib.context(self.device.index or 0)
            _lib.check(_lib.lib().bsg_ctx_enable_peer_access(ctx.handle, None), "enable peer access")
        if self.p > 1:  # nothing to map for a single rank
            mine = [reduce_tensor(t) for t in self.local]
            dist.all_gather_object(gathered, mine, group=group)
        self.mapped = [[None] * self.p for _ in range(2)]
        for w in range(self.p):
            for b in range(2):
                if w == self.me:
                    self.mapped[b][w] = self.local[b]
                else:
                    fn, args = gathered[w][b]
                    self.mapped[b][w] = fn(*args)
        self.ptrs = [[t.data_ptr() for t in self.mapped[b]] for b in range(2)]
        self._token = torch.zeros(1, dtype=torch.float32, device=self.device)

    def barrier(self) -> None:
        """Round barrier: every rank's scatter kernel has completed (and fenced
        its peer stores) before any rank continues.  NCCL: a 1-element
        all-reduce ordered on the device stream; other backends (gloo, e.g.
        two processes sharing one GPU in tests): host sync + barrier."""
        if _is_nccl(self.group):
            dist.all_reduce(self._token, group=self.group)
        else:
            torch.cuda.synchronize(self.device)
            dist.barrier(group=self.group)


def _is_nccl(group) -> bool:
    return dist.get_backend(group) == "nccl"


def _all_gather_counts(counts: torch.Tensor, p: int, group) -> torch.Tensor:
    """The count exchange of radix.hpp:275-277 as one all-gather (device
    buffers with NCCL; host-staged with other backends)."""
    if _is_nccl(group) or not counts.is_cuda:
        out = torch.empty(p * counts.numel(), dtype=counts.dtype, device=counts.device)
        dist.all_gather_into_tensor(out, counts, group=group)
        return out
    host = counts.cpu()
    parts = [torch.empty_like(host) for _ in range(p)]
    dist.all_gather(parts, host, group=group)
    return torch.cat(parts).to(counts.device)


def parallel_radix_sort(block: torch.Tensor, n_total: int, radix: int = 256, rounds: Optional[int] = None,
                        group=None, ops=None, a2a_events: Optional[list] = None, exchange: str = "nccl",
                        peer: Optional[PeerBlocks] = None, count_events: Optional[list] = None) -> torch.Tensor:
    """Sorts the globally block-distributed array (rank w holds the keys at
    Partition(n_total, p).offset_of(w) .. +size_of(w), radix.hpp:96-118).
    Returns this rank's block of the sorted array (int32 bit patterns of the
    uint32 keys).  `rounds` < 32/lg r stops early (plan.rounds override).
    If `a2a_events` is a list, CUDA event pairs around each all-to-all are
    appended to it (NVLink share of the step); with exchange="peer" they
    bracket the fused pass + round barrier.  `count_events` likewise brackets
    each round's digit count + count all-gather."""
    bits = checked_digit_bits(radix)
    p = dist.get_world_size(group)
    me = dist.get_rank(group)
    if block.dtype == torch.uint32:
        block = block.view(torch.int32)
    if block.numel() != partition_size_of(n_total, p, me):
        raise ValueError(f"rank {me} holds {block.numel()} keys; Partition({n_total}, {p}) expects "
                         f"{partition_size_of(n_total, p, me)}")
    if ops is None:
        ops = CudaStepOps(block.device)
    all_rounds = 32 // bits
    rounds = all_rounds if rounds is None else max(0, min(int(rounds), all_rounds))
    if exchange == "peer":
        return _parallel_radix_sort_peer(block, n_total, bits, rounds, group, ops, a2a_events, peer, count_events)
    if exchange != "nccl":
        raise ValueError(f"exchange must be 'nccl' or 'peer', not {exchange!r}")
    for rnd in range(rounds):
        c0 = _event(count_events, block)
        counts = ops.count(block, rnd, bits)
        counts_all = torch.empty(p * counts.numel(), dtype=counts.dtype, device=counts.device)
        dist.all_gather_into_tensor(counts_all, counts, group=group)
        _close(count_events, c0)
        sorted_ = ops.local_sort(block, rnd, bits)
        send, recv, recv_dev, delta = ops.plan(counts_all, n_total, p, me, rnd, bits)
        _check_exchange(send, recv, block.numel(), partition_size_of(n_total, p, me), me, rnd)
        recv_buf = ops.keys(sum(recv))
        if a2a_events is not None and block.is_cuda:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        dist.all_to_all_single(recv_buf, sorted_, output_split_sizes=recv, input_split_sizes=send, group=group)
        if a2a_events is not None and block.is_cuda:
            e1.record()
            a2a_events.append((e0, e1))
        block = ops.rebuild(recv_buf, recv_dev, p, rnd, bits, delta, partition_size_of(n_total, p, me))
    return block


def _check_exchange(send, recv, block_len: int, want_len, me: int, rnd: int) -> None:
    """bsp_error equivalents (radix.hpp:207-220, 283-286): this rank sends
    every key of its block exactly once and, in PR, receives exactly its
    partition's size -- before any byte moves."""
    if sum(send) != block_len:
        raise _lib.BspError(f"worker {me}, round {rnd}: send counts sum to {sum(send)}, block has {block_len} keys")
    if want_len is not None and sum(recv) != want_len:
        raise _lib.BspError(f"worker {me}, round {rnd}: receive counts sum to {sum(recv)}, "
                            f"expected {want_len} keys")


def _event(lst, block):
    if lst is None or not block.is_cuda:
        return None
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def _close(lst, e0):
    if e0 is not None:
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        lst.append((e0, e1))


def _parallel_radix_sort_peer(block, n_total, bits, rounds, group, ops, a2a_events, peer, count_events=None):
    p = dist.get_world_size(group)
    me = dist.get_rank(group)
    if peer is None:
        peer = PeerBlocks(n_total, group, block.device)
    if peer.n_total != n_total or peer.p != p:
        raise ValueError("PeerBlocks were mapped for a different (n, p)")
    size = partition_size_of(n_total, p, me)
    for rnd in range(rounds):
        c0 = _event(count_events, block)
        counts = ops.count(block, rnd, bits)
        counts_all = _all_gather_counts(counts, p, group)
        _close(count_events, c0)
        b = rnd % 2
        if a2a_events is not None and block.is_cuda:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        # the round's local pass stores straight into the owners' blocks
        ops.fused_round(block, counts_all, n_total, p, me, rnd, bits, peer.ptrs[b])
        peer.barrier()
        if a2a_events is not None and block.is_cuda:
            e1.record()
            a2a_events.append((e0, e1))
        block = peer.local[b][:size]
    return block.clone()


def digit_cuts(global_counts, p: int):
    """Balanced cut points at top-digit boundaries: rank w receives the keys
    whose top digit lies in [cuts[w], cuts[w+1]).  Deterministic on every rank
    (computed from the same all-gathered counts)."""
    total = int(sum(global_counts))
    cuts = [0]
    run = 0
    d = 0
    r = len(global_counts)
    for w in range(1, p):
        target = (total * w + p - 1) // p  # ceil(total*w/p): first w ranks hold >= w/p of the keys
        while d < r and run < target:
            run += int(global_counts[d])
            d += 1
        cuts.append(d)
    cuts.append(r)
    return cuts


def parallel_radix_sort_single_exchange(block: torch.Tensor, group=None, ops=None,
                                        a2a_events: Optional[list] = None) -> torch.Tensor:
    """Variant B: the BASELINE config-5 formulation -- local
    histogram of the top 8-bit digit, all-gather of the count vectors, one
    stable local partition by that digit (count_sort_round round 3, r=2^8),
    ONE all-to-all-v over NVLink, then a full local LSD sort of the received
    keys.  Cuts fall on digit boundaries, so per-rank sizes vary by at most one
    bucket; the concatenation of the ranks' outputs in rank order is the sorted
    array (identical to run_parallel_radix's output).  Returns this rank's
    sorted keys (int32 bit patterns)."""
    p = dist.get_world_size(group)
    me = dist.get_rank(group)
    if block.dtype == torch.uint32:
        block = block.view(torch.int32)
    if ops is None:
        ops = CudaStepOps(block.device)
    counts = ops.count(block, 3, 8)                                   # top digit, r = 2^8
    counts_all = torch.empty(p * counts.numel(), dtype=counts.dtype, device=counts.device)
    dist.all_gather_into_tensor(counts_all, counts, group=group)
    cm = counts_all.view(p, -1).cpu()                                 # p x 256 (2 KiB per rank)
    cuts = digit_cuts(cm.sum(0).tolist(), p)
    part = ops.local_sort(block, 3, 8)                                # stable partition by the top digit
    mine = cm[me]
    send = [int(mine[cuts[w]:cuts[w + 1]].sum()) for w in range(p)]
    recv = [int(cm[v, cuts[me]:cuts[me + 1]].sum()) for v in range(p)]
    _check_exchange(send, recv, block.numel(), None, me, 0)
    recv_buf = ops.keys(sum(recv))
    if a2a_events is not None and block.is_cuda:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
    dist.all_to_all_single(recv_buf, part, output_split_sizes=recv, input_split_sizes=send, group=group)
    if a2a_events is not None and block.is_cuda:
        e1.record()
        a2a_events.append((e0, e1))
    return ops.sort(recv_buf)


def network_schedule(network: int, p: int):
    """(partner, keep_low) per stage for this p (netsort.hpp:70-108)."""
    S = ctypes.c_int(0)
    L = _lib.lib()
    _lib.check(L.bsg_network_schedule(network, p, None, None, 0, ctypes.byref(S)), "schedule")
    import numpy as np

    partner = np.empty(max(1, S.value * p), dtype=np.int32)
    keep = np.empty(max(1, S.value * p), dtype=np.int32)
    _lib.check(L.bsg_network_schedule(network, p, partner.ctypes.data, keep.ctypes.data, S.value, ctypes.byref(S)),
               "schedule")
    return [[(int(partner[s * p + i]), bool(keep[s * p + i])) for i in range(p)] for s in range(S.value)]


class CudaNetworkOps(CudaStepOps):
    """merge_split on device blocks (netsort.hpp:30-51)."""

    def merge_keep(self, mine: torch.Tensor, theirs: torch.Tensor, keep_low: bool) -> torch.Tensor:
        low = torch.empty_like(mine)
        high = torch.empty_like(theirs)
        _lib.check(self.L.bsg_merge_split_u32(self.ctx.handle, mine.data_ptr(), mine.numel(), theirs.data_ptr(),
                                              theirs.numel(), low.data_ptr(), high.data_ptr(), _lib.MEM_DEVICE,
                                              self._stream()), "merge_split")
        return low if keep_low else high


def block_network_sort(block: torch.Tensor, network: int = 0, stages: Optional[int] = None, group=None,
                       ops=None) -> torch.Tensor:
    """The paper's p-processor BTN (network 0) / OET (network 1) across ranks
    (netsort.hpp:157-199 with one worker per GPU): the rank's
    block (equal sizes on every rank, padded by the caller with 0xFFFFFFFF as
    prepare_blocks does, netsort.hpp:124-141) is sorted locally, then every
    stage swaps whole blocks with the stage partner over NCCL and keeps the low
    or high half of the merge (merge_split).  `stages` < S stops early.
    Returns the rank's final block; the blocks in rank order are sorted."""
    p = dist.get_world_size(group)
    me = dist.get_rank(group)
    if block.dtype == torch.uint32:
        block = block.view(torch.int32)
    if ops is None:
        ops = CudaNetworkOps(block.device)
    sched = network_schedule(network, p)
    run = len(sched) if stages is None else max(0, min(int(stages), len(sched)))
    state = ops.sort(block)                       # superstep 0: local sort (netsort.hpp:167)
    for s in range(run):
        q, keep_low = sched[s][me]
        if q < 0:                                 # idle OET edge worker
            continue
        other = torch.empty_like(state)
        if p > 1:
            # NCCL moves device blocks peer to peer; gloo has no device
            # point-to-point, so CUDA blocks are staged through host memory
            stage = state.is_cuda and not _is_nccl(group)
            snd = state.cpu() if stage else state
            rcv = torch.empty_like(snd)
            reqs = dist.batch_isend_irecv([dist.P2POp(dist.isend, snd, q, group),
                                           dist.P2POp(dist.irecv, rcv, q, group)])
            for r in reqs:
                r.wait()
            other = rcv.to(state.device) if stage else rcv
        state = ops.merge_keep(state, other, keep_low)
    return state
