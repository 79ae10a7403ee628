"""Multi-GPU plumbing (one process per GPU, torch.distributed).

* `sharded_space_argmin`: the configuration index space shards across ranks
  with no data-path collective; the winner is one all-reduce(MIN) of the
  packed int64 key ((time << 33) | index < 2^63, so signed MIN is exact).
* `partitioned_explore`: hash-partitioned frontier exploration.  Rank r owns
  the states whose fingerprint % world == r; each round every rank expands
  its local frontier, buckets the successors by owner and exchanges them with
  one all_to_all, then inserts what it owns into its visited set.  The sweep
  ends when no rank discovered a new state (all-reduce SUM == 0).

The evaluators are injected so the same exchange logic runs over NCCL with
the GPU kernels and over gloo with CPU checkers in tests/test_distributed.py.

* `explore_multi_gpu`: the GPU sweep across ranks.  Each rank's exploration
  kernel owns one hash partition of the visited set and inserts successors
  owned by other ranks directly into their tables and queues over peer memory
  (NVLink, CUDA IPC handles exchanged here); there is no host round trip per
  frontier.  The host only exchanges the handles and reduces the statistics.
"""
from __future__ import annotations

from typing import Callable, Hashable, Iterable, List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist

KEY_INDEX_BITS = 33
KEY_SAT = (1 << 30) - 1


def shard(total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous index range [first, first+count) of `rank` (balanced to +-1)."""
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def sharded_space_argmin(total: int, local_argmin: Callable[[int, int], int],
                         group=None, device: str = "cpu",
                         local_exact: Optional[Callable[[int, int], Tuple[int, int]]] = None
                         ) -> Tuple[int, int, int]:
    """Global (key, time, index) of a space of `total` configurations.
    local_argmin(first, count) -> packed key of the rank's shard (2^63 = none).
    The key's time field saturates at KEY_SAT; when the reduced key is saturated
    every configuration has time >= KEY_SAT, and the winner is resolved exactly
    with local_exact(first, count) -> (least time or -1, least index with it):
    all-reduce(MIN) of the time, then all-reduce(MIN) of the index among the ranks
    holding that time (search.cpp:67-78's tie rule across shards)."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    first, count = shard(total, rank, world)
    key = local_argmin(first, count) if count else (1 << 63) - 1
    t = torch.tensor([min(key, (1 << 63) - 1)], dtype=torch.int64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    k = int(t.item())
    if k >= (1 << 63) - 1 or (k >> KEY_INDEX_BITS) < KEY_SAT:
        return k, k >> KEY_INDEX_BITS, k & ((1 << KEY_INDEX_BITS) - 1)
    if local_exact is None:
        raise ValueError("saturated argmin key: pass local_exact to resolve it")
    none = (1 << 63) - 1
    et, ei = local_exact(first, count) if count else (-1, none)
    v = torch.tensor([et if et >= 0 else none], dtype=torch.int64, device=device)
    if world > 1:
        dist.all_reduce(v, op=dist.ReduceOp.MIN, group=group)
    tmin = int(v.item())
    if tmin == none:
        return none, -1, none
    w = torch.tensor([ei if et == tmin else none], dtype=torch.int64, device=device)
    if world > 1:
        dist.all_reduce(w, op=dist.ReduceOp.MIN, group=group)
    idx = int(w.item())
    return (KEY_SAT << KEY_INDEX_BITS) | idx, tmin, idx


def owner(fingerprint: int, world: int) -> int:
    return fingerprint % world


def partitioned_explore(initial: Iterable[Tuple[int, Hashable]],
                        expand: Callable[[Hashable], Sequence[Tuple[int, Hashable]]],
                        encode: Callable[[Hashable], List[int]],
                        decode: Callable[[List[int]], Hashable],
                        width: int, group=None) -> Tuple[int, int]:
    """Counts the states reachable from `initial` with hash-partitioned ownership.

    initial / expand yield (fingerprint, state); encode/decode map a state to a
    fixed-width list of ints (the packed words) for the exchange.  Returns
    (states owned by this rank, global state count)."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    visited = set()
    frontier = []
    for fp, s in initial:
        if owner(fp, world) == rank and s not in visited:
            visited.add(s)
            frontier.append(s)
    while True:
        buckets: List[List[int]] = [[] for _ in range(world)]
        for s in frontier:
            for fp, succ in expand(s):
                buckets[owner(fp, world)].extend([fp & ((1 << 63) - 1)] + encode(succ))
        # exchange sizes, then payloads (one all_to_all each)
        send_counts = torch.tensor([len(b) for b in buckets], dtype=torch.int64)
        recv_counts = torch.empty(world, dtype=torch.int64)
        if world > 1:
            dist.all_to_all_single(recv_counts, send_counts, group=group)
        else:
            recv_counts.copy_(send_counts)
        send = torch.tensor([v for b in buckets for v in b], dtype=torch.int64)
        recv = torch.empty(int(recv_counts.sum()), dtype=torch.int64)
        if world > 1:
            dist.all_to_all_single(recv, send, output_split_sizes=recv_counts.tolist(),
                                   input_split_sizes=send_counts.tolist(), group=group)
        else:
            recv = send
        vals = recv.tolist()
        frontier = []
        rec = 1 + width
        for i in range(0, len(vals), rec):
            s = decode(vals[i + 1:i + rec])
            if s not in visited:
                visited.add(s)
                frontier.append(s)
        new = torch.tensor([len(frontier)], dtype=torch.int64)
        if world > 1:
            dist.all_reduce(new, op=dist.ReduceOp.SUM, group=group)
        if int(new.item()) == 0:
            break
    total = torch.tensor([len(visited)], dtype=torch.int64)
    if world > 1:
        dist.all_reduce(total, op=dist.ReduceOp.SUM, group=group)
    return len(visited), int(total.item())


def explore_multi_gpu(platform, problem, configs, max_states: int = 5_000_000,
                      check_invariants: bool = False, group=None):
    """explore_configs over all ranks of the process group (one GPU per rank): the
    same ExploreStats on every rank.  Rank r's device must be the current CUDA
    device (torch.cuda.set_device(local_rank))."""
    import ctypes as C

    from ._lib import check, i32arr, lib
    from .explore import ExploreStats, SweepInfo

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    n = len(configs)
    cfg = i32arr([v for c in configs for v in (c.wg, c.ts)])
    ctx = C.c_void_p()
    handle = C.create_string_buffer(64)
    check(lib.mctb_explore_mp_open(platform.as_array(), problem.size, problem.kernel,
                                   problem.input_array(), cfg, n, max_states, world, rank,
                                   1 if check_invariants else 0, C.byref(ctx), handle))
    try:
        handles = [bytes(handle.raw)]
        if world > 1:
            handles = [None] * world
            dist.all_gather_object(handles, bytes(handle.raw), group=group)
        check(lib.mctb_explore_mp_connect(ctx, b"".join(handles)))
        if world > 1:
            dist.barrier(group=group)
        if rank == 0:
            check(lib.mctb_explore_mp_seed(ctx))
        if world > 1:
            dist.barrier(group=group)
        out = (C.c_int64 * (8 * n))()
        info = (C.c_int64 * 4)()
        rc = lib.mctb_explore_mp_run(ctx, out, info)
        mine = (rc, list(out), list(info))
        parts = [mine]
        if world > 1:
            parts = [None] * world
            dist.all_gather_object(parts, mine, group=group)
            dist.barrier(group=group)  # no rank unmaps memory a peer's kernel still reads
    finally:
        lib.mctb_explore_mp_close(ctx)
    for rc_r, _, _ in parts:
        check(rc_r)
    res = []
    for k in range(n):
        rows = [p[1][8 * k:8 * k + 8] for p in parts]
        states = sum(r[0] for r in rows)
        terminals = sum(r[2] for r in rows)
        mn = min(r[3] for r in rows)
        mx = max(r[4] for r in rows)
        complete = states < max_states
        res.append(ExploreStats(
            complete, min(states, max_states), sum(r[1] for r in rows),
            rows[0][7] + mx if terminals else -1, mn if terminals else -1,
            mx if terminals else -1, terminals, sum(r[5] for r in rows), sum(r[6] for r in rows)))
    kern_us = max(p[2][2] for p in parts)
    return res, SweepInfo(parts[0][2][0], sum(r.states_visited for r in res), parts[0][2][1],
                          kern_us)
