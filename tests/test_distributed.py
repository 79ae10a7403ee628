"""Multi-rank logic on CPU with gloo, world size 2 (the GPU data path is the
same code with NCCL)."""
import ctypes as C
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_lib():
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from checkers import Oracle
    o = Oracle()
    o.lib.mo_successors.restype = C.c_int64
    return o


def _successors(o, plat, size, kernel, wg, ts, ser):
    cap = 256
    rec = C.c_int64()
    buf = C.create_string_buffer(cap * 4096)
    fps = (C.c_uint64 * cap)()
    n = o.lib.mo_successors((C.c_int * 4)(*plat), size, kernel, None, wg, ts, ser, buf, cap, fps,
                            C.byref(rec))
    assert n >= 0
    L = rec.value
    return [(fps[i], bytes(buf.raw[i * L:(i + 1) * L])) for i in range(n)], L


CASES = [((1, 1, 4, 4), 8, 0, 4, 4), ((2, 1, 2, 4), 8, 0, 2, 2), ((1, 1, 4, 4), 8, 1, 4, 2)]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2305_09130_b200 import distributed as D
    o = _oracle_lib()
    # 1) sharded argmin of a generalised space, oracle as the per-rank evaluator
    sd = [0, 1 << 12, 3, 1, 40, 1, 9, 0, 4, 1, 11, 1, 11]
    total = 40 * 9 * 5 * 11 * 11

    def local(first, count):
        return o.space_argmin(sd, first, count)[0]
    key, t, idx = D.sharded_space_argmin(total, local)
    # 1b) a space whose every time saturates the key: the exact resolution across ranks
    sd2 = [0, 1 << 24, 100, 1, 3, 1, 2, 0, 2, 1, 23, 1, 23]

    def local2(first, count, sd2=sd2):
        return o.space_argmin(sd2, first, count)[0]

    def exact2(first, count, sd2=sd2):
        r = o.space_argmin(sd2, first, count)
        return r[1], r[2]
    sat = D.sharded_space_argmin(3 * 2 * 3 * 23 * 23, local2, local_exact=exact2)
    # 2) hash-partitioned exploration of real model state spaces (reference fingerprints)
    counts = []
    for plat, size, kernel, wg, ts in CASES:
        init, L = _successors(o, plat, size, kernel, wg, ts, None)

        def expand(s, plat=plat, size=size, kernel=kernel, wg=wg, ts=ts):
            return _successors(o, plat, size, kernel, wg, ts, s)[0]

        def encode(s, L=L):
            return [int.from_bytes(s[i:i + 4].ljust(4, b"\0"), "little") for i in range(0, L, 4)]

        def decode(v, L=L):
            return b"".join(x.to_bytes(4, "little") for x in v)[:L]

        mine, tot = D.partitioned_explore(init, expand, encode, decode, (L + 3) // 4)
        counts.append((mine, tot))
    q.put((rank, key, t, idx, counts, sat))
    dist.destroy_process_group()


def test_two_rank_argmin_and_partitioned_exploration(oracle):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, k0, t0, i0, c0, s0), (_, k1, t1, i1, c1, s1) = res
    sd = [0, 1 << 12, 3, 1, 40, 1, 9, 0, 4, 1, 11, 1, 11]
    key, t, idx = oracle.space_argmin(sd, 0, 40 * 9 * 5 * 11 * 11)
    assert (k0, t0, i0) == (k1, t1, i1) == (key, t, idx)
    # saturated key resolved exactly across the two shards (index 8706 lies in rank 1's)
    assert s0 == s1 == (((1 << 30) - 1) << 33 | 8706, 1694498916, 8706)
    # reference state counts of these configurations (tests/golden/explore.json / oracle)
    want = [oracle.explore(p, s, k, wg, ts)["states"] for p, s, k, wg, ts in CASES]
    for (m0, tot0), (m1, tot1), w in zip(c0, c1, want):
        assert tot0 == tot1 == w and m0 + m1 == w and m0 > 0 and m1 > 0


def test_shard_bounds():
    from paper_2305_09130_b200.distributed import shard
    for total in (0, 1, 7, 10 ** 9 + 3):
        for world in (1, 2, 3, 8):
            spans = [shard(total, r, world) for r in range(world)]
            assert sum(c for _, c in spans) == total
            assert all(spans[r][0] + spans[r][1] == spans[r + 1][0] for r in range(world - 1))
