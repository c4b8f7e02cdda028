"""Multi-process (N>1) host logic of bench.py on CPU: gloo backend, world size 2.

The query path does not shard (replicas only). What N>1 adds is host
plumbing: rank 0 builds the index once with the reference builder and shares the PTRH
bytes, every rank answers its own shuffled stream, and the timing is the max over ranks.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import sys
    sys.path.insert(0, ROOT)
    import hashlib

    import bench
    from oracle.bindings import Port, corpus_u64_np

    try:
        d = bench.Dist("gloo")
        n = 20_000
        ptrh = bench.build_index_bytes(n, d, lambda m: corpus_u64_np(0, m, bench.GEN_SEED))
        port_ = Port()
        pi = port_.load(ptrh)
        # each replica answers its own shuffled stream of the full key set
        qs = port_.gen_keys("perm", 0, n, n, bench.GEN_SEED, bench.PERM_SEED + rank, threads=2)
        out = pi.query_u64(qs, True)
        ok = bool(np.array_equal(np.sort(out), np.arange(n, dtype=np.uint64)))
        t = d.max(float(rank + 1) * 1.5)
        q.put((rank, hashlib.sha1(ptrh).hexdigest(), ok, t, int(qs[0])))
        d.close()
    except Exception as e:  # pragma: no cover
        q.put((rank, "error", repr(e), None, None))


def test_two_replicas_share_one_index_and_max_over_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] != "error" for r in res), res
    assert res[0][1] == res[1][1]            # identical PTRH bytes on both ranks
    assert res[0][2] and res[1][2]           # each replica's outputs are a bijection
    assert res[0][3] == res[1][3] == 3.0     # max over ranks
    assert res[0][4] != res[1][4]            # different query streams per rank
