"""Host-side multi-process logic of the sharded paths, world_size 2 on CPU
(gloo over 127.0.0.1): document shard ranges, the error all-reduce, and the
mailbox-handle exchange.  The device-side exchange runs in
tests/test_gpu_sharded.py."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from synth import bank_corpus, init_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_1905_09598_b200 import dist as sd
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # documents sharded over ranks; local scores from the oracle stand in
        # for som_errors (no GPU here); the reduction is the product's
        C = bank_corpus(301, 120, seed=3)
        X = C.dense()
        W = init_rows(X, 12, 4)
        lo, hi = sd.shard_range(X.shape[0], rank, world)
        b1, b2, d1 = oracle.map_docs(W, X[lo:hi])
        qe_l = oracle.qerror_from_d1(d1) if hi > lo else 0.0
        te_l = oracle.topographic_error_from_bmus(3, 4, 1, b1, b2) if hi > lo else 0.0
        qe, te = sd.reduce_errors(qe_l, te_l, hi - lo)
        handles = sd.exchange_handles(bytes([rank]) * 64)
        out.put((rank, lo, hi, qe, te, handles))
    finally:
        dist.destroy_process_group()


def test_doc_sharding_and_handle_exchange_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    C = bank_corpus(301, 120, seed=3)
    X = C.dense()
    W = init_rows(X, 12, 4)
    b1, b2, d1 = oracle.map_docs(W, X)
    qe1 = oracle.qerror_from_d1(d1)
    te1 = oracle.topographic_error_from_bmus(3, 4, 1, b1, b2)
    (r0, lo0, hi0, qe_a, te_a, h0), (r1, lo1, hi1, qe_b, te_b, h1) = res
    assert (lo0, hi0, lo1, hi1) == (0, 151, 151, 301)
    assert abs(qe_a - qe1) <= 1e-12 * qe1 and abs(qe_b - qe1) <= 1e-12 * qe1
    assert te_a == te1 and te_b == te1
    assert h0 == h1 == [bytes([0]) * 64, bytes([1]) * 64]


@pytest.mark.parametrize("n,world", [(10, 3), (2, 4), (0, 2), (1000, 8)])
def test_shard_range(n, world):
    from paper_1905_09598_b200.dist import shard_range
    rs = [shard_range(n, r, world) for r in range(world)]
    assert rs[0][0] == 0 and rs[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
    sizes = [hi - lo for lo, hi in rs]
    assert max(sizes) - min(sizes) <= 1


def test_neuron_owner_partition():
    from paper_1905_09598_b200.dist import neuron_owner
    N, P = 37, 4
    seen = {}
    for u in range(N):
        r, l = neuron_owner(u, P)
        assert r + P * l == u
        seen.setdefault(r, []).append(l)
    for r in range(P):
        assert seen[r] == list(range(len(seen[r])))
        assert len(seen[r]) == (N - r + P - 1) // P
