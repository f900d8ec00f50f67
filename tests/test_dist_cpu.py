"""The multi-GPU path's host logic on CPU (gloo, world size 2 and 3):

* the product's plumbing: dist.share_unique_id gives every rank rank 0's NCCL unique id
  (vr_nccl_unique_id runs without a GPU);
* the protocol — shards, exchanges A/B/C of include/vr.h "Multi-GPU" — modelled in
  tests/_model_backend.py with the oracle as the device stage and the library's own host
  residual: the final barcode must equal the oracle's, whatever the world size.  (The
  library's C++ implementation of the same protocol is run on a GPU with emulated ranks in
  tests/test_gpu_parity.py.)"""
from __future__ import annotations

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from datagen import clouds as G
from oracle import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, lt, n, D, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from _model_backend import ModelBackend, globalize_stats, orchestrate
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        be = ModelBackend(lt, n, D, rank, world)
        bc, totals, local = orchestrate(be, D)
        bc = globalize_stats(bc, totals, local)
        q.put((rank, [p.tolist() for p in bc.pairs], [dict(s) for s in bc.stats], totals))
    finally:
        dist.destroy_process_group()


def _run(world, lt, n, D):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, lt, n, D, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out, key=lambda x: x[0])


@pytest.mark.parametrize("world,seed", [(2, 0), (2, 1), (3, 2)])
def test_sharded_orchestration_matches_oracle(world, seed):
    n, D = 8, 2
    lt = G.random_tied(n, seed, levels=4) if seed % 2 else G.random_cloud(n, seed)
    res = _run(world, lt, n, D)
    t = O.enclosing_radius(lt, n)
    ref = O.barcode(lt, n, D, t)
    first = res[0]
    for rank, pairs, stats, totals in res:
        assert pairs == first[1]  # every rank holds the same barcode
        for d in range(D + 1):
            exp = ref.positive(d).tolist()
            assert [tuple(x) for x in pairs[d]] == [tuple(x) for x in exp], (rank, d)
        for d in range(1, D + 1):
            assert stats[d]["survivors"] == ref.n_simplices[d]
            assert stats[d]["pairs_all"] == ref.num_pairs_all(d)


def _uid_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2502_05063_b200.dist import share_unique_id
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, share_unique_id()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_nccl_unique_id_shared(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_uid_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ids = set(out.values())
    assert len(ids) == 1 and len(next(iter(ids))) == 128


def test_merge_sorted_keys():
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from _model_backend import merge_sorted_keys
    rng = np.random.default_rng(0)
    allk = np.unique(rng.integers(0, 2**62, 1000, dtype=np.uint64))
    parts = [np.sort(allk[i::3]) for i in range(3)]
    assert np.array_equal(merge_sorted_keys(parts), allk)
    assert merge_sorted_keys([np.zeros(0, np.uint64)]).size == 0


def test_bitmap_sum_is_or_for_disjoint_bits():
    rng = np.random.default_rng(1)
    bits = rng.permutation(32 * 64)[:500]
    owner = rng.integers(0, 4, 500)
    words = [np.zeros(64, np.uint32) for _ in range(4)]
    for b, o in zip(bits, owner):
        words[o][b >> 5] |= np.uint32(1 << (b & 31))
    s = sum(w.view(np.int32).astype(np.int64) for w in words)  # int32 SUM all-reduce
    s = (s & 0xFFFFFFFF).astype(np.uint32)
    o = np.bitwise_or.reduce(words)
    assert np.array_equal(s, o)


def test_dense_shards_partition_rows():
    # row r of C(n,d) belongs to rank (C(n,d)-1-r) % world — every row exactly once
    for total in (1, 7, 100):
        for world in (1, 2, 3, 8):
            seen = []
            for rank in range(world):
                cnt = (total - rank + world - 1) // world if total > rank else 0
                seen += [total - 1 - (g * world + rank) for g in range(cnt)]
            assert sorted(seen) == list(range(total))
