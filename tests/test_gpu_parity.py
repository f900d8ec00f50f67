"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar: bit-exact.  Every birth/death is a copy of a distance-matrix entry, so the multiset
of (birth, death) fp32 pairs must match exactly per dimension; at the index level the
full pairing (apparent + residual + dimension-0 pairs, zero-length and essential
included) is unique for the §5.1.4 refinement and must match too.
"""
from __future__ import annotations

import math
import os

import numpy as np
import pytest

import paper_2502_05063_b200 as vr
from datagen import clouds as G
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _oracle_at(lt, n, D, t):
    return O.barcode(lt, n, D, t)


def assert_values_equal(got: vr.Barcode, ref, D):
    for d in range(D + 1):
        exp = ref.positive(d)
        assert got.pairs[d].shape == exp.shape, (d, got.pairs[d], exp)
        assert np.array_equal(got.pairs[d].view(np.uint32), exp.view(np.uint32)), d


def assert_index_equal(got: vr.Barcode, ref, D):
    for d in range(D + 1):
        g = {(int(a), int(b)) for a, b in got.index_pairs[d]}
        assert len(g) == len(got.index_pairs[d])  # no duplicates
        assert g == ref.index_pairs(d), d


def assert_counts_equal(got: vr.Barcode, ref, D):
    for d in range(D + 1):
        s = got.stats[d]
        assert s["pairs_all"] == ref.num_pairs_all(d), d
        assert s["essential"] == ref.num_essential(d), d
        if d >= 1:
            assert s["survivors"] == ref.n_simplices[d], d


def full_check(lt, n, D, threshold=math.inf, **opts):
    got = vr.barcodes(lt, n, D, threshold, index_pairs=True, **opts)
    t = got.threshold
    ref = _oracle_at(lt, n, D, t)
    assert_values_equal(got, ref, D)
    assert_index_equal(got, ref, D)
    assert_counts_equal(got, ref, D)
    if math.isinf(threshold):  # Prop 5.2.13: t = R and t = inf report the same bars
        assert_values_equal(got, _oracle_at(lt, n, D, math.inf), D)
    return got, ref


# ------------------------------------------------------------------ closed forms
def test_unit_square():
    got, _ = full_check(G.unit_square(), 4, 1)
    assert got.pairs[1].tolist() == [[1.0, np.float32(math.sqrt(2))]]


@pytest.mark.parametrize("k", [2, 3, 4])
def test_cross_polytope(k):
    got, _ = full_check(G.cross_polytope(k), 2 * k, k - 1)
    assert got.pairs[k - 1].tolist() == [[np.float32(math.sqrt(2)), 2.0]]


@pytest.mark.parametrize("n", range(6, 13))
def test_regular_ngon(n):
    full_check(G.regular_ngon(n), n, 1)


def test_single_point_and_pair():
    got = vr.barcodes(np.zeros(0, np.float32), 1, 2)
    assert got.pairs[0].tolist() == [[0.0, math.inf]] and len(got.pairs[1]) == 0
    got = vr.barcodes(np.array([5.0], np.float32), 2, 1)
    assert got.pairs[0].tolist() == [[0.0, 5.0], [0.0, math.inf]]


def test_duplicate_points_zero_length_suppressed():
    pts = np.array([[0, 0], [0, 0], [1, 0], [1, 1]], np.float64)
    lt = G.lower_tri_from_points(pts)
    got, ref = full_check(lt, 4, 2)
    assert got.stats[0]["pairs_all"] == 3 and got.stats[0]["pairs_positive"] == 2


@pytest.mark.parametrize("n,d", [(n, d) for n in (6, 9, 14, 20) for d in (1, 2)])
def test_thm542_all_equal_apparent_count(n, d):
    got = vr.barcodes(G.all_equal(n), n, 2, 1.0)
    assert got.stats[d]["apparent"] == math.comb(n - 1, d + 1)


@pytest.mark.parametrize("n", [5, 7])
def test_fig56_lex_decreasing(n):
    # §5.4.3 is a statement about the FULL Rips filtration: threshold = the max distance
    lt = G.fig56_lex_decreasing(n)
    got, _ = full_check(lt, n, 1, float(lt.max()))
    assert got.stats[1]["apparent"] == math.comb(n - 1, 2)


# ------------------------------------------------------------------ brute force on small random inputs
CASES = []
for seed in range(48):
    n = 5 + seed % 8
    D = 1 + seed % 3
    kind = ["tied", "cloud", "tied2"][seed % 3]
    thr = ["inf", "R", "q60"][(seed // 3) % 3]
    CASES.append((seed, n, D, kind, thr))


@pytest.mark.parametrize("seed,n,D,kind,thr", CASES)
def test_random_small_index_level(seed, n, D, kind, thr):
    if kind == "tied":
        lt = G.random_tied(n, seed, levels=3)
    elif kind == "tied2":
        lt = G.random_tied(n, seed, levels=8)
    else:
        lt = G.random_cloud(n, seed)
    t = math.inf if thr == "inf" else (O.enclosing_radius(lt, n) if thr == "R" else float(np.quantile(lt, 0.6)))
    full_check(lt, n, D, t)


# ------------------------------------------------------------------ configs (full where feasible, else subsampled)
def test_config1_full():
    cfg = G.CONFIGS["c1_circle64"]
    got, ref = full_check(cfg.lower_tri(), cfg.n, cfg.max_dim)
    h1 = got.pairs[1]
    assert ((h1[:, 1] - h1[:, 0]) > 1.0).sum() == 1


@pytest.mark.parametrize("name,m,D", [("c2_s3_192", 24, 3), ("c3_trefoil1000", 40, 2), ("c4a_sierpinski512", 40, 2),
                                      ("c4b_torus2000", 40, 2), ("c5_o3_4096", 36, 2), ("c5_o3_4096", 22, 3)])
def test_config_subsample(name, m, D):
    cfg = G.CONFIGS[name]
    full_check(cfg.lower_tri(m), m, D, cfg.threshold)


@pytest.mark.parametrize("steps", [1, 2, 7, 64])
def test_apparent_phase_split_invariance(steps):
    lt = G.random_cloud(60, 3)
    a = vr.barcodes(lt, 60, 2, apparent_steps=steps, index_pairs=True)
    b = vr.barcodes(lt, 60, 2, apparent_steps=16, index_pairs=True)
    for d in range(3):
        assert np.array_equal(a.pairs[d], b.pairs[d])
        assert {tuple(x) for x in a.index_pairs[d].tolist()} == {tuple(x) for x in b.index_pairs[d].tolist()}
        assert a.stats[d]["apparent"] == b.stats[d]["apparent"]


@pytest.mark.parametrize("grab", [1, 3, 16])
@pytest.mark.parametrize("D", [1, 2, 3])
def test_row_scheduling_invariance(grab, D):
    # rows_per_grab: rows per atomic grab; the scan window in shared memory is used at
    # n <= 544 and the global path above — both must agree
    for n in (70, 600):
        if n == 600 and (D == 3 or (D == 2 and grab != 3)):  # (n = 600, D = 2: 30 s of host residual each)
            continue
        lt = G.random_cloud(n, 5)
        a = vr.barcodes(lt, n, D, rows_per_grab=grab, index_pairs=True)
        b = vr.barcodes(lt, n, D, index_pairs=True)
        for d in range(D + 1):
            assert np.array_equal(a.pairs[d], b.pairs[d])
            assert {tuple(x) for x in a.index_pairs[d].tolist()} == {tuple(x) for x in b.index_pairs[d].tolist()}
            assert a.stats[d]["survivors"] == b.stats[d]["survivors"]


@pytest.mark.parametrize("n,D", [(33, 3), (100, 2), (100, 3), (544, 2), (545, 2)])
def test_flat_kernel_equals_row_kernel(n, D, monkeypatch):
    # k_enumerate_flat (d >= 2, n <= 544, shared-memory window) against the row kernel
    # (VR_NO_FLAT); n = 545 is past the window limit, so both sides run the row kernel
    lt = G.random_cloud(n, 21)
    t = float(np.quantile(lt, 0.3)) if n > 200 else math.inf
    a = vr.barcodes(lt, n, D, t, index_pairs=True)
    monkeypatch.setenv("VR_NO_FLAT", "1")
    b = vr.barcodes(lt, n, D, t, index_pairs=True)
    for d in range(D + 1):
        assert np.array_equal(a.pairs[d], b.pairs[d])
        assert {tuple(x) for x in a.index_pairs[d].tolist()} == {tuple(x) for x in b.index_pairs[d].tolist()}
        for k in ("survivors", "apparent", "cleared", "residual_columns"):
            assert a.stats[d][k] == b.stats[d][k], (d, k)


def test_residual_modes_agree():
    cfg = G.CONFIGS["c2_s3_192"]
    lt = cfg.lower_tri(60)
    a = vr.barcodes(lt, 60, 3, residual_mode=0)
    b = vr.barcodes(lt, 60, 3, residual_mode=1)
    for d in range(4):
        assert np.array_equal(a.pairs[d], b.pairs[d])


def test_device_entry_matches_host_entry():
    torch = pytest.importorskip("torch")
    cfg = G.CONFIGS["c4a_sierpinski512"]
    lt = cfg.lower_tri(120)
    a = vr.barcodes(lt, 120, 2)
    t = torch.from_numpy(lt).cuda()
    b = vr.barcodes_device(t, 120, 2)
    for d in range(3):
        assert np.array_equal(a.pairs[d], b.pairs[d])


# ------------------------------------------------------------------ full-size configs: invariants
def _triangles_le(lt, n, t):
    A = (G.square_from_lower_tri(lt, n) <= np.float32(t)).astype(np.float64)
    np.fill_diagonal(A, 0)
    return int(round(np.trace(A @ A @ A) / 6))


@pytest.mark.parametrize("name", ["c1_circle64", "c2_s3_192", "c4a_sierpinski512", "c3_trefoil1000"])
def test_full_config_invariants(name):
    cfg = G.CONFIGS[name]
    lt = cfg.lower_tri()
    got = vr.barcodes(lt, cfg.n, cfg.max_dim, cfg.threshold)
    t = got.threshold
    D = cfg.max_dim
    # survivors: edges and triangles by brute force
    assert got.stats[1]["survivors"] == int((lt <= np.float32(t)).sum())
    if D >= 2:
        assert got.stats[2]["survivors"] == _triangles_le(lt, cfg.n, t)
    # n_p = P_p + E_p + P_{p-1}
    P = [got.stats[p]["pairs_all"] for p in range(D + 1)]
    E = [got.stats[p]["essential"] for p in range(D + 1)]
    for p in range(1, D + 1):
        assert got.stats[p]["survivors"] == P[p] + E[p] + P[p - 1]
        s = got.stats[p]
        assert s["survivors"] == s["apparent"] + s["cleared"] + s["residual_columns"]
    # determinism
    again = vr.barcodes(lt, cfg.n, cfg.max_dim, cfg.threshold)
    for d in range(D + 1):
        assert np.array_equal(got.pairs[d], again.pairs[d])


def _long(pairs, frac):
    pers = pairs[:, 1] - pairs[:, 0]
    if len(pers) == 0:
        return 0
    top = np.max(np.where(np.isinf(pers), 0, pers))
    return int((pers > frac * max(top, 1e-9)).sum())


def test_betti_circle_and_s3():
    c1 = G.CONFIGS["c1_circle64"]
    b = vr.barcodes(c1.lower_tri(), c1.n, 1)
    assert ((b.pairs[1][:, 1] - b.pairs[1][:, 0]) > 1.0).sum() == 1
    c2 = G.CONFIGS["c2_s3_192"]
    b = vr.barcodes(c2.lower_tri(), c2.n, 3)
    p3 = b.pairs[3][:, 1] - b.pairs[3][:, 0]
    assert len(p3) >= 1 and np.sort(p3)[-1] > 3 * (np.sort(p3)[-2] if len(p3) > 1 else 0)


# ------------------------------------------------------------------ a4 alone: the radix sort
@pytest.mark.parametrize("n", [0, 1, 2, 100, 2048, 2049, 3001, 4096, 4097, 8192, 8193, 16385, 30000, 65537, 70000, 130122, 131072, 131073,
                               1_200_000])
@pytest.mark.parametrize("bits", [(0, 64), (0, 41), (8, 40)])
def test_radix_sort_matches_numpy(n, bits):
    rng = np.random.default_rng(n + bits[1])
    keys = rng.integers(0, 2**63, n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, n, dtype=np.uint64)
    if n > 10:
        keys[: n // 3] = keys[n // 3: 2 * (n // 3)]  # many duplicates
    got = vr.radix_sort_u64(keys, *bits)
    b0, b1 = bits
    mask = np.uint64(((1 << (b1 - b0)) - 1) << b0) if b1 - b0 < 64 else np.uint64(2**64 - 1)
    sub = keys & mask
    order = np.argsort(sub, kind="stable")  # LSD radix sort is stable on the sorted bits
    assert np.array_equal(got, keys[order])


# the residual-column sort: counting sort on the rank field + the runs of equal rank sorted
# (in registers up to 16 keys, one warp per longer run up to 4096, else the radix sort)
@pytest.mark.parametrize("n,bins,runs", [(1000, 5000, "random"), (200000, 200000, "random"), (552000, 234207, "random"),
                                         (3000, 200, "long"), (300000, 100000, "long"), (70000, 10, "huge"),
                                         (300000, 100000, "mixed")])
@pytest.mark.parametrize("mode", [-1, 0, 1])
def test_sort_columns_matches_numpy(n, bins, runs, mode):
    rng = np.random.default_rng(n + bins)
    cbits = 44
    if runs == "random":
        f = rng.integers(0, bins, n)
    elif runs == "long":  # runs of 10..40
        f = np.repeat(rng.choice(bins, n // 25, replace=False), 25)[:n]
    elif runs == "huge":  # runs of thousands (> 4096: the radix fallback)
        f = rng.integers(0, bins, n)
    else:  # every run length 1..300
        f = np.concatenate([np.full(k, i % bins) for i, k in enumerate(rng.integers(1, 300, n // 150))])[:n]
    low = rng.choice(1 << 40, len(f), replace=False).astype(np.uint64)
    keys = (f.astype(np.uint64) << np.uint64(cbits)) | low
    if len(np.unique(keys)) != len(keys):
        keys = np.unique(keys)
    rng.shuffle(keys)
    end_bit = cbits + max(1, int(bins).bit_length())
    if mode == 1 and runs == "huge":
        mode = -1  # (forcing the counting path on runs past its limit is not supported)
    got, path = vr.sort_columns_u64(keys, cbits, end_bit, bins, mode)
    assert np.array_equal(got, np.sort(keys))
    if mode == -1 and runs == "huge":
        assert path == 0
    if mode == -1 and n > 131072 and runs != "huge":
        assert path == 1  # the counting path was taken (and its runs were short enough)


# ------------------------------------------------------------------ output-sensitive (sparse) mode
@pytest.mark.parametrize("seed,n,D,kind,thr", CASES[::2])
def test_sparse_mode_index_level(seed, n, D, kind, thr):
    if kind == "tied":
        lt = G.random_tied(n, seed, levels=3)
    elif kind == "tied2":
        lt = G.random_tied(n, seed, levels=8)
    else:
        lt = G.random_cloud(n, seed)
    t = math.inf if thr == "inf" else (O.enclosing_radius(lt, n) if thr == "R" else float(np.quantile(lt, 0.6)))
    full_check(lt, n, D, t, sparse_mode=2)


@pytest.mark.parametrize("name,m,D", [("c5_o3_4096", 36, 2), ("c5_o3_4096", 22, 3), ("c3_trefoil1000", 40, 2),
                                      ("c2_s3_192", 24, 3)])
@pytest.mark.parametrize("steps", [2, 32])
def test_sparse_mode_config_subsample(name, m, D, steps):
    cfg = G.CONFIGS[name]
    thr = 1.0 if name == "c5_o3_4096" else cfg.threshold  # a sparse threshold graph
    full_check(cfg.lower_tri(m), m, D, thr, sparse_mode=2, apparent_steps=steps)


# sparse dimensions >= 2 with the clearing hash set instead of a bitmap (the path taken when
# C(n, d+1) bits cannot be allocated, e.g. config 5 at dimension 3), forced at small n
@pytest.mark.parametrize("seed,n,D,kind,thr", [c for c in CASES if c[2] >= 2][::2])
def test_sparse_clear_hash_index_level(seed, n, D, kind, thr, monkeypatch):
    monkeypatch.setenv("VR_FORCE_CLEAR_HASH", "1")
    if kind == "tied":
        lt = G.random_tied(n, seed, levels=3)
    elif kind == "tied2":
        lt = G.random_tied(n, seed, levels=8)
    else:
        lt = G.random_cloud(n, seed)
    t = math.inf if thr == "inf" else (O.enclosing_radius(lt, n) if thr == "R" else float(np.quantile(lt, 0.6)))
    full_check(lt, n, D, t, sparse_mode=2)


@pytest.mark.parametrize("name,m,D", [("c5_o3_4096", 36, 2), ("c5_o3_4096", 22, 3), ("c2_s3_192", 24, 3)])
@pytest.mark.parametrize("steps", [2, 32])
def test_sparse_clear_hash_config_subsample(name, m, D, steps, monkeypatch):
    monkeypatch.setenv("VR_FORCE_CLEAR_HASH", "1")
    cfg = G.CONFIGS[name]
    thr = 1.0 if name == "c5_o3_4096" else cfg.threshold
    full_check(cfg.lower_tri(m), m, D, thr, sparse_mode=2, apparent_steps=steps)


def test_config5_dim3_hash_equals_recompute(c5_lower_tri, monkeypatch):
    # config 5 at max_dim 3 takes the hash set at dimension 3 by itself; the recompute path
    # (VR_NO_CLEAR_HASH) must give the same barcode and the same counts
    cfg = G.CONFIGS["c5_o3_4096"]
    a = vr.barcodes(c5_lower_tri, cfg.n, 3, cfg.threshold)
    monkeypatch.setenv("VR_NO_CLEAR_HASH", "1")
    b = vr.barcodes(c5_lower_tri, cfg.n, 3, cfg.threshold)
    for d in range(4):
        assert np.array_equal(a.pairs[d], b.pairs[d])
    for k in ("survivors", "apparent", "cleared", "residual_columns"):
        assert a.stats[3][k] == b.stats[3][k], k
    assert a.stats[3]["queued"] < b.stats[3]["queued"]


@pytest.fixture(scope="module")
def c5_lower_tri():
    return G.CONFIGS["c5_o3_4096"].lower_tri()


def test_config5_dense_equals_sparse_dim2(c5_lower_tri):
    cfg = G.CONFIGS["c5_o3_4096"]
    a = vr.barcodes(c5_lower_tri, cfg.n, 2, cfg.threshold, sparse_mode=1)
    b = vr.barcodes(c5_lower_tri, cfg.n, 2, cfg.threshold, sparse_mode=2)
    for d in range(3):
        assert np.array_equal(a.pairs[d], b.pairs[d])
        for k in ("survivors", "apparent", "cleared", "residual_columns", "pairs_all", "essential"):
            assert a.stats[d][k] == b.stats[d][k], (d, k)


def test_config5_dim3_invariants(c5_lower_tri):
    cfg = G.CONFIGS["c5_o3_4096"]
    got = vr.barcodes(c5_lower_tri, cfg.n, 3, cfg.threshold)
    D = 3
    assert got.stats[1]["survivors"] == int((c5_lower_tri <= np.float32(cfg.threshold)).sum())
    P = [got.stats[p]["pairs_all"] for p in range(D + 1)]
    E = [got.stats[p]["essential"] for p in range(D + 1)]
    for p in range(1, D + 1):
        s = got.stats[p]
        assert s["survivors"] == P[p] + E[p] + P[p - 1]
        assert s["survivors"] == s["apparent"] + s["cleared"] + s["residual_columns"]
    # two O(3) components exactly 2.0 apart (> t = 1.4): beta_0 = 2 essential classes
    assert E[0] == 2


# ------------------------------------------------------------------ multi-GPU: the library's sharded path
# Ranks emulated in this process on the one GPU (dist.run_ranks: vr_comm_local, one host
# thread per rank; the collectives stage through host memory).  Every rank runs the
# library's run_distributed: its shard of each dimension, exchanges A (clearing bitmap
# all-reduce / apparent-cofacet all-gather into the sets), B (residual keys all-gather +
# device merge) and C (rank 0's residual deaths broadcast), then the result broadcast.
def _ranks(lt, n, D, world, thr=math.inf, **opts):
    from paper_2502_05063_b200.dist import barcodes_comm, run_ranks
    return run_ranks(world, lambda c: barcodes_comm(lt, n, D, thr, c, **opts))


SHARD_CASES = [("tied", 10, 2), ("cloud", 11, 3), ("c2", 24, 3), ("c5patch", 40, 2), ("c3", 36, 2)]


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("sparse", [1, 2])
@pytest.mark.parametrize("kind,m,D", SHARD_CASES)
def test_sharded_ranks_vs_oracle(world, sparse, kind, m, D):
    thr = math.inf
    if kind == "tied":
        lt = G.random_tied(m, 77, levels=4)
    elif kind == "cloud":
        lt = G.random_cloud(m, 78)
    elif kind == "c5patch":
        lt, thr = G.CONFIGS["c5_o3_4096"].patch(m), 1.4
    else:
        lt = G.CONFIGS[{"c2": "c2_s3_192", "c3": "c3_trefoil1000"}[kind]].lower_tri(m)
    res = _ranks(lt, m, D, world, thr, sparse_mode=sparse, index_pairs=True)
    ref = O.barcode(lt, m, D, res[0].threshold)
    for r, got in enumerate(res):  # every rank returns the oracle's barcode
        assert_values_equal(got, ref, D)
        assert_index_equal(got, ref, D)
        assert_counts_equal(got, ref, D)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name,m,D,sparse,hashset", [("c2_s3_192", 60, 3, 1, False), ("c3_trefoil1000", 150, 2, 2, False),
                                                     ("c2_s3_192", 60, 3, 2, True), ("c5_o3_4096", 4096, 2, 0, False)])
def test_sharded_ranks_match_single_gpu(world, name, m, D, sparse, hashset, monkeypatch):
    # larger inputs (c5 at full size: the sparse path with the clearing set at dimension 2,
    # its apparent cofacets all-gathered between the ranks) against the one-GPU result
    if hashset:
        monkeypatch.setenv("VR_FORCE_CLEAR_HASH", "1")
    cfg = G.CONFIGS[name]
    lt = cfg.lower_tri(m)
    ref = vr.barcodes(lt, m, D, cfg.threshold, sparse_mode=sparse)
    res = _ranks(lt, m, D, world, cfg.threshold, sparse_mode=sparse)
    for got in res:
        for d in range(D + 1):
            assert np.array_equal(got.pairs[d].view(np.uint32), ref.pairs[d].view(np.uint32)), d
        for d in range(1, D + 1):
            for k in ("survivors", "apparent", "cleared", "residual_columns", "pairs_all", "essential", "emergent"):
                assert got.stats[d][k] == ref.stats[d][k], (d, k)


def test_sharded_plan_replay():
    # the timed multi-rank step (bench.py): a plan per rank, replays of the sharded hot path
    # with exchanges A and B; the counters of a replay equal the first run's
    import torch
    from paper_2502_05063_b200.dist import run_ranks
    cfg = G.CONFIGS["c2_s3_192"]
    lt = cfg.lower_tri(80)
    t = torch.from_numpy(lt).cuda()
    ref = vr.barcodes(lt, 80, 3)

    def rank(c):
        s = torch.cuda.Stream()
        plan = vr.Plan(t, 80, 3, stream=s.cuda_stream, comm=c)
        first = plan.check()
        for _ in range(3):
            assert plan.replay() > 0
        again = plan.check()
        res = plan.result
        plan.close()
        return first, again, res

    for first, again, res in run_ranks(2, rank):
        assert first == again
        for d in range(4):
            assert np.array_equal(res.pairs[d], ref.pairs[d])


def test_nccl_single_rank_and_num_gpus():
    # the NCCL transport itself (one rank here: every gpurun box has one GPU) and
    # vr_options.num_gpus = 1 through vr_barcodes
    import socket
    import torch.distributed as tdist
    from paper_2502_05063_b200.dist import barcodes_sharded
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    tdist.init_process_group("gloo", rank=0, world_size=1)
    try:
        cfg = G.CONFIGS["c4a_sierpinski512"]
        lt = cfg.lower_tri(120)
        ref = vr.barcodes(lt, 120, 2)
        got = barcodes_sharded(lt, 120, 2)
        one = vr.barcodes(lt, 120, 2, num_gpus=1)
        for d in range(3):
            assert np.array_equal(got.pairs[d], ref.pairs[d])
            assert np.array_equal(one.pairs[d], ref.pairs[d])
            assert got.stats[d]["pairs_all"] == ref.stats[d]["pairs_all"]
    finally:
        tdist.destroy_process_group()


def test_merge_of_gathered_keys():
    # exchange B's device merge through the sharded path: many residual columns, 4 ranks
    cfg = G.CONFIGS["c2_s3_192"]
    lt = cfg.lower_tri(100)
    ref = vr.barcodes(lt, 100, 3)
    res = _ranks(lt, 100, 3, 4)
    assert res[0].stats[3]["residual_columns"] > 1000
    for d in range(4):
        assert np.array_equal(res[0].pairs[d], ref.pairs[d])


# ------------------------------------------------------------------ full sizes: sampled outputs vs the oracle
def _decode(c, k, n):
    out, hi = [], n
    for q in range(k):
        kk = k - q
        lo, h = kk - 1, hi - 1
        while lo < h:
            mid = (lo + h + 1) // 2
            if math.comb(mid, kk) <= c:
                lo = mid
            else:
                h = mid - 1
        out.append(lo)
        c -= math.comb(lo, kk)
        hi = lo
    return out


@pytest.mark.parametrize("name,D", [("c2_s3_192", 3), ("c3_trefoil1000", 2), ("c4a_sierpinski512", 2),
                                    ("c4b_torus2000", 2), ("c5_o3_4096", 2), ("c5_o3_4096", 3)])
def test_full_size_sampled_apparent_pairs(name, D):
    """Every config at full size, in the launch configuration bench.py times: 400 of the
    GPU's apparent pairs and 200 of its residual columns per dimension, each checked one by
    one against the oracle's per-simplex Def 5.3.4 on the explicit cofacet/facet
    sets.  The library keeps at most 2M apparent pairs per dimension here (index_pairs = k:
    an arbitrary subset), so c4b's 1.3e9 dimension-2 columns need no host copy."""
    cfg = G.CONFIGS[name]
    lt = cfg.lower_tri()
    got = vr.barcodes(lt, cfg.n, D, cfg.threshold, index_pairs=2_000_000)
    t = got.threshold
    rng = np.random.default_rng(7)
    for d in range(1, D + 1):
        ip = got.index_pairs[d]
        nres = got.stats[d]["residual_columns"]
        app, rest = ip[:len(ip) - nres], ip[len(ip) - nres:]
        assert len(app) == min(got.stats[d]["apparent"], 2_000_000)
        for k in rng.choice(len(app), size=min(400, len(app)), replace=False):
            s, tt = int(app[k, 0]), int(app[k, 1])
            assert O.apparent_one(lt, cfg.n, _decode(s, d + 1, cfg.n), t) == (True, tt), (d, s)
        for k in rng.choice(len(rest), size=min(200, len(rest)), replace=False):
            s = int(rest[k, 0])
            assert O.apparent_one(lt, cfg.n, _decode(s, d + 1, cfg.n), t) == (False, None), (d, s)


def _sorted_bars(a):
    a = np.asarray(a, np.float32).reshape(-1, 2)
    return a[np.lexsort((a[:, 1], a[:, 0]))] if len(a) else a


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c2_s3_192", "c3_trefoil1000", "c5_o3_4096"])
def test_full_config_bars_equal_cpu_ripser(name):
    """Full-size barcodes, bit-exact, against cpu_ripser — the single-threaded Ripser-style
    program (implicit cohomology + clearing + emergent pairs, §5.2) that shares no
    code with the library and is itself pinned bit-exactly to the oracle
    (tests/test_cpu_ripser.py: 48 random / tied / thresholded cases, configs 1 and 4a)."""
    import cpu_ripser as RS
    cfg = G.CONFIGS[name]
    lt = cfg.lower_tri()
    bc = vr.barcodes(lt, cfg.n, cfg.max_dim, cfg.threshold)
    pairs, st = RS.barcode(lt, cfg.n, cfg.max_dim, bc.threshold)
    for d in range(cfg.max_dim + 1):
        assert np.array_equal(_sorted_bars(pairs[d]).view(np.uint32), _sorted_bars(bc.pairs[d]).view(np.uint32)), d
    for d in range(1, cfg.max_dim + 1):
        assert st[d]["simplices"] == bc.stats[d]["survivors"], d


def test_apparent_rate_matches_paper_at_10000_points():
    # PAPER.md §5.6.6: random-permutation distance matrices, dimension 1, n = 10000:
    # average apparent fraction 0.991127743 (relative to the edges of the filtration, which
    # the enclosing-radius cut keeps).  One sample here (the paper averages 10; the sample
    # spread at this n is ~5e-5): the GPU hot path alone (hot_path_only: no residual).
    import torch
    n = 10000
    N = n * (n - 1) // 2
    perm = np.random.default_rng(1000).permutation(N).astype(np.uint32)
    vals = (perm + np.uint32(0x3F800000)).view(np.float32)  # order-preserving (Obs 5.6.8)
    lt = torch.from_numpy(vals).cuda()
    bc = vr.barcodes_device(lt, n, 1, math.inf, hot_path_only=True)
    surv, app = bc.stats[1]["survivors"], bc.stats[1]["apparent"]
    assert abs(app / surv - 0.991127743) < 3e-4
    assert app / N <= (n - 2) / n  # Theorem 5.4.2 bound


@pytest.mark.parametrize("seed", range(4))
def test_sparse_coo_input(seed):
    # SPEC's sparse input / SURVEY §8(f) NEXT-2: only some pairs given; absent pairs are
    # absent edges.  Against the oracle on the dense matrix with those entries at +inf and
    # a finite threshold (the largest given distance), and against the dense entry point
    rng = np.random.default_rng(seed)
    n, D = 24, 2
    lt = G.random_cloud(n, 30 + seed)
    keep = rng.random(lt.size) < 0.6
    ii, jj = np.tril_indices(n, -1)
    rows, cols, dist = ii[keep], jj[keep], lt[keep]
    dense = np.where(keep, lt, np.float32(np.inf)).astype(np.float32)
    t = float(dist.max())
    got = vr.barcodes_coo(n, rows, cols, dist, D, index_pairs=True)          # threshold +inf
    got2 = vr.barcodes_coo(n, cols, rows, dist, D, t)                        # transposed pairs
    ref = O.barcode(dense, n, D, t)
    for d in range(D + 1):
        exp = ref.positive(d)
        assert np.array_equal(got.pairs[d].view(np.uint32), exp.view(np.uint32)), d
        assert np.array_equal(got2.pairs[d], got.pairs[d])
    den = vr.barcodes(dense, n, D)
    for d in range(D + 1):
        assert np.array_equal(den.pairs[d], got.pairs[d])
    with pytest.raises(Exception):
        vr.barcodes_coo(n, [0], [0], [1.0], D)


# ------------------------------------------------------------------ roofline work counters
@pytest.mark.parametrize("name,D", [("c2_s3_192", 3), ("c5_o3_4096", 2), ("c4a_sierpinski512", 2)])
def test_work_counter_rate_below_alu_peak(name, D):
    # the SURVEY 8(d) op count the bench divides by kernel time must describe work the
    # kernels really do: ops / measured kernel time can never exceed the ALU peak (148 SMs x
    # 64 lanes x 2.1 GHz, a bound above any B200 clock) — a dense candidate count on the
    # sparse path once gave 500x the peak
    import torch
    cfg = G.CONFIGS[name]
    lt = torch.from_numpy(cfg.lower_tri()).cuda()
    plan = vr.Plan(lt, cfg.n, D, cfg.threshold)
    for _ in range(3):
        plan.replay()
    torch.cuda.synchronize()
    tm = plan.timing()
    plan.close()
    peak = 148 * 64 * 2.1e9
    assert tm["rank_ops_enumerate"] > 0
    assert tm["rank_ops_enumerate"] / (tm["ms_enumerate"] / 1e3) < peak
    if tm["ms_resolve"] > 0:
        assert tm["rank_ops_resolve"] / (tm["ms_resolve"] / 1e3) < peak
