"""Host-side builder tests (no GPU): the block plan decoded back from the
stored layout must reproduce A exactly, the
dense/sparse rule must follow P:96 (reading R3), the permutation must make
communities contiguous, and every error convention of
include/kur.h must be reachable."""
import ctypes
import re

import numpy as np
import pytest

import kurgen
from paper_2102_07167_b200 import kur


def reconstruct(inst, plan):
    """Dense 0/1 matrix in USER numbering rebuilt from the exported plan rows."""
    n = inst.n
    perm = plan["perm"]
    lab_int = inst.community[perm]
    rows = np.zeros((plan["n_local"], n), np.int64)
    for lj in range(plan["n_local"]):
        j = plan["row_begin"] + lj
        a = lab_int[j]
        for b in plan["D_idx"][plan["D_ptr"][a]:plan["D_ptr"][a + 1]]:
            rows[lj, lab_int == b] += 1
        s, e = plan["row_ptr"][lj], plan["row_ptr"][lj + 1]
        np.add.at(rows[lj], plan["cols"][s:e], np.where(plan["neg"][s:e] == 1, -1, 1))
    return rows


def check_plan(inst, A, **kw):
    world = kw.pop("world", 1)
    split_ok = kw.pop("split_ok", False)
    covered = []
    for rank in range(world):
        plan = kur.plan_export(inst, rank=rank, world=world, **kw)
        perm = plan["perm"]
        assert sorted(perm.tolist()) == list(range(inst.n))
        lab_int = inst.community[perm]
        assert np.all(np.diff(lab_int) >= 0), "communities must be contiguous"
        assert plan["conflicts"] == 0, "hot gathers must be bank-conflict free"
        rows = reconstruct(inst, plan)
        for lj in range(plan["n_local"]):
            j = plan["row_begin"] + lj
            u = perm[j]
            got = rows[lj].copy()
            want = A[u, perm].astype(np.int64)
            got[j] = want[j] = 0  # diagonal never contributes (reading R2)
            assert np.array_equal(got, want), (rank, j)
        covered.append((plan["row_begin"], plan["row_begin"] + plan["n_local"]))
        sr = plan["shard_row0"]
        if world > 1 and not split_ok:  # shards are whole communities
            for b in sr[1:-1]:
                assert b == 0 or b == inst.n or lab_int[b - 1] != lab_int[b]
    covered.sort()
    assert covered[0][0] == 0 and covered[-1][1] == inst.n
    for (a0, a1), (b0, b1) in zip(covered, covered[1:]):
        assert a1 == b0
    return plan


@pytest.mark.parametrize("kind", ["ones", "zeros", "auto", "random"])
@pytest.mark.parametrize("thr", [-1.0, 0.0, 0.5, 1.0])
def test_roundtrip_encodings_thresholds(kind, thr):
    A, labels = kurgen.random_dense(90, 4, seed=7, p_in=0.8, p_out=0.15, symmetric=False)
    inst = kurgen.from_dense(A, labels, kind=kind, seed=2)
    check_plan(inst, A, dense_threshold=thr)


@pytest.mark.parametrize("hot_min", [1, 1 << 30, 0])
def test_roundtrip_hot_and_remote(hot_min):
    inst = kurgen.sbm([700, 300, 5000, 1, 20], np.array(
        [[0.97, 0.3, 0.001, 0.0, 0.9], [0.3, 0.6, 0.0, 0.5, 0.0], [0.001, 0.0, 0.02, 0.0, 0.3],
         [0.0, 0.5, 0.0, 0.0, 0.0], [0.9, 0.0, 0.3, 0.0, 1.0]]), 13)
    A = inst.dense()
    check_plan(inst, A, hot_min=hot_min)


def test_roundtrip_empty_singleton_one_community():
    A, labels = kurgen.random_dense(40, 1, seed=1, p_in=0.6)
    check_plan(kurgen.from_dense(A, labels), A)
    labels = np.array([0] * 10 + [2] * 25 + [4] * 1, np.int32)  # communities 1 and 3 empty
    A, _ = kurgen.random_dense(36, 1, seed=3, p_in=0.5, symmetric=False)
    check_plan(kurgen.from_dense(A, labels, kind="random"), A)
    n = 17  # no edges at all
    check_plan(kurgen.from_dense(np.zeros((n, n), np.uint8), np.arange(n) % 3), np.zeros((n, n), np.uint8))


def test_roundtrip_many_tiles_ragged():
    # > 512 rows per community so tiles split, ragged last chunk, several windows
    inst = kurgen.sbm([1300, 4100, 77, 2600], np.array(
        [[0.95, 0.001, 0.0, 0.6], [0.001, 0.99, 0.01, 0.0], [0.0, 0.01, 0.3, 0.0], [0.6, 0.0, 0.0, 0.08]]), 5)
    A = inst.dense()
    plan = check_plan(inst, A)
    assert plan["n_tiles"] > 4
    plan2 = check_plan(inst, A, sm_count=1)  # fewer SMs -> larger tiles
    assert plan2["rows_per_tile"] == 2048
    for tr in (32, 96, 512):
        assert check_plan(inst, A, tile_rows=tr)["rows_per_tile"] == tr


@pytest.mark.parametrize("world", [2, 3])
def test_roundtrip_sharded(world):
    inst = kurgen.sbm([300, 500, 200, 400, 100], np.array(
        [[0.9, 0.01, 0.0, 0.0, 0.2], [0.01, 0.95, 0.02, 0.0, 0.0], [0.0, 0.02, 0.7, 0.01, 0.0],
         [0.0, 0.0, 0.01, 0.99, 0.0], [0.2, 0.0, 0.0, 0.0, 0.3]]), 9)
    check_plan(inst, inst.dense(), world=world)


def _census(A, labels):
    C = labels.max() + 1
    dense = set()
    for a in range(C):
        ra = np.flatnonzero(labels == a)
        for b in range(C):
            cb = np.flatnonzero(labels == b)
            blk = A[np.ix_(ra, cb)].astype(np.int64)
            total = len(ra) * len(cb)
            ones = blk.sum()
            if a == b:
                total -= len(ra)
                ones -= np.trace(blk)
            zeros = total - ones
            if total > 0 and zeros < ones:  # P:96, tie -> sparse (R3)
                dense.add((a, b))
    return dense


def test_paper_rule_matches_census():
    A, labels = kurgen.random_dense(120, 6, seed=21, p_in=0.5, p_out=0.5, symmetric=False)
    inst = kurgen.from_dense(A, labels, kind="random", seed=3)
    plan = kur.plan_export(inst)
    got = {(a, int(b)) for a in range(inst.n_comm) for b in plan["D_idx"][plan["D_ptr"][a]:plan["D_ptr"][a + 1]]}
    assert got == _census(A, labels)
    assert plan["nnz"] == int(A.sum() - np.trace(A))


def test_tie_is_sparse():
    # 2 communities of 2: block (0,1) has exactly 2 ones of 4 -> SPARSE; block (0,0) off-diag all ones -> DENSE
    A = np.array([[0, 1, 1, 0], [1, 0, 0, 1], [1, 0, 0, 1], [0, 1, 1, 0]], np.uint8)
    inst = kurgen.from_dense(A, [0, 0, 1, 1])
    plan = kur.plan_export(inst)
    D = {a: set(plan["D_idx"][plan["D_ptr"][a]:plan["D_ptr"][a + 1]].tolist()) for a in range(2)}
    assert D == {0: {0}, 1: {1}}


def test_complete_graph_plan_has_no_entries():
    inst = kurgen.complete_graph(3000, 1)
    plan = kur.plan_export(inst)
    assert plan["cols"].size == 0 and plan["D_idx"].tolist() == [0]


# ---------------------------------------------------------------- error conventions
def _build_status(**over):
    inst = kurgen.from_dense(np.array([[0, 1, 1], [1, 0, 0], [1, 0, 0]], np.uint8), [0, 0, 1], kind="ones")
    arrays = dict(community=inst.community.copy(), seg_ptr=inst.seg_ptr.copy(), seg_comm=inst.seg_comm.copy(),
                  seg_kind=inst.seg_kind.copy(), idx_ptr=inst.idx_ptr.copy(), idx=inst.idx.copy())
    n, C, thr = inst.n, inst.n_comm, over.pop("thr", -1.0)
    for k, v in over.items():
        if k == "n":
            n = v
        elif k == "C":
            C = v
        else:
            arrays[k] = np.asarray(v, arrays[k].dtype)

    class I:  # noqa: E742
        pass
    I.n, I.n_comm = n, C
    for k, v in arrays.items():
        setattr(I, k, v)
    desc, keep = kur._desc_from(I, thr)
    h = ctypes.c_void_p()
    st = kur._lib.kur_plan_build(ctypes.byref(desc), 0, 1, 148, ctypes.byref(h))
    if st == 0:
        kur._lib.kur_plan_destroy(h)
    return st


def test_error_codes():
    # row 0: [seg comm0 ONES {1}], [seg comm1 ONES {2}]; row 1: [comm0 {0}]; row 2: [comm0 {0}]
    assert _build_status() == 0
    assert _build_status(idx=[1, 5, 0, 0]) == 2          # KUR_ERR_INDEX_RANGE
    assert _build_status(community=[0, 0, 7]) == 4      # KUR_ERR_PARTITION (label)
    assert _build_status(idx=[2, 2, 0, 0]) == 4         # column outside its segment's community
    assert _build_status(seg_comm=[0, 0, 0, 0]) == 3    # community given two segments in a row
    assert _build_status(seg_kind=[0, 3, 0, 0]) == 1    # bad kind -> INVALID_ARG
    assert _build_status(thr=1.5) == 1                  # threshold > 1
    assert _build_status(n=0) == 1                      # n < 1
    assert _build_status(idx_ptr=[0, 1, 0, 3, 4]) == 5  # idx_ptr not monotone -> SIZE_MISMATCH


def test_bad_tile_rows_flag():
    A = np.ones((4, 4), np.uint8)
    inst = kurgen.from_dense(A, [0, 0, 0, 0])
    for bad in (31, 4096, 100):
        with pytest.raises(kur.KurError) as e:
            kur.plan_export(inst, tile_rows=bad)
        assert e.value.status == 1


def test_padding_is_small_on_sbm():
    """Per-part row sorting + bank-aware arrangement keep hot padding small."""
    inst = kurgen.sbm([8192, 8192], [[0.98, 2e-4], [2e-4, 0.98]], 77)
    plan = kur.plan_export(inst, tile_rows=2048)
    assert plan["conflicts"] == 0
    assert plan["slots_hot"] <= 1.16 * plan["idx_hot"], (plan["slots_hot"], plan["idx_hot"])


def test_duplicate_and_unsorted_lists():
    A = np.ones((4, 4), np.uint8)
    inst = kurgen.from_dense(A, [0, 0, 0, 0], kind="ones")
    bad = inst.idx.copy()
    bad[1] = bad[0]  # duplicate inside row 0's segment
    inst.idx = bad
    with pytest.raises(kur.KurError) as e:
        kur.plan_export(inst)
    assert e.value.status == 3
    inst = kurgen.from_dense(A, [0, 0, 0, 0], kind="ones")
    bad = inst.idx.copy()
    bad[0], bad[1] = bad[1], bad[0]
    inst.idx = bad
    with pytest.raises(kur.KurError) as e:
        kur.plan_export(inst)
    assert e.value.status == 1


def test_library_exports_every_declared_symbol():
    """Every function include/kur.h declares is exported by libkur.so (no compute calls)."""
    import os
    hdr = open(os.path.join(os.path.dirname(__file__), "..", "include", "kur.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    names = set(re.findall(r"\b(kur_[a-z_0-9]+)\s*\(", hdr))
    assert {"kur_graph_build", "kur_rhs", "kur_step", "kur_order_parameter"} <= names
    lib = ctypes.CDLL(kur.LIB_PATH)
    for name in sorted(names):
        assert hasattr(lib, name), name
    assert set(kur.EXPORTED) <= names
    assert kur._lib.kur_status_string(9) == b"KUR_ERR_NONFINITE"


@pytest.mark.parametrize("world", [1, 3])
def test_canonical_part_order(world):
    """per tile, the nown own-community hot windows first (each lying wholly inside
    the tile's community — local at any world size), then the other hot windows, then at most
    one remote part; the order does not depend on the partition into ranks."""
    sizes = [5000, 4096, 700, 9000, 33]
    inst = kurgen.sbm(sizes, np.array(
        [[0.97, 0.002, 0.6, 0.0, 0.1], [0.002, 0.9, 0.0, 0.001, 0.0], [0.6, 0.0, 0.98, 0.0, 0.0],
         [0.0, 0.001, 0.0, 0.95, 0.02], [0.1, 0.0, 0.0, 0.02, 0.5]]), 31)
    out = kur.plan_export(inst, world=world, rank=world - 1, tile_rows=512)
    off = np.concatenate([[0], np.cumsum(sizes)])
    k = 0
    seen_remote_first = False
    for row0, nrows, comm, nparts, nhot, nown, nloc in out["tiles"]:
        w = out["part_window"][k:k + nparts]
        k += nparts
        assert 0 <= nloc <= nown <= nhot <= nparts <= nhot + 1
        assert np.all(w[:nhot] >= 0) and np.all(w[nhot:] == -1)
        for q in range(nhot):
            inside = w[q] * 4096 >= off[comm] and (w[q] + 1) * 4096 <= off[comm + 1]
            assert inside == (q < nown), (comm, q, w[q])
        seen_remote_first |= nparts > nhot
    assert seen_remote_first  # the instance exercises the remote part
    assert any(t[5] > 0 for t in out["tiles"]) and any(t[4] > t[5] for t in out["tiles"])


def test_hot_chunk_lengths_every_remainder():
    """Hot chunks hold 9 positions per 16-byte unit plus an optional 4-position tail
    (plan.h): rows of 1..27 entries inside one staged window hit every remainder
    mod 9 and both tail cases; the exported layout must still decode to A."""
    n = 27 * 32
    rng = np.random.default_rng(913)
    A = np.zeros((n, n), np.uint8)
    for j in range(n):
        L = 1 + (j % 27)
        cols = rng.choice(np.delete(np.arange(n), j), size=L, replace=False)
        A[j, cols] = 1
    inst = kurgen.from_dense(A, np.zeros(n, np.int64), kind="ones")
    plan = check_plan(inst, A, hot_min=1)
    assert plan["idx_hot"] == int(A.sum())
    assert plan["slots_hot"] >= plan["idx_hot"]


def _tiles_all_ranks(inst, world, **kw):
    """(tiles without nloc, part windows, shard_row0) over all ranks of a world-size plan."""
    tiles, windows, shards = [], [], None
    for rank in range(world):
        out = kur.plan_export(inst, rank=rank, world=world, **kw)
        tiles.append(out["tiles"][:, :6])
        windows.append(out["part_window"])
        if shards is None:
            shards = out["shard_row0"]
        assert np.array_equal(out["shard_row0"], shards)
        assert out["row_begin"] == shards[rank] and out["n_local"] == shards[rank + 1] - shards[rank]
    return np.concatenate(tiles), np.concatenate(windows), shards


@pytest.mark.parametrize("case", ["sbm_small", "complete_small", "complete_2e20", "sbm5"])
def test_tiles_independent_of_world(case):
    """The tile rule depends on the graph only: tiles, their parts and windows
    (hence the fixed reduction order and every rounding) are the same at world 1, 2 and 3;
    shards are contiguous tile ranges covering all rows (builder.cpp tile rule)."""
    if case == "sbm_small":
        inst = kurgen.sbm([1000, 1000], np.array([[0.02, 0.02], [0.02, 0.02]]), 5)
    elif case == "complete_small":
        inst = kurgen.complete_graph(5000, 7)
    elif case == "complete_2e20":
        inst = kurgen.complete_graph(1 << 20, 7)
    else:
        inst = kurgen.sbm([5000, 4096, 700, 9000, 33], np.array(
            [[0.97, 0.002, 0.6, 0.0, 0.1], [0.002, 0.9, 0.0, 0.001, 0.0], [0.6, 0.0, 0.98, 0.0, 0.0],
             [0.0, 0.001, 0.0, 0.95, 0.02], [0.1, 0.0, 0.0, 0.02, 0.5]]), 31)
    t1, w1, s1 = _tiles_all_ranks(inst, 1)
    for world in (2, 3):
        tw, ww, sw = _tiles_all_ranks(inst, world)
        assert np.array_equal(tw, t1), world
        assert np.array_equal(ww, w1), world
        assert sw[0] == 0 and sw[-1] == inst.n and np.all(np.diff(sw) >= 0)
        assert set(sw.tolist()) <= set(t1[:, 0].tolist()) | {inst.n}  # boundaries between tiles
    if case == "complete_2e20":  # one community: the rows are split, every rank has tiles
        _, _, s2 = _tiles_all_ranks(inst, 2)
        assert 0 < s2[1] < inst.n


def test_split_community_plan_decodes():
    """Shards inside a community (tile granularity): every rank's layout still decodes to A and
    nloc counts only own-community windows inside the rank's rows."""
    rng = np.random.default_rng(3)
    n = 9000
    A = (rng.random((n, n)) < 0.97).astype(np.uint8)
    np.fill_diagonal(A, 0)
    inst = kurgen.from_dense(A, np.zeros(n, np.int64), kind="zeros")
    check_plan(inst, A, world=2, split_ok=True, tile_rows=512)
    for rank in range(2):
        out = kur.plan_export(inst, rank=rank, world=2, tile_rows=512)
        rb, re_ = out["row_begin"], out["row_begin"] + out["n_local"]
        assert 0 < out["n_local"] < n
        k = 0
        for row0, nrows, comm, nparts, nhot, nown, nloc in out["tiles"]:
            w = out["part_window"][k:k + nparts]
            k += nparts
            for q in range(nown):
                inside = w[q] * 4096 >= rb and (w[q] + 1) * 4096 <= re_
                if q < nloc:
                    assert inside
            assert nloc == nown or not (w[nloc] * 4096 >= rb and (w[nloc] + 1) * 4096 <= re_)
