"""Input generator checks: determinism, symmetry, no
self-loops, partition consistency, and the segment-format contract."""
import numpy as np

import kurgen


def _check_format(inst):
    n = inst.n
    assert inst.seg_ptr.shape == (n + 1,) and inst.seg_ptr[0] == 0
    assert inst.idx_ptr[-1] == inst.nidx
    for u in range(n):
        segs = range(inst.seg_ptr[u], inst.seg_ptr[u + 1])
        comms = [int(inst.seg_comm[s]) for s in segs]
        assert comms == sorted(set(comms))
        for s in segs:
            lst = inst.idx[inst.idx_ptr[s]:inst.idx_ptr[s + 1]]
            assert np.all(np.diff(lst) > 0)
            assert np.all(inst.community[lst] == inst.seg_comm[s])
            assert u not in lst


def test_determinism_and_sha():
    a = kurgen.sbm([50, 30, 20], [[0.9, 0.05, 0.0], [0.05, 0.3, 0.7], [0.0, 0.7, 0.99]], 17)
    b = kurgen.sbm([50, 30, 20], [[0.9, 0.05, 0.0], [0.05, 0.3, 0.7], [0.0, 0.7, 0.99]], 17)
    c = kurgen.sbm([50, 30, 20], [[0.9, 0.05, 0.0], [0.05, 0.3, 0.7], [0.0, 0.7, 0.99]], 18)
    assert a.sha256() == b.sha256()
    assert a.sha256() != c.sha256()


def test_sbm_symmetric_no_self_loops_partition():
    sizes = [64, 33, 1, 0, 20]
    P = np.array([[0.97, 0.02, 0.5, 0.0, 0.6], [0.02, 0.4, 0.0, 0.0, 0.0],
                  [0.5, 0.0, 0.0, 0.0, 0.0], [0.0, 0.0, 0.0, 0.0, 0.0], [0.6, 0.0, 0.0, 0.0, 0.1]])
    inst = kurgen.sbm(sizes, P, 5)
    _check_format(inst)
    A = inst.dense()
    assert (A == A.T).all()
    assert np.diag(A).sum() == 0
    assert np.bincount(inst.community, minlength=5).tolist() == sizes
    # dense (p > 0.5) blocks are emitted as KUR_ZEROS segments
    perm = inst.meta["perm_internal_to_user"]
    u0 = perm[0]  # internal node 0 is in community 0
    kinds = {int(inst.seg_comm[s]): int(inst.seg_kind[s]) for s in range(inst.seg_ptr[u0], inst.seg_ptr[u0 + 1])}
    assert kinds[0] == kurgen.KUR_ZEROS and kinds[4] == kurgen.KUR_ZEROS


def test_sbm_density_matches_p():
    inst = kurgen.sbm([400, 400], [[0.9, 0.1], [0.1, 0.3]], 3)
    A = inst.dense().astype(np.float64)
    lab = inst.community
    d00 = A[np.ix_(lab == 0, lab == 0)].sum() / (400 * 399)
    d01 = A[np.ix_(lab == 0, lab == 1)].mean()
    d11 = A[np.ix_(lab == 1, lab == 1)].sum() / (400 * 399)
    assert abs(d00 - 0.9) < 0.01 and abs(d01 - 0.1) < 0.01 and abs(d11 - 0.3) < 0.01


def test_complete_graph():
    inst = kurgen.complete_graph(10, 1)
    assert inst.nidx == 0 and inst.nseg == 10
    A = inst.dense()
    assert (A == 1 - np.eye(10, dtype=np.uint8)).all()


def test_from_dense_roundtrip():
    A, labels = kurgen.random_dense(60, 4, seed=2, symmetric=False)
    for kind in ("ones", "zeros", "auto", "random"):
        inst = kurgen.from_dense(A, labels, kind=kind, seed=1)
        _check_format(inst)
        assert (inst.dense() == A).all()


def test_config_shapes_small():
    i1 = kurgen.config(1)
    assert i1.n == 1000 and i1.nidx == 0 and i1.K == 2.0 and i1.nsteps == 50
    i3 = kurgen.config(3)
    assert i3.n == 65536 and i3.n_comm == 16
    assert 1.6e7 < i3.nidx < 1.9e7  # ~1.745e7
    sizes, P, pairs = kurgen._config4_blocks(kurgen.SEED_BASE + 4)
    assert sizes.sum() == 262144 and len(sizes) == 64 and len(pairs) == 8
    assert sizes.min() > 300 and sizes.max() < 20000
    assert set(np.round(np.diag(P), 2)) <= {0.99, 0.6, 0.05}


def test_cauchy_truncated():
    w = kurgen.cauchy_trunc(1, 1, 100000, 10.0)
    assert np.all(np.abs(w) < 10)
    # median |w| of a standard Cauchy conditioned on |w|<10 is tan(pi/2 * P(|C|<10)/2 ...) ~ 0.94
    assert 0.85 < np.median(np.abs(w)) < 1.05
