"""Entry-free plans (no stored entries: complete graphs, graphs of full or empty blocks) run a
whole RK4 kur_step as ONE cooperative launch (k_persist_rk4: state in registers / shared memory,
one grid barrier per stage, every CTA reducing all tile partials itself).  It must give the SAME
BITS as the general per-stage path (KUR_NO_PERSIST=1 at build): same tiles, same per-row
arithmetic (rhs_k), same summation shapes (finish_reduce's), and match the oracle."""
import numpy as np
import pytest
import torch

import kurgen
import oracle
from paper_2102_07167_b200 import kur
from tests.helpers import R_TOL, close, complex_rpsi

pytestmark = pytest.mark.gpu


def _run(inst, nsteps, re, monkeypatch, persist, scaling=None):
    if persist:
        monkeypatch.delenv("KUR_NO_PERSIST", raising=False)
    else:
        monkeypatch.setenv("KUR_NO_PERSIST", "1")
    g = kur.graph_build(inst, scaling=scaling)
    th = g.to_internal(torch.from_numpy(inst.theta0).cuda())
    om = g.to_internal(torch.from_numpy(inst.omega).cuda())
    kur.timing(g, True)
    rt = kur.step(g, th, om, inst.K, inst.h, nsteps, re, check=True)
    tm = kur.timing_read(g)
    kur.timing(g, False)
    torch.cuda.synchronize()
    out = g.to_user(th).cpu().numpy(), (rt.cpu().numpy() if rt is not None else None), tm
    g.close()
    return out


def _blocks_instance():
    # 4 communities, blocks full (p = 1) or empty (p = 0): no stored entries, several dense column
    # communities per row community (T_a sums of several S_b), one community of > 64 tiles
    P = np.array([[1.0, 0.0, 1.0, 0.0], [0.0, 1.0, 0.0, 1.0], [1.0, 0.0, 1.0, 1.0], [0.0, 1.0, 1.0, 1.0]])
    return kurgen.sbm([200000, 30000, 5000, 77], P, 17, K=2.5, h=0.01)


@pytest.mark.parametrize("case", ["complete_300k", "blocks", "cfg2"])
def test_persist_bitwise_equals_general_path(case, monkeypatch):
    if case == "complete_300k":
        inst = kurgen.complete_graph(300000, 21, K=3.0, h=0.01)
    elif case == "blocks":
        inst = _blocks_instance()
    else:
        inst = kurgen.config(2)
    a_th, a_rt, a_tm = _run(inst, 7, 3, monkeypatch, persist=True)
    b_th, b_rt, b_tm = _run(inst, 7, 3, monkeypatch, persist=False)
    assert a_tm["prologue_n"] == 0 and a_tm["stage_n"] == 28  # one launch did all 28 stages
    assert b_tm["prologue_n"] == 1
    assert np.array_equal(a_th, b_th)
    assert np.array_equal(a_rt, b_rt) and a_rt.shape == (3, 2)


def test_persist_degree_scaling_and_edge_cases(monkeypatch):
    inst = _blocks_instance()
    a_th, a_rt, _ = _run(inst, 4, 1, monkeypatch, persist=True, scaling=1)
    b_th, b_rt, _ = _run(inst, 4, 1, monkeypatch, persist=False, scaling=1)
    assert np.array_equal(a_th, b_th) and np.array_equal(a_rt, b_rt)
    th0, rt0, _ = _run(inst, 0, 1, monkeypatch, persist=True)  # nsteps = 0: theta unchanged, r(0) recorded
    assert np.array_equal(th0, inst.theta0) and rt0.shape == (1, 2)
    assert abs(complex_rpsi(rt0)[0] - np.exp(1j * inst.theta0).mean()) <= 1e-12


def test_persist_matches_oracle(monkeypatch):
    inst = _blocks_instance()
    og = oracle.Graph(inst)
    th, rt, _ = _run(inst, 10, 1, monkeypatch, persist=True)
    _, th10, rt_ref = oracle.rk4(og, inst.theta0, inst.omega, inst.K, inst.h, 10, 1, mode="matvec")
    ok, err = close(th, th10)
    assert ok, err
    assert np.max(np.abs(complex_rpsi(rt) - complex_rpsi(rt_ref))) <= R_TOL


def test_persist_nonfinite_flag(monkeypatch):
    inst = kurgen.complete_graph(50000, 3, K=1.0, h=0.01)
    inst.omega = inst.omega.copy()
    inst.omega[123] = np.inf
    monkeypatch.delenv("KUR_NO_PERSIST", raising=False)
    g = kur.graph_build(inst)
    th = g.to_internal(torch.from_numpy(inst.theta0).cuda())
    om = g.to_internal(torch.from_numpy(inst.omega).cuda())
    with pytest.raises(kur.KurError) as e:
        kur.step(g, th, om, inst.K, inst.h, 2, 0, check=True)
    assert e.value.status == 9
    g.close()
