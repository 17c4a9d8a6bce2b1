"""kur_step / kur_step_method with theta (and omega) in HOST memory -- the end-to-end
path bench.py times: the library copies theta in, runs the same kernels, and stores
theta_{n+1} back (pinned memory: written by the last step's final stage through the
device mapping; pageable memory, the implicit midpoint commit and the single-CTA path:
one copy after the steps).  Results must be bitwise those of the device-buffer call."""
import numpy as np
import pytest
import torch

import kurgen
from paper_2102_07167_b200 import kur

pytestmark = pytest.mark.gpu


def _device_run(g, th0, om, inst, method, nsteps):
    th = th0.clone()
    rt = kur.step_method(g, method, th, om, inst.K, inst.h, nsteps, 1)
    torch.cuda.synchronize()
    return th.cpu(), rt.cpu()


def _instance(which):
    if which == "sbm":  # short lists: theta goes back with one copy after the steps
        return kurgen.sbm([700, 900, 400], [[0.9, 0.01, 0.02], [0.01, 0.7, 0.0], [0.02, 0.0, 0.95]], 31, K=3.0)
    if which == "long":  # long lists (~700 entries per row): the final stage stores through the mapping
        return kurgen.sbm([2000, 2000], [[0.3, 0.05], [0.05, 0.3]], 34, K=3.0)
    return kurgen.sbm([20, 13], [[0.8, 0.1], [0.1, 0.9]], 32, K=2.0)  # single-CTA path


@pytest.mark.parametrize("which", ["sbm", "long", "tiny"])
@pytest.mark.parametrize("method", ["rk4", "euler", "heun", "implicit_midpoint"])
@pytest.mark.parametrize("pinned", [True, False])
@pytest.mark.parametrize("omega_host", [False, True])
def test_host_theta_matches_device(which, method, pinned, omega_host):
    inst = _instance(which)
    g = kur.graph_build(inst)
    if which == "long":  # the rule in api.cpp host_step: kernel bytes per RHS >= 60 x the bytes of theta
        assert g.info["bytes_per_rhs"] >= 60 * 8 * g.n_local
    elif which == "sbm":
        assert g.info["bytes_per_rhs"] < 60 * 8 * g.n_local
    th0 = g.to_internal(torch.from_numpy(inst.theta0).cuda())
    om = g.to_internal(torch.from_numpy(inst.omega).cuda())
    want_th, want_rt = _device_run(g, th0, om, inst, method, 3)
    th_h = th0.cpu()
    if pinned:
        th_h = th_h.pin_memory()
    om_arg = om.cpu() if omega_host else om
    if method == "rk4":
        rt = kur.step(g, th_h, om_arg, inst.K, inst.h, 3, 1)
    else:
        rt = kur.step_method(g, method, th_h, om_arg, inst.K, inst.h, 3, 1)
    torch.cuda.synchronize()
    assert torch.equal(th_h, want_th)
    assert torch.equal(rt.cpu(), want_rt)
    # again on the same handle (reused device buffers), zero steps leave theta untouched
    th_h2 = th0.cpu().pin_memory() if pinned else th0.cpu()
    kur.step(g, th_h2, om_arg, inst.K, inst.h, 0)
    torch.cuda.synchronize()
    assert torch.equal(th_h2, th0.cpu())


def test_host_theta_nonfinite_is_reported():
    inst = kurgen.sbm([600, 600], [[0.9, 0.01], [0.01, 0.9]], 33, K=1.0)
    g = kur.graph_build(inst)
    th = g.to_internal(torch.from_numpy(inst.theta0).cuda()).cpu().pin_memory()
    th[5] = float("nan")
    om = g.to_internal(torch.from_numpy(inst.omega).cuda())
    with pytest.raises(kur.KurError):
        kur.step(g, th, om, inst.K, inst.h, 1, check=True)
