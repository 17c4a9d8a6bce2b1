"""Shared helpers for the GPU parity tests: run the CUDA path through the C-ABI
binding and bring results back in USER order for comparison with oracle/."""
import numpy as np
import torch

from paper_2102_07167_b200 import kur

# north_star tolerances (BASELINE.json): per RHS / theta after 10 steps
ABS_TOL = 1e-9
REL_TOL = 1e-12
R_TOL = 1e-9  # complex order parameter r e^{i psi} along the trajectory


def close(gpu, ref, abs_tol=ABS_TOL, rel_tol=REL_TOL):
    gpu = np.asarray(gpu)
    ref = np.asarray(ref)
    err = np.abs(gpu - ref)
    ok = err <= abs_tol + rel_tol * np.abs(ref)
    return bool(np.all(ok)), float(err.max()) if err.size else 0.0


def complex_rpsi(rt):
    rt = np.asarray(rt)
    return rt[:, 0] * np.exp(1j * rt[:, 1])


class Run:
    """A built graph plus the instance's theta0/omega on the device (internal order)."""

    def __init__(self, inst, **kw):
        self.inst = inst
        self.g = kur.graph_build(inst, **kw)
        dev = f"cuda:{self.g.device}"
        self.theta_int = self.g.to_internal(torch.from_numpy(np.ascontiguousarray(inst.theta0)).to(dev))
        self.omega_int = self.g.to_internal(torch.from_numpy(np.ascontiguousarray(inst.omega)).to(dev))

    def user(self, x_int):
        out = np.empty(self.inst.n)
        out[self.g.perm] = x_int.detach().cpu().numpy()
        return out

    def rhs(self, theta_user=None, K=None):
        th = self.theta_int if theta_user is None else self.g.to_internal(
            torch.from_numpy(np.ascontiguousarray(theta_user)).to(self.theta_int.device))
        f = kur.rhs(self.g, th, self.omega_int, self.inst.K if K is None else K)
        return self.user(f)

    def step(self, nsteps, record_every=1, K=None, h=None, theta_user=None):
        th = (self.theta_int if theta_user is None else self.g.to_internal(
            torch.from_numpy(np.ascontiguousarray(theta_user)).to(self.theta_int.device))).clone()
        rt = kur.step(self.g, th, self.omega_int, self.inst.K if K is None else K,
                      self.inst.h if h is None else h, nsteps, record_every, check=True)
        torch.cuda.synchronize()
        return self.user(th), (rt.cpu().numpy() if rt is not None else None)

    def order_parameter(self, theta_user=None, local=False):
        th = self.theta_int if theta_user is None else self.g.to_internal(
            torch.from_numpy(np.ascontiguousarray(theta_user)).to(self.theta_int.device))
        out = kur.order_parameter(self.g, th, local=local)
        if local:
            return out[0].cpu().numpy(), out[1].cpu().numpy()
        return out.cpu().numpy()
