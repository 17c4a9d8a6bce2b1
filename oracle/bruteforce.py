"""Brute-force checkers for tiny inputs (N <= 64) — TEST INFRASTRUCTURE ONLY.

Independent of kur_oracle.c: works on a dense 0/1 matrix and evaluates the
definition (PAPER.md P:388 with uniform scaling M_m = M)

    f_m = omega_m + (K/M) * sum_{l != m} A_ml sin(theta_l - theta_m)

either with a correctly rounded sum of libm terms (math.fsum) or entirely in
50-digit arithmetic (mpmath).  Used by pin O2 (tests/test_oracle_pins.py).
"""
from __future__ import annotations

import math

import mpmath
import numpy as np


def rhs_fsum(A, theta, omega, K):
    A = np.asarray(A)
    n = A.shape[0]
    out = np.empty(n)
    for m in range(n):
        terms = [math.sin(theta[l] - theta[m]) for l in range(n) if l != m and A[m, l]]
        out[m] = omega[m] + (K / n) * math.fsum(terms)
    return out


def rhs_mp(A, theta, omega, K, dps=50):
    A = np.asarray(A)
    n = A.shape[0]
    with mpmath.workdps(dps):
        th = [mpmath.mpf(float(t)) for t in theta]
        out = []
        for m in range(n):
            s = mpmath.fsum(mpmath.sin(th[l] - th[m]) for l in range(n) if l != m and A[m, l])
            out.append(mpmath.mpf(float(omega[m])) + mpmath.mpf(float(K)) / n * s)
        return out


def order_parameter_mp(theta, dps=50):
    with mpmath.workdps(dps):
        n = len(theta)
        z = mpmath.fsum(mpmath.expj(mpmath.mpf(float(t))) for t in theta) / n
        return z  # complex r e^{i psi}
