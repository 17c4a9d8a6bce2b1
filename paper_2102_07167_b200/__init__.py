"""paper_2102_07167_b200 — B200-native hot path of Böhle, Kuehn & Thalhammer
(arXiv 2102.07167): the Kuramoto-on-graphs right-hand side through localised
order parameters inside fixed-step RK4, as a C-ABI library (libkur.so,
include/kur.h) with sm_100a kernels and this thin binding.
"""
from .kur import (Graph, KurError, graph_build, rhs, step, order_parameter, check,  # noqa: F401
                  nccl_unique_id, LIB_PATH, EXPORTED)
