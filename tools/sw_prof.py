"""Cycle accounting of the config-2 stepping kernel k_step_sw (library built with -DSFW_LW_CLK).

    SFW_B200_LIB=build/lwclk/libsfw.so SFW_STEP_PROF=1 python tools/sw_prof.py
Phases (per warp, per step): 0 x-build, 1 layer-1 flux + mailbox put, 2 record, 3 other fluxes,
4 phase-2 products, 5 interior leapfrogs, 6 mailbox wait, 7 layer-1 coupling + leapfrog.
"""
import ctypes as C
import math
import os
import sys

sys.path.insert(0, os.getcwd())
os.environ.setdefault("SFW_STEP_PROF", "1")
import numpy as np
import torch

import bench
from paper_1406_6923_b200 import CoupledStepper, _lib, build_models, cfl_estimate_coupled

wl, ops, alphas, _, _ = bench._workload(2)
n_sub, w, L = len(ops), wl.width, wl.layers
dev = [torch.empty(n_sub * L * w * w, dtype=torch.float64, device="cuda") for _ in range(3)]
ptrs = tuple(t.data_ptr() for t in dev)
models = build_models(ops, wl.modes_per_face, wl.n, wl.shift, device_out=ptrs)
lam, _ = cfl_estimate_coupled(models, device_coefficients=ptrs)
st = CoupledStepper(models, 0.9 * 2.0 / math.sqrt(lam), device_coefficients=ptrs)
st.initialize()
ms = C.c_float(0.0)
eb = _lib.errbuf()
K = 2000
_lib.check(st._lib.sfw_step_run_resident(st._h, 50, 1, None, C.byref(ms), eb, 1024), eb)
_lib.check(st._lib.sfw_step_run_resident(st._h, K, 1, None, C.byref(ms), eb, 1024), eb)
print("us/step", 1e3 * ms.value / K)
lib = _lib.load()
n = 148 * 8 * 16
buf = (C.c_ulonglong * n)()
lib.sfw_step_debug_prof(st._h, buf, n)
a = np.frombuffer(buf, dtype=np.uint64).reshape(148, 8, 16)[:, :, :10].astype(float) / K
live = a.sum(axis=-1) > 0
tot = a[live].sum(axis=-1)
print("cycles/step per warp: mean", tot.mean(), "max", tot.max())
for ph in range(8):
    v = a[live][:, ph]
    print(f"phase {ph}: mean {v.mean():8.0f}  max {v.max():8.0f}  frac {v.mean() / tot.mean():.3f}")
