"""Cycle accounting of the layer-split config-2 kernel k_step_sw4 (library built with -DSFW_LW_CLK).

    tools/build_variant.sh lwclk -DSFW_LW_CLK
    SFW_B200_LIB=build/lwclk/libsfw.so SFW_STEP_PROF=1 SFW_SW_NLW=2 python tools/sw4_prof.py
Phases (per warp, per step): 0 P1 x + flux products (+ mailbox put), 1 record (warp 0), 2 barrier A,
3 P2 products, 4 mailbox wait (warp 0), 5 coupling + leapfrog, 6 barrier B.
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
NWMAX = 32
n = 148 * NWMAX * 16
buf = (C.c_ulonglong * n)()
lib.sfw_step_debug_prof(st._h, buf, n)
nq = int(os.environ.get("SW4_NQ", "4"))
raw = np.frombuffer(buf, dtype=np.uint64)
nw = 4 * nq
a = raw[: 148 * nw * 16].reshape(148, nw, 16)[:, :, :8].astype(float) / K
for q in range(nq):
    sel = a[:, q::nq, :]
    live = sel.sum(axis=-1) > 0
    v = sel[live]
    print(f"warp {q}: total {v.sum(axis=-1).mean():7.0f} cycles/step  " +
          " ".join(f"p{ph}={v[:, ph].mean():6.0f}" for ph in range(7)))
