"""Cycle accounting of the default multi-shot kernel k_step_ms2 (config 4).

Needs a library built with -DSFW_MS_CLK; run with SFW_B200_LIB pointing at it:
    SFW_B200_LIB=build/clk/libsfw_b200_clk.so SFW_STEP_PROF=1 python tools/ms2_prof.py
Per compute warp: [chain-block wait, state-block wait, gemm, total, flags, phase C, tail].
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
from paper_1406_6923_b200 import CoupledStepper, SourceTerm, _lib, build_models, cfl_estimate_coupled, project_source
from paper_1406_6923_b200.configs import locate, make_workload
from paper_1406_6923_b200.pulses import ricker

wl, ops, alphas, _, _ = bench._workload(3)
wl4 = make_workload(4)
rows = {}
for ijk in wl4.sources:
    a, r = locate(ijk, wl4.counts, wl4.p)
    rows.setdefault(a, []).append(r)
n_sub, w, L = len(ops), wl.width, wl.layers
dev = [torch.empty(n_sub * L * w * w, dtype=torch.float64, device="cuda") for _ in range(3)]
ptrs = tuple(t.data_ptr() for t in dev)
models = build_models(ops, wl.modes_per_face, wl.n, wl.shift, rows=rows, device_out=ptrs)
scl = dev[2].view(n_sub, L, w, w)
idx = {a: i for i, a in enumerate(alphas)}
for a in rows:
    models[a].scales = scl[idx[a]].cpu().numpy()
lam, _ = cfl_estimate_coupled(models, device_coefficients=ptrs)
dt = 0.9 * 2.0 / math.sqrt(lam)
shots = []
for ijk in wl4.sources:
    a, r = locate(ijk, wl4.counts, wl4.p)
    shots.append(SourceTerm(a, project_source(models[a], r), ricker(wl4.f0, wl4.delay)))
st = CoupledStepper(models, dt, device_coefficients=ptrs)
st.run_shots(3, shots)
K = 20
st.run_shots(K, shots)
print("ms/step", st.last_kernel_ms / K)
lib = _lib.load()
buf = (C.c_ulonglong * (148 * 16 * 8))()
lib.sfw_step_debug_prof(st._h, buf, 148 * 16 * 8)
a = np.frombuffer(buf, dtype=np.uint64).reshape(148, 16, 8).astype(float) / K
if os.environ.get("SFW_MS2") is None:  # k_step_ms4: 8 compute warps per CTA
    a = a[:, :8, :]
names = ["c-wait", "s-wait", "gemm", "total", "flags", "C", "tail"]
for i, nm in enumerate(names):
    print(f"{nm:7s} mean {a[..., i].mean():10.0f}  max {a[..., i].max():10.0f}  frac {a[..., i].mean() / a[..., 3].mean():.3f}")
