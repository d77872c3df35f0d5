import os, sys, math, ctypes as C
sys.path.insert(0, os.getcwd())
os.environ["SFW_MS3"] = "2,3"
os.environ["SFW_STEP_PROF"] = "1"
import numpy as np, torch
import bench
from paper_1406_6923_b200 import CoupledStepper, SourceTerm, build_models, cfl_estimate_coupled, project_source, _lib
from paper_1406_6923_b200.configs import locate, make_workload
from paper_1406_6923_b200.pulses import ricker
wl, ops, alphas, (sa, sr), _ = bench._workload(3)
wl4 = make_workload(4)
rows = {}
for ijk in wl4.sources:
    a, r = locate(ijk, wl4.counts, wl4.p); rows.setdefault(a, []).append(r)
n_sub, w, L = len(ops), wl.width, wl.layers
dev = [torch.empty(n_sub * L * w * w, dtype=torch.float64, device="cuda") for _ in range(3)]
ptrs = tuple(t.data_ptr() for t in dev)
models = build_models(ops, wl.modes_per_face, wl.n, wl.shift, rows=rows, device_out=ptrs)
scl = dev[2].view(n_sub, L, w, w); idx = {a: i for i, a in enumerate(alphas)}
for a in rows: models[a].scales = scl[idx[a]].cpu().numpy()
lam, conv = cfl_estimate_coupled(models, device_coefficients=ptrs)
dt = 0.9 * 2.0 / math.sqrt(lam)
shots = []
for ijk in wl4.sources:
    a, r = locate(ijk, wl4.counts, wl4.p)
    shots.append(SourceTerm(a, project_source(models[a], r), ricker(wl4.f0, wl4.delay)))
st = CoupledStepper(models, dt, device_coefficients=ptrs)
st.run_shots(3, shots)
st.run_shots(20, shots)
print("ms/step", st.last_kernel_ms / 20, "clock GHz ~", 1.965)
lib = _lib.load()
lib.sfw_step_debug_prof.restype = C.c_int
buf = (C.c_ulonglong * (148 * 16 * 8))()
g = lib.sfw_step_debug_prof(C.c_void_p(st._h.value if hasattr(st._h, 'value') else st._h), buf, 148 * 16 * 8)
a = np.frombuffer(buf, dtype=np.uint64)[:148 * 8 * 8].reshape(148, 8, 8)[:, :, :6].astype(float)
tot = a[..., 3]
print("grid", g, "mean fractions acq/gemm/coup:", (a[..., 0] / tot).mean(), (a[..., 1] / tot).mean(), (a[..., 2] / tot).mean())
print("total cycles per step (mean, max):", tot.mean() / 20, tot.max() / 20)
print("gemm cycles per step per warp:", a[..., 1].mean() / 20)
busy = tot - a[..., 2]
print("per-step cycles: busy (total - coupling) mean/max", busy.mean() / 20, busy.max() / 20,
      " gemm mean/max", a[..., 1].mean() / 20, a[..., 1].max() / 20, " acquire mean/max", a[..., 0].mean() / 20, a[..., 0].max() / 20)
print("wait_group mean/max", a[..., 4].mean() / 20, a[..., 4].max() / 20, " F0 store+fence mean/max", a[..., 5].mean() / 20, a[..., 5].max() / 20)
