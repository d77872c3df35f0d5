"""Cold vs warm CoupledStepper.run on config 2 (K = 20000); AS_BENCH=1 replays bench.py's order."""
import math, time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_1406_6923_b200 import CoupledStepper, Probe, SourceTerm, build_models, cfl_estimate_coupled, make_probe, project_source
from paper_1406_6923_b200.pulses import ricker
wl, ops, alphas, (sa, sr), node_rx = bench._workload(2)
rows = {sa: [sr]}
for a, r in node_rx: rows.setdefault(a, []).append(r)
models = build_models(ops, wl.modes_per_face, wl.n, wl.shift, rows=rows)
lam, _ = cfl_estimate_coupled(models)
dt = 0.9 * 2 / math.sqrt(lam)
probes = []
for alpha, face in wl.face_receivers:
    for q in range(wl.modes_per_face):
        wts = np.zeros(models[alpha].state_size); wts[face * wl.modes_per_face + q] = 1.0
        probes.append(Probe(alpha, wts))
for a, r in node_rx: probes.append(make_probe(models[a], r))
src = SourceTerm(sa, project_source(models[sa], sr), ricker(wl.f0, wl.delay))
st = CoupledStepper(models, dt, sources=(src,))
st.initialize(_probes=probes)
K = 20000
lib = st._lib
orig = lib.sfw_step_run
T = {}
def run_wrap(*a):
    t0 = time.perf_counter(); r = orig(*a); T["sfw_step_run"] = time.perf_counter() - t0; return r
lib.sfw_step_run = run_wrap
orig_res = lib.sfw_step_run_resident
import ctypes as C
from paper_1406_6923_b200 import _lib
if os.environ.get("AS_BENCH"):  # the bench's order: resident kernel-only launch, L2 flush, then run()
    prof_k = np.ascontiguousarray(np.array([[src.profile(k * dt) for k in range(K)]]))
    ms = C.c_float(0.0)
    eb = _lib.errbuf()
    _lib.check(orig_res(st._h, K, 1, _lib.dptr(prof_k), C.byref(ms), eb, 1024), eb)
    print("resident kernel ms", ms.value)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    flush.fill_(1.0)
torch.cuda.synchronize()
t0 = time.perf_counter(); st.run(K, probes=probes); w1 = time.perf_counter() - t0
print("cold run wall", w1, T)
t0 = time.perf_counter(); st.run(K, probes=probes); w2 = time.perf_counter() - t0
print("warm run wall", w2, T)
a = np.empty((20001, 264)); t0 = time.perf_counter(); a[:] = 1.0; print("first-touch 42MB", time.perf_counter() - t0)
