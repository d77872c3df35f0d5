"""Host-side breakdown of CoupledStepper.run on config 2 (K = 20000, 264 probes) and the chunk count
(SFW_NCHUNK) of the overlapped row download.   python tools/e2e_prof.py   (on a B200)
"""
import math, time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_1406_6923_b200 import CoupledStepper, Probe, SourceTerm, build_models, cfl_estimate_coupled, make_probe, project_source
from paper_1406_6923_b200 import stepper as S
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
st.run(200, probes=probes)
T = {}
def wrap(obj, name):
    f = getattr(obj, name)
    def g(*a, **k):
        t0 = time.perf_counter(); r = f(*a, **k); T[name] = T.get(name, 0) + time.perf_counter() - t0; return r
    setattr(obj, name, g)
for n in ("initialize", "_profile_steps", "_limits", "_set_probes"):
    wrap(st, n)
lib = st._lib
orig = lib.sfw_step_run
def run_wrap(*a):
    t0 = time.perf_counter(); r = orig(*a); T["sfw_step_run"] = time.perf_counter() - t0; return r
lib.sfw_step_run = run_wrap
oi = lib.sfw_step_init
def init_wrap(*a):
    t0 = time.perf_counter(); r = oi(*a); T["sfw_step_init"] = time.perf_counter() - t0; return r
lib.sfw_step_init = init_wrap
K = 20000
torch.cuda.synchronize()
t0 = time.perf_counter(); st.run(K, probes=probes); wall = time.perf_counter() - t0
print("wall", wall, {k: round(v * 1e3, 2) for k, v in T.items()})
t0 = time.perf_counter(); st.run(K, probes=probes); wall = time.perf_counter() - t0
print("wall2", wall)
for env in ("SFW_NO_CHUNK", "SFW_NCHUNK=4", "SFW_NCHUNK=8", "SFW_NCHUNK=16"):
    k, _, v = env.partition("=")
    os.environ[k] = v or "1"
    t0 = time.perf_counter(); st.run(K, probes=probes); wall = time.perf_counter() - t0
    print(env, "wall", wall, "sfw_step_run", T["sfw_step_run"])
    del os.environ[k]
