"""Host-side breakdown of CoupledStepper.run_shots(K, 32 shots, 2312 probes) at config 4.
    python tools/e2e_prof4.py [K]   (on a B200)"""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
from paper_1406_6923_b200 import CoupledStepper, SourceTerm, project_source  # noqa: E402
from paper_1406_6923_b200 import stepper as S  # noqa: E402
from paper_1406_6923_b200.configs import locate, make_workload  # noqa: E402
from paper_1406_6923_b200.pulses import ricker  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
wl4 = make_workload(4)
pp = bench.prepare(3, extra_rows=wl4.sources)
models = pp["models"]
shots = [SourceTerm(a, project_source(models[a], r), ricker(wl4.f0, wl4.delay))
         for a, r in (locate(ijk, wl4.counts, wl4.p) for ijk in wl4.sources)]
st = CoupledStepper(models, pp["dt"], device_coefficients=pp["ptrs"])
st.run_shots(5, shots, probes=pp["probes"])
T = {}
lib = st._lib
orig = lib.sfw_shots_run


def w(*a):
    t0 = time.perf_counter()
    r = orig(*a)
    T["sfw_shots_run"] = T.get("sfw_shots_run", 0) + time.perf_counter() - t0
    return r


lib.sfw_shots_run = w
opt = S.profile_table


def pt(*a, **k):
    t0 = time.perf_counter()
    r = opt(*a, **k)
    T["profile_table"] = T.get("profile_table", 0) + time.perf_counter() - t0
    return r


S.profile_table = pt
out = []
for rep in range(3):
    T.clear()
    t0 = time.perf_counter()
    st.run_shots(K, shots, probes=pp["probes"])
    out.append({"wall_ms": (time.perf_counter() - t0) * 1e3, "kernel_ms": st.last_kernel_ms,
                **{k: round(v * 1e3, 3) for k, v in T.items()}})
print(json.dumps(out))
