"""Kernel time of the config-4 multi-shot launch (run_shots, K steps) for A/B of library variants;
prints ms/step.  Ignores the growth detector (timing experiments may feed the kernel fake data).
    SFW_B200_LIB=build/ab/<v>/libsfw_b200.so python tools/ms2_time.py [K]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
from paper_1406_6923_b200 import CoupledStepper, SourceTerm, project_source  # noqa: E402
from paper_1406_6923_b200.configs import locate, make_workload  # noqa: E402
from paper_1406_6923_b200.pulses import ricker  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
wl4 = make_workload(4)
pp = bench.prepare(3, extra_rows=wl4.sources)
models = pp["models"]
shots = []
for ijk in wl4.sources:
    a, r = locate(ijk, wl4.counts, wl4.p)
    shots.append(SourceTerm(a, project_source(models[a], r), ricker(wl4.f0, wl4.delay)))
st = CoupledStepper(models, pp["dt"], device_coefficients=pp["ptrs"])
res = []
for rep in range(3):
    try:
        st.run_shots(K, shots, probes=pp["probes"])
    except Exception as exc:  # noqa: BLE001
        if "diverged" not in str(exc):
            raise
    res.append(st.last_kernel_ms / K)
print(os.environ.get("SFW_B200_LIB", "default"), "ms/step", min(res), res)
