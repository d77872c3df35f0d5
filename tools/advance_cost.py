"""Per-launch cost of k_step_sw at config 2: CUDA-event time of launches of 1, 20, 200 and 2000 steps
(the fixed per-launch cost is the intercept), and the wall time of CoupledStepper.advance()."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1406_6923_b200 import CoupledStepper, _lib  # noqa: E402

pp = bench.prepare(2)
st = CoupledStepper(pp["models"], pp["dt"], sources=(pp["src"],), device_coefficients=pp["ptrs"])
st.initialize(_probes=pp["probes"])
eb = _lib.errbuf()
ms = C.c_float(0.0)
out = {}
for n in (1, 20, 200, 2000):
    prof = st._profile_steps(0, n)
    vals = []
    for _ in range(5):
        _lib.check(st._lib.sfw_step_run_resident(st._h, n, 1, _lib.dptr(prof), C.byref(ms), eb, 1024), eb)
        vals.append(ms.value * 1e3)
    out[f"launch_{n}_us"] = min(vals)
st.run(1, probes=pp["probes"])
for _ in range(10):
    st.advance()
t0 = time.perf_counter()
for _ in range(200):
    st.advance()
out["advance_wall_us"] = (time.perf_counter() - t0) / 200 * 1e6
a = np.array([[1, 20, 200, 2000]], float).T
y = np.array([out[f"launch_{n}_us"] for n in (1, 20, 200, 2000)])
coef = np.linalg.lstsq(np.hstack([np.ones_like(a), a]), y, rcond=None)[0]
out["fit_fixed_us"], out["fit_per_step_us"] = coef
print(json.dumps(out))
