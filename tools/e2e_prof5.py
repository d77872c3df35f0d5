"""Host-side breakdown of CoupledStepper.run(K, 9224 probes) at config 5 (the bench's e2e call).
    python tools/e2e_prof5.py [K]   (on a B200)"""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
from paper_1406_6923_b200 import CoupledStepper  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
pp = bench.prepare(5)
st = CoupledStepper(pp["models"], pp["dt"], sources=(pp["src"],), device_coefficients=pp["ptrs"])
probes = pp["probes"]
st.run(5, probes=probes)
T = {}


def wrap(obj, name):
    f = getattr(obj, name)

    def g(*a, **k):
        t0 = time.perf_counter()
        r = f(*a, **k)
        T[name] = T.get(name, 0) + time.perf_counter() - t0
        return r
    setattr(obj, name, g)


for n in ("initialize", "_profile_steps", "_limits", "_set_probes", "_profiles"):
    wrap(st, n)
lib = st._lib
for n in ("sfw_step_run", "sfw_step_init"):
    orig = getattr(lib, n)

    def mk(orig, n):
        def w(*a):
            t0 = time.perf_counter()
            r = orig(*a)
            T[n] = T.get(n, 0) + time.perf_counter() - t0
            return r
        return w
    setattr(lib, n, mk(orig, n))
out = []
for rep in range(3):
    T.clear()
    t0 = time.perf_counter()
    st.run(K, probes=probes)
    wall = time.perf_counter() - t0
    out.append({"wall_ms": wall * 1e3, **{k: round(v * 1e3, 3) for k, v in T.items()}})
print(json.dumps(out))
