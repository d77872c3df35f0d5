"""Debug: which fp32 W-form probe rows stay unwritten (run with SFW_POISON=w; FP64_FIRST=1 replays the
full-size test order)."""
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import test_fullsize_gpu as T
wl, models, dt, src, probes = T._build(2)
from paper_1406_6923_b200 import CoupledStepper
N = int(os.environ.get("NSTEPS", "400"))
if os.environ.get("FP64_FIRST"):
    with CoupledStepper(models, dt, sources=(src,)) as st:
        _, r1 = st.run(N, probes=probes)
with CoupledStepper(models, dt, sources=(src,), precision="fp32") as st32:
    _, r32 = st32.run(N, probes=probes)
bad = np.argwhere(~np.isfinite(r32))
print("shape", r32.shape, "nan count", len(bad))
print("rows with nan", np.unique(bad[:, 0])[:20], "cols", np.unique(bad[:, 1])[:40])
print("n probes", len(probes), "probe subdomains of nan cols", sorted(set(probes[c].alpha for c in np.unique(bad[:, 1])))[:10])
