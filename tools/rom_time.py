"""Wall time and per-stage times of the batched GPU ROM build of a config (default 3); with
--compare also builds with the one-RHS PCG (SFW_PCG1) in a subprocess-free way and reports the
largest relative difference of the chain blocks.   python tools/rom_time.py [cfg] [--compare]"""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1406_6923_b200 import build_models  # noqa: E402
from paper_1406_6923_b200.rom import LAST_BUILD_STATS  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 3
wl, ops, alphas, _, _ = bench._workload(cfg)
out = {}
for tag in (["pcg2", "pcg1"] if "--compare" in sys.argv else ["default"]):
    if tag == "pcg1":
        os.environ["SFW_PCG1"] = "1"
    t0 = time.perf_counter()
    models = build_models(ops[:512] if "--compare" in sys.argv else ops, wl.modes_per_face, wl.n, wl.shift)
    out[tag] = {"wall_s": time.perf_counter() - t0, **LAST_BUILD_STATS}
    out[tag + "_g"] = np.stack([models[a].gammas for a in sorted(models)[:64]])
    os.environ.pop("SFW_PCG1", None)
if "--compare" in sys.argv:
    d = np.abs(out["pcg2_g"] - out["pcg1_g"]).max() / np.abs(out["pcg1_g"]).max()
    out["max_rel_diff_gammas"] = float(d)
print(json.dumps({k: v for k, v in out.items() if not k.endswith("_g")}))
