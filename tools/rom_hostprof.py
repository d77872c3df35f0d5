import cProfile, pstats, sys, os, io
sys.path.insert(0, os.getcwd())
import bench
from paper_1406_6923_b200 import build_models
wl, ops, alphas, _, _ = bench._workload(3)
build_models(ops[:64], wl.modes_per_face, wl.n, wl.shift)
pr = cProfile.Profile(); pr.enable()
models = build_models(ops, wl.modes_per_face, wl.n, wl.shift)
pr.disable()
st = io.StringIO(); pstats.Stats(pr, stream=st).sort_stats("cumulative").print_stats(18); print(st.getvalue()[:3500])
from paper_1406_6923_b200.rom import LAST_BUILD_STATS
print(LAST_BUILD_STATS)
