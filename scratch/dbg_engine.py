import sys
sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import numpy as np
from conftest import golden
import test_engine_gpu as T

g = golden("sim_tiny.npz")
for method in ("buddy", "original"):
    eng = T._engine(method, g)
    out = T._run(eng)
    ev = eng.sorted_events()
    np.save(f"gpurun_out/ev_{method}.npy", ev)
    np.save(f"gpurun_out/out_{method}.npy", out)
    print(method, ev.shape, g[f"{method}_events"].shape, eng.stats())
