"""Transmitter-state build at a BASELINE size (default config 5: K=2M,
180x720): per-phase device times, for sort / tx_prep work."""
import sys, os, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_24290_b200 import capi
K = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
nt, npp = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (180, 720)
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
ctx = capi.Context(0)
scene = ctx.scene(capi.synth_scene(K, 2, 1, 7), "spectrum")
grid = capi.Grid(nt, npp, 8, 1.0)
tx = np.array([0.3, -0.2, 0.1])
for _ in range(2):
    st = scene.tx_state(tx, grid); del st
ctx.synchronize()
ctx.reset_stats(); ctx.profile(True)
t0 = time.perf_counter()
for _ in range(reps):
    st = scene.tx_state(tx, grid); del st
ctx.synchronize()
wall = (time.perf_counter() - t0) / reps * 1e3
print({n: round(ctx.kernel_stats(n)[0] / reps, 4) for n in ("tx_prep", "sort", "walk")}, "wall ms", round(wall, 3))
ctx.profile(False)
