"""Config-1 single-query latency breakdown: wall time of build_tx_state and of
render_queries (host buffers) separately, and the device time of their
kernels (per-kernel events), median of 20 after warm-up."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_24290_b200 import capi
ctx = capi.Context(0)
scene = ctx.scene(capi.synth_scene(10_000, 2, 1, 7), "spectrum")
lo, hi = scene.bounds(0.0)
cfg = capi.cond_cfg()
cond = ctx.cond(cfg, capi.synth_cond(cfg, 2, 1, lo, hi, 3, True))
olo, ohi = scene.bounds(0.1)
cond.build_occupancy(scene, 32, olo, ohi)
grid = capi.Grid(90, 360, 8, 1.0)
tx = np.array([0.3, -0.2, 0.1]); rx = np.array([[1.1, 0.7, 0.2]])
spec = np.empty((1, 90, 360), np.float32); rssi = np.empty(1, np.float32)
tb, tr = [], []
for i in range(25):
    t0 = time.perf_counter(); st = scene.tx_state(tx, grid); t1 = time.perf_counter()
    scene.render_queries(cond, st, rx, spec, rssi); t2 = time.perf_counter()
    if i >= 5: tb.append((t1 - t0) * 1e3); tr.append((t2 - t1) * 1e3)
print(f"build {np.median(tb):.3f} ms, render {np.median(tr):.3f} ms (wall, median)")
ctx.profile(True); ctx.reset_stats()
st = scene.tx_state(tx, grid); scene.render_queries(cond, st, rx, spec, rssi); ctx.synchronize()
for k in ("tx_prep", "sort", "walk", "cond_global", "cond_signal", "composite"):
    print(k, ctx.kernel_stats(k))
