"""Dump render_queries spectra / RSSI (l_max 2 and 9, conditioned) of the
library in RXGS_B200_LIB to gpurun_out/render_<tag>.npz, for bitwise A/B
between builds."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_24290_b200 import capi
tag = sys.argv[1]
ctx = capi.Context(0)
out = {}
for lm in (2, 9):
    sc = capi.synth_scene(20_000, lm, 1, 7)
    scene = ctx.scene(sc, "spectrum")
    lo, hi = scene.bounds(0.0)
    cfg = capi.cond_cfg(l_max=lm)
    cond = ctx.cond(cfg, capi.synth_cond(cfg, lm, 1, lo, hi, 3, True))
    olo, ohi = scene.bounds(0.1)
    cond.build_occupancy(scene, 32, olo, ohi)
    grid = capi.Grid(45, 90, 8, 1.0)
    rx = capi.synth_points(100, 11, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    st = scene.tx_state(np.array([0.3, -0.2, 0.1]), grid)
    s, r = scene.render_queries(cond, st, rx)
    out[f"s{lm}"], out[f"r{lm}"] = s, r
os.makedirs("gpurun_out", exist_ok=True)
np.savez(f"gpurun_out/render_{tag}.npz", **out)
