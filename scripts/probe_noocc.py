"""How much of the conditioning kernel is the occupancy probe: device time of
render_queries (config 2) with the full conditioning vs NoOcclusion (no probe)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_24290_b200 import capi
dev = torch.device("cuda", 0)
ctx = capi.Context(0)
stream = torch.cuda.Stream(dev); torch.cuda.set_stream(stream); ctx.set_stream(stream.cuda_stream)
sc = capi.synth_scene(100_000, 2, 1, 7); scene = ctx.scene(sc)
lo, hi = scene.bounds(0.0); olo, ohi = scene.bounds(0.1)
grid = capi.Grid(90, 360, 8, 1.0); tx = np.array([0.3, -0.2, 0.1])
rx = torch.from_numpy(capi.synth_points(1024, 11, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])).to(dev)
sd = torch.empty((1024, 90, 360), device=dev); rd = torch.empty(1024, device=dev)
st = scene.tx_state(tx, grid)
for mode in ("full", "no_occlusion"):
    cfg = capi.cond_cfg(mode=mode)
    cond = ctx.cond(cfg, capi.synth_cond(cfg, 2, 1, lo, hi, 3, True))
    cond.build_occupancy(scene, 32, olo, ohi)
    ctx.profile(True)
    for _ in range(3):
        scene.render_queries(cond, st, rx, sd, rd)
    ctx.synchronize(); ctx.reset_stats()
    for _ in range(10):
        scene.render_queries(cond, st, rx, sd, rd)
    ctx.synchronize()
    print(mode, "cond_signal", ctx.kernel_stats("cond_signal"), "composite", ctx.kernel_stats("composite"))
    ctx.profile(False)
