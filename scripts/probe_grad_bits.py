"""Dump the training gradient buffer (Stage II, L1 and default loss; joint)
of the library in RXGS_B200_LIB to gpurun_out/grad_<tag>.npz, for bitwise
A/B between builds."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_24290_b200 import capi
tag = sys.argv[1]
ctx = capi.Context(0)
sc = capi.synth_scene(20_000, 2, 1, 7)
out = {}
for name, hyper, geo in (("l1", capi.Trainer.L1_ONLY, None), ("default", None, None), ("joint", capi.Trainer.L1_ONLY, True)):
    scene = ctx.scene(sc, "spectrum")
    lo, hi = scene.bounds(0.0)
    cfg = capi.cond_cfg()
    cond = ctx.cond(cfg, capi.synth_cond(cfg, 2, 1, lo, hi, 3, True))
    olo, ohi = scene.bounds(0.1)
    cond.build_occupancy(scene, 32, olo, ohi)
    grid = capi.Grid(45, 90, 8, 1.0)
    rx = capi.synth_points(5, 23, "bench.train.rx", [-4, -3, -1.5], [4, 3, 1.5], 0.05)
    tg = np.random.default_rng(29).uniform(0, 2, (5, grid.cells)).astype(np.float32)
    tr = capi.Trainer(ctx, scene, cond, hyper, geometry=geo)
    st = scene.tx_state(np.array([0.3, -0.2, 0.1]), grid)
    tr.grads(st, rx, tg)
    db, dp = tr.get_grads()
    out[name + "_b"], out[name + "_p"] = db, dp
    if geo:  # positions, log-scales, quaternions, tau logits
        for q, g in enumerate(tr.get_geometry_grads()):
            out[f"{name}_geo{q}"] = np.asarray(g)
os.makedirs("gpurun_out", exist_ok=True)
np.savez(f"gpurun_out/grad_{tag}.npz", **out)
print(tag, {k: float(np.abs(v).sum()) for k, v in out.items()})
