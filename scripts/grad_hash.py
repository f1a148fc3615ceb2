"""Hash of the config-4 style gradients (for bit-identity A/B of kernel variants)."""
import hashlib, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_24290_b200 import capi
ctx = capi.Context(0)
sc = capi.synth_scene(20_000, 2, 1, 7)
scene = ctx.scene(sc, "spectrum")
lo, hi = scene.bounds(0.0)
cfg = capi.cond_cfg()
cond = ctx.cond(cfg, capi.synth_cond(cfg, 2, 1, lo, hi, 3, True))
olo, ohi = scene.bounds(0.1)
cond.build_occupancy(scene, 32, olo, ohi)
grid = capi.Grid(45, 90, 8, 1.0)
rx = capi.synth_points(8, 23, "bench.train.rx", [-4, -3, -1.5], [4, 3, 1.5], 0.05)
tg = np.random.default_rng(29).uniform(0, 2, (8, grid.cells)).astype(np.float32)
tr = capi.Trainer(ctx, scene, cond)
tr.grads(scene.tx_state(np.array([0.3, -0.2, 0.1]), grid), rx, tg)
db, dp = tr.get_grads()
print(hashlib.sha1(db.tobytes() + dp.tobytes()).hexdigest(), float(np.abs(dp).max()))
