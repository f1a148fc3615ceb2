"""Joint-step kernel breakdown (run under ncu --metrics gpu__time_duration.sum):
K=100k, 16 samples, the bench's config-4 inputs with geometry enabled."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_24290_b200 import capi
import torch

ctx = capi.Context(0)
sc = capi.synth_scene(100_000, 2, 1, 7)
scene = ctx.scene(sc, "spectrum")
lo, hi = scene.bounds(0.0)
cfg = capi.cond_cfg()
cond = ctx.cond(cfg, capi.synth_cond(cfg, 2, 1, lo, hi, 3, True))
olo, ohi = scene.bounds(0.1)
cond.build_occupancy(scene, 32, olo, ohi)
grid = capi.Grid(90, 360, 8, 1.0)
rx = capi.synth_points(16, 23, "bench.train.rx", [-4, -3, -1.5], [4, 3, 1.5], 0.05)
tg = np.random.default_rng(29).uniform(0, 2, (16, grid.cells)).astype(np.float32)
stage2 = len(sys.argv) > 1 and sys.argv[1].startswith("stage2")
hyper = capi.Trainer.L1_ONLY if len(sys.argv) > 1 and sys.argv[1] == "stage2l1" else None
tr = capi.Trainer(ctx, scene, cond, hyper, geometry=(not stage2) or None)
for _ in range(3):
    st = scene.tx_state(np.array([0.3, -0.2, 0.1]), grid)
    tr.grads(st, rx, tg)
    tr.apply()
torch.cuda.synchronize()
print("ok")
