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
# as bench.py's config-4 legs: stage2l1 (spectrum L1), stage2 (the reference's
# default loss), joint (L1, geometry on).  Stage II caches the transmitter
# state (trainer.cpp:417-427: built once, before the profiled steps); the
# joint step rebuilds it from the moving geometry every step.
mode = sys.argv[1] if len(sys.argv) > 1 else "joint"
stage2 = mode.startswith("stage2")
if mode == "stage2":
    hyper = list(capi.Trainer.DEFAULTS)
    hyper[3], hyper[4] = 0.2, 0.1
else:
    hyper = list(capi.Trainer.L1_ONLY)
tr = capi.Trainer(ctx, scene, cond, hyper, geometry=(not stage2) or None)
tx = np.array([0.3, -0.2, 0.1])
st = scene.tx_state(tx, grid)
for _ in range(3):
    if not stage2:
        st = scene.tx_state(tx, grid)
    tr.grads(st, rx, tg)
    tr.apply()
torch.cuda.synchronize()
print("ok")
