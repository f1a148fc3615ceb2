import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
from paper_2605_24290_b200 import capi
ctx = capi.Context(0)
sc = capi.synth_scene(500, 2, 1, 7)
scene = ctx.scene(sc)
lo, hi = scene.bounds(0.0)
cfg = capi.cond_cfg()
cond = ctx.cond(cfg, capi.synth_cond(cfg, 2, 1, lo, hi, 3, True))
olo, ohi = scene.bounds(0.1); cond.build_occupancy(scene, 32, olo, ohi)
grid = capi.Grid(18, 36, 8, 1.0)
rx = capi.synth_points(4, 13, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
tg = np.random.default_rng(9).uniform(0, 2, (4, grid.cells)).astype(np.float32)
TX = np.array([0.3, -0.2, 0.1])
def run(tr, st):
    l = tr.grads(st, rx, tg); return l, np.concatenate(tr.get_grads())
st = scene.tx_state(TX, grid); tr = capi.Trainer(ctx, scene, cond)
l1, a = run(tr, st); l2, b = run(tr, st)
print("same trainer+state: loss eq", np.array_equal(l1, l2), "grad eq", np.array_equal(a, b), np.abs(a-b).max())
tr2 = capi.Trainer(ctx, scene, cond); l3, c = run(tr2, st)
print("new trainer, same state (regrouped):", np.array_equal(a, c), np.array_equal(b, c))
st2 = scene.tx_state(TX, grid); l4, d = run(tr2, st2)
print("new state:", np.array_equal(a, d), np.array_equal(b, d))
l5, e = run(tr2, st2)
print("new state 2nd:", np.array_equal(d, e), np.array_equal(b, e))
n_base = tr.n_base
print("base part eq a/b", np.array_equal(a[:n_base], b[:n_base]), "param part", np.array_equal(a[n_base:], b[n_base:]))
diff = np.nonzero(a != b)[0]; print("n diff", diff.size, diff[:10], diff[-10:])
