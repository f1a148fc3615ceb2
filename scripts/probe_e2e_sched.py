"""Host-output render (config 2, pinned spectra) under the receiver-chunk
schedule in RXGS_E2E_SCHED: median and min of 15 calls."""
import os, sys, time, statistics
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_24290_b200 import capi
dev = torch.device("cuda", 0)
ctx = capi.Context(0)
stream = torch.cuda.Stream(dev); torch.cuda.set_stream(stream); ctx.set_stream(stream.cuda_stream)
sc = capi.synth_scene(100_000, 2, 1, 7); scene = ctx.scene(sc)
lo, hi = scene.bounds(0.0); cfg = capi.cond_cfg(); cond = ctx.cond(cfg, capi.synth_cond(cfg, 2, 1, lo, hi, 3, True))
olo, ohi = scene.bounds(0.1); cond.build_occupancy(scene, 32, olo, ohi)
grid = capi.Grid(90, 360, 8, 1.0); tx = np.array([0.3, -0.2, 0.1])
rx = torch.from_numpy(capi.synth_points(1024, 11, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])).pin_memory().numpy()
st = scene.tx_state(tx, grid)
sp = torch.empty((1024, 90, 360)).pin_memory().numpy(); rp = torch.empty(1024).pin_memory().numpy()
ts = []
for i in range(18):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    scene.render_queries(cond, st, rx, sp, rp)
    torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
ts = ts[3:]
print(f"sched {os.environ.get('RXGS_E2E_SCHED', '0')}: median {statistics.median(ts):.3f} min {min(ts):.3f} ms")
