"""Config-3 coverage table timeline (RXGS_COV_TRACE=1): per-transmitter build
and render intervals on the device, after two warm-up tables."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_24290_b200 import capi
import bench
dev = torch.device("cuda", 0)
ctx = capi.Context(0)
stream = torch.cuda.Stream(dev); torch.cuda.set_stream(stream); ctx.set_stream(stream.cuda_stream)
scene = ctx.scene(capi.synth_scene(500_000, 2, 1, 7), "rssi")
cond = bench._cond_for(capi, ctx, scene)
grid = capi.Grid(90, 360, 8, 1.0)
rx = capi.synth_points(1024, 11, "bench.rx", bench.BOX_LO, bench.BOX_HI, 0.05)
tx = capi.synth_points(64, 13, "bench.tx", bench.BOX_LO, bench.BOX_HI, 0.05)
txd = torch.from_numpy(tx).to(dev); rxd = torch.from_numpy(rx).to(dev); out = torch.empty((64, 1024), device=dev)
for i in range(int(os.environ.get("N_TABLES", "3"))):
    if i == 2 and not os.environ.get("NO_TRACE"): os.environ["RXGS_COV_TRACE"] = "1"
    scene.coverage_table(cond, grid, txd, rxd, out); torch.cuda.synchronize()
