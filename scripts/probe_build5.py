"""Config-5 transmitter-state build only (K=2M, 180x720): N_BUILDS builds after
one warm-up, for an ncu launch list of the binning kernels."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_24290_b200 import capi
import bench
dev = torch.device("cuda", 0)
ctx = capi.Context(0)
stream = torch.cuda.Stream(dev); torch.cuda.set_stream(stream); ctx.set_stream(stream.cuda_stream)
scene = ctx.scene(capi.synth_scene(2_000_000, 2, 1, 7), "spectrum")
grid = capi.Grid(180, 720, 8, 1.0)
tx = np.array(bench.TX)
st = scene.tx_state(tx, grid); torch.cuda.synchronize()
for _ in range(int(os.environ.get("N_BUILDS", "3"))):
    del st
    st = scene.tx_state(tx, grid)
torch.cuda.synchronize()
print(st.stats())
