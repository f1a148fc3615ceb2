"""A/B of the conditioning kernel variants (RXGS_COND_WS=0/1 in the environment):
config-2 render_queries device time per stage and a digest of the spectra, plus
the coverage local cache (YOUT) digest; run once per variant and compare."""
import hashlib, json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_24290_b200 import capi
dev = torch.device("cuda", 0)
ctx = capi.Context(0)
stream = torch.cuda.Stream(dev); torch.cuda.set_stream(stream); ctx.set_stream(stream.cuda_stream)
out = {"ws": os.environ.get("RXGS_COND_WS", "1")}
for K, l_max, n_rx, mode in ((100_000, 2, 1024, "full"), (100_000, 0, 256, "full"), (20_000, 2, 130, "no_occlusion"), (100_000, 2, 1024, "no_occlusion")):
    sc = capi.synth_scene(K, l_max, 1, 7); scene = ctx.scene(sc)
    lo, hi = scene.bounds(0.0); olo, ohi = scene.bounds(0.1)
    grid = capi.Grid(90, 360, 8, 1.0); tx = np.array([0.3, -0.2, 0.1])
    rx = torch.from_numpy(capi.synth_points(n_rx, 11, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])).to(dev)
    sd = torch.empty((n_rx, 90, 360), device=dev); rd = torch.empty(n_rx, device=dev)
    st = scene.tx_state(tx, grid)
    cfg = capi.cond_cfg(mode=mode, l_max=l_max)
    cond = ctx.cond(cfg, capi.synth_cond(cfg, l_max, 1, lo, hi, 3, True))
    cond.build_occupancy(scene, 32, olo, ohi)
    ctx.profile(True)
    for _ in range(3):
        scene.render_queries(cond, st, rx, sd, rd)
    ctx.synchronize(); ctx.reset_stats()
    for _ in range(10):
        scene.render_queries(cond, st, rx, sd, rd)
    ctx.synchronize()
    key = f"K{K}_l{l_max}_rx{n_rx}_{mode}"
    out[key] = {"cond_signal_ms": ctx.kernel_stats("cond_signal"), "composite": ctx.kernel_stats("composite"),
                "spec_md5": hashlib.md5(sd.cpu().numpy().tobytes()).hexdigest(),
                "rssi_md5": hashlib.md5(rd.cpu().numpy().tobytes()).hexdigest()}
    np.save(f"gpurun_out/ab_ws{out['ws']}_{key}.npy", sd[:4].cpu().numpy())
    ctx.profile(False)
print(json.dumps(out))
