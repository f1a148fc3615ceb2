"""Diagnostics: where does end-to-end time go (device outputs vs host outputs)."""
import os, sys, time
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
rx = capi.synth_points(1024, 11, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
def t(f, n=3):
    f(); torch.cuda.synchronize(); ts=[]
    for _ in range(n):
        t0=time.perf_counter(); f(); torch.cuda.synchronize(); ts.append((time.perf_counter()-t0)*1e3)
    return min(ts)
st = scene.tx_state(tx, grid)
print("tx_state build ms", t(lambda: scene.tx_state(tx, grid)))
rxd = torch.from_numpy(rx).to(dev); sd = torch.empty((1024, 90, 360), device=dev); rd = torch.empty(1024, device=dev)
print("render dev ms", t(lambda: scene.render_queries(cond, st, rxd, sd, rd)))
sp = torch.empty((1024, 90, 360)).pin_memory(); rp = torch.empty(1024).pin_memory()
print("render pinned-host ms", t(lambda: scene.render_queries(cond, st, rx, sp.numpy(), rp.numpy())))
sh = np.empty((1024, 90, 360), np.float32); rh = np.empty(1024, np.float32)
print("render pageable-host ms", t(lambda: scene.render_queries(cond, st, rx, sh, rh)))
print("torch D2H pinned 133MB ms", t(lambda: sp.copy_(sd, non_blocking=True)))
print("torch D2H pageable ms", t(lambda: sd.cpu()))
ctx.profile(True); ctx.reset_stats()
scene.render_queries(cond, st, rxd, sd, rd); st2 = scene.tx_state(tx, grid); ctx.synchronize()
for k in ("tx_prep", "walk", "cond_global", "cond_signal", "composite"):
    print(k, ctx.kernel_stats(k))
print("stats", st.stats())
# kernel-time totals of one device-output vs one pinned-host-output render
for name, out in (("device", (sd, rd)), ("pinned", (sp.numpy(), rp.numpy()))):
    ctx.profile(True); ctx.reset_stats()
    scene.render_queries(cond, st, rxd if name == "device" else rx, *out); ctx.synchronize()
    tot = {k: ctx.kernel_stats(k) for k in ("cond_global", "cond_signal", "composite")}
    print(name, {k: (round(v[0], 4), v[1]) for k, v in tot.items()}, "sum", round(sum(v[0] for v in tot.values()), 4))
    ctx.profile(False)
