"""Diagnose device-loop timing: events per step with/without profiling."""
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
rx = torch.from_numpy(capi.synth_points(1024, 11, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])).to(dev)
sd = torch.empty((1024, 90, 360), device=dev); rd = torch.empty(1024, device=dev)
flush = torch.empty(64 << 20, device=dev)
def step():
    st = scene.tx_state(tx, grid); scene.render_queries(cond, st, rx, sd, rd); return st
for prof in (False, True, False):
    ctx.profile(prof)
    for _ in range(3): step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
    last = None; t0 = time.perf_counter()
    for i in range(5):
        flush.fill_(float(i)); ev[i][0].record(stream); last = step(); ev[i][1].record(stream)
    torch.cuda.synchronize(); wall = (time.perf_counter() - t0) * 1e3 / 5
    print("profile", prof, "event ms/step", [round(a.elapsed_time(b), 2) for a, b in ev], "wall ms/step", round(wall, 2))
    if prof:
        for k in ("tx_prep", "walk", "cond_global", "cond_signal", "composite"): print("  ", k, ctx.kernel_stats(k))
        ctx.reset_stats()
# separate: tx_state alone and render alone
torch.cuda.synchronize()
for name, f in (("tx_state", lambda: scene.tx_state(tx, grid)), ("render", lambda: scene.render_queries(cond, last, rx, sd, rd))):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream); 
    for _ in range(5): f()
    b.record(stream); torch.cuda.synchronize(); print(name, "ms", a.elapsed_time(b) / 5)
err = ctx.selftest_tcgen05(); print("selftest", err)
