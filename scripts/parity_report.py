"""Full-size parity spot check: bench workload (K=100k, 90x360, conditioned) on
the GPU (tcgen05 and SIMT kernels) vs the C oracle for a sample of receivers."""
import json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import oracle as O
from paper_2605_24290_b200 import capi
K = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
NS = int(sys.argv[2]) if len(sys.argv) > 2 else 6
TX = np.array([0.3, -0.2, 0.1])
sc = capi.synth_scene(K, 2, 1, 7)
ctx = capi.Context(0)
scene = ctx.scene(sc)
lo, hi = scene.bounds(0.0)
cfg = capi.cond_cfg()
params = capi.synth_cond(cfg, 2, 1, lo, hi, 3, True)
cond = ctx.cond(cfg, params)
olo, ohi = scene.bounds(0.1)
occ = cond.build_occupancy(scene, 32, olo, ohi)
grid = capi.Grid(90, 360, 8, 1.0)
st = scene.tx_state(TX, grid)
rx = capi.synth_points(1024, 11, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
out = {}
for kern in ("auto", "simt"):
    ctx.set_cond_kernel(kern)
    out[kern] = scene.render_queries(cond, st, rx)
ctx.set_cond_kernel("auto")
orc = O.restatement()
og = O.Grid(90, 360, 8, 1.0)
os_ = orc.scene(sc, "spectrum"); osr = orc.scene(sc, "rssi")
oc = orc.cond(cfg, params, occ, olo, ohi)
sel = np.linspace(0, 1023, NS).astype(int)
rep = {"K": K, "receivers_checked": sel.tolist(), "tolerance": "rel_err=|a-b|/max(1,|a|,|b|) <= 1e-4"}
for kern, (spec, rssi) in out.items():
    es, er = [], []
    for j in sel:
        w = orc.predict(os_, oc, og, TX, rx[j], "spectrum").reshape(90, 360)
        es.append(float((np.abs(spec[j] - w) / np.maximum(1, np.maximum(np.abs(spec[j]), np.abs(w)))).max()))
        wr = orc.predict(osr, oc, og, TX, rx[j], "rssi")[0]
        er.append(float(abs(rssi[j] - wr) / max(1, abs(rssi[j]), abs(wr))))
    rep[kern] = {"spectrum_max_rel_err": max(es), "rssi_max_rel_err": max(er), "per_rx_spectrum": es}
s_a, r_a = out["auto"]; s_s, r_s = out["simt"]
rep["tc_vs_simt_all_1024"] = {"spectrum": float((np.abs(s_a - s_s) / np.maximum(1, np.maximum(np.abs(s_a), np.abs(s_s)))).max()),
                              "rssi": float((np.abs(r_a - r_s) / np.maximum(1, np.maximum(np.abs(r_a), np.abs(r_s)))).max())}
print(json.dumps(rep, indent=1))
