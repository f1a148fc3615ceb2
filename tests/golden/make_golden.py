"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref, the
unmodified reference sources compiled by oracle/Makefile).

These fixtures pin the C restatement (oracle/rxgs_oracle.c) wherever the
reference build is absent.  Re-run here (where /root/reference exists):
    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402

TX = np.array([0.3, -0.2, 0.1])


def case(ref, name, k, l_max, C, grid_args, cfg_kw, n_rx):
    sc = ref.synth_scene(k, l_max, C, 7)
    h = ref.scene(sc, "spectrum" if C == 1 else "csi")
    grid = O.Grid(*grid_args)
    st = ref.tx_state(h, TX, grid)
    lo, hi = ref.scene_bounds(h, 0.0)
    cfg = O.cond_cfg(l_max=l_max, C_=C, **cfg_kw)
    params = ref.synth_cond(cfg, l_max, C, lo, hi, 3, True)
    olo, ohi = ref.scene_bounds(h, 0.1)
    occ = ref.build_occupancy(h, int(cfg[4]), olo, ohi)
    cond = ref.cond(cfg, params, occ, olo, ohi)
    rx = ref.synth_points(n_rx, 11, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    co = np.stack([ref.cond_forward(cond, h, r) for r in rx])
    vals, T = ref.render(st, h, co, n_rx)
    out = dict(positions=sc["positions"], log_scales=sc["log_scales"], quaternions=sc["quaternions"],
               tau_logits=sc["tau_logits"], fle_coeffs=sc["fle_coeffs"], l_max=l_max, channels=C,
               grid=np.array(grid_args, np.float64), tx=TX, cfg=cfg, params=params, occ=occ, occ_lo=olo,
               occ_hi=ohi, rx=rx, cond_out=co, values=vals, transmittance=T,
               culled=st.data["culled"], geom=st.data["geom"], spans=st.data["spans"], basis=st.data["basis"],
               offsets=st.data["offsets"], indices=st.data["indices"],
               hash=np.array([st.data["hash"]], np.uint64))
    if C == 1:
        out["spectrum"] = ref.aggregate(vals, grid, "spectrum")
        out["rssi"] = ref.aggregate(vals, grid, "rssi")
    out["csi"] = ref.aggregate(vals, grid, "csi")
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, {k_: np.asarray(v).shape for k_, v in out.items() if k_ in ("values", "indices")})


def main():
    ref = O.reference()
    assert ref is not None, "build oracle/_ref first (make -C oracle ref)"
    tiny = dict(F=2, hidden=8, dc=3, S=4, R=8)
    case(ref, "small_spectrum", 60, 2, 1, (12, 24, 4, 0.5), tiny, 2)
    case(ref, "small_csi", 40, 1, 2, (6, 12, 4, 0.25), tiny, 2)
    case(ref, "bench_like", 400, 2, 1, (18, 36, 8, 1.0), dict(), 2)


if __name__ == "__main__":
    main()
