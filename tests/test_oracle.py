"""The checker itself: the C restatement (oracle/rxgs_oracle.c) pinned
against (a) the reference build oracle/_ref, (b) the committed golden
fixtures generated from the reference (tests/golden/make_golden.py), and
(c) the known-answer tests of the reference's own suite.  CPU only."""
import glob
import os

import numpy as np
import pytest

from conftest import rel_err

import oracle as O

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))
TX = np.array([0.3, -0.2, 0.1])


def _scene(z):
    return dict(positions=z["positions"], log_scales=z["log_scales"], quaternions=z["quaternions"],
                tau_logits=z["tau_logits"], fle_coeffs=z["fle_coeffs"], l_max=int(z["l_max"]),
                channels=int(z["channels"]))


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_restatement_matches_golden(orc, path):
    z = np.load(path)
    sc = _scene(z)
    C = sc["channels"]
    h = orc.scene(sc, "spectrum" if C == 1 else "csi")
    g = z["grid"]
    grid = O.Grid(int(g[0]), int(g[1]), int(g[2]), float(g[3]))
    st = orc.tx_state(h, z["tx"], grid)
    for key in ("culled", "geom", "spans", "basis", "offsets", "indices"):
        assert np.array_equal(st.data[key], z[key]), key
    assert st.data["hash"] == int(z["hash"][0])
    occ = orc.build_occupancy(h, int(z["cfg"][4]), z["occ_lo"], z["occ_hi"])
    assert np.array_equal(occ, z["occ"])
    cond = orc.cond(z["cfg"], z["params"], z["occ"], z["occ_lo"], z["occ_hi"])
    co = np.stack([orc.cond_forward(cond, h, r) for r in z["rx"]])
    assert np.array_equal(co, z["cond_out"])
    vals, T = orc.render(st, h, co, co.shape[0])
    assert np.array_equal(vals, z["values"]) and np.array_equal(T, z["transmittance"])
    if C == 1:
        assert np.array_equal(orc.aggregate(vals, grid, "spectrum"), z["spectrum"])
        assert np.array_equal(orc.aggregate(vals, grid, "rssi"), z["rssi"])
    assert np.array_equal(orc.aggregate(vals, grid, "csi"), z["csi"])


@pytest.mark.parametrize("k,l_max,C,seed", [(500, 2, 1, 7), (300, 3, 2, 8), (2000, 1, 1, 9)])
def test_restatement_matches_reference_build(orc, ref, k, l_max, C, seed):
    sc_o = orc.synth_scene(k, l_max, C, seed)
    sc_r = ref.synth_scene(k, l_max, C, seed)
    for key in ("positions", "log_scales", "quaternions", "tau_logits", "fle_coeffs"):
        assert np.array_equal(sc_o[key], sc_r[key]), key
    mod = "spectrum" if C == 1 else "csi"
    ho, hr = orc.scene(sc_o, mod), ref.scene(sc_r, mod)
    grid = O.Grid(36, 72, 8, 1.0)
    so, sr = orc.tx_state(ho, TX, grid), ref.tx_state(hr, TX, grid)
    for key in ("culled", "geom", "spans", "basis", "offsets", "indices", "hash"):
        assert np.array_equal(so.data[key], sr.data[key]), key
    lo, hi = orc.scene_bounds(ho)
    cfg = O.cond_cfg(l_max=l_max, C_=C)
    p_o = orc.synth_cond(cfg, l_max, C, lo, hi, 3, True)
    assert np.array_equal(p_o, ref.synth_cond(cfg, l_max, C, lo, hi, 3, True))
    olo, ohi = orc.scene_bounds(ho, 0.1)
    occ = orc.build_occupancy(ho, 32, olo, ohi)
    assert np.array_equal(occ, ref.build_occupancy(hr, 32, olo, ohi))
    for mode in ("full", "global_only", "local_only", "additive_only", "no_occlusion"):
        cfg_m = O.cond_cfg(l_max=l_max, C_=C, mode=mode)
        co_o = orc.cond_forward(orc.cond(cfg_m, p_o, occ, olo, ohi), ho, [1.1, 0.7, 0.2])
        co_r = ref.cond_forward(ref.cond(cfg_m, p_o, occ, olo, ohi), hr, [1.1, 0.7, 0.2])
        assert np.array_equal(co_o, co_r), mode
    vo, to = orc.render(so, ho, np.stack([co_o, co_o]), 2)
    vr, tr = ref.render(sr, hr, np.stack([co_o, co_o]), 2)
    assert np.array_equal(vo, vr) and np.array_equal(to, tr)


def test_restatement_error_messages(orc, ref):
    """Located errors: render_field (sphraster.cpp:197-206), condition_forward
    (conditioning.cpp:380-382), grid validation (sphraster.cpp:14-20)."""
    sc = orc.synth_scene(3, 1, 1, 45)
    for chk in (orc, ref):
        h = chk.scene(sc, "rssi")
        st = chk.tx_state(h, [0, 0, 0], O.Grid(6, 12, 4, 0.25))
        co = np.random.default_rng(0).standard_normal((2, 3, 4, 1, 2))
        co.reshape(-1)[3 * 8 + 5] = np.nan
        with pytest.raises(O.CheckerError, match="non-finite coefficient at rx 1, gaussian 0"):
            chk.render(st, h, co, 2)
        cfg = O.cond_cfg(F=2, hidden=8, dc=3, S=4, R=8, l_max=1)
        cond = chk.cond(cfg, chk.synth_cond(cfg, 1, 1, [-3] * 3, [3] * 3, 1, True))
        with pytest.raises(O.CheckerError, match="receiver coincides with gaussian 1"):
            chk.cond_forward(cond, h, sc["positions"][1])
        with pytest.raises(O.CheckerError, match="grid: radius must be > 0"):
            chk.tx_state(h, [0, 0, 0], O.Grid(6, 12, 4, 0.0))


def test_reference_kats(orc):
    """Known answers from the reference suite, restated."""
    # probe_segment: uniform 0.1 grid (test_conditioning.cpp:114-133)
    out = orc.probe(4, np.array([-10.0] * 3), np.array([10.0] * 3), np.full(64, 0.1),
                    np.array([-5.0, 0, 0]), np.array([5.0, 0, 0]), 16)
    assert rel_err(out[0], 0.1853020188851841) < 1e-7 and rel_err(out[1], 0.1) < 1e-12
    # empty grid reads T = 1, mean 0
    out = orc.probe(4, np.zeros(3), np.ones(3), None, np.zeros(3), np.ones(3), 16)
    assert out[0] == 1.0 and out[1] == 0.0
    # FLE basis closed forms (test_radiance.cpp:99-126)
    b = orc.eval_basis(0.3, 1.1, 1)
    assert rel_err(b[0, 0], 0.2820947917738781) < 1e-15 and b[0, 1] == 0.0
    b = orc.eval_basis(np.pi / 3, 0.0, 1)
    assert rel_err(b[2, 0], 0.4886025119029199 * 0.5) < 1e-14
    # bin_and_sort: depth sort with index tiebreak {1,0,2} and the seam wrap
    grid = O.Grid(6, 12, 4, 0.25)
    offs, idx = orc.bin_and_sort([0, 0, 0], [2.0, 1.0, 2.0], [[0, 1, 0, 2], [0, 0, 1, 1], [0, 0, 1, 1]], grid)
    assert list(idx[offs[1]:offs[2]]) == [1, 0, 2]
    offs, idx = orc.bin_and_sort([0], [1.0], [[0, 0, 2, 3]], grid)
    assert [list(idx[offs[t]:offs[t + 1]]) for t in range(3)] == [[0], [], [0]]
    # aggregation closed forms (test_sphraster.cpp:250-303)
    g = O.Grid(1, 1)
    assert rel_err(orc.aggregate(np.array([3.0, 4.0]).reshape(1, 1, 2, 1, 1), g, "spectrum")[0, 0, 0],
                   np.sqrt(25 + 1e-8)) < 1e-15


def test_single_gaussian_render_closed_form(orc):
    """blend of one Gaussian: C = w * s, T = 1 - w (test_sphraster.cpp:134-142)."""
    sc = dict(positions=np.array([[2.0, 0.0, 0.0]]), log_scales=np.full((1, 3), -0.5),
              quaternions=np.array([[1.0, 0, 0, 0]]), tau_logits=np.array([0.2]),
              fle_coeffs=np.array([1.5, -0.7]).reshape(1, 1, 1, 2), l_max=0, channels=1)
    h = orc.scene(sc, "spectrum")
    grid = O.Grid(6, 12, 4, 0.25)
    st = orc.tx_state(h, [0, 0, 0], grid)
    vals, T = orc.render(st, h, sc["fle_coeffs"][None], 1)
    g = st.data["geom"][0]
    s = complex(1.5, -0.7) * complex(*st.data["basis"][0, 0])
    for row in range(6):
        for col in range(12):
            th = (row + 0.5) * np.pi / 6
            ph = (col + 0.5) * 2 * np.pi / 12
            dt = th - g[0]
            dpr = np.fmod(ph - g[1], 2 * np.pi)
            dpr = dpr - 2 * np.pi if dpr > np.pi else (dpr + 2 * np.pi if dpr <= -np.pi else dpr)
            dp = np.sin(g[0]) * dpr
            m2 = g[7] * dt * dt + (g[8] + g[9]) * dt * dp + g[10] * dp * dp
            w = min(g[11] * np.exp(-0.5 * m2), 0.999)
            covered = st.data["spans"][0]
            tile = (row // 4) * 3 + (col // 4)
            inlist = 0 in list(st.data["indices"][st.data["offsets"][tile]:st.data["offsets"][tile + 1]])
            if not inlist:
                w = 0.0
            assert abs(vals[0, 0, 0, row, col] - w * s.real) < 1e-14
            assert abs(T[0, row, col] - (1 - w)) < 1e-14
            del covered


def test_reference_adjoints_match_finite_differences(orc, ref):
    """Pins the adjoint wrappers (oracle/_ref) that the GPU backward tests
    compare against: d_coeffs is exact (render is linear in the
    coefficients); d_tau_logits / d_positions by central differences of the
    restated forward; the spectrum aggregate adjoint likewise."""
    import oracle as O
    rng = np.random.default_rng(2)
    k, n_rx = 60, 1
    sc = orc.synth_scene(k, 1, 1, 5)
    g = O.Grid(8, 16, 4, 1.0)
    tx = np.array([0.3, -0.2, 0.1])
    co = rng.standard_normal((n_rx, k, 4, 1, 2))
    dv = rng.standard_normal((n_rx, 1, 2, 8, 16))
    rs = ref.scene(sc)
    b = ref.backward_render(ref.tx_state(rs, tx, g), rs, co, n_rx, dv)

    def loss(s, c=co):
        h = orc.scene(s)
        v, _ = orc.render(orc.tx_state(h, tx, g), h, c, n_rx)
        return float((v * dv).sum())

    idx = np.argsort(-np.abs(b["d_tau_logits"]))[:3]
    for kk in idx:
        for name, arr, comp in (("d_tau_logits", "tau_logits", None), ("d_positions", "positions", 0)):
            hi = {n: (v.copy() if isinstance(v, np.ndarray) else v) for n, v in sc.items()}
            lo = {n: (v.copy() if isinstance(v, np.ndarray) else v) for n, v in sc.items()}
            eps = 1e-6
            if comp is None:
                hi[arr][kk] += eps; lo[arr][kk] -= eps
                want = b[name][kk]
            else:
                hi[arr][kk, comp] += eps; lo[arr][kk, comp] -= eps
                want = b[name][kk, comp]
            fd = (loss(hi) - loss(lo)) / (2 * eps)
            assert abs(fd - want) <= 1e-4 * max(1.0, abs(want)), (name, kk, fd, want)
    e = np.zeros_like(co); e[0, idx[0], 1, 0, 1] = 1.0
    assert abs(loss(sc, e) - b["d_coeffs"][0, idx[0], 1, 0, 1]) < 1e-10
    vals = rng.standard_normal((2, 1, 2, 8, 16))
    up = rng.standard_normal((2, 8, 16))
    d = ref.aggregate_backward(vals, g, "spectrum", up)
    p = vals.copy(); p[1, 0, 0, 3, 5] += 1e-6
    m = vals.copy(); m[1, 0, 0, 3, 5] -= 1e-6
    fd = ((orc.aggregate(p, g, "spectrum") - orc.aggregate(m, g, "spectrum")) * up).sum() / 2e-6
    assert abs(fd - d[1, 0, 0, 3, 5]) < 1e-6
