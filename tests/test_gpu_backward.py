"""Parity of the materialised adjoints (rxgs_aggregate_modality_backward,
rxgs_backward_render) with the reference's own implementation
(oracle/_ref: raster::aggregate_modality_backward sphraster.cpp:383-449,
raster::backward_render sphraster.cpp:509-733).

Float tolerance: rel_err (testutil.hpp:14-20) <= 1e-4 on every gradient.
"""
import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu

TOL = 1e-4
TX = np.array([0.3, -0.2, 0.1])


def _bundle_close(got, want, tol=TOL):
    for name in ("d_positions", "d_log_scales", "d_quaternions", "d_tau_logits", "d_coeffs"):
        e = rel_err(got[name], want[name]).max() if want[name].size else 0.0
        assert e < tol, (name, e)


@pytest.mark.parametrize("modality,C", [("rssi", 1), ("csi", 1), ("csi", 3), ("spectrum", 1)])
def test_aggregate_backward_matches_reference(ctx, capi, ref, modality, C):
    import oracle as O
    rng = np.random.default_rng(5)
    n_rx = 3
    grid, og = capi.Grid(12, 20, 4, 1.0), O.Grid(12, 20, 4, 1.0)
    vals = rng.standard_normal((n_rx, C, 2, 12, 20))
    up = {"rssi": rng.standard_normal(n_rx), "csi": rng.standard_normal((n_rx, C, 2)),
          "spectrum": rng.standard_normal((n_rx, 12, 20))}[modality]
    got = ctx.aggregate_backward(vals, grid, modality, up)
    want = ref.aggregate_backward(vals, og, modality, up)
    assert rel_err(got, want).max() < 1e-12


def test_aggregate_backward_rejects_multichannel_scalar(ctx, capi):
    vals = np.zeros((1, 2, 2, 4, 4))
    with pytest.raises(capi.InvalidArgument):
        ctx.aggregate_backward(vals, capi.Grid(4, 4, 4, 1.0), "rssi", np.zeros(1))


@pytest.mark.parametrize("k,l_max,C,n_rx,ts,nt,np_", [
    (300, 2, 1, 2, 8, 16, 32),
    (400, 1, 2, 3, 4, 12, 24),   # several (rx, channel) pairs
    (600, 3, 1, 9, 8, 16, 32),   # more than one 8-pair walk pass
    (250, 2, 1, 1, 16, 32, 32),  # 16x16 tiles: four 64-cell blocks per tile
])
def test_backward_render_matches_reference(ctx, capi, ref, k, l_max, C, n_rx, ts, nt, np_):
    import oracle as O
    rng = np.random.default_rng(11)
    sc = capi.synth_scene(k, l_max, C, 7)
    grid, og = capi.Grid(nt, np_, ts, 1.0), O.Grid(nt, np_, ts, 1.0)
    scene = ctx.scene(sc, "csi")
    st = scene.tx_state(TX, grid)
    co = rng.standard_normal((n_rx, k, (l_max + 1) ** 2, C, 2))
    dv = rng.standard_normal((n_rx, C, 2, nt, np_))
    got = scene.backward_render(st, co, n_rx, dv)
    rscene = ref.scene(sc, "csi")
    rtx = ref.tx_state(rscene, TX, og)
    want = ref.backward_render(rtx, rscene, co, n_rx, dv)
    assert np.abs(want["d_positions"]).max() > 0.0
    _bundle_close(got, want)


def test_backward_chain_spectrum_matches_reference(ctx, capi, ref):
    """aggregate adjoint -> render adjoint, the reference's training chain
    (trainer.cpp:192-214) with a spectrum upstream."""
    import oracle as O
    rng = np.random.default_rng(3)
    k, n_rx = 500, 2
    sc = capi.synth_scene(k, 2, 1, 9)
    grid, og = capi.Grid(16, 32, 8, 1.0), O.Grid(16, 32, 8, 1.0)
    scene = ctx.scene(sc)
    st = scene.tx_state(TX, grid)
    co = rng.standard_normal((n_rx, k, 9, 1, 2))
    vals, _ = scene.render_field(st, co, n_rx)
    up = rng.standard_normal((n_rx, 16, 32))
    dv = ctx.aggregate_backward(vals, grid, "spectrum", up)
    got = scene.backward_render(st, co, n_rx, dv)
    rscene = ref.scene(sc)
    rtx = ref.tx_state(rscene, TX, og)
    wv, _ = ref.render(rtx, rscene, co, n_rx)
    wdv = ref.aggregate_backward(wv, og, "spectrum", up)
    assert rel_err(dv, wdv).max() < TOL
    _bundle_close(got, ref.backward_render(rtx, rscene, co, n_rx, wdv))


def test_backward_render_deterministic(ctx, capi):
    rng = np.random.default_rng(1)
    k = 400
    sc = capi.synth_scene(k, 2, 1, 4)
    grid = capi.Grid(16, 32, 8, 1.0)
    scene = ctx.scene(sc)
    st = scene.tx_state(TX, grid)
    co = rng.standard_normal((2, k, 9, 1, 2))
    dv = rng.standard_normal((2, 1, 2, 16, 32))
    a = scene.backward_render(st, co, 2, dv)
    b = scene.backward_render(st, co, 2, dv)
    for n in a:
        assert np.array_equal(a[n], b[n]), n


@pytest.mark.parametrize("mode,hidden,C,occ", [
    ("full", 64, 1, True), ("global_only", 64, 1, True), ("local_only", 64, 1, True), ("additive_only", 64, 1, True),
    ("no_occlusion", 64, 1, True), ("full", 32, 2, True), ("full", 64, 1, False)])
def test_condition_backward_matches_reference(ctx, capi, ref, mode, hidden, C, occ):
    from test_gpu_render import _setup_cond
    rng = np.random.default_rng(8)
    k = 700
    sc = capi.synth_scene(k, 2, C, 7)
    scene, cond, rscene, rcond = _setup_cond(capi, ctx, ref, sc, mode=mode, hidden=hidden, occ=occ)
    rx = np.array([0.45, -0.35, 0.2])
    d_out = rng.standard_normal((k, 9, C, 2))
    db, dp = cond.backward(scene, rx, d_out)
    wdb, wdp = ref.cond_backward(rcond, rscene, rx, d_out)
    assert rel_err(db, wdb).max() < TOL
    assert rel_err(dp, wdp).max() < TOL
    assert np.abs(wdp).max() > 0.0


def test_condition_backward_rejects_coincident_receiver(ctx, capi):
    from test_gpu_render import _setup_cond
    import oracle as O
    sc = capi.synth_scene(50, 2, 1, 7)
    scene, cond, _, _ = _setup_cond(capi, ctx, O.restatement(), sc)
    with pytest.raises(capi.InvalidArgument, match="receiver coincides with gaussian 3"):
        cond.backward(scene, sc["positions"][3], np.zeros((50, 9, 1, 2)))
