"""Coverage consumers: apps::coverage_fraction and
apps::greedy_plan (apps.cpp:69-116) on the device vs the reference build --
exact (counts, selection order, lowest-index tie break), including the
reference suite's hand instances (test_apps.cpp:118-143) and a coverage
table produced by rxgs_coverage_table."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_hand_instances(ctx, ref):
    t = np.array([-70, -90, -75, -85, -95, -60.0]).reshape(3, 2)
    assert ctx.coverage_fraction(np.full((3, 2), -10.0), [0, 1], -80) == 1.0
    assert ctx.coverage_fraction(np.full((3, 2), -99.0), [0, 1], -80) == 0.0
    assert ctx.coverage_fraction(t, [0], -80) == ref.coverage_fraction(t, [0], -80) == 2.0 / 3
    assert ctx.coverage_fraction(t, [1], -80) == 1.0 / 3
    hot, cold = -70.0, -95.0
    T = np.array([[hot, cold, cold], [hot, cold, cold], [hot, hot, cold], [cold, hot, hot], [cold, cold, hot]])
    assert list(ctx.greedy_plan(T, 2, -80)) == [0, 2]


@pytest.mark.parametrize("tx,cand,k,seed", [(64, 1024, 12, 1), (100, 37, 37, 2), (33, 500, 5, 3), (1000, 64, 20, 4)])
def test_random_tables_match_reference(ctx, ref, tx, cand, k, seed):
    rng = np.random.default_rng(seed)
    table = rng.uniform(-110, -40, size=(tx, cand))
    table[:, 3 % cand] = -200.0  # a useless candidate
    if cand > 5:
        table[:, 5] = table[:, 4]  # an exact tie: the lower index must win
    thr = -80.0
    assert np.array_equal(ctx.greedy_plan(table, k, thr), ref.greedy_plan(table, k, thr))
    sel = rng.choice(cand, size=min(7, cand), replace=False)
    assert ctx.coverage_fraction(table, sel, thr) == ref.coverage_fraction(table, sel, thr)


def test_errors_match_reference(ctx, capi):
    t = np.zeros((3, 2))
    with pytest.raises(capi.InvalidArgument, match="coverage_fraction: empty selection"):
        ctx.coverage_fraction(t, [], -80)
    with pytest.raises(capi.InvalidArgument, match="coverage_fraction: candidate index out of range"):
        ctx.coverage_fraction(t, [2], -80)
    with pytest.raises(capi.InvalidArgument, match="greedy_plan: k out of range"):
        ctx.greedy_plan(t, 3, -80)


def test_on_a_rendered_coverage_table(ctx, capi, ref):
    sc = capi.synth_scene(3000, 2, 1, 7)
    scene = ctx.scene(sc, "rssi")
    lo, hi = scene.bounds(0.0)
    cfg = capi.cond_cfg()
    cond = ctx.cond(cfg, capi.synth_cond(cfg, 2, 1, lo, hi, 3, True))
    olo, ohi = scene.bounds(0.1)
    cond.build_occupancy(scene, 32, olo, ohi)
    grid = capi.Grid(30, 60, 8, 1.0)
    tx = capi.synth_points(8, 13, "bench.tx", [-4, -3, -1.5], [4, 3, 1.5])
    rx = capi.synth_points(40, 11, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    table = scene.coverage_table(cond, grid, tx, rx).astype(np.float64)  # tx x rx (candidates)
    thr = float(np.median(table))
    assert np.array_equal(ctx.greedy_plan(table, 6, thr), ref.greedy_plan(table, 6, thr))
    assert ctx.coverage_fraction(table, [0, 5, 9], thr) == ref.coverage_fraction(table, [0, 5, 9], thr)


# ---------------------------------------------------------------- metrics
@pytest.mark.parametrize("n,h,w,opts,max_val,f32", [
    (3, 20, 30, (11, 1.5, 1.0), 1.0, False),
    (2, 90, 360, (11, 1.5, 1.0), 2.0, True),
    (4, 16, 12, (7, 2.0, 2.0), 3.0, False),
    (2, 9, 14, (8, 1.0, 1.0), 1.0, True),  # even window: half = n / 2 as in gaussian_window
])
def test_image_metrics_match_reference(ctx, ref, n, h, w, opts, max_val, f32):
    """met::mae / mse / psnr / ssim (metrics.cpp:11-112) per image on the device vs
    the reference build (rel_err <= 1e-12 in FP64; f32 predictions are widened)."""
    rng = np.random.default_rng(n * h + w)
    gt = rng.uniform(0, 2, size=(n, h, w))
    pred = gt + rng.normal(0, 0.2, size=gt.shape)
    if f32:
        pred = pred.astype(np.float32)
    got = ctx.image_metrics(pred, gt, h, w, max_val, opts)
    for i in range(n):
        want = ref.image_metrics(pred[i].astype(np.float64), gt[i], h, w, max_val, *opts)
        np.testing.assert_allclose(got[i], want, rtol=1e-12, atol=1e-14)


def test_image_metrics_edges(ctx, ref, capi):
    gt = np.random.default_rng(1).uniform(0, 1, size=(2, 12, 12))
    out = ctx.image_metrics(gt.copy(), gt, 12, 12)
    assert (out[:, 2] == 300.0).all() and (out[:, 0] == 0).all()  # kDbSentinel on identical inputs
    np.testing.assert_allclose(out[:, 3], 1.0, rtol=1e-14)
    no_ssim = ctx.image_metrics(gt + 0.1, gt, 12, 12, ssim=None)
    assert np.isnan(no_ssim[:, 3]).all()
    np.testing.assert_allclose(no_ssim[:, 0], 0.1, rtol=1e-12)
    with pytest.raises(capi.InvalidArgument, match="ssim: image smaller than the window"):
        ctx.image_metrics(gt[:, :10, :10].copy(), gt[:, :10, :10].copy(), 10, 10)
    with pytest.raises(ValueError, match="ssim: image smaller than the window"):
        ref.image_metrics(gt[0, :10, :10].ravel(), gt[0, :10, :10].ravel(), 10, 10)


def test_image_metrics_on_rendered_spectra(ctx, ref, capi):
    """Evaluation of rendered spectra (f32 on the device, as rxgs_render_queries
    writes them) against FP64 reference renders of the same queries."""
    import torch
    sc = capi.synth_scene(2000, 2, 1, 7)
    scene = ctx.scene(sc, "spectrum")
    grid = capi.Grid(18, 72, 8, 1.0)
    rx = capi.synth_points(3, 11, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    st = scene.tx_state(np.array([0.3, -0.2, 0.1]), grid)
    spec, _ = scene.render_queries(None, st, rx)
    spec = np.asarray(spec, np.float32).reshape(3, grid.cells)
    import oracle as O
    rsc = ref.scene(sc, "spectrum")
    og = O.Grid(18, 72, 8, 1.0)
    gt = np.stack([ref.predict(rsc, None, og, [0.3, -0.2, 0.1], rx[j]) for j in range(3)]).reshape(3, -1)
    got = ctx.image_metrics(torch.from_numpy(spec).cuda(), torch.from_numpy(gt).cuda(), 18, 72, 1.0)
    for j in range(3):
        want = ref.image_metrics(spec[j].astype(np.float64), gt[j], 18, 72, 1.0)
        np.testing.assert_allclose(got[j], want, rtol=1e-12, atol=1e-14)
    assert (got[:, 3] > 0.999).all()  # the B200 render agrees with the reference render


# ---------------------------------------------------------------- CSI evaluation metrics (metrics.cpp:114-149)
def test_snr_csi_matches_reference(ctx, ref):
    rng = np.random.default_rng(7)
    for n in (1, 4, 1000):
        g = rng.normal(size=(3, n)) + 1j * rng.normal(size=(3, n))
        p = g + 0.1 * (rng.normal(size=(3, n)) + 1j * rng.normal(size=(3, n)))
        got = ctx.snr_csi(p, g)
        want = [ref.snr_csi(p[i], g[i]) for i in range(3)]
        assert np.allclose(got, want, rtol=1e-12, atol=0)
    assert ctx.snr_csi(g, g)[0] == 300.0  # kDbSentinel
    import oracle as O
    with pytest.raises(ValueError, match="snr_csi: zero ground-truth energy"):
        ctx.snr_csi(np.ones((1, 3), complex), np.zeros((1, 3), complex))
    with pytest.raises(O.CheckerError, match="snr_csi: zero ground-truth energy"):
        ref.snr_csi(np.ones(3, complex), np.zeros(3, complex))


def test_per_receiver_aggregate_matches_reference(ctx, ref):
    rng = np.random.default_rng(11)
    for n, n_rx in ((1, 1), (50, 7), (20000, 300)):
        rx = rng.integers(-5, n_rx, n).astype(np.int32)
        v = rng.normal(size=n)
        g_rx, g_m, g_c, g_mu, g_sd = ctx.per_receiver_aggregate(rx, v)
        w_rx, w_m, w_c, w_mu, w_sd = ref.per_receiver_aggregate(rx, v)
        assert np.array_equal(g_rx, w_rx) and np.array_equal(g_c, w_c)
        assert np.array_equal(g_m, w_m)  # per receiver: the same sums in the same order
        assert abs(g_mu - w_mu) <= 1e-14 * max(1, abs(w_mu)) and abs(g_sd - w_sd) <= 1e-13 * max(1, w_sd)
    with pytest.raises(ValueError, match="per_receiver_aggregate: no records"):
        ctx.per_receiver_aggregate(np.zeros(0, np.int32), np.zeros(0))
