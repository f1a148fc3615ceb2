"""Training step (config 4, Stage-II chain) on the B200 vs the reference:
gradients of the base FLE coefficients and of every conditioning parameter,
summed over a batch of (tx, rx) samples, within the reference's rel_err
<= 1e-4 (the DP target is the CPU sum of per-sample
gradients); Adam update semantics; determinism."""
import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu

TX = np.array([0.3, -0.2, 0.1])
TOL = 1e-4


def _setup(capi, ctx, ref, k=600, mode="full", nt=18, np_=36, seed=7):
    import oracle as O
    sc = capi.synth_scene(k, 2, 1, seed)
    scene = ctx.scene(sc, "spectrum")
    lo, hi = scene.bounds(0.0)
    cfg = capi.cond_cfg(mode=mode)
    params = capi.synth_cond(cfg, 2, 1, lo, hi, 3, True)
    cond = ctx.cond(cfg, params)
    olo, ohi = scene.bounds(0.1)
    occ = cond.build_occupancy(scene, 32, olo, ohi)
    grid = capi.Grid(nt, np_, 8, 1.0)
    og = O.Grid(nt, np_, 8, 1.0)
    rscene = ref.scene(sc, "spectrum")
    rcond = ref.cond(cfg, params, occ, olo, ohi)
    return sc, scene, cond, grid, og, rscene, rcond, params


def _targets(n, cells, seed=5):
    rng = np.random.default_rng(seed)
    return rng.uniform(0.0, 2.0, size=(n, cells)).astype(np.float32)


@pytest.mark.parametrize("mode", ["full", "global_only", "local_only", "additive_only", "no_occlusion"])
def test_train_grads_match_reference_sum(ctx, capi, ref, mode):
    sc, scene, cond, grid, og, rscene, rcond, params = _setup(capi, ctx, ref, mode=mode)
    rx = capi.synth_points(3, 11, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    tg = _targets(3, grid.cells)
    st = scene.tx_state(TX, grid)
    tr = capi.Trainer(ctx, scene, cond, capi.Trainer.L1_ONLY)
    loss = tr.grads(st, rx, tg)
    db, dp = tr.get_grads()
    want_b = np.zeros_like(db)
    want_p = np.zeros_like(dp)
    for j in range(3):
        r = ref.train_sample(rscene, rcond, og, TX, rx[j], tg[j].astype(np.float64))
        assert rel_err(loss[j], r["loss"]) < TOL
        want_b += r["d_base"]
        want_p += r["d_params"]
    assert rel_err(db, want_b).max() < TOL
    assert rel_err(dp, want_p).max() < TOL


@pytest.mark.parametrize("n_rx", [5, 7, 13])
def test_train_tc_batches_off_the_tile_grid(ctx, capi, ref, n_rx):
    """Spectrum-L1 step on the tensor-core path (k_cond_tc forward,
    k_cond_bwd_tc rows, k_cond_grads_tc GEMMs) with receiver counts that are
    not multiples of the 4-receiver tile groups (idle warps in the last
    tiles) and row totals that are not multiples of the 64-row GEMM chunk
    (zeroed tails): summed gradients vs the reference, bitwise repeatable."""
    sc, scene, cond, grid, og, rscene, rcond, params = _setup(capi, ctx, ref, k=1500)
    rx = capi.synth_points(n_rx, 19, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    tg = _targets(n_rx, grid.cells, seed=n_rx)
    st = scene.tx_state(TX, grid)
    tr = capi.Trainer(ctx, scene, cond, capi.Trainer.L1_ONLY)
    loss = tr.grads(st, rx, tg)
    db, dp = tr.get_grads()
    tr.grads(st, rx, tg)
    db2, dp2 = tr.get_grads()
    assert np.array_equal(db, db2) and np.array_equal(dp, dp2)
    want_b, want_p = np.zeros_like(db), np.zeros_like(dp)
    for j in range(n_rx):
        r = ref.train_sample(rscene, rcond, og, TX, rx[j], tg[j].astype(np.float64))
        assert rel_err(loss[j], r["loss"]) < TOL
        want_b += r["d_base"]
        want_p += r["d_params"]
    assert rel_err(db, want_b).max() < TOL
    assert rel_err(dp, want_p).max() < TOL


@pytest.mark.parametrize("lambdas", [(0.2, 0.1), (0.5, 0.0), (0.0, 0.3)])
def test_train_full_loss_matches_reference(ctx, capi, ref, lambdas):
    """composite_loss with the SSIM and DFT terms (trainer.cpp:113-139,
    metrics.cpp:55-112): loss and summed gradients vs the reference."""
    ls, lf = lambdas
    sc, scene, cond, grid, og, rscene, rcond, params = _setup(capi, ctx, ref)
    rx = capi.synth_points(3, 11, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    tg = _targets(3, grid.cells, 8)
    st = scene.tx_state(TX, grid)
    hp = list(capi.Trainer.DEFAULTS)
    hp[3], hp[4] = ls, lf
    tr = capi.Trainer(ctx, scene, cond, hp)
    loss = tr.grads(st, rx, tg)
    db, dp = tr.get_grads()
    want_b = np.zeros_like(db)
    want_p = np.zeros_like(dp)
    for j in range(3):
        r = ref.train_sample(rscene, rcond, og, TX, rx[j], tg[j].astype(np.float64), lambda_ssim=ls, lambda_fft=lf)
        assert rel_err(loss[j], r["loss"]) < TOL
        want_b += r["d_base"]
        want_p += r["d_params"]
    assert rel_err(db, want_b).max() < TOL
    assert rel_err(dp, want_p).max() < TOL


def test_train_ssim_needs_window(ctx, capi, ref):
    sc, scene, cond, grid, og, rscene, rcond, params = _setup(capi, ctx, ref, nt=8, np_=36)
    st = scene.tx_state(TX, grid)
    hp = list(capi.Trainer.DEFAULTS)
    hp[3] = 0.2
    tr = capi.Trainer(ctx, scene, cond, hp)
    rx = capi.synth_points(1, 11, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    with pytest.raises(capi.InvalidArgument, match="ssim: image smaller than the window"):
        tr.grads(st, rx, _targets(1, grid.cells))


def test_train_deterministic_and_accumulate(ctx, capi, ref):
    sc, scene, cond, grid, og, rscene, rcond, params = _setup(capi, ctx, ref, k=500)
    rx = capi.synth_points(4, 13, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    tg = _targets(4, grid.cells, 9)
    st = scene.tx_state(TX, grid)
    tr = capi.Trainer(ctx, scene, cond, capi.Trainer.L1_ONLY)
    tr.grads(st, rx, tg)
    a = np.concatenate(tr.get_grads())
    tr.grads(st, rx, tg)
    b = np.concatenate(tr.get_grads())
    assert np.array_equal(a, b)  # fixed-order reductions: bitwise reproducible
    tr.grads(st, rx[:2], tg[:2])
    tr.grads(st, rx[2:], tg[2:], accumulate=True)
    c = np.concatenate(tr.get_grads())
    assert rel_err(c, a).max() < 1e-6


def test_train_apply_is_adam(ctx, capi, ref):
    sc, scene, cond, grid, og, rscene, rcond, params = _setup(capi, ctx, ref, k=400)
    rx = capi.synth_points(2, 17, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    tg = _targets(2, grid.cells, 3)
    st = scene.tx_state(TX, grid)
    hyper = (5e-3, 0.2, 1e-3, 0.0, 0.0, 0.9, 0.999, 1e-8)
    tr = capi.Trainer(ctx, scene, cond, hyper)
    base0 = capi.scene_coeffs(scene)
    par0 = capi.cond_params(cond)
    tr.grads(st, rx, tg)
    db, dp = tr.get_grads()
    tr.apply()
    # one Adam step from zero moments: w - lr * g / (|g| + eps) (bias-corrected), diffengine.cpp:10-34
    def adam1(w, g, lr, scale):
        m = 0.1 * g
        v = 0.001 * g * g
        return w - lr * scale * (m / 0.1) / (np.sqrt(v / 0.001) + 1e-8)
    L = 9
    scale = np.where((np.arange(db.size) // 2) % L == 0, 1.0, 0.2)
    assert rel_err(capi.scene_coeffs(scene), adam1(base0, db, 5e-3, scale)).max() < 1e-12
    assert rel_err(capi.cond_params(cond), adam1(par0, dp, 1e-3, 1.0)).max() < 1e-12
    assert tr.step_count == 1
    # the updated device parameters drive the next forward (tcgen05 path included)
    spec1, _ = scene.render_queries(cond, scene.tx_state(TX, grid), rx)
    spec0 = None
    assert np.isfinite(spec1).all()


def _nccl_one_rank_comm():
    """A 1-rank ncclComm_t from the process's libnccl (torch's, once torch is loaded)."""
    import ctypes
    import torch  # noqa: F401  (loads torch's NCCL so the library resolves the same copy)
    torch.cuda.set_device(0)
    lib = ctypes.CDLL("libnccl.so.2")

    class UniqueId(ctypes.Structure):  # ncclUniqueId, passed by value
        _fields_ = [("internal", ctypes.c_char * 128)]

    uid = UniqueId()
    assert lib.ncclGetUniqueId(ctypes.byref(uid)) == 0
    comm = ctypes.c_void_p()
    lib.ncclCommInitRank.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, UniqueId, ctypes.c_int]
    assert lib.ncclCommInitRank(ctypes.byref(comm), 1, uid, 0) == 0
    return lib, comm


def test_train_allreduce_nccl(ctx, capi, ref):
    """rxgs_train_allreduce: ncclAllReduce(sum, f64) of the flat gradient buffer
    on the library stream; over one rank the buffer is unchanged, and the
    following apply() sees it."""
    sc, scene, cond, grid, og, rscene, rcond, params = _setup(capi, ctx, ref)
    rx = capi.synth_points(2, 13, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    tg = _targets(2, grid.cells)
    st = scene.tx_state(TX, grid)
    tr = capi.Trainer(ctx, scene, cond, capi.Trainer.L1_ONLY)
    tr.grads(st, rx, tg)
    db0, dp0 = tr.get_grads()
    lib, comm = _nccl_one_rank_comm()
    try:
        tr.allreduce(comm.value)
        db1, dp1 = tr.get_grads()
        assert np.array_equal(db0, db1) and np.array_equal(dp0, dp1)
        with pytest.raises(capi.RxgsError, match="null argument"):
            tr.allreduce(0)
    finally:
        lib.ncclCommDestroy(comm)
    tr.apply()
    assert tr.step_count == 1


def _lr_at(lr_init, lr_final, total, delay_mult, delay, t):
    """opt::lr_at (diffengine.cpp:36-48)."""
    frac = t / total if total > 0 else 1.0
    base = lr_init * (lr_final / lr_init) ** frac
    ramp = 1.0
    if delay > 0:
        u = min(max(t / delay, 0.0), 1.0)
        ramp = delay_mult + (1.0 - delay_mult) * np.sin(0.5 * np.pi * u)
    return base * ramp


def _adam1(w, g, lr, scale=1.0):
    """One Adam step from zero moments (diffengine.cpp:10-34)."""
    m = 0.1 * g
    v = 0.001 * g * g
    return w - lr * scale * (m / 0.1) / (np.sqrt(v / 0.001) + 1e-8)


@pytest.mark.parametrize("mode", ["full", "no_occlusion"])
def test_train_joint_grads_match_reference_sum(ctx, capi, ref, mode):
    """Joint step (train_geometry, trainer.cpp:440-449): the geometry gradients of
    backward_render summed over the batch, next to d_base and the conditioning
    gradients, vs the reference's per-sample gradients (SURVEY.md 8c4 'joint')."""
    sc, scene, cond, grid, og, rscene, rcond, params = _setup(capi, ctx, ref, k=500, mode=mode)
    rx = capi.synth_points(3, 19, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    tg = _targets(3, grid.cells, 4)
    st = scene.tx_state(TX, grid)
    tr = capi.Trainer(ctx, scene, cond, capi.Trainer.L1_ONLY, geometry=True)
    assert tr.n == tr.n_base + cond.param_count + 11 * scene.k
    loss = tr.grads(st, rx, tg)
    db, dp = tr.get_grads()
    gpos, gls, gq, gtau = tr.get_geometry_grads()
    want = dict(d_base=0.0, d_params=0.0, d_positions=0.0, d_log_scales=0.0, d_quaternions=0.0, d_tau_logits=0.0)
    for j in range(3):
        r = ref.train_sample(rscene, rcond, og, TX, rx[j], tg[j].astype(np.float64), geometry=True)
        assert rel_err(loss[j], r["loss"]) < TOL
        for key in want:
            want[key] = want[key] + r[key]
    assert rel_err(db, want["d_base"]).max() < TOL
    assert rel_err(dp, want["d_params"]).max() < TOL
    for got, key in ((gpos, "d_positions"), (gls, "d_log_scales"), (gq, "d_quaternions"), (gtau, "d_tau_logits")):
        assert np.abs(want[key]).max() > 0, key
        assert rel_err(got, want[key]).max() < TOL, key
    # accumulate over two calls == one batch
    tr.grads(st, rx[:1], tg[:1])
    tr.grads(st, rx[1:], tg[1:], accumulate=True)
    assert rel_err(np.concatenate(tr.get_geometry_grads()), np.concatenate((gpos, gls, gq, gtau))).max() < 1e-9


def test_train_joint_apply(ctx, capi, ref):
    """Joint optimizer step (trainer.cpp:450-463): degree mask at t = 0 (only
    degree-0 coefficients move), position at lr_at(position_lr, 0), the
    constant geometry rates, quaternions renormalised; the next TxState is
    built from the updated geometry."""
    sc, scene, cond, grid, og, rscene, rcond, params = _setup(capi, ctx, ref, k=400)
    rx = capi.synth_points(2, 23, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    tg = _targets(2, grid.cells, 6)
    geo = (1.6e-4, 1.6e-6, 2000, 0.01, 200, 1e-2, 5e-3, 1e-3, 500)
    olo, ohi = scene.bounds(0.1)
    occ = cond.build_occupancy(scene, 32, olo, ohi)  # as in _setup; fixed for the run (trainer.cpp:395-397)
    tr = capi.Trainer(ctx, scene, cond, capi.Trainer.L1_ONLY, geometry=geo)
    a0 = capi.scene_arrays(scene)
    par0 = capi.cond_params(cond)
    st = scene.tx_state(TX, grid)
    tr.grads(st, rx, tg)
    db, dp = tr.get_grads()
    gpos, gls, gq, gtau = tr.get_geometry_grads()
    tr.apply()
    a1 = capi.scene_arrays(scene)
    lr_pos = _lr_at(*geo[:5], 0)
    assert rel_err(a1["positions"], _adam1(a0["positions"], gpos, lr_pos)).max() < 1e-12
    assert rel_err(a1["tau_logits"], _adam1(a0["tau_logits"], gtau, 1e-2)).max() < 1e-12
    assert rel_err(a1["log_scales"], _adam1(a0["log_scales"], gls, 5e-3)).max() < 1e-12
    q = _adam1(a0["quaternions"], gq, 1e-3).reshape(-1, 4)
    q = q * (1.0 / np.sqrt((q * q).sum(axis=1)))[:, None]
    assert rel_err(a1["quaternions"], q.ravel()).max() < 1e-12
    L = 9
    deg0 = (np.arange(db.size) // 2) % L == 0
    want_f = np.where(deg0, _adam1(a0["fle_coeffs"], db, 5e-3), a0["fle_coeffs"])
    assert rel_err(a1["fle_coeffs"], want_f).max() < 1e-12
    assert rel_err(capi.cond_params(cond), _adam1(par0, dp, 1e-3)).max() < 1e-12
    # step 2 on the updated geometry: TxState rebuilt, gradients still match the reference
    r2 = ref.scene(dict(sc, positions=a1["positions"].reshape(-1, 3), log_scales=a1["log_scales"].reshape(-1, 3),
                        quaternions=a1["quaternions"].reshape(-1, 4), tau_logits=a1["tau_logits"],
                        fle_coeffs=a1["fle_coeffs"].reshape(sc["fle_coeffs"].shape)), "spectrum")
    st2 = scene.tx_state(TX, grid)
    loss2 = tr.grads(st2, rx[:1], tg[:1])
    cfg = capi.cond_cfg(mode="full")
    rc2 = ref.cond(cfg, capi.cond_params(cond), occ, olo, ohi)
    r = ref.train_sample(r2, rc2, og, TX, rx[0], tg[0].astype(np.float64), geometry=True)
    assert rel_err(loss2[0], r["loss"]) < TOL
    assert rel_err(tr.get_geometry_grads()[0], r["d_positions"]).max() < TOL


def test_train_nonfinite_group_names(ctx, capi, ref):
    """The non-finite check names the reference's optimizer group, first in
    its step order (diffengine.cpp:50-58, trainer.cpp:258-273, 450-462);
    components hidden by the degree mask are not checked."""
    import torch
    sc, scene, cond, grid, og, rscene, rcond, params = _setup(capi, ctx, ref, k=300)
    rx = capi.synth_points(1, 29, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    tg = _targets(1, grid.cells, 8)
    st = scene.tx_state(TX, grid)
    tr = capi.Trainer(ctx, scene, cond, capi.Trainer.L1_ONLY, geometry=True)
    tr.grads(st, rx, tg)
    g = tr.grad_tensor()
    nb, npar, k = tr.n_base, cond.param_count, scene.k
    g[2 * 1] = float("nan")  # component 1 (degree 1) of Gaussian 0: masked at t = 0
    g[nb + npar - 1] = float("nan")  # cond.local.b3
    torch.cuda.synchronize()
    with pytest.raises(capi.RxgsError, match="non-finite gradient in group 'cond.local.b3'"):
        tr.apply()
    g[nb + npar + 3 * k] = float("nan")  # transmittance
    g[nb + npar + 7 * k + 2] = float("nan")  # rotation
    torch.cuda.synchronize()
    with pytest.raises(capi.RxgsError, match="non-finite gradient in group 'transmittance'"):
        tr.apply()
    g[0] = float("nan")  # features, degree 0
    g[nb + npar + 3 * k] = 0.0
    g[nb + npar + 7 * k + 2] = 0.0
    torch.cuda.synchronize()
    with pytest.raises(capi.RxgsError, match="non-finite gradient in group 'features'"):
        tr.apply()
    assert tr.step_count == 0


def _stage1_setup(capi, ctx, ref, k=400, seed=7, big=()):
    import oracle as O
    sc = capi.synth_scene(k, 2, 1, seed)
    if big:
        ls = sc["log_scales"].copy()
        ls[list(big)] = np.log(5.0)
        sc = dict(sc, log_scales=ls)
    scene = ctx.scene(sc, "spectrum")
    grid = capi.Grid(18, 36, 8, 1.0)
    return sc, scene, grid, O.Grid(18, 36, 8, 1.0)


def test_stage1_grads_match_reference(ctx, capi, ref):
    """Stage-I step (train_stage1, trainer.cpp:317-340): no conditioning, the
    scene's coefficients render; d_base = backward_render's d_coeffs and the
    geometry gradients, summed over the batch, vs the reference."""
    sc, scene, grid, og = _stage1_setup(capi, ctx, ref)
    rx = capi.synth_points(2, 31, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    tg = _targets(2, grid.cells, 12)
    tr = capi.Trainer(ctx, scene, None, capi.Trainer.L1_ONLY, geometry=True)
    assert tr.n == tr.n_base + 11 * scene.k
    loss = tr.grads(scene.tx_state(TX, grid), rx, tg)
    db, dp = tr.get_grads()
    assert dp.size == 0
    geo = tr.get_geometry_grads()
    rs = ref.scene(sc, "spectrum")
    want = [0.0] * 5
    for j in range(2):
        r = ref.train_sample(rs, None, og, TX, rx[j], tg[j].astype(np.float64), geometry=True)
        assert rel_err(loss[j], r["loss"]) < TOL
        for i, key in enumerate(("d_base", "d_positions", "d_log_scales", "d_quaternions", "d_tau_logits")):
            want[i] = want[i] + r[key]
    assert rel_err(db, want[0]).max() < TOL
    for got, w in zip(geo, want[1:]):
        assert rel_err(got, w).max() < TOL


def test_stage1_densify_and_tau_reset(ctx, capi, ref):
    """Stage-I policy ticks through the trainer (trainer.cpp:351-372):
    DensifyState accumulated per step, densify_and_prune == the reference's on
    the same state, the optimizer state remapped (training continues on the
    new row set), reset_transmittance + a fresh Adam count for that group."""
    sc, scene, grid, og = _stage1_setup(capi, ctx, ref, big=(3, 77))
    rx = capi.synth_points(1, 37, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    tg = _targets(1, grid.cells, 13)
    tr = capi.Trainer(ctx, scene, None, capi.Trainer.L1_ONLY, geometry=True)
    d_pos = []
    for _ in range(2):
        tr.grads(scene.tx_state(TX, grid), rx, tg)
        d_pos.append(tr.get_geometry_grads()[0])
        tr.apply()
    before = capi.scene_arrays(scene)
    thr, extent, seed = (1e-6, 0.01, 0.1, 0.8), 40.0, 5
    rep = tr.densify(extent, thr, seed, 2)
    h = ref.scene(dict(sc, positions=before["positions"].reshape(-1, 3),
                       log_scales=before["log_scales"].reshape(-1, 3),
                       quaternions=before["quaternions"].reshape(-1, 4), tau_logits=before["tau_logits"],
                       fle_coeffs=before["fle_coeffs"].reshape(-1, 9, 1, 2)), "spectrum")
    rrep, rsrc = ref.densify(h, np.stack(d_pos), extent, thr, seed, 2)
    assert list(rep) == list(rrep) and min(rep) > 0, rep
    got, want = capi.scene_arrays(scene), ref.scene_arrays(h)
    for key in want:
        np.testing.assert_allclose(got[key], want[key], rtol=1e-15, atol=1e-15, err_msg=key)
    assert scene.k == len(rsrc) and tr.n == tr.n_base + 11 * scene.k
    # training continues on the new rows
    loss = tr.grads(scene.tx_state(TX, grid), rx, tg)
    assert np.isfinite(loss).all()
    tr.apply()
    # transmittance reset: logit(0.01) everywhere, then that group's Adam restarts at step 1
    tr.reset_transmittance()
    tau0 = capi.scene_arrays(scene)["tau_logits"]
    assert np.array_equal(tau0, np.full(scene.k, np.log(0.01 / (1.0 - 0.01))))
    tr.grads(scene.tx_state(TX, grid), rx, tg)
    gtau = tr.get_geometry_grads()[3]
    tr.apply()
    assert rel_err(capi.scene_arrays(scene)["tau_logits"], _adam1(tau0, gtau, 1e-2)).max() < 1e-12


def test_train_geometry_api_errors(ctx, capi, ref):
    """Densification / transmittance reset need the geometry step; geometry must
    be enabled before the first step (reference-style located messages)."""
    sc, scene, grid, og = _stage1_setup(capi, ctx, ref, k=200)
    tr = capi.Trainer(ctx, scene, None, capi.Trainer.L1_ONLY)
    with pytest.raises(capi.InvalidArgument, match="densification needs rxgs_trainer_enable_geometry"):
        tr.densify(10.0)
    with pytest.raises(capi.InvalidArgument, match="transmittance reset needs rxgs_trainer_enable_geometry"):
        tr.reset_transmittance()
    with pytest.raises(capi.InvalidArgument, match="geometry gradients need rxgs_trainer_enable_geometry"):
        tr.get_geometry_grads()
    rx = capi.synth_points(1, 41, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    tr.grads(scene.tx_state(TX, grid), rx, _targets(1, grid.cells, 3))
    tr.apply()
    import ctypes
    geo = np.asarray(capi.Trainer.GEOMETRY_DEFAULTS, np.float64)
    assert capi._lib.rxgs_trainer_enable_geometry(tr.h, geo.ctypes.data) == capi.RXGS_ERR_INVALID
    assert "enable geometry before the first step" in capi._lib.rxgs_last_error().decode()


def test_train_unconditioned_stage2_matches_reference(ctx, capi, ref):
    """cond == NULL without geometry: the base coefficients alone, d_base =
    backward_render's d_coeffs summed over the batch."""
    sc, scene, grid, og = _stage1_setup(capi, ctx, ref, k=300)
    rx = capi.synth_points(2, 43, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    tg = _targets(2, grid.cells, 14)
    tr = capi.Trainer(ctx, scene, None, capi.Trainer.L1_ONLY)
    assert tr.n == tr.n_base
    loss = tr.grads(scene.tx_state(TX, grid), rx, tg)
    db, dp = tr.get_grads()
    rs = ref.scene(sc, "spectrum")
    want = 0.0
    for j in range(2):
        r = ref.train_sample(rs, None, og, TX, rx[j], tg[j].astype(np.float64))
        assert rel_err(loss[j], r["loss"]) < TOL
        want = want + r["d_base"]
    assert rel_err(db, want).max() < TOL


def test_joint_densify_keeps_conditioning(ctx, capi, ref):
    """Densifying a conditioned (joint) trainer remaps the per-Gaussian groups
    only: the conditioning parameters are untouched and training continues on
    the new row set with the conditioning gradients still matching."""
    sc, scene, cond, grid, og, rscene, rcond, params = _setup(capi, ctx, ref, k=400)
    rx = capi.synth_points(1, 47, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    tg = _targets(1, grid.cells, 15)
    tr = capi.Trainer(ctx, scene, cond, capi.Trainer.L1_ONLY, geometry=True)
    tr.grads(scene.tx_state(TX, grid), rx, tg)
    tr.apply()
    par = capi.cond_params(cond)
    k0 = scene.k
    rep = tr.densify(40.0, (1e-6, 0.01, 0.1, 0.8), 3, 0)
    assert sum(rep) > 0 and scene.k != k0
    assert np.array_equal(capi.cond_params(cond), par)
    assert tr.n == tr.n_base + cond.param_count + 11 * scene.k
    loss = tr.grads(scene.tx_state(TX, grid), rx, tg)
    assert np.isfinite(loss).all()
    tr.apply()
    assert np.isfinite(capi.scene_arrays(scene)["positions"]).all()


_FAKE_NCCL_CHILD = r"""
import ctypes, sys
import numpy as np
sys.path[:0] = [sys.argv[1], sys.argv[1] + "/tests"]
from paper_2605_24290_b200 import capi
fake = ctypes.CDLL(sys.argv[2])
fake.fake_nccl_last_count.restype = ctypes.c_size_t
ctx = capi.Context(0)
sc = capi.synth_scene(500, 2, 1, 7)
scene = ctx.scene(sc, "spectrum")
lo, hi = scene.bounds(0.0)
cfg = capi.cond_cfg()
cond = ctx.cond(cfg, capi.synth_cond(cfg, 2, 1, lo, hi, 3, True))
olo, ohi = scene.bounds(0.1)
cond.build_occupancy(scene, 32, olo, ohi)
grid = capi.Grid(18, 36, 8, 1.0)
rx = capi.synth_points(2, 13, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
tg = np.random.default_rng(5).uniform(0, 2, (2, grid.cells)).astype(np.float32)
tr = capi.Trainer(ctx, scene, cond, capi.Trainer.L1_ONLY, geometry=True)
tr.grads(scene.tx_state([0.3, -0.2, 0.1], grid), rx, tg)
g0 = tr.grad_buffer_host()
tr.allreduce(1)
g1 = tr.grad_buffer_host()
n = fake.fake_nccl_last_count()
assert n == g0.size, (n, g0.size)
geo = g0.size - 11 * 500
assert np.abs(g0[geo:]).max() > 0
assert np.array_equal(g1, 2.0 * g0), "not every segment was reduced"
print("ok", n)
"""


def test_train_allreduce_covers_geometry_segment(tmp_path):
    """ADVICE r1 (train_api.cu:366): the all-reduce must cover the whole flat
    buffer, including the joint trainer's 11 K geometry gradients.  A fake
    ncclAllReduce (tests/cpp/fake_nccl.c: a sum over two identical ranks)
    stands in for a 2-GPU communicator; every value must double."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    so = str(tmp_path / "libfake_nccl.so")
    subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-I/usr/local/cuda/include",
                           os.path.join(root, "tests", "cpp", "fake_nccl.c"), "-o", so,
                           "-L/usr/local/cuda/lib64/stubs", "-lcuda"])
    env = dict(os.environ, RXGS_NCCL_LIBRARY=so)
    out = subprocess.run([sys.executable, "-c", _FAKE_NCCL_CHILD, root, so], env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.strip().startswith("ok")
