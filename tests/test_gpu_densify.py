"""Stage-I densification on the device: densify_and_prune
(scene.cpp:178-274) and reset_transmittance (scene.cpp:276-279) vs the
reference build -- the same row set and source rows exactly, positions and
scales to the last bits (the device exp may differ from glibc's by an ulp),
including the reference suite's hand cases (test_scene.cpp:164-260)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

THR = (2e-4, 0.01, 0.1, 0.8)


def _scene_dict(pos, log_scales=None, l_max=0, channels=1):
    """init_scene-like arrays (scene.cpp:106-139): identity rotations,
    tau = logit(0.1), zero coefficients."""
    pos = np.asarray(pos, np.float64).reshape(-1, 3)
    k = len(pos)
    if log_scales is None:
        d2 = ((pos[:, None, :] - pos[None, :, :]) ** 2).sum(-1)
        np.fill_diagonal(d2, np.inf)
        log_scales = np.repeat(0.5 * np.log(d2.min(1))[:, None], 3, 1)
    q = np.zeros((k, 4))
    q[:, 0] = 1.0
    L = (l_max + 1) ** 2
    rng = np.random.default_rng(k)
    return dict(positions=pos, log_scales=np.asarray(log_scales, np.float64).reshape(k, 3), quaternions=q,
                tau_logits=np.full(k, np.log(0.1 / 0.9)), fle_coeffs=rng.normal(size=(k, L, channels, 2)),
                l_max=l_max, channels=channels)


def _run_both(ctx, ref, capi, sc, grads_list, extent, thr=THR, seed=1, pass_index=0):
    grads_list = np.asarray(grads_list, np.float64).reshape(len(grads_list), -1)
    acc = np.zeros(len(sc["tau_logits"]))
    cnt = np.zeros(len(acc), np.int32)
    for g in grads_list:  # DensifyState::accumulate (scene.cpp:141-151)
        acc += np.sqrt((g.reshape(-1, 3) ** 2).sum(1))
        cnt += 1
    scene = ctx.scene(sc, "spectrum")
    rep, src = scene.densify_and_prune(acc, cnt, extent, thr, seed, pass_index)
    h = ref.scene(sc, "spectrum")
    rrep, rsrc = ref.densify(h, grads_list, extent, thr, seed, pass_index)
    return scene, rep, src, ref.scene_arrays(h), rrep, rsrc


def _same(got, want):
    for key in ("positions", "log_scales", "quaternions", "tau_logits", "fle_coeffs"):
        assert got[key].shape == want[key].shape, key
        np.testing.assert_allclose(got[key], want[key], rtol=1e-15, atol=1e-15, err_msg=key)


def test_below_threshold_is_noop(ctx, ref, capi):
    sc = _scene_dict([[0, 0, 0], [1, 0, 0], [0, 1, 0]])
    scene, rep, src, want, rrep, rsrc = _run_both(ctx, ref, capi, sc, [np.full(9, 1e-9)], 10.0)
    assert list(rep) == [0, 0, 0] and list(src) == [0, 1, 2] == list(rsrc)
    assert np.array_equal(capi.scene_arrays(scene)["positions"], sc["positions"].ravel())


def test_small_gaussian_is_cloned(ctx, ref, capi):
    sc = _scene_dict([[0, 0, 0], [1, 0, 0]])
    scene, rep, src, want, rrep, rsrc = _run_both(ctx, ref, capi, sc, [[1.0, 0, 0, 0, 0, 0]], 1000.0)
    assert list(rep) == list(rrep) == [1, 0, 0]
    assert list(src) == list(rsrc) == [0, 1, -1]
    got = capi.scene_arrays(scene)
    assert np.array_equal(got["positions"][6:9], got["positions"][0:3])
    _same(got, want)


def test_large_gaussian_splits(ctx, ref, capi):
    sc = _scene_dict([[0, 0, 0], [1, 0, 0]], np.full((2, 3), np.log(0.5)))
    scene, rep, src, want, rrep, rsrc = _run_both(ctx, ref, capi, sc, [[1.0, 0, 0, 0, 0, 0]], 10.0)
    assert list(rep) == list(rrep) == [0, 1, 0]
    assert list(src) == list(rsrc) == [-1, 1, -1]
    got = capi.scene_arrays(scene)
    assert abs(got["log_scales"][0] - (np.log(0.5) + np.log(0.8))) < 1e-12
    a, b = got["positions"][0:3], got["positions"][6:9]
    assert abs(np.linalg.norm(a - b) - 1.0) < 1e-12
    _same(got, want)


def test_oversized_are_pruned(ctx, ref, capi):
    sc = _scene_dict([[0, 0, 0], [1, 0, 0], [0, 1, 0]], np.full((3, 3), np.log(5.0)))
    scene, rep, src, want, rrep, rsrc = _run_both(ctx, ref, capi, sc, [np.zeros(9)], 10.0)
    assert list(rep) == list(rrep) == [0, 0, 3]
    assert scene.k == 0 and len(rsrc) == 0


@pytest.mark.parametrize("k,seed,pass_index,l_max", [(3000, 1, 0, 2), (20000, 7, 3, 1), (500, 11, 1, 3)])
def test_random_states_match_reference(ctx, ref, capi, k, seed, pass_index, l_max):
    """Mixed keep / clone / split / prune over a synthetic scene with random
    rotations, several accumulate() calls, the scene-diagonal extent."""
    sc = capi.synth_scene(k, l_max, 1, seed)
    rng = np.random.default_rng(seed)
    ls = sc["log_scales"].copy()
    ls[rng.choice(k, k // 50, replace=False)] = np.log(1.5)  # some oversized
    ls[rng.choice(k, k // 10, replace=False)] -= 1.2          # some small enough to clone
    sc = dict(sc, log_scales=ls)
    grads = np.abs(rng.normal(size=(3, 3 * k))) * 1.6e-4
    lo, hi = sc["positions"].min(0), sc["positions"].max(0)
    extent = float(np.linalg.norm(hi - lo))
    scene, rep, src, want, rrep, rsrc = _run_both(ctx, ref, capi, sc, grads, extent, seed=seed,
                                                  pass_index=pass_index)
    assert list(rep) == list(rrep)
    assert min(rep) > 0, rep  # every operation occurs
    assert np.array_equal(src, rsrc)
    got = capi.scene_arrays(scene)
    _same(got, want)
    # the resized scene renders: TxState over the new row set
    st = scene.tx_state(np.array([0.3, -0.2, 0.1]), capi.Grid(18, 36, 6, 1.0))
    spec, _ = scene.render_queries(None, st, capi.synth_points(2, 3, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5]))
    assert np.isfinite(spec).all()


def test_reset_transmittance(ctx, ref, capi):
    sc = capi.synth_scene(100, 1, 1, 5)
    scene = ctx.scene(sc, "spectrum")
    scene.reset_transmittance()
    h = ref.scene(sc, "spectrum")
    ref._reset_transmittance(h.ptr)
    got = capi.scene_arrays(scene)
    assert np.array_equal(got["tau_logits"], ref.scene_arrays(h)["tau_logits"])
    assert np.array_equal(got["positions"], sc["positions"].ravel())
    scene.reset_transmittance()  # idempotent
    assert np.array_equal(capi.scene_arrays(scene)["tau_logits"], got["tau_logits"])
