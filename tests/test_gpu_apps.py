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
