"""Parity of the transmitter-side state (projection, basis, per-tile lists,
sort keys) between the CUDA path (through the C-ABI) and the CPU oracle.

Bit-exact: culled flags, tile spans, per-tile lists, sort keys.
FP64 geometry / basis: libm ulp differences only (CUDA vs glibc atan2/sin/
cos/exp), checked at 1e-12 rel_err.
"""
import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu

TX = np.array([0.3, -0.2, 0.1])


def _oracle_keys(og, otx):
    """(tile << 32) | rank with rank = position in (depth, index) order."""
    geom, culled = otx.data["geom"], otx.data["culled"]
    depth = np.where(culled == 0, geom[:, 2], np.inf)
    order = np.lexsort((np.arange(len(depth)), depth))
    rank = np.empty_like(order)
    rank[order] = np.arange(len(order))
    offs, idx = otx.data["offsets"], otx.data["indices"]
    tiles = np.repeat(np.arange(og.n_tiles, dtype=np.uint64), np.diff(offs))
    return (tiles << np.uint64(32)) | rank[idx].astype(np.uint64)


@pytest.mark.parametrize("k,nt,np_,ts", [(2000, 30, 60, 8), (10_000, 90, 360, 8), (5000, 24, 48, 4),
                                          (3000, 20, 44, 8)])
def test_tx_state_matches_oracle(ctx, capi, orc, k, nt, np_, ts):
    import oracle as O
    sc = capi.synth_scene(k, 2, 1, 7)
    grid = capi.Grid(nt, np_, ts, 1.0)
    st = ctx.scene(sc).tx_state(TX, grid)
    got = st.get()
    og = O.Grid(nt, np_, ts, 1.0)
    otx = orc.tx_state(orc.scene(sc), TX, og)
    want = otx.data
    assert np.array_equal(got["culled"], want["culled"])
    assert np.array_equal(got["spans"], want["spans"])
    vis = want["culled"] == 0
    assert rel_err(got["geom"][vis], want["geom"][vis]).max() < 1e-12
    assert rel_err(got["basis"], want["basis"]).max() < 1e-12
    assert np.array_equal(got["offsets"], want["offsets"])
    assert np.array_equal(got["indices"], want["indices"])
    assert np.array_equal(st.keys(), _oracle_keys(og, otx))


@pytest.mark.slow
@pytest.mark.parametrize("k,nt,np_", [(100_000, 90, 360), (500_000, 90, 360), (2_000_000, 180, 720)])
def test_tx_state_full_size_configs(ctx, capi, orc, k, nt, np_):
    """BASELINE configs 2/3/5 geometry: lists and keys bit-exact at full size."""
    import oracle as O
    sc = capi.synth_scene(k, 2, 1, 7)
    st = ctx.scene(sc).tx_state(TX, capi.Grid(nt, np_, 8, 1.0))
    og = O.Grid(nt, np_, 8, 1.0)
    otx = orc.tx_state(orc.scene(sc), TX, og)
    got = st.get()
    assert np.array_equal(got["spans"], otx.data["spans"])
    assert np.array_equal(got["offsets"], otx.data["offsets"])
    assert np.array_equal(got["indices"], otx.data["indices"])
    keys = st.keys()
    assert np.array_equal(keys, _oracle_keys(og, otx))
    assert np.all(np.diff(keys.astype(np.float64)) > 0) or np.all(keys[1:] > keys[:-1])


def test_bin_and_sort_on_reference_projections(ctx, capi, orc):
    """bin_and_sort fed the ORACLE's projections: isolates the sort from libm."""
    import oracle as O
    sc = capi.synth_scene(20_000, 2, 1, 9)
    og = O.Grid(90, 360, 8, 1.0)
    otx = orc.tx_state(orc.scene(sc), TX, og)
    d = otx.data
    offs, idx = ctx.bin_and_sort(d["culled"], d["geom"][:, 2], d["spans"], capi.Grid(90, 360, 8, 1.0))
    assert np.array_equal(offs, d["offsets"])
    assert np.array_equal(idx, d["indices"])


def test_many_tiles_generic_path(ctx, capi, orc):
    """More than 4096 tiles: the generic binning path ((tile, rank) pairs and
    LSD passes on the tile id, k_sort.cu) instead of the fused pass."""
    import oracle as O
    sc = capi.synth_scene(6000, 2, 1, 11)
    grid = capi.Grid(160, 720, 4, 1.0)  # 40 x 180 = 7200 tiles
    st = ctx.scene(sc).tx_state(TX, grid)
    og = O.Grid(160, 720, 4, 1.0)
    otx = orc.tx_state(orc.scene(sc), TX, og)
    got = st.get()
    assert np.array_equal(got["offsets"], otx.data["offsets"])
    assert np.array_equal(got["indices"], otx.data["indices"])
    assert np.array_equal(st.keys(), _oracle_keys(og, otx))


def test_bin_and_sort_depth_ties_and_near_ties(ctx, capi):
    """Runs of equal or nearly equal FP64 depths (equal after the 32-bit key
    truncation of the device depth rank) keep the (depth, index) order; a
    non-culled Gaussian with an empty span contributes no entries."""
    rng = np.random.default_rng(3)
    n = 5000
    depth = 1.0 + rng.integers(0, 40, n) * 0.25  # many exact ties
    depth[::7] = 3.0 + rng.integers(0, 5, len(depth[::7])) * 1e-15  # near ties, distinct bits
    depth[::11] = np.nextafter(2.0, 3.0)
    culled = (rng.uniform(size=n) < 0.1).astype(np.int32)
    t0 = rng.integers(0, 2, n)
    p0 = rng.integers(0, 6, n)
    spans = np.stack([t0, t0 + rng.integers(0, 2, n), p0, p0 + rng.integers(0, 3, n)], 1).astype(np.int32)
    spans[5] = [1, 0, 0, -1]  # empty span, not culled
    grid = capi.Grid(24, 48, 8, 0.25)  # 3 x 6 tiles; spans wrap past tiles_phi
    offs, idx = ctx.bin_and_sort(culled, depth, spans, grid)
    tp = 6
    want = [[] for _ in range(18)]
    for g in sorted(range(n), key=lambda i: (depth[i], i)):
        if culled[g]:
            continue
        t0_, t1_, p0_, p1_ = spans[g]
        for tt in range(t0_, t1_ + 1):
            for pp in range(p0_, p1_ + 1):
                want[tt * tp + pp % tp].append(g)
    got = [list(idx[offs[t]:offs[t + 1]]) for t in range(18)]
    assert got == want


def test_bin_and_sort_tie_order_and_seam(ctx, capi):
    """Reference KATs: test_sphraster.cpp:96-119 ({1,0,2}) and :121-132 (seam)."""
    grid = capi.Grid(6, 12, 4, 0.25)  # 2 x 3 tiles
    culled = [0, 0, 0]
    depth = [2.0, 1.0, 2.0]
    spans = [[0, 1, 0, 2], [0, 0, 1, 1], [0, 0, 1, 1]]
    offs, idx = ctx.bin_and_sort(culled, depth, spans, grid)
    lists = [list(idx[offs[t]:offs[t + 1]]) for t in range(6)]
    assert sum(0 in l_ for l_ in lists) == 6
    assert lists[1] == [1, 0, 2]
    offs, idx = ctx.bin_and_sort([0], [1.0], [[0, 0, 2, 3]], grid)
    lists = [list(idx[offs[t]:offs[t + 1]]) for t in range(6)]
    assert lists[0] == [0] and lists[1] == [] and lists[2] == [0]


def test_projection_kats(ctx, capi):
    """test_sphraster.cpp:59-94: axis direction, isotropic sigma^2/d^2, culling."""
    grid = capi.Grid(6, 12, 4, 0.25)
    # one isotropic Gaussian at (0, 2, 0): sigma^2 = 0.04 -> log_scale = ln(0.2)
    sc = dict(positions=np.array([[0.0, 2.0, 0.0], [1.0, 0.0, 0.0], [0.1, 0.0, 0.0]]),
              log_scales=np.log(np.full((3, 3), 0.2)), quaternions=np.tile([1.0, 0, 0, 0], (3, 1)),
              tau_logits=np.zeros(3), fle_coeffs=np.zeros((3, 1, 1, 2)), l_max=0, channels=1)
    got = ctx.scene(sc).tx_state([0, 0, 0], grid).get()
    g = got["geom"]
    assert got["culled"].tolist() == [0, 0, 1]
    assert rel_err(g[0, 3], 0.04 / 4).max() < 1e-12 and rel_err(g[0, 6], 0.04 / 4).max() < 1e-12
    assert abs(g[0, 4]) < 1e-15
    assert rel_err(g[1, 0], np.pi / 2) < 1e-14 and abs(g[1, 1]) < 1e-14 and rel_err(g[1, 2], 1.0) < 1e-14


def test_occupancy_matches_oracle(ctx, capi, orc):
    sc = capi.synth_scene(5000, 2, 1, 7)
    scene = ctx.scene(sc)
    lo, hi = scene.bounds(0.1)
    got = capi.build_occupancy(ctx, scene, 32, lo, hi)
    want = orc.build_occupancy(orc.scene(sc), 32, lo, hi)
    assert rel_err(got, want).max() < 1e-12
