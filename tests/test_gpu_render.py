"""Parity of the render path (materialised render_field, aggregation,
conditioning, fused batched queries) between the CUDA path and the oracle.

Float tolerance: the reference's rel_err (testutil.hpp:14-20) <= 1e-4 on
every float output (fields, spectra, RSSI dB, conditioned coefficients).
"""
import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu

TOL = 1e-4
TX = np.array([0.3, -0.2, 0.1])


def _random_coeffs(k, L, C, n_rx, seed=42):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((n_rx, k, L, C, 2))


def _setup_cond(capi, ctx, orc, sc, mode="full", hidden=64, S=16, R=32, nearest=0, occ=True):
    import oracle as O
    scene = ctx.scene(sc)
    lo, hi = scene.bounds(0.0)
    cfg = capi.cond_cfg(hidden=hidden, S=S, R=R, nearest=nearest, mode=mode, l_max=sc["l_max"], C_=sc["channels"])
    params = capi.synth_cond(cfg, sc["l_max"], sc["channels"], lo, hi, 3, True)
    cond = ctx.cond(cfg, params)
    oscene = orc.scene(sc)
    if occ:
        olo, ohi = scene.bounds(0.1)
        dens = cond.build_occupancy(scene, R, olo, ohi)
        ocond = orc.cond(cfg, params, dens, olo, ohi)
    else:
        ocond = orc.cond(cfg, params)
    return scene, cond, oscene, ocond


@pytest.mark.parametrize("k,l_max,C,n_rx,ts", [(800, 2, 1, 3, 8), (500, 1, 2, 2, 4), (1500, 3, 1, 5, 8)])
def test_render_field_matches_oracle(ctx, capi, orc, k, l_max, C, n_rx, ts):
    import oracle as O
    sc = capi.synth_scene(k, l_max, C, 7)
    grid = capi.Grid(24, 48, ts, 1.0)
    scene = ctx.scene(sc, "csi")
    st = scene.tx_state(TX, grid)
    co = _random_coeffs(k, (l_max + 1) ** 2, C, n_rx)
    vals, T = scene.render_field(st, co, n_rx)
    og = O.Grid(24, 48, ts, 1.0)
    oscene = orc.scene(sc, "csi")
    otx = orc.tx_state(oscene, TX, og)
    wv, wT = orc.render(otx, oscene, co, n_rx)
    assert rel_err(vals, wv).max() < TOL
    assert rel_err(T, wT).max() < 1e-12
    for m in (("csi",) if C > 1 else ("rssi", "csi", "spectrum")):
        assert rel_err(ctx.aggregate(vals, grid, m), orc.aggregate(wv, og, m)).max() < TOL


def test_render_batched_equals_sequential_bitwise(ctx, capi):
    """test_sphraster.cpp:180-199."""
    sc = capi.synth_scene(300, 2, 2, 41)
    grid = capi.Grid(6, 12, 4, 0.25)
    scene = ctx.scene(sc, "csi")
    st = scene.tx_state([0, 0, 0], grid)
    co = _random_coeffs(300, 9, 2, 3)
    vb, tb = scene.render_field(st, co, 3)
    for j in range(3):
        v1, t1 = scene.render_field(st, co[j:j + 1], 1)
        assert np.array_equal(vb[j], v1[0]) and np.array_equal(tb[j], t1[0])


def test_render_rejects_nonfinite_with_location(ctx, capi):
    """test_sphraster.cpp:211-223: first offending (rx, gaussian) in j-major order."""
    sc = capi.synth_scene(3, 1, 1, 45)
    scene = ctx.scene(sc, "rssi")
    st = scene.tx_state([0, 0, 0], capi.Grid(6, 12, 4, 0.25))
    co = _random_coeffs(3, 4, 1, 2)
    co.reshape(-1)[3 * 8 + 5] = np.nan
    with pytest.raises(capi.InvalidArgument, match=r"non-finite coefficient at rx 1, gaussian 0"):
        scene.render_field(st, co, 2)


def test_empty_scene_renders_zero_unit_T(ctx, capi):
    sc = dict(positions=np.zeros((0, 3)), log_scales=np.zeros((0, 3)), quaternions=np.zeros((0, 4)),
              tau_logits=np.zeros(0), fle_coeffs=np.zeros((0, 4, 1, 2)), l_max=1, channels=1)
    scene = ctx.scene(sc, "rssi")
    st = scene.tx_state([0, 0, 0], capi.Grid(6, 12, 4, 0.25))
    v, T = scene.render_field(st, np.zeros(0), 2)
    assert np.all(v == 0.0) and np.all(T == 1.0)


def test_aggregate_closed_forms(ctx, capi):
    """test_sphraster.cpp:250-303."""
    grid = capi.Grid(2, 3, 8, 1.0)
    f = np.zeros((1, 1, 2, 2, 3))
    assert rel_err(ctx.aggregate(f, grid, "rssi")[0], 10 * np.log10(1e-12)) < 1e-14
    f[0, 0, 0, 0, 0] = 1.0
    dom = np.sin(np.pi / 4) * (np.pi / 2) * (2 * np.pi / 3)
    assert rel_err(ctx.aggregate(f, grid, "rssi")[0], 10 * np.log10(dom + 1e-12)) < 1e-13
    g1 = capi.Grid(1, 1, 8, 1.0)
    f1 = np.array([3.0, 4.0]).reshape(1, 1, 2, 1, 1)
    assert rel_err(ctx.aggregate(f1, g1, "spectrum")[0, 0, 0], np.sqrt(25 + 1e-8)) < 1e-15
    with pytest.raises(capi.InvalidArgument, match="non-finite field"):
        ctx.aggregate(np.full((1, 1, 2, 1, 1), np.inf), g1, "spectrum")


@pytest.mark.parametrize("mode", ["full", "global_only", "local_only", "additive_only", "no_occlusion"])
def test_condition_forward_matches_oracle(ctx, capi, orc, mode):
    sc = capi.synth_scene(2000, 2, 1, 7)
    scene, cond, oscene, ocond = _setup_cond(capi, ctx, orc, sc, mode)
    for rx in ([1.1, 0.7, 0.2], [-2.5, 1.0, -0.9]):
        got = cond.forward(scene, rx)
        want = orc.cond_forward(ocond, oscene, rx)
        assert rel_err(got, want).max() < TOL


def test_condition_small_hidden_nearest(ctx, capi, orc):
    """Reference test configuration (tiny_config: hidden 8, S 4, R 8) + nearest lookup."""
    sc = capi.synth_scene(300, 1, 2, 5)
    scene, cond, oscene, ocond = _setup_cond(capi, ctx, orc, sc, "full", hidden=8, S=4, R=8, nearest=1)
    got = cond.forward(scene, [0.5, -0.5, 1.0])
    want = orc.cond_forward(ocond, oscene, [0.5, -0.5, 1.0])
    assert rel_err(got, want).max() < TOL


def test_condition_identity_bitwise_and_errors(ctx, capi):
    """test_conditioning.cpp:157-169 (fresh state = identity, bitwise), :226-241
    (receiver on a Gaussian -> located error), :292-304 (cost counters)."""
    sc = capi.synth_scene(50, 1, 2, 101)
    scene = ctx.scene(sc)
    cfg = capi.cond_cfg(F=2, hidden=8, dc=3, S=4, R=8, l_max=1, C_=2)
    params = capi.synth_cond(cfg, 1, 2, [-3, -3, -3], [3, 3, 3], 7, randomize=False)
    cond = ctx.cond(cfg, params)
    cond.build_occupancy(scene, 8, [-4, -4, -4], [4, 4, 4])
    for rx in ([0.3, 0.2, -1.0], [2.0, -1.0, 0.5]):
        assert np.array_equal(cond.forward(scene, rx), sc["fle_coeffs"])
    with pytest.raises(capi.InvalidArgument, match="receiver coincides with gaussian 7"):
        cond.forward(scene, sc["positions"][7])
    g0, l0 = cond.calls()
    cond.forward(scene, [1, 2, 0])
    g1, l1 = cond.calls()
    assert (g1 - g0, l1 - l0) == (4, 50)


def test_probe_kats(ctx, capi):
    """test_conditioning.cpp:114-133: uniform 0.1 grid -> T = 0.9^16, mean 0.1."""
    sc = capi.synth_scene(10, 0, 1, 1)
    cfg = capi.cond_cfg(F=1, hidden=8, dc=1, S=16, R=4, l_max=0)
    params = capi.synth_cond(cfg, 0, 1, [-1, -1, -1], [1, 1, 1], 1, False)
    occ = np.full((4, 4, 4), 0.1)
    cond = ctx.cond(cfg, params, occ, [-10, -10, -10], [10, 10, 10])
    out = cond.probe([-5, 0, 0], [5, 0, 0])
    assert rel_err(out[0, 0], 0.1853020188851841) < 1e-6
    assert rel_err(out[0, 1], 0.1) < 1e-6


@pytest.mark.parametrize("k,nt,np_,mode", [(3000, 30, 60, "full"), (4000, 90, 360, "full"),
                                           (2500, 30, 60, "local_only"), (2500, 30, 60, "global_only")])
def test_render_queries_matches_oracle_predict(ctx, capi, orc, k, nt, np_, mode):
    import oracle as O
    sc = capi.synth_scene(k, 2, 1, 7)
    scene, cond, oscene, ocond = _setup_cond(capi, ctx, orc, sc, mode)
    grid = capi.Grid(nt, np_, 8, 1.0)
    st = scene.tx_state(TX, grid)
    rx = capi.synth_points(5, 11, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    spec, rssi = scene.render_queries(cond, st, rx)
    og = O.Grid(nt, np_, 8, 1.0)
    oscene_r = orc.scene(sc, "rssi")
    for j in range(rx.shape[0]):
        want = orc.predict(oscene, ocond, og, TX, rx[j], "spectrum").reshape(nt, np_)
        assert rel_err(spec[j], want).max() < TOL
        wr = orc.predict(oscene_r, ocond, og, TX, rx[j], "rssi")[0]
        assert rel_err(rssi[j], wr) < TOL


@pytest.mark.parametrize("l_max,n_rx", [(4, 5), (9, 3), (9, 130)])
def test_render_queries_high_lmax_fle_gemm(ctx, capi, orc, l_max, n_rx):
    """l_max >= 3 (L >= 16) takes the FLE reduction as a tensor-core GEMM
    (k_fle_gemm.cu); l_max = 9 is the paper's spectrum setting.  130
    receivers span two 128-receiver GEMM column tiles (ragged)."""
    import oracle as O
    sc = capi.synth_scene(2500, l_max, 1, 7)
    scene, cond, oscene, ocond = _setup_cond(capi, ctx, orc, sc)
    grid = capi.Grid(30, 60, 8, 1.0)
    st = scene.tx_state(TX, grid)
    rx = capi.synth_points(n_rx, 11, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    spec, rssi = scene.render_queries(cond, st, rx)
    og = O.Grid(30, 60, 8, 1.0)
    oscene_r = orc.scene(sc, "rssi")
    for j in sorted({0, n_rx // 2, n_rx - 1}):
        want = orc.predict(oscene, ocond, og, TX, rx[j], "spectrum").reshape(30, 60)
        assert rel_err(spec[j], want).max() < TOL
        wr = orc.predict(oscene_r, ocond, og, TX, rx[j], "rssi")[0]
        assert rel_err(rssi[j], wr) < TOL


@pytest.mark.parametrize("l_max,mode", [(0, "full"), (1, "full"), (2, "global_only"), (2, "local_only")])
def test_render_queries_host_chunks_equal_device_batch(ctx, capi, orc, l_max, mode):
    """Host-output render of >= 256 receivers runs in receiver chunks with
    the global branch and (tensor-core path, l_max >= 1) the FLE GEMM
    computed once for the whole batch: spectra and RSSI identical, bit for
    bit, to the one-chunk device-resident render; spot-checked against the
    oracle."""
    import torch
    import oracle as O
    sc = capi.synth_scene(3000, l_max, 1, 7)
    scene, cond, oscene, ocond = _setup_cond(capi, ctx, orc, sc, mode=mode)
    grid, og = capi.Grid(30, 60, 8, 1.0), O.Grid(30, 60, 8, 1.0)
    n_rx = 300
    rx = capi.synth_points(n_rx, 11, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    st = scene.tx_state(TX, grid)
    spec, rssi = scene.render_queries(cond, st, rx)
    dev = torch.device("cuda", 0)
    sd = torch.empty((n_rx, 30, 60), dtype=torch.float32, device=dev)
    rd = torch.empty(n_rx, dtype=torch.float32, device=dev)
    scene.render_queries(cond, st, torch.from_numpy(rx).to(dev), sd, rd)
    torch.cuda.synchronize()
    assert np.array_equal(sd.cpu().numpy(), spec) and np.array_equal(rd.cpu().numpy(), rssi)
    for j in (0, n_rx // 2, n_rx - 1):
        want = orc.predict(oscene, ocond, og, TX, rx[j], "spectrum").reshape(30, 60)
        assert rel_err(spec[j], want).max() <= TOL


def test_render_queries_unconditioned_and_batch_invariance(ctx, capi, orc):
    import oracle as O
    sc = capi.synth_scene(3000, 2, 1, 8)
    scene = ctx.scene(sc)
    grid = capi.Grid(30, 60, 8, 1.0)
    st = scene.tx_state(TX, grid)
    rx = capi.synth_points(40, 11, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    spec, rssi = scene.render_queries(None, st, rx)
    og = O.Grid(30, 60, 8, 1.0)
    want = orc.predict(orc.scene(sc), None, og, TX, rx[0], "spectrum").reshape(30, 60)
    for j in range(40):
        assert rel_err(spec[j], want).max() < TOL
    # batch composition does not change any receiver's result (bitwise)
    s2, r2 = scene.render_queries(None, st, rx[7:9])
    assert np.array_equal(s2, spec[7:9]) and np.array_equal(r2, rssi[7:9])


def test_predict_api(ctx, capi, orc):
    import oracle as O
    sc = capi.synth_scene(1500, 2, 1, 7)
    scene, cond, oscene, ocond = _setup_cond(capi, ctx, orc, sc)
    grid = capi.Grid(18, 36, 8, 1.0)
    og = O.Grid(18, 36, 8, 1.0)
    got = scene.predict(cond, grid, TX, [1.1, 0.7, 0.2])
    want = orc.predict(oscene, ocond, og, TX, [1.1, 0.7, 0.2], "spectrum")
    assert rel_err(got, want).max() < TOL


def test_tcgen05_selftest(ctx):
    """128x64x64 bf16 GEMM with A in TMEM and in smem vs FP32 FMA of the same values."""
    e = ctx.selftest_tcgen05()
    assert e[2] == 0.0 and e[3] == 0.0 and e[4] == 0.0, e  # exact data: layouts and descriptors
    assert e[0] < 1e-2 and e[1] < 1e-2, e  # smooth data: tensor-core accumulation


def test_tcgen05_kernel_matches_simt_and_oracle(ctx, capi, orc):
    """The tcgen05 hot kernel and the FP32 SIMT kernel agree, and both match the oracle."""
    import oracle as O
    sc = capi.synth_scene(6000, 2, 1, 17)
    scene, cond, oscene, ocond = _setup_cond(capi, ctx, orc, sc)
    grid = capi.Grid(45, 90, 8, 1.0)
    st = scene.tx_state(TX, grid)
    rx = capi.synth_points(70, 19, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    s_tc, r_tc = scene.render_queries(cond, st, rx)
    ctx.set_cond_kernel("simt")
    try:
        s_si, r_si = scene.render_queries(cond, st, rx)
    finally:
        ctx.set_cond_kernel("auto")
    assert rel_err(s_tc, s_si).max() < TOL and rel_err(r_tc, r_si).max() < TOL
    og = O.Grid(45, 90, 8, 1.0)
    for j in (0, 33, 69):
        want = orc.predict(oscene, ocond, og, TX, rx[j], "spectrum").reshape(45, 90)
        assert rel_err(s_tc[j], want).max() < TOL


def test_reference_api_shim_cpp(capi, tmp_path):
    """include/rxgs_b200.hpp: reference-shaped C++ callers (tests/cpp/shim_test.cpp)
    compile against the shim, link librxgs_b200.so and pass on the B200."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.dirname(capi.LIB_PATH)
    exe = str(tmp_path / "shim_test")
    subprocess.check_call(["g++", "-std=c++17", "-O1", "-I", os.path.join(root, "include"),
                           os.path.join(root, "tests", "cpp", "shim_test.cpp"), "-L", libdir, "-lrxgs_b200",
                           "-Wl,-rpath," + libdir, "-o", exe])
    out = subprocess.run([exe], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr


def test_tcgen05_composite_matches_simt_and_oracle(ctx, capi, orc):
    """The tensor-core compositor and the SIMT compositor agree; both match the oracle."""
    import oracle as O
    sc = capi.synth_scene(8000, 2, 1, 21)
    scene, cond, oscene, ocond = _setup_cond(capi, ctx, orc, sc)
    grid = capi.Grid(45, 90, 8, 1.0)
    st = scene.tx_state(TX, grid)
    rx = capi.synth_points(100, 29, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])  # two 64-receiver chunks, ragged
    s_tc, r_tc = scene.render_queries(cond, st, rx)
    ctx.set_composite_kernel("simt")
    try:
        s_si, r_si = scene.render_queries(cond, st, rx)
    finally:
        ctx.set_composite_kernel("auto")
    assert rel_err(s_tc, s_si).max() < TOL and rel_err(r_tc, r_si).max() < TOL
    og = O.Grid(45, 90, 8, 1.0)
    for j in (0, 63, 64, 99):
        want = orc.predict(oscene, ocond, og, TX, rx[j], "spectrum").reshape(45, 90)
        assert rel_err(s_tc[j], want).max() < TOL


@pytest.mark.parametrize("mode,hidden,l_max", [("full", 64, 2), ("full", 32, 2), ("additive_only", 64, 2),
                                               ("global_only", 64, 2), (None, 64, 2), ("full", 64, 4)])
def test_coverage_table_matches_oracle_predict(ctx, capi, orc, mode, hidden, l_max):
    """Config-3 path: Tx-independent conditioning cached once, reused per Tx
    (l_max 4: the FLE-GEMM signal path)."""
    import oracle as O
    sc = capi.synth_scene(2500, l_max, 1, 7)
    grid, og = capi.Grid(18, 36, 6, 1.0), O.Grid(18, 36, 6, 1.0)
    if mode is None:
        scene, cond = ctx.scene(sc, "rssi"), None
        oscene, ocond = orc.scene(sc, "rssi"), None
    else:
        scene, cond, _, ocond = _setup_cond(capi, ctx, orc, sc, mode=mode, hidden=hidden)
        oscene = orc.scene(sc, "rssi")
    tx = capi.synth_points(3, 13, "bench.tx", [-4, -3, -1.5], [4, 3, 1.5])
    rx = capi.synth_points(37, 11, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    table = scene.coverage_table(cond, grid, tx, rx)
    for t in range(3):
        for j in range(0, 37, 4):
            want = orc.predict(oscene, ocond, og, tx[t], rx[j], "rssi")[0]
            assert rel_err(table[t, j], want) < TOL, (t, j)
    # the per-Tx fused query path gives the same table
    st = scene.tx_state(tx[1], grid)
    _, r = scene.render_queries(cond, st, rx, want=("rssi",))
    assert rel_err(table[1], r).max() < 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("n_tx", [1, 2, 7])
def test_coverage_table_builder_count_invariant(ctx, capi, orc, n_tx, monkeypatch):
    """The transmitter states of a coverage table are built by builder threads
    on helper contexts while the calling thread renders; the table is bitwise
    the same for a serial build (0), one builder and more builders than
    transmitters, and matches the oracle."""
    import oracle as O
    sc = capi.synth_scene(3000, 2, 1, 5)
    scene, cond, _, ocond = _setup_cond(capi, ctx, orc, sc)
    oscene = orc.scene(sc, "rssi")
    grid, og = capi.Grid(18, 36, 6, 1.0), O.Grid(18, 36, 6, 1.0)
    tx = capi.synth_points(n_tx, 17, "bench.tx", [-4, -3, -1.5], [4, 3, 1.5])
    rx = capi.synth_points(45, 19, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    tables = {}
    for d in (0, 1, 2, 3, 8):
        monkeypatch.setenv("RXGS_COV_BUILDERS", str(d))
        tables[d] = scene.coverage_table(cond, grid, tx, rx)
    for d, tb in tables.items():
        assert np.array_equal(tb, tables[0]), d
    for t in range(n_tx):
        j = (7 * t) % 45
        want = orc.predict(oscene, ocond, og, tx[t], rx[j], "rssi")[0]
        assert rel_err(tables[8][t, j], want) < TOL, (t, j)
