"""Scene / model load: the RXGS checkpoint container (io::save_checkpoint /
io::load_checkpoint, checkpoint.cpp:93-231).  The reference's checkpoint.cpp
is built into oracle/_ref against the nlohmann json.hpp this image ships
(oracle/Makefile); the Python restatement oracle/rxgs_checkpoint.py is pinned
to it byte for byte, and rxgs_checkpoint_save must write exactly the
reference's bytes (and each side loads the other's files).  A loaded model
must render exactly like the model it was saved from."""
import json
import struct

import numpy as np
import pytest

import rxgs_checkpoint as CK

TX = np.array([0.3, -0.2, 0.1])
GRID = dict(n_theta=18, n_phi=36, tile_size=8, radius=1.0, theta_min=0.0, theta_max=3.141592653589793)


def _tiny_scene(capi, k=50, l_max=2, seed=7):
    return capi.synth_scene(k, l_max, 1, seed)


def test_oracle_container_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    k, l_max = 5, 1
    sc = {"l_max": l_max, "channels": 1, "positions": rng.normal(size=(k, 3)), "log_scales": rng.normal(size=(k, 3)),
          "quaternions": rng.normal(size=(k, 4)), "tau_logits": rng.normal(size=k),
          "fle_coeffs": rng.normal(size=(k, 4, 1, 2))}
    p = tmp_path / "m.rxgs"
    CK.write_checkpoint(p, sc, GRID)
    raw = p.read_bytes()
    assert raw[:4] == b"RXGS" and struct.unpack_from("<I", raw, 4)[0] == 1
    hlen = struct.unpack_from("<Q", raw, 8)[0]
    text = raw[16:16 + hlen].decode()
    # insertion order of save_checkpoint (checkpoint.cpp:96-128)
    assert text.startswith('{"k":5,"l_max":1,"channels":1,"modality":"spectrum","grid":{"n_theta":18,"n_phi":36,'
                           '"tile_size":8,"radius":1.0,"theta_min":0.0,"theta_max":3.141592653589793},'
                           '"has_conditioning":false,"arrays":[{"name":"positions","dtype":"f64","shape":[5,3],'
                           '"offset":0}')
    header, arrays = CK.read_checkpoint(p)
    assert [e["name"] for e in header["arrays"]] == ["positions", "log_scales", "quaternions", "tau_logits",
                                                     "fle_coeffs"]
    for name in ("positions", "log_scales", "quaternions", "tau_logits", "fle_coeffs"):
        assert np.array_equal(arrays[name].reshape(-1), np.asarray(sc[name]).reshape(-1))
    assert len(raw) == 16 + hlen + 8 * k * (3 + 3 + 4 + 1 + 8)


def _model(capi, ctx, mode="full", k=300):
    sc = _tiny_scene(capi, k)
    scene = ctx.scene(sc, "spectrum")
    lo, hi = scene.bounds(0.0)
    cfg = capi.cond_cfg(mode=mode)
    params = capi.synth_cond(cfg, 2, 1, lo, hi, 3, True)
    cond = ctx.cond(cfg, params)
    olo, ohi = scene.bounds(0.1)
    occ = cond.build_occupancy(scene, 32, olo, ohi)
    return sc, scene, cfg, params, cond, occ, olo, ohi


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["full", "no_occlusion"])
def test_save_is_byte_identical_to_reference_format(ctx, capi, tmp_path, mode):
    sc, scene, cfg, params, cond, occ, olo, ohi = _model(capi, ctx, mode)
    grid = capi.Grid(**GRID)
    ours = tmp_path / "ours.rxgs"
    scene.save_checkpoint(ours, grid, cond)
    want = tmp_path / "want.rxgs"
    CK.write_checkpoint(want, sc, GRID, {"cfg": cfg, "params": params, "occupancy": occ, "lo": olo, "hi": ohi})
    assert ours.read_bytes() == want.read_bytes()
    # unconditioned model
    ours0, want0 = tmp_path / "o0.rxgs", tmp_path / "w0.rxgs"
    scene.save_checkpoint(ours0, grid)
    CK.write_checkpoint(want0, sc, GRID)
    assert ours0.read_bytes() == want0.read_bytes()


@pytest.mark.gpu
def test_load_renders_identically(ctx, capi, tmp_path):
    sc, scene, cfg, params, cond, occ, olo, ohi = _model(capi, ctx)
    path = tmp_path / "m.rxgs"
    CK.write_checkpoint(path, sc, GRID, {"cfg": cfg, "params": params, "occupancy": occ, "lo": olo, "hi": ohi})
    scene2, grid2, cond2 = ctx.load_checkpoint(path)
    assert (grid2.n_theta, grid2.n_phi, grid2.tile_size, grid2.radius, grid2.theta_max) == (18, 36, 8, 1.0,
                                                                                            GRID["theta_max"])
    assert scene2.k == scene.k and scene2.modality == "spectrum" and np.array_equal(cond2.cfg, cfg)
    rx = capi.synth_points(8, 11, "bench.rx", [-4, -3, -1.5], [4, 3, 1.5])
    grid = capi.Grid(**GRID)
    a = scene.render_queries(cond, scene.tx_state(TX, grid), rx)
    b = scene2.render_queries(cond2, scene2.tx_state(TX, grid2), rx)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    # and the loaded model saves back to the same bytes
    again = tmp_path / "again.rxgs"
    scene2.save_checkpoint(again, grid2, cond2)
    assert again.read_bytes() == path.read_bytes()


@pytest.mark.gpu
def test_load_partial_conditioning_uses_init(ctx, capi, tmp_path):
    """Arrays absent from the file keep init_conditioning(cfg, seed 0) values
    (checkpoint.cpp:191-193 then only the listed arrays are read)."""
    sc, scene, cfg, params, cond, occ, olo, ohi = _model(capi, ctx)
    path = tmp_path / "m.rxgs"
    CK.write_checkpoint(path, sc, GRID, {"cfg": cfg, "params": params, "occupancy": occ, "lo": olo, "hi": ohi})
    header, arrays = CK.read_checkpoint(path)
    keep = [e for e in header["arrays"] if e["name"] != "cond.local.w2"]
    # rewrite without cond.local.w2 (offsets recomputed)
    off, blobs = 0, []
    for e in keep:
        e["offset"] = off
        a = arrays[e["name"]].reshape(-1)
        blobs.append(a.astype("<f8").tobytes())
        off += a.size * 8
    header["arrays"] = keep
    text = json.dumps(header, separators=(",", ":")).encode()
    p2 = tmp_path / "partial.rxgs"
    p2.write_bytes(b"RXGS" + struct.pack("<IQ", 1, len(text)) + text + b"".join(blobs))
    _, _, cond2 = ctx.load_checkpoint(p2)
    got = capi.cond_params(cond2)
    init = capi.synth_cond(cfg, 2, 1, olo, ohi, 0, False)
    d = int(cfg[1])
    o = 3 * int(cfg[0]) + d * (6 * int(cfg[0]) + 2 + int(cfg[2])) + d + d * d + d + 4 * d + 4 + 9 * int(cfg[2])
    o_lw2 = o + d * 6 + d
    assert np.array_equal(got[o_lw2:o_lw2 + d * d], init[o_lw2:o_lw2 + d * d])
    mask = np.ones(got.size, bool)
    mask[o_lw2:o_lw2 + d * d] = False
    assert np.array_equal(got[mask], params[mask])


@pytest.mark.gpu
def test_load_errors_match_reference(ctx, capi, tmp_path):
    sc = _tiny_scene(capi, 20)
    good = tmp_path / "g.rxgs"
    CK.write_checkpoint(good, sc, GRID)
    raw = good.read_bytes()
    bad = tmp_path / "bad.rxgs"
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(capi.IoError, match=f"load_checkpoint: bad magic in {bad}"):
        ctx.load_checkpoint(bad)
    bad.write_bytes(raw[:4] + struct.pack("<I", 2) + raw[8:])
    with pytest.raises(capi.IoError, match="load_checkpoint: unsupported version 2"):
        ctx.load_checkpoint(bad)
    bad.write_bytes(raw[:-8])
    with pytest.raises(capi.IoError, match="load_checkpoint: truncated array 'fle_coeffs'"):
        ctx.load_checkpoint(bad)
    with pytest.raises(capi.IoError, match="load_checkpoint: cannot open"):
        ctx.load_checkpoint(tmp_path / "missing.rxgs")
    hlen = struct.unpack_from("<Q", raw, 8)[0]
    text = raw[16:16 + hlen].replace(b'"name":"tau_logits"', b'"name":"tau_logitz"')
    bad.write_bytes(raw[:16] + text + raw[16 + hlen:])
    with pytest.raises(capi.IoError, match="load_checkpoint: unknown array 'tau_logitz'"):
        ctx.load_checkpoint(bad)


# ---------------------------------------------------------------- pinned to the reference's checkpoint.cpp
def _ref_model(ref, k=40, seed=7, mode="full", radius=1.0, pad=0.1, bounds=None):
    import oracle as O
    sc = ref.synth_scene(k, 2, 1, seed)
    h = ref.scene(sc, "spectrum")
    lo, hi = ref.scene_bounds(h, 0.0)
    cfg = O.cond_cfg(mode=mode, R=8)
    params = ref.synth_cond(cfg, 2, 1, lo, hi, 3, True)
    olo, ohi = ref.scene_bounds(h, pad) if bounds is None else bounds
    occ = ref.build_occupancy(h, 8, olo, ohi)
    c = ref.cond(cfg, params, occ, olo, ohi)
    cond = {"cfg": cfg, "params": params, "occupancy": occ, "lo": olo, "hi": ohi}
    return sc, h, c, cond


GRIDS = [GRID,
         dict(n_theta=90, n_phi=360, tile_size=8, radius=10.0, theta_min=0.0, theta_max=3.141592653589793),
         dict(n_theta=7, n_phi=13, tile_size=4, radius=0.123456789, theta_min=0.25, theta_max=2.0000001),
         dict(n_theta=4, n_phi=4, tile_size=2, radius=12345.5, theta_min=1e-05, theta_max=0.0001)]


@pytest.mark.parametrize("gi", range(len(GRIDS)))
def test_restatement_bytes_equal_reference_save(ref, tmp_path, gi):
    """The format oracle writes exactly the bytes of io::save_checkpoint
    (checkpoint.cpp:93-155, nlohmann ordered_json dump): radius 10, integer
    and tiny doubles in the grid, occupancy bounds of +-10."""
    import oracle as O
    if not hasattr(ref, "_checkpoint_save"):
        pytest.skip("reference built without checkpoint.cpp (no json.hpp)")
    g = GRIDS[gi]
    og = O.Grid(g["n_theta"], g["n_phi"], g["tile_size"], g["radius"], g["theta_min"], g["theta_max"])
    bounds = ([-10.0, -10.0, -10.0], [10.0, 10.0, 10.0]) if gi == 1 else None
    sc, h, c, cond = _ref_model(ref, bounds=bounds)
    for with_cond in (False, True):
        a, b = tmp_path / f"ref{with_cond}.rxgs", tmp_path / f"ck{with_cond}.rxgs"
        ref.checkpoint_save(a, h, c if with_cond else None, og)
        CK.write_checkpoint(b, sc, g, cond if with_cond else None)
        assert a.read_bytes() == b.read_bytes()


def test_reference_load_reads_restatement_and_errors(ref, tmp_path):
    import oracle as O
    if not hasattr(ref, "_checkpoint_save"):
        pytest.skip("reference built without checkpoint.cpp (no json.hpp)")
    sc, h, c, cond = _ref_model(ref, mode="no_occlusion")
    p = tmp_path / "m.rxgs"
    CK.write_checkpoint(p, sc, GRIDS[2], cond)
    got = ref.checkpoint_load(p)
    g = GRIDS[2]
    assert got["grid"] == (g["n_theta"], g["n_phi"], g["tile_size"], g["radius"], g["theta_min"], g["theta_max"])
    for name in ("positions", "log_scales", "quaternions", "tau_logits", "fle_coeffs"):
        assert np.array_equal(got["scene"][name].reshape(-1), np.asarray(sc[name]).reshape(-1))
    assert np.array_equal(got["cond"]["params"], cond["params"])
    assert np.array_equal(got["cond"]["occupancy"], np.asarray(cond["occupancy"]).reshape(-1))
    assert np.array_equal(got["cond"]["cfg"], cond["cfg"])
    bad = tmp_path / "bad.rxgs"
    bad.write_bytes(b"XXXX" + p.read_bytes()[4:])
    with pytest.raises(O.CheckerError, match="bad magic"):
        ref.checkpoint_load(bad)


@pytest.mark.gpu
@pytest.mark.parametrize("gi", range(len(GRIDS)))
def test_save_is_byte_identical_to_reference_save(ctx, capi, ref, tmp_path, gi):
    """rxgs_checkpoint_save == io::save_checkpoint byte for byte (ADVICE r1:
    radius 10, occupancy bounds +-10), and each side loads the other's file."""
    import oracle as O
    if not hasattr(ref, "_checkpoint_save"):
        pytest.skip("reference built without checkpoint.cpp (no json.hpp)")
    g = GRIDS[gi]
    og = O.Grid(g["n_theta"], g["n_phi"], g["tile_size"], g["radius"], g["theta_min"], g["theta_max"])
    bounds = ([-10.0, -10.0, -10.0], [10.0, 10.0, 10.0]) if gi == 1 else None
    sc, h, c, cond = _ref_model(ref, bounds=bounds)
    scene = ctx.scene(sc, "spectrum")
    gcond = ctx.cond(cond["cfg"], cond["params"], cond["occupancy"], cond["lo"], cond["hi"])
    grid = capi.Grid(**g)
    ours, want = tmp_path / "ours.rxgs", tmp_path / "want.rxgs"
    scene.save_checkpoint(ours, grid, gcond)
    ref.checkpoint_save(want, h, c, og)
    assert ours.read_bytes() == want.read_bytes()
    # the reference loads ours; we load the reference's and save the same bytes back
    back = ref.checkpoint_load(ours)
    assert np.array_equal(back["cond"]["params"], cond["params"])
    scene2, grid2, cond2 = ctx.load_checkpoint(want)
    again = tmp_path / "again.rxgs"
    scene2.save_checkpoint(again, grid2, cond2)
    assert again.read_bytes() == want.read_bytes()
