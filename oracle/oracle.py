"""oracle/oracle.py -- TEST INFRASTRUCTURE ONLY (the checker, never the product).

ctypes front-end over the two CPU checkers:

* ``liboracle.so``      -- the plain-C restatement (oracle/rxgs_oracle.c);
* ``_ref/librxgs_ref.so`` -- the UNMODIFIED reference sources compiled by
  oracle/Makefile (present wherever it was built; /root/reference itself is
  never read at run time).

Both expose the same entry points (prefix ``or_`` / ``ref_``), so every check
can run against either.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "librxgs_ref.so")

MODALITY = {"rssi": 0, "csi": 1, "spectrum": 2}
MODE = {"full": 0, "global_only": 1, "local_only": 2, "additive_only": 3, "no_occlusion": 4}

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_lp = C.POINTER(C.c_long)
_fp = C.POINTER(C.c_float)
_u64p = C.POINTER(C.c_uint64)


def _d(a):
    if a is None:
        return None
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a.ctypes.data_as(_dp)


def _i(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a.ctypes.data_as(_ip)


def ensure_built() -> None:
    """Compile the C restatement if the prebuilt .so is missing (gcc only)."""
    if not os.path.exists(ORACLE_SO):
        subprocess.check_call(["make", "-s", "-C", HERE, "oracle"])


class Grid:
    """SphericalGrid (sphraster.hpp:15-32)."""

    def __init__(self, n_theta, n_phi, tile_size=8, radius=1.0, theta_min=0.0,
                 theta_max=3.14159265358979323846):
        self.n_theta, self.n_phi, self.tile_size = int(n_theta), int(n_phi), int(tile_size)
        self.radius, self.theta_min, self.theta_max = float(radius), float(theta_min), float(theta_max)
        self._gi = np.array([self.n_theta, self.n_phi, self.tile_size], dtype=np.int32)
        self._gd = np.array([self.radius, self.theta_min, self.theta_max], dtype=np.float64)

    @property
    def gi(self):
        return self._gi.ctypes.data_as(_ip)

    @property
    def gd(self):
        return self._gd.ctypes.data_as(_dp)

    @property
    def tiles_theta(self):
        return (self.n_theta + self.tile_size - 1) // self.tile_size

    @property
    def tiles_phi(self):
        return (self.n_phi + self.tile_size - 1) // self.tile_size

    @property
    def n_tiles(self):
        return self.tiles_theta * self.tiles_phi

    @property
    def cells(self):
        return self.n_theta * self.n_phi


class CheckerError(ValueError):
    pass


class Checker:
    """One CPU checker library (restatement or reference build)."""

    def __init__(self, path: str, prefix: str):
        self.path = path
        self.prefix = prefix
        self.lib = C.CDLL(path)
        L = self.lib
        p = prefix
        sig = {
            "abi_version": (C.c_int, []),
            "synth_scene": (None, [C.c_int, C.c_int, C.c_int, C.c_uint64, _dp, _dp, _dp, _dp, _dp]),
            "synth_points": (None, [C.c_int, C.c_uint64, C.c_char_p, _dp, _dp, C.c_double, _dp]),
            "synth_cond": (C.c_long, [_ip, C.c_int, C.c_int, _dp, _dp, C.c_uint64, C.c_int, _dp]),
            "scene_new": (C.c_void_p, [C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp]),
            "scene_free": (None, [C.c_void_p]),
            "scene_bounds": (None, [C.c_void_p, C.c_double, _dp, _dp]),
            "covariance": (None, [C.c_void_p, _dp]),
            "tx_new": (C.c_void_p, [C.c_void_p, _dp, _ip, _dp, C.c_char_p, C.c_int]),
            "tx_free": (None, [C.c_void_p]),
            "tx_entries": (C.c_long, [C.c_void_p]),
            "tx_get": (None, [C.c_void_p, _ip, _dp, _ip, _dp, _lp, _ip, _u64p]),
            "bin_and_sort": (C.c_long, [C.c_int, _ip, _dp, _ip, _ip, _dp, _lp, _ip, C.c_long]),
            "render": (C.c_int, [C.c_void_p, C.c_void_p, _dp, C.c_long, C.c_int, C.c_int, _dp, _dp,
                                 C.c_char_p, C.c_int]),
            "aggregate": (C.c_int, [C.c_int, C.c_int, _ip, _dp, _dp, C.c_int, _dp, C.c_char_p, C.c_int]),
            "cond_new": (C.c_void_p, [_ip, _dp, _dp, _dp, _dp]),
            "cond_free": (None, [C.c_void_p]),
            "cond_param_count": (C.c_long, [C.c_void_p]),
            "build_occupancy": (None, [C.c_void_p, C.c_int, _dp, _dp, _dp]),
            "probe": (None, [C.c_int, _dp, _dp, _dp, _dp, _dp, C.c_int, C.c_int, _dp]),
            "cond_forward": (C.c_int, [C.c_void_p, C.c_void_p, _dp, _dp, _dp, _dp, _dp, C.c_char_p, C.c_int]),
            "eval_basis": (None, [C.c_double, C.c_double, C.c_int, _dp]),
            "predict": (C.c_int, [C.c_void_p, C.c_void_p, _ip, _dp, _dp, _dp, C.c_int, _dp, C.c_char_p, C.c_int]),
        }
        if prefix == "ref_":
            sig.update({
                "bench_queries": (C.c_double, [C.c_void_p, C.c_void_p, _ip, _dp, _dp, _dp, C.c_int, C.c_int,
                                               _fp, _dp]),
                "bench_coverage": (C.c_double, [C.c_void_p, C.c_void_p, _ip, _dp, _dp, C.c_int, _dp, C.c_int,
                                                C.c_int, _dp, _dp]),
                "aggregate_backward": (C.c_int, [C.c_int, C.c_int, _ip, _dp, _dp, C.c_int, _dp, _dp]),
                "backward_render": (C.c_int, [C.c_void_p, C.c_void_p, _dp, C.c_long, C.c_int, _dp, C.c_long,
                                              C.c_int, _dp, _dp, _dp, _dp, _dp, C.c_char_p, C.c_int]),
                "cond_backward": (C.c_int, [C.c_void_p, C.c_void_p, _dp, _dp, _dp, _dp]),
                "cond_calls": (None, [C.c_void_p, _lp, _lp]),
                "coverage_fraction": (C.c_int, [_dp, C.c_long, C.c_long, _ip, C.c_int, C.c_double, _dp,
                                                C.c_char_p, C.c_int]),
                "greedy_plan": (C.c_int, [_dp, C.c_long, C.c_long, C.c_int, C.c_double, _ip, C.c_char_p, C.c_int]),
                "scene_count": (C.c_int, [C.c_void_p]),
                "scene_get": (None, [C.c_void_p, _dp, _dp, _dp, _dp, _dp]),
                "densify": (C.c_int, [C.c_void_p, _dp, C.c_int, C.c_double, _dp, C.c_ulong, C.c_ulong, _ip, _ip,
                                      C.c_char_p, C.c_int]),
                "reset_transmittance": (None, [C.c_void_p]),
                "image_metrics": (C.c_int, [_dp, _dp, C.c_int, C.c_int, C.c_double, C.c_int, C.c_double,
                                            C.c_double, _dp, C.c_char_p, C.c_int]),
                "snr_csi": (C.c_int, [_dp, _dp, C.c_long, _dp, C.c_char_p, C.c_int]),
                "per_receiver_aggregate": (C.c_int, [_ip, _dp, C.c_long, _ip, _dp, _lp, _ip, _dp, _dp, C.c_char_p,
                                                     C.c_int]),
                "train_sample": (C.c_int, [C.c_void_p, C.c_void_p, _ip, _dp, _dp, _dp, _dp, C.c_double,
                                           C.c_double, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                           C.c_char_p, C.c_int]),
            })
        if prefix == "ref_" and hasattr(L, "ref_has_checkpoint") and L.ref_has_checkpoint():
            sig.update({
                "checkpoint_save": (C.c_int, [C.c_char_p, C.c_void_p, C.c_void_p, _ip, _dp, C.c_char_p, C.c_int]),
                "checkpoint_load": (C.c_void_p, [C.c_char_p, C.POINTER(C.c_void_p), _ip, _dp, C.c_char_p, C.c_int]),
                "scene_modality": (C.c_int, [C.c_void_p]),
                "scene_shape": (None, [C.c_void_p, _ip]),
                "cond_export": (None, [C.c_void_p, _ip, _dp, _dp, _dp, _dp]),
            })
        for name, (res, args) in sig.items():
            fn = getattr(L, p + name)
            fn.restype = res
            fn.argtypes = args
            setattr(self, "_" + name, fn)

    # ------------------------------------------------------------ generators
    def synth_scene(self, k, l_max=2, channels=1, seed=7):
        L = (l_max + 1) ** 2
        pos = np.empty((k, 3)); ls = np.empty((k, 3)); q = np.empty((k, 4)); tau = np.empty(k)
        co = np.empty((k, L, channels, 2))
        self._synth_scene(k, l_max, channels, seed, _d(pos), _d(ls), _d(q), _d(tau), _d(co))
        return dict(positions=pos, log_scales=ls, quaternions=q, tau_logits=tau, fle_coeffs=co,
                    l_max=l_max, channels=channels)

    def synth_points(self, n, seed, tag, lo, hi, margin=0.05):
        out = np.empty((n, 3))
        lo = np.asarray(lo, np.float64); hi = np.asarray(hi, np.float64)
        self._synth_points(n, seed, tag.encode(), _d(lo), _d(hi), margin, _d(out))
        return out

    def synth_cond(self, cfg, l_max, channels, lo, hi, seed=3, randomize=True):
        cfg = np.asarray(cfg, np.int32)
        lo = np.asarray(lo, np.float64); hi = np.asarray(hi, np.float64)
        n = self._synth_cond(_i(cfg), l_max, channels, _d(lo), _d(hi), seed, int(randomize), None) \
            if self.prefix == "or_" else None
        if n is None:
            n = self._synth_cond(_i(cfg), l_max, channels, _d(lo), _d(hi), seed, int(randomize), None)
        out = np.empty(n)
        self._synth_cond(_i(cfg), l_max, channels, _d(lo), _d(hi), seed, int(randomize), _d(out))
        return out

    # ------------------------------------------------------------ scene
    def scene(self, sc, modality="spectrum"):
        return _Handle(self, self._scene_new(
            len(sc["tau_logits"]), sc["l_max"], sc["channels"], MODALITY[modality],
            _d(sc["positions"]), _d(sc["log_scales"]), _d(sc["quaternions"]), _d(sc["tau_logits"]),
            _d(sc["fle_coeffs"])), self._scene_free, sc)

    def scene_bounds(self, h, inflate=0.0):
        lo = np.empty(3); hi = np.empty(3)
        self._scene_bounds(h.ptr, inflate, _d(lo), _d(hi))
        return lo, hi

    def covariance(self, h):
        out = np.empty((len(h.data["tau_logits"]), 3, 3))
        self._covariance(h.ptr, _d(out))
        return out

    def tx_state(self, scene_h, tx, grid: Grid):
        err = C.create_string_buffer(512)
        tx = np.asarray(tx, np.float64)
        ptr = self._tx_new(scene_h.ptr, _d(tx), grid.gi, grid.gd, err, 512)
        if not ptr:
            raise CheckerError(err.value.decode())
        h = _Handle(self, ptr, self._tx_free, None)
        k = len(scene_h.data["tau_logits"])
        L = (scene_h.data["l_max"] + 1) ** 2
        n = self._tx_entries(ptr)
        culled = np.empty(k, np.int32); geom = np.empty((k, 12)); spans = np.empty((k, 4), np.int32)
        basis = np.empty((k, L, 2)); offs = np.empty(grid.n_tiles + 1, np.int64)
        idx = np.empty(max(n, 1), np.int32); hsh = np.zeros(1, np.uint64)
        self._tx_get(ptr, _i_out(culled), geom.ctypes.data_as(_dp), _i_out(spans), basis.ctypes.data_as(_dp),
                     offs.ctypes.data_as(_lp), _i_out(idx), hsh.ctypes.data_as(_u64p))
        h.data = dict(culled=culled, geom=geom, spans=spans, basis=basis, offsets=offs, indices=idx[:n],
                      hash=int(hsh[0]), grid=grid)
        return h

    def bin_and_sort(self, culled, depth, spans, grid: Grid):
        k = len(culled)
        offs = np.empty(grid.n_tiles + 1, np.int64)
        cul = np.ascontiguousarray(culled, np.int32); dep = np.ascontiguousarray(depth, np.float64)
        sp = np.ascontiguousarray(spans, np.int32)
        n = self._bin_and_sort(k, _i(cul), _d(dep), _i(sp), grid.gi, grid.gd, offs.ctypes.data_as(_lp), None, 0)
        idx = np.empty(max(n, 1), np.int32)
        self._bin_and_sort(k, _i(cul), _d(dep), _i(sp), grid.gi, grid.gd, offs.ctypes.data_as(_lp),
                           _i_out(idx), n)
        return offs, idx[:n]

    def render(self, tx_h, scene_h, coeffs, n_rx):
        grid = tx_h.data["grid"]
        C_ = scene_h.data["channels"]
        co = np.ascontiguousarray(coeffs, np.float64)
        vals = np.empty((n_rx, C_, 2, grid.n_theta, grid.n_phi))
        T = np.empty((n_rx, grid.n_theta, grid.n_phi))
        err = C.create_string_buffer(512)
        rc = self._render(tx_h.ptr, scene_h.ptr, _d(co), co.size, n_rx, 1, vals.ctypes.data_as(_dp),
                          T.ctypes.data_as(_dp), err, 512)
        if rc:
            raise CheckerError(err.value.decode())
        return vals, T

    def aggregate(self, values, grid: Grid, modality):
        values = np.ascontiguousarray(values, np.float64)
        n_rx, C_ = values.shape[0], values.shape[1]
        m = MODALITY[modality]
        out = np.empty((n_rx,) if m == 0 else ((n_rx, C_, 2) if m == 1 else (n_rx, grid.n_theta, grid.n_phi)))
        err = C.create_string_buffer(512)
        rc = self._aggregate(n_rx, C_, grid.gi, grid.gd, _d(values), m, out.ctypes.data_as(_dp), err, 512)
        if rc:
            raise CheckerError(err.value.decode())
        return out

    # ------------------------------------------------------------ conditioning
    def cond(self, cfg, params, occ=None, occ_lo=None, occ_hi=None):
        cfg = np.asarray(cfg, np.int32)
        keep = dict(cfg=cfg, params=np.ascontiguousarray(params, np.float64),
                    occ=None if occ is None else np.ascontiguousarray(occ, np.float64),
                    lo=None if occ_lo is None else np.asarray(occ_lo, np.float64),
                    hi=None if occ_hi is None else np.asarray(occ_hi, np.float64))
        ptr = self._cond_new(_i(cfg), _d(keep["params"]), _d(keep["occ"]), _d(keep["lo"]), _d(keep["hi"]))
        return _Handle(self, ptr, self._cond_free, keep)

    def build_occupancy(self, scene_h, R, lo, hi):
        out = np.empty((R, R, R))
        self._build_occupancy(scene_h.ptr, R, _d(np.asarray(lo, np.float64)), _d(np.asarray(hi, np.float64)),
                              out.ctypes.data_as(_dp))
        return out

    def probe(self, R, lo, hi, dens, frm, to, samples, nearest=False):
        out = np.empty(2)
        self._probe(R, _d(lo), _d(hi), _d(dens), _d(frm), _d(to), samples, int(nearest), out.ctypes.data_as(_dp))
        return out

    def cond_forward(self, cond_h, scene_h, rx, workspace=False):
        sc = scene_h.data
        k = len(sc["tau_logits"]); L = (sc["l_max"] + 1) ** 2; C_ = sc["channels"]
        out = np.empty((k, L, C_, 2))
        lin = np.empty((k, 6)) if workspace else None
        lout = np.empty((k, 4 * C_)) if workspace else None
        gout = np.empty((L, 4 * C_)) if workspace else None
        err = C.create_string_buffer(512)
        rc = self._cond_forward(cond_h.ptr, scene_h.ptr, _d(np.asarray(rx, np.float64)), out.ctypes.data_as(_dp),
                                None if lin is None else lin.ctypes.data_as(_dp),
                                None if lout is None else lout.ctypes.data_as(_dp),
                                None if gout is None else gout.ctypes.data_as(_dp), err, 512)
        if rc:
            raise CheckerError(err.value.decode())
        if workspace:
            return out, dict(local_in=lin, local_out=lout, global_out=gout)
        return out

    def eval_basis(self, theta, phi, l_max):
        out = np.empty(((l_max + 1) ** 2, 2))
        self._eval_basis(theta, phi, l_max, out.ctypes.data_as(_dp))
        return out

    def predict(self, scene_h, cond_h, grid: Grid, tx, rx, modality="spectrum"):
        n = grid.cells if modality == "spectrum" else (1 if modality == "rssi" else 2 * scene_h.data["channels"])
        out = np.empty(n)
        err = C.create_string_buffer(512)
        rc = self._predict(scene_h.ptr, None if cond_h is None else cond_h.ptr, grid.gi, grid.gd,
                           _d(np.asarray(tx, np.float64)), _d(np.asarray(rx, np.float64)), 1,
                           out.ctypes.data_as(_dp), err, 512)
        if rc:
            raise CheckerError(err.value.decode())
        return out

    def aggregate_backward(self, values, grid: Grid, modality, upstream):
        """raster::aggregate_modality_backward (sphraster.cpp:383-449); reference only."""
        values = np.ascontiguousarray(values, np.float64)
        n_rx, C_ = values.shape[0], values.shape[1]
        out = np.empty_like(values)
        self._aggregate_backward(n_rx, C_, grid.gi, grid.gd, _d(values), MODALITY[modality],
                                 _d(np.ascontiguousarray(upstream, np.float64)), out.ctypes.data_as(_dp))
        return out

    def cond_backward(self, cond_h, scene_h, rx, d_out):
        """cond::condition_backward (conditioning.cpp:472-587) after a forward
        at rx; reference only.  Returns (d_base, packed d_params)."""
        d_out = np.ascontiguousarray(d_out, np.float64)
        d_base = np.empty_like(d_out)
        d_params = np.empty(len(cond_h.data["params"]))
        self._cond_backward(cond_h.ptr, scene_h.ptr, _d(np.asarray(rx, np.float64)), _d(d_out),
                            d_base.ctypes.data_as(_dp), d_params.ctypes.data_as(_dp))
        return d_base, d_params

    def backward_render(self, tx_h, scene_h, coeffs, n_rx, d_values, threads=1):
        """raster::backward_render (sphraster.cpp:509-733); reference only.
        Returns the GradientBundle as a dict."""
        sc = scene_h.data
        k = len(sc["tau_logits"])
        co = np.ascontiguousarray(coeffs, np.float64)
        dv = np.ascontiguousarray(d_values, np.float64)
        out = dict(d_positions=np.empty((k, 3)), d_log_scales=np.empty((k, 3)), d_quaternions=np.empty((k, 4)),
                   d_tau_logits=np.empty(k), d_coeffs=np.empty(co.shape))
        err = C.create_string_buffer(512)
        rc = self._backward_render(tx_h.ptr, scene_h.ptr, _d(co), co.size, n_rx, _d(dv), dv.size, threads,
                                   *(out[n].ctypes.data_as(_dp) for n in ("d_positions", "d_log_scales",
                                                                          "d_quaternions", "d_tau_logits",
                                                                          "d_coeffs")), err, 512)
        if rc:
            raise CheckerError(err.value.decode())
        return out

    # ------------------------------------------------------------ reference-only extras
    def bench_queries(self, scene_h, cond_h, grid: Grid, tx, rx, threads, want_outputs=False):
        rx = np.ascontiguousarray(rx, np.float64)
        n = rx.shape[0]
        spec = np.empty((n, grid.cells), np.float32) if want_outputs else None
        rssi = np.empty(n) if want_outputs else None
        secs = self._bench_queries(scene_h.ptr, None if cond_h is None else cond_h.ptr, grid.gi, grid.gd,
                                   _d(np.asarray(tx, np.float64)), _d(rx), n, threads,
                                   None if spec is None else spec.ctypes.data_as(_fp),
                                   None if rssi is None else rssi.ctypes.data_as(_dp))
        return secs, spec, rssi


    def bench_coverage(self, scene_h, cond_h, grid: Grid, tx, rx, threads):
        """Reference CPU coverage table (config 3 rules): returns (secs, table, phases)."""
        tx = np.ascontiguousarray(tx, np.float64).reshape(-1, 3)
        rx = np.ascontiguousarray(rx, np.float64).reshape(-1, 3)
        out = np.empty((tx.shape[0], rx.shape[0]))
        ph = np.zeros(3)
        secs = self._bench_coverage(scene_h.ptr, None if cond_h is None else cond_h.ptr, grid.gi, grid.gd, _d(tx),
                                    tx.shape[0], _d(rx), rx.shape[0], threads, out.ctypes.data_as(_dp),
                                    ph.ctypes.data_as(_dp))
        return secs, out, ph

def _i_out(a):
    return a.ctypes.data_as(_ip)


class _Handle:
    def __init__(self, owner, ptr, free, data):
        self.owner, self.ptr, self._free, self.data = owner, ptr, free, data

    def __del__(self):
        try:
            if self.ptr:
                self._free(self.ptr)
                self.ptr = None
        except Exception:
            pass


_cache: dict = {}


def restatement() -> Checker:
    ensure_built()
    if "or" not in _cache:
        _cache["or"] = Checker(ORACLE_SO, "or_")
    return _cache["or"]


def reference() -> Checker | None:
    """The reference build, or None where it was never built (e.g. no /root/reference)."""
    if not os.path.exists(REF_SO):
        return None
    if "ref" not in _cache:
        _cache["ref"] = Checker(REF_SO, "ref_")
    return _cache["ref"]


def cond_cfg(F=6, hidden=64, dc=16, S=16, R=32, nearest=0, mode="full", l_max=2, C_=1):
    return np.array([F, hidden, dc, S, R, nearest, MODE[mode] if isinstance(mode, str) else mode,
                     l_max, C_], np.int32)


def _train_sample(self, scene_h, cond_h, grid: Grid, tx, rx, target, lambda_ssim=0.0, lambda_fft=0.0, geometry=False,
                  threads=1):
    """Reference one-sample Stage-II gradient (ref_train_sample, reference build only)."""
    sc = scene_h.data
    k = len(sc["tau_logits"])
    L = (sc["l_max"] + 1) ** 2
    n_par = len(cond_h.data["params"]) if cond_h is not None else 0
    loss = np.zeros(1)
    d_base = np.empty(k * L * sc["channels"] * 2)
    d_par = np.empty(n_par)
    geo = [np.empty(k * 3), np.empty(k * 3), np.empty(k * 4), np.empty(k)] if geometry else [None] * 4
    err = C.create_string_buffer(512)
    rc = self._train_sample(scene_h.ptr, None if cond_h is None else cond_h.ptr, grid.gi, grid.gd, _d(np.asarray(tx, np.float64)),
                            _d(np.asarray(rx, np.float64)), _d(np.asarray(target, np.float64)), lambda_ssim,
                            lambda_fft, threads, loss.ctypes.data_as(_dp), d_base.ctypes.data_as(_dp),
                            d_par.ctypes.data_as(_dp), *[None if g is None else g.ctypes.data_as(_dp) for g in geo],
                            err, 512)
    if rc:
        raise CheckerError(err.value.decode())
    out = dict(loss=float(loss[0]), d_base=d_base, d_params=d_par)
    if geometry:
        out.update(d_positions=geo[0], d_log_scales=geo[1], d_quaternions=geo[2], d_tau_logits=geo[3])
    return out


Checker.train_sample = _train_sample


def _coverage_fraction(self, table, selected, thr):
    """apps::coverage_fraction (reference build only)."""
    t = np.ascontiguousarray(table, np.float64)
    sel = np.ascontiguousarray(selected, np.int32)
    out = np.zeros(1)
    err = C.create_string_buffer(512)
    if self._coverage_fraction(t.ctypes.data_as(_dp), t.shape[0], t.shape[1], sel.ctypes.data_as(_ip), sel.size,
                               float(thr), out.ctypes.data_as(_dp), err, 512):
        raise ValueError(err.value.decode())
    return float(out[0])


def _greedy_plan(self, table, k, thr):
    """apps::greedy_plan (reference build only)."""
    t = np.ascontiguousarray(table, np.float64)
    order = np.zeros(max(int(k), 1), np.int32)
    err = C.create_string_buffer(512)
    if self._greedy_plan(t.ctypes.data_as(_dp), t.shape[0], t.shape[1], int(k), float(thr),
                         order.ctypes.data_as(_ip), err, 512):
        raise ValueError(err.value.decode())
    return order[:k]


def _image_metrics(self, pred, gt, h, w, max_val=1.0, window=11, sigma=1.5, dyn=1.0):
    """met::{mae, mse, psnr, ssim} of one image (reference build only)."""
    p = np.ascontiguousarray(pred, np.float64)
    g = np.ascontiguousarray(gt, np.float64)
    out = np.zeros(4)
    err = C.create_string_buffer(512)
    if self._image_metrics(p.ctypes.data_as(_dp), g.ctypes.data_as(_dp), int(h), int(w), float(max_val), int(window),
                           float(sigma), float(dyn), out.ctypes.data_as(_dp), err, 512):
        raise ValueError(err.value.decode())
    return out


def _checkpoint_save(self, path, scene_h, cond_h, grid: Grid):
    """io::save_checkpoint (checkpoint.cpp:93-155) of Model{scene, grid, cond};
    reference build only (needs checkpoint.cpp)."""
    err = C.create_string_buffer(512)
    rc = self._checkpoint_save(str(path).encode(), scene_h.ptr, None if cond_h is None else cond_h.ptr, grid.gi,
                               grid.gd, err, 512)
    if rc:
        raise CheckerError(err.value.decode())


def _checkpoint_load(self, path):
    """io::load_checkpoint (checkpoint.cpp:157-231): a dict with the scene arrays,
    modality, grid (n_theta, n_phi, tile_size, radius, theta_min, theta_max)
    and the conditioning (cfg, packed params, occupancy, lo, hi) or None."""
    cond = C.c_void_p()
    gi = np.zeros(3, np.int32)
    gd = np.zeros(3)
    err = C.create_string_buffer(512)
    ptr = self._checkpoint_load(str(path).encode(), C.byref(cond), _i(gi), _d(gd), err, 512)
    if not ptr:
        raise CheckerError(err.value.decode())
    shp = np.zeros(3, np.int32)
    self._scene_shape(ptr, _i(shp))
    k, l_max, ch = (int(v) for v in shp)
    h = _Handle(self, ptr, self._scene_free, dict(l_max=l_max, channels=ch))
    arrays = _scene_arrays(self, h)
    out = dict(scene=dict(arrays, l_max=l_max, channels=ch), handle=h,
               modality={0: "rssi", 1: "csi", 2: "spectrum"}[self._scene_modality(ptr)],
               grid=(int(gi[0]), int(gi[1]), int(gi[2]), float(gd[0]), float(gd[1]), float(gd[2])), cond=None)
    if cond.value:
        cfg = np.zeros(9, np.int32)
        lo, hi = np.zeros(3), np.zeros(3)
        self._cond_export(cond.value, _i(cfg), None, None, _d(lo), _d(hi))
        n = self._cond_param_count(cond.value)
        params = np.empty(n)
        R = int(cfg[4])
        occ = np.empty(R ** 3)
        self._cond_export(cond.value, _i(cfg), _d(params), _d(occ) if R else None, _d(lo), _d(hi))
        out["cond"] = dict(cfg=cfg, params=params, occupancy=occ, lo=lo, hi=hi)
        self._cond_free(cond.value)
    return out


Checker.checkpoint_save = _checkpoint_save
Checker.checkpoint_load = _checkpoint_load


def _scene_arrays(self, h):
    """Current arrays of a reference scene handle (after densify_and_prune)."""
    k = self._scene_count(h.ptr)
    sc = h.data
    L = (sc["l_max"] + 1) ** 2
    out = dict(positions=np.empty(3 * k), log_scales=np.empty(3 * k), quaternions=np.empty(4 * k),
               tau_logits=np.empty(k), fle_coeffs=np.empty(k * L * sc["channels"] * 2))
    self._scene_get(h.ptr, *[_d(v) for v in out.values()])
    return out


def _densify(self, h, d_pos_list, extent, thresholds=(2e-4, 0.01, 0.1, 0.8), seed=1, pass_index=0):
    """densify_and_prune (scene.cpp:178-274) on the handle's scene, in place;
    d_pos_list: accumulate() inputs (n_acc x K*3) -> (report, source_row)."""
    k = self._scene_count(h.ptr)
    acc = np.ascontiguousarray(d_pos_list, np.float64).reshape(-1, 3 * k)
    thr = np.ascontiguousarray(thresholds, np.float64)
    report = np.zeros(3, np.int32)
    src = np.zeros(2 * k + 1, np.int32)
    err = C.create_string_buffer(512)
    if self._densify(h.ptr, acc.ctypes.data_as(_dp), acc.shape[0], float(extent), thr.ctypes.data_as(_dp), int(seed),
                     int(pass_index), report.ctypes.data_as(_ip), src.ctypes.data_as(_ip), err, 512):
        raise ValueError(err.value.decode())
    return report, src[: self._scene_count(h.ptr)]


Checker.scene_arrays = _scene_arrays
Checker.densify = _densify
Checker.image_metrics = _image_metrics


def _snr_csi(self, pred, gt):
    """met::snr_csi (metrics.cpp:114-125); pred / gt complex arrays; reference only."""
    p = np.ascontiguousarray(np.asarray(pred, np.complex128)).view(np.float64)
    g = np.ascontiguousarray(np.asarray(gt, np.complex128)).view(np.float64)
    out = np.zeros(1)
    err = C.create_string_buffer(512)
    if self._snr_csi(_d(p), _d(g), len(p) // 2, out.ctypes.data_as(_dp), err, 512):
        raise CheckerError(err.value.decode())
    return float(out[0])


def _per_receiver_aggregate(self, rx, values):
    """met::per_receiver_aggregate (metrics.cpp:127-149); reference only.
    Returns (rx ids, means, counts, mean, stddev)."""
    rx = np.ascontiguousarray(rx, np.int32)
    v = np.ascontiguousarray(values, np.float64)
    n = len(rx)
    o_rx, o_mean, o_cnt = np.zeros(max(n, 1), np.int32), np.zeros(max(n, 1)), np.zeros(max(n, 1), np.int64)
    nu = np.zeros(1, np.int32)
    mean, sd = np.zeros(1), np.zeros(1)
    err = C.create_string_buffer(512)
    if self._per_receiver_aggregate(_i(rx), _d(v), n, _i(o_rx), _d(o_mean), o_cnt.ctypes.data_as(_lp), _i(nu),
                                    _d(mean), _d(sd), err, 512):
        raise CheckerError(err.value.decode())
    u = int(nu[0])
    return o_rx[:u], o_mean[:u], o_cnt[:u], float(mean[0]), float(sd[0])


Checker.snr_csi = _snr_csi
Checker.per_receiver_aggregate = _per_receiver_aggregate
Checker.coverage_fraction = _coverage_fraction
Checker.greedy_plan = _greedy_plan
