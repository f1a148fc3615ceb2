"""ctypes binding of the C-ABI in include/rxgs_b200.h (librxgs_b200.so).

This is plumbing for Python callers (tests, bench.py): every call goes
straight to the native library; there is no Python or CPU compute path.  If
the shared library is missing the import fails loudly.

Arrays may be numpy (host) or anything exposing ``data_ptr()`` (a CUDA torch
tensor, passed as a device pointer).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RXGS_B200_LIB") or os.path.join(HERE, "librxgs_b200.so")  # override: A/B builds

RXGS_OK, RXGS_ERR_INVALID, RXGS_ERR_RUNTIME, RXGS_ERR_CUDA, RXGS_ERR_IO = 0, 1, 2, 3, 4
MODALITY = {"rssi": 0, "csi": 1, "spectrum": 2}
MODE = {"full": 0, "global_only": 1, "local_only": 2, "additive_only": 3, "no_occlusion": 4}

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (the B200 path has no fallback)")

_lib = C.CDLL(LIB_PATH)
_vp = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64


class Grid(C.Structure):
    """raster::SphericalGrid (sphraster.hpp:15-32) as rxgs_grid."""
    _fields_ = [("n_theta", _i32), ("n_phi", _i32), ("tile_size", _i32), ("reserved", _i32),
                ("radius", C.c_double), ("theta_min", C.c_double), ("theta_max", C.c_double)]

    def __init__(self, n_theta=1, n_phi=1, tile_size=8, radius=1.0, theta_min=0.0,
                 theta_max=3.14159265358979323846):
        super().__init__(int(n_theta), int(n_phi), int(tile_size), 0, float(radius), float(theta_min),
                         float(theta_max))

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


_SIG = {
    "rxgs_last_error": (C.c_char_p, []),
    "rxgs_version": (C.c_int, []),
    "rxgs_ctx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "rxgs_ctx_destroy": (C.c_int, [_vp]),
    "rxgs_ctx_set_stream": (C.c_int, [_vp, _vp]),
    "rxgs_ctx_synchronize": (C.c_int, [_vp]),
    "rxgs_ctx_profile": (C.c_int, [_vp, C.c_int]),
    "rxgs_ctx_kernel_stats": (C.c_int, [_vp, C.c_char_p, C.POINTER(C.c_double), C.POINTER(_i64),
                                        C.POINTER(C.c_double)]),
    "rxgs_ctx_reset_stats": (C.c_int, [_vp]),
    "rxgs_ctx_release_cache": (C.c_int, [_vp]),
    "rxgs_ctx_launch_count": (_i64, [_vp]),
    "rxgs_ctx_set_cond_kernel": (C.c_int, [_vp, C.c_int]),
    "rxgs_ctx_set_composite_kernel": (C.c_int, [_vp, C.c_int]),
    "rxgs_selftest_tcgen05": (C.c_int, [_vp, _vp]),
    "rxgs_synth_scene": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_uint64, _vp, _vp, _vp, _vp, _vp]),
    "rxgs_synth_points": (C.c_int, [C.c_int, C.c_uint64, C.c_char_p, _vp, _vp, C.c_double, _vp]),
    "rxgs_synth_cond": (_i64, [_vp, C.c_int, C.c_int, _vp, _vp, C.c_uint64, C.c_int, _vp]),
    "rxgs_scene_create": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp,
                                    C.POINTER(_vp)]),
    "rxgs_scene_destroy": (C.c_int, [_vp]),
    "rxgs_scene_bounds": (C.c_int, [_vp, C.c_double, _vp, _vp]),
    "rxgs_tx_state_build": (C.c_int, [_vp, _vp, _vp, C.POINTER(Grid), C.POINTER(_vp)]),
    "rxgs_tx_state_destroy": (C.c_int, [_vp]),
    "rxgs_tx_state_entries": (_i64, [_vp]),
    "rxgs_tx_state_get": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "rxgs_tx_state_keys": (C.c_int, [_vp, _vp]),
    "rxgs_tx_state_stats": (C.c_int, [_vp, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(C.c_double),
                                      C.POINTER(C.c_double)]),
    "rxgs_tx_state_transmittance": (C.c_int, [_vp, _vp]),
    "rxgs_tx_state_needed": (C.c_int, [_vp, C.POINTER(_i64)]),
    "rxgs_bin_and_sort": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, C.POINTER(Grid), _vp, _vp, _i64,
                                    C.POINTER(_i64)]),
    "rxgs_render_field": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int, _vp, _vp]),
    "rxgs_aggregate_modality": (C.c_int, [_vp, C.POINTER(Grid), C.c_int, C.c_int, C.c_int, _vp, _vp]),
    "rxgs_aggregate_modality_backward": (C.c_int, [_vp, C.POINTER(Grid), C.c_int, C.c_int, C.c_int, _vp, _vp,
                                                   _vp]),
    "rxgs_backward_render": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int, _vp, _vp, _vp, _vp, _vp, _vp]),
    "rxgs_cond_create": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, C.POINTER(_vp)]),
    "rxgs_cond_destroy": (C.c_int, [_vp]),
    "rxgs_cond_param_count": (_i64, [_vp]),
    "rxgs_cond_calls": (C.c_int, [_vp, C.POINTER(_i64), C.POINTER(_i64)]),
    "rxgs_build_occupancy": (C.c_int, [_vp, _vp, C.c_int, _vp, _vp, _vp, _vp]),
    "rxgs_probe_segments": (C.c_int, [_vp, _vp, C.c_int, _vp, _vp, _vp]),
    "rxgs_condition_forward": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "rxgs_condition_backward": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "rxgs_condition_batch": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int, _vp]),
    "rxgs_render_queries": (C.c_int, [_vp, _vp, _vp, _vp, _vp, C.c_int, _vp, _vp]),
    "rxgs_coverage_table": (C.c_int, [_vp, _vp, _vp, C.POINTER(Grid), _vp, C.c_int, _vp, C.c_int, _vp]),
    "rxgs_predict": (C.c_int, [_vp, _vp, _vp, C.POINTER(Grid), _vp, _vp, _vp]),
    "rxgs_snr_csi": (C.c_int, [_vp, C.c_int, C.c_int64, _vp, _vp, _vp]),
    "rxgs_per_receiver_aggregate": (C.c_int, [_vp, C.c_int64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "rxgs_project_gaussians": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, _vp, C.POINTER(Grid), _vp, _vp, _vp]),
    "rxgs_fle_eval": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _vp]),
    "rxgs_blend_ray": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp]),
    "rxgs_occupancy_sample": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, C.c_int, _vp, C.c_int, _vp]),
    "rxgs_probe_grid": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, C.c_int, _vp, _vp, C.c_int, C.c_int, _vp]),
    "rxgs_fourier_encode": (C.c_int, [_vp, C.c_int, _vp, C.c_int, _vp, _vp]),
    "rxgs_mlp_layer_forward": (C.c_int, [_vp, C.c_int, C.c_int, _vp, _vp, C.c_int, _vp, _vp]),
    "rxgs_grid_validate": (C.c_int, [C.POINTER(Grid)]),
    "rxgs_condition_forward_base": (C.c_int, [_vp, _vp, _vp, _vp, _vp, C.c_int, _vp, _vp]),
    "rxgs_tx_state_import": (C.c_int, [_vp, _vp, C.POINTER(Grid), _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "rxgs_trainer_create": (C.c_int, [_vp, _vp, _vp, _vp, C.POINTER(_vp)]),
    "rxgs_trainer_destroy": (C.c_int, [_vp]),
    "rxgs_train_grads": (C.c_int, [_vp, _vp, _vp, C.c_int, _vp, _vp, C.c_int]),
    "rxgs_train_grad_buffer": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(_i64), C.POINTER(_i64)]),
    "rxgs_train_get_grads": (C.c_int, [_vp, _vp, _vp]),
    "rxgs_train_get_grad_buffer": (C.c_int, [_vp, _vp]),
    "rxgs_train_allreduce": (C.c_int, [_vp, _vp]),
    "rxgs_trainer_enable_geometry": (C.c_int, [_vp, _vp]),
    "rxgs_train_densify": (C.c_int, [_vp, C.c_double, _vp, C.c_uint64, C.c_uint64, _vp]),
    "rxgs_train_reset_transmittance": (C.c_int, [_vp]),
    "rxgs_train_get_geometry_grads": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "rxgs_train_apply": (C.c_int, [_vp]),
    "rxgs_train_step_count": (_i64, [_vp]),
    "rxgs_scene_get_coeffs": (C.c_int, [_vp, _vp]),
    "rxgs_checkpoint_save": (C.c_int, [C.c_char_p, _vp, C.POINTER(Grid), _vp]),
    "rxgs_checkpoint_load": (C.c_int, [_vp, C.c_char_p, C.POINTER(_vp), C.POINTER(Grid), C.POINTER(_vp)]),
    "rxgs_coverage_fraction": (C.c_int, [_vp, _vp, _i64, _i64, _vp, C.c_int, C.c_double, C.POINTER(C.c_double)]),
    "rxgs_densify_and_prune": (C.c_int, [_vp, _vp, _vp, _vp, C.c_double, _vp, C.c_uint64, C.c_uint64, _vp, _vp,
                                         C.POINTER(_i32)]),
    "rxgs_reset_transmittance": (C.c_int, [_vp]),
    "rxgs_image_metrics": (C.c_int, [_vp, _vp, C.c_int, _vp, C.c_int, C.c_int, C.c_int, C.c_double, _vp, _vp]),
    "rxgs_greedy_plan": (C.c_int, [_vp, _vp, _i64, _i64, C.c_int, C.c_double, _vp]),
    "rxgs_scene_info": (C.c_int, [_vp, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32)]),
    "rxgs_cond_config": (C.c_int, [_vp, _vp]),
    "rxgs_scene_get_arrays": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "rxgs_cond_get_occupancy": (C.c_int, [_vp, C.POINTER(_i32), _vp, _vp, _vp]),
    "rxgs_cond_get_params": (C.c_int, [_vp, _vp]),
}
for _name, (_res, _args) in _SIG.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIG)


class RxgsError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class InvalidArgument(RxgsError, ValueError):
    """The reference's std::invalid_argument."""


class IoError(RxgsError, OSError):
    """The reference's io::IoError (dataset.hpp:16)."""


def _check(rc):
    if rc != RXGS_OK:
        msg = _lib.rxgs_last_error().decode()
        if rc == RXGS_ERR_INVALID:
            raise InvalidArgument(rc, msg)
        if rc == RXGS_ERR_IO:
            raise IoError(rc, msg)
        raise RxgsError(rc, msg)


_keep: list = []


def ptr(a, dtype=None):
    """Raw pointer of a numpy array (converted to a contiguous `dtype`) or a torch tensor."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    arr = np.ascontiguousarray(a, dtype=dtype) if dtype is not None else np.ascontiguousarray(a)
    _keep.append(arr)
    if len(_keep) > 64:
        del _keep[:32]
    return C.c_void_p(arr.ctypes.data)


def _out(shape, dtype=np.float64):
    return np.empty(shape, dtype)


# ------------------------------------------------------------------ synthetic inputs
def synth_scene(k, l_max=2, channels=1, seed=7):
    L = (l_max + 1) ** 2
    pos, ls, q, tau = _out((k, 3)), _out((k, 3)), _out((k, 4)), _out(k)
    co = _out((k, L, channels, 2))
    _check(_lib.rxgs_synth_scene(k, l_max, channels, seed, pos.ctypes.data, ls.ctypes.data, q.ctypes.data,
                                 tau.ctypes.data, co.ctypes.data))
    return dict(positions=pos, log_scales=ls, quaternions=q, tau_logits=tau, fle_coeffs=co, l_max=l_max,
                channels=channels)


def synth_points(n, seed, tag, lo, hi, margin=0.05):
    out = _out((n, 3))
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    _check(_lib.rxgs_synth_points(n, seed, tag.encode(), lo.ctypes.data, hi.ctypes.data, margin, out.ctypes.data))
    return out


def cond_cfg(F=6, hidden=64, dc=16, S=16, R=32, nearest=0, mode="full", l_max=2, C_=1):
    return np.array([F, hidden, dc, S, R, nearest, MODE[mode] if isinstance(mode, str) else mode, l_max, C_],
                    np.int32)


def synth_cond(cfg, l_max, channels, lo, hi, seed=3, randomize=True):
    cfg = np.asarray(cfg, np.int32)
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    n = _lib.rxgs_synth_cond(cfg.ctypes.data, l_max, channels, lo.ctypes.data, hi.ctypes.data, seed,
                             int(randomize), None)
    out = _out(n)
    _lib.rxgs_synth_cond(cfg.ctypes.data, l_max, channels, lo.ctypes.data, hi.ctypes.data, seed, int(randomize),
                         out.ctypes.data)
    return out


# ------------------------------------------------------------------ handles
class Context:
    def __init__(self, device=0):
        h = _vp()
        _check(_lib.rxgs_ctx_create(device, C.byref(h)))
        self.h = h

    def close(self, _fn=_lib.rxgs_ctx_destroy):
        if getattr(self, "h", None):
            _fn(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def set_stream(self, stream_handle):
        _check(_lib.rxgs_ctx_set_stream(self.h, C.c_void_p(stream_handle) if stream_handle else None))

    def synchronize(self):
        _check(_lib.rxgs_ctx_synchronize(self.h))

    def profile(self, enable=True):
        _check(_lib.rxgs_ctx_profile(self.h, int(enable)))

    def kernel_stats(self, name):
        ms, n, w = C.c_double(), _i64(), C.c_double()
        _check(_lib.rxgs_ctx_kernel_stats(self.h, name.encode(), C.byref(ms), C.byref(n), C.byref(w)))
        return ms.value, n.value, w.value

    def reset_stats(self):
        _check(_lib.rxgs_ctx_reset_stats(self.h))

    def launch_count(self):
        return int(_lib.rxgs_ctx_launch_count(self.h))

    def release_cache(self):
        _check(_lib.rxgs_ctx_release_cache(self.h))

    def set_cond_kernel(self, which):
        """'auto' (tcgen05 when eligible) or 'simt'."""
        _check(_lib.rxgs_ctx_set_cond_kernel(self.h, {"auto": 0, "simt": 1}[which]))

    def set_composite_kernel(self, which):
        """'auto' (tcgen05 when eligible) or 'simt'."""
        _check(_lib.rxgs_ctx_set_composite_kernel(self.h, {"auto": 0, "simt": 1}[which]))

    def selftest_tcgen05(self):
        e = np.zeros(5)
        _check(_lib.rxgs_selftest_tcgen05(self.h, e.ctypes.data))
        return tuple(float(x) for x in e)

    # ---------------------------------------------------------- objects
    def scene(self, sc, modality="spectrum"):
        return Scene(self, sc, modality)

    def cond(self, cfg, params, occ=None, lo=None, hi=None):
        return Cond(self, cfg, params, occ, lo, hi)

    def load_checkpoint(self, path):
        """io::load_checkpoint (checkpoint.cpp:157-231) -> (Scene, Grid, Cond or None)."""
        hs, hc, grid = _vp(), _vp(), Grid()
        _check(_lib.rxgs_checkpoint_load(self.h, os.fsencode(str(path)), C.byref(hs), C.byref(grid), C.byref(hc)))
        scene = Scene._wrap(self, hs)
        cond = Cond._wrap(self, hc) if hc.value else None
        return scene, grid, cond

    def coverage_fraction(self, table, selected, threshold_dbm):
        """apps::coverage_fraction (apps.cpp:69-84) over a tx-major table."""
        table = np.ascontiguousarray(table, np.float64)
        sel = np.ascontiguousarray(selected, np.int32)
        out = C.c_double()
        _check(_lib.rxgs_coverage_fraction(self.h, table.ctypes.data, table.shape[0], table.shape[1],
                                           sel.ctypes.data if sel.size else None, int(sel.size),
                                           float(threshold_dbm), C.byref(out)))
        return out.value

    def greedy_plan(self, table, k, threshold_dbm):
        """apps::greedy_plan (apps.cpp:86-114): k candidates in selection order."""
        table = np.ascontiguousarray(table, np.float64)
        order = np.empty(max(int(k), 0), np.int32)
        _check(_lib.rxgs_greedy_plan(self.h, table.ctypes.data, table.shape[0], table.shape[1], int(k),
                                     float(threshold_dbm), order.ctypes.data if order.size else None))
        return order

    def image_metrics(self, pred, gt, h, w, max_val=1.0, ssim=(11, 1.5, 1.0)):
        """met::{mae, mse, psnr, ssim} per image (metrics.cpp:11-112) -> (n, 4).
        pred: f32 or f64 (host array or CUDA tensor), gt: f64; ssim=None skips SSIM."""
        if hasattr(pred, "data_ptr"):
            import torch
            f32 = pred.dtype == torch.float32
        else:
            pred = np.ascontiguousarray(pred)
            if pred.dtype != np.float32:
                pred = pred.astype(np.float64)
            f32 = pred.dtype == np.float32
        gt = gt if hasattr(gt, "data_ptr") else np.ascontiguousarray(gt, np.float64)
        n = max(1, (pred.numel() if hasattr(pred, "numel") else pred.size) // max(h * w, 1))
        out = np.empty((n, 4))
        opts = np.asarray(ssim if ssim is not None else (0, 1.5, 1.0), np.float64)
        _check(_lib.rxgs_image_metrics(self.h, ptr(pred), int(f32), ptr(gt), n, int(h), int(w), float(max_val),
                                       opts.ctypes.data, out.ctypes.data))
        return out

    def snr_csi(self, pred, gt):
        """met::snr_csi (metrics.cpp:114-125) per row of complex (n_sets, len) arrays -> dB."""
        p = np.ascontiguousarray(np.atleast_2d(np.asarray(pred, np.complex128)))
        g = np.ascontiguousarray(np.atleast_2d(np.asarray(gt, np.complex128)))
        if p.shape != g.shape:
            raise InvalidArgument(RXGS_ERR_INVALID, "snr_csi: need equal non-empty inputs")
        out = np.empty(p.shape[0])
        _check(_lib.rxgs_snr_csi(self.h, p.shape[0], p.shape[1], p.ctypes.data, g.ctypes.data, out.ctypes.data))
        return out

    def per_receiver_aggregate(self, rx, values):
        """met::per_receiver_aggregate (metrics.cpp:127-149) -> (rx, means, counts, mean, stddev)."""
        rx = np.ascontiguousarray(rx, np.int32)
        v = np.ascontiguousarray(values, np.float64)
        n = len(rx)
        o_rx, o_m, o_c = np.empty(max(n, 1), np.int32), np.empty(max(n, 1)), np.empty(max(n, 1), np.int64)
        nu = C.c_int32(0)
        mu, sd = C.c_double(0), C.c_double(0)
        _check(_lib.rxgs_per_receiver_aggregate(self.h, n, rx.ctypes.data, v.ctypes.data, o_rx.ctypes.data,
                                                o_m.ctypes.data, o_c.ctypes.data, C.byref(nu), C.byref(mu),
                                                C.byref(sd)))
        u = nu.value
        return o_rx[:u], o_m[:u], o_c[:u], mu.value, sd.value

    def bin_and_sort(self, culled, depth, spans, grid: Grid):
        k = len(culled)
        offs = np.empty(grid.n_tiles + 1, np.int64)
        n = _i64()
        cul = np.ascontiguousarray(culled, np.int32)
        dep = np.ascontiguousarray(depth, np.float64)
        sp = np.ascontiguousarray(spans, np.int32)
        _check(_lib.rxgs_bin_and_sort(self.h, k, cul.ctypes.data, dep.ctypes.data, sp.ctypes.data, C.byref(grid),
                                      offs.ctypes.data, None, 0, C.byref(n)))
        idx = np.empty(max(n.value, 1), np.int32)
        _check(_lib.rxgs_bin_and_sort(self.h, k, cul.ctypes.data, dep.ctypes.data, sp.ctypes.data, C.byref(grid),
                                      offs.ctypes.data, idx.ctypes.data, n.value, C.byref(n)))
        return offs, idx[:n.value]

    def aggregate(self, values, grid: Grid, modality):
        values = np.ascontiguousarray(values, np.float64)
        n_rx, ch = values.shape[0], values.shape[1]
        m = MODALITY[modality]
        shape = (n_rx,) if m == 0 else ((n_rx, ch, 2) if m == 1 else (n_rx, grid.n_theta, grid.n_phi))
        out = _out(shape)
        _check(_lib.rxgs_aggregate_modality(self.h, C.byref(grid), m, n_rx, ch, values.ctypes.data,
                                            out.ctypes.data))
        return out


    def aggregate_backward(self, values, grid: Grid, modality, upstream):
        """raster::aggregate_modality_backward (sphraster.cpp:383-449)."""
        values = np.ascontiguousarray(values, np.float64)
        n_rx, ch = values.shape[0], values.shape[1]
        out = _out(values.shape)
        _check(_lib.rxgs_aggregate_modality_backward(self.h, C.byref(grid), MODALITY[modality], n_rx, ch,
                                                     values.ctypes.data, ptr(upstream, np.float64),
                                                     out.ctypes.data))
        return out

class Scene:
    """GaussianScene upload (scene.hpp:19-48)."""

    def __init__(self, ctx: Context, sc, modality="spectrum"):
        self.ctx = ctx
        self.data = sc
        self.k = len(sc["tau_logits"])
        self.l_max = sc["l_max"]
        self.channels = sc["channels"]
        self.L = (self.l_max + 1) ** 2
        self.modality = modality
        h = _vp()
        _check(_lib.rxgs_scene_create(ctx.h, self.k, self.l_max, self.channels, MODALITY[modality],
                                      ptr(sc["positions"], np.float64), ptr(sc["log_scales"], np.float64),
                                      ptr(sc["quaternions"], np.float64), ptr(sc["tau_logits"], np.float64),
                                      ptr(sc["fle_coeffs"], np.float64), C.byref(h)))
        self.h = h

    @classmethod
    def _wrap(cls, ctx: Context, h):
        """A Scene around a handle created by the library (checkpoint load)."""
        self = cls.__new__(cls)
        self.ctx, self.h, self.data = ctx, h, None
        k, l, c, m = _i32(), _i32(), _i32(), _i32()
        _check(_lib.rxgs_scene_info(h, C.byref(k), C.byref(l), C.byref(c), C.byref(m)))
        self.k, self.l_max, self.channels = k.value, l.value, c.value
        self.L = (self.l_max + 1) ** 2
        self.modality = {v: n for n, v in MODALITY.items()}[m.value]
        return self

    def save_checkpoint(self, path, grid: Grid, cond=None):
        """io::save_checkpoint (checkpoint.cpp:93-155)."""
        _check(_lib.rxgs_checkpoint_save(os.fsencode(str(path)), self.h, C.byref(grid), cond.h if cond else None))

    def __del__(self, _fn=_lib.rxgs_scene_destroy):
        if getattr(self, "h", None):
            _fn(self.h)
            self.h = None

    def densify_and_prune(self, grad_accum, accum_count, extent, thresholds=None, seed=1, pass_index=0):
        """densify_and_prune (scene.cpp:178-274) in place -> (report, source_row)."""
        acc = grad_accum if hasattr(grad_accum, "data_ptr") else np.ascontiguousarray(grad_accum, np.float64)
        cnt = accum_count if hasattr(accum_count, "data_ptr") else np.ascontiguousarray(accum_count, np.int32)
        thr = None if thresholds is None else np.ascontiguousarray(thresholds, np.float64)
        report = np.zeros(3, np.int32)
        src = np.zeros(2 * self.k + 1, np.int32)
        nk = _i32()
        _check(_lib.rxgs_densify_and_prune(self.ctx.h, self.h, ptr(acc), ptr(cnt), float(extent),
                                           None if thr is None else thr.ctypes.data, int(seed), int(pass_index),
                                           report.ctypes.data, src.ctypes.data, C.byref(nk)))
        self.k = nk.value
        return report, src[: self.k]

    def reset_transmittance(self):
        _check(_lib.rxgs_reset_transmittance(self.h))

    def bounds(self, inflate=0.0):
        lo, hi = _out(3), _out(3)
        _check(_lib.rxgs_scene_bounds(self.h, inflate, lo.ctypes.data, hi.ctypes.data))
        return lo, hi

    def tx_state(self, tx, grid: Grid):
        return TxState(self, tx, grid)

    def render_field(self, st, coeffs, n_rx, values=None, transmittance=None):
        own = values is None
        if own:
            values = _out((n_rx, self.channels, 2, st.grid.n_theta, st.grid.n_phi))
            transmittance = _out((n_rx, st.grid.n_theta, st.grid.n_phi))
        _check(_lib.rxgs_render_field(self.ctx.h, st.h, self.h, ptr(coeffs, np.float64), n_rx, ptr(values),
                                      ptr(transmittance)))
        return values, transmittance

    def backward_render(self, st, coeffs, n_rx, d_values):
        """raster::backward_render (sphraster.cpp:509-733) -> GradientBundle dict."""
        co = np.ascontiguousarray(coeffs, np.float64)
        out = dict(d_positions=_out((self.k, 3)), d_log_scales=_out((self.k, 3)), d_quaternions=_out((self.k, 4)),
                   d_tau_logits=_out(self.k), d_coeffs=_out(co.shape))
        _check(_lib.rxgs_backward_render(self.ctx.h, st.h, self.h, co.ctypes.data, n_rx, ptr(d_values, np.float64),
                                         *(out[n].ctypes.data for n in ("d_positions", "d_log_scales",
                                                                        "d_quaternions", "d_tau_logits",
                                                                        "d_coeffs"))))
        return out

    def render_queries(self, cond, st, rx, spectrum=None, rssi=None, want=("spectrum", "rssi")):
        """Fused batched query path; numpy in -> numpy out unless torch tensors are passed."""
        n = int(rx.shape[0])
        if spectrum is None and "spectrum" in want:
            spectrum = np.empty((n, st.grid.n_theta, st.grid.n_phi), np.float32)
        if rssi is None and "rssi" in want:
            rssi = np.empty(n, np.float32)
        _check(_lib.rxgs_render_queries(self.ctx.h, self.h, None if cond is None else cond.h, st.h,
                                        ptr(rx, np.float64), n, ptr(spectrum), ptr(rssi)))
        return spectrum, rssi

    def coverage_table(self, cond, grid: Grid, tx, rx, out=None):
        """RSSI table [n_tx][n_rx] (BASELINE config 3; apps.cpp:70-116 layout)."""
        tx = tx if hasattr(tx, "data_ptr") else np.ascontiguousarray(tx, np.float64).reshape(-1, 3)
        rx = rx if hasattr(rx, "data_ptr") else np.ascontiguousarray(rx, np.float64).reshape(-1, 3)
        n_tx, n_rx = int(tx.shape[0]), int(rx.shape[0])
        if out is None:
            out = np.empty((n_tx, n_rx), np.float32)
        _check(_lib.rxgs_coverage_table(self.ctx.h, self.h, None if cond is None else cond.h, C.byref(grid),
                                        ptr(tx, np.float64), n_tx, ptr(rx, np.float64), n_rx, ptr(out)))
        return out

    def predict(self, cond, grid: Grid, tx, rx):
        m = MODALITY[self.modality]
        out = _out(grid.cells if m == 2 else (1 if m == 0 else 2 * self.channels))
        _check(_lib.rxgs_predict(self.ctx.h, self.h, None if cond is None else cond.h, C.byref(grid),
                                 ptr(tx, np.float64), ptr(rx, np.float64), out.ctypes.data))
        return out


class TxState:
    """raster::TxState (sphraster.hpp:52-61), device resident."""

    def __init__(self, scene: Scene, tx, grid: Grid):
        self.scene = scene
        self.grid = grid
        h = _vp()
        _check(_lib.rxgs_tx_state_build(scene.ctx.h, scene.h, ptr(tx, np.float64), C.byref(grid), C.byref(h)))
        self.h = h

    def __del__(self, _fn=_lib.rxgs_tx_state_destroy):
        if getattr(self, "h", None):
            _fn(self.h)
            self.h = None

    @property
    def entries(self):
        return int(_lib.rxgs_tx_state_entries(self.h))

    def get(self):
        k, L = self.scene.k, self.scene.L
        n = self.entries
        culled = np.empty(k, np.int32)
        geom = _out((k, 12))
        spans = np.empty((k, 4), np.int32)
        basis = _out((k, L, 2))
        offs = np.empty(self.grid.n_tiles + 1, np.int64)
        idx = np.empty(max(n, 1), np.int32)
        _check(_lib.rxgs_tx_state_get(self.h, culled.ctypes.data, geom.ctypes.data, spans.ctypes.data,
                                      basis.ctypes.data, offs.ctypes.data, idx.ctypes.data))
        return dict(culled=culled, geom=geom, spans=spans, basis=basis, offsets=offs, indices=idx[:n])

    def keys(self):
        out = np.empty(max(self.entries, 1), np.uint64)
        _check(_lib.rxgs_tx_state_keys(self.h, out.ctypes.data))
        return out[:self.entries]

    def stats(self):
        v, e, w, tw = _i64(), _i64(), C.c_double(), C.c_double()
        _check(_lib.rxgs_tx_state_stats(self.h, C.byref(v), C.byref(e), C.byref(w), C.byref(tw)))
        nd = _i64()
        _check(_lib.rxgs_tx_state_needed(self.h, C.byref(nd)))
        return dict(visible=v.value, entries=e.value, walk_per_cell=w.value, tile_walk_per_cell=tw.value,
                    needed=nd.value)

    def transmittance(self):
        out = _out((self.grid.n_theta, self.grid.n_phi))
        _check(_lib.rxgs_tx_state_transmittance(self.h, out.ctypes.data))
        return out


class Cond:
    """cond::ConditioningState (conditioning.hpp:72-92), device resident."""

    def __init__(self, ctx: Context, cfg, params, occ=None, lo=None, hi=None):
        self.ctx = ctx
        self.cfg = np.asarray(cfg, np.int32)
        h = _vp()
        _check(_lib.rxgs_cond_create(ctx.h, ptr(self.cfg, np.int32), ptr(params, np.float64),
                                     ptr(occ, np.float64) if occ is not None else None,
                                     ptr(lo, np.float64) if lo is not None else None,
                                     ptr(hi, np.float64) if hi is not None else None, C.byref(h)))
        self.h = h

    @classmethod
    def _wrap(cls, ctx: Context, h):
        self = cls.__new__(cls)
        self.ctx, self.h = ctx, h
        self.cfg = np.zeros(9, np.int32)
        _check(_lib.rxgs_cond_config(h, self.cfg.ctypes.data))
        return self

    def __del__(self, _fn=_lib.rxgs_cond_destroy):
        if getattr(self, "h", None):
            _fn(self.h)
            self.h = None

    @property
    def param_count(self):
        return int(_lib.rxgs_cond_param_count(self.h))

    def calls(self):
        g, l_ = _i64(), _i64()
        _check(_lib.rxgs_cond_calls(self.h, C.byref(g), C.byref(l_)))
        return g.value, l_.value

    def build_occupancy(self, scene: Scene, R, lo, hi, attach=True):
        out = _out((R, R, R))
        _check(_lib.rxgs_build_occupancy(self.ctx.h, scene.h, R, ptr(lo, np.float64), ptr(hi, np.float64),
                                         out.ctypes.data, self.h if attach else None))
        return out

    def probe(self, frm, to):
        frm = np.ascontiguousarray(frm, np.float64).reshape(-1, 3)
        to = np.ascontiguousarray(to, np.float64).reshape(-1, 3)
        out = _out((frm.shape[0], 2))
        _check(_lib.rxgs_probe_segments(self.ctx.h, self.h, frm.shape[0], frm.ctypes.data, to.ctypes.data,
                                        out.ctypes.data))
        return out

    def forward(self, scene: Scene, rx, workspace=False):
        out = _out((scene.k, scene.L, scene.channels, 2))
        lin = _out((scene.k, 6)) if workspace else None
        _check(_lib.rxgs_condition_forward(self.ctx.h, self.h, scene.h, ptr(rx, np.float64), out.ctypes.data,
                                           None if lin is None else lin.ctypes.data))
        return (out, lin) if workspace else out

    def backward(self, scene: Scene, rx, d_out):
        """cond::condition_backward (conditioning.cpp:472-587) -> (d_base, packed d_params)."""
        d_base = _out((scene.k, scene.L, scene.channels, 2))
        d_params = _out(int(_lib.rxgs_cond_param_count(self.h)))
        _check(_lib.rxgs_condition_backward(self.ctx.h, self.h, scene.h, ptr(rx, np.float64),
                                            ptr(d_out, np.float64), d_base.ctypes.data, d_params.ctypes.data))
        return d_base, d_params

    def batch(self, scene: Scene, rx):
        rx = np.ascontiguousarray(rx, np.float64).reshape(-1, 3)
        out = _out((rx.shape[0], scene.k, scene.L, scene.channels, 2))
        _check(_lib.rxgs_condition_batch(self.ctx.h, self.h, scene.h, rx.ctypes.data, rx.shape[0], out.ctypes.data))
        return out


def build_occupancy(ctx: Context, scene: Scene, R, lo, hi):
    out = _out((R, R, R))
    _check(_lib.rxgs_build_occupancy(ctx.h, scene.h, R, ptr(lo, np.float64), ptr(hi, np.float64), out.ctypes.data,
                                     None))
    return out


class _CudaArray:
    """__cuda_array_interface__ view of a device buffer owned by the library
    (lets torch.distributed all-reduce it in place, zero copy)."""

    def __init__(self, ptr, n, typestr="<f8"):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3}


class Trainer:
    """Training step of the conditioned Stage-II chain (trainer.cpp:410-466)."""

    DEFAULTS = (5e-3, 0.2, 1e-3, 0.2, 0.1, 0.9, 0.999, 1e-8)
    # spectrum L1 only (lambda_ssim = lambda_fft = 0): the config-4 headline loss
    L1_ONLY = (5e-3, 0.2, 1e-3, 0.0, 0.0, 0.9, 0.999, 1e-8)

    # TrainConfig geometry defaults (trainer.hpp:78-92): position lr schedule
    # (lr_init, lr_final, total_steps, delay_mult, delay_steps), transmittance,
    # scaling, rotation lr, fle_ramp_interval
    GEOMETRY_DEFAULTS = (1.6e-4, 1.6e-6, 2000, 0.01, 200, 1e-2, 5e-3, 1e-3, 500)

    def __init__(self, ctx: Context, scene: Scene, cond: Cond, hyper=None, geometry=None):
        """geometry: None (Stage II, geometry frozen), True (joint with the
        TrainConfig defaults) or a 9-tuple like GEOMETRY_DEFAULTS."""
        self.ctx, self.scene, self.cond = ctx, scene, cond
        hp = np.asarray(hyper if hyper is not None else self.DEFAULTS, np.float64)
        h = _vp()
        _check(_lib.rxgs_trainer_create(ctx.h, scene.h, None if cond is None else cond.h, hp.ctypes.data,
                                        C.byref(h)))
        self.h = h
        self.geometry = geometry is not None and geometry is not False
        if self.geometry:
            geo = np.asarray(self.GEOMETRY_DEFAULTS if geometry is True else geometry, np.float64)
            _check(_lib.rxgs_trainer_enable_geometry(self.h, geo.ctypes.data))
        self._refresh()

    def _refresh(self):
        p, n, nb = _vp(), _i64(), _i64()
        _check(_lib.rxgs_train_grad_buffer(self.h, C.byref(p), C.byref(n), C.byref(nb)))
        self.grad_ptr, self.n, self.n_base = p.value, n.value, nb.value

    def densify(self, extent, thresholds=None, seed=1, pass_index=0):
        """One Stage-I densification tick (trainer.cpp:359-372) -> report (cloned, split, pruned)."""
        rep = np.zeros(3, np.int32)
        thr = None if thresholds is None else np.ascontiguousarray(thresholds, np.float64)
        _check(_lib.rxgs_train_densify(self.h, float(extent), None if thr is None else thr.ctypes.data, int(seed),
                                       int(pass_index), rep.ctypes.data))
        k = _i32()
        _check(_lib.rxgs_scene_info(self.scene.h, C.byref(k), None, None, None))
        self.scene.k = k.value
        self._refresh()
        return rep

    def reset_transmittance(self):
        _check(_lib.rxgs_train_reset_transmittance(self.h))

    def __del__(self, _fn=_lib.rxgs_trainer_destroy):
        if getattr(self, "h", None):
            _fn(self.h)
            self.h = None

    def grads(self, st: TxState, rx, targets, accumulate=False):
        """Loss per sample; gradients summed into the device buffer."""
        rx = rx if hasattr(rx, "data_ptr") else np.ascontiguousarray(rx, np.float64)
        tg = targets if hasattr(targets, "data_ptr") else np.ascontiguousarray(targets, np.float32)
        n = int(rx.shape[0])
        loss = np.empty(n)
        _check(_lib.rxgs_train_grads(self.h, st.h, ptr(rx), n, ptr(tg), loss.ctypes.data, int(accumulate)))
        return loss

    def grad_tensor(self):
        """The flat f64 gradient buffer as a zero-copy CUDA torch tensor."""
        import torch
        return torch.as_tensor(_CudaArray(self.grad_ptr, self.n), device=f"cuda:{torch.cuda.current_device()}")

    def get_grads(self):
        db = np.empty(self.n_base)
        dp = np.empty(self.cond.param_count if self.cond is not None else 0)
        _check(_lib.rxgs_train_get_grads(self.h, db.ctypes.data, dp.ctypes.data))
        return db, dp

    def grad_buffer_host(self):
        """The whole flat gradient buffer [d_base | d_cond | d_geometry] (host copy)."""
        out = np.empty(self.n)
        _check(_lib.rxgs_train_get_grad_buffer(self.h, out.ctypes.data))
        return out

    def get_geometry_grads(self):
        """(d_positions K*3, d_log_scales K*3, d_quaternions K*4, d_tau_logits K)."""
        k = self.scene.k
        out = [np.empty(3 * k), np.empty(3 * k), np.empty(4 * k), np.empty(k)]
        _check(_lib.rxgs_train_get_geometry_grads(self.h, *[o.ctypes.data for o in out]))
        return tuple(out)

    def allreduce(self, nccl_comm: int):
        """Sum the gradient buffer over the ranks of an ncclComm_t (an integer
        handle: dist.nccl_comm_ptr(), or one made with ncclCommInitRank)."""
        _check(_lib.rxgs_train_allreduce(self.h, C.c_void_p(int(nccl_comm))))

    def apply(self):
        _check(_lib.rxgs_train_apply(self.h))

    @property
    def step_count(self):
        return int(_lib.rxgs_train_step_count(self.h))


def scene_coeffs(scene: Scene):
    out = np.empty(scene.k * scene.L * scene.channels * 2)
    _check(_lib.rxgs_scene_get_coeffs(scene.h, out.ctypes.data))
    return out


def scene_arrays(scene: Scene):
    """Current (possibly trained) scene arrays: positions, log_scales,
    quaternions, tau_logits, fle_coeffs (flat f64)."""
    k, L, c = scene.k, scene.L, scene.channels
    out = dict(positions=np.empty(3 * k), log_scales=np.empty(3 * k), quaternions=np.empty(4 * k),
               tau_logits=np.empty(k), fle_coeffs=np.empty(k * L * c * 2))
    _check(_lib.rxgs_scene_get_arrays(scene.h, *[v.ctypes.data for v in out.values()]))
    return out


def cond_params(cond: Cond):
    out = np.empty(cond.param_count)
    _check(_lib.rxgs_cond_get_params(cond.h, out.ctypes.data))
    return out
