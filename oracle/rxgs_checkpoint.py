"""TEST INFRASTRUCTURE (the checker, never the product): a Python restatement
of the reference's RXGS checkpoint container, io::save_checkpoint /
io::load_checkpoint (/root/reference/proj/src/checkpoint.cpp:93-231, format
include/rxgs/checkpoint.hpp:10-15).  The reference serialises its header with
nlohmann::ordered_json::dump(): compact JSON in insertion order, doubles as
the shortest round-trip digits in nlohmann's layout (dtoa_impl::format_buffer,
restated in _num).  Pinned against the reference itself: oracle/Makefile
builds checkpoint.cpp into oracle/_ref against the nlohmann json.hpp shipped
in this image, and tests/test_checkpoint.py compares bytes both ways.
"""
import json
import struct

import numpy as np

MAGIC = b"RXGS"
VERSION = 1  # kCheckpointVersion, checkpoint.hpp:14
MODALITY = ("rssi", "csi", "spectrum")  # sim::modality_name, channelsim.cpp:144-151
MODE = ("full", "global_only", "local_only", "additive_only", "no_occlusion")  # conditioning.cpp:180-189


def _mlp(prefix, p, o, d, nin, c4):
    """(name, shape, slice) of one Mlp's six tensors in the packed layout."""
    out = []
    for name, shape in (("w1", (d, nin)), ("b1", (d,)), ("w2", (d, d)), ("b2", (d,)), ("w3", (c4, d)), ("b3", (c4,))):
        n = int(np.prod(shape))
        out.append((f"{prefix}.{name}", shape, p[o:o + n]))
        o += n
    return out, o


def manifest(scene, cond):
    """manifest_for (checkpoint.cpp:31-89): [(name, shape, f64 array)]."""
    k = len(scene["tau_logits"])
    L = (scene["l_max"] + 1) ** 2
    arrays = [("positions", (k, 3), scene["positions"]), ("log_scales", (k, 3), scene["log_scales"]),
              ("quaternions", (k, 4), scene["quaternions"]), ("tau_logits", (k,), scene["tau_logits"]),
              ("fle_coeffs", (k, L, scene["channels"], 2), scene["fle_coeffs"])]
    if cond is not None:
        F, d, dc, S, R, nearest, mode, l_max, C = [int(v) for v in cond["cfg"]]
        p = np.asarray(cond["params"], np.float64)
        gin = 6 * F + 2 + dc
        arrays.append(("cond.fourier_freqs", (F, 3), p[:3 * F]))
        g, o = _mlp("cond.global", p, 3 * F, d, gin, 4 * C)
        arrays += g
        arrays.append(("cond.component_embed", (L, dc), p[o:o + L * dc]))
        loc, o = _mlp("cond.local", p, o + L * dc, d, 6, 4 * C)
        arrays += loc
        arrays.append(("cond.occupancy", (R, R, R), cond["occupancy"]))
    return [(n, s, np.ascontiguousarray(a, np.float64).reshape(-1)) for n, s, a in arrays]


def _num(v: float) -> str:
    """nlohmann::json's dump of a double: shortest round-trip digits d (k of
    them) with value d * 10^(n-k); "digits[000].0" when k <= n <= 15,
    "dig.its" when 0 < n <= 15, "0.[000]digits" when -4 < n <= 0, else
    "d.igitse+XX" (at least two exponent digits); NaN/inf -> null."""
    import math
    if not math.isfinite(v):
        return "null"
    if v == 0.0:
        return "-0.0" if math.copysign(1.0, v) < 0 else "0.0"
    sign = "-" if v < 0 else ""
    r = repr(abs(v))
    if "e" in r:
        m, e = r.split("e")
        e = int(e)
    else:
        m, e = r, 0
    if "." in m:
        ip, fp = m.split(".")
    else:
        ip, fp = m, ""
    digits = (ip + fp).lstrip("0")
    lead = len(ip + fp) - len((ip + fp).lstrip("0"))
    n = len(ip) + e - lead
    digits = digits.rstrip("0") or "0"
    k = len(digits)
    if k <= n <= 15:
        out = digits + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        out = digits[:n] + "." + digits[n:]
    elif -4 < n <= 0:
        out = "0." + "0" * (-n) + digits
    else:
        x = n - 1
        out = digits[0] + ("." + digits[1:] if k > 1 else "") + f"e{'-' if x < 0 else '+'}{abs(x):02d}"
    return sign + out


def dump_json(o) -> str:
    """nlohmann::ordered_json::dump() of the header (compact, insertion order)."""
    if isinstance(o, bool):
        return "true" if o else "false"
    if isinstance(o, int):
        return str(o)
    if isinstance(o, float):
        return _num(o)
    if isinstance(o, str):
        return json.dumps(o)
    if isinstance(o, dict):
        return "{" + ",".join(json.dumps(k) + ":" + dump_json(v) for k, v in o.items()) + "}"
    if isinstance(o, (list, tuple)):
        return "[" + ",".join(dump_json(v) for v in o) + "]"
    raise TypeError(type(o))


def write_checkpoint(path, scene, grid, cond=None, modality="spectrum"):
    """save_checkpoint (checkpoint.cpp:93-155).  grid: dict with n_theta,
    n_phi, tile_size, radius, theta_min, theta_max; cond: dict with cfg (9
    ints as rxgs_cond_create), params (packed), occupancy (R^3), lo, hi."""
    arrays = manifest(scene, cond)
    header = {"k": len(scene["tau_logits"]), "l_max": int(scene["l_max"]), "channels": int(scene["channels"]),
              "modality": modality,
              "grid": {"n_theta": int(grid["n_theta"]), "n_phi": int(grid["n_phi"]),
                       "tile_size": int(grid["tile_size"]), "radius": float(grid["radius"]),
                       "theta_min": float(grid["theta_min"]), "theta_max": float(grid["theta_max"])},
              "has_conditioning": cond is not None}
    if cond is not None:
        F, d, dc, S, R, nearest, mode, l_max, C = [int(v) for v in cond["cfg"]]
        header["conditioning"] = {"fourier_bands": F, "hidden": d, "embed_dim": dc, "probe_samples": S,
                                  "occupancy_resolution": R, "nearest_lookup": bool(nearest), "mode": MODE[mode],
                                  "occupancy_bounds": [float(v) for v in list(cond["lo"]) + list(cond["hi"])]}
    man, off = [], 0
    for name, shape, a in arrays:
        assert a.size == int(np.prod(shape)), name
        man.append({"name": name, "dtype": "f64", "shape": [int(s) for s in shape], "offset": off})
        off += a.size * 8
    header["arrays"] = man
    text = dump_json(header).encode()
    with open(path, "wb") as f:
        f.write(MAGIC + struct.pack("<IQ", VERSION, len(text)) + text)
        for _, _, a in arrays:
            f.write(a.astype("<f8").tobytes())


def read_checkpoint(path):
    """load_checkpoint's container parse (checkpoint.cpp:157-231): (header, {name: array})."""
    raw = open(path, "rb").read()
    if raw[:4] != MAGIC:
        raise IOError(f"load_checkpoint: bad magic in {path}")
    version, hlen = struct.unpack_from("<IQ", raw, 4)
    if version != VERSION:
        raise IOError(f"load_checkpoint: unsupported version {version}")
    header = json.loads(raw[16:16 + hlen])
    base = 16 + hlen
    out = {}
    for e in header["arrays"]:
        n = int(np.prod(e["shape"]))
        out[e["name"]] = np.frombuffer(raw, "<f8", n, base + e["offset"]).reshape(e["shape"])
    return header, out
