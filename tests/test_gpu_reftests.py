"""The reference's OWN test suites for the render path, compiled unchanged
against the B200 drop-in (boundary item): proj/tests/
test_sphraster.cpp, test_sphraster_grad.cpp, test_conditioning.cpp and
test_radiance.cpp, linked with librxgs_refapi.so (the reference's
rxgs::raster / rxgs::cond / rxgs::fle functions implemented on
librxgs_b200.so) in place of the reference's sphraster.cpp /
conditioning.cpp / radiance.cpp, the reference's scene container
(scene.cpp) and the doctest shim (tests/cpp/doctest).  Built by
tests/cpp/Makefile where /root/reference exists; the binaries travel with
the snapshot (oracle/_ref/reftests)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "reftests")
SUITES = ["test_sphraster", "test_sphraster_grad", "test_conditioning", "test_radiance"]


def _bin(name):
    p = os.path.join(BIN, name)
    if not os.path.exists(p):
        pytest.skip(f"{p} not built (needs the reference sources at build time)")
    return p


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_links_the_drop_in(suite):
    """The path's functions are undefined in the test binary and resolve
    from librxgs_refapi.so -- the reference implementation is not linked."""
    p = _bin(suite)
    syms = subprocess.run(["nm", "-C", p], capture_output=True, text=True).stdout
    for fn in ("rxgs::raster::render_field", "rxgs::raster::build_tx_state", "rxgs::cond::condition_forward",
               "rxgs::fle::eval_basis", "rxgs::raster::bin_and_sort"):
        defined = [l for l in syms.splitlines() if fn + "(" in l and " U " not in l]
        assert not defined, f"{fn} is defined inside {suite}: {defined[:2]}"
    ldd = subprocess.run(["ldd", p], capture_output=True, text=True).stdout
    assert "librxgs_refapi.so" in ldd and "librxgs_b200.so" in ldd


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_passes_on_b200(suite):
    p = _bin(suite)
    out = subprocess.run([p], capture_output=True, text=True, timeout=900)
    log = out.stdout + out.stderr
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"reftest_{suite}.txt"), "w") as fh:
        fh.write(log)
    assert out.returncode == 0, log[-4000:]
    assert "0 failed" in out.stdout
