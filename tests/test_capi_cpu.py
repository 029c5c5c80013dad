"""CPU checks of the C ABI library: it loads without a GPU and exports every
symbol include/moba_b200.h declares (no compute calls here)."""
import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "moba_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(moba_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_path():
    fns = declared_functions()
    for name in ("moba_centroids", "moba_route", "moba_varlen", "moba_validate_plan", "moba_fwd", "moba_bwd",
                 "moba_conv_bwd", "moba_plan_row_pos"):
        assert name in fns


def test_library_exports_every_declared_symbol():
    from paper_2511_11571_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.fail("libmoba_b200.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # every declared symbol is typed by the binding, and nothing extra
    assert set(_lib.SIGNATURES) == set(declared_functions())


def test_status_strings_and_version():
    from paper_2511_11571_b200 import _lib
    lib = _lib.load()
    assert b"sm_100a" in lib.moba_version()
    assert lib.moba_status_string(0) == b"ok"
    assert b"plan" in lib.moba_status_string(3)


def test_workspace_queries_without_gpu():
    from paper_2511_11571_b200 import _lib
    lib = _lib.load()
    assert lib.moba_route_workspace_size(16, 8192, 128, 8) > 0
    assert lib.moba_fwd_workspace_size(16, 8192, 64, 128, 9) > 16 * 8192 * 9 * 64 * 2
    assert lib.moba_bwd_workspace_size(16, 8192, 64, 128, 9, 0) >= 16 * 8192 * 64 * 4
    assert lib.moba_bwd_workspace_size(16, 8192, 64, 128, 9, 1) > lib.moba_bwd_workspace_size(16, 8192, 64, 128, 9, 0)


def test_status_maps_to_reference_exceptions():
    import paper_2511_11571_b200 as mb
    from paper_2511_11571_b200 import _lib
    for code, exc in ((1, mb.ShapeError), (2, mb.ConfigError), (3, mb.PlanValidationError),
                      (5, mb.ConfigError), (4, mb.MobaError)):
        with pytest.raises(exc):
            _lib.check(code, "probe")
    _lib.check(0, "ok")


def test_kernels_are_sm100a():
    """The shared object carries sm_100a SASS only (cuobjdump --list-elf)."""
    import shutil
    import subprocess
    from paper_2511_11571_b200 import _lib
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
