"""CPU checks of the C-ABI boundary: the in-tree library loads without a GPU and
exports every entry point include/cn_b200.h declares, and the ctypes table in
_lib.py binds exactly those names."""

import ctypes
import os
import re

from paper_2306_06946_b200 import _lib

INCLUDE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
HEADER = os.path.join(INCLUDE, "cn_b200.h")


def declared_symbols():
    """Every cnb_* function declared by include/*.h (the boundary cn_b200.h and the
    diagnostics header cn_b200_diag.h)."""
    names = set()
    for f in sorted(os.listdir(INCLUDE)):
        if f.endswith(".h"):
            text = re.sub(r"/\*.*?\*/", "", open(os.path.join(INCLUDE, f)).read(), flags=re.S)
            names.update(re.findall(r"\b(cnb_[a-z0-9_]+)\s*\(", text))
    return sorted(names)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_table_matches_header():
    assert sorted(_lib.exported_symbols()) == declared_symbols()


def test_status_codes_map_to_reference_exceptions():
    from paper_2306_06946_b200 import errors

    text = open(HEADER).read()
    codes = dict((k, int(v)) for k, v in re.findall(r"#define (CNB_E_[A-Z_]+) (\d+)", text))
    assert _lib.STATUS_ERRORS[codes["CNB_E_NOT_SPD"]] is errors.NotSPDError
    assert _lib.STATUS_ERRORS[codes["CNB_E_SINGULAR_BLOCK"]] is errors.SingularBlockError
    assert _lib.STATUS_ERRORS[codes["CNB_E_DIMENSION"]] is errors.DimensionMismatchError
    assert _lib.STATUS_ERRORS[codes["CNB_E_DEGENERATE_FRAME"]] is errors.DegenerateFrameError


def test_host_only_entry_points_run_without_gpu():
    assert _lib.lib().cnb_abi_version() == 2
    assert isinstance(_lib.lib().cnb_launch_count(), int)
    # argument validation happens before any device work
    rc = _lib.lib().cnb_pgs(4, None, 12, None, 0.01, 0.5, 1e-6, 0, None, None, None, None, None, None, None)
    assert rc == 6  # CNB_E_VALIDATION: max_iter < 1
