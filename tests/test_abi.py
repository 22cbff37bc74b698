"""C-ABI checks that need no GPU: the built library loads and exports every entry point that
include/lrcheb.h declares; context creation fails cleanly (status code + message) on a host without
a CUDA device."""
import ctypes
import os
import re

import pytest

from paper_2008_10275_b200 import lrcheb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "lrcheb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lrc_[a-z_]+)\s*\(", src)))


def test_header_declares_the_survey_entry_points():
    names = header_functions()
    for fn in ("lrc_create", "lrc_destroy", "lrc_last_error", "lrc_set_operator", "lrc_set_params",
               "lrc_solve", "lrc_apply_lowrank", "lrc_apply_dense", "lrc_truncate", "lrc_get_iterate"):
        assert fn in names


def test_library_exports_every_declared_symbol():
    lib = lrcheb.lib()
    missing = [n for n in header_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(header_functions()) == set(lrcheb.EXPORTS)


def test_version_string():
    assert "sm_100a" in lrcheb.version()


def test_create_without_gpu_fails_cleanly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("host has a GPU")
    lib = lrcheb.lib()
    h = ctypes.c_void_p()
    st = lib.lrc_create(ctypes.byref(h), 0, None)
    assert st == lrcheb.LRC_ERR_CUDA
    assert not h.value
    assert lib.lrc_last_error(None)        # a one-line message, no crash
    lib.lrc_destroy(None)                  # NULL-safe


def test_null_context_calls_return_arg_error():
    lib = lrcheb.lib()
    assert lib.lrc_set_params(None, 4, None, None, 0) == lrcheb.LRC_ERR_ARG
    assert lib.lrc_solve(None, None, 0, None, 0, 0, None, None, 0, None, 0, 0, None) == lrcheb.LRC_ERR_ARG
    assert lib.lrc_kernel_launches(None) == 0


def test_struct_layouts_match_header():
    # lrc_solve_opts: 3 doubles + 3 int64 + uint32 (padded to 8) ; info ends with chol2_cycles[3]
    assert ctypes.sizeof(lrcheb.SolveOpts) == 3 * 8 + 3 * 8 + 8
    names = [f[0] for f in lrcheb.SolveInfo._fields_]
    assert names[:3] == ["rank", "rel_residual", "b_norm"] and names[-1] == "chol2_cycles"
