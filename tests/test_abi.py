"""C-ABI boundary (include/nmq.h <-> libnmq.so <-> _lib.SIGNATURES), CPU only:
loading, exported symbols, and argument validation paths that return before
touching a GPU."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "nmq.h")


def header_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(nm_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2305_02678_b200 import _lib
    return _lib.load()


def test_header_declares_the_reference_entry_points():
    names = header_functions()
    for want in ("nm_material_create", "nm_material_destroy", "nm_fetch", "nm_eval", "nm_eval_z",
                 "nm_infer_proxy", "nm_sample", "nm_pdf", "nm_sample_pdf", "nm_query",
                 "nm_eval_multi", "nm_multi_workspace_bytes", "nm_last_error", "nm_version"):
        assert want in names


def test_library_exports_every_header_symbol(lib):
    for name in header_functions():
        assert hasattr(lib, name), f"libnmq.so does not export {name}"


def test_ctypes_table_matches_header():
    from paper_2305_02678_b200 import _lib
    assert set(header_functions()) == set(_lib.SIGNATURES)


def test_version_and_counters(lib):
    assert lib.nm_version() == 1
    assert lib.nm_launch_count() >= 0


def _desc(channels=8, width=16, height=16, n_levels=5):
    from paper_2305_02678_b200 import _lib
    d = _lib.MaterialDesc()
    d.channels = channels
    d.width, d.height, d.n_levels = width, height, n_levels
    return d


def test_create_rejects_wrong_channel_count(lib):
    from paper_2305_02678_b200 import _lib
    out = ctypes.c_void_p()
    rc = lib.nm_material_create(ctypes.byref(_desc(channels=4)), 0, ctypes.byref(out))
    assert rc == _lib.NM_ERR_UNSUPPORTED
    assert b"channels" in lib.nm_last_error()
    with pytest.raises(NotImplementedError):
        _lib.check(rc)


def test_create_rejects_corrupt_level_count(lib):
    from paper_2305_02678_b200 import _lib
    out = ctypes.c_void_p()
    rc = lib.nm_material_create(ctypes.byref(_desc(n_levels=3)), 0, ctypes.byref(out))
    assert rc == _lib.NM_ERR_INVALID
    assert b"pyramid" in lib.nm_last_error()  # latent.py:170-171 wording
    with pytest.raises(ValueError):
        _lib.check(rc)


def test_query_entry_points_validate_before_launch(lib):
    from paper_2305_02678_b200 import _lib
    assert lib.nm_eval(None, 10, None, None, 1, None, None, None, None, None, None, None) == _lib.NM_ERR_INVALID
    assert lib.nm_pdf(-1, None, None, None, None, None) == _lib.NM_ERR_INVALID
    assert lib.nm_pdf(0, None, None, None, None, None) == _lib.NM_OK  # empty batch is a no-op
    assert lib.nm_sample(5, None, None, None, None, None) == _lib.NM_ERR_INVALID
    assert lib.nm_set_kernel_path(7) == _lib.NM_ERR_INVALID
    assert lib.nm_set_kernel_path(0) == _lib.NM_OK


def test_multi_workspace_size(lib):
    assert lib.nm_multi_workspace_bytes(1000, 5) >= 1000 * 4
    assert lib.nm_multi_workspace_bytes(-1, 5) == 0


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2305_02678_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                for line in open(os.path.join(dirpath, f)):
                    assert not re.match(r"\s*(from|import)\s+oracle", line), (f, line)


def test_training_and_host_entry_points_validate_before_launch(lib):
    """The KL-loss heads, the host-buffer eval and the multi-material limits
    reject bad arguments with a status (no device work), like the query entry
    points; empty batches are no-ops."""
    from paper_2305_02678_b200 import _lib
    inv, ok = _lib.NM_ERR_INVALID, _lib.NM_OK
    assert lib.nm_kl_sample(-1, 1, 2, 0, *([None] * 9)) == inv
    assert lib.nm_kl_sample(0, 1, 2, 0, *([None] * 9)) == ok
    assert lib.nm_kl_sample(4, 1, 2, 0, *([None] * 9)) == inv
    assert lib.nm_kl_target(4, 3, *([None] * 6)) == inv
    assert lib.nm_kl_target_dir(4, 1, 2, *([None] * 6)) == inv
    assert lib.nm_kl_grad(4, 0, *([None] * 8)) == inv
    assert lib.nm_kl_grad(0, 0, *([None] * 8)) == ok
    assert lib.nm_eval_host(None, 10, None, None, 1, None, None, None, None, None, None, 0, None) == inv
    assert lib.nm_mlp_backward(None, 4, None, None, None, None, None) == inv
