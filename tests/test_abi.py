"""The C-ABI library loads without a GPU and exports exactly what include/wssr.h declares."""

import ctypes
import os
import re

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "wssr.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(wssr_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_reference_entry_points():
    names = declared_functions()
    for must in ("wssr_assemble_f64", "wssr_qr_f64", "wssr_ssi_svd_f64", "wssr_step_f64",
                 "wssr_subspace_drift_f64", "wssr_ctx_create", "wssr_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    import __graft_entry__

    __graft_entry__.build()
    from paper_2512_05749_b200 import _lib

    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(declared_functions()) == set(_lib.SIGNATURES), "ctypes prototypes out of sync"
    assert lib.wssr_version() == 1


def test_no_device_fails_loudly():
    import torch
    import pytest

    from paper_2512_05749_b200 import _lib, errors

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(errors.DeviceError):
        _lib.context()
