"""The C-ABI library loads without a GPU and exports every symbol include/ppmoe.h
declares; argument validation maps onto the reference exception types."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2411_10003_b200 import _lib
from paper_2411_10003_b200.core import DimensionMismatchError, ValidationError

HEADER = Path(__file__).resolve().parent.parent / "include" / "ppmoe.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(pp_\w+)\s*\(", text, flags=re.M)))


def test_header_symbols_exported():
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), f"{n} declared in ppmoe.h but not exported"
    assert set(names) == set(_lib.exported_symbols()), "ctypes signature table out of sync with the header"


def test_version_and_error_string():
    lib = _lib.load()
    assert lib.pp_version() == 1
    assert isinstance(lib.pp_last_error(), bytes)


def test_validation_before_any_device_work():
    lib = _lib.load()
    cm, cfg = _lib.CostModel(), _lib.PlannerCfg()
    cm.num_devices = cm.num_experts = 4
    cm.top_k = 1
    z = ctypes.c_void_p(8)  # never dereferenced: validation fails first
    cm.num_devices = 3
    rc = lib.pp_plan_greedy(z, 1, 4, ctypes.byref(cm), ctypes.byref(cfg), z, z, z, z, z, z, z, None)
    assert rc == _lib.PP_EDIM
    with pytest.raises(DimensionMismatchError):
        _lib.check(rc, "pp_plan_greedy")
    cm.num_devices = 4
    cfg.n = 4
    rc = lib.pp_plan_greedy(z, 1, 4, ctypes.byref(cm), ctypes.byref(cfg), z, z, z, z, z, z, z, None)
    assert rc == _lib.PP_EINVAL
    with pytest.raises(ValidationError):
        _lib.check(rc)
    rc = lib.pp_route_topk(z, z, None, 100, 256, 16, 2, z, z, z, z, z, None)  # T not multiple of 128
    assert rc == _lib.PP_EINVAL
    rc = lib.pp_grouped_gemm(99, z, z, z, z, z, z, 1, 128, 1, 256, 256, 0, None)
    assert rc == _lib.PP_EINVAL
    assert b"unknown mode" in lib.pp_last_error()
