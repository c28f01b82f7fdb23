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
    return sorted(set(re.findall(r"^(?:int|int64_t|const char\*)\s+(pp_\w+)\s*\(", text, flags=re.M)))


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


def test_new_entry_points_validate_before_device_work():
    """pp_plan_physical / pp_replica_* / pp_dot_bf16 reject bad shapes with the reference
    exception types, without touching (fake) device pointers."""
    lib = _lib.load()
    z = ctypes.c_void_p(8)
    cm, cfg = _lib.CostModel(), _lib.PlannerCfg()
    cm.top_k = 2
    cm.num_devices, cm.num_experts = 4, 16
    cfg.n = 0
    # E not a multiple of D
    rc = lib.pp_plan_physical(z, 1, 4, 4, 15, ctypes.byref(cm), ctypes.byref(cfg), 0, z, z, z, z, z, z, z, None)
    assert rc == _lib.PP_EINVAL
    # cost model dims disagree with the load
    cm.num_devices = 8
    rc = lib.pp_plan_physical(z, 1, 4, 4, 16, ctypes.byref(cm), ctypes.byref(cfg), 0, z, z, z, z, z, z, z, None)
    assert rc == _lib.PP_EDIM
    cm.num_devices = 4
    cfg.n = 4  # n must be < D
    rc = lib.pp_plan_physical(z, 1, 4, 4, 16, ctypes.byref(cm), ctypes.byref(cfg), 0, z, z, z, z, z, z, z, None)
    assert rc == _lib.PP_EINVAL
    cfg.n = 0
    rc = lib.pp_plan_physical(z, 1, 6, 4, 16, ctypes.byref(cm), ctypes.byref(cfg), 0, z, z, z, z, z, z, z, None)
    assert rc == _lib.PP_EINVAL  # rows not a multiple of D
    # replica kernels: rank out of range, bad parts
    assert lib.pp_replica_trans(z, z, z, 16, 4, 4, 8, 256, 256, 3, None, 0, None, None, 0, None) == _lib.PP_EINVAL
    assert lib.pp_replica_trans(z, z, z, 16, 4, 0, 8, 256, 256, 3, z, 0, None, None, 0, None) == _lib.PP_EINVAL
    assert lib.pp_replica_trans(z, z, z, 16, 4, 0, 8, 256, 256, 4, None, 0, None, None, 0, None) == _lib.PP_EINVAL
    # pp_grouped_gemm_ex: the gate serves FWD1/FWD2 and needs its epoch; the scatter FWD2/DGRAD1;
    # the adaptive reservation needs hi >= lo
    nores = (None, 0, 0, 0, 0)
    assert lib.pp_grouped_gemm_ex(0, z, z, z, z, z, z, 1, 128, 1, 256, 256, None, None, 0, z, None, 0, 2, 1,
                                  *nores, 0, None) == _lib.PP_EINVAL
    assert lib.pp_grouped_gemm_ex(2, z, z, z, z, z, z, 1, 128, 1, 256, 256, None, None, 0, z, z, 0, 2, 1,
                                  *nores, 0, None) == _lib.PP_EINVAL
    assert lib.pp_grouped_gemm_ex(0, z, z, z, z, z, z, 1, 128, 1, 256, 256, z, z, 4096, None, None, 0, 2, 1,
                                  *nores, 0, None) == _lib.PP_EINVAL
    assert lib.pp_grouped_gemm_ex(0, z, z, z, z, z, z, 1, 128, 1, 256, 256, None, None, 0, None, None, 0, 2, 1,
                                  z, 1, 2, 8, 4, 0, None) == _lib.PP_EINVAL
    # probe loss: n must be a multiple of 8, operands 16-byte aligned
    assert lib.pp_dot_bf16(z, z, 12, z, z, None) == _lib.PP_EINVAL
    assert lib.pp_dot_bf16(ctypes.c_void_p(24), z, 16, z, z, None) == _lib.PP_EINVAL
    assert b"aligned" in lib.pp_last_error()
