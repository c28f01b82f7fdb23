"""ctypes binding of libppmoe.so (the C ABI declared in include/ppmoe.h).

Loading never needs a GPU; calling compute entry points does.  If the shared
library is missing the import of any compute path raises -- there is no
CPU fallback anywhere in the product.
"""

from __future__ import annotations

import ctypes
from ctypes import POINTER, c_double, c_int32, c_uint8, c_uint64, c_void_p, c_char_p
from pathlib import Path

from .core import DimensionMismatchError, ValidationError

LIB_PATH = Path(__file__).resolve().parent / "libppmoe.so"

PP_OK, PP_EINVAL, PP_EDIM, PP_ECUDA, PP_EPEER = 0, 1, 2, 3, 4

PP_GEMM_FWD1, PP_GEMM_FWD2, PP_GEMM_DGRAD2, PP_GEMM_DGRAD1 = 0, 1, 2, 3
PP_GEMM_WGRAD2, PP_GEMM_WGRAD1, PP_GEMM_PLAIN = 4, 5, 6
PP_CHUNK = 128
PP_ROW_ALIGN = 128


class CostModel(ctypes.Structure):
    _fields_ = [
        ("input_bytes", c_double),
        ("expert_param_bytes", c_double),
        ("expert_grad_bytes", c_double),
        ("avg_bandwidth", c_double),
        ("compute_throughput", c_double),
        ("fnec_time", c_double),
        ("bnec_time", c_double),
        ("num_devices", c_int32),
        ("num_experts", c_int32),
        ("top_k", c_int32),
        ("_pad", c_int32),
    ]


class PlannerCfg(ctypes.Structure):
    _fields_ = [("alpha", c_double), ("n", c_int32), ("overlap_aware", c_int32), ("reuse_interval", c_int32),
                ("max_replicas", c_int32), ("slots_per_rank", c_int32), ("_pad", c_int32), ("iter_counter", c_void_p)]


class Group(ctypes.Structure):
    _fields_ = [
        ("row_off", c_int32),
        ("rows", c_int32),
        ("rows_pad", c_int32),
        ("wslot", c_int32),
        ("expert", c_int32),
        ("src_rank", c_int32),
        ("_pad", c_int32 * 2),
    ]


PP_DOT_PARTIALS = 592  # include/ppmoe.h
P = c_void_p  # every device pointer crosses the boundary as a plain address
I = c_int32

# name -> argtypes (restype is always int unless noted)
SIGNATURES = {
    "pp_version": [],
    "pp_plan_greedy": [P, I, I, POINTER(CostModel), POINTER(PlannerCfg), P, P, P, P, P, P, P, P],
    "pp_plan_physical": [P, I, I, I, I, POINTER(CostModel), POINTER(PlannerCfg), I, P, P, P, P, P, P, P, P],
    "pp_derive_loads": [P, P, I, I, P, P, P],
    "pp_top_m_mask": [P, I, I, I, P, P, P],
    "pp_route_topk": [P, P, P, I, I, I, I, P, P, P, P, P, P],
    "pp_slot_histogram": [P, I, I, I, P, I, I, P],
    "pp_dispatch_layout": [P, P, P, I, I, I, I, I, I, I, I, P, P, P, P, P, P, P, I, P, P, P],
    "pp_dispatch": [P, P, P, P, P, I, I, I, I, I, P, P, P, P, I, P, P, P, I, P],
    "pp_combine": [P, P, P, P, I, I, I, P, P, P],
    "pp_combine_bwd": [P, P, P, P, P, P, P, P, P, I, I, I, I, P, P, P, P, I, I, P, P],
    "pp_gate_dx": [P, P, I, I, I, I, P, P],
    "pp_dispatch_bwd": [P, P, P, P, I, I, I, P, P],
    "pp_gate_dw": [P, P, I, I, I, I, P, P, P],
    "pp_gate_dw_workspace_bytes": [I, I],
    "pp_grouped_gemm": [I, P, P, P, P, P, P, I, I, I, I, I, I, P],
    "pp_grouped_gemm_ex": [I, P, P, P, P, P, P, I, I, I, I, I, P, P, I, P, P, I, I, I, P, I, I, I, I, I, P],
    "pp_replica_trans": [P, P, P, I, I, I, I, I, I, I, P, I, P, P, I, P],
    "pp_replica_agg": [P, P, P, P, I, I, I, I, I, I, I, I, P],
    "pp_dot_bf16": [P, P, ctypes.c_int64, P, P, P],
    "pp_replica_agg_reduce": [P, P, P, P, I, I, I, I, I, I, I, P],
    "pp_copy_batch": [P, P, P, I, P],
    "pp_agg_accumulate": [P, P, P, P, I, I, I, P],
    "pp_device_alloc": [c_uint64, POINTER(c_void_p)],
    "pp_device_free": [P],
    "pp_ipc_export": [P, POINTER(c_uint8)],
    "pp_ipc_import": [POINTER(c_uint8), POINTER(c_void_p)],
    "pp_ipc_close": [P],
    "pp_peer_barrier": [P, I, I, c_uint64, P],
}

RESTYPE_I64 = {"pp_gate_dw_workspace_bytes"}

_lib = None


def load():
    """Load (once) and type the shared library.  Raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2411_10003_b200.build` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(str(LIB_PATH))
    lib.pp_last_error.restype = c_char_p
    lib.pp_last_error.argtypes = []
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = ctypes.c_int64 if name in RESTYPE_I64 else c_int32
    _lib = lib
    return lib


def exported_symbols() -> list:
    return ["pp_last_error", *SIGNATURES.keys()]


def check(rc: int, what: str = "") -> None:
    """Map a C return code onto the reference's exception types."""
    if rc == PP_OK:
        return
    msg = (load().pp_last_error() or b"").decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if rc == PP_EINVAL:
        raise ValidationError(msg)
    if rc == PP_EDIM:
        raise DimensionMismatchError(msg)
    raise RuntimeError(msg)


# kernels each entry point launches (for the bench's gpu_launches claim)
KERNELS_PER_CALL = {
    "pp_plan_greedy": 1, "pp_plan_physical": 1, "pp_derive_loads": 1, "pp_top_m_mask": 1, "pp_route_topk": 1, "pp_slot_histogram": 1,
    "pp_dispatch_layout": 1, "pp_dispatch": 1, "pp_combine": 1, "pp_combine_bwd": 1,
    "pp_gate_dx": 1, "pp_dispatch_bwd": 1, "pp_gate_dw": 2, "pp_grouped_gemm": 1, "pp_grouped_gemm_ex": 1, "pp_replica_trans": 1,
    "pp_replica_agg": 1, "pp_replica_agg_reduce": 1, "pp_dot_bf16": 2, "pp_peer_barrier": 1, "pp_agg_accumulate": 1,
}
_launches = [0]


def reset_launch_count() -> None:
    _launches[0] = 0


def launch_count() -> int:
    return _launches[0]


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
    _launches[0] += KERNELS_PER_CALL.get(name, 0)
