"""HBM plan of the layer / stack (memory.py): the cfg5 stack (BASELINE configs[4]: 12 blocks,
64 experts, d=2048, f=4096, 8 GPUs, 32K tokens/GPU) fits a B200's 180 GB under the stack's
allocation rule, and the C library's gate-dW workspace size matches the plan."""

import pytest

from paper_2411_10003_b200 import _lib, memory

GB = 1e9


def cfg5(**kw):
    args = dict(num_blocks=12, d_model=2048, d_ff=4096, num_experts=64, top_k=2, tokens=32768, world=8)
    args.update(kw)
    return memory.stack_footprint(**args)


def test_cfg5_stack_fits_8_gpus():
    fp = cfg5(capacity_factor=2.0, max_replicas=16)
    assert fp["total_with_attention"] < 160 * GB, fp["total_with_attention"] / GB
    # the largest items are what the plan says they are
    by = fp["by_buffer"]
    assert by["pre"] == 12 * fp["rows_capacity"] * 4096 * 2
    assert by["dyp"] == fp["rows_capacity"] * 2048 * 2  # one shared copy, not 12
    assert by["agg_stage"] == 2 * 8 * 7 * 2 * 2048 * 4096 * 4  # two copies alternate by block parity


def test_round1_rule_did_not_fit():
    """Worst-case receive rows (D*T*k) and E-m replica slots in every block: > 180 GB."""
    fp = cfg5(capacity_factor=None, max_replicas=None)
    assert fp["total"] > 180 * GB


@pytest.mark.parametrize("T,d", [(16384, 1024), (32768, 2048), (8192, 2048), (1024, 256), (256, 512)])
def test_gate_workspace_matches_library(T, d):
    lib = _lib.load()
    assert lib.pp_gate_dw_workspace_bytes(T, d) == memory.gate_dw_splits(T, d) * d * 128 * 4


def test_rows_capacity_rule():
    assert memory.rows_capacity(16384, 2, 16, 1) == 16384 * 2 + 16 * 128
    assert memory.rows_capacity(4096, 2, 8, 4, capacity_factor=2.0) == 2 * 4096 * 2 + 8 * 128
    assert memory.rows_capacity(4096, 2, 8, 4, capacity_factor=10.0) == 4 * 4096 * 2 + 8 * 128  # capped
    with pytest.raises(ValueError):
        memory.rows_capacity(4096, 2, 8, 4, capacity_factor=0)
