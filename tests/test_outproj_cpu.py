"""Output side on the CPU: the oracle's gated_output / attention half of
block_forward (attnkit/zoo.py:125-152) pinned to golden vectors from the reference, the
tensor-parallel restatement (per-rank gate + W_o, summed in device order) against the
single-device form for every sharding the decode path uses, and the C-ABI
validation of K4 (no GPU needed)."""

import numpy as np
import pytest

from oracle import attnkit_port as ak

from golden_util import OUT_CASES, load, regen_outproj


@pytest.mark.parametrize("name", OUT_CASES)
def test_oracle_output_side_matches_reference(name):
    meta, arr = load(name)
    cfg, w, hidden, flat = regen_outproj(meta)
    assert ak.sha(hidden) == meta["sha_hidden"] and ak.sha(flat) == meta["sha_flat"]
    assert ak.sha(w["w_o"]) == meta["sha_w_o"] and ak.sha(w["w_g"]) == meta["sha_w_g"]
    np.testing.assert_allclose(ak.gated_output(hidden, flat, w["w_g"])[:, :16], arr["gated_head"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(ak.attention_block_output(hidden, flat, w["w_o"], w["w_g"]), arr["y_gated"],
                               rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(ak.attention_block_output(hidden, flat, w["w_o"]), arr["y_plain"], rtol=1e-12,
                               atol=1e-12)


@pytest.mark.parametrize("phi", [1, 2, 4])
@pytest.mark.parametrize("by", ["heads", "branches"])
def test_tp_output_side_is_the_device_order_sum(phi, by):
    """Head sharding (MLA / GQA / GLA) and branch sharding (MLRA-4: every device holds a partial
    of every head) both reduce to the single-device block output."""
    meta, arr = load("outproj_refdims")
    cfg, w, hidden, flat = regen_outproj(meta)
    h, d_h = cfg.h, cfg.d_h
    rng = np.random.default_rng(phi)
    if by == "heads":
        per = h // phi
        parts = [(list(range(r * per, (r + 1) * per)), flat[:, r * per * d_h:(r + 1) * per * d_h]) for r in range(phi)]
    else:  # contributions of every head, summing to flat
        pieces = [rng.standard_normal(flat.shape) for _ in range(phi - 1)]
        pieces.append(flat - sum(pieces) if pieces else flat)
        parts = [(list(range(h)), p) for p in pieces]
    got = ak.tp_attention_block_output(hidden, parts, w["w_o"], w["w_g"], d_h)
    np.testing.assert_allclose(got, arr["y_gated"], rtol=1e-10, atol=1e-10)


def test_outproj_c_abi_validation():
    from paper_2603_02188_b200 import _lib

    lib = _lib.load()
    assert lib.mlra_outproj_comm_bytes(16, 3072, 4) == 2 * 4 * 16 * 3072 * 4 + 2 * 4 * 24 * 8 * 4 + 16
    assert lib.mlra_outproj_comm_bytes(0, 3072, 4) == 0
    assert lib.mlra_outproj_workspace_bytes(16, 3072) == 16 * 3072 * 2
    rc = lib.mlra_outproj(None, None, None, None, None, 65, 768, 3072, 0, 1, None, None, None)
    assert rc == -1 and b"B=65" in lib.mlra_last_error()
    rc = lib.mlra_outproj(None, None, None, None, None, 16, 764, 3072, 0, 1, None, None, None)
    assert rc == -1 and b"multiples of 8" in lib.mlra_last_error()
    rc = lib.mlra_outproj(None, None, None, None, None, 16, 768, 3072, 2, 2, None, None, None)
    assert rc == -2 and b"rank 2 of 2" in lib.mlra_last_error()
    rc = lib.mlra_outproj(None, None, None, None, None, 16, 768, 3072, 0, 2, None, None, None)
    assert rc == -2 and b"communication regions" in lib.mlra_last_error()
    rc = lib.mlra_outproj(None, None, None, None, None, 16, 768, 3072, 0, 9, None, None, None)
    assert rc == -2 and b"world 9" in lib.mlra_last_error()
    rc = lib.mlra_outproj_sim(None, None, None, None, None, 16, 768, 3072, 2, None, None, None)
    assert rc == -2
    assert lib.mlra_ipc_handle(None, None) == -2
    assert lib.mlra_comm_alloc(0, None) == -2


def test_allreduce_c_abi_validation():
    from paper_2603_02188_b200 import _lib

    lib = _lib.load()
    n, world = 49152, 4
    assert lib.mlra_allreduce_comm_bytes(n, world) == 2 * world * n * 4 + 2 * world * 4096 * 4 + 16
    assert lib.mlra_allreduce(None, None, n, 0, 2, None, None) == -2
    assert lib.mlra_allreduce(None, None, n, 2, 2, None, None) == -2
    assert lib.mlra_allreduce_sim(None, None, n, 9, None, None) == -2


def test_decode_step_tp_c_abi_validation():
    from paper_2603_02188_b200 import _lib

    lib = _lib.load()
    args = [None] * 9 + [16, 24, 128, 1, 1, 128, 64, 128, 257, 4112, 9, 0.1, 0.5]
    rc = lib.mlra_decode_step_tp(*args, 2, 2, None, None)
    assert rc == -2 and b"rank 2 of 2" in lib.mlra_last_error()
    rc = lib.mlra_decode_step_tp(*args, 0, 9, None, None)
    assert rc == -2 and b"rank 0 of 9" in lib.mlra_last_error()
    rc = lib.mlra_decode_step_tp(*args, 0, 2, None, None)
    assert rc == -2 and b"communication regions" in lib.mlra_last_error()
