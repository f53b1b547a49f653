"""C-ABI library: loads, exports every symbol include/*.h declares, validates on the host.

CPU-only: nothing here launches a kernel.
"""

import glob
import os
import re

import pytest

from paper_2505_13813_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        names |= set(re.findall(r"GRKAN_API\s+[\w\s\*]+?\b(grkan_\w+)\s*\(", src))
    return names


def test_header_declares_the_boundary():
    assert declared_symbols() == set(N.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    for sym in declared_symbols():
        assert hasattr(lib, sym), sym
    out = os.popen("nm -D --defined-only %s" % N.LIB_PATH).read()
    for sym in declared_symbols():
        assert re.search(r"\bT %s\b" % sym, out), sym


def test_library_built_for_sm100a():
    out = os.popen("cuobjdump --list-elf %s 2>&1" % N.LIB_PATH).read()
    assert "sm_100a" in out, out


def test_version_and_status_strings():
    assert "sm_100a" in N.version()
    assert N.status_string(N.OK) == "ok"
    assert N.status_string(N.ERR_LAYOUT) == "layout mismatch"
    assert N.status_string(N.ERR_ACCUM_OVERFLOW) == "accumulation overflow"


def test_host_validation_without_gpu():
    L = N.lib()
    # layout mismatch: d not divisible by groups (GroupLayout, rational.py:41-45)
    rc = L.grkan_fwd(None, None, None, None, 4, 10, 4, 6, 4, N.DT_F32, 0, None, None)
    assert rc == N.ERR_LAYOUT and "not divisible" in N.last_error()
    rc = L.grkan_fwd(None, None, None, None, 4, 0, 1, 6, 4, N.DT_F32, 0, None, None)
    assert rc == N.ERR_LAYOUT
    rc = L.grkan_fwd(None, None, None, None, 4, 8, 2, 6, 4, 9, 0, None, None)
    assert rc == N.ERR_UNSUPPORTED
    rc = L.grkan_fwd(None, None, None, None, 4, 8, 2, 13, 4, N.DT_F32, 0, None, None)
    assert rc == N.ERR_UNSUPPORTED
    rc = L.grkan_fwd(None, None, None, None, 4, 8, 2, 0, 4, N.DT_F32, 0, None, None)
    assert rc == N.ERR_INVALID
    rc = L.grkan_fwd(None, None, None, None, -1, 8, 2, 6, 4, N.DT_F32, 0, None, None)
    assert rc == N.ERR_GRID
    rc = L.grkan_fwd(None, None, None, None, 4, 8, 2, 6, 4, N.DT_F32, 0x10, None, None)
    assert rc == N.ERR_INVALID
    rc = L.grkan_fwd(None, None, None, None, 4, 8, 2, 6, 4, N.DT_F32, N.FLAG_CHECK_FINITE, None, None)
    assert rc == N.ERR_INVALID  # checked mode needs a status block
    rc = L.grkan_bwd(None, None, None, None, None, None, None, None, 0, 4, 8, 2, 6, 4, N.DT_F32, 0, None)
    assert rc == N.ERR_INVALID
    assert L.grkan_bwd_workspace_bytes(4, 10, 4, 6, 4, N.DT_F32) == 0


@pytest.mark.parametrize("dtype,es", [(N.DT_F32, 4), (N.DT_BF16, 2), (N.DT_F64, 8)])
def test_plan_geometry(dtype, es):
    for rows, d, g in [(256 * 197, 3072, 8), (128 * 197, 1536, 8), (8 * 197, 192, 8), (9, 8, 2),
                       (5 * 7, 12, 4), (2 * 9, 3072, 1), (10, 64, 64)]:
        p = N.plan(rows, d, g, 6, 4, dtype)
        dg = d // g
        w = p["vector_width"]
        assert w in (1, 16 // es)
        if (dg * es) % 16 == 0:
            assert w == 16 // es
            assert p["staged"] == (dg // w <= 768)
        else:
            assert not p["staged"]
        assert dg % w == 0
        if p["staged"]:
            assert p["threads"] == 288
            rs = p["rows_per_unit"]
            assert rs == 768 // (dg // w)
            stage_units = -(-rows // rs)
            pg = p["ctas"] // g  # persistent CTAs per group
            assert p["ctas"] == pg * g and 1 <= pg <= stage_units
            assert p["ctas"] <= 2 * 148 or pg == 1
            # one partial per consumer warp
            assert p["partials_per_group"] == pg * 8
        else:
            assert p["ctas"] == p["partials_per_group"] * g
            assert p["threads"] == 256
            R = p["rows_per_unit"]
            assert p["partials_per_group"] * R >= rows > (p["partials_per_group"] - 1) * R
        ws = N.lib().grkan_bwd_workspace_bytes(rows, d, g, 6, 4, dtype)
        acc = 8 if dtype == N.DT_F64 else 4
        assert ws >= 256 + p["ctas"] * 10 * acc
        # the staged kernels are compiled for degrees (5, 4) and (3, 2) only
        assert N.plan(rows, d, g, 4, 2, dtype)["staged"] == p["staged"]
        assert not N.plan(rows, d, g, 5, 3, dtype)["staged"]


def test_kat_b_plan_is_persistent_and_balanced():
    p = N.plan(256 * 197, 3072, 8, 6, 4, N.DT_F32)
    assert p["vector_width"] == 4 and p["staged"] and p["threads"] == 288
    assert p["rows_per_unit"] == 8  # 8 rows x 96 float4 = 768 vectors per stage
    assert p["ctas"] == 8 * (2 * 148 // 8)  # one persistent CTA per resident slot


def test_deterministic_and_fused_entry_points_validate_on_the_host():
    L = N.lib()
    # global row block: a whole number of 768-vector stages, >= 128 rows
    assert L.grkan_det_block_rows(3072, 8, N.DT_F32) == 128   # V = 96 -> 8-row stages
    assert L.grkan_det_block_rows(3072, 8, N.DT_BF16) == 128  # V = 48 -> 16-row stages
    assert L.grkan_det_block_rows(192, 8, N.DT_F32) == 128    # V = 6 -> 128-row stages
    assert L.grkan_det_block_rows(3072, 1, N.DT_F32) == 128   # V = 768 -> 1-row stages
    assert L.grkan_det_block_rows(10, 4, N.DT_F32) == 0       # layout mismatch
    assert L.grkan_det_partials_bytes(50432, 3072, 8, 6, 4, N.DT_F32) == 394 * 8 * 10 * 4
    assert L.grkan_det_partials_bytes(129, 3072, 8, 6, 4, N.DT_F64) == 2 * 8 * 10 * 8
    # partials: short buffer and null pointers are host errors
    rc = L.grkan_bwd_partials(None, None, None, None, None, None, 0, 4, 8, 2, 6, 4, N.DT_F32, 0, None, None)
    assert rc == N.ERR_INVALID and "too small" in N.last_error()
    rc = L.grkan_reduce_partials(None, -1, 2, 6, 4, None, None, N.DT_F32, None, None)
    assert rc == N.ERR_GRID
    rc = L.grkan_reduce_partials(None, 3, 2, 6, 4, None, None, N.DT_F32, None, None)
    assert rc == N.ERR_INVALID
    # fused layer backward: shape contract checked before any CUDA call
    assert L.grkan_linear_bwd_workspace_bytes(50432, 3072, 768, 8) > 256
    assert L.grkan_linear_bwd_workspace_bytes(100, 80, 64, 2) == 0    # group width 40
    rc = L.grkan_linear_bwd(None, None, None, None, None, None, None, None, None, 0, 128, 80, 64, 2, 0, None)
    assert rc == N.ERR_UNSUPPORTED and "group width" in N.last_error()
    rc = L.grkan_linear_bwd(None, None, None, None, None, None, None, None, None, 0, 128, 256, 100, 2, 0, None)
    assert rc == N.ERR_UNSUPPORTED  # K % 64
    rc = L.grkan_linear_bwd(None, None, None, None, None, None, None, None, None, 0, 128, 255, 64, 2, 0, None)
    assert rc == N.ERR_LAYOUT
    rc = L.grkan_linear_bwd(None, None, None, None, None, None, None, None, None, 0, 128, 256, 64, 2,
                            N.FLAG_EXACT, None)
    assert rc == N.ERR_UNSUPPORTED  # FAST policy only
    rc = L.grkan_linear_bwd(None, None, None, None, None, None, None, None, None, 0, 128, 256, 64, 2, 0, None)
    assert rc == N.ERR_INVALID  # null pointers


