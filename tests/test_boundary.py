"""CPU-side checks of the C-ABI boundary (no compute calls: no GPU here).

* libtinyserve.so builds for sm_100a, loads, and exports every symbol include/tinyserve.h
  declares; the binary carries sm_100a SASS with the expected instruction classes.
* host-only entry points (status strings, workspace sizes) and host-side validation
  (errors returned before any launch).
* the product package never imports the oracle, and has no CPU fallback.
"""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tinyserve.h")
PKG = os.path.join(ROOT, "paper_2509_12211_b200")


@pytest.fixture(scope="module")
def ts():
    from paper_2509_12211_b200 import _build
    _build.build()
    import paper_2509_12211_b200 as ts
    return ts


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ts_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(ts):
    declared = _declared()
    assert len(declared) >= 10
    lib = ctypes.CDLL(ts._lib.LIB_PATH)
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared) == set(ts._lib.SYMBOLS)


def test_binary_is_sm100a_with_tma_and_tensor_core_sass(ts):
    out = subprocess.run(["cuobjdump", "-sass", ts._lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    sass = out.stdout
    assert "sm_100a" in sass
    assert "UTMALDG" in sass          # TMA tile loads (cp.async.bulk.tensor)
    assert "HMMA" in sass             # tensor-core mma
    assert "SYNCS" in sass            # mbarrier transactions


def test_host_only_entry_points(ts):
    L = ts._lib.lib()
    assert L.ts_version().decode().startswith("tinyserve")
    for code in range(7):
        assert L.ts_status_str(code)
    lay = ts.Layout(32, 16, 16, 64, 16, 256, 8192, 1, 0, ts.TS_BF16)
    ws = ts.workspace_bytes(lay, 512)
    aws = ts.attn_workspace_bytes(lay, 32)
    assert ws > aws > 0
    bad = ts.Layout(32, 16, 16, 64, 0, 256, 8192, 1, 0, ts.TS_BF16)
    assert ts.workspace_bytes(bad, 512) == 0


@pytest.mark.parametrize("field,value,status", [
    ("page_size", 0, 1), ("head_dim", 0, 1), ("kv_dtype", 7, 1), ("num_q_heads", 15, 2),
    ("shard_offset", 3, 2), ("head_dim", 96, 4),
    ("max_pages", (1 << 22) + 1, 4)])  # > 2^26 tokens per row (32-bit tile arithmetic)
def test_validation_errors_before_launch(ts, field, value, status):
    lay = ts.Layout(2, 16, 4, 64, 16, 8, 16, 2, 1, ts.TS_BF16)
    setattr(lay, field, value)
    L = ts._lib.lib()
    rc = L.ts_decode_step(lay, None, None, None, None, None, None, 64, 1.0, None, None, None,
                          None, None, 0, None)
    assert rc == status
    rc = L.ts_score_pages(lay, None, None, None, None, None, None)
    assert rc == status


def test_alignment_and_workspace_errors(ts):
    L = ts._lib.lib()
    lay = ts.Layout(2, 16, 4, 64, 16, 8, 16, 1, 0, ts.TS_BF16)
    odd = 0x1008  # 8-byte aligned, not 16
    good = 0x2000
    assert L.ts_score_pages(lay, odd, good, good, good, good, None) == 3
    assert L.ts_decode_step(lay, good, good, good, good, good, good, 64, 1.0, good, good, None,
                            None, None, 0, None) == 6   # no workspace
    assert L.ts_decode_step(lay, good, good, good, good, good, good, 0, 1.0, good, good, None,
                            None, good, 1 << 30, None) == 1  # budget < 1
    lay.shard_stride = 2
    assert L.ts_decode_step(lay, good, good, good, good, good, good, 64, 1.0, good, good, None,
                            None, good, 1 << 30, None) == 4  # sharded step is composed, not fused
    assert L.ts_select_topk(good, 4, 16, None, None, 1, 0, 0, good, None, good, None) == 2
    assert L.ts_lse_merge(0, 4, 64, good, good, 0, good, good, None) == 1


def test_product_never_imports_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", src, re.M), f
                assert "tinyserve_oracle" not in src and "libtsoracle" not in src, f


def test_no_cpu_fallback(ts):
    import torch
    q = torch.zeros(1, 1, 64, dtype=torch.bfloat16)
    with pytest.raises(TypeError, match="CUDA"):
        ts.score_pages(ts.Layout(1, 1, 1, 64, 16, 4, 4, 1, 0, ts.TS_BF16), q, q, q, q)


def test_round2_entry_points_validate_before_launch(ts):
    """FP8 KV (R21), the fused sequence-sharding halves and the release / dev split."""
    L = ts._lib.lib()
    good = 0x2000
    f8 = ts.Layout(2, 16, 4, 64, 16, 8, 16, 1, 0, ts.TS_FP8E4M3)
    assert L.ts_pool_bytes(f8) == 16 * 4 * 16 * 65                 # codes + one exponent byte per row
    bf = ts.Layout(2, 16, 4, 64, 16, 8, 16, 1, 0, ts.TS_BF16)
    assert L.ts_pool_bytes(bf) == 16 * 4 * 16 * 64 * 2
    f8.head_dim = 128
    assert L.ts_pool_bytes(f8) == 0                               # FP8: head_dim 64 only
    assert L.ts_kv_quantize(-1, 64, good, good, None) == 1    # rows < 0
    assert L.ts_kv_quantize(16, 128, good, good, None) == 4   # head_dim 128 unsupported
    assert L.ts_kv_quantize(8, 64, good, good, None) == 2     # not whole 16-row sub-page records
    assert L.ts_kv_quantize(16, 64, 0x1008, good, None) == 3  # src not 16-byte aligned
    f8s = ts.Layout(2, 16, 4, 64, 8, 8, 16, 1, 0, ts.TS_FP8E4M3)
    assert L.ts_pool_bytes(f8s) == 0                          # FP8 needs page_size % 16 == 0
    sh = ts.Layout(2, 16, 4, 64, 16, 8, 16, 2, 1, ts.TS_BF16)
    assert L.ts_select_candidates(sh, good, good, good, good, 0, good, good, good, None) == 2  # k < 1
    assert L.ts_shard_attend(sh, good, good, good, good, good, good, good, 0, 0, 64, 1.0, good, good,
                             None, None, good, 1 << 30, None) == 2                            # parts < 1
    assert L.ts_shard_attend(sh, good, good, good, good, good, good, good, 2, 0, 64, 1.0, good, good,
                             None, None, None, 0, None) == 6                                  # no workspace
    f32 = ts.Layout(2, 16, 4, 64, 16, 8, 16, 2, 1, ts.TS_F32)
    assert L.ts_select_candidates(f32, good, good, good, good, 8, good, good, good, None) == 4


def test_release_library_has_no_dev_hooks(ts):
    """The A/B knobs and timestamp / debug hooks exist only in libtinyserve_dev.so."""
    lib = ctypes.CDLL(ts._lib.LIB_PATH)
    for sym in ("ts_debug_timestamps", "ts_debug_ss_timestamps", "ts_debug_error_word"):
        assert not hasattr(lib, sym), sym
    raw = open(ts._lib.LIB_PATH, "rb").read()
    assert b"TS_SC_R" not in raw and b"TS_TWO_KERNELS" not in raw  # no getenv of a knob
