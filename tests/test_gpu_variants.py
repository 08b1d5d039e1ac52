"""GPU parity of every instantiation of the fused step kernel, and the TS_DEBUG error word.

The ring depth (4 / 8 stages), the CTA-partial merge (DSMEM in the cluster leader / L2
ticket) and the select structure (one- / two-level) are chosen by the host per
configuration; the development knobs that force each choice exist only in the dev build of
the library (libtinyserve_dev.so, -DTS_DEV_KNOBS), so each variant re-runs the decode-step
parity tests in a child process that loads the dev build (TS_DEV_LIB=1) with the knob set.
"""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = "test_decode_step and (c3_small or g4_s32 or g6_s64 or two_level or c1_ragged or g3_s16 or small_budget_long)"


@pytest.mark.skipif(os.environ.get("TS_VARIANT_CHILD") == "1", reason="child process")
@pytest.mark.parametrize("env", [
    {"TS_SC_R": "4"},                      # 4-stage ring everywhere (L2 ticket merge)
    {"TS_SC_R": "8", "TS_SC_DSM": "1"},    # 8-stage ring, DSMEM merge wherever C > 1
    {"TS_SC_R": "8", "TS_SC_DSM": "0"},    # 8-stage ring, L2 ticket merge
    {"TS_SC_TWO": "1", "TS_SC_R": "8"},    # two-level select forced (C >= 2)
    {"TS_TWO_KERNELS": "1"},               # score/select kernel -> attention kernel chain
])
def test_step_variant(env):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2509_12211_b200 import _build
    _build.build(dev=True)
    child_env = dict(os.environ, TS_VARIANT_CHILD="1", TS_DEV_LIB="1", **env)
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"),
                        "-m", "gpu", "-q", "-x", "-p", "no:cacheprovider", "-k", CASES],
                       cwd=ROOT, env=child_env, capture_output=True, text=True, timeout=600)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and " failed" not in r.stdout, tail


DEBUG_CHILD = r"""
import torch, synth, paper_2509_12211_b200 as ts
from paper_2509_12211_b200 import _lib
assert _lib.LIB_PATH.endswith("libtinyserve_dev.so")
word = _lib.lib().ts_debug_error_word
word.restype = ts._lib.ctypes.c_int32
word.argtypes = [ts._lib.ctypes.c_int32]
cfg = synth.config("c3", batch=2, ctx=600, budget_tokens=128)
c = {k: (v.cuda() if isinstance(v, torch.Tensor) else v) for k, v in synth.make_case(cfg, seed=3).items()}
L = ts.make_layout(c["q"], c["k_pool"], c["page_table"])
meta = ts.meta_build(L, c["k_pool"], c["page_table"], c["seq_lens"])
ts.decode_step(L, c["q"], c["k_pool"], c["v_pool"], meta, c["page_table"], c["seq_lens"], 128, 0.125)
assert word(1) == 0, "clean inputs raised a fault bit"
bad = c["page_table"].clone(); bad[1, 3] = L.num_blocks + 5      # page-table entry out of range
ts.decode_step(L, c["q"], c["k_pool"], c["v_pool"], meta, bad, c["seq_lens"], 1 << 20, 0.125)
assert word(1) & 2, "bad block not flagged"
sl = c["seq_lens"].clone(); sl[0] = L.max_pages * L.page_size + 40  # beyond the row's capacity
ts.decode_step(L, c["q"], c["k_pool"], c["v_pool"], meta, c["page_table"], sl, 128, 0.125)
assert word(1) & 1, "seq_len overflow not flagged"
print("debug word ok")
"""


@pytest.mark.skipif(os.environ.get("TS_VARIANT_CHILD") == "1", reason="child process")
def test_debug_error_word():
    """TS_DEBUG (dev build): a page-table entry >= num_blocks and a seq_len beyond the row's
    capacity raise their bits in the device error word; clean inputs raise none."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2509_12211_b200 import _build
    _build.build(dev=True)
    env = dict(os.environ, TS_VARIANT_CHILD="1", TS_DEV_LIB="1", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", DEBUG_CHILD], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0 and "debug word ok" in r.stdout, (r.stdout + r.stderr)[-3000:]
