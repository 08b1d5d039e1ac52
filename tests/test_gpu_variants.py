"""GPU parity of every instantiation of the fused step kernel.

The ring depth (4 / 8 stages), the CTA-partial merge (DSMEM in the cluster leader / L2
ticket) and the select structure (one- / two-level) are chosen by the host per
configuration; the development knobs that force each choice are read once per process, so
each variant re-runs the decode-step parity tests in a child process with the knob set.
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
    child_env = dict(os.environ, TS_VARIANT_CHILD="1", **env)
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"),
                        "-m", "gpu", "-q", "-x", "-p", "no:cacheprovider", "-k", CASES],
                       cwd=ROOT, env=child_env, capture_output=True, text=True, timeout=600)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and " failed" not in r.stdout, tail
