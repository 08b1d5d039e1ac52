"""bench.py host logic on CPU: the sharding mode of every BASELINE config at N = 1 / 8 and the
per-GPU slices, the algorithmic-byte model against a hand computation, and the
reference arm's JSON line (this tier's reference arm is the float64 oracle)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import synth  # noqa: E402


@pytest.mark.parametrize("name,world,slice_n,mode,scaling,batch", [
    ("c2", 1, 1, "none", "weak", 32),
    ("c2", 8, 1, "batch", "weak", 32),        # one full batch per rank
    ("c3", 4, 1, "batch", "weak", 16),
    ("c4", 8, 1, "batch", "strong", 16),      # 128 sequences split over 8 ranks
    ("c4", 1, 8, "batch-slice", "strong", 16),
    ("c5", 8, 1, "sequence", "strong", 4),    # every sequence block-cyclically sharded
    ("c5", 1, 8, "sequence-slice", "strong", 4),
])
def test_rank_config_modes(name, world, slice_n, mode, scaling, batch):
    cfg, m, sc = bench.rank_config(name, world, 0, 0, slice_n)
    assert (m, sc, cfg.batch) == (mode, scaling, batch)


def test_algorithmic_bytes_c2_by_hand():
    """C2: B 32, Hq = Hkv = 16, d 64, 4k context, S 16 (P 256), K = 512 / 16 = 32, bf16."""
    cfg = synth.config("c2")
    B, H, d, P, K, S, e = 32, 16, 64, 256, 32, 16, 2
    meta = B * H * P * 2 * d * e            # [m | M] record per (page, kv head)
    kv = B * H * K * S * 2 * d * e          # K and V rows of the selected pages
    q = B * H * d * e
    o = B * H * (d + 1) * 4                 # fp32 o + lse
    pt, ids = B * P * 4, B * H * K * 4
    ab = synth.algorithmic_bytes(cfg, [4096] * B)
    assert ab["total"] == meta + kv + q + o + pt + ids == 100960256


def test_algorithmic_bytes_fp8_rows():
    """FP8 KV (reading R21): a stored row is d codes + 1 exponent byte; metadata stays bf16."""
    cfg = synth.config("c2")
    bf, f8 = synth.algorithmic_bytes(cfg, [4096] * 32), synth.algorithmic_bytes(cfg, [4096] * 32, kv="fp8")
    sel_rows = 32 * 16 * 32 * 16 * 2
    assert bf["total"] - f8["total"] == sel_rows * (64 * 2 - 65)


def test_reference_arm_json_line():
    """`bench.py --impl reference` prints the contract's line for the oracle arm (CPU only)."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "3", "--warmup", "3", "--oracle-seconds", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    j = json.loads(out.stdout.strip().splitlines()[-1])
    assert j["impl"] == "reference" and j["metric"] == "decode steps/s" and j["unit"] == "steps/s"
    assert j["steps"] == 3 and j["warmup"] == 3 and j["n_gpus"] == 1 and j["value"] > 0
    assert j["cpu_baseline"]["kind"] == "oracle" and j["cpu_baseline"]["cores"] >= 1
    assert j["e2e"]["value"] == j["value"] and j["e2e"]["h2d_bytes_per_step"] == 0
    assert j["config"]["workload"].startswith("c2")
