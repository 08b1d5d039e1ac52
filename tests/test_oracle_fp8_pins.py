"""Pins for the oracle's FP8 KV storage (reading R21; SURVEY.md §8f NEXT-3,
"FP16/INT8 KV formats" PAPER.md:94), CPU only.

Each function is pinned to something other than itself:
  * or_e4m3_value / or_e4m3_round — torch's CPU float32 -> float8_e4m3fn conversion (an
    independent library routine) on every bf16 magnitude in range, plus the format's
    closed-form anchors (1.0 = 0x38, 448 = 0x7e, 2^-9 = 0x01, 2^-6 = 0x08);
  * or_kv_exponent — its defining inequality (amax <= 448 * 2^e and not for e - 1) on
    random magnitudes, and the clamp ends;
  * or_kv_quantize / or_kv_dequantize — round-trip error within half an E4M3 ulp, exact
    bf16 representability of every dequantised value (what keeps Eq. 1 exact), and a
    hand-computed row.
"""
import math

import numpy as np
import pytest
import torch


def test_e4m3_closed_forms(orc):
    assert orc.e4m3_value(0x38) == 1.0
    assert orc.e4m3_value(0x7E) == 448.0
    assert orc.e4m3_value(0x01) == 2.0 ** -9
    assert orc.e4m3_value(0x08) == 2.0 ** -6
    assert orc.e4m3_value(0x07) == 7 * 2.0 ** -9
    assert orc.e4m3_value(0xB8) == -1.0
    assert math.isnan(orc.e4m3_value(0x7F)) and math.isnan(orc.e4m3_value(0xFF))
    # ties to even: 1.0625 is halfway between 1.0 (m=0) and 1.125 (m=1)
    assert orc.e4m3_round(1.0625) == 0x38
    assert orc.e4m3_round(1.1875) == 0x3A   # halfway 1.125 / 1.25 -> m = 2
    assert orc.e4m3_round(1e6) == 0x7E and orc.e4m3_round(-1e6) == 0xFE  # saturate
    assert orc.e4m3_round(-0.0) == 0x80 and orc.e4m3_round(2.0 ** -11) == 0x00


def test_e4m3_decode_matches_torch(orc):
    codes = torch.arange(256, dtype=torch.int32).to(torch.uint8)
    ref = codes.view(torch.float8_e4m3fn).to(torch.float64).numpy()
    mine = np.array([orc.e4m3_value(c) for c in range(256)])
    fin = np.isfinite(ref)
    assert np.array_equal(np.isnan(mine), np.isnan(ref))
    assert np.array_equal(mine[fin], ref[fin])


def test_e4m3_round_matches_torch_on_every_bf16(orc):
    """Every finite bf16 bit pattern with |x| <= 448 (x * 2^-e is such a value)."""
    bits = torch.arange(0, 1 << 16, dtype=torch.int32).to(torch.int16)
    x = bits.view(torch.bfloat16).to(torch.float32)
    x = x[torch.isfinite(x) & (x.abs() <= 448)]
    ref = x.to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    mine = np.array([orc.e4m3_round(float(v)) for v in x.tolist()], np.uint8)
    assert np.array_equal(mine, ref)


def test_e4m3_round_equals_brute_force_nearest(orc):
    """The bisection equals the plain definition: the nearest of all 127 finite magnitudes,
    ties to the even code."""
    vals = [orc.e4m3_value(c) for c in range(127)]
    rng = np.random.default_rng(3)
    xs = np.concatenate([rng.uniform(0, 470, 3000), rng.uniform(0, 2.0 ** -5, 2000),
                         np.array(vals), (np.array(vals[:-1]) + np.array(vals[1:])) / 2])
    for x in xs:
        d = [abs(v - x) for v in vals]
        m = min(d)
        best = min(c for c in range(127) if d[c] == m and (c % 2 == 0 or d.count(m) == 1)) \
            if x < 448 else 126
        assert orc.e4m3_round(float(x)) == best, x
        assert orc.e4m3_round(float(-x)) == best | 0x80, x


def test_e4m3_round_matches_torch_on_random_doubles(orc):
    rng = np.random.default_rng(7)
    x = np.concatenate([rng.normal(0, 30, 4000), rng.uniform(-448, 448, 4000),
                        rng.normal(0, 2.0 ** -8, 2000)]).astype(np.float32)
    ref = torch.from_numpy(x).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    mine = np.array([orc.e4m3_round(float(v)) for v in x], np.uint8)
    assert np.array_equal(mine, ref)


def test_kv_exponent_definition(orc):
    rng = np.random.default_rng(11)
    for a in np.concatenate([np.exp(rng.uniform(-40, 45, 3000)), [448.0, 449.0, 224.0, 1.0]]):
        e = orc.kv_exponent(float(a))
        if -64 < e < 64:
            assert a <= 448.0 * 2.0 ** e and a > 448.0 * 2.0 ** (e - 1), (a, e)
    assert orc.kv_exponent(448.0) == 0 and orc.kv_exponent(448.0 * (1 + 2 ** -20)) == 1
    assert orc.kv_exponent(0.0) == -64 and orc.kv_exponent(1e-40) == -64
    assert orc.kv_exponent(1e30) == 64


def test_kv_quantize_hand_row(orc):
    # amax 3.0 -> e = -7 (3 <= 448/128 = 3.5, 3 > 1.75); x * 2^7: 384, -96, 0.5, 0.7 * 128
    x = torch.tensor([[3.0, -0.75, 2.0 ** -8, 0.7]], dtype=torch.bfloat16)
    codes, exps = orc.kv_quantize(x)
    assert exps.tolist() == [-7]
    xs = x.to(torch.float64).numpy()[0] * 128
    assert [orc.e4m3_value(c) for c in codes[0]] == [384.0, -96.0, 0.5, orc.e4m3_value(orc.e4m3_round(xs[3]))]
    assert orc.e4m3_value(codes[0][3]) == 88.0  # 0.69921875 * 128 = 89.5 -> nearest E4M3 is 88


@pytest.mark.parametrize("scale", [1.0, 1e-3, 40.0])
def test_kv_round_trip_bounds_and_bf16_exactness(orc, scale):
    g = torch.Generator().manual_seed(5)
    x = (torch.randn(512, 64, generator=g) * scale).to(torch.bfloat16)
    codes, exps = orc.kv_quantize(x)
    deq = orc.kv_dequantize(codes, exps).astype(np.float64)
    xd = x.to(torch.float64).numpy()
    amax = np.abs(xd).max(axis=1)
    for r in range(x.shape[0]):
        e = int(exps[r])
        assert amax[r] <= 448 * 2.0 ** e and amax[r] > 448 * 2.0 ** (e - 1)
        normal = np.abs(xd[r]) >= 2.0 ** (e - 6)
        # E4M3 normals: 3 mantissa bits -> half-ulp relative error <= 2^-4
        assert np.all(np.abs(deq[r][normal] - xd[r][normal]) <= 2.0 ** -4 * np.abs(xd[r][normal]))
        # subnormal range: absolute error <= half the subnormal step 2^-10 * 2^e
        assert np.all(np.abs(deq[r][~normal] - xd[r][~normal]) <= 2.0 ** (e - 10))
    # dequantised values are exact bf16 numbers (so metadata over them stays exact)
    t = torch.from_numpy(deq.astype(np.float32))
    assert torch.equal(t.to(torch.bfloat16).to(torch.float32), t)


def test_fp8_decode_step_reduces_to_bf16_on_representable_cache(orc):
    """A cache whose rows are already E4M3 values times 2^e quantises losslessly, so the FP8
    decode step must equal the (pinned) bf16 decode step exactly."""
    import synth
    cfg = synth.config("c3", batch=2, ctx=300, budget_tokens=64)
    case = synth.make_case(cfg, seed=9, ragged=True)
    # pre-round every row to E4M3 x 2^e (the oracle's own quantiser), back to bf16
    kc, ke = orc.kv_quantize(case["k_pool"])
    vc, ve = orc.kv_quantize(case["v_pool"])
    k_rep = torch.from_numpy(orc.kv_dequantize(kc, ke)).to(torch.bfloat16)
    v_rep = torch.from_numpy(orc.kv_dequantize(vc, ve)).to(torch.bfloat16)
    kc2, ke2 = orc.kv_quantize(k_rep)  # lossless: same values (the exponent may drop by one
    assert np.array_equal(orc.kv_dequantize(kc2, ke2), orc.kv_dequantize(kc, ke))  # when amax rounded down)
    ref = orc.decode_step(case["q"], k_rep, v_rep, case["page_table"], case["seq_lens"],
                          cfg.budget_tokens, cfg.scale)
    got = orc.decode_step_fp8(case["q"], kc, ke, vc, ve, case["page_table"], case["seq_lens"],
                              cfg.budget_tokens, cfg.scale)
    assert np.array_equal(got["sel_ids"], ref["sel_ids"])
    assert np.array_equal(got["o"], ref["o"]) and np.array_equal(got["lse"], ref["lse"])
