"""GPU parity of the FP8 KV path (reading R21) vs the
float64 oracle (oracle.kv_quantize / kv_dequantize / decode_step_fp8).

Bars: E4M3 codes and row exponents bit-exact (byte work); metadata over the dequantised
keys bit-exact; page sets bit-exact on margin-enforced inputs; o max-abs <= 2e-3 and lse
<= 1e-3 against attention over the exactly dequantised values (the same bar as bf16 K/V:
the compute is bf16-class, only the storage is 8-bit).
"""
import numpy as np
import pytest
import torch

import oracle
import oracle.margin
import synth

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


@pytest.fixture(scope="module")
def ts():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2509_12211_b200 import _build
    _build.build()
    import paper_2509_12211_b200 as ts
    return ts


CASES = {
    "c3_small": ("c3", dict(batch=2, ctx=3000, budget_tokens=512)),
    "c2_small": ("c2", dict(batch=4, ctx=1500)),
    "g4_s32": ("c3", dict(batch=2, num_q_heads=16, ctx=2500, page_size=32, budget_tokens=512)),
    "g6_s64": ("c3", dict(batch=2, num_q_heads=24, ctx=6000, page_size=64, budget_tokens=1024)),
    "two_level": ("c3", dict(batch=1, ctx=36000, budget_tokens=512)),
    "small_budget_long": ("c3", dict(batch=1, ctx=32768, budget_tokens=128)),
    "c5_like": ("c5", dict(batch=1, ctx=40000, budget_tokens=1024)),
}


def make(name, seed=31, scale_kv=1.0):
    cname, over = CASES[name]
    cfg = synth.config(cname, **over)
    case = synth.make_case(cfg, seed=seed, ragged=True)
    if scale_kv != 1.0:
        case["k_pool"] = (case["k_pool"].float() * scale_kv).to(torch.bfloat16)
        case["v_pool"] = (case["v_pool"].float() * scale_kv).to(torch.bfloat16)
    return cfg, case


def quantize_both(ts, case, poison=True):
    """GPU and oracle quantisation of the case's bf16 pools; the GPU pools get garbage past
    seq_len in every partial last page (NaN codes, extreme exponents) so a kernel that reads
    them instead of masking fails."""
    cfg = case["cfg"]
    nb, Hkv, S, d = case["k_pool"].shape
    kq = ts.kv_quantize(case["k_pool"].to(DEV))
    vq = ts.kv_quantize(case["v_pool"].to(DEV))
    kc, ke = oracle.kv_quantize(case["k_pool"])
    vc, ve = oracle.kv_quantize(case["v_pool"])
    if poison:
        pt = case["page_table"].numpy()
        for pool in (kq, vq):
            codes, exps = ts.fp8_views(pool, nb, Hkv, S, d)
            for b, L in enumerate(case["seq_lens"].tolist()):
                if L % S:
                    blk = int(pt[b, L // S])
                    for sl in range(L % S, S):
                        codes[blk, :, sl // 16, sl % 16, :] = 0x7F  # E4M3 NaN
                        exps[blk, :, sl // 16, sl % 16] = 127
    return kq, vq, (kc, ke, vc, ve)


def deq_case(case, orc_q):
    kc, ke, vc, ve = orc_q
    return dict(case, k_pool=torch.from_numpy(oracle.kv_dequantize(kc, ke)),
                v_pool=torch.from_numpy(oracle.kv_dequantize(vc, ve)))


def enforce_fp8(case, orc_q, budget, rel=1e-4):
    """oracle.margin's rule on the dequantised cache (redraws q rows only)."""
    cv = deq_case(case, orc_q)  # dequantised once (= oracle.decode_step_fp8's first step)
    for attempt in range(64):
        qf = torch.from_numpy(oracle.widen(case["q"]).astype(np.float32))
        ref = oracle.decode_step(qf, cv["k_pool"], cv["v_pool"], case["page_table"], case["seq_lens"],
                                 budget, case["cfg"].scale, want_scores=True)
        bad, _ = oracle.margin.violations(cv, budget, rel, ref=ref)
        if not bad:
            return ref
        synth.resample_q_rows(case, bad, attempt)
    raise RuntimeError("margin not reached")


# ------------------------------------------------------------------ quantiser
@pytest.mark.parametrize("scale_kv", [1.0, 1e-3, 300.0])
def test_kv_quantize_bit_exact(ts, scale_kv):
    cfg, case = make("c3_small", scale_kv=scale_kv)
    kq, _, (kc, ke, _, _) = quantize_both(ts, case, poison=False)
    nb, Hkv, S, d = case["k_pool"].shape
    codes, exps = ts.fp8_split(kq, nb, Hkv, S, d)
    assert np.array_equal(exps.cpu().numpy(), ke)
    assert np.array_equal(codes.cpu().numpy(), kc)


def test_kv_quantize_edge_rows(ts):
    """all-zero rows (e = -64), a row at the exponent clamps, ties, subnormal codes."""
    rows = torch.zeros(16, 64)  # one sub-page record (rows 8..15 stay zero)
    rows[1, 0] = 448.0                       # e = 0 exactly
    rows[2, :] = torch.linspace(-1, 1, 64)   # mixed
    rows[3, 0] = 3e30                        # e clamped at 64, saturating codes
    rows[4, :] = 1e-30                       # e clamped at -64 (tiny row)
    rows[5, :8] = torch.tensor([1.0625, 1.1875, -1.0625, 2 ** -9, 2 ** -10, 3 * 2 ** -10, -2 ** -12, 0.0])
    rows[5, 8] = 448.0 / 128                 # row exponent -7 -> exact tie cases scale by 2^7
    rows[6, :] = -0.0
    rows[7, :] = torch.randn(64, generator=torch.Generator().manual_seed(3)) * 1e-5
    x = rows.to(torch.bfloat16)
    q = ts.kv_quantize(x.to(DEV))
    kc, ke = oracle.kv_quantize(x)
    assert np.array_equal(q[1024:].view(torch.int8).cpu().numpy(), ke)
    g = q[:1024].view(16, 64).cpu().numpy()
    # -0.0 rounds to the sign-bearing zero on both sides; compare values where both are zero
    zero = (kc & 0x7F) == 0
    assert np.array_equal(g[~zero], kc[~zero]) and np.all((g[zero] & 0x7F) == 0)


# ------------------------------------------------------------------ a1: metadata
@pytest.mark.parametrize("name", ["c3_small", "g4_s32", "g6_s64"])
def test_meta_build_fp8_bit_exact(ts, name):
    cfg, case = make(name)
    kq, _, oq = quantize_both(ts, case)
    d = {k: (v.to(DEV) if isinstance(v, torch.Tensor) else v) for k, v in case.items()}
    L = ts.make_layout(d["q"], kq, d["page_table"], pool_shape=tuple(case["k_pool"].shape))
    meta = ts.meta_build(L, kq, d["page_table"], d["seq_lens"])
    cv = deq_case(case, oq)
    omin, omax = oracle.meta_build(cv["k_pool"], case["page_table"], case["seq_lens"])
    m = oracle.widen(meta.cpu())
    for b, Lb in enumerate(case["seq_lens"].tolist()):
        P = -(-Lb // cfg.page_size)
        assert np.array_equal(m[b, :, :P, 0], omin[b, :, :P])
        assert np.array_equal(m[b, :, :P, 1], omax[b, :, :P])


def test_meta_append_fp8_incremental(ts):
    """Token-by-token appends of bf16 K/V into an FP8 cache == oracle quantisation of every
    row + oracle metadata over the dequantised keys (Eq. 1)."""
    cfg = synth.config("c3", batch=2, ctx=100, budget_tokens=64)
    case = synth.make_case(cfg, seed=5)
    nb, Hkv, S, d = case["k_pool"].shape
    pt = case["page_table"]
    kq, vq = ts.fp8_pool(nb, Hkv, S, d, DEV), ts.fp8_pool(nb, Hkv, S, d, DEV)
    q = case["q"].to(DEV)
    L = ts.make_layout(q, kq, pt.to(DEV), pool_shape=(nb, Hkv, S, d))
    meta = ts.new_meta(L, torch.bfloat16, DEV)
    lens = torch.zeros(cfg.batch, dtype=torch.int32, device=DEV)
    ptn = pt.numpy()
    for t in range(cfg.ctx):
        kn = torch.stack([case["k_pool"][ptn[b, t // S], :, t % S] for b in range(cfg.batch)])
        vn = torch.stack([case["v_pool"][ptn[b, t // S], :, t % S] for b in range(cfg.batch)])
        ts.meta_append(L, kn.to(DEV), vn.to(DEV), lens, pt.to(DEV), kq, vq, meta, advance=True)
    torch.cuda.synchronize()
    assert lens.cpu().tolist() == [cfg.ctx] * cfg.batch
    kc, ke = oracle.kv_quantize(case["k_pool"])
    vc, ve = oracle.kv_quantize(case["v_pool"])
    gkc, gke = ts.fp8_split(kq, nb, Hkv, S, d)
    gvc, gve = ts.fp8_split(vq, nb, Hkv, S, d)
    written = [(ptn[b, t // S], t % S) for b in range(cfg.batch) for t in range(cfg.ctx)]
    blk = np.array([w[0] for w in written])
    slot = np.array([w[1] for w in written])
    for g_, o_ in ((gkc, kc), (gke, ke), (gvc, vc), (gve, ve)):
        assert np.array_equal(g_.cpu().numpy()[blk, :, slot], o_[blk, :, slot])
    omin, omax = oracle.meta_build(torch.from_numpy(oracle.kv_dequantize(kc, ke)), pt, case["seq_lens"])
    m = oracle.widen(meta.cpu())
    assert np.array_equal(m[:, :, :, 0], omin) and np.array_equal(m[:, :, :, 1], omax)


# ------------------------------------------------------------------ a5: fused step
def _fp8_step(ts, cfg, case, kq, vq, ref, prefetch=False):
    d = {k: (v.to(DEV) if isinstance(v, torch.Tensor) else v) for k, v in case.items()}
    shape = tuple(case["k_pool"].shape)
    L = ts.make_layout(d["q"], kq, d["page_table"], pool_shape=shape)
    meta = ts.meta_build(L, kq, d["page_table"], d["seq_lens"])
    if prefetch:
        K = ts.kmax(L, cfg.budget_tokens)
        ids = torch.randint(-1, cfg.max_pages + 2, (cfg.batch, cfg.num_kv_heads, K), dtype=torch.int32, device=DEV)
        cnt = torch.full((cfg.batch, cfg.num_kv_heads), K, dtype=torch.int32, device=DEV)
        o, lse, ids, cnt = ts.decode_step_prefetch(L, d["q"], kq, vq, meta, d["page_table"], d["seq_lens"],
                                                   cfg.budget_tokens, cfg.scale, ids, cnt)
    else:
        o, lse, ids, cnt = ts.decode_step(L, d["q"], kq, vq, meta, d["page_table"], d["seq_lens"],
                                          cfg.budget_tokens, cfg.scale)
    assert ts.launch_count() == 1
    assert np.array_equal(cnt.cpu().numpy(), ref["sel_count"])
    K = ids.shape[2]
    assert np.array_equal(ids.cpu().numpy(), ref["sel_ids"][:, :, :K])
    err = np.abs(o.cpu().numpy() - ref["o"]).max()
    assert err <= 2e-3, err
    g, fin = lse.cpu().numpy(), np.isfinite(ref["lse"])
    assert np.array_equal(np.isfinite(g), fin)
    if fin.any():
        assert np.abs(g[fin] - ref["lse"][fin]).max() <= 1e-3
    return err


@pytest.mark.parametrize("name", list(CASES))
def test_decode_step_fp8(ts, name):
    cfg, case = make(name)
    kq, vq, oq = quantize_both(ts, case)
    ref = enforce_fp8(case, oq, cfg.budget_tokens)
    _fp8_step(ts, cfg, case, kq, vq, ref)


@pytest.mark.parametrize("scale", [1.0, 0.125])
def test_decode_step_fp8_scales(ts, scale):
    """paper-verbatim softmax scale 1 (reading R1) and widely varying row exponents."""
    cfg, case = make("c3_small", seed=41)
    cfg = cfg.with_(scale=scale)
    case["cfg"] = cfg
    g = torch.Generator().manual_seed(9)
    mult = torch.exp2(torch.randint(-6, 7, case["v_pool"].shape[:3] + (1,), generator=g).float())
    case["v_pool"] = (case["v_pool"].float() * mult).to(torch.bfloat16)
    kq, vq, oq = quantize_both(ts, case)
    ref = enforce_fp8(case, oq, cfg.budget_tokens)
    # outputs scale with the V magnitudes: compare relative to max |v| seen (2^6)
    d = {k: (v.to(DEV) if isinstance(v, torch.Tensor) else v) for k, v in case.items()}
    L = ts.make_layout(d["q"], kq, d["page_table"], pool_shape=tuple(case["k_pool"].shape))
    meta = ts.meta_build(L, kq, d["page_table"], d["seq_lens"])
    o, lse, ids, cnt = ts.decode_step(L, d["q"], kq, vq, meta, d["page_table"], d["seq_lens"],
                                      cfg.budget_tokens, cfg.scale)
    assert np.array_equal(ids.cpu().numpy(), ref["sel_ids"][:, :, :ids.shape[2]])
    assert np.abs(o.cpu().numpy() - ref["o"]).max() <= 2e-3 * 64


def test_decode_step_prefetch_fp8(ts):
    cfg, case = make("c3_small", seed=43)
    kq, vq, oq = quantize_both(ts, case)
    ref = enforce_fp8(case, oq, cfg.budget_tokens)
    _fp8_step(ts, cfg, case, kq, vq, ref, prefetch=True)


@pytest.mark.parametrize("name", ["c3_small", "g4_s32"])
def test_decode_step_append_fp8(ts, name):
    """ts_decode_step_append on an FP8 cache == the oracle's quantisation of the newest token,
    its metadata update, and the step over the resulting cache."""
    cfg, case = make(name, seed=47)
    nb, Hkv, S, d = case["k_pool"].shape
    pt = case["page_table"].numpy()
    lens = case["seq_lens"]
    B = cfg.batch
    k_new = torch.zeros(B, Hkv, d, dtype=torch.bfloat16)
    v_new = torch.zeros_like(k_new)
    for b, Lb in enumerate(lens.tolist()):
        blk, sl = pt[b, (Lb - 1) // S], (Lb - 1) % S
        k_new[b], v_new[b] = case["k_pool"][blk, :, sl], case["v_pool"][blk, :, sl]
    kq, vq, oq = quantize_both(ts, case, poison=False)
    ref = enforce_fp8(case, oq, cfg.budget_tokens)  # the step on the FULL cache
    gkc, gke = ts.fp8_views(kq, nb, Hkv, S, d)
    gvc, gve = ts.fp8_views(vq, nb, Hkv, S, d)
    for b, Lb in enumerate(lens.tolist()):  # stale content in the newest slot
        blk, sl = pt[b, (Lb - 1) // S], (Lb - 1) % S
        a_, r_ = sl // 16, sl % 16
        gkc[blk, :, a_, r_], gke[blk, :, a_, r_], gvc[blk, :, a_, r_], gve[blk, :, a_, r_] = 0x55, 9, 0x33, -9
    dq, dpt, dl = case["q"].to(DEV), case["page_table"].to(DEV), lens.to(DEV)
    L = ts.make_layout(dq, kq, dpt, pool_shape=(nb, Hkv, S, d))
    meta = ts.meta_build(L, kq, dpt, torch.clamp(dl - 1, min=0).to(torch.int32))
    o, lse, ids, cnt = ts.decode_step_append(L, dq, k_new.to(DEV), v_new.to(DEV), kq, vq, meta, dpt, dl,
                                             cfg.budget_tokens, cfg.scale)
    assert ts.launch_count() == 1  # the quantising append rides in the step's launch
    kc, ke, vc, ve = oq
    gkc, gke = ts.fp8_split(kq, nb, Hkv, S, d)
    gvc, gve = ts.fp8_split(vq, nb, Hkv, S, d)
    # metadata == the oracle's over the dequantised keys of the full cache (Eq. 1)
    omin, omax = oracle.meta_build(deq_case(case, oq)["k_pool"], case["page_table"], lens)
    m = oracle.widen(meta.cpu())
    for b, Lb in enumerate(lens.tolist()):
        P = -(-Lb // S)
        assert np.array_equal(m[b, :, :P, 0], omin[b, :, :P]) and np.array_equal(m[b, :, :P, 1], omax[b, :, :P])
    assert np.array_equal(gkc.cpu().numpy(), kc) and np.array_equal(gke.cpu().numpy(), ke)
    assert np.array_equal(gvc.cpu().numpy(), vc) and np.array_equal(gve.cpu().numpy(), ve)
    assert np.array_equal(ids.cpu().numpy(), ref["sel_ids"][:, :, :ids.shape[2]])
    assert np.abs(o.cpu().numpy() - ref["o"]).max() <= 2e-3


def test_fp8_full_size_c3(ts):
    """C3 at full size (B 16, 32k, K 128) in the bench's launch configuration."""
    cfg = synth.config("c3")
    case = synth.make_case(cfg, seed=42, ragged=True)
    kq, vq, oq = quantize_both(ts, case)
    ref = enforce_fp8(case, oq, cfg.budget_tokens)
    _fp8_step(ts, cfg, case, kq, vq, ref)


# ------------------------------------------------------------------ standalone entry points
def test_sparse_and_dense_attention_fp8(ts):
    """ts_sparse_decode_attn / ts_dense_decode_attn over an FP8 cache (the TMA attention
    kernel's F8 instantiation) vs the oracle's attention over the dequantised values."""
    cfg, case = make("c3_small", seed=51)
    kq, vq, oq = quantize_both(ts, case)
    cv = deq_case(case, oq)
    qf = torch.from_numpy(oracle.widen(case["q"]).astype(np.float32))
    d = {k: (v.to(DEV) if isinstance(v, torch.Tensor) else v) for k, v in case.items()}
    L = ts.make_layout(d["q"], kq, d["page_table"], pool_shape=tuple(case["k_pool"].shape))
    P = cfg.max_pages
    g = torch.Generator().manual_seed(2)
    K = 40
    ids = np.stack([np.stack([np.sort(torch.randperm(-(-int(l) // cfg.page_size), generator=g)[:K].numpy())
                              for _ in range(cfg.num_kv_heads)]) for l in case["seq_lens"].tolist()]).astype(np.int32)
    cnt = np.full((cfg.batch, cfg.num_kv_heads), K, np.int32)
    ro, rl = oracle.sparse_attn(qf, cv["k_pool"], cv["v_pool"], case["page_table"], case["seq_lens"], ids, cnt, cfg.scale)
    o, lse = ts.sparse_decode_attn(L, d["q"], kq, vq, d["page_table"], d["seq_lens"],
                                   torch.from_numpy(ids).to(DEV), torch.from_numpy(cnt).to(DEV), cfg.scale)
    assert np.abs(o.cpu().numpy() - ro).max() <= 2e-3
    assert np.abs(lse.cpu().numpy() - rl).max() <= 1e-3
    allp = np.tile(np.arange(P, dtype=np.int32), (cfg.batch, cfg.num_kv_heads, 1))
    allc = np.array([[-(-int(l) // cfg.page_size)] * cfg.num_kv_heads for l in case["seq_lens"].tolist()], np.int32)
    do, dl = oracle.sparse_attn(qf, cv["k_pool"], cv["v_pool"], case["page_table"], case["seq_lens"], allp, allc, cfg.scale)
    o2, l2 = ts.dense_decode_attn(L, d["q"], kq, vq, d["page_table"], d["seq_lens"], cfg.scale)
    assert np.abs(o2.cpu().numpy() - do).max() <= 2e-3
    assert np.abs(l2.cpu().numpy() - dl).max() <= 1e-3


@pytest.mark.parametrize("fused", [True, False])
def test_sharded_fp8_matches_oracle(ts, fused):
    """Sequence sharding over an FP8 cache (shard emulation, 4 ranks): the selection equals
    the unsharded FP8 step's and the oracle's; o within 2e-3 of the oracle."""
    from paper_2509_12211_b200 import sharded
    cfg = synth.config("c5", batch=2, ctx=20000, budget_tokens=1024)
    case = synth.make_case(cfg, seed=53, ragged=True)
    kq, vq, oq = quantize_both(ts, case)
    ref = enforce_fp8(case, oq, cfg.budget_tokens)
    d = {k: (v.to(DEV) if isinstance(v, torch.Tensor) else v) for k, v in case.items()}
    shape = tuple(case["k_pool"].shape)
    L = ts.make_layout(d["q"], kq, d["page_table"], pool_shape=shape)
    o, lse, ids, cnts = sharded.emulate(ts, L, 4, d["q"], kq, vq, d["page_table"], d["seq_lens"],
                                        cfg.budget_tokens, cfg.scale, fused=fused)
    K = ids[0].shape[-1]
    for r in range(4):
        assert np.array_equal(ids[r].cpu().numpy(), ref["sel_ids"][:, :, :K])
    assert np.abs(o.cpu().numpy().reshape(ref["o"].shape) - ref["o"]).max() <= 2e-3
