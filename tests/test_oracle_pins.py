"""Pins for the float64 oracle (oracle/), CPU only.

Each test pins an oracle function to something other than itself: the worked examples in
tests/golden/spec_examples.json (SPEC.md, cited per entry), closed forms, brute force on
tiny inputs, invariants the paper states, and an independent library routine
(torch SDPA in float64) for the K = P special case.  DESIGN.md §2 lists which pin covers
which function.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch

import synth

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ------------------------------------------------------------------ helpers (test-side)
def _pool_from_keys(keys, S, values=None):
    """One sequence, one kv head, fp32 pool holding `keys` in logical order (identity table)."""
    keys = np.asarray(keys, np.float32)
    n, d = keys.shape
    P = -(-n // S)
    kp = np.zeros((P, 1, S, d), np.float32)
    vp = np.zeros((P, 1, S, d), np.float32)
    vals = np.zeros_like(keys) if values is None else np.asarray(values, np.float32)
    for t in range(n):
        kp[t // S, 0, t % S] = keys[t]
        vp[t // S, 0, t % S] = vals[t]
    pt = np.arange(P, dtype=np.int32).reshape(1, P)
    return kp, vp, pt, np.array([n], np.int32)


def _dyadic(rng, shape, lo=-64, hi=64):
    """Values k/8 with small integer k: every product and sum below is exact in double."""
    return rng.integers(lo, hi + 1, size=shape).astype(np.float64) / 8.0


# ------------------------------------------------------------------ step 2: metadata
@pytest.mark.parametrize("ex", GOLDEN["metadata"], ids=lambda e: e["cite"].split()[0])
def test_metadata_golden(orc, ex):
    kp, _, pt, sl = _pool_from_keys(ex["keys"], ex["S"])
    mmin, mmax = orc.meta_build(kp, pt, sl)
    assert mmin[0, 0, 0].tolist() == ex["m"]
    assert mmax[0, 0, 0].tolist() == ex["M"]


def test_page_count_golden(orc):
    ex = GOLDEN["page_count"][0]
    kp, _, pt, sl = _pool_from_keys([[1.0, 1.0]] * ex["tokens"], ex["S"])
    assert pt.shape[1] == ex["pages"]
    q = np.ones((1, 1, 2), np.float32)
    out = orc.decode_step(q, kp, kp, pt, sl, budget_tokens=ex["S"] * 8, scale=1.0)
    assert out["sel_count"][0, 0] == ex["pages"]  # K = P when the budget exceeds the cache


def test_metadata_incremental_equals_batch(orc):
    """SPEC.md:73/85 + acceptance #3: >= 10 000 appends, incremental == batch bit-exactly."""
    cfg = synth.config("c2", batch=4, num_q_heads=2, num_kv_heads=2, ctx=2560, page_size=16)
    case = synth.make_case(cfg, seed=3)
    B, Hkv, d, S, mp = cfg.batch, cfg.num_kv_heads, cfg.head_dim, cfg.page_size, cfg.max_pages
    kfull = case["k_pool"]
    vfull = case["v_pool"]
    pt = case["page_table"].numpy()
    k_raw = np.zeros(kfull.view(torch.int16).shape, np.uint16)
    v_raw = np.zeros_like(k_raw)
    mmin = np.zeros((B, Hkv, mp, d))
    mmax = np.zeros((B, Hkv, mp, d))
    lens = np.zeros(B, np.int32)
    appends = 0
    for t in range(cfg.ctx):
        kn = torch.stack([kfull[pt[b, t // S], :, t % S, :] for b in range(B)])
        vn = torch.stack([vfull[pt[b, t // S], :, t % S, :] for b in range(B)])
        orc.meta_append(kn, vn, lens, pt, k_raw, v_raw, mmin, mmax)
        lens += 1
        appends += B
        if t in (0, 1, 15, 16, 17, 700):  # monotone widening spot checks
            if t > 0 and (t % S) != 0:
                assert np.all(mmin <= prev_min) and np.all(mmax >= prev_max)
        prev_min, prev_max = mmin.copy(), mmax.copy()
    assert appends >= 10_000
    assert np.array_equal(k_raw, kfull.view(torch.int16).numpy().view(np.uint16))
    bmin, bmax = orc.meta_build(kfull, pt, lens)
    assert np.array_equal(bmin, mmin) and np.array_equal(bmax, mmax)


def test_metadata_box_containment_and_partial_pages(orc):
    """Box containment over valid tokens only; partial last page (reading R7)."""
    cfg = synth.config("c2", batch=3, num_q_heads=4, num_kv_heads=4, ctx=200, page_size=16)
    case = synth.make_case(cfg, seed=5, ragged=True, poison_tail=True)
    mmin, mmax = orc.meta_build(case["k_pool"], case["page_table"], case["seq_lens"])
    kw = orc.widen(case["k_pool"])
    pt = case["page_table"].numpy()
    S = cfg.page_size
    for b, L in enumerate(case["seq_lens"].tolist()):
        for t in range(L):
            blk = pt[b, t // S]
            k = kw[blk, :, t % S, :]
            assert np.all(mmin[b, :, t // S] <= k) and np.all(k <= mmax[b, :, t // S])
        assert np.all(np.isfinite(mmin[b, :, : -(-L // S)]))  # NaN tail never enters


# ------------------------------------------------------------------ step 3: score (Eq. 2)
@pytest.mark.parametrize("ex", GOLDEN["score"], ids=lambda e: e["cite"].split()[0])
def test_score_golden(orc, ex):
    kp, _, pt, sl = _pool_from_keys(ex["keys"], S=len(ex["keys"]))
    mmin, mmax = orc.meta_build(kp, pt, sl)
    assert orc.relevance(ex["q"], mmin[0, 0, 0], mmax[0, 0, 0]) == ex["score"]
    exact = max(float(np.dot(ex["q"], k)) for k in ex["keys"])
    assert exact == ex["exact_max"]


@pytest.mark.parametrize("d,S", [(4, 4), (4, 16), (64, 4), (64, 16)])
def test_score_upper_bound_and_singleton(orc, d, S):
    """Acceptance #1: r >= max_k q.k on >= 10 000 pairs in
    total; equality for singleton pages.  Dyadic inputs make every sum exact."""
    rng = np.random.default_rng(1000 + d + S)
    n = 2500
    viol = 0
    for _ in range(n):
        q = _dyadic(rng, d)
        keys = _dyadic(rng, (S, d))
        m, M = keys.min(0), keys.max(0)
        r = orc.relevance(q, m, M)
        best = max(float(np.dot(q, k)) for k in keys)
        viol += r < best
        k1 = keys[0]
        assert orc.relevance(q, k1, k1) == float(np.dot(q, k1))
    assert viol == 0


def test_score_matches_branch_free_forms(orc):
    """Reading R3: Eq. 2 == sum_i max(q m, q M) == q+.M + q-.m when m <= M (exact inputs)."""
    rng = np.random.default_rng(7)
    for _ in range(2000):
        d = 64
        q = _dyadic(rng, d)
        a, b = _dyadic(rng, d), _dyadic(rng, d)
        m, M = np.minimum(a, b), np.maximum(a, b)
        r = orc.relevance(q, m, M)
        assert r == float(np.sum(np.maximum(q * m, q * M)))
        assert r == float(np.dot(np.maximum(q, 0), M) + np.dot(np.minimum(q, 0), m))


def test_score_pages_gqa_group_bound(orc):
    """Reading R9: s_j = max_h r_h(j) >= max_h max_{k in page j} q_h.k, and equals the max of
    the per-head relevance; -inf past P_b."""
    cfg = synth.config("c3", batch=2, ctx=300, page_size=16)
    case = synth.make_case(cfg, seed=11, ragged=True)
    mmin, mmax = orc.meta_build(case["k_pool"], case["page_table"], case["seq_lens"])
    sc = orc.score_pages(case["q"], mmin, mmax, case["seq_lens"], cfg.page_size)
    qw, kw = orc.widen(case["q"]), orc.widen(case["k_pool"])
    pt = case["page_table"].numpy()
    G, S = cfg.group, cfg.page_size
    for b, L in enumerate(case["seq_lens"].tolist()):
        P = -(-L // S)
        assert np.all(np.isneginf(sc[b, :, P:]))
        for g in range(cfg.num_kv_heads):
            for j in range(P):
                heads = range(g * G, (g + 1) * G)
                per_head = [orc.relevance(qw[b, h], mmin[b, g, j], mmax[b, g, j]) for h in heads]
                assert sc[b, g, j] == max(per_head)
                toks = [kw[pt[b, j], g, s] for s in range(min(S, L - j * S))]
                exact = max(float(qw[b, h] @ k) for h in heads for k in toks)
                assert sc[b, g, j] >= exact - 1e-12 * (1 + abs(exact))


# ------------------------------------------------------------------ step 4: top-K
@pytest.mark.parametrize("ex", GOLDEN["topk"], ids=lambda e: e["cite"].split()[0])
def test_topk_golden(orc, ex):
    s = np.array([ex["scores"]])
    ids, _, cnt = orc.select_topk(s, [len(ex["scores"])], ex["k"])
    assert ids[0, : cnt[0]].tolist() == ex["ids"]


def _brute_topk(s, k):
    """Enumerate all C(P, k) subsets, maximise the score sum, ties -> lexicographically
    smallest ascending id tuple (equivalent to 'lower id wins' at the boundary)."""
    best = None
    for sub in itertools.combinations(range(len(s)), k):
        tot = sum(s[i] for i in sub)
        if best is None or tot > best[0] or (tot == best[0] and sub < best[1]):
            best = (tot, sub)
    return list(best[1])


@pytest.mark.parametrize("seed", range(6))
def test_topk_brute_force(orc, seed):
    """C1-sized rows (P = 16, K = 4: 1820 subsets); integer scores so ties are real."""
    rng = np.random.default_rng(seed)
    for trial in range(8):
        s = rng.integers(-3, 4, size=16).astype(np.float64) if trial % 2 else rng.standard_normal(16)
        ids, _, cnt = orc.select_topk(s[None], [16], 4)
        assert cnt[0] == 4
        assert ids[0].tolist() == _brute_topk(s.tolist(), 4)


def test_topk_rank_consistency_and_ids_in(orc):
    rng = np.random.default_rng(9)
    rows, n, k = 20, 300, 37
    s = rng.integers(-20, 20, size=(rows, n)).astype(np.float64)
    s[3] = 0.0
    s[4, ::2] = -0.0  # -0.0 and +0.0 are the same score (reading R6)
    lens = rng.integers(1, n + 1, size=rows).astype(np.int32)
    ids, sc, cnt = orc.select_topk(s, lens, k)
    for r in range(rows):
        n_r, kk = lens[r], min(k, lens[r])
        assert cnt[r] == kk
        sel = ids[r, :kk]
        assert np.all(np.diff(sel) > 0) and np.all(ids[r, kk:] == -1)
        unsel = np.setdiff1d(np.arange(n_r), sel)
        for i in sel:
            for j in unsel:
                assert s[r, i] > s[r, j] or (s[r, i] == s[r, j] and i < j)
    # ids_in: a permuted candidate list with explicit ids selects the same set
    perm = np.stack([rng.permutation(n) for _ in range(rows)]).astype(np.int32)
    s_perm = np.take_along_axis(s, perm, axis=1)
    full = np.full(rows, n, np.int32)
    ids_a, _, _ = orc.select_topk(s, full, k)
    ids_b, _, _ = orc.select_topk(s_perm, full, k, ids_in=perm)
    assert np.array_equal(ids_a, ids_b)


def test_topk_neg_inf_is_no_page(orc):
    """Reading R8: -inf entries (pages that do not exist) are never selected."""
    s = np.array([[-np.inf, 1.0, -np.inf, 0.5, -np.inf, -np.inf]])
    ids, sc, cnt = orc.select_topk(s, None, 4)
    assert cnt[0] == 2 and ids[0].tolist() == [1, 3, -1, -1]
    assert np.isneginf(sc[0, 2:]).all()


def test_topk_candidate_merge_is_exact(orc):
    """global top-K == top-K of the union of per-shard top-Ks (block-cyclic
    ownership, global ids), on inputs with heavy ties."""
    rng = np.random.default_rng(21)
    n, k = 512, 24
    for G in (2, 3, 4, 8):
        s = rng.integers(-5, 5, size=n).astype(np.float64)
        gids, _, _ = orc.select_topk(s[None], [n], k)
        cand_s, cand_i = [], []
        for r in range(G):
            own = np.arange(r, n, G)
            li, ls, lc = orc.select_topk(s[own][None], [len(own)], k)
            cand_i += own[li[0, : lc[0]]].tolist()
            cand_s += ls[0, : lc[0]].tolist()
        mi, _, _ = orc.select_topk(np.array([cand_s]), [len(cand_s)], k,
                                   ids_in=np.array([cand_i], np.int32))
        assert np.array_equal(gids, mi)


# ------------------------------------------------------------------ step 5: attention
def _sdpa_dense(case, scale):
    """torch SDPA in float64 over ALL valid tokens (independent library routine)."""
    cfg = case["cfg"]
    import oracle
    qw = torch.from_numpy(oracle.widen(case["q"]))
    kw = torch.from_numpy(oracle.widen(case["k_pool"]))
    vw = torch.from_numpy(oracle.widen(case["v_pool"]))
    pt = case["page_table"]
    G = cfg.group
    outs = []
    for b, L in enumerate(case["seq_lens"].tolist()):
        P = -(-L // cfg.page_size)
        K = kw[pt[b, :P].long()].permute(1, 0, 2, 3).reshape(cfg.num_kv_heads, -1, cfg.head_dim)[:, :L]
        V = vw[pt[b, :P].long()].permute(1, 0, 2, 3).reshape(cfg.num_kv_heads, -1, cfg.head_dim)[:, :L]
        K = K.repeat_interleave(G, 0)
        V = V.repeat_interleave(G, 0)
        o = torch.nn.functional.scaled_dot_product_attention(
            qw[b][:, None, :], K, V, scale=scale)[:, 0, :]
        lse = torch.logsumexp(scale * torch.einsum("hd,htd->ht", qw[b], K), dim=-1)
        outs.append((o.numpy(), lse.numpy()))
    return outs


@pytest.mark.parametrize("cname,seed,scale", [("c1", 1, 1.0), ("c2", 2, 0.125), ("c3", 3, 1.0)])
def test_attention_k_equals_p_is_dense_sdpa(orc, cname, seed, scale):
    """SPEC.md:234 / acceptance #2 (PAPER.md:141-145 vs 169-172): K = P reproduces dense
    attention; oracle vs torch SDPA float64 within 1e-12."""
    over = {"c1": {}, "c2": dict(batch=3, ctx=500, num_q_heads=2, num_kv_heads=2),
            "c3": dict(batch=2, ctx=700)}[cname]
    cfg = synth.config(cname, **over)
    case = synth.make_case(cfg, seed=seed, ragged=(cname != "c1"), poison_tail=True)
    out = orc.decode_step(case["q"], case["k_pool"], case["v_pool"], case["page_table"],
                          case["seq_lens"], budget_tokens=cfg.ctx + cfg.page_size, scale=scale)
    ref = _sdpa_dense(case, scale)
    for b, (o_ref, lse_ref) in enumerate(ref):
        np.testing.assert_allclose(out["o"][b], o_ref, rtol=0, atol=1e-12)
        np.testing.assert_allclose(out["lse"][b], lse_ref, rtol=1e-13, atol=1e-12)


@pytest.mark.parametrize("ex", GOLDEN["attention"], ids=lambda e: e["cite"].split()[0])
def test_attention_golden(orc, ex):
    kp, vp, pt, sl = _pool_from_keys(ex["keys"], S=len(ex["keys"]), values=ex["values"])
    q = np.asarray(ex["q"], np.float32)[None, None, :]
    o, lse = orc.sparse_attn(q, kp, vp, pt, sl, np.zeros((1, 1, 1), np.int32),
                             np.ones((1, 1), np.int32), scale=1.0)
    np.testing.assert_allclose(o[0, 0], np.asarray(ex["o"], np.float64), rtol=0, atol=ex["o_tol"])


def test_attention_weights_convex_hull_and_singleton(orc):
    """output inside the convex hull of attended values; a one-token
    selection returns that token's v exactly."""
    cfg = synth.config("c2", batch=2, num_q_heads=2, num_kv_heads=2, ctx=97, page_size=16)
    case = synth.make_case(cfg, seed=4, seq_lens=[97, 1])
    kmax = 3
    ids = np.array([[[0, 2, 6]] * 2, [[0, -1, -1]] * 2], np.int32)
    cnt = np.array([[3, 3], [1, 1]], np.int32)
    o, lse = orc.sparse_attn(case["q"], case["k_pool"], case["v_pool"], case["page_table"],
                             case["seq_lens"], ids, cnt, scale=1.0)
    vw = orc.widen(case["v_pool"])
    pt = case["page_table"].numpy()
    for h in range(2):
        toks = [vw[pt[0, j], h, s] for j in (0, 2, 6) for s in range(16) if j * 16 + s < 97]
        V = np.stack(toks)
        assert np.all(o[0, h] >= V.min(0) - 1e-12) and np.all(o[0, h] <= V.max(0) + 1e-12)
        assert np.array_equal(o[1, h], vw[pt[1, 0], h, 0])


def test_attention_empty_sequence(orc):
    """Reading R8: seq_len = 0 -> o = 0, lse = -inf, no page selected."""
    cfg = synth.config("c2", batch=2, num_q_heads=2, num_kv_heads=2, ctx=64)
    case = synth.make_case(cfg, seed=8, seq_lens=[0, 64])
    out = orc.decode_step(case["q"], case["k_pool"], case["v_pool"], case["page_table"],
                          case["seq_lens"], budget_tokens=32, scale=1.0)
    assert np.all(out["o"][0] == 0) and np.all(np.isneginf(out["lse"][0]))
    assert np.all(out["sel_count"][0] == 0) and np.all(out["sel_count"][1] == 2)


def test_lse_merge_equals_unsplit(orc):
    """Split-K / multi-GPU algebra: attention over disjoint page subsets,
    merged by LSE, equals attention over their union."""
    cfg = synth.config("c3", batch=2, ctx=800)
    case = synth.make_case(cfg, seed=12, ragged=True)
    P = -(-int(case["seq_lens"].min()) // cfg.page_size)
    allp = np.arange(P, dtype=np.int32)
    parts = [allp[r::3] for r in range(3)] + [np.array([], np.int32)]
    B, Hkv = cfg.batch, cfg.num_kv_heads

    def run(pages):
        ids = np.full((B, Hkv, max(1, len(pages))), -1, np.int32)
        ids[:, :, : len(pages)] = pages
        cnt = np.full((B, Hkv), len(pages), np.int32)
        return orc.sparse_attn(case["q"], case["k_pool"], case["v_pool"], case["page_table"],
                               case["seq_lens"], ids, cnt, scale=0.125)

    o_all, lse_all = run(allp)
    outs = [run(p) for p in parts]
    rows = B * cfg.num_q_heads
    o_m, lse_m = orc.lse_merge(np.stack([o.reshape(rows, -1) for o, _ in outs]),
                               np.stack([l.reshape(rows) for _, l in outs]))
    np.testing.assert_allclose(o_m, o_all.reshape(rows, -1), rtol=0, atol=1e-13)
    np.testing.assert_allclose(lse_m, lse_all.reshape(rows), rtol=1e-14, atol=1e-13)


def test_decode_step_composes_the_steps(orc):
    """decode_step == meta_build -> score -> select(K_b = min(P, budget/S)) -> attn."""
    cfg = synth.config("c3", batch=3, ctx=1000)
    case = synth.make_case(cfg, seed=13, ragged=True)
    out = orc.decode_step(case["q"], case["k_pool"], case["v_pool"], case["page_table"],
                          case["seq_lens"], cfg.budget_tokens // 4, 0.125, want_scores=True)
    mmin, mmax = orc.meta_build(case["k_pool"], case["page_table"], case["seq_lens"])
    sc = orc.score_pages(case["q"], mmin, mmax, case["seq_lens"], cfg.page_size)
    assert np.array_equal(sc, out["scores"])
    k = cfg.budget_tokens // 4 // cfg.page_size
    P = [-(-L // cfg.page_size) for L in case["seq_lens"].tolist()]
    rl = np.repeat(np.array(P, np.int32), cfg.num_kv_heads)
    ids, _, cnt = orc.select_topk(sc.reshape(-1, cfg.max_pages), rl, k)
    assert np.array_equal(ids.reshape(out["sel_ids"].shape), out["sel_ids"])
    o, lse = orc.sparse_attn(case["q"], case["k_pool"], case["v_pool"], case["page_table"],
                             case["seq_lens"], out["sel_ids"], out["sel_count"], 0.125)
    assert np.array_equal(o, out["o"]) and np.array_equal(lse, out["lse"])


def test_oracle_thread_count_independent(orc):
    cfg = synth.config("c3", batch=2, ctx=2000)
    case = synth.make_case(cfg, seed=14)
    a = orc.decode_step(case["q"], case["k_pool"], case["v_pool"], case["page_table"],
                        case["seq_lens"], 512, 0.125, threads=1)
    b = orc.decode_step(case["q"], case["k_pool"], case["v_pool"], case["page_table"],
                        case["seq_lens"], 512, 0.125, threads=4)
    for key in a:
        assert np.array_equal(a[key], b[key])
