"""Margin enforcement for parity inputs — test infrastructure, oracle-side.

The selected page set is compared bit-exactly with the oracle, so inputs are drawn such that
the K-th and (K+1)-th largest oracle scores of every row differ by at least
    rel * max(L1_K, L1_{K+1}),   L1(j) = max_h sum_i |q_hi| * max(|m_ji|, |M_ji|),
i.e. 25x the fp32 accumulation bound d * 2^-24 * L1 (rel = 1e-4, north star "1e-4 relative").
Rows that violate it get their q redrawn (synth.resample_q_rows) — never the cache.
"""
from __future__ import annotations

import numpy as np

import synth

from . import decode_step, meta_build, widen


def l1_bounds(q, mmin, mmax, group):
    """L1(b, g, j) = max_h sum_i |q_hi| max(|m|, |M|)  (float64)."""
    qa = np.abs(widen(q))                              # [B][Hq][d]
    box = np.maximum(np.abs(mmin), np.abs(mmax))       # [B][Hkv][mp][d]
    B, Hq, d = qa.shape
    qg = qa.reshape(B, Hq // group, group, d)
    return np.einsum("bghd,bgjd->bghj", qg, box).max(axis=2)


def violations(case, budget_tokens, rel=1e-4, ref=None):
    cfg = case["cfg"]
    S, G = cfg.page_size, cfg.group
    K = max(1, budget_tokens // S)
    if ref is None:
        ref = decode_step(case["q"], case["k_pool"], case["v_pool"], case["page_table"],
                          case["seq_lens"], budget_tokens, cfg.scale, want_scores=True)
    mmin, mmax = meta_build(case["k_pool"], case["page_table"], case["seq_lens"])
    l1 = l1_bounds(case["q"], mmin, mmax, G)
    bad = []
    for b, L in enumerate(case["seq_lens"].tolist()):
        P = -(-int(L) // S)
        if P <= K:
            continue
        for g in range(cfg.num_kv_heads):
            s = ref["scores"][b, g, :P]
            order = np.lexsort((np.arange(P), -s))
            jk, jk1 = order[K - 1], order[K]
            gap = s[jk] - s[jk1]
            if gap < rel * max(l1[b, g, jk], l1[b, g, jk1]):
                bad.append((b, g))
    return bad, ref


def enforce(case, budget_tokens, rel=1e-4, max_attempts=64):
    """Redraw q rows until every row keeps the margin; returns the oracle decode_step result."""
    for attempt in range(max_attempts):
        bad, ref = violations(case, budget_tokens, rel)
        if not bad:
            return ref
        synth.resample_q_rows(case, bad, attempt)
    raise RuntimeError(f"margin not reached after {max_attempts} attempts: {len(bad)} rows")
