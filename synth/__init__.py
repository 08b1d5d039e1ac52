"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no metadata, scoring, selection or
attention).  It only draws random tensors with the shapes, dtypes and structure of the
paper's workloads and lays them out in the paged-KV format of DESIGN.md §3:

  q          [B][Hq][d]              kv dtype
  k_pool     [NB][Hkv][S][d]         kv dtype   (physical blocks, vLLM-style, head-major)
  v_pool     [NB][Hkv][S][d]         kv dtype
  page_table [B][max_pages]          int32      (logical page -> physical block)
  seq_lens   [B]                     int32      (tokens already in the cache)

Workload recipe (SURVEY.md §8d "Synthetic inputs"):
  * "clustered": per (block, kv-head) a page centre c ~ N(0, sigma_c^2 I); keys
    k_t = c + N(0, sigma_n^2 I); values v ~ N(0, 1); queries q ~ N(0, 1).  This is the
    page-structured key distribution the paper's bounding boxes exploit.
  * "int": q and k integers in [-4, 4] (exact in bf16 and fp32, so equal scores are real
    ties), v ~ N(0, 1).  Used only by the tie-break tests.
  * page table: a random permutation of the physical blocks, so gathers are scattered.
  * lengths: uniform ctx, or ragged (ctx - U[0, S) per sequence) so partial last pages occur.
  * every tensor is drawn in float32 from a torch.Generator seeded from (seed, tag) and
    cast once to the KV dtype, so every consumer sees exactly the same rounded values.

Config shapes are BASELINE.json:configs (C1..C5), with P = ceil(ctx/S) and
K = floor(budget/S) clipped to [1, P] by the method itself (not here).
"""
from __future__ import annotations

import dataclasses
import hashlib
import math
from typing import Optional

import torch

__all__ = ["Config", "CONFIGS", "make_case", "resample_q_rows", "sub_seed", "config",
           "drift_queries", "algorithmic_bytes"]


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    batch: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    ctx: int
    page_size: int
    budget_tokens: int
    dtype: str  # "bf16" | "f32"
    scale: float = 1.0  # softmax scale; reading R1 (paper has none)
    note: str = ""

    @property
    def group(self) -> int:
        return self.num_q_heads // self.num_kv_heads

    @property
    def max_pages(self) -> int:
        return -(-self.ctx // self.page_size)

    @property
    def torch_dtype(self) -> torch.dtype:
        return {"bf16": torch.bfloat16, "f32": torch.float32}[self.dtype]

    def with_(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)


# BASELINE.json "configs", in order.  C3/C4 page size: paper default 16.
CONFIGS = {
    "c1": Config("c1", 1, 1, 1, 64, 256, 16, 64, "f32",
                 note="tiny: batch 1, 1 head, d 64, 16 pages x 16 tokens, top-k 4 pages, fp32"),
    "c2": Config("c2", 32, 16, 16, 64, 4096, 16, 512, "bf16", scale=0.125,
                 note="GPT2-345M shape: 16 heads, d 64, batch 32, 4k ctx, page 16, budget 512"),
    "c3": Config("c3", 16, 32, 4, 64, 32768, 16, 2048, "bf16", scale=0.125,
                 note="TinyLLaMA-1.1B shape: 32q/4kv GQA, d 64, batch 16, 32k ctx, budget 2048"),
    "c4": Config("c4", 128, 32, 4, 64, 8192, 16, 1024, "bf16", scale=0.125,
                 note="TinyLLaMA shape, batch 128, 8k ctx, budget 1024 (batch-sharded)"),
    "c5": Config("c5", 4, 32, 4, 64, 524288, 64, 4096, "bf16", scale=0.125,
                 note="TinyLLaMA shape, batch 4, 512k ctx, page 64, budget 4096 (sequence-sharded)"),
}


def config(name: str, **overrides) -> Config:
    return CONFIGS[name].with_(**overrides) if overrides else CONFIGS[name]


def sub_seed(seed: int, *tags) -> int:
    """Deterministic 63-bit sub-seed from a base seed and tags (no RNG state sharing)."""
    h = hashlib.blake2b(repr((int(seed),) + tuple(tags)).encode(), digest_size=8)
    return int.from_bytes(h.digest(), "little") & ((1 << 63) - 1)


def _gen(seed: int, tag, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(sub_seed(seed, tag))
    return g


def _randn(shape, seed, tag, device):
    return torch.randn(shape, generator=_gen(seed, tag, device), device=device, dtype=torch.float32)


def _randint(lo, hi, shape, seed, tag, device):
    return torch.randint(lo, hi + 1, shape, generator=_gen(seed, tag, device), device=device,
                         dtype=torch.int64).to(torch.float32)


def make_case(cfg: Config, seed: int = 42, *, device="cpu", mode: str = "clustered",
              ragged: bool = False, seq_lens: Optional[list] = None,
              identity_table: bool = False, sigma_c: float = 1.0, sigma_n: float = 1.0,
              poison_tail: bool = False, spare_blocks: int = 0,
              q_local: Optional[tuple] = None) -> dict:
    """Draw one synthetic paged-KV decode case.

    seed 42 is the paper's seed.  `poison_tail` writes NaN into the
    unused slots past seq_len of every partial last page, so that a kernel that reads
    them (instead of masking) fails the parity tests loudly.

    `q_local = (n_hot, beta)` (clustered mode; SURVEY.md §8d "query locality toward n_hot
    pages", the NEXT-4 accuracy workload): per (sequence, kv head) n_hot logical pages are
    drawn among the valid ones and q head h of the group becomes
        q = beta * c_hot(h) + z,   z ~ N(0, I),
    c_hot(h) the key centre of hot page h mod n_hot, so decode attention concentrates on a
    few pages as it does for a real model's queries (random queries see near-flat
    attention over the whole context).
    """
    B, Hq, Hkv, d, S = cfg.batch, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, cfg.page_size
    mp = cfg.max_pages
    nb = B * mp + spare_blocks
    dt = cfg.torch_dtype
    dev = torch.device(device)

    if seq_lens is None:
        if ragged:
            g = _gen(seed, "lens", "cpu")
            lens = [cfg.ctx - int(torch.randint(0, S, (1,), generator=g)) for _ in range(B)]
        else:
            lens = [cfg.ctx] * B
    else:
        lens = [int(x) for x in seq_lens]
        assert len(lens) == B and all(0 <= x <= mp * S for x in lens)

    if mode == "clustered":
        centre = _randn((nb, Hkv, 1, d), seed, "kcentre", dev) * sigma_c
        k = centre + _randn((nb, Hkv, S, d), seed, "knoise", dev) * sigma_n
        q = _randn((B, Hq, d), seed, "q", dev)
    elif mode == "int":
        k = _randint(-4, 4, (nb, Hkv, S, d), seed, "kint", dev)
        q = _randint(-4, 4, (B, Hq, d), seed, "qint", dev)
    else:
        raise ValueError(mode)
    v = _randn((nb, Hkv, S, d), seed, "v", dev)

    if identity_table:
        perm = torch.arange(nb, device="cpu")
    else:
        perm = torch.randperm(nb, generator=_gen(seed, "perm", "cpu"))
    page_table = perm[: B * mp].reshape(B, mp).to(torch.int32)

    if q_local is not None:
        assert mode == "clustered"
        n_hot, beta = int(q_local[0]), float(q_local[1])
        G = Hq // Hkv
        gh = _gen(seed, "hot", "cpu")
        cen = centre.to("cpu")
        qc = q.to("cpu").clone()
        for b, L in enumerate(lens):
            P = max(1, -(-L // S))
            for g in range(Hkv):
                hot = torch.randint(0, P, (n_hot,), generator=gh)
                for h in range(G):
                    blk = int(page_table[b, int(hot[h % n_hot])])
                    qc[b, g * G + h] += beta * cen[blk, g, 0]
        q = qc.to(dev)

    k_pool = k.to(dt)
    v_pool = v.to(dt)
    if poison_tail:
        pt = page_table.to(torch.int64)
        for b, L in enumerate(lens):
            if L % S:
                blk = int(pt[b, L // S])
                k_pool[blk, :, L % S:, :] = float("nan")
                v_pool[blk, :, L % S:, :] = float("nan")

    return {
        "cfg": cfg,
        "seed": seed,
        "mode": mode,
        "q": q.to(dt).contiguous(),
        "k_pool": k_pool.contiguous(),
        "v_pool": v_pool.contiguous(),
        "page_table": page_table.to(dev).contiguous(),
        "seq_lens": torch.tensor(lens, dtype=torch.int32, device=dev),
        "num_blocks": nb,
    }


def resample_q_rows(case: dict, rows, attempt: int) -> None:
    """Redraw q for the given (b, kv_group) rows in place (margin enforcement).

    The new draw for row (b, g) depends only on (seed, b, g, attempt), never on which
    other rows were redrawn, so the procedure is reproducible.
    """
    cfg = case["cfg"]
    G, d = cfg.group, cfg.head_dim
    q = case["q"]
    for (b, g) in rows:
        gen = torch.Generator(device="cpu")
        gen.manual_seed(sub_seed(case["seed"], "qre", int(b), int(g), int(attempt)))
        if case.get("mode", "clustered") == "int":
            new = torch.randint(-4, 5, (G, d), generator=gen).to(torch.float32)
        else:
            new = torch.randn((G, d), generator=gen, dtype=torch.float32)
        q[b, g * G:(g + 1) * G, :] = new.to(q.dtype).to(q.device)


def algorithmic_bytes(cfg: Config, seq_lens, out_bytes: int = 4, kv: str = "") -> dict:
    """Bytes the method must move per decode step, by term.

    Counts: metadata of every page (2*d*e per (page, kv-head)), the K and V rows of the
    valid tokens of the selected pages (upper bound: K_b full pages, last page partial),
    q in, o (fp32) + lse out, the page-table row and the selected ids.  Pure bookkeeping
    over shapes; no scores are computed here (selected token count uses the worst case
    that the partial last page is selected, which is what the kernels read).
    """
    e = 2 if cfg.dtype == "bf16" else 4
    S, d, Hkv, Hq = cfg.page_size, cfg.head_dim, cfg.num_kv_heads, cfg.num_q_heads
    # bytes of one stored K (or V) row: d elements, or d E4M3 codes + 1 exponent byte for
    # an FP8 cache (reading R21; q and metadata stay bf16)
    row = d + 1 if kv == "fp8" else d * e
    meta = kv = pt = ids = 0
    for L in seq_lens:
        L = int(L)
        P = -(-L // S)
        K = min(P, max(1, cfg.budget_tokens // S))
        meta += Hkv * P * 2 * d * e
        toks = min(K * S, L)
        kv += Hkv * toks * 2 * row
        pt += P * 4
        ids += Hkv * K * 4
    B = len(seq_lens)
    qo = B * Hq * d * e + B * Hq * (d + 1) * out_bytes
    return {"meta": meta, "kv": kv, "q_o": qo, "page_table": pt, "ids": ids,
            "total": meta + kv + qo + pt + ids}


def drift_queries(q0: torch.Tensor, steps: int, alpha: float, seed: int) -> torch.Tensor:
    """A decode-time query stream with temporal locality (SPEC's
    "drifting" trace mode): q_0 = q0 and
        q_t = sqrt(1 - alpha^2) * q_{t-1} + alpha * z_t,   z_t ~ N(0, I)  (fp32, then cast),
    so every q_t keeps unit variance per channel and consecutive queries are correlated with
    coefficient sqrt(1 - alpha^2).  alpha = 0: a constant query; alpha = 1: independent
    queries.  Returns [steps][*q0.shape] in q0's dtype, on q0's device."""
    g = _gen(seed, ("drift", float(alpha)), q0.device)
    out = torch.empty((steps,) + tuple(q0.shape), dtype=q0.dtype, device=q0.device)
    cur = q0.to(torch.float32)
    keep = math.sqrt(max(0.0, 1.0 - alpha * alpha))
    for t in range(steps):
        if t:
            z = torch.randn(q0.shape, generator=g, device=q0.device, dtype=torch.float32)
            cur = keep * cur + alpha * z
        out[t] = cur.to(q0.dtype)
    return out
