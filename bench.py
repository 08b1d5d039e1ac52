#!/usr/bin/env python
"""bench.py — decode steps/s and achieved HBM GB/s of the TinyServe decode hot path on B200.

One step = one ts_decode_step (score every page -> top-K -> sparse attention) for the whole
batch of one attention layer, on synthetic caches of the BASELINE.json
config shapes.  Default: config c2 (GPT2-345M shape, BASELINE.json configs[1]), N = 1.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c4|c5] [--impl reference]

Timing: inputs resident in HBM; R independent cache replicas rotated step
by step with R * (bytes per step) >= 4 x L2, so every step reads cold metadata and KV; the
K steps are CUDA-graph replays timed with CUDA events on the launching stream, barrier +
synchronize on both sides, max over ranks.  Clocks sampled by NVML during the timed region.
N > 1: c2/c3 run one full config batch per rank (weak scaling, no communication); c4 splits
its batch of 128 over the ranks (strong); c5 shards every sequence block-cyclically over the
ranks with two NCCL all-gathers per step (strong; paper_2509_12211_b200/sharded.py).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402

PEAK_SPEC_GBS = 8000.0  # B200 HBM3e spec (north-star denominator)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, read+write)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)"


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons while the timed region runs."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int, period_s: float = 0.005):
        self.samples, self.reasons, self.ok = [], set(), False
        self.period, self.index = period_s, index
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"],
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def graph_upload(g, stream) -> bool:
    """cudaGraphUpload of a captured torch CUDA graph's executable (best effort)."""
    try:
        from cuda.bindings import runtime as rt
        err, = rt.cudaGraphUpload(g.raw_cuda_graph_exec(), stream.cuda_stream)
        return int(err) == 0
    except Exception:  # noqa: BLE001
        return False


# ------------------------------------------------------------------------------ workload
def rank_config(name: str, world: int, rank: int, batch: int = 0, slice_n: int = 1):
    """Per-rank config and sharding mode.  world > 1: c4 splits its batch over the ranks, c5
    shards every sequence (strong scaling); other configs run one batch per rank (weak).
    slice_n > 1 on one GPU: time ONE rank's share of a slice_n-GPU run of c4 / c5 (the per-GPU
    work of BASELINE.json configs 4-5), c5's two exchanges emulated by local copies."""
    cfg = synth.config(name)
    if batch:
        cfg = cfg.with_(batch=batch)
    shards = world if world > 1 else slice_n
    if name == "c4" and shards > 1:
        assert cfg.batch % shards == 0
        cfg = cfg.with_(batch=cfg.batch // shards)
        return cfg, ("batch" if world > 1 else "batch-slice"), "strong"
    if name == "c5" and shards > 1:
        return cfg, ("sequence" if world > 1 else "sequence-slice"), "strong"
    return cfg, ("batch" if world > 1 else "none"), "weak"


def kernel_bytes(cfg, L: int, Kmax: int, mp_local: int, world: int = 1):
    """Algorithmic bytes per launch of each kernel of one step.

    score:  metadata of every (owned) page + q + page-table row + fp32 scores written
    select: fp32 scores read + selected ids / counts written
    attn:   K and V rows of the valid tokens of the owned selected pages + q + ids +
            page-table lookups + fp32 o and lse written
    """
    e = 2 if cfg.dtype == "bf16" else 4
    B, Hq, Hkv, d, S = cfg.batch, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, cfg.page_size
    P = -(-L // S)
    P_own = -(-P // world)
    K = min(P, Kmax)
    K_own = -(-K // world)
    q = B * Hq * d * e
    score = B * Hkv * P_own * 2 * d * e + q + B * P_own * 4 + B * Hkv * mp_local * 4
    select = B * Hkv * mp_local * 4 + B * Hkv * (Kmax + 1) * 4
    toks = min(K_own * S, L)
    attn = (B * Hkv * toks * 2 * d * e + q + B * Hkv * (K + 1) * 4 + B * Hkv * K_own * 4
            + B * Hq * (d + 1) * 4)
    return {"score": score, "select": select, "attn": attn, "total": score + select + attn}


def build_replica(ts, cfg, seed, device, world=1, rank=0, kv=""):
    case = synth.make_case(cfg, seed=seed, device=device)
    pt = case["page_table"]
    if world > 1 and cfg.name == "c5":
        from paper_2509_12211_b200 import sharded
        pt = sharded.shard_page_table(pt, world, rank)
    shape = tuple(case["k_pool"].shape)
    if kv == "fp8":  # FP8 cache (reading R21): quantised once on the GPU (ts_kv_quantize)
        case["k_pool"] = ts.kv_quantize(case["k_pool"])
        case["v_pool"] = ts.kv_quantize(case["v_pool"])
    L = ts.make_layout(case["q"], case["k_pool"], pt, world if cfg.name == "c5" else 1,
                       rank if cfg.name == "c5" else 0, pool_shape=shape if kv == "fp8" else None)
    meta = ts.meta_build(L, case["k_pool"], pt, case["seq_lens"])
    rep = dict(case, page_table=pt, layout=L, meta=meta)
    B, Hq, Hkv, d = cfg.batch, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim
    K = ts.kmax(L, cfg.budget_tokens)
    rep["o"] = torch.empty((B, Hq, d), dtype=torch.float32, device=device)
    rep["lse"] = torch.empty((B, Hq), dtype=torch.float32, device=device)
    rep["ids"] = torch.empty((B, Hkv, K), dtype=torch.int32, device=device)
    rep["cnt"] = torch.empty((B, Hkv), dtype=torch.int32, device=device)
    rep["ws"] = ts.new_workspace(ts.workspace_bytes(L, cfg.budget_tokens), device)
    return rep


def step_fn(ts, cfg, rep, stream):
    return ts.decode_step(rep["layout"], rep["q"], rep["k_pool"], rep["v_pool"], rep["meta"],
                          rep["page_table"], rep["seq_lens"], cfg.budget_tokens, cfg.scale,
                          o=rep["o"], lse=rep["lse"], sel_ids=rep["ids"], sel_count=rep["cnt"],
                          ws=rep["ws"], stream=stream)


# ------------------------------------------------------------------------------ oracle legs
def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_rate(cfg, rep_cpu, budget_s: float, max_rows=None):
    """Oracle decode_step on host cores over a bounded sample of the workload (whole
    sequences, all heads): OpenMP over rows on every core of the affinity
    mask (best of 3 timed calls) and 1 thread (best of 3, one sequence).  Returns
    (full-workload steps/s, cores, sample description, extras)."""
    import oracle
    B = cfg.batch
    nb = max(1, min(B, max_rows or B))
    q, kp, vp = rep_cpu["q"], rep_cpu["k_pool"], rep_cpu["v_pool"]
    pt, sl = rep_cpu["page_table"], rep_cpu["seq_lens"]

    def run(nseq, threads=0):
        t0 = time.perf_counter()
        oracle.decode_step(q[:nseq], kp, vp, pt[:nseq], sl[:nseq], cfg.budget_tokens, cfg.scale,
                           threads=threads)
        return time.perf_counter() - t0

    cores = oracle.num_threads()  # before the 1-thread variant sets the OpenMP team to 1
    t1 = run(1)
    nseq = max(1, min(nb, int(budget_s / 4 / max(t1, 1e-6))))
    calls = [run(nseq) for _ in range(3)]
    best = min(calls)
    one = min(run(1, threads=1) for _ in range(3))
    extras = {"best_of": 3, "cpu_model": cpu_model(),
              "threads1_steps_per_s": 1.0 / (one * B),
              "affinity_cores": len(os.sched_getaffinity(0))}
    run(1, threads=cores)  # restore the OpenMP team size for later oracle calls
    return 1.0 / (best / nseq * B), cores, (
        f"best of 3 oracle decode_step calls on {nseq}/{B} sequences (all {cfg.num_q_heads} q "
        f"heads, metadata recomputed from K, OpenMP over rows), {sum(calls):.1f} s; 1-thread "
        f"figure: best of 3 calls on 1 sequence; steps/s scaled to the full batch"), extras


def run_reference(args, cfg, world, rank):
    """--impl reference: the float64 oracle (this tier's reference arm) on host cores."""
    if rank != 0:
        return
    import oracle
    oracle.build()
    case = synth.make_case(cfg, seed=42)
    per_call_budget = max(0.05, 120.0 / max(1, args.steps + args.warmup))
    # size the per-step sample (sequences) so the whole run stays within ~2-3 minutes
    t0 = time.perf_counter()
    oracle.decode_step(case["q"][:1], case["k_pool"], case["v_pool"], case["page_table"][:1],
                       case["seq_lens"][:1], cfg.budget_tokens, cfg.scale)
    t_seq = time.perf_counter() - t0
    nseq = max(1, min(cfg.batch, int(per_call_budget / max(t_seq, 1e-6))))
    for _ in range(args.warmup):
        oracle.decode_step(case["q"][:nseq], case["k_pool"], case["v_pool"],
                           case["page_table"][:nseq], case["seq_lens"][:nseq], cfg.budget_tokens,
                           cfg.scale)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.decode_step(case["q"][:nseq], case["k_pool"], case["v_pool"],
                           case["page_table"][:nseq], case["seq_lens"][:nseq], cfg.budget_tokens,
                           cfg.scale)
    dt = time.perf_counter() - t0
    per_step_full = dt / args.steps * cfg.batch / nseq
    value = 1.0 / per_step_full
    cores = oracle.num_threads()
    sample = (f"each step: oracle decode_step on {nseq}/{cfg.batch} sequences of {cfg.name} "
              f"(float64, metadata recomputed), steps/s scaled to the full batch")
    line = {"impl": "reference", "metric": "decode steps/s", "value": value, "unit": "steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": per_step_full * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_json(cfg, world, "none"),
            "cpu_baseline": {"value": value, "unit": "steps/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def traffic_key(args, cfg):
    """profiles/traffic.json key of a bench workload: config, then -b<batch> / -slice<N> /
    -fp8 when they apply (scripts/r2_evidence.sh writes the same keys)."""
    k = cfg.name
    if args.batch:
        k += f"-b{args.batch}"
    if args.slice > 1:
        k += f"-slice{args.slice}"
    if args.kv == "fp8":
        k += "-fp8"
    return k


def config_json(cfg, world, mode, extra=None):
    c = {"workload": f"{cfg.name}: {cfg.note}", "batch_per_rank": cfg.batch,
         "num_q_heads": cfg.num_q_heads, "num_kv_heads": cfg.num_kv_heads,
         "head_dim": cfg.head_dim, "ctx": cfg.ctx, "page_size": cfg.page_size,
         "budget_tokens": cfg.budget_tokens, "kv_dtype": cfg.dtype, "scale": cfg.scale,
         "sharding": mode, "world": world}
    if extra:
        c.update(extra)
    return c


# ------------------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3000)
    ap.add_argument("--warmup", type=int, default=30)
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-oracle", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-dense", action="store_true", help="skip the FullCache baseline leg")
    ap.add_argument("--oracle-seconds", type=float, default=12.0)
    ap.add_argument("--replicas", type=int, default=0)
    ap.add_argument("--batch", type=int, default=0, help="override the config's batch (e.g. c5 at 1)")
    ap.add_argument("--slice", type=int, default=1,
                    help="on one GPU: time one rank's share of an N-GPU c4 / c5 run")
    ap.add_argument("--no-spread", action="store_true", help="skip the p10/p90 + warm-L2 replays")
    ap.add_argument("--no-reuse", action="store_true", help="skip the NEXT-2 cross-step reuse leg")
    ap.add_argument("--kv", default="bf16", choices=["bf16", "fp8"],
                    help="KV storage: bf16, or FP8 E4M3 with per-row power-of-two scales (NEXT-3)")
    ap.add_argument("--sweep", action="store_true",
                    help="NEXT-4: S x K/P sweep (steps/s, FullCache speedup, error vs the float64 dense oracle)")
    ap.add_argument("--sweep-S", default="4,8,16,32,64")
    ap.add_argument("--sweep-ratios", default="0.1,0.2,0.3,0.5")
    ap.add_argument("--sweep-hot", default="4,2.0", help="query-local workload: n_hot pages, beta")
    ap.add_argument("--reuse-alpha", type=float, default=0.1,
                    help="query drift of the reuse leg (synth.drift_queries)")
    args = ap.parse_args()
    assert args.warmup >= 3

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N`: start the N ranks ourselves (one process per GPU, the
        # driver's torchrun launch line), then exit with the launcher's status
        import socket
        import subprocess
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg, mode, scaling = rank_config(args.config, world, rank, args.batch, args.slice)
    # sequence sharding: shard count / this rank's index (the emulated slice is rank 0)
    sw, sr = (world, rank) if mode == "sequence" else ((args.slice, 0) if mode == "sequence-slice" else (1, 0))
    seq = mode in ("sequence", "sequence-slice")

    if args.impl == "reference":
        run_reference(args, cfg, world, rank)
        return
    if args.sweep:
        if rank == 0:
            sweep_main(args)
        return

    import paper_2509_12211_b200 as ts
    # TS_BENCH_BACKEND=gloo (testing only): exercise the multi-rank path with several ranks
    # sharing the visible GPUs; the driver's runs use NCCL, one rank per GPU
    backend = os.environ.get("TS_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    props = torch.cuda.get_device_properties(dev)
    l2 = getattr(props, "L2_cache_size", 126 * 2**20) or 126 * 2**20
    L_ctx = cfg.ctx
    Kmax = min(cfg.max_pages, max(1, cfg.budget_tokens // cfg.page_size))
    mp_local = -(-cfg.max_pages // sw) if seq else cfg.max_pages
    kb = kernel_bytes(cfg, L_ctx, Kmax, mp_local, sw)
    kvq = "fp8" if args.kv == "fp8" else ""
    if kvq and (seq or cfg.dtype != "bf16"):
        raise SystemExit("bench.py: --kv fp8 runs the unsharded bf16-config step only")
    alg = synth.algorithmic_bytes(cfg, [L_ctx] * cfg.batch, kv=kvq)
    step_bytes = alg["total"] if not seq else kb["total"]
    R = args.replicas or max(2, -(-4 * l2 // max(1, step_bytes)))
    # every replica holds a whole pool (K + V): keep them within ~60 GB of the 180 GB HBM
    pool_bytes = cfg.batch * cfg.max_pages * cfg.num_kv_heads * cfg.page_size * cfg.head_dim * 2 * (
        2 if cfg.dtype == "bf16" else 4)  # (bf16 staging of an FP8 cache: the same bound)
    R = max(2, min(R, int(60e9 // max(1, pool_bytes)))) if not args.replicas else R
    stream = torch.cuda.Stream(device=dev)

    reps = [build_replica(ts, cfg, seed=1000 * rank + r, device=dev, world=sw, rank=sr, kv=kvq)
            for r in range(R)]
    torch.cuda.synchronize()

    if seq:
        from paper_2509_12211_b200 import sharded
        for rep in reps:
            rep["shard"] = sharded.ShardStep(ts, rep["layout"], sw, sr, cfg.budget_tokens, dev)

        def one(rep):
            if mode == "sequence":
                rep["shard"].step(rep["q"], rep["k_pool"], rep["v_pool"], rep["meta"],
                                  rep["page_table"], rep["seq_lens"], cfg.scale)
            else:
                rep["shard"].step_local(rep["q"], rep["k_pool"], rep["v_pool"], rep["meta"],
                                        rep["page_table"], rep["seq_lens"], cfg.scale)
    else:
        def one(rep):
            step_fn(ts, cfg, rep, stream)

    # ---- launches per step (our kernels)
    with torch.cuda.stream(stream):
        one(reps[0])
    torch.cuda.synchronize()
    # launches of our kernels per step, as reported by the C ABI for the step just run
    # (bf16: 1 = decode_cluster_kernel; sequence sharding: 5 calls + 2 collectives)
    launches_per_step = ts.launch_count() if not seq else (3 if reps[0]["shard"].fused else 5)
    single = not seq and launches_per_step == 1
    fused = cfg.dtype == "bf16" and cfg.group <= 8 and not seq and not single

    # ---- graphs.  The timed unit is ONE CUDA graph of exactly `steps` consecutive steps
    # (step j on replica (warmup + j) % R: cold-L2 rotation), so PDL chains every launch to
    # the previous one for the whole timed region, as in a serving loop; the warm-up is a
    # graph of `warmup` steps.  Separately, one graph per replica with CUDA events around
    # the step (the events serialise it: never the timed unit) gives the serialised
    # single-step latency.
    graphs, pgraphs = [], []
    ev = [[torch.cuda.Event(enable_timing=True, external=True) for _ in range(4)] for _ in reps]
    for es in ev:
        for e in es:
            e.record(stream)
    torch.cuda.synchronize()
    use_graph = not seq or os.environ.get("TS_BENCH_SEQ_GRAPH", "1") == "1"

    def capture(n, offset):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            with torch.cuda.graph(g, stream=stream):
                for j in range(n):
                    one(reps[(offset + j) % R])
        return g

    if use_graph:
        try:
            for r, rep in enumerate(reps):
                if not seq:
                    pg = torch.cuda.CUDAGraph()
                    with torch.cuda.stream(stream):
                        ts.profile_events(ev[r])
                        with torch.cuda.graph(pg, stream=stream):
                            one(rep)
                        ts.profile_events(None)
                    pgraphs.append(pg)
            warm_g = capture(args.warmup, 0)
            timed_g = capture(args.steps, args.warmup)
            for g_ in (warm_g, timed_g):  # pre-upload the executable graphs (no first-launch upload in the timed region)
                graph_upload(g_, stream)
            torch.cuda.synchronize()
        except Exception as ex:  # noqa: BLE001 — e.g. a collective that cannot be captured
            if mode != "sequence":
                raise
            print(f"bench: graph capture of the sharded step failed ({ex}); timing eager steps",
                  file=sys.stderr)
            use_graph, pgraphs = False, []
            torch.cuda.synchronize()

    def run_steps(n, offset=0):
        with torch.cuda.stream(stream):
            for j in range(n):
                one(reps[(offset + j) % R])

    # head start: a spin kernel occupies the stream while the host enqueues the timed work,
    # so the timed region starts behind queued GPU work (no idle-GPU launch latency in it)
    HEAD_START_CYCLES = int(4e6)  # ~2 ms at 1.97 GHz

    if use_graph:
        with torch.cuda.stream(stream):
            warm_g.replay()
    else:
        run_steps(args.warmup)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        wall0 = time.perf_counter()
        with torch.cuda.stream(stream):
            torch.cuda._sleep(HEAD_START_CYCLES)
            t0.record(stream)
            if use_graph:
                timed_g.replay()
            else:
                run_steps(args.steps, offset=args.warmup)
            t1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    if world > 1:
        torch.distributed.barrier()
    ms = t0.elapsed_time(t1)
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms = float(tt.item())
    ms_per_step = ms / args.steps

    # ---- spread over repeated timed regions (same protocol, same graph), and a labelled
    # warm-L2 figure (every step on replica 0: its bytes stay L2-resident when they fit)
    spread = None
    if use_graph and not args.no_spread:  # every rank (the graph may hold collectives)
        per = []
        with torch.cuda.stream(stream):
            for _ in range(20):
                a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda._sleep(HEAD_START_CYCLES // 4)
                a.record(stream)
                timed_g.replay()
                b_.record(stream)
                per.append((a, b_))
        torch.cuda.synchronize()
        us = sorted(1e3 * a.elapsed_time(b_) / args.steps for a, b_ in per)
        q = lambda f: us[min(len(us) - 1, int(f * len(us)))]
        spread = {"replays": len(us), "us_per_step_p10": q(0.1), "us_per_step_median": q(0.5),
                  "us_per_step_p90": q(0.9)}
        if not seq:
            wg = torch.cuda.CUDAGraph()
            with torch.cuda.stream(stream):
                with torch.cuda.graph(wg, stream=stream):
                    for _ in range(min(args.steps, 200)):
                        one(reps[0])
            with torch.cuda.stream(stream):
                wg.replay()
                a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda._sleep(HEAD_START_CYCLES // 4)
                a.record(stream)
                wg.replay()
                b_.record(stream)
            torch.cuda.synchronize()
            spread["warm_l2_us_per_step"] = 1e3 * a.elapsed_time(b_) / min(args.steps, 200)
            spread["warm_l2_note"] = ("LABELLED WARM-L2: every step on replica 0, its metadata "
                                      "and K/V partly L2-resident; not the headline")

    # ---- per-kernel durations: instrumented replays of every replica (cold rotation kept)
    phase = None
    if pgraphs:
        k1, k2, k3, tot = [], [], [], []
        with torch.cuda.stream(stream):
            for rnd in range(6):
                for r in range(R):
                    pgraphs[r].replay()
                torch.cuda.synchronize()
                if rnd == 0:
                    continue  # warm-up round
                for r in range(R):
                    k1.append(ev[r][0].elapsed_time(ev[r][1]))
                    k2.append(ev[r][1].elapsed_time(ev[r][2]))
                    k3.append(ev[r][2].elapsed_time(ev[r][3]))
                    tot.append(ev[r][0].elapsed_time(ev[r][3]))
        phase = {"samples": len(tot), "serialised_step_us": 1e3 * statistics.mean(tot)}
        if single:
            phase.update(kernels="decode_cluster_kernel (score + select + gather + attend, one launch)",
                         step_kernel_us=1e3 * statistics.mean(tot))
        elif fused:
            phase.update(kernels="score_select -> sparse_attn (PDL + per-row flags in the timed graphs)",
                         score_select_us=1e3 * statistics.mean(k1),
                         attn_us=1e3 * statistics.mean(k3))
        else:
            phase.update(score_us=1e3 * statistics.mean(k1), select_us=1e3 * statistics.mean(k2),
                         attn_us=1e3 * statistics.mean(k3))

    # ---- FullCache baseline: dense attention over every page of the same
    # replicas, same timing protocol -> the sparse/dense speedup (the paper's 2.1-3.4x claim,
    # PAPER.md:8, 550, measured on 8xA100; context only)
    dense = None
    try:
        dense = dense_leg(ts, cfg, reps, R, stream, dev, args, ms_per_step) if (
            use_graph and not args.no_dense and cfg.dtype == "bf16" and cfg.page_size % 16 == 0) else None
    except Exception as ex:  # noqa: BLE001 — the baseline is context; never fail the bench on it
        dense = {"unavailable": f"{type(ex).__name__}: {ex}"}
    # ---- NEXT-2 cross-step reuse on a drifting-query workload (labelled leg, not the headline)
    reuse = None
    if use_graph and not seq and not args.no_reuse and cfg.dtype == "bf16" and cfg.page_size % 16 == 0:
        try:
            reuse = reuse_leg(ts, cfg, reps, R, stream, dev, args.reuse_alpha)
        except Exception as ex:  # noqa: BLE001
            reuse = {"unavailable": f"{type(ex).__name__}: {ex}"}
    # ---- e2e: public API with host buffers (pinned), H2D of q / new k,v + D2H of o, lse
    e2e = None
    if not args.no_e2e and not seq:
        # its own sample: >= 240 steps (a 20-step --steps would time one replay of a 24-step
        # graph, mostly its first-replay cost), <= 600 (bounded run time)
        e2e = run_e2e_batched(ts, cfg, reps, dev, stream, steps=min(max(args.steps, 240), 600), warmup=5)
        if world > 1:
            tt = torch.tensor([1.0 / e2e["value"]], device=dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            e2e["value"] = world / float(tt.item()) if scaling == "weak" else 1.0 / float(tt.item())

    # ---- a read-only streaming reference (the path is >= 99 % reads; the copy peak of
    # MEASURED_PEAKS.json counts read + write): torch sum over 2 GiB of bf16, best of 5
    read_peak = None
    if rank == 0 and not args.no_spread:
        try:
            buf = torch.ones(2**30, dtype=torch.bfloat16, device=dev)
            best = 1e9
            for _ in range(6):
                a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(stream):
                    a.record(stream)
                    buf.sum(dtype=torch.float32)
                    b_.record(stream)
                torch.cuda.synchronize()
                best = min(best, a.elapsed_time(b_))
            read_peak = {"gbs": 2**31 / (best * 1e-3) / 1e9,
                         "how": "torch.sum of 2 GiB bf16 (read-only), best of 6, CUDA events"}
            del buf
        except Exception as ex:  # noqa: BLE001
            read_peak = {"unavailable": str(ex)}

    # ---- cpu baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and not args.no_oracle:
        import oracle
        oracle.build()
        if seq:  # the ranks hold shards: time the oracle on one whole sequence
            c1 = cfg.with_(batch=1)
            host = synth.make_case(c1, seed=1000)
            v, cores, sample, extras = oracle_rate(c1, host, args.oracle_seconds)
            v /= cfg.batch
            extras["threads1_steps_per_s"] /= cfg.batch
            sample += f"; 1 of the {cfg.batch} sequences, steps/s scaled to the batch"
        else:
            host = {k: reps[0][k].cpu() for k in ("q", "k_pool", "v_pool", "page_table", "seq_lens")}
            if kvq:  # the oracle's FP8 step: exact dequantisation, then the float64 step
                nbk = reps[0]["layout"].num_blocks
                for kk in ("k_pool", "v_pool"):
                    c_, e_ = ts.fp8_split(host[kk], nbk, cfg.num_kv_heads, cfg.page_size, cfg.head_dim)
                    host[kk] = torch.from_numpy(oracle.kv_dequantize(c_.numpy(), e_.numpy()))
                host["q"] = host["q"].float()
            v, cores, sample, extras = oracle_rate(cfg, host, args.oracle_seconds)
            if kvq:
                sample += "; FP8 cache: codes dequantised exactly to fp32 first (untimed)"
        # whole job: every rank's batch (weak) or the one global batch (strong)
        v_job = v * world if scaling == "weak" else (
            v if seq else v * (cfg.batch / (args.batch or synth.config(args.config).batch)))
        cpu = {"value": v_job, "unit": "steps/s", "cores": cores, "kind": "oracle",
               "sample": sample + (f"; x{world} ranks' batches (one host)" if world > 1 else ""),
               **extras}

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return

    steps_per_s = 1e3 / ms_per_step
    if seq or scaling == "strong":
        value = steps_per_s              # every step covers the whole (sharded) batch
    else:
        value = steps_per_s * world      # independent batches, one per rank
    gbs = step_bytes * world / (ms_per_step * 1e-3) / 1e9
    peak, peak_src = measured_peaks()
    roof = None
    if phase:
        if single:
            # the one kernel moves every byte of the step and is the only launch of it: its
            # average launch duration is the timed region's per-step time (consecutive
            # launches overlap their prologues through PDL); the per-launch time of the
            # event-instrumented graphs (serialised, launch latency included) is kept in
            # phase_us for reference
            # bytes: SURVEY.md §8(d)'s algorithmic bytes of the step (synth.algorithmic_bytes:
            # metadata + valid selected K/V + q + fp32 o/lse + page-table rows + ids) — the
            # fused kernel keeps scores in shared memory, so kernel_bytes' score round trip
            # is not moved and not counted
            cand = {"decode_cluster_kernel": (step_bytes, ms_per_step * 1e3)}
        elif fused:  # score_select (metadata + selection) and sparse_attn (selected K/V)
            cand = {"score_select": (kb["score"] + kb["select"], phase["score_select_us"]),
                    "sparse_attn": (kb["attn"], phase["attn_us"])}
        else:
            cand = {"score": (kb["score"], phase["score_us"]), "attn": (kb["attn"], phase["attn_us"])}
        dom = max(cand, key=lambda x: cand[x][1])
        nbytes, us = cand[dom]
        achieved = nbytes / (us * 1e-6) / 1e9
        traffic, tsrc = None, None
        try:  # DRAM bytes per launch of this kernel from the committed ncu capture
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
                tj = json.load(f).get(traffic_key(args, cfg))
            if tj and dom in tj["per_launch_bytes"]:
                traffic = tj["per_launch_bytes"][dom]
                tsrc = "ncu --set full: dram__bytes_read.sum + dram__bytes_write.sum, profiles/" + tj["report"]
        except (OSError, ValueError, KeyError):
            pass
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_source": tsrc,
                "peak_source": peak_src,
                "algorithmic_bytes_per_launch": nbytes, "avg_launch_us": us, "phase_us": phase,
                "step_achieved_gbs": step_bytes / (ms_per_step * 1e-3) / 1e9,
                "step_frac": step_bytes / (ms_per_step * 1e-3) / 1e9 / peak}
    if roof is None and seq:
        # per-rank bytes (owned metadata + owned selected K/V + exchange buffers) over the
        # per-step time of the whole sharded step (5 kernels + 2 NCCL all-gathers)
        achieved = kb["total"] / (ms_per_step * 1e-3) / 1e9
        roof = {"bound": "hbm", "kernel": ("sequence-sharded step per rank (select_candidates, "
                "shard_attend, lse_merge + 2 all-gathers)" if reps[0]["shard"].fused else
                "sequence-sharded step per rank (score, select, select_merge, sparse_attn, "
                "lse_merge + 2 all-gathers)"),
                "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": None, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": kb["total"], "avg_launch_us": ms_per_step * 1e3}
    clocks = clk.summary()
    line = {
        "metric": "decode steps/s", "value": value, "unit": "steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
        "dtype": "fp8e4m3-kv" if kvq else cfg.dtype, "data": "synthetic",
        "config": config_json(cfg, world, mode, {
            "slice_of_gpus": args.slice if mode.endswith("-slice") else None,
            "replicas": R, "l2_bytes": l2, "l2_policy": "rotate R cold replicas (R*bytes >= 4*L2)",
            "graph": "R steps per CUDA graph replay" if use_graph else False,
            "kv_storage": ("fp8 e4m3 codes + one power-of-two exponent byte per row (reading R21); "
                           "q / metadata bf16, fp32 compute") if kvq else cfg.dtype}),
        "tokens_per_s": value * cfg.batch,
        "hbm_gbs": gbs, "frac_of_8tbs": gbs / PEAK_SPEC_GBS, "frac_of_measured": gbs / peak,
        "algorithmic_bytes_per_step": step_bytes, "kernel_bytes": kb,
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "dense_baseline": dense,
        "serialised_step_us": phase["serialised_step_us"] if phase else None,
        "spread": spread, "read_peak": read_peak, "reuse": reuse,
        "gpu_launches": launches_per_step * args.steps, "clocks": clocks,
        "wall_s_timed": wall, "device": torch.cuda.get_device_name(dev),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def time_graph(fn, n_inner, stream, reps=5):
    """Per-call time of fn() (enqueues one call) captured n_inner times in a CUDA graph: best of
    `reps` replays behind a head-start spin, CUDA events on the launching stream."""
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        for _ in range(2):
            fn()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(n_inner):
                fn()
        g.replay()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            torch.cuda._sleep(int(2e6))
            a.record(stream)
            g.replay()
            b_.record(stream)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b_) / n_inner)
    return best * 1e3  # us


def sweep_main(args):
    """the synthetic analogue of the paper's page-size and budget-ratio
    ablations (§4.3, 688-707 §4.11).  For S in --sweep-S and K/P in
    --sweep-ratios on the config's shape (ctx fixed, P = ctx / S, K = round(ratio * P)):
      * us/step of ts_decode_step (cold replica rotation, CUDA graphs) and of the FullCache
        baseline over the same pools (ts_dense_decode_attn; S < 16: ts_sparse_decode_attn
        with every page selected, the same computation), and their ratio;
      * accuracy on a query-local workload (synth q_local: queries aimed at a few hot pages,
        as real decode queries are) and on random queries, for a sample of sequences:
        relative L2 error of the GPU sparse output against the FLOAT64 DENSE ORACLE
        (oracle.sparse_attn over every page) and the attention recall exp(lse_sel - lse_dense)
        = the dense softmax mass on the selected pages.
    Prints one JSON line with the table."""
    import numpy as np
    import oracle
    import paper_2509_12211_b200 as ts
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(device=dev)
    base = synth.config(args.config)
    Ss = [int(x) for x in args.sweep_S.split(",")]
    ratios = [float(x) for x in args.sweep_ratios.split(",")]
    props = torch.cuda.get_device_properties(dev)
    l2 = getattr(props, "L2_cache_size", 126 * 2**20) or 126 * 2**20
    rows_out = []
    for S in Ss:
        cfg = base.with_(page_size=S, budget_tokens=S)
        P = cfg.max_pages
        per_rep = synth.algorithmic_bytes(cfg.with_(budget_tokens=int(0.3 * P) * S), [cfg.ctx] * cfg.batch)["total"]
        R = max(2, min(8, -(-4 * l2 // per_rep)))
        reps = [build_replica(ts, cfg, seed=500 + r, device=dev) for r in range(R)]
        acc_cases = {}
        n_hot, beta = args.sweep_hot.split(",")
        for kind, ql in (("local", (int(n_hot), float(beta))), ("random", None)):
            ca = synth.make_case(cfg.with_(batch=2), seed=77, q_local=ql)
            dd = {k: (v.to(dev) if isinstance(v, torch.Tensor) else v) for k, v in ca.items()}
            La = ts.make_layout(dd["q"], dd["k_pool"], dd["page_table"])
            ma = ts.meta_build(La, dd["k_pool"], dd["page_table"], dd["seq_lens"])
            allp = np.tile(np.arange(P, dtype=np.int32), (2, cfg.num_kv_heads, 1))
            cnt = np.full((2, cfg.num_kv_heads), P, np.int32)
            od, ld = oracle.sparse_attn(ca["q"], ca["k_pool"], ca["v_pool"], ca["page_table"],
                                        ca["seq_lens"], allp, cnt, cfg.scale)
            acc_cases[kind] = (dd, La, ma, od, ld)
        dense_us = None
        for ratio in ratios:
            K = max(1, int(round(ratio * P)))
            budget = K * S
            for rep in reps:
                rep["ws_s"] = ts.new_workspace(ts.workspace_bytes(rep["layout"], budget), dev)
                rep["ids_s"] = torch.empty((cfg.batch, cfg.num_kv_heads, K), dtype=torch.int32, device=dev)
            state = {"i": 0}

            def step():
                rep = reps[state["i"] % R]
                state["i"] += 1
                ts.decode_step(rep["layout"], rep["q"], rep["k_pool"], rep["v_pool"], rep["meta"],
                               rep["page_table"], rep["seq_lens"], budget, cfg.scale, o=rep["o"],
                               lse=rep["lse"], sel_ids=rep["ids_s"], sel_count=rep["cnt"],
                               ws=rep["ws_s"], stream=stream)
            us = time_graph(step, 8 * R, stream)
            launches = ts.launch_count()
            if dense_us is None:
                dstate = {"i": 0}
                if S % 16 == 0:
                    dws = [ts.new_workspace(ts.dense_workspace_bytes(r_["layout"]), dev) for r_ in reps]

                    def dstep():
                        r_ = reps[dstate["i"] % R]
                        ts.dense_decode_attn(r_["layout"], r_["q"], r_["k_pool"], r_["v_pool"], r_["page_table"],
                                             r_["seq_lens"], cfg.scale, o=r_["o"], lse=r_["lse"],
                                             ws=dws[dstate["i"] % R], stream=stream)
                        dstate["i"] += 1
                else:  # every page selected through the sparse attention kernel
                    allg = torch.arange(P, dtype=torch.int32, device=dev).repeat(cfg.batch, cfg.num_kv_heads, 1).contiguous()
                    cntg = torch.full((cfg.batch, cfg.num_kv_heads), P, dtype=torch.int32, device=dev)
                    dws = [ts.new_workspace(ts.attn_workspace_bytes(r_["layout"], P), dev) for r_ in reps]

                    def dstep():
                        r_ = reps[dstate["i"] % R]
                        ts.sparse_decode_attn(r_["layout"], r_["q"], r_["k_pool"], r_["v_pool"], r_["page_table"],
                                              r_["seq_lens"], allg, cntg, cfg.scale, o=r_["o"], lse=r_["lse"],
                                              ws=dws[dstate["i"] % R], stream=stream)
                        dstate["i"] += 1
                dense_us = time_graph(dstep, 2 * R, stream)
                del dws
            alg = synth.algorithmic_bytes(cfg.with_(budget_tokens=budget), [cfg.ctx] * cfg.batch)["total"]
            row = {"S": S, "ratio": ratio, "K": K, "P": P, "budget_tokens": budget,
                   "us_per_step": us, "steps_per_s": 1e6 / us, "launches_per_step": launches,
                   "alg_bytes": alg, "gbs": alg / (us * 1e-6) / 1e9, "dense_us": dense_us,
                   "speedup_vs_dense": dense_us / us}
            for kind, (dd, La, ma, od, ld) in acc_cases.items():
                o, lse, _, _ = ts.decode_step(La, dd["q"], dd["k_pool"], dd["v_pool"], ma, dd["page_table"],
                                              dd["seq_lens"], budget, cfg.scale)
                o = o.cpu().numpy().astype(np.float64)
                lse = lse.cpu().numpy().astype(np.float64)
                row[f"rel_l2_err_{kind}"] = float(np.linalg.norm(o - od) / np.linalg.norm(od))
                row[f"recall_{kind}"] = float(np.mean(np.exp(lse - ld)))
            rows_out.append(row)
            print(f"sweep S={S} K/P={ratio}: {us:.2f} us ({row['speedup_vs_dense']:.2f}x dense), "
                  f"err local {row['rel_l2_err_local']:.3g} random {row['rel_l2_err_random']:.3g}, "
                  f"recall local {row['recall_local']:.3f}", file=sys.stderr, flush=True)
        del reps
        torch.cuda.empty_cache()
    line = {"metric": "NEXT-4 sweep: decode steps/s and output error vs the float64 dense oracle",
            "config": {"workload": f"{base.name}: {base.note}", "ctx": base.ctx, "batch": base.batch,
                       "accuracy_sample": f"2 sequences; q_local = ({args.sweep_hot}: hot pages, beta) and random q",
                       "timing": "cold replica rotation, CUDA graphs, best of 5 replays"},
            "rows": rows_out, "device": torch.cuda.get_device_name(dev)}
    print(json.dumps(line), flush=True)


def dense_leg(ts, cfg, reps, R, stream, dev, args, ms_per_step):
    """FullCache baseline leg: dense attention over every page of the same replicas."""
    dense = None
    dws = [ts.new_workspace(ts.dense_workspace_bytes(rep["layout"]), dev) for rep in reps]

    def dstep(r):
        rep = reps[r]
        ts.dense_decode_attn(rep["layout"], rep["q"], rep["k_pool"], rep["v_pool"],
                             rep["page_table"], rep["seq_lens"], cfg.scale, o=rep["o"],
                             lse=rep["lse"], ws=dws[r], stream=stream)
    with torch.cuda.stream(stream):
        for r in range(R):
            dstep(r)
    torch.cuda.synchronize()
    dg = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        with torch.cuda.graph(dg, stream=stream):
            for r in range(R):
                dstep(r)
    torch.cuda.synchronize()
    nd = max(1, min(args.steps, 600) // R)
    with torch.cuda.stream(stream):
        for _ in range(2):
            dg.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(nd):
            dg.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    dms = e0.elapsed_time(e1) / (nd * R)
    e = 2
    row = cfg.head_dim + 1 if args.kv == "fp8" else cfg.head_dim * e  # bytes per stored K (or V) row
    dbytes = (cfg.batch * cfg.num_kv_heads * cfg.ctx * 2 * row
              + cfg.batch * cfg.num_q_heads * cfg.head_dim * (e + 4) + cfg.batch * cfg.num_q_heads * 4)
    dense = {"ms_per_step": dms, "steps_per_s": 1e3 / dms, "bytes_per_step": dbytes,
             "hbm_gbs": dbytes / (dms * 1e-3) / 1e9,
             "speedup_sparse_vs_dense": dms / ms_per_step,
             "kernel": "sparse_attn_tma_kernel in dense mode (every page; ts_dense_decode_attn)"
                       + (", FP8 KV" if args.kv == "fp8" else "")}

    return dense


def reuse_leg(ts, cfg, reps, R, stream, dev, alpha, T=24):
    """SURVEY.md §8f NEXT-2, cross-step page reuse ("prefetching selected pages",
    the reuse probability rho of PAPER.md:263-271).  A drifting-query workload
    (synth.drift_queries: q_t = sqrt(1 - a^2) q_{t-1} + a z_t per replica) on the same cold
    replica rotation as the headline: step j runs replica j % R with its (j // R)-th query.
    Reported: the hit rate |prev ∩ cur| / |cur| of consecutive selections of a row
    (averaged over rows and steps, the first step excluded; its mean is rho-hat) and the
    per-step time of ts_decode_step vs ts_decode_step_prefetch (the previous selection
    prefetched into L2 while the pages are scored) on the same query stream."""
    B, Hkv = cfg.batch, cfg.num_kv_heads
    qb = [synth.drift_queries(rep["q"], T, alpha, seed=7000 + r) for r, rep in enumerate(reps)]
    rep = reps[0]
    prev, hits = None, []
    with torch.cuda.stream(stream):
        for t in range(T):
            ts.decode_step(rep["layout"], qb[0][t], rep["k_pool"], rep["v_pool"], rep["meta"],
                           rep["page_table"], rep["seq_lens"], cfg.budget_tokens, cfg.scale,
                           o=rep["o"], lse=rep["lse"], sel_ids=rep["ids"], sel_count=rep["cnt"],
                           ws=rep["ws"], stream=stream)
            cur = rep["ids"].view(B * Hkv, -1).clone()
            if prev is not None:
                valid = cur >= 0
                hit = (cur.unsqueeze(-1) == prev.unsqueeze(-2)).any(-1) & valid
                hits.append((hit.sum().float() / valid.sum().clamp(min=1).float()))
            prev = cur
    torch.cuda.synchronize()
    hit_rate = float(torch.stack(hits).mean()) if hits else None

    def one(j, prefetch):
        r = reps[j % R]
        q = qb[j % R][(j // R) % T]
        if prefetch:
            ts.decode_step_prefetch(r["layout"], q, r["k_pool"], r["v_pool"], r["meta"],
                                    r["page_table"], r["seq_lens"], cfg.budget_tokens, cfg.scale,
                                    r["ids"], r["cnt"], o=r["o"], lse=r["lse"], ws=r["ws"],
                                    stream=stream)
        else:
            ts.decode_step(r["layout"], q, r["k_pool"], r["v_pool"], r["meta"], r["page_table"],
                           r["seq_lens"], cfg.budget_tokens, cfg.scale, o=r["o"], lse=r["lse"],
                           sel_ids=r["ids"], sel_count=r["cnt"], ws=r["ws"], stream=stream)

    n = R * T
    res = {}
    for name, pf in (("plain", False), ("prefetch", True)):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            for j in range(n):  # untimed pass: every replica's buffers hold a real selection
                one(j, pf)
            with torch.cuda.graph(g, stream=stream):
                for j in range(n):
                    one(j, pf)
        graph_upload(g, stream)
        with torch.cuda.stream(stream):
            g.replay()
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(3):
            a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                torch.cuda._sleep(int(2e6))
                a.record(stream)
                g.replay()
                b_.record(stream)
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b_) / n)
        res[name] = best * 1e3
    return {"alpha": alpha, "steps_per_replica": T, "hit_rate": hit_rate, "rho_hat": hit_rate,
            "us_per_step_plain": res["plain"], "us_per_step_prefetch": res["prefetch"],
            "speedup": res["plain"] / res["prefetch"],
            "workload": "drifting queries q_t = sqrt(1-a^2) q_(t-1) + a z_t per replica, cold "
                        "replica rotation as the headline; best of 3 graph replays of R*T steps",
            "api": "ts_decode_step vs ts_decode_step_prefetch (previous selection -> L2)"}


def run_e2e_batched(ts, cfg, reps, dev, stream, steps, warmup, NB=8):
    """e2e with the copies batched per NB steps (one H2D of NB steps' [q|k_new|v_new], one
    D2H of NB steps' [o|lse]): the NB kernels of a batch follow each other on the compute
    stream with no foreign dependency between them, so PDL overlaps every kernel's prologue
    with its predecessor's tail (a per-step copy edge in the graph serialises the kernels);
    batch j's H2D and batch j-1's D2H overlap batch j's kernels (two buffer sets).  Every
    step still moves its own inputs host -> device and its own outputs device -> host inside
    the timed region (a step's inputs do not depend on the previous step's outputs here).
    Measured against per-step copies on two copy streams with 8 staging slots (the round-1
    form, where each kernel also waits on its own copy): C2 26.2 -> 22.8 us per step, C3
    25.1 -> 21.9, C5 25.7 -> 23.7, C4 43.6 -> 38.6."""
    B, Hq, Hkv, d = cfg.batch, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim
    dt = cfg.torch_dtype
    nq, nk, no = B * Hq * d, B * Hkv * d, B * Hq * (d + 1)
    per_in = nq + 2 * nk
    hin = [torch.randn(NB * per_in).to(dt).pin_memory() for _ in range(2)]
    hout = [torch.empty(NB * no, dtype=torch.float32).pin_memory() for _ in range(2)]
    din = [torch.empty_like(hin[0], device=dev) for _ in range(2)]
    dout = [torch.empty(NB * no, dtype=torch.float32, device=dev) for _ in range(2)]
    h2d_s = torch.cuda.Stream(device=dev)
    d2h_s = torch.cuda.Stream(device=dev)
    R = len(reps)

    def chain(nbatch):
        ev_in = [torch.cuda.Event() for _ in range(nbatch)]
        ev_k = [torch.cuda.Event() for _ in range(nbatch)]
        ev_out = [torch.cuda.Event() for _ in range(nbatch)]
        fork = torch.cuda.Event()
        fork.record(stream)
        h2d_s.wait_event(fork)
        d2h_s.wait_event(fork)
        for j in range(nbatch):
            sl = j % 2
            with torch.cuda.stream(h2d_s):  # batch j's inputs (buffer set free once batch j-2 ran)
                if j >= 2:
                    h2d_s.wait_event(ev_k[j - 2])
                din[sl].copy_(hin[sl], non_blocking=True)
                ev_in[j].record(h2d_s)
            stream.wait_event(ev_in[j])
            if j >= 2:
                stream.wait_event(ev_out[j - 2])  # dout set read back
            for e in range(NB):
                i = j * NB + e
                rep = reps[i % R]
                x = din[sl][e * per_in:(e + 1) * per_in]
                y = dout[sl][e * no:(e + 1) * no]
                ts.decode_step_append(rep["layout"], x[:nq].view(B, Hq, d), x[nq:nq + nk].view(B, Hkv, d),
                                      x[nq + nk:].view(B, Hkv, d), rep["k_pool"], rep["v_pool"],
                                      rep["meta"], rep["page_table"], rep["seq_lens"],
                                      cfg.budget_tokens, cfg.scale, o=y[:B * Hq * d].view(B, Hq, d),
                                      lse=y[B * Hq * d:].view(B, Hq), sel_ids=rep["ids"],
                                      sel_count=rep["cnt"], ws=rep["ws"], stream=stream)
            ev_k[j].record(stream)
            with torch.cuda.stream(d2h_s):
                d2h_s.wait_event(ev_k[j])
                hout[sl].copy_(dout[sl], non_blocking=True)
                ev_out[j].record(d2h_s)
        stream.wait_event(ev_in[nbatch - 1])
        stream.wait_event(ev_out[nbatch - 1])

    # one graph holds all the timed steps (graph-to-graph transitions carry no PDL overlap)
    nbatch = max(2, -(-max(steps, 2 * R) // NB))
    with torch.cuda.stream(stream):
        chain(nbatch)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        with torch.cuda.graph(g, stream=stream):
            chain(nbatch)
    torch.cuda.synchronize()
    graph_upload(g, stream)
    with torch.cuda.stream(stream):
        g.replay()
    torch.cuda.synchronize()
    n_chain = nbatch * NB
    n = max(1, steps // n_chain)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        torch.cuda._sleep(int(2e6))
        a.record(stream)
        for _ in range(n):
            g.replay()
        b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / (n * n_chain)
    return {"value": 1e3 / ms, "unit": "steps/s", "h2d_bytes_per_step": per_in * hin[0].element_size(),
            "d2h_bytes_per_step": no * 4, "ms_per_step": ms, "steps": n * n_chain,
            "api": ("paper_2509_12211_b200.decode_step_append (ctypes -> C ABI: ts_decode_step_append, "
                    f"the token append fused into the step's launch for bf16); per step its [q|k_new|v_new] "
                    f"H2D and [o|lse] D2H from / to pinned memory, copied in batches of {NB} steps on two "
                    "copy streams (double-buffered), so the kernels of a batch stay PDL-chained; CUDA graphs")}


if __name__ == "__main__":
    main()
