#!/usr/bin/env python
"""Benchmark: trained words/sec of skip-gram HS training (BASELINE.json metric).

A "step" is one training pass of the hot path over one GPU's shard of the synthetic
corpus. Default: BASELINE config 5 (the largest single-GPU configuration: 1B tokens of
Zipf(1.2) over a 1M vocabulary, D 300, W 5, sample 1e-5, K 31 -- the reference default,
BASELINE.json leaves it to the K sweep). Inputs (id stream, tree, model) are resident in
HBM before the timed region. Each timed step = K3 subsampling/pair generation + K1
Hogwild training (+ the replicas' delta sync at N > 1). K1 is the library's default
kernel (v8: each center's products on the tensor cores, fp16-rounded operands, fp32 sums,
fp32 model and updates; `dtype` says so); the same step on the all-FP32 kernel (v5) is
timed in the same run and reported as `fp32_kernel`.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

Under torchrun each rank trains its own full-size shard (weak scaling) on its own GPU and
sums the replicas' deltas with NCCL every --sync-words words per GPU (default 1M; 50M at
C5, sized so the dense 2.4 GB delta all-reduce stays under 10% of the pass at N = 8:
20 syncs x ~9 ms against a 2.3 s pass).
Rank 0 prints ONE JSON line. `--impl reference` times the reference's own CPU
implementation (the reference headers compiled unchanged, oracle/_ref) on this host's
cores on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "trained words/sec (skip-gram HS)"
UNIT = "words/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c5", choices=["c1", "c2", "c3", "c4", "c5"])
    p.add_argument("--cache-nodes", type=int, default=31)
    p.add_argument("--sync-words", type=int, default=0,
                   help="delta all-reduce interval per GPU at N > 1 (0 = 50M at C5, else 1M)")
    p.add_argument("--sync-mode", default="delta", choices=["delta", "average"])
    p.add_argument("--e2e-steps", type=int, default=2)
    p.add_argument("--e2e-text-max-tokens", type=int, default=20_000_000,
                   help="also time train(corpus_path) on the corpus written as text when it has at most this many tokens")
    p.add_argument("--cpu-sample-tokens", type=int, default=0, help="reference sample size (0 = auto)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--warps", type=int, default=0)
    p.add_argument("--cpw", type=int, default=0)
    p.add_argument("--rows", type=int, default=-1)
    p.add_argument("--blocks", type=int, default=0)
    p.add_argument("--hot-flush-scale", type=float, default=0.0)
    p.add_argument("--flush-centers", type=int, default=0)
    p.add_argument("--min-cache-rows", type=int, default=0)
    p.add_argument("--kernel", type=int, default=0, help="K1 version (0 = default: v8; 5 = the all-FP32 kernel)")
    p.add_argument("--fp32-steps", type=int, default=2,
                   help="also time this many passes of the all-FP32 K1 (kernel 5) when the timed kernel is v8 (0 = skip)")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------ workload
def workload(cfg_name: str, rank: int, world: int, device: bool = False):
    """Per-rank shard of the configured corpus plus the shared vocabulary/tree.
    Each rank's shard has the configuration's full token count (weak scaling) and is
    drawn with its own seed; the vocabulary comes from shard 0 with ties broken by
    first occurrence in shard 0, so every rank builds the identical tree without
    communication. C4/C5 are generated on the GPU (`device=True`): ids come back as a
    CUDA int32 tensor, otherwise as a numpy array."""
    from paper_1606_07822_b200 import corpus_gen as G

    c = G.CONFIGS[cfg_name]
    if device and not c.clusters:
        import torch

        raw0 = G.zipf_raw_ids_device(c.tokens, c.vocab, c.zipf_s, c.seed)
        vocab, ids0 = G.vocab_from_raw_device(raw0, c.min_count, c.vocab)
        del raw0
        if rank == 0:
            return c, vocab, ids0
        raw = G.zipf_raw_ids_device(c.tokens, c.vocab, c.zipf_s, c.seed * 1000 + rank)
        rank_of = torch.full((c.vocab,), -1, dtype=torch.int32, device=raw.device)
        rank_of[torch.from_numpy(vocab.raw_of_id).to(raw.device).long()] = torch.arange(
            vocab.size(), dtype=torch.int32, device=raw.device)
        ids = rank_of[raw.long()]
        return c, vocab, ids[ids >= 0].contiguous()
    if c.clusters:
        raw0, _ = G.cluster_raw_ids(c)
        space = c.clusters * c.cluster_size
    else:
        raw0 = G.zipf_raw_ids(c.tokens, c.vocab, c.zipf_s, c.seed)
        space = c.vocab
    vocab, ids0 = G.vocab_from_raw(raw0, c.min_count, space)
    if rank == 0:
        return c, vocab, ids0
    raw = G.zipf_raw_ids(c.tokens, c.vocab, c.zipf_s, c.seed * 1000 + rank) if not c.clusters else raw0
    rank_of = np.full(space, -1, np.int32)
    rank_of[vocab.raw_of_id] = np.arange(vocab.size(), dtype=np.int32)
    ids = rank_of[raw]
    return c, vocab, np.ascontiguousarray(ids[ids >= 0])


def host_ids(ids, n: int | None = None) -> np.ndarray:
    if isinstance(ids, np.ndarray):
        return ids if n is None else ids[:n]
    t = ids if n is None else ids[:n]
    return t.cpu().numpy()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.active", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, r[3:7]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ reference arm / CPU baseline
def write_text(ids, words_of_id, path: str, n: int) -> None:
    """The id stream as text (token of id i = words_of_id[i]), a newline every 1000 tokens."""
    words = np.array([w if isinstance(w, bytes) else w.encode() for w in words_of_id], dtype=object)
    with open(path, "wb") as f:
        for a in range(0, n, 1_000_000):
            toks = words[ids[a:min(n, a + 1_000_000)]]
            f.write(b"\n".join(b" ".join(toks[i:i + 1000].tolist()) for i in range(0, toks.size, 1000)) + b"\n")


def reference_sample(c, vocab, ids, sample_tokens: int, workdir: str):
    """Writes the first `sample_tokens` tokens of the id stream as text (`w<id>`, newline
    every 1000) for the reference's file-based train(); its vocabulary is built from the
    full-corpus counts so keep probabilities and the tree match the GPU run."""
    sys.path.insert(0, str(ROOT / "tests"))
    import ctypes as C

    import oracle_lib as O

    n = min(sample_tokens, len(ids))
    ids = host_ids(ids, n)
    path = os.path.join(workdir, f"ref_sample_{c.name}.txt")
    write_text(ids, [b"w%d" % i for i in range(vocab.size())], path, n)  # ref_open_counts names word i "w<i>"
    counts = np.ascontiguousarray(vocab.counts, np.int64)
    h = O.ref().ref_open_counts(counts.ctypes.data_as(C.POINTER(C.c_int64)), counts.size)
    return O, h, path, n


def run_reference(c, vocab, ids, threads: int, sample_tokens: int, reps: int, cache_nodes: int):
    with tempfile.TemporaryDirectory() as d:
        O, h, path, n = reference_sample(c, vocab, ids, sample_tokens, d)
        cfg = dict(dim=c.dim, window=c.window, min_count=1, sample=c.sample, iterations=1, cache_nodes=cache_nodes,
                   flush_interval=10, seed=c.seed)
        rates, walls = [], []
        for _ in range(reps):
            _, _, words, wall = O.ref_train(h, path, cfg, workers=threads)
            rates.append(words / wall)
            walls.append(wall)
        O.ref().ref_close(h)
    return rates, walls, n


def _has_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_topology() -> dict:
    """Host threads this process may use and the machine's physical cores (psutil), so a
    CPU number says whether its threads were hardware threads or cores."""
    info = {"threads_available": cpu_threads(), "logical_cpus": os.cpu_count()}
    try:
        import psutil

        info["physical_cores"] = psutil.cpu_count(logical=False)
    except Exception:
        info["physical_cores"] = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["model"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return info


def auto_sample(c) -> int:
    """Tokens per reference pass: about 10-30 s of CPU work on a 16-32 core host."""
    return {"c1": 1_000_000, "c2": 17_000_000, "c3": 20_000_000, "c4": 6_000_000, "c5": 20_000_000}[c.name]


# ------------------------------------------------------------------ main
def main():
    args = parse()
    rank, world, local = dist_env()

    if args.impl == "reference":
        if rank != 0:
            return 0
        c, vocab, ids = workload(args.config, 0, 1, device=args.config in ("c4", "c5") and _has_cuda())
        threads = cpu_threads()
        sample = args.cpu_sample_tokens or auto_sample(c)
        for _ in range(max(args.warmup, 0) and 1):
            run_reference(c, vocab, ids, threads, min(sample, 200_000), 1, args.cache_nodes)
        rates, walls, n = run_reference(c, vocab, ids, threads, sample, args.steps, args.cache_nodes)
        words = n * args.steps
        value = words / sum(walls)
        line = {
            "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(walls) / len(walls),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.config}: {c.tokens // 10**6}M-token Zipf({c.zipf_s}) V {vocab.size()} "
                                   f"D {c.dim} W {c.window} sample {c.sample} K {args.cache_nodes}",
                       "sample_tokens_per_step": n},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "host": cpu_topology(),
                             "sample": f"first {n} tokens of the {args.config} corpus, 1 pass per step, "
                                       f"reference train() with workers={threads}"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return 0

    import torch
    import torch.distributed as dist

    # One process per GPU. CG_BENCH_BACKEND=gloo (tests only) runs the N > 1 code path
    # with every rank on the visible GPUs round-robin; timings of such a run mean nothing.
    backend = os.environ.get("CG_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_1606_07822_b200 import api

    c, vocab, ids = workload(args.config, rank, world, device=args.config in ("c4", "c5"))
    tree = api.build_huffman_tree(vocab)
    sel = api.select_cached_nodes(tree, args.cache_nodes)
    cfg = api.TrainConfig(dim=c.dim, window=c.window, min_count=c.min_count, sample=c.sample, iterations=1,
                          cache_nodes=args.cache_nodes, seed=c.seed, mode="hogwild")
    stream = torch.cuda.current_stream()
    sess = api.Session(vocab, tree, sel, cfg, device=local, stream=stream.cuda_stream)
    sess.tune(args.blocks, args.warps, args.cpw, args.rows, args.hot_flush_scale, args.flush_centers,
              args.min_cache_rows, args.kernel)
    if isinstance(ids, np.ndarray):
        sess.upload_ids(ids)
    else:
        sess.upload_ids_device(ids)
    model_t = sess.model_tensor() if world > 1 else None
    if not args.sync_words:
        args.sync_words = 50_000_000 if args.config == "c5" else 1_000_000
    l2_flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    T = int(len(ids))
    launches = {"n": 0}
    agg = {"train_ms": 0.0, "bytes": 0.0, "pairs": 0, "steps": 0, "kept": 0, "launch_count": 0}
    record = {"on": False}

    def local_step(epoch, a, b, base, mult):
        e = sess.train_range(epoch, a, b, base, mult)
        if record["on"]:
            launches["n"] += e.train_launches + e.other_launches
            agg["train_ms"] += e.train_ms
            agg["bytes"] += 4.0 * c.dim * (2.0 * e.steps + 2.0 * e.pairs)
            agg["pairs"] += e.pairs
            agg["steps"] += e.steps
            agg["kept"] += e.kept
            agg["launch_count"] += e.train_launches
            agg["geometry"] = {"blocks": e.blocks, "worker_warps": e.worker_warps, "ctx_batch": e.ctx_batch,
                               "cached_rows_per_cta": e.cached_rows, "smem_rows": e.smem_rows,
                               "floor_rows": e.floor_rows, "flush_centers": e.flush_centers, "kernel": e.kernel}
        return e

    from paper_1606_07822_b200.replicas import ReplicaTrainer

    trainer = ReplicaTrainer(local_step, model_t, world, rank, args.sync_words, replica=sess, mode=args.sync_mode)

    def one_step(epoch: int, rec: bool):
        record["on"] = rec
        trainer.run_pass(epoch, T, tokens_before=0)

    # The clock sampler starts with the warm-up: nvidia-smi needs ~0.2 s to report its
    # first sample, longer than a whole timed region of the small configs. Extra untimed
    # warm-up steps run until it has reported at least once (bounded), so the reported
    # clocks are those of the loaded GPU from the warm-up through the timed region.
    clocks = ClockSampler(local)
    clocks.start()
    for w in range(args.warmup):
        one_step(10_000 + w, False)
    torch.cuda.synchronize()
    t_wait = time.perf_counter()
    extra = 0
    while clocks.proc is not None and not clocks.rows and time.perf_counter() - t_wait < 5.0:
        one_step(20_000 + extra, False)
        torch.cuda.synchronize()
        extra += 1
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = []
    for s in range(args.steps):
        l2_flush.fill_(float(s))  # > L2 (126 MB): evicts the previous step's lines
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        one_step(s, True)
        ev1.record(stream)
        ev1.synchronize()
        step_ms.append(ev0.elapsed_time(ev1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    clk["window"] = "from the warm-up through the timed region (GPU under load throughout)"
    total_ms = float(sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    words_all = float(T) * args.steps * world  # every rank's shard has the same size
    value = words_all / (total_ms / 1e3)

    # The all-FP32 K1 (v5: packed FFMA2, no tensor cores) on the same resident inputs, for
    # readers who want the number without fp16 operand rounding: same step, device-timed.
    fp32_arm = None
    kernel_run = (agg.get("geometry") or {}).get("kernel")
    if world == 1 and kernel_run == 8 and args.fp32_steps > 0:
        sess.tune(args.blocks, args.warps, args.cpw, args.rows, args.hot_flush_scale, args.flush_centers,
                  args.min_cache_rows, 5)
        record["on"] = False
        sess.train_range(30_000, 0, T)
        torch.cuda.synchronize()
        ms5 = []
        geo5 = None
        for s in range(args.fp32_steps):
            l2_flush.fill_(float(s))
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            e5 = sess.train_range(40_000 + s, 0, T)
            ev1.record(stream)
            ev1.synchronize()
            ms5.append(ev0.elapsed_time(ev1))
            geo5 = {"worker_warps": e5.worker_warps, "ctx_batch": e5.ctx_batch, "kernel": e5.kernel,
                    "k1_ms": e5.train_ms}
        fp32_arm = {"value": float(T) * len(ms5) / (sum(ms5) / 1e3), "unit": UNIT, "ms_per_step": sum(ms5) / len(ms5),
                    "steps": len(ms5), "kernel": "hog5_kernel (K1 v5, FP32 FMA arithmetic end to end)", "geometry": geo5}
        sess.tune(args.blocks, args.warps, args.cpw, args.rows, args.hot_flush_scale, args.flush_centers,
                  args.min_cache_rows, args.kernel)

    # Roofline of the dominant kernel (K1). The HBM roofline is graded on
    # DRAM bytes: `achieved` = ncu-measured DRAM bytes per K1 launch (profiles/, captured
    # for this kernel source: `traffic_current`) / this run's CUDA-event K1 time. The
    # algorithmic bytes (4 D (2 L + 2) per pair) are reported beside it, not as the
    # fraction: K1 loads each path row once per center and keeps hot rows on chip, so they
    # exceed what crosses HBM. K1 is bound by SM issue; `fp32` is its FMA throughput
    # (3 D FMAs per pair and path step) against the FP32 pipe (SMs x 128 x the SM clock).
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    n_launch = max(agg["launch_count"], 1)
    per_launch_bytes = agg["bytes"] / n_launch
    per_launch_ms = agg["train_ms"] / n_launch
    algorithmic_gbs = per_launch_bytes / (per_launch_ms / 1e3) / 1e9
    sys.path.insert(0, str(ROOT / "tools"))
    from ncu_summary import kernel_sha16

    src_sha = kernel_sha16()
    traffic = l2_traffic = None
    ncu_pcts = {}
    traffic_current = False
    prof = ROOT / "profiles" / f"ncu_traffic_{args.config}.json"
    if prof.exists():
        try:
            tj = json.loads(prof.read_text())
            traffic, l2_traffic = tj.get("dram_bytes_per_launch"), tj.get("l2_bytes_per_launch")
            ncu_pcts = {k: tj.get(k) for k in ("lts_throughput_pct", "l1tex_throughput_pct", "issue_active_pct",
                                                "l2_hit_rate_pct") if tj.get(k) is not None}
            traffic_current = tj.get("kernel_sha16") == src_sha
        except Exception:
            traffic = l2_traffic = None
    dram_gbs = traffic / (per_launch_ms / 1e3) / 1e9 if traffic else None
    props = torch.cuda.get_device_properties(local)
    f_sm = 1e6 * float(clk.get("sm_mhz") or clk.get("sm_max_mhz") or 1965.0)
    fma_per_launch = 3.0 * c.dim * agg["steps"] / n_launch
    fp32_peak = props.multi_processor_count * 128 * f_sm
    fp32_achieved = fma_per_launch / (per_launch_ms / 1e3)
    roofline = {
        "bound": "hbm", "unit": "GB/s", "peak": peak, "peak_source": peak_src,
        "achieved": dram_gbs, "frac": dram_gbs / peak if dram_gbs else None, "traffic": traffic,
        "traffic_source": f"profiles/{prof.name} (ncu --set full, one K1 launch)",
        "traffic_current": traffic_current, "kernel_sha16": src_sha,
        "dram_frac": dram_gbs / peak if dram_gbs else None,
        "l2_traffic": l2_traffic,
        "l2": {"achieved_gbs": l2_traffic / (per_launch_ms / 1e3) / 1e9 if l2_traffic else None,
               "ncu": ncu_pcts or None,
               "note": "L2 bytes of the same ncu capture / this run's K1 time; ncu percentages are the capture's"},
        "algorithmic_bytes_per_launch": per_launch_bytes, "algorithmic_gbs": algorithmic_gbs,
        "algorithmic_gbs_over_hbm_peak": algorithmic_gbs / peak,
        "fp32": {"fma_per_launch": fma_per_launch, "achieved_tfma_s": fp32_achieved / 1e12,
                 "peak_tfma_s": fp32_peak / 1e12, "frac": fp32_achieved / fp32_peak,
                 "note": "3 D FMAs per (pair, path step); peak = SMs x 128 FMA/clk x median SM clock"},
        "fp32_frac": fp32_achieved / fp32_peak,
        "kernel": {8: "hog8_kernel (K1 v8)", 5: "hog5_kernel (K1 v5)", 0: "hog_generic_kernel (K1)"}.get(
            (agg.get("geometry") or {}).get("kernel"), "K1"), "kernel_ms_per_launch": per_launch_ms,
    }

    # end to end through the public API with host buffers (pinned): ids H2D, model init,
    # subsampling + training (+ averaging at N > 1), model D2H. N = 1 goes through the
    # reference-facing C-ABI call cg_train(); N > 1 through api.Session + ReplicaTrainer.
    e2e = None
    if args.e2e_steps > 0:
        ids_pin = torch.from_numpy(host_ids(ids)).pin_memory()
        out0 = torch.empty((vocab.size(), c.dim), dtype=torch.float32).pin_memory()
        out1 = torch.empty((vocab.size() - 1, c.dim), dtype=torch.float32).pin_memory()
        import ctypes as C

        from paper_1606_07822_b200._lib import CgTrainStats, check, load, ptr

        keep: list = []
        desc = api.model_desc(vocab, tree, sel, keep)
        ccfg = cfg.to_c()
        walls = []
        for it in range(args.e2e_steps + 1):  # the first call warms the device memory pool (untimed)
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            if world == 1:
                st = CgTrainStats()
                check(load().cg_train(C.byref(ccfg), 0, C.byref(desc), ptr(ids_pin.numpy(), C.c_int32), T,
                                      ptr(out0.numpy(), C.c_float), ptr(out1.numpy(), C.c_float), C.byref(st)))
            else:
                s2 = api.Session(vocab, tree, sel, cfg, device=local, stream=stream.cuda_stream)
                s2.upload_ids(ids_pin.numpy())
                rt2 = ReplicaTrainer(lambda e, a, b, base, mult: s2.train_range(e, a, b, base, mult),
                                     s2.model_tensor(), world, rank, args.sync_words, replica=s2, mode=args.sync_mode)
                rt2.run_pass(0, T)
                m = s2.download()
                s2.close()
            if it > 0:
                walls.append(time.perf_counter() - t0)
        e2e_wall = float(np.median(walls))
        if world > 1:
            t = torch.tensor([e2e_wall], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_wall = float(t.item())
        e2e = {"value": float(T) * world / e2e_wall, "unit": UNIT, "h2d_bytes_per_step": int(T * 4),
               "d2h_bytes_per_step": int(out0.numel() * 4 + out1.numel() * 4),
               "note": ("cg_train()" if world == 1 else "api.Session + ReplicaTrainer") +
                       ": host ids -> device, model init, subsample + train, device -> host model"}

    # end to end through the drop-in train(corpus_path, ...): the corpus as a text file
    # (page cache), tokenised on the GPU (cg_train_file), trained, model back on the host --
    # the same work the reference's train() does in its timed region.
    e2e_text = None
    if rank == 0 and world == 1 and args.e2e_steps > 0 and T <= args.e2e_text_max_tokens:
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "corpus.txt")
            write_text(host_ids(ids), [vocab.word(i) for i in range(vocab.size())], path, T)
            walls = []
            for it in range(args.e2e_steps + 1):
                st = api.TrainStats()
                t0 = time.perf_counter()
                api.train(path, vocab, tree, sel, cfg, st)
                if it > 0:
                    walls.append(time.perf_counter() - t0)
                assert st.words_processed == T, (st.words_processed, T)
            w = float(np.median(walls))
            e2e_text = {"value": T / w, "unit": UNIT, "text_bytes_per_step": os.path.getsize(path),
                        "d2h_bytes_per_step": int(vocab.size() * c.dim * 4 + (vocab.size() - 1) * c.dim * 4),
                        "note": "train(corpus_path) -> cg_train_file(): text file read + GPU tokenise + train + model D2H"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = cpu_threads()
            sample = args.cpu_sample_tokens or auto_sample(c)
            rates, walls, n = run_reference(c, vocab, ids, threads, sample, 1, args.cache_nodes)
            extra = {}
            if args.config == "c1" and threads != 4:  # BASELINE config 1 states 4 CPU threads in the reference
                r4, _, _ = run_reference(c, vocab, ids, 4, sample, 1, args.cache_nodes)
                extra = {"value_4_threads": float(np.median(r4))}
            cpu = {"value": float(np.median(rates)), "unit": UNIT, "cores": threads, "kind": "reference", **extra,
                   "host": cpu_topology(),
                   "sample": f"first {n} tokens of the {args.config} corpus, 1 pass, reference train() "
                             f"(headers compiled unchanged, -O3) with workers={threads}"}
        except Exception as ex:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "reference", "sample": f"failed: {ex}"}

    sess.close()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f32 model, sums and updates; fp16 mma operands (K1 v8)" if kernel_run == 8 else "f32",
            "data": "synthetic",
            "config": {"workload": f"{args.config}: {c.tokens / 1e6:g}M-token Zipf({c.zipf_s}) per GPU, V {vocab.size()}, "
                                   f"D {c.dim}, W {c.window}, sample {c.sample}, K {args.cache_nodes}, 1 pass per step",
                       "l2": "256 MB buffer written between timed steps", "parallelism": f"replicas{world}",
                       "sync_words_per_gpu": args.sync_words if world > 1 else None,
                       "sync": (f"{args.sync_mode}: replicas' deltas all-reduced (SUM) and applied with the per-row "
                                "sync scale" if args.sync_mode == "delta" else "whole-model all-reduce (AVG)")
                       if world > 1 else None},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_text": e2e_text,
            "fp32_kernel": fp32_arm,
            "gpu_launches": launches["n"],
            "clocks": clk,
            "detail": {"syncs": trainer.syncs, "sync_bytes": trainer.sync_bytes,
                       "sync_ms_total": 1e3 * trainer.sync_seconds,
                       "pairs_per_step": agg["pairs"] / args.steps, "path_steps_per_step": agg["steps"] / args.steps,
                       "kept_per_step": agg["kept"] / args.steps, "step_ms": step_ms,
                       "k1_geometry": agg.get("geometry")},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
