"""Multi-replica orchestration (shards, sync cadence, global-progress estimate, the delta
reduction) on CPU with torch.distributed gloo, world_size 2. The local step is the
oracle's single-worker trainer (test infrastructure) standing in for the device kernels,
and a host stand-in applies the library's sync rule (cg_sync_row_scale); the expected
result is recomputed sequentially in one process."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_lib as O
from paper_1606_07822_b200.replicas import ReplicaTrainer, plan_chunks, shard_bounds

V, D = 60, 8


def corpus():
    rng = np.random.default_rng(7)
    p = 1.0 / np.arange(1, V + 1)
    ids = rng.choice(V, size=24_000, p=p / p.sum()).astype(np.int32)
    counts = np.bincount(ids, minlength=V).astype(np.int64)
    order = np.argsort(-counts, kind="stable")
    rank = np.empty(V, np.int32)
    rank[order] = np.arange(V)
    return rank[ids], counts[order]


def local_step_factory(ids, counts, model_np):
    tree = O.orc_tree(counts)
    hot, slot = O.orc_select(tree.usage, 7)
    import ctypes as C

    def step(epoch, a, b, base, mult):
        cfg = O.OrcConfig(D, 3, 1, 1e-3, 0.025, 1, 1, 7, 10, 11 + epoch)
        st = O.OrcStats()
        seg = np.ascontiguousarray(ids[a:b])
        syn0 = model_np[: V * D].reshape(V, D)
        syn1 = model_np[V * D:].reshape(V - 1, D)
        s0 = np.ascontiguousarray(syn0)
        s1 = np.ascontiguousarray(syn1)
        O.oracle().orc_train_single(O._p(seg, C.c_int32), seg.size, V, O._p(counts, C.c_int64), int(counts.sum()),
                                    O._p(tree.off, C.c_int64), O._p(tree.nodes, C.c_int32),
                                    O._p(tree.turns, C.c_uint8), O._p(hot, C.c_int32), hot.size,
                                    O._p(slot, C.c_int32), C.byref(cfg), O._p(s0, C.c_float), O._p(s1, C.c_float),
                                    C.byref(st))
        syn0[:] = s0
        syn1[:] = s1
        return (epoch, a, b, base, mult)

    return step


def init_model():
    s0, s1 = O.orc_init(V, D, 3)
    return np.concatenate([s0.ravel(), s1.ravel()]).astype(np.float32)


def row_shares(counts, window=3):
    """Per-row update shares in the model layout: syn0 row w, (W + 1) x its share of the
    stream; syn1 node n, its usage over the root's (what the session uses)."""
    tree = O.orc_tree(counts)
    q0 = np.minimum(1.0, (window + 1) * counts / counts.sum())
    q1 = tree.usage / tree.usage[-1]
    return np.concatenate([q0, q1])


class HostReplica:
    """Host stand-in for a session's sync operations (cg_session_sync_*): the same
    snapshot/delta/apply steps on a numpy model, with the library's row scale."""

    def __init__(self, model_np, counts):
        from paper_1606_07822_b200 import api

        self.m = model_np
        self.q = row_shares(counts)
        self.api = api

    def sync_begin(self):
        self.snap = self.m.copy()

    def sync_delta_tensor(self):
        # the delta in the model's layout, one squared norm per row, and the squared norms
        # of the two matrices (cg_session_sync_delta)
        d = self.m - self.snap
        self.delta = torch.from_numpy(np.concatenate([d, _row_sumsq(d), _matrix_sumsq(self.m)]).astype(np.float32))
        return self.delta

    def sync_apply(self, n, words):
        total = self.delta.numpy()
        d, sumsq, mats = total[: self.m.size], total[self.m.size:-2], total[-2:]
        prior = np.array([self.api.sync_row_scale(q, n, words) for q in self.q], np.float32)
        self.m[:] = self.snap + _sync_rows(d, sumsq, mats, prior, n) * d
        self.snap = self.m.copy()


TRUST = 0.25  # kSyncTrust (cg_capi.cu); the rms norms cover the 1024 hottest rows: all of them here


def _sync_rows(total, sumsq, mats, prior, n):
    """cg_session_sync_apply's per-row scale, repeated over each row's D floats:
    s = min(prior, max(ratio, trust)), ratio = clamp(sum |delta_r|^2 / |sum delta_r|^2, 1/n, 1),
    trust = min(1, TRUST / (rms row norm of the other matrix x |sum delta_r|))."""
    norm2 = _row_sumsq(total)
    ratio = np.clip(np.divide(sumsq, norm2, out=np.ones_like(sumsq), where=norm2 > 0), 1.0 / n, 1.0)
    rms0, rms1 = np.sqrt(mats[0] / n / V), np.sqrt(mats[1] / n / (V - 1))
    other = np.maximum(np.concatenate([np.full(V, rms1), np.full(V - 1, rms0)]), 1e-12)
    trust = np.minimum(1.0, TRUST / (other * np.sqrt(np.maximum(norm2, 1e-30))))
    sc = np.minimum(prior, np.maximum(ratio, trust)).astype(np.float32)
    return np.concatenate([np.repeat(sc[:V], D), np.repeat(sc[V:], D)])


def _matrix_sumsq(flat):
    r = _row_sumsq(flat)
    return np.array([r[:V].sum(), r[V:].sum()], np.float32)


def _row_sumsq(flat):
    """Squared norm of every model row: V syn0 rows, then V - 1 syn1 rows of D floats."""
    return (flat.reshape(2 * V - 1, D).astype(np.float32) ** 2).sum(axis=1, dtype=np.float32)


def _worker(rank, world, port, out, mode):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ids, counts = corpus()
    a, b = shard_bounds(ids.size, world, rank)
    model = torch.from_numpy(init_model())
    rt = ReplicaTrainer(local_step_factory(ids[a:b], counts, model.numpy()), model, world, rank, sync_words=5000,
                        replica=HostReplica(model.numpy(), counts), mode=mode)
    calls = rt.run_pass(0, b - a) + rt.run_pass(1, b - a, tokens_before=b - a)
    out[rank] = (model.numpy().copy(), calls, rt.syncs)
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_plan_and_shards():
    assert [(c.begin, c.end) for c in plan_chunks(10, 4)] == [(0, 4), (4, 8), (8, 10)]
    assert plan_chunks(0, 4) == []
    bounds = [shard_bounds(10, 3, r) for r in range(3)]
    assert bounds == [(0, 3), (3, 6), (6, 10)]


def test_sync_row_scale():
    """The delta reduction's per-row scale (cg_sync_row_scale): one replica is the plain
    sum; a row few replicas touch is summed as in the reference; a row every replica
    updates from the same snapshot is capped at 128 stale updates' worth but never below
    the replicas' average; monotone in the row's share."""
    from paper_1606_07822_b200 import api

    assert api.sync_row_scale(1.0, 1, 1e6) == 1.0
    for n in (2, 4, 8):
        assert api.sync_row_scale(1e-9, n, 1e5) == 1.0  # touched by at most one replica
        assert api.sync_row_scale(1.0, n, 1e5) == pytest.approx(1.0 / n)  # the root: the average
        assert api.sync_row_scale(1.0, n, 8.0) == pytest.approx(1.0)  # <= 128 stale updates: still a sum
        qs = np.logspace(-8, 0, 40)
        sc = [api.sync_row_scale(q, n, 1e5) for q in qs]
        assert all(1.0 / n - 1e-7 <= x <= 1.0 for x in sc)
        assert all(a >= b - 1e-7 for a, b in zip(sc, sc[1:]))


@pytest.mark.parametrize("mode", ["delta", "average"])
def test_two_replicas_gloo_match_sequential_simulation(mode):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), out, mode), nprocs=world, start_method="spawn", join=True)
    m0, calls0, syncs0 = out[0]
    m1, calls1, _ = out[1]
    assert np.array_equal(m0, m1)  # replicas agree after every sync point
    ids, counts = corpus()
    n = [shard_bounds(ids.size, world, r) for r in range(world)]
    # progress estimate: base = world x local tokens before the chunk, mult = world
    assert calls0[0] == (0, 0, 5000, 0, 2) and calls0[1] == (0, 5000, 10000, 10000, 2)
    assert calls0[len(plan_chunks(n[0][1] - n[0][0], 5000))][3] == (n[0][1] - n[0][0]) * world
    assert syncs0 == 2 * len(plan_chunks(n[0][1] - n[0][0], 5000))
    # sequential simulation of the same schedule
    models = [init_model() for _ in range(world)]
    steps = [local_step_factory(ids[a:b], counts, models[r]) for r, (a, b) in enumerate(n)]
    snap = models[0].copy()
    q = row_shares(counts)
    from paper_1606_07822_b200 import api

    prior = np.array([api.sync_row_scale(x, world, 5000) for x in q], np.float32)
    for epoch in range(2):
        chunks = [plan_chunks(b - a, 5000) for a, b in n]
        for i in range(max(len(c) for c in chunks)):
            for r in range(world):
                if i < len(chunks[r]):
                    ch = chunks[r][i]
                    steps[r](epoch, ch.begin, ch.end, 0, world)
            if mode == "average":
                new = (models[0] + models[1]) / 2
            else:  # the summed deltas since the last sync, scaled per row (_sync_rows)
                d = [(models[r] - snap).astype(np.float32) for r in range(world)]
                total = d[0] + d[1]
                sumsq = _row_sumsq(d[0]) + _row_sumsq(d[1])
                mats = _matrix_sumsq(models[0]) + _matrix_sumsq(models[1])
                new = snap + _sync_rows(total, sumsq, mats, prior, world) * total
            for r in range(world):
                models[r][:] = new
            snap = new.copy()
    np.testing.assert_allclose(m0, models[0], rtol=0, atol=1e-6)
    if mode == "delta":  # a row one replica alone touched keeps its whole update
        assert not np.allclose(m0, (models[0] + init_model()) / 2)


@pytest.mark.gpu
def test_bench_two_ranks_functional(tmp_path):
    """bench.py's N > 1 path end to end (sessions, shards, averaging through the device
    model buffer, max-over-ranks timing, one JSON line from rank 0) with 2 ranks on the
    one available GPU over gloo. Functional only: the ranks share the GPU."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    port = _free_port()
    env = dict(os.environ, CG_BENCH_BACKEND="gloo", MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(root / "bench.py"), "--gpus", "2",
           "--config", "c1", "--steps", "2", "--warmup", "1", "--no-cpu-baseline", "--e2e-steps", "1",
           "--sync-words", "200000"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=str(root), env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["parallelism"] == "replicas2"
    assert d["e2e"]["value"] > 0


@pytest.mark.gpu
def test_bench_two_ranks_nccl_on_two_gpus():
    """The driver's N > 1 launch exactly (NCCL, one rank per GPU); runs only where at
    least two GPUs are visible (the round-1 boxes have one)."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    root = Path(__file__).resolve().parents[1]
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(root / "bench.py"), "--gpus", "2",
           "--config", "c1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=str(root),
                       env=dict(os.environ, MASTER_ADDR="127.0.0.1"))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "weak" and d["e2e"]["value"] > 0
