"""Multi-rank host logic of the frame-sharded path on CPU with gloo, world size 2."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_0902_0657_b200.dist import shard_frame_ids, reduce_run, frame_counters, COUNTERS


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shards_partition_the_frames():
    for ws in (1, 2, 3, 8):
        ids = np.concatenate([shard_frame_ids(100, r, ws) for r in range(ws)])
        assert np.array_equal(np.sort(ids), np.arange(100 * ws))
    with pytest.raises(ValueError):
        shard_frame_ids(4, 2, 2)


def test_frame_counters():
    from paper_0902_0657_b200._ffi import STATS_FIELDS
    st = np.zeros(3, dtype=STATS_FIELDS)
    st["lp_solves"] = [1, 2, 3]
    st["pcg_iters"] = [10, 0, 5]
    st["pcg_bytes"] = [1.5, 0, 2.5]
    st["pcg_solves"] = [4, 0, 2]
    st["pcg_p4_fail"] = [1, 0, 0]
    hard = np.array([[0, 1], [1, 1], [0, 0]])
    cw = np.array([[0, 1], [0, 1], [0, 0]])
    c = frame_counters(hard, cw, [1, 0, 1], [0, 2 | 4, 4], st)
    d = dict(zip(COUNTERS, c))
    assert d == dict(frames=3, frame_errors=1, not_certified=1, lp_solves=6, ipm_iters=0,
                     pcg_iters=15, frames_capped=1, pcg_bytes=4.0, pcg_solves=6,
                     pcg_p4_failed_solves=1, pcg_true_failed_solves=0, frames_alp_maxiter=0,
                     frames_ipm_maxiter=1, frames_pcg_maxiter=2, frames_pcg_breakdown=0,
                     frames_numeric=0)


def _worker(rank, ws, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    ids = shard_frame_ids(5, rank, ws)
    counters = np.array([ids.size, rank, 1, 0, 0, 10 * (rank + 1), 0, 0.5], dtype=np.float64)
    tot, t = reduce_run(counters, seconds=1.0 + rank)
    q.put((rank, ids.tolist(), tot.tolist(), t))
    dist.destroy_process_group()


def test_gloo_world_size_2_reduction():
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(ws)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    all_ids = sorted(res[0][1] + res[1][1])
    assert all_ids == list(range(10))
    for _, _, tot, t in res:
        assert tot == [10, 1, 2, 0, 0, 30, 0, 1.0]
        assert t == 2.0


def test_single_process_reduce_is_identity():
    c, t = reduce_run(np.array([1.0, 2.0]), 3.5)
    assert c.tolist() == [1.0, 2.0] and t == 3.5


def test_bench_launches_its_own_ranks():
    """`bench.py --gpus 2` without a torch.distributed environment launches 2 ranks itself
    (torch.distributed.run on 127.0.0.1); exercised on CPU through the oracle reference arm,
    where rank 0 alone prints the JSON line and reports n_gpus = 2."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--impl", "reference",
                          "--steps", "1", "--warmup", "0", "--cpu-seconds", "2"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    assert lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"
