"""World-size-2 gloo test of the batch-sharded multi-GPU plumbing: disjoint
frames per rank, max-over-ranks timing, whole-job throughput. Runs on CPU."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2107_11627_b200 import dist as pdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    r, w, lr = pdist.env_rank_world()
    d = pdist.init("gloo")
    frames = list(pdist.rank_frames(r, 3))
    t = pdist.max_over_ranks(10.0 + 5.0 * r, d)
    import torch
    gathered = [None] * w
    d.all_gather_object(gathered, frames)
    q.put((r, w, lr, frames, t, gathered, pdist.throughput(3, w, 4, t)))
    pdist.shutdown(d)


def test_two_rank_sharding_and_max_time():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    all_frames = res[0][5]
    assert all_frames[0] == [0, 1, 2] and all_frames[1] == [3, 4, 5]  # disjoint, contiguous
    for r, w, lr, frames, t, gathered, thr in res:
        assert w == 2 and lr == r
        assert t == 15.0                     # slowest rank's time
        assert thr == pytest.approx(3 * 2 * 4 / 0.015)


def test_single_process_defaults():
    assert pdist.max_over_ranks(3.5, None) == 3.5
    assert list(pdist.rank_frames(0, 1)) == [0]
    with pytest.raises(ValueError):
        pdist.throughput(1, 1, 1, 0.0)


def test_bench_gpus_flag_launches_ranks_dry_run():
    """`python bench.py --gpus 2 --dry-run` (no torchrun around it) re-launches itself as two ranks
    (torch.distributed.run, gloo, 127.0.0.1) and rank 0 prints n_gpus = 2 with disjoint frame blocks."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run", "--steps", "3"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["dry_run"] and d["rank_frames"] == [[0], [1]]
    assert d["max_over_ranks_probe"] == 2.0 and d["scaling"] == "weak"
