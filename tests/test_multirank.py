"""Multi-rank host logic on CPU (gloo, world_size 2): point sharding, bit-plane
gather and job totals reproduce the single-process result bit for bit.  The
per-rank compute stand-in is the C restatement (test infrastructure), since
this container has no GPU; the GPU path itself is covered by
test_gpu_parity.py::test_multi_shard_identical."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2306_04316_b200.dist import shard_range


def test_shard_ranges_cover_and_align():
    for n in (0, 1, 31, 32, 33, 1000, 100_003, 10**8):
        for world in (1, 2, 3, 4, 8):
            parts = [shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c
            for lo, hi in parts:
                assert lo <= hi and (lo % 32 == 0 or lo == hi)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2306_04316_b200 import pack_bits
    from paper_2306_04316_b200 import workloads as W
    from paper_2306_04316_b200.dist import gather_bit_planes, job_totals, max_over_ranks

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        poly = W.star_polygon(300)
        n = 20_011
        xy = W.uniform_points(n, W.bounds(poly), 9)
        lo, hi = shard_range(n, rank, world)
        v, st = oracle.port_classify(xy[lo:hi], poly.vx, poly.vy, poly.ring_off, 0)
        local = torch.from_numpy(pack_bits(v == 0).view(np.int32).copy())
        full = gather_bit_planes(local, n, world)
        units, pts = job_totals((hi - lo) * poly.n_edges, hi - lo, world)
        mx = max_over_ranks(float(rank + 1), world)
        if rank == 0:
            q.put((full, units, pts, mx))
    finally:
        dist.destroy_process_group()


def test_two_rank_gather_matches_single_process():
    import oracle
    from paper_2306_04316_b200 import pack_bits
    from paper_2306_04316_b200 import workloads as W

    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    full, units, pts, mx = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    poly = W.star_polygon(300)
    n = 20_011
    xy = W.uniform_points(n, W.bounds(poly), 9)
    v, _ = oracle.port_classify(xy, poly.vx, poly.vy, poly.ring_off, 0)
    assert np.array_equal(full, pack_bits(v == 0))
    assert units == n * poly.n_edges and pts == n and mx == 2.0


def test_bench_torchrun_path_gloo():
    """bench.py's own torchrun code path (two ranks, gloo, CPU): per-rank shard
    generation, bit-plane all-gather, job totals and max over ranks."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    port = _free_port()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(root, "bench.py"),
                        "--gpus", "2", "--dist-check", "--dist-check-points", "300007"],
                       capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["dist_check"] == "ok" and line["world"] == 2
