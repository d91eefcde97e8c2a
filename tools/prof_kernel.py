"""Small driver for ncu: runs one classify call (device pointers) of a config,
`--reps` times, so `ncu -k regex:pip_ -s <skip> -c <count>` can capture the hot
kernel.  Usage: python tools/prof_kernel.py --workload c4 --points 4000000 --mode 0 --reps 3"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_04316_b200 import Engine  # noqa: E402
from paper_2306_04316_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c1", choices=["c1", "c2", "c4", "c3", "c5"])
ap.add_argument("--n", type=int, default=1000, help="polygon vertices for c2")
ap.add_argument("--points", type=int, default=1_000_000)
ap.add_argument("--polys", type=int, default=200_000)
ap.add_argument("--mode", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--bucket", type=int, default=-1)
ap.add_argument("--tree", type=int, default=-1, help="PC_OPT_TREE: -1 auto, 0 scan kernel, 1 segment tree")
a = ap.parse_args()

dev = torch.device("cuda:0")
torch.cuda.set_stream(torch.cuda.Stream())
eng = Engine(devices=[0])
eng.set_bucketing(a.bucket)
eng.set_tree(a.tree)
st = torch.cuda.current_stream().cuda_stream


def u64(x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).to(dev)


if a.workload in ("c1", "c2", "c4"):
    if a.workload == "c1":
        poly = W.star_polygon(1000)
        xy = W.uniform_points(a.points, (-1.0, -1.0, 1.0, 1.0), 1)
    elif a.workload == "c2":
        poly = W.star_polygon(a.n)
        xy = W.uniform_points(a.points, W.bounds(poly), 2)
    else:
        poly = W.fractal_polygon(200_000)
        xy = W.uniform_points(a.points, W.bounds(poly), 4)
    d_xy, d_vx, d_vy, d_ro = (torch.from_numpy(xy).to(dev), torch.from_numpy(poly.vx).to(dev),
                              torch.from_numpy(poly.vy).to(dev), u64(poly.ring_off))
    nw = (len(xy) + 31) // 32
    bits = torch.zeros(2 * nw, dtype=torch.int32, device=dev)
    stats = torch.zeros(4, dtype=torch.int64, device=dev)
    for _ in range(a.reps):
        eng.classify_dev(0, st, d_xy, len(xy), d_vx, d_vy, d_ro, poly.n_rings, poly.n_verts, a.mode, 1e-12, True,
                         bits[:nw], bits[nw:], stats)
else:
    s = W.footprints(a.polys) if a.workload == "c3" else W.degenerate(a.polys)
    t = {k: (u64(getattr(s, k)) if getattr(s, k).dtype == np.uint64 else torch.from_numpy(getattr(s, k)).to(dev))
         for k in ("xy", "pt_off", "vx", "vy", "ring_off", "poly_ring_off")}
    nw = (s.n_points + 31) // 32
    bits = torch.zeros(2 * nw, dtype=torch.int32, device=dev)
    stats = torch.zeros(4, dtype=torch.int64, device=dev)
    for _ in range(a.reps):
        eng.classify_csr_dev(0, st, t["xy"], t["pt_off"], s.n_polys, s.n_points, t["vx"], t["vy"], t["ring_off"],
                             t["poly_ring_off"], a.mode, 1e-12, bits[:nw], bits[nw:], stats)
torch.cuda.synchronize()
print("stats", stats.cpu().numpy())
