"""Times one device-pointer classify call per small polygon size with the scan
kernel and with the literal binary64 kernel (PC_OPT_EXACT): which is faster for
few edges?  python tools/time_small_n.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_04316_b200 import Engine  # noqa: E402
from paper_2306_04316_b200 import workloads as W  # noqa: E402

dev = torch.device("cuda:0")
torch.cuda.set_stream(torch.cuda.Stream())
st = torch.cuda.current_stream().cuda_stream
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for n in (4, 10, 32, 63, 64, 100, 200, 1000):
    poly = W.star_polygon(n)
    xy = W.uniform_points(1_000_000, W.bounds(poly), 2)
    d_xy, d_vx, d_vy = torch.from_numpy(xy).to(dev), torch.from_numpy(poly.vx).to(dev), torch.from_numpy(poly.vy).to(dev)
    d_ro = torch.from_numpy(np.ascontiguousarray(poly.ring_off).view(np.int64)).to(dev)
    nw = (len(xy) + 31) // 32
    out = {}
    for exact in (False, True):
        eng = Engine(devices=[0])
        eng.set_exact(exact)
        for mode in (0, 1, 2):
            bits = torch.zeros(2 * nw, dtype=torch.int32, device=dev)
            stats = torch.zeros(4, dtype=torch.int64, device=dev)
            ts = []
            for rep in range(8):
                flush.fill_(rep)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                eng.classify_dev(0, st, d_xy, len(xy), d_vx, d_vy, d_ro, poly.n_rings, poly.n_verts, mode, 1e-12, True,
                                 bits[:nw], bits[nw:], stats)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            out[(exact, mode)] = (min(ts[3:]), bits.clone())
        eng.close()
    for mode in (0, 1, 2):
        same = bool(torch.equal(out[(False, mode)][1], out[(True, mode)][1]))
        print(f"n={n} mode={mode} scan {out[(False, mode)][0]*1e3:.1f} us  exact {out[(True, mode)][0]*1e3:.1f} us  equal={same}", flush=True)
