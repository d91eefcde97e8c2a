#!/bin/bash
# scan vs tree per polygon size (1e6 points each), C1
cat > /tmp/thr.py <<'PY'
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2306_04316_b200 import Engine
from paper_2306_04316_b200 import workloads as W
eng = Engine(devices=[0])
dev = torch.device('cuda:0')
st = torch.cuda.Stream(dev)
for n in (100, 300, 1000, 3000, 10000, 100000, 1000000):
    poly = W.star_polygon(n); xy = W.uniform_points(1_000_000, W.bounds(poly), 2 + n)
    d_xy = torch.from_numpy(xy).to(dev); d_vx = torch.from_numpy(poly.vx).to(dev); d_vy = torch.from_numpy(poly.vy).to(dev)
    d_ro = torch.from_numpy(poly.ring_off.view(np.int64)).to(dev)
    nw = (len(xy) + 31) // 32
    bits = torch.zeros(2 * nw, dtype=torch.int32, device=dev); stats = torch.zeros(4, dtype=torch.int64, device=dev)
    res = {}
    for mode in (0, 1):
        eng.set_tree(mode)
        for _ in range(3):
            eng.classify_dev(0, st.cuda_stream, d_xy, len(xy), d_vx, d_vy, d_ro, poly.n_rings, poly.n_verts, 0, 1e-12, True, bits[:nw], bits[nw:], stats)
        st.synchronize(); t = time.perf_counter()
        for _ in range(5):
            eng.classify_dev(0, st.cuda_stream, d_xy, len(xy), d_vx, d_vy, d_ro, poly.n_rings, poly.n_verts, 0, 1e-12, True, bits[:nw], bits[nw:], stats)
        st.synchronize(); res[mode] = (time.perf_counter() - t) / 5 * 1e3
    eng.set_tree(-1)
    print(f"n={n:8d}  scan {res[0]:8.3f} ms  tree {res[1]:8.3f} ms", flush=True)
PY
python /tmp/thr.py
