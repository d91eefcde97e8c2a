"""TEST INFRASTRUCTURE — full-size reference goldens for the large configs.

BASELINE.md §4: "Full-size golden flags for parity are generated once with the
multi-threaded oracle and cached outside git."  This script runs the UNMODIFIED
reference classify_batch (oracle/_ref/libpolycast_ref.so, built from
/root/reference/proj/include by oracle/Makefile; workers = all host threads) on

  c4/C1      all 1e8 points of configs[3] (fractal star, 2e5 vertices)  2e13 tests
  c4/C2      the first 1e7 points                                       2e12 tests
  c4/Robust  the first 1e7 points (tol 1e-12)                           2e12 tests
  c2/n1e5    all 1e6 points of the sweep's 1e5-vertex star, 3 modes     3e11 tests
  c2/n1e6    all 1e6 points of the sweep's 1e6-vertex star, 3 modes     3e12 tests
  c1         all 1e6 points of configs[0], 3 modes                      3e9 tests
  c3         all 6.4e7 points of configs[2] (1e6 footprints; the reference
             classify_batch per polygon, its CSR loop), 3 modes

and writes the bit planes (inside, aux; bit i%32 of word i//32) to
golden_cache/ (git-ignored, NOT gpurun-ignored: it travels to the GPU box),
in 1e7-point parts so an interrupted run resumes.  The manifest with the
sha256 of every plane file and of the input bytes is committed as
tests/golden/full_manifest.json; tests/test_full_parity.py regenerates the
inputs on the box (same seeded generator), checks their sha256 against the
manifest, and compares the GPU planes with these files.

Run here (the reference exists only in this container):
    nice -n 10 python tools/make_full_goldens.py [--only c4_C1,...]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2306_04316_b200 import workloads as W  # noqa: E402
from paper_2306_04316_b200.engine import verdicts_to_bits  # noqa: E402

CACHE = os.path.join(ROOT, "golden_cache")
MANIFEST = os.path.join(ROOT, "tests", "golden", "full_manifest.json")
PART = 10_000_000
TOL = 1e-12


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8)).hexdigest()


def cases():
    """name -> (input builder, mode, n_points)"""
    out = {}
    out["c4_C1"] = ("c4", 0, 100_000_000)
    out["c4_C2"] = ("c4", 1, 10_000_000)
    out["c4_Robust"] = ("c4", 2, 10_000_000)
    for n in (100_000, 1_000_000):
        for m, mn in ((0, "C1"), (1, "C2"), (2, "Robust")):
            out[f"c2_n{n}_{mn}"] = (f"c2:{n}", m, 1_000_000)
    for m, mn in ((0, "C1"), (1, "C2"), (2, "Robust")):
        out[f"c1_{mn}"] = ("c1", m, 1_000_000)
        out[f"c3_{mn}"] = ("c3", m, 64_000_000)
    return out


_inputs = {}


def inputs(kind):
    if kind not in _inputs:
        if kind == "c4":
            _inputs[kind] = W.config4()
        elif kind == "c1":
            _inputs[kind] = W.config1()
        elif kind == "c3":
            _inputs[kind] = W.footprints()
        else:
            _inputs[kind] = W.config2(int(kind.split(":")[1]))
    return _inputs[kind]


def run_csr_case(name, kind, mode):
    s = inputs(kind)
    f = os.path.join(CACHE, "parts", name + ".npz")
    os.makedirs(os.path.dirname(f), exist_ok=True)
    if not os.path.exists(f):
        t0 = time.time()
        v, st = oracle.ref_classify_csr(s, mode, TOL, threads=0)
        i_b, a_b = verdicts_to_bits(v, mode)
        np.savez(f, inside=i_b, aux=a_b, stats=st)
        print(f"[{name}] {s.n_points} points: {time.time() - t0:.1f} s", flush=True)
    z = np.load(f)
    np.save(os.path.join(CACHE, f"{name}_inside.npy"), z["inside"])
    np.save(os.path.join(CACHE, f"{name}_aux.npy"), z["aux"])
    return {
        "config": kind, "mode": mode, "n_points": int(s.n_points), "tol": TOL, "csr": True,
        "points_sha256": sha(s.xy), "vx_sha256": sha(s.vx), "vy_sha256": sha(s.vy),
        "pt_off_sha256": sha(s.pt_off), "ring_off_sha256": sha(s.ring_off), "poly_ring_off_sha256": sha(s.poly_ring_off),
        "inside_file": f"{name}_inside.npy", "inside_sha256": sha(z["inside"]),
        "aux_file": f"{name}_aux.npy", "aux_sha256": sha(z["aux"]),
        "stats": [int(x) for x in z["stats"]],
        "source": "reference classify_batch per polygon (oracle/_ref ref_classify_csr, unmodified "
                  "/root/reference/proj/include), all host threads",
    }


def run_case(name, kind, mode, n):
    if kind == "c3":
        return run_csr_case(name, kind, mode)
    poly, xy = inputs(kind)
    xy = xy[:n]
    parts_dir = os.path.join(CACHE, "parts", name)
    os.makedirs(parts_dir, exist_ok=True)
    stats = np.zeros(4, np.uint64)
    ins, aux = [], []
    for lo in range(0, n, PART):
        hi = min(n, lo + PART)
        f = os.path.join(parts_dir, f"{lo:012d}.npz")
        if not os.path.exists(f):
            t0 = time.time()
            v, st = oracle.ref_classify(xy[lo:hi], poly.vx, poly.vy, poly.ring_off, mode, TOL, workers=0)
            i_b, a_b = verdicts_to_bits(v, mode)
            np.savez(f + ".tmp.npz", inside=i_b, aux=a_b, stats=st)
            os.replace(f + ".tmp.npz", f)
            print(f"[{name}] points {lo}..{hi}: {time.time() - t0:.1f} s", flush=True)
        z = np.load(f)
        ins.append(z["inside"])
        aux.append(z["aux"])
        stats += z["stats"]
    inside = np.concatenate(ins)  # PART is a multiple of 32: parts concatenate word-aligned
    auxp = np.concatenate(aux)
    np.save(os.path.join(CACHE, f"{name}_inside.npy"), inside)
    np.save(os.path.join(CACHE, f"{name}_aux.npy"), auxp)
    return {
        "config": kind, "mode": mode, "n_points": n, "tol": TOL,
        "points_sha256": sha(xy), "vx_sha256": sha(poly.vx), "vy_sha256": sha(poly.vy),
        "ring_off": [int(v) for v in poly.ring_off],
        "inside_file": f"{name}_inside.npy", "inside_sha256": sha(inside),
        "aux_file": f"{name}_aux.npy", "aux_sha256": sha(auxp),
        "stats": [int(s) for s in stats],
        "source": "reference classify_batch (oracle/_ref, unmodified /root/reference/proj/include), workers=all",
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    assert oracle.ref_available(), "build oracle/_ref first (make -C oracle)"
    os.makedirs(CACHE, exist_ok=True)
    man = {}
    if os.path.exists(MANIFEST):
        man = json.load(open(MANIFEST))
    want = [s for s in args.only.split(",") if s] or list(cases())
    # cheap ones first, then the headline c4/C1, so partial runs still leave usable goldens
    pri = ["c1_C1", "c1_C2", "c1_Robust", "c3_C1", "c3_C2", "c3_Robust",
           "c2_n100000_C1", "c2_n100000_C2", "c2_n100000_Robust", "c2_n1000000_C1", "c4_C1",
           "c2_n1000000_C2", "c4_C2", "c2_n1000000_Robust", "c4_Robust"]
    done = {k for k, v in man.items() if os.path.exists(os.path.join(CACHE, v["inside_file"]))}
    want = [k for k in want if k not in done or args.only]
    order = sorted(want, key=lambda k: pri.index(k) if k in pri else len(pri))
    for name in order:
        kind, mode, n = cases()[name]
        t0 = time.time()
        man[name] = run_case(name, kind, mode, n)
        man[name]["ref_seconds"] = round(time.time() - t0, 1)
        with open(MANIFEST + ".tmp", "w") as fh:
            json.dump(man, fh, indent=1, sort_keys=True)
        os.replace(MANIFEST + ".tmp", MANIFEST)
        print(f"[{name}] done in {time.time() - t0:.0f} s; stats {man[name]['stats']}", flush=True)


if __name__ == "__main__":
    main()
