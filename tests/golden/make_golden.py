"""Generates tests/golden/golden_v1.npz — golden input/output vectors for the
batched point-in-polygon path, produced by the UNMODIFIED reference
implementation (classify_batch from /root/reference/proj/include/polycast,
built into oracle/_ref/libpolycast_ref.so by oracle/Makefile).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The .npz is committed; tests read it on machines without the reference.

Cases whose polygons have consecutive duplicate vertices cannot be built with
the reference's Ring type (geometry.hpp:54-59, SURVEY §8 rule P8); their
expected verdicts come from the C restatement (oracle/pip_oracle.c) and are
tagged source="port" — that restatement is itself pinned to the reference on
every duplicate-free case below.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import adversarial  # noqa: E402
import oracle  # noqa: E402
from paper_2306_04316_b200 import workloads as W  # noqa: E402

OUT = os.path.join(HERE, "golden_v1.npz")


def subset_csr(s, n_polys):
    """First n_polys polygons of a CSR set."""
    p = n_polys
    r1 = int(s.poly_ring_off[p])
    v1 = int(s.ring_off[r1])
    t = int(s.pt_off[p])
    return dict(xy=s.xy[:t].copy(), pt_off=s.pt_off[:p + 1].copy(), vx=s.vx[:v1].copy(), vy=s.vy[:v1].copy(),
                ring_off=s.ring_off[:r1 + 1].copy(), poly_ring_off=s.poly_ring_off[:p + 1].copy())


def main():
    assert oracle.ref_available(), "build oracle/_ref first (make -C oracle)"
    data = {}
    names = []

    def single(name, poly, xy, source):
        names.append(name)
        data[f"{name}/kind"] = np.array("single")
        data[f"{name}/source"] = np.array(source)
        data[f"{name}/xy"] = np.ascontiguousarray(xy, np.float64)
        data[f"{name}/vx"] = poly.vx
        data[f"{name}/vy"] = poly.vy
        data[f"{name}/ring_off"] = poly.ring_off
        for mode in (0, 1, 2):
            if source == "reference":
                v, st = oracle.ref_classify(xy, poly.vx, poly.vy, poly.ring_off, mode)
            else:
                v, st = oracle.port_classify(xy, poly.vx, poly.vy, poly.ring_off, mode)
            data[f"{name}/verdicts{mode}"] = v
            data[f"{name}/stats{mode}"] = st
            # contains() semantics (no prefilter): reference single-point calls
            if source == "reference" and len(xy) <= 4096:
                cv = np.array([oracle.ref_contains(p, poly.vx, poly.vy, poly.ring_off, mode) for p in xy], np.uint8)
            else:
                cv, _ = oracle.port_classify(xy, poly.vx, poly.vy, poly.ring_off, mode, prefilter=False)
            data[f"{name}/contains{mode}"] = cv

    def csr(name, d, source):
        names.append(name)
        data[f"{name}/kind"] = np.array("csr")
        data[f"{name}/source"] = np.array(source)
        for k, v in d.items():
            data[f"{name}/{k}"] = v
        from paper_2306_04316_b200.engine import CsrSet
        s = CsrSet(**d)
        for mode in (0, 1, 2):
            if source == "reference":
                v, st = oracle.ref_classify_csr(s, mode)
            else:
                v, st = oracle.port_classify_csr(s, mode)
            data[f"{name}/verdicts{mode}"] = v
            data[f"{name}/stats{mode}"] = st

    for name, poly, xy in adversarial.cases(include_dups=True):
        single(name, poly, xy, "port" if name == "dup_vertices" else "reference")

    poly = W.star_polygon(1000)
    single("c1_star1000_sample", poly, W.uniform_points(4096, (-1.0, -1.0, 1.0, 1.0), 11), "reference")
    poly = W.star_polygon(10)
    single("c2_star10_sample", poly, W.uniform_points(4096, W.bounds(poly), 12), "reference")
    poly = W.fractal_polygon(20_000)
    single("c4_fractal20k_sample", poly, W.uniform_points(2048, W.bounds(poly), 13), "reference")
    csr("c3_footprints_sample", subset_csr(W.footprints(4096), 96), "reference")
    csr("c5_degenerate_nodup_sample", subset_csr(W.degenerate(4096, allow_dups=False), 96), "reference")
    csr("c5_degenerate_dups_sample", subset_csr(W.degenerate(4096, allow_dups=True), 96), "port")

    data["__names__"] = np.array(names)
    np.savez_compressed(OUT, **data)
    print(f"wrote {OUT}: {len(names)} cases, {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
