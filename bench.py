#!/usr/bin/env python
"""Benchmark of the batched point-in-polygon path on B200 (one JSON line).

Default workload = BASELINE.json configs[1], the O(n) scaling sweep: star
polygons with n in {10, 1e2, 1e3, 1e4, 1e5, 1e6} vertices, 1e6 float64 query
points uniform in each polygon's bbox.  One step = classify all six point sets
(C1 mode, classify_batch semantics) with inputs resident in HBM.  Other
configs: --workload c1 | c4 | c3 | c5.

metric = point-edge tests/s (N_points x edges summed over the step); points/s
is reported alongside.  Multi-GPU: one process per GPU (torchrun); sweep/c1/
c3/c5 scale weakly (each rank its own seeded points), c4 strongly (1e8 points
sharded).  Bit planes are gathered to rank 0 with NCCL at the end of each step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload ...] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------- workloads
class Item:
    """One classify call of a step: a single polygon + points, or a CSR set."""

    def __init__(self, label, poly=None, xy=None, csr=None):
        self.label, self.poly, self.xy, self.csr = label, poly, xy, csr
        if csr is None:
            self.n_points = len(xy)
            self.tests = self.n_points * poly.n_edges
            self.bytes = 16 * self.n_points + self.n_points / 8 + 16 * poly.n_verts
        else:
            self.n_points = csr.n_points
            self.tests = csr.work()
            # 16 B/pt + 1/8 B/pt flags + 16 B/vertex + 8 B/polygon offsets (pt_off and ring CSR)
            self.bytes = (16 * self.n_points + self.n_points / 8 + 16 * len(csr.vx) + 8 * (csr.n_polys + 1) * 2
                          + 8 * len(csr.ring_off))


def build_items(workload, rank, world):
    from paper_2306_04316_b200 import workloads as W
    seed = W.SEED + 1000 * rank
    if workload == "c2_sweep":
        items = []
        for n in W.SWEEP_N:
            poly = W.star_polygon(n, W.SEED)
            items.append(Item(f"n={n}", poly, W.uniform_points(1_000_000, W.bounds(poly), seed + 2 + n)))
        return items
    if workload == "c1":
        poly = W.star_polygon(1000, W.SEED)
        return [Item("star1000", poly, W.uniform_points(1_000_000, (-1.0, -1.0, 1.0, 1.0), seed + 1))]
    if workload == "c4":
        poly = W.fractal_polygon(200_000, W.SEED)
        from paper_2306_04316_b200.dist import shard_range
        total = 100_000_000
        lo, hi = shard_range(total, rank, world)
        xy = W.uniform_points(total, W.bounds(poly), W.SEED + 4)
        return [Item("fractal200k", poly, np.ascontiguousarray(xy[lo:hi]) if world > 1 else xy)]
    if workload == "c3":
        return [Item("footprints1e6", csr=W.footprints(1_000_000, seed=seed))]
    if workload == "c5":
        return [Item("degenerate1e5", csr=W.degenerate(100_000, seed=seed))]
    raise SystemExit(f"unknown workload {workload}")


def cpu_sample(item, workload):
    """Bounded CPU sample of an item: (xy_sample, tests) — sized ~1e9-1e10 tests."""
    if item.csr is not None:
        s = item.csr
        k = min(s.n_polys, 20_000)
        return ("csr", k), None
    m = item.n_points
    if workload == "c2_sweep":
        m = max(10_000, min(item.n_points, int(1e9 // max(item.poly.n_edges, 1))))
    elif workload == "c4":
        m = 50_000
    return np.ascontiguousarray(item.xy[:m]), m * item.poly.n_edges


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev, self.lines, self.proc = dev, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.dev)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return
    import oracle
    items = build_items(args.workload, 0, 1)
    threads = oracle.host_threads()
    prepared, tests, pts, desc = [], 0, 0, []
    for it in items:
        if it.csr is not None:
            from paper_2306_04316_b200.engine import CsrSet
            s = it.csr
            k = min(s.n_polys, 20_000)
            sub = CsrSet(s.xy[:int(s.pt_off[k])], s.pt_off[:k + 1], s.vx, s.vy, s.ring_off, s.poly_ring_off[:k + 1])
            prepared.append(("csr", sub))
            tests += sub.work()
            pts += sub.n_points
            desc.append(f"{it.label}: first {k} polygons")
        else:
            xy, t = cpu_sample(it, args.workload)
            prepared.append(("single", oracle.RefPrepared(xy, it.poly.vx, it.poly.vy, it.poly.ring_off)))
            tests += t
            pts += len(xy)
            desc.append(f"{it.label}: {len(xy)} pts")

    def csr_run(sub):
        try:
            return oracle.ref_classify_csr(sub, args.mode, threads=threads)
        except oracle.RefError:  # duplicate vertices (config 5): the pinned C restatement
            return oracle.port_classify_csr(sub, args.mode, threads=threads)

    def step():
        for kind, h in prepared:
            if kind == "csr":
                csr_run(h)
            else:
                h.run(args.mode, workers=0)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    value = tests / dt
    line = {"metric": "point-edge tests/s", "value": value, "unit": "tests/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak" if args.workload != "c4" else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": WORKLOAD_NAMES[args.workload], "mode": MODE_NAMES[args.mode]},
            "points_per_s": pts / dt,
            "cpu_baseline": {"value": value, "unit": "tests/s", "cores": threads,
                             "kind": "port" if args.workload == "c5" else "reference",
                             "sample": "; ".join(desc) + " per step (reference classify_batch, workers=all)"},
            "e2e": {"value": value, "unit": "tests/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


WORKLOAD_NAMES = {
    "c2_sweep": "configs[1] O(n) sweep: star n in {1e1..1e6}, 1e6 f64 points each",
    "c1": "configs[0] star n=1000, 1e6 f64 points in [-1,1]^2",
    "c4": "configs[3] fractal star n=200000, 1e8 f64 points (sharded)",
    "c3": "configs[2] 1e6 building footprints x 64 points (CSR)",
    "c5": "configs[4] 1e5 degenerate integer-grid polygons, ~1e7 points (CSR)",
}
MODE_NAMES = {0: "C1", 1: "C2", 2: "Robust"}


# ---------------------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2306_04316_b200 import Engine

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    # an explicit stream: the library and the timing events must share it
    # (the legacy default stream's handle is 0, which the C-ABI reads as "context stream")
    torch.cuda.set_stream(torch.cuda.Stream(device=dev))
    eng = Engine(devices=[local_rank])
    if args.bucket is not None:
        eng.set_bucketing(args.bucket)
    if args.tree is not None:
        eng.set_tree(args.tree)
    items = build_items(args.workload, rank, world)
    log(f"[rank {rank}] workload {args.workload}: {len(items)} items, "
        f"{sum(i.tests for i in items):.3e} tests/step, {sum(i.n_points for i in items)} points/step")

    def u64(a):
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)

    # device-resident inputs and outputs
    dv = []
    for it in items:
        d = {}
        if it.csr is None:
            d["xy"] = torch.from_numpy(it.xy).to(dev)
            d["vx"] = torch.from_numpy(it.poly.vx).to(dev)
            d["vy"] = torch.from_numpy(it.poly.vy).to(dev)
            d["ro"] = u64(it.poly.ring_off)
        else:
            s = it.csr
            d["xy"] = torch.from_numpy(s.xy).to(dev)
            d["pt_off"], d["ro"], d["pro"] = u64(s.pt_off), u64(s.ring_off), u64(s.poly_ring_off)
            d["vx"], d["vy"] = torch.from_numpy(s.vx).to(dev), torch.from_numpy(s.vy).to(dev)
        nw = (it.n_points + 31) // 32
        d["bits"] = torch.zeros(2 * nw, dtype=torch.int32, device=dev)
        d["stats"] = torch.zeros(4, dtype=torch.int64, device=dev)
        d["nw"] = nw
        if world > 1:
            d["gather"] = torch.zeros(world * nw, dtype=torch.int32, device=dev)
        dv.append(d)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)  # 256 MiB > 126 MB L2
    eng.set_profiling(True)
    launches = [0]

    def step():
        stream = torch.cuda.current_stream().cuda_stream
        for it, d in zip(items, dv):
            nw = d["nw"]
            if it.csr is None:
                eng.classify_dev(0, stream, d["xy"], it.n_points, d["vx"], d["vy"], d["ro"], it.poly.n_rings,
                                 it.poly.n_verts, args.mode, 1e-12, True, d["bits"][:nw], d["bits"][nw:],
                                 d["stats"])
            else:
                eng.classify_csr_dev(0, stream, d["xy"], d["pt_off"], it.csr.n_polys, it.n_points, d["vx"], d["vy"],
                                     d["ro"], d["pro"], args.mode, 1e-12, d["bits"][:nw], d["bits"][nw:],
                                     d["stats"])
            launches[0] += eng.last_launch_count
            if world > 1:  # final-result gather of the inside plane (NCCL over NVLink)
                dist.all_gather_into_tensor(d["gather"], d["bits"][:nw])

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    eng.profile_take(0)
    if world > 1:
        dist.barrier()
    launches[0] = 0
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for k in range(args.steps):
            flush.zero_()  # L2 flush between timed steps, outside the events
            starts[k].record()
            step()
            ends[k].record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    kern_ms = eng.profile_take(0)
    tot_ms = sum(step_ms)
    from paper_2306_04316_b200.dist import max_over_ranks
    max_ms = max_over_ranks(tot_ms, world, dev)
    tot_units, tot_pts = job_totals(items, world, dev)
    value = tot_units / (max_ms / args.steps / 1e3)

    # ---- roofline of the dominant kernel (rank 0's device) -----------------------------
    per_item_ms = np.array(kern_ms, dtype=np.float64).reshape(args.steps, len(items)).mean(0)
    csr = items[0].csr is not None
    # configs 3 (and 2 at n <= ~25) are HBM-bound, configs 1, 2, 4
    # and 5 (~35 edges per point) FP64-bound
    if args.workload == "c3":
        bytes_launch = sum(i.bytes for i in items) / len(items)
        achieved = bytes_launch / (per_item_ms.mean() / 1e3) / 1e9
        peak_src = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
            os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
        peak = peak_src.get("hbm_gbs", 6650.0)
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if peak_src else "fallback 6650 GB/s"}
    else:
        fp64 = eng.fp64_rate(0, 300.0)
        flops = 2.0 * sum(i.tests for i in items)
        achieved = flops / (per_item_ms.sum() / 1e3) / 1e12
        roof = {"bound": "fp64", "achieved": achieved, "peak": fp64 / 1e12, "unit": "TFLOP/s",
                "frac": achieved / (fp64 / 1e12),
                "peak_source": "measured live: unfused DMUL+DADD probe (pc_measure_fp64_rate) on this GPU",
                "flops_per_test": 2}
    roof["kernel"] = "pip_csr_kernel" if csr else "pip_single_kernel"
    if not csr and args.mode in (0, 1) and args.tree != 0:
        # C1 / C2 single polygons with >= 4096 vertices take the segment-tree path
        # (pip_tree.cu, PC_OPT_TREE auto): O(log^2 n) comparisons per point instead
        # of a scan over the edges, so the reference-equivalent FP64 work per
        # second exceeds the FP64 peak by the algorithmic factor
        roof["kernel"] = "segment tree (pip_tree.cu) for n_verts >= 4096, scan kernel (pip_single.cu) below"
        roof["note"] = ("achieved = reference-equivalent work (2 FP64 flops per point-edge test) / time; "
                        "the tree does O(log^2 n) work per point, so frac > 1 is the algorithmic gain")
    roof["kernel_ms_per_step"] = float(per_item_ms.sum())
    roof["kernel_share_of_step"] = float(per_item_ms.sum() / (tot_ms / args.steps))
    # DRAM bytes per launch of the dominant kernel from the committed ncu --set full
    # capture (tools/summarize_profiles.py); the sweep's is its n = 1e6 launch
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf) and args.mode == 0:
        # C1 sweep / c4 run the segment tree: its query kernel's capture; c1 the scan kernel
        ent = json.load(open(tf)).get({"c2_sweep": "tree_query"}.get(args.workload, args.workload))
        if ent:
            traffic = ent["dram_bytes_per_launch"]
            roof["traffic_source"] = ent["source"]
    roof["traffic"] = traffic

    line = {"metric": "point-edge tests/s", "value": value, "unit": "tests/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
            "higher_is_better": True, "scaling": "strong" if args.workload == "c4" else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.json shapes)",
            "config": {"workload": WORKLOAD_NAMES[args.workload], "mode": MODE_NAMES[args.mode],
                       "points_per_step": tot_pts, "tests_per_step": tot_units,
                       "parallelism": f"points sharded over {world} GPU(s)",
                       "l2": "256 MiB buffer written between timed steps (L2 flush)"},
            "points_per_s": tot_pts / (max_ms / args.steps / 1e3),
            "per_item_tests_per_s": {i.label: i.tests / (ms / 1e3) for i, ms in zip(items, per_item_ms)},
            "roofline": roof, "gpu_launches": launches[0]}

    if args.workload == "c2_sweep":
        line["sweep_fit"] = sweep_fit(items, per_item_ms)

    # ---- clocks -------------------------------------------------------------------------
    line["clocks"] = clk.summary()
    if max_over_ranks(float(line["clocks"]["samples"] < 3), world, dev) > 0:
        # the timed region was shorter than nvidia-smi's sampling period: repeat the
        # same step (untimed, right after the timed region) for ~1 s under the
        # sampler; the repeat count comes from the max-over-ranks step time, so
        # every rank runs the same number of steps (they may hold collectives)
        n_rep = int(min(100_000, max(1, 1000.0 / max(max_ms / args.steps, 1e-3))))
        with ClockSampler(local_rank) as clk2:
            for _ in range(n_rep):
                step()
            torch.cuda.synchronize()
        line["clocks"] = dict(clk2.summary(), window="repeat of the step right after the timed region "
                                                      f"(timed region {tot_ms:.1f} ms < sampler period)")
        eng.profile_take(0)

    # ---- e2e through the public host API (pinned host buffers, copies timed) --------------
    if not args.no_e2e:
        e2e = run_e2e(args, eng, items, world, rank)
        line["e2e"] = e2e

    # ---- CPU baseline: reference on the host cores (rank 0, N=1) ----------------------
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = run_cpu_baseline(args, items)
    if rank == 0:
        print(json.dumps(line), flush=True)
    eng.close()


def sweep_fit(items, per_item_ms):
    """The paper's O(n) claim on the GPU: least-squares line of kernel time vs n
    (vertices) over the sweep, solved on centred data as the reference's
    least_squares_fit (bench.hpp:120-148), with its per-sample relative
    prediction error (error_report, bench.hpp:172-199) and R^2."""
    n = np.array([it.tests / it.n_points for it in items], dtype=np.float64)  # edges
    t = np.asarray(per_item_ms, dtype=np.float64) / 1e3
    dn, dt = n - n.mean(), t - t.mean()
    slope = float((dn * dt).sum() / (dn * dn).sum())
    icpt = float(t.mean() - slope * n.mean())
    pred = slope * n + icpt
    ss_res, ss_tot = float(((t - pred) ** 2).sum()), float((dt * dt).sum())
    return {"x": "edges n", "y": "kernel seconds per 1e6-point launch", "slope_s_per_edge": slope,
            "intercept_s": icpt, "r2": 1.0 - ss_res / ss_tot if ss_tot > 0 else 1.0,
            "rel_err": {it.label: float(abs(p - a) / a) for it, p, a in zip(items, pred, t)}}


def job_totals(items, world, dev):
    """(tests, points) processed by all ranks in one step."""
    from paper_2306_04316_b200.dist import job_totals as jt
    return jt(sum(i.tests for i in items), sum(i.n_points for i in items), world, dev)


def run_e2e(args, eng, items, world, rank):
    import torch
    import torch.distributed as dist
    from paper_2306_04316_b200.engine import CsrSet

    from paper_2306_04316_b200.engine import Polygon

    def pinned(a):
        """A page-locked copy of array a (the caller's buffers, as a user would pin them)."""
        a = np.ascontiguousarray(a)
        t = torch.empty(max(a.nbytes, 1), dtype=torch.uint8, pin_memory=True).numpy()[:a.nbytes]
        t = t.view(a.dtype).reshape(a.shape)
        t[...] = a
        return t

    def pinned_out(nw):
        return torch.empty(nw, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)

    host = []
    h2d = d2h = 0
    for it in items:
        nw = (it.n_points + 31) // 32
        if it.csr is None:
            xy = pinned(it.xy)
            poly = Polygon(pinned(it.poly.vx), pinned(it.poly.vy), pinned(it.poly.ring_off))
            host.append((xy, poly, None, (None, pinned_out(nw), pinned_out(nw))))
            h2d += xy.nbytes + poly.vx.nbytes * 2 + poly.ring_off.nbytes
        else:
            s = it.csr
            cs = CsrSet(pinned(s.xy), pinned(s.pt_off), pinned(s.vx), pinned(s.vy), pinned(s.ring_off),
                        pinned(s.poly_ring_off))
            host.append((None, None, cs, (None, pinned_out(nw), pinned_out(nw))))
            h2d += cs.xy.nbytes + cs.pt_off.nbytes + cs.vx.nbytes * 2 + cs.ring_off.nbytes + cs.poly_ring_off.nbytes
        d2h += 2 * nw * 4 + 32

    def step():
        for xy, poly, cs, out in host:
            if cs is None:
                eng.classify(xy, poly, args.mode, out=out)
            else:
                eng.classify_csr(cs, args.mode, out=out)

    for _ in range(max(1, args.warmup)):
        step()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    from paper_2306_04316_b200.dist import max_over_ranks
    dev = torch.device("cuda", torch.cuda.current_device())
    dt = max_over_ranks(dt, world, dev) / args.steps
    units, _ = job_totals(items, world, dev)
    return {"value": units / dt, "unit": "tests/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": dt * 1e3, "api": "pc_classify / pc_classify_csr (host pointers; all input and output buffers pinned)"}


def run_cpu_baseline(args, items):
    import oracle
    if not oracle.ref_available():
        return None
    threads = oracle.host_threads()
    tests = 0
    tsum = 0.0
    desc = []
    for it in items:
        if it.csr is not None:
            from paper_2306_04316_b200.engine import CsrSet
            s = it.csr
            k = min(s.n_polys, 20_000)
            sub = CsrSet(s.xy[:int(s.pt_off[k])], s.pt_off[:k + 1], s.vx, s.vy, s.ring_off, s.poly_ring_off[:k + 1])
            try:
                oracle.ref_classify_csr(sub, args.mode, threads=threads)
                run, kind = (lambda: oracle.ref_classify_csr(sub, args.mode, threads=threads)), "reference"
            except oracle.RefError:
                # config 5 has consecutive duplicate vertices, which the reference Ring
                # rejects: the pinned C restatement stands in
                run, kind = (lambda: oracle.port_classify_csr(sub, args.mode, threads=threads)), "port"
            t0 = time.perf_counter()
            run()
            tsum += time.perf_counter() - t0
            tests += sub.work()
            desc.append(f"{it.label}: first {k} polygons ({kind})")
            continue
        xy, t = cpu_sample(it, args.workload)
        h = oracle.RefPrepared(xy, it.poly.vx, it.poly.vy, it.poly.ring_off)
        warm = oracle.RefPrepared(xy[: max(1, len(xy) // 10)], it.poly.vx, it.poly.vy, it.poly.ring_off)
        warm.run(args.mode, workers=0)
        t0 = time.perf_counter()
        h.run(args.mode, workers=0)
        tsum += time.perf_counter() - t0
        tests += t
        desc.append(f"{it.label}: {len(xy)} pts")
    kind = "port" if any("(port)" in d for d in desc) else "reference"
    return {"value": tests / tsum, "unit": "tests/s", "cores": threads, "kind": kind,
            "sample": "; ".join(desc) + " (reference classify_batch, all host threads, 1 timed run after warm-up)",
            "seconds": tsum}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2_sweep", choices=list(WORKLOAD_NAMES))
    ap.add_argument("--mode", type=int, default=0, choices=[0, 1, 2])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--bucket", type=int, default=None, choices=[-1, 0, 1], help="y-bucketing: auto/off/on")
    ap.add_argument("--tree", type=int, default=None, choices=[-1, 0, 1],
                    help="segment tree for single polygons: auto/off (the linear scan only)/on")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)  # timing rule: at least 3 untimed warm-up steps (reported as run)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
