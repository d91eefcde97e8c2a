#!/usr/bin/env python
"""Benchmark of the batched point-in-polygon path on B200 (one JSON line).

Default workload = BASELINE.json configs[3] ("Large region polygon"): one
200,000-vertex fractal star, 1e8 float64 query points uniform in its bbox,
C1 mode with classify_batch semantics, the points sharded over the GPUs (one
process per GPU under torchrun; strong scaling).  This is the configuration
BASELINE's "1/2/4/8 B200" metric is defined on and the largest single-GPU one.
One step = classify all 1e8 points (inputs resident in HBM; the polygon's
per-call prep, the y-ordering of the points, the scan and the bit-plane
finalize all inside the timed region).  Other configs: --workload c1 |
c2_sweep | c3 | c5.  The default line also carries the configs[1] O(n) sweep
(kernel time vs n, least-squares fit, R^2) measured after the timed region.

metric = point-edge tests/s (N_points x edges, the reference's linear-scan
work); points/s alongside.  The roofline of the scan kernel is its real bound
(warp-instruction issue, from the committed ncu capture of the same kernel),
with the reference-equivalent FP64 ratio reported separately and labelled.

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


def build_items(workload, rank, world, c4_total=100_000_000):
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
        from paper_2306_04316_b200.dist import shard_range
        total = c4_total
        lo, hi = shard_range(total, rank, world)
        poly, xy = W.config4(W.SEED, total, shard=(lo, hi))  # this rank's shard only
        return [Item("fractal200k", poly, xy)]
    if workload == "c3":
        return [Item("footprints1e6", csr=W.footprints(1_000_000, seed=seed))]
    if workload == "c5":
        return [Item("degenerate1e5", csr=W.degenerate(100_000, seed=seed))]
    raise SystemExit(f"unknown workload {workload}")


def cpu_sample(item, workload, scale=1.0):
    """Bounded CPU sample of an item: (xy_sample, tests) -- ~1e9-1e10 tests (x scale)."""
    if item.csr is not None:
        s = item.csr
        k = min(s.n_polys, 20_000)
        return ("csr", k), None
    m = item.n_points
    if workload == "c2_sweep":
        m = max(10_000, min(item.n_points, int(1e9 // max(item.poly.n_edges, 1))))
    elif workload == "c4":
        m = 100_000
    m = min(item.n_points, int(m * scale))
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
            "config": workload_config(args, world),
            "points_per_s": pts / dt,
            "cpu_baseline": {"value": value, "unit": "tests/s", "cores": threads,
                             "kind": "port" if args.workload == "c5" else "reference",
                             "sample": "; ".join(desc) + " per step (a bounded sample of the workload; reference "
                                       "classify_batch, workers=all)"},
            "e2e": {"value": value, "unit": "tests/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(args, world):
    """The config dict of the JSON line -- identical for both arms (the workload,
    not how an arm ran it)."""
    full = {"c4": (100_000_000, 100_000_000 * 200_000)}
    cfg = {"workload": WORKLOAD_NAMES[args.workload], "mode": MODE_NAMES[args.mode],
           "algorithm": "segment tree (opt-in extension, not the reference scan)" if args.tree == 1
           else "linear scan over every (point, edge) pair (geometry.hpp:182-203)",
           "parallelism": f"points sharded over {world} GPU(s)" if args.workload == "c4"
           else f"each of {world} GPU(s) classifies its own seeded point set",
           "l2": "inputs > L2 (1.6 GB of points); 256 MiB buffer also written between timed steps"
           if args.workload == "c4" else "256 MiB buffer written between timed steps (L2 flush)"}
    if args.workload in full:
        cfg["points_per_step"], cfg["tests_per_step"] = full[args.workload]
    return cfg


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
    # timed steps run as the library runs repeated device-pointer calls: replayed
    # CUDA graphs (PC_OPT_GRAPH; captured during the warm-up); the kernel times of
    # the roofline come from separate profiled steps right after the timed region
    eng.set_profiling(False)
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
    tot_ms = sum(step_ms)
    timed_launches = launches[0]
    n_prof = min(args.steps, 5)
    eng.set_profiling(True)  # per-kernel events (no graph replay while profiling)
    for _ in range(n_prof):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    kern_ms = eng.profile_take(0)
    eng.set_profiling(False)
    from paper_2306_04316_b200.dist import max_over_ranks
    max_ms = max_over_ranks(tot_ms, world, dev)
    tot_units, tot_pts = job_totals(items, world, dev)
    value = tot_units / (max_ms / args.steps / 1e3)

    # ---- roofline of the dominant kernel (rank 0's device) -----------------------------
    per_item_ms = np.array(kern_ms, dtype=np.float64).reshape(n_prof, len(items)).mean(0)
    roof = roofline(args, eng, items, per_item_ms, tot_ms)

    line = {"metric": "point-edge tests/s", "value": value, "unit": "tests/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
            "higher_is_better": True, "scaling": "strong" if args.workload == "c4" else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.json shapes)",
            "config": dict(workload_config(args, world), points_per_step=tot_pts, tests_per_step=tot_units),
            "points_per_s": tot_pts / (max_ms / args.steps / 1e3),
            "per_item_tests_per_s": {i.label: i.tests / (ms / 1e3) for i, ms in zip(items, per_item_ms)},
            "roofline": roof, "gpu_launches": timed_launches}

    if args.workload == "c2_sweep":
        line["sweep_fit"] = sweep_fit(items, per_item_ms)
    elif args.workload == "c4" and world == 1 and not args.no_sweep:
        # the second line: configs[1]'s O(n) sweep on the same scan (after the timed region)
        line["sweep"] = run_sweep(args, eng, dev)

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


def ncu_entry(workload, mode):
    """The committed ncu --set full summary of this config's dominant kernel
    (tools/summarize_profiles.py -> profiles/ncu_kernels.json), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_kernels.json")
    if not os.path.exists(path):
        return None
    return json.load(open(path)).get(f"{workload}_{MODE_NAMES[mode]}")


def roofline(args, eng, items, per_item_ms, tot_ms):
    """Roofline of the step's dominant kernel.

    c3 (many small polygons) is HBM-bound by design: algorithmic bytes (SURVEY
    §8(d)) / kernel time vs MEASURED_PEAKS.json hbm_gbs.  The single-polygon
    scan (c1, c2, c4) and c5 decide almost every (point, edge) pair with
    integer keys and certified fp32, so the FP64 pipe is not
    their bound; what they saturate is warp-instruction issue: achieved =
    instructions per launch (the committed ncu capture of the same kernel on
    the same config) / live kernel time, peak = 4 warp-instructions per cycle
    per SM x SMs x SM clock.  The reference-equivalent FP64 rate (2 flops per
    point-edge test of the reference's scan / time) is reported beside it,
    labelled: it is an algorithmic ratio, not a pipe utilisation."""
    import torch
    step_kern_ms = float(per_item_ms.sum())
    if args.workload == "c2_sweep":  # the sweep's dominant launch: its n = 1e6 item (the capture's config)
        items, per_item_ms = items[-1:], per_item_ms[-1:]
    kern_ms = float(per_item_ms.sum())
    kern_s = kern_ms / 1e3
    tests = float(sum(i.tests for i in items))
    props = torch.cuda.get_device_properties(torch.cuda.current_device())
    sms = props.multi_processor_count
    peaks = {}
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        peaks = json.load(open(pk))
    clk_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    ent = ncu_entry(args.workload, args.mode)
    if args.workload == "c3":
        bytes_launch = sum(i.bytes for i in items) / len(items)
        achieved = bytes_launch / (per_item_ms.mean() / 1e3) / 1e9
        peak = float(peaks.get("hbm_gbs", 6650.0))
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if peaks else "fallback 6650 GB/s",
                "algorithmic_bytes_per_launch": bytes_launch, "kernel": "pip_csr_tile_kernel"}
        if ent and ent.get("inst_per_launch"):  # what the kernel actually saturates
            issue_peak = 4.0 * sms * clk_mhz * 1e6
            ach_i = float(ent["inst_per_launch"]) / (per_item_ms.mean() / 1e3)
            roof["issue"] = {"achieved": ach_i, "peak": issue_peak, "unit": "warp-inst/s", "frac": ach_i / issue_peak,
                             "inst_per_launch": float(ent["inst_per_launch"]), "ipc": ent.get("ipc"),
                             "inst_source": ent["source"],
                             "peak_source": f"4 warp-inst/cycle/SM x {sms} SMs x {clk_mhz:.0f} MHz"}
    else:
        issue_peak = 4.0 * sms * clk_mhz * 1e6
        roof = {"bound": "issue", "unit": "warp-inst/s", "peak": issue_peak,
                "peak_source": f"4 warp-inst/cycle/SM x {sms} SMs x {clk_mhz:.0f} MHz (MEASURED_PEAKS sm_max_mhz)",
                "kernel": "pip_csr_tile_kernel" if items[0].csr is not None else "pip_tile_kernel (the linear scan)"}
        if ent and ent.get("inst_per_launch"):
            inst = float(ent["inst_per_launch"]) * len(items)
            roof["achieved"] = inst / kern_s
            roof["frac"] = roof["achieved"] / issue_peak
            roof["inst_per_launch"] = float(ent["inst_per_launch"])
            roof["inst_per_point_edge_test"] = inst / tests
            for k in ("ipc", "alu_pct", "fma_pct", "fp64_pct", "lsu_pct", "lts_pct", "dram_pct"):
                if k in ent:
                    roof[k] = ent[k]
            roof["inst_source"] = ent["source"]
        else:
            roof["achieved"] = None
            roof["frac"] = None
            roof["inst_source"] = "no committed ncu capture for this config/mode"
        fp64 = eng.fp64_rate(0, 300.0)
        ach = 2.0 * tests / kern_s / 1e12
        roof["fp64_reference_equivalent"] = {
            "achieved_tflops": ach, "peak_tflops": fp64 / 1e12, "ratio": ach / (fp64 / 1e12),
            "peak_source": "measured live: unfused DMUL+DADD probe (pc_measure_fp64_rate) on this GPU",
            "note": "2 FP64 flops per point-edge test of the reference's linear scan / kernel time; the kernel decides "
                    "pairs with exact integer keys and certified fp32 (DESIGN.md s3), so this is an algorithmic ratio, "
                    "not FP64-pipe utilisation (see fp64_pct)"}
    roof["kernel_ms_per_step"] = step_kern_ms
    roof["kernel_share_of_step"] = step_kern_ms / (tot_ms / args.steps)
    roof["traffic"] = None
    if ent and ent.get("dram_bytes_per_launch") is not None:
        roof["traffic"] = float(ent["dram_bytes_per_launch"])
        roof["traffic_source"] = ent["source"]
    return roof


def run_sweep(args, eng, dev):
    """configs[1]: star n in {1e1..1e6}, 1e6 points each: scan-kernel time per n
    (device events around the kernel, 3 runs after a warm-up), tests/s per n and
    the least-squares line of time vs n (the paper's O(n) claim)."""
    import torch
    items = build_items("c2_sweep", 0, 1)
    stream = torch.cuda.current_stream().cuda_stream
    ms = np.zeros(len(items))
    eng.set_profiling(True)
    for j, it in enumerate(items):
        xy = torch.from_numpy(it.xy).to(dev)
        vx, vy = torch.from_numpy(it.poly.vx).to(dev), torch.from_numpy(it.poly.vy).to(dev)
        ro = torch.from_numpy(np.ascontiguousarray(it.poly.ring_off).view(np.int64)).to(dev)
        nw = (it.n_points + 31) // 32
        bits = torch.zeros(2 * nw, dtype=torch.int32, device=dev)
        stats = torch.zeros(4, dtype=torch.int64, device=dev)
        eng.profile_take(0)
        for r in range(4):
            eng.classify_dev(0, stream, xy, it.n_points, vx, vy, ro, it.poly.n_rings, it.poly.n_verts, args.mode,
                             1e-12, True, bits[:nw], bits[nw:], stats)
        torch.cuda.synchronize()
        ms[j] = float(np.mean(eng.profile_take(0)[1:]))
    eng.set_profiling(False)
    return {"workload": WORKLOAD_NAMES["c2_sweep"], "mode": MODE_NAMES[args.mode],
            "kernel_ms": {it.label: float(m) for it, m in zip(items, ms)},
            "tests_per_s": {it.label: it.tests / (m / 1e3) for it, m in zip(items, ms)},
            "fit": sweep_fit(items, ms)}


def lsq_fit(x, t):
    """Least-squares line t = slope * x + intercept, solved exactly as the
    reference's least_squares_fit (proj/include/polycast/bench.hpp:123-150):
    sequential means, centred sums Sxx, Sxy, slope = Sxy / Sxx, intercept =
    mean_t - slope * mean_x (same operation order, so bit-identical results;
    tests/test_lsq_fit.py checks it against the reference)."""
    x = [float(v) for v in x]
    t = [float(v) for v in t]
    if len(x) < 2:
        raise ValueError("least_squares_fit: need at least 2 samples")
    mx = mt = 0.0
    for a, b in zip(x, t):
        mx += a
        mt += b
    mx /= len(x)
    mt /= len(x)
    sxx = sxy = 0.0
    for a, b in zip(x, t):
        d = a - mx
        sxx += d * d
        sxy += d * (b - mt)
    if sxx == 0.0:
        raise ValueError("least_squares_fit: all samples share one n_points value")
    slope = sxy / sxx
    return slope, mt - slope * mx


def error_rows(slope, intercept, x, t):
    """The reference's error_report (bench.hpp:176-198) for one fit:
    (predicted, absolute error, relative error or None) per sample."""
    out = []
    for a, b in zip(x, t):
        pred = slope * float(a) + intercept
        ab = abs(pred - float(b))
        out.append((pred, ab, ab / float(b) if float(b) > 0.0 else None))
    return out


def sweep_fit(items, per_item_ms):
    """The paper's O(n) claim on the GPU: least-squares line of kernel time vs n
    (edges) over the sweep (lsq_fit, the reference's least_squares_fit), its
    per-sample relative prediction error (error_rows, the reference's
    error_report) and R^2."""
    n = [it.tests / it.n_points for it in items]  # edges
    t = [float(m) / 1e3 for m in per_item_ms]
    slope, icpt = lsq_fit(n, t)
    rows = error_rows(slope, icpt, n, t)
    mt = sum(t) / len(t)
    ss_res = sum((b - r[0]) ** 2 for b, r in zip(t, rows))
    ss_tot = sum((b - mt) ** 2 for b in t)
    return {"x": "edges n", "y": "kernel seconds per 1e6-point launch", "slope_s_per_edge": slope,
            "intercept_s": icpt, "r2": 1.0 - ss_res / ss_tot if ss_tot > 0 else 1.0,
            "rel_err": {it.label: r[2] for it, r in zip(items, rows)}}


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
    out = {"value": units / dt, "unit": "tests/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
           "ms_per_step": dt * 1e3, "api": "pc_classify / pc_classify_csr (host pointers; all input and output buffers pinned)"}
    out["link"] = link_bound(host, dev, h2d, d2h, dt)
    return out


def link_bound(host, dev, h2d, d2h, dt):
    """The host link's share of the e2e step: the pinned host->device copy rate
    measured on this box (the largest input array of the step, copied 3 times
    into a device buffer, CUDA events on a side stream), the time the step's
    h2d + d2h bytes need at that rate, and that time / the measured e2e step."""
    import torch
    arrs = [a for xy, poly, cs, _ in host for a in ((xy,) if cs is None else (cs.xy,))]
    src = max(arrs, key=lambda a: a.nbytes)
    h = torch.from_numpy(src.view(np.uint8).reshape(-1))
    d = torch.empty(h.numel(), dtype=torch.uint8, device=dev)
    st = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(st):
        d.copy_(h, non_blocking=True)  # warm
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(3):
            d.copy_(h, non_blocking=True)
        e1.record(st)
    e1.synchronize()
    gbs = 3 * h.numel() / (e0.elapsed_time(e1) * 1e-3) / 1e9
    need_ms = (h2d + d2h) / (gbs * 1e9) * 1e3
    del d
    return {"h2d_gbs_measured": gbs, "copy_bytes": int(h.numel()), "achieved_gbs": (h2d + d2h) / dt / 1e9,
            "link_ms_per_step": need_ms, "frac": need_ms / (dt * 1e3),
            "note": "pinned torch copy_ of the step's largest input array, 3 reps, CUDA events; frac = (h2d + d2h bytes at that rate) / e2e ms"}


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
            run()  # warm-up
            best = float("inf")
            for _ in range(3):  # min of 3 timed runs (bench.hpp:109-117)
                t0 = time.perf_counter()
                run()
                best = min(best, time.perf_counter() - t0)
            tsum += best
            tests += sub.work()
            desc.append(f"{it.label}: first {k} polygons ({kind})")
            continue
        # cpu_baseline: ~10-30 s of CPU work in all (warm-up + 3 timed runs)
        xy, t = cpu_sample(it, args.workload, scale=5.0 if args.workload == "c4" else 1.0)
        h = oracle.RefPrepared(xy, it.poly.vx, it.poly.vy, it.poly.ring_off)
        warm = oracle.RefPrepared(xy[: max(1, len(xy) // 10)], it.poly.vx, it.poly.vy, it.poly.ring_off)
        warm.run(args.mode, workers=0)
        best = float("inf")
        for _ in range(3):  # min of 3 timed runs after a warm-up (bench.hpp:109-117)
            t0 = time.perf_counter()
            h.run(args.mode, workers=0)
            best = min(best, time.perf_counter() - t0)
        tsum += best
        tests += t
        desc.append(f"{it.label}: {len(xy)} pts")
    kind = "port" if any("(port)" in d for d in desc) else "reference"
    return {"value": tests / tsum, "unit": "tests/s", "cores": threads, "kind": kind,
            "sample": "; ".join(desc) + " (reference classify_batch, all host threads, min of 3 timed runs after a warm-up)",
            "seconds": tsum}


def run_dist_check(args, rank, world):
    """CPU check of this script's torchrun path (gloo, any world size): each rank
    builds only its configs[3] shard (build_items), a per-point stand-in flag
    (y above the bbox centre: no classification happens here) is packed into a
    bit plane and all-gathered with the same helper the GPU run uses, and the
    job totals / max-over-ranks reductions run; rank 0 checks everything
    against the single-process result and prints one JSON line."""
    import torch.distributed as dist

    from paper_2306_04316_b200 import pack_bits
    from paper_2306_04316_b200 import workloads as W
    from paper_2306_04316_b200.dist import gather_bit_planes, job_totals, max_over_ranks, shard_range
    import torch
    total = args.dist_check_points
    items = build_items("c4", rank, world, c4_total=total)
    it = items[0]
    lo, hi = shard_range(total, rank, world)
    assert it.n_points == hi - lo
    box = W.bounds(it.poly)
    cy = 0.5 * (box[1] + box[3])
    local = torch.from_numpy(pack_bits(it.xy[:, 1] > cy).view(np.int32).copy())
    full = gather_bit_planes(local, total, world)
    units, pts = job_totals(it.tests, it.n_points, world)
    mx = max_over_ranks(float(rank + 1), world)
    ok = True
    if rank == 0:
        _, xy = W.config4(W.SEED, total)
        ok = (np.array_equal(full, pack_bits(xy[:, 1] > cy)) and pts == total
              and units == total * it.poly.n_edges and mx == float(world))
        print(json.dumps({"dist_check": "ok" if ok else "FAILED", "world": world, "points": total,
                          "backend": dist.get_backend()}), flush=True)
    return ok


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=list(WORKLOAD_NAMES))
    ap.add_argument("--no-sweep", action="store_true", help="c4: skip the configs[1] sweep sub-line")
    ap.add_argument("--dist-check", action="store_true",
                    help="CPU/gloo check of the torchrun plumbing (shards, gather, reductions); no GPU, no timing")
    ap.add_argument("--dist-check-points", type=int, default=1_000_003)
    ap.add_argument("--mode", type=int, default=0, choices=[0, 1, 2])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--bucket", type=int, default=None, choices=[-1, 0, 1], help="y-bucketing: auto/off/on")
    ap.add_argument("--tree", type=int, default=None, choices=[0, 1],
                    help="opt-in segment tree (an extension outside the reference's linear scan): 0 off (default), 1 on")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)  # timing rule: at least 3 untimed warm-up steps (reported as run)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.dist_check:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        try:
            ok = run_dist_check(args, rank, world)
        finally:
            dist.destroy_process_group()
        raise SystemExit(0 if ok else 1)
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
