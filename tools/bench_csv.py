"""Points-CSV ingest benchmark: the GPU reader
(pc_parse_points_csv[_dev], paper_2306_04316_b200/csrc/pip_csv.cu) on a
synthetic 'id,lon,lat' file of N rows with 17-significant-digit coordinates
(the format the reference's write_results_csv emits, io.hpp:137-141), against
the reference's read_points_csv (oracle/_ref, single-threaded like the
reference) on a bounded sample of the same file.

  python tools/bench_csv.py [--rows N] [--steps K] [--warmup W]

Prints one JSON line:
  value     rows/s of the kernel alone, text resident in HBM, L2 flushed
            between timed launches (CUDA events on the launching stream);
  e2e       rows/s through the host C-ABI call (pageable text in, points out:
            upload, kernel, download inside the timed region);
  roofline  HBM: algorithmic bytes = text bytes read once + 16 B per row
            written, over the kernel time, against MEASURED_PEAKS.json;
  cpu_baseline  the reference reader on the first --cpu-rows rows.
"""
import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def make_text(n, seed=11):
    rng = np.random.default_rng(seed)
    lon = rng.uniform(-180.0, 180.0, n)
    lat = rng.uniform(-90.0, 90.0, n)
    parts = [b"id,lon,lat\n"]
    step = 1 << 18
    for s in range(0, n, step):
        e = min(n, s + step)
        parts.append("".join("%d,%.17g,%.17g\n" % (i, a, b)
                             for i, a, b in zip(range(s, e), lon[s:e].tolist(), lat[s:e].tolist())).encode())
    return b"".join(parts), np.stack([lon, lat], 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=10_000_000)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cpu-rows", type=int, default=1_000_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    import torch
    from paper_2306_04316_b200 import Engine

    t0 = time.perf_counter()
    text, want = make_text(args.rows)
    print(f"generated {len(text) / 1e6:.1f} MB in {time.perf_counter() - t0:.1f} s", file=sys.stderr)
    data_start = text.index(b"\n") + 1
    eng = Engine(devices=[0])
    dev = torch.device("cuda:0")
    d_text = torch.frombuffer(bytearray(text), dtype=torch.uint8).to(dev)
    d_out = torch.empty((args.rows, 2), dtype=torch.float64, device=dev)
    d_res = torch.zeros(4, dtype=torch.int64, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)
    stream = torch.cuda.Stream(dev)  # a real stream: the C-ABI launches on it (null = the context's own)
    sp = stream.cuda_stream

    def launch():
        eng.parse_points_csv_dev(0, sp, d_text, len(text), data_start, 1, 2, ",", d_out, args.rows, d_res)

    for _ in range(max(3, args.warmup)):
        launch()
    torch.cuda.synchronize()
    res = d_res.cpu().numpy().view(np.uint64)
    assert int(res[0]) == args.rows and int(res[1]) == 0, res
    assert d_out.cpu().numpy().tobytes() == want.tobytes(), "parity: GPU points differ from the written doubles"

    # kernel time: the C-ABI's own event pair around the launch, on its stream
    eng.set_profiling(True)
    eng.profile_take(0)
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()  # L2 flush, outside the event pair
        launch()
        stream.synchronize()
    ms = eng.profile_take(0)
    eng.set_profiling(False)
    assert len(ms) == args.steps
    kern_ms = float(np.median(ms))

    # end to end through the host C-ABI (pageable bytes in, points out)
    eng.parse_points_csv(text, data_start, 1, 2, ",")
    e2e_s = []
    for _ in range(max(3, args.steps // 2)):
        t = time.perf_counter()
        xy, n_bad, _, _ = eng.parse_points_csv(text, data_start, 1, 2, ",")
        e2e_s.append(time.perf_counter() - t)
    assert len(xy) == args.rows and n_bad == 0
    e2e = float(np.median(e2e_s))

    # where the end-to-end time goes (stderr only): pageable and pinned uploads of the text
    src = torch.frombuffer(bytearray(text), dtype=torch.uint8)
    pin = src.pin_memory()
    for name, h in (("pageable", src), ("pinned", pin)):
        torch.cuda.synchronize()
        t = time.perf_counter()
        d_text.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        print(f"h2d {name}: {len(text) / (time.perf_counter() - t) / 1e9:.1f} GB/s", file=sys.stderr)
    del pin

    peaks = {}
    pp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pp):
        peaks = json.load(open(pp))
    peak = peaks.get("hbm_gbs", 7672.0)
    traffic = {}  # DRAM bytes per launch from the last committed ncu --set full capture
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        traffic = json.load(open(tf))
    alg = len(text) + 16 * args.rows
    achieved = alg / (kern_ms * 1e-3) / 1e9

    cpu = None
    if not args.no_cpu_baseline:
        import oracle
        if oracle.ref_available():
            k = min(args.cpu_rows, args.rows)
            end = 0
            for _ in range(k + 1):
                end = text.index(b"\n", end) + 1
            with tempfile.NamedTemporaryFile(suffix=".csv", delete=False) as f:
                f.write(text[:end])
                path = f.name
            oracle.ref_read_points_csv(path, "lon", "lat", cap=k + 16)  # warm (page cache)
            t = time.perf_counter()
            r = oracle.ref_read_points_csv(path, "lon", "lat", cap=k + 16)
            cs = time.perf_counter() - t
            os.unlink(path)
            assert r["kind"] == 0 and len(r["points"]) == k
            assert r["points"].tobytes() == want[:k].tobytes()
            cpu = {"value": k / cs, "unit": "rows/s", "cores": 1, "kind": "reference",
                   "sample": f"reference read_points_csv on the first {k} rows ({end / 1e6:.1f} MB, file in page "
                             f"cache), 1 timed run after a warm-up; the reference reader is single-threaded"}

    line = {"metric": "csv_ingest_rows_per_s", "value": args.rows / (kern_ms * 1e-3), "unit": "rows/s",
            "n_gpus": 1, "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": kern_ms,
            "higher_is_better": True, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"points CSV id,lon,lat: {args.rows} rows, %.17g coordinates, "
                                   f"{len(text)} bytes", "l2": "256 MiB buffer written between timed launches"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": (traffic.get("csv_parse") or {}).get("dram_bytes_per_launch"),
                         "algorithmic_bytes": alg, "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else
                         "B200_PROFILING.md fallback"},
            "e2e": {"value": args.rows / e2e, "unit": "rows/s", "h2d_bytes_per_step": len(text),
                    "d2h_bytes_per_step": 16 * args.rows + 32, "seconds": e2e},
            "gpu_launches": 3, "cpu_baseline": cpu, "kernel_ms_all": ms}
    print(json.dumps(line), flush=True)

    # ---- results-CSV writer (write_results_csv): the parsed points as records
    from paper_2306_04316_b200.engine import RESULT_RECORD
    rng = np.random.default_rng(5)
    n = args.rows
    recs = np.zeros(n, dtype=RESULT_RECORD)
    recs["index"] = np.arange(n)
    recs["x"], recs["y"] = want[:, 0], want[:, 1]
    recs["verdict"] = rng.integers(0, 4, n).astype(np.uint8)
    d_recs = torch.from_numpy(recs.view(np.uint8)).to(dev)
    cap = 18 + 80 * n
    d_txt = torch.empty(cap, dtype=torch.uint8, device=dev)
    d_len = torch.zeros(1, dtype=torch.int64, device=dev)

    def emit():
        eng.format_results_csv_dev(0, sp, d_recs, n, d_txt, cap, d_len)

    for _ in range(3):
        emit()
    torch.cuda.synchronize()
    out_len = int(d_len.item())
    eng.set_profiling(True)
    eng.profile_take(0)
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        emit()
        stream.synchronize()
    ems = eng.profile_take(0)
    eng.set_profiling(False)
    emit_ms = float(np.median(ems))
    host_text = eng.format_results_csv(recs)  # records in host memory, as write_results_csv gets them
    assert len(host_text) == out_len
    ee = []
    for _ in range(max(3, args.steps // 2)):
        t = time.perf_counter()
        eng.format_results_csv(recs)
        ee.append(time.perf_counter() - t)
    e2e_emit = float(np.median(ee))
    cpu2 = None
    if not args.no_cpu_baseline:
        import oracle
        if oracle.ref_available():
            k = min(args.cpu_rows, n)
            with tempfile.NamedTemporaryFile(suffix=".csv", delete=False) as f:
                path = f.name
            t = time.perf_counter()
            rc = oracle.ref_write_results_csv(path, recs["index"][:k], want[:k], recs["verdict"][:k])
            cs = time.perf_counter() - t
            ref_bytes = open(path, "rb").read()
            os.unlink(path)
            assert rc == 0
            gpu_k = eng.format_results_csv(np.ascontiguousarray(recs[:k])).tobytes()
            assert gpu_k == ref_bytes, "parity: GPU text differs from the reference writer"
            cpu2 = {"value": k / cs, "unit": "rows/s", "cores": 1, "kind": "reference",
                    "sample": f"reference write_results_csv of the first {k} records (to a file in /tmp, page "
                              f"cache), 1 timed run; byte-identical to the GPU text"}
    alg2 = 32 * n + out_len
    ach2 = alg2 / (emit_ms * 1e-3) / 1e9
    line2 = {"metric": "csv_emit_rows_per_s", "value": n / (emit_ms * 1e-3), "unit": "rows/s", "n_gpus": 1,
             "steps": args.steps, "warmup": 3, "ms_per_step": emit_ms, "higher_is_better": True, "dtype": "f64",
             "data": "synthetic",
             "config": {"workload": f"write_results_csv text of {n} records ({out_len} bytes), the parsed points, "
                                    f"random verdicts", "l2": "256 MiB buffer written between timed launches"},
             "roofline": {"bound": "hbm", "achieved": ach2, "peak": peak, "unit": "GB/s", "frac": ach2 / peak,
                          "traffic": (traffic.get("csv_emit") or {}).get("dram_bytes_per_launch"), "algorithmic_bytes": alg2},
             "e2e": {"value": n / e2e_emit, "unit": "rows/s", "h2d_bytes_per_step": 32 * n,
                     "d2h_bytes_per_step": out_len, "seconds": e2e_emit},
             "gpu_launches": 3, "cpu_baseline": cpu2, "kernel_ms_all": ems}
    print(json.dumps(line2), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
