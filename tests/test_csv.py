"""Points-CSV ingest: the GPU reader behind
pc_parse_points_csv / polycast::read_points_csv against the reference's
read_points_csv and detail::parse_double (proj/include/polycast/io.hpp:111-119,
148-225), compiled unmodified into oracle/_ref.

CPU: the device number parser compiled as host code vs std::from_chars
(tests/cpp/parse_test, ~2M strings) and the reference parser's own semantics.
GPU: cell-by-cell parity with the reference parser, whole files (header,
CRLF, empty lines, short rows, bad cells, no final newline) in lenient mode
vs the reference reader, and the 17-significant-digit round trip of 2^20
random doubles (bit-exact)."""
import os
import subprocess

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def test_device_parser_vs_from_chars():
    subprocess.run(["make", "-s", "-C", CPP, os.path.join(CPP, "parse_test")], check=True)
    r = subprocess.run([os.path.join(CPP, "parse_test")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:]
    assert " 0 mismatches" in r.stdout


def test_device_formatter_vs_printf():
    """The GPU writer's %.17g formatter, compiled as host code, vs glibc snprintf (4.4M values)."""
    subprocess.run(["make", "-s", "-C", CPP, os.path.join(CPP, "format_test")], check=True)
    r = subprocess.run([os.path.join(CPP, "format_test")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:]
    assert " 0 mismatches" in r.stdout


@needs_ref
@pytest.mark.parametrize("cell,ok,val", [
    (b"1.5", True, 1.5), (b" 2.25\t", True, 2.25), (b'"-3"', True, -3.0), (b"+1", False, None),
    (b"1e400", False, None), (b"1e-400", False, None), (b"nan", False, None), (b"inf", False, None),
    (b"", False, None), (b'""', False, None), (b"1,5", False, None), (b"4.9e-324", True, 5e-324),
    (b"0x10", False, None), (b"-0", True, -0.0), (b"1.", True, 1.0), (b".5", True, 0.5)])
def test_reference_parse_double_semantics(cell, ok, val):
    """Pins the reference semantics the GPU parser follows (io.hpp:111-119)."""
    got_ok, got = oracle.ref_parse_double(cell)
    assert got_ok == ok
    if ok:
        assert np.float64(got).tobytes() == np.float64(val).tobytes()


def _cells(rng, n):
    """A mix of well-formed numbers in many formats and malformed cells."""
    u = rng.integers(0, 2 ** 63, n, dtype=np.uint64) | (rng.integers(0, 2, n, dtype=np.uint64) << np.uint64(63))
    d = u.view(np.float64)
    out = []
    fmts = ["%.17g", "%.16g", "%.6e", "%.25g", "%.3f", "%.20e"]
    bad = [b"abc", b"", b"+1.5", b"1e999", b"nan", b"-inf", b"1e-400", b"1..2", b"--1", b"1e", b" ", b'"', b"0x1p3"]
    for i in range(n):
        k = int(rng.integers(0, 12))
        v = d[i]
        if not np.isfinite(v):
            v = float(rng.standard_normal())
        if k < 6:
            s = (fmts[k] % v).encode()
        elif k == 6:
            s = bad[int(rng.integers(0, len(bad)))]
        elif k == 7:
            s = b'"' + (b"%.17g" % v) + b'"'
        elif k == 8:
            s = b" \t" + (b"%.9g" % (rng.standard_normal() * 10.0 ** rng.integers(-30, 30))) + b"\t "
        elif k == 9:  # long digit strings
            s = "".join(map(str, rng.integers(0, 10, int(rng.integers(18, 60))))).encode()
            s = s[:5] + b"." + s[5:] + b"e" + str(int(rng.integers(-330, 300))).encode()
        elif k == 10:  # subnormal / boundary magnitudes
            s = b"%.17g" % (float(rng.random()) * 10.0 ** float(rng.integers(-325, -300)))
        else:
            s = b"%d" % int(rng.integers(-(2 ** 62), 2 ** 62))
        out.append(s)
    return out


@needs_ref
@pytest.mark.gpu
def test_cells_match_reference_parser(engine):
    rng = np.random.default_rng(5)
    cells = _cells(rng, 60_000)
    # one cell per row in column 1 (x), a fixed good y in column 2
    text = b"id,x,y\n" + b"".join(b"%d,%s,0.5\n" % (i, c) for i, c in enumerate(cells))
    ref = [oracle.ref_parse_double(c) for c in cells]
    xy, n_bad, first_bad, kind = engine.parse_points_csv(text, 7, 1, 2, ",")
    want = np.array([v for ok, v in ref if ok], np.float64)
    assert n_bad == sum(1 for ok, _ in ref if not ok)
    assert len(xy) == len(want)
    assert xy[:, 0].tobytes() == want.tobytes()
    assert np.all(xy[:, 1] == 0.5)
    bad_rows = [i for i, (ok, _) in enumerate(ref) if not ok]
    if bad_rows:
        assert first_bad == text.index(b"\n%d," % bad_rows[0]) + 1 and kind == 3


def _rand_file(rng, path, delim, header, crlf, final_nl, rows):
    eol = b"\r\n" if crlf else b"\n"
    d = delim.encode()
    lines = []
    if header:
        lines.append(b"id" + d + b"lon" + d + b"lat")
    for r in range(rows):
        if rng.random() < 0.03:
            lines.append(b"")
        nc = int(rng.integers(1, 5)) if rng.random() < 0.2 else 3
        cells = [b"%d" % r]
        for c in range(1, nc):
            p = rng.random()
            if p < 0.05:
                cells.append(b"bad")
            elif p < 0.08:
                cells.append(b"")
            else:
                cells.append(b"%.17g" % (rng.uniform(-180, 180)))
        lines.append(d.join(cells))
    text = eol.join(lines) + (eol if final_nl else b"")
    with open(path, "wb") as f:
        f.write(text)
    return text


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("trial", range(8))
def test_files_match_reference_reader(engine, tmp_path, trial):
    """Lenient read: same points (bitwise) and skipped count as the reference;
    the first bad line is the reference's strict-mode error row."""
    rng = np.random.default_rng(100 + trial)
    delim = ",;\t,"[trial % 4]
    header = trial % 3 != 2
    path = tmp_path / f"p{trial}.csv"
    rows = [0, 1, 7, 500, 3000, 20000, 64, 100_000][trial]
    text = _rand_file(rng, path, delim, header, crlf=trial % 2 == 1, final_nl=trial % 4 != 3, rows=rows)
    ref = oracle.ref_read_points_csv(str(path), 1, 2, has_header=header, delim=delim, lenient=True)
    assert ref["kind"] == 0, ref["msg"]
    data_start = text.index(b"\n") + 1 if header else 0  # the header is the first line
    xy, n_bad, first_bad, kind = engine.parse_points_csv(text, data_start, 1, 2, delim)
    assert n_bad == ref["skipped"]
    assert xy.shape == ref["points"].shape
    assert xy.tobytes() == ref["points"].tobytes()
    strict = oracle.ref_read_points_csv(str(path), 1, 2, has_header=header, delim=delim, lenient=False)
    if strict["kind"] == 1:
        lines = text[data_start:first_bad].split(b"\n")[:-1]  # the lines before the bad one
        data_row = 1 + sum(1 for ln in lines if ln.rstrip(b"\r"))
        assert data_row == strict["row"]
        assert ("row has only" in strict["msg"]) == (kind == 2)
    else:
        assert first_bad is None


@pytest.mark.gpu
def test_round_trip_17_digits(engine):
    """%.17g of any finite double parses back to the same bits (2^20 rows)."""
    rng = np.random.default_rng(9)
    u = rng.integers(0, 2 ** 64, (1 << 20, 2), dtype=np.uint64)
    v = u.view(np.float64).copy()
    v[~np.isfinite(v)] = 1.0
    text = "\n".join("%.17g,%.17g" % (a, b) for a, b in v).encode()
    xy, n_bad, first_bad, _ = engine.parse_points_csv(text, 0, 0, 1, ",")
    assert n_bad == 0 and first_bad is None
    assert xy.tobytes() == v.tobytes()


@pytest.mark.gpu
def test_empty_and_degenerate_texts(engine):
    assert engine.parse_points_csv(b"", 0, 0, 1)[0].shape == (0, 2)
    xy, n_bad, fb, _ = engine.parse_points_csv(b"\n\r\n\n", 0, 0, 1)
    assert len(xy) == 0 and n_bad == 0 and fb is None
    xy, n_bad, fb, kind = engine.parse_points_csv(b"1,2\n3\n4,5", 0, 0, 1)
    assert xy.tolist() == [[1.0, 2.0], [4.0, 5.0]] and n_bad == 1 and fb == 4 and kind == 2
    xy, n_bad, fb, kind = engine.parse_points_csv(b"1,x\r\n", 0, 0, 1)
    assert len(xy) == 0 and n_bad == 1 and fb == 0 and kind == 4


def _tile_texts():
    """Inputs aimed at the reader's 8 KiB tiles: lines ending on / starting at
    tile boundaries, lines longer than a tile plus its spill, tiles of empty
    lines, tiles of minimal rows, a header longer than a tile."""
    T = 8192
    out = {}
    # '\n' exactly at byte T-1 and at T: rows of a fixed width that divides T
    out["width16"] = b"".join(b"%07d,%07d\n" % (i, -i) for i in range(5000))  # 16-byte rows
    out["width17"] = b"".join(b"%07d,%08d\n" % (i, i) for i in range(5000))
    out["min_rows"] = b"1,2\n" * 9000 + b"3,4"                                 # 2048 good rows per tile
    out["empty_tiles"] = b"5,6\n" + b"\n" * (3 * T) + b"7,8\r\n" + b"\r\n" * T + b"9,1"
    long_cell = b" " * (3 * T) + b"2.5"
    out["long_line"] = b"1,1\n" + long_cell + b"," + long_cell + b"\n2,2\n" + b"x" * (T - 2) + b"\n3,3"
    out["spill_edge"] = b"a" * (T - 3) + b"\n" + b"4," + b"0" * 600 + b"7\n5,5"
    out["no_newline"] = b"1.25,2.5"
    rng = np.random.default_rng(3)
    rows = []
    for i in range(20000):
        w = int(rng.integers(0, 40))
        rows.append(b" " * w + b"%.17g,%.17g" % tuple(rng.standard_normal(2)))
    out["ragged"] = b"\n".join(rows)
    return out


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("name", list(_tile_texts()))
def test_tile_boundaries_match_reference_reader(engine, tmp_path, name):
    text = _tile_texts()[name]
    path = tmp_path / f"{name}.csv"
    path.write_bytes(text)
    ref = oracle.ref_read_points_csv(str(path), 0, 1, has_header=False, lenient=True)
    assert ref["kind"] == 0, ref["msg"]
    xy, n_bad, first_bad, kind = engine.parse_points_csv(text, 0, 0, 1, ",")
    assert n_bad == ref["skipped"]
    assert xy.tobytes() == ref["points"].tobytes()


@needs_ref
@pytest.mark.gpu
def test_header_longer_than_a_tile(engine, tmp_path):
    head = b",".join(b"col%05d" % i for i in range(3000))  # ~27 KB header
    body = b"".join(b"%d,%d\n" % (i, 2 * i) for i in range(3000))
    text = b"\n\n" + head + b"\n" + body
    path = tmp_path / "wide.csv"
    path.write_bytes(text)
    ref = oracle.ref_read_points_csv(str(path), "col00000", "col00001", has_header=True, lenient=False)
    assert ref["kind"] == 0, ref["msg"]
    xy, n_bad, first_bad, _ = engine.parse_points_csv(text, len(text) - len(body), 0, 1, ",")
    assert n_bad == 0 and first_bad is None
    assert xy.tobytes() == ref["points"].tobytes()


@pytest.mark.gpu
def test_device_pointer_csv_api(engine):
    """pc_parse_points_csv_dev on an unaligned device pointer, capacity short."""
    import torch
    rows = b"".join(b"%d.5,%d\n" % (i, -i) for i in range(100_000))
    buf = torch.zeros(len(rows) + 3, dtype=torch.uint8)
    buf[3:] = torch.frombuffer(bytearray(rows), dtype=torch.uint8)
    d_text = buf.cuda()[3:]
    assert d_text.data_ptr() % 16 != 0
    d_out = torch.zeros((50_000, 2), dtype=torch.float64, device="cuda")
    d_res = torch.zeros(4, dtype=torch.int64, device="cuda")
    engine.parse_points_csv_dev(0, None, d_text, len(rows), 0, 0, 1, ",", d_out, 50_000, d_res)
    torch.cuda.synchronize()
    res = d_res.cpu().numpy().view(np.uint64)
    assert res[0] == 100_000 and res[1] == 0 and res[2] == np.uint64(2 ** 64 - 1)
    want = np.stack([np.arange(50_000) + 0.5, -np.arange(50_000.0)], 1)
    want[0, 1] = 0.0  # "0" parses to +0
    assert d_out.cpu().numpy().tobytes() == want.tobytes()


def _records(rng, n):
    u = rng.integers(0, 2 ** 64, (n, 2), dtype=np.uint64)
    xy = u.view(np.float64).copy()
    xy[~np.isfinite(xy)] = 0.25
    k = n // 4  # coordinates and the io_test magnitudes too
    xy[:k, 0] = rng.uniform(-180, 180, k)
    xy[:k, 1] = rng.uniform(-90, 90, k)
    xy[k:2 * k, 0] = rng.integers(0, 2 ** 63, k).astype(np.float64) / 1e3 * -1e-7
    if n >= 8:
        xy[2 * k:2 * k + 4] = [[0.0, -0.0], [5e-324, 1e17], [1e-5, 123456789012345678.0],
                               [-1e-300, 1.7976931348623157e308]]
    index = rng.integers(0, 2 ** 64, n, dtype=np.uint64)
    index[: n // 2] = np.arange(n // 2)
    verdict = rng.integers(0, 4, n).astype(np.uint8)
    return index, xy, verdict


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("n", [0, 1, 255, 256, 257, 100_000])
def test_results_text_matches_reference_writer(engine, tmp_path, n):
    """write_results_csv's bytes: the GPU writer vs the reference's own file."""
    rng = np.random.default_rng(n + 1)
    index, xy, verdict = _records(rng, n)
    from paper_2306_04316_b200.engine import make_records
    got = engine.format_results_csv(make_records(index, xy, verdict)).tobytes()
    path = tmp_path / "ref.csv"
    assert oracle.ref_write_results_csv(path, index, xy, verdict) == 0
    want = path.read_bytes()
    assert got == want
    names = [b"inside", b"outside", b"boundary", b"error"]
    py = b"index,x,y,verdict\n" + b"".join(b"%d,%s,%s,%s\n" % (int(i), (b"%.17g" % a), (b"%.17g" % b), names[v])
                                           for i, (a, b), v in zip(index, xy.tolist(), verdict))
    assert got == py


@pytest.mark.gpu
def test_results_round_trip_through_points_reader(engine):
    """17 significant digits round-trip: format on the GPU, parse on the GPU, same bits (2^20 rows)."""
    rng = np.random.default_rng(12)
    index, xy, verdict = _records(rng, 1 << 20)
    from paper_2306_04316_b200.engine import make_records
    text = engine.format_results_csv(make_records(index, xy, verdict)).tobytes()
    back, n_bad, fb, _ = engine.parse_points_csv(text, len(b"index,x,y,verdict\n"), 1, 2, ",")
    assert n_bad == 0 and fb is None
    assert back.tobytes() == xy.tobytes()
