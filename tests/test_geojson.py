"""GeoJSON ingest: include/polycast/io.hpp
read_polygon_geojson over include/polycast/json.hpp against the unmodified
reference (oracle/_ref: read_polygon_geojson over nlohmann::json,
proj/include/polycast/io.hpp:229-309).  Host code, no GPU: the reference's own
io_test cases (io_test.cpp:123-176), semantic errors (same exception type and
message), every JSON number form (same doubles, bit for bit), syntax errors and
accepted syntax variants (same exception type), 400 random documents.  The GPU
leg (read_polygons_geojson -> classify_batch_many) is in tests/cpp/api_test.cpp."""
import os
import subprocess

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_geojson_matches_reference():
    subprocess.run(["make", "-s", "-C", CPP, os.path.join(CPP, "geojson_test")], check=True)
    r = subprocess.run([os.path.join(CPP, "geojson_test"), oracle.REF_LIB], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout[-4000:]
    assert " 0 failures" in r.stdout
