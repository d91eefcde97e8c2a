// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// C-ABI shim around the *unmodified* reference CSV reader and number parser
// (proj/include/polycast/io.hpp: detail::parse_double :116-124,
// read_points_csv :148-225, read_polygon_geojson :280-309, write_results_csv
// :325-335), included from /root/reference at build time.
// Checker for the GPU CSV reader (paper_2306_04316_b200/csrc/pip_csv.cu) in
// tests/ and the CPU baseline of bench.py's csv workload; never the product.
#include <polycast/io.hpp>

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

using namespace polycast;

extern "C" {

// 1 if the reference parses [s, s+n) as a finite double (its value in *out)
int ref_parse_double(const char* s, uint64_t n, double* out) {
    double v = 0.0;
    const bool ok = detail::parse_double(std::string_view(s, n), v);
    if (ok) *out = v;
    return ok ? 1 : 0;
}

// read_points_csv; kind: 0 ok, 1 CsvParseError, 2 ColumnMissing, 3 FileNotFound,
// 4 IoError, 5 std::invalid_argument, 6 other.  x_name / y_name NULL: use the index.
int ref_read_points_csv(const char* path, const char* x_name, uint64_t x_idx, const char* y_name, uint64_t y_idx,
                        int has_header, char delim, int lenient, double* out_xy, uint64_t cap, uint64_t* n_points,
                        uint64_t* skipped, uint64_t* err_row, char* msg, uint64_t msg_cap) {
    PointsFileSpec spec;
    spec.path = path;
    if (x_name) spec.x_column = std::string(x_name);
    else spec.x_column = std::size_t(x_idx);
    if (y_name) spec.y_column = std::string(y_name);
    else spec.y_column = std::size_t(y_idx);
    spec.has_header = has_header != 0;
    spec.delimiter = delim;
    spec.lenient = lenient != 0;
    auto put = [&](const char* w) {
        if (msg && msg_cap) {
            std::strncpy(msg, w, msg_cap - 1);
            msg[msg_cap - 1] = 0;
        }
    };
    *n_points = *skipped = *err_row = 0;
    try {
        const CsvPoints r = read_points_csv(spec);
        *n_points = r.batch.size();
        *skipped = r.skipped_rows;
        for (std::size_t i = 0; i < r.batch.size() && i < cap; ++i) {
            out_xy[2 * i] = r.batch.points[i].x;
            out_xy[2 * i + 1] = r.batch.points[i].y;
        }
        return 0;
    } catch (const CsvParseError& e) {
        *err_row = e.row;
        put(e.what());
        return 1;
    } catch (const ColumnMissing& e) {
        put(e.what());
        return 2;
    } catch (const FileNotFound& e) {
        put(e.what());
        return 3;
    } catch (const IoError& e) {
        put(e.what());
        return 4;
    } catch (const std::invalid_argument& e) {
        put(e.what());
        return 5;
    } catch (const std::exception& e) {
        put(e.what());
        return 6;
    }
}

// write_results_csv of n records given as arrays; 0 ok, 4 IoError, 6 other
int ref_write_results_csv(const char* path, const uint64_t* index, const double* xy, const uint8_t* verdict,
                          uint64_t n) {
    try {
        std::vector<ResultRecord> recs(n);
        for (uint64_t i = 0; i < n; ++i)
            recs[i] = ResultRecord{index[i], xy[2 * i], xy[2 * i + 1], static_cast<Verdict>(verdict[i])};
        write_results_csv(recs, path);
        return 0;
    } catch (const IoError&) {
        return 4;
    } catch (const std::exception&) {
        return 6;
    }
}

// read_polygon_geojson; kind: 0 ok, 1 GeoJsonError, 2 UnsupportedGeometry, 3 RingTooShort,
// 4 FileNotFound, 5 IoError, 6 other std::exception.  Rings: ring_sizes[k] vertices each
// (closing vertex included), all vertices in out_xy.
int ref_read_polygon_geojson(const char* path, double* out_xy, uint64_t cap_verts, uint64_t* ring_sizes,
                             uint64_t cap_rings, uint64_t* n_rings, uint64_t* n_verts, char* msg, uint64_t msg_cap) {
    auto put = [&](const char* w) {
        if (msg && msg_cap) {
            std::strncpy(msg, w, msg_cap - 1);
            msg[msg_cap - 1] = 0;
        }
    };
    *n_rings = *n_verts = 0;
    try {
        const Polygon poly = read_polygon_geojson(path);
        uint64_t v = 0, r = 0;
        for (const Ring& ring : poly.rings()) {
            if (r < cap_rings) ring_sizes[r] = ring.size();
            ++r;
            for (const Point2& q : ring.vertices()) {
                if (v < cap_verts) {
                    out_xy[2 * v] = q.x;
                    out_xy[2 * v + 1] = q.y;
                }
                ++v;
            }
        }
        *n_rings = r;
        *n_verts = v;
        return 0;
    } catch (const RingTooShort& e) {
        put(e.what());
        return 3;
    } catch (const UnsupportedGeometry& e) {
        put(e.what());
        return 2;
    } catch (const GeoJsonError& e) {
        put(e.what());
        return 1;
    } catch (const FileNotFound& e) {
        put(e.what());
        return 4;
    } catch (const IoError& e) {
        put(e.what());
        return 5;
    } catch (const std::exception& e) {
        put(e.what());
        return 6;
    }
}

} // extern "C"
