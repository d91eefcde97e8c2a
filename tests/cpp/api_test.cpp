// Drop-in C++ API test: the reference's own known-answer tests and properties
// (proj/tests/unit/geometry_test.cpp, batch_test.cpp, acceptance.cpp checks
// 3, 7, 8, 9), re-expressed against include/polycast/*.hpp, which evaluates
// on the GPU through libpolycast_cuda.so.  Random cases are cross-checked
// against the unmodified reference (oracle/_ref/libpolycast_ref.so, loaded
// with dlopen) when it is present.  Exit code = number of failed checks.
#include <dlfcn.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <numbers>
#include <random>
#include <string>
#include <vector>

#include <polycast/io.hpp>
#include <polycast/polycast.hpp>

using namespace polycast;

static int g_checks = 0, g_fail = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        ++g_checks;                                                              \
        if (!(cond)) {                                                           \
            ++g_fail;                                                            \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                        \
    } while (0)
#define CHECK_THROWS(expr, Ex)                   \
    do {                                         \
        bool thrown_ = false;                    \
        try {                                    \
            (void)(expr);                        \
        } catch (const Ex&) {                    \
            thrown_ = true;                      \
        }                                        \
        CHECK(thrown_ && #expr " throws " #Ex);  \
    } while (0)

namespace {

double uni(std::mt19937_64& g, double lo, double hi) { return lo + (double)(g() >> 11) * 0x1.0p-53 * (hi - lo); }

Ring square() { return Ring({{0, 0}, {1, 0}, {1, 1}, {0, 1}, {0, 0}}); }

Ring star(std::mt19937_64& g, std::size_t n, Point2 c, double r0, double r1) {
    std::vector<Point2> v;
    const double step = 2.0 * std::numbers::pi / (double)n;
    for (std::size_t i = 0; i < n; ++i) {
        const double th = step * ((double)i + uni(g, 0.05, 0.95));
        const double r = uni(g, r0, r1);
        v.emplace_back(c.x + r * std::cos(th), c.y + r * std::sin(th));
    }
    v.push_back(v.front());
    return Ring(std::move(v));
}

Polygon random_polygon(std::mt19937_64& g, std::size_t n) {
    const Point2 c(uni(g, -10, 10), uni(g, -10, 10));
    const double R = uni(g, 0.5, 20.0);
    if (g() % 2 == 0) return Polygon(star(g, n, c, R, R));
    return Polygon(star(g, n, c, 0.35 * R, R));
}

// reference classify_batch through the oracle shim (optional)
using RefClassify = int (*)(const double*, uint64_t, const double*, const double*, const uint64_t*, uint32_t, int,
                            double, uint64_t, uint8_t*, uint64_t*);
RefClassify g_ref = nullptr;
using RefReadCsv = int (*)(const char*, const char*, uint64_t, const char*, uint64_t, int, char, int, double*, uint64_t,
                           uint64_t*, uint64_t*, uint64_t*, char*, uint64_t);
RefReadCsv g_ref_csv = nullptr;
using RefWriteResults = int (*)(const char*, const uint64_t*, const double*, const uint8_t*, uint64_t);
RefWriteResults g_ref_write = nullptr;
using RefRandomBatch = void (*)(const double*, uint64_t, uint64_t, double*);
RefRandomBatch g_ref_rb = nullptr;

std::string what_of(const std::function<void()>& f) {
    try {
        f();
    } catch (const std::exception& e) {
        return e.what();
    }
    return "";
}

// DegenerateEdge text names the first degenerate edge (geometry.hpp:219-220),
// through count_crossings_c2 and through contains (which propagates it)
void degenerate_messages() {
    const Ring sq = square();
    CHECK(what_of([&] { (void)count_crossings_c2({0.5, 0.0}, sq); }) ==
          "count_crossings_c2: horizontal edge 0 lies on the query ray");
    CHECK(what_of([&] { (void)count_crossings_c2({0.5, 1.0}, sq); }) ==
          "count_crossings_c2: horizontal edge 2 lies on the query ray");
    CHECK(what_of([&] { (void)contains({0.5, 0.0}, Polygon(sq), CrossingMode::C2); }) ==
          "count_crossings_c2: horizontal edge 0 lies on the query ray");
    // a hole's horizontal edge (index 1 of the hole ring), the outer ring clean at y = 5
    const Ring outer({{0, 0}, {10, 1}, {11, 11}, {-1, 10}, {0, 0}});
    const Ring hole({{2, 4}, {2, 5}, {4, 5}, {4, 4}, {2, 4}});
    const Polygon holed(outer, {hole});
    CHECK(what_of([&] { (void)contains({3.0, 5.0}, holed, CrossingMode::C2); }) ==
          "count_crossings_c2: horizontal edge 1 lies on the query ray");
}

// bench.hpp: random_batch identical to the reference's; a GPU scaling run
void bench_harness() {
    const BBox box(-2.0, -1.0, 3.0, 4.0);
    const PointBatch b = random_batch(box, 1000, 42);
    if (g_ref_rb) {
        std::vector<double> ref(2000);
        const double bx[4] = {-2.0, -1.0, 3.0, 4.0};
        g_ref_rb(bx, 1000, 42, ref.data());
        bool eq = true;
        for (std::size_t i = 0; i < 1000; ++i) eq = eq && b.points[i].x == ref[2 * i] && b.points[i].y == ref[2 * i + 1];
        CHECK(eq);
    }
    std::mt19937_64 g(5);
    const Polygon poly(star(g, 500, {0, 0}, 0.5, 1.0));
    const std::vector<std::size_t> sizes{10000, 20000, 40000, 80000};
    const auto samples = run_scaling_bench(poly, sizes, CrossingMode::C1, 4, 2, 9);
    CHECK(samples.size() == 4 && samples[0].algorithm == "c1_p" && samples[3].n_points == 80000);
    bool pos = true;
    for (const auto& s : samples) pos = pos && s.elapsed_seconds > 0.0;
    CHECK(pos);
    const GroupedFits fits = fit_per_algorithm(samples);
    CHECK(fits.fits.size() == 1 && fits.degenerate.empty());
    const ErrorReport rep = error_report(fits.fits, samples);
    CHECK(rep.size() == 4 && rep[0].relative_error.has_value());
    CHECK_THROWS(run_scaling_bench(poly, std::vector<std::size_t>{5, 5}, CrossingMode::C1, 1, 1, 0), std::invalid_argument);
    CHECK_THROWS(least_squares_fit(std::vector<TimingSample>{{5, "a", 1.0}}), DegenerateFit);
    CHECK_THROWS(error_report(fits.fits, std::vector<TimingSample>{{5, "zz", 1.0}}), MissingFit);
}

void kats() {
    const Ring sq = square();
    const Polygon sqp(sq);
    // geometry_test.cpp:34-50 — type validation
    CHECK_THROWS(Point2(std::nan(""), 0.0), std::invalid_argument);
    CHECK_THROWS(Point2(0.0, INFINITY), std::invalid_argument);
    CHECK_THROWS(Ring({{0, 0}, {1, 0}, {0, 0}}), std::invalid_argument);
    CHECK_THROWS(Ring({{0, 0}, {1, 0}, {1, 1}, {0, 1}}), std::invalid_argument);
    CHECK_THROWS(Ring({{0, 0}, {1, 0}, {1, 0}, {0, 1}, {0, 0}}), std::invalid_argument);
    // composed helpers (geometry_test.cpp:52-93)
    CHECK((signed_offsets(sq, 0.5) == std::vector<double>{-0.5, -0.5, 0.5, 0.5, -0.5}));
    CHECK((detect_sign_changes(std::vector<double>{0, 0, 1, 1, 0}) == std::vector<std::size_t>{0, 1, 3}));
    CHECK(crossing_x({0, 0}, {2, 4}, 2.0) == 1.0);
    CHECK_THROWS(crossing_x({3, 2}, {5, 2}, 2.0), DegenerateEdge);
    CHECK(edge_normal({0, 1}, {0, 0}).nx == 1.0);
    CHECK(edge_normal({0, 0}, {2, 4}).ny == -2.0);
    CHECK(segment_distance({5, 0}, {0, 0}, {1, 0}) == 4.0);
    // unit-square crossing counts (geometry_test.cpp:95-105) — on the GPU
    CHECK(count_crossings_c1({0.5, 0.5}, sq) == 1);
    CHECK(count_crossings_c1({-1.0, 0.5}, sq) == 2);
    CHECK(count_crossings_c1({2.0, 0.5}, sq) == 0);
    CHECK(count_crossings_c2({0.5, 0.5}, sq) == 1);
    CHECK(count_crossings_c2({-1.0, 0.5}, sq) == 2);
    CHECK_THROWS(count_crossings_c2({0.5, 0.0}, sq), DegenerateEdge);
    // verdicts (geometry_test.cpp:107-121; acceptance check 3)
    for (CrossingMode m : {CrossingMode::C1, CrossingMode::C2, CrossingMode::Robust}) {
        CHECK(contains({0.5, 0.5}, sqp, m) == Classification::Inside);
        CHECK(contains({5.0, 5.0}, sqp, m) == Classification::Outside);
    }
    CHECK(contains({1.0, 0.5}, sqp, CrossingMode::Robust) == Classification::Boundary);
    CHECK_THROWS(contains({0.5, 0.0}, sqp, CrossingMode::C2), DegenerateEdge);
    CHECK(contains({0.5, 0.0}, sqp, CrossingMode::Robust) == Classification::Boundary);
    // holes (geometry_test.cpp:123-137)
    const Polygon holed(square(), {Ring({{0.25, 0.25}, {0.75, 0.25}, {0.75, 0.75}, {0.25, 0.75}, {0.25, 0.25}})});
    CHECK(contains({0.5, 0.5}, holed, CrossingMode::Robust) == Classification::Outside);
    CHECK(contains({0.1, 0.5}, holed, CrossingMode::Robust) == Classification::Inside);
    CHECK(contains({0.5, 0.5}, holed, CrossingMode::C1) == Classification::Outside);
    // vertex on ray (geometry_test.cpp:145-160)
    const Ring diamond({{0, 0}, {2, 2}, {4, 0}, {2, -2}, {0, 0}});
    CHECK(count_crossings_c1({-3.0, 0.0}, diamond) == 4);
    CHECK(contains({-3.0, 0.0}, Polygon(diamond), CrossingMode::C1) == Classification::Outside);
    CHECK(contains({2.0, 0.0}, Polygon(diamond), CrossingMode::Robust) == Classification::Inside);
    // prefilter changes C1 verdicts on degenerate rays
    CHECK(contains({-1.0, 1.0}, sqp, CrossingMode::C1) == Classification::Inside);
    {
        PointBatch b;
        b.points = {{-1.0, 1.0}};
        CHECK(classify_batch(b, sqp, CrossingMode::C1).verdicts[0] == Verdict::Outside);
    }
    // batch probes (batch_test.cpp:65-85; acceptance check 9)
    {
        PointBatch b;
        b.points = {{0.5, 0.5}, {1.5, 0.5}, {0.5, -0.5}, {-0.5, 0.5}};
        const BatchResult r = classify_batch(b, sqp, CrossingMode::Robust);
        CHECK((r.verdicts == std::vector<Verdict>{Verdict::Inside, Verdict::Outside, Verdict::Outside, Verdict::Outside}));
        CHECK(r.stats.inside == 1 && r.stats.outside == 3 && r.stats.total() == 4);
    }
    {
        PointBatch b;
        b.points = {{0.5, 0.0}, {0.5, 0.5}, {-2.0, 0.5}};
        const BatchResult r = classify_batch(b, sqp, CrossingMode::C2);
        CHECK(r.verdicts[0] == Verdict::Error && r.verdicts[1] == Verdict::Inside && r.verdicts[2] == Verdict::Outside);
        CHECK(r.stats.error == 1 && r.stats.total() == 3);
    }
    {
        PointBatch b;
        b.points = {{0.5, 0.0}, {-5.0, 0.0}, {0.5, 0.5}};
        const BatchResult r = classify_batch(b, sqp, CrossingMode::C2, 2);
        CHECK(r.verdicts[0] == Verdict::Error && r.verdicts[1] == Verdict::Outside && r.verdicts[2] == Verdict::Inside);
    }
    CHECK(classify_batch(PointBatch{}, sqp, CrossingMode::Robust).verdicts.empty());
    CHECK(bbox_of(Polygon(Ring({{-2, 3}, {5, 3}, {5, 7}, {-2, 7}, {-2, 3}}))) == BBox(-2, 3, 5, 7));
}

void randomized() {
    std::mt19937_64 g(42);
    int compared = 0;
    for (int trial = 0; trial < 30; ++trial) {
        const Polygon poly = trial % 5 == 4 ? Polygon(star(g, 40, {0, 0}, 5, 9), {star(g, 12, {0, 0}, 1, 3)})
                                            : random_polygon(g, 5 + g() % 300);
        const BBox box = bbox_of(poly).inflated(0.3);
        PointBatch b;
        for (int i = 0; i < 20000; ++i) b.points.emplace_back(uni(g, box.min_x, box.max_x), uni(g, box.min_y, box.max_y));
        for (CrossingMode m : {CrossingMode::C1, CrossingMode::C2, CrossingMode::Robust}) {
            const BatchResult r = classify_batch(b, poly, m);
            CHECK(r.stats.total() == b.size());
            // identical for any "workers" value (batch_test.cpp:87-105)
            CHECK(classify_batch(b, poly, m, 3) == r);
            if (g_ref) {
                std::vector<double> x, y;
                std::vector<uint64_t> off{0};
                for (const Ring& ring : poly.rings()) {
                    for (const Point2& v : ring.vertices()) { x.push_back(v.x); y.push_back(v.y); }
                    off.push_back(x.size());
                }
                std::vector<uint8_t> want(b.size());
                uint64_t st[4];
                g_ref(&b.points[0].x, b.size(), x.data(), y.data(), off.data(), (uint32_t)(off.size() - 1), (int)m,
                      kDefaultBoundaryTol, 0, want.data(), st);
                bool same = std::memcmp(want.data(), r.verdicts.data(), b.size()) == 0;
                CHECK(same && "classify_batch bit-identical to the reference");
                CHECK(st[0] == r.stats.inside && st[1] == r.stats.outside && st[2] == r.stats.boundary &&
                      st[3] == r.stats.error);
                ++compared;
            }
        }
    }
    // many-polygon extension == per-polygon classify_batch
    std::vector<Polygon> polys;
    std::vector<PointBatch> batches;
    for (int i = 0; i < 50; ++i) {
        polys.push_back(random_polygon(g, 4 + g() % 12));
        const BBox box = bbox_of(polys.back()).inflated(0.5);
        PointBatch b;
        const int np = (int)(g() % 70);
        for (int k = 0; k < np; ++k) b.points.emplace_back(uni(g, box.min_x, box.max_x), uni(g, box.min_y, box.max_y));
        batches.push_back(std::move(b));
    }
    for (CrossingMode m : {CrossingMode::C1, CrossingMode::C2, CrossingMode::Robust}) {
        const BatchResult many = classify_batch_many(batches, polys, m);
        std::size_t off = 0;
        bool ok = true;
        for (std::size_t i = 0; i < polys.size(); ++i) {
            const BatchResult one = classify_batch(batches[i], polys[i], m);
            for (std::size_t k = 0; k < one.verdicts.size(); ++k) ok = ok && one.verdicts[k] == many.verdicts[off + k];
            off += one.verdicts.size();
        }
        CHECK(ok && off == many.verdicts.size());
    }
    std::printf("randomized: %d polygon x mode cases compared against the reference\n", compared);
}

// batch_test.cpp:37-63 (prefilter_bbox, scatter_verdicts) and the bbox
// property of :107-124, now GPU compaction / scatter behind the same API
void prefilter_scatter() {
    PointBatch batch;
    batch.points = {{0.5, 0.5}, {2, 2}};
    const PrefilterResult pre = prefilter_bbox(batch, BBox(0, 0, 1, 1));
    CHECK(pre.inside_box.size() == 1);
    CHECK(pre.inside_box.size() == 1 && pre.inside_box.points[0] == Point2(0.5, 0.5));
    CHECK(pre.original_indices == std::vector<std::size_t>{0});
    CHECK(pre.outside_count == 1);
    PointBatch edge_case;
    edge_case.points = {{1.0, 0.5}};
    CHECK(prefilter_bbox(edge_case, BBox(0, 0, 1, 1)).inside_box.size() == 1); // closed interval

    PointBatch b2;
    b2.points = {{0.5, 0.5}, {2, 2}, {0.1, 0.1}, {-3, 0}};
    const PrefilterResult p2 = prefilter_bbox(b2, BBox(0, 0, 1, 1));
    CHECK(p2.inside_box.size() == 2);
    const std::vector<Verdict> sc = scatter_verdicts(p2, {Verdict::Inside, Verdict::Boundary});
    CHECK((sc == std::vector<Verdict>{Verdict::Inside, Verdict::Outside, Verdict::Boundary, Verdict::Outside}));
    CHECK_THROWS(scatter_verdicts(p2, {Verdict::Inside}), std::invalid_argument);
    CHECK(prefilter_bbox(PointBatch{}, BBox(0, 0, 1, 1)).inside_box.empty());

    // order, indices and counts vs the reference loop on random batches (1e5 points)
    std::mt19937_64 g(17);
    for (int trial = 0; trial < 5; ++trial) {
        const Polygon poly = random_polygon(g, 5 + g() % 50);
        const BBox box = bbox_of(poly);
        const BBox big = box.inflated(1.0);
        PointBatch pb;
        for (int k = 0; k < 100000; ++k) pb.points.emplace_back(uni(g, big.min_x, big.max_x), uni(g, big.min_y, big.max_y));
        pb.points.emplace_back(box.min_x, box.max_y); // corners are inside (closed)
        const PrefilterResult pr = prefilter_bbox(pb, box);
        std::vector<std::size_t> want;
        for (std::size_t i = 0; i < pb.size(); ++i)
            if (box.contains(pb.points[i])) want.push_back(i);
        bool ok = pr.original_indices == want && pr.outside_count + want.size() == pb.size();
        for (std::size_t k = 0; ok && k < want.size(); ++k) ok = pr.inside_box.points[k] == pb.points[want[k]];
        CHECK(ok);
        const BatchResult in = classify_batch(pr.inside_box, poly, CrossingMode::C1);
        const std::vector<Verdict> full = scatter_verdicts(pr, in.verdicts);
        CHECK(full == classify_batch(pb, poly, CrossingMode::C1).verdicts); // the CLI pipeline == classify_batch
    }
}

// read_points_csv (io.hpp:148-225) against the unmodified reference on
// generated files: number formats, quotes, spaces, CRLF, empty lines, BOM +
// named columns, delimiters, short rows, bad cells; strict and lenient.
std::string rand_cell(std::mt19937_64& g) {
    char b[64];
    const double v = uni(g, -1e3, 1e3) * std::pow(10.0, (double)((int)(g() % 40) - 20));
    switch (g() % 16) {
    case 0: return "abc";
    case 1: return "";
    case 2: return " " + std::to_string(v) + "\t";
    case 3: std::snprintf(b, sizeof b, "\"%.17g\"", v); return b;
    case 4: return "+1.5";
    case 5: return "1e999";
    case 6: return "nan";
    case 7: std::snprintf(b, sizeof b, "%.3e", v); return b;
    case 8: return "1e-400";
    case 9: return "-0";
    default: std::snprintf(b, sizeof b, "%.17g", v); return b;
    }
}

void csv_vs_reference() {
    if (!g_ref_csv) {
        std::printf("note: reference CSV reader not available; skipped\n");
        return;
    }
    std::mt19937_64 g(23);
    int compared = 0;
    for (int trial = 0; trial < 60; ++trial) {
        const char delim = "x,;\t"[1 + trial % 3];
        const bool header = trial % 4 != 3, lenient = trial % 2, crlf = trial % 5 == 0, bom = trial % 7 == 1;
        std::string text;
        if (header) text += std::string(bom ? "\xEF\xBB\xBF" : "") + "id" + delim + "lon" + delim + "\"lat\"" + (crlf ? "\r\n" : "\n");
        const int rows = 1 + (int)(g() % 300);
        const bool clean = trial % 3 == 0; // clean files: no bad rows (strict mode succeeds)
        for (int r = 0; r < rows; ++r) {
            if (g() % 23 == 0) text += crlf ? "\r\n" : "\n"; // empty line
            char b[64];
            std::snprintf(b, sizeof b, "%d", r);
            std::string row = b;
            const int ncells = clean ? 3 : (int)(g() % 4) + 1;
            for (int c = 1; c < ncells; ++c) {
                std::string cell;
                if (clean) {
                    std::snprintf(b, sizeof b, "%.17g", uni(g, -180, 180));
                    cell = b;
                } else {
                    cell = rand_cell(g);
                }
                row += delim + cell;
            }
            text += row + (crlf ? "\r\n" : "\n");
        }
        if (trial % 6 == 2 && !text.empty()) text.pop_back(); // no final newline
        const std::string path = "/tmp/pc_csv_test_" + std::to_string(trial) + ".csv";
        FILE* f = std::fopen(path.c_str(), "wb");
        std::fwrite(text.data(), 1, text.size(), f);
        std::fclose(f);
        PointsFileSpec spec;
        spec.path = path;
        spec.delimiter = delim;
        spec.has_header = header;
        spec.lenient = lenient;
        const bool named = header && trial % 2 == 0;
        if (named) {
            spec.x_column = std::string("lon");
            spec.y_column = std::string("lat");
        } else {
            spec.x_column = std::size_t(1);
            spec.y_column = std::size_t(2);
        }
        std::vector<double> ref(2 * (rows + 4));
        uint64_t rn = 0, rs = 0, rrow = 0;
        char msg[512] = {0};
        const int rk = g_ref_csv(path.c_str(), named ? "lon" : nullptr, 1, named ? "lat" : nullptr, 2, header, delim,
                                 lenient, ref.data(), rows + 4, &rn, &rs, &rrow, msg, sizeof msg);
        int k = 0;
        std::string what;
        CsvPoints got;
        try {
            got = read_points_csv(spec);
        } catch (const CsvParseError& e) {
            k = 1;
            what = e.what();
            CHECK(e.row == rrow);
        } catch (const ColumnMissing& e) {
            k = 2;
            what = e.what();
        } catch (const IoError& e) {
            k = 4;
            what = e.what();
        }
        CHECK(k == rk);
        if (k != rk || (k && what != msg)) std::fprintf(stderr, "trial %d: kind %d vs %d, '%s' vs '%s'\n", trial, k, rk, what.c_str(), msg);
        if (k == 0 && rk == 0) {
            bool ok = got.batch.size() == rn && got.skipped_rows == rs;
            for (std::size_t i = 0; ok && i < rn; ++i)
                ok = std::memcmp(&got.batch.points[i].x, &ref[2 * i], 8) == 0 &&
                     std::memcmp(&got.batch.points[i].y, &ref[2 * i + 1], 8) == 0;
            CHECK(ok);
        } else {
            CHECK(what == msg);
        }
        ++compared;
        std::remove(path.c_str());
    }
    // the reference's own error cases
    CHECK_THROWS(read_points_csv(PointsFileSpec{"/nonexistent/file.csv"}), FileNotFound);
    PointsFileSpec same;
    same.path = "/nonexistent/file.csv";
    same.y_column = std::size_t(0);
    CHECK_THROWS(read_points_csv(same), std::invalid_argument);
    std::printf("csv: %d files compared against the reference reader\n", compared);
}

std::string slurp(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    return std::string((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
}

// io_test.cpp:197-225 (results round-trip bitwise) re-expressed, plus the
// written bytes against the reference's writer and awkward doubles
void results_csv() {
    std::mt19937_64 rng(99);
    std::vector<ResultRecord> records;
    for (std::size_t i = 0; i < 10000; ++i) {
        const double x = (static_cast<double>(rng()) / 1e3) * (rng() % 2 ? 1 : -1e-7);
        const double y = static_cast<double>(rng() >> 11) * 0x1.0p-53;
        records.push_back({i, x, y, static_cast<Verdict>(rng() % 4)});
    }
    // awkward values: signed zeros, subnormals, extremes, powers of ten, huge indices
    const double odd[] = {0.0, -0.0, 5e-324, -2.2250738585072014e-308, 1.7976931348623157e308, 1e-5, 1e16, 1e17,
                          0.1, 123456789012345678.0, -1e-300, 9.999999999999999e22};
    for (double v : odd) records.push_back({~std::size_t(0) - records.size(), v, -v, Verdict::Boundary});
    for (int k = 0; k < 20000; ++k) { // random bit patterns
        uint64_t a = rng(), b = rng();
        double x, y;
        std::memcpy(&x, &a, 8);
        std::memcpy(&y, &b, 8);
        if (!std::isfinite(x)) x = 1.5;
        if (!std::isfinite(y)) y = -2.5;
        records.push_back({rng(), x, y, static_cast<Verdict>(rng() % 4)});
    }
    const std::string out = "/tmp/pc_results_test.csv", ref = "/tmp/pc_results_ref.csv";
    write_results_csv(records, out);
    const std::vector<ResultRecord> back = read_results_csv(out);
    CHECK(back.size() == records.size());
    bool same = back.size() == records.size();
    for (std::size_t i = 0; same && i < records.size(); ++i)
        same = back[i].index == records[i].index && std::memcmp(&back[i].x, &records[i].x, 8) == 0 &&
               std::memcmp(&back[i].y, &records[i].y, 8) == 0 && back[i].verdict == records[i].verdict;
    CHECK(same);
    // coordinates also survive re-reading through the points reader
    PointsFileSpec spec;
    spec.path = out;
    spec.x_column = std::string("x");
    spec.y_column = std::string("y");
    const CsvPoints pts = read_points_csv(spec);
    CHECK(pts.batch.size() == records.size());
    bool same_pts = pts.batch.size() == records.size();
    for (std::size_t i = 0; same_pts && i < records.size(); ++i)
        same_pts = pts.batch.points[i].x == records[i].x && pts.batch.points[i].y == records[i].y;
    CHECK(same_pts);
    // byte-identical to the reference's writer
    if (g_ref_write) {
        std::vector<uint64_t> idx(records.size());
        std::vector<double> xy(2 * records.size());
        std::vector<uint8_t> v(records.size());
        for (std::size_t i = 0; i < records.size(); ++i) {
            idx[i] = records[i].index;
            xy[2 * i] = records[i].x;
            xy[2 * i + 1] = records[i].y;
            v[i] = static_cast<uint8_t>(records[i].verdict);
        }
        CHECK(g_ref_write(ref.c_str(), idx.data(), xy.data(), v.data(), records.size()) == 0);
        const std::string a = slurp(out), b = slurp(ref);
        CHECK(a == b);
        if (a != b) {
            std::size_t k = 0;
            while (k < a.size() && k < b.size() && a[k] == b[k]) ++k;
            std::fprintf(stderr, "results differ at byte %zu: '%.60s' vs '%.60s'\n", k, a.c_str() + (k > 20 ? k - 20 : 0),
                         b.c_str() + (k > 20 ? k - 20 : 0));
        }
        std::printf("results: %zu records, %zu bytes, identical to the reference writer: %s\n", records.size(),
                    a.size(), a == b ? "yes" : "NO");
        std::remove(ref.c_str());
    }
    // empty batch: header only (io_test.cpp:184-194)
    write_results_csv(std::vector<ResultRecord>{}, out);
    CHECK(slurp(out) == "index,x,y,verdict\n");
    CHECK(read_results_csv(out).empty());
    // reader errors
    {
        std::FILE* f = std::fopen(out.c_str(), "wb");
        std::fputs("index,x,y,verdict\n0,1,2,inside\n1,1,2,sideways\n", f);
        std::fclose(f);
        CHECK_THROWS(read_results_csv(out), CsvParseError);
    }
    CHECK_THROWS(read_results_csv("/nonexistent/results.csv"), FileNotFound);
    CHECK_THROWS(write_results_csv(records, "/nonexistent/dir/results.csv"), IoError);
    std::remove(out.c_str());
}

// read_polygons_geojson (extension) feeding classify_batch_many: a
// FeatureCollection of random polygons with holes, written with %.17g, reads
// back bit-exactly and classifies like per-polygon classify_batch
void geojson_to_csr() {
    std::mt19937_64 g(31);
    std::vector<Polygon> polys;
    std::string doc = R"({"type":"FeatureCollection","features":[)";
    char b[64];
    auto ring_json = [&](const Ring& r) {
        std::string s = "[";
        for (std::size_t i = 0; i < r.size(); ++i) {
            std::snprintf(b, sizeof b, "%s[%.17g,%.17g]", i ? "," : "", r[i].x, r[i].y);
            s += b;
        }
        return s + "]";
    };
    for (int k = 0; k < 60; ++k) {
        const Polygon base = random_polygon(g, 5 + g() % 60);
        std::vector<Ring> holes;
        if (k % 3 == 0) { // a small square hole around the polygon's first vertex's midpoint to its centroid
            const Point2 v = base.outer()[0];
            const double h = 1e-3;
            holes.emplace_back(std::vector<Point2>{Point2(v.x * 0.5 - h, v.y * 0.5 - h), Point2(v.x * 0.5 + h, v.y * 0.5 - h),
                                                   Point2(v.x * 0.5 + h, v.y * 0.5 + h), Point2(v.x * 0.5 - h, v.y * 0.5 + h),
                                                   Point2(v.x * 0.5 - h, v.y * 0.5 - h)});
        }
        Ring outer(std::vector<Point2>(base.outer().vertices().begin(), base.outer().vertices().end()));
        const Polygon poly(outer, holes);
        std::string coords = ring_json(poly.outer());
        for (const Ring& hr : poly.holes()) coords += "," + ring_json(hr);
        doc += std::string(k ? "," : "") + R"({"type":"Feature","properties":{"id":)" + std::to_string(k) +
               R"(},"geometry":{"type":"Polygon","coordinates":[)" + coords + "]}}";
        polys.push_back(poly);
    }
    doc += "]}";
    const std::string path = "/tmp/pc_geojson_csr.json";
    FILE* f = std::fopen(path.c_str(), "wb");
    std::fwrite(doc.data(), 1, doc.size(), f);
    std::fclose(f);
    const std::vector<Polygon> back = read_polygons_geojson(path);
    CHECK(back.size() == polys.size());
    bool same = back.size() == polys.size();
    for (std::size_t i = 0; same && i < polys.size(); ++i) {
        same = back[i].rings().size() == polys[i].rings().size();
        for (std::size_t r = 0; same && r < polys[i].rings().size(); ++r) {
            const Ring &a = back[i].rings()[r], &c = polys[i].rings()[r];
            same = a.size() == c.size() &&
                   std::memcmp(a.vertices().data(), c.vertices().data(), a.size() * sizeof(Point2)) == 0;
        }
    }
    CHECK(same);
    CHECK(read_polygon_geojson(path).outer().size() == polys[0].outer().size()); // the first feature
    std::vector<PointBatch> batches(polys.size());
    for (std::size_t i = 0; i < polys.size(); ++i) {
        const BBox bb = bbox_of(polys[i]);
        for (int j = 0; j < 300; ++j)
            batches[i].points.emplace_back(uni(g, bb.min_x - 1, bb.max_x + 1), uni(g, bb.min_y - 1, bb.max_y + 1));
    }
    for (CrossingMode m : {CrossingMode::C1, CrossingMode::C2, CrossingMode::Robust}) {
        const BatchResult all = classify_batch_many(batches, polys, m);
        std::size_t at = 0;
        bool eq = true;
        for (std::size_t i = 0; i < polys.size(); ++i) {
            const BatchResult one = classify_batch(batches[i], polys[i], m);
            for (std::size_t j = 0; j < one.verdicts.size(); ++j) eq = eq && all.verdicts[at + j] == one.verdicts[j];
            at += one.verdicts.size();
        }
        CHECK(eq);
    }
    std::remove(path.c_str());
    std::printf("geojson: %zu polygons read back bit-exactly and classified through the CSR path\n", back.size());
}

} // namespace

int main(int argc, char** argv) {
    const char* ref_path = argc > 1 ? argv[1] : "oracle/_ref/libpolycast_ref.so";
    if (void* h = dlopen(ref_path, RTLD_NOW)) {
        g_ref = reinterpret_cast<RefClassify>(dlsym(h, "ref_classify"));
        g_ref_csv = reinterpret_cast<RefReadCsv>(dlsym(h, "ref_read_points_csv"));
        g_ref_write = reinterpret_cast<RefWriteResults>(dlsym(h, "ref_write_results_csv"));
        g_ref_rb = reinterpret_cast<RefRandomBatch>(dlsym(h, "ref_random_batch"));
    }
    else std::printf("note: reference shim not found at %s; reference cross-check skipped\n", ref_path);
    try {
        kats();
        degenerate_messages();
        bench_harness();
        randomized();
        prefilter_scatter();
        csv_vs_reference();
        results_csv();
        geojson_to_csr();
    } catch (const std::exception& e) {
        std::fprintf(stderr, "FAIL: uncaught exception: %s\n", e.what());
        return 100;
    }
    std::printf("api_test: %d checks, %d failed\n", g_checks, g_fail);
    return g_fail;
}
