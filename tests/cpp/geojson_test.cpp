// GeoJSON ingest (include/polycast/io.hpp read_polygon_geojson over
// include/polycast/json.hpp) against the unmodified reference
// (oracle/_ref: read_polygon_geojson over nlohmann::json, io.hpp:229-309).
// Host-only: no GPU needed.  Same exception kind for every document; same
// message for the semantic errors (the text of a JSON syntax error comes from
// the JSON library and differs); identical vertex bits on success.  The one
// documented divergence: a number overflowing to infinity is a GeoJsonError
// here, nlohmann's out_of_range (kind 6) in the reference.
// usage: geojson_test <path to libpolycast_ref.so>; exit code = failures (capped)
#include <dlfcn.h>

#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include <polycast/io.hpp>

using namespace polycast;

using RefGeo = int (*)(const char*, double*, uint64_t, uint64_t*, uint64_t, uint64_t*, uint64_t*, char*, uint64_t);
static RefGeo g_ref = nullptr;
static int fails = 0, total = 0, compared_ok = 0;

static int ours(const std::string& path, std::vector<double>& xy, std::vector<uint64_t>& sizes, std::string& msg) {
    try {
        const Polygon p = read_polygon_geojson(path);
        for (const Ring& r : p.rings()) {
            sizes.push_back(r.size());
            for (const Point2& q : r.vertices()) {
                xy.push_back(q.x);
                xy.push_back(q.y);
            }
        }
        return 0;
    } catch (const RingTooShort& e) {
        msg = e.what();
        return 3;
    } catch (const UnsupportedGeometry& e) {
        msg = e.what();
        return 2;
    } catch (const GeoJsonError& e) {
        msg = e.what();
        return 1;
    } catch (const FileNotFound& e) {
        msg = e.what();
        return 4;
    } catch (const IoError& e) {
        msg = e.what();
        return 5;
    } catch (const std::exception& e) {
        msg = e.what();
        return 6;
    }
}

static void check(const std::string& name, const std::string& doc, bool overflow = false) {
    const std::string path = "/tmp/pc_geojson_test.json";
    FILE* f = std::fopen(path.c_str(), "wb");
    std::fwrite(doc.data(), 1, doc.size(), f);
    std::fclose(f);
    std::vector<double> xy, rxy(2 * 4096);
    std::vector<uint64_t> sizes, rsizes(512);
    std::string msg;
    char rmsg[1024] = {0};
    uint64_t nr = 0, nv = 0;
    const int k = ours(path, xy, sizes, msg);
    const int rk = g_ref(path.c_str(), rxy.data(), 4096, rsizes.data(), 512, &nr, &nv, rmsg, sizeof rmsg);
    ++total;
    bool ok = k == rk || (overflow && k == 1 && rk == 6);
    const bool syntax = std::strstr(rmsg, "[json.exception") != nullptr;
    if (ok && k != 0 && !syntax && !overflow) ok = msg == rmsg;
    if (ok && k == 0) {
        ok = nr == sizes.size() && nv * 2 == xy.size() && std::memcmp(xy.data(), rxy.data(), xy.size() * 8) == 0;
        for (std::size_t i = 0; ok && i < nr; ++i) ok = rsizes[i] == sizes[i];
        if (ok) ++compared_ok;
    }
    if (!ok) {
        ++fails;
        if (fails <= 20)
            std::printf("MISMATCH %s: ours %d '%s' / ref %d '%s'\n  doc: %.200s\n", name.c_str(), k, msg.c_str(), rk,
                        rmsg, doc.c_str());
    }
}

static std::string num(std::mt19937_64& g, double v) {
    char b[64];
    switch (g() % 6) {
    case 0: std::snprintf(b, sizeof b, "%.17g", v); break;
    case 1: std::snprintf(b, sizeof b, "%.6e", v); break;
    case 2: std::snprintf(b, sizeof b, "%.3f", v); break;
    case 3: std::snprintf(b, sizeof b, "%.0f", v); break; // integer tokens (incl. "-0")
    case 4: std::snprintf(b, sizeof b, "%.20E", v); break;
    default: std::snprintf(b, sizeof b, "%.25g", v); break;
    }
    return b;
}

static std::string ring(std::mt19937_64& g, int n, double cx, double cy, double r, bool close, bool ws) {
    std::string s = "[";
    std::vector<std::pair<std::string, std::string>> pts;
    for (int i = 0; i < n; ++i) {
        const double a = 2 * 3.141592653589793 * i / n;
        const double rr = r * (0.6 + 0.4 * std::uniform_real_distribution<double>(0, 1)(g));
        pts.emplace_back(num(g, cx + rr * std::cos(a)), num(g, cy + rr * std::sin(a)));
    }
    if (close) pts.push_back(pts[0]);
    for (std::size_t i = 0; i < pts.size(); ++i) {
        if (i) s += ws ? " ,\n " : ",";
        s += "[" + pts[i].first + (ws ? " , " : ",") + pts[i].second + (g() % 5 == 0 ? ",7.5" : "") + "]";
    }
    return s + "]";
}

int main(int argc, char** argv) {
    const char* ref_path = argc > 1 ? argv[1] : "oracle/_ref/libpolycast_ref.so";
    void* h = dlopen(ref_path, RTLD_NOW);
    if (!h || !(g_ref = reinterpret_cast<RefGeo>(dlsym(h, "ref_read_polygon_geojson")))) {
        std::printf("reference shim not available at %s\n", ref_path);
        return 1;
    }
    const std::string sq = R"({"type":"Polygon","coordinates":[[[0,0],[1,0],[1,1],[0,1],[0,0]]]})";
    // the reference's own cases (io_test.cpp:123-176)
    check("square", sq);
    check("open", R"({"type":"Polygon","coordinates":[[[0,0],[1,0],[1,1],[0,1]]]})");
    check("feature", R"({"type":"Feature","properties":{},"geometry":)" + sq + "}");
    check("collection", R"({"type":"FeatureCollection","features":[{"type":"Feature","geometry":)" + sq + "}]}");
    check("hole", R"({"type":"Polygon","coordinates":[[[0,0],[1,0],[1,1],[0,1],[0,0]],
            [[0.25,0.25],[0.75,0.25],[0.75,0.75],[0.25,0.75],[0.25,0.25]]]})");
    check("point", R"({"type":"Point","coordinates":[0,0]})");
    check("multi", R"({"type":"MultiPolygon","coordinates":[[[[0,0],[1,0],[1,1],[0,0]]]]})");
    check("short", R"({"type":"Polygon","coordinates":[[[0,0],[1,0]]]})");
    check("junk", "{not json");
    // semantic errors
    const char* sem[] = {
        R"([1,2])", R"({"coordinates":[]})", R"({"type":5})", R"({"type":"Polygon"})",
        R"({"type":"Polygon","coordinates":{}})", R"({"type":"Polygon","coordinates":[]})",
        R"({"type":"Polygon","coordinates":[5]})", R"({"type":"Polygon","coordinates":[[]]})",
        R"({"type":"Polygon","coordinates":[[[0,0],[1,0],[0,0]]]})",
        R"({"type":"Polygon","coordinates":[[[0,0],[1,0],[1,0],[0,1]]]})",
        R"({"type":"Polygon","coordinates":[[[0],[1,0],[1,1]]]})",
        R"({"type":"Polygon","coordinates":[[[0,"1"],[1,0],[1,1]]]})",
        R"({"type":"Polygon","coordinates":[[[0,0],[1,0],[1,1]],[[0,0]]]})",
        R"({"type":"Polygon","coordinates":[[[0,0],[1,0],[1,1]],7]})",
        R"({"type":"Polygon","coordinates":[[[0,0],[1,0],[1,1]],[[0,0],[1,0],[1,0],[0,0]]]})",
        R"({"type":"FeatureCollection"})", R"({"type":"FeatureCollection","features":[]})",
        R"({"type":"FeatureCollection","features":{}})", R"({"type":"FeatureCollection","features":[5]})",
        R"({"type":"FeatureCollection","features":[{"type":"Feature"}]})",
        R"({"type":"FeatureCollection","features":[{"geometry":null}]})", R"({"type":"Feature"})",
        R"({"type":"Feature","geometry":null})", R"({"type":"Feature","geometry":{"type":"LineString"}})",
        R"({"type":"GeometryCollection","geometries":[]})", R"({"type":"Point","type":"Polygon","coordinates":[[[0,0],[1,0],[1,1]]]})",
        R"({"type":"Polygon","coordinates":[[[0,0],[1,0],[1,1]]],"coordinates":[[[5,5],[6,5],[6,6]]]})",
        R"({"type":"Polygon","coordinates":[[[true,0],[1,0],[1,1]]]})",
        R"({"type":"Polygon","coordinates":[[[null,0],[1,0],[1,1]]]})",
    };
    for (const char* d : sem) check("semantic", d);
    // numbers: every JSON number form, edge magnitudes
    const char* nums[] = {"0", "-0", "0.0", "-0.0", "1", "-1", "1e5", "1E+5", "1e-5", "-1.5e-310", "4.9e-324",
                          "2.4703282292062328e-324", "1e-400", "-1e-400", "123456789012345678901234567890",
                          "18446744073709551615", "18446744073709551616", "-9223372036854775808",
                          "-9223372036854775809", "9007199254740993", "0.1", "1.7976931348623157e308",
                          "0.30000000000000004", "12345678901234567890.123456789", "1.00000000000000011102230246251565404236316680908203125"};
    for (const char* a : nums)
        check(std::string("number ") + a,
              std::string(R"({"type":"Polygon","coordinates":[[[)") + a + R"(,0],[2,0.5],[1,3],[-1,2]]]})");
    // syntax errors and accepted syntax variants
    const char* syn[] = {
        "", " ", "{", "}", "[", "{\"type\":\"Polygon\",}", "{\"type\":\"Polygon\" \"coordinates\":[]}",
        "{\"type\":\"Polygon\",\"coordinates\":[[[0,0],[1,0],[1,1],]]}", "// c\n" "{}", "{} x", "{}{}",
        "{\"type\":'Polygon'}", "{type:\"Polygon\"}", "{\"type\":\"Poly\ngon\"}", "{\"type\":\"Poly\\xgon\"}",
        "{\"type\":\"\\ud800\"}", "{\"type\":\"\\udc00\"}", "{\"type\":\"\\ud800\\u0041\"}", "{\"type\":\"\\u12\"}",
        "{\"type\":\"\xC0\x80\"}", "{\"type\":\"\xFF\"}", "{\"type\":\"\xED\xA0\x80\"}", "{\"type\":\"\xF4\x90\x80\x80\"}",
        "{\"type\":\"\xE2\x82\"}", "{\"a\":01}", "{\"a\":1.}", "{\"a\":.5}", "{\"a\":+1}", "{\"a\":-}", "{\"a\":1e}",
        "{\"a\":NaN}", "{\"a\":Infinity}", "{\"a\":tru}", "{\"a\":nul}", "{\"a\":[1 2]}", "{\"a\"}", "{\"a\":}",
        "\xEF\xBB\xBF{\"type\":\"Point\"}", "\xEF\xBB{\"type\":\"Point\"}", "  {\"type\" : \"Point\" }  \n",
        "{\"type\":\"\\u00e9\\ud83d\\ude00 \\\" \\\\ \\/ \\b \\f \\n \\r \\t\"}", "{\"type\":\"caf\xC3\xA9 \xF0\x9F\x98\x80\"}",
        "{\"\\u0074ype\":\"Point\"}", "{\"type\":\"Point\",\"p\":[true,false,null,{},[],\"\"]}",
        "\t\r\n{\"type\":\"Point\"}", "null", "\"Polygon\"", "[]",
    };
    for (const char* d : syn) check(std::string("syntax ") + d, d);
    check("trailing NUL", sq + std::string(1, '\0'));
    check("NUL then junk", sq + std::string(1, '\0') + "junk");
    check("NUL inside", std::string(R"({"type":"Pol)") + std::string(1, '\0') + R"(ygon"})");
    check("NUL first", std::string(1, '\0') + sq);
    check("overflow", R"({"type":"Polygon","coordinates":[[[1e400,0],[1,0],[1,1]]]})", true);
    // random valid documents (wrappers, holes, whitespace, number forms, BOM, escapes in properties)
    std::mt19937_64 g(2024);
    for (int t = 0; t < 400; ++t) {
        const bool ws = g() & 1;
        const double cx = std::uniform_real_distribution<double>(-180, 180)(g);
        const double cy = std::uniform_real_distribution<double>(-80, 80)(g);
        const double r = std::pow(10.0, -(double)(g() % 8));
        std::string rings = ring(g, 3 + (int)(g() % 40), cx, cy, r, g() & 1, ws);
        const int holes = (int)(g() % 3);
        for (int k = 0; k < holes; ++k) rings += (ws ? " ,\n" : ",") + ring(g, 3 + (int)(g() % 8), cx, cy, r * 0.2, g() & 1, ws);
        std::string geom = std::string(R"({"type":"Polygon",)") + (ws ? "\n  " : "") + R"("coordinates":[)" + rings + "]}";
        std::string doc;
        switch (g() % 3) {
        case 0: doc = geom; break;
        case 1: doc = R"({"type":"Feature","properties":{"name":"b\u00e9t \"x\"","id":)" + std::to_string(t) + R"(},"geometry":)" + geom + "}"; break;
        default:
            doc = R"({"type":"FeatureCollection","features":[{"type":"Feature","geometry":)" + geom +
                  R"(},{"type":"Feature","geometry":{"type":"Point","coordinates":[1,2]}}]})";
        }
        if (g() % 10 == 0) doc = "\xEF\xBB\xBF" + doc;
        check("random", doc);
    }
    std::printf("geojson_test: %d documents, %d parsed identically, %d failures\n", total, compared_ok, fails);
    return fails > 100 ? 100 : fails;
}
