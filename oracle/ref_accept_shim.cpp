// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// C-ABI shim over the reference's own acceptance corpus and winding-number
// oracle (proj/tests/acceptance/acceptance.cpp:82-101 corpus_polygon /
// corpus_points, proj/tests/support/random_shapes.hpp, winding_oracle.hpp),
// included from /root/reference at build time, so tests/test_acceptance_gpu.py
// can re-run acceptance checks 1 and 2 through the GPU path on exactly the
// reference's inputs.  Never the product.
#include <polycast/batch.hpp>
#include <polycast/bench.hpp>
#include <polycast/geometry.hpp>

#include <support/random_shapes.hpp>
#include <support/winding_oracle.hpp>

#include <cstdint>
#include <thread>
#include <vector>

using namespace polycast;

namespace {
constexpr std::size_t kCorpus = 50; // acceptance.cpp:83

// acceptance.cpp:87-95 (restated call for call: same seeds, same draws)
Polygon corpus_polygon(std::size_t idx) {
    std::mt19937_64 rng(9000 + idx);
    const std::size_t verts = 5 + (495 * idx) / (kCorpus - 1);
    const Point2 center(testing::uniform_in(rng, -5.0, 5.0), testing::uniform_in(rng, -5.0, 5.0));
    const double radius = testing::uniform_in(rng, 1.0, 15.0);
    if (idx % 2 == 0) return Polygon(testing::convex_ring(rng, verts, center, radius));
    return Polygon(testing::star_ring(rng, verts, center, 0.35 * radius, radius));
}
} // namespace

extern "C" {

// outer ring of corpus polygon idx into vx/vy (cap entries); returns its vertex count
uint64_t ref_corpus_polygon(uint64_t idx, double* vx, double* vy, uint64_t cap) {
    const Polygon p = corpus_polygon(idx);
    const Ring& r = p.outer();
    for (std::size_t i = 0; i < r.size() && i < cap; ++i) {
        vx[i] = r[i].x;
        vy[i] = r[i].y;
    }
    return r.size();
}

// acceptance.cpp:97-99: random_batch(bbox_of(poly).inflated(0.20), n, 4242 + idx)
void ref_corpus_points(uint64_t idx, uint64_t n, double* xy) {
    const Polygon p = corpus_polygon(idx);
    const PointBatch b = random_batch(bbox_of(p).inflated(0.20), n, 4242 + idx);
    for (std::size_t i = 0; i < n; ++i) {
        xy[2 * i] = b.points[i].x;
        xy[2 * i + 1] = b.points[i].y;
    }
}

// winding_oracle.hpp oracle_classify of n points against corpus polygon idx
// (0 Inside, 1 Outside, 2 Boundary), on all host threads
void ref_winding_oracle(uint64_t idx, const double* xy, uint64_t n, uint8_t* out) {
    const Polygon p = corpus_polygon(idx);
    const unsigned nt = std::max(1u, std::thread::hardware_concurrency());
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            for (uint64_t i = t; i < n; i += nt)
                out[i] = static_cast<uint8_t>(testing::oracle_classify(Point2(xy[2 * i], xy[2 * i + 1]), p));
        });
    for (auto& x : th) x.join();
}

} // extern "C"
