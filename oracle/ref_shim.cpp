// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// C-ABI shim around the *unmodified* reference implementation of the hot path
// (polycast, header-only C++20).  The reference headers are included straight
// from /root/reference/proj/include at build time (see oracle/Makefile); no
// reference source is copied into this repository.  The built library lands in
// oracle/_ref/libpolycast_ref.so and is used only by tests/, by
// __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
// arm, always as the checker or the CPU baseline, never as the product path.
//
// Entry points wrap:
//   classify_batch  proj/include/polycast/batch.hpp:184-230
//   contains        proj/include/polycast/geometry.hpp:281-300
//   count_crossings_c1 / _c2  proj/include/polycast/geometry.hpp:182-229
//   bbox_of         proj/include/polycast/batch.hpp:121-133
#include <polycast/batch.hpp>
#include <polycast/geometry.hpp>

#include <atomic>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

using namespace polycast;

namespace {

thread_local std::string g_err;

CrossingMode to_mode(int m) {
    switch (m) {
    case 0: return CrossingMode::C1;
    case 1: return CrossingMode::C2;
    default: return CrossingMode::Robust;
    }
}

Ring make_ring(const double* vx, const double* vy, uint64_t lo, uint64_t hi) {
    std::vector<Point2> v;
    v.reserve(hi - lo);
    for (uint64_t i = lo; i < hi; ++i) v.emplace_back(vx[i], vy[i]);
    return Ring(std::move(v));
}

Polygon make_polygon(const double* vx, const double* vy, const uint64_t* ring_off, uint64_t r0,
                     uint64_t r1) {
    Ring outer = make_ring(vx, vy, ring_off[r0], ring_off[r0 + 1]);
    std::vector<Ring> holes;
    for (uint64_t r = r0 + 1; r < r1; ++r) holes.push_back(make_ring(vx, vy, ring_off[r], ring_off[r + 1]));
    return Polygon(std::move(outer), std::move(holes));
}

PointBatch make_batch(const double* xy, uint64_t lo, uint64_t hi) {
    PointBatch b;
    b.points.reserve(hi - lo);
    for (uint64_t i = lo; i < hi; ++i) b.points.emplace_back(xy[2 * i], xy[2 * i + 1]);
    return b;
}

void put_stats(const BatchStats& s, uint64_t* stats) {
    stats[0] = s.inside;
    stats[1] = s.outside;
    stats[2] = s.boundary;
    stats[3] = s.error;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Builds the Polygon (validating exactly as the reference types do) and runs
// the reference classify_batch.  Returns 0, or 1 when the reference rejects the
// input (message in ref_last_error()).
int ref_classify(const double* xy, uint64_t n, const double* vx, const double* vy,
                 const uint64_t* ring_off, uint32_t n_rings, int mode, double tol, uint64_t workers,
                 uint8_t* verdicts, uint64_t* stats) {
    try {
        const Polygon poly = make_polygon(vx, vy, ring_off, 0, n_rings);
        const PointBatch batch = make_batch(xy, 0, n);
        const BatchResult r = classify_batch(batch, poly, to_mode(mode), workers, tol);
        if (verdicts) std::memcpy(verdicts, r.verdicts.data(), n);
        if (stats) put_stats(r.stats, stats);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Same, but only the timed classify_batch call: the Polygon and PointBatch are
// prebuilt by ref_prepare() (outside any timer, as BASELINE.md §4 asks).
struct RefPrepared {
    Polygon poly;
    PointBatch batch;
};

void* ref_prepare(const double* xy, uint64_t n, const double* vx, const double* vy,
                  const uint64_t* ring_off, uint32_t n_rings) {
    try {
        return new RefPrepared{make_polygon(vx, vy, ring_off, 0, n_rings), make_batch(xy, 0, n)};
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_prepared_free(void* h) { delete static_cast<RefPrepared*>(h); }

int ref_run_prepared(void* h, int mode, double tol, uint64_t workers, uint64_t* stats) {
    auto* p = static_cast<RefPrepared*>(h);
    const BatchResult r = classify_batch(p->batch, p->poly, to_mode(mode), workers, tol);
    if (stats) put_stats(r.stats, stats);
    return 0;
}

// Single-point contains(): returns Classification (0 Inside, 1 Outside,
// 2 Boundary), 3 when DegenerateEdge was thrown, -1 on invalid input.
int ref_contains(double px, double py, const double* vx, const double* vy, const uint64_t* ring_off,
                 uint32_t n_rings, int mode, double tol) {
    try {
        const Polygon poly = make_polygon(vx, vy, ring_off, 0, n_rings);
        return static_cast<int>(contains(Point2(px, py), poly, to_mode(mode), tol));
    } catch (const DegenerateEdge& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// count_crossings_c1 (mode 0) / count_crossings_c2 (mode 1) of one ring.
// Returns 0 and *count, 3 on DegenerateEdge, -1 on invalid input.
int ref_count_crossings(double px, double py, const double* vx, const double* vy, uint64_t nv,
                        int mode, uint64_t* count) {
    try {
        const Ring ring = make_ring(vx, vy, 0, nv);
        const Point2 p(px, py);
        *count = mode == 0 ? count_crossings_c1(p, ring) : count_crossings_c2(p, ring);
        return 0;
    } catch (const DegenerateEdge& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// bbox_of(poly) -> out[4] = {min_x, min_y, max_x, max_y}.
int ref_bbox_of(const double* vx, const double* vy, const uint64_t* ring_off, uint32_t n_rings,
                double* out) {
    try {
        const BBox b = bbox_of(make_polygon(vx, vy, ring_off, 0, n_rings));
        out[0] = b.min_x;
        out[1] = b.min_y;
        out[2] = b.max_x;
        out[3] = b.max_y;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Multi-polygon CSR batch (no reference symbol): an outer
// work-stealing pool over polygons, each calling the reference
// classify_batch(points_i, poly_i, mode, 1).  Polygons are built inside the
// call when `prepared` is null.  Returns 0, or 1 if any polygon is rejected by
// the reference types (message in ref_last_error()).
int ref_classify_csr(const double* xy, const uint64_t* pt_off, uint64_t n_polys, const double* vx,
                     const double* vy, const uint64_t* ring_off, const uint64_t* poly_ring_off,
                     int mode, double tol, uint64_t threads, uint8_t* verdicts, uint64_t* stats) {
    std::vector<Polygon> polys;
    polys.reserve(n_polys);
    try {
        for (uint64_t p = 0; p < n_polys; ++p)
            polys.push_back(make_polygon(vx, vy, ring_off, poly_ring_off[p], poly_ring_off[p + 1]));
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
    const uint64_t nthr = threads ? threads : default_worker_count();
    std::atomic<uint64_t> next{0};
    std::vector<BatchStats> part(nthr);
    auto work = [&](uint64_t t) {
        for (;;) {
            const uint64_t p = next.fetch_add(1);
            if (p >= n_polys) return;
            const PointBatch b = make_batch(xy, pt_off[p], pt_off[p + 1]);
            const BatchResult r = classify_batch(b, polys[p], to_mode(mode), 1, tol);
            if (verdicts) std::memcpy(verdicts + pt_off[p], r.verdicts.data(), r.verdicts.size());
            part[t].add(r.stats);
        }
    };
    std::vector<std::thread> th;
    for (uint64_t t = 0; t < nthr; ++t) th.emplace_back(work, t);
    for (auto& t : th) t.join();
    BatchStats tot;
    for (auto& s : part) tot.add(s);
    if (stats) put_stats(tot, stats);
    return 0;
}

uint64_t ref_default_worker_count() { return default_worker_count(); }

} // extern "C"
