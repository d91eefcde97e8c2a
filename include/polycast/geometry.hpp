// polycast-b200 — geometry layer of the drop-in C++ API.
//
// Same public surface as the reference header proj/include/polycast/geometry.hpp
// (types :14-107, composed helpers :115-177, crossing counts :182-229,
// contains :281-300, to_string/mode_token :302-321): same names, enum orders,
// default arguments and exception types.  What differs is where the work runs:
// the crossing counts and contains() are evaluated by the sm_100a kernels of
// libpolycast_cuda.so through the C-ABI in include/polycast_cuda.h, with
// bit-identical results.  The composed per-ring helpers, which return per-edge
// vectors rather than verdicts, stay host-inline.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "device.hpp"

namespace polycast {

/// A crossing test needed a usable edge and did not get one: identical
/// endpoints, or (C2) a horizontal edge lying exactly on the query ray.
struct DegenerateEdge : std::runtime_error {
    explicit DegenerateEdge(const std::string& what) : std::runtime_error(what) {}
};

/// Query point / vertex; both coordinates must be finite.
struct Point2 {
    double x = 0.0;
    double y = 0.0;

    Point2() = default;
    Point2(double px, double py) : x(px), y(py) {
        if (!(std::isfinite(px) && std::isfinite(py)))
            throw std::invalid_argument("Point2: coordinates must be finite");
    }

    friend bool operator==(const Point2& a, const Point2& b) { return a.x == b.x && a.y == b.y; }
};

// Point2[] is passed to the GPU engine as interleaved x,y doubles.
static_assert(sizeof(Point2) == 16 && std::is_standard_layout_v<Point2>, "Point2 must be two packed doubles");

/// Closed vertex loop stored with its closing vertex (front() == back()), at
/// least a closed triangle, no zero-length edges.
class Ring {
  public:
    explicit Ring(std::vector<Point2> vertices) : v_(std::move(vertices)) {
        if (v_.size() < 4) throw std::invalid_argument("Ring: need at least 4 vertices (closed triangle)");
        if (!(v_.front() == v_.back())) throw std::invalid_argument("Ring: first and last vertex must be equal");
        for (std::size_t k = 1; k < v_.size(); ++k)
            if (v_[k - 1] == v_[k])
                throw std::invalid_argument("Ring: consecutive duplicate vertex at index " + std::to_string(k - 1));
    }

    std::size_t size() const { return v_.size(); }
    std::size_t edge_count() const { return v_.size() - 1; }
    const Point2& operator[](std::size_t i) const { return v_[i]; }
    std::span<const Point2> vertices() const { return v_; }

  private:
    std::vector<Point2> v_;
};

/// Outer ring plus holes; rings combine by even-odd parity.
class Polygon {
  public:
    explicit Polygon(Ring outer, std::vector<Ring> holes = {}) {
        rings_.reserve(holes.size() + 1);
        rings_.push_back(std::move(outer));
        rings_.insert(rings_.end(), std::make_move_iterator(holes.begin()), std::make_move_iterator(holes.end()));
    }

    const Ring& outer() const { return rings_[0]; }
    std::span<const Ring> holes() const { return std::span<const Ring>(rings_).subspan(1); }
    std::span<const Ring> rings() const { return rings_; }

  private:
    std::vector<Ring> rings_;
};

/// Edge normal oriented so that nx >= 0.
struct EdgeNormal {
    double nx = 0.0;
    double ny = 0.0;
};

enum class Classification { Inside, Outside, Boundary };

/// C1: inclusive sign-change scan + side-of-normal test (p - r_i).n <= 0.
/// C2: inclusive sign-change scan + parametric crossing x > p_x (DegenerateEdge
///     on a horizontal edge on the ray).
/// Robust: half-open rule with Boundary detection within boundary_tol.
enum class CrossingMode { C1, C2, Robust };

inline constexpr double kDefaultBoundaryTol = 1e-12;

// ---- composed per-ring helpers (host-inline; not on the batched path) -------

/// f_i = y_i - p_y for every stored vertex of the ring.
inline std::vector<double> signed_offsets(const Ring& ring, double p_y) {
    std::vector<double> f(ring.size());
    for (std::size_t i = 0; i < f.size(); ++i) f[i] = ring[i].y - p_y;
    return f;
}

/// Edges i whose offsets satisfy f_i * f_{i+1} <= 0 (zero counts on both sides).
inline std::vector<std::size_t> detect_sign_changes(std::span<const double> offsets) {
    if (offsets.size() < 2) throw std::invalid_argument("detect_sign_changes: need at least 2 offsets");
    std::vector<std::size_t> idx;
    for (std::size_t i = 1; i < offsets.size(); ++i)
        if (offsets[i - 1] * offsets[i] <= 0.0) idx.push_back(i - 1);
    return idx;
}

inline EdgeNormal edge_normal(const Point2& a, const Point2& b) {
    if (a == b) throw DegenerateEdge("edge_normal: zero-length edge");
    const EdgeNormal n{b.y - a.y, a.x - b.x};
    return n.nx < 0.0 ? EdgeNormal{-n.nx, -n.ny} : n;
}

inline EdgeNormal edge_normal_c1(const Ring& ring, std::size_t edge_index) {
    return edge_normal(ring[edge_index], ring[edge_index + 1]);
}

inline double crossing_x(const Point2& a, const Point2& b, double p_y) {
    const double dy = b.y - a.y;
    if (dy == 0.0) throw DegenerateEdge("crossing_x: horizontal edge has no unique crossing");
    const double lambda = (p_y - a.y) / dy;
    return a.x + lambda * (b.x - a.x);
}

inline double crossing_x_c2(const Ring& ring, std::size_t edge_index, double p_y) {
    return crossing_x(ring[edge_index], ring[edge_index + 1], p_y);
}

/// Distance from p to the closed segment ab.
inline double segment_distance(const Point2& p, const Point2& a, const Point2& b) {
    const double ux = b.x - a.x, uy = b.y - a.y;
    const double wx = p.x - a.x, wy = p.y - a.y;
    const double uu = ux * ux + uy * uy;
    double t = uu > 0.0 ? (wx * ux + wy * uy) / uu : 0.0;
    t = t < 0.0 ? 0.0 : (1.0 < t ? 1.0 : t);
    const double ex = wx - t * ux, ey = wy - t * uy;
    return std::sqrt(ex * ex + ey * ey);
}

// ---- GPU-evaluated crossing tests ------------------------------------------

namespace detail {

/// SoA flattening of a polygon for the C-ABI (closing vertices kept).
struct FlatPolygon {
    std::vector<double> x, y;
    std::vector<uint64_t> ring_off{0};

    explicit FlatPolygon(const Polygon& poly) {
        std::size_t total = 0;
        for (const Ring& r : poly.rings()) total += r.size();
        x.reserve(total);
        y.reserve(total);
        for (const Ring& r : poly.rings()) {
            for (const Point2& v : r.vertices()) {
                x.push_back(v.x);
                y.push_back(v.y);
            }
            ring_off.push_back(x.size());
        }
    }
    uint32_t rings() const { return static_cast<uint32_t>(ring_off.size() - 1); }
};

inline int mode_code(CrossingMode m) { return static_cast<int>(m); }

inline std::size_t ring_count(const Point2& p, const Ring& ring, int mode, const char* who) {
    std::vector<double> x(ring.size()), y(ring.size());
    for (std::size_t i = 0; i < ring.size(); ++i) {
        x[i] = ring[i].x;
        y[i] = ring[i].y;
    }
    uint64_t cnt = 0;
    uint8_t deg = 0;
    pc_ctx* ctx = device::context();
    device::throw_on(pc_count_crossings(ctx, &p.x, 1, x.data(), y.data(), x.size(), mode, &cnt, &deg), ctx, who);
    // the reference's message names the first degenerate edge (geometry.hpp:219-220);
    // the engine reports its index in place of the count
    if (deg) throw DegenerateEdge(std::string(who) + ": horizontal edge " + std::to_string(cnt) + " lies on the query ray");
    return static_cast<std::size_t>(cnt);
}

} // namespace detail

/// Rightward-ray crossings of one ring, side-of-normal test (paper Algorithm 1).
inline std::size_t count_crossings_c1(const Point2& p, const Ring& ring) {
    return detail::ring_count(p, ring, PC_MODE_C1, "count_crossings_c1");
}

/// Rightward-ray crossings of one ring, parametric crossing (paper Algorithm 2).
inline std::size_t count_crossings_c2(const Point2& p, const Ring& ring) {
    return detail::ring_count(p, ring, PC_MODE_C2, "count_crossings_c2");
}

/// Even-odd classification of one point (no bounding-box short-circuit).
inline Classification contains(const Point2& p, const Polygon& poly, CrossingMode mode,
                               double boundary_tol = kDefaultBoundaryTol) {
    const detail::FlatPolygon f(poly);
    uint8_t verdict = PC_OUTSIDE;
    pc_ctx* ctx = device::context();
    device::throw_on(pc_classify(ctx, &p.x, 1, f.x.data(), f.y.data(), f.ring_off.data(), f.rings(),
                                 detail::mode_code(mode), boundary_tol, 0, &verdict, nullptr, nullptr, nullptr),
                     ctx, "contains");
    switch (verdict) {
    case PC_INSIDE: return Classification::Inside;
    case PC_BOUNDARY: return Classification::Boundary;
    case PC_ERROR:
        // the reference's contains propagates count_crossings_c2's exception from
        // the first ring (in ring order) whose loop meets a horizontal edge on the ray
        for (const Ring& ring : poly.rings()) detail::ring_count(p, ring, PC_MODE_C2, "count_crossings_c2");
        throw DegenerateEdge("count_crossings_c2: horizontal edge lies on the query ray");
    default: return Classification::Outside;
    }
}

inline const char* to_string(Classification c) {
    switch (c) {
    case Classification::Inside: return "inside";
    case Classification::Outside: return "outside";
    case Classification::Boundary: return "boundary";
    }
    return "?";
}

inline const char* mode_token(CrossingMode mode) {
    switch (mode) {
    case CrossingMode::C1: return "c1";
    case CrossingMode::C2: return "c2";
    case CrossingMode::Robust: return "robust";
    }
    return "?";
}

} // namespace polycast
