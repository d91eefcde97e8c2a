// Seeded synthetic workloads for the five BASELINE.json configs.
//
// The paper's data (Google Open Buildings points, GADM Ghana boundary —
// PAPER.md:258-271) is not available; these generators stand in for it with
// the shapes, sizes and value distributions BASELINE.json names.  Everything is
// drawn from std::mt19937_64 (fully specified by the C++ standard) mapped to
// [0,1) through the 53-bit mantissa, the reference's own idiom
// (proj/include/polycast/bench.hpp:63-70, proj/tests/support/random_shapes.hpp:16-18),
// so a (config, seed) pair always yields the same bytes.  Large point sets are
// generated in fixed-size chunks, each with its own seed_seq, so the output is
// independent of the thread count.
//
// Layouts (the framework's device layout):
//   points    AoS interleaved x,y doubles (== reference Point2[])
//   vertices  SoA vx[], vy[]; each ring stored closed (first == last)
//   ring_off  CSR into vertices, poly_ring_off CSR into rings, pt_off CSR into points
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numbers>
#include <random>
#include <thread>
#include <vector>

namespace {

constexpr double kMetersPerDegLat = 111320.0;
constexpr uint64_t kChunk = 1u << 20; // points per independently seeded chunk

struct Rng {
    std::mt19937_64 eng;
    explicit Rng(std::initializer_list<uint64_t> key) {
        std::vector<uint32_t> w;
        for (uint64_t k : key) {
            w.push_back(static_cast<uint32_t>(k));
            w.push_back(static_cast<uint32_t>(k >> 32));
        }
        std::seed_seq sq(w.begin(), w.end());
        eng.seed(sq);
    }
    double u() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + u() * (hi - lo); }
    uint64_t below(uint64_t n) { return eng() % n; }
};

template <class Fn>
void parallel_chunks(uint64_t nchunks, int threads, Fn&& fn) {
    if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    threads = static_cast<int>(std::min<uint64_t>(threads, std::max<uint64_t>(nchunks, 1)));
    std::vector<std::thread> th;
    for (int t = 0; t < threads; ++t)
        th.emplace_back([&, t] {
            for (uint64_t c = t; c < nchunks; c += threads) fn(c);
        });
    for (auto& x : th) x.join();
}

struct CsrSet {
    std::vector<double> vx, vy, xy;
    std::vector<uint64_t> ring_off{0}, poly_ring_off{0}, pt_off{0};

    void add_ring(const std::vector<double>& x, const std::vector<double>& y) {
        vx.insert(vx.end(), x.begin(), x.end());
        vy.insert(vy.end(), y.begin(), y.end());
        ring_off.push_back(vx.size());
    }
    void end_polygon() {
        poly_ring_off.push_back(ring_off.size() - 1);
        pt_off.push_back(xy.size() / 2);
    }
    void append(const CsrSet& o) {
        const uint64_t v0 = vx.size(), r0 = ring_off.size() - 1, p0 = xy.size() / 2;
        vx.insert(vx.end(), o.vx.begin(), o.vx.end());
        vy.insert(vy.end(), o.vy.begin(), o.vy.end());
        xy.insert(xy.end(), o.xy.begin(), o.xy.end());
        for (size_t i = 1; i < o.ring_off.size(); ++i) ring_off.push_back(v0 + o.ring_off[i]);
        for (size_t i = 1; i < o.poly_ring_off.size(); ++i) poly_ring_off.push_back(r0 + o.poly_ring_off[i]);
        for (size_t i = 1; i < o.pt_off.size(); ++i) pt_off.push_back(p0 + o.pt_off[i]);
    }
};

// ---- c3: building footprints ------------------------------------------------
// Staircase outline with k steps (k=0 rotated rectangle, k=1 L-shape, ...),
// 4 + 2k distinct vertices, k in 0..6 -> 4..16 vertices; sides W,H in [10,50] m.
void footprint(Rng& rng, uint64_t pts_per_poly, CsrSet& out) {
    const int k = static_cast<int>(rng.below(7));
    const double W = rng.uniform(10.0, 50.0), H = rng.uniform(10.0, 50.0);
    std::vector<double> lx{0.0, W}, ly{0.0, 0.0};
    double xprev = W;
    for (int i = 1; i <= k; ++i) {
        const double xi = W * (1.0 - (i + rng.uniform(-0.3, 0.3)) / (k + 1));
        const double yi = H * ((i + rng.uniform(-0.3, 0.3)) / (k + 1));
        lx.push_back(xprev); ly.push_back(yi);
        lx.push_back(xi);    ly.push_back(yi);
        xprev = xi;
    }
    lx.push_back(xprev); ly.push_back(H);
    lx.push_back(0.0);   ly.push_back(H);

    const double clon = rng.uniform(-0.5, 0.5), clat = rng.uniform(5.0, 6.0);
    const double phi = rng.uniform(0.0, 2.0 * std::numbers::pi);
    const double c = std::cos(phi), s = std::sin(phi);
    const double mlat = 1.0 / kMetersPerDegLat;
    const double mlon = 1.0 / (kMetersPerDegLat * std::cos(clat * std::numbers::pi / 180.0));
    std::vector<double> x, y;
    for (size_t i = 0; i < lx.size(); ++i) {
        const double dx = lx[i] - 0.5 * W, dy = ly[i] - 0.5 * H;
        x.push_back(clon + (c * dx - s * dy) * mlon);
        y.push_back(clat + (s * dx + c * dy) * mlat);
    }
    const size_t nd = x.size();
    x.push_back(x[0]);
    y.push_back(y[0]);
    double x0 = x[0], x1 = x[0], y0 = y[0], y1 = y[0];
    for (size_t i = 0; i < nd; ++i) {
        x0 = std::min(x0, x[i]); x1 = std::max(x1, x[i]);
        y0 = std::min(y0, y[i]); y1 = std::max(y1, y[i]);
    }
    out.add_ring(x, y);
    const uint64_t half = pts_per_poly / 2;
    for (uint64_t i = 0; i < pts_per_poly; ++i) {
        if (i < half) {
            const double px = rng.uniform(x0, x1);
            const double py = rng.uniform(y0, y1);
            out.xy.push_back(px);
            out.xy.push_back(py);
        } else {
            const size_t v = rng.below(nd);
            const double jx = rng.uniform(-5.0, 5.0) * mlon;
            const double jy = rng.uniform(-5.0, 5.0) * mlat;
            out.xy.push_back(x[v] + jx);
            out.xy.push_back(y[v] + jy);
        }
    }
    out.end_polygon();
}

// ---- c5: degenerate / tie-breaking stress ---------------------------------
// Integer-grid rectilinear outline with rectangular notches (concave) cut into
// the top and bottom edges, an optional 45-degree chamfer, optional rectangular
// hole, inserted collinear vertices and (when allow_dups) consecutive duplicate
// vertices.  4..64 stored vertices per outer ring.  Half of the points sit
// exactly on vertices / edges / vertex y-levels, half are uniform in the bbox.
void degenerate_poly(Rng& rng, bool allow_dups, CsrSet& out) {
    const int mt = static_cast<int>(rng.below(5)), mb = static_cast<int>(rng.below(4));
    const int W = 2 * std::max(mt, mb) * 2 + 4 + static_cast<int>(rng.below(6));
    const int D = 1 + static_cast<int>(rng.below(2)); // notch depth
    const int H = 2 * D + 4 + static_cast<int>(rng.below(6));
    const double ox = static_cast<double>(static_cast<int64_t>(rng.below(2001)) - 1000);
    const double oy = static_cast<double>(static_cast<int64_t>(rng.below(2001)) - 1000);
    const bool chamfer = rng.below(2) == 0;

    std::vector<double> x, y;
    auto push = [&](double a, double b) { x.push_back(ox + a); y.push_back(oy + b); };
    // bottom edge, left -> right, notches pushing up
    push(0, 0);
    for (int i = 0; i < mb; ++i) {
        const int l = 2 + 4 * i, r = l + 1 + static_cast<int>(rng.below(2));
        push(l, 0); push(l, D); push(r, D); push(r, 0);
    }
    if (chamfer) { push(W - 1, 0); push(W, 1); } else { push(W, 0); }
    // right edge up, then top edge right -> left, notches pushing down
    push(W, H);
    for (int i = mt - 1; i >= 0; --i) {
        const int l = 2 + 4 * i, r = l + 1 + static_cast<int>(rng.below(2));
        push(r, H); push(r, H - D); push(l, H - D); push(l, H);
    }
    push(0, H);
    // collinear insertions on axis-aligned edges of length >= 2 (integer midpoints)
    std::vector<double> cx, cy;
    const size_t n = x.size();
    for (size_t i = 0; i < n; ++i) {
        cx.push_back(x[i]); cy.push_back(y[i]);
        const size_t j = (i + 1) % n;
        const double dx = x[j] - x[i], dy = y[j] - y[i];
        const bool axis = dx == 0.0 || dy == 0.0;
        if (axis && std::abs(dx + dy) >= 2.0 && rng.below(3) == 0) {
            cx.push_back(std::floor((x[i] + x[j]) / 2.0)); cy.push_back(std::floor((y[i] + y[j]) / 2.0));
        }
        if (allow_dups && rng.below(6) == 0) { cx.push_back(cx.back()); cy.push_back(cy.back()); }
    }
    // never start with a duplicate of the closing vertex
    cx.push_back(cx[0]); cy.push_back(cy[0]);
    out.add_ring(cx, cy);
    const bool hole = H >= 2 * D + 5 && W >= 6 && rng.below(4) == 0;
    if (hole) {
        const double hx0 = ox + 2, hx1 = ox + W - 2, hy0 = oy + D + 1, hy1 = oy + H - D - 1;
        out.add_ring({hx0, hx0, hx1, hx1, hx0}, {hy0, hy1, hy1, hy0, hy0});
    }
    // points
    const uint64_t npts = 50 + rng.below(101);
    const size_t nv = cx.size() - 1;
    for (uint64_t i = 0; i < npts; ++i) {
        double px, py;
        const uint64_t kind = rng.below(8);
        if (kind < 4) { // uniform in the outer bbox
            px = ox + rng.uniform(0.0, W);
            py = oy + rng.uniform(0.0, H);
        } else if (kind == 4) { // exactly on a vertex
            const size_t v = rng.below(nv);
            px = cx[v]; py = cy[v];
        } else if (kind == 5) { // on an edge at a half-integer step (exact for axis / 45-degree edges)
            const size_t v = rng.below(nv);
            const double dx = cx[v + 1] - cx[v], dy = cy[v + 1] - cy[v];
            const double len = std::max(std::abs(dx), std::abs(dy));
            const double steps = std::max(1.0, 2.0 * len);
            const double t = static_cast<double>(rng.below(static_cast<uint64_t>(steps) + 1)) / steps;
            px = cx[v] + t * dx; py = cy[v] + t * dy;
        } else if (kind == 6) { // on a vertex's y-level, integer or half-integer x
            const size_t v = rng.below(nv);
            py = cy[v];
            px = ox - 1.0 + 0.5 * static_cast<double>(rng.below(2 * W + 5));
        } else { // on a vertex's y-level, uniform x
            const size_t v = rng.below(nv);
            py = cy[v];
            px = ox + rng.uniform(-1.0, W + 1.0);
        }
        out.xy.push_back(px);
        out.xy.push_back(py);
    }
    out.end_polygon();
}

} // namespace

extern "C" {

// c1/c2: star polygon with n vertices, vertex k at angle 2*pi*k/n and radius
// uniform in [rmin, rmax]; writes n+1 closed vertices.
void wl_star(uint64_t n, uint64_t seed, double rmin, double rmax, double* vx, double* vy) {
    Rng rng({seed, n, 0x57A2});
    for (uint64_t k = 0; k < n; ++k) {
        const double th = 2.0 * std::numbers::pi * static_cast<double>(k) / static_cast<double>(n);
        const double r = rng.uniform(rmin, rmax);
        vx[k] = r * std::cos(th);
        vy[k] = r * std::sin(th);
    }
    vx[n] = vx[0];
    vy[n] = vy[0];
}

// c4: star polygon whose radius is 1 + amp * nu(theta), nu = sum_j cos(j*theta
// + phi_j)/j (1/f noise, seeded phases) normalised to [-1, 1]; r > 0 so the
// ring is simple.  Writes n+1 closed vertices.
void wl_fractal_star(uint64_t n, uint64_t seed, double amp, int terms, double* vx, double* vy,
                     int threads) {
    Rng rng({seed, n, 0xF4AC});
    std::vector<double> phase(terms);
    for (int j = 0; j < terms; ++j) phase[j] = rng.uniform(0.0, 2.0 * std::numbers::pi);
    std::vector<double> nu(n);
    const uint64_t nchunks = (n + 4095) / 4096;
    parallel_chunks(nchunks, threads, [&](uint64_t c) {
        for (uint64_t k = c * 4096; k < std::min(n, (c + 1) * 4096); ++k) {
            const double th = 2.0 * std::numbers::pi * static_cast<double>(k) / static_cast<double>(n);
            double s = 0.0;
            for (int j = 1; j <= terms; ++j) s += std::cos(j * th + phase[j - 1]) / j;
            nu[k] = s;
        }
    });
    double m = 0.0;
    for (double v : nu) m = std::max(m, std::abs(v));
    if (m == 0.0) m = 1.0;
    for (uint64_t k = 0; k < n; ++k) {
        const double th = 2.0 * std::numbers::pi * static_cast<double>(k) / static_cast<double>(n);
        const double r = 1.0 + amp * (nu[k] / m);
        vx[k] = r * std::cos(th);
        vy[k] = r * std::sin(th);
    }
    vx[n] = vx[0];
    vy[n] = vy[0];
}

// Uniform points in [x0,x1] x [y0,y1] (x drawn before y, as random_batch does).
void wl_uniform_points(uint64_t n, double x0, double y0, double x1, double y1, uint64_t seed,
                       double* xy, int threads) {
    const uint64_t nchunks = (n + kChunk - 1) / kChunk;
    parallel_chunks(nchunks, threads, [&](uint64_t c) {
        Rng rng({seed, c, 0x9017});
        for (uint64_t i = c * kChunk; i < std::min(n, (c + 1) * kChunk); ++i) {
            xy[2 * i] = rng.uniform(x0, x1);
            xy[2 * i + 1] = rng.uniform(y0, y1);
        }
    });
}

// Points [lo, hi) of the same seeded sequence as wl_uniform_points(n, ...) for
// any n >= hi (a rank generates only its shard; identical bytes).
void wl_uniform_points_range(uint64_t lo, uint64_t hi, double x0, double y0, double x1, double y1,
                             uint64_t seed, double* xy, int threads) {
    if (hi <= lo) return;
    const uint64_t c0 = lo / kChunk, c1 = (hi + kChunk - 1) / kChunk;
    parallel_chunks(c1 - c0, threads, [&](uint64_t k) {
        const uint64_t c = c0 + k;
        Rng rng({seed, c, 0x9017});
        for (uint64_t i = c * kChunk; i < std::min(hi, (c + 1) * kChunk); ++i) {
            const double x = rng.uniform(x0, x1), y = rng.uniform(y0, y1);
            if (i >= lo) {
                xy[2 * (i - lo)] = x;
                xy[2 * (i - lo) + 1] = y;
            }
        }
    });
}

// Tight bounds of a vertex range (used to place points "in the bounding box").
void wl_bounds(const double* vx, const double* vy, uint64_t n, double* box) {
    box[0] = box[2] = vx[0];
    box[1] = box[3] = vy[0];
    for (uint64_t i = 1; i < n; ++i) {
        box[0] = std::min(box[0], vx[i]); box[2] = std::max(box[2], vx[i]);
        box[1] = std::min(box[1], vy[i]); box[3] = std::max(box[3], vy[i]);
    }
}

// CSR multi-polygon sets (c3 footprints, c5 degenerate) behind a handle:
// kind 3 = footprints (pts_per_poly points each), kind 5 = degenerate.
void* wl_csr_new(int kind, uint64_t n_polys, uint64_t seed, uint64_t pts_per_poly, int allow_dups,
                 int threads) {
    constexpr uint64_t kPolyChunk = 4096;
    const uint64_t nchunks = (n_polys + kPolyChunk - 1) / kPolyChunk;
    std::vector<CsrSet> parts(nchunks);
    parallel_chunks(nchunks, threads, [&](uint64_t c) {
        Rng rng({seed, c, static_cast<uint64_t>(kind), 0xC5u});
        for (uint64_t p = c * kPolyChunk; p < std::min(n_polys, (c + 1) * kPolyChunk); ++p) {
            if (kind == 3) footprint(rng, pts_per_poly, parts[c]);
            else degenerate_poly(rng, allow_dups != 0, parts[c]);
        }
    });
    auto* out = new CsrSet();
    size_t nv = 0, np = 0;
    for (auto& p : parts) { nv += p.vx.size(); np += p.xy.size(); }
    out->vx.reserve(nv); out->vy.reserve(nv); out->xy.reserve(np);
    for (auto& p : parts) { out->append(p); CsrSet().vx.swap(p.vx); }
    return out;
}

void wl_csr_sizes(void* h, uint64_t* n_polys, uint64_t* n_rings, uint64_t* n_verts, uint64_t* n_points) {
    auto* s = static_cast<CsrSet*>(h);
    *n_polys = s->pt_off.size() - 1;
    *n_rings = s->ring_off.size() - 1;
    *n_verts = s->vx.size();
    *n_points = s->xy.size() / 2;
}

void wl_csr_copy(void* h, double* vx, double* vy, uint64_t* ring_off, uint64_t* poly_ring_off,
                 double* xy, uint64_t* pt_off) {
    auto* s = static_cast<CsrSet*>(h);
    std::memcpy(vx, s->vx.data(), s->vx.size() * 8);
    std::memcpy(vy, s->vy.data(), s->vy.size() * 8);
    std::memcpy(ring_off, s->ring_off.data(), s->ring_off.size() * 8);
    std::memcpy(poly_ring_off, s->poly_ring_off.data(), s->poly_ring_off.size() * 8);
    std::memcpy(xy, s->xy.data(), s->xy.size() * 8);
    std::memcpy(pt_off, s->pt_off.data(), s->pt_off.size() * 8);
}

void wl_csr_free(void* h) { delete static_cast<CsrSet*>(h); }

} // extern "C"
