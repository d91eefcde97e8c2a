/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * Plain-C restatement of the reference's batched point-in-polygon path over
 * raw arrays (SoA vertices + ring CSR), used as the parity checker where the
 * reference types cannot express the input (consecutive duplicate vertices,
 * SURVEY §8 rule P8) and cross-validated bit-for-bit against the reference
 * itself (oracle/_ref/libpolycast_ref.so) on every duplicate-free input in
 * tests/.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it.
 *
 * Restated from (file:line into /root/reference):
 *   count_crossings_c1        proj/include/polycast/geometry.hpp:182-203
 *   count_crossings_c2        proj/include/polycast/geometry.hpp:208-229
 *   robust_ray_crossings      proj/include/polycast/geometry.hpp:237-273
 *   contains (even-odd)       proj/include/polycast/geometry.hpp:281-300
 *   bbox_of / BBox::contains  proj/include/polycast/batch.hpp:121-133, :39-41
 *   classify_batch per point  proj/include/polycast/batch.hpp:196-210
 *
 * Build: gcc -O2 -ffp-contract=off (never -ffast-math): every operation is a
 * single IEEE double op in the reference's expression order (rule P1).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

enum { ORC_INSIDE = 0, ORC_OUTSIDE = 1, ORC_BOUNDARY = 2, ORC_ERROR = 3 };
enum { MODE_C1 = 0, MODE_C2 = 1, MODE_ROBUST = 2 };

/* geometry.hpp:182-203 — returns the crossing count of one ring. */
static uint64_t ring_c1(double px, double py, const double* vx, const double* vy, uint64_t lo,
                        uint64_t hi) {
    uint64_t count = 0;
    if (hi - lo < 2) return 0;
    double f_prev = vy[lo] - py;
    for (uint64_t i = lo; i + 1 < hi; ++i) {
        const double ax = vx[i], ay = vy[i], bx = vx[i + 1], by = vy[i + 1];
        const double f_next = by - py;
        if (f_prev * f_next <= 0.0) {
            double nx = by - ay;
            double ny = ax - bx;
            if (nx < 0.0) {
                nx = -nx;
                ny = -ny;
            }
            const double side = (px - ax) * nx + (py - ay) * ny;
            if (side <= 0.0) ++count;
        }
        f_prev = f_next;
    }
    return count;
}

/* geometry.hpp:208-229 — *degenerate set to 1 where the reference throws. */
static uint64_t ring_c2(double px, double py, const double* vx, const double* vy, uint64_t lo,
                        uint64_t hi, int* degenerate) {
    uint64_t count = 0;
    if (hi - lo < 2) return 0;
    double f_prev = vy[lo] - py;
    for (uint64_t i = lo; i + 1 < hi; ++i) {
        const double ax = vx[i], ay = vy[i], bx = vx[i + 1], by = vy[i + 1];
        const double f_next = by - py;
        if (f_prev * f_next <= 0.0) {
            const double dy = by - ay;
            if (dy == 0.0) {
                *degenerate = 1;
                return count;
            }
            const double lambda = (py - ay) / dy;
            const double x = ax + lambda * (bx - ax);
            if (x > px) ++count;
        }
        f_prev = f_next;
    }
    return count;
}

/* std::clamp(v, 0.0, 1.0) as libstdc++ evaluates it (NaN propagates). */
static double clamp01(double v) { return (v < 0.0) ? 0.0 : ((1.0 < v) ? 1.0 : v); }

/* geometry.hpp:237-273 */
static uint64_t ring_robust(double px, double py, const double* vx, const double* vy, uint64_t lo,
                            uint64_t hi, double tol, int* on_boundary) {
    uint64_t count = 0;
    const double tol2 = tol * tol;
    if (hi - lo < 2) return 0;
    for (uint64_t i = lo; i + 1 < hi; ++i) {
        const double ax = vx[i], ay = vy[i], bx = vx[i + 1], by = vy[i + 1];
        const double ylo = by < ay ? by : ay; /* std::min(a.y, b.y): returns a if !(b < a) */
        const double yhi = ay < by ? by : ay; /* std::max(a.y, b.y): returns a if !(a < b) */
        if (py + tol < ylo || py - tol > yhi) continue;
        const double abx = bx - ax;
        const double aby = by - ay;
        const double apx = px - ax;
        const double apy = py - ay;
        const double len2 = abx * abx + aby * aby;
        double t = (apx * abx + apy * aby) / len2;
        t = clamp01(t);
        const double dx = apx - t * abx;
        const double dyp = apy - t * aby;
        if (dx * dx + dyp * dyp <= tol2) {
            *on_boundary = 1;
            return count;
        }
        const int upward = ay <= py && py < by;
        const int downward = by <= py && py < ay;
        if (upward || downward) {
            const double x = ax + (py - ay) / aby * abx;
            if (x > px) ++count;
        }
    }
    return count;
}

/* contains(): geometry.hpp:281-300, mapped to the batch Verdict enum. */
static uint8_t classify_point(double px, double py, const double* vx, const double* vy,
                              const uint64_t* ring_off, uint64_t r0, uint64_t r1, int mode,
                              double tol) {
    uint64_t total = 0;
    for (uint64_t r = r0; r < r1; ++r) {
        const uint64_t lo = ring_off[r], hi = ring_off[r + 1];
        if (mode == MODE_C1) {
            total += ring_c1(px, py, vx, vy, lo, hi);
        } else if (mode == MODE_C2) {
            int deg = 0;
            total += ring_c2(px, py, vx, vy, lo, hi, &deg);
            if (deg) return ORC_ERROR;
        } else {
            int ob = 0;
            total += ring_robust(px, py, vx, vy, lo, hi, tol, &ob);
            if (ob) return ORC_BOUNDARY;
        }
    }
    return (total % 2 == 1) ? ORC_INSIDE : ORC_OUTSIDE;
}

/* bbox_of(): batch.hpp:121-133 (outer ring only; std::min/std::max order). */
void orc_bbox(const double* vx, const double* vy, const uint64_t* ring_off, uint64_t r0,
              double* box) {
    double mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
    for (uint64_t i = ring_off[r0]; i < ring_off[r0 + 1]; ++i) {
        mnx = vx[i] < mnx ? vx[i] : mnx; /* std::min(min_x, v.x) returns min_x unless v.x < min_x */
        mny = vy[i] < mny ? vy[i] : mny;
        mxx = mxx < vx[i] ? vx[i] : mxx; /* std::max(max_x, v.x) returns max_x unless max_x < v.x */
        mxy = mxy < vy[i] ? vy[i] : mxy;
    }
    box[0] = mnx;
    box[1] = mny;
    box[2] = mxx;
    box[3] = mxy;
}

typedef struct {
    const double* xy;
    const double* vx;
    const double* vy;
    const uint64_t* ring_off;
    const uint64_t* pt_off;        /* CSR only */
    const uint64_t* poly_ring_off; /* CSR only */
    uint32_t n_rings;
    int mode;
    double tol;
    int prefilter;
    uint8_t* verdicts;
    uint64_t lo, hi; /* point range (single) or polygon range (CSR) */
    uint64_t stats[4];
} job_t;

static void* run_single(void* arg) {
    job_t* j = (job_t*)arg;
    double box[4];
    orc_bbox(j->vx, j->vy, j->ring_off, 0, box);
    for (uint64_t i = j->lo; i < j->hi; ++i) {
        const double px = j->xy[2 * i], py = j->xy[2 * i + 1];
        uint8_t v = ORC_OUTSIDE;
        const int inbox = px >= box[0] && px <= box[2] && py >= box[1] && py <= box[3];
        if (!j->prefilter || inbox)
            v = classify_point(px, py, j->vx, j->vy, j->ring_off, 0, j->n_rings, j->mode, j->tol);
        j->verdicts[i] = v;
        j->stats[v]++;
    }
    return NULL;
}

static void* run_csr(void* arg) {
    job_t* j = (job_t*)arg;
    for (uint64_t p = j->lo; p < j->hi; ++p) {
        const uint64_t r0 = j->poly_ring_off[p], r1 = j->poly_ring_off[p + 1];
        double box[4];
        if (r1 > r0) orc_bbox(j->vx, j->vy, j->ring_off, r0, box);
        for (uint64_t i = j->pt_off[p]; i < j->pt_off[p + 1]; ++i) {
            const double px = j->xy[2 * i], py = j->xy[2 * i + 1];
            uint8_t v = ORC_OUTSIDE;
            if (r1 > r0 && px >= box[0] && px <= box[2] && py >= box[1] && py <= box[3])
                v = classify_point(px, py, j->vx, j->vy, j->ring_off, r0, r1, j->mode, j->tol);
            j->verdicts[i] = v;
            j->stats[v]++;
        }
    }
    return NULL;
}

static void run_jobs(job_t* base, uint64_t total, int nthreads, void* (*fn)(void*),
                     uint64_t* stats) {
    if (nthreads < 1) nthreads = 1;
    if ((uint64_t)nthreads > total) nthreads = total ? (int)total : 1;
    job_t* jobs = (job_t*)calloc((size_t)nthreads, sizeof(job_t));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    const uint64_t chunk = (total + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = *base;
        jobs[t].lo = t * chunk < total ? t * chunk : total;
        jobs[t].hi = (t + 1) * chunk < total ? (t + 1) * chunk : total;
        pthread_create(&th[t], NULL, fn, &jobs[t]);
    }
    for (int k = 0; k < 4; ++k) stats[k] = 0;
    for (int t = 0; t < nthreads; ++t) {
        pthread_join(th[t], NULL);
        for (int k = 0; k < 4; ++k) stats[k] += jobs[t].stats[k];
    }
    free(jobs);
    free(th);
}

/* classify_batch (prefilter=1) or per-point contains (prefilter=0) over one
 * polygon given as rings [ring_off[r], ring_off[r+1]) of closed vertex loops.
 * stats[4] = {inside, outside, boundary, error} (BatchStats order). */
void orc_classify(const double* xy, uint64_t n, const double* vx, const double* vy,
                  const uint64_t* ring_off, uint32_t n_rings, int mode, double tol, int prefilter,
                  uint8_t* verdicts, uint64_t* stats, int nthreads) {
    job_t j = {0};
    j.xy = xy;
    j.vx = vx;
    j.vy = vy;
    j.ring_off = ring_off;
    j.n_rings = n_rings;
    j.mode = mode;
    j.tol = tol;
    j.prefilter = prefilter;
    j.verdicts = verdicts;
    run_jobs(&j, n, nthreads, run_single, stats);
}

/* Multi-polygon CSR batch: polygon p owns points [pt_off[p], pt_off[p+1]) and
 * rings [poly_ring_off[p], poly_ring_off[p+1]); classify_batch semantics
 * (bbox prefilter on the polygon's outer ring) per polygon. */
void orc_classify_csr(const double* xy, const uint64_t* pt_off, uint64_t n_polys, const double* vx,
                      const double* vy, const uint64_t* ring_off, const uint64_t* poly_ring_off,
                      int mode, double tol, uint8_t* verdicts, uint64_t* stats, int nthreads) {
    job_t j = {0};
    j.xy = xy;
    j.vx = vx;
    j.vy = vy;
    j.ring_off = ring_off;
    j.pt_off = pt_off;
    j.poly_ring_off = poly_ring_off;
    j.mode = mode;
    j.tol = tol;
    j.verdicts = verdicts;
    run_jobs(&j, n_polys, nthreads, run_csr, stats);
}

/* count_crossings_c1 / _c2 of one ring for n points; err[i] = 1 where the
 * reference throws DegenerateEdge (C2). */
void orc_count_crossings(const double* xy, uint64_t n, const double* vx, const double* vy,
                         uint64_t nv, int mode, uint64_t* counts, uint8_t* err) {
    for (uint64_t i = 0; i < n; ++i) {
        int deg = 0;
        counts[i] = mode == MODE_C1 ? ring_c1(xy[2 * i], xy[2 * i + 1], vx, vy, 0, nv)
                                    : ring_c2(xy[2 * i], xy[2 * i + 1], vx, vy, 0, nv, &deg);
        err[i] = (uint8_t)deg;
    }
}
