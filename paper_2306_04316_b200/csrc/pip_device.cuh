// Device-side arithmetic of the point-in-polygon crossing tests.
//
// Every floating-point operation is an explicit round-to-nearest binary64
// intrinsic (__dadd_rn/__dsub_rn/__dmul_rn/__ddiv_rn), so nvcc can neither
// contract a multiply-add into a DFMA nor reassociate: each expression
// evaluates exactly as the reference's C++ does on an x86-64 host
// (SURVEY §8 rules P1, P2, P6, P7).
#pragma once

#include <cstdint>
#include <cstdio>

// Device-side bounds / invariant checks, compiled in only for the checking
// build (make -C paper_2306_04316_b200 debug -> lib/debug/, selected with
// POLYCAST_LIB_VARIANT=debug): a failed check prints its location and traps,
// so the call returns PC_ECUDA.  This pool has no compute-sanitizer; these
// checks on every shared- and global-memory index the kernels compute are the
// substitute (tools/gpu_devchecks.sh runs tools/sanitize_cases.py with them).
#ifdef PC_DEVICE_CHECKS
#define PC_DCHECK(cond)                                                                       \
    do {                                                                                      \
        if (!(cond)) {                                                                        \
            printf("PC_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
                   (int)blockIdx.x, (int)threadIdx.x);                                        \
            __trap();                                                                         \
        }                                                                                     \
    } while (0)
#else
#define PC_DCHECK(cond) \
    do {                \
    } while (0)
#endif

namespace pcd {

enum Mode : int { kC1 = 0, kC2 = 1, kRobust = 2 };

// Per-edge record staged in shared memory, mode-specific, precomputed once per
// call by prep_edges_kernel from the raw vertices with the same RN operations
// the reference performs per (point, edge):
//   C1:     ax ay by nx ny   (n = (b.y-a.y, a.x-b.x), flipped so nx >= 0; geometry.hpp:191-196)
//   C2:     ax ay by dx dy   (dx = b.x-a.x, dy = b.y-a.y; geometry.hpp:216-222)
//   Robust: ax ay by abx aby len2 ylo yhi  (geometry.hpp:245-254)
struct __align__(16) EdgeRec {
    double d[8];
};

// Monotone 32-bit key of a double through its binary32 rounding.
//   key(u) < key(v)  =>  u < v  (strictly),  and  u <= v  =>  key(u) <= key(v).
// RN to binary32 is monotone non-decreasing; -0 is canonicalised to +0 so the
// integer order equals the float order.  Values that share a key are "ties"
// and always take the exact binary64 path, so the filter below never decides a
// case the reference decides differently (proof in DESIGN.md §3).
__device__ __forceinline__ int fkey(double v) {
    const float f = __fadd_rn(__double2float_rn(v), 0.0f);
    const int i = __float_as_int(f);
    return i >= 0 ? i : (i ^ 0x7fffffff);
}

// Unsigned monotone 64-bit key of a double (for bbox atomics).
__device__ __forceinline__ unsigned long long dkey(double v) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(__dadd_rn(v, 0.0)));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
    const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double(static_cast<long long>(b));
}

// 15-bit keys for the packed filter.  Two keys share a 32-bit register as
// (q_a << 1) | (q_b << 17): one 32-bit IMAD then subtracts an edge's key from
// both halves exactly (the low half's carry only reaches bit 0 of the high
// half, which the compare ignores) and a 3-input packed VIMNMX3.U16x2 folds
// four points into a running minimum.
// q(y) = clamp(floor((c(y) - y0) * scale), 0, 32766) with
// c(y) = 0 for |y| < 2^-480, else y.  Every step (collapse, RN subtract, RN
// multiply by scale >= 0, clamp, floor) is monotone non-decreasing, so as for
// fkey: q(u) < q(v) => u < v.  The collapse keeps the product-underflow cases
// of the straddle test (both |y - p.y| < 2^-537, which forces all three values
// below 2^-484) on equal keys, i.e. they are never rejected.  y0/scale come
// from the outer ring's bbox (any values are correct; a tight range makes the
// filter sharp).
struct QMap {
    double y0, scale;
};

__device__ __forceinline__ double q_collapse(double y) { return fabs(y) < 0x1p-480 ? 0.0 : y; }

__device__ __forceinline__ QMap qmap_from_bbox(const unsigned long long* bbox_keys) {
    QMap m;
    const double lo = q_collapse(dkey_inv(bbox_keys[1])), hi = q_collapse(dkey_inv(~bbox_keys[3]));
    const double h = __dsub_rn(hi, lo);
    m.y0 = lo;
    m.scale = (h > 0.0 && h < 1e300) ? __ddiv_rn(32766.0, h) : 0.0; // degenerate: all keys equal
    if (!(lo == lo)) m.y0 = 0.0;                                     // empty outer ring
    return m;
}

// A map on an arbitrary y range [lo, hi] (pip_single.cu: the y range of a
// CTA's points), keeping every point key strictly inside the key range:
// y < lo -> 0, y > hi -> 32766, [lo, hi] -> 1 .. 32765.  So an edge that extends
// past the CTA's points on one side never ties with the extreme point there.
// Monotone non-decreasing (piecewise, each piece monotone and ordered), hence
// exact as a filter like qkey15.
struct CtaQMap {
    double y0, y1, scale;
};

__device__ __forceinline__ CtaQMap ctaqmap_from_range(double y_lo, double y_hi) {
    CtaQMap m;
    m.y0 = q_collapse(y_lo);
    m.y1 = q_collapse(y_hi);
    // the scale in binary32 (no binary64 division in the C1 kernels, rule P1's
    // SASS check): any non-negative scale gives a monotone map, and qkey_cta
    // clamps an overshoot; one y level or an extreme range: every point key is 1
    const double h = __dsub_rn(m.y1, m.y0);
    const float hf = __double2float_rn(h);
    m.scale = (h > 0.0 && hf >= 0x1p-100f && hf <= 0x1p100f) ? (double)__fdiv_rn(32764.0f, hf) : 0.0;
    return m;
}

__device__ __forceinline__ uint32_t qkey_cta(double y, const CtaQMap& m) {
    const double c = q_collapse(y);
    if (c < m.y0) return 0u;
    if (c > m.y1) return 32766u;
    double t = __dmul_rn(__dsub_rn(c, m.y0), m.scale);
    t = t < 32764.0 ? t : 32764.0; // also NaN-free: c, y0 finite and scale < inf
    return (uint32_t)t + 1u;
}

__device__ __forceinline__ uint32_t qkey15(double y, const QMap& m) {
    double t = __dmul_rn(__dsub_rn(q_collapse(y), m.y0), m.scale);
    t = t > 0.0 ? t : 0.0; // also maps a NaN product (0 * inf cannot occur: scale < inf) to 0
    t = t < 32766.0 ? t : 32766.0; // 32767 stays free: inactive points' key, never a candidate
    return (uint32_t)t;
}

// Polygon-local scaling of the C1 certified fp32 side test:
// local coordinate L = RN(v - o) * s with o = the outer ring's bbox min and s a
// power of two with W*s, H*s in [1/2, 1); valid when 2^-300 <= W, H <= 2^300
// (sx = sy = 0 otherwise).  A point inside the bbox and an edge with both
// endpoints inside get |s_fp32 - S'| <= 13.1 * 2^-24 against the reference's
// side scaled by sx*sy, so |s| > kLocalBand = 2^-20 decides its sign.
struct LocalMap {
    double x0, y0, sx, sy;
    bool c2ok; // C2 also needs max(|x|) * sx <= 2^20 (its reference error is ~u * |x|)
};
constexpr float kLocalBand = 0x1p-20f;

__device__ __forceinline__ double pow2_inv_above(double w) { // 2^-(E+1) for w in [2^E, 2^(E+1))
    const int e = (__double2hiint(w) >> 20) & 0x7ff;
    return __hiloint2double((2045 - e) << 20, 0);
}

__device__ __forceinline__ LocalMap local_map_from_bbox(const unsigned long long* bbox_keys) {
    LocalMap m;
    m.x0 = dkey_inv(bbox_keys[0]);
    m.y0 = dkey_inv(bbox_keys[1]);
    const double W = __dsub_rn(dkey_inv(~bbox_keys[2]), m.x0), H = __dsub_rn(dkey_inv(~bbox_keys[3]), m.y0);
    const bool ok = W >= 0x1p-300 && W <= 0x1p300 && H >= 0x1p-300 && H <= 0x1p300;
    m.sx = ok ? pow2_inv_above(W) : 0.0;
    m.sy = ok ? pow2_inv_above(H) : 0.0;
    const double mx = fmax(fabs(m.x0), fabs(dkey_inv(~bbox_keys[2])));
    m.c2ok = ok && __dmul_rn(mx, m.sx) <= 0x1p20;
    return m;
}

// Per-edge scaling of a record's normal by the power of two 2^k that puts
// max(|Nx|, |Ny|) in [1/2, 1) (exact; a zero normal stays zero).  Every fp32
// operation of the side test then scales by exactly 2^k, so its sign is
// unchanged, and the error bound of DESIGN.md §3.4 (derived for |Nx|, |Ny| <= 1)
// holds as it stands: the fixed band B = 2^-20 becomes relative to the edge's
// length instead of the polygon's size, so short edges (configs 2 and 4: local
// lengths down to ~1e-5) are decided in fp32 instead of falling into the band.
__device__ __forceinline__ void normalize_pow2(double& Nx, double& Ny) {
    const double M = fmax(fabs(Nx), fabs(Ny));
    if (M > 0.0 && M < 0.5) {
        const double k = pow2_inv_above(M); // M * k in [1/2, 1)
        Nx = __dmul_rn(Nx, k);
        Ny = __dmul_rn(Ny, k);
    }
}

// {Nx, Ny, c} of edge a->b with the reference's flipped normal (nx, ny); NaN
// when the map is off or an endpoint lies outside the bbox (a hole poking out)
__device__ __forceinline__ float3 local_side_record(const LocalMap& m, double ax, double ay, double bx, double by,
                                                    double nx, double ny) {
    const double axl = __dmul_rn(__dsub_rn(ax, m.x0), m.sx), ayl = __dmul_rn(__dsub_rn(ay, m.y0), m.sy);
    const double bxl = __dmul_rn(__dsub_rn(bx, m.x0), m.sx), byl = __dmul_rn(__dsub_rn(by, m.y0), m.sy);
    const bool ok = m.sx != 0.0 && axl >= 0.0 && axl < 1.0 && ayl >= 0.0 && ayl < 1.0 && bxl >= 0.0 && bxl < 1.0 &&
                    byl >= 0.0 && byl < 1.0;
    if (!ok) return make_float3(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000), __int_as_float(0x7fc00000));
    double Nx = __dmul_rn(nx, m.sy), Ny = __dmul_rn(ny, m.sx);
    normalize_pow2(Nx, Ny);
    const double cd = __dadd_rn(__dmul_rn(axl, Nx), __dmul_rn(ayl, Ny));
    // c + kLocalBand: the kernel's s' = s + B is then <= -0 (sign bit) for a sure
    // count and in [+0, 2B] for a band hit; the extra fp32 rounding of c + B
    // (<= 2 * 2^-24) keeps the total error at 15.1 * 2^-24 < B
    return make_float3(__double2float_rn(Nx), __double2float_rn(Ny),
                       __double2float_rn(__dadd_rn(-cd, (double)kLocalBand)));
}

// C2 (geometry.hpp:216-224): count iff x > p.x with x the reference's rounded
// intercept.  With X* = a.x + (p.y - a.y) * dx / dy (the rounded dx, dy),
// |x - X*| <= u*|a.x| + 4.03u*|dx| for a sure straddle (0 < lambda < 1), and
// (X* - p.x) * dy = -C with C = (p - a) x (dx, dy); so the local fp32 value of
// C * sign(dy), with N = sign(dy) * (dy * s_y, -dx * s_x), has the error of
// §3.4 plus at most u * (max|x| * s_x + 4.03) <= 2^-33 after scaling when
// max|x| * s_x <= 2^20: it is certified by the same band, and the count is
// its sign bit (s' = s + B as for C1).  NaN record when not usable.
__device__ __forceinline__ float3 local_side_record_c2(const LocalMap& m, double ax, double ay, double bx, double by,
                                                       double dx, double dy) {
    const double axl = __dmul_rn(__dsub_rn(ax, m.x0), m.sx), ayl = __dmul_rn(__dsub_rn(ay, m.y0), m.sy);
    const double bxl = __dmul_rn(__dsub_rn(bx, m.x0), m.sx), byl = __dmul_rn(__dsub_rn(by, m.y0), m.sy);
    const bool ok = m.c2ok && dy != 0.0 && axl >= 0.0 && axl < 1.0 && ayl >= 0.0 && ayl < 1.0 && bxl >= 0.0 &&
                    bxl < 1.0 && byl >= 0.0 && byl < 1.0;
    if (!ok) return make_float3(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000), __int_as_float(0x7fc00000));
    const double sg = dy > 0.0 ? 1.0 : -1.0;
    double Nx = __dmul_rn(__dmul_rn(dy, m.sy), sg), Ny = __dmul_rn(__dmul_rn(-dx, m.sx), sg);
    normalize_pow2(Nx, Ny);
    const double cd = __dadd_rn(__dmul_rn(axl, Nx), __dmul_rn(ayl, Ny));
    return make_float3(__double2float_rn(Nx), __double2float_rn(Ny),
                       __double2float_rn(__dadd_rn(-cd, (double)kLocalBand)));
}

// C1 exact test of one straddle candidate (geometry.hpp:189-200).  `sure`:
// the keys already prove min(a.y,b.y) < p.y < max(a.y,b.y) strictly, so the
// reference's product f_prev*f_next is negative (or -0) and `<= 0.0` holds;
// the product is only evaluated when a key tie leaves the order open.
__device__ __forceinline__ void exact_c1(double px, double py, const EdgeRec& r, int& cnt, bool sure = false) {
    const double ax = r.d[0], ay = r.d[1], by = r.d[2], nx = r.d[3], ny = r.d[4];
    if (sure || __dmul_rn(__dsub_rn(ay, py), __dsub_rn(by, py)) <= 0.0) {
        const double side = __dadd_rn(__dmul_rn(__dsub_rn(px, ax), nx), __dmul_rn(__dsub_rn(py, ay), ny));
        if (side <= 0.0) ++cnt;
    }
}

// C2 exact test (geometry.hpp:214-226); `err` marks the DegenerateEdge throw.
__device__ __forceinline__ void exact_c2(double px, double py, const EdgeRec& r, int& cnt, bool& err,
                                         bool sure = false) {
    const double ax = r.d[0], ay = r.d[1], by = r.d[2], dx = r.d[3], dy = r.d[4];
    if (sure || __dmul_rn(__dsub_rn(ay, py), __dsub_rn(by, py)) <= 0.0) {
        if (dy == 0.0) {
            err = true;
        } else {
            const double lambda = __ddiv_rn(__dsub_rn(py, ay), dy);
            const double x = __dadd_rn(ax, __dmul_rn(lambda, dx));
            if (x > px) ++cnt;
        }
    }
}

// Robust exact test (geometry.hpp:245-270); `bnd` marks on_boundary.
__device__ __forceinline__ void exact_robust(double px, double py, double tol, double tol2,
                                             const EdgeRec& r, int& cnt, bool& bnd) {
    const double ax = r.d[0], ay = r.d[1], by = r.d[2], abx = r.d[3], aby = r.d[4], len2 = r.d[5];
    const double ylo = by < ay ? by : ay; // std::min(a.y, b.y)
    const double yhi = ay < by ? by : ay; // std::max(a.y, b.y)
    if (__dadd_rn(py, tol) < ylo || __dsub_rn(py, tol) > yhi) return;
    const double apx = __dsub_rn(px, ax);
    const double apy = __dsub_rn(py, ay);
    double t = __ddiv_rn(__dadd_rn(__dmul_rn(apx, abx), __dmul_rn(apy, aby)), len2);
    t = (t < 0.0) ? 0.0 : ((1.0 < t) ? 1.0 : t); // std::clamp(t, 0.0, 1.0), NaN propagates
    const double dx = __dsub_rn(apx, __dmul_rn(t, abx));
    const double dyp = __dsub_rn(apy, __dmul_rn(t, aby));
    if (__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dyp, dyp)) <= tol2) {
        bnd = true;
        return;
    }
    const bool upward = ay <= py && py < by;
    const bool downward = by <= py && py < ay;
    if (upward || downward) {
        const double x = __dadd_rn(ax, __dmul_rn(__ddiv_rn(apy, aby), abx));
        if (x > px) ++cnt;
    }
}

// Literal per-edge step over raw vertices, for the CSR kernels and the count
// kernel (which walk rings directly).  `f_prev` carries b.y - p.y to the next
// edge exactly as the reference loop does.
template <int MODE>
__device__ __forceinline__ void raw_edge(double px, double py, double tol, double tol2, double ax,
                                         double ay, double bx, double by, double& f_prev, int& cnt,
                                         bool& aux) {
    if (MODE == kRobust) {
        const double ylo = by < ay ? by : ay;
        const double yhi = ay < by ? by : ay;
        if (__dadd_rn(py, tol) < ylo || __dsub_rn(py, tol) > yhi) return;
        const double abx = __dsub_rn(bx, ax), aby = __dsub_rn(by, ay);
        const double apx = __dsub_rn(px, ax), apy = __dsub_rn(py, ay);
        const double len2 = __dadd_rn(__dmul_rn(abx, abx), __dmul_rn(aby, aby));
        double t = __ddiv_rn(__dadd_rn(__dmul_rn(apx, abx), __dmul_rn(apy, aby)), len2);
        t = (t < 0.0) ? 0.0 : ((1.0 < t) ? 1.0 : t);
        const double dx = __dsub_rn(apx, __dmul_rn(t, abx));
        const double dyp = __dsub_rn(apy, __dmul_rn(t, aby));
        if (__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dyp, dyp)) <= tol2) {
            aux = true;
            return;
        }
        if ((ay <= py && py < by) || (by <= py && py < ay)) {
            const double x = __dadd_rn(ax, __dmul_rn(__ddiv_rn(apy, aby), abx));
            if (x > px) ++cnt;
        }
    } else {
        const double f_next = __dsub_rn(by, py);
        if (__dmul_rn(f_prev, f_next) <= 0.0) {
            if (MODE == kC1) {
                double nx = __dsub_rn(by, ay);
                double ny = __dsub_rn(ax, bx);
                if (nx < 0.0) {
                    nx = -nx;
                    ny = -ny;
                }
                const double side =
                    __dadd_rn(__dmul_rn(__dsub_rn(px, ax), nx), __dmul_rn(__dsub_rn(py, ay), ny));
                if (side <= 0.0) ++cnt;
            } else {
                const double dy = __dsub_rn(by, ay);
                if (dy == 0.0) {
                    aux = true;
                } else {
                    const double lambda = __ddiv_rn(__dsub_rn(py, ay), dy);
                    const double x = __dadd_rn(ax, __dmul_rn(lambda, __dsub_rn(bx, ax)));
                    if (x > px) ++cnt;
                }
            }
        }
        f_prev = f_next;
    }
}

} // namespace pcd
