// CSR batch kernel for C1 (the paper's side-of-normal test, configs 3 and 5)
// and C2 (parametric crossing): many small polygons, each with its own
// contiguous run of query points.
//
// Every warp works on its own: it takes a group of 32 consecutive polygons
// (lane = polygon), resolves their point / vertex / ring ranges, and then
// processes them in batches whose vertices fit its shared-memory slice
// (kWV vertices).  Per batch the warp
//   1. loads the batch's vertices into shared memory (lanes stride over the
//      batch's vertices, so a 10-vertex footprint does not leave 22 lanes
//      idle), and marks ring ends;
//   2. lane per polygon: the exact closed bbox of the outer ring with the
//      reference's std::min / std::max order (batch.hpp:121-133) and the
//      polygon-local scaling of the C1 fast path (pip_csr_common.cuh);
//   3. lanes stride over the vertices again: one fast-path record per edge;
//   4. classifies each polygon of the batch, 64 points per step (2 per lane):
//      ~9 instructions per (point, edge) pair; the rare undecided points (a
//      tie, or |s| within the band) re-run the polygon in binary64 in the
//      reference's expression order (geometry.hpp:182-203).
// No block-wide barriers: a warp waiting on its loads never holds up others.
// Polygons with more than kWV vertices are appended to a list and handled
// afterwards by the warp-per-polygon kernel (pip_csr.cu), which streams
// edges in chunks.
//
// Reference semantics per polygon: classify_batch(points_i, poly_i, mode)
// (batch.hpp:184-230) -> bbox short-circuit (batch.hpp:200) -> contains
// (geometry.hpp:281-300) -> count_crossings_c1 / _c2 over every ring; a C2
// DegenerateEdge (a horizontal edge on the ray) makes the point Error (aux
// plane).  C2 uses the same fast pass with the intercept-side record of
// pip_device.cuh local_side_record_c2 (gate: max|x| * s_x <= 2^20).
#include "pip_kernels.h"

#include <cuda_runtime.h>

#include <algorithm>

#include "pip_csr_common.cuh"
#include "pip_device.cuh"

namespace pcd {

namespace {

constexpr int kBThreads = 128;
constexpr int kBWarps = kBThreads / 32;
#ifndef PC_CSR_WV
#define PC_CSR_WV 96
#endif
#ifndef PC_CSR_WALK_NS
#define PC_CSR_WALK_NS 16
#endif
#ifndef PC_CSR_WALK_ROBUST
#define PC_CSR_WALK_ROBUST 1
#endif
#ifndef PC_CSR_MINB
#define PC_CSR_MINB 7
#endif
constexpr int kWV = PC_CSR_WV; // vertex budget of one batch (per warp)

struct BPoly {
    double bx0, by0, bx1, by1; // exact closed bbox of the outer ring
    double sx, sy;             // fast-path scaling (powers of two)
    unsigned long long s;      // first point (shard-local index)
    uint32_t np;               // points
    uint32_t e0, e1;           // vertex range in the batch
    uint32_t nloop;            // records the fast pass must visit (a closed single ring's
                               // last vertex repeats the first: its sentinel is skipped),
                               // bit 31: fast path usable
};

struct WarpSmem {
    double2 vert[kWV];
    // C1 / C2: rec = (K(a), Nx, Ny, c + B) with K the packed 14-bit key of the
    //          vertex (see classify_item), rec2 = (q_lo + 1, q_hi) on 30-bit keys
    //          (the exact path's candidate test);
    // Robust:  rec = (q_lo + 1, q_hi, q(a), Nx), rec2 = (Ny, c + B)
    int4 rec[kWV];
    int2 rec2[kWV];
    BPoly bp[32];
    unsigned long long v0s[32]; // first vertex (shard-local) of batch polygon k
    uint32_t off[32];           // batch offset of batch polygon k's first vertex
    uint32_t nvo[32];           // outer-ring vertices of batch polygon k
    uint32_t ring_end[kWV / 32]; // bit i: batch vertex i is the last vertex of its ring
    uint32_t starts[kWV / 32];   // bit i: batch vertex i is the first vertex of a batch polygon
    unsigned char owner[kWV];
    // the current group of 32 polygons (lane = polygon), kept here rather than
    // in registers across the batches
    unsigned long long gs[32], gr0[32], gv0[32];
    uint32_t gnp[32], gnr[32], gnv[32], gnvo[32];
};

__device__ __forceinline__ bool is_ring_end(const WarpSmem& ws, uint32_t i) {
    return (ws.ring_end[i >> 5] >> (i & 31)) & 1u;
}

// One step of a batch polygon: points cc .. cc+63 (2 per lane, already loaded
// into qc) against all of its edges.
// walk_all (warp-uniform): skip the fp32 pass and walk every candidate edge in
// binary64 -- cheaper when most points tie vertex keys anyway (returns the
// number of undecided points so the caller can pick the mode adaptively).
template <int MODE>
__device__ __forceinline__ int classify_item(const WarpSmem& ws, int j, uint32_t cc, const double2 (&qc)[2],
                                             int lane, const double2* __restrict__ pts,
                                             uint32_t* __restrict__ inside_bits, uint32_t* __restrict__ aux_bits,
                                             double tol, double tol2, bool walk_all) {
    const BPoly& tp = ws.bp[j];
    const uint32_t np = tp.np, e0 = tp.e0, e1 = tp.e1;
    const double bx0 = tp.bx0, by0 = tp.by0, bx1 = tp.bx1, by1 = tp.by1;
    const double sx = tp.sx, sy = tp.sy;
    const bool fast = tp.nloop >> 31;
    float lx[2], ly[2];
    int qy[2], qm[2], qp[2]; // keys of p.y; Robust: of RN(p.y - tol), RN(p.y + tol) (else = qy)
    uint32_t act = 0, qok = 0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const double2 q = qc[k];
        // classify_batch short-circuit (batch.hpp:200): outside the closed bbox -> Outside
        const bool a = cc + 32 * k + lane < np && q.x >= bx0 && q.x <= bx1 && q.y >= by0 && q.y <= by1;
        act |= (uint32_t)a << k;
        const double yl = __dmul_rn(__dsub_rn(q.y, by0), sy);
        lx[k] = __double2float_rn(__dmul_rn(__dsub_rn(q.x, bx0), sx));
        ly[k] = __double2float_rn(yl);
        if (MODE == kRobust) { // the band reject's own rounded values (geometry.hpp:248)
            qy[k] = __double2int_rz(__dmul_rn(yl, 0x1p30)); // = trunc((y - o_y) * s_y * 2^30): exact scaling
            qm[k] = __double2int_rz(__dmul_rn(__dmul_rn(__dsub_rn(__dsub_rn(q.y, tol), by0), sy), 0x1p30));
            qp[k] = __double2int_rz(__dmul_rn(__dmul_rn(__dsub_rn(__dadd_rn(q.y, tol), by0), sy), 0x1p30));
        } else {
            qy[k] = qm[k] = qp[k] = 0; // C1 / C2: the 30-bit key is formed on the exact path only
        }
        qok |= (uint32_t)(a && fast) << k;
    }
    // the key filters are exact only for |p.y| >= 2^-400 (pip_csr_common.cuh);
    // bit 30 of nloop: the polygon's whole closed bbox is clear of that range
    // (integer form: |y| >= 2^-400 iff the high word without its sign is >= 0x26f00000)
    if (!(tp.nloop >> 30 & 1u))
        qok &= (uint32_t)((__double2hiint(qc[0].y) & 0x7fffffff) >= 0x26f00000) |
               ((uint32_t)((__double2hiint(qc[1].y) & 0x7fffffff) >= 0x26f00000) << 1);
    if (!__any_sync(kFull, act != 0)) return 0;
    uint32_t par = 0, slow = act & ~qok, band = 0, err = 0;
    if (fast && walk_all) {
        slow = act;
        band = act; // every candidate edge of every point
    } else if (fast && MODE != kRobust) {
        // Packed pass, both points of the lane in one 32-bit word per quantity.
        // Keys: k(y) = bits 8..21 of RN32(RN32(y_local) * 0.5 + 1) -- a monotone
        // 14-bit function of y, the same for points and vertices.  Q holds
        // (k0 << 1 | 1) and (k1 << 1 | 1) in its halves, K(v) holds k(v) << 1 in
        // both; in d = Q - K the half of point j has its sign bit (15 / 31) set
        // iff k_j < k(v) (the low half's borrow only clears the high half's guard
        // bit), and the half is 0 or 1 iff k_j == k(v) (a tie).  With no tie,
        // edge a -> b surely straddles iff the sign bits of d(a) and d(b) differ
        // (strict: k(a) < k < k(b) => a.y < p.y < b.y), and surely does not iff
        // they agree (both ends strictly above / below; the product cannot
        // underflow since |p.y| >= 2^-400).  The side test's s' = s + B as in the
        // Robust branch below; its high halves of both points are packed into P
        // (sign bits 15 / 31), so (d(a) ^ d(b)) & P toggles the parity bits.
        // A point with a tie or a band hit (P half <= 0x3600, i.e. 0 <= s' <
        // 2B (1 + 2^-7)) is decided by the exact path instead.
        const uint32_t t0 = __float_as_uint(fmaf(ly[0], 0.5f, 1.0f)), t1 = __float_as_uint(fmaf(ly[1], 0.5f, 1.0f));
        const uint32_t Q = ((t0 >> 7) & 0x7ffeu) | ((t1 << 9) & 0x7ffe0000u) | 0x00010001u;
        uint32_t acc = 0u, tm = 0xffffffffu, bm = 0xffffffffu;
        const uint32_t dfirst = Q - (uint32_t)ws.rec[e0].x;
        uint32_t dprev = dfirst, pprev = 0u;
        // both points' local coordinates as packed pairs: one FFMA2 per term and
        // record serves the two points (each half an IEEE fmaf: the same values)
        const unsigned long long LX = f32x2(lx[0], lx[1]), LY = f32x2(ly[0], ly[1]);
        // every stored vertex of the polygon (a ring's last vertex carries the
        // no-toggle sentinel record) -- except a closed single ring's last vertex,
        // which repeats the first: its edge closes with d(first) below.  Two
        // records per iteration; an odd count re-reads the last record as the
        // second (d ^ d = 0: no toggle, the same tie / band values).
        const uint32_t stop = e0 + (tp.nloop & 0x3fffffffu), last = stop - 1u;
        for (uint32_t i = e0; i < stop; i += 2) {
            const int4 fi = ws.rec[i], fj = ws.rec[min(i + 1u, last)];
            const uint32_t di = Q - (uint32_t)fi.x, dj = Q - (uint32_t)fj.x;
            const uint32_t pi = hi16x2(ffma2_b(LX, __int_as_float(fi.y), ffma2_bb(LY, __int_as_float(fi.z), __int_as_float(fi.w))));
            const uint32_t pj = hi16x2(ffma2_b(LX, __int_as_float(fj.y), ffma2_bb(LY, __int_as_float(fj.z), __int_as_float(fj.w))));
            acc ^= ((dprev ^ di) & pprev) ^ ((di ^ dj) & pi);
            tm = __vimin3_u16x2(tm, di, dj);
            bm = __vimin3_u16x2(bm, pi, pj);
            dprev = dj;
            pprev = pj;
        }
        acc ^= (dprev ^ dfirst) & pprev; // the closing edge (a sentinel's pprev is +: no toggle)
        const uint32_t fpar = (acc >> 15 & 1u) | (acc >> 30 & 2u);
        band = ((uint32_t)((bm & 0xffffu) <= 0x3600u) | ((uint32_t)((bm >> 16) <= 0x3600u) << 1) |
                (uint32_t)((tm & 0xffffu) <= 1u) | ((uint32_t)((tm >> 16) <= 1u) << 1)) & act;
        slow |= band;
        par = fpar & qok & ~band;
    } else if (fast) {
        // per record and point: x = q - q_hi < 0 and y = q - (q_lo + 1) >= 0 iff
        // q_lo < q < q_hi (a sure straddle); s' = s + B (B folded into the
        // record's offset) has its sign bit set iff the side test counts, so the
        // sign bit of x & ~y & s' toggles the parity; +0 <= s' <= 2B is a band hit
        int acc0 = 0, acc1 = 0;
        uint32_t t0 = 0xffffffffu, t1 = 0xffffffffu, u0 = 0xffffffffu, u1 = 0xffffffffu;
        const unsigned long long LX = f32x2(lx[0], lx[1]), LY = f32x2(ly[0], ly[1]);
        auto rec = [&](uint32_t i) {
            const int4 f = ws.rec[i];
            const int2 g = ws.rec2[i];
            // both points in one FFMA2 per term (each half an IEEE fmaf)
            const unsigned long long s = ffma2_b(LX, __int_as_float(f.w), ffma2_bb(LY, __int_as_float(g.x), __int_as_float(g.y)));
            const float s0 = __uint_as_float((uint32_t)s), s1 = __uint_as_float((uint32_t)(s >> 32));
            acc0 ^= (qp[0] - f.y) & ~(qm[0] - f.x) & __float_as_int(s0);
            acc1 ^= (qp[1] - f.y) & ~(qm[1] - f.x) & __float_as_int(s1);
            u0 = min(u0, __float_as_uint(s0)); // band hits
            u1 = min(u1, __float_as_uint(s1));
            t0 = min(t0, (unsigned)(f.z - qm[0])); // ties: a vertex key in [qm, qp]
            t1 = min(t1, (unsigned)(f.z - qm[1]));
        };
        // four records per iteration; reads past the polygon's last record
        // re-read it (the final vertex's sentinel: no toggle, no band hit, a
        // repeated tie check), so no remainder loop is needed
        const uint32_t last = e1 - 1u, stop = e0 + (tp.nloop & 0x3fffffffu);
        uint32_t i = e0;
        for (; i + 4 <= stop; i += 4) { // whole groups: consecutive records, fixed offsets
#pragma unroll
            for (int k = 0; k < 4; ++k) rec(i + k);
        }
        if (i < stop) { // the remainder, clamped
#pragma unroll
            for (int k = 0; k < 4; ++k) rec(min(i + k, last));
        }
        constexpr uint32_t k2B = 0x36000000u; // bits of 2^-19 = 2 * kFastBand
        const uint32_t fpar = ((uint32_t)acc0 >> 31) | (((uint32_t)acc1 >> 31) << 1);
        band = ((uint32_t)(u0 <= k2B) | ((uint32_t)(u1 <= k2B) << 1)) & act;
        const uint32_t tie =
            ((uint32_t)(t0 <= (unsigned)(qp[0] - qm[0])) | ((uint32_t)(t1 <= (unsigned)(qp[1] - qm[1])) << 1)) & act;
        slow |= band | tie;
        // decided contributions (ties never toggle fpar); points with a band hit
        // redo every candidate edge
        par = fpar & qok & ~band;
    }
    int ns = 0; // undecided points of the step (the caller's adaptive mode)
    if (__any_sync(kFull, slow != 0)) {
        ns = __popc(__ballot_sync(kFull, slow & 1u)) + __popc(__ballot_sync(kFull, slow >> 1 & 1u));
        // exact binary64 path, count_crossings_c1 (geometry.hpp:182-203), on the
        // undecided (point, edge) pairs: a point with only key ties redoes the
        // edges whose key range it ties (q == q_lo or q == q_hi); a point with a
        // band hit redoes every candidate edge (q_lo <= q <= q_hi); a point whose
        // key filter is not exact redoes every edge
        const double2* P = pts + tp.s;
        double px[2], py[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const double2 q = (slow >> k & 1u) ? P[cc + 32 * k + lane] : make_double2(0.0, 0.0);
            px[k] = q.x;
            py[k] = q.y;
        }
        // one selection rule per warp: if any point has a band hit, every
        // undecided point redoes all its candidate edges (and drops fpar)
        // a slow point redoes every candidate edge (C1 / C2: 30-bit keys formed here)
        par &= ~slow;
        if (MODE != kRobust) {
#pragma unroll
            for (int k = 0; k < 2; ++k) qy[k] = __double2int_rz(__dmul_rn(__dmul_rn(__dsub_rn(py[k], by0), sy), 0x1p30));
        }
        const int qy1[2] = {qy[0] + 1, qy[1] + 1};
        for (uint32_t i0 = e0; i0 < e1; i0 += 32) {
            const int n = (int)min(32u, e1 - i0);
            // real edges of the chunk: not a ring's last vertex, inside the chunk
            const uint32_t w = i0 >> 5, sh = i0 & 31;
            uint32_t ends = ws.ring_end[w] >> sh;
            if (sh && w + 1 < (uint32_t)(kWV / 32)) ends |= ws.ring_end[w + 1] << (32 - sh);
            const uint32_t real = ~ends & (n == 32 ? 0xffffffffu : ((1u << n) - 1u));
            uint32_t cm0 = 0u, cm1 = 0u;
            // record: f.x = q_lo + 1, f.y = q_hi
            if (MODE == kRobust) { // edges the band reject may keep: q_lo <= q(RN(p.y + tol)), q(RN(p.y - tol)) <= q_hi
                for (int u = n - 1; u >= 0; --u) {
                    const int2 f = *reinterpret_cast<const int2*>(&ws.rec[i0 + u]);
                    cm0 = (cm0 << 1) | (uint32_t)(((qp[0] + 1 - f.x) | (f.y - qm[0])) >= 0);
                    cm1 = (cm1 << 1) | (uint32_t)(((qp[1] + 1 - f.x) | (f.y - qm[1])) >= 0);
                }
            } else { // C1 / C2: q_lo <= q <= q_hi (rec2 = (q_lo + 1, q_hi))
                for (int u = n - 1; u >= 0; --u) {
                    const int2 f = ws.rec2[i0 + u];
                    const unsigned r = (unsigned)(f.y - f.x + 1);
                    cm0 = (cm0 << 1) | (uint32_t)((unsigned)(qy1[0] - f.x) <= r);
                    cm1 = (cm1 << 1) | (uint32_t)((unsigned)(qy1[1] - f.x) <= r);
                }
            }
            // points whose key filter is not exact: every edge
            cm0 = (slow & 1u) ? real & ((qok & 1u) ? cm0 : 0xffffffffu) : 0u;
            cm1 = (slow & 2u) ? real & ((qok & 2u) ? cm1 : 0xffffffffu) : 0u;
            // walk both points' undecided edges side by side
            while (__any_sync(kFull, (cm0 | cm1) != 0)) {
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    uint32_t& m = k ? cm1 : cm0;
                    if (m == 0) continue;
                    const uint32_t i = i0 + __ffs(m) - 1;
                    m &= m - 1;
                    PC_DCHECK(i + 1 < e1 && i >= e0);
                    const double2 a = ws.vert[i], b = ws.vert[i + 1];
                    if (MODE == kRobust) { // robust_ray_crossings (geometry.hpp:242-270), literally
                        int c = 0;
                        bool bnd = false;
                        double f_prev = 0.0; // unused by the Robust step
                        raw_edge<kRobust>(px[k], py[k], tol, tol2, a.x, a.y, b.x, b.y, f_prev, c, bnd);
                        if (c) par ^= 1u << k;
                        if (bnd) err |= 1u << k; // Boundary
                    } else if (__dmul_rn(__dsub_rn(a.y, py[k]), __dsub_rn(b.y, py[k])) <= 0.0) {
                        if (MODE == kC1) { // count_crossings_c1 (geometry.hpp:189-200)
                            double nx = __dsub_rn(b.y, a.y), ny = __dsub_rn(a.x, b.x);
                            if (nx < 0.0) {
                                nx = -nx;
                                ny = -ny;
                            }
                            const double side =
                                __dadd_rn(__dmul_rn(__dsub_rn(px[k], a.x), nx), __dmul_rn(__dsub_rn(py[k], a.y), ny));
                            if (side <= 0.0) par ^= 1u << k;
                        } else { // count_crossings_c2 (geometry.hpp:216-224)
                            const double dy = __dsub_rn(b.y, a.y);
                            if (dy == 0.0) {
                                err |= 1u << k; // DegenerateEdge
                            } else {
                                const double lambda = __ddiv_rn(__dsub_rn(py[k], a.y), dy);
                                const double x = __dadd_rn(a.x, __dmul_rn(lambda, __dsub_rn(b.x, a.x)));
                                if (x > px[k]) par ^= 1u << k;
                            }
                        }
                    }
                }
            }
        }
    }
    const uint32_t b0 = __ballot_sync(kFull, act & par & ~err & 1u);
    const uint32_t b1 = __ballot_sync(kFull, (act & par & ~err) >> 1 & 1u);
    or_bits64(inside_bits, tp.s + cc, b0, b1, lane);
    if (MODE != kC1 && __any_sync(kFull, err != 0)) { // C2: Error (DegenerateEdge), Robust: Boundary
        const uint32_t e0 = __ballot_sync(kFull, act & err & 1u);
        const uint32_t e1 = __ballot_sync(kFull, (act & err) >> 1 & 1u);
        or_bits64(aux_bits, tp.s + cc, e0, e1, lane);
    }
    return ns;
}

template <int MODE>
__global__ void __launch_bounds__(kBThreads, PC_CSR_MINB) pip_csr_tile_kernel(
    const double2* __restrict__ pts, const unsigned long long* __restrict__ pt_off, unsigned long long n_polys,
    const double* __restrict__ vx, const double* __restrict__ vy, const unsigned long long* __restrict__ ring_off,
    const unsigned long long* __restrict__ poly_ring_off, unsigned long long pt_base, unsigned long long ring_base,
    unsigned long long vert_base, double tol, double tol2, uint32_t* __restrict__ inside_bits,
    uint32_t* __restrict__ aux_bits, uint32_t* __restrict__ defer_list, uint32_t* __restrict__ defer_count) {
    __shared__ WarpSmem smem[kBWarps];
    const int lane = threadIdx.x & 31;
    WarpSmem& ws = smem[threadIdx.x >> 5];
    const unsigned long long nw = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    const unsigned long long ngroups = (n_polys + 31) / 32;

    int walk_left = 0; // adaptive mode of classify_item (warp-uniform)
    for (unsigned long long g = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < ngroups; g += nw) {
        // ---- ranges: lane = polygon g*32 + lane --------------------------------
        const unsigned long long p = g * 32 + lane;
        unsigned long long s = 0, e = 0, r0 = 0, r1 = 0, v0 = 0, vo1 = 0, vend = 0;
        if (p < n_polys) {
            s = pt_off[p] - pt_base;
            e = pt_off[p + 1] - pt_base;
            r0 = poly_ring_off[p] - ring_base;
            r1 = poly_ring_off[p + 1] - ring_base;
            v0 = ring_off[r0] - vert_base;
            vend = ring_off[r1] - vert_base;
            vo1 = r1 > r0 ? ring_off[r0 + 1] - vert_base : v0;
        }
        // no points or no rings: nothing to classify (no rings -> nothing is inside;
        // no vertices: an empty outer ring has an empty bbox -> nothing is inside)
        const bool work = p < n_polys && e > s && r1 > r0 && vend > v0;
        const bool big = work && vend - v0 > (unsigned long long)kWV;
        if (big) defer_list[atomicAdd(defer_count, 1u)] = (uint32_t)p;
        ws.gs[lane] = s;
        ws.gr0[lane] = r0;
        ws.gv0[lane] = v0;
        ws.gnp[lane] = (uint32_t)(e - s);
        ws.gnr[lane] = (uint32_t)(r1 - r0);
        ws.gnv[lane] = work && !big ? (uint32_t)(vend - v0) : 0u;
        ws.gnvo[lane] = (uint32_t)(vo1 - v0);
        uint32_t todo = __ballot_sync(kFull, work && !big);
        while (todo) {
            // ---- batch: a prefix of the remaining polygons that fits kWV ----------
            const uint32_t nv = ws.gnv[lane];
            const uint32_t mine = (todo >> lane & 1u) ? nv : 0u;
            uint32_t cum = mine;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, cum, o);
                if (lane >= o) cum += y;
            }
            const uint32_t batch = todo & __ballot_sync(kFull, cum <= (uint32_t)kWV);
            const int nb = __popc(batch);
            const bool inb = batch >> lane & 1u;
            const uint32_t excl = cum - mine;
            const int k = __popc(batch & ((1u << lane) - 1u)); // compact index of this lane's polygon
            const uint32_t total = __shfl_sync(kFull, cum, 31 - __clz(batch));
            if (lane < kWV / 32) ws.ring_end[lane] = ws.starts[lane] = 0u;
            __syncwarp();
            if (inb) {
                ws.off[k] = excl;
                ws.nvo[k] = ws.gnvo[lane];
                ws.v0s[k] = ws.gv0[lane];
                atomicOr(&ws.starts[excl >> 5], 1u << (excl & 31)); // distinct: every batch polygon has >= 1 vertex
            }
            __syncwarp();
            if (inb) { // ring ends
                const unsigned long long r0 = ws.gr0[lane], r1 = r0 + ws.gnr[lane], v0 = ws.gv0[lane];
                if (r1 - r0 == 1) {
                    atomicOr(&ws.ring_end[(excl + nv - 1) >> 5], 1u << ((excl + nv - 1) & 31));
                } else {
                    for (unsigned long long r = r0; r < r1; ++r) {
                        const uint32_t i = excl + (uint32_t)(ring_off[r + 1] - vert_base - v0) - 1u;
                        atomicOr(&ws.ring_end[i >> 5], 1u << (i & 31));
                    }
                }
            }
            // ---- 1. vertices -> shared memory ------------------------------------
#pragma unroll
            for (int u = 0; u < kWV / 32; ++u) {
                const uint32_t i = lane + 32 * u;
                if (i < total) {
                    PC_DCHECK(i < (uint32_t)kWV);
                    // owner: the last batch polygon whose first vertex is <= i
                    int o = __popc(ws.starts[u] & (0xffffffffu >> (31 - lane))) - 1;
#pragma unroll
                    for (int w = 0; w < u; ++w) o += __popc(ws.starts[w]);
                    PC_DCHECK(o >= 0 && o < nb);
                    ws.owner[i] = (unsigned char)o;
                    const unsigned long long v = ws.v0s[o] + (i - ws.off[o]);
                    ws.vert[i] = make_double2(vx[v], vy[v]);
                }
            }
            __syncwarp();
            // ---- 2. bbox of the outer ring and scaling --------------------------------
            {
                // 2^floor(log2(32 / nb)) lanes per polygon, each a strided part of the
                // outer ring, then a butterfly.  The reference's std::min / std::max
                // (batch.hpp:121-133) pick the first of equal values; the only equal
                // but distinguishable values are +0 / -0, which compare equal in the
                // prefilter and give the same fast-path keys and signs (a zero origin
                // only flips the sign of exact zero local coordinates).
                const int lg = 31 - __clz(32 / nb);
                const int kk = lane >> lg, sub = lane & ((1 << lg) - 1);
                double bx0 = INFINITY, by0 = INFINITY, bx1 = -INFINITY, by1 = -INFINITY;
                if (kk < nb) {
                    const uint32_t st = ws.off[kk], en = st + ws.nvo[kk];
                    for (uint32_t i = st + sub; i < en; i += 1u << lg) {
                        const double2 q = ws.vert[i];
                        bx0 = q.x < bx0 ? q.x : bx0; // std::min(min_x, v.x)
                        by0 = q.y < by0 ? q.y : by0;
                        bx1 = bx1 < q.x ? q.x : bx1; // std::max(max_x, v.x)
                        by1 = by1 < q.y ? q.y : by1;
                    }
                }
                for (int o = 1; o < (1 << lg); o <<= 1) {
                    const double x0 = __shfl_xor_sync(kFull, bx0, o), y0 = __shfl_xor_sync(kFull, by0, o);
                    const double x1 = __shfl_xor_sync(kFull, bx1, o), y1 = __shfl_xor_sync(kFull, by1, o);
                    bx0 = x0 < bx0 ? x0 : bx0;
                    by0 = y0 < by0 ? y0 : by0;
                    bx1 = bx1 < x1 ? x1 : bx1;
                    by1 = by1 < y1 ? y1 : by1;
                }
                if (kk < nb && sub == 0) {
                    ws.bp[kk].bx0 = bx0;
                    ws.bp[kk].by0 = by0;
                    ws.bp[kk].bx1 = bx1;
                    ws.bp[kk].by1 = by1;
                }
            }
            __syncwarp();
            if (inb) {
                BPoly& b = ws.bp[k];
                const double bx0 = b.bx0, by0 = b.by0, bx1 = b.bx1, by1 = b.by1;
                const double W = __dsub_rn(bx1, bx0), H = __dsub_rn(by1, by0);
                bool fast = W >= 0x1p-300 && W <= 0x1p300 && H >= 0x1p-300 && H <= 0x1p300;
                b.sx = fast ? pow2_below_inv(W) : 1.0;
                b.sy = fast ? pow2_below_inv(H) : 1.0;
                // C2 / Robust: the reference's intercept rounding scales with |x|
                // (pip_device.cuh local_side_record_c2)
                if (MODE != kC1) fast = fast && __dmul_rn(fmax(fabs(bx0), fabs(bx1)), b.sx) <= 0x1p20;
                // Robust: a decided sign must also rule out the boundary -- the point is
                // then >= 0.64 * 2^-24 / max(s_x, s_y) from the edge's line,
                // >= 2.5 tol under this gate
                if (MODE == kRobust)
                    fast = fast && tol >= 0.0 && __dmul_rn(__dmul_rn(tol, 2.0), fmax(b.sx, b.sy)) <= 0x1p-25;
                b.s = ws.gs[lane];
                b.np = ws.gnp[lane];
                b.e0 = excl;
                b.e1 = excl + nv;
                const double2 vf = ws.vert[excl], vl = ws.vert[excl + nv - 1];
                b.nloop = (ws.gnr[lane] == 1 && nv > 1 && vf.x == vl.x && vf.y == vl.y ? nv - 1 : nv) |
                          ((uint32_t)fast << 31) | ((uint32_t)(by0 >= 0x1p-400 || by1 <= -0x1p-400) << 30);
            }
            __syncwarp();
            // ---- 3. fast-path record per edge -----------------------------------
            for (uint32_t i = lane; i < total; i += 32) {
                const int o = ws.owner[i];
                const double bx0 = ws.bp[o].bx0, by0 = ws.bp[o].by0;
                const double sx = ws.bp[o].sx, sy = ws.bp[o].sy;
                const double2 a = ws.vert[i];
                const double axl = __dmul_rn(__dsub_rn(a.x, bx0), sx), ayl = __dmul_rn(__dsub_rn(a.y, by0), sy);
                const int qa = __double2int_rz(__dmul_rn(ayl, 0x1p30));
                if (!(axl >= 0.0 && axl < 1.0 && ayl >= 0.0 && ayl < 1.0)) atomicAnd(&ws.bp[o].nloop, 0x7fffffffu); // a hole poking out
                // C1 / C2: the packed 14-bit key of the vertex (classify_item)
                const uint32_t kt = (__float_as_uint(fmaf(__double2float_rn(ayl), 0.5f, 1.0f)) >> 8) & 0x3fffu;
                const int kv = (int)((kt << 1) | (kt << 17));
                int4 f = MODE == kRobust ? make_int4(kFastSentinelLo, 0, qa, 0)
                                         : make_int4(kv, 0, 0, __float_as_int(1.f));
                int2 gg = MODE == kRobust ? make_int2(0, __float_as_int(1.f)) : make_int2(kFastSentinelLo, 0);
                if (!is_ring_end(ws, i)) {
                    PC_DCHECK(i + 1 < total);
                    const double2 b = ws.vert[i + 1];
                    const int qb = __double2int_rz(__dmul_rn(__dmul_rn(__dsub_rn(b.y, by0), sy), 0x1p30));
                    double Nx, Ny;
                    if (MODE == kC1) { // the reference's normal (geometry.hpp:190-195)
                        double nx = __dsub_rn(b.y, a.y), ny = __dsub_rn(a.x, b.x);
                        if (nx < 0.0) {
                            nx = -nx;
                            ny = -ny;
                        }
                        Nx = __dmul_rn(nx, sy);
                        Ny = __dmul_rn(ny, sx);
                    } else { // C2: sign(dy) * (dy, -dx): the count is the sign of C * sign(dy) < 0
                        const double dy = __dsub_rn(b.y, a.y), dx = __dsub_rn(b.x, a.x);
                        const double sg = dy > 0.0 ? 1.0 : -1.0;
                        Nx = __dmul_rn(__dmul_rn(dy, sy), sg);
                        Ny = __dmul_rn(__dmul_rn(-dx, sx), sg);
                    }
                    const int qlo = min(qa, qb), qhi = max(qa, qb);
                    const double cd = __dadd_rn(__dmul_rn(axl, Nx), __dmul_rn(ayl, Ny));
                    // offset c + B (see classify_item): the extra fp32 rounding (<= 2 * 2^-24)
                    // keeps the error at 15.1 * 2^-24 < B
                    const float nxf = __double2float_rn(Nx), nyf = __double2float_rn(Ny);
                    const float cf = __double2float_rn(__dadd_rn(-cd, (double)kFastBand));
                    if (MODE == kRobust) {
                        f = make_int4(qlo + 1, qhi, qa, __float_as_int(nxf));
                        gg = make_int2(__float_as_int(nyf), __float_as_int(cf));
                    } else {
                        f = make_int4(kv, __float_as_int(nxf), __float_as_int(nyf), __float_as_int(cf));
                        gg = make_int2(qlo + 1, qhi);
                    }
                }
                ws.rec[i] = f;
                ws.rec2[i] = gg;
            }
            __syncwarp();
            // ---- 4. classify the batch's polygons ---------------------------------
            // items (polygon j, points c..c+63) in order; the points of the next
            // item are loaded while the current one is classified
            int j = 0;
            uint32_t c = 0;
            double2 qn0, qn1;
            auto load = [&](int jj, uint32_t cc, double2& a0, double2& a1) {
                // past the polygon's last point: re-read it (such lanes are inactive)
                const uint32_t n1 = ws.bp[jj].np - 1u;
                const double2* P = pts + ws.bp[jj].s;
                a0 = P[min(cc + lane, n1)];
                a1 = P[min(cc + 32 + lane, n1)];
            };
            load(0, 0, qn0, qn1);
            while (j < nb) {
                const double2 qc[2] = {qn0, qn1};
                const int cj = j;
                const uint32_t cc = c;
                c += 64;
                if (c >= ws.bp[j].np) {
                    c = 0;
                    ++j;
                }
                if (j < nb) load(j, c, qn0, qn1);
                const int ns =
                    classify_item<MODE>(ws, cj, cc, qc, lane, pts, inside_bits, aux_bits, tol, tol2, walk_left > 0);
                // mode choice: after an fp32 pass that left >= 1/4 of the points
                // undecided, walk everything for the next 16 steps, then probe again
                if (walk_left > 0) --walk_left;
                else if (ns >= PC_CSR_WALK_NS && (MODE != kRobust || PC_CSR_WALK_ROBUST)) walk_left = 16;
            }
            __syncwarp(); // the next batch rewrites this warp's shared slice
            todo &= ~batch;
        }
    }
}

int sms(int dev) {
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
}

} // namespace

namespace {

template <int MODE>
cudaError_t launch_tile(const CsrArgs& a, uint32_t* list, uint32_t* count, cudaStream_t st, int dev,
                        uint64_t* launches) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pip_csr_tile_kernel<MODE>, kBThreads, 0);
    per_sm = std::max(per_sm, 1);
    const uint64_t ngroups = (a.n_polys + 31) / 32;
    const uint64_t want = (ngroups + kBWarps - 1) / kBWarps;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)sms(dev) * per_sm));
    pip_csr_tile_kernel<MODE><<<grid, kBThreads, 0, st>>>(
        reinterpret_cast<const double2*>(a.pts), reinterpret_cast<const unsigned long long*>(a.pt_off), a.n_polys,
        a.vx, a.vy, reinterpret_cast<const unsigned long long*>(a.ring_off),
        reinterpret_cast<const unsigned long long*>(a.poly_ring_off), a.pt_base, a.ring_base, a.vert_base,
        a.tol, a.tol2, a.inside_bits, a.aux_bits, list, count);
    ++*launches;
    return cudaGetLastError();
}

} // namespace

cudaError_t launch_csr_tile(const CsrArgs& a, uint32_t* list, uint32_t* count, cudaStream_t st, int dev,
                            uint64_t* launches) {
    if (a.n_polys > 0xffffffffull) return cudaErrorInvalidValue; // 32-bit deferred-polygon list
    if (a.mode == kC2) return launch_tile<kC2>(a, list, count, st, dev, launches);
    if (a.mode == kRobust) return launch_tile<kRobust>(a, list, count, st, dev, launches);
    return launch_tile<kC1>(a, list, count, st, dev, launches);
}

} // namespace pcd
