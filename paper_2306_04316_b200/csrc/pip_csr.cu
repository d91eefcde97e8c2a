// CSR multi-polygon kernel (configs 3 and 5): many small
// polygons, each with its own contiguous run of query points.
//
// A metadata prepass (csr_meta_kernel, one thread per polygon) resolves each
// polygon's point / vertex / ring ranges and the exact bbox of its outer ring.
// Then one warp per polygon (grid-stride, next polygon's record prefetched):
//   1. reads the polygon's 80-byte metadata record (uniform loads);
//   2. walks its points 64 at a time (2 per lane) and, for each chunk of up to
//      31 edges, loads the chunk's 32 vertices (one per lane), derives the
//      per-edge data (filter keys, normal / direction) lane-parallel into a
//      per-warp shared-memory scratch; then (a) the integer key filter builds,
//      per point, a bitmask of candidate edges, and (b) every lane walks its
//      own candidate edges (ffs loop) running the reference's binary64 test --
//      the warp iterates max-popcount (~2-4 for footprints) times, not once
//      per edge, so the FP64 work follows the candidates, not the SIMT width;
//   3. masks the result with the closed bbox of the outer ring -- points
//      outside it are Outside with no Error / Boundary, exactly as
//      classify_batch's short-circuit (batch.hpp:200);
//   4. ORs one ballot word per 32 points into the bit planes.
//
// Reference semantics per polygon: classify_batch(points_i, poly_i, mode)
// (batch.hpp:184-230) -> contains (geometry.hpp:281-300) ->
// count_crossings_c1/_c2 / robust_ray_crossings (geometry.hpp:182-273).
#include "pip_kernels.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>

#include "pip_csr_common.cuh"
#include "pip_device.cuh"

namespace pcd {

namespace {

constexpr int kCsrThreads = 256;
constexpr int kWarps = kCsrThreads / 32;
constexpr int kNoEdge = 0x7ffffffe; // klo of a ring seam: no point key equals it

struct __align__(16) EdgeScratch { // one warp's current chunk of <= 31 edges
    int2 kr[32];                     // (klo, C1/C2: khi-klo | Robust: khi)
    double2 a[32];                   // (a.x, a.y)
    double2 q[32];                   // C1 (nx, ny) | C2 (dx, dy) | Robust (abx, aby)
    double by[32];
    double len2[32];                 // Robust only
    int4 fr[32];                     // C1 fast path: (qlo+1, max(qhi-qlo-1,0), q(a), Nx)
    float2 fr2[32];                  //               (Ny, c)
};

// Per-polygon metadata, one thread per polygon (csr_meta_kernel): the exact
// closed bbox of the outer ring (batch.hpp:121-133, std::min/std::max order)
// and the resolved point / vertex / ring ranges.  A thread per polygon costs
// ~1/32 of a warp per polygon, so the classify kernel's warps start straight
// at the points and edges.
struct __align__(16) PolyMeta {
    double bx0, by0, bx1, by1;        // empty outer ring: +inf/-inf (nothing inside)
    unsigned long long s;             // first point (local index)
    unsigned long long v0;            // first vertex (local index)
    unsigned long long r0;            // first ring (local index)
    uint32_t np, nv, nvo, nr;         // points, vertices (all rings), outer-ring vertices, rings
};

// list == nullptr: record k describes polygon k (k < n_polys); otherwise
// record k describes polygon list[k] for k < *count (the polygons of the tiles
// the C1 tile kernel deferred, see pip_csr_tile.cu).
__global__ void __launch_bounds__(256) csr_meta_kernel(
    const unsigned long long* __restrict__ pt_off, unsigned long long n_polys, const double* __restrict__ vx,
    const double* __restrict__ vy, const unsigned long long* __restrict__ ring_off,
    const unsigned long long* __restrict__ poly_ring_off, unsigned long long pt_base, unsigned long long ring_base,
    unsigned long long vert_base, PolyMeta* __restrict__ meta, const uint32_t* __restrict__ list,
    const uint32_t* __restrict__ count) {
    const unsigned long long n = count ? min((unsigned long long)*count, n_polys) : n_polys;
    for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; k < n;
         k += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long p = list ? list[k] : k;
        PolyMeta m;
        const unsigned long long s = pt_off[p] - pt_base, t = pt_off[p + 1] - pt_base;
        const unsigned long long r0 = poly_ring_off[p] - ring_base, r1 = poly_ring_off[p + 1] - ring_base;
        m.s = s;
        m.r0 = r0;
        m.np = (uint32_t)(t - s);
        m.nr = (uint32_t)min(r1 - r0, 0xffffffffull);
        m.bx0 = m.by0 = INFINITY;
        m.bx1 = m.by1 = -INFINITY;
        m.v0 = 0;
        m.nv = m.nvo = 0;
        if (r1 > r0) {
            const unsigned long long v0 = ring_off[r0] - vert_base, vo1 = ring_off[r0 + 1] - vert_base;
            const unsigned long long vend = ring_off[r1] - vert_base;
            m.v0 = v0;
            m.nv = (uint32_t)(vend - v0);
            m.nvo = (uint32_t)(vo1 - v0);
            for (unsigned long long v = v0; v < vo1; ++v) {
                const double x = vx[v], y = vy[v];
                m.bx0 = x < m.bx0 ? x : m.bx0;
                m.by0 = y < m.by0 ? y : m.by0;
                m.bx1 = m.bx1 < x ? x : m.bx1;
                m.by1 = m.by1 < y ? y : m.by1;
            }
        }
        meta[k] = m;
    }
}

template <int MODE>
__global__ void __launch_bounds__(kCsrThreads, MODE == kC1 ? 3 : 4) pip_csr_warp_kernel(
    const double2* __restrict__ pts, const unsigned long long* __restrict__ pt_off, unsigned long long n_polys,
    const double* __restrict__ vx, const double* __restrict__ vy, const unsigned long long* __restrict__ ring_off,
    const unsigned long long* __restrict__ poly_ring_off, unsigned long long pt_base, unsigned long long ring_base,
    unsigned long long vert_base, double tol, double tol2, uint32_t* __restrict__ inside_bits,
    uint32_t* __restrict__ aux_bits, const PolyMeta* __restrict__ meta, const uint32_t* __restrict__ count) {
    if (count) n_polys = min((unsigned long long)*count, n_polys); // deferred polygons only
    __shared__ EdgeScratch scratch[kWarps];
    const int lane = threadIdx.x & 31;
    EdgeScratch& es = scratch[threadIdx.x >> 5];
    const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    unsigned long long p = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;

    // metadata records: lanes 0-4 copy the next polygon's 80 bytes into this
    // warp's shared double buffer (cp.async) while the warp works on the current one
    __shared__ PolyMeta meta_s[kWarps][2];
    PolyMeta* mbuf = meta_s[threadIdx.x >> 5];
    auto fetch = [&](unsigned long long q, int slot) {
        if (lane < 5) {
            const unsigned dst = (unsigned)__cvta_generic_to_shared(reinterpret_cast<char*>(mbuf + slot) + 16 * lane);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                         "l"(reinterpret_cast<const char*>(meta + q) + 16 * lane)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int slot = 0;
    if (p < n_polys) fetch(p, 0);
    for (; p < n_polys; p += nwarps, slot ^= 1) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        const PolyMeta& m = mbuf[slot];
        const unsigned long long pn = p + nwarps;
        if (pn < n_polys) fetch(pn, slot ^ 1); // the slot last read one polygon ago
        if (m.np == 0 || m.nr == 0) continue;  // no points, or no rings (nothing is inside)
        const int nr = (int)min(m.nr, 1u << 20);
        const unsigned long long v0 = m.v0, r0 = m.r0;
        // ring starts (only for polygons with holes): lane i holds ring_off[r0 + i]
        const uint32_t rs_lane = (nr > 1 && lane < nr) ? (uint32_t)(ring_off[r0 + lane] - vert_base - v0) : 0u;
        const double* X = vx + v0;
        const double* Y = vy + v0;
        const double2* P = pts + m.s;
        const unsigned long long s = m.s;
        const uint32_t np = m.np, nv = m.nv;
        const double bx0 = m.bx0, by0 = m.by0, bx1 = m.bx1, by1 = m.by1;

        // C1 fast path scaling (uniform per polygon); see the comment at kFastBand
        const double Wb = __dsub_rn(bx1, bx0), Hb = __dsub_rn(by1, by0);
        const bool fast = MODE == kC1 && Wb >= 0x1p-300 && Wb <= 0x1p300 && Hb >= 0x1p-300 && Hb <= 0x1p300;
        const double sxl = fast ? pow2_below_inv(Wb) : 1.0, syl = fast ? pow2_below_inv(Hb) : 1.0;
        const double sy30 = __dmul_rn(syl, 0x1p30);

        for (uint32_t c = 0; c < np; c += 64) {
            double px[2], py[2];
            int ka[2], kb[2];
            float lx[2], ly[2];
            int qy[2];
            uint32_t par = 0, auxm = 0, act = 0, slow0 = 0;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const uint32_t i = c + 32 * j + lane;
                double2 q = make_double2(0.0, 0.0);
                if (i < np) q = P[i];
                px[j] = q.x;
                py[j] = q.y;
                // classify_batch short-circuit (batch.hpp:200): outside the closed bbox -> Outside
                const bool a = i < np && q.x >= bx0 && q.x <= bx1 && q.y >= by0 && q.y <= by1;
                act |= (uint32_t)a << j;
                if (MODE == kRobust) {
                    ka[j] = a ? fkey(__dadd_rn(q.y, tol)) : INT_MIN;
                    kb[j] = a ? fkey(__dsub_rn(q.y, tol)) : INT_MAX;
                } else {
                    ka[j] = a ? fkey(q.y) : INT_MAX;
                    kb[j] = 0;
                }
                if (MODE == kC1) {
                    const double dyp = __dsub_rn(q.y, by0);
                    lx[j] = __double2float_rn(__dmul_rn(__dsub_rn(q.x, bx0), sxl));
                    ly[j] = __double2float_rn(__dmul_rn(dyp, syl));
                    qy[j] = __double2int_rz(__dmul_rn(dyp, sy30));
                    slow0 |= (uint32_t)(a && !(fast && fabs(q.y) >= 0x1p-400)) << j;
                } else {
                    slow0 |= (uint32_t)a << j;
                }
            }
            if (!__any_sync(kFull, act != 0)) continue;
            for (uint32_t cv = 0;; cv += 31) {
                // vertices cv .. cv+31 (one per lane); edges cv+i -> cv+i+1 for i < 31
                const uint32_t v = cv + lane;
                double x = 0.0, y = 0.0;
                if (v < nv) {
                    x = X[v];
                    y = Y[v];
                }
                const double xn = __shfl_down_sync(kFull, x, 1), yn = __shfl_down_sync(kFull, y, 1);
                bool edge = lane < 31 && v + 1 < nv;
                for (int r = 1; r < nr; ++r) { // a ring's last vertex does not start an edge (P5)
                    const uint32_t rs = r < 32 ? __shfl_sync(kFull, rs_lane, r)
                                               : (uint32_t)(ring_off[r0 + r] - vert_base - v0);
                    edge = edge && v + 1 != rs;
                }
                // C1 fast path: local coordinates and key of this lane's vertex; a
                // vertex outside the outer bbox (a hole poking out) disables the
                // fast path for the chunk (the scaled terms would exceed 1)
                double axl = 0.0, ayl = 0.0;
                int qa = -1;
                bool chunk_fast = false;
                if (MODE == kC1) {
                    const double dya = __dsub_rn(y, by0);
                    axl = __dmul_rn(__dsub_rn(x, bx0), sxl);
                    ayl = __dmul_rn(dya, syl);
                    const bool inb = v >= nv || (axl >= 0.0 && axl < 1.0 && ayl >= 0.0 && ayl < 1.0);
                    if (v < nv) qa = __double2int_rz(__dmul_rn(dya, sy30));
                    chunk_fast = fast && __all_sync(kFull, inb);
                    if (lane == 31) {
                        es.fr[31] = make_int4(kFastSentinelLo, 0, qa, 0);
                        es.fr2[31] = make_float2(0.f, 1.f);
                    }
                }
                const int qb = __shfl_down_sync(kFull, qa, 1);
                if (lane < 31) {
                    const double ylo = yn < y ? yn : y, yhi = y < yn ? yn : y;
                    const int klo = fkey(ylo), khi = fkey(yhi);
                    int2 kr;
                    double2 q;
                    if (MODE == kC1) {
                        double nx = __dsub_rn(yn, y), ny = __dsub_rn(x, xn);
                        if (nx < 0.0) {
                            nx = -nx;
                            ny = -ny;
                        }
                        q = make_double2(nx, ny);
                        kr = make_int2(klo, (int)((unsigned)khi - (unsigned)klo));
                        // fast record: keys of the endpoints, scaled normal, offset
                        const int qlo = min(qa, qb), qhi = max(qa, qb);
                        const double Nx = __dmul_rn(nx, syl), Ny = __dmul_rn(ny, sxl);
                        const double cd = __dadd_rn(__dmul_rn(axl, Nx), __dmul_rn(ayl, Ny));
                        int4 f = make_int4(qlo + 1, max(qhi - qlo - 1, 0), qa, __float_as_int(__double2float_rn(Nx)));
                        float2 g = make_float2(__double2float_rn(Ny), __double2float_rn(-cd));
                        if (!edge) {
                            f = make_int4(kFastSentinelLo, 0, qa, 0);
                            g = make_float2(0.f, 1.f);
                        }
                        es.fr[lane] = f;
                        es.fr2[lane] = g;
                    } else if (MODE == kC2) {
                        q = make_double2(__dsub_rn(xn, x), __dsub_rn(yn, y));
                        kr = make_int2(klo, (int)((unsigned)khi - (unsigned)klo));
                    } else {
                        const double abx = __dsub_rn(xn, x), aby = __dsub_rn(yn, y);
                        q = make_double2(abx, aby);
                        es.len2[lane] = __dadd_rn(__dmul_rn(abx, abx), __dmul_rn(aby, aby));
                        kr = make_int2(klo, khi);
                    }
                    if (!edge) kr = make_int2(kNoEdge, MODE == kRobust ? INT_MIN : 0);
                    es.kr[lane] = kr;
                    es.a[lane] = make_double2(x, y);
                    es.q[lane] = q;
                    es.by[lane] = yn;
                }
                __syncwarp();
                const int ne = (int)min(31u, nv - cv - 1);
                // C1 fast pass over records 0..ne (vertex ne closes the chunk's
                // last edge; records past it are sentinels), four at a time
                uint32_t slow = slow0;
                if (MODE == kC1) {
                    if (chunk_fast) {
                        uint32_t fpar = 0, t0 = 0xffffffffu, t1 = 0xffffffffu;
                        float m0 = 1.f, m1 = 1.f;
                        const int nrec = (ne + 4) & ~3;
                        for (int i = 0; i < nrec; i += 4) {
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                const int4 f = es.fr[i + k];
                                const float2 g = es.fr2[i + k];
                                const float nxf = __int_as_float(f.w);
                                const float s0 = fmaf(lx[0], nxf, fmaf(ly[0], g.x, g.y));
                                const float s1 = fmaf(lx[1], nxf, fmaf(ly[1], g.x, g.y));
                                fast_toggle(fpar, 1u, (unsigned)(qy[0] - f.x), (unsigned)f.y, s0);
                                fast_toggle(fpar, 2u, (unsigned)(qy[1] - f.x), (unsigned)f.y, s1);
                                m0 = fminf(m0, fabsf(s0)); // band hits
                                m1 = fminf(m1, fabsf(s1));
                                t0 = min(t0, (unsigned)(qy[0] - f.z)); // ties: 0 iff q(p.y) == q(vertex)
                                t1 = min(t1, (unsigned)(qy[1] - f.z));
                            }
                        }
                        const bool u0 = m0 <= kFastBand || t0 == 0u, u1 = m1 <= kFastBand || t1 == 0u;
                        slow = (slow | (uint32_t)u0 | ((uint32_t)u1 << 1)) & act;
                        par ^= fpar & ~slow;
                    } else {
                        slow = act;
                    }
                }
                // pass 1 (integer filter) for the points on the exact path: per
                // point, the bitmask of this chunk's candidate edges -- key(p.y)
                // inside the edge's key range
                uint32_t cmask[2] = {0u, 0u};
                if (__any_sync(kFull, slow != 0)) {
                    int kx[2];
#pragma unroll
                    for (int j = 0; j < 2; ++j) kx[j] = (slow >> j & 1u) ? ka[j] : (MODE == kRobust ? INT_MIN : INT_MAX);
                    for (int i = ne - 1; i >= 0; --i) {
                        const int2 kr = es.kr[i];
#pragma unroll
                        for (int j = 0; j < 2; ++j) {
                            const bool c = MODE == kRobust ? (kx[j] >= kr.x && kb[j] <= kr.y)
                                                           : (unsigned)(kx[j] - kr.x) <= (unsigned)kr.y;
                            cmask[j] = (cmask[j] << 1) | (uint32_t)c;
                        }
                    }
                }
                // pass 2 (exact): every lane walks its *own* candidate edges, so the
                // warp iterates max-popcount times instead of once per edge
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    uint32_t m = cmask[j];
                    while (__any_sync(kFull, m != 0)) {
                        if (m == 0) continue;
                        const int i = __ffs(m) - 1;
                        m &= m - 1;
                        const int2 kr = es.kr[i];
                        const double2 a = es.a[i], q = es.q[i];
                        const unsigned d = (unsigned)(ka[j] - kr.x);
                        // sure: key(ylo) < key(p.y) < key(yhi) -> the reference straddles (P2)
                        const bool sure = kr.y != 0 && d - 1u < (unsigned)kr.y - 1u;
                        if (MODE == kC1) {
                            bool st = sure;
                            if (!st) st = __dmul_rn(__dsub_rn(a.y, py[j]), __dsub_rn(es.by[i], py[j])) <= 0.0;
                            const double side = __dadd_rn(__dmul_rn(__dsub_rn(px[j], a.x), q.x),
                                                          __dmul_rn(__dsub_rn(py[j], a.y), q.y));
                            if (st && side <= 0.0) par ^= 1u << j;
                        } else {
                            EdgeRec rr;
                            rr.d[0] = a.x;
                            rr.d[1] = a.y;
                            rr.d[2] = es.by[i];
                            rr.d[3] = q.x;
                            rr.d[4] = q.y;
                            rr.d[5] = MODE == kRobust ? es.len2[i] : 0.0;
                            int cnt = 0;
                            bool ax = false;
                            if (MODE == kRobust) exact_robust(px[j], py[j], tol, tol2, rr, cnt, ax);
                            else exact_c2(px[j], py[j], rr, cnt, ax, sure);
                            par ^= (uint32_t)(cnt & 1) << j;
                            auxm |= (uint32_t)ax << j;
                        }
                    }
                }
                __syncwarp();
                if (cv + 32 >= nv) break;
            }
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const uint32_t bi = __ballot_sync(kFull, (act & par & ~auxm) >> j & 1u);
                const uint32_t ba = __ballot_sync(kFull, (act & auxm) >> j & 1u);
                if (lane == 0) {
                    const unsigned long long g0 = s + c + 32 * j;
                    or_bits(inside_bits, g0, bi);
                    or_bits(aux_bits, g0, ba);
                }
            }
        }
    }
}

int sms(int dev) {
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
}

template <int MODE>
cudaError_t launch_warp(const CsrArgs& a, const uint32_t* list, const uint32_t* count, cudaStream_t st, int dev,
                        uint64_t* launches) {
    PolyMeta* meta = reinterpret_cast<PolyMeta*>(a.meta);
    const unsigned mgrid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((a.n_polys + 255) / 256, (uint64_t)sms(dev) * 8));
    csr_meta_kernel<<<mgrid, 256, 0, st>>>(
        reinterpret_cast<const unsigned long long*>(a.pt_off), a.n_polys, a.vx, a.vy,
        reinterpret_cast<const unsigned long long*>(a.ring_off), reinterpret_cast<const unsigned long long*>(a.poly_ring_off),
        a.pt_base, a.ring_base, a.vert_base, meta, list, count);
    ++*launches;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pip_csr_warp_kernel<MODE>, kCsrThreads, 0);
    per_sm = std::max(per_sm, 1);
    const uint64_t want = (a.n_polys + kWarps - 1) / kWarps;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)sms(dev) * per_sm));
    pip_csr_warp_kernel<MODE><<<grid, kCsrThreads, 0, st>>>(
        reinterpret_cast<const double2*>(a.pts), reinterpret_cast<const unsigned long long*>(a.pt_off), a.n_polys,
        a.vx, a.vy, reinterpret_cast<const unsigned long long*>(a.ring_off),
        reinterpret_cast<const unsigned long long*>(a.poly_ring_off), a.pt_base, a.ring_base, a.vert_base, a.tol,
        a.tol2, a.inside_bits, a.aux_bits, meta, count);
    ++*launches;
    return cudaGetLastError();
}

} // namespace

// scratch: per-polygon records, then the deferred-polygon list and its count
size_t csr_meta_bytes(uint64_t n_polys) {
    return (size_t)n_polys * sizeof(PolyMeta) + ((size_t)n_polys + 4) * sizeof(uint32_t);
}

cudaError_t launch_csr(const CsrArgs& a, cudaStream_t st, int dev, uint64_t* launches) {
    if (a.n_polys == 0) return cudaSuccess;
    // small polygons in the tile kernel (pip_csr_tile.cu); polygons whose
    // vertices do not fit its shared-memory slice are deferred to the
    // warp-per-polygon kernel
    uint32_t* list = reinterpret_cast<uint32_t*>(static_cast<char*>(a.meta) + (size_t)a.n_polys * sizeof(PolyMeta));
    uint32_t* count = list + a.n_polys;
    cudaError_t e = cudaMemsetAsync(count, 0, sizeof(uint32_t), st);
    if (e != cudaSuccess) return e;
    e = launch_csr_tile(a, list, count, st, dev, launches);
    if (e != cudaSuccess) return e;
    if (a.mode == kC1) return launch_warp<kC1>(a, list, count, st, dev, launches);
    if (a.mode == kC2) return launch_warp<kC2>(a, list, count, st, dev, launches);
    return launch_warp<kRobust>(a, list, count, st, dev, launches);
}

} // namespace pcd
