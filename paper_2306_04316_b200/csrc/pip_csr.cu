// CSR multi-polygon kernel (configs 3 and 5): many small
// polygons, each with its own contiguous run of query points.
//
// One warp per polygon (grid-stride, next polygon's offsets prefetched).  Per
// polygon the warp:
//   1. reads the polygon's CSR offsets with a single load (lanes 0-3) and
//      broadcasts them with shuffles;
//   2. walks its points 64 at a time (2 per lane) and, for each chunk of up to
//      31 edges, loads the chunk's 32 vertices (one per lane), derives the
//      per-edge data (filter keys, normal / direction) lane-parallel into a
//      per-warp shared-memory scratch and then scans the edges: integer key
//      filter for all points, the exact binary64 test of the reference for the
//      straddle candidates;
//   3. masks the result with the closed bbox of the outer ring (reduced from
//      the same vertex loads) — points outside it are Outside with no Error /
//      Boundary, exactly as classify_batch's short-circuit (batch.hpp:200);
//   4. ORs one ballot word per 32 points into the bit planes.
//
// Reference semantics per polygon: classify_batch(points_i, poly_i, mode)
// (batch.hpp:184-230) -> contains (geometry.hpp:281-300) ->
// count_crossings_c1/_c2 / robust_ray_crossings (geometry.hpp:182-273).
#include "pip_kernels.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>

#include "pip_device.cuh"

namespace pcd {

namespace {

constexpr int kCsrThreads = 256;
constexpr int kWarps = kCsrThreads / 32;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kNoEdge = 0x7ffffffe; // klo of a ring seam: no point key equals it

struct __align__(16) EdgeScratch { // one warp's current chunk of <= 31 edges
    int2 kr[32];                     // (klo, C1/C2: khi-klo | Robust: khi)
    double2 a[32];                   // (a.x, a.y)
    double2 q[32];                   // C1 (nx, ny) | C2 (dx, dy) | Robust (abx, aby)
    double by[32];
    double len2[32];                 // Robust only
};

__device__ __forceinline__ unsigned long long shfl64(unsigned long long v, int src) {
    return __shfl_sync(kFull, v, src);
}

__device__ __forceinline__ void or_bits(uint32_t* plane, unsigned long long g0, uint32_t bits) {
    if (!bits) return;
    const unsigned long long w = g0 >> 5;
    const unsigned sh = (unsigned)(g0 & 31);
    atomicOr(&plane[w], bits << sh);
    if (sh && (bits >> (32 - sh))) atomicOr(&plane[w + 1], bits >> (32 - sh));
}

// Exact min / max of a double over a lane group via its monotone 64-bit key
// and two 32-bit REDUX steps (high word, then low word among the lanes that tie).
__device__ __forceinline__ unsigned long long group_min_key(unsigned mask, unsigned long long k) {
    const unsigned hi = __reduce_min_sync(mask, (unsigned)(k >> 32));
    const unsigned lo = __reduce_min_sync(mask, (unsigned)(k >> 32) == hi ? (unsigned)k : 0xffffffffu);
    return ((unsigned long long)hi << 32) | lo;
}
__device__ __forceinline__ unsigned long long group_max_key(unsigned mask, unsigned long long k) {
    const unsigned hi = __reduce_max_sync(mask, (unsigned)(k >> 32));
    const unsigned lo = __reduce_max_sync(mask, (unsigned)(k >> 32) == hi ? (unsigned)k : 0u);
    return ((unsigned long long)hi << 32) | lo;
}

// Half-warp per polygon: lanes 0-15 classify polygon 2w, lanes 16-31 polygon
// 2w+1, 4 points per lane (64 per pass).  All loops run to the maximum of the
// two halves with per-half validity, so every warp-collective instruction is
// executed by the full warp; per-half values travel through half-local lanes
// and the per-half shared scratch.
template <int MODE>
__global__ void __launch_bounds__(kCsrThreads, 2) pip_csr_warp_kernel(
    const double2* __restrict__ pts, const unsigned long long* __restrict__ pt_off, unsigned long long n_polys,
    const double* __restrict__ vx, const double* __restrict__ vy, const unsigned long long* __restrict__ ring_off,
    const unsigned long long* __restrict__ poly_ring_off, unsigned long long pt_base, unsigned long long ring_base,
    unsigned long long vert_base, double tol, double tol2, uint32_t* __restrict__ inside_bits,
    uint32_t* __restrict__ aux_bits) {
    __shared__ EdgeScratch scratch[kWarps];
    const int lane = threadIdx.x & 31;
    const int h = lane >> 4, hl = lane & 15, hb = lane & 16; // half, lane in half, half's first lane
    const unsigned hmask = 0xffffu << hb;
    EdgeScratch& es = scratch[threadIdx.x >> 5];
    const unsigned long long npairs = (n_polys + 1) >> 1;
    const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    unsigned long long w = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;

    auto load_hdr = [&](unsigned long long pair) -> unsigned long long {
        const unsigned long long q = 2 * pair + h;
        if (q >= n_polys || hl >= 4) return 0ull;
        return hl < 2 ? pt_off[q + hl] : poly_ring_off[q + hl - 2];
    };
    unsigned long long hv = w < npairs ? load_hdr(w) : 0ull;
    for (; w < npairs; w += nwarps) {
        const bool has_poly = 2 * w + h < n_polys;
        const unsigned long long s = shfl64(hv, hb + 0) - pt_base, t = shfl64(hv, hb + 1) - pt_base;
        const unsigned long long r0 = shfl64(hv, hb + 2) - ring_base, r1 = shfl64(hv, hb + 3) - ring_base;
        if (w + nwarps < npairs) hv = load_hdr(w + nwarps);
        const bool live = has_poly && t > s && r1 > r0;
        const int nr = live ? (int)min(r1 - r0, 1ull << 20) : 0;
        // lane hl of each half holds ring_off[r0 + hl] (hl <= nr, hl < 16); more rings come from global
        const unsigned long long ro = live && hl <= nr ? ring_off[r0 + hl] - vert_base : 0ull;
        const unsigned long long v0 = shfl64(ro, hb);
        const unsigned long long ro_last = shfl64(ro, hb + min(nr, 15)); // shuffles run on all lanes
        const unsigned long long ro_1 = shfl64(ro, hb + 1);
        const unsigned long long vend = !live ? v0 : (nr < 16 ? ro_last : ring_off[r1] - vert_base);
        const double* X = vx + v0;
        const double* Y = vy + v0;
        const double2* P = pts + s;
        const uint32_t np = live ? (uint32_t)(t - s) : 0u, nv = (uint32_t)(vend - v0);
        const uint32_t nvo = live ? (uint32_t)(ro_1 - v0) : 0u; // outer ring vertices
        const uint32_t rs_lane = (uint32_t)(ro - v0);                         // start of ring hl
        const uint32_t np_max = max(np, __shfl_xor_sync(kFull, np, 16));
        const uint32_t nv_max = max(nv, __shfl_xor_sync(kFull, nv, 16));
        const uint32_t nvo_max = max(nvo, __shfl_xor_sync(kFull, nvo, 16));
        const int nr_max = max(nr, __shfl_xor_sync(kFull, nr, 16));
        if (np_max == 0) continue;

        // closed bbox of the outer ring, exactly (monotone keys + REDUX per half)
        unsigned long long kx0 = ~0ull, ky0 = ~0ull, kx1 = 0ull, ky1 = 0ull;
        for (uint32_t cv = 0; cv < nvo_max; cv += 16) {
            const uint32_t v = cv + hl;
            unsigned long long kx = ~0ull, ky = ~0ull, qx = 0ull, qy = 0ull;
            if (v < nvo) {
                kx = qx = dkey(X[v]);
                ky = qy = dkey(Y[v]);
            }
            kx0 = min(kx0, group_min_key(hmask, kx));
            ky0 = min(ky0, group_min_key(hmask, ky));
            kx1 = max(kx1, group_max_key(hmask, qx));
            ky1 = max(ky1, group_max_key(hmask, qy));
        }
        const double bx0 = dkey_inv(kx0), by0 = dkey_inv(ky0), bx1 = dkey_inv(kx1), by1 = dkey_inv(ky1);

        for (uint32_t c = 0; c < np_max; c += 64) {
            double px[4], py[4];
            int ka[4], kb[4];
            uint32_t par = 0, auxm = 0, act = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t i = c + 16 * j + hl;
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
            }
            if (__any_sync(kFull, act != 0)) {
                for (uint32_t cv = 0;; cv += 15) {
                    // vertices cv .. cv+15 (one per half-lane); edges cv+i -> cv+i+1 for i < 15
                    const uint32_t v = cv + hl;
                    double x = 0.0, y = 0.0;
                    if (v < nv) {
                        x = X[v];
                        y = Y[v];
                    }
                    const double xn = __shfl_down_sync(kFull, x, 1, 16), yn = __shfl_down_sync(kFull, y, 1, 16);
                    bool edge = hl < 15 && v + 1 < nv;
                    for (int r = 1; r < nr_max; ++r) { // a ring's last vertex does not start an edge (P5)
                        const uint32_t rs_sh = __shfl_sync(kFull, rs_lane, hb + min(r, 15));
                        if (r < nr) {
                            const uint32_t rs = r < 16 ? rs_sh : (uint32_t)(ring_off[r0 + r] - vert_base - v0);
                            edge = edge && v + 1 != rs;
                        }
                    }
                    if (hl < 15) {
                        const int slot = h * 16 + hl;
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
                        } else if (MODE == kC2) {
                            q = make_double2(__dsub_rn(xn, x), __dsub_rn(yn, y));
                            kr = make_int2(klo, (int)((unsigned)khi - (unsigned)klo));
                        } else {
                            const double abx = __dsub_rn(xn, x), aby = __dsub_rn(yn, y);
                            q = make_double2(abx, aby);
                            es.len2[slot] = __dadd_rn(__dmul_rn(abx, abx), __dmul_rn(aby, aby));
                            kr = make_int2(klo, khi);
                        }
                        if (!edge) kr = make_int2(kNoEdge, MODE == kRobust ? INT_MIN : 0);
                        es.kr[slot] = kr;
                        es.a[slot] = make_double2(x, y);
                        es.q[slot] = q;
                        es.by[slot] = yn;
                    }
                    __syncwarp();
                    const int ne = (int)min(15u, nv > cv + 1 ? nv - cv - 1 : 0u);
                    const int ne_max = max(ne, __shfl_xor_sync(kFull, ne, 16));
                    for (int i = 0; i < ne_max; ++i) {
                        const int slot = h * 16 + i;
                        const int2 kr = i < ne ? es.kr[slot] : make_int2(kNoEdge, MODE == kRobust ? INT_MIN : 0);
                        bool cand[4];
                        uint32_t dd[4];
                        bool anyc = false;
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            dd[j] = (unsigned)(ka[j] - kr.x);
                            cand[j] = MODE == kRobust ? (ka[j] >= kr.x && kb[j] <= kr.y) : dd[j] <= (unsigned)kr.y;
                            anyc |= cand[j];
                        }
                        if (!__any_sync(kFull, anyc)) continue;
                        const double2 a = es.a[slot], q = es.q[slot];
                        if (MODE == kC1) {
                            // key tie (d == 0 or d == range): the reference's product decides
                            bool anyt = false;
                            bool tie[4];
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                tie[j] = cand[j] && dd[j] - 1u >= (unsigned)kr.y - 1u;
                                anyt |= tie[j];
                            }
                            if (__any_sync(kFull, anyt)) {
                                const double byv = es.by[slot];
#pragma unroll
                                for (int j = 0; j < 4; ++j)
                                    if (tie[j])
                                        cand[j] = __dmul_rn(__dsub_rn(a.y, py[j]), __dsub_rn(byv, py[j])) <= 0.0;
                            }
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                const double side = __dadd_rn(__dmul_rn(__dsub_rn(px[j], a.x), q.x),
                                                              __dmul_rn(__dsub_rn(py[j], a.y), q.y));
                                if (cand[j] && side <= 0.0) par ^= 1u << j;
                            }
                        } else {
                            EdgeRec rr;
                            rr.d[0] = a.x;
                            rr.d[1] = a.y;
                            rr.d[2] = es.by[slot];
                            rr.d[3] = q.x;
                            rr.d[4] = q.y;
                            rr.d[5] = MODE == kRobust ? es.len2[slot] : 0.0;
                            rr.d[6] = rr.d[2] < a.y ? rr.d[2] : a.y;
                            rr.d[7] = a.y < rr.d[2] ? rr.d[2] : a.y;
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                if (!cand[j]) continue;
                                int cnt = 0;
                                bool ax = false;
                                if (MODE == kRobust) exact_robust(px[j], py[j], tol, tol2, rr, cnt, ax);
                                else exact_c2(px[j], py[j], rr, cnt, ax, dd[j] - 1u < (unsigned)kr.y - 1u);
                                par ^= (uint32_t)(cnt & 1) << j;
                                auxm |= (uint32_t)ax << j;
                            }
                        }
                    }
                    __syncwarp();
                    if (cv + 16 >= nv_max) break;
                }
            }
            // one 32-point word per (half, j-pair): points c+32m .. c+32m+31 of the half's polygon
#pragma unroll
            for (int m = 0; m < 2; ++m) {
                const uint32_t b0 = __ballot_sync(kFull, (act & par & ~auxm) >> (2 * m) & 1u);
                const uint32_t b1 = __ballot_sync(kFull, (act & par & ~auxm) >> (2 * m + 1) & 1u);
                const uint32_t a0 = __ballot_sync(kFull, (act & auxm) >> (2 * m) & 1u);
                const uint32_t a1 = __ballot_sync(kFull, (act & auxm) >> (2 * m + 1) & 1u);
                if (hl == 0 && live) {
                    const uint32_t bi = ((b0 >> hb) & 0xffffu) | (((b1 >> hb) & 0xffffu) << 16);
                    const uint32_t ba = ((a0 >> hb) & 0xffffu) | (((a1 >> hb) & 0xffffu) << 16);
                    const unsigned long long g0 = s + c + 32 * m;
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
cudaError_t launch_t(const CsrArgs& a, cudaStream_t st, int dev, uint64_t* launches) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pip_csr_warp_kernel<MODE>, kCsrThreads, 0);
    per_sm = std::max(per_sm, 1);
    const uint64_t want = (a.n_polys + 2 * kWarps - 1) / (2 * kWarps);
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)sms(dev) * per_sm));
    pip_csr_warp_kernel<MODE><<<grid, kCsrThreads, 0, st>>>(
        reinterpret_cast<const double2*>(a.pts), reinterpret_cast<const unsigned long long*>(a.pt_off), a.n_polys,
        a.vx, a.vy, reinterpret_cast<const unsigned long long*>(a.ring_off),
        reinterpret_cast<const unsigned long long*>(a.poly_ring_off), a.pt_base, a.ring_base, a.vert_base, a.tol,
        a.tol2, a.inside_bits, a.aux_bits);
    ++*launches;
    return cudaGetLastError();
}

} // namespace

cudaError_t launch_csr(const CsrArgs& a, cudaStream_t st, int dev, uint64_t* launches) {
    if (a.n_polys == 0) return cudaSuccess;
    switch (a.mode) {
    case kC1: return launch_t<kC1>(a, st, dev, launches);
    case kC2: return launch_t<kC2>(a, st, dev, launches);
    default: return launch_t<kRobust>(a, st, dev, launches);
    }
}

} // namespace pcd
