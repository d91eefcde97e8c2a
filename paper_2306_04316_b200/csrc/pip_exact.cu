// The literal binary64 path (PC_OPT_EXACT): every point walks every edge of
// its polygon with the reference's own loop, no filter keys, no fp32
// certification, no y-bucketing, no bbox keys.  It exists so that the fast
// kernels (pip_single.cu, pip_csr_tile.cu, pip_csr.cu) can be checked on ALL
// points of the large configs on the GPU itself (tests/test_full_parity.py),
// where the CPU reference would take hours; it is pinned to the reference by
// the same golden vectors as the fast path.
//
// Per point (thread), per ring (geometry.hpp:281-300):
//   C1      f_prev = ring[0].y - p.y; per edge raw_edge<C1>   (geometry.hpp:182-203)
//   C2      same with the intercept test, DegenerateEdge -> aux (geometry.hpp:208-229)
//   Robust  raw_edge<Robust>, on_boundary -> aux            (geometry.hpp:237-273)
// classify_batch's bbox short-circuit (batch.hpp:121-133, :39-41, :200) uses
// the outer ring's literal min/max (std::min/std::max order) when prefilter is on.
// Bits leave as one ballot word per warp (32 consecutive points), stored, not
// accumulated: the planes need no clearing.
#include "pip_kernels.h"

#include <cuda_runtime.h>

#include <algorithm>

#include "pip_device.cuh"

namespace pcd {

namespace {

constexpr int kXTPB = 256;
constexpr int kXTile = 1024; // vertices per shared-memory stage (16 KB)

// bbox_of (batch.hpp:121-133) over the outer ring, std::min / std::max order
__device__ __forceinline__ void outer_bbox(const double* vx, const double* vy, uint64_t lo, uint64_t hi, double* b) {
    double mnx = __longlong_as_double(0x7ff0000000000000ll), mny = mnx;
    double mxx = -mnx, mxy = -mnx;
    for (uint64_t i = lo; i < hi; ++i) {
        const double x = vx[i], y = vy[i];
        mnx = x < mnx ? x : mnx;
        mny = y < mny ? y : mny;
        mxx = mxx < x ? x : mxx;
        mxy = mxy < y ? y : mxy;
    }
    b[0] = mnx;
    b[1] = mny;
    b[2] = mxx;
    b[3] = mxy;
}

__global__ void exact_bbox_kernel(const double* __restrict__ vx, const double* __restrict__ vy,
                                  const uint64_t* __restrict__ ring_off, double* __restrict__ box) {
    // one CTA: strided partial boxes, then a serial fold by thread 0 (the
    // order of min/max over finite values never changes a closed-box test)
    __shared__ double part[kXTPB][4];
    const uint64_t lo = ring_off[0], hi = ring_off[1];
    double mnx = __longlong_as_double(0x7ff0000000000000ll), mny = mnx, mxx = -mnx, mxy = -mnx;
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const double x = vx[i], y = vy[i];
        mnx = x < mnx ? x : mnx;
        mny = y < mny ? y : mny;
        mxx = mxx < x ? x : mxx;
        mxy = mxy < y ? y : mxy;
    }
    part[threadIdx.x][0] = mnx;
    part[threadIdx.x][1] = mny;
    part[threadIdx.x][2] = mxx;
    part[threadIdx.x][3] = mxy;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int t = 1; t < (int)blockDim.x; ++t) {
            mnx = part[t][0] < mnx ? part[t][0] : mnx;
            mny = part[t][1] < mny ? part[t][1] : mny;
            mxx = mxx < part[t][2] ? part[t][2] : mxx;
            mxy = mxy < part[t][3] ? part[t][3] : mxy;
        }
        box[0] = mnx;
        box[1] = mny;
        box[2] = mxx;
        box[3] = mxy;
    }
}

template <int MODE>
__global__ void __launch_bounds__(kXTPB) exact_single_kernel(const double2* __restrict__ pts, uint64_t n,
                                                             const double* __restrict__ vx,
                                                             const double* __restrict__ vy,
                                                             const uint64_t* __restrict__ ring_off, uint32_t n_rings,
                                                             const double* __restrict__ box, double tol, double tol2,
                                                             uint32_t* __restrict__ inside_bits,
                                                             uint32_t* __restrict__ aux_bits) {
    __shared__ double2 tile[kXTile];
    const uint64_t i = blockIdx.x * (uint64_t)kXTPB + threadIdx.x;
    const bool live = i < n;
    const double2 p = live ? pts[i] : make_double2(0.0, 0.0);
    bool run = live;
    if (run && box) run = p.x >= box[0] && p.x <= box[2] && p.y >= box[1] && p.y <= box[3]; // batch.hpp:39-41
    const uint64_t nv = ring_off[n_rings];
    int cnt = 0;
    bool aux = false;
    double f_prev = 0.0, ax = 0.0, ay = 0.0;
    uint32_t r = 0;
    uint64_t ring_start = ring_off[0], ring_end = ring_off[1];
    const bool any = __syncthreads_or(run); // CTA-uniform: nothing to walk for a CTA outside the box
    for (uint64_t t0 = 0; any && t0 < nv; t0 += kXTile) {
        const uint32_t nt = (uint32_t)min((uint64_t)kXTile, nv - t0);
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < nt; k += kXTPB) tile[k] = make_double2(vx[t0 + k], vy[t0 + k]);
        __syncthreads();
        for (uint32_t k = 0; k < nt; ++k) {
            const uint64_t v = t0 + k;
            while (v >= ring_end) { // next ring (uniform); rings are non-empty
                ++r;
                ring_start = ring_off[r];
                ring_end = ring_off[r + 1];
            }
            const double2 b = tile[k];
            if (v == ring_start) { // geometry.hpp:185: f_prev = ring[0].y - p.y
                f_prev = __dsub_rn(b.y, p.y);
            } else if (run) {
                raw_edge<MODE>(p.x, p.y, tol, tol2, ax, ay, b.x, b.y, f_prev, cnt, aux);
            }
            ax = b.x;
            ay = b.y;
        }
    }
    const uint32_t in_w = __ballot_sync(0xffffffffu, run && (cnt & 1));
    const uint32_t aux_w = __ballot_sync(0xffffffffu, run && aux);
    if ((threadIdx.x & 31) == 0 && i < n) {
        inside_bits[i >> 5] = in_w;
        aux_bits[i >> 5] = aux_w;
    }
}

// CSR: thread per point; its polygon by binary search in pt_off; the polygon's
// rings straight from global memory (a footprint's vertices stay in L1).
template <int MODE>
__global__ void __launch_bounds__(kXTPB) exact_csr_kernel(const double2* __restrict__ pts, uint64_t n,
                                                          const uint64_t* __restrict__ pt_off, uint64_t n_polys,
                                                          const double* __restrict__ vx, const double* __restrict__ vy,
                                                          const uint64_t* __restrict__ ring_off,
                                                          const uint64_t* __restrict__ poly_ring_off,
                                                          uint64_t pt_base, uint64_t ring_base, uint64_t vert_base,
                                                          double tol, double tol2, uint32_t* __restrict__ inside_bits,
                                                          uint32_t* __restrict__ aux_bits) {
    const uint64_t i = blockIdx.x * (uint64_t)kXTPB + threadIdx.x;
    bool run = false;
    int cnt = 0;
    bool aux = false;
    if (i < n) {
        const uint64_t g = pt_base + i;
        uint64_t lo = 0, hi = n_polys; // largest p with pt_off[p] <= g (empty polygons skipped)
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) >> 1;
            if (pt_off[mid] <= g) lo = mid; else hi = mid;
        }
        const uint64_t p = lo;
        PC_DCHECK(p < n_polys && pt_off[p] <= g && g < pt_off[p + 1]);
        const uint64_t r0 = poly_ring_off[p] - ring_base, r1 = poly_ring_off[p + 1] - ring_base;
        const double2 q = pts[i];
        if (r1 > r0) {
            double b[4];
            outer_bbox(vx, vy, ring_off[r0] - vert_base, ring_off[r0 + 1] - vert_base, b);
            run = q.x >= b[0] && q.x <= b[2] && q.y >= b[1] && q.y <= b[3];
        }
        if (run) {
            for (uint64_t r = r0; r < r1; ++r) {
                const uint64_t v0 = ring_off[r] - vert_base, v1 = ring_off[r + 1] - vert_base;
                if (v1 <= v0) continue;
                double f_prev = __dsub_rn(vy[v0], q.y);
                double ax = vx[v0], ay = vy[v0];
                for (uint64_t v = v0 + 1; v < v1; ++v) {
                    const double bx = vx[v], by = vy[v];
                    raw_edge<MODE>(q.x, q.y, tol, tol2, ax, ay, bx, by, f_prev, cnt, aux);
                    ax = bx;
                    ay = by;
                }
            }
        }
    }
    const uint32_t in_w = __ballot_sync(0xffffffffu, run && (cnt & 1));
    const uint32_t aux_w = __ballot_sync(0xffffffffu, run && aux);
    if ((threadIdx.x & 31) == 0 && i < n) {
        inside_bits[i >> 5] = in_w;
        aux_bits[i >> 5] = aux_w;
    }
}

} // namespace

cudaError_t launch_exact_single(const double* pts, uint64_t n, const double* vx, const double* vy,
                                const uint64_t* ring_off, uint32_t n_rings, int prefilter, double* box_scratch,
                                int mode, double tol, uint32_t* inside_bits, uint32_t* aux_bits, cudaStream_t st,
                                uint64_t* launches) {
    if (n == 0) return cudaSuccess;
    const double* box = nullptr;
    if (prefilter) {
        exact_bbox_kernel<<<1, kXTPB, 0, st>>>(vx, vy, ring_off, box_scratch);
        ++*launches;
        box = box_scratch;
    }
    const unsigned grid = (unsigned)((n + kXTPB - 1) / kXTPB);
    const double tol2 = tol * tol;
    const double2* p = reinterpret_cast<const double2*>(pts);
    switch (mode) {
    case kC1:
        exact_single_kernel<kC1><<<grid, kXTPB, 0, st>>>(p, n, vx, vy, ring_off, n_rings, box, tol, tol2, inside_bits,
                                                         aux_bits);
        break;
    case kC2:
        exact_single_kernel<kC2><<<grid, kXTPB, 0, st>>>(p, n, vx, vy, ring_off, n_rings, box, tol, tol2, inside_bits,
                                                         aux_bits);
        break;
    default:
        exact_single_kernel<kRobust><<<grid, kXTPB, 0, st>>>(p, n, vx, vy, ring_off, n_rings, box, tol, tol2,
                                                             inside_bits, aux_bits);
    }
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_outer_bbox(const double* vx, const double* vy, const uint64_t* ring_off, double* box,
                              cudaStream_t st, uint64_t* launches) {
    exact_bbox_kernel<<<1, kXTPB, 0, st>>>(vx, vy, ring_off, box);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_exact_csr(const CsrArgs& a, uint64_t n_points, cudaStream_t st, uint64_t* launches) {
    if (n_points == 0) return cudaSuccess;
    const unsigned grid = (unsigned)((n_points + kXTPB - 1) / kXTPB);
    const double2* p = reinterpret_cast<const double2*>(a.pts);
#define PC_EXACT_CSR(M)                                                                                              \
    exact_csr_kernel<M><<<grid, kXTPB, 0, st>>>(p, n_points, a.pt_off, a.n_polys, a.vx, a.vy, a.ring_off,            \
                                                a.poly_ring_off, a.pt_base, a.ring_base, a.vert_base, a.tol, a.tol2, \
                                                a.inside_bits, a.aux_bits)
    switch (a.mode) {
    case kC1: PC_EXACT_CSR(kC1); break;
    case kC2: PC_EXACT_CSR(kC2); break;
    default: PC_EXACT_CSR(kRobust);
    }
#undef PC_EXACT_CSR
    ++*launches;
    return cudaGetLastError();
}

} // namespace pcd
