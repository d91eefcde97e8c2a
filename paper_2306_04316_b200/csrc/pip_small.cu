// Small calls (the single-point contains / count_crossings_c1/_c2 of the
// drop-in API, and classify_batch on a few points): one launch, a CTA per
// point, the CTA's threads striding over the polygon's edges with the
// reference's own loop body (raw_edge: geometry.hpp:182-273, literal binary64),
// then a block reduction of the count (sum), the aux outcome (OR) and the
// first degenerate edge (min vertex index, for DegenerateEdge's message).
//
// Every (point, edge) term of the reference is independent of the others
// (f_prev of an edge is RN(a.y - p.y) for its own first vertex a, the value the
// reference carries over), so splitting a ring's edges across threads
// reproduces count_crossings_c1/_c2 exactly; Robust's boundary and C2's
// DegenerateEdge abort the reference loop, which only matters for the count,
// not for the verdict (Boundary / Error dominate), and the count API reports
// the first degenerate edge instead of a count, as the reference throws there.
//
// Output of a classify call (one device buffer, zeroed by the caller):
//   verdict bytes [n] | inside plane [ceil(n/32)] | aux plane | stats[4] (u64)
#include "pip_kernels.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>

#include "pip_device.cuh"

namespace pcd {

namespace {

constexpr int kSTPB = 256;

__device__ __forceinline__ uint32_t ring_of_small(const uint64_t* ring_off, uint32_t n_rings, uint64_t v) {
    uint32_t lo = 0, hi = n_rings; // largest r with ring_off[r] <= v
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (ring_off[mid] <= v) lo = mid; else hi = mid;
    }
    return lo;
}

// COUNT: count_crossings of one ring (ring_off = {0, nv}); else classify.
template <int MODE, bool COUNT>
__global__ void __launch_bounds__(kSTPB) small_kernel(const double2* __restrict__ pts, uint64_t n,
                                                      const double* __restrict__ vx, const double* __restrict__ vy,
                                                      const uint64_t* __restrict__ ring_off, uint32_t n_rings,
                                                      const double* __restrict__ box, double tol, double tol2,
                                                      unsigned char* __restrict__ out,
                                                      unsigned long long* __restrict__ counts,
                                                      uint8_t* __restrict__ degen) {
    __shared__ int s_cnt[kSTPB / 32];
    __shared__ unsigned long long s_deg[kSTPB / 32];
    const uint64_t i = blockIdx.x;
    const double2 p = pts[i];
    const bool run = box == nullptr || (p.x >= box[0] && p.x <= box[2] && p.y >= box[1] && p.y <= box[3]);
    int cnt = 0;
    bool aux = false;
    unsigned long long first = ~0ull; // first vertex of the first aux edge (vertex order = the reference's loop order)
    const uint64_t nv = ring_off[n_rings];
    if (run && nv >= 2) { // CTA-uniform
        for (uint64_t v = threadIdx.x; v + 1 < nv; v += kSTPB) {
            if (n_rings > 1) {
                const uint32_t r = ring_of_small(ring_off, n_rings, v);
                if (v + 1 >= ring_off[r + 1]) continue; // last vertex of its ring: no edge
            }
            PC_DCHECK(v + 1 < nv);
            const double ax = vx[v], ay = vy[v], bx = vx[v + 1], by = vy[v + 1];
            double f_prev = __dsub_rn(ay, p.y); // geometry.hpp:185/:223 (carried as b.y - p.y of the previous edge)
            bool a = false;
            raw_edge<MODE>(p.x, p.y, tol, tol2, ax, ay, bx, by, f_prev, cnt, a);
            if (a) {
                aux = true;
                first = min(first, (unsigned long long)v);
            }
        }
    }
    // block reduction: sum of counts, min of the first aux edge
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_cnt[w] = cnt;
        s_deg[w] = first;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    int total = 0;
    for (int k = 0; k < kSTPB / 32; ++k) {
        total += s_cnt[k];
        first = min(first, s_deg[k]);
    }
    aux = first != ~0ull;
    if (COUNT) {
        counts[i] = aux ? (unsigned long long)(first - ring_off[0]) : (unsigned long long)total;
        degen[i] = aux ? 1 : 0;
        return;
    }
    const uint64_t nw = (n + 31) >> 5;
    uint8_t* verdicts = out;
    uint32_t* inside = reinterpret_cast<uint32_t*>(out + ((n + 15) & ~15ull));
    uint32_t* auxp = inside + nw;
    unsigned long long* stats = reinterpret_cast<unsigned long long*>(auxp + nw); // 2 nw words: 8-byte aligned
    uint8_t v = 1; // Outside
    if (aux) v = MODE == kRobust ? 2 : 3;           // Boundary / Error
    else if (total & 1) v = 0;                       // Inside
    verdicts[i] = v;
    if (v == 0) atomicOr(&inside[i >> 5], 1u << (i & 31));
    if (v >= 2) atomicOr(&auxp[i >> 5], 1u << (i & 31));
    atomicAdd(&stats[v], 1ull);
}

} // namespace

size_t small_out_bytes(uint64_t n) {
    const uint64_t nw = (n + 31) >> 5;
    return ((n + 15) & ~15ull) + 4 * (2 * nw) + 32;
}

cudaError_t launch_small(const double* pts, uint64_t n, const double* vx, const double* vy, const uint64_t* ring_off,
                         uint32_t n_rings, const double* box, int mode, double tol, void* out,
                         unsigned long long* counts, uint8_t* degen, cudaStream_t st, uint64_t* launches) {
    if (n == 0) return cudaSuccess;
    const double2* p = reinterpret_cast<const double2*>(pts);
    const double tol2 = tol * tol;
    unsigned char* o = static_cast<unsigned char*>(out);
    const unsigned grid = (unsigned)n;
    if (counts) {
        if (mode == kC1) small_kernel<kC1, true><<<grid, kSTPB, 0, st>>>(p, n, vx, vy, ring_off, n_rings, nullptr, 0.0, 0.0, o, counts, degen);
        else small_kernel<kC2, true><<<grid, kSTPB, 0, st>>>(p, n, vx, vy, ring_off, n_rings, nullptr, 0.0, 0.0, o, counts, degen);
    } else {
        switch (mode) {
        case kC1: small_kernel<kC1, false><<<grid, kSTPB, 0, st>>>(p, n, vx, vy, ring_off, n_rings, box, tol, tol2, o, nullptr, nullptr); break;
        case kC2: small_kernel<kC2, false><<<grid, kSTPB, 0, st>>>(p, n, vx, vy, ring_off, n_rings, box, tol, tol2, o, nullptr, nullptr); break;
        default: small_kernel<kRobust, false><<<grid, kSTPB, 0, st>>>(p, n, vx, vy, ring_off, n_rings, box, tol, tol2, o, nullptr, nullptr);
        }
    }
    ++*launches;
    return cudaGetLastError();
}

} // namespace pcd
