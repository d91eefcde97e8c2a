// y-bucketing of query points (SIMT coherence for the single-polygon kernel).
//
// Why: a warp classifies 32 points per step against one staged edge.  When the
// 32 points have unrelated y, the chance that *some* lane needs the exact
// binary64 test of an edge is ~1-(1-s)^32 (s = the edge's y-span fraction):
// for the star polygons of configs 1/2, s ~ 0.05, so ~60% of edges take the
// slow path for some lane and the whole warp pays for it.  Counting-sorting
// the points by y over the polygon's bbox (4096 bins) makes each warp's
// points y-adjacent, so they straddle the same edges and the slow path runs
// for ~s of the edges instead.  Points the bbox prefilter rejects
// (classify_batch, batch.hpp:200) land in a trailing bin and are never
// classified (they are Outside), which is the GPU form of prefilter_bbox
// (batch.hpp:145-156).  Results are mapped back to the original order by
// index, so the output does not depend on the (nondeterministic) order inside
// a bin.  The scan over every (point, edge) pair is unchanged.
#include "pip_kernels.h"

#include <cuda_runtime.h>

#include <algorithm>

#include "pip_device.cuh"

namespace pcd {

namespace {

struct BinMap {
    double minx, miny, maxx, maxy, scale;
    int prefilter;

    __device__ __forceinline__ int bin(double x, double y) const {
        if (prefilter && !(x >= minx && x <= maxx && y >= miny && y <= maxy)) return kBuckets;
        const double t = (y - miny) * scale; // ordering only: no exactness needed
        int b = t > 0.0 ? (int)t : 0;
        return b < kBuckets ? b : kBuckets - 1;
    }
};

__device__ __forceinline__ BinMap make_map(const unsigned long long* bbox_keys, int prefilter) {
    BinMap m;
    m.minx = dkey_inv(bbox_keys[0]);
    m.miny = dkey_inv(bbox_keys[1]);
    m.maxx = dkey_inv(~bbox_keys[2]);
    m.maxy = dkey_inv(~bbox_keys[3]);
    const double h = m.maxy - m.miny;
    m.scale = (h > 0.0 && h < 1e300) ? kBuckets / h : 0.0;
    m.prefilter = prefilter;
    return m;
}

// Atomic-free (in global memory) counting sort over P CTAs:
//   count    CTA b histograms its contiguous chunk of points in shared memory
//            and writes the counts to blk[bin][b] (bin-major);
//   colscan  a warp per bin: exclusive prefix over the CTAs (blk[bin][b]
//            becomes CTA b's offset inside the bin) and the bin total;
//   scan     exclusive scan of the bin totals -> bin base (and n_in);
//   scatter  CTA b re-reads its chunk and places each point at base[bin] +
//            blk[bin][b] + (shared-memory cursor), no global atomics.
__global__ void __launch_bounds__(1024) bucket_count_kernel(const double2* __restrict__ pts, uint64_t n,
                                                            uint64_t chunk,
                                                            const unsigned long long* __restrict__ bbox_keys,
                                                            int prefilter, uint32_t* __restrict__ blk) {
    __shared__ uint32_t h[kBuckets + 1];
    for (int j = threadIdx.x; j <= kBuckets; j += blockDim.x) h[j] = 0;
    __syncthreads();
    const BinMap m = make_map(bbox_keys, prefilter);
    const uint64_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const double2 p = pts[i];
        atomicAdd(&h[m.bin(p.x, p.y)], 1u);
    }
    __syncthreads();
    // bin-major: blk[bin * n_blk + block], so the per-bin scan over blocks reads contiguous memory
    for (int j = threadIdx.x; j <= kBuckets; j += blockDim.x) blk[(uint64_t)j * gridDim.x + blockIdx.x] = h[j];
}

// Per bin (one warp each): exclusive scan over the blocks of blk[bin][*]
// (contiguous) -> each block's offset inside the bin; hist[bin] = bin total.
__global__ void __launch_bounds__(256) bucket_colscan_kernel(uint32_t* __restrict__ blk, int n_blk,
                                                             uint32_t* __restrict__ hist) {
    const int bin = (int)((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (bin > kBuckets) return;
    uint32_t* col = blk + (uint64_t)bin * n_blk;
    uint32_t run = 0;
    for (int b0 = 0; b0 < n_blk; b0 += 32) {
        const int b = b0 + lane;
        const uint32_t v = b < n_blk ? col[b] : 0u;
        uint32_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (b < n_blk) col[b] = run + incl - v;
        run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) hist[bin] = run;
}

// Exclusive scan of the kBuckets+1 counts (one CTA of 1024 threads): every
// thread loads its 64 counts of a coalesced tile layout up front (one memory
// latency), then the CTA scans tile after tile with a carried running sum;
// hist becomes the write cursor of each bin, hist[kBuckets+1] = in-box count.
__global__ void __launch_bounds__(1024) bucket_scan_kernel(uint32_t* __restrict__ hist) {
    constexpr int kTiles = (kBuckets + 1 + 1023) / 1024;
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t carry_s;
    const int t = threadIdx.x;
    uint32_t v[kTiles];
#pragma unroll
    for (int q = 0; q < kTiles; ++q) {
        const int j = q * 1024 + t;
        v[q] = j <= kBuckets ? hist[j] : 0u;
    }
    if (t == 0) carry_s = 0;
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kTiles; ++q) {
        uint32_t incl = v[q];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if ((t & 31) >= o) incl += y;
        }
        if ((t & 31) == 31) warp_sums[t >> 5] = incl;
        __syncthreads();
        if (t < 32) {
            uint32_t w = warp_sums[t];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (t >= o) w += y;
            }
            warp_sums[t] = w;
        }
        __syncthreads();
        const uint32_t carry = carry_s;
        const uint32_t excl = carry + incl - v[q] + ((t >> 5) ? warp_sums[(t >> 5) - 1] : 0u);
        const int j = q * 1024 + t;
        if (j <= kBuckets) {
            hist[j] = excl;
            if (j == kBuckets) hist[kBuckets + 1] = excl; // in-box count = start of the reject bin
        }
        __syncthreads();
        if (t == 1023) carry_s = carry + warp_sums[31];
        __syncthreads();
    }
}

__global__ void __launch_bounds__(1024) bucket_scatter_kernel(const double2* __restrict__ pts, uint64_t n,
                                                              uint64_t chunk,
                                                              const unsigned long long* __restrict__ bbox_keys,
                                                              int prefilter, const uint32_t* __restrict__ blk,
                                                              const uint32_t* __restrict__ base,
                                                              double2* __restrict__ sorted_pts,
                                                              uint32_t* __restrict__ sorted_idx) {
    __shared__ uint32_t cur[kBuckets + 1];
    for (int j = threadIdx.x; j <= kBuckets; j += blockDim.x) cur[j] = base[j] + blk[(uint64_t)j * gridDim.x + blockIdx.x];
    __syncthreads();
    const BinMap m = make_map(bbox_keys, prefilter);
    const uint64_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const double2 p = pts[i];
        const int b = m.bin(p.x, p.y);
        if (b == kBuckets) continue; // rejected by the bbox prefilter: Outside, never classified
        const uint32_t pos = atomicAdd(&cur[b], 1u);
        sorted_pts[pos] = p;
        sorted_idx[pos] = (uint32_t)i;
    }
}

// Bucketed bit planes -> original order (planes pre-zeroed).  Only set bits
// cost an atomic; a warp reads each bucketed word once.
__global__ void __launch_bounds__(256) unbucket_kernel(uint64_t n, const uint32_t* __restrict__ n_dev,
                                                       const uint32_t* __restrict__ sorted_idx,
                                                       const uint32_t* __restrict__ s_inside,
                                                       const uint32_t* __restrict__ s_aux,
                                                       uint32_t* __restrict__ inside_bits,
                                                       uint32_t* __restrict__ aux_bits) {
    const uint64_t n_in = min(n, (uint64_t)*n_dev);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_in; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t wi = s_inside[i >> 5], wa = s_aux[i >> 5];
        const uint32_t bit = 1u << (i & 31);
        if ((wi | wa) & bit) {
            const uint32_t o = sorted_idx[i];
            if (wi & bit) atomicOr(&inside_bits[o >> 5], 1u << (o & 31));
            if (wa & bit) atomicOr(&aux_bits[o >> 5], 1u << (o & 31));
        }
    }
}

int sms(int dev) {
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
}

} // namespace

cudaError_t launch_bucket(const BucketArgs& a, cudaStream_t st, int dev, uint64_t* launches) {
    const double2* p = reinterpret_cast<const double2*>(a.pts);
    const int n_blk = a.n_blk;
    const uint64_t chunk = (a.n + n_blk - 1) / n_blk;
    bucket_count_kernel<<<n_blk, 1024, 0, st>>>(p, a.n, chunk, a.bbox_keys, a.prefilter, a.blk);
    bucket_colscan_kernel<<<(kBuckets + 1 + 7) / 8, 256, 0, st>>>(a.blk, n_blk, a.hist);
    bucket_scan_kernel<<<1, 1024, 0, st>>>(a.hist);
    bucket_scatter_kernel<<<n_blk, 1024, 0, st>>>(p, a.n, chunk, a.bbox_keys, a.prefilter, a.blk, a.hist,
                                                  reinterpret_cast<double2*>(a.sorted_pts), a.sorted_idx);
    *launches += 4;
    return cudaGetLastError();
}

int bucket_blocks(uint64_t n, int dev) {
    return (int)std::max<uint64_t>(1, std::min<uint64_t>((n + 4095) / 4096, (uint64_t)sms(dev)));
}

cudaError_t launch_unbucket(uint64_t n, const uint32_t* n_dev, const uint32_t* sorted_idx, const uint32_t* s_inside,
                            const uint32_t* s_aux, uint32_t* inside_bits, uint32_t* aux_bits, cudaStream_t st, int dev,
                            uint64_t* launches) {
    const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)sms(dev) * 8));
    unbucket_kernel<<<blocks, 256, 0, st>>>(n, n_dev, sorted_idx, s_inside, s_aux, inside_bits, aux_bits);
    ++*launches;
    return cudaGetLastError();
}

} // namespace pcd
