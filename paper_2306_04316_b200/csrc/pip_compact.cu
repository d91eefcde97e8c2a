// GPU prefilter_bbox / scatter_verdicts (reference
// batch.hpp:137-170, used by the CLI pipeline polycast_cli.cpp:78-80).
//
// prefilter_bbox: an order-preserving stream compaction of the points inside
// the closed box (BBox::contains, batch.hpp:39-41), with the original index of
// every retained point and the count of the others.  Three launches, all
// HBM-bound:
//   count    block b counts its chunk's in-box points (ballot + popc);
//   scan     exclusive scan of the per-block counts (one CTA) -> block bases,
//            total at [n_blk];
//   scatter  block b re-reads its chunk and writes each in-box point and its
//            index at base[b] + (in-block rank), in input order: warp ranks
//            from ballots, warp offsets from a shared-memory scan.
// scatter_verdicts: out[] is set to Outside, then out[idx[k]] = verdict[k]
// (batch.hpp:157-168); an index >= n_total raises a device flag (the host
// reports PC_EINVAL) instead of writing out of bounds.
#include "pip_kernels.h"

#include <cuda_runtime.h>

#include <algorithm>

namespace pcd {

namespace {

constexpr int kCThreads = 1024;
constexpr int kCWarps = kCThreads / 32;
constexpr unsigned kFullMask = 0xffffffffu;

struct Box {
    double x0, y0, x1, y1;
    __device__ __forceinline__ bool contains(double2 p) const {
        return p.x >= x0 && p.x <= x1 && p.y >= y0 && p.y <= y1;
    }
};

__global__ void __launch_bounds__(kCThreads) compact_count_kernel(const double2* __restrict__ pts, uint64_t n,
                                                                  uint64_t chunk, Box box,
                                                                  unsigned long long* __restrict__ blk) {
    __shared__ unsigned wsum[kCWarps];
    const uint64_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
    unsigned c = 0;
    for (uint64_t i = lo + threadIdx.x; i < hi; i += kCThreads) c += box.contains(pts[i]);
    c = __reduce_add_sync(kFullMask, c);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x < 32) {
        unsigned v = wsum[threadIdx.x];
        v = __reduce_add_sync(kFullMask, v);
        if (threadIdx.x == 0) blk[blockIdx.x] = v;
    }
}

// exclusive scan of blk[0 .. n_blk) in place; blk[n_blk] = total
__global__ void __launch_bounds__(kCThreads) compact_scan_kernel(unsigned long long* __restrict__ blk, int n_blk) {
    __shared__ unsigned long long wsum[kCWarps];
    __shared__ unsigned long long carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int base = 0; base < n_blk; base += kCThreads) {
        const int j = base + threadIdx.x;
        const unsigned long long v = j < n_blk ? blk[j] : 0ull;
        unsigned long long incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(kFullMask, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[w] = incl;
        __syncthreads();
        if (w == 0) {
            unsigned long long s = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(kFullMask, s, o);
                if (lane >= o) s += y;
            }
            wsum[lane] = s;
        }
        __syncthreads();
        const unsigned long long c0 = carry;
        if (j < n_blk) blk[j] = c0 + incl - v + (w ? wsum[w - 1] : 0ull);
        __syncthreads();
        if (threadIdx.x == kCThreads - 1) carry = c0 + wsum[kCWarps - 1];
        __syncthreads();
    }
    if (threadIdx.x == 0) blk[n_blk] = carry;
}

__global__ void __launch_bounds__(kCThreads) compact_scatter_kernel(const double2* __restrict__ pts, uint64_t n,
                                                                    uint64_t chunk, Box box,
                                                                    const unsigned long long* __restrict__ base,
                                                                    double2* __restrict__ out_pts,
                                                                    unsigned long long* __restrict__ out_idx) {
    __shared__ unsigned wcnt[kCWarps];
    __shared__ unsigned long long run_s;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
    if (threadIdx.x == 0) run_s = base[blockIdx.x];
    __syncthreads();
    for (uint64_t i0 = lo; i0 < hi; i0 += kCThreads) {
        const uint64_t i = i0 + threadIdx.x;
        double2 p = make_double2(0.0, 0.0);
        bool in = false;
        if (i < hi) {
            p = pts[i];
            in = box.contains(p);
        }
        const unsigned b = __ballot_sync(kFullMask, in);
        if (lane == 0) wcnt[w] = __popc(b);
        __syncthreads();
        // warp offsets: every warp scans the 32 warp counts with shuffles
        const unsigned c = wcnt[lane];
        unsigned incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(kFullMask, incl, o);
            if (lane >= o) incl += y;
        }
        const unsigned before = __shfl_sync(kFullMask, incl - c, w); // in-box points of the earlier warps
        const unsigned total = __shfl_sync(kFullMask, incl, 31);     // ... of the whole pass
        const unsigned long long run = run_s;
        if (in) {
            const unsigned long long pos = run + before + __popc(b & ((1u << lane) - 1u));
            out_pts[pos] = p;
            out_idx[pos] = i;
        }
        __syncthreads(); // everyone has read wcnt and run_s
        if (threadIdx.x == 0) run_s = run + total;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) scatter_verdicts_kernel(const unsigned long long* __restrict__ idx,
                                                               const uint8_t* __restrict__ v, uint64_t n_in,
                                                               uint64_t n_total, uint8_t* __restrict__ out,
                                                               unsigned* __restrict__ bad) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n_in; k += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long o = idx[k];
        if (o < n_total) out[o] = v[k];
        else atomicOr(bad, 1u);
    }
}

int sms(int dev) {
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
}

} // namespace

int compact_blocks(uint64_t n, int dev) {
    // >= 16 points per thread per block, at most 4 blocks per SM
    const uint64_t want = (n + 16ull * kCThreads - 1) / (16ull * kCThreads);
    return (int)std::max<uint64_t>(1, std::min<uint64_t>(want, 4ull * sms(dev)));
}

cudaError_t launch_prefilter(const double* pts, uint64_t n, const double box[4], int n_blk,
                             unsigned long long* blk, double* out_pts, unsigned long long* out_idx, cudaStream_t st,
                             uint64_t* launches) {
    const Box b{box[0], box[1], box[2], box[3]};
    const uint64_t chunk = (n + n_blk - 1) / n_blk;
    const double2* p = reinterpret_cast<const double2*>(pts);
    compact_count_kernel<<<n_blk, kCThreads, 0, st>>>(p, n, chunk, b, blk);
    compact_scan_kernel<<<1, kCThreads, 0, st>>>(blk, n_blk);
    compact_scatter_kernel<<<n_blk, kCThreads, 0, st>>>(p, n, chunk, b, blk, reinterpret_cast<double2*>(out_pts),
                                                         out_idx);
    *launches += 3;
    return cudaGetLastError();
}

cudaError_t launch_scatter_verdicts(const unsigned long long* idx, const uint8_t* v, uint64_t n_in, uint64_t n_total,
                                    uint8_t* out, unsigned* bad, cudaStream_t st, int dev, uint64_t* launches) {
    cudaError_t e = cudaMemsetAsync(out, 1 /* Verdict::Outside */, n_total, st);
    if (e != cudaSuccess || n_in == 0) return e;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n_in + 255) / 256, 8ull * sms(dev)));
    scatter_verdicts_kernel<<<grid, 256, 0, st>>>(idx, v, n_in, n_total, out, bad);
    ++*launches;
    return cudaGetLastError();
}

} // namespace pcd
