// y-ordering of query points (SIMT coherence for the single-polygon kernel).
//
// Why: the scan kernel (pip_single.cu) tests every edge's key range against the
// y range of a CTA's 4096 points, and classifies a warp's 512 points against
// the candidates together.  With points in input order both ranges are the
// whole polygon and every edge is a candidate; ordered by y, a CTA spans a thin
// slab and only the edges crossing it remain.  Points the bbox prefilter rejects
// (classify_batch, batch.hpp:200) get the largest key and are never classified
// (they are Outside), which is the GPU form of prefilter_bbox
// (batch.hpp:145-156).  Results are mapped back to the original order by index,
// so nothing depends on the order.  The scan over every (point, edge) pair is
// unchanged.
//
// Sort: 16-bit keys (65280 y levels over the outer ring's bbox, 0xffff =
// rejected), two LSD passes of 8 bits over (key, point, index), stable at tile
// granularity (rk_scatter_kernel); each
// pass reads its tile coalesced, ranks it in shared memory and writes
// contiguous runs per digit, so the points move in whole lines (a gather by
// index would pull a 128-byte line per 16-byte point).
//   rk_key_kernel      keys + per-tile digit counts (pass 1's re-counted over
//                      the pass-0 output by rk_count_hi_kernel)
//   rk_colscan_kernel  per (digit, tile) offsets: a CTA per digit scans its
//                      tiles, then one warp scans the 256 digit totals (two
//                      passes); one pass (<= 4M points) uses a decoupled
//                      look-back inside the scatter instead
//   rk_scatter_kernel  per tile: rank in shared memory (atomics on the tile's
//                      digit histogram), staged by digit, written out in
//                      contiguous runs per digit
#include "pip_kernels.h"

#include <cuda_runtime.h>

#include <algorithm>

#include "pip_device.cuh"

namespace pcd {

namespace {

#ifndef PC_RK_THREADS
#define PC_RK_THREADS 512
#endif
#ifndef PC_RK_MINB
#define PC_RK_MINB 2
#endif
#ifndef PC_RK_PF
#define PC_RK_PF 1
#endif
#ifndef PC_RK_PF_DIST
#define PC_RK_PF_DIST 64
#endif
constexpr int kRkThreads = PC_RK_THREADS;
constexpr int kRkItems = 8;                        // per thread
constexpr int kRkTile = kRkThreads * kRkItems;     // 4096 elements per tile (default)
constexpr int kRkWarps = kRkThreads / 32;
constexpr uint32_t kRkLevels = 65280;              // in-box keys 0 .. 65279 (high byte < 0xff)
constexpr uint16_t kRkReject = 0xffff;
constexpr uint64_t kRkOnePassMax = 1ull << 22; // up to this many points: one pass on the high byte

struct KeyMap {
    double minx, miny, maxx, maxy, scale;
    int prefilter;

    __device__ __forceinline__ uint32_t key(double x, double y) const {
        if (prefilter && !(x >= minx && x <= maxx && y >= miny && y <= maxy)) return kRkReject;
        const double t = (y - miny) * scale; // ordering only: no exactness needed
        const uint32_t k = t > 0.0 ? (uint32_t)fmin(t, (double)(kRkLevels - 1)) : 0u;
        return k;
    }
};

__device__ __forceinline__ KeyMap make_keymap(const unsigned long long* bbox_keys, int prefilter) {
    KeyMap m;
    m.minx = dkey_inv(bbox_keys[0]);
    m.miny = dkey_inv(bbox_keys[1]);
    m.maxx = dkey_inv(~bbox_keys[2]);
    m.maxy = dkey_inv(~bbox_keys[3]);
    const double h = m.maxy - m.miny;
    m.scale = (h > 0.0 && h < 1e300) ? kRkLevels / h : 0.0;
    m.prefilter = prefilter;
    return m;
}

// keys[i] for tile blockIdx.x; pass-0 digit counts, digit-major:
// cnt[0][digit * n_tiles + tile] (one pass: the high-digit totals instead)
__global__ void __launch_bounds__(kRkThreads) rk_key_kernel(const double2* __restrict__ pts, uint64_t n,
                                                            const unsigned long long* __restrict__ bbox_keys,
                                                            int prefilter, uint16_t* __restrict__ keys,
                                                            uint32_t* __restrict__ cnt, uint32_t n_tiles,
                                                            unsigned int* __restrict__ ticket,
                                                            uint32_t* __restrict__ tot1, uint32_t* __restrict__ status) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *ticket = 0u; // the colscan's completion counter
    __shared__ uint32_t h[2][256];
    for (int j = threadIdx.x; j < 512; j += blockDim.x) (&h[0][0])[j] = 0;
    __syncthreads();
    const KeyMap m = make_keymap(bbox_keys, prefilter);
    const uint64_t lo = (uint64_t)blockIdx.x * kRkTile, hi = min(n, lo + kRkTile);
    for (uint64_t i = lo + threadIdx.x; i < hi; i += kRkThreads) {
        const double2 p = pts[i];
        const uint32_t k = m.key(p.x, p.y);
        keys[i] = (uint16_t)k;
        if (tot1) atomicAdd(&h[1][k >> 8], 1u); // one pass: the high digit only
        else atomicAdd(&h[0][k & 0xff], 1u);    // two passes: pass 1 is recounted over the pass-0 output
    }
    __syncthreads();
    if (tot1) { // one pass with a look-back scan: high-digit totals, this tile's status row cleared
        for (int d = threadIdx.x; d < 256; d += blockDim.x) {
            if (h[1][d]) atomicAdd(&tot1[d], h[1][d]);
            status[(uint64_t)blockIdx.x * 256 + d] = 0u;
        }
        return;
    }
    for (int d = threadIdx.x; d < 256; d += blockDim.x) cnt[(uint64_t)d * n_tiles + blockIdx.x] = h[0][d];
}

// Pass-1 digit counts per tile of the pass-0 OUTPUT order (an LSD pass ranks
// within the order it reads): overwrites cnt[1][*][*].
__global__ void __launch_bounds__(kRkThreads) rk_count_hi_kernel(const uint16_t* __restrict__ keys, uint64_t n,
                                                                 uint32_t* __restrict__ cnt, uint32_t n_tiles) {
    __shared__ uint32_t h[256];
    for (int j = threadIdx.x; j < 256; j += blockDim.x) h[j] = 0;
    __syncthreads();
    const uint64_t lo = (uint64_t)blockIdx.x * kRkTile, hi = min(n, lo + kRkTile);
    for (uint64_t i = lo + threadIdx.x; i < hi; i += kRkThreads) atomicAdd(&h[keys[i] >> 8], 1u);
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += blockDim.x) cnt[256ull * n_tiles + (uint64_t)d * n_tiles + blockIdx.x] = h[d];
}

// One warp per (pass, digit): exclusive prefix over the tiles (in place) and
// the digit total; then (last CTA, one warp per pass) the exclusive scan of the
// 256 totals is added to every entry by the scatter kernel via base[pass][digit].
// Exclusive scan of 256 digit totals (one warp): base[digit]; the in-box
// count (keys below the reject key, i.e. everything before high digit 0xff)
// is the last pass's base[255].
__device__ __forceinline__ void rk_digit_bases(const uint32_t* tot, uint32_t* base, uint32_t* n_in, int lane) {
    uint32_t run = 0;
    for (int d0 = 0; d0 < 256; d0 += 32) {
        const uint32_t v = tot[d0 + lane];
        uint32_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        base[d0 + lane] = run + incl - v;
        if (n_in && d0 + lane == 255) *n_in = run + incl - v;
        run += __shfl_sync(0xffffffffu, incl, 31);
    }
}

// One CTA per (pass, digit) column in [first, last): exclusive prefix over the
// column's tiles (in place) and the digit total, 2048 tiles per round (8
// consecutive counts per thread, a block scan of the 256 thread sums); the last
// CTA to finish (ticket) then forms the digit bases of the passes it covered
// and resets the ticket.
constexpr int kCsThreads = 256;
__global__ void __launch_bounds__(kCsThreads) rk_colscan_kernel(uint32_t* __restrict__ cnt, uint32_t n_tiles,
                                                                uint32_t* __restrict__ tot, uint32_t first,
                                                                uint32_t last, uint32_t* __restrict__ base,
                                                                uint32_t* __restrict__ n_in,
                                                                unsigned int* __restrict__ ticket) {
    __shared__ uint32_t wsum[kCsThreads / 32];
    __shared__ bool is_last;
    const uint32_t wid = first + blockIdx.x; // pass * 256 + digit
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t* col = cnt + (uint64_t)wid * n_tiles;
    uint32_t run = 0;
    for (uint32_t c0 = 0; c0 < n_tiles; c0 += 8 * kCsThreads) {
        const uint32_t b = c0 + 8u * (uint32_t)tid;
        uint32_t v[8], ts = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            v[j] = b + j < n_tiles ? col[b + j] : 0u;
            ts += v[j];
        }
        // block-wide exclusive scan of the thread sums
        uint32_t incl = ts;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        uint32_t wpre = 0, rtot = 0;
#pragma unroll
        for (int w = 0; w < kCsThreads / 32; ++w) {
            const uint32_t x = wsum[w];
            wpre += w < warp ? x : 0u;
            rtot += x;
        }
        __syncthreads(); // wsum is rewritten next round
        uint32_t r = run + wpre + incl - ts;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (b + j < n_tiles) col[b + j] = r;
            r += v[j];
        }
        run += rtot;
    }
    if (tid == 0) tot[wid] = run;
    __threadfence();
    __syncthreads();
    if (tid == 0) is_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    for (uint32_t pass = first / 256; pass < last / 256; ++pass)
        if (warp == (int)(pass - first / 256)) rk_digit_bases(tot + pass * 256, base + pass * 256, pass == 1 ? n_in : nullptr, lane);
    if (tid == 0) *ticket = 0u;
}

struct RkShared {
    double2 spts[kRkTile];
    uint32_t hist[256];  // per digit: the tile's running count, then its start in the tile
    uint32_t gbase[256]; // global start of this tile's run of each digit
    uint32_t sidx[kRkTile];
    uint16_t skey[kRkTile];
};

// One counting-sort pass over tile blockIdx.x: (key, idx) -> position
// base[digit] + cnt[digit][tile] + (rank of the element among the tile's
// elements with that digit).  The rank inside a tile comes from shared-memory
// atomics, so elements of one digit may leave a tile in any order: the runs
// keep the tile order (the passes stay stable at tile granularity), and in the
// second pass a tile's elements of one high digit nearly all share the low
// digit too.  The y-order only steers performance -- every result is exact for
// any order (pip_single.cu) -- so this is all the scan kernel needs.
// PASS 0: idx = element position (implicit), writes keys_out and idx_out;
// PASS 1: writes idx_out only.
// LOOKBACK (one pass on the high digit, n <= kRkOnePassMax): instead of the
// column scan's offsets, the digit bases come from the totals rk_key_kernel
// accumulated and each tile's offsets from a decoupled look-back over the
// earlier tiles' published per-digit counts (status word: 1 << 30 | own count
// once counted, 2 << 30 | inclusive prefix once known); CTAs start in tile
// order, so a tile only ever waits on tiles already running.
template <int PASS, bool IMPLICIT = PASS == 0, bool LOOKBACK = false>
__global__ void __launch_bounds__(kRkThreads, PC_RK_MINB) rk_scatter_kernel(uint64_t n, const uint16_t* __restrict__ keys_in,
                                                                const double2* __restrict__ pts_in,
                                                                double2* __restrict__ pts_out,
                                                                const uint32_t* __restrict__ idx_in,
                                                                const uint32_t* __restrict__ cnt,
                                                                const uint32_t* __restrict__ base, uint32_t n_tiles,
                                                                uint16_t* __restrict__ keys_out,
                                                                uint32_t* __restrict__ idx_out,
                                                                const uint32_t* __restrict__ tot1 = nullptr,
                                                                uint32_t* status = nullptr,
                                                                uint32_t* __restrict__ n_in = nullptr) {
    extern __shared__ __align__(16) unsigned char rk_smem[];
    RkShared& S = *reinterpret_cast<RkShared*>(rk_smem);
    const int tid = threadIdx.x;
    const int shift = 8 * PASS;
    const uint64_t t0 = (uint64_t)blockIdx.x * kRkTile;
    const uint32_t tn = (uint32_t)min((uint64_t)kRkTile, n - t0);
#if PC_RK_PF
    // L2 prefetch of a later CTA's whole tile (keys, points, indices), as in the
    // scan kernel: that CTA's up-front requests then hit L2
    if (tid == 0) {
        const uint64_t nb = t0 + (uint64_t)PC_RK_PF_DIST * kRkTile;
        if (nb + kRkTile <= n) {
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pts_in + nb), "r"(kRkTile * 16u) : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(keys_in + nb), "r"(kRkTile * 2u) : "memory");
            if constexpr (!IMPLICIT)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(idx_in + nb), "r"(kRkTile * 4u) : "memory");
        }
    }
#endif
    // this thread's elements e = j * kRkThreads + tid: keys, indices and points
    // are all requested before the ranking, so their latency overlaps it
    uint32_t key[kRkItems], idx[IMPLICIT ? 1 : kRkItems];
    double2 pt[kRkItems];
#pragma unroll
    for (int j = 0; j < kRkItems; ++j) {
        const uint32_t e = j * kRkThreads + tid;
        const bool live = e < tn;
        key[j] = live ? (uint32_t)keys_in[t0 + e] : 0xffffffffu;
        if constexpr (!IMPLICIT) idx[j] = live ? idx_in[t0 + e] : 0u;
        pt[j] = live ? pts_in[t0 + e] : make_double2(0.0, 0.0);
    }
    if constexpr (LOOKBACK) {
        if (tid < 256) S.hist[tid] = 0;
        if (tid < 32) { // digit bases: exclusive scan of the totals (8 per lane)
            uint32_t v[8], sum = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                v[q] = tot1[tid * 8 + q];
                sum += v[q];
            }
            uint32_t incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (tid >= o) incl += y;
            }
            uint32_t run = incl - sum;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                S.gbase[tid * 8 + q] = run;
                run += v[q];
            }
            if (blockIdx.x == 0 && tid == 31 && n_in) *n_in = run - v[7]; // points below high digit 0xff: in the box
        }
    } else {
        for (int d = tid; d < 256; d += kRkThreads) {
            S.hist[d] = 0;
            S.gbase[d] = base[PASS * 256 + d] + cnt[(uint64_t)PASS * 256 * n_tiles + (uint64_t)d * n_tiles + blockIdx.x];
        }
    }
    __syncthreads();
    uint32_t rank[kRkItems];
#pragma unroll
    for (int j = 0; j < kRkItems; ++j)
        if (key[j] != 0xffffffffu) rank[j] = atomicAdd(&S.hist[(key[j] >> shift) & 0xffu], 1u);
    __syncthreads();
    if constexpr (LOOKBACK) {
        if (tid < 256) {
            volatile uint32_t* st = status;
            const uint32_t own = S.hist[tid];
            const uint64_t me = (uint64_t)blockIdx.x * 256 + tid;
            st[me] = (blockIdx.x == 0 ? 2u << 30 : 1u << 30) | own;
            uint32_t excl = 0;
            for (int64_t t = (int64_t)blockIdx.x - 1; t >= 0; --t) {
                uint32_t v;
                do {
                    v = st[(uint64_t)t * 256 + tid];
                } while ((v >> 30) == 0u);
                excl += v & 0x3fffffffu;
                if ((v >> 30) == 2u) break;
            }
            if (blockIdx.x > 0) st[me] = (2u << 30) | (excl + own);
            S.gbase[tid] += excl;
        }
        __syncthreads();
    }
    if (tid < 32) { // exclusive scan of the 256 digit counts by one warp (8 per lane)
        uint32_t v[8], sum = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            v[q] = S.hist[tid * 8 + q];
            sum += v[q];
        }
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (tid >= o) incl += y;
        }
        uint32_t run = incl - sum;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            S.hist[tid * 8 + q] = run;
            run += v[q];
        }
    }
    __syncthreads();
    // staged in digit order
#pragma unroll
    for (int j = 0; j < kRkItems; ++j) {
        if (key[j] == 0xffffffffu) continue;
        const uint32_t pos = S.hist[(key[j] >> shift) & 0xffu] + rank[j];
        PC_DCHECK(pos < tn);
        S.skey[pos] = (uint16_t)key[j];
        S.spts[pos] = pt[j];
        if constexpr (IMPLICIT) S.sidx[pos] = (uint32_t)(t0 + j * kRkThreads + tid);
        else S.sidx[pos] = idx[j];
    }
    __syncthreads();
    // contiguous runs per digit: element at tile position L goes to gbase[d] + (L - hist[d])
    for (uint32_t L = tid; L < tn; L += kRkThreads) {
        const uint32_t k = S.skey[L], d = (k >> shift) & 0xffu;
        const uint64_t g = (uint64_t)S.gbase[d] + (L - S.hist[d]);
        PC_DCHECK(g < n && L >= S.hist[d]);
        if (PASS == 0) keys_out[g] = (uint16_t)k;
        pts_out[g] = S.spts[L];
        idx_out[g] = S.sidx[L];
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
            PC_DCHECK(o < n);
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


uint64_t bucket_tiles(uint64_t n) { return std::max<uint64_t>(1, (n + kRkTile - 1) / kRkTile); }

size_t bucket_scratch_bytes(uint64_t n) {
    const uint64_t nt = bucket_tiles(n);
    // keys, keys1 (u16), idx1 (u32), pts1 (2 x f64), counts (2 x 256 x tiles), totals + bases (2 x 512),
    // look-back totals (256) and status (256 x tiles)
    return 2 * ((n * 2 + 15) / 16 * 16) + (n * 4 + 15) / 16 * 16 + n * 16 + 2 * 256 * nt * 4 + 4 * 512 * 4 + 80 +
           256 * 4 + 256 * nt * 4 + 32;
}

cudaError_t launch_bucket(const BucketArgs& a, cudaStream_t st, int dev, uint64_t* launches) {
    const double2* p = reinterpret_cast<const double2*>(a.pts);
    const uint64_t n = a.n, nt = bucket_tiles(n);
    char* sp = static_cast<char*>(a.scratch);
    auto take = [&](size_t bytes) {
        char* r = sp;
        sp += (bytes + 15) / 16 * 16;
        return r;
    };
    uint16_t* keys = reinterpret_cast<uint16_t*>(take(n * 2));
    uint16_t* keys1 = reinterpret_cast<uint16_t*>(take(n * 2));
    uint32_t* idx1 = reinterpret_cast<uint32_t*>(take(n * 4));
    double2* pts1 = reinterpret_cast<double2*>(take(n * 16));
    uint32_t* cnt = reinterpret_cast<uint32_t*>(take(2 * 256 * nt * 4));
    uint32_t* tot = reinterpret_cast<uint32_t*>(take(512 * 4));
    uint32_t* base = reinterpret_cast<uint32_t*>(take(512 * 4));
    unsigned int* ticket = reinterpret_cast<unsigned int*>(take(16));
    uint32_t* tot1 = reinterpret_cast<uint32_t*>(take(256 * 4));
    uint32_t* status = reinterpret_cast<uint32_t*>(take(256 * nt * 4));
    const bool one_pass = n <= kRkOnePassMax;
    if (one_pass) {
        const cudaError_t e = cudaMemsetAsync(tot1, 0, 256 * 4, st);
        if (e != cudaSuccess) return e;
    }
    rk_key_kernel<<<(unsigned)nt, kRkThreads, 0, st>>>(p, n, a.bbox_keys, a.prefilter, keys, cnt, (uint32_t)nt,
                                                       ticket, one_pass ? tot1 : nullptr, status);
    static bool attr[64] = {};
    if (dev >= 0 && dev < 64 && !attr[dev]) {
        cudaFuncSetAttribute(rk_scatter_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(RkShared));
        cudaFuncSetAttribute(rk_scatter_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(RkShared));
        cudaFuncSetAttribute(rk_scatter_kernel<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(RkShared));
        cudaFuncSetAttribute(rk_scatter_kernel<1, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(RkShared));
        attr[dev] = true;
    }
    const size_t sm = sizeof(RkShared);
    if (one_pass) {
        // one pass on the high byte (255 y levels): for up to ~4M points a CTA's
        // 4096 points span a slab this thin anyway; the tile offsets by look-back,
        // so the key pass and the scatter are the only launches
        rk_scatter_kernel<1, true, true><<<(unsigned)nt, kRkThreads, sm, st>>>(
            n, keys, p, reinterpret_cast<double2*>(a.sorted_pts), nullptr, cnt, base, (uint32_t)nt, nullptr,
            a.sorted_idx, tot1, status, a.n_in);
        *launches += 2;
        return cudaGetLastError();
    }
    // pass-0 offsets, totals and bases (pass 1's come from its recount below)
    rk_colscan_kernel<<<256, kCsThreads, 0, st>>>(cnt, (uint32_t)nt, tot, 0u, 256u, base, a.n_in, ticket);
    rk_scatter_kernel<0><<<(unsigned)nt, kRkThreads, sm, st>>>(n, keys, p, pts1, nullptr, cnt, base, (uint32_t)nt,
                                                              keys1, idx1);
    rk_count_hi_kernel<<<(unsigned)nt, kRkThreads, 0, st>>>(keys1, n, cnt, (uint32_t)nt);
    rk_colscan_kernel<<<256, kCsThreads, 0, st>>>(cnt, (uint32_t)nt, tot, 256u, 512u, base, a.n_in, ticket);
    rk_scatter_kernel<1><<<(unsigned)nt, kRkThreads, sm, st>>>(n, keys1, pts1,
                                                              reinterpret_cast<double2*>(a.sorted_pts), idx1, cnt,
                                                              base, (uint32_t)nt, nullptr, a.sorted_idx);
    *launches += 6;
    return cudaGetLastError();
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
