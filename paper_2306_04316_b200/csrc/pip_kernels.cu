// sm_100a kernels of the batched point-in-polygon path.
//
//   prep_edges_kernel   raw rings -> per-edge filter keys + exact records, bbox
//   pip_single_kernel   one polygon, (point tile x edge chunk) CTAs, edges staged
//                       through shared memory, K points per thread, XOR parity
//   pip_csr_kernel      many small polygons (CSR), one warp per polygon
//   finalize_kernel     bit planes -> verdict bytes + BatchStats
//   count_kernel        per-ring crossing counts (count_crossings_c1/_c2)
//
// Reference path replaced: classify_batch (proj/include/polycast/batch.hpp:184-230)
// -> contains (geometry.hpp:281-300) -> count_crossings_c1/_c2 /
// robust_ray_crossings (geometry.hpp:182-273).  See DESIGN.md for the layout
// and the exactness argument of the two-stage (filter + exact) edge test.
#include "pip_kernels.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>

#include "pip_device.cuh"

namespace pcd {

namespace {

constexpr int kTPB = 256;       // threads per CTA, single-polygon kernel
constexpr int kTile = 512;      // edges per shared-memory tile
constexpr int kWarpsCsr = 8;    // warps per CTA, CSR kernel

__device__ __forceinline__ uint32_t ring_of(const uint64_t* ring_off, uint32_t n_rings, uint64_t v) {
    // largest r with ring_off[r] <= v
    uint32_t lo = 0, hi = n_rings; // invariant: ring_off[lo] <= v < ring_off[hi]
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (ring_off[mid] <= v) lo = mid; else hi = mid;
    }
    return lo;
}

// One thread per vertex v: if (v, v+1) is an edge of the same ring, write its
// filter key pair and exact record at edge index e = v - ring(v).  Also folds
// the outer ring's vertices into the bbox (monotone-key atomics on memory
// pre-set to 0xff) and zeroes the output bit planes and stats.
template <int MODE>
__global__ void __launch_bounds__(256) prep_edges_kernel(
    const double* __restrict__ vx, const double* __restrict__ vy, const uint64_t* __restrict__ ring_off,
    uint32_t n_rings, uint64_t n_verts, uint2* __restrict__ filt, EdgeRec* __restrict__ rec,
    unsigned long long* __restrict__ bbox_keys, uint32_t* __restrict__ zero_words, uint64_t n_zero_words,
    unsigned long long* __restrict__ stats) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w = tid; w < n_zero_words; w += stride) zero_words[w] = 0u;
    if (tid < 4) stats[tid] = 0ull;

    const uint64_t outer_end = ring_off[1];
    unsigned long long kminx = ~0ull, kminy = ~0ull, kmaxx = ~0ull, kmaxy = ~0ull;
    for (uint64_t v = tid; v < n_verts; v += stride) {
        const double ax = vx[v], ay = vy[v];
        if (v < outer_end) {
            const unsigned long long kx = dkey(ax), ky = dkey(ay);
            kminx = min(kminx, kx);
            kminy = min(kminy, ky);
            kmaxx = min(kmaxx, ~kx);
            kmaxy = min(kmaxy, ~ky);
        }
        const uint32_t r = ring_of(ring_off, n_rings, v);
        if (v + 1 >= ring_off[r + 1]) continue; // last (closing) vertex of its ring
        const uint64_t e = v - r;
        const double bx = vx[v + 1], by = vy[v + 1];
        EdgeRec er;
#pragma unroll
        for (int i = 0; i < 8; ++i) er.d[i] = 0.0;
        er.d[0] = ax;
        er.d[1] = ay;
        er.d[2] = by;
        const double ylo = by < ay ? by : ay; // std::min(a.y, b.y)
        const double yhi = ay < by ? by : ay; // std::max(a.y, b.y)
        const int klo = fkey(ylo), khi = fkey(yhi);
        if (MODE == kC1) {
            double nx = __dsub_rn(by, ay), ny = __dsub_rn(ax, bx);
            if (nx < 0.0) {
                nx = -nx;
                ny = -ny;
            }
            er.d[3] = nx;
            er.d[4] = ny;
            filt[e] = make_uint2((uint32_t)klo, (uint32_t)khi - (uint32_t)klo);
        } else if (MODE == kC2) {
            er.d[3] = __dsub_rn(bx, ax);
            er.d[4] = __dsub_rn(by, ay);
            filt[e] = make_uint2((uint32_t)klo, (uint32_t)khi - (uint32_t)klo);
        } else {
            const double abx = __dsub_rn(bx, ax), aby = __dsub_rn(by, ay);
            er.d[3] = abx;
            er.d[4] = aby;
            er.d[5] = __dadd_rn(__dmul_rn(abx, abx), __dmul_rn(aby, aby));
            er.d[6] = ylo;
            er.d[7] = yhi;
            filt[e] = make_uint2((uint32_t)klo, (uint32_t)khi);
        }
        rec[e] = er;
    }
    // warp-reduce then one atomic per warp and key
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kminx = min(kminx, __shfl_xor_sync(0xffffffffu, kminx, o));
        kminy = min(kminy, __shfl_xor_sync(0xffffffffu, kminy, o));
        kmaxx = min(kmaxx, __shfl_xor_sync(0xffffffffu, kmaxx, o));
        kmaxy = min(kmaxy, __shfl_xor_sync(0xffffffffu, kmaxy, o));
    }
    if ((threadIdx.x & 31) == 0 && kminx != ~0ull) {
        atomicMin(&bbox_keys[0], kminx);
        atomicMin(&bbox_keys[1], kminy);
        atomicMin(&bbox_keys[2], kmaxx);
        atomicMin(&bbox_keys[3], kmaxy);
    }
}

// Single-polygon kernel.  CTA (bx, by) classifies points [bx*kTPB*K, +kTPB*K)
// against edges [by*chunk, +chunk).  Thread t owns points base + k*kTPB + t.
// Per staged edge: a 2-instruction integer range test per point decides
// "certainly not straddling" (exactly, see fkey); only candidates run the
// binary64 test of the reference.  Partial parities are XOR-ed into the
// inside plane, Error/Boundary OR-ed into the aux plane.
template <int MODE, int K>
__global__ void __launch_bounds__(kTPB) pip_single_kernel(
    const double2* __restrict__ pts, uint64_t n, const uint2* __restrict__ filt,
    const EdgeRec* __restrict__ rec, uint32_t n_edges, uint32_t edges_per_chunk,
    const unsigned long long* __restrict__ bbox_keys, int prefilter, double tol, double tol2,
    uint32_t* __restrict__ inside_bits, uint32_t* __restrict__ aux_bits, const uint32_t* __restrict__ n_dev) {
    __shared__ uint2 s_filt[kTile];
    extern __shared__ __align__(16) unsigned char s_dyn[];
    EdgeRec* s_rec = reinterpret_cast<EdgeRec*>(s_dyn);

    const uint32_t e_begin = blockIdx.y * edges_per_chunk;
    const uint32_t e_end = min(n_edges, e_begin + edges_per_chunk);
    const uint64_t base = (uint64_t)blockIdx.x * (kTPB * K);
    const int tid = threadIdx.x;
    if (n_dev) n = min(n, (uint64_t)*n_dev); // bucketed input: only the in-box prefix is live
    if (base >= n) return;

    double minx = 0, miny = 0, maxx = 0, maxy = 0;
    if (prefilter) {
        minx = dkey_inv(bbox_keys[0]);
        miny = dkey_inv(bbox_keys[1]);
        maxx = dkey_inv(~bbox_keys[2]);
        maxy = dkey_inv(~bbox_keys[3]);
    }

    double px[K], py[K];
    int ka[K], kb[K]; // C1/C2: ka = kb = key(p.y); Robust: ka = key(p.y+tol), kb = key(p.y-tol)
    int cnt[K];
    bool aux[K], act[K];
    bool any_act = false;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const uint64_t i = base + (uint64_t)k * kTPB + tid;
        cnt[k] = 0;
        aux[k] = false;
        act[k] = i < n;
        double2 p = make_double2(0.0, 0.0);
        if (act[k]) p = pts[i];
        px[k] = p.x;
        py[k] = p.y;
        if (act[k] && prefilter)
            act[k] = p.x >= minx && p.x <= maxx && p.y >= miny && p.y <= maxy; // batch.hpp:39-41
        if (MODE == kRobust) {
            ka[k] = act[k] ? fkey(__dadd_rn(p.y, tol)) : INT_MIN;
            kb[k] = act[k] ? fkey(__dsub_rn(p.y, tol)) : INT_MAX;
        } else {
            ka[k] = act[k] ? fkey(p.y) : INT_MAX;
            kb[k] = ka[k];
        }
        any_act |= act[k];
    }
    if (!__syncthreads_or(any_act)) return;

    for (uint32_t t0 = e_begin; t0 < e_end; t0 += kTile) {
        const uint32_t nt = min((uint32_t)kTile, e_end - t0);
        __syncthreads();
        for (uint32_t j = tid; j < nt; j += kTPB) s_filt[j] = filt[t0 + j];
        {
            const float4* src = reinterpret_cast<const float4*>(rec + t0);
            float4* dst = reinterpret_cast<float4*>(s_rec);
            for (uint32_t j = tid; j < nt * 4; j += kTPB) dst[j] = src[j];
        }
        __syncthreads();
        if (!any_act) continue;
#pragma unroll 2
        for (uint32_t e = 0; e < nt; ++e) {
            const uint2 f = s_filt[e];
            bool c[K];
            bool any = false;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (MODE == kRobust)
                    c[k] = ka[k] >= (int)f.x && kb[k] <= (int)f.y;
                else
                    c[k] = (uint32_t)(ka[k] - (int)f.x) <= f.y;
                any |= c[k];
            }
            if (any) {
                const EdgeRec r = s_rec[e];
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    if (c[k]) {
                        if (MODE == kRobust) {
                            exact_robust(px[k], py[k], tol, tol2, r, cnt[k], aux[k]);
                        } else {
                            const uint32_t d = (uint32_t)(ka[k] - (int)f.x); // 0..range; strict inside => sure
                            const bool sure = d != 0u && d != f.y;
                            if (MODE == kC1) exact_c1(px[k], py[k], r, cnt[k], sure);
                            else exact_c2(px[k], py[k], r, cnt[k], aux[k], sure);
                        }
                    }
                }
            }
        }
    }

    const int lane = tid & 31;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const uint64_t i0 = base + (uint64_t)k * kTPB + (tid & ~31);
        const uint32_t b = __ballot_sync(0xffffffffu, act[k] && (cnt[k] & 1));
        const uint32_t a = __ballot_sync(0xffffffffu, act[k] && aux[k]);
        if (lane == 0 && i0 < n) {
            if (b) atomicXor(&inside_bits[i0 >> 5], b);
            if (a) atomicOr(&aux_bits[i0 >> 5], a);
        }
    }
}

// CSR kernel: one warp per polygon (grid-stride).  The warp reduces the outer
// ring's bbox, then walks its points 32 at a time; each lane runs the literal
// reference loop over every ring edge (vertex loads are warp-uniform
// broadcasts).  Flags are OR-ed into the bit planes (polygon point ranges need
// not be 32-aligned).
template <int MODE>
__global__ void __launch_bounds__(kWarpsCsr * 32) pip_csr_kernel(
    const double2* __restrict__ pts, const uint64_t* __restrict__ pt_off, uint64_t n_polys,
    const double* __restrict__ vx, const double* __restrict__ vy, const uint64_t* __restrict__ ring_off,
    const uint64_t* __restrict__ poly_ring_off, uint64_t pt_base, uint64_t ring_base, uint64_t vert_base,
    double tol, double tol2, uint32_t* __restrict__ inside_bits, uint32_t* __restrict__ aux_bits) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t p = warp; p < n_polys; p += nwarps) {
        const uint64_t r0 = poly_ring_off[p] - ring_base, r1 = poly_ring_off[p + 1] - ring_base;
        const uint64_t s = pt_off[p] - pt_base, t = pt_off[p + 1] - pt_base;
        if (s == t) continue;
        double minx = INFINITY, miny = INFINITY, maxx = -INFINITY, maxy = -INFINITY;
        if (r1 > r0) {
            for (uint64_t v = ring_off[r0] - vert_base + lane; v < ring_off[r0 + 1] - vert_base; v += 32) {
                const double x = vx[v], y = vy[v];
                minx = x < minx ? x : minx;
                miny = y < miny ? y : miny;
                maxx = maxx < x ? x : maxx;
                maxy = maxy < y ? y : maxy;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double a = __shfl_xor_sync(0xffffffffu, minx, o);
                const double b = __shfl_xor_sync(0xffffffffu, miny, o);
                const double c = __shfl_xor_sync(0xffffffffu, maxx, o);
                const double d = __shfl_xor_sync(0xffffffffu, maxy, o);
                minx = a < minx ? a : minx;
                miny = b < miny ? b : miny;
                maxx = maxx < c ? c : maxx;
                maxy = maxy < d ? d : maxy;
            }
        }
        for (uint64_t c0 = s; c0 < t; c0 += 32) {
            const uint64_t i = c0 + lane;
            bool act = i < t;
            double2 q = make_double2(0.0, 0.0);
            if (act) q = pts[i];
            act = act && r1 > r0 && q.x >= minx && q.x <= maxx && q.y >= miny && q.y <= maxy;
            int cnt = 0;
            bool aux = false;
            if (__any_sync(0xffffffffu, act)) {
                for (uint64_t r = r0; r < r1; ++r) {
                    const uint64_t lo = ring_off[r] - vert_base, hi = ring_off[r + 1] - vert_base;
                    if (hi - lo < 2) continue;
                    double ax = vx[lo], ay = vy[lo];
                    double f_prev = __dsub_rn(ay, q.y);
                    for (uint64_t v = lo + 1; v < hi; ++v) {
                        const double bx = vx[v], by = vy[v];
                        raw_edge<MODE>(q.x, q.y, tol, tol2, ax, ay, bx, by, f_prev, cnt, aux);
                        ax = bx;
                        ay = by;
                    }
                }
            }
            const uint32_t bi = __ballot_sync(0xffffffffu, act && (cnt & 1) && !aux);
            const uint32_t ba = __ballot_sync(0xffffffffu, act && aux);
            if (lane == 0) {
                const uint64_t w = c0 >> 5;
                const uint32_t sh = (uint32_t)(c0 & 31);
                if (bi) {
                    atomicOr(&inside_bits[w], bi << sh);
                    if (sh && (bi >> (32 - sh))) atomicOr(&inside_bits[w + 1], bi >> (32 - sh));
                }
                if (ba) {
                    atomicOr(&aux_bits[w], ba << sh);
                    if (sh && (ba >> (32 - sh))) atomicOr(&aux_bits[w + 1], ba >> (32 - sh));
                }
            }
        }
    }
}

// Bit planes -> verdict bytes + stats.  One thread per 32-point word.
// stats = {inside, outside, boundary, error}; aux counts go to slot aux_slot.
__global__ void __launch_bounds__(256) finalize_kernel(uint64_t n, uint32_t* __restrict__ inside_bits,
                                                       const uint32_t* __restrict__ aux_bits,
                                                       uint8_t* __restrict__ verdicts, int aux_verdict,
                                                       unsigned long long* __restrict__ stats) {
    const uint64_t nwords = (n + 31) >> 5;
    unsigned long long c_in = 0, c_aux = 0, c_out = 0;
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords;
         w += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t a = aux_bits[w];
        const uint32_t in = inside_bits[w] & ~a;
        inside_bits[w] = in;
        const uint64_t lo = w << 5;
        const uint32_t valid = (uint32_t)min((uint64_t)32, n - lo);
        const uint32_t vmask = valid == 32 ? 0xffffffffu : ((1u << valid) - 1u);
        c_in += __popc(in & vmask);
        c_aux += __popc(a & vmask);
        c_out += valid - __popc((in | a) & vmask);
        if (verdicts) {
            uint8_t* dst = verdicts + lo;
            if (valid == 32 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
                uint32_t wv[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    uint32_t word = 0;
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        const int bit = q * 4 + b;
                        const uint32_t v = ((a >> bit) & 1u) ? (uint32_t)aux_verdict
                                                              : (((in >> bit) & 1u) ? 0u : 1u);
                        word |= v << (8 * b);
                    }
                    wv[q] = word;
                }
                reinterpret_cast<uint4*>(dst)[0] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
                reinterpret_cast<uint4*>(dst)[1] = make_uint4(wv[4], wv[5], wv[6], wv[7]);
            } else {
                for (uint32_t bit = 0; bit < valid; ++bit)
                    dst[bit] = ((a >> bit) & 1u) ? (uint8_t)aux_verdict : (((in >> bit) & 1u) ? 0 : 1);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        c_in += __shfl_xor_sync(0xffffffffu, c_in, o);
        c_aux += __shfl_xor_sync(0xffffffffu, c_aux, o);
        c_out += __shfl_xor_sync(0xffffffffu, c_out, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (c_in) atomicAdd(&stats[0], c_in);
        if (c_out) atomicAdd(&stats[1], c_out);
        if (c_aux) atomicAdd(&stats[aux_verdict == 2 ? 2 : 3], c_aux);
    }
}

// count_crossings_c1/_c2 of one ring: one thread per point, literal loop.
template <int MODE>
__global__ void __launch_bounds__(256) count_kernel(const double2* __restrict__ pts, uint64_t n,
                                                    const double* __restrict__ vx,
                                                    const double* __restrict__ vy, uint64_t nv,
                                                    unsigned long long* __restrict__ counts,
                                                    uint8_t* __restrict__ degenerate) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double2 q = pts[i];
    int cnt = 0;
    bool aux = false;
    if (nv >= 2) {
        double ax = vx[0], ay = vy[0];
        double f_prev = __dsub_rn(ay, q.y);
        for (uint64_t v = 1; v < nv; ++v) {
            const double bx = vx[v], by = vy[v];
            raw_edge<MODE>(q.x, q.y, 0.0, 0.0, ax, ay, bx, by, f_prev, cnt, aux);
            ax = bx;
            ay = by;
        }
    }
    counts[i] = (unsigned long long)cnt;
    degenerate[i] = aux ? 1 : 0;
}

// FP64 add/multiply throughput probe: 8 independent DMUL->DADD chains per
// thread (no FMA), the instruction mix of the binary64 crossing test.
__global__ void __launch_bounds__(256) fp64_probe_kernel(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = 1.0 + 1e-3 * (threadIdx.x + k);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = __dadd_rn(__dmul_rn(x[k], a), b);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s = __dadd_rn(s, x[k]);
    if (s == 12345.678) out[0] = s; // practically never; keeps the chains live
}

int sm_count(int dev) {
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
}

template <int MODE, int K>
cudaError_t launch_single_t(const SingleArgs& a, cudaStream_t st, int dev, uint64_t* launches) {
    const uint32_t pts_per_cta = kTPB * K;
    const uint64_t n_ptiles = (a.n + pts_per_cta - 1) / pts_per_cta;
    const size_t dyn = sizeof(EdgeRec) * kTile;
    static bool attr_set[64] = {};
    if (dev < 64 && !attr_set[dev]) {
        cudaFuncSetAttribute(pip_single_kernel<MODE, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        attr_set[dev] = true;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pip_single_kernel<MODE, K>, kTPB, dyn);
    if (per_sm < 1) per_sm = 1;
    const uint64_t slots = (uint64_t)sm_count(dev) * per_sm;
    // Split the edge range so the grid covers >= ~4 waves, chunks >= one tile.
    const uint64_t max_chunks = std::max<uint64_t>(1, (a.n_edges + kTile - 1) / kTile);
    uint64_t chunks = std::max<uint64_t>(1, (4 * slots + n_ptiles - 1) / std::max<uint64_t>(n_ptiles, 1));
    chunks = std::min<uint64_t>(std::min<uint64_t>(chunks, max_chunks), 65535);
    const uint32_t per_chunk = (uint32_t)((a.n_edges + chunks - 1) / chunks);
    chunks = a.n_edges ? (a.n_edges + per_chunk - 1) / per_chunk : 1;
    dim3 grid((unsigned)n_ptiles, (unsigned)chunks);
    pip_single_kernel<MODE, K><<<grid, kTPB, dyn, st>>>(
        reinterpret_cast<const double2*>(a.pts), a.n, a.filt, reinterpret_cast<const EdgeRec*>(a.rec),
        a.n_edges, per_chunk ? per_chunk : 1, a.bbox_keys, a.prefilter, a.tol, a.tol2, a.inside_bits,
        a.aux_bits, a.n_dev);
    ++*launches;
    return cudaGetLastError();
}

} // namespace

size_t edge_rec_bytes() { return sizeof(EdgeRec); }

cudaError_t launch_fp64_probe(double* out, int iters, int dev, cudaStream_t st, double* flops) {
    const unsigned blocks = (unsigned)sm_count(dev) * 8;
    fp64_probe_kernel<<<blocks, 256, 0, st>>>(out, iters, 0.9999999, 1e-7);
    *flops = (double)blocks * 256.0 * iters * 8.0 * 2.0;
    return cudaGetLastError();
}

cudaError_t launch_prep(const PrepArgs& a, cudaStream_t st, int dev, uint64_t* launches) {
    cudaError_t e = cudaMemsetAsync(a.bbox_keys, 0xff, 4 * sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    const uint64_t work = std::max<uint64_t>(a.n_verts, a.n_zero_words);
    const unsigned blocks = (unsigned)std::min<uint64_t>((work + 255) / 256 + 1, (uint64_t)sm_count(dev) * 16);
    switch (a.mode) {
    case kC1:
        prep_edges_kernel<kC1><<<blocks, 256, 0, st>>>(a.vx, a.vy, a.ring_off, a.n_rings, a.n_verts, a.filt,
                                                       reinterpret_cast<EdgeRec*>(a.rec), a.bbox_keys,
                                                       a.zero_words, a.n_zero_words, a.stats);
        break;
    case kC2:
        prep_edges_kernel<kC2><<<blocks, 256, 0, st>>>(a.vx, a.vy, a.ring_off, a.n_rings, a.n_verts, a.filt,
                                                       reinterpret_cast<EdgeRec*>(a.rec), a.bbox_keys,
                                                       a.zero_words, a.n_zero_words, a.stats);
        break;
    default:
        prep_edges_kernel<kRobust><<<blocks, 256, 0, st>>>(a.vx, a.vy, a.ring_off, a.n_rings, a.n_verts,
                                                           a.filt, reinterpret_cast<EdgeRec*>(a.rec),
                                                           a.bbox_keys, a.zero_words, a.n_zero_words,
                                                           a.stats);
        break;
    }
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_single(const SingleArgs& a, cudaStream_t st, int dev, uint64_t* launches) {
    if (a.n == 0) return cudaSuccess;
    switch (a.mode) {
    case kC1: return launch_single_t<kC1, 8>(a, st, dev, launches);
    case kC2: return launch_single_t<kC2, 8>(a, st, dev, launches);
    default: return launch_single_t<kRobust, 8>(a, st, dev, launches);
    }
}

cudaError_t launch_csr(const CsrArgs& a, cudaStream_t st, int dev, uint64_t* launches) {
    if (a.n_polys == 0) return cudaSuccess;
    const uint64_t want = (a.n_polys + kWarpsCsr - 1) / kWarpsCsr;
    const unsigned blocks = (unsigned)std::min<uint64_t>(want, (uint64_t)sm_count(dev) * 64);
    const dim3 tpb(kWarpsCsr * 32);
    const double2* p = reinterpret_cast<const double2*>(a.pts);
    switch (a.mode) {
    case kC1:
        pip_csr_kernel<kC1><<<blocks, tpb, 0, st>>>(p, a.pt_off, a.n_polys, a.vx, a.vy, a.ring_off, a.poly_ring_off,
                                                    a.pt_base, a.ring_base, a.vert_base, a.tol, a.tol2, a.inside_bits, a.aux_bits);
        break;
    case kC2:
        pip_csr_kernel<kC2><<<blocks, tpb, 0, st>>>(p, a.pt_off, a.n_polys, a.vx, a.vy, a.ring_off, a.poly_ring_off,
                                                    a.pt_base, a.ring_base, a.vert_base, a.tol, a.tol2, a.inside_bits, a.aux_bits);
        break;
    default:
        pip_csr_kernel<kRobust><<<blocks, tpb, 0, st>>>(p, a.pt_off, a.n_polys, a.vx, a.vy, a.ring_off,
                                                        a.poly_ring_off, a.pt_base, a.ring_base, a.vert_base, a.tol, a.tol2, a.inside_bits,
                                                        a.aux_bits);
        break;
    }
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_finalize(uint64_t n, uint32_t* inside_bits, const uint32_t* aux_bits, uint8_t* verdicts,
                            int mode, unsigned long long* stats, cudaStream_t st, int dev, uint64_t* launches) {
    if (n == 0) return cudaSuccess;
    const uint64_t nwords = (n + 31) >> 5;
    const unsigned blocks = (unsigned)std::min<uint64_t>((nwords + 255) / 256, (uint64_t)sm_count(dev) * 8);
    finalize_kernel<<<blocks, 256, 0, st>>>(n, inside_bits, aux_bits, verdicts, mode == kRobust ? 2 : 3, stats);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_count(const double* pts, uint64_t n, const double* vx, const double* vy, uint64_t nv, int mode,
                         unsigned long long* counts, uint8_t* degenerate, cudaStream_t st, uint64_t* launches) {
    if (n == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)((n + 255) / 256);
    const double2* p = reinterpret_cast<const double2*>(pts);
    if (mode == kC1) count_kernel<kC1><<<blocks, 256, 0, st>>>(p, n, vx, vy, nv, counts, degenerate);
    else count_kernel<kC2><<<blocks, 256, 0, st>>>(p, n, vx, vy, nv, counts, degenerate);
    ++*launches;
    return cudaGetLastError();
}

} // namespace pcd
