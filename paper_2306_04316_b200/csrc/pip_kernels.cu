// sm_100a kernels of the batched point-in-polygon path.
//
//   prep_bbox_kernel    outer-ring bbox, zeroed planes/stats
//   prep_edges_kernel   raw rings -> per-edge filter keys + exact records
//   (the single-polygon kernel lives in pip_single.cu)
//   (the CSR multi-polygon kernel lives in pip_csr.cu, bucketing in pip_sort.cu)
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


__device__ __forceinline__ uint32_t ring_of(const uint64_t* ring_off, uint32_t n_rings, uint64_t v) {
    // largest r with ring_off[r] <= v
    uint32_t lo = 0, hi = n_rings; // invariant: ring_off[lo] <= v < ring_off[hi]
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (ring_off[mid] <= v) lo = mid; else hi = mid;
    }
    return lo;
}

// Outer-ring bbox (monotone-key atomics on memory pre-set to 0xff), plus
// zeroing of the output plane and stats.  Runs before prep_edges_kernel, which
// needs the bbox for the 16-bit key map.
__global__ void __launch_bounds__(256) prep_bbox_kernel(const double* __restrict__ vx, const double* __restrict__ vy,
                                                        const uint64_t* __restrict__ ring_off,
                                                        unsigned long long* __restrict__ bbox_keys,
                                                        uint32_t* __restrict__ zero_words, uint32_t* __restrict__ zero_words2,
                                                        uint64_t n_zero_words, unsigned long long* __restrict__ stats) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w = tid; w < n_zero_words; w += stride) {
        zero_words[w] = 0u;
        zero_words2[w] = 0u;
    }
    if (tid < 4) stats[tid] = 0ull;
    const uint64_t outer_end = ring_off[1];
    unsigned long long kminx = ~0ull, kminy = ~0ull, kmaxx = ~0ull, kmaxy = ~0ull;
    for (uint64_t v = tid; v < outer_end; v += stride) {
        const unsigned long long kx = dkey(vx[v]), ky = dkey(vy[v]);
        kminx = min(kminx, kx);
        kminy = min(kminy, ky);
        kmaxx = min(kmaxx, ~kx);
        kmaxy = min(kmaxy, ~ky);
    }
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

// One thread per vertex v: if (v, v+1) is an edge of the same ring, write its
// filter word, key word and exact record at edge index e = v - ring(v).
//   key halves (all modes), on the 15-bit map, for the phase-1 key scan of
//          pip_single.cu: per group of 8 edges, 8 words = 16 halves: half j is
//          q(ylo) of edge j, half 8 + j is 0x7fff - q(yhi) of edge j (word 2i
//          / 2i+1 thus pairs edges 2i, 2i+1 in its low / high half, so one
//          packed add-max tests two edges); padding edges (>= n_edges up to
//          qk_words) have both halves 0x7fff, which never matches (keys <= 0x7ffe)
//   filter word C1/C2: {(-q(ylo) mod 2^15) << 1 in both 16-bit halves,
//          ((q(yhi) - q(ylo)) << 1) + 2 in both halves} (15-bit keys)
//   filter word Robust: {fkey(ylo), fkey(yhi)} (32-bit keys)
template <int MODE>
__device__ __forceinline__ void prep_edges_body(
    const double* __restrict__ vx, const double* __restrict__ vy, const uint64_t* __restrict__ ring_off,
    uint32_t n_rings, uint64_t n_verts, uint2* __restrict__ filt, uint32_t* __restrict__ qk, uint64_t n_qk,
    EdgeRec* __restrict__ rec, unsigned long long* __restrict__ bbox_keys, double tol, uint64_t tid,
    uint64_t stride) {
    const QMap qm = qmap_from_bbox(bbox_keys);
    const LocalMap lm = local_map_from_bbox(bbox_keys);
    if (tid == 0) { // published for the classify kernels (bbox_keys[4..7])
        reinterpret_cast<double*>(bbox_keys)[4] = qm.y0;
        reinterpret_cast<double*>(bbox_keys)[5] = qm.scale;
        reinterpret_cast<double*>(bbox_keys)[6] = lm.sx;
        reinterpret_cast<double*>(bbox_keys)[7] = lm.sy;
    }
    uint16_t* const qh = reinterpret_cast<uint16_t*>(qk);
    for (uint64_t e = n_verts - n_rings + tid; e < n_qk; e += stride) {
        qh[qk_half(e)] = 0x7fffu;
        qh[qk_half(e) + 8] = 0x7fffu;
    }
    for (uint64_t v = tid; v < n_verts; v += stride) {
        const uint32_t r = ring_of(ring_off, n_rings, v);
        if (v + 1 >= ring_off[r + 1]) continue; // last (closing) vertex of its ring
        const uint64_t e = v - r;
        const double ax = vx[v], ay = vy[v], bx = vx[v + 1], by = vy[v + 1];
        EdgeRec er;
#pragma unroll
        for (int i = 0; i < 8; ++i) er.d[i] = 0.0;
        er.d[0] = ax;
        er.d[1] = ay;
        er.d[2] = by;
        const double ylo = by < ay ? by : ay; // std::min(a.y, b.y)
        const double yhi = ay < by ? by : ay; // std::max(a.y, b.y)
        if (MODE == kRobust) {
            const double abx = __dsub_rn(bx, ax), aby = __dsub_rn(by, ay);
            er.d[3] = abx;
            er.d[4] = aby;
            er.d[5] = __dadd_rn(__dmul_rn(abx, abx), __dmul_rn(aby, aby));
            // fp32 record of the intercept sign (as C2: same expression), valid only
            // while tol is far below the polygon's size (then a decided sign also
            // rules out the boundary): d[6] = {Nx, Ny}, d[7] = {c + B, 0}
            LocalMap lr = lm;
            lr.c2ok = lm.c2ok && tol >= 0.0 && __dmul_rn(__dmul_rn(tol, 2.0), fmax(lm.sx, lm.sy)) <= 0x1p-30;
            const float3 fr = local_side_record_c2(lr, ax, ay, bx, by, abx, aby);
            er.d[6] = __hiloint2double(__float_as_int(fr.y), __float_as_int(fr.x));
            er.d[7] = __hiloint2double(0, __float_as_int(fr.z));
            filt[e] = make_uint2((uint32_t)fkey(ylo), (uint32_t)fkey(yhi));
        } else {
            if (MODE == kC1) {
                double nx = __dsub_rn(by, ay), ny = __dsub_rn(ax, bx);
                if (nx < 0.0) {
                    nx = -nx;
                    ny = -ny;
                }
                er.d[3] = nx;
                er.d[4] = ny;
                // fp32 side-test record (d[5] = {Nx, Ny}, d[6] = {c, 0}): see
                // LocalMap; NaN when unusable (every test then goes exact)
                const float3 fr = local_side_record(lm, ax, ay, bx, by, nx, ny);
                er.d[5] = __hiloint2double(__float_as_int(fr.y), __float_as_int(fr.x));
                er.d[6] = __hiloint2double(0, __float_as_int(fr.z));
            } else {
                er.d[3] = __dsub_rn(bx, ax);
                er.d[4] = __dsub_rn(by, ay);
                // fp32 side-test record of the intercept sign (d[5] = {Nx, Ny}, d[6] = {c + B, 0})
                const float3 fr = local_side_record_c2(lm, ax, ay, bx, by, er.d[3], er.d[4]);
                er.d[5] = __hiloint2double(__float_as_int(fr.y), __float_as_int(fr.x));
                er.d[6] = __hiloint2double(0, __float_as_int(fr.z));
            }
            const uint32_t klo = qkey15(ylo, qm), khi = qkey15(yhi, qm);
            const uint32_t neg = ((0x8000u - klo) & 0x7fffu) << 1; // -q(ylo) mod 2^15, guard bit clear
            // threshold + 1 in both halves: candidate iff min(d_lo, d_hi) < ((khi - klo) << 1) + 2
            // (<= 65534 since keys are <= 32766), see lane_candidate (pip_single.cu)
            const uint32_t thr1 = ((khi - klo) << 1) + 2u;
            filt[e] = make_uint2(neg | (neg << 16), thr1 | (thr1 << 16));
        }
        qh[qk_half(e)] = (uint16_t)qkey15(ylo, qm);
        qh[qk_half(e) + 8] = (uint16_t)(0x7fffu - qkey15(yhi, qm));
        rec[e] = er;
    }
}

template <int MODE>
__global__ void __launch_bounds__(256) prep_edges_kernel(
    const double* __restrict__ vx, const double* __restrict__ vy, const uint64_t* __restrict__ ring_off,
    uint32_t n_rings, uint64_t n_verts, uint2* __restrict__ filt, uint32_t* __restrict__ qk, uint64_t n_qk,
    EdgeRec* __restrict__ rec, unsigned long long* __restrict__ bbox_keys, double tol) {
    prep_edges_body<MODE>(vx, vy, ring_off, n_rings, n_verts, filt, qk, n_qk, rec, bbox_keys, tol,
                          blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, (uint64_t)gridDim.x * blockDim.x);
}

// Polygons of up to kPrepSmall vertices: the whole prep in one launch -- CTA 0
// does the stats zeroing, the outer-ring bbox (a block reduction instead of
// atomics, so no pre-set) and the edge records, the other CTAs clear the
// output planes -- one launch instead of a memset and two.
constexpr int kPrepThreads = 1024;
constexpr uint64_t kPrepSmall = 16384;
constexpr uint64_t kPrepZero = 8192; // plane words cleared per extra CTA of prep_small_kernel
template <int MODE>
__global__ void __launch_bounds__(kPrepThreads) prep_small_kernel(
    const double* __restrict__ vx, const double* __restrict__ vy, const uint64_t* __restrict__ ring_off,
    uint32_t n_rings, uint64_t n_verts, uint2* __restrict__ filt, uint32_t* __restrict__ qk, uint64_t n_qk,
    EdgeRec* __restrict__ rec, unsigned long long* __restrict__ bbox_keys, double tol,
    uint32_t* __restrict__ zero_words, uint32_t* __restrict__ zero_words2, uint64_t n_zero_words,
    unsigned long long* __restrict__ stats) {
    __shared__ unsigned long long red[kPrepThreads / 32][4];
    const uint32_t tid = threadIdx.x;
    if (blockIdx.x > 0) { // the other CTAs clear the output planes, kPrepZero words each
        const uint64_t w0 = (uint64_t)(blockIdx.x - 1) * kPrepZero, w1 = min(n_zero_words, w0 + kPrepZero);
        for (uint64_t w = w0 + tid; w < w1; w += kPrepThreads) {
            zero_words[w] = 0u;
            zero_words2[w] = 0u;
        }
        return;
    }
    if (tid < 4) stats[tid] = 0ull;
    unsigned long long k[4] = {~0ull, ~0ull, ~0ull, ~0ull};
    for (uint64_t v = tid; v < ring_off[1]; v += kPrepThreads) {
        const unsigned long long kx = dkey(vx[v]), ky = dkey(vy[v]);
        k[0] = min(k[0], kx);
        k[1] = min(k[1], ky);
        k[2] = min(k[2], ~kx);
        k[3] = min(k[3], ~ky);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int j = 0; j < 4; ++j) k[j] = min(k[j], __shfl_xor_sync(0xffffffffu, k[j], o));
    if ((tid & 31) == 0)
#pragma unroll
        for (int j = 0; j < 4; ++j) red[tid >> 5][j] = k[j];
    __syncthreads();
    if (tid < 4) {
        unsigned long long m = ~0ull;
        for (int w = 0; w < kPrepThreads / 32; ++w) m = min(m, red[w][tid]);
        bbox_keys[tid] = m;
    }
    __syncthreads(); // the bbox keys are visible to the whole CTA
    prep_edges_body<MODE>(vx, vy, ring_off, n_rings, n_verts, filt, qk, n_qk, rec, bbox_keys, tol, tid,
                          kPrepThreads);
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
    uint64_t first = 0; // the reference throws DegenerateEdge at the first such edge: report its index
    if (nv >= 2) {
        double ax = vx[0], ay = vy[0];
        double f_prev = __dsub_rn(ay, q.y);
        for (uint64_t v = 1; v < nv && !aux; ++v) {
            const double bx = vx[v], by = vy[v];
            raw_edge<MODE>(q.x, q.y, 0.0, 0.0, ax, ay, bx, by, f_prev, cnt, aux);
            first = v - 1;
            ax = bx;
            ay = by;
        }
    }
    counts[i] = aux ? (unsigned long long)first : (unsigned long long)cnt;
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

} // namespace

size_t filt_words(uint64_t n_edges) { return std::max<uint64_t>(n_edges, 1); }
size_t qk_words(uint64_t n_edges) { return (std::max<uint64_t>(n_edges, 1) + kKeyTile - 1) / kKeyTile * kKeyTile; }

size_t edge_rec_bytes() { return sizeof(EdgeRec); }

cudaError_t launch_fp64_probe(double* out, int iters, int dev, cudaStream_t st, double* flops) {
    const unsigned blocks = (unsigned)sm_count(dev) * 8;
    fp64_probe_kernel<<<blocks, 256, 0, st>>>(out, iters, 0.9999999, 1e-7);
    *flops = (double)blocks * 256.0 * iters * 8.0 * 2.0;
    return cudaGetLastError();
}

cudaError_t launch_prep(const PrepArgs& a, cudaStream_t st, int dev, uint64_t* launches) {
    const uint64_t nqk = qk_words(a.n_verts - a.n_rings);
    EdgeRec* rec = reinterpret_cast<EdgeRec*>(a.rec);
    if (a.n_verts <= kPrepSmall) {
#define PC_PREP_SMALL(M)                                                                                        \
    prep_small_kernel<M><<<(unsigned)(1 + (a.n_zero_words + kPrepZero - 1) / kPrepZero), kPrepThreads, 0, st>>>(a.vx, a.vy, a.ring_off, a.n_rings, a.n_verts, a.filt, a.qk, \
                                                     nqk, rec, a.bbox_keys, a.tol, a.zero_words, a.zero_words2,  \
                                                     a.n_zero_words, a.stats)
        switch (a.mode) {
        case kC1: PC_PREP_SMALL(kC1); break;
        case kC2: PC_PREP_SMALL(kC2); break;
        default: PC_PREP_SMALL(kRobust);
        }
#undef PC_PREP_SMALL
        *launches += 1;
        return cudaGetLastError();
    }
    cudaError_t e = cudaMemsetAsync(a.bbox_keys, 0xff, 4 * sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    const unsigned bb = (unsigned)std::min<uint64_t>(std::max<uint64_t>(a.n_verts, a.n_zero_words) / 256 + 1,
                                                     (uint64_t)sm_count(dev) * 8);
    prep_bbox_kernel<<<bb, 256, 0, st>>>(a.vx, a.vy, a.ring_off, a.bbox_keys, a.zero_words, a.zero_words2,
                                         a.n_zero_words, a.stats);
    const unsigned blocks = (unsigned)std::min<uint64_t>(a.n_verts / 256 + 1, (uint64_t)sm_count(dev) * 16);
    switch (a.mode) {
    case kC1:
        prep_edges_kernel<kC1><<<blocks, 256, 0, st>>>(a.vx, a.vy, a.ring_off, a.n_rings, a.n_verts, a.filt, a.qk,
                                                       nqk, rec, a.bbox_keys, a.tol);
        break;
    case kC2:
        prep_edges_kernel<kC2><<<blocks, 256, 0, st>>>(a.vx, a.vy, a.ring_off, a.n_rings, a.n_verts, a.filt, a.qk,
                                                       nqk, rec, a.bbox_keys, a.tol);
        break;
    default:
        prep_edges_kernel<kRobust><<<blocks, 256, 0, st>>>(a.vx, a.vy, a.ring_off, a.n_rings, a.n_verts, a.filt,
                                                           a.qk, nqk, rec, a.bbox_keys, a.tol);
        break;
    }
    *launches += 2;
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
