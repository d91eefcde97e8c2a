// CSR multi-polygon kernel (configs 3 and 5): many small
// polygons, each with its own contiguous run of query points.
//
// The work per byte is tiny (c3: ~10 point-edge tests per 16-byte point), so
// this path is HBM-bound and the design is about keeping bytes in flight:
//
//   * persistent CTAs, each owning a contiguous range of polygons;
//   * warp 0 is a producer: it reads the CSR offsets of the next group of
//     polygons (up to kG polygons, kPmax points, kVmax vertices, kRmax rings),
//     and moves the group's points and vertices into a shared-memory stage
//     with TMA bulk copies (cp.async.bulk ... mbarrier::complete_tx), two
//     stages deep, so the next group streams in while this one is computed;
//   * warps 1..7 are consumers: per group they derive per-edge data once
//     (filter keys, normals / direction vectors) and then classify, one warp
//     per polygon, 64 points per pass (2 per lane), every ring edge of the
//     polygon from shared memory: the integer key filter first, the exact
//     binary64 test of the reference only for straddle candidates;
//   * flags leave as ballot words OR-ed into the bit planes.
//
// Reference semantics per polygon: classify_batch(points_i, poly_i, mode)
// (batch.hpp:184-230): closed bbox of the outer ring, then even-odd over rings
// of count_crossings_c1/_c2 / robust_ray_crossings (geometry.hpp:182-300).
// A polygon too large for a stage is classified by the consumer warps straight
// from global memory with the same arithmetic.
#include "pip_kernels.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>

#include "pip_device.cuh"

namespace pcd {

namespace {

constexpr int kCsrThreads = 256;          // warp 0 producer + 7 consumer warps
constexpr int kConsumers = kCsrThreads / 32 - 1;
constexpr int kG = 32;                    // polygons per stage (max)
constexpr int kPmax = 1024;               // points per stage
constexpr int kVmax = 512;                // vertices per stage
constexpr int kRmax = 128;                // rings per stage

struct __align__(16) Stage {
    double2 pts[kPmax];
    double vx[kVmax + 2];                 // +2: the 16-byte aligned bulk window may start one element early
    double vy[kVmax + 2];
    unsigned long long pt_off[kG + 1];    // raw values (global indices)
    unsigned long long pring[kG + 1];
    unsigned long long ring_off[kRmax + 1];
    int n_polys;                          // polygons in the stage; -1 = no more work
    int oversize;                         // 1: single polygon too big for the stage (global path)
    unsigned long long p_first;           // first polygon (local to this call)
    unsigned long long v_win;             // vertex index of vx[0] (window start)
    unsigned long long s_first;           // first point (raw pt_off value)
};

constexpr int kStages = 3;
constexpr int kEChunk = 64;               // edges derived per warp pass

struct WarpScratch {                      // per consumer warp: data of up to kEChunk edges
    int klo[kEChunk];
    unsigned rng[kEChunk];                // C1/C2: khi-klo; Robust: khi
    double e0[kEChunk], e1[kEChunk], e2[kEChunk];
};

struct CsrShared {
    Stage stage[kStages];
    WarpScratch ws[kConsumers];
    unsigned long long full[kStages], empty[kStages];
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// OR the bits of a 32-point ballot (point g0 = first) into a bit plane.
__device__ __forceinline__ void or_bits(uint32_t* plane, unsigned long long g0, uint32_t bits) {
    if (!bits) return;
    const unsigned long long w = g0 >> 5;
    const unsigned sh = (unsigned)(g0 & 31);
    atomicOr(&plane[w], bits << sh);
    if (sh && (bits >> (32 - sh))) atomicOr(&plane[w + 1], bits >> (32 - sh));
}

template <int MODE>
__device__ __forceinline__ void warp_bbox(const double* x, const double* y, unsigned long long lo,
                                          unsigned long long hi, double& minx, double& miny, double& maxx,
                                          double& maxy) {
    const int lane = threadIdx.x & 31;
    minx = miny = INFINITY;
    maxx = maxy = -INFINITY;
    for (unsigned long long v = lo + lane; v < hi; v += 32) {
        const double a = x[v], b = y[v];
        minx = fmin(minx, a);
        miny = fmin(miny, b);
        maxx = fmax(maxx, a);
        maxy = fmax(maxy, b);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        minx = fmin(minx, __shfl_xor_sync(0xffffffffu, minx, o));
        miny = fmin(miny, __shfl_xor_sync(0xffffffffu, miny, o));
        maxx = fmax(maxx, __shfl_xor_sync(0xffffffffu, maxx, o));
        maxy = fmax(maxy, __shfl_xor_sync(0xffffffffu, maxy, o));
    }
}

// Derive the per-edge data of edges [e0, e0+ne) (vertex indices into vx/vy,
// edge e = (e, e+1)) into the warp's scratch; one lane per edge.
template <int MODE>
__device__ __forceinline__ void derive_chunk(const double* vx, const double* vy, unsigned long long e0, int ne,
                                             WarpScratch& w) {
    const int lane = threadIdx.x & 31;
    for (int i = lane; i < ne; i += 32) {
        const unsigned long long v = e0 + i;
        const double ax = vx[v], ay = vy[v], bx = vx[v + 1], by = vy[v + 1];
        const double ylo = by < ay ? by : ay, yhi = ay < by ? by : ay;
        const int klo = fkey(ylo), khi = fkey(yhi);
        w.klo[i] = klo;
        if (MODE == kC1) {
            double nx = __dsub_rn(by, ay), ny = __dsub_rn(ax, bx);
            if (nx < 0.0) {
                nx = -nx;
                ny = -ny;
            }
            w.e0[i] = nx;
            w.e1[i] = ny;
            w.rng[i] = (unsigned)khi - (unsigned)klo;
        } else if (MODE == kC2) {
            w.e0[i] = __dsub_rn(bx, ax);
            w.e1[i] = __dsub_rn(by, ay);
            w.rng[i] = (unsigned)khi - (unsigned)klo;
        } else {
            const double abx = __dsub_rn(bx, ax), aby = __dsub_rn(by, ay);
            w.e0[i] = abx;
            w.e1[i] = aby;
            w.e2[i] = __dadd_rn(__dmul_rn(abx, abx), __dmul_rn(aby, aby));
            w.rng[i] = (unsigned)khi;
        }
    }
    __syncwarp();
}

// Classify points [s, t) (indices into `pts`) of one polygon whose rings are
// [rl0, rl1) with vertex offsets roff[r] - vbase (indices into vx/vy), 64 points
// per pass (2 per lane).  Per ring, edges are derived kEChunk at a time into
// the warp's scratch, then every edge is tested against the 64 points: the
// integer key filter (is p.y inside the edge's y-range?) for all, the exact
// binary64 test of the reference only when a lane has a candidate.
template <int MODE>
__device__ __forceinline__ void classify_polygon(const double2* pts, unsigned long long s, unsigned long long t,
                                 unsigned long long plane0, const double* vx, const double* vy,
                                 const unsigned long long* roff, unsigned long long vbase, int rl0, int rl1,
                                 WarpScratch& w, double tol, double tol2, uint32_t* inside_bits, uint32_t* aux_bits,
                                 int chunk_stride, int first_chunk) {
    const int lane = threadIdx.x & 31;
    if (t <= s) return;
    double minx, miny, maxx, maxy;
    if (rl1 > rl0) {
        warp_bbox<MODE>(vx, vy, roff[rl0] - vbase, roff[rl0 + 1] - vbase, minx, miny, maxx, maxy);
    } else {
        minx = miny = 1.0;
        maxx = maxy = -1.0; // no rings: nothing inside
    }
    for (unsigned long long c = s + 64ull * first_chunk; c < t; c += 64ull * chunk_stride) {
        double px[2], py[2];
        int ka[2], kb[2], cnt[2];
        bool act[2], aux[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const unsigned long long i = c + 32 * j + lane;
            act[j] = i < t;
            double2 p = make_double2(0.0, 0.0);
            if (act[j]) p = pts[i];
            px[j] = p.x;
            py[j] = p.y;
            act[j] = act[j] && p.x >= minx && p.x <= maxx && p.y >= miny && p.y <= maxy; // batch.hpp:200
            cnt[j] = 0;
            aux[j] = false;
            if (MODE == kRobust) {
                ka[j] = act[j] ? fkey(__dadd_rn(p.y, tol)) : INT_MIN;
                kb[j] = act[j] ? fkey(__dsub_rn(p.y, tol)) : INT_MAX;
            } else {
                ka[j] = act[j] ? fkey(p.y) : INT_MAX;
                kb[j] = ka[j];
            }
        }
        if (__any_sync(0xffffffffu, act[0] || act[1])) {
            for (int r = rl0; r < rl1; ++r) {
                const unsigned long long lo = roff[r] - vbase, hi = roff[r + 1] - vbase;
                for (unsigned long long e0 = lo; e0 + 1 < hi; e0 += kEChunk) {
                    const int ne = (int)min((unsigned long long)kEChunk, hi - 1 - e0);
                    __syncwarp();
                    derive_chunk<MODE>(vx, vy, e0, ne, w);
                    for (int i = 0; i < ne; ++i) {
                        const int klo = w.klo[i];
                        const unsigned rg = w.rng[i];
                        bool cand[2];
#pragma unroll
                        for (int j = 0; j < 2; ++j)
                            cand[j] = MODE == kRobust ? (ka[j] >= klo && kb[j] <= (int)rg)
                                                      : ((unsigned)(ka[j] - klo) <= rg);
                        if (!__any_sync(0xffffffffu, cand[0] || cand[1])) continue;
                        const unsigned long long e = e0 + i;
                        const double ax = vx[e], ay = vy[e];
                        const double q0 = w.e0[i], q1 = w.e1[i];
                        if (MODE == kC1) {
                            // key ties leave the straddle open: the reference product decides
                            bool tie[2];
#pragma unroll
                            for (int j = 0; j < 2; ++j) {
                                const unsigned d = (unsigned)(ka[j] - klo);
                                tie[j] = cand[j] && (d == 0u || d == rg);
                            }
                            if (__any_sync(0xffffffffu, tie[0] || tie[1])) {
                                const double by = vy[e + 1];
#pragma unroll
                                for (int j = 0; j < 2; ++j)
                                    if (tie[j])
                                        cand[j] = __dmul_rn(__dsub_rn(ay, py[j]), __dsub_rn(by, py[j])) <= 0.0;
                            }
#pragma unroll
                            for (int j = 0; j < 2; ++j) {
                                const double side = __dadd_rn(__dmul_rn(__dsub_rn(px[j], ax), q0),
                                                              __dmul_rn(__dsub_rn(py[j], ay), q1));
                                cnt[j] += (cand[j] && side <= 0.0) ? 1 : 0;
                            }
                        } else {
                            const double by = vy[e + 1];
#pragma unroll
                            for (int j = 0; j < 2; ++j) {
                                if (!cand[j]) continue;
                                if (MODE == kRobust) {
                                    EdgeRec rr;
                                    rr.d[0] = ax;
                                    rr.d[1] = ay;
                                    rr.d[2] = by;
                                    rr.d[3] = q0;
                                    rr.d[4] = q1;
                                    rr.d[5] = w.e2[i];
                                    rr.d[6] = by < ay ? by : ay;
                                    rr.d[7] = ay < by ? by : ay;
                                    exact_robust(px[j], py[j], tol, tol2, rr, cnt[j], aux[j]);
                                } else {
                                    const unsigned d = (unsigned)(ka[j] - klo);
                                    EdgeRec rr;
                                    rr.d[0] = ax;
                                    rr.d[1] = ay;
                                    rr.d[2] = by;
                                    rr.d[3] = q0;
                                    rr.d[4] = q1;
                                    exact_c2(px[j], py[j], rr, cnt[j], aux[j], d != 0u && d != rg);
                                }
                            }
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const uint32_t bi = __ballot_sync(0xffffffffu, act[j] && (cnt[j] & 1) && !aux[j]);
            const uint32_t ba = __ballot_sync(0xffffffffu, act[j] && aux[j]);
            if (lane == 0) {
                const unsigned long long g0 = plane0 + (c - s) + 32 * j;
                or_bits(inside_bits, g0, bi);
                or_bits(aux_bits, g0, ba);
            }
        }
    }
}

template <int MODE>
__global__ void __launch_bounds__(kCsrThreads, 2) pip_csr_tma_kernel(
    const double2* __restrict__ pts, const unsigned long long* __restrict__ pt_off, unsigned long long n_polys,
    const double* __restrict__ vx, const double* __restrict__ vy, const unsigned long long* __restrict__ ring_off,
    const unsigned long long* __restrict__ poly_ring_off, unsigned long long pt_base, unsigned long long ring_base,
    unsigned long long vert_base, double tol, double tol2, uint32_t* __restrict__ inside_bits,
    uint32_t* __restrict__ aux_bits) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    CsrShared& sh = *reinterpret_cast<CsrShared*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // contiguous polygon range of this CTA
    const unsigned long long p_begin = n_polys * blockIdx.x / gridDim.x;
    const unsigned long long p_end = n_polys * (blockIdx.x + 1) / gridDim.x;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&sh.full[i], 1);
            mbar_init(&sh.empty[i], kConsumers);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == 0) {
        // ---------------- producer -----------------
        unsigned long long p = p_begin;
        int s = 0;
        unsigned phase = 0;
        for (;;) {
            mbar_wait(&sh.empty[s], phase ^ 1);
            Stage& st = sh.stage[s];
            if (p >= p_end) {
                if (lane == 0) {
                    st.n_polys = -1;
                    mbar_arrive(&sh.full[s]);
                }
                break;
            }
            const unsigned long long avail = min((unsigned long long)kG, p_end - p);
            // offsets of up to kG+1 polygons (values are raw; local = value - base)
            for (int i = lane; i <= (int)avail; i += 32) {
                st.pt_off[i] = pt_off[p + i];
                st.pring[i] = poly_ring_off[p + i];
            }
            __syncwarp();
            // largest m with points <= kPmax and rings <= kRmax
            int m_ok = 0;
            for (int i = lane + 1; i <= (int)avail; i += 32) {
                const bool fit = st.pt_off[i] - st.pt_off[0] <= (unsigned long long)kPmax &&
                                 st.pring[i] - st.pring[0] <= (unsigned long long)kRmax;
                if (fit) m_ok = max(m_ok, i);
            }
            // fit is monotone in i, so the max over lanes is the answer
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m_ok = max(m_ok, __shfl_xor_sync(0xffffffffu, m_ok, o));
            int m = m_ok;
            const unsigned long long r0 = st.pring[0] - ring_base;
            if (m > 0) {
                const int nr = (int)(st.pring[m] - st.pring[0]);
                for (int i = lane; i <= nr; i += 32) st.ring_off[i] = ring_off[r0 + i];
                __syncwarp();
                // shrink m until the vertices fit
                int m_v = 0;
                for (int i = lane + 1; i <= m; i += 32) {
                    const unsigned long long nv = st.ring_off[st.pring[i] - st.pring[0]] - st.ring_off[0];
                    if (nv <= (unsigned long long)kVmax) m_v = max(m_v, i);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) m_v = max(m_v, __shfl_xor_sync(0xffffffffu, m_v, o));
                m = m_v;
            }
            if (m == 0) {
                // one polygon that does not fit a stage: consumers read it from global memory
                if (lane == 0) {
                    st.n_polys = 1;
                    st.oversize = 1;
                    st.p_first = p;
                    mbar_arrive(&sh.full[s]);
                }
                p += 1;
            } else {
                const unsigned long long v0 = st.ring_off[0] - vert_base;
                const unsigned long long v1 = st.ring_off[st.pring[m] - st.pring[0]] - vert_base;
                const unsigned long long s0 = st.pt_off[0] - pt_base, s1 = st.pt_off[m] - pt_base;
                const unsigned long long win = v0 & ~1ull;               // 16-byte aligned window start
                const unsigned long long a0 = (v0 + 1) & ~1ull;          // aligned interior [a0, a1)
                const unsigned long long a1 = v1 & ~1ull;
                if (lane == 0) {
                    st.n_polys = m;
                    st.oversize = 0;
                    st.p_first = p;
                    st.v_win = win + vert_base;
                    st.s_first = st.pt_off[0];
                }
                // ragged vertex ends (at most one element each) with plain loads
                if (lane == 1 && (v0 & 1ull) && v0 < v1) {
                    st.vx[v0 - win] = vx[v0];
                    st.vy[v0 - win] = vy[v0];
                }
                if (lane == 2 && (v1 & 1ull) && v1 - 1 >= a0 && v1 > v0) {
                    st.vx[v1 - 1 - win] = vx[v1 - 1];
                    st.vy[v1 - 1 - win] = vy[v1 - 1];
                }
                __syncwarp();
                if (lane == 0) {
                    const unsigned pbytes = (unsigned)((s1 - s0) * 16);
                    const unsigned vbytes = a1 > a0 ? (unsigned)((a1 - a0) * 8) : 0u;
                    mbar_arrive_expect_tx(&sh.full[s], pbytes + 2 * vbytes);
                    if (pbytes) bulk_g2s(st.pts, pts + s0, pbytes, &sh.full[s]);
                    if (vbytes) {
                        bulk_g2s(st.vx + (a0 - win), vx + a0, vbytes, &sh.full[s]);
                        bulk_g2s(st.vy + (a0 - win), vy + a0, vbytes, &sh.full[s]);
                    }
                }
                p += m;
            }
            if (++s == kStages) {
                s = 0;
                phase ^= 1;
            }
        }
        return;
    }

    // ---------------- consumers (warps 1..7) -----------------
    const int cw = warp - 1;
    WarpScratch& w = sh.ws[cw];
    int s = 0;
    unsigned phase = 0;
    for (;;) {
        mbar_wait(&sh.full[s], phase);
        const Stage& st = sh.stage[s];
        const int np = st.n_polys;
        if (np < 0) break;
        if (st.oversize) {
            // global-memory path: the consumer warps share the polygon's 64-point chunks
            const unsigned long long p = st.p_first;
            const unsigned long long r0 = poly_ring_off[p] - ring_base, r1 = poly_ring_off[p + 1] - ring_base;
            const unsigned long long ps = pt_off[p] - pt_base, pe = pt_off[p + 1] - pt_base;
            classify_polygon<MODE>(pts, ps, pe, ps, vx, vy, ring_off + r0, vert_base, 0, (int)(r1 - r0), w, tol, tol2,
                                   inside_bits, aux_bits, kConsumers, cw);
        } else {
            for (int i = cw; i < np; i += kConsumers) {
                const unsigned long long ps = st.pt_off[i] - st.s_first, pe = st.pt_off[i + 1] - st.s_first;
                const int rl0 = (int)(st.pring[i] - st.pring[0]), rl1 = (int)(st.pring[i + 1] - st.pring[0]);
                classify_polygon<MODE>(st.pts, ps, pe, st.pt_off[i] - pt_base, st.vx, st.vy, st.ring_off, st.v_win,
                                       rl0, rl1, w, tol, tol2, inside_bits, aux_bits, 1, 0);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sh.empty[s]); // this warp is done with the stage
        if (++s == kStages) {
            s = 0;
            phase ^= 1;
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
    const size_t smem = sizeof(CsrShared);
    static bool attr[64] = {};
    if (dev < 64 && !attr[dev]) {
        cudaFuncSetAttribute(pip_csr_tma_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr[dev] = true;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pip_csr_tma_kernel<MODE>, kCsrThreads, smem);
    per_sm = std::max(per_sm, 1);
    const uint64_t want = (a.n_polys + kG - 1) / kG;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)sms(dev) * per_sm));
    pip_csr_tma_kernel<MODE><<<grid, kCsrThreads, smem, st>>>(
        reinterpret_cast<const double2*>(a.pts), reinterpret_cast<const unsigned long long*>(a.pt_off), a.n_polys,
        a.vx, a.vy, reinterpret_cast<const unsigned long long*>(a.ring_off),
        reinterpret_cast<const unsigned long long*>(a.poly_ring_off), a.pt_base, a.ring_base, a.vert_base, a.tol,
        a.tol2, a.inside_bits, a.aux_bits);
    ++*launches;
    return cudaGetLastError();
}

} // namespace

size_t csr_smem_bytes() { return sizeof(CsrShared); }

cudaError_t launch_csr(const CsrArgs& a, cudaStream_t st, int dev, uint64_t* launches) {
    if (a.n_polys == 0) return cudaSuccess;
    switch (a.mode) {
    case kC1: return launch_t<kC1>(a, st, dev, launches);
    case kC2: return launch_t<kC2>(a, st, dev, launches);
    default: return launch_t<kRobust>(a, st, dev, launches);
    }
}

} // namespace pcd
