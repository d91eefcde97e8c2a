// Single-polygon kernel (configs 1, 2, 4; classify_batch / contains over one
// polygon with holes): the point-edge scan of count_crossings_c1/_c2 /
// robust_ray_crossings (geometry.hpp:182-273) for every point of a batch.
//
// Work decomposition: CTA (bx, by) classifies points [bx*kTPB*K, +kTPB*K)
// against edges [by*chunk, +chunk); partial parities are XOR-ed and
// Error/Boundary flags OR-ed into the bit planes, so edge chunks combine
// exactly like the reference's per-ring sums (geometry.hpp:285-299).
//
// Per thread: K points, of which only the 32-bit filter keys live in
// registers (coordinates sit in shared memory, loaded once per CTA by one TMA
// bulk copy); parity and aux flags are K-bit masks.  Warp w owns K*32
// consecutive points (k-slice k = 32 consecutive points), which after
// y-bucketing (pip_sort.cu) are y-adjacent, so an edge either misses the whole
// warp or is a candidate for most of it.
//
// Per edge (fast path, all points): d_k = key(p.y) - key(ylo) (mod 2^32) and
// the running minimum of the d_k — one fused add+min (VIADDMNMX) per point —
// then a single compare of the minimum against key(yhi)-key(ylo) decides, for
// the whole warp, whether any point may straddle the edge (exactness argument
// in DESIGN.md §3).  Only then (warp-uniform branch) does the slow path
// re-derive which points are candidates and run the binary64 test of the
// reference for them.
//
// Edge tiles (filter keys + exact records, precomputed by prep_edges_kernel)
// stream into shared memory with TMA bulk copies, double-buffered on
// mbarriers, while the previous tile is scanned.
#include "pip_kernels.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <climits>
#include <type_traits>

#include "pip_device.cuh"

namespace pcd {

namespace {

constexpr int kTPB = 256;
constexpr int kK = 16;      // points per thread
constexpr int kTile = 256;  // edges per shared-memory stage (multiple of 2: 16-byte bulk copies)

struct __align__(128) TileStage {
    EdgeRec rec[kTile];
    uint2 wkr[kTile];  // key range per edge (warp-level test)   } one bulk copy:
    uint2 filt[kTile]; // per-point filter word                   } the tile-blocked block
};
static_assert(kTile == kEdgeTile, "the stage holds one filter block");

// Every mode keeps only the polygon-local fp32 coordinates of its points in
// shared memory (the certified fp32 side / intercept test); the binary64
// fallbacks re-read the point from global memory (L2).
template <int MODE>
struct SingleShared {
    using PointT = float2;
    PointT pts[kTPB * kK]; // this CTA's points (bucketed order)
    TileStage st[2];
    unsigned long long full[2];
    unsigned long long pbar;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// explicit shared-memory loads from a 32-bit shared address (kept in a
// register by the caller, see the edge loop)
__device__ __forceinline__ uint2 lds_u2(unsigned a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ EdgeRec lds_rec(unsigned a) {
    EdgeRec r;
#pragma unroll
    for (int i = 0; i < 8; i += 2)
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.d[i]), "=d"(r.d[i + 1]) : "r"(a + 8u * i));
    return r;
}

__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
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

// One elected thread: load tile [t0, t0+nt) of the edge arrays into stage s.
template <class Shared>
__device__ __forceinline__ void issue_tile(Shared& sh, int s, const uint2* filt, const EdgeRec* rec,
                                           uint32_t t0, uint32_t nt) {
    const unsigned fb = 2u * kTile * 8u; // the whole block of ranges + words (t0 is tile-aligned)
    const unsigned rb = nt * (unsigned)sizeof(EdgeRec);
    const unsigned bar = smem_u32(&sh.full[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(fb + rb) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sh.st[s].wkr)),
                 "l"(filt + 2ull * t0), "r"(fb), "r"(bar)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sh.st[s].rec)),
                 "l"(rec + t0), "r"(rb), "r"(bar)
                 : "memory");
}

// Per-thread point keys.  C1/C2: 15-bit keys (qkey15), two points per
// register as (q_2i << 1) | (q_2i+1 << 17).  Robust: 32-bit keys of p.y+tol
// and p.y-tol.
template <int MODE>
struct Keys;
template <>
struct Keys<kC1> {
    uint32_t k2[kK / 2];
    // d_k = q_k - q(ylo) mod 2^15 for the edge whose filter word is fx
    __device__ __forceinline__ uint32_t diff(int k, uint32_t fx) const {
        return ((k2[k >> 1] + fx) >> (16 * (k & 1) + 1)) & 0x7fffu;
    }
};
template <>
struct Keys<kC2> : Keys<kC1> {};
template <>
struct Keys<kRobust> {
    int ka[kK], kb[kK];
};

// Fast path: may any of this lane's points straddle the edge?
// C1/C2: d_k = q_k - q(ylo) (mod 2^15); candidate iff d_k <= q(yhi) - q(ylo).
// Per pair of points one 32-bit IMAD (FMA pipe) forms both d_k << 1 (+ a
// guard bit); one VIMNMX3.U16x2 (ALU pipe) folds four points into the running
// packed minimum, compared once against (range << 1) | 1.
template <int MODE>
__device__ __forceinline__ bool lane_candidate(const Keys<MODE>& K, uint2 f) {
    if constexpr (MODE == kRobust) {
        bool c = false;
#pragma unroll
        for (int k = 0; k < kK; ++k) c |= (K.ka[k] >= (int)f.x) & (K.kb[k] <= (int)f.y);
        return c;
    } else {
        static_assert(kK / 2 >= 4 && (kK / 2) % 2 == 0, "fold below assumes an even number of key registers");
        uint32_t d[kK / 2];
#pragma unroll
        for (int i = 0; i < kK / 2; ++i) d[i] = K.k2[i] + f.x;
        uint32_t m = __vimin3_u16x2(d[0], d[1], d[2]);
#pragma unroll
        for (int i = 3; i + 1 < kK / 2; i += 2) m = __vimin3_u16x2(m, d[i], d[i + 1]);
        // f.y = (threshold + 1) in both halves: the fold's last input, so the
        // result differs from f.y iff some half of some d is below it
        m = __vimin3_u16x2(m, d[kK / 2 - 1], f.y);
        return m != f.y;
    }
}

// C1 slow path (geometry.hpp:189-200) for one candidate edge, branch-free
// over the 16 points.  Straddle: if the warp's whole key range lies strictly
// inside the edge's, every active point straddles for sure; otherwise per-point
// candidate / tie masks, ties evaluating the reference product.  Side: the
// certified fp32 test on the polygon-local coordinates (LocalMap, DESIGN.md
// §3.4) -- two FFMAs per point; a point within the band (or without local
// coordinates) re-reads its binary64 coordinates and runs the reference's
// expression.
__device__ __forceinline__ void slow_c1(const float2* my_l, const double2* __restrict__ my_g, const Keys<kC1>& K,
                                        uint32_t act, uint32_t nonloc, uint2 f, const EdgeRec& r, uint32_t& par,
                                        uint32_t wkey_lo, uint32_t wkey_hi) {
    const double ax = r.d[0], ay = r.d[1];
    const uint32_t rng = ((f.y & 0xffffu) - 2u) >> 1;
    const uint32_t klo = (0x8000u - ((f.x & 0xffffu) >> 1)) & 0x7fffu;
    uint32_t cm = act;
    if (!(klo < wkey_lo && wkey_hi < klo + rng)) {
        uint32_t tm = 0;
        cm = 0;
#pragma unroll
        for (int k = 0; k < kK; ++k) {
            const uint32_t d = K.diff(k, f.x);
            cm |= (uint32_t)(d <= rng) << k;
            tm |= (uint32_t)(d == 0u || d == rng) << k;
        }
        cm &= act;
        tm &= cm;
        if (__any_sync(0xffffffffu, tm != 0)) {
            const double by = r.d[2];
#pragma unroll 1
            for (int k = 0; k < kK; ++k) {
                if (tm >> k & 1u) {
                    const double py = my_g[k * 32].y;
                    if (!(__dmul_rn(__dsub_rn(ay, py), __dsub_rn(by, py)) <= 0.0)) cm &= ~(1u << k);
                }
            }
        }
    }
    const float nxf = __int_as_float(__double2loint(r.d[5])), nyf = __int_as_float(__double2hiint(r.d[5]));
    const float cf = __int_as_float(__double2loint(r.d[6])); // c + B
    // s' = s + B: counted iff the sign bit is set (s' <= -0); band hit iff
    // +0 <= s' <= 2B, i.e. its bits (as unsigned) are <= those of 2B
    constexpr uint32_t k2B = 0x36000000u; // bits of 2^-19 = 2 * kLocalBand
    uint32_t hit = 0, umin = 0xffffffffu;
#pragma unroll
    for (int k = kK - 1; k >= 0; --k) {
        const float2 l = my_l[k * 32];
        const uint32_t u = __float_as_uint(fmaf(l.x, nxf, fmaf(l.y, nyf, cf)));
        hit = (hit << 1) | (u >> 31);
        umin = min(umin, u);
    }
    // undecided: band hits (rare: per point only then), points without local
    // coordinates (nonloc) and edges without a record (NaN: every point)
    uint32_t und = nonloc | ((nxf == nxf) ? 0u : 0xffffu);
    if (umin <= k2B) {
#pragma unroll
        for (int k = 0; k < kK; ++k) {
            const float2 l = my_l[k * 32];
            und |= (uint32_t)(__float_as_uint(fmaf(l.x, nxf, fmaf(l.y, nyf, cf))) <= k2B) << k;
        }
    }
    und &= cm;
    if (__any_sync(0xffffffffu, und != 0)) {
        const double nx = r.d[3], ny = r.d[4];
#pragma unroll 1
        for (int k = 0; k < kK; ++k) {
            if (und >> k & 1u) {
                const double2 p = my_g[k * 32];
                const double side = __dadd_rn(__dmul_rn(__dsub_rn(p.x, ax), nx), __dmul_rn(__dsub_rn(p.y, ay), ny));
                hit = (hit & ~(1u << k)) | ((uint32_t)(side <= 0.0) << k);
            }
        }
    }
    par ^= hit & cm;
}

// C2 slow path (geometry.hpp:216-224) for one candidate edge: sure straddles
// decide the intercept sign with the certified fp32 test (local_side_record_c2);
// key ties, band hits and points without local coordinates run the
// reference's expression (division included, DegenerateEdge -> Error).
__device__ __forceinline__ void slow_c2(const float2* my_l, const double2* __restrict__ my_g, const Keys<kC2>& K,
                                        uint32_t act, uint32_t nonloc, uint2 f, const EdgeRec& r, uint32_t& par,
                                        uint32_t& auxm, uint32_t wkey_lo, uint32_t wkey_hi) {
    const uint32_t rng = ((f.y & 0xffffu) - 2u) >> 1;
    const uint32_t klo = (0x8000u - ((f.x & 0xffffu) >> 1)) & 0x7fffu;
    uint32_t cm = act, tm = 0;
    if (!(klo < wkey_lo && wkey_hi < klo + rng)) {
        cm = 0;
#pragma unroll
        for (int k = 0; k < kK; ++k) {
            const uint32_t d = K.diff(k, f.x);
            cm |= (uint32_t)(d <= rng) << k;
            tm |= (uint32_t)(d == 0u || d == rng) << k;
        }
        cm &= act;
        tm &= cm;
    }
    const uint32_t sure = cm & ~tm;
    const float nxf = __int_as_float(__double2loint(r.d[5])), nyf = __int_as_float(__double2hiint(r.d[5]));
    const float cf = __int_as_float(__double2loint(r.d[6])); // c + B
    constexpr uint32_t k2B = 0x36000000u;                   // bits of 2^-19 = 2 * kLocalBand
    uint32_t hit = 0, umin = 0xffffffffu;
#pragma unroll
    for (int k = kK - 1; k >= 0; --k) {
        const float2 l = my_l[k * 32];
        const uint32_t u = __float_as_uint(fmaf(l.x, nxf, fmaf(l.y, nyf, cf)));
        hit = (hit << 1) | (u >> 31);
        umin = min(umin, u);
    }
    uint32_t und = nonloc | ((nxf == nxf) ? 0u : 0xffffu);
    if (umin <= k2B) {
#pragma unroll
        for (int k = 0; k < kK; ++k) {
            const float2 l = my_l[k * 32];
            und |= (uint32_t)(__float_as_uint(fmaf(l.x, nxf, fmaf(l.y, nyf, cf))) <= k2B) << k;
        }
    }
    und &= sure;
    par ^= hit & sure & ~und;
    const uint32_t ex = und | tm; // binary64: band hits / no local coordinates (sure) and key ties
    if (__any_sync(0xffffffffu, ex != 0)) {
#pragma unroll 1
        for (int k = 0; k < kK; ++k) {
            if (ex >> k & 1u) {
                const double2 p = my_g[k * 32];
                int cnt = 0;
                bool err = false;
                exact_c2(p.x, p.y, r, cnt, err, (und >> k) & 1u);
                par ^= (uint32_t)(cnt & 1) << k;
                auxm |= (uint32_t)err << k;
            }
        }
    }
}

// Robust slow path (geometry.hpp:237-273) for one candidate edge.  Keys of
// p.y + tol and p.y - tol strictly inside the edge's key range imply
// y_lo < p.y - tol and p.y + tol < y_hi: no band reject, and exactly one of
// upward / downward holds; the crossing is then C2's intercept sign (the
// reference evaluates the same expression), certified in fp32, and a decided
// sign also rules out the boundary when tol <= 2^-30 * min(W, H) (the record
// is NaN otherwise): the point's distance to the edge's line is then at least
// ~29 tol.  Everything else runs the reference's expression.
__device__ __forceinline__ void slow_robust(const float2* my_l, const double2* __restrict__ my_g,
                                            const Keys<kRobust>& K, uint32_t act, uint32_t nonloc, uint2 f,
                                            const EdgeRec& r, double tol, double tol2, uint32_t& par, uint32_t& auxm,
                                            int wka_max, int wkb_min) {
    const int flo = (int)f.x, fhi = (int)f.y;
    uint32_t cm = act, sure = act;
    if (!(flo < wkb_min && wka_max < fhi)) {
        cm = sure = 0;
#pragma unroll
        for (int k = 0; k < kK; ++k) {
            cm |= (uint32_t)(K.ka[k] >= flo && K.kb[k] <= fhi) << k;
            sure |= (uint32_t)(flo < K.kb[k] && K.ka[k] < fhi) << k;
        }
        cm &= act;
        sure &= cm;
    }
    const float nxf = __int_as_float(__double2loint(r.d[6])), nyf = __int_as_float(__double2hiint(r.d[6]));
    const float cf = __int_as_float(__double2loint(r.d[7])); // c + B
    constexpr uint32_t k2B = 0x36000000u;                   // bits of 2^-19 = 2 * kLocalBand
    uint32_t hit = 0, umin = 0xffffffffu;
#pragma unroll
    for (int k = kK - 1; k >= 0; --k) {
        const float2 l = my_l[k * 32];
        const uint32_t u = __float_as_uint(fmaf(l.x, nxf, fmaf(l.y, nyf, cf)));
        hit = (hit << 1) | (u >> 31);
        umin = min(umin, u);
    }
    uint32_t und = nonloc | ((nxf == nxf) ? 0u : 0xffffu);
    if (umin <= k2B) {
#pragma unroll
        for (int k = 0; k < kK; ++k) {
            const float2 l = my_l[k * 32];
            und |= (uint32_t)(__float_as_uint(fmaf(l.x, nxf, fmaf(l.y, nyf, cf))) <= k2B) << k;
        }
    }
    und &= sure;
    par ^= hit & sure & ~und;
    const uint32_t ex = und | (cm & ~sure);
    if (__any_sync(0xffffffffu, ex != 0)) {
#pragma unroll 1
        for (int k = 0; k < kK; ++k) {
            if (ex >> k & 1u) {
                const double2 p = my_g[k * 32];
                int cnt = 0;
                bool bnd = false;
                exact_robust(p.x, p.y, tol, tol2, r, cnt, bnd);
                par ^= (uint32_t)(cnt & 1) << k;
                auxm |= (uint32_t)bnd << k;
            }
        }
    }
}

template <int MODE>
__global__ void __launch_bounds__(kTPB, MODE == kRobust ? 2 : 3) pip_tile_kernel(const double2* __restrict__ pts, uint64_t n,
                                                        const uint2* __restrict__ filt,
                                                        const EdgeRec* __restrict__ rec, uint32_t n_edges,
                                                        uint32_t edges_per_chunk,
                                                        const unsigned long long* __restrict__ bbox_keys,
                                                        int prefilter, double tol, double tol2,
                                                        uint32_t* __restrict__ inside_bits,
                                                        uint32_t* __restrict__ aux_bits,
                                                        const uint32_t* __restrict__ n_dev) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SingleShared<MODE>& sh = *reinterpret_cast<SingleShared<MODE>*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (n_dev) n = min(n, (uint64_t)*n_dev); // bucketed input: only the in-box prefix is live
    const uint64_t cta_base = (uint64_t)blockIdx.x * (kTPB * kK);
    if (cta_base >= n) return;
    const uint32_t e_begin = blockIdx.y * edges_per_chunk;
    const uint32_t e_end = min(n_edges, e_begin + edges_per_chunk);
    const uint64_t wbase = cta_base + (uint64_t)warp * 32 * kK; // this warp's first point (global)

    const uint32_t cta_n = (uint32_t)min((uint64_t)(kTPB * kK), n - cta_base);
    if (tid == 0) {
        mbar_init(&sh.full[0], 1);
        mbar_init(&sh.full[1], 1);
        mbar_init(&sh.pbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint32_t n_tiles = (e_end - e_begin + kTile - 1) / kTile;
    if (tid == 0) {
        for (uint32_t q = 0; q < 2 && q < n_tiles; ++q)
            issue_tile(sh, (int)q, filt, rec, e_begin + q * kTile, min((uint32_t)kTile, e_end - e_begin - q * kTile));
    }

    // ---- keys of this thread's points (coordinates stay in shared memory) ----
    double minx = 0, miny = 0, maxx = 0, maxy = 0;
    if (prefilter) {
        minx = dkey_inv(bbox_keys[0]);
        miny = dkey_inv(bbox_keys[1]);
        maxx = dkey_inv(~bbox_keys[2]);
        maxy = dkey_inv(~bbox_keys[3]);
    }
    const uint32_t wloc = (uint32_t)warp * 32 * kK; // this warp's first point within the CTA
    LocalMap lm{};
    {
        lm.x0 = dkey_inv(bbox_keys[0]);
        lm.y0 = dkey_inv(bbox_keys[1]);
        lm.sx = reinterpret_cast<const double*>(bbox_keys)[6];
        lm.sy = reinterpret_cast<const double*>(bbox_keys)[7];
    }
    Keys<MODE> K;
    uint32_t act = 0, nonloc = 0; // nonloc (C1): active points without local fp32 coordinates
    const QMap qm = {reinterpret_cast<const double*>(bbox_keys)[4], reinterpret_cast<const double*>(bbox_keys)[5]};
#pragma unroll
    for (int k = 0; k < kK; ++k) {
        const uint32_t li = wloc + k * 32 + lane;
        bool a = li < cta_n;
        double2 p = make_double2(0.0, 0.0);
        {
            if (a) p = pts[cta_base + li];
            if ((k & 3) == 3) asm volatile("" ::: "memory"); // at most 4 point loads in flight (registers)
        }
        if (a && prefilter) a = p.x >= minx && p.x <= maxx && p.y >= miny && p.y <= maxy; // batch.hpp:39-41
        {
            // polygon-local fp32 coordinates; NaN outside the bbox / without a map (-> exact side test)
            const double lxd = __dmul_rn(__dsub_rn(p.x, lm.x0), lm.sx), lyd = __dmul_rn(__dsub_rn(p.y, lm.y0), lm.sy);
            const bool ok = lm.sx != 0.0 && lxd >= 0.0 && lxd < 1.0 && lyd >= 0.0 && lyd < 1.0;
            const float nan = __int_as_float(0x7fc00000);
            sh.pts[li] = ok ? make_float2(__double2float_rn(lxd), __double2float_rn(lyd)) : make_float2(nan, nan);
            nonloc |= (uint32_t)(a && !ok) << k;
        }
        if constexpr (MODE == kRobust) {
            K.ka[k] = a ? fkey(__dadd_rn(p.y, tol)) : INT_MIN;
            K.kb[k] = a ? fkey(__dsub_rn(p.y, tol)) : INT_MAX;
        } else {
            const uint32_t q = (a ? qkey15(p.y, qm) : 0x7fffu) << 1; // inactive: masked by `act` (slow path)
            if (k & 1) K.k2[k >> 1] |= q << 16;
            else K.k2[k >> 1] = q;
        }
        act |= (uint32_t)a << k;
    }
    const bool warp_live = __any_sync(0xffffffffu, act != 0);
    // key range of the warp's active points (C1 "all sure" shortcut)
    uint32_t wkey_lo = 0xffffu, wkey_hi = 0u;
    if constexpr (MODE != kRobust) {
        uint32_t lo = 0xffffu, hi = 0u;
#pragma unroll
        for (int k = 0; k < kK; ++k) {
            if (act >> k & 1u) {
                const uint32_t q = (K.k2[k >> 1] >> (16 * (k & 1) + 1)) & 0x7fffu;
                lo = min(lo, q);
                hi = max(hi, q);
            }
        }
        wkey_lo = __reduce_min_sync(0xffffffffu, lo);
        wkey_hi = __reduce_max_sync(0xffffffffu, hi);
    }
    // warp-level interval test (Robust): some point may straddle only if
    // max key(p.y + tol) >= key(ylo) and min key(p.y - tol) <= key(yhi)
    int wka_max = INT_MIN, wkb_min = INT_MAX;
    if constexpr (MODE == kRobust) {
        int hi = INT_MIN, lo = INT_MAX;
#pragma unroll
        for (int k = 0; k < kK; ++k) {
            if (act >> k & 1u) {
                hi = max(hi, K.ka[k]);
                lo = min(lo, K.kb[k]);
            }
        }
        wka_max = __reduce_max_sync(0xffffffffu, hi);
        wkb_min = __reduce_min_sync(0xffffffffu, lo);
    }
    // may any active point of the warp straddle edge f?  (exact: the keys are
    // monotone; the per-point filter and the slow path then decide per point)
    auto warp_may = [&](uint32_t lo, uint32_t hi) {
        if constexpr (MODE == kRobust) return ((int)lo <= wka_max) & ((int)hi >= wkb_min);
        else return (lo <= wkey_hi) & (hi >= wkey_lo);
    };

    uint32_t par = 0, auxm = 0;
    for (uint32_t q = 0; q < n_tiles; ++q) {
        const int s = (int)(q & 1);
        const uint32_t t0 = e_begin + q * kTile;
        const uint32_t nt = min((uint32_t)kTile, e_end - t0);
        mbar_wait(&sh.full[s], (q >> 1) & 1);
        const TileStage& T = sh.st[s];
        if (warp_live) {
            // the stage's shared address, opaque to the compiler: kept in a
            // register instead of being re-derived from the CTA's shared window
            // base on every step of the edge loop
            unsigned st_s = smem_u32(&T);
            asm volatile("" : "+r"(st_s));
            const unsigned filt_s = st_s + (unsigned)offsetof(TileStage, filt);
            // process one group of 4 edges that passed the warp-level test
            auto group = [&](uint32_t e0) {
                // per-point filter of the 4 edges, then one warp-wide OR says
                // which of them need the slow path
                bool c[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) c[u] = lane_candidate<MODE>(K, lds_u2(filt_s + 8u * (e0 + u)));
                // common case: no candidate in the warp for any of the 4 edges
                if (!__any_sync(0xffffffffu, c[0] | c[1] | c[2] | c[3])) return;
                uint32_t bits = 0;
#pragma unroll
                for (int u = 0; u < 4; ++u) bits |= (uint32_t)c[u] << u;
                uint32_t todo = __reduce_or_sync(0xffffffffu, bits);
                if (nt - e0 < 4) todo &= (1u << (nt - e0)) - 1u; // stale tail entries
                while (todo) {
                    const uint32_t e = e0 + (__ffs(todo) - 1);
                    todo &= todo - 1;
                    const uint2 f = lds_u2(filt_s + 8u * e);
                    const EdgeRec rec_e = lds_rec(st_s + (unsigned)sizeof(EdgeRec) * e);
                    // ---- slow path: exact binary64 test for the candidate points ----
                    if constexpr (MODE == kC1)
                        slow_c1(sh.pts + wloc + lane, pts + cta_base + wloc + lane, K, act, nonloc, f, rec_e, par,
                                wkey_lo, wkey_hi);
                    else if constexpr (MODE == kC2)
                        slow_c2(sh.pts + wloc + lane, pts + cta_base + wloc + lane, K, act, nonloc, f, rec_e, par,
                                auxm, wkey_lo, wkey_hi);
                    else
                        slow_robust(sh.pts + wloc + lane, pts + cta_base + wloc + lane, K, act, nonloc, f, rec_e,
                                    tol, tol2, par, auxm, wka_max, wkb_min);
                }
            };
            // warp-level interval test (warp-uniform: the key range of the warp's
            // points against each edge's key range), 8 edges per step with the
            // loads of both halves issued together; the stage's shared address is
            // formed once per tile
            const unsigned wkr_s = st_s + (unsigned)offsetof(TileStage, wkr);
            for (uint32_t e0 = 0; e0 < nt; e0 += 8) {
                uint4 r[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(r[j].x), "=r"(r[j].y), "=r"(r[j].z), "=r"(r[j].w)
                                 : "r"(wkr_s + (e0 + 2 * j) * 8u));
                const bool pa = warp_may(r[0].x, r[0].y) | warp_may(r[0].z, r[0].w) | warp_may(r[1].x, r[1].y) |
                                warp_may(r[1].z, r[1].w);
                const bool pb = warp_may(r[2].x, r[2].y) | warp_may(r[2].z, r[2].w) | warp_may(r[3].x, r[3].y) |
                                warp_may(r[3].z, r[3].w);
                if (pa) group(e0);
                if (pb && e0 + 4 < nt) group(e0 + 4);
            }
        }
        __syncthreads(); // stage s fully consumed
        if (tid == 0 && q + 2 < n_tiles)
            issue_tile(sh, s, filt, rec, t0 + 2 * kTile, min((uint32_t)kTile, e_end - (t0 + 2 * kTile)));
    }

    // ---- flags: one ballot word per k-slice ----
#pragma unroll
    for (int k = 0; k < kK; ++k) {
        const uint32_t b = __ballot_sync(0xffffffffu, (par & act) >> k & 1u);
        const uint32_t a = __ballot_sync(0xffffffffu, (auxm & act) >> k & 1u);
        const uint64_t i0 = wbase + k * 32;
        if (lane == 0 && i0 < n) {
            if (b) atomicXor(&inside_bits[i0 >> 5], b);
            if (a) atomicOr(&aux_bits[i0 >> 5], a);
        }
    }
}

int sms(int dev) {
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
}

template <int MODE>
cudaError_t launch_t(const SingleArgs& a, cudaStream_t st, int dev, uint64_t* launches) {
    const size_t smem = sizeof(SingleShared<MODE>);
    static bool attr[64] = {};
    if (dev < 64 && !attr[dev]) {
        cudaFuncSetAttribute(pip_tile_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr[dev] = true;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pip_tile_kernel<MODE>, kTPB, smem);
    per_sm = std::max(per_sm, 1);
    const uint64_t pts_per_cta = (uint64_t)kTPB * kK;
    const uint64_t n_ptiles = (a.n + pts_per_cta - 1) / pts_per_cta;
    const uint64_t slots = (uint64_t)sms(dev) * per_sm;
    // Split the edges so the grid covers >= ~4 waves; chunks are whole tiles.
    const uint64_t tiles = std::max<uint64_t>(1, (a.n_edges + kTile - 1) / kTile);
    uint64_t chunks = std::max<uint64_t>(1, (4 * slots + n_ptiles - 1) / std::max<uint64_t>(n_ptiles, 1));
    chunks = std::min<uint64_t>(std::min<uint64_t>(chunks, tiles), 65535);
    const uint64_t tiles_per_chunk = (tiles + chunks - 1) / chunks;
    const uint32_t per_chunk = (uint32_t)(tiles_per_chunk * kTile);
    chunks = (tiles + tiles_per_chunk - 1) / tiles_per_chunk;
    dim3 grid((unsigned)n_ptiles, (unsigned)chunks);
    pip_tile_kernel<MODE><<<grid, kTPB, smem, st>>>(reinterpret_cast<const double2*>(a.pts), a.n, a.filt,
                                                   reinterpret_cast<const EdgeRec*>(a.rec), a.n_edges, per_chunk,
                                                   a.bbox_keys, a.prefilter, a.tol, a.tol2, a.inside_bits,
                                                   a.aux_bits, a.n_dev);
    ++*launches;
    return cudaGetLastError();
}

} // namespace

cudaError_t launch_single(const SingleArgs& a, cudaStream_t st, int dev, uint64_t* launches) {
    if (a.n == 0) return cudaSuccess;
    switch (a.mode) {
    case kC1: return launch_t<kC1>(a, st, dev, launches);
    case kC2: return launch_t<kC2>(a, st, dev, launches);
    default: return launch_t<kRobust>(a, st, dev, launches);
    }
}

} // namespace pcd
