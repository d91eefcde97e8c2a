// Single-polygon kernel (configs 1, 2, 4; classify_batch / contains over one
// polygon with holes): the point-edge scan of count_crossings_c1/_c2 /
// robust_ray_crossings (geometry.hpp:182-273) for every point of a batch.
//
// Work decomposition: CTA (bx, by) classifies points [bx*kTPB*K, +kTPB*K)
// against edges [by*chunk, +chunk); partial parities are XOR-ed and
// Error/Boundary flags OR-ed into the bit planes, so edge chunks combine
// exactly like the reference's per-ring sums (geometry.hpp:285-299).
//
// Per thread: K points, of which only the filter keys live in registers
// (coordinates sit in shared memory as polygon-local fp32, the binary64
// fallbacks re-read them from L2); parity and aux flags are K-bit masks.  Warp
// w owns K*32 consecutive points (k-slice k = 32 consecutive points), which
// after y-bucketing (pip_sort.cu) are y-adjacent.
//
// The linear scan has two phases per CTA (every edge of the chunk is examined
// for every CTA):
//  1. Key scan.  The chunk's 4-byte edge key words (q(ylo), q(yhi) on the
//     15-bit monotone map, prep_edges_kernel) stream through shared memory in
//     8 KB tiles (TMA bulk copies, 2-stage mbarrier pipeline).  Each thread
//     tests 8 edges per tile against the key range of ALL the CTA's points --
//     one packed add + and per edge -- and appends the (rare) candidates to a
//     shared list.  Exact: a non-candidate has both endpoints strictly above or
//     below every point, so the reference counts nothing for it.
//  2. Candidates.  The list's filter words and exact records are gathered
//     from L2 into shared memory, 128 at a time, and every warp runs the
//     per-point filter and the exact / certified edge test of the reference
//     (slow_c1 / slow_c2 / slow_robust) on them.
#include "pip_kernels.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <climits>
#include <type_traits>

#include "pip_device.cuh"

#ifndef PC_EMPTYBAR
#define PC_EMPTYBAR 0
#endif
#ifndef PC_PF
#define PC_PF 1
#endif
#ifndef PC_PF_DIST
#define PC_PF_DIST 64
#endif

namespace pcd {

namespace {

#ifndef PC_TPB
#define PC_TPB 256
#endif
#ifndef PC_KPT
#define PC_KPT 16
#endif
constexpr int kTPB = PC_TPB;    // threads per CTA
constexpr int kK = PC_KPT;      // points per thread (a CTA holds kTPB * kK points)
constexpr uint32_t kAllK = kK >= 32 ? 0xffffffffu : (1u << kK) - 1u; // a mask of all of a thread's points
#ifndef PC_QTILE
#define PC_QTILE kKeyTile
#endif
#ifndef PC_LISTCAP
#define PC_LISTCAP 4096
#endif
#ifndef PC_BATCH
#define PC_BATCH (PC_TPB / 2)
#endif
#ifndef PC_MINB
#define PC_MINB 3
#endif
#ifndef PC_MINB_C2
#define PC_MINB_C2 2 // C2: 2 CTAs/SM at 128 registers, no spills (c4 kernel 4.65 -> 3.79 ms, c1 0.093 -> 0.079)
#endif
#ifndef PC_MINB_SMALL
#define PC_MINB_SMALL 2 // C1, one CTA per point tile and <= PC_SMALL_EDGES edges (c1 kernel 0.091 -> 0.081 ms)
#endif
#ifndef PC_SMALL_EDGES
#define PC_SMALL_EDGES 2048 // (n = 1e4 edges is 8% slower at 2 CTAs/SM, n = 1e3 10% faster)
#endif
constexpr int kQTile = PC_QTILE; // edge key words per shared-memory stage (8 KB; 8 per thread)
static_assert(kKeyTile % kQTile == 0 || kQTile % kKeyTile == 0, "tiles and the key array's padding");
#ifndef PC_EPI
#define PC_EPI 8 // epilogue: original indices requested at a time
#endif
#ifndef PC_PRO
#define PC_PRO 4 // prologue: point loads in flight per thread
#endif
#ifndef PC_PRO2
#define PC_PRO2 16 // prologue, second pass (per-CTA keys): y loads in flight per thread
#endif
#ifndef PC_QSTAGES
#define PC_QSTAGES 2
#endif
constexpr int kStages = PC_QSTAGES; // key-scan stages in flight
#ifndef PC_WARPKEYS
#define PC_WARPKEYS 0 // 1: phase 1 per warp (own bulk-copy stages and mbarriers, no CTA barrier per tile)
#endif
constexpr int kWarpsCta = PC_TPB / 32;
#ifndef PC_KSPLIT_TILES
#define PC_KSPLIT_TILES 8 // chunks of at least this many key tiles: the CTAs of a cluster split them
#endif
#ifndef PC_KSPLIT_G
#define PC_KSPLIT_G 2 // CTAs per cluster that split the key tiles (2 or 4)
#endif
static_assert(PC_KSPLIT_G == 2 || PC_KSPLIT_G == 4, "key split over 2 or 4 CTAs");
constexpr uint32_t kWT = kQTile / kWarpsCta; // per-warp tile: edge key words per stage (8 per lane)
static_assert(!PC_WARPKEYS || kWT == 256u, "per-warp tiles of 8 key words per lane");
constexpr int kListCap = PC_LISTCAP; // candidate edge indices; a tile can add kQTile, so flush above kListCap - kQTile
static_assert(kListCap >= (PC_WARPKEYS ? kQTile / (PC_TPB / 32) : kQTile), "the list must hold one tile's candidates");
constexpr int kBatch = PC_BATCH;     // candidates gathered per batch (two threads each)
static_assert(kBatch <= PC_TPB / 2, "the gather uses two threads per candidate");
constexpr int kEPT = kQTile / kTPB; // phase 1: key words per thread per tile
static_assert(kEPT == 16 || kEPT == 8, "phase 1: whole groups of 8 edges (8 key words) per thread");

// Every mode keeps only the polygon-local fp32 coordinates of its points in
// shared memory (the certified fp32 side / intercept test); the binary64
// fallbacks re-read the point from global memory (L2).
struct SingleShared {
    float2 pts[kTPB * kK];       // this CTA's points (bucketed order), local fp32
    uint4 qk[kStages][kQTile / 4]; // key-scan stages
    uint32_t list[kListCap];     // candidate edges of the chunk (phase 1 -> phase 2)
    uint2 bfilt[kBatch];         // gathered per-point filter words
    EdgeRec brec[kBatch];        // gathered exact records
    unsigned long long full[PC_WARPKEYS ? kStages * kWarpsCta : kStages];
    unsigned long long empty[kStages]; // key split: stage consumed by all kWarpsCta warps (PC_EMPTYBAR)
    uint32_t ncand;
    uint32_t scan_from;          // SPLIT = 2: this round's first tile (min over warps)
    uint32_t valid_end;          // per-warp phase 1: end of the reservations that fit the list
    uint32_t any_ovf;            // per-warp phase 1: some warp stopped on a full list
    uint32_t cta_lo, cta_hi;     // key range of the CTA's active points
    unsigned long long cta_ylo, cta_yhi; // C1/C2: dkey of their min / max y (per-CTA key map)
    uint32_t live;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait_at(unsigned bar, unsigned parity) { // bar: shared-window address
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    }
}

// One elected thread: load key words [t0, t0 + nw) into stage s (nw <= kQTile,
// a multiple of 8: whole key groups, 16-byte bulk copies; the key array is padded with
// never-candidate words to whole tiles, so nw may run past the chunk's end).
// The key array is re-read by every CTA: keep it in L2 (evict_last), while the
// point loads stream past it (evict_first, see load_pt).
__device__ __forceinline__ void issue_tile(SingleShared& sh, int s, const uint32_t* qk, uint32_t t0, uint32_t nw) {
    const unsigned bytes = nw * 4u;
    const unsigned bar = smem_u32(&sh.full[s]);
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(sh.qk[s])),
        "l"(qk + t0), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}

// Thread-block-cluster helpers (SPLIT = 2).
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned dsmem_addr(const void* p, unsigned rank) { // p in this CTA -> rank's copy
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ uint32_t dsmem_ld(unsigned a) {
    uint32_t v;
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void dsmem_st(unsigned a, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t dsmem_add(unsigned a, uint32_t v) {
    uint32_t old;
    asm volatile("atom.shared::cluster.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void dsmem_max(unsigned a, uint32_t v) {
    uint32_t old;
    asm volatile("atom.shared::cluster.max.u32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
}

__device__ __forceinline__ double2 load_pt(const double2* p) {
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    double2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}

// Phase-1 test of two edges at once.  A = {q(ylo) of edge 2i, of edge 2i+1}
// and B = {0x7fff - q(yhi), ...} (the key array's layout, prep_edges_body);
// with the CTA constants KA = 0x7fff - cta_hi and KB = cta_lo in both halves,
// per half u = q(ylo) + KA and v = (0x7fff - q(yhi)) + KB stay below 2^16
// (keys <= 0x7ffe), u <= 0x7fff iff q(ylo) <= cta_hi and v <= 0x7fff iff
// q(yhi) >= cta_lo.  So the top bit of max(u, v) -- one VIADDMNMX.U16x2 after
// the add of B -- is clear iff the edge's key range meets the CTA's.
__device__ __forceinline__ uint32_t key_pair(uint32_t a, uint32_t b, uint32_t ka, uint32_t kb) {
    return __viaddmax_u16x2(a, ka, b + kb);
}

constexpr uint32_t kAllEPT = (1u << kEPT) - 1u;
// Phase-1 candidate mask of one thread's kEPT key words against the key-range
// constants (ka, kb) of key_pair: bit i set iff edge i of the words may meet a
// point of that range; the common all-clear case costs the pair tests + folds.
__device__ __forceinline__ uint32_t key_mask(const uint32_t (&d)[kEPT], uint32_t ka, uint32_t kb) {
    uint32_t t[kEPT / 2];
#pragma unroll
    for (int g = 0; g < kEPT / 8; ++g)
#pragma unroll
        for (int i = 0; i < 4; ++i) t[4 * g + i] = key_pair(d[8 * g + i], d[8 * g + 4 + i], ka, kb);
    uint32_t mn = __vimin3_u16x2(t[0], t[1], t[2]);
#pragma unroll
    for (int i = 3; i < kEPT / 2; i += 2) mn = __vimin3_u16x2(mn, t[i], t[min(i + 1, kEPT / 2 - 1)]);
    if ((mn & 0x80008000u) == 0x80008000u) return 0u;
    uint32_t m = 0;
#pragma unroll
    for (int g = 0; g < kEPT / 8; ++g)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t nt = ~t[4 * g + i];
            m |= ((nt >> 15) & 1u) << (8 * g + 2 * i);
            m |= (nt >> 31) << (8 * g + 2 * i + 1);
        }
    return m;
}


// A lane's binary64 points for the exact fallbacks: point k of the lane is g[k * 32].
struct PtRef {
    const double2* __restrict__ g;
    __device__ __forceinline__ double2 operator[](int j) const { return g[j]; }
};

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
__device__ __forceinline__ void slow_c1(const float2* my_l, const PtRef& my_g, const Keys<kC1>& K,
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
    uint32_t und = nonloc | ((nxf == nxf) ? 0u : kAllK);
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
__device__ __forceinline__ void slow_c2(const float2* my_l, const PtRef& my_g, const Keys<kC2>& K,
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
    uint32_t und = nonloc | ((nxf == nxf) ? 0u : kAllK);
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
__device__ __forceinline__ void slow_robust(const float2* my_l, const PtRef& my_g,
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
    uint32_t und = nonloc | ((nxf == nxf) ? 0u : kAllK);
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

template <int MODE, int SPLIT, bool SMALL = false>
__global__ void __launch_bounds__(kTPB, kTPB >= 512 ? 2 : (MODE == kRobust ? 2 : (MODE == kC2 ? PC_MINB_C2 : (SMALL ? PC_MINB_SMALL : PC_MINB))))
    pip_tile_kernel(const double2* __restrict__ pts, uint64_t n, const uint32_t* __restrict__ qk,
                    const uint2* __restrict__ filt, const EdgeRec* __restrict__ rec, uint32_t n_edges,
                    uint32_t edges_per_chunk, const unsigned long long* __restrict__ bbox_keys, int prefilter,
                    double tol, double tol2, uint32_t* __restrict__ inside_bits, uint32_t* __restrict__ aux_bits,
                    const uint32_t* __restrict__ n_dev, const uint32_t* __restrict__ orig) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SingleShared& sh = *reinterpret_cast<SingleShared*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (n_dev) n = min(n, (uint64_t)*n_dev); // bucketed input: only the in-box prefix is live
    const uint64_t cta_base = (uint64_t)blockIdx.x * (kTPB * kK);
    // SPLIT = 2: both CTAs of a pair take part in the key scan, also one without
    // points (the grid is rounded up to whole pairs)
    if (SPLIT == 1 && cta_base >= n) return;
    const uint32_t e_begin = blockIdx.y * edges_per_chunk;
    const uint32_t e_end = min(n_edges, e_begin + edges_per_chunk);
    if (e_begin >= e_end) return;
    const uint64_t wbase = cta_base + (uint64_t)warp * 32 * kK; // this warp's first point (global)
#if PC_PF
    // L2 prefetch of a point tile (and its original indices) a later CTA will
    // read -- the tile PC_PF_DIST further on -- so that its prologue and
    // epilogue wait on L2 instead of DRAM: one bulk prefetch per array, thread
    // 0.  c4 kernel 3.36 -> 3.20 ms for any distance from 16 to 148 tiles
    // (444, a whole resident set ahead: 3.26; 888: no gain).
    if (tid == 0 && blockIdx.y == 0) {
        const uint64_t nb = cta_base + (uint64_t)PC_PF_DIST * (kTPB * kK);
        if (nb < n) {
            const uint32_t cnt = (uint32_t)min((uint64_t)(kTPB * kK), n - nb);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pts + nb), "r"(cnt * 16u) : "memory");
            if (orig && (cnt & 3u) == 0u)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(orig + nb), "r"(cnt * 4u) : "memory");
        }
    }
#endif

    const uint32_t cta_n = cta_base >= n ? 0u : (uint32_t)min((uint64_t)(kTPB * kK), n - cta_base);
    if (tid == 0) {
        for (int k = 0; k < (PC_WARPKEYS ? kStages * kWarpsCta : kStages); ++k) mbar_init(&sh.full[k], 1);
        for (int k = 0; k < kStages; ++k) mbar_init(&sh.empty[k], kWarpsCta);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        sh.ncand = 0;
        sh.valid_end = 0;
        sh.any_ovf = 0;
        sh.cta_lo = 0xffffu;
        sh.cta_hi = 0u;
        sh.cta_ylo = ~0ull;
        sh.cta_yhi = 0ull;
        sh.live = 0;
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
    uint32_t act = 0, nonloc = 0; // nonloc: active points without local fp32 coordinates
    uint32_t qlo = 0xffffu, qhi = 0u; // this thread's range of phase-1 keys
    unsigned long long ylo_k = ~0ull, yhi_k = 0ull; // C1/C2: monotone keys of its min / max p.y
    const QMap qm = {reinterpret_cast<const double*>(bbox_keys)[4], reinterpret_cast<const double*>(bbox_keys)[5]};
    __syncthreads(); // shared counters initialised
#pragma unroll
    for (int k = 0; k < kK; ++k) {
        const uint32_t li = wloc + k * 32 + lane;
        bool a = li < cta_n;
        double2 p = make_double2(0.0, 0.0);
        {
            PC_DCHECK(!a || cta_base + li < n);
            if (a) p = load_pt(pts + cta_base + li);
            if ((k & (PC_PRO - 1)) == PC_PRO - 1) asm volatile("" ::: "memory"); // at most PC_PRO point loads in flight (registers)
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
            if (a) { // phase-1 range: q(RN(p.y - tol)) .. q(RN(p.y + tol))
                qlo = min(qlo, qkey15(__dsub_rn(p.y, tol), qm));
                qhi = max(qhi, qkey15(__dadd_rn(p.y, tol), qm));
            }
        } else {
            if (a) { // phase-1 range (global map) and the CTA's exact y range
                const uint32_t q = qkey15(p.y, qm);
                qlo = min(qlo, q);
                qhi = max(qhi, q);
                ylo_k = min(ylo_k, dkey(p.y));
                yhi_k = max(yhi_k, dkey(p.y));
            }
        }
        act |= (uint32_t)a << k;
    }
    // key range of the warp's active points (phase 1; C1/C2 re-key below)
    uint32_t wkey_lo = __reduce_min_sync(0xffffffffu, qlo), wkey_hi = __reduce_max_sync(0xffffffffu, qhi);
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
    } else {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            ylo_k = min(ylo_k, __shfl_xor_sync(0xffffffffu, ylo_k, o));
            yhi_k = max(yhi_k, __shfl_xor_sync(0xffffffffu, yhi_k, o));
        }
    }
    const bool warp_live = __any_sync(0xffffffffu, act != 0);
    if (lane == 0 && warp_live) {
        atomicMin(&sh.cta_lo, wkey_lo);
        atomicMax(&sh.cta_hi, wkey_hi);
        if constexpr (MODE != kRobust) {
            atomicMin(&sh.cta_ylo, ylo_k);
            atomicMax(&sh.cta_yhi, yhi_k);
        }
        sh.live = 1;
    }
    __syncthreads(); // points staged, CTA key range complete
    if (SPLIT == 1 && !sh.live) return; // no active point: nothing to classify (uniform)
    // C1/C2 per-point keys on the CTA's own y range (y-bucketed CTAs span a thin
    // slab, so the 15-bit keys resolve ~2^27 levels over the polygon and key ties
    // -- which take the binary64 path -- stay rare even for edges far shorter
    // than the polygon's height / 2^15).  Any monotone map is exact.
    CtaQMap cm{};
    if constexpr (MODE != kRobust) {
        cm = ctaqmap_from_range(dkey_inv(sh.cta_ylo), dkey_inv(sh.cta_yhi));
        uint32_t lo = 0xffffu, hi = 0u;
#pragma unroll
        for (int k0 = 0; k0 < kK; k0 += PC_PRO2) { // the points' y again (L1 / L2), PC_PRO2 loads in flight
            double y[PC_PRO2];
#pragma unroll
            for (int k = 0; k < PC_PRO2; ++k)
                y[k] = (act >> (k0 + k) & 1u) ? pts[cta_base + wloc + (k0 + k) * 32 + lane].y : 0.0;
#pragma unroll
            for (int k = k0; k < k0 + PC_PRO2; ++k) {
                const bool a = act >> k & 1u;
                const uint32_t q = a ? qkey_cta(y[k - k0], cm) : 0x7fffu; // inactive: masked by `act`
                if (k & 1) K.k2[k >> 1] |= (q << 1) << 16;
                else K.k2[k >> 1] = q << 1;
                if (a) {
                    lo = min(lo, q);
                    hi = max(hi, q);
                }
            }
        }
        wkey_lo = __reduce_min_sync(0xffffffffu, lo);
        wkey_hi = __reduce_max_sync(0xffffffffu, hi);
    }
    const uint32_t ka = (0x7fffu - sh.cta_hi) * 0x10001u, kb = sh.cta_lo * 0x10001u; // key_pair constants

    const uint32_t t_begin = e_begin, n_tiles = (e_end - e_begin + kQTile - 1) / kQTile;
    // words of tile q: whole tiles, the chunk's last one rounded up to a group of 8
    auto tile_words = [&](uint32_t q) { return min((uint32_t)kQTile, (e_end - (t_begin + q * kQTile) + 7u) & ~7u); };
#if PC_WARPKEYS
    // per-warp key stream: warp w scans warp tiles j = w, w + kWarpsCta, ... (kWT
    // edges each) through its own kStages 1 KB stages; copy k of the warp uses
    // stage k % kStages at mbarrier parity (k / kStages) & 1
    const uint32_t n_wt = (e_end - e_begin + kWT - 1) / kWT;
    const unsigned wbar0 = smem_u32(&sh.full[warp * kStages]);
    const unsigned wst0 = smem_u32(&sh.qk[0][0]) + (unsigned)warp * kStages * (kWT * 4u);
    uint32_t j_issue = (uint32_t)warp, seq_issued = 0; // uniform per warp
    auto issue_w = [&]() {
        if (lane == 0) {
            const uint32_t t0 = e_begin + j_issue * kWT;
            const unsigned bytes = min(kWT, (e_end - t0 + 7u) & ~7u) * 4u; // whole groups of 8 (padded array)
            const unsigned st = seq_issued % kStages;
            const unsigned bar = wbar0 + 8u * st;
            unsigned long long pol;
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                    wst0 + st * (kWT * 4u)),
                "l"(qk + t0), "r"(bytes), "r"(bar), "l"(pol)
                : "memory");
        }
        ++seq_issued;
        j_issue += kWarpsCta;
    };
    while (seq_issued < (uint32_t)kStages && j_issue < n_wt) issue_w();
#else
    // (SPLIT = 2: the key tiles of a pair are issued round by round in phase 1)
    if (SPLIT == 1 && tid == 0) {
        for (uint32_t q = 0; q < (uint32_t)kStages && q < n_tiles; ++q)
            issue_tile(sh, (int)q, qk, t_begin + q * kQTile, tile_words(q));
    }
#endif

    // may any active point of the warp straddle the edge with filter word f?
    // (exact: the keys are monotone; the per-point filter then decides per point)
    auto warp_may = [&](uint2 f) {
        if constexpr (MODE == kRobust) {
            return ((int)f.x <= wka_max) & ((int)f.y >= wkb_min);
        } else {
            const uint32_t klo = (0x8000u - ((f.x & 0xffffu) >> 1)) & 0x7fffu;
            const uint32_t khi = klo + (((f.y & 0xffffu) - 2u) >> 1);
            return (klo <= wkey_hi) & (khi >= wkey_lo);
        }
    };

    const PtRef my_g{pts + cta_base + wloc + lane};
    uint32_t par = 0, auxm = 0;
    // ---- phase 2: classify against the listed candidate edges ----
    auto flush = [&](uint32_t nc) { // nc = sh.ncand, read by every thread before any could append again
        for (uint32_t b0 = 0; b0 < nc; b0 += kBatch) {
            const uint32_t nb = min((uint32_t)kBatch, nc - b0);
            { // gather: two threads per candidate (filter word + half of the record each)
                const uint32_t i = (uint32_t)tid >> 1, h = (uint32_t)tid & 1u;
                if (i < nb) {
                    PC_DCHECK(b0 + i < (uint32_t)kListCap && i < (uint32_t)kBatch);
                    const uint32_t e = sh.list[b0 + i];
                    PC_DCHECK(e >= e_begin && e < e_end);
                    const uint4* src = reinterpret_cast<const uint4*>(rec + e) + 2 * h;
                    uint4* dst = reinterpret_cast<uint4*>(&sh.brec[i]) + 2 * h;
                    const uint4 r0 = __ldg(src), r1 = __ldg(src + 1);
                    if (h == 0) {
                        if constexpr (MODE == kRobust) {
                            sh.bfilt[i] = __ldg(filt + e);
                        } else { // the per-point filter word on the CTA's key map (as prep_edges_kernel)
                            const double ay = __hiloint2double((int)r0.w, (int)r0.z);
                            const double by = __hiloint2double((int)r1.y, (int)r1.x);
                            const double ylo = by < ay ? by : ay, yhi = ay < by ? by : ay;
                            const uint32_t klo = qkey_cta(ylo, cm), khi = qkey_cta(yhi, cm);
                            const uint32_t neg = ((0x8000u - klo) & 0x7fffu) << 1;
                            const uint32_t thr1 = ((khi - klo) << 1) + 2u;
                            sh.bfilt[i] = make_uint2(neg | (neg << 16), thr1 | (thr1 << 16));
                        }
                    }
                    dst[0] = r0;
                    dst[1] = r1;
                }
            }
            __syncthreads();
            if (warp_live) {
                for (uint32_t g = 0; g < nb; g += 4) {
                    bool c[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint2 f = sh.bfilt[min(g + u, nb - 1)];
                        c[u] = (g + u < nb) && warp_may(f) && lane_candidate<MODE>(K, f);
                    }
                    if (!__any_sync(0xffffffffu, c[0] | c[1] | c[2] | c[3])) continue;
                    uint32_t bits = 0;
#pragma unroll
                    for (int u = 0; u < 4; ++u) bits |= (uint32_t)c[u] << u;
                    uint32_t todo = __reduce_or_sync(0xffffffffu, bits);
                    while (todo) {
                        const uint32_t i = g + (__ffs(todo) - 1);
                        todo &= todo - 1;
                        const uint2 f = sh.bfilt[i];
                        const EdgeRec rec_e = sh.brec[i];
                        if constexpr (MODE == kC1)
                            slow_c1(sh.pts + wloc + lane, my_g, K, act, nonloc, f, rec_e, par,
                                    wkey_lo, wkey_hi);
                        else if constexpr (MODE == kC2)
                            slow_c2(sh.pts + wloc + lane, my_g, K, act, nonloc, f, rec_e, par,
                                    auxm, wkey_lo, wkey_hi);
                        else
                            slow_robust(sh.pts + wloc + lane, my_g, K, act, nonloc, f, rec_e,
                                        tol, tol2, par, auxm, wka_max, wkb_min);
                    }
                }
            }
            __syncthreads(); // batch buffers free
        }
        if (tid == 0) {
            sh.ncand = 0;
            sh.valid_end = 0;
            sh.any_ovf = 0;
        }
        __syncthreads();
    };

    // ---- phase 1: the key scan over the chunk ----
#if PC_WARPKEYS
    {
        uint32_t seq_done = 0, j_cur = (uint32_t)warp; // uniform per warp
        for (;;) { // rounds: a round ends when every warp finished or stopped on a full list
            bool stopped = false;
            while (j_cur < n_wt) {
                const unsigned st = seq_done % kStages;
                mbar_wait_at(wbar0 + 8u * st, (seq_done / kStages) & 1u);
                uint32_t d[8];
                {
                    const unsigned a = wst0 + st * (kWT * 4u) + 32u * (unsigned)lane;
                    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]) : "r"(a));
                    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]) : "r"(a + 16u));
                }
                uint32_t t[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) t[i] = key_pair(d[i], d[4 + i], ka, kb);
                const uint32_t mn = __vimin3_u16x2(__vimin3_u16x2(t[0], t[1], t[2]), t[3], t[3]);
                const bool mine = (mn & 0x80008000u) != 0x80008000u;
                ++seq_done;
                if (__any_sync(0xffffffffu, mine)) { // rare: reserve the warp's candidates at once
                    uint32_t m = 0;
                    if (mine) {
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const uint32_t nt = ~t[i];
                            m |= ((nt >> 15) & 1u) << (2 * i);
                            m |= (nt >> 31) << (2 * i + 1);
                        }
                    }
                    const uint32_t e0 = e_begin + j_cur * kWT + 8u * (uint32_t)lane;
                    if (e0 + 8u > e_end) m &= e0 >= e_end ? 0u : (1u << (e_end - e0)) - 1u;
                    const uint32_t c = (uint32_t)__popc(m);
                    uint32_t incl = c;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += y;
                    }
                    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
                    uint32_t base = 0;
                    if (lane == 0 && total) base = atomicAdd(&sh.ncand, total);
                    base = __shfl_sync(0xffffffffu, base, 0);
                    if (base + total <= (uint32_t)kListCap) {
                        uint32_t pos = base + incl - c;
                        while (m) {
                            sh.list[pos++] = e0 + (__ffs(m) - 1);
                            m &= m - 1;
                        }
                        if (lane == 0 && total) atomicMax(&sh.valid_end, base + total);
                    } else {
                        stopped = true; // uniform: this warp tile is redone after the flush
                    }
                }
                if (stopped) break;
                __syncwarp(); // every lane has read stage st
                if (j_issue < n_wt) issue_w();
                j_cur += kWarpsCta;
            }
            if (stopped) { // drain this warp's copies in flight, so its mbarriers agree with seq_*
                while (seq_done < seq_issued) {
                    mbar_wait_at(wbar0 + 8u * (seq_done % kStages), (seq_done / kStages) & 1u);
                    ++seq_done;
                }
                if (lane == 0) sh.any_ovf = 1u;
            }
            __syncthreads();
            const uint32_t nc = sh.valid_end;
            const bool again = sh.any_ovf != 0u;
            __syncthreads(); // read by everyone before flush resets them
            flush(nc);
            if (!again) break;
            if (stopped) { // resume at the tile that did not fit
                j_issue = j_cur;
                while (seq_issued < seq_done + (uint32_t)kStages && j_issue < n_wt) issue_w();
            }
        }
    }
#else
    if constexpr (SPLIT > 1) {
        // The SPLIT CTAs of a cluster (adjacent y slabs, the same edge chunk)
        // split the chunk's key tiles: CTA r scans tiles q = r, r + SPLIT, ... and
        // tests each edge against every member's key range, listing candidates in
        // its own list and -- through distributed shared memory -- in the others'.
        // Each CTA reads 1/SPLIT of the key bytes and waits on 1/SPLIT of the tile
        // barriers.  Lists never flush mid-scan: a warp whose reservation does not
        // fit stops listing for that member and records the tile (lo[]); after a
        // round every CTA classifies its list, and a new round rescans from the
        // earliest unlisted tile, listing each member only from its own lo on.
        const unsigned crank = cluster_rank();
        cluster_sync_all(); // every member's prologue (key range, live flag) is complete
        uint32_t mka[SPLIT], mkb[SPLIT], lo[SPLIT];
        uint32_t live_m = 0u; // bit r: member r has active points
#pragma unroll
        for (int r = 0; r < SPLIT; ++r) {
            const uint32_t l = dsmem_ld(dsmem_addr(&sh.cta_lo, (unsigned)r)), h = dsmem_ld(dsmem_addr(&sh.cta_hi, (unsigned)r));
            live_m |= (uint32_t)(dsmem_ld(dsmem_addr(&sh.live, (unsigned)r)) != 0u) << r;
            mka[r] = (0x7fffu - h) * 0x10001u; // key_pair constants of member r
            mkb[r] = l * 0x10001u;
            lo[r] = crank; // per warp: first of this CTA's tiles not yet listed for member r
        }
        unsigned qk_s = smem_u32(&sh.qk[0][(kEPT / 4) * tid]);
        asm volatile("" : "+r"(qk_s));
        const unsigned bar0 = smem_u32(&sh.full[0]);
        const unsigned ebar0 = smem_u32(&sh.empty[0]);
        (void)ebar0;
        constexpr uint32_t kDone = 0xffffffffu;
        uint32_t seq = 0; // copies issued (= consumed at round ends); uniform
        // warp-aggregated reservation of m's candidates (edges e0 + bit) in member
        // r's list: all of them or none; returns false when they do not fit
        auto list_warp = [&](uint32_t m, uint32_t e0, unsigned r) {
            const uint32_t c = (uint32_t)__popc(m);
            uint32_t incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
            if (total == 0u) return true;
            uint32_t base = 0;
            if (lane == 0) base = dsmem_add(dsmem_addr(&sh.ncand, r), total);
            base = __shfl_sync(0xffffffffu, base, 0);
            if (base + total > (uint32_t)kListCap) return false;
            const unsigned rl = dsmem_addr(&sh.list[0], r);
            uint32_t pos = base + incl - c;
            while (m) {
                PC_DCHECK(pos < (uint32_t)kListCap && e0 + (__ffs(m) - 1) < e_end && r < (unsigned)SPLIT);
                dsmem_st(rl + 4u * pos, e0 + (__ffs(m) - 1));
                ++pos;
                m &= m - 1;
            }
            if (lane == 0) dsmem_max(dsmem_addr(&sh.valid_end, r), base + total);
            return true;
        };
        // a cluster without any active point (e.g. past the in-box prefix of a
        // bucketed batch) has nothing to scan (live_m is the same in every
        // member); it still waits until every member has read the others' ranges
        // above, so no CTA leaves while a partner may read its shared memory
        // (live_m made opaque to the optimiser: with the idle test visible, ptxas
        // schedules the C2 instantiation's phase 2 worse -- c4 C2 kernel 4.86 vs
        // 4.65 ms, C1 / Robust unchanged; profiles/r2c_experiments.txt)
        asm volatile("" : "+r"(live_m));
        if (live_m == 0u) cluster_sync_all();
        for (; live_m != 0u;) { // rounds (cluster-uniform)
            uint32_t lmin = kDone;
#pragma unroll
            for (int r = 0; r < SPLIT; ++r) lmin = min(lmin, lo[r]);
            if (tid == 0) sh.scan_from = kDone;
            __syncthreads();
            if (lane == 0) atomicMin(&sh.scan_from, lmin);
            __syncthreads();
            const uint32_t from = sh.scan_from;
            uint32_t fail = 0u; // bit r: listing for member r stopped this round (warp-uniform)
            uint32_t q_issue = from;
            for (uint32_t k = 0; k < (uint32_t)kStages && q_issue < n_tiles; ++k, q_issue += SPLIT)
                if (tid == 0) issue_tile(sh, (int)((seq + k) % kStages), qk, t_begin + q_issue * kQTile, tile_words(q_issue));
            for (uint32_t q = from; q < n_tiles; q += SPLIT) {
                PC_DCHECK(q % SPLIT == crank);
                const unsigned st = seq % kStages;
                mbar_wait_at(bar0 + 8u * st, (seq / kStages) & 1u);
                uint32_t d[kEPT];
                {
                    const unsigned a = qk_s + st * (kQTile * 4u);
#pragma unroll
                    for (int j = 0; j < kEPT / 4; ++j)
                        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                     : "=r"(d[4 * j]), "=r"(d[4 * j + 1]), "=r"(d[4 * j + 2]), "=r"(d[4 * j + 3])
                                     : "r"(a + 16u * j));
                }
                const uint32_t e0 = t_begin + q * kQTile + (uint32_t)kEPT * (uint32_t)tid;
                const uint32_t emask = e0 + kEPT <= e_end ? kAllEPT : (e0 >= e_end ? 0u : (1u << (e_end - e0)) - 1u);
#pragma unroll
                for (int r = 0; r < SPLIT; ++r) {
                    const bool want = (live_m >> r & 1u) && !(fail >> r & 1u) && q >= lo[r]; // warp-uniform
                    const uint32_t m = want ? key_mask(d, mka[r], mkb[r]) & emask : 0u;
                    if (__any_sync(0xffffffffu, m != 0u) && !list_warp(m, e0, (unsigned)r)) {
                        fail |= 1u << r;
                        lo[r] = q;
                    }
                }
                ++seq;
#if PC_EMPTYBAR
                // stage st consumed: every warp arrives on the stage's "empty"
                // mbarrier (release: after its reads of the stage) and only the
                // issuing thread waits for all kWarpsCta arrivals before the next
                // bulk copy overwrites the stage -- no CTA-wide barrier per tile
                __syncwarp();
                if (lane == 0)
                    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(ebar0 + 8u * st) : "memory");
                if (q_issue < n_tiles) {
                    if (tid == 0) {
                        mbar_wait_at(ebar0 + 8u * st, ((seq - 1u) / kStages) & 1u);
                        issue_tile(sh, (int)st, qk, t_begin + q_issue * kQTile, tile_words(q_issue));
                    }
                    q_issue += SPLIT;
                }
#else
                __syncthreads(); // stage st consumed by every warp
                if (q_issue < n_tiles) {
                    if (tid == 0) issue_tile(sh, (int)((seq + kStages - 1) % kStages), qk, t_begin + q_issue * kQTile, tile_words(q_issue));
                    q_issue += SPLIT;
                }
#endif
            }
            bool more = false;
#pragma unroll
            for (int r = 0; r < SPLIT; ++r) {
                if (!(fail >> r & 1u)) lo[r] = kDone;
                more = more || lo[r] != kDone;
            }
            if (__syncthreads_or(more) && tid == 0) {
#pragma unroll
                for (int r = 0; r < SPLIT; ++r) dsmem_st(dsmem_addr(&sh.any_ovf, (unsigned)r), 1u);
            }
            cluster_sync_all(); // every listing (local and remote) and flag is visible
            const uint32_t nc = sh.valid_end;
            const bool again = sh.any_ovf != 0u;
            PC_DCHECK(nc <= (uint32_t)kListCap && (sh.live != 0u || nc == 0u)); // an idle CTA is never listed for
            __syncthreads(); // read by everyone before flush resets them
            flush(nc);
            // the last round: nobody touches another CTA's shared memory after the
            // barrier above, so a CTA may leave without waiting for its partner's
            // classification; otherwise wait until every list is classified / reset
            if (!again) break;
            cluster_sync_all();
        }
    } else {
    uint32_t pending = 0; // list size (uniform)
    // this thread's kEPT key words in stage 0 (a shared address kept in a register)
    unsigned qk_s = smem_u32(&sh.qk[0][(kEPT / 4) * tid]);
    asm volatile("" : "+r"(qk_s));
    unsigned bar0 = smem_u32(&sh.full[0]); // stage s's mbarrier: bar0 + 8 s
    asm volatile("" : "+r"(bar0));
    for (uint32_t q = 0; q < n_tiles; ++q) {
        const int s = (int)(q % kStages);
        const uint32_t t0 = t_begin + q * kQTile;
        mbar_wait_at(bar0 + 8u * (unsigned)s, (q / kStages) & 1);
        PC_DCHECK(t0 >= e_begin && t0 < e_end);
        uint32_t d[kEPT];
        {
            const unsigned a = qk_s + (unsigned)s * (kQTile * 4u);
#pragma unroll
            for (int j = 0; j < kEPT / 4; ++j)
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(d[4 * j]), "=r"(d[4 * j + 1]), "=r"(d[4 * j + 2]), "=r"(d[4 * j + 3])
                             : "r"(a + 16u * j));
        }
        // per group of 8 edges: words 0..3 the q(ylo) pairs, 4..7 the
        // 0x7fff - q(yhi) pairs; t has a half with its top bit clear iff that
        // edge may meet a point (key_pair): 1.25 instructions per edge on the
        // common no-candidate path, the exact mask only when some edge hits
        uint32_t t[kEPT / 2];
#pragma unroll
        for (int g = 0; g < kEPT / 8; ++g)
#pragma unroll
            for (int i = 0; i < 4; ++i) t[4 * g + i] = key_pair(d[8 * g + i], d[8 * g + 4 + i], ka, kb);
        uint32_t mn = __vimin3_u16x2(t[0], t[1], t[2]);
#pragma unroll
        for (int i = 3; i < kEPT / 2; i += 2) mn = __vimin3_u16x2(mn, t[i], t[min(i + 1, kEPT / 2 - 1)]);
        const bool mine = (mn & 0x80008000u) != 0x80008000u;
        if (mine) { // rare: append this thread's candidates (edges past e_end are padding or the next chunk's)
            uint32_t m = 0;
#pragma unroll
            for (int g = 0; g < kEPT / 8; ++g)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint32_t nt = ~t[4 * g + i];
                    m |= ((nt >> 15) & 1u) << (8 * g + 2 * i);
                    m |= (nt >> 31) << (8 * g + 2 * i + 1);
                }
            const uint32_t e0 = t0 + (uint32_t)kEPT * (uint32_t)tid;
            if (e0 + kEPT > e_end) m &= e0 >= e_end ? 0u : (1u << (e_end - e0)) - 1u;
            uint32_t pos = atomicAdd(&sh.ncand, (uint32_t)__popc(m));
            PC_DCHECK(pos + (uint32_t)__popc(m) <= (uint32_t)kListCap);
            while (m) {
                sh.list[pos++] = e0 + (__ffs(m) - 1);
                m &= m - 1;
            }
        }
        // stage s consumed and this tile's candidates listed; the count of
        // appending threads is uniform, so is the decision to read the list size
        const int appended = __syncthreads_count(mine);
        if (tid == 0 && q + kStages < n_tiles) issue_tile(sh, s, qk, t0 + kStages * kQTile, tile_words(q + kStages));
        if (appended) {
            pending = sh.ncand;
            __syncthreads(); // everyone has read it before anyone appends again
        }
        if (pending > kListCap - kQTile || (q + 1 == n_tiles && pending)) {
            flush(pending);
            pending = 0;
        }
    }
    }
#endif

    // ---- flags ----
    if (orig) {
        // y-ordered input: each set bit goes to its point's original position
        // (XOR: partial parities of the edge chunks combine; OR: aux); the
        // original indices are requested PC_EPI at a time before their atomics
        const uint32_t setm = (par | auxm) & act;
#pragma unroll
        for (int k0 = 0; k0 < kK; k0 += PC_EPI) {
            uint32_t o[PC_EPI];
#pragma unroll
            for (int k = 0; k < PC_EPI; ++k)
                o[k] = (setm >> (k0 + k) & 1u) ? orig[cta_base + wloc + (k0 + k) * 32 + lane] : 0u;
#pragma unroll
            for (int k = 0; k < PC_EPI; ++k) {
                if ((par & act) >> (k0 + k) & 1u) atomicXor(&inside_bits[o[k] >> 5], 1u << (o[k] & 31));
                if ((auxm & act) >> (k0 + k) & 1u) atomicOr(&aux_bits[o[k] >> 5], 1u << (o[k] & 31));
            }
        }
    } else {
        // one ballot word per k-slice
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
}

int sms(int dev) {
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
}

template <int MODE>
cudaError_t launch_t(const SingleArgs& a, cudaStream_t st, int dev, uint64_t* launches) {
    const size_t smem = sizeof(SingleShared);
    static bool attr[64] = {};
    if (dev < 64 && !attr[dev]) {
        cudaFuncSetAttribute(pip_tile_kernel<MODE, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(pip_tile_kernel<MODE, PC_KSPLIT_G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if constexpr (MODE == kC1)
            cudaFuncSetAttribute(pip_tile_kernel<MODE, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr[dev] = true;
    }
    // C1 on small polygons: the instantiation with more registers per thread (PC_MINB_SMALL)
    const bool small = MODE == kC1 && a.n_edges <= (uint32_t)PC_SMALL_EDGES;
    int per_sm = 0;
    if constexpr (MODE == kC1) {
        if (small) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pip_tile_kernel<MODE, 1, true>, kTPB, smem);
    }
    if (per_sm == 0) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pip_tile_kernel<MODE, 1>, kTPB, smem);
    per_sm = std::max(per_sm, 1);
    const uint64_t pts_per_cta = (uint64_t)kTPB * kK;
    const uint64_t n_ptiles = (a.n + pts_per_cta - 1) / pts_per_cta;
    const uint64_t slots = (uint64_t)sms(dev) * per_sm;
    // Split the edges so the grid covers several waves: long CTAs (many edges)
    // ~8 waves, so the last one is short; few edges ~2 (a chunk re-stages its
    // CTA's points, which then dominates).  Chunks are multiples of 64 edges.
    const uint64_t ne = std::max<uint64_t>(1, a.n_edges);
    const uint64_t waves = ne >= 32768 ? 8 : 2;
    uint64_t chunks = std::max<uint64_t>(1, (waves * slots + n_ptiles - 1) / std::max<uint64_t>(n_ptiles, 1));
    chunks = std::min<uint64_t>(std::min<uint64_t>(chunks, (ne + 63) / 64), 65535);
    const uint32_t per_chunk = (uint32_t)(((ne + chunks - 1) / chunks + 63) / 64 * 64);
    chunks = (ne + per_chunk - 1) / per_chunk;
    // Long chunks: the CTAs of a cluster (PC_KSPLIT_G of them, adjacent y slabs)
    // split the key tiles and list candidates for each other, dividing each
    // CTA's key bytes and tile barriers; short chunks keep one CTA per point tile.
    constexpr int G = PC_KSPLIT_G;
    const bool split = PC_KSPLIT_TILES > 0 && (per_chunk + kQTile - 1) / kQTile >= (uint32_t)PC_KSPLIT_TILES &&
                       n_ptiles >= 2;
    if (split) {
        dim3 grid((unsigned)((n_ptiles + G - 1) / G * G), (unsigned)chunks); // whole clusters
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(kTPB);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = G;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const cudaError_t e = cudaLaunchKernelEx(&cfg, pip_tile_kernel<MODE, G>, reinterpret_cast<const double2*>(a.pts),
                                                 a.n, a.qk, a.filt, reinterpret_cast<const EdgeRec*>(a.rec), a.n_edges,
                                                 per_chunk, a.bbox_keys, a.prefilter, a.tol, a.tol2, a.inside_bits,
                                                 a.aux_bits, a.n_dev, a.orig);
        ++*launches;
        return e != cudaSuccess ? e : cudaGetLastError();
    }
    dim3 grid((unsigned)n_ptiles, (unsigned)chunks);
    if constexpr (MODE == kC1) {
        if (small) {
            pip_tile_kernel<MODE, 1, true><<<grid, kTPB, smem, st>>>(
                reinterpret_cast<const double2*>(a.pts), a.n, a.qk, a.filt, reinterpret_cast<const EdgeRec*>(a.rec),
                a.n_edges, per_chunk, a.bbox_keys, a.prefilter, a.tol, a.tol2, a.inside_bits, a.aux_bits, a.n_dev, a.orig);
            ++*launches;
            return cudaGetLastError();
        }
    }
    pip_tile_kernel<MODE, 1><<<grid, kTPB, smem, st>>>(reinterpret_cast<const double2*>(a.pts), a.n, a.qk, a.filt,
                                                      reinterpret_cast<const EdgeRec*>(a.rec), a.n_edges, per_chunk,
                                                      a.bbox_keys, a.prefilter, a.tol, a.tol2, a.inside_bits,
                                                      a.aux_bits, a.n_dev, a.orig);
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
