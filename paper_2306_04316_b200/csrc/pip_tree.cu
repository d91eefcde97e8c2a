// Segment-tree crossing count for one large polygon in C1 mode (the paper's
// side-of-normal test; reference count_crossings_c1, geometry.hpp:182-203,
// over every ring, contains :281-300) and C2 (count_crossings_c2 :208-229: the
// same straddle, the intercept-side record of pip_device.cuh, DegenerateEdge
// on the fallback points' horizontal edges -> aux plane).
//
// The scan kernel (pip_single.cu) tests every edge whose y-range holds a
// point; for a spiky polygon ~5% of all (point, edge) pairs truly straddle and
// each needs a side test.  Here a point's count comes from O(log^2 n)
// comparisons instead:
//
//   keys      q(y) = trunc(RN(RN(y - o_y) s_y) 2^53) on the polygon-local map of
//             DESIGN.md §3.4 (monotone, 64-bit); V = the sorted distinct vertex
//             keys.  53 bits make a key tie (a point on a vertex's y, or within
//             2^-53 local of it) rare even for 10^6 vertices.
//             A point whose key is not a vertex key ("clean") straddles edge e
//             iff q_lo(e) < q < q_hi(e) -- exactly the reference's
//             f_prev * f_next <= 0 (§3.4, |p.y| >= 2^-400);
//   tree      leaves = the open key intervals (V_j, V_j+1); edge e is stored
//             at the O(log n) canonical nodes of its leaf range.  The edges
//             of a node span the node's whole key range, so for a simple
//             polygon they never cross inside it and are totally ordered in x;
//             each node's list is sorted by x at the range's middle;
//   verify    consecutive edges of a node must stay ordered (within 2^-30
//             local, far inside the fp32 test's band) at both ends of the
//             range, else the node is flagged and queried by a linear scan
//             (non-simple input);
//   query     thread per clean point: walk leaf -> root; per node count the
//             edges right of the point (the reference counts iff
//             (p - a).n <= 0 with n_x >= 0, i.e. the edge lies right of p):
//             a binary search with the certified fp32 side test of §3.4 as the
//             comparator (the reference's binary64 expression when the
//             fp32 value is inside the band), then a scan from the boundary
//             in both directions over the edges the fp32 test cannot decide,
//             stopping at the first decided one.  Decided (|s| > B) edges are
//             farther than ~2^-24 local from the point, far beyond the
//             rounding of the order, so only undecided edges can be out of
//             order with respect to the point and all of them are evaluated.
//   fallback  points with a key tie, |p.y| < 2^-400 or outside the local map
//             are compacted and classified literally (few) or by the scan
//             kernel (many).
#include "pip_kernels.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <utility>
#include <cub/block/block_radix_sort.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include "pip_device.cuh"

namespace pcd {

namespace {

constexpr float kBand = 0x1p-20f;
constexpr uint32_t k2BBits = 0x36000000u; // bits of 2^-19 = 2 kBand

struct Map {
    double x0, y0, sx, sy;
};

__device__ __forceinline__ Map map_of(const unsigned long long* bbox_keys) {
    Map m;
    m.x0 = dkey_inv(bbox_keys[0]);
    m.y0 = dkey_inv(bbox_keys[1]);
    m.sx = reinterpret_cast<const double*>(bbox_keys)[6];
    m.sy = reinterpret_cast<const double*>(bbox_keys)[7];
    return m;
}

// 53-bit key of y on the local map (valid for y in the bbox; clamped otherwise):
// trunc of the local y (in [0, 1)) scaled by 2^53, exact for local y >= 1/2 and
// monotone everywhere, so a point ties a vertex key essentially only when it
// sits on that vertex's y
__device__ __forceinline__ uint64_t key53(double y, const Map& m) {
    double t = __dmul_rn(__dmul_rn(__dsub_rn(y, m.y0), m.sy), 0x1p53);
    t = t > 0.0 ? t : 0.0;
    t = t < 0x1.fffffffffffffp52 ? t : 0x1.fffffffffffffp52;
    return (uint64_t)t;
}

// number of keys < v (lower_bound) / <= v (upper_bound) in V[0, m)
__device__ __forceinline__ uint32_t lower_bound(const uint64_t* __restrict__ V, uint32_t m, uint64_t v) {
    uint32_t lo = 0, hi = m;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(V + mid) < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}
__device__ __forceinline__ uint32_t upper_bound(const uint64_t* __restrict__ V, uint32_t m, uint64_t v) {
    uint32_t lo = 0, hi = m;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(V + mid) <= v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// ring of vertex v (ring_off[r] <= v < ring_off[r+1])
__device__ __forceinline__ uint32_t ring_of(const unsigned long long* __restrict__ ring_off, uint32_t n_rings,
                                            unsigned long long v) {
    uint32_t lo = 0, hi = n_rings;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (ring_off[mid] <= v) lo = mid;
        else hi = mid;
    }
    return lo;
}

__global__ void vkey_kernel(const double* __restrict__ vy, uint64_t nv, const unsigned long long* __restrict__ bbox_keys,
                            uint64_t* __restrict__ vk, uint32_t* __restrict__ vhi, uint32_t* __restrict__ vid) {
    const Map m = map_of(bbox_keys);
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv; v += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = key53(vy[v], m);
        vk[v] = k;
        vhi[v] = (uint32_t)(k >> 21); // the top 32 of the 53 bits: the radix sort's key
        vid[v] = (uint32_t)v;
    }
}

// full keys in the order of the 32-bit sort
__global__ void vgather_kernel(const uint64_t* __restrict__ vk, const uint32_t* __restrict__ vsid, uint64_t nv,
                               uint64_t* __restrict__ vs) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < nv; p += (uint64_t)gridDim.x * blockDim.x)
        vs[p] = vk[vsid[p]];
}

// runs of equal top 32 bits (rare: y values within 2^-32 local of each other)
// sorted by the full key, one thread per run (insertion sort, the ids move along)
__global__ void vfix_kernel(const uint32_t* __restrict__ vhs, uint64_t nv, uint64_t* __restrict__ vs,
                            uint32_t* __restrict__ vsid) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p + 1 < nv;
         p += (uint64_t)gridDim.x * blockDim.x) {
        if (vhs[p + 1] != vhs[p] || (p > 0 && vhs[p - 1] == vhs[p])) continue; // not a run start
        uint64_t e = p + 1;
        while (e < nv && vhs[e] == vhs[p]) ++e;
        for (uint64_t i = p + 1; i < e; ++i) {
            const uint64_t k = vs[i];
            const uint32_t id = vsid[i];
            uint64_t j = i;
            for (; j > p && vs[j - 1] > k; --j) {
                vs[j] = vs[j - 1];
                vsid[j] = vsid[j - 1];
            }
            vs[j] = k;
            vsid[j] = id;
        }
    }
}

// first occurrence of each key in the sorted keys (its inclusive sum is the rank + 1)
__global__ void newkey_kernel(const uint64_t* __restrict__ vs, uint64_t nv, uint32_t* __restrict__ isnew) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < nv; p += (uint64_t)gridDim.x * blockDim.x)
        isnew[p] = p == 0 || vs[p] != vs[p - 1];
}

// rank of every vertex's key among the distinct keys (= its leaf boundary index)
__global__ void vrank_kernel(const uint32_t* __restrict__ csum, const uint32_t* __restrict__ vsid, uint64_t nv,
                             uint32_t* __restrict__ vrank) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < nv; p += (uint64_t)gridDim.x * blockDim.x)
        vrank[vsid[p]] = csum[p] - 1u;
}

// canonical nodes of leaf range [lo, hi) in a tree of L leaves (node ids 1 ..
// 2L-1), level by level from the leaves: at most a left and a right node per
// level.  Warp-collective (all lanes call it; inactive lanes pass lo == hi) so
// lanes that emit the same node share one atomic: f(node, rank, leader_count)
// gets the lane's rank among the lanes emitting that node and, for the
// lowest such lane, their number (0 for the others).
template <class F>
__device__ __forceinline__ void canonical_warp(uint32_t lo, uint32_t hi, uint32_t L, F f) {
    const unsigned lane = threadIdx.x & 31;
    uint32_t l = lo + L, r = hi + L;
    while (__any_sync(0xffffffffu, l < r)) {
        uint32_t nodes[2] = {0u, 0u};
        if (l < r) {
            if (l & 1u) nodes[0] = l++;
            if (r & 1u) nodes[1] = --r;
            l >>= 1;
            r >>= 1;
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const uint32_t nd = nodes[k];
            const uint32_t same = __match_any_sync(0xffffffffu, nd);
            if (nd) {
                const uint32_t rank = __popc(same & ((1u << lane) - 1u));
                f(nd, rank, rank == 0 ? (uint32_t)__popc(same) : 0u, same);
            }
        }
    }
}

// count (fill == false) or fill (fill == true) the node lists
template <bool kFill>
__global__ void edges_kernel(const double* __restrict__ vx, const double* __restrict__ vy,
                             const unsigned long long* __restrict__ ring_off, uint32_t n_rings, uint64_t nv,
                             const unsigned long long* __restrict__ bbox_keys, const uint32_t* __restrict__ vrank,
                             const uint64_t* __restrict__ V, const uint32_t* __restrict__ m_dev, uint32_t L,
                             uint32_t* __restrict__ cnt,
                             const uint2* __restrict__ okh, const double* __restrict__ nmid,
                             unsigned long long* __restrict__ keys, uint32_t* __restrict__ vals,
                             double4* __restrict__ line) {
    const Map mp = map_of(bbox_keys);
    const uint32_t m = *m_dev;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    // whole warps iterate together (canonical_warp is warp-collective)
    for (uint64_t v0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) & ~31ull; v0 < nv; v0 += stride) {
        const uint64_t v = v0 + (threadIdx.x & 31);
        uint32_t lo = 0, hi = 0, e = 0;
        double axl = 0, ayl = 0, slope = 0;
        if (v < nv) {
            const uint32_t r = ring_of(ring_off, n_rings, v);
            if (v + 1 < ring_off[r + 1]) { // a ring's last vertex starts no edge
                e = (uint32_t)(v - r);
                const double ay = vy[v], by = vy[v + 1];
                // leaf range: the ranks of the endpoint keys among the distinct vertex keys
                const uint32_t ra = vrank[v], rb = vrank[v + 1];
                lo = min(ra, rb);
                hi = max(ra, rb);
                if (kFill && hi > lo) { // local endpoints for the x order at each node's middle
                    const double ax = vx[v], bx = vx[v + 1];
                    axl = __dmul_rn(__dsub_rn(ax, mp.x0), mp.sx);
                    ayl = __dmul_rn(__dsub_rn(ay, mp.y0), mp.sy);
                    const double bxl = __dmul_rn(__dsub_rn(bx, mp.x0), mp.sx);
                    const double byl = __dmul_rn(__dsub_rn(by, mp.y0), mp.sy);
                    slope = __ddiv_rn(__dsub_rn(bxl, axl), __dsub_rn(byl, ayl));
                    line[e] = make_double4(axl, ayl, slope, 0.0); // x(y) = axl + (y - ayl) slope, local units
                }
            }
        }
        // flat in key space (hi == lo): never a sure straddle, stored nowhere
        if (!kFill) {
            canonical_warp(lo, hi, L, [&](uint32_t nd, uint32_t, uint32_t lead, uint32_t) {
                if (lead) atomicAdd(&cnt[nd], lead);
            });
        } else {
            canonical_warp(lo, hi, L, [&](uint32_t nd, uint32_t rank, uint32_t lead, uint32_t same) {
                uint32_t base = 0;
                if (lead) base = atomicAdd(&cnt[nd], lead);
                base = __shfl_sync(same, base, __ffs(same) - 1);
                const double ym = nmid[nd];   // the node's middle y, local units
                const uint2 ok = okh[nd];      // {list offset, key high word}
                // x at the middle as 32-bit fixed point: two edges the key misorders are
                // within 2^-32 there, hence within 2^-31 over the whole range (the
                // difference of two non-crossing segments is linear and keeps its sign)
                double xm = __dmul_rn(__dadd_rn(axl, __dmul_rn(__dsub_rn(ym, ayl), slope)), 0x1p32);
                xm = xm > 0.0 ? xm : 0.0;
                xm = xm < 4294967294.0 ? xm : 4294967294.0; // below the mid-node sort's padding key
                const uint32_t key = (uint32_t)xm;
                const uint32_t slot = ok.x + base + rank;
                keys[slot] = (unsigned long long)ok.y << 32 | key; // (node or big-node rank, x)
                vals[slot] = e;
            });
        }
    }
}

// per edge: its packed fp32 record {Nx, Ny, c + B, edge} (the record of
// pip_kernels.cu prep_edges_kernel), 16 B instead of the 64 B EdgeRec
__global__ void erec_kernel(const EdgeRec* __restrict__ rec, uint32_t ne, float4* __restrict__ erec) {
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += gridDim.x * blockDim.x) {
        const double d5 = rec[e].d[5], d6 = rec[e].d[6];
        erec[e] = make_float4(__int_as_float(__double2loint(d5)), __int_as_float(__double2hiint(d5)),
                              __int_as_float(__double2loint(d6)), __uint_as_float(e));
    }
}

// per entry: its packed record (erec of its edge: the query's binary search
// probes one 16 B load per step), and the order check against the next entry
// of the same node at both ends of the node's key range (x from the edge's
// local line; a violation beyond 2^-30 flags the node)
__global__ void verify_pack_kernel(const uint32_t* __restrict__ vals, const unsigned long long* __restrict__ keys,
                                   const uint32_t* __restrict__ tot, const uint32_t* __restrict__ bignode, uint32_t L,
                                   const uint64_t* __restrict__ V, const uint32_t* __restrict__ m_dev,
                                   const double4* __restrict__ line, const float4* __restrict__ erec,
                                   float4* __restrict__ packed, uint8_t* __restrict__ flag) {
    const uint32_t m = *m_dev, tsm = tot[0] + tot[1], total = tsm + tot[2];
    // node of entry j: the key's high word is the node id for small and mid nodes,
    // the huge-node rank after them
    auto node = [&](uint32_t j) { const uint32_t h = (uint32_t)(keys[j] >> 32); return j < tsm ? h : bignode[h]; };
    auto x = [](const double4& l, double y) { return __dadd_rn(l.x, __dmul_rn(__dsub_rn(y, l.y), l.z)); };
    const unsigned lane = threadIdx.x & 31;
    const uint32_t stride = gridDim.x * blockDim.x;
    // whole warps step together: entry i + 1 is the next lane's entry, so its node
    // and its x at this node's ends come by shuffle (lane 31 computes its own)
    for (uint32_t i0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; i0 < total; i0 += stride) {
        const uint32_t i = i0 + lane;
        uint32_t nd = 0xffffffffu, e0 = 0;
        double x0 = 0.0, x1 = 0.0, y0 = 0.0, y1 = 0.0;
        if (i < total) {
            e0 = vals[i];
            packed[i] = erec[e0];
            nd = node(i);
            const int d = 31 - __clz(nd);
            const uint32_t span = L >> d, a = (nd - (1u << d)) * span, b = min(a + span, m - 1);
            y0 = (double)V[a] * 0x1p-53;
            y1 = (double)V[b] * 0x1p-53;
            const double4 l0 = line[e0];
            x0 = x(l0, y0);
            x1 = x(l0, y1);
        }
        uint32_t nd1 = __shfl_down_sync(0xffffffffu, nd, 1);
        double n0 = __shfl_down_sync(0xffffffffu, x0, 1), n1 = __shfl_down_sync(0xffffffffu, x1, 1);
        if (lane == 31 && i + 1 < total) {
            nd1 = node(i + 1);
            if (nd1 == nd) {
                const double4 l1 = line[vals[i + 1]];
                n0 = x(l1, y0);
                n1 = x(l1, y1);
            }
        }
        // consecutive entries of one node must stay ordered within 2^-30 at both ends
        if (i + 1 < total && nd1 == nd && (x0 > __dadd_rn(n0, 0x1p-30) || x1 > __dadd_rn(n1, 0x1p-30))) flag[nd] = 1;
    }
}

// per node, what a query needs in one 8-byte load: {offset, count | linear << 31}
__global__ void meta_kernel(const uint32_t* __restrict__ off, const uint32_t* __restrict__ cnt,
                            const uint8_t* __restrict__ flag, uint32_t n, uint2* __restrict__ meta) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        meta[i] = make_uint2(off[i], cnt[i] | (uint32_t)(flag[i] != 0) << 31);
}

// F: the reference's C1 count decision for a sure straddle, from a packed node
// entry {Nx, Ny, c + B, edge}: 1 counted, 0 not; *certain: decided by the fp32
// test (else the binary64 expression of the edge's record ran)
template <int MODE>
__device__ __forceinline__ int decide(const float4 pk, const EdgeRec* __restrict__ rec, float lx, float ly, double px,
                                      double py, bool* certain) {
    const float s = fmaf(lx, pk.x, fmaf(ly, pk.y, pk.z)); // s' = s + B
    const uint32_t u = __float_as_uint(s);
    if (s == s && u > k2BBits) { // sign bit set (count) or s' > 2B (no count)
        *certain = true;
        return (int)(u >> 31);
    }
    *certain = false;
    int cnt = 0;
    if (MODE == kC1) {
        exact_c1(px, py, rec[__float_as_uint(pk.w)], cnt, true); // keys proved the straddle (geometry.hpp:189-200)
    } else {
        bool err = false; // a sure straddle has dy != 0: no DegenerateEdge
        exact_c2(px, py, rec[__float_as_uint(pk.w)], cnt, err, true); // geometry.hpp:214-226
    }
    return cnt;
}

// edges of one node list that the point counts
template <int MODE>
__device__ __forceinline__ uint32_t node_count(const float4* __restrict__ packed, uint32_t o, uint32_t k, bool linear,
                                               const EdgeRec* __restrict__ rec, float lx, float ly, double px,
                                               double py) {
    bool cert;
    const float4* P = packed + o;
    if (linear) { // non-simple input: every edge
        uint32_t c = 0;
        for (uint32_t i = 0; i < k; ++i) c += decide<MODE>(__ldg(P + i), rec, lx, ly, px, py, &cert);
        return c;
    }
    // lists run left to right: not counted, then counted.  b = first counted
    uint32_t lo = 0, hi = k;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (decide<MODE>(__ldg(P + mid), rec, lx, ly, px, py, &cert)) hi = mid;
        else lo = mid + 1;
    }
    const uint32_t b = lo;
    uint32_t c = k - b; // [b, k) counted, corrected below
    // right of b: undecided edges may be "not counted" after all
    for (uint32_t i = b; i < k; ++i) {
        const int f = decide<MODE>(__ldg(P + i), rec, lx, ly, px, py, &cert);
        if (cert && f) break;
        c -= (uint32_t)(1 - f);
    }
    // left of b: undecided edges may be counted
    for (uint32_t i = b; i-- > 0;) {
        const int f = decide<MODE>(__ldg(P + i), rec, lx, ly, px, py, &cert);
        if (cert && !f) break;
        c += (uint32_t)f;
    }
    return c;
}

template <int MODE>
__global__ void __launch_bounds__(256) query_kernel(const double2* __restrict__ pts, uint64_t n, int prefilter,
                                                    const unsigned long long* __restrict__ bbox_keys,
                                                    const uint64_t* __restrict__ V, const uint32_t* __restrict__ m_dev,
                                                    uint32_t L, const uint2* __restrict__ meta,
                                                    const float4* __restrict__ packed,
                                                    const EdgeRec* __restrict__ rec, uint32_t* __restrict__ inside_bits,
                                                    uint32_t* __restrict__ fb_idx, uint32_t* __restrict__ fb_count,
                                                    const uint32_t* __restrict__ n_dev) {
    if (n_dev) n = min(n, (uint64_t)*n_dev); // y-bucketed input: the in-box prefix
    const Map mp = map_of(bbox_keys);
    const uint32_t m = *m_dev;
    const double minx = dkey_inv(bbox_keys[0]), miny = dkey_inv(bbox_keys[1]);
    const double maxx = dkey_inv(~bbox_keys[2]), maxy = dkey_inv(~bbox_keys[3]);
    const int lane = threadIdx.x & 31;
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t wi = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; wi * 32 < n; wi += warps) {
        const uint64_t i = wi * 32 + lane;
        bool in = false, fb = false;
        if (i < n) {
            const double2 p = pts[i];
            bool act = true;
            if (prefilter) act = p.x >= minx && p.x <= maxx && p.y >= miny && p.y <= maxy; // batch.hpp:39-41
            if (act) {
                const double lxd = __dmul_rn(__dsub_rn(p.x, mp.x0), mp.sx);
                const double lyd = __dmul_rn(__dsub_rn(p.y, mp.y0), mp.sy);
                const bool ok = mp.sx != 0.0 && lxd >= 0.0 && lxd < 1.0 && lyd >= 0.0 && lyd < 1.0 &&
                                fabs(p.y) >= 0x1p-400;
                if (!ok) {
                    fb = true;
                } else {
                    const uint64_t q = (uint64_t)__dmul_rn(lyd, 0x1p53);
                    const uint32_t j = upper_bound(V, m, q); // keys <= q
                    if (j > 0 && __ldg(V + j - 1) == q) {
                        fb = true; // a vertex key: the exact straddle products decide
                    } else if (j > 0 && j < m) {
                        const float lx = __double2float_rn(lxd), ly = __double2float_rn(lyd);
                        uint32_t c = 0;
                        for (uint32_t nd = L + j - 1; nd; nd >>= 1) {
                            const uint2 md = __ldg(meta + nd); // {offset, count | linear << 31}
                            const uint32_t k = md.y & 0x7fffffffu;
                            if (k) c += node_count<MODE>(packed, md.x, k, md.y >> 31, rec, lx, ly, p.x, p.y);
                        }
                        in = c & 1u;
                    }
                }
            }
        }
        const uint32_t w = __ballot_sync(0xffffffffu, in);
        const uint32_t fbm = __ballot_sync(0xffffffffu, fb);
        if (lane == 0) inside_bits[wi] = w;
        if (fbm) {
            uint32_t pos = 0;
            if (lane == 0) pos = atomicAdd(fb_count, (uint32_t)__popc(fbm));
            pos = __shfl_sync(0xffffffffu, pos, 0);
            if (fb) fb_idx[pos + __popc(fbm & ((1u << lane) - 1u))] = (uint32_t)i;
        }
    }
}

__global__ void gather_kernel(const double2* __restrict__ pts, const uint32_t* __restrict__ idx,
                              const uint32_t* __restrict__ count, double2* __restrict__ out) {
    const uint32_t n = *count;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) out[k] = pts[idx[k]];
}

// the fallback points (few) against every edge, the reference's literal C1 step
// (geometry.hpp:189-200: straddle product, then the side of the flipped
// normal); block (chunk of kFbEdges edges, group of 256 points), parity bits
// XOR-combined across chunks
constexpr int kFbEdges = 256;
template <int MODE>
__global__ void __launch_bounds__(256) fallback_kernel(const double2* __restrict__ pts, const uint32_t* __restrict__ idx,
                                                       const uint32_t* __restrict__ count, const EdgeRec* __restrict__ rec,
                                                       uint32_t n_edges, uint32_t* __restrict__ bits,
                                                       uint32_t* __restrict__ ebits) {
    __shared__ double sa[5][kFbEdges];
    const uint32_t e0 = blockIdx.x * kFbEdges, ne = min((uint32_t)kFbEdges, n_edges - e0);
    for (uint32_t i = threadIdx.x; i < ne; i += blockDim.x) {
        const EdgeRec& r = rec[e0 + i];
#pragma unroll
        for (int f = 0; f < 5; ++f) sa[f][i] = r.d[f];
    }
    __syncthreads();
    const uint32_t n = *count, k = blockIdx.y * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double2 p = pts[idx[k]];
    uint32_t par = 0, err = 0;
    for (uint32_t i = 0; i < ne; ++i) {
        const double ax = sa[0][i], ay = sa[1][i], by = sa[2][i];
        if (__dmul_rn(__dsub_rn(ay, p.y), __dsub_rn(by, p.y)) <= 0.0) {
            if (MODE == kC1) { // geometry.hpp:189-200 (record: nx, ny)
                const double side =
                    __dadd_rn(__dmul_rn(__dsub_rn(p.x, ax), sa[3][i]), __dmul_rn(__dsub_rn(p.y, ay), sa[4][i]));
                par ^= side <= 0.0;
            } else { // geometry.hpp:214-226 (record: dx, dy)
                const double dy = sa[4][i];
                if (dy == 0.0) {
                    err = 1; // DegenerateEdge
                } else {
                    const double x = __dadd_rn(ax, __dmul_rn(__ddiv_rn(__dsub_rn(p.y, ay), dy), sa[3][i]));
                    par ^= x > p.x;
                }
            }
        }
    }
    if (par) atomicXor(&bits[k >> 5], 1u << (k & 31));
    if (err) atomicOr(&ebits[k >> 5], 1u << (k & 31));
}

__global__ void scatter_kernel(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ count,
                               const uint32_t* __restrict__ bits, const uint32_t* __restrict__ ebits,
                               uint32_t* __restrict__ inside_bits, uint32_t* __restrict__ aux_bits) {
    const uint32_t n = *count;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const uint32_t i = idx[k], b = 1u << (i & 31);
        if ((bits[k >> 5] >> (k & 31)) & 1u) atomicOr(&inside_bits[i >> 5], b);
        if ((ebits[k >> 5] >> (k & 31)) & 1u) atomicOr(&aux_bits[i >> 5], b);
    }
}

int sms(int dev) {
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
}

uint32_t tree_leaves(uint64_t nv) {
    uint32_t L = 1;
    while (L < nv) L <<= 1;
    return L;
}

// Node lists by size: at most kTinySeg entries (a thread each, a sorting network
// in registers), at most kSmallSeg (a warp each, a bitonic sort over shuffles),
// up to kMidSeg (one CTA each, cub::BlockRadixSort in shared memory, three size
// classes), and bigger ("huge", a few hundred nodes near the root): one
// device-wide radix sort on (huge-node rank, x).  Small, mid and huge lists are
// laid out one after another, each node's list contiguous.
constexpr uint32_t kTinySeg = 16, kSmallSeg = 64, kMidSeg = 4096;
constexpr uint32_t kMidClass[3] = {256, 1024, 4096}; // CTA capacities of the mid classes
constexpr int kClasses = 5;                          // tiny, small, mid x 3

__global__ void split_kernel(const uint32_t* __restrict__ cnt, uint32_t n, uint32_t* __restrict__ cs,
                             uint32_t* __restrict__ cm, uint32_t* __restrict__ ch, uint32_t* __restrict__ fh) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t c = cnt[i];
        const bool mid = c > kSmallSeg && c <= kMidSeg, huge = c > kMidSeg;
        cs[i] = mid || huge ? 0u : c;
        cm[i] = mid ? c : 0u;
        ch[i] = huge ? c : 0u;
        fh[i] = huge;
    }
}

// node offsets, the key high words (node id; huge: rank), the huge-node list and
// the lists of the other non-empty nodes by size class;
// tot = {small, mid, huge entries, huge nodes, nodes of class 0 .. 4}
__global__ void offsets_kernel(const uint32_t* __restrict__ cnt, uint32_t n, const uint32_t* __restrict__ os,
                               const uint32_t* __restrict__ om, const uint32_t* __restrict__ oh,
                               const uint32_t* __restrict__ rh, uint32_t* __restrict__ off,
                               uint32_t* __restrict__ khi,
                               uint32_t* __restrict__ bignode, uint32_t* __restrict__ mlist, uint32_t mcap,
                               uint32_t* __restrict__ tot, const uint64_t* __restrict__ V,
                               const uint32_t* __restrict__ m_dev, uint32_t L, uint2* __restrict__ okh,
                               double* __restrict__ nmid) {
    const uint32_t m = *m_dev;
    // cnt[n - 1] == 0: the last exclusive sums are the totals
    const uint32_t ts = os[n - 1], tm = om[n - 1];
    const uint32_t lane = threadIdx.x & 31;
    // whole warps step together (the class lists are appended warp-aggregated)
    for (uint32_t i0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; i0 < n; i0 += gridDim.x * blockDim.x) {
        const uint32_t i = i0 + lane;
        const uint32_t c = i < n ? cnt[i] : 0u;
        const bool mid = c > kSmallSeg && c <= kMidSeg, huge = c > kMidSeg;
        if (i < n) {
            const uint32_t o = huge ? ts + tm + oh[i] : mid ? ts + om[i] : os[i], h = huge ? rh[i] : i;
            off[i] = o;
            khi[i] = h;
            okh[i] = make_uint2(o, h);
            if (huge) bignode[rh[i]] = i;
            if (c) { // the middle of the node's key range, local units (the fill's x-order point)
                const int d = 31 - __clz(i);
                const uint32_t span = L >> d, a = (i - (1u << d)) * span, b = a + span;
                nmid[i] = ((double)V[a] + (double)V[min(b, m - 1)]) * 0x1p-54;
            }
        }
        const int k = !c || huge ? kClasses
                      : c <= kTinySeg ? 0 : c <= kSmallSeg ? 1 : c <= kMidClass[0] ? 2 : c <= kMidClass[1] ? 3 : 4;
        const uint32_t peers = __match_any_sync(0xffffffffu, k);
        const int leader = __ffs(peers) - 1;
        uint32_t base = 0;
        if (k < kClasses && (int)lane == leader) base = atomicAdd(&tot[4 + k], (uint32_t)__popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (k < kClasses) mlist[k * mcap + base + __popc(peers & ((1u << lane) - 1u))] = i;
        if (i == 0) {
            tot[0] = ts;
            tot[1] = tm;
            tot[2] = oh[n - 1];
            tot[3] = rh[n - 1];
        }
    }
}

// one thread per listed tiny node (<= kTinySeg entries): an odd-even transposition
// network over registers (padding keys 0xffffffff sort last)
__global__ void tiny_sort_kernel(const uint32_t* __restrict__ list, const uint32_t* __restrict__ list_count,
                                 const uint32_t* __restrict__ off, const uint32_t* __restrict__ cnt,
                                 const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ vals,
                                 unsigned long long* __restrict__ keys2, uint32_t* __restrict__ vals2) {
    const uint32_t nl = *list_count;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nl; t += gridDim.x * blockDim.x) {
        const uint32_t nd = list[t], o = off[nd], k = cnt[nd];
        uint32_t kk[kTinySeg], vv[kTinySeg];
#pragma unroll
        for (uint32_t q = 0; q < kTinySeg; ++q) {
            kk[q] = q < k ? (uint32_t)keys[o + q] : 0xffffffffu;
            vv[q] = q < k ? vals[o + q] : 0u;
        }
        // n rounds sort n elements; most tiny lists have <= 4 entries
        auto network = [&](auto nn) {
            constexpr uint32_t N = decltype(nn)::value;
#pragma unroll
            for (uint32_t r = 0; r < N; ++r) {
#pragma unroll
                for (uint32_t q = r & 1; q + 1 < N; q += 2) {
                    const bool sw = kk[q] > kk[q + 1];
                    const uint32_t a = kk[q], b = kk[q + 1], va = vv[q], vb = vv[q + 1];
                    kk[q] = sw ? b : a;
                    kk[q + 1] = sw ? a : b;
                    vv[q] = sw ? vb : va;
                    vv[q + 1] = sw ? va : vb;
                }
            }
        };
        if (k > 4) network(std::integral_constant<uint32_t, kTinySeg>{});
        else if (k > 1) network(std::integral_constant<uint32_t, 4>{});
#pragma unroll
        for (uint32_t q = 0; q < kTinySeg; ++q)
            if (q < k) {
                keys2[o + q] = (unsigned long long)nd << 32 | kk[q];
                vals2[o + q] = vv[q];
            }
    }
}

// one warp per listed small node (<= kSmallSeg entries): a bitonic sort of 64
// (two per lane: positions lane and lane + 32) over shuffles
__global__ void warp_sort_kernel(const uint32_t* __restrict__ list, const uint32_t* __restrict__ list_count,
                                 const uint32_t* __restrict__ off, const uint32_t* __restrict__ cnt,
                                 const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ vals,
                                 unsigned long long* __restrict__ keys2, uint32_t* __restrict__ vals2) {
    const uint32_t nl = *list_count, lane = threadIdx.x & 31;
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nl; w += warps) {
        const uint32_t nd = list[w], o = off[nd], k = cnt[nd];
        uint32_t ka = lane < k ? (uint32_t)keys[o + lane] : 0xffffffffu;
        uint32_t va = lane < k ? vals[o + lane] : 0u;
        uint32_t kb = lane + 32 < k ? (uint32_t)keys[o + lane + 32] : 0xffffffffu;
        uint32_t vb = lane + 32 < k ? vals[o + lane + 32] : 0u;
        // element at position p: p < 32 in (ka, va) of lane p, else (kb, vb) of lane p - 32
#pragma unroll
        for (uint32_t size = 2; size <= 64; size <<= 1) {
#pragma unroll
            for (uint32_t j = size >> 1; j > 0; j >>= 1) {
                if (j == 32) { // partners are the two elements of one lane (size == 64: ascending)
                    const bool sw = ka > kb;
                    const uint32_t k0 = sw ? kb : ka, k1 = sw ? ka : kb, v0 = sw ? vb : va, v1 = sw ? va : vb;
                    ka = k0, kb = k1, va = v0, vb = v1;
                } else {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        uint32_t& kx = h ? kb : ka;
                        uint32_t& vx = h ? vb : va;
                        const uint32_t p = lane + 32 * h;
                        const uint32_t ko = __shfl_xor_sync(0xffffffffu, kx, j), vo = __shfl_xor_sync(0xffffffffu, vx, j);
                        const bool up = (p & size) == 0, lower = (p & j) == 0;
                        // the lower position keeps the min when ascending, the max when descending
                        const bool take = lower == up ? ko < kx : ko > kx;
                        kx = take ? ko : kx;
                        vx = take ? vo : vx;
                    }
                }
            }
        }
        if (lane < k) {
            keys2[o + lane] = (unsigned long long)nd << 32 | ka;
            vals2[o + lane] = va;
        }
        if (lane + 32 < k) {
            keys2[o + lane + 32] = (unsigned long long)nd << 32 | kb;
            vals2[o + lane + 32] = vb;
        }
    }
}

// one CTA per listed mid node: its list (keys' low words = x) sorted in shared
// memory; padding keys 0xffffffff sort last (real keys are clamped below it)
template <int T, int I>
__global__ void __launch_bounds__(T) node_sort_kernel(const uint32_t* __restrict__ list,
                                                      const uint32_t* __restrict__ list_count,
                                                      const uint32_t* __restrict__ off, const uint32_t* __restrict__ cnt,
                                                      const unsigned long long* __restrict__ keys,
                                                      const uint32_t* __restrict__ vals,
                                                      unsigned long long* __restrict__ keys2,
                                                      uint32_t* __restrict__ vals2) {
    using BRS = cub::BlockRadixSort<uint32_t, T, I, uint32_t>;
    __shared__ typename BRS::TempStorage tmp;
    const uint32_t nl = *list_count;
    for (uint32_t b = blockIdx.x; b < nl; b += gridDim.x) {
        const uint32_t nd = list[b], o = off[nd], k = cnt[nd];
        uint32_t kk[I], vv[I];
#pragma unroll
        for (int q = 0; q < I; ++q) { // striped (coalesced); equal x keys have no required order
            const uint32_t j = q * T + threadIdx.x;
            kk[q] = j < k ? (uint32_t)keys[o + j] : 0xffffffffu;
            vv[q] = j < k ? vals[o + j] : 0u;
        }
        BRS(tmp).SortBlockedToStriped(kk, vv);
#pragma unroll
        for (int q = 0; q < I; ++q) {
            const uint32_t j = q * T + threadIdx.x;
            if (j < k) {
                keys2[o + j] = (unsigned long long)nd << 32 | kk[q];
                vals2[o + j] = vv[q];
            }
        }
        __syncthreads(); // tmp is reused by the next node
    }
}

struct Layout {
    uint64_t nv, ne, L, emax;
    size_t o_meta, o_okh, o_nmid, o_cs, o_cm, o_ch, o_fh, o_os, o_om, o_oh, o_rh, o_khi, o_big, o_mlist, o_tot;
    size_t o_vk, o_vs, o_vid, o_vhi, o_vhs, o_vsid, o_vrank, o_V, o_m, o_cnt, o_off, o_keys, o_vals, o_keys2, o_vals2, o_erec, o_packed, o_flag, o_fbidx, o_fbcnt,
        o_fbpts, o_fbbits, o_fbebits, o_line, o_tmp, tmp_bytes, total;
};

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

Layout layout(uint64_t nv, uint64_t ne, uint64_t n_pts) {
    Layout l{};
    l.nv = nv;
    l.ne = ne;
    l.L = tree_leaves(std::max<uint64_t>(nv, 2));
    const int depth = 63 - __builtin_clzll(l.L);
    l.emax = std::max<uint64_t>(ne * 2ull * (depth + 1), nv);
    // CUB temporary storage: the largest of the four primitives
    size_t t1 = 0, t2 = 0, t3 = 0, t4 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t1, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (uint32_t*)nullptr, (int)nv, 0, 32);
    size_t t6 = 0;
    cub::DeviceScan::InclusiveSum(nullptr, t6, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)nv);
    t1 = std::max(t1, t6);
    cub::DeviceSelect::Unique(nullptr, t2, (uint64_t*)nullptr, (uint64_t*)nullptr, (uint32_t*)nullptr, (int)nv);
    cub::DeviceScan::ExclusiveSum(nullptr, t3, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)(2 * l.L + 1));
    cub::DeviceRadixSort::SortPairs(nullptr, t4, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                    (uint32_t*)nullptr, (uint32_t*)nullptr, (int)l.emax, 0, 64);
    l.tmp_bytes = std::max({t1, t2, t3, t4, (size_t)256});
    size_t o = 0;
    auto put = [&](size_t bytes) {
        const size_t at = o;
        o = align256(o + bytes);
        return at;
    };
    l.o_vk = put(nv * 8);
    l.o_vs = put(nv * 8);
    l.o_vid = put(nv * 4);
    l.o_vhi = put(nv * 4);
    l.o_vhs = put(nv * 4);
    l.o_vsid = put(nv * 4);
    l.o_vrank = put(nv * 4);
    l.o_V = put(nv * 8);
    l.o_m = put(16);
    l.o_cnt = put((2 * l.L + 1) * 4);
    l.o_off = put((2 * l.L + 1) * 4);
    for (size_t* o_split : {&l.o_cs, &l.o_cm, &l.o_ch, &l.o_fh, &l.o_os, &l.o_om, &l.o_oh, &l.o_rh,
                            &l.o_khi, &l.o_big})
        *o_split = put((2 * l.L + 1) * 4);
    l.o_mlist = put(kClasses * (2 * l.L + 1) * 4);
    l.o_tot = put(64);
    l.o_keys = put(l.emax * 8);
    l.o_vals = put(l.emax * 4);
    l.o_keys2 = put(l.emax * 8);
    l.o_vals2 = put(l.emax * 4);
    l.o_erec = put(std::max<uint64_t>(ne, 1) * 16);
    l.o_packed = put(l.emax * 16);
    l.o_flag = put(2 * l.L);
    l.o_meta = put(2 * l.L * 8);
    l.o_okh = put((2 * l.L + 1) * 8);
    l.o_nmid = put((2 * l.L + 1) * 8);
    l.o_fbidx = put(n_pts * 4 + 4);
    l.o_fbcnt = put(16);
    l.o_fbpts = put(n_pts * 16 + 16);
    l.o_fbbits = put(((n_pts + 31) / 32) * 4 + 4);
    l.o_fbebits = put(((n_pts + 31) / 32) * 4 + 4);
    l.o_line = put(std::max<uint64_t>(ne, 1) * 32);
    l.o_tmp = put(l.tmp_bytes);
    l.total = o;
    return l;
}

} // namespace

bool tree_eligible(uint64_t n_verts, uint64_t n_pts, bool forced) {
    // 32-bit node lists and point indices; (auto) big enough to pay for the build
    if (n_verts < 4 || n_verts > (1ull << 22) || n_pts == 0 || n_pts >= 0xffffffffull) return false;
    return forced || (n_verts >= 4096 && n_pts >= 16384);
}

size_t tree_scratch_bytes(uint64_t n_verts, uint64_t n_edges, uint64_t n_pts) {
    return layout(n_verts, n_edges, n_pts).total;
}

cudaError_t launch_tree(const TreeArgs& a, void* scratch, cudaStream_t st, int dev, uint64_t* launches) {
    const cudaError_t e = launch_tree_phase(a, scratch, st, dev, launches, kTreeBuild);
    return e != cudaSuccess ? e : launch_tree_phase(a, scratch, st, dev, launches, kTreeQuery);
}

// kTreeBuild reads only the polygon (and the records of prep); kTreeQuery the points
cudaError_t launch_tree_phase(const TreeArgs& a, void* scratch, cudaStream_t st, int dev, uint64_t* launches,
                              int phase) {
    const Layout l = layout(a.n_verts, a.n_edges, a.n_layout ? a.n_layout : a.n);
    char* s = static_cast<char*>(scratch);
    uint64_t* vk = reinterpret_cast<uint64_t*>(s + l.o_vk);
    uint64_t* vs = reinterpret_cast<uint64_t*>(s + l.o_vs);
    uint32_t* vid = reinterpret_cast<uint32_t*>(s + l.o_vid);
    uint32_t* vhi = reinterpret_cast<uint32_t*>(s + l.o_vhi);
    uint32_t* vhs = reinterpret_cast<uint32_t*>(s + l.o_vhs);
    uint32_t* vsid = reinterpret_cast<uint32_t*>(s + l.o_vsid);
    uint32_t* vrank = reinterpret_cast<uint32_t*>(s + l.o_vrank);
    uint64_t* V = reinterpret_cast<uint64_t*>(s + l.o_V);
    uint32_t* m_dev = reinterpret_cast<uint32_t*>(s + l.o_m);
    uint32_t* cnt = reinterpret_cast<uint32_t*>(s + l.o_cnt);
    uint32_t* off = reinterpret_cast<uint32_t*>(s + l.o_off);
    auto u32 = [&](size_t o) { return reinterpret_cast<uint32_t*>(s + o); };
    uint32_t *cs = u32(l.o_cs), *cm = u32(l.o_cm), *ch = u32(l.o_ch), *fh = u32(l.o_fh), *os = u32(l.o_os),
             *om = u32(l.o_om), *oh = u32(l.o_oh), *rh = u32(l.o_rh), *khi = u32(l.o_khi),
             *bignode = u32(l.o_big), *mlist = u32(l.o_mlist), *tot = u32(l.o_tot);
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(s + l.o_keys);
    uint32_t* vals = reinterpret_cast<uint32_t*>(s + l.o_vals);
    unsigned long long* keys2 = reinterpret_cast<unsigned long long*>(s + l.o_keys2);
    uint32_t* vals2 = reinterpret_cast<uint32_t*>(s + l.o_vals2);
    float4* erec = reinterpret_cast<float4*>(s + l.o_erec);
    float4* packed = reinterpret_cast<float4*>(s + l.o_packed);
    uint8_t* flag = reinterpret_cast<uint8_t*>(s + l.o_flag);
    uint2* meta = reinterpret_cast<uint2*>(s + l.o_meta);
    uint2* okh = reinterpret_cast<uint2*>(s + l.o_okh);
    double* nmid = reinterpret_cast<double*>(s + l.o_nmid);
    uint32_t* fb_idx = reinterpret_cast<uint32_t*>(s + l.o_fbidx);
    uint32_t* fb_cnt = reinterpret_cast<uint32_t*>(s + l.o_fbcnt);
    double* fb_pts = reinterpret_cast<double*>(s + l.o_fbpts);
    uint32_t* fb_bits = reinterpret_cast<uint32_t*>(s + l.o_fbbits);
    uint32_t* fb_ebits = reinterpret_cast<uint32_t*>(s + l.o_fbebits);
    double4* line = reinterpret_cast<double4*>(s + l.o_line);
    void* tmp = s + l.o_tmp;
    size_t tmp_bytes = l.tmp_bytes;
    const uint32_t L = (uint32_t)l.L;
    const int grid = sms(dev) * 8;
    const EdgeRec* rec = static_cast<const EdgeRec*>(a.rec);
    const unsigned long long* ro = reinterpret_cast<const unsigned long long*>(a.ring_off);
    cudaError_t e;
#define PC_TRY(x)                                                                                                      \
    if ((e = (x)) != cudaSuccess) return e
    if (phase == kTreeBuild) {
        // ---- build ----
        // vertex keys sorted on their top 32 bits (4 radix passes instead of 7), then
        // runs of equal top bits fixed up on the full 53
        vkey_kernel<<<grid, 256, 0, st>>>(a.vy, a.n_verts, a.bbox_keys, vk, vhi, vid);
        PC_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, vhi, vhs, vid, vsid, (int)a.n_verts, 0, 32, st));
        vgather_kernel<<<grid, 256, 0, st>>>(vk, vsid, a.n_verts, vs);
        vfix_kernel<<<grid, 256, 0, st>>>(vhs, a.n_verts, vs, vsid);
        tmp_bytes = l.tmp_bytes;
        PC_TRY(cub::DeviceSelect::Unique(tmp, tmp_bytes, vs, V, m_dev, (int)a.n_verts, st));
        // vertex ranks among the distinct keys (vid is free again: first-occurrence flags, then their sums)
        newkey_kernel<<<grid, 256, 0, st>>>(vs, a.n_verts, vid);
        tmp_bytes = l.tmp_bytes;
        PC_TRY(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, vid, vrank, (int)a.n_verts, st));
        vrank_kernel<<<grid, 256, 0, st>>>(vrank, vsid, a.n_verts, vid);
        uint32_t* const vr = vid;
        PC_TRY(cudaMemsetAsync(cnt, 0, (2 * l.L + 1) * 4, st));
        PC_TRY(cudaMemsetAsync(flag, 0, 2 * l.L, st));
        edges_kernel<false><<<grid, 256, 0, st>>>(a.vx, a.vy, ro, a.n_rings, a.n_verts, a.bbox_keys, vr, V, m_dev, L, cnt,
                                                  nullptr, nullptr, nullptr, nullptr, nullptr);
        const int n_nodes = (int)(2 * l.L + 1);
        split_kernel<<<grid, 256, 0, st>>>(cnt, (uint32_t)n_nodes, cs, cm, ch, fh);
        for (auto [in, out] : {std::pair{cs, os}, std::pair{cm, om}, std::pair{ch, oh}, std::pair{fh, rh}}) {
            tmp_bytes = l.tmp_bytes;
            PC_TRY(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, in, out, n_nodes, st));
        }
        PC_TRY(cudaMemsetAsync(tot, 0, 64, st));
        offsets_kernel<<<grid, 256, 0, st>>>(cnt, (uint32_t)n_nodes, os, om, oh, rh, off, khi, bignode, mlist,
                                             (uint32_t)n_nodes, tot, V, m_dev, L, okh, nmid);
        PC_TRY(cudaMemsetAsync(cnt, 0, (2 * l.L + 1) * 4, st));
        edges_kernel<true><<<grid, 256, 0, st>>>(a.vx, a.vy, ro, a.n_rings, a.n_verts, a.bbox_keys, vr, V, m_dev, L, cnt,
                                                 okh, nmid, keys, vals, line);
        // the split sizes come to the host (item counts of the sorts, grid sizes)
        uint32_t h_tot[4 + kClasses] = {};
        PC_TRY(cudaMemcpyAsync(h_tot, tot, sizeof(h_tot), cudaMemcpyDeviceToHost, st));
        PC_TRY(cudaStreamSynchronize(st));
        auto cls_grid = [&](uint32_t k, uint32_t per_block) {
            return std::max(1u, std::min((k + per_block - 1) / per_block, (uint32_t)grid * 4));
        };
        const uint32_t* lists = mlist;
        if (h_tot[4]) tiny_sort_kernel<<<cls_grid(h_tot[4], 256), 256, 0, st>>>(lists, tot + 4, off, cnt, keys, vals, keys2,
                                                                               vals2);
        if (h_tot[5]) warp_sort_kernel<<<cls_grid(h_tot[5], 8), 256, 0, st>>>(lists + n_nodes, tot + 5, off, cnt, keys,
                                                                             vals, keys2, vals2);
        if (h_tot[6])
            node_sort_kernel<64, 4><<<cls_grid(h_tot[6], 1), 64, 0, st>>>(lists + 2 * n_nodes, tot + 6, off, cnt, keys,
                                                                         vals, keys2, vals2);
        if (h_tot[7])
            node_sort_kernel<128, 8><<<cls_grid(h_tot[7], 1), 128, 0, st>>>(lists + 3 * n_nodes, tot + 7, off, cnt,
                                                                           keys, vals, keys2, vals2);
        if (h_tot[8])
            node_sort_kernel<256, 16><<<cls_grid(h_tot[8], 1), 256, 0, st>>>(lists + 4 * n_nodes, tot + 8, off, cnt,
                                                                            keys, vals, keys2, vals2);
        if (h_tot[2]) {
            const uint32_t o = h_tot[0] + h_tot[1];
            const int bits = 32 + (32 - __builtin_clz(std::max(h_tot[3], 1u)));
            tmp_bytes = l.tmp_bytes;
            PC_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys + o, keys2 + o, vals + o, vals2 + o,
                                                   (int)h_tot[2], 0, bits, st));
        }
        erec_kernel<<<grid, 256, 0, st>>>(rec, (uint32_t)a.n_edges, erec);
        verify_pack_kernel<<<grid, 256, 0, st>>>(vals2, keys2, tot, bignode, L, V, m_dev, line, erec, packed, flag);
        meta_kernel<<<grid, 256, 0, st>>>(off, cnt, flag, (uint32_t)(2 * l.L), meta);
        *launches += 19;
        return cudaGetLastError();
    }
    // ---- query ----
    PC_TRY(cudaMemsetAsync(fb_cnt, 0, 4, st));
    const unsigned qgrid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((a.n + 255) / 256, (uint64_t)grid * 4));
    if (a.mode == kC1)
        query_kernel<kC1><<<qgrid, 256, 0, st>>>(reinterpret_cast<const double2*>(a.pts), a.n, a.prefilter, a.bbox_keys,
                                                 V, m_dev, L, meta, packed, rec, a.inside_bits, fb_idx, fb_cnt,
                                                 a.n_dev);
    else
        query_kernel<kC2><<<qgrid, 256, 0, st>>>(reinterpret_cast<const double2*>(a.pts), a.n, a.prefilter, a.bbox_keys,
                                                 V, m_dev, L, meta, packed, rec, a.inside_bits, fb_idx, fb_cnt,
                                                 a.n_dev);
    *launches += 4;
    // ---- fallback points through the scan kernel, its grid sized for their number ----
    uint32_t n_fb = 0;
    PC_TRY(cudaMemcpyAsync(&n_fb, fb_cnt, 4, cudaMemcpyDeviceToHost, st));
    PC_TRY(cudaStreamSynchronize(st));
    if (n_fb) {
        PC_TRY(cudaMemsetAsync(fb_bits, 0, ((n_fb + 31) / 32) * 4, st));
        PC_TRY(cudaMemsetAsync(fb_ebits, 0, ((n_fb + 31) / 32) * 4, st));
        if ((double)n_fb * (double)a.n_edges <= 2e10) { // few points: every edge, literally
            const dim3 fgrid((unsigned)((a.n_edges + kFbEdges - 1) / kFbEdges), (unsigned)((n_fb + 255) / 256));
            if (a.mode == kC1)
                fallback_kernel<kC1><<<fgrid, 256, 0, st>>>(reinterpret_cast<const double2*>(a.pts), fb_idx, fb_cnt,
                                                            rec, (uint32_t)a.n_edges, fb_bits, fb_ebits);
            else
                fallback_kernel<kC2><<<fgrid, 256, 0, st>>>(reinterpret_cast<const double2*>(a.pts), fb_idx, fb_cnt,
                                                            rec, (uint32_t)a.n_edges, fb_bits, fb_ebits);
            ++*launches;
        } else { // many: the scan kernel (its filters), grid sized for their number
            gather_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const double2*>(a.pts), fb_idx, fb_cnt,
                                                reinterpret_cast<double2*>(fb_pts));
            SingleArgs sa = a.single;
            sa.pts = fb_pts;
            sa.n = n_fb;
            sa.n_dev = nullptr;
            sa.prefilter = 0; // gathered points were active
            sa.inside_bits = fb_bits;
            sa.aux_bits = fb_ebits;
            PC_TRY(launch_single(sa, st, dev, launches));
            ++*launches;
        }
        scatter_kernel<<<grid, 256, 0, st>>>(fb_idx, fb_cnt, fb_bits, fb_ebits, a.inside_bits, a.aux_bits);
        ++*launches;
    }
#undef PC_TRY
    return cudaGetLastError();
}

} // namespace pcd
