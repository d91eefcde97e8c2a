// C-ABI of libpolycast_cuda.so (include/polycast_cuda.h).
//
// Replaces the reference's batch engine (proj/include/polycast/batch.hpp:184-230):
// the std::thread fork/join over contiguous point chunks becomes contiguous
// point shards over the context's GPUs (one stream each), the per-point loop
// becomes the sm_100a kernels of pip_kernels.cu, and per-point DegenerateEdge
// / Boundary outcomes come back as bit planes + verdict bytes + BatchStats.
#include "../../include/polycast_cuda.h"
#include "pip_kernels.h"
#include "host_stage.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

namespace {

// bumped whenever a scratch buffer is (re)allocated: captured graphs that
// embed the old addresses are then stale
std::atomic<uint64_t> g_alloc_gen{0};

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        ++g_alloc_gen;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        const size_t want = std::max<size_t>(bytes + bytes / 8, 256);
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

struct DevState {
    int dev = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t copy = nullptr; // points upload, overlapping polygon-only work on `stream` (made on first use)
    std::vector<cudaEvent_t> up_evs; // one per uploaded chunk
    DevBuf pts, vx, vy, ring_off, pt_off, poly_ring_off, filt, qk, rec, bbox, bits, verdicts, stats, counts, degen;
    DevBuf bucket_scratch, sorted_pts, sorted_idx;            // y order (pip_sort.cu)
    DevBuf csr_meta;                                          // per-polygon records (pip_csr.cu)
    DevBuf cmp_blk, cmp_pts, cmp_idx, cmp_v, cmp_out;         // prefilter / scatter (pip_compact.cu)
    DevBuf csv_text, csv_state, csv_res, csv_out;             // CSV reader (pip_csv.cu)
    DevBuf emit_recs, emit_scratch, emit_out;                 // results-CSV writer (pip_emit.cu)
    DevBuf tree;                                              // segment tree + fallback (pip_tree.cu)
    // small calls (pip_small.cu): the last polygon, by content (host copy for the
    // comparison), with its outer bbox; pinned staging of points in / results out
    std::vector<double> cvx, cvy;
    std::vector<uint64_t> cro;
    bool cvalid = false;
    DevBuf c_vx, c_vy, c_ro, c_box, small_pts, small_out;
    unsigned char* h_small = nullptr;
    size_t h_small_cap = 0;
    unsigned long long* h_stats = nullptr; // pinned 4 x u64
    uint64_t launches = 0;                 // kernels this device launched in the current call
    // device-pointer calls replayed as CUDA graphs (PC_OPT_GRAPH): key = every
    // argument and option of the call; exec == nullptr: seen once (the next
    // identical call is captured, after this one settled the scratch sizes)
    struct Graph {
        std::vector<uint64_t> key;
        cudaGraphExec_t exec = nullptr;
        uint64_t gen = 0, launches = 0;
        bool failed = false;
    };
    std::vector<Graph> graphs;
    pch::Stager* stager = nullptr;         // pageable host copies (host_stage.h), made on first use
    // profiling: one event pair per main-kernel launch since the last take
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> evs;
    std::vector<uint8_t> ev_cont; // pair i continues pair i - 1 (one logical measurement)
    size_t ev_used = 0;
};

} // namespace

// points per upload chunk of a big single-polygon shard (128 MB)
constexpr uint64_t kUploadChunk = 1ull << 23;

struct pc_ctx {
    std::vector<DevState> devs;
    std::string err;
    std::mutex mu;
    bool profiling = false;
    int64_t bucket_mode = -1; // PC_OPT_BUCKET_POINTS: -1 auto, 0 off, 1 on
    int64_t tree_mode = 0;    // PC_OPT_TREE: 0 off (default), 1 on (opt-in extension, not the reference scan)
    bool exact = false;       // PC_OPT_EXACT: the literal binary64 loop only (pip_exact.cu)
    bool graphs = true;       // PC_OPT_GRAPH: replay repeated device-pointer calls as CUDA graphs
};

namespace {

// An error carries its message, so per-device host threads never write the
// context's shared error string concurrently (guarded() publishes it).
struct Fail {
    int code;
    std::string msg;
};

void check(pc_ctx*, cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    std::string m = std::string(what) + ": " + cudaGetErrorString(e);
    cudaGetLastError(); // clear sticky-free errors
    throw Fail{e == cudaErrorMemoryAllocation ? PC_ENOMEM : PC_ECUDA, std::move(m)};
}

void invalid(pc_ctx*, const char* msg) { throw Fail{PC_EINVAL, msg}; }

// Runs fn(i) for every device index i, each on its own host thread when there
// are several (enqueue, copies and the final wait of one device never wait on
// another's); rethrows the first failure.
template <class Fn>
void per_device(size_t n, Fn&& fn) {
    if (n <= 1) {
        if (n == 1) fn(size_t(0));
        return;
    }
    std::vector<Fail> errs(n, Fail{PC_OK, {}});
    std::vector<std::thread> th;
    th.reserve(n);
    for (size_t i = 0; i < n; ++i)
        th.emplace_back([&, i] {
            try {
                fn(i);
            } catch (const Fail& f) {
                errs[i] = f;
            } catch (const std::exception& e) {
                errs[i] = Fail{PC_ENOMEM, e.what()};
            }
        });
    for (auto& t : th) t.join();
    for (auto& f : errs)
        if (f.code != PC_OK) throw f;
}

template <class Fn>
int guarded(pc_ctx* c, Fn&& fn) {
    if (!c) return PC_EINVAL;
    std::lock_guard<std::mutex> lk(c->mu);
    for (auto& d : c->devs) d.launches = 0;
    try {
        fn();
        c->err.clear();
        return PC_OK;
    } catch (const Fail& f) {
        c->err = f.msg;
        return f.code;
    } catch (const std::exception& e) {
        c->err = e.what();
        return PC_ENOMEM;
    }
}

void validate_rings(pc_ctx* c, const uint64_t* ring_off, uint64_t n_rings) {
    if (n_rings < 1) invalid(c, "polygon needs at least one (outer) ring");
    if (ring_off[0] != 0) invalid(c, "ring_off[0] must be 0");
    for (uint64_t r = 0; r < n_rings; ++r)
        if (ring_off[r + 1] <= ring_off[r]) invalid(c, "every ring needs at least one vertex (ring_off must increase)");
}

// cont: this pair continues the previous one (pc_profile_take reports their sum)
void mark_begin(pc_ctx* c, DevState& d, cudaStream_t st, bool cont = false) {
    if (!c->profiling) return;
    if (d.ev_used == d.evs.size()) {
        cudaEvent_t a, b;
        check(c, cudaEventCreate(&a), "event");
        check(c, cudaEventCreate(&b), "event");
        d.evs.emplace_back(a, b);
        d.ev_cont.push_back(0);
    }
    d.ev_cont[d.ev_used] = cont;
    check(c, cudaEventRecord(d.evs[d.ev_used].first, st), "event record");
}

void mark_end(pc_ctx* c, DevState& d, cudaStream_t st) {
    if (!c->profiling) return;
    check(c, cudaEventRecord(d.evs[d.ev_used].second, st), "event record");
    ++d.ev_used;
}

// Enqueue the whole single-polygon pipeline for one device; inputs already on
// the device.  prep (edge records, bbox, zeroed planes) -> classify -> finalize.
void enqueue_single(pc_ctx* c, DevState& d, cudaStream_t st, const double* d_pts, uint64_t n, const double* d_vx,
                    const double* d_vy, const uint64_t* d_ring_off, uint32_t n_rings, uint64_t n_verts, int mode,
                    double tol, int prefilter, uint8_t* d_verdicts, uint32_t* d_inside, uint32_t* d_aux,
                    unsigned long long* d_stats, const cudaEvent_t* ready = nullptr, uint64_t chunk = 0) {
    // ready (nullable): the points are still being uploaded on another stream,
    // in chunks of `chunk` points (0: one piece), ready[k] recorded after chunk
    // k; everything that reads only the polygon (prep, the segment-tree build)
    // is enqueued before the first wait, so it overlaps the upload, and chunk k
    // is classified while chunk k + 1 uploads
    const uint64_t n_edges = n_verts - n_rings;
    if (n_edges > 0xffffffffull) invalid(c, "too many edges for one polygon (>= 2^32)");
    const uint64_t nwords = (n + 31) / 32;
    if (c->exact) { // PC_OPT_EXACT: the literal loop over every (point, edge), then the same finalize
        if (ready) {
            const uint64_t cn = chunk && chunk < n ? chunk : n;
            for (uint64_t lo = 0, k = 0; lo < n; lo += cn, ++k)
                check(c, cudaStreamWaitEvent(st, ready[k], 0), "wait for the points upload");
        }
        check(c, d.bbox.ensure(8 * sizeof(double)), "alloc bbox");
        check(c, cudaMemsetAsync(d_stats, 0, 4 * sizeof(unsigned long long), st), "clear stats");
        mark_begin(c, d, st);
        check(c, pcd::launch_exact_single(d_pts, n, d_vx, d_vy, d_ring_off, n_rings, prefilter, d.bbox.as<double>(),
                                          mode, tol, d_inside, d_aux, st, &d.launches),
              "exact kernel");
        mark_end(c, d, st);
        check(c, pcd::launch_finalize(n, d_inside, d_aux, d_verdicts, mode, d_stats, st, d.dev, &d.launches),
              "finalize kernel");
        return;
    }
    check(c, d.filt.ensure(pcd::filt_words(n_edges) * sizeof(uint2)), "alloc edge filter words");
    check(c, d.qk.ensure(pcd::qk_words(n_edges) * sizeof(uint32_t)), "alloc edge keys");
    check(c, d.rec.ensure(std::max<uint64_t>(n_edges, 1) * pcd::edge_rec_bytes()), "alloc edge records");
    check(c, d.bbox.ensure(8 * sizeof(unsigned long long)), "alloc bbox"); // 4 keys + key map
    pcd::PrepArgs pa{};
    pa.mode = mode;
    pa.vx = d_vx;
    pa.vy = d_vy;
    pa.ring_off = d_ring_off;
    pa.n_rings = n_rings;
    pa.n_verts = n_verts;
    pa.filt = d.filt.as<uint2>();
    pa.qk = d.qk.as<uint32_t>();
    pa.rec = d.rec.p;
    pa.bbox_keys = d.bbox.as<unsigned long long>();
    pa.stats = d_stats;
    pa.tol = tol;
    pa.zero_words = d_inside;
    pa.zero_words2 = d_aux;
    pa.n_zero_words = nwords;
    check(c, pcd::launch_prep(pa, st, d.dev, &d.launches), "prep kernel");
    const bool tree = (mode == 0 || mode == 1) /* C1, C2 */ && c->tree_mode == 1 && pcd::tree_eligible(n_verts, n, true);
    // y-ordering pays from ~24 edges on (measured break-even, tools/time_bucket_threshold.py:
    // 1e6 points: 24 edges 59 vs 59 us, 63 edges 63 vs 106 us; 1e5 points: 16-20 edges)
    const bool bucket = !tree && n < 0xffffffffull &&
                        (c->bucket_mode == 1 || (c->bucket_mode < 0 && n_edges >= 24 && n >= 4096));
    pcd::SingleArgs sa{};
    sa.mode = mode;
    sa.pts = d_pts;
    sa.n = n;
    sa.qk = d.qk.as<uint32_t>();
    sa.filt = d.filt.as<uint2>();
    sa.rec = d.rec.p;
    sa.n_edges = (uint32_t)n_edges;
    sa.bbox_keys = d.bbox.as<unsigned long long>();
    sa.prefilter = prefilter;
    sa.tol = tol;
    sa.tol2 = tol * tol;
    sa.inside_bits = d_inside;
    sa.aux_bits = d_aux;
    sa.n_dev = nullptr;
    sa.orig = nullptr;
    pcd::TreeArgs ta{};
    if (tree) { // segment-tree build (polygon only)
        ta.mode = mode;
        ta.n = n;
        ta.n_layout = chunk && chunk < n ? chunk : n; // per-chunk fallback buffers
        ta.vx = d_vx;
        ta.vy = d_vy;
        ta.ring_off = d_ring_off;
        ta.n_rings = n_rings;
        ta.n_verts = n_verts;
        ta.n_edges = n_edges;
        ta.rec = d.rec.p;
        ta.bbox_keys = d.bbox.as<unsigned long long>();
        check(c, d.tree.ensure(pcd::tree_scratch_bytes(n_verts, n_edges, ta.n_layout)), "alloc segment tree");
        mark_begin(c, d, st);
        check(c, pcd::launch_tree_phase(ta, d.tree.p, st, d.dev, &d.launches, pcd::kTreeBuild), "segment-tree build");
        mark_end(c, d, st);
    }
    // the points in chunks of `chunk` (one chunk when the caller uploads them in one
    // piece): chunk k waits for its upload event, then bucket -> classify ->
    // unbucket on its own range of the bit planes (chunks are 32-point aligned)
    const uint64_t cn = chunk && chunk < n ? chunk : n;
    for (uint64_t lo = 0, k = 0; lo < n; lo += cn, ++k) {
        const uint64_t m = std::min(cn, n - lo), mw = (m + 31) / 32;
        if (ready) check(c, cudaStreamWaitEvent(st, ready[k], 0), "wait for the points upload");
        pcd::SingleArgs sc = sa;
        sc.pts = d_pts + 2 * lo;
        sc.n = m;
        sc.inside_bits = d_inside + lo / 32;
        sc.aux_bits = d_aux + lo / 32;
        if (bucket) {
            // y order by a radix sort of (key, point, index); the scan kernel reads
            // the y-ordered points and sets the bits of their original positions
            check(c, d.bucket_scratch.ensure(pcd::bucket_scratch_bytes(m) + 16), "alloc bucket scratch");
            check(c, d.sorted_idx.ensure(m * 4), "alloc bucket index");
            check(c, d.sorted_pts.ensure(m * 16), "alloc y-ordered points");
            uint32_t* n_in = reinterpret_cast<uint32_t*>(d.bucket_scratch.as<char>() + pcd::bucket_scratch_bytes(m));
            pcd::BucketArgs ba{sc.pts, m, d.bbox.as<unsigned long long>(), prefilter, d.bucket_scratch.p,
                               d.sorted_pts.as<double>(), d.sorted_idx.as<uint32_t>(), n_in};
            check(c, pcd::launch_bucket(ba, st, d.dev, &d.launches), "bucket kernels");
            sc.pts = d.sorted_pts.as<double>();
            sc.prefilter = 0; // rejected points sort last and are left out (n_dev)
            sc.orig = d.sorted_idx.as<uint32_t>();
            sc.n_dev = n_in;
        }
        if (tree) { // segment-tree counts; key-tie / off-map points through the scan kernel
            // (y-bucketed points: a warp's queries walk nearby leaves, sharing nodes)
            ta.pts = sc.pts;
            ta.n = m;
            ta.n_dev = sc.n_dev;
            ta.prefilter = sc.prefilter;
            ta.inside_bits = sc.inside_bits;
            ta.aux_bits = sc.aux_bits;
            ta.single = sc;
            ta.single.n_dev = nullptr;
            mark_begin(c, d, st, true); // one measurement with the build
            check(c, pcd::launch_tree_phase(ta, d.tree.p, st, d.dev, &d.launches, pcd::kTreeQuery),
                  "segment-tree query");
            mark_end(c, d, st);
        } else {
            mark_begin(c, d, st, k > 0);
            check(c, pcd::launch_single(sc, st, d.dev, &d.launches), "classify kernel");
            mark_end(c, d, st);
        }
    }
    check(c, pcd::launch_finalize(n, d_inside, d_aux, d_verdicts, mode, d_stats, st, d.dev, &d.launches),
          "finalize kernel");
}

void enqueue_csr(pc_ctx* c, DevState& d, cudaStream_t st, const double* d_pts, uint64_t n_points,
                 const uint64_t* d_pt_off, uint64_t n_polys, const double* d_vx, const double* d_vy,
                 const uint64_t* d_ring_off, const uint64_t* d_poly_ring_off, uint64_t pt_base, uint64_t ring_base,
                 uint64_t vert_base, int mode, double tol, uint8_t* d_verdicts, uint32_t* d_inside, uint32_t* d_aux,
                 unsigned long long* d_stats) {
    const uint64_t nwords = (n_points + 31) / 32;
    check(c, cudaMemsetAsync(d_inside, 0, nwords * 4, st), "clear inside plane");
    check(c, cudaMemsetAsync(d_aux, 0, nwords * 4, st), "clear aux plane");
    check(c, cudaMemsetAsync(d_stats, 0, 4 * sizeof(unsigned long long), st), "clear stats");
    pcd::CsrArgs a{};
    a.mode = mode;
    a.pts = d_pts;
    a.pt_off = d_pt_off;
    a.n_polys = n_polys;
    a.vx = d_vx;
    a.vy = d_vy;
    a.ring_off = d_ring_off;
    a.poly_ring_off = d_poly_ring_off;
    a.pt_base = pt_base;
    a.ring_base = ring_base;
    a.vert_base = vert_base;
    a.tol = tol;
    a.tol2 = tol * tol;
    a.inside_bits = d_inside;
    a.aux_bits = d_aux;
    mark_begin(c, d, st);
    if (c->exact) {
        check(c, pcd::launch_exact_csr(a, n_points, st, &d.launches), "exact csr kernel");
    } else {
        check(c, d.csr_meta.ensure(std::max<size_t>(pcd::csr_meta_bytes(n_polys), 16)), "alloc polygon metadata");
        a.meta = d.csr_meta.p;
        check(c, pcd::launch_csr(a, st, d.dev, &d.launches), "csr kernel");
    }
    mark_end(c, d, st);
    check(c, pcd::launch_finalize(n_points, d_inside, d_aux, d_verdicts, mode, d_stats, st, d.dev, &d.launches),
          "finalize kernel");
}

pch::Stager& stager(DevState& d) {
    if (!d.stager) d.stager = new pch::Stager();
    return *d.stager;
}

// upload (pageable sources of >= 4 MiB go through the pinned staging chunks)
void h2d(pc_ctx* c, DevState& d, DevBuf& b, const void* src, size_t bytes, cudaStream_t st, const char* what) {
    check(c, b.ensure(std::max<size_t>(bytes, 16)), what);
    if (bytes) check(c, stager(d).h2d(b.p, src, bytes, st), what);
}

// download after the work queued on st; complete on return
void d2h(pc_ctx* c, DevState& d, void* dst, const void* src, size_t bytes, cudaStream_t st, const char* what) {
    if (bytes) check(c, stager(d).d2h(dst, src, bytes, st), what);
}

// OR `nbits` bits from src (bit 0 = point `bit_off` of the destination) into dst.
void merge_bits(uint32_t* dst, const uint32_t* src, uint64_t bit_off, uint64_t nbits) {
    const uint64_t nw = (nbits + 31) / 32;
    const uint32_t sh = (uint32_t)(bit_off & 31);
    const uint64_t w0 = bit_off >> 5;
    const uint64_t dst_words = (bit_off + nbits + 31) / 32;
    for (uint64_t i = 0; i < nw; ++i) {
        uint32_t v = src[i];
        if (i == nw - 1 && (nbits & 31)) v &= (1u << (nbits & 31)) - 1u;
        dst[w0 + i] |= v << sh;
        if (sh && w0 + i + 1 < dst_words) dst[w0 + i + 1] |= v >> (32 - sh);
    }
}

// Runs `enqueue` (which launches the whole call on stream st) directly, or --
// for the second and later identical device-pointer calls -- as a captured
// CUDA graph: one launch instead of one per kernel and memset.  Profiling, the
// opt-in segment tree (host syncs) and the first call of a key run directly.
template <class Fn>
void run_maybe_graph(pc_ctx* c, DevState& d, cudaStream_t st, std::vector<uint64_t> key, bool allow, Fn&& enqueue) {
    if (!c->graphs || c->profiling || !allow) {
        enqueue();
        return;
    }
    key.push_back(c->bucket_mode);
    key.push_back(c->tree_mode);
    key.push_back(c->exact);
    DevState::Graph* g = nullptr;
    for (auto& e : d.graphs)
        if (e.key == key) g = &e;
    const uint64_t gen = g_alloc_gen.load();
    if (g && g->exec && g->gen == gen) {
        check(c, cudaGraphLaunch(g->exec, st), "graph launch");
        d.launches = g->launches;
        return;
    }
    if (!g || g->failed || (g->exec && g->gen != gen) || !g->exec) {
        const bool capture_now = g && !g->failed && g->gen == gen && !g->exec; // seen once, sizes settled
        if (!capture_now) {
            if (!g) {
                if (d.graphs.size() >= 16) { // bounded cache: drop the oldest
                    if (d.graphs.front().exec) cudaGraphExecDestroy(d.graphs.front().exec);
                    d.graphs.erase(d.graphs.begin());
                }
                d.graphs.push_back(DevState::Graph{key, nullptr, 0, 0, false});
                g = &d.graphs.back();
            } else if (g->exec) {
                cudaGraphExecDestroy(g->exec);
                g->exec = nullptr;
            }
            enqueue();
            g->gen = g_alloc_gen.load();
            return;
        }
    }
    // capture the call's launches
    cudaGraph_t graph = nullptr;
    const uint64_t l0 = d.launches;
    check(c, cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "begin capture");
    try {
        enqueue();
    } catch (...) {
        cudaStreamEndCapture(st, &graph);
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();
        g->failed = true;
        enqueue(); // outside capture
        return;
    }
    const cudaError_t ce = cudaStreamEndCapture(st, &graph);
    cudaGraphExec_t exec = nullptr;
    if (ce != cudaSuccess || g_alloc_gen.load() != gen ||
        cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();
        g->failed = true;
        enqueue();
        return;
    }
    cudaGraphDestroy(graph);
    g->exec = exec;
    g->gen = gen;
    g->launches = d.launches - l0;
    check(c, cudaGraphLaunch(exec, st), "graph launch");
}

// The polygon of a small call on the device: reused while the caller passes the
// same vertices (compared by content, so a changed polygon is never stale).
void cache_polygon(pc_ctx* c, DevState& d, const double* vx, const double* vy, const uint64_t* ring_off,
                   uint32_t n_rings, cudaStream_t st) {
    const uint64_t nv = ring_off[n_rings];
    if (d.cvalid && d.cro.size() == (size_t)n_rings + 1 && d.cvx.size() == nv &&
        std::memcmp(d.cro.data(), ring_off, (n_rings + 1) * sizeof(uint64_t)) == 0 &&
        std::memcmp(d.cvx.data(), vx, nv * 8) == 0 && std::memcmp(d.cvy.data(), vy, nv * 8) == 0)
        return;
    d.cvalid = false;
    d.cvx.assign(vx, vx + nv);
    d.cvy.assign(vy, vy + nv);
    d.cro.assign(ring_off, ring_off + n_rings + 1);
    check(c, d.c_vx.ensure(std::max<uint64_t>(nv * 8, 16)), "alloc cached polygon");
    check(c, d.c_vy.ensure(std::max<uint64_t>(nv * 8, 16)), "alloc cached polygon");
    check(c, d.c_ro.ensure((n_rings + 1) * 8ull), "alloc cached polygon");
    check(c, d.c_box.ensure(4 * sizeof(double)), "alloc cached bbox");
    check(c, cudaMemcpyAsync(d.c_vx.p, d.cvx.data(), nv * 8, cudaMemcpyHostToDevice, st), "upload polygon");
    check(c, cudaMemcpyAsync(d.c_vy.p, d.cvy.data(), nv * 8, cudaMemcpyHostToDevice, st), "upload polygon");
    check(c, cudaMemcpyAsync(d.c_ro.p, d.cro.data(), (n_rings + 1) * 8ull, cudaMemcpyHostToDevice, st),
          "upload polygon");
    if (nv > 0) check(c, pcd::launch_outer_bbox(d.c_vx.as<double>(), d.c_vy.as<double>(), d.c_ro.as<uint64_t>(),
                                                d.c_box.as<double>(), st, &d.launches), "bbox kernel");
    check(c, cudaStreamSynchronize(st), "upload polygon"); // the host copies may change with the next call
    d.cvalid = true;
}

unsigned char* small_staging(pc_ctx* c, DevState& d, size_t bytes) {
    if (bytes > d.h_small_cap) {
        if (d.h_small) cudaFreeHost(d.h_small);
        d.h_small = nullptr;
        d.h_small_cap = 0;
        const size_t want = std::max<size_t>(bytes, 1 << 16);
        check(c, cudaMallocHost(&d.h_small, want), "alloc pinned staging");
        d.h_small_cap = want;
    }
    return d.h_small;
}

// classify_batch / contains on at most kSmallN points: one upload, one launch, one download
constexpr uint64_t kSmallN = 2048;

void classify_small(pc_ctx* c, const double* pts_xy, uint64_t n, const double* vx, const double* vy,
                    const uint64_t* ring_off, uint32_t n_rings, int mode, double tol, int prefilter,
                    uint8_t* verdicts, uint32_t* inside_bits, uint32_t* aux_bits, uint64_t* stats) {
    DevState& d = c->devs[0];
    check(c, cudaSetDevice(d.dev), "cudaSetDevice");
    cudaStream_t st = d.stream;
    cache_polygon(c, d, vx, vy, ring_off, n_rings, st);
    const size_t ob = pcd::small_out_bytes(n), ib = n * 16;
    unsigned char* h = small_staging(c, d, ib + ob);
    std::memcpy(h, pts_xy, ib);
    check(c, d.small_pts.ensure(ib), "alloc points");
    check(c, d.small_out.ensure(ob), "alloc results");
    check(c, cudaMemcpyAsync(d.small_pts.p, h, ib, cudaMemcpyHostToDevice, st), "upload points");
    check(c, cudaMemsetAsync(d.small_out.p, 0, ob, st), "clear results");
    mark_begin(c, d, st);
    check(c, pcd::launch_small(d.small_pts.as<double>(), n, d.c_vx.as<double>(), d.c_vy.as<double>(),
                               d.c_ro.as<uint64_t>(), n_rings, prefilter ? d.c_box.as<double>() : nullptr, mode, tol,
                               d.small_out.p, nullptr, nullptr, st, &d.launches),
          "small classify kernel");
    mark_end(c, d, st);
    check(c, cudaMemcpyAsync(h + ib, d.small_out.p, ob, cudaMemcpyDeviceToHost, st), "download results");
    check(c, cudaStreamSynchronize(st), "classify");
    const uint64_t nw = (n + 31) / 32;
    const unsigned char* o = h + ib;
    if (verdicts) std::memcpy(verdicts, o, n);
    const unsigned char* planes = o + ((n + 15) & ~15ull);
    if (inside_bits) std::memcpy(inside_bits, planes, nw * 4);
    if (aux_bits) std::memcpy(aux_bits, planes + nw * 4, nw * 4);
    if (stats) std::memcpy(stats, planes + 2 * nw * 4, 32);
}

} // namespace

extern "C" {

const char* pc_version(void) { return "polycast-b200 0.1 (sm_100a)"; }

int pc_create_devices(pc_ctx** out, const int* device_ids, int n) {
    if (!out) return PC_EINVAL;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return PC_ECUDA;
    }
    if (n < 1) return PC_EINVAL;
    auto* c = new pc_ctx();
    for (int i = 0; i < n; ++i) {
        if (device_ids[i] < 0 || device_ids[i] >= count) {
            delete c;
            return PC_EINVAL;
        }
        DevState d;
        d.dev = device_ids[i];
        if (cudaSetDevice(d.dev) != cudaSuccess || cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaMallocHost(&d.h_stats, 4 * sizeof(unsigned long long)) != cudaSuccess) {
            cudaGetLastError();
            delete c;
            return PC_ECUDA;
        }
        c->devs.push_back(d);
    }
    *out = c;
    return PC_OK;
}

int pc_create(pc_ctx** out, int num_gpus) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        if (out) *out = nullptr;
        return PC_ECUDA;
    }
    if (num_gpus == 0) num_gpus = count;
    if (num_gpus < 0 || num_gpus > count) return PC_EINVAL;
    std::vector<int> ids(num_gpus);
    for (int i = 0; i < num_gpus; ++i) ids[i] = i;
    return pc_create_devices(out, ids.data(), num_gpus);
}

void pc_destroy(pc_ctx* c) {
    if (!c) return;
    for (auto& d : c->devs) {
        cudaSetDevice(d.dev);
        cudaStreamSynchronize(d.stream);
        for (DevBuf* b : {&d.pts, &d.vx, &d.vy, &d.ring_off, &d.pt_off, &d.poly_ring_off, &d.filt, &d.qk, &d.rec, &d.bbox,
                          &d.bits, &d.verdicts, &d.stats, &d.counts, &d.degen, &d.bucket_scratch,
                          &d.sorted_pts, &d.sorted_idx, &d.csr_meta, &d.cmp_blk, &d.cmp_pts, &d.cmp_idx, &d.cmp_v,
                          &d.cmp_out, &d.csv_text, &d.csv_state, &d.csv_res, &d.csv_out, &d.emit_recs,
                          &d.emit_scratch, &d.emit_out, &d.tree})
            b->release();
        if (d.h_stats) cudaFreeHost(d.h_stats);
        if (d.h_small) cudaFreeHost(d.h_small);
        for (DevBuf* b : {&d.c_vx, &d.c_vy, &d.c_ro, &d.c_box, &d.small_pts, &d.small_out}) b->release();
        delete d.stager;
        for (auto& e : d.evs) {
            cudaEventDestroy(e.first);
            cudaEventDestroy(e.second);
        }
        for (auto& g : d.graphs)
            if (g.exec) cudaGraphExecDestroy(g.exec);
        if (d.copy) cudaStreamDestroy(d.copy);
        for (cudaEvent_t e : d.up_evs) cudaEventDestroy(e);
        cudaStreamDestroy(d.stream);
    }
    delete c;
}

const char* pc_last_error(const pc_ctx* c) { return c ? c->err.c_str() : "null context"; }
int pc_device_count(const pc_ctx* c) { return c ? (int)c->devs.size() : 0; }
uint64_t pc_last_launch_count(const pc_ctx* c) {
    uint64_t n = 0;
    if (c)
        for (const auto& d : c->devs) n += d.launches;
    return n;
}

int pc_set_option(pc_ctx* c, int option, int64_t value) {
    if (!c) return PC_EINVAL;
    std::lock_guard<std::mutex> lk(c->mu);
    if (option == PC_OPT_BUCKET_POINTS && value >= -1 && value <= 1) {
        c->bucket_mode = value;
        return PC_OK;
    }
    if (option == PC_OPT_TREE && value >= -1 && value <= 1) {
        c->tree_mode = value == 1 ? 1 : 0;
        return PC_OK;
    }
    if (option == PC_OPT_EXACT && (value == 0 || value == 1)) {
        c->exact = value == 1;
        return PC_OK;
    }
    if (option == PC_OPT_GRAPH && (value == 0 || value == 1)) {
        c->graphs = value == 1;
        return PC_OK;
    }
    c->err = "unknown option or value";
    return PC_EINVAL;
}

int pc_set_profiling(pc_ctx* c, int on) {
    if (!c) return PC_EINVAL;
    std::lock_guard<std::mutex> lk(c->mu);
    c->profiling = on != 0;
    return PC_OK;
}

int pc_profile_take(pc_ctx* c, int dev_index, double* ms_out, int cap) {
    if (!c || dev_index < 0 || dev_index >= (int)c->devs.size()) return -1;
    std::lock_guard<std::mutex> lk(c->mu);
    DevState& d = c->devs[dev_index];
    cudaSetDevice(d.dev);
    int k = 0;
    for (size_t i = 0; i < d.ev_used; ++i) {
        float ms = -1.0f;
        if (cudaEventSynchronize(d.evs[i].second) != cudaSuccess ||
            cudaEventElapsedTime(&ms, d.evs[i].first, d.evs[i].second) != cudaSuccess) {
            cudaGetLastError();
            ms = -1.0f;
        }
        if (d.ev_cont[i] && k > 0) {
            if (k - 1 < cap && ms_out) ms_out[k - 1] += ms;
            continue;
        }
        if (k < cap && ms_out) ms_out[k] = ms;
        ++k;
    }
    d.ev_used = 0;
    return k;
}

int pc_measure_fp64_rate(pc_ctx* c, int dev_index, double ms, double* flops_per_s) {
    return guarded(c, [&] {
        if (dev_index < 0 || dev_index >= (int)c->devs.size() || !flops_per_s) invalid(c, "bad arguments");
        DevState& d = c->devs[dev_index];
        check(c, cudaSetDevice(d.dev), "cudaSetDevice");
        DevBuf out;
        check(c, out.ensure(64), "alloc");
        cudaEvent_t e0, e1;
        check(c, cudaEventCreate(&e0), "event");
        check(c, cudaEventCreate(&e1), "event");
        double flops = 0.0;
        int iters = 1 << 14;
        float el = 0.0f;
        for (int pass = 0; pass < 4; ++pass) { // calibrate to ~ms, keep the last (warm) pass
            check(c, cudaEventRecord(e0, d.stream), "event");
            check(c, pcd::launch_fp64_probe(out.as<double>(), iters, d.dev, d.stream, &flops), "fp64 probe");
            check(c, cudaEventRecord(e1, d.stream), "event");
            check(c, cudaEventSynchronize(e1), "fp64 probe");
            check(c, cudaEventElapsedTime(&el, e0, e1), "event");
            if (pass < 3 && el > 0.0f) iters = std::max(1, (int)(iters * (ms / el)));
        }
        *flops_per_s = flops / (el * 1e-3);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        out.release();
    });
}

int pc_classify(pc_ctx* c, const double* pts_xy, uint64_t n, const double* vx, const double* vy,
                const uint64_t* ring_off, uint32_t n_rings, int mode, double tol, int prefilter, uint8_t* verdicts,
                uint32_t* inside_bits, uint32_t* aux_bits, uint64_t stats[4]) {
    return guarded(c, [&] {
        if (mode < 0 || mode > 2) invalid(c, "mode must be 0 (C1), 1 (C2) or 2 (Robust)");
        if (!ring_off || !vx || !vy) invalid(c, "null polygon arrays");
        validate_rings(c, ring_off, n_rings);
        if (n && !pts_xy) invalid(c, "null points");
        uint64_t tot[4] = {0, 0, 0, 0};
        if (n == 0) {
            if (stats) std::memset(stats, 0, 4 * sizeof(uint64_t));
            return;
        }
        const uint64_t n_verts = ring_off[n_rings];
        if (n <= kSmallN) { // the drop-in API's single-point calls and tiny batches
            classify_small(c, pts_xy, n, vx, vy, ring_off, n_rings, mode, tol, prefilter, verdicts, inside_bits,
                           aux_bits, stats);
            return;
        }
        // contiguous shards, 32-point aligned so every device owns whole words
        const uint64_t ndev = std::min<uint64_t>(c->devs.size(), std::max<uint64_t>(1, n / 32));
        uint64_t shard = (n + ndev - 1) / ndev;
        shard = (shard + 31) & ~31ull;
        struct Part {
            uint64_t lo, hi;
        };
        std::vector<Part> parts;
        for (uint64_t d = 0; d < ndev; ++d) {
            const uint64_t lo = std::min(n, d * shard), hi = std::min(n, (d + 1) * shard);
            if (hi > lo) parts.push_back({lo, hi});
        }
        // one host thread per device: upload, enqueue, download and wait for its shard
        per_device(parts.size(), [&](size_t i) {
            DevState& d = c->devs[i];
            const uint64_t m = parts[i].hi - parts[i].lo, nwords = (m + 31) / 32;
            check(c, cudaSetDevice(d.dev), "cudaSetDevice");
            cudaStream_t st = d.stream;
            // polygon first on the compute stream; the points on the copy stream, so
            // prep and the segment-tree build run while they upload (an async
            // copy for pinned points; pageable ones are staged by this thread)
            h2d(c, d, d.vx, vx, n_verts * 8, st, "upload vx");
            h2d(c, d, d.vy, vy, n_verts * 8, st, "upload vy");
            h2d(c, d, d.ring_off, ring_off, (n_rings + 1) * 8ull, st, "upload ring_off");
            if (!d.copy) check(c, cudaStreamCreateWithFlags(&d.copy, cudaStreamNonBlocking), "create copy stream");
            // big shards upload in chunks, each classified while the next one uploads
            const uint64_t chunk = m > 2 * kUploadChunk ? kUploadChunk : 0;
            const uint64_t nchunks = chunk ? (m + chunk - 1) / chunk : 1;
            while (d.up_evs.size() < nchunks) {
                cudaEvent_t ev;
                check(c, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "create upload event");
                d.up_evs.push_back(ev);
            }
            check(c, d.pts.ensure(std::max<uint64_t>(m * 16, 16)), "upload points");
            for (uint64_t k = 0; k < nchunks; ++k) {
                const uint64_t lo = k * (chunk ? chunk : m), cnt = std::min(chunk ? chunk : m, m - lo);
                check(c, stager(d).h2d(d.pts.as<double>() + 2 * lo, pts_xy + 2 * (parts[i].lo + lo), cnt * 16, d.copy),
                      "upload points");
                check(c, cudaEventRecord(d.up_evs[k], d.copy), "record upload event");
            }
            check(c, d.bits.ensure(2 * nwords * 4), "alloc bit planes");
            check(c, d.stats.ensure(4 * 8), "alloc stats");
            uint8_t* dv = nullptr;
            if (verdicts) {
                check(c, d.verdicts.ensure(m), "alloc verdicts");
                dv = d.verdicts.as<uint8_t>();
            }
            uint32_t* din = d.bits.as<uint32_t>();
            uint32_t* daux = din + nwords;
            enqueue_single(c, d, st, d.pts.as<double>(), m, d.vx.as<double>(), d.vy.as<double>(),
                           d.ring_off.as<uint64_t>(), n_rings, n_verts, mode, tol, prefilter, dv, din, daux,
                           d.stats.as<unsigned long long>(), d.up_evs.data(), chunk);
            if (inside_bits)
                check(c, cudaMemcpyAsync(inside_bits + parts[i].lo / 32, din, nwords * 4, cudaMemcpyDeviceToHost, st),
                      "download inside plane");
            if (aux_bits)
                check(c, cudaMemcpyAsync(aux_bits + parts[i].lo / 32, daux, nwords * 4, cudaMemcpyDeviceToHost, st),
                      "download aux plane");
            if (verdicts)
                check(c, cudaMemcpyAsync(verdicts + parts[i].lo, dv, m, cudaMemcpyDeviceToHost, st),
                      "download verdicts");
            check(c, cudaMemcpyAsync(d.h_stats, d.stats.p, 32, cudaMemcpyDeviceToHost, st), "download stats");
            check(c, cudaStreamSynchronize(st), "classify");
        });
        for (size_t i = 0; i < parts.size(); ++i)
            for (int k = 0; k < 4; ++k) tot[k] += c->devs[i].h_stats[k];
        if (stats) std::memcpy(stats, tot, sizeof(tot));
    });
}

int pc_classify_csr(pc_ctx* c, const double* pts_xy, const uint64_t* pt_off, uint64_t n_polys, const double* vx,
                    const double* vy, const uint64_t* ring_off, const uint64_t* poly_ring_off, int mode, double tol,
                    uint8_t* verdicts, uint32_t* inside_bits, uint32_t* aux_bits, uint64_t stats[4]) {
    return guarded(c, [&] {
        if (mode < 0 || mode > 2) invalid(c, "mode must be 0 (C1), 1 (C2) or 2 (Robust)");
        if (!pt_off || !poly_ring_off) invalid(c, "null CSR offsets");
        uint64_t tot[4] = {0, 0, 0, 0};
        const uint64_t n_points = n_polys ? pt_off[n_polys] - pt_off[0] : 0;
        if (n_points == 0) {
            if (stats) std::memset(stats, 0, sizeof(tot));
            return;
        }
        if (!pts_xy || !vx || !vy || !ring_off) invalid(c, "null arrays");
        for (uint64_t p = 0; p < n_polys; ++p)
            if (pt_off[p + 1] < pt_off[p] || poly_ring_off[p + 1] < poly_ring_off[p])
                invalid(c, "CSR offsets must be non-decreasing");
        const uint64_t P0 = pt_off[0];
        const uint64_t nwords_all = (n_points + 31) / 32;
        std::mutex merge_mu;
        if (inside_bits) std::memset(inside_bits, 0, nwords_all * 4);
        if (aux_bits) std::memset(aux_bits, 0, nwords_all * 4);
        // shard polygons so each device gets ~n_points/ndev points
        const uint64_t ndev = std::min<uint64_t>(c->devs.size(), n_polys);
        std::vector<uint64_t> cut{0};
        for (uint64_t d = 1; d < ndev; ++d) {
            const uint64_t target = P0 + n_points * d / ndev;
            uint64_t p = std::lower_bound(pt_off, pt_off + n_polys + 1, target) - pt_off;
            p = std::max(p, cut.back());
            cut.push_back(std::min(p, n_polys));
        }
        cut.push_back(n_polys);
        // one host thread per device; its bit planes come back into pinned
        // per-device buffers and are OR-ed into the caller's planes at the
        // shard's bit offset (a shard starts at a polygon, not a word boundary)
        per_device(ndev, [&](size_t i) {
            const uint64_t p0 = cut[i], p1 = cut[i + 1];
            if (p1 == p0) return;
            DevState& d = c->devs[i];
            const uint64_t s = pt_off[p0], t = pt_off[p1], m = t - s, nwords = (m + 31) / 32;
            check(c, cudaSetDevice(d.dev), "cudaSetDevice");
            cudaStream_t st = d.stream;
            const uint64_t r0 = poly_ring_off[p0], r1 = poly_ring_off[p1];
            const uint64_t v0 = r1 > r0 ? ring_off[r0] : 0, v1 = r1 > r0 ? ring_off[r1] : 0;
            h2d(c, d, d.pts, pts_xy + 2 * (s - P0), m * 16, st, "upload points");
            h2d(c, d, d.pt_off, pt_off + p0, (p1 - p0 + 1) * 8, st, "upload pt_off");
            h2d(c, d, d.poly_ring_off, poly_ring_off + p0, (p1 - p0 + 1) * 8, st, "upload poly_ring_off");
            h2d(c, d, d.ring_off, ring_off + r0, (r1 - r0 + 1) * 8, st, "upload ring_off");
            h2d(c, d, d.vx, vx + v0, (v1 - v0) * 8, st, "upload vx");
            h2d(c, d, d.vy, vy + v0, (v1 - v0) * 8, st, "upload vy");
            check(c, d.bits.ensure(2 * nwords * 4), "alloc bit planes");
            check(c, d.stats.ensure(32), "alloc stats");
            uint8_t* dv = nullptr;
            if (verdicts) {
                check(c, d.verdicts.ensure(m), "alloc verdicts");
                dv = d.verdicts.as<uint8_t>();
            }
            uint32_t* din = d.bits.as<uint32_t>();
            uint32_t* daux = din + nwords;
            enqueue_csr(c, d, st, d.pts.as<double>(), m, d.pt_off.as<uint64_t>(), p1 - p0, d.vx.as<double>(),
                        d.vy.as<double>(), d.ring_off.as<uint64_t>(), d.poly_ring_off.as<uint64_t>(), s, r0, v0, mode,
                        tol, dv, din, daux, d.stats.as<unsigned long long>());
            uint32_t* hp = nullptr;
            if (inside_bits || aux_bits) {
                hp = reinterpret_cast<uint32_t*>(small_staging(c, d, 2 * nwords * 4));
                check(c, cudaMemcpyAsync(hp, din, 2 * nwords * 4, cudaMemcpyDeviceToHost, st), "download planes");
            }
            if (verdicts)
                check(c, cudaMemcpyAsync(verdicts + (s - P0), dv, m, cudaMemcpyDeviceToHost, st), "download verdicts");
            check(c, cudaMemcpyAsync(d.h_stats, d.stats.p, 32, cudaMemcpyDeviceToHost, st), "download stats");
            check(c, cudaStreamSynchronize(st), "classify_csr");
            if (hp) {
                std::lock_guard<std::mutex> lk(merge_mu); // neighbouring shards share boundary words
                if (inside_bits) merge_bits(inside_bits, hp, s - P0, m);
                if (aux_bits) merge_bits(aux_bits, hp + nwords, s - P0, m);
            }
        });
        for (uint64_t i = 0; i < ndev; ++i)
            if (cut[i + 1] != cut[i])
                for (int k = 0; k < 4; ++k) tot[k] += c->devs[i].h_stats[k];
        if (stats) std::memcpy(stats, tot, sizeof(tot));
    });
}

int pc_count_crossings(pc_ctx* c, const double* pts_xy, uint64_t n, const double* vx, const double* vy, uint64_t nv,
                       int mode, uint64_t* counts, uint8_t* degenerate) {
    return guarded(c, [&] {
        if (mode != 0 && mode != 1) invalid(c, "count_crossings: mode must be 0 (C1) or 1 (C2)");
        if (n == 0) return;
        if (!pts_xy || !counts || !degenerate || (nv && (!vx || !vy))) invalid(c, "null arrays");
        DevState& d = c->devs[0];
        check(c, cudaSetDevice(d.dev), "cudaSetDevice");
        cudaStream_t st = d.stream;
        if (n <= kSmallN) { // cached ring, a CTA per point, one round trip
            const uint64_t ro[2] = {0, nv};
            cache_polygon(c, d, vx, vy, ro, 1, st);
            const size_t ib = n * 16, cb = n * 8;
            unsigned char* h = small_staging(c, d, ib + cb + n);
            std::memcpy(h, pts_xy, ib);
            check(c, d.small_pts.ensure(ib), "alloc points");
            check(c, d.small_out.ensure(cb + n + 16), "alloc results");
            check(c, cudaMemcpyAsync(d.small_pts.p, h, ib, cudaMemcpyHostToDevice, st), "upload points");
            unsigned long long* dc = d.small_out.as<unsigned long long>();
            check(c, pcd::launch_small(d.small_pts.as<double>(), n, d.c_vx.as<double>(), d.c_vy.as<double>(),
                                       d.c_ro.as<uint64_t>(), 1, nullptr, mode, 0.0, nullptr, dc,
                                       reinterpret_cast<uint8_t*>(dc + n), st, &d.launches),
                  "count kernel");
            check(c, cudaMemcpyAsync(h + ib, d.small_out.p, cb + n, cudaMemcpyDeviceToHost, st), "download counts");
            check(c, cudaStreamSynchronize(st), "count_crossings");
            std::memcpy(counts, h + ib, cb);
            std::memcpy(degenerate, h + ib + cb, n);
            return;
        }
        h2d(c, d, d.pts, pts_xy, n * 16, st, "upload points");
        h2d(c, d, d.vx, vx, nv * 8, st, "upload vx");
        h2d(c, d, d.vy, vy, nv * 8, st, "upload vy");
        check(c, d.counts.ensure(n * 8), "alloc counts");
        check(c, d.degen.ensure(n), "alloc flags");
        check(c, pcd::launch_count(d.pts.as<double>(), n, d.vx.as<double>(), d.vy.as<double>(), nv, mode,
                                   d.counts.as<unsigned long long>(), d.degen.as<uint8_t>(), st, &d.launches),
              "count kernel");
        check(c, cudaMemcpyAsync(counts, d.counts.p, n * 8, cudaMemcpyDeviceToHost, st), "download counts");
        check(c, cudaMemcpyAsync(degenerate, d.degen.p, n, cudaMemcpyDeviceToHost, st), "download flags");
        check(c, cudaStreamSynchronize(st), "count_crossings");
    });
}

namespace {

void check_box(pc_ctx* c, const double* box) {
    if (!box) invalid(c, "null box");
    if (!(box[0] <= box[2]) || !(box[1] <= box[3])) invalid(c, "BBox: min must not exceed max");
}

// prefilter on device d, stream st; blk scratch from d; count left at blk[n_blk]
unsigned long long* enqueue_prefilter(pc_ctx* c, DevState& d, cudaStream_t st, const double* d_pts, uint64_t n,
                                      const double* box, double* d_out, unsigned long long* d_idx) {
    const int nb = pcd::compact_blocks(n, d.dev);
    check(c, d.cmp_blk.ensure((size_t)(nb + 1) * 8), "alloc prefilter scratch");
    unsigned long long* blk = d.cmp_blk.as<unsigned long long>();
    check(c, pcd::launch_prefilter(d_pts, n, box, nb, blk, d_out, d_idx, st, &d.launches), "prefilter kernels");
    return blk + nb;
}

} // namespace

int pc_prefilter_bbox(pc_ctx* c, const double* pts_xy, uint64_t n, const double box[4], double* out_xy,
                      uint64_t* out_idx, uint64_t* n_inside) {
    return guarded(c, [&] {
        check_box(c, box);
        if (!n_inside) invalid(c, "null n_inside");
        *n_inside = 0;
        if (n == 0) return;
        if (!pts_xy || !out_xy || !out_idx) invalid(c, "null arrays");
        DevState& d = c->devs[0];
        check(c, cudaSetDevice(d.dev), "cudaSetDevice");
        cudaStream_t st = d.stream;
        h2d(c, d, d.cmp_pts, pts_xy, n * 16, st, "upload points");
        check(c, d.cmp_out.ensure(n * 16), "alloc compacted points");
        check(c, d.cmp_idx.ensure(n * 8), "alloc indices");
        const unsigned long long* cnt = enqueue_prefilter(c, d, st, d.cmp_pts.as<double>(), n, box,
                                                          d.cmp_out.as<double>(), d.cmp_idx.as<unsigned long long>());
        unsigned long long k = 0;
        check(c, cudaMemcpyAsync(&k, cnt, 8, cudaMemcpyDeviceToHost, st), "download count");
        check(c, cudaStreamSynchronize(st), "prefilter");
        if (k) {
            d2h(c, d, out_xy, d.cmp_out.p, k * 16, st, "download points");
            d2h(c, d, out_idx, d.cmp_idx.p, k * 8, st, "download indices");
        }
        *n_inside = k;
    });
}

int pc_scatter_verdicts(pc_ctx* c, const uint64_t* idx, const uint8_t* inbox_verdicts, uint64_t n_inbox,
                        uint64_t n_total, uint8_t* out) {
    return guarded(c, [&] {
        if (n_inbox > n_total) invalid(c, "scatter_verdicts: verdict count does not match index map");
        if (n_total == 0) return;
        if (!out || (n_inbox && (!idx || !inbox_verdicts))) invalid(c, "null arrays");
        DevState& d = c->devs[0];
        check(c, cudaSetDevice(d.dev), "cudaSetDevice");
        cudaStream_t st = d.stream;
        h2d(c, d, d.cmp_idx, idx, n_inbox * 8, st, "upload indices");
        h2d(c, d, d.cmp_v, inbox_verdicts, n_inbox, st, "upload verdicts");
        const size_t off = (n_total + 7) & ~7ull; // the out-of-range flag after the verdicts
        check(c, d.cmp_out.ensure(off + 16), "alloc verdicts");
        uint8_t* o = d.cmp_out.as<uint8_t>();
        unsigned* bad = reinterpret_cast<unsigned*>(o + off);
        check(c, cudaMemsetAsync(bad, 0, 4, st), "clear flag");
        check(c, pcd::launch_scatter_verdicts(d.cmp_idx.as<unsigned long long>(), d.cmp_v.as<uint8_t>(), n_inbox,
                                              n_total, o, bad, st, d.dev, &d.launches),
              "scatter kernel");
        unsigned b = 0;
        check(c, cudaMemcpyAsync(&b, bad, 4, cudaMemcpyDeviceToHost, st), "download flag");
        d2h(c, d, out, o, n_total, st, "download verdicts");
        check(c, cudaStreamSynchronize(st), "scatter_verdicts");
        if (b) invalid(c, "scatter_verdicts: original index out of range");
    });
}

int pc_prefilter_bbox_dev(pc_ctx* c, int dev_index, void* stream, const double* d_pts_xy, uint64_t n,
                          const double box[4], double* d_out_xy, uint64_t* d_out_idx, uint64_t* d_n_inside) {
    return guarded(c, [&] {
        if (dev_index < 0 || dev_index >= (int)c->devs.size()) invalid(c, "bad device index");
        check_box(c, box);
        if (!d_n_inside) invalid(c, "null count");
        DevState& d = c->devs[dev_index];
        check(c, cudaSetDevice(d.dev), "cudaSetDevice");
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d.stream;
        if (n == 0) {
            check(c, cudaMemsetAsync(d_n_inside, 0, 8, st), "clear count");
            return;
        }
        if (!d_pts_xy || !d_out_xy || !d_out_idx) invalid(c, "null arrays");
        const unsigned long long* cnt = enqueue_prefilter(c, d, st, d_pts_xy, n, box, d_out_xy,
                                                          reinterpret_cast<unsigned long long*>(d_out_idx));
        check(c, cudaMemcpyAsync(d_n_inside, cnt, 8, cudaMemcpyDeviceToDevice, st), "copy count");
    });
}

int pc_scatter_verdicts_dev(pc_ctx* c, int dev_index, void* stream, const uint64_t* d_idx,
                            const uint8_t* d_inbox_verdicts, uint64_t n_inbox, uint64_t n_total, uint8_t* d_out,
                            uint32_t* d_bad) {
    return guarded(c, [&] {
        if (dev_index < 0 || dev_index >= (int)c->devs.size()) invalid(c, "bad device index");
        if (n_inbox > n_total) invalid(c, "scatter_verdicts: verdict count does not match index map");
        if (n_total == 0) return;
        if (!d_out || !d_bad || (n_inbox && (!d_idx || !d_inbox_verdicts))) invalid(c, "null arrays");
        DevState& d = c->devs[dev_index];
        check(c, cudaSetDevice(d.dev), "cudaSetDevice");
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d.stream;
        check(c, pcd::launch_scatter_verdicts(reinterpret_cast<const unsigned long long*>(d_idx), d_inbox_verdicts,
                                              n_inbox, n_total, d_out, d_bad, st, d.dev, &d.launches),
              "scatter kernel");
    });
}

int pc_parse_points_csv(pc_ctx* c, const char* text, uint64_t len, uint64_t data_start, uint32_t x_col,
                        uint32_t y_col, char delim, double* out_xy, uint64_t cap_points, uint64_t* n_points,
                        uint64_t* n_bad, uint64_t* first_bad_offset, uint32_t* first_bad_kind) {
    return guarded(c, [&] {
        if (!n_points || !n_bad || !first_bad_offset || !first_bad_kind) invalid(c, "null outputs");
        *first_bad_kind = 0;
        *n_points = *n_bad = 0;
        *first_bad_offset = ~0ull;
        if (x_col == y_col) invalid(c, "read_points_csv: x and y columns must differ");
        if (len == 0) return;
        if (!text) invalid(c, "null text");
        DevState& d = c->devs[0];
        check(c, cudaSetDevice(d.dev), "cudaSetDevice");
        cudaStream_t st = d.stream;
        h2d(c, d, d.csv_text, text, len, st, "upload text");
        check(c, d.csv_state.ensure(pcd::csv_scratch_bytes(len)), "alloc csv scratch");
        // a good row spans >= 4 bytes ("d,d\n") except the file's last: (len + 1) / 4 bounds the rows
        const uint64_t dev_cap = std::min<uint64_t>(cap_points, (len + 1) / 4 + 1);
        check(c, d.csv_out.ensure(std::max<uint64_t>(dev_cap, 1) * 16), "alloc points");
        check(c, d.csv_res.ensure(4 * 8), "alloc results");
        unsigned long long* res = d.csv_res.as<unsigned long long>();
        mark_begin(c, d, st);
        check(c, pcd::launch_csv_points(d.csv_text.as<char>(), len, data_start, x_col, y_col, delim,
                                        d.csv_out.as<double>(), dev_cap, d.csv_state.p,
                                        res, st, &d.launches),
              "csv kernel");
        mark_end(c, d, st);
        check(c, cudaMemcpyAsync(d.h_stats, res, 32, cudaMemcpyDeviceToHost, st), "download counts");
        check(c, cudaStreamSynchronize(st), "csv");
        const uint64_t n_ok = d.h_stats[0], fb = d.h_stats[2];
        *n_points = n_ok;
        *n_bad = d.h_stats[1];
        if (fb != ~0ull) {
            *first_bad_offset = fb >> 3;
            *first_bad_kind = (uint32_t)(fb & 7);
        }
        if (n_ok > cap_points) invalid(c, "read_points_csv: output capacity too small (n_points holds the need)");
        if (n_ok) {
            if (!out_xy) invalid(c, "null out_xy");
            d2h(c, d, out_xy, d.csv_out.p, n_ok * 16, st, "download points");
        }
    });
}

int pc_parse_points_csv_dev(pc_ctx* c, int dev_index, void* stream, const char* d_text, uint64_t len,
                            uint64_t data_start, uint32_t x_col, uint32_t y_col, char delim, double* d_out_xy,
                            uint64_t cap_points, uint64_t* d_result) {
    return guarded(c, [&] {
        if (dev_index < 0 || dev_index >= (int)c->devs.size()) invalid(c, "bad device index");
        if (x_col == y_col) invalid(c, "read_points_csv: x and y columns must differ");
        if (!d_result || (len && !d_text) || (cap_points && !d_out_xy)) invalid(c, "null arrays");
        DevState& d = c->devs[dev_index];
        check(c, cudaSetDevice(d.dev), "cudaSetDevice");
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d.stream;
        check(c, d.csv_state.ensure(pcd::csv_scratch_bytes(len)), "alloc csv scratch");
        mark_begin(c, d, st);
        check(c, pcd::launch_csv_points(d_text, len, data_start, x_col, y_col, delim, d_out_xy, cap_points,
                                        d.csv_state.p,
                                        reinterpret_cast<unsigned long long*>(d_result), st, &d.launches),
              "csv kernel");
        mark_end(c, d, st);
    });
}

int pc_format_results_csv(pc_ctx* c, const pc_result_record* recs, uint64_t n, char* out, uint64_t cap,
                          uint64_t* len) {
    return guarded(c, [&] {
        if (!len) invalid(c, "null length");
        *len = 0;
        if (n && !recs) invalid(c, "null records");
        DevState& d = c->devs[0];
        check(c, cudaSetDevice(d.dev), "cudaSetDevice");
        cudaStream_t st = d.stream;
        h2d(c, d, d.emit_recs, recs, n * sizeof(pc_result_record), st, "upload records");
        check(c, d.emit_scratch.ensure(pcd::emit_scratch_bytes(n)), "alloc emit scratch");
        const uint64_t dev_cap = pcd::emit_max_bytes(n);
        check(c, d.emit_out.ensure(dev_cap), "alloc text");
        check(c, d.csv_res.ensure(4 * 8), "alloc results");
        unsigned long long* dl = d.csv_res.as<unsigned long long>();
        mark_begin(c, d, st);
        check(c, pcd::launch_emit_results(d.emit_recs.p, n, d.emit_out.as<char>(), dev_cap, d.emit_scratch.p, dl, st,
                                          &d.launches),
              "emit kernels");
        mark_end(c, d, st);
        check(c, cudaMemcpyAsync(d.h_stats, dl, 8, cudaMemcpyDeviceToHost, st), "download length");
        check(c, cudaStreamSynchronize(st), "emit");
        const uint64_t total = d.h_stats[0];
        *len = total;
        if (total > cap) invalid(c, "write_results_csv: output capacity too small (len holds the need)");
        if (!out) invalid(c, "null out");
        d2h(c, d, out, d.emit_out.p, total, st, "download text");
    });
}

int pc_format_results_csv_dev(pc_ctx* c, int dev_index, void* stream, const pc_result_record* d_recs, uint64_t n,
                              char* d_out, uint64_t cap, uint64_t* d_len) {
    return guarded(c, [&] {
        if (dev_index < 0 || dev_index >= (int)c->devs.size()) invalid(c, "bad device index");
        if (!d_len || (n && !d_recs) || (cap && !d_out)) invalid(c, "null arrays");
        DevState& d = c->devs[dev_index];
        check(c, cudaSetDevice(d.dev), "cudaSetDevice");
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d.stream;
        check(c, d.emit_scratch.ensure(pcd::emit_scratch_bytes(n)), "alloc emit scratch");
        mark_begin(c, d, st);
        check(c, pcd::launch_emit_results(d_recs, n, d_out, cap, d.emit_scratch.p,
                                          reinterpret_cast<unsigned long long*>(d_len), st, &d.launches),
              "emit kernels");
        mark_end(c, d, st);
    });
}

int pc_classify_dev(pc_ctx* c, int dev_index, void* stream, const double* d_pts_xy, uint64_t n, const double* d_vx,
                    const double* d_vy, const uint64_t* d_ring_off, uint32_t n_rings, uint64_t n_verts, int mode,
                    double tol, int prefilter, uint8_t* d_verdicts, uint32_t* d_inside, uint32_t* d_aux,
                    uint64_t* d_stats) {
    return guarded(c, [&] {
        if (dev_index < 0 || dev_index >= (int)c->devs.size()) invalid(c, "bad device index");
        if (mode < 0 || mode > 2) invalid(c, "mode must be 0 (C1), 1 (C2) or 2 (Robust)");
        if (n_rings < 1 || n_verts < n_rings) invalid(c, "bad ring layout");
        if (!d_inside || !d_aux || !d_stats) invalid(c, "null output planes");
        if (reinterpret_cast<uintptr_t>(d_pts_xy) & 15) invalid(c, "device points must be 16-byte aligned");
        DevState& d = c->devs[dev_index];
        check(c, cudaSetDevice(d.dev), "cudaSetDevice");
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d.stream;
        if (n == 0) {
            check(c, cudaMemsetAsync(d_stats, 0, 32, st), "clear stats");
            return;
        }
        uint64_t tolbits;
        std::memcpy(&tolbits, &tol, 8);
        const std::vector<uint64_t> key{0, (uint64_t)dev_index, (uint64_t)(uintptr_t)st, (uint64_t)(uintptr_t)d_pts_xy,
                                        n, (uint64_t)(uintptr_t)d_vx, (uint64_t)(uintptr_t)d_vy,
                                        (uint64_t)(uintptr_t)d_ring_off, n_rings, n_verts, (uint64_t)mode, tolbits,
                                        (uint64_t)prefilter, (uint64_t)(uintptr_t)d_verdicts,
                                        (uint64_t)(uintptr_t)d_inside, (uint64_t)(uintptr_t)d_aux,
                                        (uint64_t)(uintptr_t)d_stats};
        run_maybe_graph(c, d, st, key, c->tree_mode != 1, [&] {
            enqueue_single(c, d, st, d_pts_xy, n, d_vx, d_vy, d_ring_off, n_rings, n_verts, mode, tol, prefilter,
                           d_verdicts, d_inside, d_aux, reinterpret_cast<unsigned long long*>(d_stats));
        });
    });
}

int pc_classify_csr_dev(pc_ctx* c, int dev_index, void* stream, const double* d_pts_xy, const uint64_t* d_pt_off,
                        uint64_t n_polys, uint64_t n_points, const double* d_vx, const double* d_vy,
                        const uint64_t* d_ring_off, const uint64_t* d_poly_ring_off, int mode, double tol,
                        uint8_t* d_verdicts, uint32_t* d_inside, uint32_t* d_aux, uint64_t* d_stats) {
    return guarded(c, [&] {
        if (dev_index < 0 || dev_index >= (int)c->devs.size()) invalid(c, "bad device index");
        if (mode < 0 || mode > 2) invalid(c, "mode must be 0 (C1), 1 (C2) or 2 (Robust)");
        if (!d_inside || !d_aux || !d_stats) invalid(c, "null output planes");
        DevState& d = c->devs[dev_index];
        check(c, cudaSetDevice(d.dev), "cudaSetDevice");
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d.stream;
        if (n_points == 0) {
            check(c, cudaMemsetAsync(d_stats, 0, 32, st), "clear stats");
            return;
        }
        uint64_t tolbits;
        std::memcpy(&tolbits, &tol, 8);
        const std::vector<uint64_t> key{1, (uint64_t)dev_index, (uint64_t)(uintptr_t)st, (uint64_t)(uintptr_t)d_pts_xy,
                                        (uint64_t)(uintptr_t)d_pt_off, n_polys, n_points, (uint64_t)(uintptr_t)d_vx,
                                        (uint64_t)(uintptr_t)d_vy, (uint64_t)(uintptr_t)d_ring_off,
                                        (uint64_t)(uintptr_t)d_poly_ring_off, (uint64_t)mode, tolbits,
                                        (uint64_t)(uintptr_t)d_verdicts, (uint64_t)(uintptr_t)d_inside,
                                        (uint64_t)(uintptr_t)d_aux, (uint64_t)(uintptr_t)d_stats};
        run_maybe_graph(c, d, st, key, true, [&] {
            enqueue_csr(c, d, st, d_pts_xy, n_points, d_pt_off, n_polys, d_vx, d_vy, d_ring_off, d_poly_ring_off, 0,
                        0, 0, mode, tol, d_verdicts, d_inside, d_aux, reinterpret_cast<unsigned long long*>(d_stats));
        });
    });
}

} // extern "C"
