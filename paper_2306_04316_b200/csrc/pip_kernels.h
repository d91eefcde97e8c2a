// Host-side launch interface of the sm_100a point-in-polygon kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace pcd {

struct PrepArgs {
    int mode;
    const double* vx;
    const double* vy;
    const uint64_t* ring_off;
    uint32_t n_rings;
    uint64_t n_verts;
    uint2* filt;                  // per-edge per-point filter words (see prep_edges_kernel)
    uint32_t* qk;                 // per-edge key words of the phase-1 key scan, padded to qk_words()
    void* rec;                    // n_edges EdgeRec (edge_rec_bytes() each)
    unsigned long long* bbox_keys; // 4 monotone keys: min x, min y, ~max x, ~max y; [4..5] 16-bit key map
    uint32_t* zero_words;          // output bit planes to clear: inside ...
    uint32_t* zero_words2;         // ... and aux (n_zero_words each)
    uint64_t n_zero_words;
    unsigned long long* stats;     // 4 counters to clear
    double tol;                    // Robust boundary tolerance (gates its fp32 side records)
};

struct SingleArgs {
    int mode;
    const double* pts;
    uint64_t n;
    const uint32_t* qk;
    const uint2* filt;
    const void* rec;
    uint32_t n_edges;
    const unsigned long long* bbox_keys;
    int prefilter;
    double tol, tol2;
    uint32_t* inside_bits;
    uint32_t* aux_bits;
    const uint32_t* n_dev; // optional device-side point count (bucketed input)
    const uint32_t* orig;  // optional (y-ordered input): results of point i go to bit orig[i] of the planes
};

struct CsrArgs {
    int mode;
    const double* pts;
    const uint64_t* pt_off;
    uint64_t n_polys;
    const double* vx;
    const double* vy;
    const uint64_t* ring_off;
    const uint64_t* poly_ring_off;
    uint64_t pt_base, ring_base, vert_base; // subtracted from pt_off / poly_ring_off / ring_off values
    double tol, tol2;
    uint32_t* inside_bits;
    uint32_t* aux_bits;
    void* meta; // csr_meta_bytes(n_polys) of device scratch (per-polygon records)
};

size_t edge_rec_bytes();
constexpr int kKeyTile = 2048;       // edge key words per stage of pip_single.cu's key scan
size_t filt_words(uint64_t n_edges); // uint2 entries of the filter array
size_t qk_words(uint64_t n_edges);   // uint32 entries of the key array (whole tiles, padding never matches)
// position of edge e's q(ylo) half in the key array (its 0x7fff - q(yhi) half is 8 further):
// groups of 8 edges, 16 halves each (pip_kernels.cu prep_edges_body)
__host__ __device__ __forceinline__ uint64_t qk_half(uint64_t e) { return (e >> 3) * 16 + (e & 7); }
size_t csr_meta_bytes(uint64_t n_polys);
cudaError_t launch_prep(const PrepArgs& a, cudaStream_t st, int dev, uint64_t* launches);
cudaError_t launch_single(const SingleArgs& a, cudaStream_t st, int dev, uint64_t* launches);
cudaError_t launch_csr(const CsrArgs& a, cudaStream_t st, int dev, uint64_t* launches);
// C1 tile kernel (pip_csr_tile.cu): appends the polygons of oversized tiles to
// list[*count ...] for the warp-per-polygon kernel
cudaError_t launch_csr_tile(const CsrArgs& a, uint32_t* list, uint32_t* count, cudaStream_t st, int dev,
                            uint64_t* launches);
cudaError_t launch_finalize(uint64_t n, uint32_t* inside_bits, const uint32_t* aux_bits, uint8_t* verdicts,
                            int mode, unsigned long long* stats, cudaStream_t st, int dev, uint64_t* launches);
cudaError_t launch_count(const double* pts, uint64_t n, const double* vx, const double* vy, uint64_t nv, int mode,
                         unsigned long long* counts, uint8_t* degenerate, cudaStream_t st, uint64_t* launches);

// GPU prefilter_bbox / scatter_verdicts (pip_compact.cu): blk needs
// compact_blocks(n)+1 entries; box = {min_x, min_y, max_x, max_y}; the in-box
// count lands in blk[n_blk].
int compact_blocks(uint64_t n, int dev);
cudaError_t launch_prefilter(const double* pts, uint64_t n, const double box[4], int n_blk,
                             unsigned long long* blk, double* out_pts, unsigned long long* out_idx, cudaStream_t st,
                             uint64_t* launches);
cudaError_t launch_scatter_verdicts(const unsigned long long* idx, const uint8_t* v, uint64_t n_in, uint64_t n_total,
                                    uint8_t* out, unsigned* bad, cudaStream_t st, int dev, uint64_t* launches);

// GPU points-CSV reader (pip_csv.cu): three launches (parse tiles, scan the
// tile counts, emit); scratch = csv_scratch_bytes(len) bytes of device memory;
// res = 4 words ([0] rows kept, [1] bad rows, [2] first bad row as (line start
// offset << 3 | kind), [3] unused), reset here.
uint64_t csv_tiles(uint64_t len);
uint64_t csv_scratch_bytes(uint64_t len);
cudaError_t launch_csv_points(const char* text, uint64_t len, uint64_t data_start, uint32_t x_idx, uint32_t y_idx,
                              char delim, double* out, uint64_t cap, void* scratch, unsigned long long* res,
                              cudaStream_t st, uint64_t* launches);

// Segment-tree C1 path for one large polygon (pip_tree.cu): builds the tree
// from the prepared polygon (prep_edges_kernel's records and map), counts the
// clean points' crossings and sends the rest through launch_single(single);
// writes every word of inside_bits.
struct TreeArgs {
    int mode; // kC1 or kC2
    const double* pts;
    uint64_t n;
    uint64_t n_layout;     // points the scratch layout is sized for (>= n; 0: n) -- the same in both phases
    const uint32_t* n_dev; // optional device-side point count (y-bucketed input)
    int prefilter;
    const double* vx;
    const double* vy;
    const uint64_t* ring_off;
    uint32_t n_rings;
    uint64_t n_verts, n_edges;
    const void* rec;
    const unsigned long long* bbox_keys;
    uint32_t* inside_bits;
    uint32_t* aux_bits; // C2: DegenerateEdge (zeroed by the caller)
    SingleArgs single;  // the prepared scan-kernel arguments (for the fallback points)
};
bool tree_eligible(uint64_t n_verts, uint64_t n_pts, bool forced);
size_t tree_scratch_bytes(uint64_t n_verts, uint64_t n_edges, uint64_t n_pts);
cudaError_t launch_tree(const TreeArgs& a, void* scratch, cudaStream_t st, int dev, uint64_t* launches);
// the two halves of launch_tree: the build (polygon only) and the query (points);
// the query phase must follow the build phase on the same scratch
constexpr int kTreeBuild = 1, kTreeQuery = 2;
cudaError_t launch_tree_phase(const TreeArgs& a, void* scratch, cudaStream_t st, int dev, uint64_t* launches,
                              int phase);

// GPU results-CSV writer (pip_emit.cu): recs = n 32-byte records
// (pc_result_record); out gets the header and the rows (at most cap bytes
// written), *out_len (device) the full length; scratch = emit_scratch_bytes(n).
uint64_t emit_tiles(uint64_t n);
uint64_t emit_scratch_bytes(uint64_t n);
uint64_t emit_max_bytes(uint64_t n);
cudaError_t launch_emit_results(const void* recs, uint64_t n, char* out, uint64_t cap, void* scratch,
                                unsigned long long* out_len, cudaStream_t st, uint64_t* launches);

// y-ordering of the points of one polygon (pip_sort.cu): a stable 2-pass
// radix sort of (16-bit y key over the outer ring's bbox, point, index); points the
// bbox prefilter rejects sort last and are not classified.
struct BucketArgs {
    const double* pts;                    // n interleaved points
    uint64_t n;                           // < 2^32
    const unsigned long long* bbox_keys;  // from prep
    int prefilter;
    void* scratch;                        // bucket_scratch_bytes(n)
    double* sorted_pts;                   // n points in y order
    uint32_t* sorted_idx;                 // n: original index of each point in y order
    uint32_t* n_in;                       // (device) number of points not rejected
};
size_t bucket_scratch_bytes(uint64_t n);
cudaError_t launch_bucket(const BucketArgs& a, cudaStream_t st, int dev, uint64_t* launches);
// ORs the set bits of the bucketed planes back to the original point order.
cudaError_t launch_unbucket(uint64_t n, const uint32_t* n_dev, const uint32_t* sorted_idx, const uint32_t* s_inside,
                            const uint32_t* s_aux, uint32_t* inside_bits, uint32_t* aux_bits, cudaStream_t st, int dev,
                            uint64_t* launches);

// The literal binary64 checker path (pip_exact.cu, PC_OPT_EXACT): writes every
// word of both planes; box_scratch = 4 doubles of device memory (prefilter).
cudaError_t launch_exact_single(const double* pts, uint64_t n, const double* vx, const double* vy,
                                const uint64_t* ring_off, uint32_t n_rings, int prefilter, double* box_scratch,
                                int mode, double tol, uint32_t* inside_bits, uint32_t* aux_bits, cudaStream_t st,
                                uint64_t* launches);
cudaError_t launch_exact_csr(const CsrArgs& a, uint64_t n_points, cudaStream_t st, uint64_t* launches);

// bbox_of (batch.hpp:121-133) of the outer ring into box[4] (one CTA).
cudaError_t launch_outer_bbox(const double* vx, const double* vy, const uint64_t* ring_off, double* box,
                              cudaStream_t st, uint64_t* launches);

// Small calls (pip_small.cu): a CTA per point over all edges.  classify (counts
// == nullptr): out = small_out_bytes(n) zeroed bytes -> verdicts | inside |
// aux | stats; box = outer bbox (prefilter) or nullptr.  count (counts != nullptr,
// ring_off = {0, nv}, n_rings = 1, mode C1/C2): counts[i] = crossings, or the
// first degenerate edge's index where degen[i] = 1.
size_t small_out_bytes(uint64_t n);
cudaError_t launch_small(const double* pts, uint64_t n, const double* vx, const double* vy, const uint64_t* ring_off,
                         uint32_t n_rings, const double* box, int mode, double tol, void* out,
                         unsigned long long* counts, uint8_t* degen, cudaStream_t st, uint64_t* launches);

cudaError_t launch_fp64_probe(double* out, int iters, int dev, cudaStream_t st, double* flops);

} // namespace pcd
