/* polycast_cuda.h — C-ABI of libpolycast_cuda.so, the B200 (sm_100a) batched
 * point-in-polygon engine.
 *
 * This is the drop-in boundary of SURVEY.md §8(b).  The reference (polycast,
 * header-only C++20) has no FFI: its hot path is the C++ call
 *     classify_batch(const PointBatch&, const Polygon&, CrossingMode,
 *                    size_t workers = 0, double boundary_tol = 1e-12)
 *     (/root/reference/proj/include/polycast/batch.hpp:184-186)
 * which runs contains() (geometry.hpp:281-300) -> count_crossings_c1/_c2 /
 * robust_ray_crossings (geometry.hpp:182-273) per point.  The entry points
 * below replace that call below the C++ types; include/polycast/*.hpp keeps
 * the reference's public C++ API on top of them.
 *
 * Conventions
 *  - Plain pointers and sizes only; no exceptions cross this boundary.
 *  - Status codes: PC_OK, PC_EINVAL, PC_ECUDA, PC_ENOMEM, PC_ENCCL; the message
 *    of the last failure of a context is returned by pc_last_error().
 *  - mode: 0 = C1, 1 = C2, 2 = Robust  (CrossingMode order, geometry.hpp:107).
 *  - Verdict bytes: 0 Inside, 1 Outside, 2 Boundary, 3 Error (batch.hpp:60).
 *  - stats[4] = {inside, outside, boundary, error} (BatchStats, batch.hpp:81-109).
 *  - Points: interleaved x,y doubles (== reference Point2[], 16 B each).
 *  - Polygons: SoA vertex arrays vx[], vy[] holding closed rings (first vertex
 *    repeated at the end, as the reference Ring stores it, geometry.hpp:41-60);
 *    ring r spans vertices [ring_off[r], ring_off[r+1]); ring 0 is the outer
 *    ring, the rest are holes, combined by even-odd parity (geometry.hpp:281-300).
 *  - Bit planes: bit (i % 32) of word i/32 belongs to point i.  inside_bits
 *    marks Inside verdicts; aux_bits marks Error (C2) or Boundary (Robust).
 *  - Host buffers are borrowed for the duration of a synchronous call (pinned
 *    buffers make the copies faster but are not required).  Inputs are not
 *    validated for finiteness (the C++ types do that, SURVEY §8 rule P9).
 *  - Results are bit-identical to the reference CPU implementation for every
 *    mode, input and device count (IEEE binary64, round-to-nearest, no FMA
 *    contraction, the reference's expression order).
 *  - A context serialises its own use; concurrent callers use separate contexts.
 *  - There is no CPU fallback: with no usable GPU, pc_create fails.
 */
#ifndef POLYCAST_CUDA_H
#define POLYCAST_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PC_OK 0
#define PC_EINVAL 1
#define PC_ECUDA 2
#define PC_ENOMEM 3
#define PC_ENCCL 4

#define PC_MODE_C1 0
#define PC_MODE_C2 1
#define PC_MODE_ROBUST 2

#define PC_INSIDE 0
#define PC_OUTSIDE 1
#define PC_BOUNDARY 2
#define PC_ERROR 3

typedef struct pc_ctx pc_ctx;

/* Creates a context over GPUs 0..num_gpus-1 (num_gpus = 0: all visible).
 * Replaces the reference's std::thread worker pool (batch.hpp:172-175,
 * :212-229): points are sharded contiguously across the context's GPUs. */
int pc_create(pc_ctx** out, int num_gpus);
/* Creates a context over an explicit device list (e.g. one rank's LOCAL_RANK). */
int pc_create_devices(pc_ctx** out, const int* device_ids, int n);
void pc_destroy(pc_ctx* ctx);
const char* pc_last_error(const pc_ctx* ctx);
int pc_device_count(const pc_ctx* ctx);
/* Library version string. */
const char* pc_version(void);

/* Batched classification of n points against one polygon; replaces
 * classify_batch (batch.hpp:184-230) when bbox_prefilter = 1 and per-point
 * contains() (geometry.hpp:281-300) when bbox_prefilter = 0.
 * Every output pointer is optional (NULL = not wanted); inside_bits/aux_bits
 * hold ceil(n/32) words, verdicts n bytes, stats 4 counters. */
int pc_classify(pc_ctx* ctx, const double* pts_xy, uint64_t n, const double* vx, const double* vy,
                const uint64_t* ring_off, uint32_t n_rings, int mode, double boundary_tol,
                int bbox_prefilter, uint8_t* verdicts, uint32_t* inside_bits, uint32_t* aux_bits,
                uint64_t stats[4]);

/* Multi-polygon CSR batch: polygon p owns points
 * [pt_off[p], pt_off[p+1]) and rings [poly_ring_off[p], poly_ring_off[p+1]);
 * each polygon is classified with classify_batch semantics (bbox of its outer
 * ring, closed interval).  Polygons are sharded across the context's GPUs. */
int pc_classify_csr(pc_ctx* ctx, const double* pts_xy, const uint64_t* pt_off, uint64_t n_polys,
                    const double* vx, const double* vy, const uint64_t* ring_off,
                    const uint64_t* poly_ring_off, int mode, double boundary_tol,
                    uint8_t* verdicts, uint32_t* inside_bits, uint32_t* aux_bits,
                    uint64_t stats[4]);

/* count_crossings_c1 (mode 0) / count_crossings_c2 (mode 1) of one closed
 * ring of nv vertices for n points (geometry.hpp:182-229).  counts[i] is the
 * crossing count; degenerate[i] = 1 where the reference throws DegenerateEdge
 * (C2, horizontal edge on the ray), and counts[i] is then the index of the
 * first such edge (the index in the reference's message, geometry.hpp:219). */
int pc_count_crossings(pc_ctx* ctx, const double* pts_xy, uint64_t n, const double* vx,
                       const double* vy, uint64_t nv, int mode, uint64_t* counts,
                       uint8_t* degenerate);

/* Device-pointer variants on the context's GPU `dev_index`, enqueued on
 * `stream` (a cudaStream_t; NULL = the context's stream) and NOT synchronised
 * (the opt-in segment-tree path of pc_classify_dev waits on the stream twice
 * for sizes it needs on the host).  d_pts_xy must be 16-byte aligned (the
 * kernels load points as double2; cudaMalloc memory always is).
 * d_inside_bits / d_aux_bits (ceil(n/32) words) and d_stats (4 x u64) are
 * required; d_verdicts is optional.  Repeated identical calls replay a
 * captured CUDA graph (PC_OPT_GRAPH).  Used for kernel-only timing and by
 * callers that keep their data resident in HBM. */
int pc_classify_dev(pc_ctx* ctx, int dev_index, void* stream, const double* d_pts_xy, uint64_t n,
                    const double* d_vx, const double* d_vy, const uint64_t* d_ring_off,
                    uint32_t n_rings, uint64_t n_verts, int mode, double boundary_tol,
                    int bbox_prefilter, uint8_t* d_verdicts, uint32_t* d_inside_bits,
                    uint32_t* d_aux_bits, uint64_t* d_stats);

int pc_classify_csr_dev(pc_ctx* ctx, int dev_index, void* stream, const double* d_pts_xy,
                        const uint64_t* d_pt_off, uint64_t n_polys, uint64_t n_points,
                        const double* d_vx, const double* d_vy, const uint64_t* d_ring_off,
                        const uint64_t* d_poly_ring_off, int mode, double boundary_tol,
                        uint8_t* d_verdicts, uint32_t* d_inside_bits, uint32_t* d_aux_bits,
                        uint64_t* d_stats);

/* prefilter_bbox (batch.hpp:137-153) on the GPU: the points of pts_xy[n]
 * inside the closed box {min_x, min_y, max_x, max_y} (BBox::contains,
 * batch.hpp:39-41), in input order, to out_xy (capacity n points) with their
 * original indices to out_idx (capacity n); *n_inside = how many.  The
 * outside count is n - *n_inside.  PC_EINVAL if min > max on an axis (the
 * BBox constructor's check, batch.hpp:32-36) or a needed pointer is NULL. */
int pc_prefilter_bbox(pc_ctx* ctx, const double* pts_xy, uint64_t n, const double box[4], double* out_xy,
                      uint64_t* out_idx, uint64_t* n_inside);

/* scatter_verdicts (batch.hpp:157-168) on the GPU: out[n_total] = Outside,
 * then out[idx[k]] = inbox_verdicts[k] for k < n_inbox.  PC_EINVAL if
 * n_inbox > n_total (the reference's size check) or an index is >= n_total. */
int pc_scatter_verdicts(pc_ctx* ctx, const uint64_t* idx, const uint8_t* inbox_verdicts, uint64_t n_inbox,
                        uint64_t n_total, uint8_t* out);

/* Device-pointer variants (not synchronised).  d_n_inside receives the count
 * (one u64 in device memory); d_bad (one u32, zeroed by the caller) is set
 * to non-zero when an index is out of range. */
int pc_prefilter_bbox_dev(pc_ctx* ctx, int dev_index, void* stream, const double* d_pts_xy, uint64_t n,
                          const double box[4], double* d_out_xy, uint64_t* d_out_idx, uint64_t* d_n_inside);
int pc_scatter_verdicts_dev(pc_ctx* ctx, int dev_index, void* stream, const uint64_t* d_idx,
                            const uint8_t* d_inbox_verdicts, uint64_t n_inbox, uint64_t n_total,
                            uint8_t* d_out, uint32_t* d_bad);

/* The data-row loop of read_points_csv (io.hpp:148-225) on GPU 0 of the
 * context: text[len] is the file's bytes; lines split at '\n' (a trailing
 * '\r' is removed, empty lines skipped); lines starting before byte
 * data_start (the header and the empty lines before it) are not data rows.
 * Each data row is split at `delim` and cells x_col / y_col are parsed as the
 * reference's parse_double does (one pair of surrounding quotes and
 * spaces/tabs stripped, then a correctly rounded, finite binary64).  Good rows
 * are written to out_xy in file order, *n_points of them; *n_bad counts the
 * rows that have too few cells or a cell that is not a finite number (the rows
 * lenient mode skips), *first_bad_offset is the byte offset of the first such
 * row's line (UINT64_MAX if none) -- strict mode reports it -- with
 * *first_bad_kind = 2 (too few cells), 3 (x cell) or 4 (y cell).  If
 * cap_points < *n_points, nothing is copied and PC_EINVAL is returned with
 * *n_points set.  x_col == y_col is PC_EINVAL (io.hpp:149-156). */
int pc_parse_points_csv(pc_ctx* ctx, const char* text, uint64_t len, uint64_t data_start, uint32_t x_col,
                        uint32_t y_col, char delim, double* out_xy, uint64_t cap_points, uint64_t* n_points,
                        uint64_t* n_bad, uint64_t* first_bad_offset, uint32_t* first_bad_kind);

/* Device-pointer variant (not synchronised): d_text in device memory, points
 * to d_out_xy (at most cap_points written); d_result = 4 x u64 in device
 * memory: [0] good rows (may exceed cap_points), [1] bad rows, [2] first bad
 * row as (line offset << 3 | kind) or UINT64_MAX, [3] scratch.  One kernel. */
int pc_parse_points_csv_dev(pc_ctx* ctx, int dev_index, void* stream, const char* d_text, uint64_t len,
                            uint64_t data_start, uint32_t x_col, uint32_t y_col, char delim, double* d_out_xy,
                            uint64_t cap_points, uint64_t* d_result);

/* One row of write_results_csv (io.hpp:312-322): layout-compatible with
 * polycast::ResultRecord (32 bytes; verdict = PC_INSIDE .. PC_ERROR). */
typedef struct pc_result_record {
    uint64_t index;
    double x;
    double y;
    uint8_t verdict;
    uint8_t pad[7];
} pc_result_record;

/* The text write_results_csv (io.hpp:325-335) puts in its file, on GPU 0:
 * "index,x,y,verdict\n" and one "index,x,y,verdict\n" row per record, x and y
 * as printf("%.17g") prints them (byte-identical; every finite double reads
 * back exactly), verdict as to_string(Verdict) (batch.hpp:71-79).  *len = the
 * text's length; if cap < *len nothing is copied and PC_EINVAL is returned
 * (18 + 80 n bytes always suffice). */
int pc_format_results_csv(pc_ctx* ctx, const pc_result_record* recs, uint64_t n, char* out, uint64_t cap,
                          uint64_t* len);

/* Device-pointer variant (not synchronised): at most cap bytes to d_out,
 * the full length to d_len (one u64 in device memory). */
int pc_format_results_csv_dev(pc_ctx* ctx, int dev_index, void* stream, const pc_result_record* d_recs, uint64_t n,
                              char* d_out, uint64_t cap, uint64_t* d_len);

/* Number of GPU kernels the last call on this context launched (all devices). */
uint64_t pc_last_launch_count(const pc_ctx* ctx);

/* Tuning options (none changes any result).
 *  PC_OPT_BUCKET_POINTS: -1 auto (default), 0 off, 1 on — y-bucket the points of
 *  a single-polygon call before classifying, for SIMT coherence (pip_sort.cu). */
#define PC_OPT_BUCKET_POINTS 1
/*  PC_OPT_TREE: 0 off (default; -1 means the default), 1 on — an opt-in
 *  extension OUTSIDE the reference's linear scan: C1/C2 single
 *  polygons count a point's crossings through a segment tree over the
 *  vertices' y-order (pip_tree.cu) instead of scanning the edges.  Never used
 *  by the headline measurement. */
#define PC_OPT_TREE 2
/*  PC_OPT_EXACT: 0 off (default), 1 on — run only the literal binary64 loop of
 *  the reference (pip_exact.cu: thread per point, every edge, __dadd_rn /
 *  __dmul_rn in the reference's order; no filter keys, no fp32 certification,
 *  no bucketing, no tree).  A checker for the fast path on full-size inputs;
 *  results are identical by construction of the fast path. */
#define PC_OPT_EXACT 3
/*  PC_OPT_GRAPH: 1 on (default), 0 off — a device-pointer call (pc_classify_dev,
 *  pc_classify_csr_dev) repeated with identical arguments is captured once as
 *  a CUDA graph and replayed (one launch for the call's kernels and memsets).
 *  Not used while profiling (pc_set_profiling) or with PC_OPT_TREE. */
#define PC_OPT_GRAPH 4
int pc_set_option(pc_ctx* ctx, int option, int64_t value);

/* Measurement hooks (bench.py).  With profiling on, every call records a pair
 * of CUDA events around its main classify kernel(s), on the stream they are
 * launched on (the segment-tree path: the build and the query, reported as one
 * duration).  pc_profile_take() waits for the pairs recorded on device
 * `dev_index` since the previous take, writes up to `cap` kernel durations
 * (ms) to ms_out, clears them and returns how many there were. */
int pc_set_profiling(pc_ctx* ctx, int on);
int pc_profile_take(pc_ctx* ctx, int dev_index, double* ms_out, int cap);

/* Runs an FP64 add/multiply throughput probe (no FMA: the instruction mix of
 * the crossing test) on device `dev_index` for about `ms` milliseconds and
 * returns the achieved rate in FP64 operations per second. */
int pc_measure_fp64_rate(pc_ctx* ctx, int dev_index, double ms, double* flops_per_s);

#ifdef __cplusplus
}
#endif

#endif /* POLYCAST_CUDA_H */
