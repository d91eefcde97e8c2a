// GPU points-CSV reader: the data-row loop of the
// reference's read_points_csv (io.hpp:148-225) on the device.  The host reads
// the file bytes, resolves the header / column names (io.hpp:126-140, cheap)
// and composes error messages; the GPU finds the lines, splits the cells and
// parses the two coordinates of every row with the correctly rounded parser
// of pip_parse.cuh (the reference's from_chars + isfinite), and writes the
// good rows in file order.
//
// One pass, one launch (csv_points_kernel), the text read from HBM once:
//   * the text is cut into kTile-byte tiles; a line belongs to the tile that
//     holds its first byte.  A CTA stages its tile (plus kSpill bytes of the
//     next one, where its last line usually ends) in shared memory;
//   * line starts: each thread scans 32 contiguous staged bytes for '\n'
//     (4-byte SIMD compares), a block scan orders them;
//   * thread per line: '\r' strip, empty-line skip (getline loop, io.hpp:
//     166-172), split at the delimiter (split_line: no quoting rules), strip
//     one pair of quotes and spaces/tabs and parse x and y (parse_double);
//   * the good rows of the tile are compacted in order into shared memory;
//     the tile's offset in the output comes from a decoupled look-back over
//     the tiles before it (tiles are numbered in launch order by an atomic
//     counter, so every predecessor is resident or done); then one coalesced
//     16-byte store per point.
// Bad rows (too few cells, x or y not a finite number) are counted and the
// first one reported as (byte offset of its line << 3 | kind).
#include "pip_kernels.h"

#include <cuda_runtime.h>

#include <algorithm>

#include "pip_parse.cuh"

namespace pcd {

namespace {

constexpr int kT = 256;         // threads per CTA
constexpr int kTile = 8192;     // text bytes per tile (32 per thread)
constexpr int kSpill = 512;     // staged bytes past the tile
constexpr int kStage = kTile + kSpill;
constexpr unsigned kSlot = 512;   // good rows a tile keeps from pass 1 (a tile of short rows is parsed again)
constexpr unsigned kFullMask = 0xffffffffu;

struct CsvSmem {
    uint16_t starts[kTile];
    char text[kStage];
    uint32_t dmask[kStage / 32]; // bit b of word k: staged byte 32 k + b is the delimiter
    unsigned wsum[kT / 32];
    unsigned long long scratch[2];
};

// parse_double's cell preparation (io.hpp:111-119): one pair of surrounding
// quotes, then spaces / tabs on both ends
__device__ __forceinline__ bool parse_cell(const char* c, int n, double* out) {
    if (n >= 2 && c[0] == '"' && c[n - 1] == '"') {
        ++c;
        n -= 2;
    }
    while (n > 0 && (c[0] == ' ' || c[0] == '\t')) {
        ++c;
        --n;
    }
    while (n > 0 && (c[n - 1] == ' ' || c[n - 1] == '\t')) --n;
    if (n == 0) return false;
    return parse::parse_f64(c, n, out);
}

// status of one line: 0 not a row (empty), 1 ok, 2 too few cells, 3 x bad, 4 y bad
__device__ __forceinline__ int parse_row(const char* s, uint64_t n, uint32_t x_idx, uint32_t y_idx, char delim,
                                         double2& p) {
    if (n > 0 && s[n - 1] == '\r') --n; // getline + '\r' strip (io.hpp:171)
    if (n == 0) return 0;
    const uint32_t need = max(x_idx, y_idx);
    uint32_t cell = 0;
    uint64_t cs = 0, xs = 0, xe = 0, ys = 0, ye = 0;
    bool hx = false, hy = false;
    for (uint64_t i = 0; i <= n; ++i) {
        if (i == n || s[i] == delim) {
            if (cell == x_idx) {
                xs = cs;
                xe = i;
                hx = true;
            }
            if (cell == y_idx) {
                ys = cs;
                ye = i;
                hy = true;
            }
            if (++cell > need) break;
            cs = i + 1;
        }
    }
    if (!hx || !hy) return 2;
    if (!parse_cell(s + xs, (int)min(xe - xs, (uint64_t)(1u << 30)), &p.x)) return 3;
    if (!parse_cell(s + ys, (int)min(ye - ys, (uint64_t)(1u << 30)), &p.y)) return 4;
    return 1;
}

// parse_row for a line staged in shared memory: cells from the delimiter
// bit mask instead of a byte loop
__device__ __forceinline__ int parse_row_staged(const char* text, const uint32_t* dmask, uint32_t s, uint32_t e,
                                                uint32_t x_idx, uint32_t y_idx, double2& p) {
    if (e > s && text[e - 1] == '\r') --e;
    if (e == s) return 0;
    const uint32_t need = max(x_idx, y_idx);
    uint32_t cell = 0, cs = s, xs = 0, xe = 0, ys = 0, ye = 0;
    bool hx = false, hy = false, done = false;
    for (uint32_t wi = s >> 5; wi <= (e - 1) >> 5 && !done; ++wi) {
        uint32_t m = dmask[wi];
        if (wi == s >> 5) m &= ~0u << (s & 31);
        if (wi == (e - 1) >> 5 && (e & 31)) m &= ~(~0u << (e & 31));
        while (m) {
            const uint32_t q = wi * 32 + __ffs(m) - 1;
            m &= m - 1;
            if (cell == x_idx) {
                xs = cs;
                xe = q;
                hx = true;
            }
            if (cell == y_idx) {
                ys = cs;
                ye = q;
                hy = true;
            }
            cs = q + 1;
            if (++cell > need) {
                done = true;
                break;
            }
        }
    }
    if (!done) { // the last cell runs to the end of the line
        if (cell == x_idx) {
            xs = cs;
            xe = e;
            hx = true;
        }
        if (cell == y_idx) {
            ys = cs;
            ye = e;
            hy = true;
        }
    }
    if (!hx || !hy) return 2;
    if (!parse_cell(text + xs, (int)(xe - xs), &p.x)) return 3;
    if (!parse_cell(text + ys, (int)(ye - ys), &p.y)) return 4;
    return 1;
}

// block-wide exclusive scan of one unsigned per thread; the total in `total`
__device__ __forceinline__ unsigned block_scan(unsigned v, unsigned* wsum, unsigned& total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(kFullMask, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    unsigned before = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < kT / 32; ++k) {
        const unsigned c = wsum[k];
        before += k < w ? c : 0u;
        tot += c;
    }
    __syncthreads(); // wsum is reused
    total = tot;
    return before + incl - v;
}

// One tile: stage it, find its data lines, parse them (thread per line) and
// hand every good row to sink(k, p) with k its rank among the tile's good rows
// (file order).  Returns the number of good rows; bad rows are counted in
// n_bad / first_bad of thread 0..kT-1 (each thread its own lines).
template <class Sink>
__device__ __forceinline__ unsigned parse_tile(CsvSmem& sm, const char* __restrict__ text, uint64_t len,
                                               uint64_t tile, uint64_t data_start, uint32_t x_idx, uint32_t y_idx,
                                               char delim, bool aligned, unsigned& n_bad,
                                               unsigned long long& first_bad, Sink sink) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint64_t base = tile * kTile;
    const uint64_t staged = min((uint64_t)kStage, len - base);
    const uint64_t tile_len = min((uint64_t)kTile, len - base);

    // ---- stage the tile (+ spill) in shared memory --------------------------------
    if (aligned && staged == kStage) {
        const uint4* src = reinterpret_cast<const uint4*>(text + base);
        uint4* dst = reinterpret_cast<uint4*>(sm.text);
        for (int i = tid; i < kStage / 16; i += kT) dst[i] = __ldg(src + i);
    } else {
        for (uint64_t i = tid; i < staged; i += kT) sm.text[i] = text[base + i];
        for (uint64_t i = staged + tid; i < kStage; i += kT) sm.text[i] = 0;
    }
    __syncthreads();

    // ---- line starts and delimiter masks: thread t scans bytes [32 t, 32 t + 32) ----
    // A line starts at 0 (file start) or after a '\n'; it is a data line if it
    // starts at or after data_start and before len.
    const uint32_t dd = 0x01010101u * (uint8_t)delim;
    auto masks = [&](const char* p, uint32_t* nl) { // 32 bytes -> delimiter bit mask (+ '\n' bytes per word)
        const uint4* t4 = reinterpret_cast<const uint4*>(p);
        const uint4 a = t4[0], b = t4[1];
        const uint32_t wv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        uint32_t dm = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (nl) nl[k] = __vcmpeq4(wv[k], 0x0a0a0a0au) & 0x80808080u;
            const uint32_t q = __vcmpeq4(wv[k], dd) & 0x80808080u;
            dm |= (((q >> 7) | (q >> 14) | (q >> 21) | (q >> 28)) & 0xfu) << (4 * k);
        }
        return dm;
    };
    uint32_t nlm[8]; // per word: 0x80 in each byte that is '\n'
    sm.dmask[tid] = masks(sm.text + tid * 32, nlm);
    if (tid < kSpill / 32) sm.dmask[kTile / 32 + tid] = masks(sm.text + kTile + tid * 32, nullptr);
    auto is_start = [&](uint64_t rel) { // rel: tile-relative start candidate
        const uint64_t g = base + rel;
        return rel < tile_len && g < len && g >= data_start;
    };
    unsigned cnt = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        uint32_t m = nlm[k];
        while (m) {
            const int b = (__ffs(m) - 1) >> 3;
            m &= m - 1;
            cnt += is_start((uint64_t)tid * 32 + k * 4 + b + 1);
        }
    }
    // a line starting at the tile's first byte: the file start, or a '\n' ending the previous tile
    const bool first = tid == 0 && is_start(0) && (base == 0 || text[base - 1] == '\n');
    cnt += first;
    unsigned n_lines;
    unsigned pos = block_scan(cnt, sm.wsum, n_lines);
    if (first) sm.starts[pos++] = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        uint32_t m = nlm[k];
        while (m) {
            const int b = (__ffs(m) - 1) >> 3;
            m &= m - 1;
            const uint64_t rel = (uint64_t)tid * 32 + k * 4 + b + 1;
            if (is_start(rel)) sm.starts[pos++] = (uint16_t)rel;
        }
    }
    __syncthreads();

    // ---- thread per line; good rows ranked in file order with ballots ---------------
    unsigned n_ok = 0;
    for (unsigned r0 = 0; r0 < n_lines; r0 += kT) {
        const unsigned i = r0 + tid;
        int st = 0;
        double2 p = make_double2(0.0, 0.0);
        if (i < n_lines) {
            const uint64_t s = sm.starts[i];
            uint64_t e; // tile-relative end (exclusive) of the line before its '\n'
            if (i + 1 < n_lines) {
                e = sm.starts[i + 1] - 1;
            } else { // the tile's last line: search for its end
                e = s;
                const uint64_t lim = len - base;
                while (e < staged && sm.text[e] != '\n') ++e;
                if (e == staged)
                    while (e < lim && text[base + e] != '\n') ++e;
            }
            st = e <= staged ? parse_row_staged(sm.text, sm.dmask, (uint32_t)s, (uint32_t)e, x_idx, y_idx, p)
                             : parse_row(text + base + s, e - s, x_idx, y_idx, delim, p);
            if (st >= 2) {
                ++n_bad;
                first_bad = min(first_bad, ((base + s) << 3) | (unsigned long long)st);
            }
        }
        const unsigned b = __ballot_sync(kFullMask, st == 1);
        if (lane == 0) sm.wsum[w] = __popc(b);
        __syncthreads();
        unsigned before = 0, tot = 0;
#pragma unroll
        for (int k = 0; k < kT / 32; ++k) {
            const unsigned c = sm.wsum[k];
            before += k < w ? c : 0u;
            tot += c;
        }
        if (st == 1) sink(n_ok + before + __popc(b & ((1u << lane) - 1u)), p);
        n_ok += tot;
        __syncthreads();
    }
    return n_ok;
}

// pass 1: CTA per tile; the first kSlot good rows go to the tile's slot in
// `slots`, the count to counts[tile]; bad rows to res[1] / res[2]
__global__ void __launch_bounds__(kT) csv_parse_kernel(const char* __restrict__ text, uint64_t len,
                                                       uint64_t data_start, uint32_t x_idx, uint32_t y_idx,
                                                       char delim, double2* __restrict__ slots,
                                                       unsigned* __restrict__ counts,
                                                       unsigned long long* __restrict__ res, bool aligned) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    CsvSmem& sm = *reinterpret_cast<CsvSmem*>(smem_raw);
    const uint64_t tile = blockIdx.x;
    unsigned n_bad = 0;
    unsigned long long first_bad = ~0ull;
    double2* slot = slots + tile * kSlot;
    const unsigned n_ok = parse_tile(sm, text, len, tile, data_start, x_idx, y_idx, delim, aligned, n_bad, first_bad,
                                     [&](unsigned k, double2 p) {
                                         if (k < kSlot) slot[k] = p;
                                     });
    if (threadIdx.x == 0) counts[tile] = n_ok;
    n_bad = __reduce_add_sync(kFullMask, n_bad);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) first_bad = min(first_bad, __shfl_xor_sync(kFullMask, first_bad, o));
    if ((threadIdx.x & 31) == 0 && n_bad) {
        atomicAdd(res + 1, (unsigned long long)n_bad);
        atomicMin(res + 2, first_bad);
    }
}

// pass 2: exclusive scan of the tile counts (one CTA) -> offs[], total -> res[0]
__global__ void __launch_bounds__(1024) csv_scan_kernel(const unsigned* __restrict__ counts, uint64_t n,
                                                        unsigned long long* __restrict__ offs,
                                                        unsigned long long* __restrict__ res) {
    __shared__ unsigned long long ws[32];
    __shared__ unsigned long long carry;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint64_t b0 = 0; b0 < n; b0 += 1024) {
        const uint64_t j = b0 + threadIdx.x;
        const unsigned long long v = j < n ? counts[j] : 0ull;
        unsigned long long incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(kFullMask, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) ws[w] = incl;
        __syncthreads();
        if (w == 0) {
            unsigned long long t = ws[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(kFullMask, t, o);
                if (lane >= o) t += y;
            }
            ws[lane] = t;
        }
        __syncthreads();
        const unsigned long long c0 = carry;
        if (j < n) offs[j] = c0 + incl - v + (w ? ws[w - 1] : 0ull);
        __syncthreads();
        if (threadIdx.x == 1023) carry = c0 + ws[31];
        __syncthreads();
    }
    if (threadIdx.x == 0) res[0] = carry;
}

// pass 3: CTA per tile; copy its slot to the output, or parse the tile again
// when it has more good rows than a slot holds
__global__ void __launch_bounds__(kT) csv_emit_kernel(const char* __restrict__ text, uint64_t len,
                                                      uint64_t data_start, uint32_t x_idx, uint32_t y_idx,
                                                      char delim, const double2* __restrict__ slots,
                                                      const unsigned* __restrict__ counts,
                                                      const unsigned long long* __restrict__ offs,
                                                      double2* __restrict__ out, uint64_t cap, bool aligned) {
    const uint64_t tile = blockIdx.x;
    const unsigned n = counts[tile];
    const uint64_t off = offs[tile];
    if (n <= kSlot) {
        const double2* slot = slots + tile * kSlot;
        for (unsigned k = threadIdx.x; k < n; k += kT)
            if (off + k < cap) out[off + k] = slot[k];
        return;
    }
    extern __shared__ __align__(16) unsigned char smem_raw[];
    CsvSmem& sm = *reinterpret_cast<CsvSmem*>(smem_raw);
    unsigned n_bad = 0;
    unsigned long long first_bad = ~0ull;
    parse_tile(sm, text, len, tile, data_start, x_idx, y_idx, delim, aligned, n_bad, first_bad,
               [&](unsigned k, double2 p) {
                   if (off + k < cap) out[off + k] = p;
               });
}

} // namespace

uint64_t csv_tiles(uint64_t len) { return (len + kTile - 1) / kTile; }
uint64_t csv_scratch_bytes(uint64_t len) { return csv_tiles(len) * (kSlot * 16ull + 4 + 8) + 64; }

cudaError_t launch_csv_points(const char* text, uint64_t len, uint64_t data_start, uint32_t x_idx, uint32_t y_idx,
                              char delim, double* out, uint64_t cap, void* scratch, unsigned long long* res,
                              cudaStream_t st, uint64_t* launches) {
    const uint64_t n_tiles = csv_tiles(len);
    cudaError_t e = cudaMemsetAsync(res, 0, 4 * sizeof(unsigned long long), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(res + 2, 0xff, sizeof(unsigned long long), st);
    if (e != cudaSuccess || n_tiles == 0) return e;
    for (const void* f : {(const void*)csv_parse_kernel, (const void*)csv_emit_kernel}) {
        e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(CsvSmem));
        if (e != cudaSuccess) return e;
    }
    double2* slots = static_cast<double2*>(scratch);
    unsigned long long* offs = reinterpret_cast<unsigned long long*>(slots + n_tiles * kSlot);
    unsigned* counts = reinterpret_cast<unsigned*>(offs + n_tiles);
    const bool aligned = (reinterpret_cast<uintptr_t>(text) & 15) == 0;
    csv_parse_kernel<<<(unsigned)n_tiles, kT, sizeof(CsvSmem), st>>>(text, len, data_start, x_idx, y_idx, delim,
                                                                    slots, counts, res, aligned);
    csv_scan_kernel<<<1, 1024, 0, st>>>(counts, n_tiles, offs, res);
    csv_emit_kernel<<<(unsigned)n_tiles, kT, sizeof(CsvSmem), st>>>(text, len, data_start, x_idx, y_idx, delim,
                                                                   slots, counts, offs,
                                                                   reinterpret_cast<double2*>(out), cap, aligned);
    *launches += 3;
    return cudaGetLastError();
}

} // namespace pcd
