// GPU results-CSV writer: the row loop of the
// reference's write_results_csv (io.hpp:312-335) on the device -- the text of
// "index,x,y,verdict\n" followed by one "index,x,y,verdict" row per record,
// coordinates in "%.17g" (pip_format.cuh: byte-identical to glibc, so every
// finite double round-trips), verdict names of to_string(Verdict)
// (batch.hpp:71-79).  The host writes the bytes to the file.
//
// Three launches:
//   format  CTA per tile of kT records: thread per record formats its row into
//           a shared-memory slot, a block scan of the row lengths packs the
//           tile's text in shared memory, coalesced 16-byte stores put it in
//           the tile's scratch slot; the tile's length to lens[tile];
//   scan    exclusive scan of the tile lengths (one CTA), the header bytes;
//   copy    CTA per tile: its text to the output at its offset (byte-wide,
//           coalesced).
#include "pip_kernels.h"

#include <cuda_runtime.h>

#include "pip_format.cuh"

namespace pcd {

namespace {

constexpr int kT = 256;
constexpr int kRowMax = 80; // 20 (index) + 24 + 24 (coordinates) + 8 (verdict) + 4 separators
constexpr int kTileBytes = kT * kRowMax;
constexpr unsigned kFullMask = 0xffffffffu;
__device__ __constant__ const char kHeader[] = "index,x,y,verdict\n";
constexpr int kHeaderLen = 18;

struct Rec { // polycast::ResultRecord / pc_result_record
    unsigned long long index;
    double x, y;
    unsigned char verdict, pad[7];
};

__device__ __forceinline__ int put_verdict(char* p, unsigned v) {
    const char* s = v == 0 ? "inside" : v == 1 ? "outside" : v == 2 ? "boundary" : v == 3 ? "error" : "?";
    int n = 0;
    while (s[n]) {
        p[n] = s[n];
        ++n;
    }
    return n;
}

struct EmitSmem {
    char rows[kTileBytes];         // row t at kRowMax * t
    __align__(16) char packed[kTileBytes + 16];
    unsigned wsum[kT / 32];
};

__global__ void __launch_bounds__(kT) emit_format_kernel(const Rec* __restrict__ recs, uint64_t n,
                                                         char* __restrict__ slots, unsigned* __restrict__ lens) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    EmitSmem& sm = *reinterpret_cast<EmitSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint64_t i = blockIdx.x * (uint64_t)kT + tid;
    int len = 0;
    char* row = sm.rows + kRowMax * tid;
    if (i < n) {
        const Rec r = recs[i];
        len = fmt::put_u64(row, r.index);
        row[len++] = ',';
        len += fmt::format_17g(r.x, row + len);
        row[len++] = ',';
        len += fmt::format_17g(r.y, row + len);
        row[len++] = ',';
        len += put_verdict(row + len, r.verdict);
        row[len++] = '\n';
    }
    // block scan of the row lengths
    unsigned incl = (unsigned)len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(kFullMask, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) sm.wsum[w] = incl;
    __syncthreads();
    unsigned before = 0, total = 0;
#pragma unroll
    for (int k = 0; k < kT / 32; ++k) {
        const unsigned c = sm.wsum[k];
        before += k < w ? c : 0u;
        total += c;
    }
    const unsigned at = before + incl - (unsigned)len;
    for (int k = 0; k < len; ++k) sm.packed[at + k] = row[k];
    __syncthreads();
    uint4* dst = reinterpret_cast<uint4*>(slots + blockIdx.x * (uint64_t)kTileBytes);
    const uint4* src = reinterpret_cast<const uint4*>(sm.packed);
    for (unsigned k = tid; k < (total + 15) / 16; k += kT) dst[k] = src[k];
    if (tid == 0) lens[blockIdx.x] = total;
}

// exclusive scan of the tile lengths -> offs (after the header), total -> *out_len; header bytes
__global__ void __launch_bounds__(1024) emit_scan_kernel(const unsigned* __restrict__ lens, uint64_t n_tiles,
                                                         unsigned long long* __restrict__ offs, char* __restrict__ out,
                                                         unsigned long long* __restrict__ out_len, uint64_t cap) {
    __shared__ unsigned long long ws[32];
    __shared__ unsigned long long carry;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = kHeaderLen;
    if (threadIdx.x < kHeaderLen && threadIdx.x < cap) out[threadIdx.x] = kHeader[threadIdx.x];
    __syncthreads();
    for (uint64_t b0 = 0; b0 < n_tiles; b0 += 1024) {
        const uint64_t j = b0 + threadIdx.x;
        const unsigned long long v = j < n_tiles ? lens[j] : 0ull;
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
        if (j < n_tiles) offs[j] = c0 + incl - v + (w ? ws[w - 1] : 0ull);
        __syncthreads();
        if (threadIdx.x == 1023) carry = c0 + ws[31];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out_len = carry;
}

__global__ void __launch_bounds__(kT) emit_copy_kernel(const char* __restrict__ slots,
                                                       const unsigned* __restrict__ lens,
                                                       const unsigned long long* __restrict__ offs,
                                                       char* __restrict__ out, uint64_t cap) {
    const unsigned len = lens[blockIdx.x];
    const uint64_t off = offs[blockIdx.x];
    const char* src = slots + blockIdx.x * (uint64_t)kTileBytes;
    if (off + len <= cap) {
        for (unsigned k = threadIdx.x; k < len; k += kT) out[off + k] = src[k];
    } else {
        for (unsigned k = threadIdx.x; k < len; k += kT)
            if (off + k < cap) out[off + k] = src[k];
    }
}

} // namespace

uint64_t emit_tiles(uint64_t n) { return (n + kT - 1) / kT; }
uint64_t emit_scratch_bytes(uint64_t n) { return emit_tiles(n) * ((uint64_t)kTileBytes + 4 + 8) + 64; }
uint64_t emit_max_bytes(uint64_t n) { return kHeaderLen + n * (uint64_t)kRowMax; }

cudaError_t launch_emit_results(const void* recs, uint64_t n, char* out, uint64_t cap, void* scratch,
                                unsigned long long* out_len, cudaStream_t st, uint64_t* launches) {
    const uint64_t n_tiles = emit_tiles(n);
    char* slots = static_cast<char*>(scratch);
    unsigned long long* offs = reinterpret_cast<unsigned long long*>(slots + n_tiles * (uint64_t)kTileBytes);
    unsigned* lens = reinterpret_cast<unsigned*>(offs + n_tiles);
    cudaError_t e = cudaSuccess;
    if (n_tiles) {
        e = cudaFuncSetAttribute(emit_format_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sizeof(EmitSmem));
        if (e != cudaSuccess) return e;
        emit_format_kernel<<<(unsigned)n_tiles, kT, sizeof(EmitSmem), st>>>(static_cast<const Rec*>(recs), n, slots,
                                                                           lens);
    }
    emit_scan_kernel<<<1, 1024, 0, st>>>(lens, n_tiles, offs, out, out_len, cap);
    if (n_tiles) emit_copy_kernel<<<(unsigned)n_tiles, kT, 0, st>>>(slots, lens, offs, out, cap);
    *launches += n_tiles ? 3 : 1;
    return cudaGetLastError();
}

} // namespace pcd
