// GPU points-CSV reader: the data-row loop of the
// reference's read_points_csv (io.hpp:148-225) on the device.  The host reads
// the file bytes, resolves the header / column names (io.hpp:126-140, cheap)
// and composes error messages; the GPU finds the lines, splits the cells and
// parses the two coordinates of every row with the correctly rounded parser
// of pip_parse.cuh (the reference's from_chars + isfinite), then compacts
// the good rows in file order.
//
// Launches (all byte- or line-parallel, HBM-bound):
//   nl_count   per block: '\n' bytes in its chunk
//   scan       exclusive scan of the block counts (one CTA)
//   nl_write   line end offsets, in order
//   rows       thread per line: '\r' strip, empty / header skip, split on the
//              delimiter (split_line: no quoting rules), strip one pair of
//              quotes and spaces/tabs (parse_double), parse x and y;
//              status per line, first failing line (atomicMin)
//   ok_count / scan / ok_write  order-preserving compaction of the good rows
#include "pip_kernels.h"

#include <cuda_runtime.h>

#include <algorithm>

#include "pip_parse.cuh"

namespace pcd {

namespace {

constexpr int kT = 512;
constexpr unsigned kFullMask = 0xffffffffu;

__global__ void __launch_bounds__(kT) nl_count_kernel(const char* __restrict__ text, uint64_t len, uint64_t chunk,
                                                      unsigned long long* __restrict__ blk) {
    const uint64_t lo = blockIdx.x * chunk, hi = min(len, lo + chunk);
    unsigned c = 0;
    for (uint64_t i = lo + threadIdx.x; i < hi; i += kT) c += text[i] == '\n';
    c = __reduce_add_sync(kFullMask, c);
    __shared__ unsigned ws[kT / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x < 32) {
        unsigned v = threadIdx.x < kT / 32 ? ws[threadIdx.x] : 0u;
        v = __reduce_add_sync(kFullMask, v);
        if (threadIdx.x == 0) blk[blockIdx.x] = v;
    }
}

// exclusive scan of blk[0 .. n) in place, blk[n] = total (one CTA)
__global__ void __launch_bounds__(1024) scan_kernel(unsigned long long* __restrict__ blk, int n) {
    __shared__ unsigned long long ws[32];
    __shared__ unsigned long long carry;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < n; base += 1024) {
        const int j = base + threadIdx.x;
        const unsigned long long v = j < n ? blk[j] : 0ull;
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
        if (j < n) blk[j] = c0 + incl - v + (w ? ws[w - 1] : 0ull);
        __syncthreads();
        if (threadIdx.x == 1023) carry = c0 + ws[31];
        __syncthreads();
    }
    if (threadIdx.x == 0) blk[n] = carry;
}

// positions of the '\n' bytes, in order (block b writes from base[b])
__global__ void __launch_bounds__(kT) nl_write_kernel(const char* __restrict__ text, uint64_t len, uint64_t chunk,
                                                      const unsigned long long* __restrict__ base,
                                                      unsigned long long* __restrict__ ends) {
    __shared__ unsigned wc[kT / 32];
    __shared__ unsigned long long run_s;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t lo = blockIdx.x * chunk, hi = min(len, lo + chunk);
    if (threadIdx.x == 0) run_s = base[blockIdx.x];
    __syncthreads();
    for (uint64_t i0 = lo; i0 < hi; i0 += kT) {
        const uint64_t i = i0 + threadIdx.x;
        const bool nl = i < hi && text[i] == '\n';
        const unsigned b = __ballot_sync(kFullMask, nl);
        if (lane == 0) wc[w] = __popc(b);
        __syncthreads();
        unsigned before = 0, total = 0;
#pragma unroll
        for (int k = 0; k < kT / 32; ++k) {
            const unsigned c = wc[k];
            before += k < w ? c : 0u;
            total += c;
        }
        const unsigned long long run = run_s;
        if (nl) ends[run + before + __popc(b & ((1u << lane) - 1u))] = i;
        __syncthreads();
        if (threadIdx.x == 0) run_s = run + total;
        __syncthreads();
    }
}

// parse_double's cell preparation (io.hpp:117-119): one pair of surrounding
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

// thread per line: status 0 = not a data row (empty / header / before it),
// 1 = ok, 2 = too few columns, 3 = x not a finite number, 4 = y not
__global__ void __launch_bounds__(256) rows_kernel(const char* __restrict__ text, uint64_t len,
                                                   const unsigned long long* __restrict__ ends, uint64_t n_lines,
                                                   uint64_t first_data_line, uint32_t x_idx, uint32_t y_idx,
                                                   char delim, uint8_t* __restrict__ status, double2* __restrict__ xy,
                                                   unsigned long long* __restrict__ first_bad) {
    const uint64_t l = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (l >= n_lines) return;
    const uint64_t b = l == 0 ? 0 : ends[l - 1] + 1;
    uint64_t e = l < n_lines - 1 || (len > 0 && text[len - 1] == '\n') ? ends[l] : len;
    if (e > len) e = len;
    if (e > b && text[e - 1] == '\r') --e; // getline + '\r' strip (io.hpp:171)
    uint8_t st = 0;
    double2 p = make_double2(0.0, 0.0);
    if (e > b && l >= first_data_line) {
        // split_line: cells are the ranges between delimiters; locate x_idx and y_idx
        const uint32_t need = max(x_idx, y_idx);
        uint32_t cell = 0;
        uint64_t cs = b, xs = 0, xe = 0, ys = 0, ye = 0;
        bool hx = false, hy = false;
        for (uint64_t i = b; i <= e; ++i) {
            if (i == e || text[i] == delim) {
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
                ++cell;
                cs = i + 1;
                if (cell > need) break;
            }
        }
        if (!hx || !hy) {
            st = 2;
        } else if (!parse_cell(text + xs, (int)min(xe - xs, (uint64_t)(1u << 30)), &p.x)) {
            st = 3;
        } else if (!parse_cell(text + ys, (int)min(ye - ys, (uint64_t)(1u << 30)), &p.y)) {
            st = 4;
        } else {
            st = 1;
        }
        if (st >= 2) atomicMin(first_bad, (unsigned long long)l);
    }
    status[l] = st;
    xy[l] = p;
}

__global__ void __launch_bounds__(kT) ok_count_kernel(const uint8_t* __restrict__ status, uint64_t n, uint64_t chunk,
                                                      unsigned long long* __restrict__ blk) {
    const uint64_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
    unsigned c = 0;
    for (uint64_t i = lo + threadIdx.x; i < hi; i += kT) c += status[i] == 1;
    c = __reduce_add_sync(kFullMask, c);
    __shared__ unsigned ws[kT / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x < 32) {
        unsigned v = threadIdx.x < kT / 32 ? ws[threadIdx.x] : 0u;
        v = __reduce_add_sync(kFullMask, v);
        if (threadIdx.x == 0) blk[blockIdx.x] = v;
    }
}

__global__ void __launch_bounds__(kT) ok_write_kernel(const uint8_t* __restrict__ status, const double2* __restrict__ xy,
                                                      uint64_t n, uint64_t chunk,
                                                      const unsigned long long* __restrict__ base,
                                                      double2* __restrict__ out) {
    __shared__ unsigned wc[kT / 32];
    __shared__ unsigned long long run_s;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
    if (threadIdx.x == 0) run_s = base[blockIdx.x];
    __syncthreads();
    for (uint64_t i0 = lo; i0 < hi; i0 += kT) {
        const uint64_t i = i0 + threadIdx.x;
        const bool ok = i < hi && status[i] == 1;
        const unsigned b = __ballot_sync(kFullMask, ok);
        if (lane == 0) wc[w] = __popc(b);
        __syncthreads();
        unsigned before = 0, total = 0;
#pragma unroll
        for (int k = 0; k < kT / 32; ++k) {
            const unsigned c = wc[k];
            before += k < w ? c : 0u;
            total += c;
        }
        const unsigned long long run = run_s;
        if (ok) out[run + before + __popc(b & ((1u << lane) - 1u))] = xy[i];
        __syncthreads();
        if (threadIdx.x == 0) run_s = run + total;
        __syncthreads();
    }
}

int sms(int dev) {
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
}

} // namespace

int csv_blocks(uint64_t n, int dev) {
    const uint64_t want = (n + 16ull * kT - 1) / (16ull * kT);
    return (int)std::max<uint64_t>(1, std::min<uint64_t>(want, 4ull * sms(dev)));
}

cudaError_t launch_csv_lines(const char* text, uint64_t len, int nb, unsigned long long* blk,
                             unsigned long long* ends, cudaStream_t st, uint64_t* launches) {
    const uint64_t chunk = (len + nb - 1) / nb;
    nl_count_kernel<<<nb, kT, 0, st>>>(text, len, chunk, blk);
    scan_kernel<<<1, 1024, 0, st>>>(blk, nb);
    nl_write_kernel<<<nb, kT, 0, st>>>(text, len, chunk, blk, ends);
    *launches += 3;
    return cudaGetLastError();
}

cudaError_t launch_csv_rows(const char* text, uint64_t len, const unsigned long long* ends, uint64_t n_lines,
                            uint64_t first_data_line, uint32_t x_idx, uint32_t y_idx, char delim, uint8_t* status,
                            double* xy, unsigned long long* first_bad, cudaStream_t st, uint64_t* launches) {
    if (n_lines == 0) return cudaSuccess;
    rows_kernel<<<(unsigned)((n_lines + 255) / 256), 256, 0, st>>>(text, len, ends, n_lines, first_data_line, x_idx,
                                                                   y_idx, delim, status,
                                                                   reinterpret_cast<double2*>(xy), first_bad);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_csv_compact(const uint8_t* status, const double* xy, uint64_t n_lines, int nb,
                               unsigned long long* blk, double* out, cudaStream_t st, uint64_t* launches) {
    if (n_lines == 0) return cudaSuccess;
    const uint64_t chunk = (n_lines + nb - 1) / nb;
    ok_count_kernel<<<nb, kT, 0, st>>>(status, n_lines, chunk, blk);
    scan_kernel<<<1, 1024, 0, st>>>(blk, nb);
    ok_write_kernel<<<nb, kT, 0, st>>>(status, reinterpret_cast<const double2*>(xy), n_lines, chunk, blk,
                                        reinterpret_cast<double2*>(out));
    *launches += 3;
    return cudaGetLastError();
}

} // namespace pcd
