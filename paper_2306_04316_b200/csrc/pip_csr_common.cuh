// Helpers shared by the CSR kernels (pip_csr.cu warp kernel, pip_csr_tile.cu
// tile kernel): the C1 certified fast path and bit-plane output.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace pcd {

constexpr unsigned kFull = 0xffffffffu;

// ---- C1 certified fast path -------------------------------------------------
// For a polygon whose bbox W x H is well scaled (2^-300 <= W, H <= 2^300), map
// coordinates to polygon-local units: L = (v - o) * s with o the bbox min and s
// a power of two with W*s, H*s in [1/2, 1).  Then, per (point, edge):
//   * y: q(y) = trunc((y - o_y) * s_y * 2^30) is monotone, so
//       q_lo < q(p.y) < q_hi        =>  y_lo < p.y < y_hi  => the reference's
//                                       f_prev * f_next <= 0 holds (P2);
//       q(p.y) outside [q_lo, q_hi] =>  p.y outside [y_lo, y_hi] strictly, and
//       with |p.y| >= 2^-400 both differences are >= 2^-453 so the product is
//       > 0 (no underflow): the edge is not a straddle;
//     q(p.y) equal to some vertex key is a tie -> the exact path.
//   * side: s = fma(lx, Nx, fma(ly, Ny, c)) in fp32 approximates
//       S' = (p - a) . n * s_x * s_y  (n = the reference's rounded, flipped
//       normal) with |s - S'| <= 13.1 * 2^-24 (all local terms are <= 1 in
//       magnitude, |c| <= 2), while the reference's binary64
//       value differs from S' by <= 4.1 * 2^-53 (+ underflow terms < 2^-470).
//       So |s| > kFastBand = 2^-20 decides the sign of the reference's side;
//       |s| <= kFastBand is sent to the exact path.
// A point with any tie / band hit in a chunk of edges takes the exact binary64
// path (binary64, the reference's expression order) for that chunk; every other (point, edge)
// contribution is the reference's, so parities stay bit-exact.
constexpr float kFastBand = 0x1p-20f;
constexpr int kFastSentinelLo = 0x40000000; // qlo+1 of a non-edge: never "sure"

// fpar ^= bit when d1 < rng1 (unsigned: q_lo < q(p.y) < q_hi) and s < -kFastBand,
// as two predicate-combining compares and one predicated xor
__device__ __forceinline__ void fast_toggle(uint32_t& fpar, uint32_t bit, unsigned d1, unsigned rng1, float s) {
    asm("{\n\t.reg .pred p, q;\n\t"
        "setp.lt.f32 p, %2, %5;\n\t"
        "setp.lt.and.u32 q, %3, %4, p;\n\t"
        "@q xor.b32 %0, %0, %1;\n\t}"
        : "+r"(fpar)
        : "r"(bit), "f"(s), "r"(d1), "r"(rng1), "f"(-kFastBand));
}

// Packed binary32 pairs (sm_100 FFMA2): each half is an IEEE fma.rn of its own,
// bit-identical to a scalar fmaf on that half.  A broadcast operand (f, f) is
// folded by ptxas into FFMA2's scalar-operand form (no register pair needed).
__device__ __forceinline__ unsigned long long f32x2(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
// (a.lo, a.hi) * (f, f) + (g, g)
__device__ __forceinline__ unsigned long long ffma2_bb(unsigned long long a, float f, float g) {
    return ffma2(a, f32x2(f, f), f32x2(g, g));
}
// (a.lo, a.hi) * (f, f) + c
__device__ __forceinline__ unsigned long long ffma2_b(unsigned long long a, float f, unsigned long long c) {
    return ffma2(a, f32x2(f, f), c);
}
// the high 16 bits of both halves in one word (sign bits at 15 / 31)
__device__ __forceinline__ uint32_t hi16x2(unsigned long long s) {
    return __byte_perm((uint32_t)s, (uint32_t)(s >> 32), 0x7632);
}

__device__ __forceinline__ double pow2_below_inv(double w) { // 2^-(E+1) for w in [2^E, 2^(E+1))
    const int e = (__double2hiint(w) >> 20) & 0x7ff;
    return __hiloint2double((2045 - e) << 20, 0);
}

__device__ __forceinline__ void or_bits(uint32_t* plane, unsigned long long g0, uint32_t bits) {
    if (!bits) return;
    const unsigned long long w = g0 >> 5;
    const unsigned sh = (unsigned)(g0 & 31);
    atomicOr(&plane[w], bits << sh);
    if (sh && (bits >> (32 - sh))) atomicOr(&plane[w + 1], bits >> (32 - sh));
}

// 64 consecutive bits (lo: points g0 .. g0+31, hi: g0+32 .. g0+63; warp-uniform)
// into a bit plane: lanes 0..2 each OR one of the (at most) three words they touch
__device__ __forceinline__ void or_bits64(uint32_t* plane, unsigned long long g0, uint32_t lo, uint32_t hi,
                                          int lane) {
    // word `lane` of (0 : hi : lo : 0) << sh, i.e. the high word of (b : a) << sh
    // with (a, b) = (0, lo), (lo, hi), (hi, 0) for lanes 0, 1, 2
    const uint32_t a = lane == 1 ? lo : hi, b = lane == 0 ? lo : hi;
    const uint32_t w = __funnelshift_l(lane == 0 ? 0u : a, lane == 2 ? 0u : b, (unsigned)g0 & 31u);
    if (lane < 3 && w) atomicOr(plane + (g0 >> 5) + lane, w);
}

} // namespace pcd
