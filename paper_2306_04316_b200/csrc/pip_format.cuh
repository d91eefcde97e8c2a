// binary64 -> "%.17g" text and u64 -> decimal, for the GPU results-CSV writer
// (pip_emit.cu).  Output is byte-identical to glibc's
// printf("%.17g") (the reference's detail::format_17g, io.hpp:137-141): 17
// significant digits, correctly rounded (ties to even), fixed notation when
// the decimal exponent X satisfies -4 <= X < 17 and exponential otherwise
// ("d.ddde+XX", at least two exponent digits), trailing zeros and a bare '.'
// removed, "-0" for negative zero.
//
// Algorithm (restated, not copied): v = m 2^e.  The 17-digit integer
// D = round(v 10^(16-X)) comes from one 64 x 128-bit product with the
// normalised 5^k of pow5_128.inc (the CSV parser's table): the bits below
// D's are the fraction, known to within m units of the product's last bit
// because the table entry is truncated.  When the fraction is within that
// error of one half (exact ties included) the decision is redone exactly with
// big integers (the parser's Big helpers).  Header-only and __host__
// __device__: tests/cpp/format_test.cpp checks it against snprintf.
#pragma once

#include "pip_parse.cuh"

namespace pcd {
namespace fmt {

using parse::Big;
using parse::Pow5;

PC_HD uint64_t dbl_bits(double v) {
#if defined(__CUDA_ARCH__)
    return (uint64_t)__double_as_longlong(v);
#else
    uint64_t b;
    __builtin_memcpy(&b, &v, 8);
    return b;
#endif
}

// 8 decimal digits of v < 10^8 (32-bit arithmetic), most significant first
PC_HD void put8(char* p, uint32_t v) {
    for (int i = 7; i >= 0; --i) {
        p[i] = (char)('0' + v % 10u);
        v /= 10u;
    }
}

// the 17 digits of D < 10^17
PC_HD void put_digits17(char* p, uint64_t D) {
    const uint64_t a = D / 100000000ull;
    put8(p + 9, (uint32_t)(D - a * 100000000ull));
    const uint32_t top = (uint32_t)(a / 100000000ull);
    put8(p + 1, (uint32_t)(a - (uint64_t)top * 100000000ull));
    p[0] = (char)('0' + top);
}

// decimal u64 (no leading zeros); returns the length
PC_HD int put_u64(char* p, uint64_t v) {
    char t[20];
    int n = 0;
    // 8-digit groups through 32-bit arithmetic
    while (v >= 100000000ull) {
        uint32_t g = (uint32_t)(v % 100000000ull);
        v /= 100000000ull;
        for (int i = 0; i < 8; ++i) {
            t[n++] = (char)('0' + g % 10);
            g /= 10;
        }
    }
    uint32_t g = (uint32_t)v;
    do {
        t[n++] = (char)('0' + g % 10);
        g /= 10;
    } while (g);
    for (int i = 0; i < n; ++i) p[i] = t[n - 1 - i];
    return n;
}

// Exact decision for a fraction near one half: compares v 10^k = m 2^e 10^k
// with D + 1/2.  Returns >0, 0 or <0.
PC_HD int cmp_half_exact(uint64_t m, int e, int k, uint64_t D) {
    Big A, B;
    parse::big_set(A, m);
    parse::big_set(B, 2 * D + 1); // compare 2 m 2^e 2^k 5^k with 2 D + 1
    if (k >= 0) parse::big_mul_pow5(A, k);
    else parse::big_mul_pow5(B, -k);
    const int sh = e + k + 1;
    if (sh >= 0) parse::big_shl(A, sh);
    else parse::big_shl(B, -sh);
    return parse::big_cmp(A, B);
}

// Writes "%.17g" of v to p (at most 24 bytes); returns the length.
PC_HD int format_17g(double v, char* p) {
    uint64_t b = dbl_bits(v);
    int n = 0;
    if (b >> 63) p[n++] = '-';
    b &= ~(1ull << 63);
    if (b == 0) {
        p[n++] = '0';
        return n;
    }
    const int ef = (int)(b >> 52);
    uint64_t m = b & ((1ull << 52) - 1);
    int e;
    if (ef == 0) {
        e = -1074;
    } else {
        m |= 1ull << 52;
        e = ef - 1075;
    }
    const int lz = parse::clz64(m);
    const uint64_t wn = m << lz;
    const int e2 = e - lz; // v = wn 2^e2, wn in [2^63, 2^64)
    // X ~ floor(log10 v); v in [2^(e2+63), 2^(e2+64)); 78913 / 2^18 ~ log10(2)
    int X = (int)(((int64_t)(e2 + 63) * 78913) >> 18);
    uint64_t D = 0;
    uint64_t z[3];
    int s = 0;
    bool raised = false;
    for (int tries = 0; tries < 4; ++tries) {
        const int k = 16 - X;
        const Pow5& P = parse::kPow5[k - parse::kQMin];
        const uint64_t p0 = wn * P.lo, p1 = parse::mulhi64(wn, P.lo);
        const uint64_t p2 = wn * P.hi, p3 = parse::mulhi64(wn, P.hi);
        z[0] = p0;
        z[1] = p1 + p2;
        z[2] = p3 + (z[1] < p1 ? 1u : 0u);
        s = -(P.e - 127 + e2 + k); // v 10^k ~ z 2^-s
        D = parse::bits_at192(z, s, 64);
        if (D >= 100000000000000000ull) {
            ++X;
            raised = true;
        } else if (D < 10000000000000000ull && !raised) {
            --X;
        } else {
            break; // (after a raise, D = 10^16 - 1 is an underestimate of 10^16: it rounds up)
        }
    }
    // rounding: the fraction is z mod 2^s, true value in [z, z + wn) unless 5^k is exact
    const int k = 16 - X;
    const bool exact = k >= 0 && k <= 55;
    // D >= 10^16 > 2^53 and z < 2^192 put the half bit s - 1 in z[2] (s in [134, 138])
    const uint64_t lowm = (1ull << (s - 1 - 128)) - 1; // z[2] bits under the half bit
    const bool half = (z[2] >> (s - 1 - 128)) & 1u;
    const bool below = (z[2] & lowm) || z[1] || z[0]; // bits under the half bit
    bool up;
    // near one half: the bits [64, s-1) are all ones (just under) or all zeros (half or just over);
    // the error of the truncated 5^k is below 2^64 units
    bool near = false;
    if (!exact) {
        const bool all0 = z[1] == 0 && (z[2] & lowm) == 0;
        const bool all1 = z[1] == ~0ull && (z[2] & lowm) == lowm;
        near = half ? all0 : all1;
    }
    if (near) {
        const int c = cmp_half_exact(m, e, k, D);
        up = c > 0 || (c == 0 && (D & 1));
    } else if (exact) {
        up = half && (below || (D & 1));
    } else {
        up = half; // strictly above or below one half
    }
    if (up && ++D == 100000000000000000ull) {
        D = 10000000000000000ull;
        ++X;
    }
    // layout
    char dg[17];
    put_digits17(dg, D);
    int nd = 17;
    while (nd > 1 && dg[nd - 1] == '0') --nd; // significant digits without trailing zeros
    if (X < -4 || X >= 17) {
        p[n++] = dg[0];
        if (nd > 1) {
            p[n++] = '.';
            for (int i = 1; i < nd; ++i) p[n++] = dg[i];
        }
        p[n++] = 'e';
        int ax = X;
        if (ax < 0) {
            p[n++] = '-';
            ax = -ax;
        } else {
            p[n++] = '+';
        }
        if (ax >= 100) {
            p[n++] = (char)('0' + ax / 100);
            ax %= 100;
            p[n++] = (char)('0' + ax / 10);
            p[n++] = (char)('0' + ax % 10);
        } else {
            p[n++] = (char)('0' + ax / 10);
            p[n++] = (char)('0' + ax % 10);
        }
    } else if (X >= 0) {
        for (int i = 0; i <= X; ++i) p[n++] = dg[i];
        if (nd > X + 1) {
            p[n++] = '.';
            for (int i = X + 1; i < nd; ++i) p[n++] = dg[i];
        }
    } else {
        p[n++] = '0';
        p[n++] = '.';
        for (int i = 0; i < -X - 1; ++i) p[n++] = '0';
        for (int i = 0; i < nd; ++i) p[n++] = dg[i];
    }
    return n;
}

} // namespace fmt
} // namespace pcd
