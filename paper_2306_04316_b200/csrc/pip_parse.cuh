// Decimal text -> binary64, correctly rounded, for the GPU CSV reader
// (pip_csv.cu).  Semantics of the reference's
// detail::parse_double (io.hpp:116-124): std::from_chars (general format) on
// the whole cell, then std::isfinite -- i.e.
//   [-] (digits [. [digits]] | . digits) [(e|E) [+|-] digits]
// with no leading '+', no whitespace, no hex, no inf/nan (they parse but are
// not finite); a value that overflows, or a non-zero value that rounds to
// zero, is out of range (libstdc++ reports result_out_of_range) and fails.
//
// Algorithm (restated, not copied): the first 19 significant digits give w,
// the value is w * 10^q (plus truncated digits).  (1) Clinger's exact case:
// w <= 2^53 and |q| <= 22 -> one IEEE multiply or divide.  (2) Otherwise the
// 128-bit truncation M_q of 5^q (pow5_128.inc, tools/gen_pow5.py) gives
// w * M_q, a lower bound of the scaled value, and (w + truncated) * (M_q + 1)
// an upper bound; when both round to the same double that is the result.
// (3) Else an exact comparison of all digits against the midpoint of the two
// candidates in big-integer arithmetic (ties to even).
// Header-only and __host__ __device__, so the CPU test suite checks it
// against std::from_chars without a GPU (tests/test_csv.py).
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define PC_HD __host__ __device__ __forceinline__
#else
#define PC_HD inline
#endif

namespace pcd {
namespace parse {

struct Pow5 {
    uint64_t hi, lo;
    int e; // floor(log2(5^q))
};

#if defined(__CUDA_ARCH__)
__device__ __constant__ const Pow5 kPow5[] = {
#include "pow5_128.inc"
};
__device__ __constant__ const double kPow10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,
                                                  1e8,  1e9,  1e10, 1e11, 1e12, 1e13, 1e14, 1e15,
                                                  1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
#else
static const Pow5 kPow5[] = {
#include "pow5_128.inc"
};
static const double kPow10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                                  1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
#endif
constexpr int kQMin = -342, kQMax = 308; // parser range; the table runs to 342 (formatter)
constexpr int kMaxDigits = 800; // digits beyond this only act as a sticky bit in the exact comparison

PC_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

PC_HD int clz64(uint64_t x) {
#if defined(__CUDA_ARCH__)
    return __clzll((long long)x);
#else
    return x ? __builtin_clzll(x) : 64;
#endif
}

PC_HD double bits_to_double(uint64_t b) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double((long long)b);
#else
    double d;
    __builtin_memcpy(&d, &b, 8);
    return d;
#endif
}

// 192-bit helpers (z[0] least significant)
PC_HD bool bit192(const uint64_t z[3], int i) { return i >= 0 && i < 192 && ((z[i >> 6] >> (i & 63)) & 1u); }
PC_HD bool any_below192(const uint64_t z[3], int i) { // any set bit at positions < i
    if (i <= 0) return false;
    for (int w = 0; w < 3; ++w) {
        const int lo = w * 64;
        if (i >= lo + 64) {
            if (z[w]) return true;
        } else if (i > lo) {
            if (z[w] & ((1ull << (i - lo)) - 1ull)) return true;
        }
    }
    return false;
}
PC_HD uint64_t word192(const uint64_t z[3], int w) { return w >= 0 && w < 3 ? z[w] : 0ull; }
PC_HD uint64_t bits_at192(const uint64_t z[3], int lo, int n) { // bits [lo, lo+n), 0 <= lo, 1 <= n <= 64
    const int w = lo >> 6, r = lo & 63;
    uint64_t v = word192(z, w) >> r;
    if (r) v |= word192(z, w + 1) << (64 - r);
    return n == 64 ? v : (v & ((1ull << n) - 1ull));
}

// Rounds Z * 2^f (Z = 192-bit value, its top bit at `top`) to binary64 with
// round-half-even.  Returns the bit pattern (sign not set) or ~0 on overflow;
// 0 means the value rounds to zero.
PC_HD uint64_t round192(const uint64_t z[3], int top, int f) {
    int e2 = top + f; // value in [2^e2, 2^(e2+1))
    int drop = top - 52; // bits below the 53-bit mantissa
    if (e2 < -1022) drop += -1022 - e2; // subnormal: fewer mantissa bits
    if (drop > 192) return 0;
    uint64_t mant = drop >= 0 ? bits_at192(z, drop, 53) : 0;
    if (drop < 0) { // cannot happen for our inputs (top >= 190)
        mant = bits_at192(z, 0, 53) << (-drop);
    }
    const bool rnd = drop > 0 && bit192(z, drop - 1);
    const bool sticky = drop > 1 && any_below192(z, drop - 1);
    if (rnd && (sticky || (mant & 1u))) ++mant;
    if (e2 < -1022) { // subnormal (mant < 2^52), or rounded up into the normal range
        if (mant >= (1ull << 52)) return (1ull << 52) | (mant & ((1ull << 52) - 1)); // exponent field 1
        return mant;
    }
    if (mant >= (1ull << 53)) { // carry out of the mantissa
        mant >>= 1;
        ++e2;
    }
    if (e2 > 1023) return ~0ull;
    return ((uint64_t)(e2 + 1023) << 52) | (mant & ((1ull << 52) - 1));
}

// Rounding of w * M * 2^(e5 - 127 + q) where M = {mhi, mlo} (a 128-bit value).
// With near_half != nullptr, also reports whether the bits below the
// rounding position are within 2^64 units of one half: then w * (M + 1) --
// the product's upper bound when M is a truncation -- may round differently.
PC_HD uint64_t round_product(uint64_t w, uint64_t mhi, uint64_t mlo, int e5, int q, bool* near_half = nullptr) {
    const int lz = clz64(w);
    const uint64_t wn = w << lz;
    // Z = wn * (mhi * 2^64 + mlo), 192 bits
    const uint64_t p0 = wn * mlo, p1 = mulhi64(wn, mlo);
    const uint64_t p2 = wn * mhi, p3 = mulhi64(wn, mhi);
    uint64_t z[3];
    z[0] = p0;
    z[1] = p1 + p2;
    z[2] = p3 + (z[1] < p1 ? 1u : 0u);
    const int top = (z[2] >> 63) ? 191 : 190;
    const int f = e5 - 127 + q - lz;
    if (near_half) {
        // the rounding position of round192: bits below `drop` are rounded off
        const int e2 = top + f;
        int drop = top - 52;
        if (e2 < -1022) drop += -1022 - e2;
        if (drop <= 66 || drop > 192) {
            *near_half = true; // the error window reaches the half bit: decide exactly
        } else {
            // bits [64, drop - 1): z[1] whole, then z[2] below bit drop - 1 - 128 (if drop - 1 > 128)
            const int hb = drop - 1;
            const bool half = bit192(z, hb);
            uint64_t m1 = z[1], m2 = 0, full2 = 0;
            if (hb > 128) {
                full2 = (hb - 128 >= 64) ? ~0ull : ((1ull << (hb - 128)) - 1ull);
                m2 = z[2] & full2;
            } else { // hb in (66, 128]: only z[1] bits [0, hb - 64)
                const uint64_t k = (1ull << (hb - 64)) - 1ull;
                m1 &= k;
                full2 = 0;
                *near_half = half ? (m1 == 0) : (m1 == k);
                return round192(z, top, f);
            }
            *near_half = half ? (m1 == 0 && m2 == 0) : (m1 == ~0ull && m2 == full2);
        }
    }
    return round192(z, top, f);
}

// ---- exact comparison (rare path) ------------------------------------------
constexpr int kLimbs = 200; // 6400 bits

struct Big {
    uint32_t v[kLimbs];
    int n; // used limbs
};

PC_HD void big_set(Big& b, uint64_t x) {
    b.v[0] = (uint32_t)x;
    b.v[1] = (uint32_t)(x >> 32);
    b.n = b.v[1] ? 2 : (b.v[0] ? 1 : 0);
}
PC_HD void big_mul_small(Big& b, uint32_t m, uint32_t add = 0) {
    uint64_t carry = add;
    for (int i = 0; i < b.n; ++i) {
        const uint64_t t = (uint64_t)b.v[i] * m + carry;
        b.v[i] = (uint32_t)t;
        carry = t >> 32;
    }
    if (carry && b.n < kLimbs) b.v[b.n++] = (uint32_t)carry;
}
PC_HD void big_mul_pow5(Big& b, int k) {
    while (k >= 13) { // 5^13 < 2^32
        big_mul_small(b, 1220703125u);
        k -= 13;
    }
    uint32_t m = 1;
    while (k-- > 0) m *= 5;
    if (m != 1) big_mul_small(b, m);
}
PC_HD void big_shl(Big& b, int s) {
    const int w = s >> 5, r = s & 31;
    if (b.n == 0) return;
    int n = b.n + w + 1;
    if (n > kLimbs) n = kLimbs;
    for (int i = n - 1; i >= 0; --i) {
        const int j = i - w;
        uint32_t hi = (j >= 0 && j < b.n) ? b.v[j] : 0u;
        uint32_t lo = (j - 1 >= 0 && j - 1 < b.n) ? b.v[j - 1] : 0u;
        b.v[i] = r ? (hi << r) | (lo >> (32 - r)) : hi;
    }
    b.n = n;
    while (b.n > 0 && b.v[b.n - 1] == 0) --b.n;
}
PC_HD int big_cmp(const Big& a, const Big& b) {
    if (a.n != b.n) return a.n < b.n ? -1 : 1;
    for (int i = a.n - 1; i >= 0; --i)
        if (a.v[i] != b.v[i]) return a.v[i] < b.v[i] ? -1 : 1;
    return 0;
}

// Decides between the adjacent doubles lo_bits and lo_bits + 1 (both
// non-negative patterns) by comparing all digits with their midpoint.
PC_HD uint64_t exact_decide(const char* s, int n, int64_t exp10, uint64_t lo_bits) {
    // all significant digits -> A, q_all = exp10 - (digits after the point) (+ skipped beyond the cap)
    // value = A * 10^(exp10 - frac + dropped) (+ the dropped digits: sticky)
    Big A, B;
    A.n = 0;
    int nd = 0, frac = 0, dropped = 0;
    bool seen_nz = false, point = false, sticky = false;
    for (int i = 0; i < n; ++i) {
        const char c = s[i];
        if (c == '.') {
            point = true;
            continue;
        }
        if (c < '0' || c > '9') break;
        if (point) ++frac;
        if (!seen_nz && c == '0') continue;
        seen_nz = true;
        if (nd < kMaxDigits) {
            big_mul_small(A, 10u, (uint32_t)(c - '0'));
            ++nd;
        } else {
            if (c != '0') sticky = true;
            ++dropped;
        }
    }
    int64_t qa = exp10 - frac + dropped;
    // midpoint of lo and lo+1: (2 m + 1) * 2^(E - 1)
    uint64_t m;
    int E;
    const int ef = (int)(lo_bits >> 52);
    if (ef == 0) {
        m = lo_bits & ((1ull << 52) - 1);
        E = -1074;
    } else {
        m = (lo_bits & ((1ull << 52) - 1)) | (1ull << 52);
        E = ef - 1075;
    }
    big_set(B, 2 * m + 1);
    int64_t pow2;
    if (qa >= 0) {
        big_mul_pow5(A, (int)qa);
        pow2 = qa - (E - 1); // compare A * 2^qa  vs  B * 2^(E-1)
    } else {
        big_mul_pow5(B, (int)(-qa));
        pow2 = -(E - 1) + qa; // compare A  vs  B * 2^(E-1) * 2^(-qa)  ->  A * 2^(-(E-1)+qa) vs B
    }
    if (pow2 >= 0) big_shl(A, (int)pow2);
    else big_shl(B, (int)(-pow2));
    int c = big_cmp(A, B);
    if (c == 0 && sticky) c = 1;
    if (c > 0) return lo_bits + 1;
    if (c < 0) return lo_bits;
    return (lo_bits & 1u) ? lo_bits + 1 : lo_bits; // tie: to even
}

// ---- SWAR digit runs (8 or 4 ASCII bytes at once, little-endian) ---------------
PC_HD uint64_t load_le(const char* p, int k) {
    uint64_t v = 0;
    for (int j = 0; j < k; ++j) v |= (uint64_t)(uint8_t)p[j] << (8 * j);
    return v;
}
// every byte in '0'..'9': high nibble 3, and adding 6 does not carry out of the low nibble
PC_HD bool all_digits8(uint64_t v) {
    return ((v & 0xf0f0f0f0f0f0f0f0ull) | (((v + 0x0606060606060606ull) & 0xf0f0f0f0f0f0f0f0ull) >> 4)) ==
           0x3333333333333333ull;
}
PC_HD bool all_digits4(uint32_t v) {
    return ((v & 0xf0f0f0f0u) | (((v + 0x06060606u) & 0xf0f0f0f0u) >> 4)) == 0x33333333u;
}
// value of 8 digit bytes (first digit in the low byte): pairs, then quads, then the two halves
PC_HD uint32_t digits8(uint64_t v) {
    v -= 0x3030303030303030ull;
    v = v * 10 + (v >> 8);                                  // byte 2k: 2-digit value of digits 2k, 2k+1
    v = ((v & 0x000000ff000000ffull) * (100 + (1000000ull << 32)) +
         ((v >> 16) & 0x000000ff000000ffull) * (1 + (10000ull << 32))) >> 32;
    return (uint32_t)v;
}
PC_HD uint32_t digits4(uint32_t v) {
    v -= 0x30303030u;
    v = v * 10 + (v >> 8);                      // bytes 0 and 2: 2-digit values
    return (v & 0xff) * 100 + ((v >> 16) & 0xff);
}

// Parses the whole range [s, s+n).  Returns true and *out on success.
PC_HD bool parse_f64(const char* s, int n, double* out) {
    int i = 0;
    bool neg = false;
    if (i < n && s[i] == '-') {
        neg = true;
        ++i;
    }
    const int start = i;
    uint64_t w = 0;
    int nsig = 0, frac = 0, ndig = 0;
    bool trunc = false, point = false;
    for (; i < n; ++i) {
        // runs of digits inside the 19-digit window, 8 or 4 at a time (after the first significant one)
        if (nsig > 0 && nsig <= 11 && i + 8 <= n) {
            const uint64_t v = load_le(s + i, 8);
            if (all_digits8(v)) {
                w = w * 100000000ull + digits8(v);
                nsig += 8;
                ndig += 8;
                if (point) frac += 8;
                i += 7;
                continue;
            }
        }
        if (nsig > 0 && nsig <= 15 && i + 4 <= n) {
            const uint32_t v = (uint32_t)load_le(s + i, 4);
            if (all_digits4(v)) {
                w = w * 10000ull + digits4(v);
                nsig += 4;
                ndig += 4;
                if (point) frac += 4;
                i += 3;
                continue;
            }
        }
        const char c = s[i];
        if (c == '.') {
            if (point) break;
            point = true;
            continue;
        }
        if (c < '0' || c > '9') break;
        ++ndig;
        if (point) ++frac;
        if (nsig == 0 && c == '0') continue; // leading zeros
        if (nsig < 19) w = w * 10 + (uint64_t)(c - '0');
        else if (c != '0') trunc = true;
        ++nsig;
    }
    if (ndig == 0) return false; // "", "-", ".", "-."
    const int mant_end = i;
    int64_t exp10 = 0;
    if (i < n && (s[i] == 'e' || s[i] == 'E')) {
        int j = i + 1;
        bool eneg = false;
        if (j < n && (s[j] == '+' || s[j] == '-')) {
            eneg = s[j] == '-';
            ++j;
        }
        if (j < n && s[j] >= '0' && s[j] <= '9') {
            int64_t e = 0;
            for (; j < n && s[j] >= '0' && s[j] <= '9'; ++j)
                if (e < 100000000) e = e * 10 + (s[j] - '0');
            exp10 = eneg ? -e : e;
            i = j;
        }
    }
    if (i != n) return false; // trailing characters (incl. an exponent without digits)
    const uint64_t sign = neg ? (1ull << 63) : 0ull;
    if (w == 0) { // all digits zero: +-0 regardless of the exponent
        *out = bits_to_double(sign);
        return true;
    }
    // value = w * 10^q (+ truncated digits)
    const int64_t q = exp10 - frac + (nsig > 19 ? nsig - 19 : 0);
    if (!trunc && w <= (1ull << 53) && q >= -22 && q <= 22) { // Clinger: exact operands, one rounding
        double d = (double)w;
        d = q >= 0 ? d * kPow10[q] : d / kPow10[-q];
        *out = neg ? -d : d;
        return true;
    }
    if (q < kQMin) return false; // < 1e-323: rounds to zero (out of range)
    if (q > kQMax) return false; // overflow
    const Pow5& P = kPow5[q - kQMin];
    const bool exact5 = q >= 0 && q <= 55;
    uint64_t bits;
    if (!trunc) {
        // w is exact: the scaled value lies in [w M, w (M + 1)) (M exact for 0 <= q <= 55);
        // one product decides unless its rounded-off bits sit within w of one half
        bool near = false;
        const uint64_t r = round_product(w, P.hi, P.lo, P.e, (int)q, exact5 ? nullptr : &near);
        if (!near) {
            bits = r;
        } else {
            if (r == ~0ull) return false; // overflow even from below
            // candidates r - 1 / r when z rounded up (half bit set), r / r + 1 otherwise:
            // decide between the two around the half
            bits = exact_decide(s + start, mant_end - start, exp10, r);
            const uint64_t b2 = r ? exact_decide(s + start, mant_end - start, exp10, r - 1) : r;
            bits = (b2 == r - 1 && r) ? b2 : bits;
        }
    } else {
        const uint64_t lo = round_product(w, P.hi, P.lo, P.e, (int)q);
        // upper bound: (w + 1) (M + 1 unless exact); rounding of that product stands in
        // for the rounding of the exclusive bound (can only make the bounds disagree)
        uint64_t mhi = P.hi, mlo = P.lo;
        if (!exact5 && ++mlo == 0) ++mhi;
        const uint64_t hi = round_product(w + 1, mhi, mlo, P.e, (int)q);
        if (lo == hi) {
            bits = lo;
        } else {
            if (lo == ~0ull) return false; // even the lower bound overflows
            bits = exact_decide(s + start, mant_end - start, exp10, lo);
        }
    }
    if (bits == 0 || bits >= (0x7ffull << 52)) return false; // rounded to zero / overflow
    *out = bits_to_double(bits | sign);
    return true;
}

} // namespace parse
} // namespace pcd
