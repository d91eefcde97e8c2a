// CPU test of the GPU results-CSV writer's number formatter (paper_2306_04316_b200/
// csrc/pip_format.cuh, compiled here as host code) against glibc's
// snprintf("%.17g") -- the reference's detail::format_17g (io.hpp:137-141) --
// and of put_u64 against "%llu".  Random bit patterns (normal, subnormal),
// integers and exact decimal ties, powers of ten and their neighbours.
// Exit code = number of mismatches (capped).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>

#include "pip_format.cuh"

static long fails = 0, total = 0;

static void check(double v) {
    char want[64], got[64];
    std::snprintf(want, sizeof want, "%.17g", v);
    const int n = pcd::fmt::format_17g(v, got);
    got[n] = 0;
    ++total;
    if (std::strcmp(want, got) != 0) {
        if (fails < 20) std::printf("MISMATCH %a: want '%s' got '%s'\n", v, want, got);
        ++fails;
    }
}

static void check_u64(unsigned long long v) {
    char want[32], got[32];
    std::snprintf(want, sizeof want, "%llu", v);
    const int n = pcd::fmt::put_u64(got, v);
    got[n] = 0;
    ++total;
    if (std::strcmp(want, got) != 0) {
        if (fails < 20) std::printf("MISMATCH u64 want '%s' got '%s'\n", want, got);
        ++fails;
    }
}

int main() {
    const double fixed[] = {0.0, -0.0, 1.0, -1.0, 0.1, 0.5, 1e-4, 1e-5, 9.9999999999999995e-5, 1e16, 1e17, 1e22,
                            1e23, 123456789012345678.0, 5e-324, 1e-323, 2.2250738585072014e-308,
                            2.2250738585072009e-308, 1.7976931348623157e308, 4503599627370496.5, 0.3, 2.0 / 3.0,
                            100.0, 1e21, 9007199254740993.0, 12345678901234567890.0, 0.000123, 1.5e-300,
                            180.0, -180.0, 90.0, -89.999999999999986};
    for (double v : fixed) check(v);
    std::mt19937_64 g(17);
    for (int k = 0; k < 2000000; ++k) {
        uint64_t u = g();
        double d;
        std::memcpy(&d, &u, 8);
        if (!std::isfinite(d)) continue;
        check(d);
    }
    for (int k = 0; k < 300000; ++k) { // subnormals and coordinates
        uint64_t u = g() & 0x800fffffffffffffull;
        double d;
        std::memcpy(&d, &u, 8);
        check(d);
        check(std::uniform_real_distribution<double>(-180, 180)(g));
        check((double)(g() >> 11) * 0x1.0p-53);
        check((double)g() / 1e3 * ((g() & 1) ? 1 : -1e-7)); // io_test.cpp's awkward magnitudes
    }
    // integers with more than 17 digits: exact ties at the 17th digit and neighbours
    for (int k = 0; k < 200000; ++k) {
        const int sh = 4 + (int)(g() % 60);
        const double base = std::ldexp((double)((g() >> 11) | 1), sh);
        check(base);
        check(std::nextafter(base, 0.0));
        check(std::nextafter(base, INFINITY));
    }
    // exact decimal ties: d * 10^j + 5 * 10^(j-1) style values (representable ones)
    for (unsigned long long a = 1; a < 200000; ++a) {
        const double t = (double)(a * 10ull + 5ull) * 1e16; // 18+ digits, 5 in the 18th place
        check(t);
        check((double)(100000000000000000ull + a * 10ull + 5ull)); // 18-digit integers ending in 5
    }
    for (int j = -330; j <= 310; ++j) { // powers of ten and their neighbours
        const double p = std::pow(10.0, (double)j);
        if (!std::isfinite(p)) continue;
        check(p);
        check(std::nextafter(p, 0.0));
        check(std::nextafter(p, INFINITY));
    }
    const unsigned long long ints[] = {0, 1, 9, 10, 99999999, 100000000, 18446744073709551615ull,
                                       10000000000000000000ull, 12345678901234567ull};
    for (auto v : ints) check_u64(v);
    for (int k = 0; k < 200000; ++k) check_u64(g() >> (g() % 64));
    std::printf("format_test: %ld checks, %ld mismatches\n", total, fails);
    return fails > 100 ? 100 : (int)fails;
}
