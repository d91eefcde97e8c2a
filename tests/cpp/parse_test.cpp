// CPU test of the GPU CSV reader's number parser (paper_2306_04316_b200/csrc/
// pip_parse.cuh, compiled here as host code) against std::from_chars +
// std::isfinite -- the reference's detail::parse_double (io.hpp:116-124).
// Random doubles printed in several formats, random digit strings with
// exponents, exact midpoints between adjacent doubles (ties), just above /
// below them, subnormals, the overflow / underflow boundaries and long digit
// strings.  Exit code = number of mismatches (capped).
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>

#include "pip_parse.cuh"

static long fails = 0, total = 0;

static void check(const std::string& t) {
    double a = 0;
    const auto [p, ec] = std::from_chars(t.data(), t.data() + t.size(), a);
    const bool ok_ref = ec == std::errc{} && p == t.data() + t.size() && std::isfinite(a);
    double b = 0;
    const bool ok = pcd::parse::parse_f64(t.data(), (int)t.size(), &b);
    ++total;
    uint64_t ba, bb;
    std::memcpy(&ba, &a, 8);
    std::memcpy(&bb, &b, 8);
    if (ok != ok_ref || (ok && ba != bb)) {
        if (fails < 20) std::printf("MISMATCH '%.80s' ref(%d,%.17g) got(%d,%.17g)\n", t.c_str(), ok_ref, a, ok, b);
        ++fails;
    }
}

int main() {
    const char* fixed[] = {
        "1e-400", "2e-324", "2.4703282292062327e-324", "2.4703282292062328e-324", "3e-324", "4.9e-324", "1e400",
        "1.7976931348623157e308", "1.7976931348623158e308", "1.7976931348623159e308", "-0", "+1", ".5", "5.", ".",
        "inf", "nan", "-inf", "infinity", "1e", "1e+", "1e-", "0x10", " 1", "1 ", "1e+400", "-1e-400", "123456789012345678901234567890",
        "00000000000000001", "1E5", "1e0005", "-.5e-2", "9007199254740993", "9007199254740992", "9007199254740995",
        "1.00000000000000011102230246251565404236316680908203125", "-", "-.", "1..2", "1.2.3", "1e5e5", "e5", "-e5",
        "0e9999999999", "0.0", "-0.0e-5", "2.2250738585072011e-308", "2.2250738585072014e-308", "1e23", "0.1", "0.3",
        "1e22", "1e-22", "4294967295", "18446744073709551615", "18446744073709551616", "99999999999999999999",
        "5e-324", "1e-323", "1e308", "--1", "1-", "1.e5", ".e5", "1.5E-3", "1_0", "١"};
    for (const char* t : fixed) check(t);
    std::mt19937_64 g(7);
    char buf[160];
    const char* fmts[] = {"%.17g", "%.16g", "%.15g", "%.20e", "%.6e", "%.25g", "%.3g", "%.40f"};
    for (int k = 0; k < 1000000; ++k) {
        uint64_t u = g();
        double d;
        std::memcpy(&d, &u, 8);
        if (!std::isfinite(d)) continue;
        std::snprintf(buf, sizeof buf, fmts[k % 8], d);
        check(buf);
    }
    for (int k = 0; k < 1000000; ++k) {
        std::string t;
        if (g() & 1) t += '-';
        const int nd = 1 + (int)(g() % 30), pt = (int)(g() % (nd + 2));
        for (int i = 0; i < nd; ++i) {
            if (i == pt) t += '.';
            t += char('0' + g() % 10);
        }
        if (g() % 3 == 0) t += (g() & 1 ? "e" : "E") + std::to_string((int)(g() % 700) - 350);
        check(t);
    }
    // exact midpoints (long double holds them exactly), ties and their neighbours
    for (int k = 0; k < 40000; ++k) {
        uint64_t u = g();
        switch (k % 3) {
        case 0: u &= 0x000fffffffffffffull; break; // subnormal
        case 1: u = 0x7fe0000000000000ull | (u & 0x000fffffffffffffull); break; // near the top
        default: u &= 0x7fefffffffffffffull;
        }
        double d;
        std::memcpy(&d, &u, 8);
        const double nx = std::nextafter(d, INFINITY);
        const long double mid = ((long double)d + (long double)nx) / 2;
        std::snprintf(buf, sizeof buf, "%.40Lg", mid);
        check(buf);
        std::snprintf(buf, sizeof buf, "%.21Lg", mid);
        check(buf);
        std::string s = buf;
        if (s.find('e') == std::string::npos && s.find('.') != std::string::npos) check(s + "000000000000000000001");
    }
    // long digit strings (beyond 19 and beyond the exact path's 800-digit cap)
    for (int k = 0; k < 2000; ++k) {
        std::string t = std::to_string(1 + g() % 9) + ".";
        const int nd = 20 + (int)(g() % 1200);
        for (int i = 0; i < nd; ++i) t += char('0' + (k % 2 ? 0 : g() % 10));
        if (k % 4 == 1) t += "1";
        t += "e" + std::to_string((int)(g() % 600) - 300);
        check(t);
    }
    std::printf("parse_test: %ld checks, %ld mismatches\n", total, fails);
    return fails > 100 ? 100 : (int)fails;
}
