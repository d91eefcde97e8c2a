// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// C-ABI shim around the *unmodified* reference benchmark harness
// (proj/include/polycast/bench.hpp: random_batch :62-80, least_squares_fit
// :123-150, error_report :176-198), included from /root/reference at build time.
// Checker for bench.py's sweep_fit / lsq_fit and for include/polycast/bench.hpp
// (tests/test_lsq_fit.py); never the product.
#include <polycast/bench.hpp>

#include <cstdint>
#include <string>
#include <vector>

using namespace polycast;

namespace {
std::vector<TimingSample> samples(const uint64_t* n, const double* t, uint64_t k, const char* label) {
    std::vector<TimingSample> s(k);
    for (uint64_t i = 0; i < k; ++i) s[i] = TimingSample{static_cast<std::size_t>(n[i]), label, t[i]};
    return s;
}
} // namespace

extern "C" {

// 0 ok, 1 DegenerateFit
int ref_least_squares_fit(const uint64_t* n, const double* t, uint64_t k, double* slope, double* intercept) {
    try {
        const auto s = samples(n, t, k, "a");
        const FitCoefficients f = least_squares_fit(s);
        *slope = f.slope;
        *intercept = f.intercept;
        return 0;
    } catch (const DegenerateFit&) {
        return 1;
    }
}

// fit (slope, intercept) applied to k samples: predicted, absolute error, relative error (NaN if absent)
void ref_error_report(double slope, double intercept, const uint64_t* n, const double* t, uint64_t k, double* pred,
                      double* abs_err, double* rel_err) {
    std::map<std::string, FitCoefficients> fits{{"a", FitCoefficients{slope, intercept}}};
    const auto s = samples(n, t, k, "a");
    const ErrorReport r = error_report(fits, s);
    for (uint64_t i = 0; i < k; ++i) {
        pred[i] = r[i].predicted_seconds;
        abs_err[i] = r[i].absolute_error;
        rel_err[i] = r[i].relative_error ? *r[i].relative_error : __builtin_nan("");
    }
}

void ref_random_batch(const double* box, uint64_t n, uint64_t seed, double* xy) {
    const PointBatch b = random_batch(BBox{box[0], box[1], box[2], box[3]}, n, seed);
    for (uint64_t i = 0; i < n; ++i) {
        xy[2 * i] = b.points[i].x;
        xy[2 * i + 1] = b.points[i].y;
    }
}

} // extern "C"
