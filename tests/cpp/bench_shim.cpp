// C-ABI over include/polycast/bench.hpp (the drop-in harness) for
// tests/test_lsq_fit.py: compared there with the unmodified reference
// (oracle/_ref ref_bench_shim.cpp) and with bench.py's Python fit.
#include <polycast/bench.hpp>

#include <cstdint>
#include <map>
#include <string>
#include <vector>

using namespace polycast;

namespace {
std::vector<TimingSample> samples(const uint64_t* n, const double* t, uint64_t k) {
    std::vector<TimingSample> s(k);
    for (uint64_t i = 0; i < k; ++i) s[i] = TimingSample{static_cast<std::size_t>(n[i]), "a", t[i]};
    return s;
}
} // namespace

extern "C" {

int our_least_squares_fit(const uint64_t* n, const double* t, uint64_t k, double* slope, double* intercept) {
    try {
        const auto s = samples(n, t, k);
        const FitCoefficients f = least_squares_fit(s);
        *slope = f.slope;
        *intercept = f.intercept;
        return 0;
    } catch (const DegenerateFit&) {
        return 1;
    }
}

void our_error_report(double slope, double intercept, const uint64_t* n, const double* t, uint64_t k, double* pred,
                      double* abs_err, double* rel_err) {
    std::map<std::string, FitCoefficients> fits{{"a", FitCoefficients{slope, intercept}}};
    const auto s = samples(n, t, k);
    const ErrorReport r = error_report(fits, s);
    for (uint64_t i = 0; i < k; ++i) {
        pred[i] = r[i].predicted_seconds;
        abs_err[i] = r[i].absolute_error;
        rel_err[i] = r[i].relative_error ? *r[i].relative_error : __builtin_nan("");
    }
}

void our_random_batch(const double* box, uint64_t n, uint64_t seed, double* xy) {
    const PointBatch b = random_batch(BBox{box[0], box[1], box[2], box[3]}, n, seed);
    for (uint64_t i = 0; i < n; ++i) {
        xy[2 * i] = b.points[i].x;
        xy[2 * i + 1] = b.points[i].y;
    }
}

// emit_report + read_samples_csv round trip through a temp file: returns the
// number of samples read back (-1 on an exception)
int our_report_roundtrip(const uint64_t* n, const double* t, uint64_t k, const char* json_path, const char* csv_path) {
    try {
        const auto s = samples(n, t, k);
        const GroupedFits g = fit_per_algorithm(s);
        emit_report(s, g.fits, error_report(g.fits, s), json_path);
        {
            std::ofstream f(csv_path, std::ios::binary);
            f << "algorithm,seconds,n\n";
            for (const auto& x : s) f << x.algorithm << ',' << detail::format_17g_host(x.elapsed_seconds) << ',' << x.n_points << '\n';
        }
        const auto back = read_samples_csv(csv_path);
        for (uint64_t i = 0; i < k; ++i)
            if (back[i].n_points != s[i].n_points || back[i].elapsed_seconds != s[i].elapsed_seconds) return -2;
        return static_cast<int>(back.size());
    } catch (const std::exception&) {
        return -1;
    }
}

} // extern "C"
