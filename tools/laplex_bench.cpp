// laplex_bench -- CPU-vs-GPU benchmark CLI over the drop-in C++ API (include/laplex).
//
// Reproduces the reference harness's bench-matvec, accuracy and bench-gram
// subcommands (reference proj/tools/laplex_bench.cpp:32-34 CSV schema,
// :191-345 experiments, :141-142,170-187 trial protocol) on the B200 library,
// with three columns appended to the same CSV schema:
//   gpus          devices used (1)
//   gbs           algorithmic bytes of the timed call / wall time (GB/s);
//                 the model of SURVEY.md 8(d) (cached-plan matvec:
//                 12n + 8k + B(4n + 4k) per call, Gram: 8k reads + 8n^2 writes)
//   roofline_frac gbs / HBM peak (LAPLEX_HBM_GBS, default 6452 measured on
//                 this pool's B200s)
// The drop-in API takes host vectors, so wall times include the PCIe copies
// of x and y (as a caller of the reference API would see them).
//
// Methods: laplex (this library, on the GPU) and dense (explicit O(nk) CPU
// kernel, the reference harness's comparison method).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include <sys/resource.h>

#include "laplex/laplex.hpp"

using namespace laplex;

namespace {

const char* kHeader =
    "experiment,method,precision,n,k,batch,feature_count,trial,wall_ns,peak_bytes,rel_err_l2,seed,gpus,gbs,"
    "roofline_frac";

struct Row {
    std::string experiment, method, precision;
    std::size_t n = 0, k = 0, batch = 1;
    long long feature_count = -1;
    std::size_t trial = 0;
    double wall_ns = 0;
    long long peak_bytes = -1;
    double rel_err_l2 = -1;
    std::uint64_t seed = 0;
    double model_bytes = -1;  // algorithmic bytes of the timed call (-1: not modelled)
};

double hbm_peak_gbs() {
    const char* e = std::getenv("LAPLEX_HBM_GBS");
    return e ? std::atof(e) : 6452.0;
}

class Csv {
  public:
    explicit Csv(const std::string& path) {
        if (!path.empty()) {
            f_.open(path);
            if (!f_) throw std::runtime_error("cannot open output file " + path);
        }
        out() << kHeader << "\n";
    }
    void write(const Row& r) {
        std::ostringstream s;
        s << r.experiment << ',' << r.method << ',' << r.precision << ',' << r.n << ',' << r.k << ',' << r.batch
          << ',' << r.feature_count << ',' << r.trial << ',' << std::llround(r.wall_ns) << ',' << r.peak_bytes
          << ',';
        if (r.rel_err_l2 < 0)
            s << -1;
        else
            s << std::scientific << r.rel_err_l2 << std::defaultfloat;
        s << ',' << r.seed << ',' << (r.method == "laplex" ? 1 : 0) << ',';
        if (r.model_bytes > 0 && r.wall_ns > 0) {
            const double gbs = r.model_bytes / r.wall_ns;  // bytes per ns == GB/s
            s << gbs << ',' << gbs / hbm_peak_gbs();
        } else {
            s << "-1,-1";
        }
        out() << s.str() << "\n";
    }

  private:
    std::ostream& out() { return f_.is_open() ? f_ : std::cout; }
    std::ofstream f_;
};

double now_ns() {
    return double(std::chrono::duration_cast<std::chrono::nanoseconds>(
                      std::chrono::steady_clock::now().time_since_epoch())
                      .count());
}

long long peak_rss() {
    rusage ru{};
    return getrusage(RUSAGE_SELF, &ru) == 0 ? (long long)ru.ru_maxrss * 1024 : -1;
}

struct Opts {
    std::size_t n_min = 1 << 10, n_max = 1 << 14, k = 0, batch = 1, trials = 5, warmups = 2, gram_n = 64;
    std::uint64_t seed = 42;
    std::string precision = "f64", methods = "laplex", out;
    long long mem_cap_bytes = 2LL << 30, time_cap_ms = 2000;
};

[[noreturn]] void usage(int code) {
    std::cerr << "usage: laplex_bench <bench-matvec|accuracy|bench-gram> [--n-min N] [--n-max N] [--k K]\n"
                 "       [--batch B] [--trials T] [--warmups W] [--seed S] [--precision f32|f64]\n"
                 "       [--methods laplex,dense] [--mem-cap-bytes X] [--time-cap-ms X] [--gram-n N] [--out PATH]\n";
    std::exit(code);
}

std::vector<std::size_t> pow2_sweep(std::size_t lo, std::size_t hi) {
    auto p2 = [](std::size_t v) { return v && !(v & (v - 1)); };
    if (!p2(lo) || !p2(hi) || lo > hi) throw InvalidSize("size range must be powers of two with n-min <= n-max");
    std::vector<std::size_t> v;
    for (std::size_t s = lo; s <= hi; s <<= 1) v.push_back(s);
    return v;
}

std::vector<std::string> methods_of(const std::string& s) {
    std::vector<std::string> out;
    std::stringstream ss(s);
    std::string t;
    while (std::getline(ss, t, ','))
        if (!t.empty()) out.push_back(t);
    if (out.empty()) throw std::invalid_argument("--methods list is empty");
    for (auto& m : out)
        if (m != "laplex" && m != "dense") throw std::invalid_argument("methods are laplex,dense");
    return out;
}

template <typename Real>
std::vector<Real> uniform(std::mt19937_64& g, std::size_t n, double lo = -1.0, double hi = 1.0) {
    std::uniform_real_distribution<double> d(lo, hi);
    std::vector<Real> v(n);
    for (auto& x : v) x = Real(d(g));
    return v;
}

template <typename Real>
double rel_l2(const std::vector<Real>& got, const std::vector<double>& want) {
    double num = 0, den = 0;
    for (std::size_t i = 0; i < want.size(); ++i) {
        const double d = double(got[i]) - want[i];
        num += d * d;
        den += want[i] * want[i];
    }
    return den == 0 ? std::sqrt(num) : std::sqrt(num / den);
}

// warmups, then one row per timed trial; median trial ms, or -1 past the time cap
template <typename Fn>
double trials(Csv& csv, Row row, const Opts& o, Fn&& fn) {
    for (std::size_t w = 0; w < o.warmups; ++w) fn();
    std::vector<double> ts;
    for (std::size_t t = 0; t < o.trials; ++t) {
        const double t0 = now_ns();
        fn();
        row.wall_ns = now_ns() - t0;
        row.trial = t;
        row.peak_bytes = peak_rss();
        csv.write(row);
        ts.push_back(row.wall_ns);
        if (row.wall_ns > double(o.time_cap_ms) * 1e6) return -1;
    }
    std::sort(ts.begin(), ts.end());
    return ts[ts.size() / 2] / 1e6;
}

template <typename Real>
void bench_matvec(Csv& csv, const Opts& o, const char* prec) {
    for (const auto& method : methods_of(o.methods)) {
        for (std::size_t n : pow2_sweep(o.n_min, o.n_max)) {
            const std::size_t k = o.k ? o.k : n;
            std::mt19937_64 g(o.seed);
            auto a = uniform<Real>(g, n, -100.0, 100.0);
            auto b = uniform<Real>(g, k, -100.0, 100.0);
            auto x = uniform<Real>(g, k);
            Row r;
            r.experiment = "bench-matvec";
            r.method = method;
            r.precision = prec;
            r.n = n;
            r.k = k;
            r.batch = o.batch;
            r.seed = o.seed;
            double med;
            if (method == "dense") {
                const long long bytes = (long long)n * (long long)k * sizeof(Real);
                if (bytes > o.mem_cap_bytes) {
                    std::cerr << "bench-matvec: dense cap-skipped at n=" << n << "\n";
                    continue;
                }
                std::vector<Real> K(n * k), y(n);
                for (std::size_t i = 0; i < n; ++i)
                    for (std::size_t j = 0; j < k; ++j) K[i * k + j] = std::exp(-std::abs(a[i] - b[j]));
                r.model_bytes = double(bytes) + sizeof(Real) * double(n + k);
                volatile Real sink = 0;
                med = trials(csv, r, o, [&] {
                    for (std::size_t i = 0; i < n; ++i) {
                        Real s = 0;
                        for (std::size_t j = 0; j < k; ++j) s += K[i * k + j] * x[j];
                        y[i] = s;
                    }
                    sink = sink + y[0];
                });
            } else {
                LaplexOperator<Real> op(a, b, Real(1));
                // cached plan: 12n + 8k metadata + B(4n + 4k) payload (fp32 units)
                r.model_bytes = (sizeof(Real) / 4.0) * (12.0 * n + 8.0 * k + 4.0 * (n + k));
                volatile Real sink = 0;
                med = trials(csv, r, o, [&] { sink = sink + op.matvec(x)[0]; });
            }
            if (med < 0) {
                std::cerr << "bench-matvec: " << method << " stopped at n=" << n << " (time cap)\n";
                break;
            }
        }
    }
}

// f32 device path and f32 dense row sums, both against a streamed f64 dense
// reference; one row per (method, size, batch column)
void accuracy(Csv& csv, const Opts& o) {
    for (std::size_t n : pow2_sweep(o.n_min, o.n_max)) {
        const std::size_t k = o.k ? o.k : n;
        std::mt19937_64 g(o.seed + n);
        auto a64 = uniform<double>(g, n, -3.0, 3.0);
        auto b64 = uniform<double>(g, k, -3.0, 3.0);
        std::vector<float> a32(a64.begin(), a64.end()), b32(b64.begin(), b64.end());
        LaplexOperator<float> op(a32, b32, 1.0f);
        for (std::size_t col = 0; col < o.batch; ++col) {
            auto x64 = uniform<double>(g, k);
            std::vector<float> x32(x64.begin(), x64.end());
            std::vector<double> ref(n, 0.0);
            for (std::size_t i = 0; i < n; ++i)
                for (std::size_t j = 0; j < k; ++j) ref[i] += std::exp(-std::abs(a64[i] - b64[j])) * x64[j];
            double t0 = now_ns();
            auto y = op.matvec(x32);
            const double t_gpu = now_ns() - t0;
            std::vector<float> yd(n, 0.0f);
            t0 = now_ns();
            for (std::size_t i = 0; i < n; ++i) {
                float s = 0.0f;
                for (std::size_t j = 0; j < k; ++j) s += std::exp(-std::abs(a32[i] - b32[j])) * x32[j];
                yd[i] = s;
            }
            const double t_dense = now_ns() - t0;
            Row r;
            r.experiment = "accuracy";
            r.precision = "f32";
            r.n = n;
            r.k = k;
            r.batch = o.batch;
            r.trial = col;
            r.seed = o.seed;
            r.peak_bytes = peak_rss();
            r.method = "laplex";
            r.wall_ns = t_gpu;
            r.rel_err_l2 = rel_l2(y, ref);
            csv.write(r);
            r.method = "dense";
            r.wall_ns = t_dense;
            r.rel_err_l2 = rel_l2(yd, ref);
            csv.write(r);
        }
    }
}

void bench_gram(Csv& csv, const Opts& o) {
    for (const auto& method : methods_of(o.methods)) {
        for (std::size_t k : pow2_sweep(o.n_min, o.n_max)) {
            const std::size_t n = o.gram_n;
            std::mt19937_64 g(o.seed);
            auto a = uniform<double>(g, n, -10.0, 10.0);
            auto b = uniform<double>(g, k, -10.0, 10.0);
            auto w = uniform<double>(g, k, 0.1, 1.0);
            Row r;
            r.experiment = "bench-gram";
            r.method = method;
            r.precision = "f64";
            r.n = n;
            r.k = k;
            r.seed = o.seed;
            double med;
            if (method == "dense") {
                const long long bytes = (long long)n * (long long)k * 8;
                if (bytes > o.mem_cap_bytes) {
                    std::cerr << "bench-gram: dense cap-skipped at k=" << k << "\n";
                    continue;
                }
                std::vector<double> K(n * k), M(n * n);
                for (std::size_t i = 0; i < n; ++i)
                    for (std::size_t j = 0; j < k; ++j) K[i * k + j] = std::exp(-std::abs(a[i] - b[j]));
                volatile double sink = 0;
                med = trials(csv, r, o, [&] {
                    for (std::size_t i = 0; i < n; ++i)
                        for (std::size_t j = 0; j <= i; ++j) {
                            double s = 0;
                            for (std::size_t t = 0; t < k; ++t) s += K[i * k + t] * w[t] * K[j * k + t];
                            M[i * n + j] = M[j * n + i] = s;
                        }
                    sink = sink + M[0];
                });
            } else {
                LaplexOperator<double> op(a, b, 1.0);
                r.model_bytes = 8.0 * k + 8.0 * double(n) * double(n);
                volatile double sink = 0;
                med = trials(csv, r, o, [&] { sink = sink + op.weighted_gram(w).matrix(0, 0); });
            }
            if (med < 0) {
                std::cerr << "bench-gram: " << method << " stopped at k=" << k << " (time cap)\n";
                break;
            }
        }
    }
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) usage(2);
    const std::string cmd = argv[1];
    if (cmd == "-h" || cmd == "--help") usage(0);
    if (cmd != "bench-matvec" && cmd != "accuracy" && cmd != "bench-gram") {
        std::cerr << "unknown subcommand " << cmd << "\n";
        usage(2);
    }
    Opts o;
    try {
        for (int i = 2; i < argc; ++i) {
            const std::string f = argv[i];
            if (f == "-h" || f == "--help") usage(0);
            if (i + 1 >= argc) throw std::invalid_argument("missing value for " + f);
            const std::string v = argv[++i];
            if (f == "--n-min") o.n_min = std::stoull(v);
            else if (f == "--n-max") o.n_max = std::stoull(v);
            else if (f == "--k") o.k = std::stoull(v);
            else if (f == "--batch") o.batch = std::stoull(v);
            else if (f == "--trials") o.trials = std::stoull(v);
            else if (f == "--warmups") o.warmups = std::stoull(v);
            else if (f == "--seed") o.seed = std::stoull(v);
            else if (f == "--precision") o.precision = v;
            else if (f == "--methods") o.methods = v;
            else if (f == "--mem-cap-bytes") o.mem_cap_bytes = std::stoll(v);
            else if (f == "--time-cap-ms") o.time_cap_ms = std::stoll(v);
            else if (f == "--gram-n") o.gram_n = std::stoull(v);
            else if (f == "--out") o.out = v;
            else throw std::invalid_argument("unknown flag " + f);
        }
        if (o.precision != "f32" && o.precision != "f64") throw std::invalid_argument("--precision is f32 or f64");
        if (o.trials == 0) throw std::invalid_argument("--trials must be positive");
        Csv csv(o.out);
        if (cmd == "bench-matvec") {
            if (o.precision == "f32")
                bench_matvec<float>(csv, o, "f32");
            else
                bench_matvec<double>(csv, o, "f64");
        } else if (cmd == "accuracy") {
            accuracy(csv, o);
        } else {
            bench_gram(csv, o);
        }
    } catch (const std::exception& e) {
        std::cerr << "laplex_bench: " << e.what() << "\n";
        return 1;
    }
    return 0;
}
