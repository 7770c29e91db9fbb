// dashsvd_b200 — the reference CLI (tools/dashsvd.cpp) over the B200 library.
//
// Same subcommands, flags, report keys, CSV columns and exit codes as the
// reference front end (dashsvd.cpp:151-329, exit mapping :404-422):
//   run      load (.dsh cache or Matrix Market, both built on the GPU), solve,
//            optionally write PREFIX.S.txt / .U.mtx / .V.mtx, print the report
//   metrics  eps_pve, eps_res, eps_spec, eps_sigma of stored factors (GPU)
//   bench    parameter sweeps as long-format CSV (GPU solves and metrics)
// Exit codes: 0 ok; 2 usage / configuration / input errors (dashsvd::Error);
// 3 RankDeficient, NumericalError, DegenerateReference, HypothesisError; 1 other.
//
// Differences, all on paths the GPU build does not carry: `--reference oracle`
// (the reference's dense host Jacobi SVD) and the dense1/dense2 synthetic
// families exit with a ConfigError (2). Timing keys come from the device:
// iterate_seconds is the solve minus its finalize (device-timed finalize and
// D2H), as the reference splits at its last observer callback.
//
// The flag parser is a small restatement of the CLI11 behaviour the reference
// relies on (options with values, --opt=value, comma lists, negatable flag,
// required options, mutually exclusive options); CLI11 itself is not vendored.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "dashsvd_b200.hpp"

namespace {

using Clock = std::chrono::steady_clock;

double seconds_between(Clock::time_point a, Clock::time_point b) {
    return std::chrono::duration<double>(b - a).count();
}

// ---- flag parsing -------------------------------------------------------------------

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct Spec {
    std::string name;  // without the leading dashes
    bool takes_value = true;
    bool required = false;
    bool list = false;
    std::string help;
};

struct Parsed {
    std::map<std::string, std::vector<std::string>> values;
    std::set<std::string> seen;
    bool has(const std::string& n) const { return seen.count(n) > 0; }
    const std::string& one(const std::string& n) const { return values.at(n).back(); }
};

Parsed parse_flags(const std::vector<Spec>& specs, const std::vector<std::string>& args,
                   const std::vector<std::pair<std::string, std::string>>& excludes) {
    Parsed p;
    for (std::size_t i = 0; i < args.size(); ++i) {
        std::string a = args[i];
        if (a.rfind("--", 0) != 0) throw UsageError("The following argument was not expected: " + a);
        std::string name = a.substr(2), value;
        bool inline_value = false;
        const auto eq = name.find('=');
        if (eq != std::string::npos) {
            value = name.substr(eq + 1);
            name = name.substr(0, eq);
            inline_value = true;
        }
        const Spec* spec = nullptr;
        for (const Spec& s : specs)
            if (s.name == name) spec = &s;
        if (!spec) throw UsageError("The following argument was not expected: " + a);
        if (spec->takes_value) {
            if (!inline_value) {
                if (i + 1 >= args.size()) throw UsageError("--" + name + ": 1 required TEXT missing");
                value = args[++i];
            }
            if (spec->list) {
                std::size_t start = 0;
                while (true) {
                    const auto comma = value.find(',', start);
                    p.values[name].push_back(value.substr(start, comma - start));
                    if (comma == std::string::npos) break;
                    start = comma + 1;
                }
            } else {
                p.values[name].push_back(value);
            }
        } else {
            if (inline_value) throw UsageError("--" + name + " does not take a value");
            p.values[name].push_back("1");
        }
        p.seen.insert(name);
    }
    for (const auto& ex : excludes)
        if (p.has(ex.first) && p.has(ex.second))
            throw UsageError("--" + ex.first + " excludes --" + ex.second);
    for (const Spec& s : specs)
        if (s.required && !p.has(s.name)) throw UsageError("--" + s.name + " is required");
    return p;
}

int64_t to_int(const std::string& flag, const std::string& v) {
    char* end = nullptr;
    const long long x = std::strtoll(v.c_str(), &end, 10);
    if (v.empty() || *end != '\0') throw UsageError("Could not convert: --" + flag + " = " + v);
    return x;
}
uint64_t to_uint(const std::string& flag, const std::string& v) {
    char* end = nullptr;
    if (!v.empty() && v[0] == '-') throw UsageError("Could not convert: --" + flag + " = " + v);
    const unsigned long long x = std::strtoull(v.c_str(), &end, 10);
    if (v.empty() || *end != '\0') throw UsageError("Could not convert: --" + flag + " = " + v);
    return x;
}
double to_double(const std::string& flag, const std::string& v) {
    char* end = nullptr;
    const double x = std::strtod(v.c_str(), &end);
    if (v.empty() || *end != '\0') throw UsageError("Could not convert: --" + flag + " = " + v);
    return x;
}

void print_help(const char* title, const std::vector<Spec>& specs) {
    std::printf("%s\nOptions:\n  --help  print this message and exit\n", title);
    for (const Spec& s : specs)
        std::printf("  --%s%s  %s%s\n", s.name.c_str(), s.takes_value ? " VALUE" : "", s.help.c_str(),
                    s.required ? " (required)" : "");
}

// ---- shared helpers (dashsvd.cpp:29-121) ------------------------------------------------

dashsvd::Algorithm parse_alg(const std::string& name) {
    static const std::map<std::string, dashsvd::Algorithm> table{
        {"basic", dashsvd::Algorithm::basic},
        {"shifted", dashsvd::Algorithm::shifted},
        {"fixed-shift", dashsvd::Algorithm::fixed_shift},
        {"fixed_shift", dashsvd::Algorithm::fixed_shift},
        {"dash", dashsvd::Algorithm::dash},
    };
    auto it = table.find(name);
    if (it == table.end())
        throw dashsvd::ConfigError("unknown algorithm '" + name +
                                   "' (expected basic, shifted, fixed-shift or dash)");
    return it->second;
}

const char* alg_name(dashsvd::Algorithm alg) {
    switch (alg) {
        case dashsvd::Algorithm::basic: return "basic";
        case dashsvd::Algorithm::shifted: return "shifted";
        case dashsvd::Algorithm::fixed_shift: return "fixed-shift";
        case dashsvd::Algorithm::dash: return "dash";
    }
    return "?";
}

const char* stop_name(dashsvd::StopReason r) {
    switch (r) {
        case dashsvd::StopReason::fixed_p: return "fixed_p";
        case dashsvd::StopReason::tol_met: return "tol_met";
        case dashsvd::StopReason::p_max_reached: return "p_max_reached";
    }
    return "?";
}

// flag > DASHSVD_THREADS > all cores; host threads only (the solve runs on the GPU)
int resolve_threads(int flag_value) {
    if (flag_value > 0) return flag_value;
    const char* env = std::getenv("DASHSVD_THREADS");
    if (!env || !*env) return static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    char* end = nullptr;
    const long v = std::strtol(env, &end, 10);
    if (*end != '\0' || v < 1)
        throw dashsvd::ConfigError("DASHSVD_THREADS must be a positive integer, got '" + std::string(env) + "'");
    return static_cast<int>(v);
}

// --synthetic sparse:R:C:NPR (dashsvd.cpp:86-121); dense1/dense2 are not carried
dashsvd::SparseMatrix make_synthetic(const std::string& spec) {
    const auto bad = [&]() {
        throw dashsvd::ConfigError("bad --synthetic spec '" + spec +
                                   "' (expected dense1:N, dense2:N or sparse:R:C:NPR)");
    };
    std::vector<std::string> parts;
    std::size_t start = 0;
    while (true) {
        const std::size_t colon = spec.find(':', start);
        parts.push_back(spec.substr(start, colon - start));
        if (colon == std::string::npos) break;
        start = colon + 1;
    }
    auto as_count = [&](const std::string& s) -> dashsvd::index_t {
        char* end = nullptr;
        const long long v = std::strtoll(s.c_str(), &end, 10);
        if (s.empty() || *end != '\0' || v < 1) bad();
        return static_cast<dashsvd::index_t>(v);
    };
    if ((parts[0] == "dense1" || parts[0] == "dense2") && parts.size() == 2) {
        as_count(parts[1]);
        throw dashsvd::ConfigError("--synthetic " + parts[0] +
                                   " (dense test matrices) is not available in the B200 build; use sparse:R:C:NPR");
    }
    if (parts[0] == "sparse" && parts.size() == 4)
        return dashsvd::sparse_random(as_count(parts[1]), as_count(parts[2]), as_count(parts[3]), 0, true);
    bad();
    return {};
}

dashsvd::ReferenceSpectrum reference_for(const std::string& flag) {
    if (flag.empty() || flag == "oracle")
        throw dashsvd::ConfigError(
            "--reference oracle (the host dense Jacobi SVD) is not available in the B200 build; pass a spectrum "
            "file");
    return dashsvd::load_reference_spectrum(flag);
}

// ---- run (dashsvd.cpp:150-223) ------------------------------------------------------------

const std::vector<Spec> kRunSpecs = {
    {"input", true, true, false, "Matrix Market file (.mtx) or CSR cache (.dsh)"},
    {"k", true, true, false, "target rank"},
    {"s", true, false, false, "oversampling (default k/2)"},
    {"p", true, false, false, "power-iteration count (basic/shifted)"},
    {"tol", true, false, false, "accuracy tolerance (dash)"},
    {"pmax", true, false, false, "iteration cap (dash)"},
    {"alg", true, false, false, "basic | shifted | fixed-shift | dash (default dash)"},
    {"orth", true, false, false, "eigsvd | qr (basic only; default eigsvd)"},
    {"seed", true, false, false, "sketch seed (default 0)"},
    {"threads", true, false, false, "host threads (default: DASHSVD_THREADS or all)"},
    {"deterministic", false, false, false, "bitwise reproducible runs (default on)"},
    {"no-deterministic", false, false, false, "accepted for compatibility (runs stay deterministic)"},
    {"out-prefix", true, false, false, "write PREFIX.S.txt, PREFIX.U.mtx, PREFIX.V.mtx"},
};

int cmd_run(const Parsed& f) {
    dashsvd::SolverConfig cfg;
    const std::string input = f.one("input");
    cfg.k = to_int("k", f.one("k"));
    if (f.has("s")) cfg.s = to_int("s", f.one("s"));
    if (f.has("p")) cfg.p = to_int("p", f.one("p"));
    if (f.has("tol")) cfg.tol = to_double("tol", f.one("tol"));
    if (f.has("pmax")) cfg.p_max = to_int("pmax", f.one("pmax"));
    const std::string alg = f.has("alg") ? f.one("alg") : "dash";
    const std::string orth = f.has("orth") ? f.one("orth") : "eigsvd";
    if (f.has("seed")) cfg.seed = to_uint("seed", f.one("seed"));
    const int threads_flag = f.has("threads") ? static_cast<int>(to_int("threads", f.one("threads"))) : 0;
    if (f.has("deterministic") && f.has("no-deterministic"))
        throw UsageError("--deterministic excludes --no-deterministic");
    cfg.deterministic = !f.has("no-deterministic");
    const std::string out_prefix = f.has("out-prefix") ? f.one("out-prefix") : "";
    cfg.alg = parse_alg(alg);
    if (orth == "eigsvd") cfg.orth = dashsvd::Orthonormalizer::eigsvd;
    else if (orth == "qr") cfg.orth = dashsvd::Orthonormalizer::qr;
    else throw dashsvd::ConfigError("unknown orthonormalizer '" + orth + "'");
    if (cfg.alg == dashsvd::Algorithm::dash) {
        if (f.has("p")) throw dashsvd::ConfigError("--p applies to fixed-power algorithms; dash uses --tol");
    } else if (f.has("tol") || f.has("pmax")) {
        throw dashsvd::ConfigError("--tol/--pmax apply to the dash algorithm only");
    }
    const int threads = resolve_threads(threads_flag);

    const auto t0 = Clock::now();
    const dashsvd::b200::DeviceMatrix a = dashsvd::b200::DeviceMatrix::load(input);
    const auto t_loaded = Clock::now();
    dsvd_stats stats{};
    dashsvd::SolveResult r = a.solve(cfg, &stats);
    const auto t_solved = Clock::now();
    const double solve_s = seconds_between(t_loaded, t_solved);
    const double finalize_s = std::min(solve_s, (stats.finalize_ms + stats.d2h_ms) * 1e-3);

    std::string s_file, u_file, v_file;
    if (!out_prefix.empty()) {
        s_file = out_prefix + ".S.txt";
        u_file = out_prefix + ".U.mtx";
        v_file = out_prefix + ".V.mtx";
        dashsvd::write_reference_spectrum(s_file, r.svd.s);
        dashsvd::write_dense_array(u_file, r.svd.u);
        dashsvd::write_dense_array(v_file, r.svd.v);
    }
    const auto t_end = Clock::now();

    std::printf("matrix: %s\n", input.c_str());
    std::printf("rows: %lld\n", static_cast<long long>(a.rows()));
    std::printf("cols: %lld\n", static_cast<long long>(a.cols()));
    std::printf("nnz: %lld\n", static_cast<long long>(a.nnz()));
    std::printf("alg: %s\n", alg_name(cfg.alg));
    std::printf("k: %lld\n", static_cast<long long>(cfg.k));
    std::printf("s: %lld\n", static_cast<long long>(cfg.effective_s(cfg.k)));
    std::printf("l: %lld\n", static_cast<long long>(cfg.sketch_width()));
    if (cfg.alg == dashsvd::Algorithm::dash) {
        std::printf("tol: %.17g\n", cfg.tol);
        std::printf("p_max: %lld\n", static_cast<long long>(cfg.p_max));
    } else {
        std::printf("p: %lld\n", static_cast<long long>(cfg.p));
    }
    std::printf("orth: %s\n", orth.c_str());
    std::printf("seed: %llu\n", static_cast<unsigned long long>(cfg.seed));
    std::printf("threads: %d\n", threads);
    std::printf("deterministic: %s\n", cfg.deterministic ? "true" : "false");
    std::printf("load_seconds: %.6f\n", seconds_between(t0, t_loaded));
    std::printf("iterate_seconds: %.6f\n", solve_s - finalize_s);
    std::printf("finalize_seconds: %.6f\n", finalize_s);
    std::printf("total_seconds: %.6f\n", seconds_between(t0, t_end));
    std::printf("iterations: %lld\n", static_cast<long long>(r.trace.iterations));
    std::printf("stop_reason: %s\n", stop_name(r.trace.stop_reason));
    std::printf("alphas:");
    for (double alpha : r.trace.alphas) std::printf(" %.17g", alpha);
    std::printf("\n");
    std::printf("sigma:");
    for (double s : r.svd.s) std::printf(" %.17g", s);
    std::printf("\n");
    std::printf("max_triplet_residual: %.6e\n", dashsvd::max_triplet_residual(a, r.svd));
    if (!out_prefix.empty()) {
        std::printf("s_file: %s\n", s_file.c_str());
        std::printf("u_file: %s\n", u_file.c_str());
        std::printf("v_file: %s\n", v_file.c_str());
    }
    return 0;
}

// ---- metrics (dashsvd.cpp:225-255) ----------------------------------------------------------

const std::vector<Spec> kMetricsSpecs = {
    {"input", true, true, false, "matrix the factors approximate"},
    {"factors", true, true, false, "prefix written by run --out-prefix"},
    {"reference", true, true, false, "spectrum file ('oracle' is not available on the GPU build)"},
    {"power-iters", true, false, false, "spectral-norm power iterations (default 300)"},
    {"threads", true, false, false, "host threads"},
};

int cmd_metrics(const Parsed& f) {
    const int64_t power_iters = f.has("power-iters") ? to_int("power-iters", f.one("power-iters")) : 300;
    resolve_threads(f.has("threads") ? static_cast<int>(to_int("threads", f.one("threads"))) : 0);
    const dashsvd::b200::DeviceMatrix a = dashsvd::b200::DeviceMatrix::load(f.one("input"));
    dashsvd::TruncatedSvd approx;
    const std::string prefix = f.one("factors");
    approx.u = dashsvd::load_dense_array(prefix + ".U.mtx");
    approx.v = dashsvd::load_dense_array(prefix + ".V.mtx");
    approx.s = dashsvd::load_reference_spectrum(prefix + ".S.txt").sigmas;
    const dashsvd::ReferenceSpectrum ref = reference_for(f.one("reference"));
    const double pve = dashsvd::eps_pve(a, approx.u, ref);
    const double res = dashsvd::eps_res(a, approx, ref);
    const double spec = dashsvd::eps_spec(a, approx, ref, power_iters);
    const double sig = dashsvd::eps_sigma(approx.s, ref);
    std::printf("eps_pve,eps_res,eps_spec,eps_sigma\n");
    std::printf("%.9e,%.9e,%.9e,%.9e\n", pve, res, spec, sig);
    return 0;
}

// ---- bench (dashsvd.cpp:257-329) ------------------------------------------------------------

const std::vector<Spec> kBenchSpecs = {
    {"input", true, false, false, "matrix file"},
    {"synthetic", true, false, false, "sparse:R:C:NPR instead of --input"},
    {"reference", true, false, false, "spectrum file"},
    {"k", true, true, false, "target rank"},
    {"s", true, false, false, "oversampling (default k/2)"},
    {"alg", true, true, true, "algorithms to sweep (comma separated)"},
    {"p-list", true, false, true, "power counts to sweep"},
    {"tol-list", true, false, true, "tolerances to sweep"},
    {"repeats", true, false, false, "seeds per configuration (default 1)"},
    {"seed-base", true, false, false, "first seed (default 1)"},
    {"threads", true, false, false, "host threads"},
};

int cmd_bench(const Parsed& f) {
    resolve_threads(f.has("threads") ? static_cast<int>(to_int("threads", f.one("threads"))) : 0);
    const int64_t k = to_int("k", f.one("k"));
    const int64_t s = f.has("s") ? to_int("s", f.one("s")) : -1;
    const int64_t repeats = f.has("repeats") ? to_int("repeats", f.one("repeats")) : 1;
    const uint64_t seed_base = f.has("seed-base") ? to_uint("seed-base", f.one("seed-base")) : 1;
    std::vector<int64_t> p_list;
    std::vector<double> tol_list;
    if (f.has("p-list"))
        for (const auto& v : f.values.at("p-list")) p_list.push_back(to_int("p-list", v));
    if (f.has("tol-list"))
        for (const auto& v : f.values.at("tol-list")) tol_list.push_back(to_double("tol-list", v));

    const dashsvd::b200::DeviceMatrix a = f.has("synthetic")
                                              ? dashsvd::b200::DeviceMatrix(make_synthetic(f.one("synthetic")))
                                              : dashsvd::b200::DeviceMatrix::load(f.has("input") ? f.one("input")
                                                                                                 : std::string());
    const dashsvd::ReferenceSpectrum ref = reference_for(f.has("reference") ? f.one("reference") : "");
    if (p_list.empty() == tol_list.empty())
        throw dashsvd::ConfigError("exactly one of --p-list and --tol-list is required");

    std::printf("alg,param,seed,time_s,iterations,stop_reason,eps_pve,eps_res,eps_spec,eps_sigma\n");
    for (const std::string& alg_str : f.values.at("alg")) {
        const dashsvd::Algorithm alg = parse_alg(alg_str);
        const bool fixed_power = alg != dashsvd::Algorithm::dash;
        if (fixed_power && p_list.empty())
            throw dashsvd::ConfigError("algorithm '" + alg_str + "' sweeps --p-list");
        if (!fixed_power && tol_list.empty()) throw dashsvd::ConfigError("algorithm 'dash' sweeps --tol-list");
        const std::size_t params = fixed_power ? p_list.size() : tol_list.size();
        for (std::size_t pi = 0; pi < params; ++pi) {
            for (int64_t rep = 0; rep < repeats; ++rep) {
                dashsvd::SolverConfig cfg;
                cfg.alg = alg;
                cfg.k = k;
                cfg.s = s;
                cfg.seed = seed_base + static_cast<uint64_t>(rep);
                char param_text[64];
                if (fixed_power) {
                    cfg.p = p_list[pi];
                    std::snprintf(param_text, sizeof param_text, "%lld", static_cast<long long>(cfg.p));
                } else {
                    cfg.tol = tol_list[pi];
                    std::snprintf(param_text, sizeof param_text, "%g", cfg.tol);
                }
                const auto t0 = Clock::now();
                dashsvd::SolveResult r = a.solve(cfg);
                const double elapsed = seconds_between(t0, Clock::now());
                const double pve = dashsvd::eps_pve(a, r.svd.u, ref);
                const double res = dashsvd::eps_res(a, r.svd, ref);
                const double spec = dashsvd::eps_spec(a, r.svd, ref);
                const double sig = dashsvd::eps_sigma(r.svd.s, ref);
                std::printf("%s,%s,%llu,%.6f,%lld,%s,%.9e,%.9e,%.9e,%.9e\n", alg_name(alg), param_text,
                            static_cast<unsigned long long>(cfg.seed), elapsed,
                            static_cast<long long>(r.trace.iterations), stop_name(r.trace.stop_reason), pve, res,
                            spec, sig);
            }
        }
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    const char* title = "randomized truncated SVD for large sparse matrices (B200)";
    std::vector<std::string> args(argv + 1, argv + argc);
    if (args.empty() || args[0] == "--help" || args[0] == "-h") {
        std::printf("%s\nSubcommands:\n  run      factor a matrix and write the results\n"
                    "  metrics  error metrics of stored factors\n  bench    parameter sweeps as long-format CSV\n",
                    title);
        if (args.empty()) {
            std::fprintf(stderr, "A subcommand is required\n");
            return 2;
        }
        return 0;
    }
    const std::string sub = args[0];
    const std::vector<std::string> rest(args.begin() + 1, args.end());
    const std::vector<Spec>* specs = sub == "run" ? &kRunSpecs
                                     : sub == "metrics" ? &kMetricsSpecs
                                     : sub == "bench" ? &kBenchSpecs
                                                      : nullptr;
    if (!specs) {
        std::fprintf(stderr, "The following argument was not expected: %s\nRun with --help for more information.\n",
                     sub.c_str());
        return 2;
    }
    for (const auto& a : rest)
        if (a == "--help" || a == "-h") {
            print_help(sub.c_str(), *specs);
            return 0;
        }
    Parsed parsed;
    try {
        std::vector<std::pair<std::string, std::string>> excludes;
        if (sub == "run") excludes = {{"p", "tol"}};
        if (sub == "bench") excludes = {{"input", "synthetic"}, {"p-list", "tol-list"}};
        parsed = parse_flags(*specs, rest, excludes);
    } catch (const UsageError& e) {
        std::fprintf(stderr, "%s\nRun with --help for more information.\n", e.what());
        return 2;
    }
    try {
        if (sub == "run") return cmd_run(parsed);
        if (sub == "metrics") return cmd_metrics(parsed);
        return cmd_bench(parsed);
    } catch (const UsageError& e) {
        std::fprintf(stderr, "%s\nRun with --help for more information.\n", e.what());
        return 2;
    } catch (const dashsvd::RankDeficient& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 3;
    } catch (const dashsvd::NumericalError& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 3;
    } catch (const dashsvd::DegenerateReference& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 3;
    } catch (const dashsvd::HypothesisError& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 3;
    } catch (const dashsvd::Error& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
