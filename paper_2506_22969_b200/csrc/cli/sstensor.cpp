// sstensor — command-line front end, drop-in for the reference CLI
// (proj/tools/main.cpp:75-193; the reference uses CLI11, absent here, so the
// option parser is a small hand-written one with the same subcommands, options,
// defaults, output lines and exit codes: 0 ok, 1 verification failure, 2 error).
//
//   sstensor compile --stencil S --grid 64x64 [--hw H] [--r1 N --r2 N] [--fuse T]
//                    [--precision exact64|round16] [--seed N] [--out DIR] [--no-verify]
//                    [--device D]
//   sstensor explore --stencil S --grid G [--hw H] [--fuse T] [--csv FILE]
//   sstensor verify  [--hw H] [--precision P] [--seed N] [--device D]
//   sstensor presets
//   sstensor run     --stencil S --grid G --steps T [--fuse F] [--seed N] [--device D]
//                    (engine extension: the B200 time loop, GStencil/s)
//   sstensor model   --stencil S --grid G [--fuse T] [--storage f16|f32] [--tyb N]
//                    (engine extension: the B200 execution model of one launch,
//                    hwmodel.hpp estimate_device; no device needed)
//
// compile / verify run the desk-scale verification on the GPU (the reference
// emulates it on the CPU); --no-verify skips it.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "sparstencil.h"
#include "stensor/hwmodel.hpp"
#include "stensor/pipeline.hpp"
#include "stensor/spec.hpp"

namespace {

struct Args {
    std::string cmd;
    std::map<std::string, std::string> opt;
    std::set<std::string> flags;
    bool has(const std::string& k) const { return opt.count(k) != 0; }
    std::string get(const std::string& k, const std::string& def = "") const {
        auto it = opt.find(k);
        return it == opt.end() ? def : it->second;
    }
};

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

Args parse(int argc, char** argv) {
    static const std::map<std::string, std::set<std::string>> kOpts = {
        {"compile", {"stencil", "grid", "hw", "fuse", "precision", "seed", "r1", "r2", "out", "device"}},
        {"explore", {"stencil", "grid", "hw", "fuse", "precision", "seed", "csv"}},
        {"verify", {"hw", "precision", "seed", "device"}},
        {"presets", {}},
        {"run", {"stencil", "grid", "steps", "fuse", "seed", "device"}},
        {"model", {"stencil", "grid", "fuse", "storage", "tyb"}},
    };
    static const std::map<std::string, std::set<std::string>> kFlags = {
        {"compile", {"corrupt-permutation", "no-verify"}}, {"verify", {"no-verify"}}};
    if (argc < 2) throw UsageError("a subcommand is required: compile | explore | verify | presets | run | model");
    Args a;
    a.cmd = argv[1];
    if (!kOpts.count(a.cmd)) throw UsageError("unknown subcommand: " + a.cmd);
    for (int i = 2; i < argc; ++i) {
        std::string t = argv[i];
        if (t.rfind("--", 0) != 0) throw UsageError("unexpected argument: " + t);
        t = t.substr(2);
        std::string val;
        const auto eq = t.find('=');
        const bool inline_val = eq != std::string::npos;
        if (inline_val) {
            val = t.substr(eq + 1);
            t = t.substr(0, eq);
        }
        if (kFlags.count(a.cmd) && kFlags.at(a.cmd).count(t)) {
            a.flags.insert(t);
            continue;
        }
        if (!kOpts.at(a.cmd).count(t)) throw UsageError("unknown option --" + t + " for " + a.cmd);
        if (!inline_val) {
            if (i + 1 >= argc) throw UsageError("option --" + t + " needs a value");
            val = argv[++i];
        }
        a.opt[t] = val;
    }
    return a;
}

std::string slurp(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot read " + path);
    std::ostringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

stensor::StencilSpec load_stencil(const std::string& arg) {
    if (stensor::is_preset(arg)) return stensor::stencil_preset(arg);
    return stensor::parse_stencil_spec(slurp(arg));
}

stensor::HardwareDescriptor load_hw(const std::string& arg) {
    for (const auto& n : stensor::hw_preset_names())
        if (n == arg) return stensor::hw_preset(arg);
    return stensor::parse_hw_descriptor(slurp(arg));
}

std::vector<std::size_t> parse_grid(const std::string& arg) {
    std::vector<std::size_t> dims;
    std::string tok;
    for (char c : arg + ",") {
        if (c == ',' || c == 'x' || c == 'X') {
            if (!tok.empty()) dims.push_back(std::stoull(tok));
            tok.clear();
        } else {
            tok += c;
        }
    }
    if (dims.empty() || dims.size() > 3) throw std::runtime_error("grid must list 1-3 extents, e.g. 64x64");
    return dims;
}

stensor::Precision parse_precision(const std::string& p) {
    if (p == "exact64") return stensor::Precision::exact64;
    if (p == "round16") return stensor::Precision::round16;
    throw std::runtime_error("precision must be exact64 or round16");
}

void print_candidates(std::ostream& out, const std::vector<stensor::PerfEstimate>& ranked, bool csv) {
    if (csv)
        out << "r1,r2,t_compute,t_memory,t_total,n_mma,m_prime,k_prime,n_prime\n";
    else
        std::printf("%4s %4s %14s %14s %14s %12s\n", "r1", "r2", "t_compute", "t_memory", "t_total", "n_mma");
    for (const auto& e : ranked) {
        if (csv)
            out << e.r1 << ',' << e.r2 << ',' << e.t_compute << ',' << e.t_memory << ',' << e.t_total << ','
                << e.n_mma << ',' << e.m_prime << ',' << e.k_prime << ',' << e.n_prime << '\n';
        else
            std::printf("%4d %4d %14.6e %14.6e %14.6e %12llu\n", e.r1, e.r2, e.t_compute, e.t_memory, e.t_total,
                        static_cast<unsigned long long>(e.n_mma));
    }
}

void ck(sst_status s) {
    if (s != SST_OK) throw std::runtime_error(sst_last_error());
}

int cmd_run(const Args& a) {
    if (!a.has("stencil") || !a.has("grid") || !a.has("steps")) throw UsageError("run needs --stencil --grid --steps");
    const auto dims = parse_grid(a.get("grid"));
    const std::uint64_t steps = std::stoull(a.get("steps"));
    const std::uint64_t fuse = std::stoull(a.get("fuse", "1"));
    const int device = std::stoi(a.get("device", "0"));
    const std::string st = a.get("stencil");
    const std::string text = stensor::is_preset(st) ? st : slurp(st);
    std::vector<uint64_t> d(dims.begin(), dims.end());
    sst_compiled* c = nullptr;
    ck(sst_compile(text.c_str(), d.data(), static_cast<int>(d.size()), 16, 8, fuse, &c));  // device layout (1D: folded)
    sst_plan_desc desc;
    ck(sst_compiled_plan_desc(c, &desc));
    sst_plan* p = nullptr;
    ck(sst_plan_create(&desc, device, &p));
    ck(sst_plan_bind(p, nullptr, nullptr));
    std::size_t cells = 1;
    for (auto x : dims) cells *= x;
    std::vector<float> g(cells);
    ck(sst_random_grid(static_cast<int>(d.size()), d.data(), std::stoull(a.get("seed", "1")), g.data()));
    ck(sst_upload(p, 0, g.data(), 0, nullptr));
    int dst = 0;
    ck(sst_run_steps(p, 0, fuse, nullptr, &dst));  // warm-up launch
    if (cudaDeviceSynchronize() != cudaSuccess) throw std::runtime_error("device error in warm-up");
    const auto t0 = std::chrono::steady_clock::now();
    ck(sst_run_steps(p, dst, steps, nullptr, &dst));
    if (cudaDeviceSynchronize() != cudaSuccess) throw std::runtime_error("device error");
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const auto tp = stensor::gstencil_rate(steps, dims, s);
    sst_plan_stats stats;
    ck(sst_plan_stats_get(p, &stats));
    std::printf("%s grid %s steps %llu: %.3f ms, %.2f GStencil/s (launches %llu, ctas %d)\n", st.c_str(),
                a.get("grid").c_str(), static_cast<unsigned long long>(steps), s * 1e3, tp.gstencils_per_sec,
                static_cast<unsigned long long>(stats.launches), stats.ctas);
    sst_plan_destroy(p);
    sst_compiled_destroy(c);
    return 0;
}

int cmd_model(const Args& a) {
    if (!a.has("stencil") || !a.has("grid")) throw UsageError("model needs --stencil --grid");
    const auto dims = parse_grid(a.get("grid"));
    const std::string st = a.get("stencil");
    const std::string text = stensor::is_preset(st) ? st : slurp(st);
    const std::string storage = a.get("storage", "f16");
    if (storage != "f16" && storage != "f32") throw UsageError("--storage must be f16 or f32");
    std::vector<uint64_t> d(dims.begin(), dims.end());
    double o[12];
    ck(sst_estimate_device(text.c_str(), d.data(), static_cast<int>(d.size()), std::stoull(a.get("fuse", "1")),
                           storage == "f16" ? 2 : 4, std::stoi(a.get("tyb", "0")), o));
    static const char* kBound[] = {"hbm", "smem", "tensor"};
    std::printf("updates %.0f  batches %.0f  k_pad %.0f\n", o[0], o[1], o[11]);
    std::printf("hbm %.1f MB -> %.2f us | smem %.0f wavefronts -> %.2f us | tensor %.0f issues -> %.2f us\n",
                o[2] / 1e6, o[5] * 1e6, o[3], o[6] * 1e6, o[4], o[7] * 1e6);
    std::printf("predicted %.2f us per launch, %.1f GStencil/s, bound: %s\n", o[8] * 1e6, o[9],
                kBound[static_cast<int>(o[10])]);
    return 0;
}

int run(const Args& a) {
    if (a.cmd == "presets") {
        for (const auto& n : stensor::preset_names()) {
            const auto s = stensor::stencil_preset(n);
            std::printf("%-12s dims=%d k=%d points=%zu %s\n", n.c_str(), s.dims, s.k, s.points.size(),
                        s.shape == stensor::StencilShape::star ? "star" : "box");
        }
        for (const auto& n : stensor::hw_preset_names()) std::printf("hw: %s\n", n.c_str());
        return 0;
    }
    if (a.cmd == "run") return cmd_run(a);
    if (a.cmd == "model") return cmd_model(a);
    const auto hw = load_hw(a.get("hw", "a100-sparse"));
    const auto prec = parse_precision(a.get("precision", "exact64"));
    const std::uint64_t seed = std::stoull(a.get("seed", "1"));
    const int device = std::stoi(a.get("device", "0"));
    if (a.cmd == "verify") {
        bool all_ok = true;
        for (const auto& n : stensor::preset_names()) {
            stensor::CompileRequest req;
            req.spec = stensor::stencil_preset(n);
            req.grid_dims = req.spec.dims == 1   ? std::vector<std::size_t>{256}
                            : req.spec.dims == 2 ? std::vector<std::size_t>{64, 64}
                                                 : std::vector<std::size_t>{24, 24, 24};
            req.hw = hw;
            req.precision = prec;
            req.seed = seed;
            req.r_max = 4;
            req.device = device;
            req.verify = !a.flags.count("no-verify");
            const auto res = stensor::run_compile(req);
            std::printf("%-12s %-10s max_abs=%.3e max_rel=%.3e\n", n.c_str(), res.verification.status.c_str(),
                        res.verification.max_abs_err, res.verification.max_rel_err);
            all_ok = all_ok && res.verification.status == "verified";
        }
        return all_ok ? 0 : 1;
    }
    if (!a.has("stencil") || !a.has("grid")) throw UsageError(a.cmd + " needs --stencil and --grid");
    stensor::CompileRequest req;
    req.spec = load_stencil(a.get("stencil"));
    req.grid_dims = parse_grid(a.get("grid"));
    req.hw = hw;
    req.fuse = std::stoull(a.get("fuse", "1"));
    req.precision = prec;
    req.seed = seed;
    req.device = device;
    if (a.cmd == "explore") {
        stensor::StencilSpec spec = req.spec;
        if (req.fuse > 1) spec = stensor::fuse_time_steps(spec, req.fuse);
        const auto ex = stensor::explore_layouts(req.hw, spec, req.grid_dims);
        print_candidates(std::cout, ex.ranked, false);
        if (a.has("csv")) {
            std::ofstream csv(a.get("csv"));
            print_candidates(csv, ex.ranked, true);
        }
        return 0;
    }
    const int r1 = std::stoi(a.get("r1", "0")), r2 = std::stoi(a.get("r2", "0"));
    if (r1 > 0) req.r1 = r1;
    if (r2 > 0) req.r2 = r2;
    if (r1 > 0 && r2 == 0) req.r2 = 1;
    req.out_dir = a.get("out");
    req.corrupt_permutation = a.flags.count("corrupt-permutation") != 0;
    req.verify = !a.flags.count("no-verify");
    const auto res = stensor::run_compile(req);
    std::printf("r1=%d r2=%d p=%zu n_mma=%llu issued_mma=%llu status=%s\n", res.plan.layout.r1, res.plan.layout.r2,
                res.plan.p, static_cast<unsigned long long>(res.perf.n_mma),
                static_cast<unsigned long long>(res.issued_mma), res.verification.status.c_str());
    std::printf("model: t_total=%.6e s, %.6f GStencil/s\n", res.perf.t_total, res.model_gstencil);
    if (res.emulation_seconds > 0) std::printf("device verification time: %.3f ms\n", res.emulation_seconds * 1e3);
    return res.ok ? 0 : 1;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        return run(parse(argc, argv));
    } catch (const UsageError& e) {
        std::fprintf(stderr, "usage error: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
}
