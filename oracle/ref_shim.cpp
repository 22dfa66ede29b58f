// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference sources
// (/root/reference/proj/core/src/{stencil,layout,convert,emulator,perf}.cpp),
// compiled by oracle/Makefile into oracle/_ref/libstensor_ref.so. It exposes
// exactly the reference calls the checker needs:
//   ref_direct_apply   stensor::direct_apply   (stencil.cpp:231-270)
//   ref_random_grid    stensor::random_grid    (stencil.cpp:361-369)
//   ref_compile        explore/crush/convert/compress as run_compile does
//                      (pipeline.cpp:56-78, 112; codegen.cpp:94) -> .s24 bytes
//   ref_hier_match     stensor::hierarchical_match (convert.cpp:206-269)
//   ref_estimate       stensor::estimate (perf.cpp:39-70)
// Used by tests/ (golden fixtures, parity) and by bench.py's reference arm.
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "stensor/convert.hpp"
#include "stensor/emulator.hpp"
#include "stensor/layout.hpp"
#include "stensor/perf.hpp"
#include "stensor/stencil.hpp"

using namespace stensor;

namespace {
thread_local std::string g_err;

StencilSpec spec_of(const char* s) {
    const std::string t(s);
    if (is_preset(t)) return stencil_preset(t);
    return parse_stencil_spec(t);
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_random_grid(int ndims, const uint64_t* dims, uint64_t seed, double* out) {
    try {
        std::vector<std::size_t> d(dims, dims + ndims);
        const Grid g = random_grid(d, seed);
        std::memcpy(out, g.values.data(), g.values.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// out receives prod(dims - steps*(k-1)) doubles
int ref_direct_apply(const char* stencil, int ndims, const uint64_t* dims, const double* in,
                     uint64_t steps, double* out) {
    try {
        const StencilSpec spec = spec_of(stencil);
        Grid g;
        g.dims.assign(dims, dims + ndims);
        g.values.assign(in, in + g.size());
        const Grid r = direct_apply(spec, g, steps);
        std::memcpy(out, r.values.data(), r.values.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Reference sweep over `nthreads` disjoint slabs of the slowest axis, each an
// independent direct_apply call on its own (haloed) sub-grid. One step only:
// output identical to direct_apply(spec, grid, 1). The reference itself is
// single-threaded; this is how its own code is spread over the host cores.
int ref_direct_apply_slabs(const char* stencil, int ndims, const uint64_t* dims, const double* in,
                           double* out, int nthreads) {
    try {
        const StencilSpec spec = spec_of(stencil);
        const std::size_t k = static_cast<std::size_t>(spec.k);
        std::vector<std::size_t> d(dims, dims + ndims);
        const std::size_t out0 = d[0] - k + 1;
        std::size_t in_row = 1, out_row = 1;
        for (int a = 1; a < ndims; ++a) {
            in_row *= d[static_cast<std::size_t>(a)];
            out_row *= d[static_cast<std::size_t>(a)] - k + 1;
        }
        if (nthreads < 1) nthreads = 1;
        std::vector<std::thread> pool;
        std::vector<std::string> errs(static_cast<std::size_t>(nthreads));
        for (int t = 0; t < nthreads; ++t) {
            const std::size_t lo = out0 * static_cast<std::size_t>(t) / static_cast<std::size_t>(nthreads);
            const std::size_t hi = out0 * static_cast<std::size_t>(t + 1) / static_cast<std::size_t>(nthreads);
            if (hi <= lo) continue;
            pool.emplace_back([&, t, lo, hi] {
                try {
                    Grid g;
                    g.dims = d;
                    g.dims[0] = hi - lo + k - 1;
                    g.values.assign(in + lo * in_row, in + (hi + k - 1) * in_row);
                    const Grid r = direct_apply(spec, g, 1);
                    std::memcpy(out + lo * out_row, r.values.data(), r.values.size() * sizeof(double));
                } catch (const std::exception& e) {
                    errs[static_cast<std::size_t>(t)] = e.what();
                }
            });
        }
        for (auto& th : pool) th.join();
        for (const auto& e : errs)
            if (!e.empty()) {
                g_err = e;
                return 1;
            }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// info[0..7] = p, align_cols, used_blossom, refined, cols, k_prime, r1, r2
// r1 = r2 = 0 -> explore_layouts(a100-sparse, r_max) as run_compile does
int ref_compile(const char* stencil, int ndims, const uint64_t* dims, int r1, int r2, int r_max,
                uint32_t tag, uint8_t* s24, size_t cap, size_t* len, uint64_t* info,
                uint64_t* col_origin, size_t co_cap) {
    try {
        const StencilSpec spec = spec_of(stencil);
        std::vector<std::size_t> d(dims, dims + ndims);
        if (r1 <= 0 || r2 <= 0) {
            const auto ex = explore_layouts(hw_preset("a100-sparse"), spec, d, r_max, r_max);
            r1 = ex.best.r1;
            r2 = ex.best.r2;
        }
        if (spec.dims == 1) r2 = 1;
        const auto lay = crush(flatten(spec, d), r1, r2);
        const Conversion cv = convert_layout(lay);
        const Sparse24Matrix a2 = compress_24(cv.converted.a);
        std::ostringstream os(std::ios::binary);
        dump_sparse24(os, a2, tag ? Precision::round16 : Precision::exact64);
        const std::string bytes = os.str();
        *len = bytes.size();
        if (s24) {
            if (cap < bytes.size()) throw std::invalid_argument("s24 buffer too small");
            std::memcpy(s24, bytes.data(), bytes.size());
        }
        if (info) {
            info[0] = cv.p;
            info[1] = cv.align_cols;
            info[2] = cv.used_blossom ? 1 : 0;
            info[3] = cv.matching.refined ? 1 : 0;
            info[4] = cv.converted.a.cols;
            info[5] = lay.k_prime;
            info[6] = static_cast<uint64_t>(r1);
            info[7] = static_cast<uint64_t>(r2);
        }
        if (col_origin) {
            if (co_cap < cv.converted.col_origin.size()) throw std::invalid_argument("col_origin buffer too small");
            for (std::size_t i = 0; i < cv.converted.col_origin.size(); ++i)
                col_origin[i] = cv.converted.col_origin[i] == npos ? UINT64_MAX : cv.converted.col_origin[i];
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// pairs as (left, right) u64 pairs; returns count in *npairs
int ref_hier_match(uint64_t m, uint64_t g, int k, uint64_t* pairs, size_t cap, size_t* npairs,
                   uint64_t* p, int* refined) {
    try {
        const Matching mm = hierarchical_match(m, g, k);
        *npairs = mm.pairs.size();
        if (pairs) {
            if (cap < 2 * mm.pairs.size()) throw std::invalid_argument("pair buffer too small");
            for (std::size_t i = 0; i < mm.pairs.size(); ++i) {
                pairs[2 * i] = mm.pairs[i].left;
                pairs[2 * i + 1] = mm.pairs[i].right;
            }
        }
        *p = mm.zero_columns;
        *refined = mm.refined ? 1 : 0;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

int ref_estimate(const char* hw, int dims, const uint64_t* grid, int k, int r1, int r2, double* out4,
                 uint64_t* n_mma_out) {
    try {
        std::vector<std::size_t> d(grid, grid + dims);
        const auto e = estimate(hw_preset(hw), dims, d, k, r1, r2);
        out4[0] = e.t_compute;
        out4[1] = e.t_memory;
        out4[2] = e.t_total;
        out4[3] = static_cast<double>(e.n_prime);
        *n_mma_out = e.n_mma;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// the reference's own .hw parser (perf.cpp:93-134) on a descriptor text, then its
// estimate (perf.cpp:39-70): pins presets/b200-sparse.hw against the reference model
int ref_estimate_hw_text(const char* hw_text, int dims, const uint64_t* grid, int k, int r1, int r2,
                         double* out4, uint64_t* n_mma_out) {
    try {
        std::vector<std::size_t> d(grid, grid + dims);
        const auto e = estimate(parse_hw_descriptor(hw_text), dims, d, k, r1, r2);
        out4[0] = e.t_compute;
        out4[1] = e.t_memory;
        out4[2] = e.t_total;
        out4[3] = static_cast<double>(e.n_prime);
        *n_mma_out = e.n_mma;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

}  // extern "C"
