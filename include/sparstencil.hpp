// sparstencil.hpp — header-only C++ drop-in for the reference's stencil sweep.
//
// Reference (proj/core/include/stensor/stencil.hpp:72):
//     Grid direct_apply(const StencilSpec& spec, const Grid& grid, std::uint64_t steps);
// Engine:
//     Grid sst::sparse_apply(const StencilSpec& spec, const Grid& grid, std::uint64_t steps);
//
// Templated on the caller's own StencilSpec / Grid types (the reference's
// stensor:: types, or this engine's identical ones): the spec is written out as a
// spec document (docs/formats.md:3-30) and compiled by sst_compile, the sweep runs
// on the B200 through the C ABI (sparstencil.h), and the result is the valid
// region, extent N - steps*(k-1) per axis, like direct_apply's. Status codes come
// back as the reference's exception types (std::invalid_argument, std::logic_error,
// std::out_of_range, std::runtime_error). No CPU fallback: no device throws.
#ifndef SPARSTENCIL_HPP_
#define SPARSTENCIL_HPP_

#include <cstdint>
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "sparstencil.h"

namespace sst {

inline void check(sst_status s) {
    if (s == SST_OK) return;
    const std::string msg = sst_last_error();
    switch (s) {
        case SST_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case SST_ERR_LOGIC: throw std::logic_error(msg);
        case SST_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
        default: throw std::runtime_error(msg);
    }
}

// Spec document of a StencilSpec-like value: name, dims, shape (enum: star first),
// k and points {off[3], weight}; weights printed to round-trip exactly.
template <class StencilSpec>
std::string spec_document(const StencilSpec& spec) {
    std::string doc = "name = " + std::string(spec.name.empty() ? "stencil" : spec.name) + "\n";
    doc += "dims = " + std::to_string(spec.dims) + "\n";
    doc += std::string("shape = ") + (static_cast<int>(spec.shape) == 0 ? "star" : "box") + "\n";
    doc += "k = " + std::to_string(spec.k) + "\n";
    for (const auto& pt : spec.points) {
        doc += "point =";
        for (int a = 0; a < spec.dims; ++a) doc += " " + std::to_string(pt.off[static_cast<std::size_t>(a)]);
        char w[40];
        std::snprintf(w, sizeof w, " : %.17g\n", static_cast<double>(pt.weight));
        doc += w;
    }
    return doc;
}

enum class Precision { f16 = SST_PREC_F16, f16x2 = SST_PREC_F16X2 };

template <class StencilSpec, class Grid>
Grid sparse_apply(const StencilSpec& spec, const Grid& grid, std::uint64_t steps, int device = 0,
                  Precision precision = Precision::f16) {
    if (steps == 0) throw std::invalid_argument("steps must be >= 1");
    if (grid.dims.size() != static_cast<std::size_t>(spec.dims))
        throw std::invalid_argument("grid dimensionality does not match stencil");
    const std::size_t k = static_cast<std::size_t>(spec.k), shrink = steps * (k - 1);
    std::vector<std::uint64_t> dims(grid.dims.begin(), grid.dims.end());
    std::size_t cells = 1;
    for (auto d : dims) {
        if (d < k + shrink - (k - 1)) throw std::invalid_argument("grid smaller than kernel");
        cells *= static_cast<std::size_t>(d);
    }
    if (grid.values.size() != cells) throw std::invalid_argument("grid values do not match its dims");

    const std::string doc = spec_document(spec);
    sst_compiled* c = nullptr;
    check(sst_compile(doc.c_str(), dims.data(), static_cast<int>(dims.size()), 16, 8, 1, &c));
    std::unique_ptr<sst_compiled, void (*)(sst_compiled*)> cg(c, sst_compiled_destroy);
    sst_plan_desc desc;
    check(sst_compiled_plan_desc(c, &desc));
    desc.precision = static_cast<int32_t>(precision);
    sst_plan* p = nullptr;
    check(sst_plan_create(&desc, device, &p));
    std::unique_ptr<sst_plan, void (*)(sst_plan*)> pg(p, sst_plan_destroy);

    std::vector<float> in(grid.values.begin(), grid.values.end()), out(cells);
    check(sst_apply_host(p, in.data(), out.data(), steps));

    // the valid region [steps*r, N - steps*r) of every axis (row-major)
    const std::size_t c0 = shrink / 2, nd = dims.size();
    Grid res = grid;
    res.dims.clear();
    for (auto d : dims) res.dims.push_back(static_cast<std::size_t>(d) - shrink);
    std::size_t n_out = 1;
    for (auto d : res.dims) n_out *= d;
    res.values.assign(n_out, 0.0);
    std::vector<std::size_t> idx(nd, 0);
    for (std::size_t flat = 0; flat < n_out; ++flat) {
        std::size_t rem = flat, src = 0;
        for (std::size_t a = nd; a-- > 0;) {
            idx[a] = rem % res.dims[a];
            rem /= res.dims[a];
        }
        for (std::size_t a = 0; a < nd; ++a) src = src * static_cast<std::size_t>(dims[a]) + idx[a] + c0;
        res.values[flat] = static_cast<double>(out[src]);
    }
    return res;
}

// The same sweep slab-decomposed along the slowest axis over devices.size() slabs
// (sst_run_steps_multi; several slabs may share a GPU, neighbours on different GPUs
// must be peer-accessible): bitwise the single-domain result.
template <class StencilSpec, class Grid>
Grid sparse_apply_multi(const StencilSpec& spec, const Grid& grid, std::uint64_t steps,
                        const std::vector<int>& devices, Precision precision = Precision::f16) {
    if (steps == 0) throw std::invalid_argument("steps must be >= 1");
    if (devices.empty()) throw std::invalid_argument("need at least one device");
    if (grid.dims.size() != static_cast<std::size_t>(spec.dims))
        throw std::invalid_argument("grid dimensionality does not match stencil");
    const std::size_t k = static_cast<std::size_t>(spec.k), shrink = steps * (k - 1);
    std::vector<std::uint64_t> dims(grid.dims.begin(), grid.dims.end());
    std::size_t cells = 1;
    for (auto d : dims) {
        if (d < k + shrink - (k - 1)) throw std::invalid_argument("grid smaller than kernel");
        cells *= static_cast<std::size_t>(d);
    }
    if (grid.values.size() != cells) throw std::invalid_argument("grid values do not match its dims");
    const std::string doc = spec_document(spec);
    sst_compiled* c = nullptr;
    check(sst_compile(doc.c_str(), dims.data(), static_cast<int>(dims.size()), 16, 8, 1, &c));
    std::unique_ptr<sst_compiled, void (*)(sst_compiled*)> cg(c, sst_compiled_destroy);
    sst_plan_desc desc;
    check(sst_compiled_plan_desc(c, &desc));
    desc.precision = static_cast<int32_t>(precision);
    std::vector<float> in(grid.values.begin(), grid.values.end()), out(cells);
    check(sst_run_steps_multi(&desc, static_cast<int>(devices.size()), devices.data(), in.data(), out.data(),
                              steps));
    const std::size_t c0 = shrink / 2, nd = dims.size();
    Grid res = grid;
    res.dims.clear();
    for (auto d : dims) res.dims.push_back(static_cast<std::size_t>(d) - shrink);
    std::size_t n_out = 1;
    for (auto d : res.dims) n_out *= d;
    res.values.assign(n_out, 0.0);
    std::vector<std::size_t> idx(nd, 0);
    for (std::size_t flat = 0; flat < n_out; ++flat) {
        std::size_t rem = flat, src = 0;
        for (std::size_t a = nd; a-- > 0;) {
            idx[a] = rem % res.dims[a];
            rem /= res.dims[a];
        }
        for (std::size_t a = 0; a < nd; ++a) src = src * static_cast<std::size_t>(dims[a]) + idx[a] + c0;
        res.values[flat] = static_cast<double>(out[src]);
    }
    return res;
}

}  // namespace sst

#endif  // SPARSTENCIL_HPP_
