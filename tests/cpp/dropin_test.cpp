// Drop-in test (TEST INFRASTRUCTURE): a reference C++ caller switches
//     stensor::direct_apply(spec, grid, steps)            (the reference, oracle/_ref)
// to  sst::sparse_apply(spec, grid, steps)                (include/sparstencil.hpp)
// with the REFERENCE's own StencilSpec / Grid types, presets, random_grid and spec
// parser (compiled from /root/reference/proj/core, headers unchanged). 1 step must
// be bit-identical; T steps within the f16-operand tolerance 2^-11 (1 + T/4). The
// slab-decomposed sst::sparse_apply_multi (sst_run_steps_multi) must equal the
// single-domain sweep bitwise.
// Built by oracle/Makefile (target dropin) into tests/cpp/build/dropin_test.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "sparstencil.hpp"
#include "stensor/stencil.hpp"

int main() {
    int checks = 0, failures = 0;
    auto compare = [&](const std::string& what, const stensor::Grid& want, const stensor::Grid& got,
                       std::uint64_t steps) {
        ++checks;
        bool ok = want.dims == got.dims && want.values.size() == got.values.size();
        double err = 0;
        for (std::size_t i = 0; ok && i < want.values.size(); ++i)
            err = std::max(err, std::fabs(want.values[i] - got.values[i]));
        const double tol = steps == 1 ? 0.0 : std::ldexp(1.0, -11) * (1.0 + steps / 4.0);
        ok = ok && err <= tol;
        if (!ok) ++failures;
        std::printf("%-28s steps %llu  max|err| %.3g  %s\n", what.c_str(), static_cast<unsigned long long>(steps),
                    err, ok ? "ok" : "FAIL");
    };
    for (const auto& name : stensor::preset_names()) {
        const auto spec = stensor::stencil_preset(name);
        const std::vector<std::size_t> dims = spec.dims == 1   ? std::vector<std::size_t>{5003}
                                              : spec.dims == 2 ? std::vector<std::size_t>{97, 131}
                                                               : std::vector<std::size_t>{19, 23, 41};
        const auto grid = stensor::random_grid(dims, 7);
        for (std::uint64_t steps : {1ull, 3ull})
            compare(name, stensor::direct_apply(spec, grid, steps), sst::sparse_apply(spec, grid, steps), steps);
    }
    // a spec document through the reference parser
    const auto custom = stensor::parse_stencil_spec(
        "name = aniso\ndims = 2\nshape = box\nk = 3\n"
        "point = -1 -1 : 0.0625\npoint = 0 0 : 0.5\npoint = 1 1 : 0.0625\npoint = 0 1 : 0.25\n");
    const auto g = stensor::random_grid(std::vector<std::size_t>{64, 80}, 3);
    compare("custom spec", stensor::direct_apply(custom, g, 2), sst::sparse_apply(custom, g, 2), 2);
    // slab decomposition in one process (sst_run_steps_multi): 2 and 3 slabs sharing
    // device 0 must equal the single-domain sweep bitwise
    for (const char* name : {"Box-2D9P", "Star-2D13P", "Box-3D27P", "Heat-3D"}) {
        const auto spec = stensor::stencil_preset(name);
        const std::vector<std::size_t> dims =
            spec.dims == 2 ? std::vector<std::size_t>{150, 131} : std::vector<std::size_t>{40, 23, 41};
        const auto grid = stensor::random_grid(dims, 11);
        const auto one = sst::sparse_apply(spec, grid, 4);
        for (int n : {2, 3}) {
            ++checks;
            const auto multi = sst::sparse_apply_multi(spec, grid, 4, std::vector<int>(static_cast<std::size_t>(n), 0));
            const bool ok = multi.dims == one.dims && multi.values == one.values;
            if (!ok) ++failures;
            std::printf("%-28s %d slabs, 4 steps: %s\n", name, n, ok ? "bitwise equal" : "FAIL");
        }
    }
    // the reference's exception types
    ++checks;
    try {
        sst::sparse_apply(custom, g, 0);
        ++failures;
    } catch (const std::invalid_argument&) {
    }
    std::printf("%d checks, %d failures\n", checks, failures);
    return failures ? 1 : 0;
}
