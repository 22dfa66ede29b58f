// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Runs the UNMODIFIED reference run_compile (/root/reference/proj/core/src/
// pipeline.cpp:52-198, with codegen.cpp's emit_report / build_lut) for one
// request per stdin line and writes its artefacts (report.json, a2.s24,
// lut.bin, kernel.cu) under the given directory. Built by `make -C oracle ref`
// into oracle/_ref/ref_compile; oracle/make_golden_compile.py turns its output
// into tests/golden/compile/.
//
// line: <out_dir> <stencil preset> <grid e.g. 64x64> <hw> <r1|0> <r2|0> <fuse>
//       <exact64|round16> <seed> <corrupt 0|1>
#include <cstdio>
#include <iostream>
#include <sstream>
#include <string>

#include "stensor/pipeline.hpp"

int main() {
    std::string line;
    int rc = 0;
    while (std::getline(std::cin, line)) {
        if (line.empty() || line[0] == '#') continue;
        std::istringstream in(line);
        std::string out, stencil, grid, hw, prec;
        int r1 = 0, r2 = 0, corrupt = 0;
        unsigned long long fuse = 1, seed = 1;
        in >> out >> stencil >> grid >> hw >> r1 >> r2 >> fuse >> prec >> seed >> corrupt;
        try {
            stensor::CompileRequest req;
            req.spec = stensor::stencil_preset(stencil);
            std::string tok;
            for (char c : grid + "x") {
                if (c == 'x') {
                    req.grid_dims.push_back(std::stoull(tok));
                    tok.clear();
                } else {
                    tok += c;
                }
            }
            req.hw = stensor::hw_preset(hw);
            if (r1 > 0) req.r1 = r1;
            if (r1 > 0) req.r2 = r2 > 0 ? r2 : 1;
            req.fuse = fuse;
            req.precision = prec == "round16" ? stensor::Precision::round16 : stensor::Precision::exact64;
            req.seed = seed;
            req.out_dir = out;
            req.corrupt_permutation = corrupt != 0;
            const auto res = stensor::run_compile(req);
            std::printf("%s ok=%d status=%s\n", out.c_str(), res.ok ? 1 : 0, res.verification.status.c_str());
        } catch (const std::exception& e) {
            std::printf("%s error=%s\n", out.c_str(), e.what());
            rc = 1;
        }
    }
    return rc;
}
