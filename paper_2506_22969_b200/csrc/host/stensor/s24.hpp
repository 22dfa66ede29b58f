// Compressed 2:4 operand and its byte-exact `.s24` artifact — drop-in for the
// reference emulator API's compress/dump half (proj/core/include/stensor/
// emulator.hpp:28-48, 67-69; docs/formats.md:49-63). The reference's
// software fragment-MMA emulator is replaced by the sm_100a tcgen05.mma.sp
// kernel (engine.hpp); it is not reproduced here.
#pragma once

#include <cstddef>
#include <cstdint>
#include <iosfwd>
#include <string>
#include <vector>

#include "stensor/morph.hpp"
#include "stensor/spec.hpp"

namespace stensor {

/// Two kept values per 4-group plus metadata byte pos0 | pos1 << 2 (pos0 < pos1).
struct Sparse24Matrix {
    std::size_t rows = 0;
    std::size_t logical_cols = 0;    // divisible by 4
    std::vector<double> values;      // rows x logical_cols/2
    std::vector<std::uint8_t> meta;  // rows x logical_cols/4

    std::size_t groups_per_row() const { return logical_cols / 4; }
    double value_at(std::size_t r, std::size_t slot) const {
        return values[r * (logical_cols / 2) + slot];
    }
    std::uint8_t meta_at(std::size_t r, std::size_t grp) const {
        return meta[r * (logical_cols / 4) + grp];
    }
};

Sparse24Matrix compress_24(const Matrix& dense);
Matrix decompress(const Sparse24Matrix& sparse);

void dump_sparse24(std::ostream& out, const Sparse24Matrix& s, Precision tag);
Sparse24Matrix load_sparse24(std::istream& in, Precision* tag_out = nullptr);
std::string sparse24_bytes(const Sparse24Matrix& s, Precision tag);

}  // namespace stensor
