// 2:4 compression and the `.s24` container.
//   compress_24   proj/core/src/emulator.cpp:40-80 — 0:4 groups canonicalise to
//                 slots {0,1}; a 1:4 group puts its zero in the smallest unused
//                 slot and keeps pos0 < pos1 (values follow the positions)
//   decompress    emulator.cpp:82-93
//   dump / load   emulator.cpp:195-230, docs/formats.md:49-63 (little endian:
//                 "S24\0", u64 rows, u64 cols, u32 tag, f64 values, u8 meta)
#include <cstring>
#include <istream>
#include <ostream>
#include <sstream>
#include <stdexcept>
#include <utility>

#include "stensor/s24.hpp"

namespace stensor {

namespace {

void write_le(std::ostream& out, std::uint64_t v, int nbytes) {
    char buf[8];
    for (int i = 0; i < nbytes; ++i) buf[i] = static_cast<char>((v >> (8 * i)) & 0xffu);
    out.write(buf, nbytes);
}

std::uint64_t read_le(std::istream& in, int nbytes) {
    unsigned char buf[8];
    in.read(reinterpret_cast<char*>(buf), nbytes);
    if (!in) throw std::runtime_error("truncated sparse24 stream");
    std::uint64_t v = 0;
    for (int i = 0; i < nbytes; ++i) v |= static_cast<std::uint64_t>(buf[i]) << (8 * i);
    return v;
}

}  // namespace

Sparse24Matrix compress_24(const Matrix& dense) {
    if (dense.cols % 4 != 0) throw std::invalid_argument("column count must be divisible by 4");
    Sparse24Matrix s;
    s.rows = dense.rows;
    s.logical_cols = dense.cols;
    s.values.assign(dense.rows * dense.cols / 2, 0.0);
    s.meta.assign(dense.rows * dense.cols / 4, 0);
    const std::size_t half = dense.cols / 2, quarter = dense.cols / 4;
    for (std::size_t r = 0; r < dense.rows; ++r)
        for (std::size_t g = 0; g < quarter; ++g) {
            int slot[2] = {0, 1};  // 0:4 canonical positions
            double kept[2] = {0.0, 0.0};
            int found = 0;
            for (int l = 0; l < 4; ++l) {
                const double v = dense.at(r, 4 * g + static_cast<std::size_t>(l));
                if (v == 0.0) continue;
                if (found == 2) throw std::invalid_argument("4-group has more than 2 nonzeros");
                slot[found] = l;
                kept[found] = v;
                ++found;
            }
            if (found == 1) {
                // the zero partner takes the smallest slot the nonzero does not use
                const int zero_slot = slot[0] == 0 ? 1 : 0;
                if (zero_slot > slot[0]) {
                    slot[1] = zero_slot;
                } else {
                    slot[1] = slot[0];
                    kept[1] = kept[0];
                    slot[0] = zero_slot;
                    kept[0] = 0.0;
                }
            }
            s.values[r * half + 2 * g] = kept[0];
            s.values[r * half + 2 * g + 1] = kept[1];
            s.meta[r * quarter + g] = static_cast<std::uint8_t>(slot[0] | (slot[1] << 2));
        }
    return s;
}

Matrix decompress(const Sparse24Matrix& s) {
    Matrix d(s.rows, s.logical_cols);
    for (std::size_t r = 0; r < s.rows; ++r)
        for (std::size_t g = 0; g < s.groups_per_row(); ++g) {
            const std::uint8_t m = s.meta_at(r, g);
            const std::size_t p0 = m & 3u, p1 = (m >> 2) & 3u;
            if (p0 >= p1) throw std::invalid_argument("metadata positions must be increasing");
            d.at(r, 4 * g + p0) = s.value_at(r, 2 * g);
            d.at(r, 4 * g + p1) = s.value_at(r, 2 * g + 1);
        }
    return d;
}

void dump_sparse24(std::ostream& out, const Sparse24Matrix& s, Precision tag) {
    out.write("S24\0", 4);
    write_le(out, s.rows, 8);
    write_le(out, s.logical_cols, 8);
    write_le(out, tag == Precision::round16 ? 1u : 0u, 4);
    for (double v : s.values) {
        std::uint64_t bits;
        std::memcpy(&bits, &v, sizeof bits);
        write_le(out, bits, 8);
    }
    out.write(reinterpret_cast<const char*>(s.meta.data()),
              static_cast<std::streamsize>(s.meta.size()));
}

Sparse24Matrix load_sparse24(std::istream& in, Precision* tag_out) {
    char magic[4];
    in.read(magic, 4);
    if (!in || std::memcmp(magic, "S24\0", 4) != 0) throw std::runtime_error("bad sparse24 magic");
    Sparse24Matrix s;
    s.rows = read_le(in, 8);
    s.logical_cols = read_le(in, 8);
    const auto tag = static_cast<std::uint32_t>(read_le(in, 4));
    if (s.logical_cols % 4 != 0) throw std::runtime_error("bad sparse24 column count");
    if (tag_out) *tag_out = tag ? Precision::round16 : Precision::exact64;
    s.values.resize(s.rows * s.logical_cols / 2);
    for (double& v : s.values) {
        const std::uint64_t bits = read_le(in, 8);
        std::memcpy(&v, &bits, sizeof v);
    }
    s.meta.resize(s.rows * s.logical_cols / 4);
    in.read(reinterpret_cast<char*>(s.meta.data()), static_cast<std::streamsize>(s.meta.size()));
    if (!in) throw std::runtime_error("truncated sparse24 stream");
    return s;
}

std::string sparse24_bytes(const Sparse24Matrix& s, Precision tag) {
    std::ostringstream os(std::ios::binary);
    dump_sparse24(os, s, tag);
    return os.str();
}

}  // namespace stensor
