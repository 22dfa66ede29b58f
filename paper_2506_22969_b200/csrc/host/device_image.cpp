// Constant-operand images for the tcgen05.mma.sp (kind::f16) stencil kernels.
//
// A (sparse, K-major, SWIZZLE_NONE): per 32-wide logical K step a 4 KiB block
//   of 128 rows x 16 stored halves; core matrices are 8 rows x 16 B,
//   LBO (K direction) = 128 B, SBO (M direction) = 256 B.
// E (metadata, TMEM): per K step one 32-bit TMEM column. Lane
//   L = m0 + 8*k1 + 16*m2 holds, in nibble (g + 4*m1), the 2:4 selector of
//   A row m0 + 8*m1 + 16*m2, 4-group 4*k1 + g of the step. The nibble is the
//   reference metadata byte pos0 | pos1 << 2 verbatim (emulator.cpp:74-75);
//   layout confirmed on B200 by tools/probes/probe_sparse_mma.cu.
// koff: B''[q, tile] = patch[tile_origin + koff[q]] with koff from the PIT'd
//   col_origin (layout.cpp:162-188 restated for a shared-memory patch).
#include <algorithm>
#include <array>
#include <cstdint>
#include <cmath>
#include <cstring>
#include <numeric>
#include <random>
#include <stdexcept>

#include "stensor/device_image.hpp"
#include "stensor/morph.hpp"

namespace stensor {

std::uint16_t f32_to_f16_bits(float f) {
    std::uint32_t x;
    std::memcpy(&x, &f, 4);
    const std::uint32_t sign = (x >> 16) & 0x8000u;
    std::uint32_t mag = x & 0x7fffffffu;
    if (mag >= 0x7f800000u) return static_cast<std::uint16_t>(sign | (mag > 0x7f800000u ? 0x7e00u : 0x7c00u));
    if (mag >= 0x477ff000u) return static_cast<std::uint16_t>(sign | 0x7c00u);  // overflow
    if (mag < 0x38800000u) {                                                     // subnormal / zero
        const int e = static_cast<int>(mag >> 23);
        const int shift = 126 - e;
        if (shift > 24) return static_cast<std::uint16_t>(sign);
        const std::uint32_t m = (mag & 0x7fffffu) | 0x800000u;
        std::uint32_t q = m >> shift;
        const std::uint32_t rem = m & ((1u << shift) - 1u), halfway = 1u << (shift - 1);
        if (rem > halfway || (rem == halfway && (q & 1u))) ++q;
        return static_cast<std::uint16_t>(sign | q);
    }
    std::uint32_t h = mag >> 13;
    const std::uint32_t rem = mag & 0x1fffu;
    if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ++h;
    return static_cast<std::uint16_t>(sign | (h - (112u << 10)));
}

double f16_bits_to_double(std::uint16_t h) {
    const int e = (h >> 10) & 0x1f, m = h & 0x3ff;
    const double v = e == 0 ? std::ldexp(static_cast<double>(m), -24)
                            : std::ldexp(static_cast<double>(m | 0x400), e - 25);
    return (h & 0x8000) ? -v : v;
}

namespace {

// distinct 4-byte words per bank among the 32 lanes of one gather LDS (addresses
// in patch elements of `elem` bytes: two binary16 lanes may share a word)
int bank_degree(const std::array<std::int32_t, 32>& addr, int elem) {
    std::array<std::vector<std::int32_t>, 32> per_bank;
    for (std::int32_t e : addr) {
        const std::int32_t a = e * elem / 4;
        auto& v = per_bank[static_cast<std::size_t>(((a % 32) + 32) % 32)];
        if (std::find(v.begin(), v.end(), a) == v.end()) v.push_back(a);
    }
    std::size_t worst = 0;
    for (const auto& v : per_bank) worst = std::max(worst, v.size());
    return static_cast<int>(worst);
}

int schedule_cost(const std::vector<std::uint8_t>& order, const std::vector<std::int32_t>& koff, int elem,
                  int* worst_out) {
    int total = 0, worst = 0;
    for (std::size_t it = 0; it * 4 < order.size(); ++it) {
        std::array<std::int32_t, 32> addr{};
        for (int lane = 0; lane < 32; ++lane)
            addr[static_cast<std::size_t>(lane)] =
                koff[static_cast<std::size_t>(order[it * 4 + static_cast<std::size_t>(lane / 8)]) * 8 +
                     static_cast<std::size_t>(lane % 8)];
        const int d = bank_degree(addr, elem);
        total += d;
        worst = std::max(worst, d);
    }
    if (worst_out) *worst_out = worst;
    return total;
}

}  // namespace

DeviceImage build_device_image(const BatchGeometry& geo_in, std::size_t rows, std::size_t cols,
                               const double* values, const std::uint8_t* meta,
                               const std::size_t* col_origin, std::size_t wv, std::size_t wu) {
    if (rows != 128) throw std::invalid_argument("device image needs m' = 128 (r1 * r2)");
    if (cols % 4 != 0) throw std::invalid_argument("A'' column count must be 4-aligned");
    DeviceImage img;
    img.geo = geo_in;
    BatchGeometry& g = img.geo;
    // z_slices > 1 (3D z-streaming): A'' is cut into kz z-slices of C columns
    // each (expand_units orders the PIT'd columns z-major, convert.cpp:376-396),
    // every slice padded to its own K; B'' is gathered per input plane.
    const std::size_t nsl = static_cast<std::size_t>(std::max(1, g.z_slices));
    if (cols % nsl != 0) throw std::invalid_argument("A'' columns do not split into z slices");
    const std::size_t C = cols / nsl;
    if (nsl > 1 && C % 4 != 0) throw std::invalid_argument("z slice is not 4-group aligned");
    g.k_pad = static_cast<int>((C + 31) / 32 * 32);
    const std::size_t k_pad = static_cast<std::size_t>(g.k_pad), ksteps = k_pad / 32;
    const std::size_t half_cols = cols / 2, quarter_cols = cols / 4;

    // ---- A image: slice dz occupies K steps [dz*ksteps, (dz+1)*ksteps)
    img.a_smem.assign(nsl * 128 * k_pad / 2, 0);
    for (std::size_t dz = 0; dz < nsl; ++dz)
        for (std::size_t m = 0; m < 128; ++m)
            for (std::size_t jl = 0; jl < C / 2; ++jl) {
                const std::size_t j = dz * (C / 2) + jl;  // stored index in the reference order
                const std::size_t s = dz * ksteps + jl / 16, jj = jl % 16;
                const std::size_t at = s * 2048 + (m / 8) * 128 + (jj / 8) * 64 + (m % 8) * 8 + jj % 8;
                img.a_smem[at] = f32_to_f16_bits(static_cast<float>(values[m * half_cols + j]));
            }

    // ---- E words
    img.e_words.assign(nsl * ksteps * 128, 0);
    for (std::size_t dz = 0; dz < nsl; ++dz)
        for (std::size_t s = 0; s < ksteps; ++s)
            for (std::size_t m = 0; m < 128; ++m)
                for (std::size_t gl = 0; gl < 8; ++gl) {
                    const std::size_t grp = s * 8 + gl;  // group inside the slice
                    const std::uint32_t nib =
                        grp < C / 4 ? (meta[m * quarter_cols + dz * (C / 4) + grp] & 0xfu)
                                    : 0x4u;  // padding: canonical {0,1}
                    const std::size_t m0 = m % 8, m1 = (m / 8) % 2, m2 = m / 16;
                    const std::size_t lane = m0 + 8 * (gl / 4) + 16 * m2;
                    img.e_words[(dz * ksteps + s) * 128 + lane] |= nib << (4 * ((gl % 4) + 4 * m1));
                }

    // ---- K-row offsets into the shared-memory patch (one slice: positions [0, C))
    const std::int32_t plane = g.patch_w * g.patch_h;
    img.koff.assign(k_pad, 0);  // zero columns read a real (finite) patch cell; A'' is 0 there
    std::vector<std::int64_t> uv(C, -1);
    for (std::size_t dz = 0; dz < nsl; ++dz)
        for (std::size_t ql = 0; ql < C; ++ql) {
            const std::size_t j = col_origin[dz * C + ql];
            std::int64_t here = -1;
            std::size_t z = 0;
            if (j != npos) {
                z = j / (wu * wv);
                here = static_cast<std::int64_t>(j % (wu * wv));
            }
            if (nsl > 1) {
                if (j != npos && z != dz) throw std::invalid_argument("z slice holds a foreign plane");
                if (dz == 0) uv[ql] = here;
                else if (uv[ql] != here) throw std::invalid_argument("z slices differ in (u, v) order");
            }
            if (dz > 0 || j == npos) continue;
            const std::size_t u = static_cast<std::size_t>(here) / wv, v = static_cast<std::size_t>(here) % wv;
            img.koff[ql] = static_cast<std::int32_t>(nsl > 1 ? 0 : z) * plane +
                           static_cast<std::int32_t>(u) * g.patch_w + static_cast<std::int32_t>(v) +
                           g.x_shift;
        }

    // ---- gather schedule: partition 8-row groups into 32-row sweeps with few
    // shared-memory bank conflicts (deterministic local search)
    const std::size_t ngroups = k_pad / 8;
    img.kgroup_order.resize(ngroups);
    std::iota(img.kgroup_order.begin(), img.kgroup_order.end(), std::uint8_t{0});
    int best = schedule_cost(img.kgroup_order, img.koff, g.elem_bytes, nullptr);
    std::mt19937 rng(12345);
    for (int trial = 0; trial < 4000 && ngroups > 4; ++trial) {
        const std::size_t a = rng() % ngroups, b = rng() % ngroups;
        if (a / 4 == b / 4) continue;
        std::swap(img.kgroup_order[a], img.kgroup_order[b]);
        const int c = schedule_cost(img.kgroup_order, img.koff, g.elem_bytes, nullptr);
        if (c <= best)
            best = c;
        else
            std::swap(img.kgroup_order[a], img.kgroup_order[b]);
    }
    schedule_cost(img.kgroup_order, img.koff, g.elem_bytes, &img.worst_bank_conflict);

    // ---- per-lane gather tables: sweep j, lane -> (patch byte offset, B byte offset)
    img.gather_src.resize(k_pad / 32 * 32);
    img.gather_dst.resize(k_pad / 32 * 32);
    for (std::size_t j = 0; j < k_pad / 32; ++j)
        for (std::size_t lane = 0; lane < 32; ++lane) {
            const std::size_t k = static_cast<std::size_t>(img.kgroup_order[4 * j + lane / 8]) * 8 + lane % 8;
            img.gather_src[j * 32 + lane] = img.koff[k] * g.elem_bytes;
            img.gather_dst[j * 32 + lane] = static_cast<std::int32_t>(k) * 16;
        }
    img.lo_sweep0 = static_cast<int>(k_pad / 32);
    if (g.terms == 2) {
        // split operand: every z slice's K becomes [K rows -> B_hi; K rows -> B_lo]
        // and A'' (with its metadata) is repeated for the second half, so the MMA
        // accumulates A'' B_hi + A'' B_lo. Exact only if A'' itself is binary16.
        for (std::size_t i = 0; i < rows * half_cols; ++i) {
            const double v = values[i];
            if (f16_bits_to_double(f32_to_f16_bits(static_cast<float>(v))) != v)
                throw std::invalid_argument("f16x2 needs A'' weights exact in binary16 (use f16)");
        }
        std::vector<std::uint16_t> a2(2 * img.a_smem.size());
        std::vector<std::uint32_t> e2(2 * img.e_words.size());
        for (std::size_t dz = 0; dz < nsl; ++dz)
            for (std::size_t t = 0; t < 2 * ksteps; ++t) {
                const std::size_t from = dz * ksteps + t % ksteps, to = dz * 2 * ksteps + t;
                std::copy_n(img.a_smem.begin() + static_cast<std::ptrdiff_t>(from * 2048), 2048,
                            a2.begin() + static_cast<std::ptrdiff_t>(to * 2048));
                std::copy_n(img.e_words.begin() + static_cast<std::ptrdiff_t>(from * 128), 128,
                            e2.begin() + static_cast<std::ptrdiff_t>(to * 128));
            }
        img.a_smem = std::move(a2);
        img.e_words = std::move(e2);
        const std::size_t sweeps = k_pad / 32;
        img.koff.resize(2 * k_pad);
        std::copy_n(img.koff.begin(), k_pad, img.koff.begin() + static_cast<std::ptrdiff_t>(k_pad));
        img.gather_src.resize(2 * sweeps * 32);
        img.gather_dst.resize(2 * sweeps * 32);
        for (std::size_t i = 0; i < sweeps * 32; ++i) {
            img.gather_src[sweeps * 32 + i] = img.gather_src[i];
            img.gather_dst[sweeps * 32 + i] = img.gather_dst[i] + static_cast<std::int32_t>(k_pad) * 16;
        }
        g.k_pad = static_cast<int>(2 * k_pad);
    }
    // the kernels read ONE 32-bit word per lane and sweep: half the patch byte offset
    // (low 16 bits; offsets are even, patches < 128 KiB) | the B'' row (high 16 bits)
    img.gather_packed.resize(img.gather_src.size());
    for (std::size_t i = 0; i < img.gather_src.size(); ++i) {
        const std::int32_t src = img.gather_src[i], row = img.gather_dst[i] / 16;
        if (src < 0 || src >= (1 << 17) || (src & 1) || row >= (1 << 16))
            throw std::invalid_argument("gather table entry out of the packed range");
        img.gather_packed[i] = (src >> 1) | (row << 16);
    }
    return img;
}

}  // namespace stensor
