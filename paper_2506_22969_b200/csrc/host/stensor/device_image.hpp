// Host-side construction of the constant operands the sm_100a kernels consume.
// Replaces the reference's per-block int64 lookup table (codegen.cpp:19-59,
// 839 MB at 8192^2) with a K-entry offset table: B''[q, tile] =
// patch[tile_origin + koff[q]] holds for every tile.
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

namespace stensor {

/// Geometry of one CTA batch of output tiles (all sizes in elements).
struct BatchGeometry {
    int dims = 2;
    int k = 3;                 // kernel extent per axis
    int r1 = 16, r2 = 8;       // tile = r1 (x) by r2 (y) outputs; r1*r2 == 128
    int tiles_x = 8;           // TXB: tiles per batch along x
    int tiles_y = 8;           // TYB: tiles per batch along y
    int patch_w = 0;           // TMA box width (multiple of 4 elements)
    int patch_h = 0;           // rows per plane
    int patch_planes = 1;      // kz (3D) or 1
    int k_pad = 0;             // logical K rounded to the MMA K step (32)
    int z_slices = 1;          // 1: whole A'' per MMA pass; kz: 3D z-streaming slices
    int terms = 1;             // 2: split B'' = B_hi + B_lo (SST_PREC_F16X2); K doubled
    int x_shift = 0;           // patch column of the window origin (TMA boxes start
                               // 16-byte aligned, so the patch begins lp cells early)
    int elem_bytes = 4;        // patch element: 4 (fp32 storage) or 2 (binary16 inter-step storage)
    int n_tiles() const { return tiles_x * tiles_y; }
};

struct DeviceImage {
    BatchGeometry geo;
    std::vector<std::uint16_t> a_smem;    // fp16 bits, UMMA K-major interleaved image
    std::vector<std::uint32_t> e_words;   // [k_steps][128] TMEM metadata words
    std::vector<std::int32_t> koff;       // [k_pad] patch element offset of B'' row q
    std::vector<std::uint8_t> kgroup_order;  // [k_pad/8] gather schedule (groups of 8 rows)
    // flattened schedule, [k_pad/32][32]: lane's patch byte offset and its
    // byte offset inside one 8-tile B'' group (MN-major: row k at k * 16 B)
    std::vector<std::int32_t> gather_src, gather_dst;
    // what the kernels load: (gather_src / 2) | (gather_dst / 16) << 16 per lane and sweep
    std::vector<std::int32_t> gather_packed;
    int worst_bank_conflict = 0;          // max lanes per bank over gather LDS sweeps
    int lo_sweep0 = 0;                    // first gather sweep producing B_lo rows (= sweeps if terms 1)
};

/// Inputs are the reference compile products: compressed A'' (values as
/// double, meta bytes pos0|pos1<<2) and col_origin (pre-PIT window index,
/// npos == SIZE_MAX for zero columns), with window extents wv (x), wu (y).
DeviceImage build_device_image(const BatchGeometry& geo_in, std::size_t rows, std::size_t cols,
                               const double* values, const std::uint8_t* meta,
                               const std::size_t* col_origin, std::size_t wv, std::size_t wu);

/// fp32 -> fp16 bits, round to nearest even (host side, for the A operand)
std::uint16_t f32_to_f16_bits(float f);
/// fp16 bits -> value (exact)
double f16_bits_to_double(std::uint16_t h);

}  // namespace stensor
