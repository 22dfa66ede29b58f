// Plan aggregation and compile artefacts (reference: proj/core/src/codegen.cpp).
//   default_block_config   codegen.cpp:10-17
//   build_lut / lut.bin    codegen.cpp:19-59, pipeline.cpp:177-191, formats.md:65-72
//   make_plan              codegen.cpp:75-102
//   emit_report            codegen.cpp:203-242, formats.md:74-103 (nlohmann dump(2) layout)
#include "stensor/codegen.hpp"

#include <charconv>
#include <cmath>
#include <cstring>
#include <stdexcept>

namespace stensor {

BlockConfig default_block_config(int dims) {
    switch (dims) {
        case 1: return {1024, 1};
        case 2: return {32, 64};
        case 3: return {8, 64};
        default: throw std::invalid_argument("unsupported dimensionality");
    }
}

LookupTable build_lut(const MorphedLayout& layout, const BlockConfig& block) {
    if (block.x == 0 || block.y == 0) throw std::invalid_argument("empty block config");
    const auto d = static_cast<std::size_t>(layout.dims);
    const std::size_t gx = layout.grid_dims[d - 1];
    const std::size_t gy = d >= 2 ? layout.grid_dims[d - 2] : 1;
    std::size_t cells = 1;
    for (auto g : layout.grid_dims) cells *= g;
    const auto r1 = static_cast<std::size_t>(layout.r1), r2 = static_cast<std::size_t>(layout.r2);
    // operand columns are output tiles, tx fastest, then ty, then the output plane
    const std::size_t ntx = layout.padded_out_x / r1, nty = layout.padded_out_y / r2;

    LookupTable lut;
    lut.block_config = block;
    lut.b_rows = layout.a.cols;
    lut.cols_per_block = block.x < layout.n_prime ? block.x : layout.n_prime;
    lut.block_count = lut.cols_per_block ? (layout.n_prime + lut.cols_per_block - 1) / lut.cols_per_block : 0;
    lut.base.assign(lut.block_count, 0);
    lut.entries.assign(lut.block_count * lut.b_rows * lut.cols_per_block, kLutZero);
    for (std::size_t blk = 0; blk < lut.block_count; ++blk) {
        const std::size_t first = blk * lut.cols_per_block;
        const std::size_t tx = first % ntx, ty = (first / ntx) % nty, zo = first / (ntx * nty);
        const std::size_t base = (zo * gy + ty * r2) * gx + tx * r1;
        lut.base[blk] = static_cast<std::int64_t>(base);
        const std::size_t ncol = std::min(lut.cols_per_block, layout.n_prime - first);
        std::int64_t* out = lut.entries.data() + blk * lut.b_rows * lut.cols_per_block;
        for (std::size_t c = 0; c < ncol; ++c)
            for (std::size_t row = 0; row < lut.b_rows; ++row) {
                const BRef ref = layout.b_at(row, first + c);
                if (ref.is_zero()) continue;
                if (ref.flat >= cells) throw std::out_of_range("lookup slot maps outside the grid");
                out[row * lut.cols_per_block + c] =
                    static_cast<std::int64_t>(ref.flat) - static_cast<std::int64_t>(base);
            }
    }
    return lut;
}

std::string lut_bytes(const LookupTable& lut) {
    std::string out;
    out.reserve(8 * (3 + lut.base.size() + lut.entries.size()));
    auto put = [&out](std::int64_t v) {
        const auto u = static_cast<std::uint64_t>(v);
        for (int i = 0; i < 8; ++i) out.push_back(static_cast<char>((u >> (8 * i)) & 0xffu));
    };
    put(static_cast<std::int64_t>(lut.block_count));
    put(static_cast<std::int64_t>(lut.b_rows));
    put(static_cast<std::int64_t>(lut.cols_per_block));
    for (auto b : lut.base) put(b);
    for (auto e : lut.entries) put(e);
    return out;
}

KernelPlan make_plan(std::string stencil_name, const MorphedLayout& layout, const Conversion& cv,
                     const HardwareDescriptor& hw, Precision precision, bool with_lut) {
    if (!check_24(cv.converted.a)) throw std::invalid_argument("plan operand violates the 2:4 constraint");
    std::vector<std::uint8_t> hit(cv.perm.size(), 0);
    for (std::size_t pos : cv.perm.order) {
        if (pos >= hit.size() || hit[pos]) throw std::invalid_argument("plan permutation is not a bijection");
        hit[pos] = 1;
    }
    KernelPlan plan;
    plan.stencil_name = std::move(stencil_name);
    plan.dims = layout.dims;
    plan.k = layout.kext[static_cast<std::size_t>(layout.dims) - 1];
    plan.grid_dims = layout.grid_dims;
    plan.layout = cv.converted;
    plan.perm = cv.perm;
    plan.a2 = compress_24(cv.converted.a);
    plan.fragment = hw.fragment;
    plan.block = default_block_config(layout.dims);
    if (with_lut) plan.lut = build_lut(cv.converted, plan.block);
    plan.precision = precision;
    plan.p = cv.p;
    plan.align_cols = cv.align_cols;
    plan.used_blossom = cv.used_blossom;
    return plan;
}

// ------------------------------------------------------------------ JSON text

std::string json_number(double v) {
    if (!std::isfinite(v)) return "null";
    if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
    std::string out;
    if (v < 0) {
        out.push_back('-');
        v = -v;
    }
    // shortest round-trip digits d1.d2d3...e<exp>
    char sci[64];
    const auto res = std::to_chars(sci, sci + sizeof sci - 1, v, std::chars_format::scientific);
    *res.ptr = '\0';  // to_chars does not terminate; atoi below reads the exponent
    std::string digits;
    const char* p = sci;
    for (; p < res.ptr && *p != 'e'; ++p)
        if (*p != '.') digits.push_back(*p);
    const int e10 = std::atoi(p + 1);
    const int k = static_cast<int>(digits.size());
    const int n = e10 + 1;  // position of the decimal point relative to the digits
    constexpr int kMinExp = -4, kMaxExp = 15;
    if (k <= n && n <= kMaxExp) {  // integral: digits, zeros, ".0"
        out += digits + std::string(static_cast<std::size_t>(n - k), '0') + ".0";
    } else if (0 < n && n <= kMaxExp) {  // fixed with a fraction
        out += digits.substr(0, static_cast<std::size_t>(n)) + "." + digits.substr(static_cast<std::size_t>(n));
    } else if (kMinExp < n && n <= 0) {  // 0.000ddd
        out += "0." + std::string(static_cast<std::size_t>(-n), '0') + digits;
    } else {  // d.ddde+XX
        out.push_back(digits[0]);
        if (k > 1) out += "." + digits.substr(1);
        const int x = n - 1;
        out.push_back('e');
        out.push_back(x < 0 ? '-' : '+');
        const int ax = x < 0 ? -x : x;
        if (ax < 10) out.push_back('0');
        out += std::to_string(ax);
    }
    return out;
}

namespace {

std::string json_string(const std::string& s) {
    std::string out = "\"";
    for (unsigned char c : s) {
        switch (c) {
            case '"': out += "\\\""; break;
            case '\\': out += "\\\\"; break;
            case '\b': out += "\\b"; break;
            case '\f': out += "\\f"; break;
            case '\n': out += "\\n"; break;
            case '\r': out += "\\r"; break;
            case '\t': out += "\\t"; break;
            default:
                if (c < 0x20) {
                    char buf[8];
                    std::snprintf(buf, sizeof buf, "\\u%04x", c);
                    out += buf;
                } else {
                    out.push_back(static_cast<char>(c));
                }
        }
    }
    return out + "\"";
}

// Minimal ordered writer reproducing the reference's dump(2) output: two-space
// indent, one member per line, "key": value separators.
class JsonObject {
  public:
    explicit JsonObject(int depth) : depth_(depth) {}
    void raw(const std::string& key, const std::string& text) { items_.emplace_back(key, text); }
    void str(const std::string& key, const std::string& v) { raw(key, json_string(v)); }
    void num(const std::string& key, double v) { raw(key, json_number(v)); }
    void uint(const std::string& key, std::uint64_t v) { raw(key, std::to_string(v)); }
    void sint(const std::string& key, std::int64_t v) { raw(key, std::to_string(v)); }
    void boolean(const std::string& key, bool v) { raw(key, v ? "true" : "false"); }
    void uint_array(const std::string& key, const std::vector<std::size_t>& v) {
        // the reference build's json.hpp (cudnn_frontend's vendored v3.11.3) prints
        // arrays of numbers on one line without separators' spaces: [64,64]
        std::string t = "[";
        for (std::size_t i = 0; i < v.size(); ++i) t += (i ? "," : "") + std::to_string(v[i]);
        raw(key, t + "]");
    }
    std::string text() const {
        if (items_.empty()) return "{}";
        const std::string in(static_cast<std::size_t>(2 * (depth_ + 1)), ' ');
        std::string t = "{\n";
        for (std::size_t i = 0; i < items_.size(); ++i)
            t += in + json_string(items_[i].first) + ": " + items_[i].second + (i + 1 < items_.size() ? ",\n" : "\n");
        return t + std::string(static_cast<std::size_t>(2 * depth_), ' ') + "}";
    }

  private:
    int depth_;
    std::vector<std::pair<std::string, std::string>> items_;
};

}  // namespace

std::string emit_report(const KernelPlan& plan, const PerfEstimate& perf, const VerificationResult& verification,
                        std::uint64_t issued_mma, double model_gstencil) {
    JsonObject j(0);
    j.sint("schema_version", 1);
    j.str("stencil", plan.stencil_name);
    j.sint("dims", plan.dims);
    j.sint("k", plan.k);
    j.uint_array("grid", plan.grid_dims);
    j.str("precision", plan.precision == Precision::round16 ? "round16" : "exact64");
    j.sint("r1", plan.layout.r1);
    j.sint("r2", plan.layout.r2);
    j.uint("m_prime", plan.layout.a.rows);
    j.uint("k_prime", plan.layout.a.cols);
    j.uint("n_prime", plan.layout.n_prime);
    j.uint("zero_columns", plan.p);
    j.uint("align_columns", plan.align_cols);
    j.boolean("used_blossom", plan.used_blossom);
    std::size_t nnz = 0;
    for (double v : plan.layout.a.data) nnz += v != 0.0;
    j.num("sparsity_ratio",
          1.0 - static_cast<double>(nnz) / static_cast<double>(plan.layout.a.rows * plan.layout.a.cols));
    j.uint("n_mma", perf.n_mma);
    j.uint("issued_mma", issued_mma);
    j.num("t_compute", perf.t_compute);
    j.num("t_memory", perf.t_memory);
    j.num("t_total", perf.t_total);
    j.num("model_gstencils_per_sec", model_gstencil);
    JsonObject v(1);
    v.str("status", verification.status);
    v.num("max_abs_err", verification.max_abs_err);
    v.num("max_rel_err", verification.max_rel_err);
    if (verification.status == "conversion-failed") {
        v.uint("bad_row", verification.bad_row);
        v.uint("bad_col", verification.bad_col);
    }
    j.raw("verification", v.text());
    return j.text() + "\n";
}

}  // namespace stensor
