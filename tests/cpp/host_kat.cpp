// Known-answer tests for the engine's host compile library (namespace stensor),
// restating the reference unit tests' fixtures (proj/tests/unit/*.cpp) against
// our implementation. Built and run by tests/test_host_kat.py.
//
//   host_kat                 run every check, exit 1 on any failure
//   host_kat perf HW K R1 R2 D0 [D1 [D2]]   print estimate() as JSON
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "stensor/device_image.hpp"
#include "stensor/hwmodel.hpp"
#include "stensor/morph.hpp"
#include "stensor/s24.hpp"
#include "stensor/sparsify.hpp"
#include "stensor/spec.hpp"

using namespace stensor;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                            \
    do {                                                                       \
        ++g_checks;                                                            \
        if (!(cond)) {                                                         \
            ++g_fail;                                                          \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);        \
        }                                                                      \
    } while (0)
#define CHECK_THROWS(expr)                                                     \
    do {                                                                       \
        bool thrown_ = false;                                                  \
        try {                                                                  \
            (void)(expr);                                                      \
        } catch (...) {                                                        \
            thrown_ = true;                                                    \
        }                                                                      \
        CHECK(thrown_);                                                        \
    } while (0)

// independent valid-region sweep used as the test oracle (brute force)
static std::vector<double> brute(const StencilSpec& s, const Grid& g) {
    const int r = s.radius();
    std::array<std::size_t, 3> in{1, 1, 1}, out{1, 1, 1};
    for (int a = 0; a < s.dims; ++a) {
        in[3 - s.dims + a] = g.dims[a];
        out[3 - s.dims + a] = g.dims[a] - s.k + 1;
    }
    std::vector<double> res(out[0] * out[1] * out[2]);
    for (std::size_t z = 0; z < out[0]; ++z)
        for (std::size_t y = 0; y < out[1]; ++y)
            for (std::size_t x = 0; x < out[2]; ++x) {
                double acc = 0;
                for (const auto& p : s.points) {
                    std::array<long, 3> o{0, 0, 0};
                    for (int a = 0; a < s.dims; ++a) o[3 - s.dims + a] = p.off[a] + r;
                    acc += p.weight *
                           g.values[((z + o[0]) * in[1] + (y + o[1])) * in[2] + x + o[2]];
                }
                res[(z * out[1] + y) * out[2] + x] = acc;
            }
    return res;
}

static Matrix random_24(std::size_t rows, std::size_t groups, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    Matrix a(rows, groups * 4);
    for (std::size_t r = 0; r < rows; ++r)
        for (std::size_t g = 0; g < groups; ++g) {
            const int count = static_cast<int>(rng() % 3);
            std::array<int, 4> slots{0, 1, 2, 3};
            std::shuffle(slots.begin(), slots.end(), rng);
            for (int i = 0; i < count; ++i)
                a.at(r, 4 * g + static_cast<std::size_t>(slots[static_cast<std::size_t>(i)])) =
                    static_cast<double>(1 + rng() % 9);
        }
    return a;
}

static void spec_tests() {
    // presets: counts, shapes, weights sum to 1 (test_stencil.cpp:57-82)
    const std::vector<std::pair<std::string, std::size_t>> counts = {
        {"Heat-1D", 3}, {"1D5P", 5}, {"Heat-2D", 5}, {"Box-2D9P", 9}, {"Star-2D13P", 13},
        {"Box-2D49P", 49}, {"Heat-3D", 7}, {"Box-3D27P", 27}};
    for (const auto& [n, c] : counts) {
        const auto s = stencil_preset(n);
        CHECK(s.points.size() == c);
        double sum = 0;
        for (const auto& p : s.points) sum += p.weight;
        CHECK(sum == 1.0);
        for (std::size_t i = 1; i < s.points.size(); ++i) CHECK(s.points[i - 1].off < s.points[i].off);
    }
    CHECK_THROWS(stencil_preset("nope"));
    CHECK(preset_names().size() == 8 && is_preset("Heat-3D") && !is_preset("heat-3d"));
    // parser (formats.md:3-30; test_stencil.cpp:84-100)
    const auto p = parse_stencil_spec(
        "name = h\ndims = 2\nshape = star\nk = 3  # kernel\npoint = -1 0 : 0.125\n"
        "point = 0 -1 : 0.125\npoint = 0 0 : 0.5\npoint = 0 1 : 0.125\npoint = 1 0 : 0.125\n");
    const auto h = stencil_preset("Heat-2D");
    CHECK(p.points.size() == h.points.size());
    for (std::size_t i = 0; i < p.points.size(); ++i)
        CHECK(p.points[i].off == h.points[i].off && p.points[i].weight == h.points[i].weight);
    CHECK_THROWS(parse_stencil_spec("name = x\ndims = 2\nshape = star\nk = 3\npoint = 1 1 : 1\n"));
    CHECK_THROWS(parse_stencil_spec("name = x\ndims = 2\nshape = box\nk = 3\npoint = 2 0 : 1\n"));
    CHECK_THROWS(parse_stencil_spec("name = x\ndims = 2\nshape = box\nk = 3\npoint = 0 0 : 1\npoint = 0 0 : 1\n"));
    CHECK_THROWS(parse_stencil_spec("name = x\nshape = box\nk = 3\npoint = 0 0 : 1\n"));
    CHECK_THROWS(parse_stencil_spec("name = x\ndims = 2\nshape = box\nk = 3\npoint = 0 : 1\n"));
    CHECK_THROWS(parse_stencil_spec("garbage\n"));
    CHECK_THROWS(parse_stencil_spec("name = x\ndims = 2\nshape = hex\nk = 3\n"));
    // fusion: impulse response of Heat-1D twice = [1,4,6,4,1]/16 (test_stencil.cpp:139-162)
    const auto f = fuse_time_steps(stencil_preset("Heat-1D"), 2);
    CHECK(f.k == 5 && f.points.size() == 5);
    const double want[5] = {1 / 16.0, 4 / 16.0, 6 / 16.0, 4 / 16.0, 1 / 16.0};
    for (int i = 0; i < 5; ++i) CHECK(f.points[static_cast<std::size_t>(i)].weight == want[i]);
    CHECK(f.name == "Heat-1D-fused2");
    CHECK(fuse_time_steps(stencil_preset("Box-2D9P"), 3).k == 7);
    CHECK_THROWS(fuse_time_steps(h, 0));
    // fusion soundness: fused(t) on dyadic data == t direct steps (exact)
    {
        const auto s = stencil_preset("Box-2D9P");
        const std::array<std::size_t, 2> dims{17, 19};
        Grid g = random_grid(dims, 3);
        Grid cur = g;
        for (int t = 0; t < 2; ++t) {
            auto v = brute(s, cur);
            cur.dims = {cur.dims[0] - 2, cur.dims[1] - 2};
            cur.values = v;
        }
        const auto fused = brute(fuse_time_steps(s, 2), g);
        CHECK(fused == cur.values);
    }
    // metric (test_stencil.cpp:200-211)
    const std::array<std::size_t, 2> d2{1000, 1000};
    CHECK(std::fabs(gstencil_rate(10, d2, 0.01).gstencils_per_sec - 1.0) < 1e-12);
    CHECK_THROWS(gstencil_rate(1, d2, 0.0));
    // random_grid: deterministic, dyadic in [0,1) (test_stencil.cpp:213-222)
    const auto a = random_grid(d2, 9), b = random_grid(d2, 9), c = random_grid(d2, 10);
    CHECK(a.values == b.values && a.values != c.values);
    for (double v : a.values) CHECK(v >= 0 && v < 1 && v * 256 == std::floor(v * 256));
    // validate (test_stencil.cpp:224-...)
    StencilSpec bad = h;
    bad.k = 4;
    CHECK_THROWS(validate(bad));
    bad = h;
    bad.points.clear();
    CHECK_THROWS(validate(bad));
    bad = h;
    bad.dims = 4;
    CHECK_THROWS(validate(bad));
}

static void layout_tests() {
    const auto box = stencil_preset("Box-2D9P");
    // flatten 3x3 on 5x5 (test_layout.cpp:39-51)
    const std::array<std::size_t, 2> d55{5, 5};
    const auto flat = flatten(box, d55);
    CHECK(flat.a_vector.size() == 9 && flat.b_rows == 9 && flat.b_cols == 9);
    CHECK_THROWS(flatten(box, std::array<std::size_t, 2>{2, 5}));
    CHECK_THROWS(flatten(box, std::array<std::size_t, 1>{5}));
    // crush k=3 (2,2) -> 4x16 (test_layout.cpp:97-107)
    const auto lay = crush(flatten(box, std::array<std::size_t, 2>{6, 6}), 2, 2);
    CHECK(lay.a.rows == 4 && lay.a.cols == 16 && lay.n_prime == 4 && verify_staircase(lay).ok);
    CHECK_THROWS(crush(flat, 17, 1));
    CHECK_THROWS(crush(flatten(stencil_preset("Heat-1D"), std::array<std::size_t, 1>{12}), 2, 2));
    // morph_dims incl. the 10240^2 golden (test_layout.cpp:132-147)
    auto md = morph_dims(3, 6, 6, 2, 2);
    CHECK(md.m_prime == 4 && md.k_prime == 16 && md.n_prime == 4);
    md = morph_dims(3, 9, 11, 1, 1);
    CHECK(md.m_prime == 1 && md.k_prime == 9 && md.n_prime == 63);
    md = morph_dims(7, 10240, 10240, 4, 2);
    CHECK(md.m_prime == 8 && md.k_prime == 80 && md.n_prime == std::size_t{5117} * 2559);
    // crush product == brute force under output_position, bijective (test_layout.cpp:109-130, 220-256)
    for (const char* name : {"Heat-2D", "Box-2D9P", "Star-2D13P", "Heat-3D", "Box-3D27P", "Heat-1D"}) {
        const auto s = stencil_preset(name);
        std::vector<std::size_t> dims = s.dims == 1 ? std::vector<std::size_t>{23}
                                       : s.dims == 2 ? std::vector<std::size_t>{13, 17}
                                                     : std::vector<std::size_t>{7, 8, 9};
        const Grid g = random_grid(dims, 13);
        const auto want = brute(s, g);
        const auto fl = flatten(s, dims);
        for (const auto [r1, r2] : {std::pair{3, 1}, {2, 2}, {1, 3}, {4, 2}, {16, 8}}) {
            if (s.dims == 1 && r2 != 1) continue;
            const auto L = crush(fl, r1, r2);
            for (const auto& M : {L, convert_layout(L).converted}) {
                const Matrix prod = matmul(M.a, materialize_b(M, g));
                std::size_t covered = 0;
                bool ok = true;
                for (std::size_t r = 0; r < prod.rows; ++r)
                    for (std::size_t c = 0; c < prod.cols; ++c) {
                        const auto pos = M.output_position(r, c);
                        if (!pos.valid) continue;
                        ++covered;
                        ok = ok && prod.at(r, c) == want[pos.flat];
                    }
                CHECK(ok && covered == want.size());
            }
        }
    }
    // staircase checks (test_layout.cpp:149-170)
    Matrix st(4, 6);
    for (std::size_t r = 0; r < 4; ++r)
        for (std::size_t c = r; c < r + 3; ++c) st.at(r, c) = 1.0;
    CHECK(staircase_check(st, 3).ok);
    Matrix dense(3, 6);
    for (auto& v : dense.data) v = 1.0;
    CHECK(!staircase_check(dense, 3).ok);
    auto corrupt = crush(flatten(box, std::array<std::size_t, 2>{8, 8}), 2, 2);
    corrupt.structural[5] ^= 1;
    CHECK(!verify_staircase(corrupt).ok);
    // ZERO slots and out_of_range (test_layout.cpp:172-192)
    const auto l31 = crush(flatten(box, std::array<std::size_t, 2>{6, 6}), 3, 1);
    bool zero = false;
    for (std::size_t r = 0; r < l31.a.cols; ++r)
        for (std::size_t c = 0; c < l31.n_prime; ++c) zero = zero || l31.b_at(r, c).is_zero();
    CHECK(zero);
    CHECK_THROWS(l31.b_at(0, l31.n_prime));
    // duplicates crushed: a grid cell appears once per column (test_layout.cpp:194-208)
    const auto l49 = crush(flatten(stencil_preset("Box-2D49P"), std::array<std::size_t, 2>{12, 12}), 3, 4);
    bool unique = true;
    for (std::size_t c = 0; c < l49.n_prime; ++c) {
        std::set<std::size_t> seen;
        for (std::size_t r = 0; r < l49.a.cols; ++r) {
            const auto ref = l49.b_at(r, c);
            if (!ref.is_zero()) unique = unique && seen.insert(ref.flat).second;
        }
    }
    CHECK(unique);
}

static void convert_tests() {
    // conflict graphs (test_convert.cpp:46-76, 275-280)
    Matrix id(4, 4);
    for (std::size_t i = 0; i < 4; ++i) id.at(i, i) = 1;
    CHECK(build_conflict_graph(id).edges.empty());
    Matrix row(1, 3);
    for (auto& v : row.data) v = 1;
    CHECK(dump_conflict_graph(build_conflict_graph(row)) == "0: 1 2\n1: 0 2\n2: 0 1\n");
    Matrix blocks(2, 8);
    blocks.at(0, 0) = 1;
    blocks.at(1, 5) = 1;
    const auto bg = build_conflict_graph_blocks(blocks, 2, 2);
    CHECK(bg.node_count == 4 && bg.edges.size() == 1 && bg.has_edge(0, 2));
    CHECK_THROWS(build_conflict_graph_blocks(blocks, 2, 3));
    CHECK_THROWS(build_conflict_graph(Matrix{}));
    // hierarchical traces (test_convert.cpp:78-103)
    auto m = hierarchical_match(2, 4, 2);
    CHECK(m.zero_columns == 0 && m.pairs.size() == 4 && m.pairs[0].left == 0 &&
          m.pairs[0].right == 2 && m.pairs[1].right == 3 && m.pairs[2].left == 4 &&
          m.pairs[2].right == 6);
    m = hierarchical_match(1, 3, 2);
    CHECK(m.zero_columns == 1 && m.pairs.size() == 2 && m.pairs[0].right == 2 && m.pairs[1].right == 3);
    m = hierarchical_match(1, 4, 3);
    CHECK(m.zero_columns == 2 && m.pairs.size() == 3 && m.pairs[0].right == 3);
    // padding == brute force minimum (test_convert.cpp:133-143)
    for (std::size_t mm = 1; mm <= 6; ++mm)
        for (std::size_t g = 1; g <= 6; ++g) {
            if (mm * g > 12) continue;
            for (int k = 1; k <= static_cast<int>(g); ++k)
                CHECK(hierarchical_match(mm, g, k).zero_columns ==
                      min_padding_bruteforce(descriptor_conflict_graph(mm, g, k)));
        }
    // blossom vs brute force on random graphs (test_convert.cpp:145-168)
    for (std::uint64_t seed = 0; seed < 30; ++seed) {
        std::mt19937_64 rng(seed);
        ConflictGraph g;
        g.node_count = 8;
        g.adj.assign(64, 0);
        for (std::size_t i = 0; i < 8; ++i)
            for (std::size_t j = i + 1; j < 8; ++j)
                if (std::uniform_real_distribution<>(0, 1)(rng) < 0.4) {
                    g.adj[i * 8 + j] = g.adj[j * 8 + i] = 1;
                    g.edges.emplace_back(i, j);
                }
        const auto bm = blossom_match(g);
        CHECK(bm.zero_columns == min_padding_bruteforce(g));
        for (const auto& pr : bm.pairs)
            if (pr.right < 8) CHECK(!g.has_edge(pr.left, pr.right));
    }
    ConflictGraph k3;
    k3.node_count = 3;
    k3.adj = {0, 1, 1, 1, 0, 1, 1, 1, 0};
    CHECK(blossom_match(k3).zero_columns == 3);
    ConflictGraph big;
    big.node_count = 13;
    CHECK_THROWS(min_padding_bruteforce(big));
    // permutation order (test_convert.cpp:187-203)
    Matching mt;
    mt.node_count = 6;
    mt.pairs = {{0, 3}, {1, 4}, {2, 5}};
    CHECK(build_permutation(mt, 6, 0).order == (std::vector<std::size_t>{0, 2, 4, 1, 3, 5}));
    Matching badm;
    badm.node_count = 4;
    badm.pairs = {{0, 1}};
    CHECK_THROWS(build_permutation(badm, 4, 0));
    // check_24 (test_convert.cpp:230-242)
    Matrix ok(1, 4), bad(1, 4);
    ok.at(0, 0) = 1;
    ok.at(0, 2) = 2;
    bad.at(0, 0) = bad.at(0, 1) = bad.at(0, 2) = 1;
    CHECK(check_24(ok) && !check_24(bad) && check_24(Matrix(3, 8)));
    CHECK_THROWS(check_24(Matrix(1, 6)));
    // blossom fallback on a shuffled staircase (test_convert.cpp:258-273)
    auto lay = crush(flatten(stencil_preset("Heat-2D"), std::array<std::size_t, 2>{8, 8}), 2, 2);
    for (std::size_t r = 0; r < lay.a.rows; ++r) {
        std::swap(lay.a.at(r, 0), lay.a.at(r, 7));
        std::swap(lay.structural[r * lay.a.cols + 0], lay.structural[r * lay.a.cols + 7]);
    }
    std::swap(lay.col_origin[0], lay.col_origin[7]);
    CHECK(!verify_staircase(lay).ok);
    const auto cv = convert_layout(lay);
    CHECK(cv.used_blossom && check_24(cv.converted.a));
    // PIT keeps the product (test_convert.cpp:205-228)
    const auto l2 = crush(flatten(stencil_preset("Box-2D9P"), std::array<std::size_t, 2>{7, 7}), 2, 2);
    const Grid g7 = random_grid(std::array<std::size_t, 2>{7, 7}, 31);
    const auto cv2 = convert_layout(l2);
    CHECK(matmul(cv2.converted.a, materialize_b(cv2.converted, g7)) == matmul(l2.a, materialize_b(l2, g7)));
}

static void s24_tests() {
    // group encodings (test_emulator.cpp:34-65)
    Matrix a(1, 4);
    a.at(0, 1) = 5;
    a.at(0, 3) = 7;
    auto s = compress_24(a);
    CHECK(s.value_at(0, 0) == 5 && s.value_at(0, 1) == 7 && s.meta_at(0, 0) == (1 | (3 << 2)));
    s = compress_24(Matrix(1, 4));
    CHECK(s.meta_at(0, 0) == (0 | (1 << 2)) && s.value_at(0, 0) == 0 && s.value_at(0, 1) == 0);
    Matrix one(1, 4);
    one.at(0, 0) = 9;
    CHECK(compress_24(one).meta_at(0, 0) == (0 | (1 << 2)));
    one = Matrix(1, 4);
    one.at(0, 2) = 9;
    s = compress_24(one);
    CHECK(s.meta_at(0, 0) == (0 | (2 << 2)) && s.value_at(0, 0) == 0 && s.value_at(0, 1) == 9);
    Matrix bad(1, 4);
    bad.at(0, 0) = bad.at(0, 1) = bad.at(0, 2) = 1;
    CHECK_THROWS(compress_24(bad));
    CHECK_THROWS(compress_24(Matrix(1, 6)));
    // round trip (test_emulator.cpp:67-78)
    for (std::uint64_t seed = 0; seed < 50; ++seed) {
        const Matrix m = random_24(4, 5, seed);
        CHECK(decompress(compress_24(m)) == m);
    }
    // .s24 byte-exact round trip (test_emulator.cpp:177-201)
    const auto c = compress_24(random_24(5, 3, 77));
    const std::string bytes = sparse24_bytes(c, Precision::round16);
    CHECK(bytes.size() == 4 + 8 + 8 + 4 + c.values.size() * 8 + c.meta.size());
    std::istringstream in(bytes, std::ios::binary);
    Precision tag;
    const auto back = load_sparse24(in, &tag);
    CHECK(tag == Precision::round16 && back.values == c.values && back.meta == c.meta);
    CHECK(sparse24_bytes(c, Precision::round16) == bytes);
    std::istringstream trunc(bytes.substr(0, 10), std::ios::binary);
    CHECK_THROWS(load_sparse24(trunc));
}

static void perf_tests() {
    // A100 golden fixture Heat-2D 10240^2 at (2,2) (test_perf.cpp:41-69)
    const std::array<std::size_t, 2> d{10240, 10240};
    const auto e = estimate(hw_preset("a100-sparse"), 2, d, 3, 2, 2);
    CHECK(e.n_prime == 26204161 && e.n_mma == 3275521);
    CHECK(e.t_total == 2.6967748424437297e-4);
    CHECK(n_mma(16, 32, 8, kFragSparse) == 1 && n_mma(17, 33, 9, kFragSparse) == 8);
    // explorer: argmin + tie-break (test_perf.cpp:71-106)
    const auto ex = explore_layouts(hw_preset("a100-sparse"), stencil_preset("Heat-2D"), d, 16, 16);
    CHECK(ex.ranked.size() == 256 && ex.best.t_total == ex.ranked.front().t_total);
    for (const auto& r : ex.ranked) CHECK(r.t_total >= ex.best.t_total);
    // descriptor parsing (test_perf.cpp:145-172)
    const auto hw = parse_hw_descriptor("name = t\ncpi_tcu = 16\nf = 1e9\nn_tcu = 4\nbw_g = 1e12\n"
                                        "bw_s = 1e13\nfrag_m = 16\nfrag_k = 32\nfrag_n = 8\n");
    CHECK(hw.name == "t" && hw.fragment.k == 32);
    CHECK_THROWS(parse_hw_descriptor("cpi_tcu = 16\n"));
    CHECK_THROWS(parse_hw_descriptor("cpi_tcu = x\nf=1\nn_tcu=1\nbw_g=1\nbw_s=1\n"));
    CHECK_THROWS(parse_hw_descriptor("bogus = 1\n"));
    CHECK_THROWS(hw_preset("h100"));
    // b200 tcgen05 explorer picks a legal M=128 layout, wide in x
    const auto t = explore_layouts_tcgen05(hw_preset("b200-sparse"), stencil_preset("Box-2D9P"),
                                           std::array<std::size_t, 2>{8192, 8192}, 128);
    CHECK(t.best.r1 * t.best.r2 == 128 && t.best.r1 == 16);
    // tall-narrow grids: the model may rank (8, 16) first, but the choice is the
    // layout sst_plan_create runs
    for (const auto& g : {std::vector<std::size_t>{8000, 40}, std::vector<std::size_t>{8000, 40, 20}}) {
        const auto s = stencil_preset(g.size() == 2 ? "Box-2D9P" : "Box-3D27P");
        const auto e = explore_layouts_tcgen05(hw_preset("b200-sparse"), s, g, 128);
        CHECK(e.best.r1 == 16 && e.best.r2 == 8 && device_runnable(e.best.r1, e.best.r2));
    }
}

// Emulate the sm_100a kernel's data path on the CPU from the device image the
// runtime uploads (A smem image, TMEM metadata words, koff) and compare with a
// brute-force sweep: proves the operand layouts (with the hardware conventions
// pinned by tools/probes/probe_sparse_mma.cu) and the patch/offset arithmetic.
static void image_tests() {
    for (const char* name : {"Heat-2D", "Box-2D9P", "Star-2D13P", "Box-2D49P", "Heat-3D", "Box-3D27P"}) {
        const auto s = stencil_preset(name);
        const int r = s.radius();
        std::vector<std::size_t> dims = s.dims == 2 ? std::vector<std::size_t>{83, 301}
                                                    : std::vector<std::size_t>{9, 21, 150};
        const auto L = crush(flatten(s, dims), 16, 8);
        const auto cv = convert_layout(L);
        const auto a2 = compress_24(cv.converted.a);
        BatchGeometry geo;
        geo.dims = s.dims;
        geo.k = s.k;
        geo.tiles_x = 8;
        geo.tiles_y = s.dims == 2 ? 8 : 2;
        geo.patch_planes = s.dims == 3 ? s.k : 1;
        const int lp = (4 - r % 4) % 4;
        geo.x_shift = lp;
        const std::size_t wv = cv.converted.stair.block_size, wu = cv.converted.stair.block_count;
        geo.patch_w = static_cast<int>((lp + wv + 16 * 7 + 3) / 4 * 4);
        geo.patch_h = static_cast<int>(wu) + 8 * (geo.tiles_y - 1);
        const auto img = build_device_image(geo, 128, cv.converted.a.cols, a2.values.data(),
                                            a2.meta.data(), cv.converted.col_origin.data(), wv, wu);
        const int k_pad = img.geo.k_pad;
        // the packed gather table the kernels read (one word per lane and sweep) covers
        // every K row exactly once with its patch offset, for fp32 and binary16 patches
        auto packed_ok = [&](const DeviceImage& im) {
            std::vector<int> seen(static_cast<std::size_t>(im.geo.k_pad), 0);
            bool good = im.gather_packed.size() == static_cast<std::size_t>(im.geo.k_pad);
            for (std::size_t i = 0; good && i < im.gather_packed.size(); ++i) {
                const uint32_t e = static_cast<uint32_t>(im.gather_packed[i]);
                const uint32_t src = (e & 0xffffu) << 1, row = e >> 16;
                good = row < seen.size() && src == static_cast<uint32_t>(im.koff[row] * im.geo.elem_bytes);
                if (good) ++seen[row];
            }
            for (int c : seen) good = good && c == 1;
            return good;
        };
        CHECK(packed_ok(img));
        {
            BatchGeometry gh = geo;
            gh.elem_bytes = 2;
            gh.x_shift = (8 - r % 8) % 8 & 7;
            gh.patch_w = static_cast<int>((gh.x_shift + wv + 16 * 7 + 7) / 8 * 8);
            const auto img_h = build_device_image(gh, 128, cv.converted.a.cols, a2.values.data(), a2.meta.data(),
                                                  cv.converted.col_origin.data(), wv, wu);
            CHECK(packed_ok(img_h));
        }
        // decode A'' (dense, k_pad wide) back from the smem image + metadata words
        std::vector<double> A(128 * static_cast<std::size_t>(k_pad), 0.0);
        for (int m = 0; m < 128; ++m)
            for (int g = 0; g < k_pad / 4; ++g) {
                const int st = g / 8, gl = g % 8;
                const int m0 = m % 8, m1 = (m / 8) % 2, m2 = m / 16;
                const uint32_t word = img.e_words[static_cast<std::size_t>(st * 128 + m0 + 8 * (gl / 4) + 16 * m2)];
                const uint32_t nib = (word >> (4 * ((gl % 4) + 4 * m1))) & 0xf;
                for (int slot = 0; slot < 2; ++slot) {
                    const int j = 2 * g + slot, jj = j % 16;
                    const std::size_t at = static_cast<std::size_t>((j / 16) * 2048 + (m / 8) * 128 +
                                                                    (jj / 8) * 64 + (m % 8) * 8 + jj % 8);
                    const uint16_t h = img.a_smem[at];
                    // fp16 -> double (normal/zero only: preset weights)
                    const int e = (h >> 10) & 0x1f;
                    const double v = h == 0 ? 0.0 : std::ldexp(1.0 + (h & 0x3ff) / 1024.0, e - 15) * ((h & 0x8000) ? -1 : 1);
                    const int pos = (nib >> (2 * slot)) & 3;
                    A[static_cast<std::size_t>(m) * k_pad + 4 * g + pos] += v;
                }
            }
        bool a_ok = true;
        for (std::size_t m = 0; m < 128; ++m)
            for (std::size_t q = 0; q < cv.converted.a.cols; ++q)
                a_ok = a_ok && A[m * k_pad + q] == cv.converted.a.at(m, q);
        CHECK(a_ok);
        // storage + patches + gather + MMA, every batch of the grid
        const Grid grid = random_grid(dims, 4);
        const auto want = brute(s, grid);
        const std::size_t gx = dims.back(), gy = dims[dims.size() - 2], gz = s.dims == 3 ? dims[0] : 1;
        const std::size_t pitch = (lp + gx + 3) / 4 * 4;
        auto stor = [&](long z, long y, long xs) -> double {  // storage coordinates, TMA OOB -> 0
            if (z < 0 || y < 0 || xs < 0 || z >= long(gz) || y >= long(gy) || xs >= long(pitch)) return 0.0;
            const long x = xs - lp;
            if (x < 0 || x >= long(gx)) return 0.0;  // pads hold zeros after bind
            return grid.values[(static_cast<std::size_t>(z) * gy + static_cast<std::size_t>(y)) * gx + static_cast<std::size_t>(x)];
        };
        const std::size_t ox = gx - 2 * r, oy = gy - 2 * r, oz = s.dims == 3 ? gz - 2 * r : 1;
        const int bw = 128, bh = 8 * geo.tiles_y;
        std::size_t checked = 0;
        bool ok = true;
        for (std::size_t Z0 = 0; Z0 < oz; ++Z0)
            for (std::size_t Y0 = 0; Y0 < oy; Y0 += bh)
                for (std::size_t X0 = 0; X0 < ox; X0 += bw) {
                    std::vector<double> patch(static_cast<std::size_t>(geo.patch_planes * geo.patch_h * geo.patch_w));
                    for (int z = 0; z < geo.patch_planes; ++z)
                        for (int u = 0; u < geo.patch_h; ++u)
                            for (int v = 0; v < geo.patch_w; ++v)
                                patch[static_cast<std::size_t>((z * geo.patch_h + u) * geo.patch_w + v)] =
                                    stor(long(Z0) + z, long(Y0) + u, long(X0) + v);
                    for (int ty = 0; ty < geo.tiles_y; ++ty)
                        for (int tx = 0; tx < 8; ++tx) {
                            std::vector<double> B(static_cast<std::size_t>(k_pad));
                            for (int q = 0; q < k_pad; ++q)
                                B[static_cast<std::size_t>(q)] = patch[static_cast<std::size_t>(
                                    img.koff[static_cast<std::size_t>(q)] + ty * 8 * geo.patch_w + tx * 16)];
                            for (int m = 0; m < 128; ++m) {
                                const std::size_t x = X0 + tx * 16 + m / 8, y = Y0 + ty * 8 + m % 8;
                                if (x >= ox || y >= oy) continue;
                                double d = 0;
                                for (int q = 0; q < k_pad; ++q) d += A[static_cast<std::size_t>(m) * k_pad + q] * B[static_cast<std::size_t>(q)];
                                ok = ok && d == want[(Z0 * oy + y) * ox + x];
                                ++checked;
                            }
                        }
                }
        CHECK(ok && checked == want.size());
        if (!ok) std::printf("  image emulation mismatch for %s\n", name);
    }
}

int main(int argc, char** argv) {
    if (argc >= 2 && std::string(argv[1]) == "image") {
        image_tests();
        std::printf("%d checks, %d failures\n", g_checks, g_fail);
        return g_fail ? 1 : 0;
    }
    if (argc >= 7 && std::string(argv[1]) == "perf") {
        std::vector<std::size_t> dims;
        for (int i = 6; i < argc; ++i) dims.push_back(std::strtoull(argv[i], nullptr, 10));
        const auto e = estimate(hw_preset(argv[2]), static_cast<int>(dims.size()), dims,
                                std::atoi(argv[3]), std::atoi(argv[4]), std::atoi(argv[5]));
        std::printf("{\"t_compute\": %.17g, \"t_memory\": %.17g, \"t_total\": %.17g, \"n_prime\": %zu, "
                    "\"n_mma\": %llu}\n",
                    e.t_compute, e.t_memory, e.t_total, e.n_prime,
                    static_cast<unsigned long long>(e.n_mma));
        return 0;
    }
    spec_tests();
    layout_tests();
    convert_tests();
    s24_tests();
    perf_tests();
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
