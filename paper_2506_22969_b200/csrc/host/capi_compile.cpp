// C ABI, compile tier: host-only entry points (no GPU needed). The compile
// order mirrors the reference pipeline (proj/core/src/pipeline.cpp:56-78, 112):
// fuse -> choose (r1, r2) -> flatten -> crush -> convert_layout -> compress_24.
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "capi_internal.hpp"
#include "sparstencil.h"
#include "stensor/hwmodel.hpp"
#include "stensor/pipeline.hpp"
#include "stensor/morph.hpp"
#include "stensor/s24.hpp"
#include "stensor/sparsify.hpp"
#include "stensor/spec.hpp"

struct sst_compile_result {
    stensor::CompileResult res;
};

struct sst_compiled {
    stensor::StencilSpec spec;
    std::vector<std::size_t> dims;
    stensor::Conversion cv;
    stensor::Sparse24Matrix a2;
    std::vector<std::uint64_t> col_origin_u64;
    std::uint64_t fuse = 1;
    std::uint64_t fold_n = 0, fold_w = 0;  // 1D grid folded into a 2D view (device layout)
};

namespace sstc {

thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

sst_status from_current_exception() {
    try {
        throw;
    } catch (const std::invalid_argument& e) {
        set_error(e.what());
        return SST_ERR_INVALID_ARGUMENT;
    } catch (const std::out_of_range& e) {
        set_error(e.what());
        return SST_ERR_OUT_OF_RANGE;
    } catch (const std::logic_error& e) {
        set_error(e.what());
        return SST_ERR_LOGIC;
    } catch (const CudaError& e) {
        set_error(e.what());
        return e.no_device ? SST_ERR_NO_DEVICE : SST_ERR_CUDA;
    } catch (const std::exception& e) {
        set_error(e.what());
        return SST_ERR_RUNTIME;
    } catch (...) {
        set_error("unknown error");
        return SST_ERR_RUNTIME;
    }
}

}  // namespace sstc

namespace {

stensor::StencilSpec resolve_stencil(const char* text) {
    if (!text) throw std::invalid_argument("null stencil");
    const std::string s(text);
    if (stensor::is_preset(s)) return stensor::stencil_preset(s);
    if (s.find('=') != std::string::npos) return stensor::parse_stencil_spec(s);
    throw std::invalid_argument("unknown stencil preset: " + s);
}

stensor::HardwareDescriptor resolve_hw(const char* text) {
    const std::string s = text ? text : "a100-sparse";
    for (const auto& n : stensor::hw_preset_names())
        if (n == s) return stensor::hw_preset(s);
    if (s.find('=') != std::string::npos) return stensor::parse_hw_descriptor(s);
    throw std::invalid_argument("unknown hardware preset: " + s);
}

template <class T>
sst_status copy_out(const std::vector<T>& src, T* buf, size_t cap, size_t* len) {
    if (len) *len = src.size();
    if (!buf) return SST_OK;
    if (cap < src.size()) throw std::invalid_argument("output buffer too small");
    std::memcpy(buf, src.data(), src.size() * sizeof(T));
    return SST_OK;
}

}  // namespace

extern "C" {

sst_status sst_compile(const char* stencil, const uint64_t* grid_dims, int ndims, int r1, int r2,
                       uint64_t fuse, sst_compiled** out) {
    try {
        if (!out) throw std::invalid_argument("null output handle");
        *out = nullptr;
        auto c = std::make_unique<sst_compiled>();
        c->spec = resolve_stencil(stencil);
        if (fuse > 1) c->spec = stensor::fuse_time_steps(c->spec, fuse);
        c->fuse = fuse > 1 ? fuse : 1;
        if (ndims != c->spec.dims || !grid_dims)
            throw std::invalid_argument("grid dimensionality does not match stencil");
        c->dims.assign(grid_dims, grid_dims + ndims);
        if (c->spec.dims == 1 && r1 == 16 && r2 == 8) {
            // 1D on the device layout: fold the grid into a 2D view (rows of W interior
            // cells, W a multiple of the 128-wide batch) and embed the stencil as a 2D
            // star stencil along the rows; the kernel's patch rows overlap by the halo,
            // so the 1D neighbourhood of every cell is one view row.
            const std::size_t N = c->dims[0], k = static_cast<std::size_t>(c->spec.k), r = (k - 1) / 2;
            if (N < k) throw std::invalid_argument("grid smaller than kernel");
            const std::size_t n_int = N - 2 * r;
            const std::size_t W = std::min<std::size_t>(8192, (n_int + 127) / 128 * 128);
            const std::size_t R = (n_int + W - 1) / W;
            stensor::StencilSpec s2 = c->spec;
            s2.dims = 2;
            s2.shape = stensor::StencilShape::star;
            for (auto& pt : s2.points) pt.off = {0, pt.off[0], 0};
            stensor::validate(s2);
            c->spec = s2;
            c->dims = {R + 2 * r, W + 2 * r};
            c->fold_n = N;
            c->fold_w = W;
        }
        if (r1 <= 0 || r2 <= 0) {
            const auto ex = stensor::explore_layouts_tcgen05(stensor::hw_preset("b200-sparse"),
                                                             c->spec, c->dims, 128);
            r1 = ex.best.r1;
            r2 = ex.best.r2;
        }
        if (c->spec.dims == 1) r2 = 1;
        const auto flat = stensor::flatten(c->spec, c->dims);
        const auto morphed = stensor::crush(flat, r1, r2);
        c->cv = stensor::convert_layout(morphed);
        c->a2 = stensor::compress_24(c->cv.converted.a);
        c->col_origin_u64.resize(c->cv.converted.col_origin.size());
        for (std::size_t i = 0; i < c->col_origin_u64.size(); ++i)
            c->col_origin_u64[i] = c->cv.converted.col_origin[i] == stensor::npos
                                       ? UINT64_MAX
                                       : static_cast<uint64_t>(c->cv.converted.col_origin[i]);
        *out = c.release();
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

void sst_compiled_destroy(sst_compiled* c) { delete c; }

sst_status sst_compiled_info(const sst_compiled* c, sst_compile_info* info) {
    try {
        if (!c || !info) throw std::invalid_argument("null argument");
        const auto& L = c->cv.converted;
        *info = sst_compile_info{};
        info->dims = L.dims;
        info->k = c->spec.k;
        info->r1 = L.r1;
        info->r2 = L.r2;
        info->m_prime = L.m_prime;
        info->k_prime = L.k_prime;
        info->n_prime = L.n_prime;
        info->cols = L.a.cols;
        info->p = c->cv.p;
        info->align_cols = c->cv.align_cols;
        info->used_blossom = c->cv.used_blossom ? 1 : 0;
        info->refined = c->cv.matching.refined ? 1 : 0;
        info->window_w = L.stair.block_size;
        info->window_h = L.stair.block_count;
        info->window_d = L.z_factor;
        for (std::size_t a = 0; a < c->dims.size() && a < 3; ++a) info->grid_dims[a] = c->dims[a];
        info->fold_n = c->fold_n;
        info->fold_w = c->fold_w;
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_compiled_s24(const sst_compiled* c, uint32_t tag, uint8_t* buf, size_t cap,
                            size_t* len) {
    try {
        if (!c) throw std::invalid_argument("null compiled handle");
        const std::string bytes = stensor::sparse24_bytes(
            c->a2, tag ? stensor::Precision::round16 : stensor::Precision::exact64);
        std::vector<uint8_t> v(bytes.begin(), bytes.end());
        return copy_out(v, buf, cap, len);
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_compiled_perm(const sst_compiled* c, uint64_t* buf, size_t cap, size_t* len) {
    try {
        if (!c) throw std::invalid_argument("null compiled handle");
        std::vector<uint64_t> v(c->cv.perm.order.begin(), c->cv.perm.order.end());
        return copy_out(v, buf, cap, len);
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_compiled_col_origin(const sst_compiled* c, uint64_t* buf, size_t cap, size_t* len) {
    try {
        if (!c) throw std::invalid_argument("null compiled handle");
        return copy_out(c->col_origin_u64, buf, cap, len);
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_compiled_matrix(const sst_compiled* c, double* buf, size_t cap, size_t* len) {
    try {
        if (!c) throw std::invalid_argument("null compiled handle");
        return copy_out(c->cv.converted.a.data, buf, cap, len);
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_compiled_plan_desc(const sst_compiled* c, sst_plan_desc* d) {
    try {
        if (!c || !d) throw std::invalid_argument("null argument");
        const auto& L = c->cv.converted;
        *d = sst_plan_desc{};
        d->dims = L.dims;
        d->k = c->spec.k;
        d->r1 = L.r1;
        d->r2 = L.r2;
        for (std::size_t a = 0; a < c->dims.size() && a < 3; ++a) d->grid_dims[a] = c->dims[a];
        d->rows = c->a2.rows;
        d->cols = c->a2.logical_cols;
        d->a_values = c->a2.values.data();
        d->a_meta = c->a2.meta.data();
        d->col_origin = c->col_origin_u64.data();
        d->window_w = L.stair.block_size;
        d->window_h = L.stair.block_count;
        d->window_d = L.z_factor;
        d->precision = SST_PREC_F16;
        d->fuse = static_cast<uint32_t>(c->fuse);
        d->fold_n = c->fold_n;
        d->fold_w = c->fold_w;
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_random_grid(int ndims, const uint64_t* dims, uint64_t seed, float* out) {
    try {
        if (!dims || !out || ndims < 1 || ndims > 3) throw std::invalid_argument("bad grid");
        std::vector<std::size_t> d(dims, dims + ndims);
        const stensor::Grid g = stensor::random_grid(d, seed);
        for (std::size_t i = 0; i < g.values.size(); ++i) out[i] = static_cast<float>(g.values[i]);
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_run_compile(const sst_compile_request* q, sst_compile_result** out) {
    try {
        if (!q || !out) throw std::invalid_argument("null argument");
        *out = nullptr;
        if (!q->grid_dims || q->ndims < 1 || q->ndims > 3) throw std::invalid_argument("bad grid");
        stensor::CompileRequest req;
        req.spec = resolve_stencil(q->stencil);
        req.grid_dims.assign(q->grid_dims, q->grid_dims + q->ndims);
        req.hw = resolve_hw(q->hw);
        if (q->r1 > 0) {
            req.r1 = q->r1;
            req.r2 = q->r2 > 0 ? q->r2 : 1;
        }
        if (q->r_max > 0) req.r_max = q->r_max;
        req.fuse = q->fuse > 1 ? q->fuse : 1;
        req.precision = q->precision ? stensor::Precision::round16 : stensor::Precision::exact64;
        req.seed = q->seed ? q->seed : 1;
        if (q->out_dir) req.out_dir = q->out_dir;
        req.verify = q->verify != 0;
        req.device = q->device;
        req.corrupt_permutation = q->corrupt_permutation != 0;
        auto r = std::make_unique<sst_compile_result>();
        r->res = stensor::run_compile(req);
        *out = r.release();
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

void sst_compile_result_destroy(sst_compile_result* r) { delete r; }

sst_status sst_compile_result_summary(const sst_compile_result* r, sst_compile_summary* s) {
    try {
        if (!r || !s) throw std::invalid_argument("null argument");
        const auto& R = r->res;
        *s = sst_compile_summary{};
        s->ok = R.ok ? 1 : 0;
        s->r1 = R.plan.layout.r1;
        s->r2 = R.plan.layout.r2;
        s->used_blossom = R.plan.used_blossom ? 1 : 0;
        s->p = R.plan.p;
        s->align_cols = R.plan.align_cols;
        s->n_mma = R.perf.n_mma;
        s->issued_mma = R.issued_mma;
        s->m_prime = R.plan.layout.a.rows;
        s->k_prime = R.plan.layout.a.cols;
        s->n_prime = R.plan.layout.n_prime;
        s->t_compute = R.perf.t_compute;
        s->t_memory = R.perf.t_memory;
        s->t_total = R.perf.t_total;
        s->model_gstencil = R.model_gstencil;
        s->max_abs_err = R.verification.max_abs_err;
        s->max_rel_err = R.verification.max_rel_err;
        s->verify_seconds = R.emulation_seconds;
        std::strncpy(s->status, R.verification.status.c_str(), sizeof(s->status) - 1);
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_compile_result_report(const sst_compile_result* r, char* buf, size_t cap, size_t* len) {
    try {
        if (!r) throw std::invalid_argument("null result");
        const std::string& t = r->res.report_json;
        std::vector<char> v(t.begin(), t.end());
        return copy_out(v, buf, cap, len);
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_compile_result_lut(const sst_compile_result* r, uint8_t* buf, size_t cap, size_t* len) {
    try {
        if (!r) throw std::invalid_argument("null result");
        const std::string t = stensor::lut_bytes(r->res.plan.lut);
        std::vector<uint8_t> v(t.begin(), t.end());
        return copy_out(v, buf, cap, len);
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_explore(const char* stencil, const uint64_t* grid_dims, int ndims, const char* hw, uint64_t fuse,
                       int r_max, double* buf, size_t cap, size_t* len) {
    try {
        if (!grid_dims || ndims < 1 || ndims > 3) throw std::invalid_argument("bad grid");
        stensor::StencilSpec spec = resolve_stencil(stencil);
        if (fuse > 1) spec = stensor::fuse_time_steps(spec, fuse);
        const std::vector<std::size_t> dims(grid_dims, grid_dims + ndims);
        const int rm = r_max > 0 ? r_max : 16;
        const auto ex = stensor::explore_layouts(resolve_hw(hw), spec, dims, rm, rm);
        std::vector<double> v;
        for (const auto& e : ex.ranked)
            for (double x : {double(e.r1), double(e.r2), e.t_compute, e.t_memory, e.t_total, double(e.n_mma),
                             double(e.m_prime), double(e.k_prime), double(e.n_prime)})
                v.push_back(x);
        return copy_out(v, buf, cap, len);
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_estimate_device(const char* stencil, const uint64_t* grid_dims, int ndims, uint64_t fuse,
                               int storage, int tyb, double out[12]) {
    try {
        if (!out) throw std::invalid_argument("null argument");
        if (storage != 2 && storage != 4) throw std::invalid_argument("storage must be 2 (binary16) or 4 (fp32)");
        sst_compiled* c = nullptr;
        sst_status st = sst_compile(stencil, grid_dims, ndims, 16, 8, fuse, &c);
        if (st != SST_OK) return st;
        std::unique_ptr<sst_compiled, void (*)(sst_compiled*)> hold(c, sst_compiled_destroy);
        const auto& L = c->cv.converted;
        const int dims = L.dims;  // 1D grids are folded into a 2D view by sst_compile
        const int kz = dims == 3 && L.z_factor > 1 && L.a.cols % L.z_factor == 0 ? static_cast<int>(L.z_factor) : 1;
        const int t = tyb > 0 ? tyb : (dims == 3 && storage == 2 ? 8 : 4);
        const auto e = stensor::estimate_device(stensor::DeviceModel{}, dims, c->dims, c->spec.k, L.r1, L.r2,
                                                L.a.cols, kz, t, storage, storage, static_cast<int>(c->fuse));
        const double v[12] = {e.updates, e.batches, e.hbm_bytes, e.smem_wavefronts, e.mma_issues, e.t_hbm, e.t_smem,
                              e.t_mma, e.t_total, e.gstencil,
                              std::string(e.bound) == "hbm" ? 0.0 : std::string(e.bound) == "smem" ? 1.0 : 2.0,
                              std::ceil(static_cast<double>(L.a.cols) / kz / 32.0) * 32.0};
        std::memcpy(out, v, sizeof v);
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

const char* sst_last_error(void) { return sstc::g_last_error.c_str(); }

const char* sst_version(void) { return "sparstencil-b200 0.1.0 (sm_100a, tcgen05.mma.sp kind::f16)"; }

}  // extern "C"
