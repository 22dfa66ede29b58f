// multi.cu — slab decomposition of one compiled operator over several slabs
// (GPUs of one node, or several slabs per GPU) inside ONE process, behind the C
// ABI (sst_multi_*, sst_run_steps_multi).
//
// The reference has no multi-device path: its sweep is direct_apply(spec, grid,
// steps) (stencil.hpp:72) on one host thread. Here slab i owns global slices
// [a_i, b_i) of the slowest axis and stores r halo slices per neighbour; every
// step is ONE launch per slab whose epilogue also TMA-stores the first / last r
// interior slices straight into the neighbours' halo slices (sst_plan_set_peer:
// NVLink peer memory, or the same GPU). Slabs are ordered on their streams by flag
// words: after launch u a slab writes u + 1 into both neighbours' flags
// (cuStreamWriteValue32), before launch u it waits until its own flags are >= u
// (cuStreamWaitValue32): its halos for step u are in place and the neighbours no
// longer read the buffers its halo stores go to. No host synchronisation and no
// exchange step inside a run.
//
// Not a CUDA graph: the stream waits compare against absolute launch counts, which a
// replayed graph would repeat; the host enqueue (5 calls per slab and step) costs
// a few microseconds per step against >= 160 us of device time per step for the
// 1024^3 north-star grid on 8 GPUs.
#include <cuda_runtime.h>

#include <algorithm>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../host/capi_internal.hpp"
#include "launch_util.cuh"
#include "sparstencil.h"

namespace {

using sstl::ck;

void check(sst_status s) {
    if (s != SST_OK) {
        const std::string msg = sst_last_error();
        switch (s) {
            case SST_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
            case SST_ERR_LOGIC: throw std::logic_error(msg);
            case SST_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
            case SST_ERR_NO_DEVICE: throw sstc::CudaError(msg, true);
            case SST_ERR_CUDA: throw sstc::CudaError(msg, false);
            default: throw std::runtime_error(msg);
        }
    }
}

struct Slab {
    int device = 0;
    uint64_t a = 0, b = 0;    // owned global slices [a, b)
    uint64_t lo = 0, hi = 0;  // stored global slices [lo, hi) (owned + halos)
    sst_plan* plan = nullptr;
    cudaStream_t stream = nullptr;
    uint32_t* flags = nullptr;  // [from upper neighbour, from lower neighbour]: its finished launches
};

}  // namespace

struct sst_multi {
    std::vector<Slab> slabs;
    int dims = 2, r = 1;
    uint64_t fuse = 1;
    uint64_t global[3] = {0, 0, 0};
    uint64_t slice_elems = 0;  // cells per slice of the slowest axis
    uint32_t launches = 0;     // launches every slab has enqueued (flag epoch)
    int cur = 0;               // buffer holding the current state (same parity on every slab)

    ~sst_multi() {
        for (auto& s : slabs) {
            cudaSetDevice(s.device);
            if (s.stream) cudaStreamSynchronize(s.stream);
        }
        for (auto& s : slabs) {
            cudaSetDevice(s.device);
            if (s.plan) sst_plan_destroy(s.plan);
            if (s.flags) cudaFree(s.flags);
            if (s.stream) cudaStreamDestroy(s.stream);
        }
    }

    void sync_all() {
        for (auto& s : slabs) {
            ck(cudaSetDevice(s.device), "cudaSetDevice");
            ck(cudaStreamSynchronize(s.stream), "cudaStreamSynchronize");
        }
    }
};

extern "C" {

sst_status sst_multi_create(const sst_plan_desc* global, int nslabs, const int* devs, sst_multi** out) {
    try {
        if (!global || !devs || !out) throw std::invalid_argument("null argument");
        *out = nullptr;
        if (nslabs < 1) throw std::invalid_argument("need at least one slab");
        if (global->fold_n) throw std::invalid_argument("slab decomposition of a 1D fold is not supported");
        if (global->dims != 2 && global->dims != 3) throw std::invalid_argument("device path supports 2D and 3D");
        auto M = std::make_unique<sst_multi>();
        M->dims = global->dims;
        M->r = (global->k - 1) / 2;  // halo of one (possibly fused) launch
        M->fuse = global->fuse > 1 ? global->fuse : 1;
        for (int a = 0; a < 3; ++a) M->global[a] = global->grid_dims[a];
        const uint64_t G = global->grid_dims[0];
        M->slice_elems = 1;
        for (int a = 1; a < global->dims; ++a) M->slice_elems *= global->grid_dims[a];
        const uint64_t r = static_cast<uint64_t>(M->r);
        // even split of the slowest axis; every slab needs >= 2r owned slices so the
        // slices it sends are its own computed interior (the edge slabs' owned slices
        // include the global boundary ring)
        const uint64_t n = static_cast<uint64_t>(nslabs), base = G / n, extra = G % n;
        uint64_t a = 0;
        for (int i = 0; i < nslabs; ++i) {
            Slab s;
            s.device = devs[i];
            s.a = a;
            s.b = a + base + (static_cast<uint64_t>(i) < extra ? 1 : 0);
            a = s.b;
            s.lo = s.a >= r ? s.a - r : 0;
            s.hi = std::min(G, s.b + r);
            if (s.b - s.a < 2 * r)
                throw std::invalid_argument("slab " + std::to_string(i) + " owns too few slices for its halos");
            M->slabs.push_back(s);
        }
        for (auto& s : M->slabs) {
            sst_plan_desc d = *global;
            d.grid_dims[0] = s.hi - s.lo;
            check(sst_plan_create(&d, s.device, &s.plan));
            check(sst_plan_bind(s.plan, nullptr, nullptr));  // plan-owned (guard rows for peer maps)
            ck(cudaSetDevice(s.device), "cudaSetDevice");
            ck(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking), "cudaStreamCreate");
            ck(cudaMalloc(&s.flags, 8), "cudaMalloc(flags)");
            ck(cudaMemset(s.flags, 0, 8), "cudaMemset(flags)");
        }
        // neighbours on other GPUs: their memory must be reachable (NVLink / NVSwitch)
        for (std::size_t i = 0; i + 1 < M->slabs.size(); ++i) {
            const int d0 = M->slabs[i].device, d1 = M->slabs[i + 1].device;
            if (d0 == d1) continue;
            for (auto [x, y] : {std::pair<int, int>{d0, d1}, std::pair<int, int>{d1, d0}}) {
                int ok = 0;
                ck(cudaDeviceCanAccessPeer(&ok, x, y), "cudaDeviceCanAccessPeer");
                if (!ok)
                    throw sstc::CudaError("GPU " + std::to_string(x) + " cannot access peer GPU " + std::to_string(y),
                                          false);
                ck(cudaSetDevice(x), "cudaSetDevice");
                const cudaError_t e = cudaDeviceEnablePeerAccess(y, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled)
                    cudaGetLastError();
                else
                    ck(e, "cudaDeviceEnablePeerAccess");
            }
        }
        // binary16 pairs too (f16 plans), so runs keep binary16 between steps
        const bool h16 = global->precision == SST_PREC_F16;
        auto wire = [&](Slab& s, int which, const Slab& nb) {
            void *b0 = nullptr, *b1 = nullptr;
            check(sst_plan_buffers(nb.plan, &b0, &b1));
            check(sst_plan_set_peer(s.plan, which, b0, b1, nb.hi - nb.lo));
            void *h0 = nullptr, *h1 = nullptr;
            if (h16 && sst_plan_buffers_h(nb.plan, &h0, &h1) == SST_OK)
                check(sst_plan_set_peer_h(s.plan, which, h0, h1));
        };
        for (std::size_t i = 0; i < M->slabs.size(); ++i) {
            auto& s = M->slabs[i];
            if (i > 0) wire(s, 0, M->slabs[i - 1]);
            if (i + 1 < M->slabs.size()) wire(s, 1, M->slabs[i + 1]);
        }
        *out = M.release();
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

void sst_multi_destroy(sst_multi* m) { delete m; }

sst_status sst_multi_upload(sst_multi* m, const float* grid, int grid_on_device) {
    try {
        if (!m || !grid) throw std::invalid_argument("null argument");
        // neighbours' late halo stores must not land after (and overwrite) the upload
        m->sync_all();
        for (auto& s : m->slabs)
            check(sst_upload(s.plan, 0, grid + s.lo * m->slice_elems, grid_on_device, s.stream));
        // every slab loaded before any neighbour's first step stores halos into it
        m->sync_all();
        m->cur = 0;
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_multi_run(sst_multi* m, uint64_t steps) {
    try {
        if (!m) throw std::invalid_argument("null argument");
        if (steps % m->fuse != 0) throw std::invalid_argument("steps must be a multiple of the fusion factor");
        const std::size_t n = m->slabs.size();
        const uint64_t L = steps / m->fuse;
        // binary16 between steps when every slab's run qualifies (sstc::plan_h16_runner)
        std::vector<sst_plan*> hp(n, nullptr);
        bool h16 = L > 1;
        for (std::size_t i = 0; i < n && h16; ++i) h16 = (hp[i] = sstc::plan_h16_runner(m->slabs[i].plan, L)) != nullptr;
        if (h16) {
            std::vector<uint64_t> l0(n), h0(n);
            for (std::size_t i = 0; i < n; ++i) {
                auto& s = m->slabs[i];
                ck(cudaSetDevice(s.device), "cudaSetDevice");
                l0[i] = sstc::plan_launches(hp[i], false);
                h0[i] = sstc::plan_launches(hp[i], true);
                sstc::plan_h16_begin(hp[i], m->cur, s.stream);
            }
            for (uint64_t t = 0; t < L; ++t) {
                const uint32_t u = m->launches;
                for (std::size_t i = 0; i < n; ++i) {
                    auto& s = m->slabs[i];
                    ck(cudaSetDevice(s.device), "cudaSetDevice");
                    if (i > 0) sstl::stream_wait_geq(s.stream, s.flags + 0, u);
                    if (i + 1 < n) sstl::stream_wait_geq(s.stream, s.flags + 1, u);
                    sstc::plan_h16_step(hp[i], m->cur, t, L, s.stream);
                    if (i > 0) sstl::stream_write(s.stream, m->slabs[i - 1].flags + 1, u + 1);
                    if (i + 1 < n) sstl::stream_write(s.stream, m->slabs[i + 1].flags + 0, u + 1);
                }
                m->launches = u + 1;
            }
            for (std::size_t i = 0; i < n; ++i)
                if (hp[i] != m->slabs[i].plan)
                    sstc::plan_add_launches(m->slabs[i].plan, sstc::plan_launches(hp[i], false) - l0[i],
                                            sstc::plan_launches(hp[i], true) - h0[i]);
            m->cur = static_cast<int>((static_cast<uint64_t>(m->cur) + L) & 1);
            return SST_OK;
        }
        for (uint64_t t = 0; t < L; ++t) {
            const uint32_t u = m->launches;
            int dst = m->cur;
            for (std::size_t i = 0; i < n; ++i) {
                auto& s = m->slabs[i];
                ck(cudaSetDevice(s.device), "cudaSetDevice");
                if (i > 0) sstl::stream_wait_geq(s.stream, s.flags + 0, u);
                if (i + 1 < n) sstl::stream_wait_geq(s.stream, s.flags + 1, u);
                check(sst_run_steps(s.plan, m->cur, m->fuse, s.stream, &dst));
                if (i > 0) sstl::stream_write(s.stream, m->slabs[i - 1].flags + 1, u + 1);
                if (i + 1 < n) sstl::stream_write(s.stream, m->slabs[i + 1].flags + 0, u + 1);
            }
            m->cur = dst;
            m->launches = u + 1;
        }
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_multi_sync(sst_multi* m) {
    try {
        if (!m) throw std::invalid_argument("null argument");
        m->sync_all();
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_multi_download(sst_multi* m, float* grid, int grid_on_device) {
    try {
        if (!m || !grid) throw std::invalid_argument("null argument");
        for (auto& s : m->slabs)
            check(sst_download_slices(s.plan, m->cur, s.a - s.lo, s.b - s.a, grid + s.a * m->slice_elems,
                                      grid_on_device, s.stream));
        m->sync_all();
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_multi_slab(const sst_multi* m, int i, sst_plan** plan, void** stream, uint64_t owned[2]) {
    try {
        if (!m || i < 0 || static_cast<std::size_t>(i) >= m->slabs.size())
            throw std::invalid_argument("no such slab");
        const auto& s = m->slabs[static_cast<std::size_t>(i)];
        if (plan) *plan = s.plan;
        if (stream) *stream = s.stream;
        if (owned) {
            owned[0] = s.a;
            owned[1] = s.b;
        }
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_run_steps_multi(const sst_plan_desc* global, int ngpu, const int* devs, const float* h_in,
                               float* h_out, uint64_t steps) {
    try {
        if (!h_in || !h_out) throw std::invalid_argument("null argument");
        sst_multi* m = nullptr;
        check(sst_multi_create(global, ngpu, devs, &m));
        std::unique_ptr<sst_multi, void (*)(sst_multi*)> guard(m, sst_multi_destroy);
        check(sst_multi_upload(m, h_in, 0));
        check(sst_multi_run(m, steps));
        // boundary ring (first / last r global slices) and every owned slice
        check(sst_multi_download(m, h_out, 0));
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

}  // extern "C"
