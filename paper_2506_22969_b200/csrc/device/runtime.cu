// runtime.cu — C ABI device tier: plan creation (constant operands to HBM),
// storage layout, TMA descriptors, the ping-pong time loop and host e2e.
// Replaces make_plan (proj/core/src/codegen.cpp:75-102) and the verification
// loop of run_compile (pipeline.cpp:115-153) with real device execution.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../host/capi_internal.hpp"
#include "sparstencil.h"
#include "stencil3d_kernel.cuh"
#include "launch_util.cuh"
#include "stencil_kernel.cuh"
#include "stensor/device_image.hpp"
#include "stensor/morph.hpp"

namespace {

using sstc::CudaError;

using namespace sstl;

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        ck(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q),
           "cudaGetDriverEntryPoint(cuTensorMapEncodeTiled)");
        if (!p || q != cudaDriverEntryPointSuccess)
            throw CudaError("cuTensorMapEncodeTiled unavailable", false);
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// One compiled instantiation of the step kernel: (dims, tile rows per batch,
// patch pipeline depth, A'' in TMEM or smem). Plans pick the first variant in
// preference order whose smem and TMEM budgets fit.
struct Variant {
    int dims, tyb, np;
    int kz;         // 0: whole-window kernel; > 0: 3D z-streaming kernel with kz z slices
    bool a_tmem;    // compressed A'' in TMEM
    int acc_cols;   // TMEM columns of the accumulator ring
    sst::SmemLayout (*layout)(int nks, int k_pad, int pw, int ph, int planes);
    void (*configure)(int smem);
    bool multistep;  // one launch can run many time steps (2D dataflow kernel)
    int ctas_per_sm = 1;  // co-resident CTAs the variant is built for (smem / TMEM / registers)
    void (*launch)(int grid, int smem, cudaStream_t st, const sst::MapSet& maps, const sst::StepParams& p,
                   bool cooperative);
    std::vector<sstl::TypedFns> h16c;  // binary16 inter-step storage instantiations (step_h16.cu), if any
};

template <int D, int TYB, int NP, bool AT, int NS = sst::kStageBufs, int CPS = 1>
Variant make_variant() {
    Variant v{};
    v.dims = D;
    v.tyb = TYB;
    v.np = NP;
    v.a_tmem = AT;
    v.acc_cols = 2 * sst::kTXB * TYB;
    v.ctas_per_sm = CPS;
    v.layout = [](int nks, int k_pad, int pw, int ph, int planes) {
        return sst::smem_layout<TYB, NP, AT, NS>(nks, k_pad, pw, ph, planes);
    };
    // 2D: one instantiation per time-loop mode (static / dynamic / multi-step)
    v.configure = [](int smem) {
        auto setup = [smem](KernelFn kernel) { raise_smem_attr(kernel, smem); };
        setup(sst::stencil_step_kernel<D, TYB, NP, AT, sst::kModeStatic, NS, CPS>);
        if constexpr (D == 2) {
            setup(sst::stencil_step_kernel<D, TYB, NP, AT, sst::kModeDynamic, NS, CPS>);
            setup(sst::stencil_step_kernel<D, TYB, NP, AT, sst::kModeMulti, NS, CPS>);
            setup(sst::stencil_step_kernel<D, TYB, NP, AT, sst::kModePeer, NS, CPS>);
            setup(sst::stencil_step_kernel<D, TYB, NP, AT, sst::kModeMultiDyn, NS, CPS>);
        }
    };
    v.multistep = D == 2;
    if constexpr (D == 2) v.h16c = sstl::typed_fns_2d(TYB, NP, AT, NS, CPS);
    v.launch = [](int grid, int smem, cudaStream_t st, const sst::MapSet& maps, const sst::StepParams& p,
                  bool coop) {
        if constexpr (D == 2) {
            if (p.multi_dyn)
                return launch_pdl(sst::stencil_step_kernel<D, TYB, NP, AT, sst::kModeMultiDyn, NS, CPS>, grid, smem, st,
                                  maps, p, coop);
            if (p.nsteps > 1)
                return launch_pdl(sst::stencil_step_kernel<D, TYB, NP, AT, sst::kModeMulti, NS, CPS>, grid, smem, st,
                                  maps, p, coop);
            if (p.sched && (p.peer_mask || p.nby1 != p.nby))
                return launch_pdl(sst::stencil_step_kernel<D, TYB, NP, AT, sst::kModePeer, NS, CPS>, grid, smem, st,
                                  maps, p, coop);
            if (p.sched)
                return launch_pdl(sst::stencil_step_kernel<D, TYB, NP, AT, sst::kModeDynamic, NS, CPS>, grid, smem, st,
                                  maps, p, coop);
        }
        launch_pdl(sst::stencil_step_kernel<D, TYB, NP, AT, sst::kModeStatic, NS, CPS>, grid, smem, st, maps, p, coop);
    };
    return v;
}

template <int TYB, int NP, int KZ, bool AT, int NB = 2, int NACC = KZ + 1, int NS = 1>
Variant make_stream_variant() {
    Variant v{};
    v.dims = 3;
    v.tyb = TYB;
    v.np = NP;
    v.kz = KZ;
    v.a_tmem = AT;
    v.acc_cols = NACC * sst::kTXB * TYB;
    v.layout = [](int nks, int k_pad, int pw, int ph, int) {
        return sst::smem_layout_stream<TYB, NP, KZ, NB, NACC, NS, AT>(nks, k_pad, pw, ph);
    };
    v.configure = [](int smem) {
        raise_smem_attr(sst::stencil3d_stream_kernel<TYB, NP, KZ, NB, NACC, NS, AT, false>, smem);
        raise_smem_attr(sst::stencil3d_stream_kernel<TYB, NP, KZ, NB, NACC, NS, AT, true>, smem);
    };
    v.multistep = false;
    v.h16c = sstl::typed_fns_3d(TYB, NP, KZ, AT, NB, NACC, NS);
    v.launch = [](int grid, int smem, cudaStream_t st, const sst::MapSet& maps, const sst::StepParams& p,
                  bool coop) {
        if (p.peer_mask)
            return launch_pdl(sst::stencil3d_stream_kernel<TYB, NP, KZ, NB, NACC, NS, AT, true>, grid, smem, st, maps,
                              p, coop);
        launch_pdl(sst::stencil3d_stream_kernel<TYB, NP, KZ, NB, NACC, NS, AT, false>, grid, smem, st, maps, p, coop);
    };
    return v;
}

// preference order per dimensionality: 3D z-streaming first, A'' in TMEM first,
// then the deepest TMA pipeline that fits (SST_VARIANT=<index> forces one, for
// experiments; SST_A_SMEM=1 skips the A''-in-TMEM variants)
const Variant* variants(int& n) {
    static const Variant v[] = {
        // 2D (measured order, tools/ablate.py): 0 TMEM-A 4x2 built for TWO co-resident CTAs
        // per SM (each CTA's pipeline bubbles filled by the other's; 81 KiB smem, <= 256 TMEM
        // columns, <= 102 registers): Box-2D9P 8192^2 83.0 us vs 83.2 for the best one-CTA
        // variant, Heat-2D 4096^2 24.8 vs 25.1, Star-2D13P 16384^2 341 vs 354, fused Box-2D9P
        // t = 3 / 4: 2254 / 2964 GSt/s vs 2166 / 2854; then the one-CTA variants: 1 TMEM-A 8x3
        // with two staging buffers, 2 TMEM-A 8x3, 3 TMEM-A 8x2, 4 TMEM-A 4x4, then smem-A
        make_variant<2, 4, 2, true, 1, 2>(), make_variant<2, 8, 3, true, 2>(), make_variant<2, 8, 3, true>(),
        make_variant<2, 8, 2, true>(), make_variant<2, 4, 4, true>(), make_variant<2, 8, 3, false>(),
        make_variant<2, 4, 4, false>(), make_variant<2, 4, 2, true>(), make_variant<2, 8, 2, false>(),
        make_variant<2, 4, 2, false>(),
        // 3D z-streaming (10-16): TMEM-A TYB 4 NP 4 (Box-3D27P 512^3: 206 us vs 222 smem-A), ...
        make_stream_variant<4, 4, 3, true>(), make_stream_variant<4, 3, 3, true>(),
        make_stream_variant<8, 3, 3, true>(), make_stream_variant<4, 2, 3, true>(),
        make_stream_variant<4, 6, 3, true>(), make_stream_variant<4, 4, 3, false>(),
        make_stream_variant<8, 2, 3, false>(),
        // pipeline-depth experiments with A'' in TMEM (19-24): <TYB, NP, KZ, AT, NB, NACC, NS>
        make_stream_variant<4, 6, 3, true, 4, 8, 2>(), make_stream_variant<4, 4, 3, true, 4, 8, 2>(),
        make_stream_variant<4, 6, 3, true, 6, 8, 2>(), make_stream_variant<4, 4, 3, true, 4, 8, 1>(),
        make_stream_variant<4, 4, 3, true, 2, 8, 1>(), make_stream_variant<8, 3, 3, true, 3, 5, 1>(),
        make_stream_variant<8, 2, 3, true, 2, 5, 2>(), make_stream_variant<8, 2, 3, true, 2, 4, 2>(),
        // 3D whole-window kernel (kz != 3 or non-streamable layouts): 25-27
        make_variant<3, 2, 4, false>(), make_variant<3, 2, 3, false>(), make_variant<3, 2, 2, false>(),
        // more 2D (28-31): <D, TYB, NP, AT, NS, CPS>
        make_variant<2, 8, 4, false>(), make_variant<2, 4, 3, true, 1, 2>(), make_variant<2, 4, 4, true, 2>(),
        make_variant<2, 8, 2, true, 2>(),
        // 3D z-streaming with KZ = 5 (temporally fused 3D stencils, k = 5: 40 K steps of A''):
        // 32-35 <TYB, NP, KZ, AT>
        make_stream_variant<2, 4, 5, true>(), make_stream_variant<2, 6, 5, true>(),
        make_stream_variant<4, 3, 5, false>(), make_stream_variant<2, 4, 5, false>(),
    };
    n = static_cast<int>(sizeof(v) / sizeof(v[0]));
    return v;
}

}  // namespace

namespace {
// Boundary ring of an fp32 storage buffer -> binary16 in both f16 buffers, one thread
// per ring cell (a flat index over the full ring rows — 2D: y < r, y >= gy - r; 3D also
// the whole ring planes — then the r left + r right cells of every other row). A
// warp-per-row loop serialised the full ring rows behind the possible aliasing of its
// loads and stores (8192-cell rows: 114 us per run; this: a few us).
// 3D slabs (halo_lo / halo_hi): the r planes at that z end are a neighbour's interior,
// written by its epilogue every step: only their x / y ring cells are converted
// (as for an interior plane), never their interior, which the neighbour may already
// have stored for this run.
__global__ void ring_to_half_kernel(const float* __restrict__ src, __half* __restrict__ d0,
                                    __half* __restrict__ d1, int gx, int gy, int gz, int r, long long rp,
                                    long long pp, int lp, long long rph, long long pph, int lph, int halo_lo,
                                    int halo_hi) {
    const bool d3 = gz > 1;
    // z planes converted whole: [0, zl) and [gz - zh, gz); the others [zl, gz - zh) like interior planes
    const int zl = d3 && !halo_lo ? r : 0, zh = d3 && !halo_hi ? r : 0;
    const int nin = d3 ? gz - zl - zh : 1;  // planes converted ring-only
    // 2D slabs: the r halo rows at a peer end are converted like interior rows (x ring only)
    const int yl = !d3 && halo_lo ? 0 : r, yh = !d3 && halo_hi ? 0 : r;  // whole ring rows per plane
    const long long full_planes_rows = static_cast<long long>(zl + zh) * gy;  // rows of the whole planes
    const long long full_rows = full_planes_rows + static_cast<long long>(yl + yh) * nin;  // + y ring rows
    const long long inner_rows = static_cast<long long>(gy - yl - yh) * nin;
    const long long n_full = full_rows * gx, n_all = n_full + inner_rows * 2 * r;
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n_all;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        int x, y, z;
        if (i < n_full) {
            const long long f = i / gx;
            x = static_cast<int>(i % gx);
            if (f < full_planes_rows) {
                const int pz = static_cast<int>(f / gy);
                y = static_cast<int>(f % gy);
                z = pz < zl ? pz : gz - zh - zl + pz;
            } else {
                const long long g = f - full_planes_rows;
                const int j = static_cast<int>(g % (yl + yh));
                z = d3 ? zl + static_cast<int>(g / (yl + yh)) : 0;
                y = j < yl ? j : gy - yl - yh + j;
            }
        } else {
            const long long g = i - n_full;
            const long long row = g / (2 * r);
            const int j = static_cast<int>(g % (2 * r));
            x = j < r ? j : gx - 2 * r + j;
            y = yl + static_cast<int>(row % (gy - yl - yh));
            z = d3 ? zl + static_cast<int>(row / (gy - yl - yh)) : 0;
        }
        const __half h = __float2half_rn(src[z * pp + y * rp + lp + x]);
        const long long o = z * pph + y * rph + lph + x;
        d0[o] = h;
        d1[o] = h;
    }
}
}  // namespace

void sstl::launch_ring_to_half(const float* src, __half* d0, __half* d1, int gx, int gy, int gz, int r, long long rp,
                               long long pp, int lp, long long rph, long long pph, int lph, cudaStream_t st,
                               bool halo_lo, bool halo_hi) {
    if (r == 0) return;
    ring_to_half_kernel<<<148 * 8, 256, 0, st>>>(src, d0, d1, gx, gy, gz, r, rp, pp, lp, rph, pph, lph,
                                                 halo_lo ? 1 : 0, halo_hi ? 1 : 0);
    launch_counter().fetch_add(1, std::memory_order_relaxed);
}

struct sst_plan {
    int device = 0;
    int dims = 2, k = 3, r = 1;
    int gx = 0, gy = 1, gz = 1;
    stensor::DeviceImage img;
    int tiles_y = 8;
    const Variant* variant = nullptr;
    sst_storage storage{};
    int smem = 0, num_sms = 0;
    int tmem_cols = 256;  // TMEM allocation of the chosen variant
    int zchunk = 0;       // 3D stream kernel unit order (SST_ZCHUNK; 0 = whole columns)
    unsigned long long* trace = nullptr;  // profiling: per-CTA timestamps (sst_plan_set_trace)
    // device constants
    void* d_a = nullptr;
    uint32_t* d_e = nullptr;
    int32_t* d_gsrc = nullptr;
    int32_t* d_gdst = nullptr;
    // ping-pong storage
    float* buf[2] = {nullptr, nullptr};
    bool owns_buf = false;
    float* alloc_base[2] = {nullptr, nullptr};  // owned buffers: allocation start (guard rows first)
    // owned 2D buffers start with kGuardRows rows that nothing reads: a lower
    // neighbour's halo stores may start up to a box height above its halo rows
    // (TMA store boxes cannot start at negative coordinates)
    static constexpr int64_t kGuardRows = 64;
    int64_t guard_elems() const { return dims == 2 ? kGuardRows * static_cast<int64_t>(storage.row_pitch) : 0; }
    sst::MapSet maps{};       // in[i]: patch loads over buffer i (whole storage);
                              // out[i]: stores into buffer i, clipped to the interior (and row window)
    uint32_t* d_sched = nullptr;  // dynamic batch counter of single-step 2D launches
    uint32_t sched_base = 0;
    uint32_t* d_flags = nullptr;  // progress words of multi-step launches (per CTA / per batch)
    int flag_mode = 0;            // what d_flags counts: 1 per-CTA iterations, 2 per-batch steps
    int flags_n = 0;
    uint32_t flag_base = 0;
    bool tmap_ok = false;
    int64_t map_lo = -1, map_hi = -1;  // row window the output maps were built for
    int64_t y_lo = 0, y_hi = -1;  // interior row window (two windows: their hull)
    int64_t y_hi1 = 0, y_lo2 = 0;  // two-window launches (2D): first window end, second start
    uint64_t launches = 0;
    int debug_mode = 0;  // SST_DEBUG_MODE (ablation experiments only)
    uint64_t fuse = 1;   // original time steps per launch
    int load_x0 = 0;     // storage column of a batch's patch start, relative to X0
    uint64_t fold_n = 0, fold_w = 0;  // 1D grid folded into the 2D view (see sst_compile)
    // slab P2P halos (sst_plan_set_peer): neighbour buffers by parity and slab size
    float* peer_buf[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [0 up, 1 down][parity]
    sst::PeerMaps peer_maps_h{};              // encoded here, copied to d_peer_maps
    sst::PeerMaps* d_peer_maps = nullptr;
    uint64_t peer_slices[2] = {0, 0};
    float* d_ring_save = nullptr;     // fold: the r right-ring cells, restored after a run
    // binary16 inter-step storage (SST_PREC_F16 runs of >= 2 steps, full window, no
    // peers / fold): steps 1 .. T-1 live in hbuf (ring: the f32 ring rounded once per
    // run), the last step writes the f32 buffer. img_h: gather tables for f16 patches.
    bool h16_ok = false;              // plan / variant support it
    sstl::TypedFns h16{};             // the chosen binary16 instantiations
    int smem_h = 0, smem_f32_h = 0;   // dynamic smem of the binary16-input / fp32-input typed kernels
    int occ_smem = 0;                 // smem floor keeping CTAs per SM within the TMEM budget
    int tmem_cols_h = 0;              // TMEM allocation of the typed kernels
    stensor::DeviceImage img_h;
    int32_t* d_gsrc_h = nullptr;
    int32_t* d_gdst_h = nullptr;
    sst_storage storage_h{};
    int load_x0_h = 0;
    __half* hbuf[2] = {nullptr, nullptr};
    __half* hbuf_base[2] = {nullptr, nullptr};  // allocations (2D: kGuardRows rows before hbuf, as buf)
    int64_t guard_elems_h() const { return dims == 2 ? kGuardRows * static_cast<int64_t>(storage_h.row_pitch) : 0; }
    CUtensorMap hin[2]{}, hout[2]{};  // f16 patch loads / interior stores
    CUtensorMap hring[2]{};           // 3D: the f16 buffers' right-edge ring chunks (kEdgeRing)
    // 3D slabs with P2P halos in binary16 runs: the neighbours' binary16 buffers
    // (sst_plan_set_peer_h) and, per launch kind, the PeerMaps the kernel reads at
    // [p.src ^ 1] = [1]: {f16 out hbuf[0], f16 out hbuf[1], fp32 out buf[0], fp32 out buf[1]}
    __half* peer_hbuf[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    sst::PeerMaps* d_peer_maps_run = nullptr;
    bool run_maps_ok = false;
    sst::GroupMaps* d_group = nullptr;  // grouped batch runs (h16_run_group)
    std::size_t group_cap = 0;
    bool hmaps_ok = false;
    uint64_t h16_launches = 0;        // launches that read or wrote binary16 storage
    int variant_index = -1;
    // 3D: binary16 runs go through a companion plan over the SAME fp32 buffers built
    // for the variant that is fastest with binary16 storage (TYB = 8: N = 64 MMAs,
    // half the MMA issues per output; Box-3D27P 512^3 146 vs 180 us per step), while
    // this plan keeps the variant that is fastest for fp32 single steps (TYB = 4:
    // 194 vs 224 us), which the slab / peer paths use
    std::unique_ptr<sst_plan> typed;

    ~sst_plan() {
        cudaSetDevice(device);
        cudaFree(d_a);
        cudaFree(d_e);
        cudaFree(d_gsrc);
        cudaFree(d_gdst);
        cudaFree(d_flags);
        cudaFree(d_sched);
        cudaFree(d_ring_save);
        cudaFree(d_peer_maps);
        cudaFree(d_peer_maps_run);
        cudaFree(d_group);
        cudaFree(d_gsrc_h);
        cudaFree(d_gdst_h);
        cudaFree(hbuf_base[0]);
        cudaFree(hbuf_base[1]);
        if (owns_buf) {
            cudaFree(alloc_base[0]);
            cudaFree(alloc_base[1]);
        }
    }

    // L2 sector promotion of TMA traffic (SST_L2_PROMO=0/64/128/256 overrides;
    // experiments only): 128 B keeps a patch row's tail sector from dragging a
    // neighbour's 256 B into L2 when that neighbour is not running concurrently
    static CUtensorMapL2promotion l2_promotion() {
        const char* e = std::getenv("SST_L2_PROMO");
        const int v = e ? std::atoi(e) : 128;
        return v == 0     ? CU_TENSOR_MAP_L2_PROMOTION_NONE
               : v == 64  ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
               : v == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                          : CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    }

    static void encode(CUtensorMap* m, int rank, void* base, const cuuint64_t* dim,
                       const cuuint64_t* stride, const cuuint32_t* box, CUtensorMapSwizzle swz,
                       CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT32) {
        cuuint32_t estride[3] = {1, 1, 1};
        const CUresult rc = encode_fn()(m, dt, static_cast<cuuint32_t>(rank),
                                        base, dim, stride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                        swz, l2_promotion(),
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (rc != CUDA_SUCCESS)
            throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(rc) + ")", false);
    }

    // active interior window of the slowest axis, clamped
    void window(int32_t& lo, int32_t& hi) const {
        const int64_t slow = (dims == 3 ? gz : gy) - 2 * r;
        lo = static_cast<int32_t>(y_hi > y_lo ? std::min<int64_t>(y_lo, slow) : 0);
        hi = static_cast<int32_t>(y_hi > y_lo ? std::min<int64_t>(y_hi, slow) : slow);
    }

    void make_tmaps() {
        const cuuint64_t gstride[2] = {storage.row_pitch * 4, storage.plane_pitch * 4};
        int32_t lo, hi;
        window(lo, hi);
        if (fold_n) {
            // 1D fold: view row i = storage cells [i W, i W + lp + W + 2r) — rows overlap
            // by the halo (a TMA map may have row stride < row extent) — so every cell's
            // 1D neighbourhood lies in its view row; stores: rows of W interior cells
            // starting at the first interior cell lp + r
            if (y_hi > y_lo) throw std::invalid_argument("row windows are not supported for a 1D fold");
            const cuuint64_t fstride[1] = {fold_w * 4};
            const cuuint64_t rows = static_cast<cuuint64_t>(gy - 2 * r);
            for (int i = 0; i < 2; ++i) {
                const cuuint64_t gdim[2] = {(storage.left_pad + fold_w + 2 * r + 3) / 4 * 4, rows};
                const cuuint32_t box[2] = {static_cast<cuuint32_t>(img.geo.patch_w),
                                           static_cast<cuuint32_t>(img.geo.patch_h)};
                encode(&maps.in[i], 2, buf[i], gdim, fstride, box, CU_TENSOR_MAP_SWIZZLE_NONE);
                const cuuint64_t odim[2] = {fold_w, rows};
                const cuuint32_t obox[2] = {static_cast<cuuint32_t>(sst::kBoxW),
                                            static_cast<cuuint32_t>(tiles_y * sst::kTileH)};
                encode(&maps.out[i], 2, buf[i] + storage.left_pad + r, odim, fstride, obox,
                       CU_TENSOR_MAP_SWIZZLE_128B);
            }
            map_lo = lo;
            map_hi = hi;
            tmap_ok = true;
            return;
        }
        for (int i = 0; i < 2; ++i) {
            // loads: the whole storage buffer; boxes start on 16-byte aligned columns
            const cuuint64_t gdim[3] = {storage.row_pitch, static_cast<cuuint64_t>(gy),
                                        static_cast<cuuint64_t>(gz)};
            const cuuint32_t box[3] = {static_cast<cuuint32_t>(img.geo.patch_w),
                                       static_cast<cuuint32_t>(img.geo.patch_h),
                                       static_cast<cuuint32_t>(img.geo.patch_planes)};
            encode(&maps.in[i], dims, buf[i], gdim, gstride, box, CU_TENSOR_MAP_SWIZZLE_NONE);
            // stores: interior origin (16-byte aligned by the left pad), interior
            // extents, 2D rows restricted to the active window -> TMA clips the
            // boundary ring, ragged edges and everything outside the window
            const int64_t row0 = r + (dims == 2 ? lo : 0);
            const int64_t plane0 = dims == 3 ? r : 0;
            float* base = buf[i] + plane0 * static_cast<int64_t>(storage.plane_pitch) +
                          row0 * static_cast<int64_t>(storage.row_pitch) +
                          static_cast<int64_t>(storage.left_pad) + r;
            // inner extent ends on the last 16-byte boundary of the interior (TMA
            // clips the innermost dimension in 16-byte units); the kernel writes
            // the <= 3 remaining columns directly
            // the 3D stream kernel also stores the last 16-byte chunk [ox4, ox4 + 4),
            // staging its ring / pad cells with their current values (kEdgeRing)
            const int ox = gx - 2 * r;
            const int oxs = (variant && variant->kz > 0 && (ox & 3)) ? (ox & ~3) + 4 : (ox & ~3);
            const cuuint64_t odim[3] = {static_cast<cuuint64_t>(std::max(oxs, 4)),
                                        static_cast<cuuint64_t>(dims == 2 ? std::max(hi - lo, 1) : gy - 2 * r),
                                        static_cast<cuuint64_t>(gz - 2 * r)};
            const cuuint32_t obox[3] = {static_cast<cuuint32_t>(sst::kBoxW),
                                        static_cast<cuuint32_t>(tiles_y * sst::kTileH), 1u};
            encode(&maps.out[i], dims, base, odim, gstride, obox, CU_TENSOR_MAP_SWIZZLE_128B);
            if (dims == 3) {  // right-edge ring chunk loads of the 3D stream kernel
                const cuuint32_t rbox[3] = {4u, static_cast<cuuint32_t>(tiles_y * sst::kTileH), 1u};
                encode(&maps.ring[i], 3, buf[i], gdim, gstride, rbox, CU_TENSOR_MAP_SWIZZLE_NONE);
            }
            // neighbours' halo slices: the upper neighbour's last r slices receive this
            // rank's interior slices [0, r) (coordinates as for the local map); the
            // lower neighbour's first r slices receive [n_int - r, n_int) (the kernel
            // subtracts peer_down0 from the slow coordinate)
            const int64_t slice_pitch = dims == 3 ? static_cast<int64_t>(storage.plane_pitch)
                                                  : static_cast<int64_t>(storage.row_pitch);
            const int64_t inner0 = (dims == 3 ? r * static_cast<int64_t>(storage.row_pitch) : 0) +
                                   static_cast<int64_t>(storage.left_pad) + r;
            for (int w = 0; w < 2; ++w) {
                if (!peer_buf[w][i]) continue;
                // (2D lower peer: the map starts kGuardRows rows early, in its guard)
                const int64_t guard = (w == 1 && dims == 2) ? kGuardRows : 0;
                const int64_t first = w == 0 ? static_cast<int64_t>(peer_slices[0]) - r : -guard;  // peer slice
                float* pbase = peer_buf[w][i] + first * slice_pitch + inner0;
                cuuint64_t pdim[3] = {odim[0], odim[1], odim[2]};
                if (dims == 2)
                    pdim[1] = static_cast<cuuint64_t>(r + guard);
                else
                    pdim[2] = static_cast<cuuint64_t>(r);
                encode(w == 0 ? &peer_maps_h.up[i] : &peer_maps_h.down[i], dims, pbase, pdim, gstride, obox,
                       CU_TENSOR_MAP_SWIZZLE_128B);
            }
        }
        if (peer_buf[0][0] || peer_buf[1][0]) {
            if (!d_peer_maps) ck(cudaMalloc(&d_peer_maps, sizeof(sst::PeerMaps)), "cudaMalloc(peer maps)");
            ck(cudaMemcpy(d_peer_maps, &peer_maps_h, sizeof(sst::PeerMaps), cudaMemcpyHostToDevice),
               "cudaMemcpy(peer maps)");
        }
        map_lo = lo;
        map_hi = hi;
        tmap_ok = true;
    }

    sst::StepParams step_params(int src) const {
        sst::StepParams p{};
        p.a_img = static_cast<const uint4*>(d_a);
        p.e_words = d_e;
        p.gsrc = d_gsrc;
        p.gdst = d_gdst;
        p.buf[0] = buf[0];
        p.buf[1] = buf[1];
        p.src = src;
        p.nsteps = 1;
        p.flags = d_flags;
        p.flag_base = flag_base;
        p.row_pitch = static_cast<int64_t>(storage.row_pitch);
        p.plane_pitch = static_cast<int64_t>(storage.plane_pitch);
        p.left_pad = static_cast<int32_t>(storage.left_pad);
        p.load_x0 = load_x0;
        p.gx = gx;
        p.gy = gy;
        p.gz = gz;
        p.r = r;
        window(p.slow_lo, p.slow_hi);
        p.y_end = gy - 2 * r;
        const int bw = img.geo.tiles_x * sst::kTileW, bh = tiles_y * sst::kTileH;
        p.nbx = (gx - 2 * r + bw - 1) / bw;
        p.nby1 = 0;
        p.slow_lo2 = 0;
        if (dims == 2 && y_lo2 > 0 && y_hi > y_lo) {
            // two windows [slow_lo, hi1) and [lo2, slow_hi): the out maps span the hull; a
            // first-window batch running past hi1 rewrites rows the preceding interior
            // launch of the step already wrote, with the same values
            const int64_t slow = gy - 2 * r;
            const int32_t hi1 = static_cast<int32_t>(std::min<int64_t>(y_hi1, slow));
            p.slow_lo2 = static_cast<int32_t>(std::min<int64_t>(y_lo2, slow));
            p.nby1 = (hi1 - p.slow_lo + bh - 1) / bh;
            p.nby = p.nby1 + (p.slow_hi - p.slow_lo2 + bh - 1) / bh;
            p.nbz = 1;
        } else if (dims == 2) {
            p.nby = (p.slow_hi - p.slow_lo + bh - 1) / bh;
            p.nbz = 1;
        } else {
            p.nby = (p.y_end + bh - 1) / bh;
            p.nbz = std::max(0, p.slow_hi - p.slow_lo);
        }
        p.nbatch = p.nbx * p.nby * p.nbz;
        if (p.nby1 == 0) p.nby1 = p.nby;
        p.k_pad = img.geo.k_pad;
        p.nks = static_cast<int32_t>(img.a_smem.size() * 2 / 4096);  // K steps of the A'' image
        p.patch_w = img.geo.patch_w;
        p.patch_h = img.geo.patch_h;
        p.patch_planes = img.geo.patch_planes;
        p.debug_mode = debug_mode;
        p.tmem_cols = tmem_cols;
        p.zchunk = zchunk;
        p.lo_sweep0 = img.lo_sweep0;
        p.load_y0 = fold_n ? -r : 0;  // fold: view rows have no ring rows above them
        {   // slab P2P halos
            const int64_t n_int = (dims == 3 ? gz : gy) - 2 * r;
            p.peer_mask = (peer_buf[0][0] ? 1 : 0) | (peer_buf[1][0] ? 2 : 0);
            p.peer_maps = d_peer_maps;
            p.peer_down0 = static_cast<int32_t>(n_int - r);
            p.peer_down_c0 = static_cast<int32_t>(n_int - r - (dims == 2 ? kGuardRows : 0));
            p.peer_up_shift = static_cast<int64_t>(peer_slices[0]) - 2 * r;
            p.peer_down_shift = -n_int;
            for (int i = 0; i < 2; ++i) {
                p.peer_up_buf[i] = peer_buf[0][i];
                p.peer_down_buf[i] = peer_buf[1][i];
            }
        }
        p.trace = trace;
        if (fold_n && r > 0) {
            p.fold_ring = d_ring_save;
            p.fold_nint = static_cast<int64_t>(fold_n) - 2 * r;
            p.fold_w = static_cast<int32_t>(fold_w);
        }
        return p;
    }

    // SST_H16=0 keeps fp32 storage between steps (A/B experiments, tests; read per call)
    static bool h16_enabled() {
        const char* e = std::getenv("SST_H16");
        return !(e && std::atoi(e) == 0);
    }

    // binary16 storage buffers and their tensor maps (allocated on first use)
    void ensure_h16() {
        if (hmaps_ok) return;
        const size_t bytes = storage_h.bytes + static_cast<size_t>(guard_elems_h()) * 2;
        for (int i = 0; i < 2; ++i) {
            if (!hbuf_base[i]) {
                ck(cudaMalloc(&hbuf_base[i], bytes), "cudaMalloc(f16 grid)");
                ck(cudaMemset(hbuf_base[i], 0, bytes), "cudaMemset(f16 grid)");
                hbuf[i] = hbuf_base[i] + guard_elems_h();
            }
        }
        const cuuint64_t gstride[2] = {storage_h.row_pitch * 2, storage_h.plane_pitch * 2};
        const int ox = gx - 2 * r, ox8 = ox & ~7;
        // the 3D stream kernel stores the whole last 16-byte chunk (kEdgeRing)
        const int oxs = (variant->kz > 0 && (ox & 7)) ? ox8 + 8 : ox8;
        for (int i = 0; i < 2; ++i) {
            const cuuint64_t gdim[3] = {storage_h.row_pitch, static_cast<cuuint64_t>(gy), static_cast<cuuint64_t>(gz)};
            const cuuint32_t box[3] = {static_cast<cuuint32_t>(img_h.geo.patch_w),
                                       static_cast<cuuint32_t>(img_h.geo.patch_h),
                                       static_cast<cuuint32_t>(img_h.geo.patch_planes)};
            encode(&hin[i], dims, hbuf[i], gdim, gstride, box, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
            __half* base = hbuf[i] + (dims == 3 ? r * static_cast<int64_t>(storage_h.plane_pitch) : 0) +
                           static_cast<int64_t>(r) * static_cast<int64_t>(storage_h.row_pitch) +
                           static_cast<int64_t>(storage_h.left_pad) + r;
            const cuuint64_t odim[3] = {static_cast<cuuint64_t>(std::max(oxs, 8)),
                                        static_cast<cuuint64_t>(gy - 2 * r), static_cast<cuuint64_t>(gz - 2 * r)};
            const cuuint32_t obox[3] = {64u, static_cast<cuuint32_t>(tiles_y * sst::kTileH), 1u};
            encode(&hout[i], dims, base, odim, gstride, obox, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
            if (dims == 3) {
                const cuuint32_t rbox[3] = {8u, static_cast<cuuint32_t>(tiles_y * sst::kTileH), 1u};
                encode(&hring[i], 3, hbuf[i], gdim, gstride, rbox, CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
            }
        }
        hmaps_ok = true;
    }

    // A run of nsteps >= 2 with binary16 inter-step storage: f32 buf[src] -> hbuf[0]
    // -> hbuf[1] -> ... -> f32 buf[(src + nsteps) & 1] (the index plain ping-pong
    // would end on; when that is buf[src] itself, step 1 read it long before).
    // h16_begin converts the ring; h16_step(t) issues launch t of the run (the batch
    // driver, sst_run_steps_batch, interleaves the launches of several plans).
    void h16_begin(int src, cudaStream_t st) {
        ensure_h16();
        sstl::launch_ring_to_half(buf[src], hbuf[0], hbuf[1], gx, gy, gz, r,
                                  static_cast<long long>(storage.row_pitch), static_cast<long long>(storage.plane_pitch),
                                  static_cast<int>(storage.left_pad), static_cast<long long>(storage_h.row_pitch),
                                  static_cast<long long>(storage_h.plane_pitch), static_cast<int>(storage_h.left_pad),
                                  st, peer_buf[0][0] != nullptr, peer_buf[1][0] != nullptr);
        ck(cudaGetLastError(), "ring_to_half launch");
        if ((peer_buf[0][0] || peer_buf[1][0]) && !run_maps_ok) make_run_peer_maps();
    }

    // the PeerMaps of binary16 slab runs (see d_peer_maps_run): the neighbours' binary16
    // halo slices as this rank's interior coordinates address them (2D: rows, the lower
    // neighbour's map starting in its guard rows; 3D: planes), and the fp32 ones
    void make_run_peer_maps() {
        sst::PeerMaps pm[4]{};
        const int ox = gx - 2 * r, ox8 = ox & ~7;
        const int oxs = (dims == 3 && (ox & 7)) ? ox8 + 8 : ox8;  // (3D: kEdgeRing stores the last chunk)
        const cuuint64_t gstride[2] = {storage_h.row_pitch * 2, storage_h.plane_pitch * 2};
        const cuuint32_t obox[3] = {64u, static_cast<cuuint32_t>(tiles_y * sst::kTileH), 1u};
        const int64_t slice_pitch = static_cast<int64_t>(dims == 3 ? storage_h.plane_pitch : storage_h.row_pitch);
        const int64_t inner0 = (dims == 3 ? static_cast<int64_t>(r) * static_cast<int64_t>(storage_h.row_pitch) : 0) +
                               static_cast<int64_t>(storage_h.left_pad) + r;
        for (int w = 0; w < 2; ++w) {
            if (!peer_buf[w][0]) continue;
            const int64_t guard = (w == 1 && dims == 2) ? kGuardRows : 0;
            const int64_t first = w == 0 ? static_cast<int64_t>(peer_slices[0]) - r : -guard;
            for (int i = 0; i < 2; ++i) {
                __half* base = peer_hbuf[w][i] + first * slice_pitch + inner0;
                const cuuint64_t pdim[3] = {static_cast<cuuint64_t>(std::max(oxs, 8)),
                                            static_cast<cuuint64_t>(dims == 2 ? r + guard : gy - 2 * r),
                                            static_cast<cuuint64_t>(r)};
                encode(w == 0 ? &pm[i].up[1] : &pm[i].down[1], dims, base, pdim, gstride, obox,
                       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
                (w == 0 ? pm[2 + i].up[1] : pm[2 + i].down[1]) = w == 0 ? peer_maps_h.up[i] : peer_maps_h.down[i];
            }
        }
        if (!d_peer_maps_run) ck(cudaMalloc(&d_peer_maps_run, sizeof pm), "cudaMalloc(run peer maps)");
        ck(cudaMemcpy(d_peer_maps_run, pm, sizeof pm, cudaMemcpyHostToDevice), "cudaMemcpy(run peer maps)");
        run_maps_ok = true;
    }

    // launch t of a binary16 run of nsteps launches: parameters and tensor maps
    sst::StepParams h16_params(int src, uint64_t t, uint64_t nsteps, sst::MapSet& m) const {
        const int fin = static_cast<int>((static_cast<uint64_t>(src) + nsteps) & 1);
        const bool hi = t > 0, ho = t + 1 < nsteps;
        sst::StepParams p = step_params(src);
        m = sst::MapSet{};
        m.in[0] = m.in[1] = hi ? hin[(t - 1) & 1] : maps.in[src];
        m.out[0] = m.out[1] = ho ? hout[t & 1] : maps.out[fin];
        // 3D: the output storage's ring chunks (binary16: the output buffer's own,
        // converted from buf[src]; fp32: the input buffer's, never rewritten)
        m.ring[0] = m.ring[1] = ho ? hring[t & 1] : maps.ring[src];
        float* outp = ho ? reinterpret_cast<float*>(hbuf[t & 1]) : buf[fin];
        p.src = 0;
        p.buf[0] = p.buf[1] = outp;
        p.tmem_cols = tmem_cols_h;
        if (ho) {
            p.row_pitch = static_cast<int64_t>(storage_h.row_pitch);
            p.plane_pitch = static_cast<int64_t>(storage_h.plane_pitch);
            p.left_pad = static_cast<int32_t>(storage_h.left_pad);
        }
        if (hi) {
            p.load_x0 = load_x0_h;
            p.patch_w = img_h.geo.patch_w;
            p.gsrc = d_gsrc_h;
            p.gdst = d_gdst_h;
        }
        if (p.peer_mask) {  // the launch's output parity is [1] (p.src = 0)
            p.peer_maps = d_peer_maps_run + (ho ? static_cast<int>(t & 1) : 2 + fin);
            for (int w = 0; w < 2; ++w) {  // 2D plain right-edge peer stores
                float* nb = ho ? reinterpret_cast<float*>(peer_hbuf[w][t & 1]) : peer_buf[w][fin];
                (w == 0 ? p.peer_up_buf : p.peer_down_buf)[1] = nb;
            }
        }
        return p;
    }

    // issue one launch of a binary16 run (items: batches to draw; group launches
    // draw the batches of every grid of the group)
    void h16_issue(sst::StepParams& p, const sst::MapSet& m, bool hi, bool ho, int items, cudaStream_t st) {
        const int grid = grid_size(p);
        const char* dyn_e = std::getenv("SST_DYN");
        // (the store-only ablation, debug bit 32, has no producer to draw batches)
        // (the 3D stream kernel splits its work statically)
        // (2D slab peers and groups: only the dynamic instantiations carry them)
        const bool dyn = variant->kz == 0 && !(debug_mode & 32) &&
                         (p.peer_mask != 0 || p.group != nullptr ||
                          (dyn_e ? std::atoi(dyn_e) != 0 : p.nbatch >= 8 * grid));
        if (dyn && !d_sched) {
            ck(cudaMalloc(&d_sched, 4), "cudaMalloc(sched)");
            ck(cudaMemsetAsync(d_sched, 0, 4, st), "cudaMemsetAsync(sched)");
            sched_base = 0;
        }
        p.sched = dyn ? d_sched : nullptr;
        p.sched_base = sched_base;
        h16.launch(dyn, hi, ho, grid, hi ? smem_h : smem_f32_h, st, m, p);
        if (dyn)
            sched_base += static_cast<uint32_t>((items + sst::kDrawGroup - 1) / sst::kDrawGroup +
                                                grid * (sst::kDrawAhead - 1));
        ck(cudaGetLastError(), "kernel launch");
        ++launches;
        ++h16_launches;
    }

    void h16_step(int src, uint64_t t, uint64_t nsteps, cudaStream_t st) {
        sst::MapSet m;
        sst::StepParams p = h16_params(src, t, nsteps, m);
        // odd launches of a run draw batches in reverse order: they start on the rows the
        // previous launch stored last (still in L2); SST_REVERSE=0 off
        const char* rv = std::getenv("SST_REVERSE");
        p.reverse = (rv && std::atoi(rv) == 0) ? 0 : static_cast<int32_t>(t & 1);
        h16_issue(p, m, t > 0, t + 1 < nsteps, p.nbatch, st);
    }

    // A grouped binary16 run: `this` (the runner of the group's first plan) launches
    // every step once for all grids of `grp` (identical geometry and operators, see
    // sst_run_steps_batch); d_group holds 4 x G GroupMaps: first launch, middle launches
    // of even / odd t, last launch.
    void h16_run_group(const std::vector<sst_plan*>& grp, const int* src, uint64_t L, cudaStream_t st) {
        const std::size_t G = grp.size();
        for (sst_plan* q : grp) q->ensure_h16();
        std::vector<sst::GroupMaps> gm(4 * G);
        for (std::size_t i = 0; i < G; ++i) {
            const sst_plan* q = grp[i];
            const int s0 = src[i], fin = static_cast<int>((static_cast<uint64_t>(s0) + L) & 1);
            gm[i].in = q->maps.in[s0];  // first: fp32 in, binary16 out
            gm[i].out = q->hout[0];
            gm[i].out_buf = reinterpret_cast<float*>(q->hbuf[0]);
            for (int par = 0; par < 2; ++par) {  // middle launch t (t & 1 = par): binary16 both ways
                sst::GroupMaps& e = gm[(1 + par) * G + i];
                e.in = q->hin[(par + 1) & 1];
                e.out = q->hout[par];
                e.out_buf = reinterpret_cast<float*>(q->hbuf[par]);
            }
            sst::GroupMaps& e = gm[3 * G + i];  // last: binary16 in, fp32 out
            e.in = q->hin[(L - 2) & 1];
            e.out = q->maps.out[fin];
            e.out_buf = q->buf[fin];
        }
        if (group_cap < 4 * G) {
            cudaFree(d_group);
            d_group = nullptr;
            ck(cudaMalloc(&d_group, 4 * G * sizeof(sst::GroupMaps)), "cudaMalloc(group maps)");
            group_cap = 4 * G;
        }
        // pageable source: staged by the driver at the call, copied in stream order
        ck(cudaMemcpyAsync(d_group, gm.data(), 4 * G * sizeof(sst::GroupMaps), cudaMemcpyHostToDevice, st),
           "cudaMemcpyAsync(group maps)");
        for (std::size_t i = 0; i < G; ++i) grp[i]->h16_begin(src[i], st);
        for (uint64_t t = 0; t < L; ++t) {
            sst::MapSet m;
            sst::StepParams p = h16_params(src[0], t, L, m);
            const int kind = t == 0 ? 0 : t + 1 == L ? 3 : 1 + static_cast<int>(t & 1);
            p.group = d_group + static_cast<std::size_t>(kind) * G;
            p.group_n = static_cast<int32_t>(G);
            const char* rv = std::getenv("SST_REVERSE");  // (as h16_step: odd launches in reverse)
            p.reverse = (rv && std::atoi(rv) == 0) ? 0 : static_cast<int32_t>(t & 1);
            h16_issue(p, m, t > 0, t + 1 < L, p.nbatch * static_cast<int>(G), st);
        }
    }

    // grids another runner can launch together with this one (same shape, stencil
    // operator and storage: the constant operands and the tensor-map geometry agree)
    bool groupable_with(const sst_plan* o) const {
        return o->variant == variant && o->h16.launch == h16.launch && o->gx == gx && o->gy == gy && o->gz == gz &&
               o->dims == dims && o->r == r && o->fuse == fuse && o->device == device && !fold_n && !o->fold_n &&
               o->storage.row_pitch == storage.row_pitch && o->storage_h.row_pitch == storage_h.row_pitch &&
               o->img.a_smem == img.a_smem && o->img.e_words == img.e_words &&
               o->img.gather_packed == img.gather_packed && o->img_h.gather_packed == img_h.gather_packed &&
               o->smem_h == smem_h && o->smem_f32_h == smem_f32_h && o->tmem_cols_h == tmem_cols_h;
    }

    int launch_h16(int src, uint64_t nsteps, cudaStream_t st) {
        h16_begin(src, st);
        for (uint64_t t = 0; t < nsteps; ++t) h16_step(src, t, nsteps, st);
        return static_cast<int>((static_cast<uint64_t>(src) + nsteps) & 1);
    }

    // the plan that runs binary16 launches of `nsteps` operator steps, or null when the
    // run takes the fp32 path (same conditions as launch())
    sst_plan* h16_runner(uint64_t nsteps) {
        const char* ms_e = std::getenv("SST_MULTISTEP");
        const bool ms_env = ms_e && std::atoi(ms_e) != 0;
        const bool full = !(y_hi > y_lo);
        const bool multi = ms_env && variant->multistep && full && nsteps > 1 && !fold_n && !peer_buf[0][0] &&
                           !peer_buf[1][0];
        sst_plan* hp = typed ? typed.get() : this;
        // slab peers: every fp32 peer must have its binary16 pair registered too
        bool peers_ok = true;
        for (int w = 0; w < 2; ++w)
            if (peer_buf[w][0]) peers_ok &= hp->peer_buf[w][0] && hp->peer_hbuf[w][0];
        if (hp->h16_ok && h16_enabled() && !multi && full && nsteps > 1 && peers_ok) return hp;
        return nullptr;
    }

    // streaming kernels: (row-band groups) x nbx CTAs, see stencil3d_kernel.cuh;
    // the others: persistent CTAs striding over batches
    // cooperative: the multi-step launch with static ownership needs every CTA resident;
    // the driver's occupancy check for cooperative launches admits one CTA per SM here
    int grid_size(const sst::StepParams& p, bool cooperative = false) const {
        if (variant->kz > 0) {
            const int64_t bands = static_cast<int64_t>(p.nby) * p.nbz;
            const int64_t groups = std::max<int64_t>(1, std::min<int64_t>(num_sms / p.nbx, bands));
            return static_cast<int>(groups * p.nbx);
        }
        return std::min(p.nbatch, num_sms * (cooperative ? 1 : variant->ctas_per_sm));
    }

    // Launch `nsteps` operator applications starting from buffer src; returns the
    // buffer holding the result. Multi-step launches (opt-in, SST_MULTISTEP=1) need
    // the full window and a multi-step variant.
    int launch(int src, uint64_t nsteps, cudaStream_t st) {
        sst::StepParams p = step_params(src);
        if (p.nbatch <= 0 || nsteps == 0) return src;
        if (p.slow_lo != map_lo || p.slow_hi != map_hi) make_tmaps();  // window changed
        // Default: one launch per step, batches drawn dynamically, PDL overlapping
        // consecutive steps (Box-2D9P 8192^2: 83.4 us/step vs 86.4 for the
        // multi-step dataflow launch, whose static batch ownership inherits the
        // 15-20 % spread of per-SM speed). SST_MULTISTEP=1 selects the multi-step
        // launch (read per call: tests toggle it).
        // SST_MULTISTEP=2: the multi-step launch with dynamic batch ownership
        const char* ms_e = std::getenv("SST_MULTISTEP");
        const bool ms_env = ms_e && std::atoi(ms_e) != 0;
        const bool ms_dyn = ms_e && std::atoi(ms_e) == 2;
        const bool full = !(y_hi > y_lo);
        // (a fold's view rows depend on the next row's first cells: outside the
        // multi-step kernel's 3 x 3 batch neighbourhood, so folds run per step)
        const bool multi = ms_env && variant->multistep && full && nsteps > 1 && !fold_n && !peer_buf[0][0] &&
                           !peer_buf[1][0];
        const bool mdyn = multi && ms_dyn;
        if (sst_plan* hp = h16_runner(nsteps)) {
            if (hp == this) return launch_h16(src, nsteps, st);
            const uint64_t l0 = hp->launches, h0 = hp->h16_launches;
            const int fin = hp->launch_h16(src, nsteps, st);
            launches += hp->launches - l0;
            h16_launches += hp->h16_launches - h0;
            return fin;
        }
        const int grid = grid_size(p, multi && !mdyn);
        if (multi && flags_n < p.nbatch) {
            cudaFree(d_flags);
            d_flags = nullptr;
            ck(cudaMalloc(&d_flags, static_cast<size_t>(p.nbatch) * 4), "cudaMalloc(flags)");
            ck(cudaMemsetAsync(d_flags, 0, static_cast<size_t>(p.nbatch) * 4, st), "cudaMemsetAsync(flags)");
            flags_n = p.nbatch;
            flag_base = 0;
        }
        // the two multi-step modes count different things in the flag words (per CTA /
        // per batch): restart the counters when the mode changes
        if (multi && flag_mode != (mdyn ? 2 : 1)) {
            ck(cudaMemsetAsync(d_flags, 0, static_cast<size_t>(flags_n) * 4, st), "cudaMemsetAsync(flags)");
            flag_base = 0;
            flag_mode = mdyn ? 2 : 1;
        }
        int cur = src;
        uint64_t left = nsteps;
        // fold: the last view row's store boxes also cover the r right-ring cells; the
        // kernel stages their input values (saved here) in place of computed ones, so
        // the ring is fixed across steps as in 2D / 3D (fold_keep_ring)
        const size_t ring_off = static_cast<size_t>(storage.left_pad + fold_n - r);
        if (fold_n && r > 0) {
            if (!d_ring_save) ck(cudaMalloc(&d_ring_save, static_cast<size_t>(r) * 4), "cudaMalloc(ring)");
            ck(cudaMemcpyAsync(d_ring_save, buf[src] + ring_off, static_cast<size_t>(r) * 4,
                               cudaMemcpyDeviceToDevice, st), "cudaMemcpyAsync(ring save)");
        }
        while (left > 0) {
            // chunks keep flag counters far from wrap-around between resets
            // (mdyn: items t * nbatch + b stay below 2^31)
            const uint64_t cap = mdyn ? std::max<uint64_t>(1, 0x7fffffffu / static_cast<uint64_t>(p.nbatch)) : 1u << 16;
            const uint64_t chunk = multi ? std::min<uint64_t>({left, uint64_t{1} << 16, cap}) : 1;
            p = step_params(cur);
            p.nsteps = static_cast<int32_t>(chunk);
            p.flags = d_flags;
            p.flag_base = flag_base;
            // single-step 2D launches draw batches from a counter (load balance: the
            // static stride leaves a 15-20 % spread of CTA finish times); SST_DYN=0 off
            const char* dyn_e = std::getenv("SST_DYN");
            // (few batches per CTA: static striding; Heat-2D 4096^2, 14 batches per CTA,
            // back to back: dynamic 25.3-25.4 vs static 25.6-26.0 us; SST_DYN=1 forces
            // dynamic, 0 static)
            // (2D P2P halos: only the dynamic-peer instantiation carries the peer stores)
            // (the store-only ablation, debug bit 32, has no producer to draw batches)
            const bool dyn = mdyn || (!multi && variant->multistep && !(debug_mode & 32) &&
                                      (p.peer_mask != 0 || p.nby1 != p.nby ||
                                       (dyn_e ? std::atoi(dyn_e) != 0 : p.nbatch >= 8 * grid)));
            if (dyn && !d_sched) {
                ck(cudaMalloc(&d_sched, 4), "cudaMalloc(sched)");
                ck(cudaMemsetAsync(d_sched, 0, 4, st), "cudaMemsetAsync(sched)");
                sched_base = 0;
            }
            p.sched = dyn ? d_sched : nullptr;
            p.sched_base = sched_base;
            p.multi_dyn = mdyn ? 1 : 0;
            variant->launch(grid, smem, st, maps, p, multi && !mdyn);
            // (items - grid draws, plus one final draw per CTA)
            if (dyn)
                sched_base += static_cast<uint32_t>(
                    (p.nbatch * (mdyn ? chunk : 1) + sst::kDrawGroup - 1) / sst::kDrawGroup +
                    grid * (sst::kDrawAhead - 1));
            ck(cudaGetLastError(), "kernel launch");
            ++launches;
            if (mdyn) {  // per-batch step counters
                flag_base += static_cast<uint32_t>(chunk);
            } else if (multi) {  // per-CTA progress counters advance by nper iterations per step
                const uint64_t nper = (static_cast<uint64_t>(p.nbatch) + grid - 1) / grid;
                flag_base += static_cast<uint32_t>(nper * chunk);
            }
            cur = (cur + static_cast<int>(chunk & 1)) & 1;
            left -= chunk;
        }
        return cur;
    }
};

extern "C" {

unsigned long long sst_launch_count(void) { return sstl::launch_counter().load(); }

int sst_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

namespace {
// forced_variant >= 0: only that variant (else SST_VARIANT or the preference order)
std::unique_ptr<sst_plan> create_plan(const sst_plan_desc* d, int device, int forced_variant) {
        if (d->precision != SST_PREC_F16 && d->precision != SST_PREC_F16X2)
            throw std::invalid_argument("unsupported precision");
        const int terms = d->precision == SST_PREC_F16X2 ? 2 : 1;
        if (d->dims != 2 && d->dims != 3)
            throw std::invalid_argument("device path supports 2D and 3D stencils (m' = 128 needs r2 > 1)");
        if (d->fold_n && (d->dims != 2 || d->fold_w % 128 != 0 || d->fold_w == 0))
            throw std::invalid_argument("bad 1D fold");
        if (d->r1 != sst::kTileW || d->r2 != sst::kTileH || d->rows != 128)
            throw std::invalid_argument("device path needs the (r1, r2) = (16, 8) layout");
        if (d->k < 1 || d->k % 2 == 0) throw std::invalid_argument("k must be odd and >= 1");
        int ndev = 0;
        ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
        if (device < 0 || device >= ndev) throw CudaError("no such CUDA device", true);
        ck(cudaSetDevice(device), "cudaSetDevice");
        auto P = std::make_unique<sst_plan>();
        P->device = device;
        P->dims = d->dims;
        P->k = d->k;
        P->r = (d->k - 1) / 2;
        P->fuse = d->fuse > 1 ? d->fuse : 1;
        P->gx = static_cast<int>(d->grid_dims[d->dims - 1]);
        P->gy = static_cast<int>(d->grid_dims[d->dims - 2]);
        P->gz = d->dims == 3 ? static_cast<int>(d->grid_dims[0]) : 1;
        if (P->gx < d->k || P->gy < d->k || P->gz < (d->dims == 3 ? d->k : 1))
            throw std::invalid_argument("grid smaller than kernel");

        // storage: the first interior column (r) of every row lands on a 16-byte
        // boundary (TMA store requirement) in 2D. 3D: rows start on 128-byte lines (the z-streaming kernel's TMA stores then
        // write whole 32-byte sectors only; with its ring-chunk store the row ends
        // are whole sectors too. Measured: Box-3D27P 512^3 204 -> 196 us). 2D: 16 B.
        // SST_ALIGN=16|128 overrides (experiments).
        const char* al = std::getenv("SST_ALIGN");
        const int al_bytes = al ? std::atoi(al) : (d->dims == 3 ? 128 : 16);
        const uint64_t aln = al_bytes == 128 ? 32 : 4;  // elements
        const uint64_t lp = (aln - static_cast<uint64_t>(P->r) % aln) % aln;
        P->load_x0 = static_cast<int>(lp & ~uint64_t{3});  // 16-byte aligned patch start
        int max_smem = 0;
        ck(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device),
           "cudaDeviceGetAttribute");
        int smem_per_sm = 0;
        ck(cudaDeviceGetAttribute(&smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device),
           "cudaDeviceGetAttribute");
        ck(cudaDeviceGetAttribute(&P->num_sms, cudaDevAttrMultiProcessorCount, device),
           "cudaDeviceGetAttribute");
        const int k_pad = static_cast<int>((d->cols + 31) / 32 * 32) * terms;
        stensor::BatchGeometry geo;
        geo.dims = d->dims;
        geo.k = d->k;
        geo.tiles_x = 8;
        geo.terms = terms;
        geo.patch_planes = d->dims == 3 ? d->k : 1;
        // the patch is loaded from the 16-byte aligned storage column X0 + load_x0,
        // lp & 3 cells left of the window origin (TMA box starts must be aligned)
        geo.x_shift = static_cast<int>(lp & 3);
        geo.patch_w = static_cast<int>(sst::align_up(
            static_cast<uint32_t>((lp & 3) + d->window_w + sst::kTileW * (geo.tiles_x - 1)), 4));
        std::vector<std::size_t> origin(d->cols);
        for (std::size_t i = 0; i < d->cols; ++i)
            origin[i] = d->col_origin[i] == UINT64_MAX ? stensor::npos
                                                       : static_cast<std::size_t>(d->col_origin[i]);
        // 3D z-streaming needs A'' to split into kz 4-group-aligned z slices with
        // identical (u, v) order (true for expand_units layouts); probe it
        const int kz = d->dims == 3 ? static_cast<int>(d->window_d) : 0;
        bool can_stream = false;
        int k_pad_z = 0;
        if (kz > 1 && d->cols % static_cast<uint64_t>(kz) == 0) {
            try {
                stensor::BatchGeometry g2 = geo;
                g2.z_slices = kz;
                g2.patch_planes = 1;
                g2.patch_h = static_cast<int>(d->window_h);
                const auto probe = stensor::build_device_image(g2, d->rows, d->cols, d->a_values,
                                                               d->a_meta, origin.data(), d->window_w,
                                                               d->window_h);
                k_pad_z = probe.geo.k_pad;
                can_stream = true;
            } catch (const std::invalid_argument&) {
                can_stream = false;
            }
        }
        int nvar = 0;
        const Variant* vars = variants(nvar);
        const char* force = std::getenv("SST_VARIANT");
        const int forced = forced_variant >= 0 ? forced_variant : force ? std::atoi(force) : -1;
        const char* asm_env = std::getenv("SST_A_SMEM");
        const bool no_a_tmem = asm_env && std::atoi(asm_env) != 0;
        for (int i = 0; i < nvar && !P->variant; ++i) {
            const Variant& v = vars[i];
            if (v.dims != d->dims || (forced >= 0 && i != forced)) continue;
            if (v.kz > 0 && (!can_stream || v.kz != kz)) continue;
            if (v.a_tmem && no_a_tmem && forced < 0) continue;
            const int ph = static_cast<int>(d->window_h) + sst::kTileH * (v.tyb - 1);
            const int kp = v.kz > 0 ? k_pad_z : k_pad;
            const int nks = v.kz > 0 ? kz * k_pad_z / 32 : k_pad / 32;
            const int planes = v.kz > 0 ? 1 : geo.patch_planes;
            const sst::SmemLayout L = v.layout(nks, kp, geo.patch_w, ph, planes);
            const int need = static_cast<int>(L.total) + 1024;  // slack for the 1 KiB base alignment
            if (need > max_smem || ph > 256) continue;
            // co-resident CTAs: each takes its smem plus the 1 KiB the driver reserves per CTA
            if (v.ctas_per_sm > 1 && v.ctas_per_sm * (need + 1024) > smem_per_sm) continue;
            const uint32_t tneed =
                sst::tmem_budget(static_cast<uint32_t>(v.acc_cols), static_cast<uint32_t>(nks), v.a_tmem).need;
            if (tneed > 512) continue;
            if (v.ctas_per_sm > 1 && tneed > 512u / static_cast<uint32_t>(v.ctas_per_sm)) continue;
            if (sst::prologue_scratch_bytes(nks, v.a_tmem) > L.gsrc - L.b) continue;
            P->variant = &v;
            P->variant_index = i;
            P->smem = need;
            P->tmem_cols = tneed <= 32 ? 32 : tneed <= 64 ? 64 : tneed <= 128 ? 128 : tneed <= 256 ? 256 : 512;
            geo.tiles_y = v.tyb;
            geo.patch_h = ph;
            if (v.kz > 0) {
                geo.z_slices = kz;
                geo.patch_planes = 1;
            }
        }
        if (!P->variant)
            throw std::invalid_argument("stencil too wide for one CTA's shared memory");
        // Occupancy guard: a CTA that finds no free TMEM blocks in tcgen05.alloc until a
        // co-resident CTA retires — for a persistent CTA holding its first batch, the end
        // of the launch. So never let more CTAs share an SM than its 512 TMEM columns
        // hold: pad the dynamic smem instead (binary16 patches made the typed kernels
        // small enough for a third CTA per SM: Box-2D9P 78 -> 127 us per step).
        P->occ_smem = [&] {
            const int allowed = std::max(P->variant->ctas_per_sm, 512 / P->tmem_cols);
            return std::min(max_smem, smem_per_sm / (allowed + 1));
        }();
        P->smem = std::max(P->smem, P->occ_smem);
        P->tiles_y = geo.tiles_y;
        P->img = stensor::build_device_image(geo, d->rows, d->cols, d->a_values, d->a_meta,
                                             origin.data(), d->window_w, d->window_h);
        P->variant->configure(P->smem);
        if (const char* dm = std::getenv("SST_DEBUG_MODE")) P->debug_mode = std::atoi(dm);
        if (const char* zc = std::getenv("SST_ZCHUNK")) P->zchunk = std::atoi(zc);

        P->fold_n = d->fold_n;
        P->fold_w = d->fold_w;
        P->storage.left_pad = lp;
        P->storage.row_pitch = (lp + static_cast<uint64_t>(P->gx) + aln - 1) / aln * aln;
        {  // room for the 3D stream kernel's full last 16-byte store chunk
            const uint64_t ox = static_cast<uint64_t>(P->gx - 2 * P->r);
            const uint64_t need = lp + static_cast<uint64_t>(P->r) + (ox + 3) / 4 * 4;
            if (P->storage.row_pitch < need) P->storage.row_pitch = (need + aln - 1) / aln * aln;
        }
        P->storage.plane_pitch = P->storage.row_pitch * static_cast<uint64_t>(P->gy);
        P->storage.bytes = P->storage.plane_pitch * static_cast<uint64_t>(P->gz) * 4;
        if (P->fold_n) {  // 1D: contiguous cells, element p at left_pad + p; room for the
                          // last view row's loads (W + 2r + 3 past its start)
            const uint64_t rows = static_cast<uint64_t>(P->gy - 2 * P->r);
            P->storage.row_pitch = P->fold_w;
            P->storage.plane_pitch = rows * P->fold_w;
            const uint64_t cells = std::max<uint64_t>(lp + P->fold_n, rows * P->fold_w + lp + 2 * P->r + 4);
            P->storage.bytes = (cells + 3) / 4 * 4 * 4;
        }

        // binary16 inter-step storage: f16 operands only, full-grid runs (see launch)
        if (terms == 1 && !P->fold_n && !P->variant->h16c.empty()) {
            // the interior starts 16-byte aligned (2D) / 128-byte aligned (3D: whole-sector
            // TMA stores, as for the fp32 storage)
            const uint64_t alh = d->dims == 3 ? 64 : 8;  // elements
            const uint64_t lph = (alh - static_cast<uint64_t>(P->r) % alh) % alh;
            P->storage_h.left_pad = lph;
            P->storage_h.row_pitch = (lph + static_cast<uint64_t>(P->gx) + alh - 1) / alh * alh;
            {  // room for the 3D stream kernel's full last 16-byte store chunk
                const uint64_t ox = static_cast<uint64_t>(P->gx - 2 * P->r);
                const uint64_t need = lph + static_cast<uint64_t>(P->r) + (ox + 7) / 8 * 8;
                if (P->storage_h.row_pitch < need) P->storage_h.row_pitch = (need + alh - 1) / alh * alh;
            }
            P->storage_h.plane_pitch = P->storage_h.row_pitch * static_cast<uint64_t>(P->gy);
            P->storage_h.bytes = P->storage_h.plane_pitch * static_cast<uint64_t>(P->gz) * 2;
            P->load_x0_h = static_cast<int>(lph & ~uint64_t{7});
            stensor::BatchGeometry gh = geo;
            gh.elem_bytes = 2;
            gh.x_shift = static_cast<int>(lph & 7);
            gh.patch_w = static_cast<int>(
                sst::align_up(static_cast<uint32_t>(gh.x_shift + d->window_w + sst::kTileW * (gh.tiles_x - 1)), 8));
            const int nks = static_cast<int>(P->img.a_smem.size() * 2 / 4096);
            const auto& G = P->img.geo;
            const int cps = P->variant->ctas_per_sm;
            for (const auto& T : P->variant->h16c) {  // deepest pipeline that fits
                const uint32_t tneed = sst::tmem_budget(static_cast<uint32_t>(T.nacc * sst::kTXB * P->variant->tyb),
                                                        static_cast<uint32_t>(nks), true).need;
                const int tcols = tneed <= 32 ? 32 : tneed <= 64 ? 64 : tneed <= 128 ? 128 : tneed <= 256 ? 256 : 512;
                if (tneed > 512u / static_cast<uint32_t>(cps)) continue;
                // occupancy guard as for the plan's own kernels (TMEM-blocked CTAs)
                const int occ = std::min(max_smem, smem_per_sm / (std::max(cps, 512 / tcols) + 1));
                const int s32 = std::max(occ, T.smem(false, nks, G.k_pad, G.patch_w, G.patch_h, G.patch_planes));
                const int s16 = std::max(occ, T.smem(true, nks, G.k_pad, gh.patch_w, G.patch_h, G.patch_planes));
                const int worst = std::max(s32, s16);
                if (worst <= max_smem && (cps == 1 || cps * (worst + 1024) <= smem_per_sm)) {
                    P->h16 = T;
                    P->smem_f32_h = s32;
                    P->smem_h = s16;
                    P->tmem_cols_h = tcols;
                    break;
                }
            }
            if (gh.patch_w <= 256 && P->h16.launch) {
                P->img_h = stensor::build_device_image(gh, d->rows, d->cols, d->a_values, d->a_meta, origin.data(),
                                                       d->window_w, d->window_h);
                ck(cudaMalloc(&P->d_gsrc_h, P->img_h.gather_packed.size() * 4), "cudaMalloc");
                ck(cudaMemcpy(P->d_gsrc_h, P->img_h.gather_packed.data(), P->img_h.gather_packed.size() * 4,
                              cudaMemcpyHostToDevice), "cudaMemcpy");
                ck(cudaMalloc(&P->d_gdst_h, P->img_h.gather_dst.size() * 4), "cudaMalloc");
                ck(cudaMemcpy(P->d_gdst_h, P->img_h.gather_dst.data(), P->img_h.gather_dst.size() * 4,
                              cudaMemcpyHostToDevice), "cudaMemcpy");
                P->h16.configure(P->smem_f32_h, P->smem_h);
                P->h16_ok = true;
            }
        }
        ck(cudaMalloc(&P->d_a, P->img.a_smem.size() * 2), "cudaMalloc");
        ck(cudaMemcpy(P->d_a, P->img.a_smem.data(), P->img.a_smem.size() * 2, cudaMemcpyHostToDevice),
           "cudaMemcpy");
        ck(cudaMalloc(&P->d_e, P->img.e_words.size() * 4), "cudaMalloc");
        ck(cudaMemcpy(P->d_e, P->img.e_words.data(), P->img.e_words.size() * 4, cudaMemcpyHostToDevice),
           "cudaMemcpy");
        ck(cudaMalloc(&P->d_gsrc, P->img.gather_packed.size() * 4), "cudaMalloc");
        ck(cudaMemcpy(P->d_gsrc, P->img.gather_packed.data(), P->img.gather_packed.size() * 4,
                      cudaMemcpyHostToDevice),
           "cudaMemcpy");
        ck(cudaMalloc(&P->d_gdst, P->img.gather_dst.size() * 4), "cudaMalloc");
        ck(cudaMemcpy(P->d_gdst, P->img.gather_dst.data(), P->img.gather_dst.size() * 4,
                      cudaMemcpyHostToDevice),
           "cudaMemcpy");
        return P;
}

// 3D z-streaming variants in preference order for binary16 runs (see sst_plan::typed)
constexpr int kTyped3D[] = {12, 10};
}  // namespace

sst_status sst_plan_create(const sst_plan_desc* d, int device, sst_plan** out) {
    try {
        if (!d || !out) throw std::invalid_argument("null argument");
        *out = nullptr;
        auto P = create_plan(d, device, -1);
        const char* sub_e = std::getenv("SST_H16_SUBPLAN");
        if (P->dims == 3 && P->variant->kz > 0 && !P->fold_n && !std::getenv("SST_VARIANT") &&
            !(sub_e && std::atoi(sub_e) == 0) && d->precision == SST_PREC_F16) {
            for (const int vi : kTyped3D) {
                if (vi == P->variant_index) break;  // the plan's own variant is the typed choice
                std::unique_ptr<sst_plan> T;
                try {
                    T = create_plan(d, device, vi);
                } catch (const std::invalid_argument&) {
                    continue;  // does not fit this stencil
                }
                if (!T->h16_ok || T->variant->kz != P->variant->kz) continue;
                P->typed = std::move(T);
                break;
            }
        }
        *out = P.release();
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

void sst_plan_destroy(sst_plan* plan) { delete plan; }

sst_status sst_plan_storage(const sst_plan* plan, sst_storage* st) {
    try {
        if (!plan || !st) throw std::invalid_argument("null argument");
        *st = plan->storage;
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_plan_stats_get(const sst_plan* plan, sst_plan_stats* s) {
    try {
        if (!plan || !s) throw std::invalid_argument("null argument");
        const auto& G = plan->img.geo;
        *s = sst_plan_stats{};
        s->k_pad = G.k_pad;
        s->k_steps = G.k_pad / 32;
        s->tiles_x = G.tiles_x;
        s->tiles_y = plan->tiles_y;
        s->patch_w = G.patch_w;
        s->patch_h = G.patch_h;
        s->patch_planes = G.patch_planes;
        s->worst_bank_conflict = plan->img.worst_bank_conflict;
        s->patch_stages = plan->variant->np;
        s->smem_bytes = plan->smem;
        const sst::StepParams p = plan->step_params(0);
        s->batches = p.nbatch;
        s->ctas = plan->grid_size(p);
        s->launches = plan->launches;
        s->h16_launches = plan->h16_launches;
        const sst_plan* hp = plan->typed ? plan->typed.get() : plan;  // the plan binary16 runs use
        s->h16_capable = hp->h16_ok ? 1 : 0;
        s->h16_patch_stages = hp->h16_ok ? hp->h16.np_h16 * 100 + hp->h16.nbb * 10 + hp->h16.nacc : 0;
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_plan_bind(sst_plan* plan, void* b0, void* b1) {
    try {
        if (!plan) throw std::invalid_argument("null plan");
        ck(cudaSetDevice(plan->device), "cudaSetDevice");
        if (plan->owns_buf) {
            cudaFree(plan->alloc_base[0]);
            cudaFree(plan->alloc_base[1]);
            plan->alloc_base[0] = plan->alloc_base[1] = nullptr;
            plan->owns_buf = false;
        }
        if (!b0 && !b1) {
            const size_t guard = static_cast<size_t>(plan->guard_elems()) * 4;
            for (int i = 0; i < 2; ++i) {
                void* a = nullptr;
                ck(cudaMalloc(&a, plan->storage.bytes + guard), "cudaMalloc(grid)");
                ck(cudaMemset(a, 0, guard), "cudaMemset(guard)");
                plan->alloc_base[i] = static_cast<float*>(a);
                plan->buf[i] = plan->alloc_base[i] + plan->guard_elems();
            }
            plan->owns_buf = true;
        } else {
            if (!b0 || !b1) throw std::invalid_argument("bind needs two buffers (or none)");
            if ((reinterpret_cast<uintptr_t>(b0) | reinterpret_cast<uintptr_t>(b1)) & 15u)
                throw std::invalid_argument("grid buffers must be 16-byte aligned");
            plan->buf[0] = static_cast<float*>(b0);
            plan->buf[1] = static_cast<float*>(b1);
        }
        ck(cudaMemset(plan->buf[0], 0, plan->storage.bytes), "cudaMemset");
        ck(cudaMemset(plan->buf[1], 0, plan->storage.bytes), "cudaMemset");
        plan->make_tmaps();
        // binary16 storage pair up front (not inside the first timed run)
        if (plan->typed) {  // the companion plan works on the same fp32 buffers
            plan->typed->buf[0] = plan->buf[0];
            plan->typed->buf[1] = plan->buf[1];
            plan->typed->make_tmaps();
            plan->typed->ensure_h16();
        } else if (plan->h16_ok) {
            plan->ensure_h16();
        }
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

static void copy_dense(sst_plan* plan, int which, const float* src, float* dst, bool to_storage,
                       bool other_on_device, cudaStream_t st) {
    if (which < 0 || which > 1) throw std::invalid_argument("buffer index must be 0 or 1");
    if (!plan->buf[0]) throw std::invalid_argument("plan has no bound buffers");
    const bool fold = plan->fold_n != 0;  // 1D: one contiguous row of fold_n cells
    const size_t w = (fold ? static_cast<size_t>(plan->fold_n) : static_cast<size_t>(plan->gx)) * 4;
    const size_t rows = fold ? 1 : static_cast<size_t>(plan->gy) * static_cast<size_t>(plan->gz);
    const size_t pitch = fold ? w : plan->storage.row_pitch * 4;
    float* base = plan->buf[which] + plan->storage.left_pad;
    if (to_storage) {
        ck(cudaMemcpy2DAsync(base, pitch, src, w, w, rows,
                             other_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st),
           "cudaMemcpy2DAsync(upload)");
    } else {
        ck(cudaMemcpy2DAsync(dst, w, base, pitch, w, rows,
                             other_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st),
           "cudaMemcpy2DAsync(download)");
    }
}

sst_status sst_upload(sst_plan* plan, int which, const float* src, int src_on_device, void* stream) {
    try {
        if (!plan || !src) throw std::invalid_argument("null argument");
        ck(cudaSetDevice(plan->device), "cudaSetDevice");
        const auto st = static_cast<cudaStream_t>(stream);
        copy_dense(plan, which, src, nullptr, true, src_on_device != 0, st);
        // the partner buffer carries the same boundary ring (ping-pong semantics)
        ck(cudaMemcpyAsync(plan->buf[which ^ 1], plan->buf[which], plan->storage.bytes,
                           cudaMemcpyDeviceToDevice, st),
           "cudaMemcpyAsync(ring)");
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_download(sst_plan* plan, int which, float* dst, int dst_on_device, void* stream) {
    try {
        if (!plan || !dst) throw std::invalid_argument("null argument");
        ck(cudaSetDevice(plan->device), "cudaSetDevice");
        const auto st = static_cast<cudaStream_t>(stream);
        copy_dense(plan, which, nullptr, dst, false, dst_on_device != 0, st);
        if (!dst_on_device) ck(cudaStreamSynchronize(st), "cudaStreamSynchronize(download)");
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_download_slices(sst_plan* plan, int which, uint64_t first, uint64_t count, float* dst,
                               int dst_on_device, void* stream) {
    try {
        if (!plan || !dst) throw std::invalid_argument("null argument");
        if (which < 0 || which > 1) throw std::invalid_argument("buffer index must be 0 or 1");
        if (!plan->buf[0]) throw std::invalid_argument("plan has no bound buffers");
        if (plan->fold_n) throw std::invalid_argument("slices of a 1D fold");
        const uint64_t slices = static_cast<uint64_t>(plan->dims == 3 ? plan->gz : plan->gy);
        if (first + count > slices) throw std::out_of_range("slice range beyond the grid");
        ck(cudaSetDevice(plan->device), "cudaSetDevice");
        const auto st = static_cast<cudaStream_t>(stream);
        const size_t w = static_cast<size_t>(plan->gx) * 4;
        const size_t rows_per_slice = plan->dims == 3 ? static_cast<size_t>(plan->gy) : 1;
        const size_t pitch = plan->storage.row_pitch * 4;
        const float* base = plan->buf[which] + plan->storage.left_pad +
                            static_cast<int64_t>(first) * static_cast<int64_t>(rows_per_slice) *
                                static_cast<int64_t>(plan->storage.row_pitch);
        ck(cudaMemcpy2DAsync(dst, w, base, pitch, w, static_cast<size_t>(count) * rows_per_slice,
                             dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st),
           "cudaMemcpy2DAsync(download slices)");
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_plan_set_trace(sst_plan* plan, void* dev_buf) {
    try {
        if (!plan) throw std::invalid_argument("null plan");
        plan->trace = static_cast<unsigned long long*>(dev_buf);
        if (plan->typed) plan->typed->trace = plan->trace;
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_plan_set_peer(sst_plan* plan, int which, void* buf0, void* buf1, uint64_t peer_slices) {
    try {
        if (!plan) throw std::invalid_argument("null plan");
        if (which != 0 && which != 1) throw std::invalid_argument("peer must be 0 (upper) or 1 (lower)");
        if (plan->fold_n) throw std::invalid_argument("peers are not supported for a 1D fold");
        if ((buf0 == nullptr) != (buf1 == nullptr)) throw std::invalid_argument("peer needs both buffers");
        if (buf0 && peer_slices < static_cast<uint64_t>(2 * plan->r))
            throw std::invalid_argument("peer slab smaller than its halos");
        // peers are plan-owned allocations (sst_plan_buffers): skip their guard rows
        plan->peer_buf[which][0] = buf0 ? static_cast<float*>(buf0) + plan->guard_elems() : nullptr;
        plan->peer_buf[which][1] = buf1 ? static_cast<float*>(buf1) + plan->guard_elems() : nullptr;
        plan->peer_slices[which] = buf0 ? peer_slices : 0;
        if (plan->tmap_ok) plan->make_tmaps();
        plan->run_maps_ok = false;
        if (!buf0) plan->peer_hbuf[which][0] = plan->peer_hbuf[which][1] = nullptr;
        if (plan->typed) {  // the companion plan runs the binary16 launches of the same slab
            sst_plan* T = plan->typed.get();
            T->peer_buf[which][0] = plan->peer_buf[which][0];
            T->peer_buf[which][1] = plan->peer_buf[which][1];
            T->peer_slices[which] = plan->peer_slices[which];
            if (T->tmap_ok) T->make_tmaps();
            T->run_maps_ok = false;
            if (!buf0) T->peer_hbuf[which][0] = T->peer_hbuf[which][1] = nullptr;
        }
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_plan_buffers(const sst_plan* plan, void** buf0, void** buf1) {
    try {
        if (!plan || !buf0 || !buf1) throw std::invalid_argument("null argument");
        if (!plan->owns_buf) throw std::invalid_argument("plan buffers are caller-owned");
        *buf0 = plan->alloc_base[0];
        *buf1 = plan->alloc_base[1];
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_plan_buffers_h(sst_plan* plan, void** h0, void** h1) {
    try {
        if (!plan || !h0 || !h1) throw std::invalid_argument("null argument");
        sst_plan* hp = plan->typed ? plan->typed.get() : plan;
        if (!hp->h16_ok) throw std::invalid_argument("plan has no binary16 storage");
        ck(cudaSetDevice(hp->device), "cudaSetDevice");
        hp->ensure_h16();
        *h0 = hp->hbuf_base[0];  // allocation starts (2D: guard rows first), like sst_plan_buffers
        *h1 = hp->hbuf_base[1];
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_plan_set_peer_h(sst_plan* plan, int which, void* h0, void* h1) {
    try {
        if (!plan) throw std::invalid_argument("null plan");
        if (which != 0 && which != 1) throw std::invalid_argument("peer must be 0 (upper) or 1 (lower)");
        if ((h0 == nullptr) != (h1 == nullptr)) throw std::invalid_argument("peer needs both buffers");
        if (h0 && !plan->peer_buf[which][0]) throw std::invalid_argument("set the fp32 peer (sst_plan_set_peer) first");
        sst_plan* hp = plan->typed ? plan->typed.get() : plan;
        // peers are sst_plan_buffers_h allocations: skip their guard rows
        hp->peer_hbuf[which][0] = h0 ? static_cast<__half*>(h0) + hp->guard_elems_h() : nullptr;
        hp->peer_hbuf[which][1] = h1 ? static_cast<__half*>(h1) + hp->guard_elems_h() : nullptr;
        hp->run_maps_ok = false;
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_device_alloc(int device, size_t bytes, void** ptr) {
    try {
        if (!ptr) throw std::invalid_argument("null argument");
        ck(cudaSetDevice(device), "cudaSetDevice");
        ck(cudaMalloc(ptr, bytes), "cudaMalloc");
        ck(cudaMemset(*ptr, 0, bytes), "cudaMemset");
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_device_free(void* ptr) {
    try {
        ck(cudaFree(ptr), "cudaFree");
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_ipc_handle(void* dev_ptr, uint8_t handle[64]) {
    try {
        if (!dev_ptr || !handle) throw std::invalid_argument("null argument");
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
        cudaIpcMemHandle_t h;
        ck(cudaIpcGetMemHandle(&h, dev_ptr), "cudaIpcGetMemHandle");
        std::memcpy(handle, &h, 64);
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_ipc_open(int device, const uint8_t handle[64], void** dev_ptr) {
    try {
        if (!dev_ptr || !handle) throw std::invalid_argument("null argument");
        ck(cudaSetDevice(device), "cudaSetDevice");
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, 64);
        ck(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_ipc_close(void* dev_ptr) {
    try {
        ck(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle");
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

namespace {
using StreamValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
StreamValueFn stream_fn(const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    ck(cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q), "cudaGetDriverEntryPoint");
    if (!p || q != cudaDriverEntryPointSuccess) throw CudaError(std::string(name) + " unavailable", false);
    return reinterpret_cast<StreamValueFn>(p);
}
}  // namespace

extern "C++" {
void sstl::stream_write(cudaStream_t st, uint32_t* dev_addr, uint32_t value) {
    static StreamValueFn fn = stream_fn("cuStreamWriteValue32");
    const CUresult rc = fn(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(dev_addr), value,
                           CU_STREAM_WRITE_VALUE_DEFAULT);
    if (rc != CUDA_SUCCESS) throw CudaError("cuStreamWriteValue32 failed (" + std::to_string(rc) + ")", false);
}

void sstl::stream_wait_geq(cudaStream_t st, uint32_t* dev_addr, uint32_t value) {
    static StreamValueFn fn = stream_fn("cuStreamWaitValue32");
    const CUresult rc = fn(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(dev_addr), value,
                           CU_STREAM_WAIT_VALUE_GEQ);
    if (rc != CUDA_SUCCESS) throw CudaError("cuStreamWaitValue32 failed (" + std::to_string(rc) + ")", false);
}
}  // extern "C++"

sst_status sst_stream_write_u32(void* stream, uint32_t* dev_addr, uint32_t value) {
    try {
        sstl::stream_write(static_cast<cudaStream_t>(stream), dev_addr, value);
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_stream_wait_geq_u32(void* stream, uint32_t* dev_addr, uint32_t value) {
    try {
        sstl::stream_wait_geq(static_cast<cudaStream_t>(stream), dev_addr, value);
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_set_row_window(sst_plan* plan, uint64_t y0, uint64_t y1) {
    try {
        if (!plan) throw std::invalid_argument("null plan");
        plan->y_lo = static_cast<int64_t>(y0);
        plan->y_hi = static_cast<int64_t>(y1);
        plan->y_hi1 = plan->y_lo2 = 0;
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_set_row_windows(sst_plan* plan, uint64_t y0, uint64_t y1, uint64_t y2, uint64_t y3) {
    try {
        if (!plan) throw std::invalid_argument("null plan");
        if (plan->dims != 2 || plan->fold_n) throw std::invalid_argument("two row windows need a 2D plan");
        if (!(y0 < y1 && y1 <= y2 && y2 < y3)) throw std::invalid_argument("row windows must be y0 < y1 <= y2 < y3");
        plan->y_lo = static_cast<int64_t>(y0);
        plan->y_hi = static_cast<int64_t>(y3);
        plan->y_hi1 = static_cast<int64_t>(y1);
        plan->y_lo2 = static_cast<int64_t>(y2);
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_run_steps(sst_plan* plan, int src, uint64_t steps, void* stream, int* dst_out) {
    try {
        if (!plan) throw std::invalid_argument("null plan");
        if (src < 0 || src > 1) throw std::invalid_argument("buffer index must be 0 or 1");
        if (!plan->tmap_ok) throw std::invalid_argument("plan has no bound buffers");
        ck(cudaSetDevice(plan->device), "cudaSetDevice");
        const auto st = static_cast<cudaStream_t>(stream);
        if (steps % plan->fuse != 0)
            throw std::invalid_argument("steps must be a multiple of the fusion factor");
        const int cur = plan->launch(src, steps / plan->fuse, st);
        if (dst_out) *dst_out = cur;
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

}  // extern "C"

// binary16 runs of slab plans for the in-process multi-slab driver (multi.cu)
namespace sstc {
sst_plan* plan_h16_runner(sst_plan* p, uint64_t launches) { return p->h16_runner(launches); }
void plan_h16_begin(sst_plan* hp, int src, void* st) { hp->h16_begin(src, static_cast<cudaStream_t>(st)); }
void plan_h16_step(sst_plan* hp, int src, uint64_t t, uint64_t launches, void* st) {
    hp->h16_step(src, t, launches, static_cast<cudaStream_t>(st));
}
uint64_t plan_launches(const sst_plan* p, bool h16) { return h16 ? p->h16_launches : p->launches; }
void plan_add_launches(sst_plan* p, uint64_t launches, uint64_t h16) {
    p->launches += launches;
    p->h16_launches += h16;
}
}  // namespace sstc

extern "C" {

sst_status sst_run_steps_batch(sst_plan* const* plans, int n, const int* src, uint64_t steps, void* stream,
                               int* dst_out) {
    try {
        if (!plans || n < 1 || !src) throw std::invalid_argument("null argument");
        for (int i = 0; i < n; ++i) {
            if (!plans[i]) throw std::invalid_argument("null plan");
            if (src[i] < 0 || src[i] > 1) throw std::invalid_argument("buffer index must be 0 or 1");
            if (!plans[i]->tmap_ok) throw std::invalid_argument("plan has no bound buffers");
            if (plans[i]->device != plans[0]->device) throw std::invalid_argument("plans on different devices");
            if (plans[i]->fuse != plans[0]->fuse) throw std::invalid_argument("plans with different fusion factors");
            if (plans[i]->peer_buf[0][0] || plans[i]->peer_buf[1][0])
                throw std::invalid_argument("slab plans with peers step through sst_run_steps_peer / sst_multi_run");
            for (int j = 0; j < i; ++j)
                if (plans[j] == plans[i]) throw std::invalid_argument("a plan appears twice in the batch");
        }
        if (steps % plans[0]->fuse != 0) throw std::invalid_argument("steps must be a multiple of the fusion factor");
        ck(cudaSetDevice(plans[0]->device), "cudaSetDevice");
        const auto st = static_cast<cudaStream_t>(stream);
        const uint64_t L = steps / plans[0]->fuse;
        std::vector<sst_plan*> hp(static_cast<std::size_t>(n));
        bool all_h16 = true;
        for (int i = 0; i < n; ++i) all_h16 &= (hp[static_cast<std::size_t>(i)] = plans[i]->h16_runner(L)) != nullptr;
        std::vector<int> cur(src, src + n);
        // identical 2D grids: ONE launch per step for the whole group (SST_GROUP=0: interleaved)
        const char* grp_e = std::getenv("SST_GROUP");
        bool group = all_h16 && n > 1 && L > 1 && !(grp_e && std::atoi(grp_e) == 0) && hp[0]->dims == 2;
        for (int i = 1; i < n && group; ++i) group = hp[0]->groupable_with(hp[static_cast<std::size_t>(i)]);
        if (group) {
            sst_plan* h0p = hp[0];
            const uint64_t l0 = h0p->launches, hh0 = h0p->h16_launches;
            h0p->h16_run_group(hp, src, L, st);
            const uint64_t dl = h0p->launches - l0, dh = h0p->h16_launches - hh0;
            h0p->launches = l0;
            h0p->h16_launches = hh0;
            for (int i = 0; i < n; ++i) {  // every grid advanced L steps: count them on its plan
                plans[i]->launches += dl;
                plans[i]->h16_launches += dh;
                cur[static_cast<std::size_t>(i)] = static_cast<int>((static_cast<uint64_t>(src[i]) + L) & 1);
            }
            if (dst_out)
                for (int i = 0; i < n; ++i) dst_out[i] = cur[static_cast<std::size_t>(i)];
            return SST_OK;
        }
        if (all_h16) {
            std::vector<uint64_t> l0(static_cast<std::size_t>(n)), h0(static_cast<std::size_t>(n));
            for (int i = 0; i < n; ++i) {
                sst_plan* h = hp[static_cast<std::size_t>(i)];
                l0[static_cast<std::size_t>(i)] = h->launches;
                h0[static_cast<std::size_t>(i)] = h->h16_launches;
                h->h16_begin(src[i], st);
            }
            for (uint64_t t = 0; t < L; ++t)
                for (int i = 0; i < n; ++i) hp[static_cast<std::size_t>(i)]->h16_step(src[i], t, L, st);
            for (int i = 0; i < n; ++i) {
                sst_plan* h = hp[static_cast<std::size_t>(i)];
                if (h != plans[i]) {  // companion plan: count on the caller's plan
                    plans[i]->launches += h->launches - l0[static_cast<std::size_t>(i)];
                    plans[i]->h16_launches += h->h16_launches - h0[static_cast<std::size_t>(i)];
                }
                cur[static_cast<std::size_t>(i)] = static_cast<int>((static_cast<uint64_t>(src[i]) + L) & 1);
            }
        } else {
            for (uint64_t t = 0; t < L; ++t)
                for (int i = 0; i < n; ++i)
                    cur[static_cast<std::size_t>(i)] = plans[i]->launch(cur[static_cast<std::size_t>(i)], 1, st);
        }
        if (dst_out)
            for (int i = 0; i < n; ++i) dst_out[i] = cur[static_cast<std::size_t>(i)];
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_run_steps_peer(sst_plan* plan, int src, uint64_t steps, void* stream, uint32_t* my_flags,
                              uint32_t* up_flag, uint32_t* down_flag, uint32_t launch0, int* dst_out) {
    try {
        if (!plan) throw std::invalid_argument("null plan");
        if (src < 0 || src > 1) throw std::invalid_argument("buffer index must be 0 or 1");
        if (!plan->tmap_ok) throw std::invalid_argument("plan has no bound buffers");
        if (steps % plan->fuse != 0) throw std::invalid_argument("steps must be a multiple of the fusion factor");
        const bool up = plan->peer_buf[0][0] != nullptr, down = plan->peer_buf[1][0] != nullptr;
        if ((up && !up_flag) || (down && !down_flag) || ((up || down) && !my_flags))
            throw std::invalid_argument("peer flags missing");
        ck(cudaSetDevice(plan->device), "cudaSetDevice");
        const auto st = static_cast<cudaStream_t>(stream);
        int cur = src;
        const uint64_t launches = steps / plan->fuse;
        if (sst_plan* hp = plan->h16_runner(launches)) {  // binary16 between steps (3D slabs)
            const uint64_t l0 = hp->launches, h0 = hp->h16_launches;
            hp->h16_begin(src, st);
            for (uint64_t i = 0; i < launches; ++i) {
                const uint32_t u = launch0 + static_cast<uint32_t>(i);
                if (up) sstl::stream_wait_geq(st, my_flags + 0, u);
                if (down) sstl::stream_wait_geq(st, my_flags + 1, u);
                hp->h16_step(src, i, launches, st);
                if (up) sstl::stream_write(st, up_flag, u + 1);
                if (down) sstl::stream_write(st, down_flag, u + 1);
            }
            if (hp != plan) {
                plan->launches += hp->launches - l0;
                plan->h16_launches += hp->h16_launches - h0;
            }
            if (dst_out) *dst_out = static_cast<int>((static_cast<uint64_t>(src) + launches) & 1);
            return SST_OK;
        }
        for (uint64_t i = 0; i < launches; ++i) {
            const uint32_t u = launch0 + static_cast<uint32_t>(i);
            // both neighbours finished launch u - 1: this launch's input halos are in
            // place and they no longer read the buffers its halo stores go to
            if (up) sstl::stream_wait_geq(st, my_flags + 0, u);
            if (down) sstl::stream_wait_geq(st, my_flags + 1, u);
            cur = plan->launch(cur, 1, st);
            if (up) sstl::stream_write(st, up_flag, u + 1);
            if (down) sstl::stream_write(st, down_flag, u + 1);
        }
        if (dst_out) *dst_out = cur;
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

sst_status sst_apply_host(sst_plan* plan, const float* h_in, float* h_out, uint64_t steps) {
    try {
        if (!plan || !h_in || !h_out) throw std::invalid_argument("null argument");
        if (!plan->buf[0]) {
            sst_status s = sst_plan_bind(plan, nullptr, nullptr);
            if (s != SST_OK) return s;
        }
        ck(cudaSetDevice(plan->device), "cudaSetDevice");
        cudaStream_t st = nullptr;
        if (steps % plan->fuse != 0)
            throw std::invalid_argument("steps must be a multiple of the fusion factor");
        copy_dense(plan, 0, h_in, nullptr, true, false, st);
        // identical boundary ring in both buffers (device-side copy)
        ck(cudaMemcpyAsync(plan->buf[1], plan->buf[0], plan->storage.bytes, cudaMemcpyDeviceToDevice, st),
           "cudaMemcpyAsync(ring)");
        const int cur = plan->launch(0, steps / plan->fuse, st);
        copy_dense(plan, cur, nullptr, h_out, false, false, st);
        ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
        return SST_OK;
    } catch (...) {
        return sstc::from_current_exception();
    }
}

}  // extern "C"
