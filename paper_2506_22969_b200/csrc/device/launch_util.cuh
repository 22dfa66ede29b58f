// launch_util.cuh — host-side launch helpers shared by the translation units that
// instantiate step kernels (runtime.cu, step_h16.cu): error checks, the smem
// attribute bookkeeping and the programmatic-dependent launch.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../host/capi_internal.hpp"
#include "stencil_common.cuh"

namespace sstl {

inline void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        const bool nodev = e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver;
        throw sstc::CudaError(std::string(what) + ": " + cudaGetErrorString(e), nodev);
    }
}

// Every step kernel is launched with programmatic stream serialization: its
// prologue (barrier init, TMEM alloc, constant staging) runs while the previous
// step drains, and griddepcontrol.wait in the kernel orders all grid-buffer
// accesses after that step completes. SST_PDL=0 disables it (A/B experiments).
inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SST_PDL");
        return !(e && std::atoi(e) == 0);
    }();
    return on;
}

using KernelFn = void (*)(sst::MapSet, sst::StepParams);

// kernel launches the library has issued, process-wide (sst_launch_count)
inline std::atomic<unsigned long long>& launch_counter() {
    static std::atomic<unsigned long long> n{0};
    return n;
}

// cudaFuncAttributeMaxDynamicSharedMemorySize belongs to a kernel instantiation on a
// device, not to a plan, and a plan's smem depends on its stencil. So the attribute
// is only ever raised: lowering it for a narrower stencil would make every later
// launch of a still-live plan with more smem on the same instantiation fail.
inline void raise_smem_attr(KernelFn kernel, int smem) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> configured;
    int dev = 0;
    ck(cudaGetDevice(&dev), "cudaGetDevice");
    std::lock_guard<std::mutex> lock(mu);
    int& cur = configured[{reinterpret_cast<const void*>(kernel), dev}];
    if (smem <= cur) return;
    ck(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), "cudaFuncSetAttribute");
    // max shared-memory carveout: the co-residency a variant is built for (CPS CTAs
    // per SM) must also hold for the occupancy check of cooperative launches
    ck(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100),
       "cudaFuncSetAttribute(carveout)");
    cur = smem;
}

// cooperative: a multi-step launch relies on all its CTAs being co-resident
// (CTAs wait on each other's step flags); the attribute makes that a launch-time
// guarantee instead of an assumption.
inline void launch_pdl(KernelFn fn, int grid, int smem, cudaStream_t st, const sst::MapSet& maps,
                       const sst::StepParams& p, bool cooperative) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(sst::kThreads);
    cfg.dynamicSmemBytes = static_cast<size_t>(smem);
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (pdl_enabled()) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (cooperative) {
        attr[na].id = cudaLaunchAttributeCooperative;
        attr[na].val.cooperative = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = static_cast<unsigned>(na);
    ck(cudaLaunchKernelEx(&cfg, fn, maps, p), "cudaLaunchKernelEx");
    launch_counter().fetch_add(1, std::memory_order_relaxed);
}

// Binary16-storage instantiations of one 2D variant (step_h16.cu): single-step
// launches, static or dynamic batches, input / output storage f32 or f16.
struct TypedFns {
    // dynamic smem of the launches reading fp32 (hin = false) or binary16 patches;
    // the binary16-input kernels keep a deeper patch ring (half-size patches)
    int (*smem)(bool hin, int nks, int k_pad, int patch_w, int patch_h, int planes) = nullptr;
    int np_h16 = 0;  // patch ring depth of the binary16-input kernels
    int nbb = 2;     // B'' operand stages
    int nacc = 2;    // accumulator stages (TMEM columns: nacc * 8 * TYB)
    void (*configure)(int smem_f32_in, int smem_h16_in) = nullptr;
    void (*launch)(bool dyn, bool hin, bool hout, int grid, int smem, cudaStream_t st, const sst::MapSet& maps,
                   const sst::StepParams& p) = nullptr;
};
// candidates in preference order (empty when the variant has no binary16 instantiations)
std::vector<TypedFns> typed_fns_2d(int tyb, int np, bool a_tmem, int ns, int cps);

// 3D z-streaming kernel with binary16 storage (step_h16.cu), same contract
std::vector<TypedFns> typed_fns_3d(int tyb, int np, int kz, bool a_tmem, int nb, int nacc, int ns);

// Boundary ring (and everything outside the interior the kernels read) of an f32
// storage buffer -> binary16 in two f16 storage buffers (runtime.cu).
// halo_lo / halo_hi: 3D slab ends whose r planes a P2P neighbour writes (ring cells only)
void launch_ring_to_half(const float* src, __half* d0, __half* d1, int gx, int gy, int gz, int r,
                         long long rp, long long pp, int lp, long long rph, long long pph, int lph,
                         cudaStream_t st, bool halo_lo = false, bool halo_hi = false);

// Stream-ordered flag write / wait >= (cuStreamWriteValue32 / cuStreamWaitValue32,
// resolved at run time through the driver entry points; runtime.cu).
void stream_write(cudaStream_t st, uint32_t* dev_addr, uint32_t value);
void stream_wait_geq(cudaStream_t st, uint32_t* dev_addr, uint32_t value);

}  // namespace sstl
