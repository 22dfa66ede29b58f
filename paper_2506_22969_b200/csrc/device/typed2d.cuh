// typed2d.cuh — binary16 inter-step storage instantiations of the 2D step kernel
// (included by the step_h16_*.cu translation units, which compile in parallel).
//
// A SST_PREC_F16 run of T >= 2 steps reads the f32 input once, keeps steps
// 1 .. T-1 in binary16 and writes the last step as f32. Every consumer of an
// intermediate grid is the next step's gather, which rounds to binary16 RNE
// anyway (the reference round16 semantics, fp16.hpp:13-59), so rounding in the
// producing epilogue instead is bitwise the same result at 4 B per update
// (2 read + 2 write) instead of 8.
#pragma once

#include <stdexcept>
#include <vector>

#include "launch_util.cuh"
#include "stencil_kernel.cuh"

namespace sstl {

// NP32 / NP16: patch ring depth of the kernels reading fp32 / binary16 patches;
// NBB / NACC: B'' and accumulator stages (binary16 halves the bytes per update, so
// more batches must be in flight per SM for the same HBM rate)
template <int TYB, int NP32, int NP16, bool AT, int NS, int CPS, int NBB, int NACC>
struct Typed2D {
    template <int MODE, bool HI, bool HO>
    static KernelFn k() {
        return sst::stencil_step_kernel<2, TYB, HI ? NP16 : NP32, AT, MODE, NS, CPS, HI, HO, NBB, NACC>;
    }
    static int smem(bool hin, int nks, int k_pad, int pw, int ph, int planes) {
        const sst::SmemLayout L =
            hin ? sst::smem_layout<TYB, NP16, AT, NS, NBB, NACC>(nks, k_pad, pw, ph, planes, 2)
                : sst::smem_layout<TYB, NP32, AT, NS, NBB, NACC>(nks, k_pad, pw, ph, planes, 4);
        return static_cast<int>(L.total) + 1024;  // slack for the 1 KiB base alignment
    }
    static void configure(int smem32, int smem16) {
        raise_smem_attr(k<sst::kModeStatic, false, true>(), smem32);
        raise_smem_attr(k<sst::kModeStatic, true, true>(), smem16);
        raise_smem_attr(k<sst::kModeStatic, true, false>(), smem16);
        raise_smem_attr(k<sst::kModeDynamic, false, true>(), smem32);
        raise_smem_attr(k<sst::kModeDynamic, true, true>(), smem16);
        raise_smem_attr(k<sst::kModeDynamic, true, false>(), smem16);
        raise_smem_attr(k<sst::kModePeer, false, true>(), smem32);
        raise_smem_attr(k<sst::kModePeer, true, true>(), smem16);
        raise_smem_attr(k<sst::kModePeer, true, false>(), smem16);
        raise_smem_attr(k<sst::kModeGroup, false, true>(), smem32);
        raise_smem_attr(k<sst::kModeGroup, true, true>(), smem16);
        raise_smem_attr(k<sst::kModeGroup, true, false>(), smem16);
    }
    static void launch(bool dyn, bool hin, bool hout, int grid, int smem, cudaStream_t st, const sst::MapSet& maps,
                       const sst::StepParams& p) {
        if (!hin && !hout) throw std::logic_error("typed launch without binary16 storage");
        KernelFn f = nullptr;
        if (p.group) {  // grouped launch over identical grids (sst_run_steps_batch)
            if (!p.sched) throw std::logic_error("grouped launches draw batches dynamically");
            f = hin ? (hout ? k<sst::kModeGroup, true, true>() : k<sst::kModeGroup, true, false>())
                    : k<sst::kModeGroup, false, true>();
        } else if (p.peer_mask) {  // slab P2P halos: the dynamic-peer instantiations (p.sched set)
            if (!p.sched) throw std::logic_error("peer launches draw batches dynamically");
            f = hin ? (hout ? k<sst::kModePeer, true, true>() : k<sst::kModePeer, true, false>())
                    : k<sst::kModePeer, false, true>();
        } else if (dyn)
            f = hin ? (hout ? k<sst::kModeDynamic, true, true>() : k<sst::kModeDynamic, true, false>())
                    : k<sst::kModeDynamic, false, true>();
        else
            f = hin ? (hout ? k<sst::kModeStatic, true, true>() : k<sst::kModeStatic, true, false>())
                    : k<sst::kModeStatic, false, true>();
        launch_pdl(f, grid, smem, st, maps, p, false);
    }
    static TypedFns fns() {
        TypedFns t;
        t.smem = &smem;
        t.np_h16 = NP16;
        t.nbb = NBB;
        t.nacc = NACC;
        t.configure = &configure;
        t.launch = &launch;
        return t;
    }
};

std::vector<TypedFns> typed_fns_tyb4();  // step_h16_a.cu: the two-CTA TYB = 4 variant
std::vector<TypedFns> typed_fns_tyb8();  // step_h16_b.cu: the one-CTA TYB = 8 variants

}  // namespace sstl
