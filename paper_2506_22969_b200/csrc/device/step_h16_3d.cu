// step_h16_3d.cu — binary16 inter-step storage instantiations of the 3D z-streaming
// kernel (stencil3d_kernel.cuh, HIN / HOUT), same contract as the 2D ones
// (typed2d.cuh): a SST_PREC_F16 run of T >= 2 steps reads the f32 input once, keeps
// steps 1 .. T-1 in binary16 (every consumer is the next step's gather, which rounds
// to binary16 RNE anyway: bitwise the fp32-storage result) and writes the last step
// as f32 — 4 B per update instead of 8.
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

#include "launch_util.cuh"
#include "stencil3d_kernel.cuh"

namespace sstl {

namespace {

// NP32 / NP16: patch ring depth of the kernels reading fp32 / binary16 patches
template <int TYB, int NP32, int NP16, int KZ, bool AT, int NB, int NACC, int NS>
struct Typed3D {
    // PR: the slab P2P halo stores (launched when peers are registered)
    template <bool HI, bool HO, bool PR = false>
    static KernelFn k() {
        return sst::stencil3d_stream_kernel<TYB, HI ? NP16 : NP32, KZ, NB, NACC, NS, AT, PR, HI, HO>;
    }
    static int smem(bool hin, int nks, int k_pad, int pw, int ph, int) {
        const sst::SmemLayout L =
            hin ? sst::smem_layout_stream<TYB, NP16, KZ, NB, NACC, NS, AT>(nks, k_pad, pw, ph, 2)
                : sst::smem_layout_stream<TYB, NP32, KZ, NB, NACC, NS, AT>(nks, k_pad, pw, ph, 4);
        return static_cast<int>(L.total) + 1024;  // slack for the 1 KiB base alignment
    }
    static void configure(int smem32, int smem16) {
        raise_smem_attr(k<false, true>(), smem32);
        raise_smem_attr(k<true, true>(), smem16);
        raise_smem_attr(k<true, false>(), smem16);
        raise_smem_attr(k<false, true, true>(), smem32);
        raise_smem_attr(k<true, true, true>(), smem16);
        raise_smem_attr(k<true, false, true>(), smem16);
    }
    static void launch(bool, bool hin, bool hout, int grid, int smem, cudaStream_t st, const sst::MapSet& maps,
                       const sst::StepParams& p) {
        if (!hin && !hout) throw std::logic_error("typed launch without binary16 storage");
        const KernelFn f = p.peer_mask ? (hin ? (hout ? k<true, true, true>() : k<true, false, true>())
                                              : k<false, true, true>())
                                       : (hin ? (hout ? k<true, true>() : k<true, false>()) : k<false, true>());
        launch_pdl(f, grid, smem, st, maps, p, false);
    }
    static TypedFns fns() {
        TypedFns t;
        t.smem = &smem;
        t.np_h16 = NP16;
        t.nbb = NB;
        t.nacc = NACC;
        t.configure = &configure;
        t.launch = &launch;
        return t;
    }
};

}  // namespace

std::vector<TypedFns> typed_fns_3d(int tyb, int np, int kz, bool a_tmem, int nb, int nacc, int ns) {
    // candidates deepest first (binary16 patches are half the bytes: twice the ring
    // depth for the same smem); SST_H16_CFG=<np16>,<nbb>,<nacc> keeps only that one
    std::vector<TypedFns> v;
    if (kz == 3 && a_tmem && nb == 2 && nacc == 4 && ns == 1) {
        if (tyb == 4 && np == 4)
            v = {Typed3D<4, 4, 8, 3, true, 2, 4, 1>::fns(), Typed3D<4, 4, 6, 3, true, 2, 4, 1>::fns(),
                 Typed3D<4, 4, 4, 3, true, 2, 4, 1>::fns()};
        else if (tyb == 8 && np == 3)
            v = {Typed3D<8, 3, 6, 3, true, 2, 4, 1>::fns(), Typed3D<8, 3, 4, 3, true, 2, 4, 1>::fns()};
    }
    if (const char* e = std::getenv("SST_H16_CFG")) {
        int a = 0, b = 0, c = 0;
        std::sscanf(e, "%d,%d,%d", &a, &b, &c);
        std::vector<TypedFns> only;
        for (const auto& t : v)
            if (t.np_h16 == a && t.nbb == b && t.nacc == c) only.push_back(t);
        v = only;
    }
    return v;
}

}  // namespace sstl
