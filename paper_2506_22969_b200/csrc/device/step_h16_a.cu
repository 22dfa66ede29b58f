// step_h16_a.cu — binary16-storage instantiations of the two-CTA TYB = 4 variant
// (variant 0, the first 2D choice), deepest pipelines first (typed2d.cuh).
#include "typed2d.cuh"

namespace sstl {

std::vector<TypedFns> typed_fns_tyb4() {
    // <TYB, NP32, NP16, AT, NS, CPS, NBB, NACC>
    return {Typed2D<4, 2, 4, true, 1, 2, 4, 4>::fns(), Typed2D<4, 2, 3, true, 1, 2, 4, 4>::fns(),
            Typed2D<4, 2, 6, true, 1, 2, 2, 4>::fns(), Typed2D<4, 2, 4, true, 1, 2, 3, 4>::fns(),
            Typed2D<4, 2, 4, true, 1, 2, 2, 4>::fns(), Typed2D<4, 2, 4, true, 1, 2, 2, 2>::fns(),
            // wide (fused) operators: shallow rings so two CTAs still fit an SM
            Typed2D<4, 2, 3, true, 1, 2, 2, 2>::fns(), Typed2D<4, 2, 2, true, 1, 2, 2, 2>::fns()};
}

}  // namespace sstl
