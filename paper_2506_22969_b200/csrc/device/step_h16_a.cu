// step_h16_a.cu — binary16-storage instantiations of the two-CTA TYB = 4 variant
// (variant 0, the first 2D choice), deepest pipelines first (typed2d.cuh).
#include "typed2d.cuh"

namespace sstl {

std::vector<TypedFns> typed_fns_tyb4() {
    // <TYB, NP32, NP16, AT, NS, CPS, NBB, NACC>
    // (4, 2, 2) first: Box-2D9P 8192^2 55.8 vs 56.7 us for (4, 4, 4), Star-2D13P equal
    return {Typed2D<4, 2, 4, true, 2, 2, 2, 2>::fns(), Typed2D<4, 2, 4, true, 1, 2, 2, 2>::fns(), Typed2D<4, 2, 4, true, 1, 2, 4, 4>::fns(), Typed2D<4, 2, 3, true, 1, 2, 4, 4>::fns(),
            Typed2D<4, 2, 6, true, 1, 2, 2, 4>::fns(), Typed2D<4, 2, 4, true, 1, 2, 3, 4>::fns(),
            Typed2D<4, 2, 4, true, 1, 2, 2, 4>::fns(), Typed2D<4, 2, 4, true, 1, 2, 2, 2>::fns(),
            // wide (fused) operators: shallow rings so two CTAs still fit an SM
            Typed2D<4, 2, 3, true, 1, 2, 2, 2>::fns(), Typed2D<4, 2, 2, true, 1, 2, 2, 2>::fns()};
}

}  // namespace sstl
