// step_h16_b.cu — binary16-storage instantiations of the one-CTA TYB = 8
// variants (typed2d.cuh).
#include "typed2d.cuh"

namespace sstl {

std::vector<TypedFns> typed_fns_tyb8() {
    // <TYB, NP32, NP16, AT, NS, CPS, NBB, NACC>
    return {Typed2D<8, 3, 6, true, 2, 1, 2, 4>::fns(), Typed2D<8, 3, 4, true, 2, 1, 2, 2>::fns()};
}

}  // namespace sstl
