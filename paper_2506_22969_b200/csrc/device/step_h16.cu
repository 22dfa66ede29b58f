// step_h16.cu — which binary16-storage instantiations (typed2d.cuh) belong to
// which 2D variant of runtime.cu.
#include <cstdio>
#include <cstdlib>

#include "typed2d.cuh"

namespace sstl {

std::vector<TypedFns> typed_fns_2d(int tyb, int np, bool a_tmem, int ns, int cps) {
    // candidates deepest first: the plan takes the first that fits the variant's
    // co-residency (smem, TMEM). SST_H16_CFG=<np16>,<nbb>,<nacc> keeps only that
    // configuration (experiments).
    std::vector<TypedFns> v;
    if (a_tmem && tyb == 4 && np == 2 && ns == 1 && cps == 2) v = typed_fns_tyb4();
    else if (a_tmem && tyb == 8 && np == 3 && ns == 2 && cps == 1) v = typed_fns_tyb8();
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
