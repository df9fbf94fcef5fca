// kr_div_hsw.cu -- the divergence-horizon kernels with exact cosines in
// OpenBLAS' Haswell ddot order (kr_div.cuh); a translation unit of its own so
// the two orders compile in parallel.
#include "kr_div.cuh"

namespace kr {

int div_run_hsw(const DivArgs& a) { return div_run<kDotHaswell>(a); }

}  // namespace kr
