// kr_div_skx.cu -- the divergence-horizon kernels with exact cosines in
// OpenBLAS' SkylakeX ddot order (kr_div.cuh); a translation unit of its own so
// the two orders compile in parallel.
#include "kr_div.cuh"

namespace kr {

int div_run_skx(const DivArgs& a) { return div_run<kDotSkylakeX>(a); }

}  // namespace kr
