// interact_d3.cu — instantiates the interaction kernel for D = 3.
#include "interact.cuh"

namespace h2b {
template <>
void interact_all_d<3>(int kind, const DevH2& h, int64_t R, int64_t r0, int nr, const KParams& kp,
                        cudaStream_t s) {
  interact_all_d_impl<3>(kind, h, R, r0, nr, kp, s);
}
}  // namespace h2b
