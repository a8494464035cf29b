// interact_d3.cu — instantiates the interaction kernel for D = 3.
#include "interact_sym.cuh"

namespace h2b {
template <>
void interact_all_d<3>(int kind, const DevH2& h, int64_t R, int64_t r0, int nr, const KParams& kp,
                        cudaStream_t s) {
  interact_all_d_impl<3>(kind, h, R, r0, nr, kp, s);
}
template <>
void interact_sym_d<3>(int kind, const DevH2& h, int64_t R, int64_t r0, const KParams& kp, cudaStream_t s) {
  interact_sym_d_impl<3>(kind, h, R, r0, kp, s);
}
template <>
void pack_coords_dim<3>(const DevH2& h, int nr, cudaStream_t s) {
  if (nr == 16) pack_coords_d<3, 16>(h, s);
  else pack_coords_d<3, 1>(h, s);
}
}  // namespace h2b
