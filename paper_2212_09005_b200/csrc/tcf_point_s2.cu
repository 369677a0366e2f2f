// tcf_point_s2.cu -- point-TCF kernels for 16-bit slot words (explicit instantiation).
#include "tcf_point_impl.cuh"

namespace fk {
template int tcf_run<uint16_t>(int, int, int, const TcfDev &, const TcfCall &, cudaStream_t);
}  // namespace fk
