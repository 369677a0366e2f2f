// tcf_point_s1.cu -- point-TCF kernels for 8-bit slot words (explicit instantiation).
#include "tcf_point_impl.cuh"

namespace fk {
template int tcf_run<uint8_t>(int, int, int, const TcfDev &, const TcfCall &, cudaStream_t);
}  // namespace fk
