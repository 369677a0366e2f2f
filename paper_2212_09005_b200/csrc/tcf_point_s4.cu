// tcf_point_s4.cu -- point-TCF kernels for 32-bit slot words (explicit instantiation).
#include "tcf_point_impl.cuh"

namespace fk {
template int tcf_run<uint32_t>(int, int, int, const TcfDev &, const TcfCall &, cudaStream_t);
}  // namespace fk
