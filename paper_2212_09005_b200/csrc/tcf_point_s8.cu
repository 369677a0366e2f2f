// tcf_point_s8.cu -- point-TCF kernels for 64-bit slot words (explicit instantiation).
#include "tcf_point_impl.cuh"

namespace fk {
template int tcf_run<uint64_t>(int, int, int, const TcfDev &, const TcfCall &, cudaStream_t);
}  // namespace fk
