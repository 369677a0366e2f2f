// fk_scratch.cuh -- stream-ordered scratch for the multi-kernel host
// pipelines (GQF apply, bulk TCF): cudaMallocAsync from the device's default
// memory pool, released with cudaFreeAsync on the same stream when the
// pipeline function returns, so nothing outlives the call and repeated calls
// reuse pooled memory without a device synchronisation.
#pragma once
#include <cuda_runtime.h>

#include <vector>

namespace fk {

// Stream-ordered scratch that frees itself (cudaMallocAsync pool).
struct Scratch {
  cudaStream_t st;
  std::vector<void *> ptrs;
  cudaError_t err = cudaSuccess;
  explicit Scratch(cudaStream_t s) : st(s) {}
  ~Scratch() {
    for (void *p : ptrs) cudaFreeAsync(p, st);
  }
  template <typename T>
  T *get(size_t count) {
    void *p = nullptr;
    size_t bytes = count * sizeof(T);
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMallocAsync(&p, bytes, st);
    if (e != cudaSuccess) {
      err = e;
      return nullptr;
    }
    ptrs.push_back(p);
    return reinterpret_cast<T *>(p);
  }
};

}  // namespace fk
