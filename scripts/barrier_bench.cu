// Grid-barrier microbenchmark (sm_100a): cost of one grid-wide barrier for
// a cooperative grid of `per_sm` x 148 CTAs of 256 threads, for
//   0: cooperative_groups grid.sync()
//   1: flat arrive counter + generation flag (one atomic per CTA)
//   2: two-level arrive (groups of 16 CTAs, then one atomic per group)
// The ordered point-TCF kernels pay one grid barrier per round (~1000 rounds
// per 2^28-slot batch), so this bounds what a faster barrier can save.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/barrier_bench scripts/barrier_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
namespace cg = cooperative_groups;

struct Bar {
  unsigned count[64 * 32];  // [group * 32]: padded counters
  unsigned top;
  unsigned pad[31];
  unsigned gen;
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned *p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned *p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

template <int MODE>
__global__ void __launch_bounds__(256) k_bar(Bar *b, int iters, unsigned *sink) {
  cg::grid_group grid = cg::this_grid();
  unsigned acc = 0;
  const unsigned nb = gridDim.x;
  constexpr unsigned GS = 16;
  const unsigned ngroups = (nb + GS - 1) / GS;
  for (int it = 0; it < iters; it++) {
    acc += threadIdx.x ^ it;
    if constexpr (MODE == 0) {
      grid.sync();
    } else {
      __syncthreads();
      if (threadIdx.x == 0) {
        unsigned gen = ld_acquire(&b->gen);
        bool last;
        if constexpr (MODE == 1) {
          last = atom_add_acqrel(&b->count[0], 1u) == nb - 1;
          if (last) b->count[0] = 0;
        } else {
          unsigned g = blockIdx.x / GS;
          unsigned gsize = (g == ngroups - 1) ? nb - g * GS : GS;
          last = false;
          if (atom_add_acqrel(&b->count[g * 32], 1u) == gsize - 1) {
            b->count[g * 32] = 0;
            last = atom_add_acqrel(&b->top, 1u) == ngroups - 1;
            if (last) b->top = 0;
          }
        }
        if (last) st_release(&b->gen, gen + 1);
        else
          while (ld_acquire(&b->gen) == gen) {
          }
      }
      __syncthreads();
    }
  }
  if (acc == 0xFFFFFFFFu) *sink = acc;
}

template <int MODE>
static float run(int per_sm, int iters, Bar *b, unsigned *sink) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int grid = per_sm * sms;
  void *args[] = {(void *)&b, (void *)&iters, (void *)&sink};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchCooperativeKernel((const void *)k_bar<MODE>, grid, 256, args, 0, 0);  // warm-up
  cudaEventRecord(e0);
  cudaLaunchCooperativeKernel((const void *)k_bar<MODE>, grid, 256, args, 0, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  return ms * 1e3f / iters;
}

int main() {
  Bar *b;
  unsigned *sink;
  cudaMalloc(&b, sizeof(Bar));
  cudaMemset(b, 0, sizeof(Bar));
  cudaMalloc(&sink, 4);
  const int iters = 20000;
  for (int per_sm = 1; per_sm <= 4; per_sm++) {
    float t0 = run<0>(per_sm, iters, b, sink);
    float t1 = run<1>(per_sm, iters, b, sink);
    float t2 = run<2>(per_sm, iters, b, sink);
    printf("{\"ctas_per_sm\": %d, \"us_per_barrier\": {\"cg_grid_sync\": %.3f, \"flat\": %.3f, \"two_level\": %.3f}}\n",
           per_sm, t0, t1, t2);
  }
  return 0;
}
