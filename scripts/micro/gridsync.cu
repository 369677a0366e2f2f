// grid.sync() cost on B200 for a co-resident cooperative grid
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__global__ void k(int iters, unsigned *x) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; i++) { if (threadIdx.x == 0) atomicAdd(x, 1); g.sync(); }
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *x; cudaMalloc(&x, 4);
  for (int per : {1, 2, 4, 8}) for (int bs : {128, 256}) {
    int grid = sms * per; int iters = 2000;
    void *args[] = {&iters, &x};
    cudaLaunchCooperativeKernel((void *)k, grid, bs, args, 0, 0); cudaDeviceSynchronize();
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); cudaLaunchCooperativeKernel((void *)k, grid, bs, args, 0, 0); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("grid %d x %d: %.2f us per grid.sync (%s)\n", grid, bs, ms * 1000 / iters, cudaGetErrorString(cudaGetLastError()));
  }
}
