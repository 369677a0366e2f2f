// Random 32-byte gather microbenchmark: what does one random sector cost on B200?
// Variants of the load instruction; reports ns, effective GB/s of useful bytes.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL; x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL; return x ^ (x >> 31);
}

template <int V>
__global__ void gather(const uint32_t *__restrict__ buf, uint64_t nblk, int64_t n, uint32_t *out) {
  uint32_t acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t b = mix(i) & (nblk - 1);
    const uint32_t *p = buf + b * 8;
    uint32_t r[8];
    if (V == 0) {
      asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]) : "l"(p));
    } else if (V == 1) {
      asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]) : "l"(p));
    } else if (V == 2) {
      asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]) : "l"(p));
    } else if (V == 3) {
      asm volatile("ld.global.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]) : "l"(p));
    } else if (V == 4) {
      asm volatile("ld.global.L2::64B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]) : "l"(p));
    } else if (V == 5) {
      uint4 a = *(const uint4 *)p, c = *(const uint4 *)(p + 4);
      r[0]=a.x;r[1]=a.y;r[2]=a.z;r[3]=a.w;r[4]=c.x;r[5]=c.y;r[6]=c.z;r[7]=c.w;
    } else if (V == 6) {  // only 8 bytes of the sector
      uint2 a = *(const uint2 *)p; r[0]=a.x; r[1]=a.y; for (int j=2;j<8;j++) r[j]=0;
    } else if (V == 7) {
      asm volatile("ld.global.lu.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]) : "l"(p));
    }
    for (int j = 0; j < 8; j++) acc ^= r[j];
  }
  if (acc == 0x12345678) out[0] = acc;
}

// sequential copy reference
__global__ void copyk(const uint4 *a, uint4 *b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) b[i] = a[i];
}

template <int V>
float run(const uint32_t *buf, uint64_t nblk, int64_t n, uint32_t *out, int grid, int block) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  gather<V><<<grid, block>>>(buf, nblk, n, out);
  cudaEventRecord(a);
  for (int r = 0; r < 5; r++) gather<V><<<grid, block>>>(buf, nblk, n, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms / 5;
}

int main(int argc, char **argv) {
  size_t bytes = 1ull << 31;  // 2 GiB table
  uint64_t nblk = bytes / 32;
  int64_t n = 1ll << 28;
  uint32_t *buf, *out; cudaMalloc(&buf, bytes); cudaMalloc(&out, 64); cudaMemset(buf, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int fetch = argc > 1 ? atoi(argv[1]) : 0;
  if (fetch) { cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, fetch); size_t v; cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity); printf("set L2 fetch %d -> %s, now %zu\n", fetch, cudaGetErrorString(e), v); }
  int grid = sms * 8, block = 256;
  const char *names[] = {"v8", "cg.v8", "nc.v8", "L1::no_allocate.v8", "L2::64B.v8", "2x v4", "8B only", "lu.v8"};
  float ms[8];
  ms[0] = run<0>(buf, nblk, n, out, grid, block);
  ms[1] = run<1>(buf, nblk, n, out, grid, block);
  ms[2] = run<2>(buf, nblk, n, out, grid, block);
  ms[3] = run<3>(buf, nblk, n, out, grid, block);
  ms[4] = run<4>(buf, nblk, n, out, grid, block);
  ms[5] = run<5>(buf, nblk, n, out, grid, block);
  ms[6] = run<6>(buf, nblk, n, out, grid, block);
  ms[7] = run<7>(buf, nblk, n, out, grid, block);
  for (int v = 0; v < 8; v++)
    printf("%-20s %8.3f ms  %7.1f Gsectors/s  useful %7.1f GB/s\n", names[v], ms[v], n / ms[v] / 1e6, n * 32.0 / ms[v] / 1e6);
  for (int occ : {1, 2, 4, 16}) {
    float m = run<1>(buf, nblk, n, out, sms * occ, block);
    printf("cg.v8 grid %d x 256: %8.3f ms  %7.1f Gsectors/s\n", sms * occ, m, n / m / 1e6);
  }
  // copy bandwidth reference
  uint4 *dst; cudaMalloc(&dst, bytes / 2);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  copyk<<<sms * 8, 256>>>((const uint4 *)buf, dst, bytes / 2 / 16);
  cudaEventRecord(a); for (int r = 0; r < 5; r++) copyk<<<sms * 8, 256>>>((const uint4 *)buf, dst, bytes / 2 / 16); cudaEventRecord(b); cudaEventSynchronize(b);
  float mc; cudaEventElapsedTime(&mc, a, b); mc /= 5;
  printf("copy 1 GiB: %.3f ms -> %.1f GB/s (read+write)\n", mc, 2.0 * (bytes / 2) / mc / 1e6);
  return 0;
}
