// Probe: %cluster_ctarank under cudaLaunchKernelEx with a 2-CTA cluster (sm_100a).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* out) {
  unsigned r, id, nr;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(id));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(nr));
  if (threadIdx.x == 0) { out[3 * blockIdx.x] = r; out[3 * blockIdx.x + 1] = id; out[3 * blockIdx.x + 2] = nr; }
}
int main() {
  int* d; cudaMalloc(&d, 3 * 8 * sizeof(int));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(8); cfg.blockDim = dim3(64);
  cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = 2; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
  cfg.attrs = a; cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, d);
  printf("launch: %s\n", cudaGetErrorString(e));
  int h[24]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  for (int b = 0; b < 8; ++b) printf("block %d: rank %d cluster %d nranks %d\n", b, h[3*b], h[3*b+1], h[3*b+2]);
}
