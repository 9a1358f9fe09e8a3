#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* o) { extern __shared__ int d[]; __shared__ int s[868]; s[threadIdx.x] = threadIdx.x; d[threadIdx.x] = s[threadIdx.x ^ 1]; o[threadIdx.x] = d[threadIdx.x ^ 2]; }
int main() {
  cudaFuncAttributes a; cudaFuncGetAttributes(&a, k);
  printf("static %zu maxDynamic(default) %d\n", a.sharedSizeBytes, a.maxDynamicSharedSizeBytes);
  for (int x = 232448; x >= 200000; x -= 512) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, x);
    if (e == cudaSuccess) { printf("max dynamic accepted %d (+static %zu = %zu)\n", x, a.sharedSizeBytes, x + a.sharedSizeBytes); break; }
    cudaGetLastError();
  }
  return 0;
}
