#include <cstdio>
#include <cuda_runtime.h>
__global__ void __maxnreg__(176) kk(float* p) { p[threadIdx.x] = 1; }
int main() {
  int v; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kk, 352, 0); printf("occ352=%d\n", v);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kk, 384, 0); printf("occ384=%d\n", v);
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, kk); printf("regs %d maxthr %d\n", fa.numRegs, fa.maxThreadsPerBlock);
  cudaDeviceProp pr; cudaGetDeviceProperties(&pr, 0); printf("regsPerBlock %d regsPerSM %d\n", pr.regsPerBlock, pr.regsPerMultiprocessor);
}
