// Microbenchmark for the B200 numbers MEASURED_PEAKS.json lacks:
// FP64 / FP32 FMA issue rates, L2 size, and whether a cooperative launch can be
// captured into a CUDA graph (the align kernel uses a grid barrier).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe tools/probe_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("ERR %s at %s:%d: %s\n", #x, __FILE__, __LINE__, cudaGetErrorString(e)); } } while (0)

template <typename T>
__global__ void fma_loop(T* out, int iters, T a, T b) {
  T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
      x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void coop_kernel(unsigned* bar, int* out) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    while (atomicAdd(bar, 0u) < gridDim.x) {}
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = 1;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int l2 = 0; CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
  int clk = 0; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  printf("{\"name\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"smem_optin\":%zu,\"clock_khz\":%d,\"regs_per_sm\":%d}\n",
         p.name, p.multiProcessorCount, l2, p.sharedMemPerBlockOptin, clk, p.regsPerMultiprocessor);
  const int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
  void* buf; CK(cudaMalloc(&buf, blocks * threads * 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    fma_loop<double><<<blocks, threads>>>((double*)buf, iters, 0.999, 1e-3);
    cudaEventRecord(e0);
    fma_loop<double><<<blocks, threads>>>((double*)buf, iters, 0.999, 1e-3);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 64 * (double)iters * blocks * threads;
    printf("{\"fp64_fma_tflops\":%.2f}\n", flops / ms / 1e9);
    fma_loop<float><<<blocks, threads>>>((float*)buf, iters, 0.999f, 1e-3f);
    cudaEventRecord(e0);
    fma_loop<float><<<blocks, threads>>>((float*)buf, iters, 0.999f, 1e-3f);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"fp32_fma_tflops\":%.2f}\n", flops / ms / 1e9);
  }
  // cooperative launch under stream capture
  unsigned* bar; int* out; CK(cudaMalloc(&bar, 4)); CK(cudaMalloc(&out, 4096 * 4));
  cudaStream_t s; cudaStreamCreate(&s);
  cudaGraph_t g; cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  CK(cudaMemsetAsync(bar, 0, 4, s));
  cudaLaunchConfig_t cfg = {}; cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1;
  cfg.gridDim = dim3(p.multiProcessorCount * 4); cfg.blockDim = dim3(256); cfg.stream = s;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaError_t le = cudaLaunchKernelEx(&cfg, coop_kernel, bar, out);
  printf("{\"coop_launch_in_capture\":\"%s\"}\n", cudaGetErrorString(le));
  cudaError_t ce = cudaStreamEndCapture(s, &g);
  printf("{\"end_capture\":\"%s\"}\n", cudaGetErrorString(ce));
  if (ce == cudaSuccess) {
    CK(cudaGraphInstantiate(&ge, g, 0));
    for (int i = 0; i < 3; ++i) CK(cudaGraphLaunch(ge, s));
    CK(cudaStreamSynchronize(s));
    cudaEventRecord(e0, s);
    for (int i = 0; i < 100; ++i) CK(cudaGraphLaunch(ge, s));
    cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"graph_memset_coop_us\":%.2f}\n", ms * 10.0);
  }
  // plain launch latency
  cudaEventRecord(e0, s);
  for (int i = 0; i < 1000; ++i) coop_kernel<<<1, 32, 0, s>>>(bar, out);
  cudaEventRecord(e1, s); cudaEventSynchronize(e1);
  { float ms; cudaEventElapsedTime(&ms, e0, e1); printf("{\"stream_launch_us\":%.2f}\n", ms); }
  CK(cudaGetLastError());
  return 0;
}
