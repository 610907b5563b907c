// Fixed cost of launching a persistent kernel, measured like bench.py (events
// build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o tools/micro/launch/launch tools/micro/launch/launch.cu
// around the launch, a 256 MiB memset between steps so the host runs ahead).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_empty(int* out) {
  extern __shared__ int sm[];
  if (threadIdx.x == 0) { sm[0] = blockIdx.x; out[blockIdx.x] = sm[0]; }
}
__global__ void k_fill(uint4* p, size_t n, unsigned v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(v, v, v, v);
}
static int g_kflush = 0;
static float run(int grid, int threads, int smem, int kernels, bool graph) {
  static int* out = nullptr; static void* flush = nullptr;
  if (!out) { cudaMalloc(&out, 4096); cudaMalloc(&flush, 256 << 20); }
  cudaStream_t st; cudaStreamCreate(&st);
  cudaGraphExec_t ge = nullptr;
  if (graph) {
    cudaGraph_t g;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int k = 0; k < kernels; ++k) k_empty<<<grid, threads, smem, st>>>(out);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
  }
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float tot = 0; int n = 50;
  for (int i = 0; i < n + 3; ++i) {
    if (g_kflush) k_fill<<<148 * 4, 512, 0, st>>>((uint4*)flush, (256 << 20) / 16, i);
    else cudaMemsetAsync(flush, i, 256 << 20, st);
    cudaEventRecord(a, st);
    if (graph) cudaGraphLaunch(ge, st);
    else for (int k = 0; k < kernels; ++k) k_empty<<<grid, threads, smem, st>>>(out);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (i >= 3) tot += ms;
  }
  cudaStreamDestroy(st);
  return 1000 * tot / n;
}
int main() {
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  printf("grid 1 x 32, 16 B smem        : %.2f us\n", run(1, 32, 16, 1, false));
  printf("grid 148 x 768, 16 B          : %.2f us\n", run(148, 768, 16, 1, false));
  printf("grid 148 x 768, 208 KB        : %.2f us\n", run(148, 768, 208 * 1024, 1, false));
  printf("2 kernels 148 x 768, 208 KB   : %.2f us\n", run(148, 768, 208 * 1024, 2, false));
  printf("graph 1 kernel 148x768 208KB  : %.2f us\n", run(148, 768, 208 * 1024, 1, true));
  printf("graph 2 kernels               : %.2f us\n", run(148, 768, 208 * 1024, 2, true));
  g_kflush = 1;
  printf("kernel flush: grid 1 x 32     : %.2f us\n", run(1, 32, 16, 1, false));
  printf("kernel flush: graph 148x768   : %.2f us\n", run(148, 768, 208 * 1024, 1, true));
  printf("kernel flush: 2 kernels       : %.2f us\n", run(148, 768, 208 * 1024, 2, false));
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
