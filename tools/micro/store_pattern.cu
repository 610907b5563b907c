// Micro-benchmark: L2 cost of per-lane-region 16-byte stores vs coalesced ones.
// Output 50 MB.  Pattern A: warp writes 512 B contiguous per instruction.
// Pattern B: lane l owns a contiguous region of R chunks; per instruction the 32
// lanes write chunk i of their own regions (32 different lines).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void coalesced(uint4* out, size_t nchunks) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nchunks; i += stride)
    out[i] = make_uint4(i, i + 1, i + 2, i + 3);
}

template <int R>
__global__ void per_lane(uint4* out, size_t nchunks) {
  // each warp handles 32*R consecutive chunks; lane l owns chunks [l*R, l*R+R)
  size_t warps = (size_t)gridDim.x * blockDim.x / 32;
  size_t w = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) / 32;
  int lane = threadIdx.x & 31;
  for (size_t base = w * 32 * R; base < nchunks; base += warps * 32 * R) {
#pragma unroll 4
    for (int i = 0; i < R; ++i) {
      size_t c = base + (size_t)lane * R + i;
      if (c < nchunks) out[c] = make_uint4(c, c + 1, c + 2, c + 3);
    }
  }
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < 20; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 20;
}

int main() {
  size_t bytes = 50u << 20;
  size_t n = bytes / 16;
  uint4* out;
  cudaMalloc(&out, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int blocks : {sms * 4, sms * 8}) {
    float t = timeit([&] { coalesced<<<blocks, 512>>>(out, n); });
    printf("coalesced      blocks=%d: %.2f us  %.0f GB/s\n", blocks, t * 1e3, bytes / t / 1e6);
    t = timeit([&] { per_lane<10><<<blocks, 512>>>(out, n); });
    printf("per-lane R=10  blocks=%d: %.2f us  %.0f GB/s\n", blocks, t * 1e3, bytes / t / 1e6);
    t = timeit([&] { per_lane<3><<<blocks, 512>>>(out, n); });
    printf("per-lane R=3   blocks=%d: %.2f us  %.0f GB/s\n", blocks, t * 1e3, bytes / t / 1e6);
    t = timeit([&] { per_lane<20><<<blocks, 512>>>(out, n); });
    printf("per-lane R=20  blocks=%d: %.2f us  %.0f GB/s\n", blocks, t * 1e3, bytes / t / 1e6);
  }
  return 0;
}
