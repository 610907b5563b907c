// book.cu -- codebook construction on the device: symbol
// histogram and Huffman code lengths, byte-identical to the reference's
// build_lengths (codebook.py:38-83).
//
// The reference pops a heap of (count, order, node): leaves get their rank in
// symbol order, merged nodes later orders, so ties go to (count, symbol) among
// leaves and leaves before merged subtrees.  Merged counts are created in
// non-decreasing order, so the same sequence of pops comes out of two queues
// (the classic two-queue Huffman construction): the leaves sorted by
// (count, symbol) and the merged nodes in creation order, taking the leaf on a
// count tie.  Depths follow from the parent pointers by pointer jumping.
#include "common.cuh"

namespace bh {

constexpr int HIST_THREADS = 512;
constexpr uint32_t HIST_SMEM_SYMS = 8192;  // shared-memory bins; larger symbols go straight to global
constexpr int LEN_THREADS = 1024;
constexpr uint32_t LEN_MAX_SYMS = 4096;    // distinct symbols the one-CTA builder takes

// counts[s] += occurrences of s (u64 global counters, zeroed by the caller)
__global__ void __launch_bounds__(HIST_THREADS) k_histogram(const uint16_t* __restrict__ sym, uint64_t n,
                                                            unsigned long long* __restrict__ counts) {
  __shared__ uint32_t h[HIST_SMEM_SYMS];
  for (uint32_t i = threadIdx.x; i < HIST_SMEM_SYMS; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const uint64_t nvec = n / 8;
  const uint4* v = reinterpret_cast<const uint4*>(sym);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  auto add = [&](uint32_t s) {
    if (s < HIST_SMEM_SYMS) atomicAdd(&h[s], 1u);
    else atomicAdd(&counts[s], 1ull);
  };
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nvec; i += stride) {
    const uint4 q = __ldg(v + i);
    add(q.x & 0xffffu); add(q.x >> 16);
    add(q.y & 0xffffu); add(q.y >> 16);
    add(q.z & 0xffffu); add(q.z >> 16);
    add(q.w & 0xffffu); add(q.w >> 16);
  }
  if (blockIdx.x == 0)
    for (uint64_t i = nvec * 8 + threadIdx.x; i < n; i += blockDim.x) add(sym[i]);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < HIST_SMEM_SYMS; i += blockDim.x)
    if (h[i]) atomicAdd(&counts[i], (unsigned long long)h[i]);
}

// One CTA: lengths[s] for s < alphabet (0 = absent) from counts; *status gets
// BH_OK, BH_LENGTHOVERFLOW (a code longer than 32 bits), BH_EMPTY (no symbol)
// or BH_BAD_ARGUMENT (more distinct symbols than LEN_MAX_SYMS).
__global__ void __launch_bounds__(LEN_THREADS) k_build_lengths(const unsigned long long* __restrict__ counts,
                                                               uint32_t alphabet, uint8_t* __restrict__ lengths,
                                                               int32_t* status) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned long long* key = reinterpret_cast<unsigned long long*>(smem);        // [P] count << 16 | symbol
  unsigned long long* mc = key + LEN_MAX_SYMS;                                  // [m-1] merged counts
  uint16_t* par = reinterpret_cast<uint16_t*>(mc + LEN_MAX_SYMS);               // [2m-1] parent
  uint16_t* par2 = par + 2 * LEN_MAX_SYMS;                                      // pointer-jumping copy
  uint8_t* dep = reinterpret_cast<uint8_t*>(par2 + 2 * LEN_MAX_SYMS);           // [2m-1] depth
  uint8_t* dep2 = dep + 2 * LEN_MAX_SYMS;
  __shared__ uint32_t s_wsum[LEN_THREADS / 32];
  __shared__ uint32_t s_m;
  __shared__ int s_big;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // 1. compact the nonzero counts (in symbol order) into key[]
  if (tid == 0) { s_m = 0; s_big = 0; }
  __syncthreads();
  for (uint32_t b0 = 0; b0 < alphabet; b0 += LEN_THREADS) {
    const uint32_t s = b0 + tid;
    const unsigned long long c = s < alphabet ? counts[s] : 0ull;
    const bool nz = c != 0;
    if (c >> 47) s_big = 1;  // the sort key holds the count in 48 bits
    const unsigned m = __ballot_sync(0xffffffffu, nz);
    if (lane == 0) s_wsum[warp] = __popc(m);
    __syncthreads();
    uint32_t before = s_m;
    for (uint32_t w = 0; w < warp; ++w) before += s_wsum[w];
    before += __popc(m & ((1u << lane) - 1u));
    if (nz && before < LEN_MAX_SYMS) key[before] = (c << 16) | s;
    __syncthreads();
    if (tid == 0)
      for (uint32_t w = 0; w < LEN_THREADS / 32; ++w) s_m += s_wsum[w];
    __syncthreads();
  }
  const uint32_t m = s_m;
  for (uint32_t s = tid; s < alphabet; s += LEN_THREADS) lengths[s] = 0;
  if (m == 0 || m > LEN_MAX_SYMS || s_big) {
    if (tid == 0) *status = m == 0 ? BH_EMPTY : BH_BAD_ARGUMENT;
    return;
  }
  __syncthreads();
  if (m == 1) {  // codebook.py:49-50: a single symbol gets a 1-bit code
    if (tid == 0) { lengths[key[0] & 0xffffu] = 1; *status = BH_OK; }
    return;
  }
  // 2. bitonic sort of key[0..P) by (count, symbol); padding sorts last
  uint32_t P = 1;
  while (P < m) P <<= 1;
  for (uint32_t i = m + tid; i < P; i += LEN_THREADS) key[i] = ~0ull;
  __syncthreads();
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = tid; i < P; i += LEN_THREADS) {
        const uint32_t l = i ^ j;
        if (l > i) {
          const unsigned long long a = key[i], b = key[l];
          const bool up = (i & k) == 0;
          if ((a > b) == up) { key[i] = b; key[l] = a; }
        }
      }
      __syncthreads();
    }
  }
  // 3. two-queue merge (one thread): leaves 0..m-1, merged m..2m-2
  if (tid == 0) {
    uint32_t i = 0, j = 0;
    unsigned long long f1 = key[0] >> 16, f2 = 0;
    for (uint32_t k = 0; k + 1 < m; ++k) {
      uint32_t node[2];
      unsigned long long c[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        if (i < m && (j >= k || f1 <= f2)) {  // a leaf wins a count tie (lower heap order)
          node[t] = i;
          c[t] = f1;
          ++i;
          f1 = i < m ? key[i] >> 16 : 0ull;
        } else {
          node[t] = m + j;
          c[t] = f2;
          ++j;
          f2 = j < k ? mc[j] : 0ull;
        }
      }
      mc[k] = c[0] + c[1];
      if (j == k) f2 = mc[k];  // the merged queue was empty: its new front
      par[node[0]] = (uint16_t)(m + k);
      par[node[1]] = (uint16_t)(m + k);
    }
    par[2 * m - 2] = (uint16_t)(2 * m - 2);  // root points to itself
  }
  __syncthreads();
  // 4. depth by pointer jumping: 6 rounds resolve depths up to 64
  const uint32_t nn = 2 * m - 1;
  for (uint32_t v = tid; v < nn; v += LEN_THREADS) dep[v] = v == nn - 1 ? 0 : 1;
  __syncthreads();
  uint16_t* pa = par;
  uint16_t* pb = par2;
  uint8_t* da = dep;
  uint8_t* db = dep2;
  for (int r = 0; r < 6; ++r) {
    for (uint32_t v = tid; v < nn; v += LEN_THREADS) {
      const uint32_t p = pa[v];
      const uint32_t d = da[v] + da[p];
      db[v] = (uint8_t)(d > 255 ? 255 : d);
      pb[v] = pa[p];
    }
    __syncthreads();
    uint16_t* tp = pa; pa = pb; pb = tp;
    uint8_t* td = da; da = db; db = td;
  }
  __shared__ int s_over;
  if (tid == 0) s_over = 0;
  __syncthreads();
  for (uint32_t v = tid; v < m; v += LEN_THREADS) {
    const uint32_t d = da[v];
    if (d > 32) s_over = 1;
    lengths[key[v] & 0xffffu] = (uint8_t)d;
  }
  __syncthreads();
  if (tid == 0) *status = s_over ? BH_LENGTHOVERFLOW : BH_OK;
}

constexpr size_t LEN_SMEM = (size_t)LEN_MAX_SYMS * 8 * 2 + (size_t)LEN_MAX_SYMS * 2 * 2 * 2 +
                            (size_t)LEN_MAX_SYMS * 2 * 2;

}  // namespace bh

using namespace bh;

extern "C" size_t bh_book_workspace_bytes(uint32_t alphabet) {
  return align16(8 * (size_t)(alphabet > HIST_SMEM_SYMS ? alphabet : HIST_SMEM_SYMS)) + 16;
}

extern "C" int bh_symbol_histogram(const uint16_t* symbols_dev, uint64_t n, uint32_t alphabet,
                                   uint64_t* counts_dev, void* cuda_stream) {
  if (!counts_dev || (n && !symbols_dev) || alphabet == 0 || alphabet > 65536u) return BH_BAD_ARGUMENT;
  if (reinterpret_cast<uintptr_t>(symbols_dev) & 15u) return BH_BAD_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  const size_t cells = alphabet > HIST_SMEM_SYMS ? alphabet : HIST_SMEM_SYMS;
  if (cudaMemsetAsync(counts_dev, 0, 8 * cells, st) != cudaSuccess) return BH_CUDA_ERROR;
  if (n) {
    const int sms = device_sm_count();
    uint64_t grid = (n / 8 + HIST_THREADS - 1) / HIST_THREADS;
    if (grid > (uint64_t)sms * 4) grid = (uint64_t)sms * 4;
    if (grid < 1) grid = 1;
    k_histogram<<<(unsigned)grid, HIST_THREADS, 0, st>>>(symbols_dev, n,
                                                         reinterpret_cast<unsigned long long*>(counts_dev));
  }
  return cudaGetLastError() == cudaSuccess ? BH_OK : BH_CUDA_ERROR;
}

extern "C" int bh_build_lengths(const uint64_t* counts_dev, uint32_t alphabet, uint8_t* lengths_dev,
                                int32_t* status_dev, void* cuda_stream) {
  if (!counts_dev || !lengths_dev || !status_dev || alphabet == 0 || alphabet > 65536u) return BH_BAD_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  // per-device opt-in: set it on every call (cheap, and right on any device)
  if (cudaFuncSetAttribute(k_build_lengths, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LEN_SMEM) !=
      cudaSuccess)
    return BH_CUDA_ERROR;
  k_build_lengths<<<1, LEN_THREADS, LEN_SMEM, st>>>(reinterpret_cast<const unsigned long long*>(counts_dev),
                                                    alphabet, lengths_dev, status_dev);
  return cudaGetLastError() == cudaSuccess ? BH_OK : BH_CUDA_ERROR;
}
