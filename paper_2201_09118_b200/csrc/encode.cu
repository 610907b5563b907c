// encode.cu -- GPU encoder with inline gap emission and the
// unit repacker.  Produces exactly what encoder.py:33-97 / kernels.py:151-179
// produce: codewords concatenated MSB-first, and the forward-skip gap array
// (g[i] = first codeword start >= boundary i, minus the boundary; boundaries
// past the last start skip to total_bits, encoder.py:81-85).  Bits are packed
// into 32-bit words; units of 8/16 bits are the same bit sequence.
#include "common.cuh"

namespace bh {

constexpr int ENC_THREADS = 1024;
constexpr int ENC_ITEMS = 4;
constexpr int ENC_TILE = ENC_THREADS * ENC_ITEMS;

struct EncWork {               // workspace layout
  unsigned long long total;    // sum of lengths
  unsigned long long bad;      // first symbol without a codeword
  unsigned long long tiles;    // dynamic tile counter
  int32_t status;
  int32_t pad;
  unsigned long long desc[1];  // look-back descriptors, one per tile
};

__global__ void k_enc_init(EncWork* w, uint64_t ntiles) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i == 0) { w->total = 0; w->bad = ~0ull; w->tiles = 0; w->status = BH_OK; }
  for (; i < ntiles; i += (uint64_t)gridDim.x * blockDim.x) w->desc[i] = 0;
}

__global__ void k_enc_size(const uint16_t* __restrict__ sym, uint64_t n, const uint8_t* __restrict__ lens,
                           uint32_t alphabet, EncWork* w) {
  unsigned long long acc = 0;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    uint32_t s = sym[i];
    uint32_t ln = s < alphabet ? lens[s] : 0;
    if (!ln) atomicMin(&w->bad, (unsigned long long)i);
    acc += ln;
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(&w->total, acc);
}

// Block-wide exclusive scan of one u32 per thread; returns the block total.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t& total, uint32_t* s_warp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t t = lane < nw ? s_warp[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    s_warp[lane] = t;  // inclusive warp prefix
  }
  __syncthreads();
  total = s_warp[nw - 1];
  uint32_t before = warp ? s_warp[warp - 1] : 0;
  __syncthreads();
  return before + x - v;
}

// Single pass: tile scan + decoupled look-back for the tile's start bit, pack
// into a shared-memory word window, store interior words, OR the two edge words.
__global__ void __launch_bounds__(ENC_THREADS) k_enc_pack(
    const uint16_t* __restrict__ sym, uint64_t n, const uint32_t* __restrict__ codes,
    const uint8_t* __restrict__ lens, uint64_t total_bits, uint32_t subseq_bits,
    uint32_t* __restrict__ words, uint8_t* __restrict__ gap, uint64_t nsub, uint64_t chunk,
    unsigned long long* __restrict__ chunk_off, EncWork* w) {
  __shared__ uint32_t s_words[ENC_TILE + 2];
  __shared__ uint32_t s_warp[32];
  __shared__ unsigned long long s_tile, s_start;
  if (threadIdx.x == 0) s_tile = atomicAdd(&w->tiles, 1ull);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t base = tile * ENC_TILE + (uint64_t)threadIdx.x * ENC_ITEMS;
  uint32_t ln[ENC_ITEMS], cw[ENC_ITEMS];
  uint32_t mine = 0;
#pragma unroll
  for (int k = 0; k < ENC_ITEMS; ++k) {
    uint64_t i = base + k;
    uint32_t s = i < n ? sym[i] : 0;
    ln[k] = i < n ? lens[s] : 0;
    cw[k] = i < n ? codes[s] : 0;
    mine += ln[k];
  }
  uint32_t tile_bits;
  uint32_t off = block_excl_scan(mine, tile_bits, s_warp);
  if (threadIdx.x < 32) {
    unsigned long long excl = 0;
    if (tile == 0) {
      if (threadIdx.x == 0) st_release(&w->desc[0], LB_FLAG_INC | tile_bits);
    } else {
      if (threadIdx.x == 0) st_release(&w->desc[tile], LB_FLAG_AGG | tile_bits);
      excl = warp_lookback(w->desc, tile);
      if (threadIdx.x == 0) st_release(&w->desc[tile], LB_FLAG_INC | (excl + tile_bits));
    }
    if (threadIdx.x == 0) s_start = excl;
  }
  for (int i = threadIdx.x; i < ENC_TILE + 2; i += blockDim.x) s_words[i] = 0;
  __syncthreads();
  const uint64_t tstart = s_start;
  const uint64_t w0 = tstart >> 5;              // first global word touched
  const uint32_t sh0 = (uint32_t)(tstart & 31);
  uint64_t p = tstart + off;                    // this thread's first codeword start
#pragma unroll
  for (int k = 0; k < ENC_ITEMS; ++k) {
    const uint64_t i = base + k;
    if (i >= n) break;
    const uint32_t len = ln[k];
    // pack into the shared word window (bit offset relative to word w0)
    const uint32_t rel = (uint32_t)(p - (w0 << 5));
    const uint32_t wi = rel >> 5, bo = rel & 31;
    const uint64_t v = ((((uint64_t)cw[k]) << (64 - len))) >> bo;  // left-justified
    atomicOr(&s_words[wi], (uint32_t)(v >> 32));
    if ((uint32_t)v) atomicOr(&s_words[wi + 1], (uint32_t)v);
    if (chunk && (i % chunk) == 0) chunk_off[i / chunk] = p;
    if (gap) {
      // boundaries j*sb in (previous start, p] skip forward to p
      // (kernels.py:167-169; boundary 0 has gap 0, encoder.py:60-61)
      uint64_t jlo = 0;
      if (i > 0) {
        const uint32_t plen = k > 0 ? ln[k - 1] : lens[sym[i - 1]];
        jlo = (p - plen) / subseq_bits + 1;
      }
      for (uint64_t j = jlo; j <= p / subseq_bits && j < nsub; ++j) {
        const uint64_t g = p - j * subseq_bits;
        if (g >= 256) w->status = BH_GAPOVERFLOW;
        gap[j] = (uint8_t)g;
      }
      if (i == n - 1) {
        // the end of the stream acts as a final virtual start (encoder.py:81-85)
        for (uint64_t j = p / subseq_bits + 1; j < nsub; ++j) {
          const uint64_t g = total_bits - j * subseq_bits;
          if (g >= 256) w->status = BH_GAPOVERFLOW;
          gap[j] = (uint8_t)g;
        }
      }
    }
    p += len;
  }
  __syncthreads();
  // store: interior words plainly, the two edge words (shared with neighbour
  // tiles) with atomicOr
  const uint32_t nwords = (sh0 + tile_bits + 31) >> 5;
  for (uint32_t i = threadIdx.x; i < nwords; i += blockDim.x) {
    uint32_t v = s_words[i];
    if (i == 0 || i == nwords - 1) {
      if (v) atomicOr(words + w0 + i, v);
    } else {
      words[w0 + i] = v;
    }
  }
}

// units (uint32 holding `unit_bits` meaningful bits, MSB-first) -> 32-bit words
__global__ void k_repack(const uint32_t* __restrict__ units, uint64_t n_units, uint32_t unit_bits,
                         uint32_t* __restrict__ words, uint64_t n_words) {
  const uint32_t per = 32 / unit_bits;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_words; i += stride) {
    uint32_t v = 0;
    for (uint32_t k = 0; k < per; ++k) {
      uint64_t u = i * per + k;
      uint32_t x = u < n_units ? units[u] : 0;
      v = (unit_bits == 32) ? x : ((v << unit_bits) | (x & ((1u << unit_bits) - 1)));
    }
    words[i] = v;
  }
}

}  // namespace bh

using namespace bh;

static uint64_t enc_tiles(uint64_t n) { return (n + ENC_TILE - 1) / ENC_TILE; }

extern "C" size_t bh_encode_workspace_bytes(uint64_t n) {
  return sizeof(EncWork) + sizeof(unsigned long long) * (enc_tiles(n) + 1);
}

extern "C" int bh_encode_size(const uint16_t* symbols_dev, uint64_t n, const uint8_t* lens_dev,
                              uint32_t alphabet, void* ws, size_t ws_bytes,
                              uint64_t* total_bits_host, uint64_t* bad_symbol_host, void* cuda_stream) {
  if (ws_bytes < bh_encode_workspace_bytes(n) || !total_bits_host) return BH_BAD_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  EncWork* w = static_cast<EncWork*>(ws);
  k_enc_init<<<64, 256, 0, st>>>(w, enc_tiles(n));
  if (n) k_enc_size<<<1184, 256, 0, st>>>(symbols_dev, n, lens_dev, alphabet, w);
  unsigned long long hv[2];
  if (cudaMemcpyAsync(hv, w, sizeof(hv), cudaMemcpyDeviceToHost, st) != cudaSuccess) return BH_CUDA_ERROR;
  if (cudaStreamSynchronize(st) != cudaSuccess) return BH_CUDA_ERROR;
  *total_bits_host = hv[0];
  if (bad_symbol_host) *bad_symbol_host = hv[1];
  return BH_OK;
}

extern "C" int bh_encode_pack(const uint16_t* symbols_dev, uint64_t n, const uint32_t* codes_dev,
                              const uint8_t* lens_dev, uint64_t total_bits, uint32_t subseq_bits,
                              uint32_t* words_dev, uint8_t* gap_dev, uint64_t chunk,
                              uint64_t* chunk_offsets_dev, void* ws, size_t ws_bytes,
                              void* cuda_stream) {
  if (ws_bytes < bh_encode_workspace_bytes(n) || !words_dev || subseq_bits == 0) return BH_BAD_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  EncWork* w = static_cast<EncWork*>(ws);
  uint64_t nwords = (total_bits + 31) / 32 + BH_WORD_PAD;
  if (cudaMemsetAsync(words_dev, 0, nwords * 4, st) != cudaSuccess) return BH_CUDA_ERROR;
  k_enc_init<<<64, 256, 0, st>>>(w, enc_tiles(n));
  uint64_t nsub = (total_bits + subseq_bits - 1) / subseq_bits;
  if (n) {
    k_enc_pack<<<(unsigned)enc_tiles(n), ENC_THREADS, 0, st>>>(
        symbols_dev, n, codes_dev, lens_dev, total_bits, subseq_bits, words_dev, gap_dev, nsub,
        chunk_offsets_dev ? chunk : 0, reinterpret_cast<unsigned long long*>(chunk_offsets_dev), w);
  }
  if (cudaGetLastError() != cudaSuccess) return BH_CUDA_ERROR;
  int32_t status = BH_OK;
  if (cudaMemcpyAsync(&status, &w->status, sizeof(status), cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return BH_CUDA_ERROR;
  if (cudaStreamSynchronize(st) != cudaSuccess) return BH_CUDA_ERROR;
  return status;
}

extern "C" int bh_repack_units(const uint32_t* units_dev, uint64_t n_units, uint32_t unit_bits,
                               uint32_t* words_dev, uint64_t n_words, void* cuda_stream) {
  if (!(unit_bits == 8 || unit_bits == 16 || unit_bits == 32)) return BH_BAD_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  if (n_words) k_repack<<<592, 256, 0, st>>>(units_dev, n_units, unit_bits, words_dev, n_words);
  return cudaGetLastError() == cudaSuccess ? BH_OK : BH_CUDA_ERROR;
}
