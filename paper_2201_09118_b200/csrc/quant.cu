// quant.cu -- dequantization of decoded quantization codes on the device
// (the cuSZ decompression step after the decode path).
//
// The reference reconstruction (kernels.py:216-227 dequantize_chain, called
// by quant.py:64-74) is a sequential recurrence rounded through float32:
//     pred = f64(f32(pred + twice_eb * (code - midpoint)))     (outliers reset
//     pred to their stored float64 value)
// Exact regime: when twice_eb = 2^e (-149 <= e <= 104) and every running sum
// S_i of (code - midpoint) since the last outlier (plus the outlier's value in
// units of 2^e) stays below 2^24 in magnitude, every step is exact -- the f64
// product and sum are exact and the f32 rounding keeps all 24 significant
// bits -- so pred_i = 2^e * S_i: a segmented prefix sum, computed here in one
// pass with a decoupled look-back across tiles.  The kernel raises a device
// flag when a running sum leaves that range; the caller then runs the exact
// sequential chain on the device (k_dequant_chain, one thread: slow but
// bit-identical in every regime).
#include "common.cuh"

namespace bh {

constexpr int DQ_THREADS = 256;
constexpr int DQ_ITEMS = 16;                        // codes per thread
constexpr int DQ_TILE = DQ_THREADS * DQ_ITEMS;      // 4096 codes per tile
constexpr long long DQ_LIMIT = 1ll << 24;

// descriptor: [63:62] 0 empty / 1 aggregate / 2 inclusive, [61] segment reset
// inside, [60:0] sum (two's complement)
constexpr unsigned long long DQ_AGG = 1ull << 62, DQ_INC = 2ull << 62, DQ_RST = 1ull << 61;
constexpr unsigned long long DQ_VAL = (1ull << 61) - 1;

struct DqWork {
  unsigned long long tiles;  // dynamic tile counter
  int32_t inexact;           // a running sum left +-2^24 (or a flagged outlier)
  int32_t pad;
  unsigned long long desc[1];
};

__device__ __forceinline__ long long dq_sext(unsigned long long v) {
  return (long long)(v << 3) >> 3;  // 61-bit two's complement
}

struct Seg {  // segmented-sum scan element
  long long s;
  uint32_t r;  // a reset (outlier) inside: s is the running value after it
};
__device__ __forceinline__ Seg seg_op(Seg a, Seg b) { return b.r ? b : Seg{a.s + b.s, a.r}; }

__global__ void __launch_bounds__(DQ_THREADS) k_dequant(const uint16_t* __restrict__ codes, uint64_t n,
                                                        const int64_t* __restrict__ oidx,
                                                        const long long* __restrict__ ounits, uint64_t nout,
                                                        double twice_eb, int32_t mid, double* __restrict__ out,
                                                        DqWork* w) {
  __shared__ uint32_t s_tile;
  __shared__ Seg s_warp[DQ_THREADS / 32];
  __shared__ long long s_prefix;
  __shared__ uint32_t s_rst[DQ_TILE / 32];  // outlier positions of the tile (bitmask)
  __shared__ long long s_oval[64];          // their values in units of twice_eb (first 64 per tile)
  __shared__ uint32_t s_nout, s_o0;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = (uint32_t)atomicAdd(&w->tiles, 1ull);
  for (uint32_t i = tid; i < DQ_TILE / 32; i += DQ_THREADS) s_rst[i] = 0;
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t t0 = tile * DQ_TILE;
  if (t0 >= n) return;
  // outliers of this tile: binary search for the first index >= t0
  if (tid == 0) {
    uint64_t lo = 0, hi = nout;
    while (lo < hi) {
      const uint64_t m = (lo + hi) >> 1;
      if ((uint64_t)oidx[m] < t0) lo = m + 1; else hi = m;
    }
    uint64_t e = lo;
    while (e < nout && (uint64_t)oidx[e] < t0 + DQ_TILE) ++e;
    s_o0 = (uint32_t)lo;
    s_nout = (uint32_t)(e - lo);
    if (e - lo > 64) w->inexact = 1;  // more than 64 outliers in 4096 codes: take the exact chain
  }
  __syncthreads();
  const uint32_t no = min(s_nout, 64u);
  for (uint32_t k = tid; k < no; k += DQ_THREADS) {
    const uint32_t p = (uint32_t)(oidx[s_o0 + k] - t0);
    atomicOr(&s_rst[p >> 5], 1u << (p & 31));
    s_oval[k] = ounits[s_o0 + k];
  }
  __syncthreads();
  // this thread's 16 codes: deltas, local segmented scan
  const uint64_t i0 = t0 + (uint64_t)tid * DQ_ITEMS;
  long long v[DQ_ITEMS];
  uint32_t rmask = 0;
  const uint32_t rbits = (s_rst[(tid * DQ_ITEMS) >> 5] >> ((tid * DQ_ITEMS) & 31)) & 0xffffu;
  if (i0 + DQ_ITEMS <= n) {
    const uint4* src = reinterpret_cast<const uint4*>(codes + i0);
    const uint4 a = __ldg(src), b = __ldg(src + 1);
    const uint32_t wv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int k = 0; k < DQ_ITEMS; ++k) v[k] = (long long)((wv[k >> 1] >> ((k & 1) * 16)) & 0xffffu) - mid;
  } else {
#pragma unroll
    for (int k = 0; k < DQ_ITEMS; ++k) v[k] = i0 + k < n ? (long long)codes[i0 + k] - mid : 0ll;
  }
  if (rbits) {
    uint32_t oi = 0;  // rank of this thread's first outlier among the tile's
    for (uint32_t q = 0; q < (tid * DQ_ITEMS) >> 5; ++q) oi += __popc(s_rst[q]);
    oi += __popc(s_rst[(tid * DQ_ITEMS) >> 5] & ((1u << ((tid * DQ_ITEMS) & 31)) - 1u));
#pragma unroll
    for (int k = 0; k < DQ_ITEMS; ++k)
      if ((rbits >> k) & 1u) { v[k] = s_oval[oi++]; rmask |= 1u << k; }
  }
  Seg t{0, 0};
#pragma unroll
  for (int k = 0; k < DQ_ITEMS; ++k) {
    if ((rmask >> k) & 1u) t = Seg{v[k], 1};
    else t.s += v[k];
  }
  // block-wide exclusive segmented scan of the thread totals
  Seg x = t;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Seg y{__shfl_up_sync(0xffffffffu, x.s, o), __shfl_up_sync(0xffffffffu, x.r, o)};
    if ((int)lane >= o) x = seg_op(y, x);
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    Seg z = lane < DQ_THREADS / 32 ? s_warp[lane] : Seg{0, 0};
#pragma unroll
    for (int o = 1; o < DQ_THREADS / 32; o <<= 1) {
      Seg y{__shfl_up_sync(0xffffffffu, z.s, o), __shfl_up_sync(0xffffffffu, z.r, o)};
      if ((int)lane >= o) z = seg_op(y, z);
    }
    if (lane < DQ_THREADS / 32) s_warp[lane] = z;  // inclusive per warp
    // tile aggregate -> look-back (lane 0 publishes, the warp looks back)
    const Seg agg{__shfl_sync(0xffffffffu, z.s, DQ_THREADS / 32 - 1),
                  __shfl_sync(0xffffffffu, z.r, DQ_THREADS / 32 - 1)};
    long long excl = 0;
    if (tile == 0) {
      if (lane == 0)
        st_release(&w->desc[0], DQ_INC | (agg.r ? DQ_RST : 0ull) | ((unsigned long long)agg.s & DQ_VAL));
    } else {
      // a tile with an outlier knows its inclusive value at once; its codes
      // before the outlier still need the prefix of the tiles before it
      if (lane == 0)
        st_release(&w->desc[tile], (agg.r ? DQ_INC : DQ_AGG) | (agg.r ? DQ_RST : 0ull) |
                                       ((unsigned long long)agg.s & DQ_VAL));
      {
        // walk back until an inclusive prefix or a reset (a segment start)
        int64_t base = (int64_t)tile - 1;
        while (base >= 0) {
          const int64_t idx = base - (int64_t)lane;
          unsigned long long d;
          while (true) {
            d = idx >= 0 ? ld_acquire(&w->desc[idx]) : DQ_INC;
            if (__all_sync(0xffffffffu, (d >> 62) != 0)) break;
            __nanosleep(32);
          }
          const bool stop = idx < 0 || (d >> 62) == 2 || (d & DQ_RST);
          const unsigned m = __ballot_sync(0xffffffffu, stop);
          const uint32_t sl = m ? __ffs(m) - 1 : 31;
          const long long val = (lane <= sl && idx >= 0) ? dq_sext(d & DQ_VAL) : 0ll;
          excl += warp_sum(val);
          if (m) break;
          base -= 32;
        }
        if (lane == 0 && !agg.r) st_release(&w->desc[tile], DQ_INC | ((unsigned long long)(excl + agg.s) & DQ_VAL));
      }
    }
    if (lane == 0) s_prefix = excl;
  }
  __syncthreads();
  // this thread's exclusive prefix: tile prefix, then warps and lanes before it
  Seg pre{s_prefix, 0};
  if (warp) pre = seg_op(pre, s_warp[warp - 1]);
  Seg lp{__shfl_up_sync(0xffffffffu, x.s, 1), __shfl_up_sync(0xffffffffu, x.r, 1)};
  if (lane) pre = seg_op(pre, lp);
  long long run = pre.s;
  bool bad = false;
  double r[DQ_ITEMS];
#pragma unroll
  for (int k = 0; k < DQ_ITEMS; ++k) {
    run = ((rmask >> k) & 1u) ? v[k] : run + v[k];
    bad |= run >= DQ_LIMIT || run <= -DQ_LIMIT;
    r[k] = (double)run * twice_eb;  // exact: |run| < 2^24, twice_eb a power of two
  }
  if (bad) w->inexact = 1;
  if (i0 + DQ_ITEMS <= n) {
    double2* dst = reinterpret_cast<double2*>(out + i0);
#pragma unroll
    for (int k = 0; k < DQ_ITEMS / 2; ++k) dst[k] = make_double2(r[2 * k], r[2 * k + 1]);
  } else {
#pragma unroll
    for (int k = 0; k < DQ_ITEMS; ++k)
      if (i0 + k < n) out[i0 + k] = r[k];
  }
}

// The reference recurrence itself (kernels.py:216-227), one thread: exact in
// every regime (any twice_eb, any outlier values).
__global__ void k_dequant_chain(const uint16_t* __restrict__ codes, uint64_t n, const int64_t* __restrict__ oidx,
                                const double* __restrict__ oval, uint64_t nout, double twice_eb, int32_t mid,
                                double* __restrict__ out) {
  if (threadIdx.x || blockIdx.x) return;
  double pred = 0.0;
  uint64_t j = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (j < nout && (uint64_t)oidx[j] == i) {
      pred = oval[j];
      ++j;
    } else {
      pred = (double)__double2float_rn(pred + twice_eb * (double)((int32_t)codes[i] - mid));
    }
    out[i] = pred;
  }
}

__global__ void k_dq_init(DqWork* w, uint64_t ntiles) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i == 0) { w->tiles = 0; w->inexact = 0; }
  for (; i < ntiles; i += (uint64_t)gridDim.x * blockDim.x) w->desc[i] = 0;
}

}  // namespace bh

using namespace bh;

static uint64_t dq_tiles(uint64_t n) { return (n + DQ_TILE - 1) / DQ_TILE; }

extern "C" size_t bh_dequant_workspace_bytes(uint64_t n) {
  return sizeof(DqWork) + 8 * (dq_tiles(n) + 1);
}

// twice_eb = 2^e with -149 <= e <= 104 (f32 keeps every multiple below 2^24)
static bool pow2_in_range(double x, int* e) {
  if (!(x > 0)) return false;
  int ex = 0;
  const double m = frexp(x, &ex);  // x = m * 2^ex, m in [0.5, 1)
  if (m != 0.5) return false;
  *e = ex - 1;
  return *e >= -149 && *e <= 104;
}

extern "C" int bh_dequantize(const uint16_t* codes_dev, uint64_t n, const int64_t* outlier_idx_dev,
                             const double* outlier_val_dev, const int64_t* outlier_units_dev, uint64_t n_outliers,
                             double twice_eb, uint32_t midpoint, int exact_scan, double* out_dev, void* ws,
                             size_t ws_bytes, int32_t* inexact_dev, void* cuda_stream) {
  if ((n && (!codes_dev || !out_dev)) || (n_outliers && !outlier_idx_dev) || !(twice_eb > 0)) return BH_BAD_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  int e = 0;
  if (exact_scan) {
    if (!pow2_in_range(twice_eb, &e) || !ws || ws_bytes < bh_dequant_workspace_bytes(n) || !inexact_dev ||
        (n_outliers && !outlier_units_dev) || (reinterpret_cast<uintptr_t>(codes_dev) & 15u) ||
        (reinterpret_cast<uintptr_t>(out_dev) & 15u))
      return BH_BAD_ARGUMENT;
    DqWork* w = static_cast<DqWork*>(ws);
    k_dq_init<<<64, 256, 0, st>>>(w, dq_tiles(n));
    if (n)
      k_dequant<<<(unsigned)dq_tiles(n), DQ_THREADS, 0, st>>>(codes_dev, n, outlier_idx_dev,
                                                             reinterpret_cast<const long long*>(outlier_units_dev),
                                                             n_outliers, twice_eb, (int32_t)midpoint, out_dev, w);
    if (cudaMemcpyAsync(inexact_dev, &w->inexact, 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return BH_CUDA_ERROR;
  } else {
    if (n_outliers && !outlier_val_dev) return BH_BAD_ARGUMENT;
    k_dequant_chain<<<1, 32, 0, st>>>(codes_dev, n, outlier_idx_dev, outlier_val_dev, n_outliers, twice_eb,
                                      (int32_t)midpoint, out_dev);
  }
  return cudaGetLastError() == cudaSuccess ? BH_OK : BH_CUDA_ERROR;
}
