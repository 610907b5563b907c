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
// bits -- so pred_i = 2^e * S_i: a segmented prefix sum, computed here as
// reduce (tile aggregates) -> scan (one CTA) -> apply.  (A one-pass decoupled
// look-back spent half its time with whole CTAs parked at the look-back
// barrier: 1.48 ms for 281 M codes, 28 % of HBM; profiles/r02.)  The kernel raises a device
// flag when a running sum leaves that range; the caller then runs the exact
// sequential chain on the device (k_dequant_chain, one thread: slow but
// bit-identical in every regime).
#include "common.cuh"

namespace bh {

constexpr int DQ_THREADS = 256;
constexpr int DQ_ITEMS = 16;                        // codes per thread
constexpr int DQ_TILE = DQ_THREADS * DQ_ITEMS;      // 4096 codes per tile
constexpr long long DQ_LIMIT = 1ll << 24;


struct DqWork {
  int32_t inexact;  // a running sum left +-2^24 (or a tile held more than 64 outliers)
  int32_t pad[3];
};

struct Seg {  // segmented-sum scan element
  long long s;
  uint32_t r;  // a reset (outlier) inside: s is the running value after it
};
__device__ __forceinline__ Seg seg_op(Seg a, Seg b) { return b.r ? b : Seg{a.s + b.s, a.r}; }

// Per tile (DQ_TILE codes): this thread's 16 deltas (code - midpoint, or an
// outlier's value in units of twice_eb with its reset bit), and the block's
// segmented scan of the thread totals.  Shared by the reduce and apply passes.
struct DqTile {
  long long v[DQ_ITEMS];
  uint32_t rmask;
  Seg x;    // inclusive scan of thread totals within its warp
  Seg agg;  // tile aggregate
};

__device__ __forceinline__ void dq_tile(const uint16_t* __restrict__ codes, uint64_t n,
                                        const int64_t* __restrict__ oidx, const long long* __restrict__ ounits,
                                        uint64_t nout, int32_t mid, uint64_t tile, DqWork* w, DqTile& T,
                                        Seg* s_warp) {
  __shared__ uint32_t s_rst[DQ_TILE / 32];  // outlier positions of the tile (bitmask)
  __shared__ long long s_oval[64];          // their values in units of twice_eb (first 64 per tile)
  __shared__ uint32_t s_nout, s_o0;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t t0 = tile * DQ_TILE;
  for (uint32_t i = tid; i < DQ_TILE / 32; i += DQ_THREADS) s_rst[i] = 0;
  if (tid == 0) {  // outliers of this tile: first index >= t0
    uint64_t lo = 0, hi = nout;
    while (lo < hi) {
      const uint64_t m = (lo + hi) >> 1;
      if ((uint64_t)oidx[m] < t0) lo = m + 1; else hi = m;
    }
    uint64_t e = lo;
    while (e < nout && (uint64_t)oidx[e] < t0 + DQ_TILE) ++e;
    s_o0 = (uint32_t)lo;
    s_nout = (uint32_t)(e - lo);
    if (e - lo > 64 && w) w->inexact = 1;  // more than 64 outliers in 4096 codes: take the exact chain
  }
  __syncthreads();
  const uint32_t no = min(s_nout, 64u);
  for (uint32_t k = tid; k < no; k += DQ_THREADS) {
    const uint32_t p = (uint32_t)(oidx[s_o0 + k] - t0);
    atomicOr(&s_rst[p >> 5], 1u << (p & 31));
    s_oval[k] = ounits[s_o0 + k];
  }
  __syncthreads();
  const uint64_t i0 = t0 + (uint64_t)tid * DQ_ITEMS;
  const uint32_t rbits = (s_rst[(tid * DQ_ITEMS) >> 5] >> ((tid * DQ_ITEMS) & 31)) & 0xffffu;
  if (i0 + DQ_ITEMS <= n) {
    const uint4* src = reinterpret_cast<const uint4*>(codes + i0);
    const uint4 a = __ldg(src), b = __ldg(src + 1);
    const uint32_t wv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int k = 0; k < DQ_ITEMS; ++k) T.v[k] = (long long)((wv[k >> 1] >> ((k & 1) * 16)) & 0xffffu) - mid;
  } else {
#pragma unroll
    for (int k = 0; k < DQ_ITEMS; ++k) T.v[k] = i0 + k < n ? (long long)codes[i0 + k] - mid : 0ll;
  }
  T.rmask = 0;
  if (rbits) {
    uint32_t oi = 0;  // rank of this thread's first outlier among the tile's
    for (uint32_t q = 0; q < (tid * DQ_ITEMS) >> 5; ++q) oi += __popc(s_rst[q]);
    oi += __popc(s_rst[(tid * DQ_ITEMS) >> 5] & ((1u << ((tid * DQ_ITEMS) & 31)) - 1u));
#pragma unroll
    for (int k = 0; k < DQ_ITEMS; ++k)
      if ((rbits >> k) & 1u) { T.v[k] = s_oval[oi++]; T.rmask |= 1u << k; }
  }
  Seg t{0, 0};
#pragma unroll
  for (int k = 0; k < DQ_ITEMS; ++k) {
    if ((T.rmask >> k) & 1u) t = Seg{T.v[k], 1};
    else t.s += T.v[k];
  }
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
  }
  __syncthreads();
  T.x = x;
  T.agg = s_warp[DQ_THREADS / 32 - 1];
}

// pass 1: the segmented aggregate of every tile (aggs[tile] = sum, resets[tile])
__global__ void __launch_bounds__(DQ_THREADS) k_dq_reduce(const uint16_t* __restrict__ codes, uint64_t n,
                                                          const int64_t* __restrict__ oidx,
                                                          const long long* __restrict__ ounits, uint64_t nout,
                                                          int32_t mid, long long* __restrict__ aggs,
                                                          uint8_t* __restrict__ resets, DqWork* w) {
  __shared__ Seg s_warp[DQ_THREADS / 32];
  DqTile T;
  dq_tile(codes, n, oidx, ounits, nout, mid, blockIdx.x, w, T, s_warp);
  if (threadIdx.x == 0) {
    aggs[blockIdx.x] = T.agg.s;
    resets[blockIdx.x] = (uint8_t)T.agg.r;
  }
}

// pass 2: exclusive segmented scan of the tile aggregates in two levels --
// every CTA scans 1024 aggregates (coalesced) and keeps its total, one CTA
// scans the totals; the apply pass combines the two prefixes
__device__ __forceinline__ Seg block_excl_seg(Seg v, Seg& total) {
  __shared__ Seg s_w[32];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Seg x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Seg y{__shfl_up_sync(0xffffffffu, x.s, o), __shfl_up_sync(0xffffffffu, x.r, o)};
    if ((int)lane >= o) x = seg_op(y, x);
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  if (warp == 0) {
    Seg z = lane < (blockDim.x >> 5) ? s_w[lane] : Seg{0, 0};
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      Seg y{__shfl_up_sync(0xffffffffu, z.s, o), __shfl_up_sync(0xffffffffu, z.r, o)};
      if ((int)lane >= o) z = seg_op(y, z);
    }
    s_w[lane] = z;
  }
  __syncthreads();
  total = s_w[(blockDim.x >> 5) - 1];
  Seg pre{0, 0};
  if (warp) pre = s_w[warp - 1];
  const Seg lp{__shfl_up_sync(0xffffffffu, x.s, 1), __shfl_up_sync(0xffffffffu, x.r, 1)};
  if (lane) pre = seg_op(pre, lp);
  __syncthreads();
  return pre;
}

__global__ void __launch_bounds__(1024) k_dq_scan_local(long long* __restrict__ aggs, uint8_t* __restrict__ resets,
                                                        uint64_t ntiles, long long* __restrict__ bsum,
                                                        uint8_t* __restrict__ breset) {
  const uint64_t i = (uint64_t)blockIdx.x * 1024 + threadIdx.x;
  const Seg a = i < ntiles ? Seg{aggs[i], resets[i]} : Seg{0, 0};
  Seg tot;
  const Seg pre = block_excl_seg(a, tot);
  if (i < ntiles) {
    aggs[i] = pre.s;                 // prefix within the block
    resets[i] = (uint8_t)pre.r;      // a reset before this tile inside the block
  }
  if (threadIdx.x == 0) {
    bsum[blockIdx.x] = tot.s;
    breset[blockIdx.x] = (uint8_t)tot.r;
  }
}

__global__ void __launch_bounds__(1024) k_dq_scan_top(long long* __restrict__ bsum, uint8_t* __restrict__ breset,
                                                      uint64_t nb) {
  Seg carry{0, 0};
  for (uint64_t b0 = 0; b0 < nb; b0 += 1024) {
    const uint64_t i = b0 + threadIdx.x;
    const Seg a = i < nb ? Seg{bsum[i], breset[i]} : Seg{0, 0};
    Seg tot;
    const Seg pre = seg_op(carry, block_excl_seg(a, tot));
    if (i < nb) bsum[i] = pre.s;     // exclusive prefix of the block totals
    carry = seg_op(carry, tot);
  }
}

// pass 1 without outliers: each tile's sum of (code - midpoint), lean enough
// for eight CTAs per SM (bytes in flight)
__global__ void __launch_bounds__(DQ_THREADS) k_dq_reduce_plain(const uint16_t* __restrict__ codes, uint64_t n,
                                                                int32_t mid, long long* __restrict__ aggs,
                                                                uint8_t* __restrict__ resets) {
  __shared__ long long s_w[DQ_THREADS / 32];
  const uint64_t i0 = (uint64_t)blockIdx.x * DQ_TILE + (uint64_t)threadIdx.x * DQ_ITEMS;
  long long acc = 0;
  if (i0 + DQ_ITEMS <= n) {
    const uint4* src = reinterpret_cast<const uint4*>(codes + i0);
    const uint4 a = __ldg(src), b = __ldg(src + 1);
    uint32_t sm = 0;
    const uint32_t wv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int k = 0; k < 8; ++k) sm += (wv[k] & 0xffffu) + (wv[k] >> 16);
    acc = (long long)sm - (long long)DQ_ITEMS * mid;
  } else {
    for (uint64_t i = i0; i < n && i < i0 + DQ_ITEMS; ++i) acc += (long long)codes[i] - mid;
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
#pragma unroll
    for (int w = 0; w < DQ_THREADS / 32; ++w) t += s_w[w];
    aggs[blockIdx.x] = t;
    resets[blockIdx.x] = 0;
  }
}

// pass 3: values = 2^e * (tile prefix + in-tile segmented scan), float64 out
__global__ void __launch_bounds__(DQ_THREADS) k_dequant(const uint16_t* __restrict__ codes, uint64_t n,
                                                        const int64_t* __restrict__ oidx,
                                                        const long long* __restrict__ ounits, uint64_t nout,
                                                        double twice_eb, int32_t mid,
                                                        const long long* __restrict__ prefix,
                                                        const uint8_t* __restrict__ resets_pre,
                                                        const long long* __restrict__ bpre,
                                                        double* __restrict__ out, DqWork* w) {
  __shared__ Seg s_warp[DQ_THREADS / 32];
  DqTile T;
  dq_tile(codes, n, oidx, ounits, nout, mid, blockIdx.x, nullptr, T, s_warp);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // tile prefix: the block prefix unless a reset precedes the tile in its block
  Seg pre{resets_pre[blockIdx.x] ? prefix[blockIdx.x] : bpre[blockIdx.x >> 10] + prefix[blockIdx.x], 0};
  if (warp) pre = seg_op(pre, s_warp[warp - 1]);
  const Seg lp{__shfl_up_sync(0xffffffffu, T.x.s, 1), __shfl_up_sync(0xffffffffu, T.x.r, 1)};
  if (lane) pre = seg_op(pre, lp);
  long long run = pre.s;
  bool bad = false;
  double r[DQ_ITEMS];
#pragma unroll
  for (int k = 0; k < DQ_ITEMS; ++k) {
    run = ((T.rmask >> k) & 1u) ? T.v[k] : run + T.v[k];
    bad |= run >= DQ_LIMIT || run <= -DQ_LIMIT;
    r[k] = (double)run * twice_eb;  // exact: |run| < 2^24, twice_eb a power of two
  }
  if (bad) w->inexact = 1;
  // through shared memory (rows of 16 padded to 17 doubles: conflict-free),
  // so each warp store covers 512 consecutive bytes
  extern __shared__ double s_out[];
#pragma unroll
  for (int k = 0; k < DQ_ITEMS; ++k) s_out[threadIdx.x * (DQ_ITEMS + 1) + k] = r[k];
  __syncthreads();
  const uint64_t t0 = (uint64_t)blockIdx.x * DQ_TILE;
#pragma unroll
  for (int j = 0; j < DQ_ITEMS / 2; ++j) {
    const uint32_t q = (uint32_t)j * 2 * DQ_THREADS + 2 * threadIdx.x;  // item pair within the tile
    const uint32_t sa = (q / DQ_ITEMS) * (DQ_ITEMS + 1) + (q % DQ_ITEMS);
    const uint64_t g = t0 + q;
    if (g + 2 <= n) {
      *reinterpret_cast<double2*>(out + g) = make_double2(s_out[sa], s_out[sa + 1]);
    } else if (g < n) {
      out[g] = s_out[sa];
    }
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

__global__ void k_dq_init(DqWork* w) {
  if (threadIdx.x == 0) w->inexact = 0;
}

}  // namespace bh

using namespace bh;

static uint64_t dq_tiles(uint64_t n) { return (n + DQ_TILE - 1) / DQ_TILE; }

extern "C" size_t bh_dequant_workspace_bytes(uint64_t n) {
  const uint64_t nt = dq_tiles(n), nb = (nt + 1023) / 1024 + 1;
  return align16(sizeof(DqWork)) + align16(8 * (nt + 1)) + align16(nt + 1) + align16(8 * nb) + align16(nb);
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
    const uint64_t nt = dq_tiles(n);
    long long* aggs = reinterpret_cast<long long*>(static_cast<char*>(ws) + align16(sizeof(DqWork)));
    uint8_t* resets = reinterpret_cast<uint8_t*>(aggs) + align16(8 * (nt + 1));
    const long long* un = reinterpret_cast<const long long*>(outlier_units_dev);
    k_dq_init<<<1, 32, 0, st>>>(w);
    if (n) {
      // reduce -> scan of the tile aggregates -> apply: every pass streams at
      // HBM speed with no inter-CTA waiting (12 B per code in all)
      if (n_outliers)
        k_dq_reduce<<<(unsigned)nt, DQ_THREADS, 0, st>>>(codes_dev, n, outlier_idx_dev, un, n_outliers,
                                                         (int32_t)midpoint, aggs, resets, w);
      else
        k_dq_reduce_plain<<<(unsigned)nt, DQ_THREADS, 0, st>>>(codes_dev, n, (int32_t)midpoint, aggs, resets);
      const uint64_t nb = (nt + 1023) / 1024;
      long long* bsum = reinterpret_cast<long long*>(resets + align16(nt + 1));
      uint8_t* breset = reinterpret_cast<uint8_t*>(bsum) + align16(8 * (nb + 1));
      k_dq_scan_local<<<(unsigned)nb, 1024, 0, st>>>(aggs, resets, nt, bsum, breset);
      k_dq_scan_top<<<1, 1024, 0, st>>>(bsum, breset, nb);
      k_dequant<<<(unsigned)nt, DQ_THREADS, DQ_THREADS * (DQ_ITEMS + 1) * sizeof(double), st>>>(
          codes_dev, n, outlier_idx_dev, un, n_outliers, twice_eb, (int32_t)midpoint, aggs, resets, bsum, out_dev,
          w);
    }
    if (cudaMemcpyAsync(inexact_dev, &w->inexact, 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return BH_CUDA_ERROR;
  } else {
    if (n_outliers && !outlier_val_dev) return BH_BAD_ARGUMENT;
    k_dequant_chain<<<1, 32, 0, st>>>(codes_dev, n, outlier_idx_dev, outlier_val_dev, n_outliers, twice_eb,
                                      (int32_t)midpoint, out_dev);
  }
  return cudaGetLastError() == cudaSuccess ? BH_OK : BH_CUDA_ERROR;
}
