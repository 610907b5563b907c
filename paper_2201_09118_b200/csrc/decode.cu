// decode.cu -- reference-structured decode kernels (K2, K3, K4, K5, K6, K7, K8).
//
// These kernels keep the reference's phase structure and its SyncState arrays
// (int64 entry/exit/count per subsequence, state.py:16-41) so every sub-step of
// the parhuff API has a GPU twin whose intermediate state can be compared with
// the reference bit-for-bit.  The single-pass fused kernels in fused.cu are the
// fast path used by bh_decode; they produce identical symbols.
#include "common.cuh"

namespace bh {

constexpr int MODE_GAP = 1;   // windows [e_i, e_{i+1}), last [e, tb) (gap_decoder.py:50-53)
constexpr int MODE_SYNC = 2;  // windows [e_i, (i+1)*sb) (sync_decoder.py:112-113)

__global__ void k_report_init(DevReport* rep) {
  if (threadIdx.x == 0) {
    rep->status = 0x7fffffff;
    rep->fail_slot = ~0ull;
    rep->bits_sync = rep->bits_count = rep->bits_write = 0;
    rep->write_rounds = rep->staged_slots = rep->bypass_slots = 0;
    rep->total_symbols = rep->stale_seams = rep->seam_passes = rep->repair_needed = 0;
    rep->pad[0] = rep->pad[1] = rep->pad[2] = rep->pad[3] = 0;
    rep->phase_ns[0] = ~0ull;  // min over CTAs
    for (int k = 1; k < 6; ++k) rep->phase_ns[k] = 0;
  }
}

__global__ void k_stamp(DevReport* rep, int k) {
  const unsigned long long t = global_ns();
  if (k == 0) atomicMin(&rep->phase_ns[0], t);
  else atomicMax(&rep->phase_ns[k], t);
}

// CTA-uniform early exit (one thread reads, everyone agrees).
__device__ __forceinline__ bool cta_should_skip(const DevReport* rep, const unsigned long long* gate) {
  __shared__ int s_skip;
  if (threadIdx.x == 0)
    s_skip = (*(volatile const int32_t*)&rep->status != 0x7fffffff) ||
             (gate && *(volatile const unsigned long long*)gate == 0);
  __syncthreads();
  return s_skip != 0;
}

__device__ __forceinline__ TableView dev_table(const void* blob, uint32_t max_codes) {
  const TableHdr* h = static_cast<const TableHdr*>(blob);
  return table_view(blob, max_codes, h->ncodes);
}

// gap_decoder.py:24-33
__global__ void k_entries_from_gap(const uint8_t* __restrict__ gap, uint64_t nsub, uint32_t sb,
                                   int64_t* __restrict__ entries) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nsub; i += stride)
    entries[i] = (int64_t)(i * sb + gap[i]);
}

// kernels.py:47-76 for every slot, one thread per slot.
__global__ void __launch_bounds__(256) k_count_windows(
    const uint32_t* __restrict__ words, const void* table, uint32_t max_codes, int mode,
    const int64_t* __restrict__ entries, uint64_t nsub, uint32_t sb, uint64_t tb,
    int64_t* __restrict__ counts, int64_t* __restrict__ exits, DevReport* rep, int stats) {
  __shared__ __align__(16) uint32_t s_lut[LUT_SIZE];
  __shared__ __align__(16) uint16_t s_cnt[LUT_SIZE];
  TableView t = dev_table(table, max_codes);
  load_luts(t, s_lut, s_cnt);
  __syncthreads();
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  unsigned long long bits = 0;
  if (i < nsub) {
    uint64_t entry = (uint64_t)entries[i];
    uint64_t stop;
    if (mode == MODE_GAP) stop = (i + 1 < nsub) ? (uint64_t)entries[i + 1] : tb;
    else stop = (i + 1) * (uint64_t)sb;
    if (stop > tb) stop = tb;
    uint64_t pos = entry;
    uint32_t n = 0;
    bool ok = true;
    if (pos < stop) {
      BitReader r;
      r.init(words, pos);
      ok = count_window(r, pos, stop, s_lut, s_cnt, t, n);
    }
    counts[i] = n;
    exits[i] = (int64_t)pos;
    bits = pos - entry;
    if (!ok) report_error(rep, BH_INVALID, i);
  }
  if (stats) {
    bits = warp_sum(bits);
    if ((threadIdx.x & 31) == 0 && bits) atomicAdd(&rep->bits_count, bits);
  }
}

// One window decode for the sync kernels; returns false on an invalid code.
__device__ __forceinline__ bool sync_window(const uint32_t* words, const uint32_t* s_lut,
                                            const uint16_t* s_cnt, const TableView& t,
                                            uint64_t slot, uint64_t entry, uint32_t sb, uint64_t tb,
                                            uint32_t& n, uint64_t& exit_pos) {
  uint64_t stop = (slot + 1) * (uint64_t)sb;
  if (stop > tb) stop = tb;
  uint64_t pos = entry;
  n = 0;
  bool ok = true;
  if (pos < stop) {
    BitReader r;
    r.init(words, pos);
    ok = count_window(r, pos, stop, s_lut, s_cnt, t, n);
  }
  exit_pos = pos;
  return ok;
}

// K2 (reference-exact form): sync_decoder.py:62-109 with one warp per sequence.
// Round 1 decodes every slot from its boundary (or only the first slot from
// `seed`); round k hands each re-decoded slot's exit to its right neighbour,
// which retires when the exit equals its entry and re-decodes otherwise.
// flags_a/flags_b hold "decoded in the previous/current round" per slot.
__global__ void __launch_bounds__(128) k_intra_sync(
    const uint32_t* __restrict__ words, const void* table, uint32_t max_codes, uint64_t nsub,
    uint64_t nseq, uint32_t sb, uint32_t sps, uint64_t tb, const int64_t* __restrict__ seeds,
    int64_t* __restrict__ entries, int64_t* __restrict__ exits, int64_t* __restrict__ counts,
    uint8_t* __restrict__ synced, int32_t* __restrict__ iterations, uint8_t* __restrict__ flags_a,
    uint8_t* __restrict__ flags_b, uint32_t round_cap, DevReport* rep, int stats,
    const unsigned long long* gate) {
  __shared__ __align__(16) uint32_t s_lut[LUT_SIZE];
  __shared__ __align__(16) uint16_t s_cnt[LUT_SIZE];
  if (cta_should_skip(rep, gate)) return;  // earlier failure, or nothing stale this pass
  TableView t = dev_table(table, max_codes);
  load_luts(t, s_lut, s_cnt);
  __syncthreads();
  const uint32_t lane = lane_id();
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  unsigned long long bits = 0;
  for (uint64_t q = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); q < nseq; q += warps) {
    // seeds: -1 = leave this sequence alone, -2 = unseeded, >= 0 = seed bit
    const int64_t seed = seeds ? seeds[q] : -2;
    if (seed == -1) continue;
    const bool seeded = seed >= 0;
    const uint64_t j0 = q * sps;
    const uint64_t j1 = min(j0 + sps, nsub);
    const uint64_t nslots = j1 - j0;
    const uint64_t cap = round_cap ? round_cap : nslots;
    bool fail = false;
    uint64_t fail_slot = ~0ull;
    // round 1
    for (uint64_t slot = j0 + lane; slot < j1; slot += 32) {
      bool dec = !seeded || slot == j0;
      if (!seeded) entries[slot] = (int64_t)(slot * sb);
      else if (slot == j0) entries[slot] = seed;
      flags_a[slot] = dec ? 1 : 0;
      if (dec) {
        uint32_t n;
        uint64_t ex;
        if (!sync_window(words, s_lut, s_cnt, t, slot, (uint64_t)entries[slot], sb, tb, n, ex)) {
          fail = true;
          fail_slot = min(fail_slot, slot);
        }
        counts[slot] = n;
        exits[slot] = (int64_t)ex;
        bits += ex - (uint64_t)entries[slot];
      }
    }
    __syncwarp();
    uint8_t* prev = flags_a;
    uint8_t* cur = flags_b;
    uint64_t rounds = 1, last_active = 1;
    bool any_fail = __any_sync(0xffffffffu, fail);
    while (!any_fail && rounds < cap) {
      bool live = false;
      for (uint64_t slot = j0 + 1 + lane; slot < j1; slot += 32) live |= prev[slot - 1] != 0;
      if (!__any_sync(0xffffffffu, live)) break;  // early exit (results identical either way)
      ++rounds;
      last_active = rounds;
      // phase A: adopt incoming exits (snapshot of the previous round)
      for (uint64_t slot = j0 + lane; slot < j1; slot += 32) {
        uint8_t d = 0;
        if (slot > j0 && prev[slot - 1]) {
          int64_t in = exits[slot - 1];
          if (in != entries[slot]) { entries[slot] = in; d = 1; }
        }
        cur[slot] = d;
      }
      __syncwarp();
      // phase B: re-decode
      for (uint64_t slot = j0 + lane; slot < j1; slot += 32) {
        if (!cur[slot]) continue;
        uint32_t n;
        uint64_t ex;
        if (!sync_window(words, s_lut, s_cnt, t, slot, (uint64_t)entries[slot], sb, tb, n, ex)) {
          fail = true;
          fail_slot = min(fail_slot, slot);
        }
        counts[slot] = n;
        exits[slot] = (int64_t)ex;
        bits += ex - (uint64_t)entries[slot];
      }
      __syncwarp();
      uint8_t* tmp = prev; prev = cur; cur = tmp;
      any_fail = __any_sync(0xffffffffu, fail);
    }
    if (fail) report_error(rep, BH_INVALID, fail_slot);
    if (any_fail) continue;
    bool pending = false;
    for (uint64_t slot = j0 + lane; slot + 1 < j1; slot += 32) pending |= prev[slot] != 0;
    if (__any_sync(0xffffffffu, pending)) {
      if (lane == 0) report_error(rep, BH_NOFIXPOINT, q);
      continue;
    }
    for (uint64_t slot = j0 + lane; slot < j1; slot += 32) synced[slot] = 1;
    if (lane == 0) iterations[q] = (int32_t)last_active;
  }
  if (stats) {
    bits = warp_sum(bits);
    if (lane == 0 && bits) atomicAdd(&rep->bits_sync, bits);
  }
}

// K3 seam check (sync_decoder.py:133-135): snapshot seeds for the pass.
__global__ void k_seam_check(const int64_t* __restrict__ entries, const int64_t* __restrict__ exits,
                             uint64_t nseq, uint32_t sps, int64_t* __restrict__ seeds,
                             unsigned long long* stale_ctr) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  unsigned long long stale = 0;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nseq; q += stride) {
    int64_t s = -1;
    if (q > 0) {
      uint64_t f = q * sps;
      int64_t seed = exits[f - 1];
      if (seed != entries[f]) { s = seed; ++stale; }
    }
    seeds[q] = s;
  }
  stale = warp_sum(stale);
  if ((threadIdx.x & 31) == 0 && stale) atomicAdd(stale_ctr, stale);
}

__global__ void k_zero_u64(unsigned long long* p, uint64_t n) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) p[i] = 0;
}

// K5: decoupled look-back exclusive scan of int64 counts (state.py:44-53).
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_i64(const int64_t* __restrict__ counts,
                                                           uint64_t n, int64_t* __restrict__ oi,
                                                           unsigned long long* desc,
                                                           unsigned long long* tile_ctr) {
  __shared__ unsigned long long s_warp[SCAN_THREADS / 32];
  __shared__ unsigned long long s_tile, s_excl;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1ull);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t base = tile * SCAN_TILE + (uint64_t)threadIdx.x * SCAN_ITEMS;
  unsigned long long v[SCAN_ITEMS], sum = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    v[k] = base + k < n ? (unsigned long long)counts[base + k] : 0ull;
    sum += v[k];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long x = sum;
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    unsigned long long tw = lane < SCAN_THREADS / 32 ? s_warp[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, tw, o);
      if (lane >= o) tw += y;
    }
    if (lane < SCAN_THREADS / 32) s_warp[lane] = tw;
    __syncwarp();
    unsigned long long total = s_warp[SCAN_THREADS / 32 - 1];
    unsigned long long excl = 0;
    if (tile == 0) {
      if (lane == 0) st_release(desc, LB_FLAG_INC | total);
    } else {
      if (lane == 0) st_release(desc + tile, LB_FLAG_AGG | total);
      excl = warp_lookback(desc, tile);
      if (lane == 0) st_release(desc + tile, LB_FLAG_INC | (excl + total));
    }
    if (lane == 0) s_excl = excl;
  }
  __syncthreads();
  unsigned long long run = s_excl + (warp ? s_warp[warp - 1] : 0ull) + x - sum;
  if (tile == 0 && threadIdx.x == 0) oi[0] = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    run += v[k];
    if (base + k < n) oi[base + k + 1] = (int64_t)run;
  }
}

// Decode exactly c symbols from `entry` into dst[0..c); returns false on an
// invalid code; adds the consumed bits.  (kernels.py:79-99 for one slot)
__device__ __forceinline__ bool decode_symbols(const uint32_t* words, const uint32_t* s_lut,
                                               const TableView& t, uint64_t entry, uint64_t c,
                                               uint16_t* dst, unsigned long long& bits) {
  if (c == 0) return true;
  BitReader r;
  r.init(words, entry);
  uint64_t consumed = 0;
  for (uint64_t k = 0; k < c; ++k) {
    uint32_t e = lookup(s_lut, t, r.peek());
    uint32_t len = (e >> 16) & 0xffu;
    if (len == 0) { bits += consumed; return false; }
    dst[k] = (uint16_t)e;
    r.skip(len);
    consumed += len;
  }
  bits += consumed;
  return true;
}

// K7 (reference-exact form): staging.py:113-147 per sequence, one warp per
// sequence, staging buffer of `capacity` symbols per warp in shared memory.
constexpr int DW_WARPS = 4;
__global__ void __launch_bounds__(DW_WARPS * 32) k_decode_write(
    const uint32_t* __restrict__ words, const void* table, uint32_t max_codes, uint64_t nsub,
    uint64_t nseq, uint32_t sps, const int64_t* __restrict__ entries,
    const int64_t* __restrict__ counts, const int64_t* __restrict__ oi,
    const int64_t* __restrict__ seq_ids, uint64_t nids, uint32_t capacity, uint32_t stage_stride,
    uint16_t* __restrict__ out, uint64_t out_len, DevReport* rep, int stats,
    const int64_t* __restrict__ classes, const uint32_t* __restrict__ caps) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ __align__(16) uint32_t s_lut[LUT_SIZE];
  __shared__ __align__(16) uint16_t s_cnt[LUT_SIZE];
  if (cta_should_skip(rep, nullptr)) return;  // an earlier phase failed
  TableView t = dev_table(table, max_codes);
  load_luts(t, s_lut, s_cnt);
  __syncthreads();
  const uint32_t lane = lane_id(), wib = threadIdx.x >> 5;
  uint16_t* staging = reinterpret_cast<uint16_t*>(dyn) + (size_t)wib * stage_stride;
  const uint64_t warps = (uint64_t)gridDim.x * DW_WARPS;
  unsigned long long bits = 0, rounds = 0, staged = 0, bypass = 0;
  bool fail = false;
  uint64_t fail_slot = ~0ull;
  for (uint64_t w = blockIdx.x * (uint64_t)DW_WARPS + wib; w < nids; w += warps) {
    const uint64_t q = seq_ids ? (uint64_t)seq_ids[w] : w;
    if (q >= nseq) continue;
    // tuner.py:150-191: a sequence's class selects its staging capacity
    const uint64_t cap = classes ? caps[classes[q] - 1] : capacity;
    const uint64_t j0 = q * sps, j1 = min(j0 + sps, nsub);
    uint64_t si = (uint64_t)oi[j0];
    const uint64_t ei = (uint64_t)oi[j1];
    uint64_t j = j0;
    while (si < ei) {
      ++rounds;
      const uint64_t window = si + cap;
      while ((uint64_t)oi[j + 1] <= si) ++j;
      uint64_t k = j;
      while (k < j1 && (uint64_t)oi[k + 1] <= window) ++k;
      if (k == j) {
        // bypass: slot j's range alone exceeds the buffer
        if (lane == 0) {
          uint64_t d = (uint64_t)oi[j], c = (uint64_t)counts[j];
          if (d + c <= out_len) {
            if (!decode_symbols(words, s_lut, t, (uint64_t)entries[j], c, out + d, bits)) {
              fail = true;
              fail_slot = min(fail_slot, j);
            }
          }
        }
        si = (uint64_t)oi[j + 1];
        ++j;
        ++bypass;
        continue;
      }
      const uint64_t temp_end = k < j1 ? (uint64_t)oi[k] : ei;
      for (uint64_t x = j + lane; x < k; x += 32) {
        uint64_t d = (uint64_t)oi[x] - si, c = (uint64_t)counts[x];
        if (!decode_symbols(words, s_lut, t, (uint64_t)entries[x], c, staging + d, bits)) {
          fail = true;
          fail_slot = min(fail_slot, x);
        }
      }
      __syncwarp();
      const uint64_t len = temp_end - si;
      if (si + len <= out_len)
        for (uint64_t x = lane; x < len; x += 32) out[si + x] = staging[x];
      __syncwarp();
      staged += k - j;
      si = temp_end;
      j = k;
    }
  }
  if (fail) report_error(rep, BH_INVALID, fail_slot);
  if (stats) {
    bits = warp_sum(bits);
    if (lane == 0) {
      if (bits) atomicAdd(&rep->bits_write, bits);
      if (rounds) atomicAdd(&rep->write_rounds, rounds);
      if (staged) atomicAdd(&rep->staged_slots, staged);
      if (bypass) atomicAdd(&rep->bypass_slots, bypass);
    }
  }
}

// Compare the scanned total with the header (sync: Truncated, gap: BadGap).
__global__ void k_check_total(const int64_t* __restrict__ oi, uint64_t nsub, uint64_t expect,
                              int status_on_mismatch, DevReport* rep) {
  if (threadIdx.x == 0) {
    uint64_t tot = oi ? (uint64_t)oi[nsub] : 0;
    rep->total_symbols = tot;
    if (tot != expect) report_error(rep, status_on_mismatch, ~0ull);
  }
}

// tuner.py:109-114
__global__ void k_seq_counts(const int64_t* __restrict__ counts, uint64_t nsub, uint64_t nseq,
                             uint32_t sps, int64_t* __restrict__ seqc) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nseq; q += stride) {
    uint64_t j0 = q * sps, j1 = min(j0 + sps, nsub);
    int64_t s = 0;
    for (uint64_t j = j0; j < j1; ++j) s += counts[j];
    seqc[q] = s;
  }
}

// K6 (tuner.py:117-147): classify + per-tile class histogram, 1024 sequences/tile.
constexpr int TUNE_TILE = 1024;
__global__ void __launch_bounds__(TUNE_TILE) k_tune_classify(
    const int64_t* __restrict__ seqc, uint64_t nseq, uint64_t seq_bits, uint64_t last_bits,
    uint32_t width, uint32_t t_high, int64_t* __restrict__ classes, uint32_t* __restrict__ hist) {
  extern __shared__ uint32_t s_hist[];
  const uint32_t C = t_high + 1;
  for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) s_hist[c] = 0;
  __syncthreads();
  uint64_t q = blockIdx.x * (uint64_t)TUNE_TILE + threadIdx.x;
  if (q < nseq) {
    uint64_t bits = (q == nseq - 1) ? last_bits : seq_bits;
    uint64_t cnt = (uint64_t)seqc[q];
    uint64_t c = cnt ? (cnt * width + bits - 1) / bits : 1;  // integer ceil
    if (c > C) c = C;
    classes[q] = (int64_t)c;
    atomicAdd(&s_hist[c - 1], 1u);
  }
  __syncthreads();
  for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) hist[(uint64_t)blockIdx.x * C + c] = s_hist[c];
}

// single CTA: per-class exclusive offsets for every tile, freq and start.
__global__ void k_tune_offsets(uint32_t* __restrict__ hist, uint64_t ntiles, uint32_t t_high,
                               int64_t* __restrict__ freq, int64_t* __restrict__ start) {
  const uint32_t C = t_high + 1;
  __shared__ unsigned long long s_tot[256];
  for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) {
    unsigned long long acc = 0;
    for (uint64_t tl = 0; tl < ntiles; ++tl) acc += hist[tl * C + c];
    s_tot[c] = acc;
    freq[c] = (int64_t)acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long a = 0;
    for (uint32_t c = 0; c < C; ++c) { unsigned long long f = s_tot[c]; s_tot[c] = a; a += f; start[c] = (int64_t)s_tot[c]; }
  }
  __syncthreads();
  for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) {
    unsigned long long run = s_tot[c];
    for (uint64_t tl = 0; tl < ntiles; ++tl) {
      uint32_t h = hist[tl * C + c];
      hist[tl * C + c] = (uint32_t)run;  // overwritten with the tile offset (fits: < 2^32 seqs)
      run += h;
    }
  }
}

// stable counting-sort placement: perm[offset(tile, class) + rank within tile]
__global__ void __launch_bounds__(TUNE_TILE) k_tune_perm(const int64_t* __restrict__ classes,
                                                         uint64_t nseq, uint32_t t_high,
                                                         const uint32_t* __restrict__ tile_off,
                                                         int64_t* __restrict__ perm) {
  extern __shared__ uint32_t s_wc[];  // [32 warps][C]
  const uint32_t C = t_high + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (uint32_t i = threadIdx.x; i < 32 * C; i += blockDim.x) s_wc[i] = 0;
  __syncthreads();
  uint64_t q = blockIdx.x * (uint64_t)TUNE_TILE + threadIdx.x;
  uint32_t c = q < nseq ? (uint32_t)classes[q] - 1 : 0xffffffffu;
  unsigned peers = __match_any_sync(0xffffffffu, c);
  uint32_t wrank = __popc(peers & ((1u << lane) - 1));
  if (c != 0xffffffffu && wrank == 0) s_wc[warp * C + c] = __popc(peers);
  __syncthreads();
  if (c != 0xffffffffu) {
    uint32_t r = tile_off[(uint64_t)blockIdx.x * C + c] + wrank;
    for (int w = 0; w < warp; ++w) r += s_wc[w * C + c];
    perm[r] = (int64_t)q;
  }
}

// K8: cuSZ-style coarse-grained decoder -- one thread per fixed chunk of
// symbols starting at a recorded bit offset, bit-serial canonical matching
// (the per-length first-code loop of kernels.py:35-44), direct global writes.
__global__ void __launch_bounds__(256) k_coarse(const uint32_t* __restrict__ words, const void* table,
                                                uint32_t max_codes, const uint64_t* __restrict__ offs,
                                                uint64_t chunk, uint64_t n, uint16_t* __restrict__ out,
                                                DevReport* rep) {
  __shared__ uint32_t s_lim[34];   // left-justified limit per length, 64-bit saturated to 2^32-1
  __shared__ uint32_t s_first[34]; // canonical index of the first code of each length
  __shared__ uint32_t s_fcode[34];
  __shared__ uint32_t s_max;
  TableView t = dev_table(table, max_codes);
  if (threadIdx.x == 0) {
    // derive per-length (first code, first index) from the canonical lj array
    uint32_t ml = t.hdr->max_len;
    s_max = ml;
    uint32_t idx = 0;
    unsigned long long code = 0;
    for (uint32_t ln = 1; ln <= 32; ++ln) {
      uint32_t cnt = 0;
      while (idx + cnt < t.ncodes && t.ljlen[idx + cnt] == ln) ++cnt;
      s_fcode[ln] = (uint32_t)code;
      s_first[ln] = idx;
      s_lim[ln] = cnt;  // count per length
      code = (code + cnt) << 1;
      idx += cnt;
    }
  }
  __syncthreads();
  uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t k0 = c * chunk;
  if (k0 >= n) return;
  uint64_t k1 = min(k0 + chunk, n);
  uint64_t pos = offs[c];
  const uint32_t ml = s_max;
  for (uint64_t k = k0; k < k1; ++k) {
    uint32_t code = 0, ln = 1;
    uint32_t word = __ldg(words + (pos >> 5));
    for (; ln <= ml; ++ln) {
      uint32_t b = (word >> (31 - (uint32_t)(pos & 31))) & 1u;
      ++pos;
      if ((pos & 31) == 0) word = __ldg(words + (pos >> 5));
      code = (code << 1) | b;
      uint32_t d = code - s_fcode[ln];
      if (code >= s_fcode[ln] && d < s_lim[ln]) {
        out[k] = t.ljsym[s_first[ln] + d];
        break;
      }
    }
    if (ln > ml) { report_error(rep, BH_INVALID, k); return; }
  }
}

}  // namespace bh

// ---------------------------------------------------------------------------
// extern "C" entry points for the reference-structured sub-steps
// ---------------------------------------------------------------------------
using namespace bh;

namespace {
inline cudaStream_t S(void* p) { return static_cast<cudaStream_t>(p); }
inline int last_status() { return cudaGetLastError() == cudaSuccess ? BH_OK : BH_CUDA_ERROR; }
inline uint64_t nsub_of(const bh_stream* s) { return s->subseq_bits ? (s->total_bits + s->subseq_bits - 1) / s->subseq_bits : 0; }
inline uint64_t nseq_of(const bh_stream* s) { return s->subseqs_per_seq ? (nsub_of(s) + s->subseqs_per_seq - 1) / s->subseqs_per_seq : 0; }
inline unsigned grid_for(uint64_t n, unsigned threads, unsigned cap = 65535u * 16) {
  uint64_t g = (n + threads - 1) / threads;
  if (g == 0) g = 1;
  return (unsigned)(g > cap ? cap : g);
}
inline bool bad_stream(const bh_stream* s) {
  return !s || s->subseq_bits == 0 || s->subseqs_per_seq == 0 || (s->total_bits && !s->words_dev) ||
         !s->table_dev;
}
int sm_count() { return device_sm_count(); }
}  // namespace

extern "C" int bh_device_sm_count(void) { return sm_count(); }

extern "C" size_t bh_report_bytes(void) { return sizeof(DevReport); }

int bh::stamp_phase(void* report_dev, int k, cudaStream_t st) {
  k_stamp<<<1, 1, 0, st>>>(static_cast<DevReport*>(report_dev), k);
  return cudaGetLastError() == cudaSuccess ? BH_OK : BH_CUDA_ERROR;
}

extern "C" int bh_report_init(void* report_dev, void* cuda_stream) {
  k_report_init<<<1, 32, 0, S(cuda_stream)>>>(static_cast<DevReport*>(report_dev));
  return last_status();
}

extern "C" int bh_report_read(const void* report_dev, bh_report* out, void* cuda_stream) {
  DevReport r;
  if (cudaMemcpyAsync(&r, report_dev, sizeof(r), cudaMemcpyDeviceToHost, S(cuda_stream)) != cudaSuccess)
    return BH_CUDA_ERROR;
  if (cudaStreamSynchronize(S(cuda_stream)) != cudaSuccess) return BH_CUDA_ERROR;
  out->status = r.status == 0x7fffffff ? BH_OK : r.status;
  if (r.pad[2] == 0xF05EDull) {  // written by a fused kernel: status epoch-tagged in pad[0]
    const uint32_t ep = (uint32_t)r.pad[1];
    const unsigned long long tag = r.pad[0];
    out->status = (uint32_t)(tag >> 32) == ep ? (int32_t)(0x7fffffffu - (uint32_t)tag) : BH_OK;
    if (ep && (uint32_t)r.pad[3] == ep) out->status = BH_NEED_STAGED;  // fused path declined
  }
  out->fail_slot = r.fail_slot;
  out->bits_sync = r.bits_sync;
  out->bits_count = r.bits_count;
  out->bits_write = r.bits_write;
  out->write_rounds = r.write_rounds;
  out->staged_slots = r.staged_slots;
  out->bypass_slots = r.bypass_slots;
  out->total_symbols = r.total_symbols;
  out->stale_seams = r.stale_seams;
  out->seam_passes = r.seam_passes;
  out->repair_needed = r.repair_needed;
  for (int k = 0; k < 6; ++k) out->phase_ns[k] = r.phase_ns[k];
  return BH_OK;
}

extern "C" int bh_entries_from_gap(const bh_stream* s, int64_t* entries_dev, void* cuda_stream) {
  if (bad_stream(s)) return BH_BAD_ARGUMENT;
  if (!s->gap_dev) return BH_NOTPRESENT;
  uint64_t ns = nsub_of(s);
  if (ns) k_entries_from_gap<<<grid_for(ns, 256, 4096), 256, 0, S(cuda_stream)>>>(s->gap_dev, ns, s->subseq_bits, entries_dev);
  return last_status();
}

extern "C" int bh_count_windows(const bh_stream* s, int mode, const int64_t* entries_dev,
                                int64_t* counts_dev, int64_t* exits_dev, void* report_dev,
                                void* cuda_stream) {
  if (bad_stream(s) || (mode != MODE_GAP && mode != MODE_SYNC)) return BH_BAD_ARGUMENT;
  uint64_t ns = nsub_of(s);
  if (ns)
    k_count_windows<<<(unsigned)((ns + 255) / 256), 256, 0, S(cuda_stream)>>>(
        s->words_dev, s->table_dev, s->max_codes, mode, entries_dev, ns, s->subseq_bits,
        s->total_bits, counts_dev, exits_dev, static_cast<DevReport*>(report_dev), 1);
  return last_status();
}

extern "C" size_t bh_scan_workspace_bytes(uint64_t n) {
  return sizeof(unsigned long long) * (2 + (n + SCAN_TILE - 1) / SCAN_TILE);
}

extern "C" int bh_output_index(const int64_t* counts_dev, uint64_t n, int64_t* oi_dev, void* ws,
                               size_t ws_bytes, void* cuda_stream) {
  if (ws_bytes < bh_scan_workspace_bytes(n)) return BH_BAD_ARGUMENT;
  unsigned long long* w = static_cast<unsigned long long*>(ws);
  uint64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (n == 0) return cudaMemsetAsync(oi_dev, 0, sizeof(int64_t), S(cuda_stream)) == cudaSuccess ? BH_OK : BH_CUDA_ERROR;
  k_zero_u64<<<grid_for(tiles + 2, 256, 1024), 256, 0, S(cuda_stream)>>>(w, tiles + 2);
  k_scan_i64<<<(unsigned)tiles, SCAN_THREADS, 0, S(cuda_stream)>>>(counts_dev, n, oi_dev, w + 2, w);
  return last_status();
}

extern "C" int bh_intra_sync_ex(const bh_stream* s, const int64_t* seeds_dev, uint32_t round_cap,
                                const unsigned long long* gate,
                                int64_t* entries_dev, int64_t* exits_dev, int64_t* counts_dev,
                                uint8_t* synced_dev, int32_t* iterations_dev, void* ws,
                                size_t ws_bytes, void* report_dev, void* cuda_stream) {
  if (bad_stream(s)) return BH_BAD_ARGUMENT;
  uint64_t ns = nsub_of(s), nq = nseq_of(s);
  if (ws_bytes < 2 * ns) return BH_BAD_ARGUMENT;
  if (!nq) return BH_OK;
  uint8_t* fa = static_cast<uint8_t*>(ws);
  uint8_t* fb = fa + ns;
  unsigned grid = grid_for(nq, 4, (unsigned)sm_count() * 64);
  k_intra_sync<<<grid, 128, 0, S(cuda_stream)>>>(s->words_dev, s->table_dev, s->max_codes, ns, nq,
                                                 s->subseq_bits, s->subseqs_per_seq, s->total_bits,
                                                 seeds_dev, entries_dev, exits_dev, counts_dev,
                                                 synced_dev, iterations_dev, fa, fb, round_cap,
                                                 static_cast<DevReport*>(report_dev), 1, gate);
  return last_status();
}

extern "C" int bh_intra_sync(const bh_stream* s, int early_exit, int64_t* entries_dev,
                             int64_t* exits_dev, int64_t* counts_dev, uint8_t* synced_dev,
                             int32_t* iterations_dev, void* ws, size_t ws_bytes, void* report_dev,
                             void* cuda_stream) {
  (void)early_exit;  // the final state and iterations do not depend on it (test_sync_decoder.py:34-42)
  return bh_intra_sync_ex(s, nullptr, 0, nullptr, entries_dev, exits_dev, counts_dev, synced_dev,
                          iterations_dev, ws, ws_bytes, report_dev, cuda_stream);
}

// workspace: [2*nsub flags][pad][nseq int64 seeds]
extern "C" int bh_inter_sync_pass(const bh_stream* s, int64_t* entries_dev, int64_t* exits_dev,
                                  int64_t* counts_dev, uint8_t* synced_dev, int32_t* iterations_dev,
                                  void* ws, size_t ws_bytes, void* report_dev, uint64_t* stale_host,
                                  void* cuda_stream) {
  if (bad_stream(s)) return BH_BAD_ARGUMENT;
  uint64_t ns = nsub_of(s), nq = nseq_of(s);
  size_t off = align16(2 * ns);
  if (ws_bytes < off + 8 * nq) return BH_BAD_ARGUMENT;
  int64_t* seeds = reinterpret_cast<int64_t*>(static_cast<char*>(ws) + off);
  DevReport* rep = static_cast<DevReport*>(report_dev);
  if (stale_host) *stale_host = 0;
  if (nq <= 1) return BH_OK;
  cudaStream_t st = S(cuda_stream);
  // reset the stale counter, snapshot seeds, read the count
  unsigned long long zero = 0;
  if (cudaMemcpyAsync(&rep->stale_seams, &zero, sizeof(zero), cudaMemcpyHostToDevice, st) != cudaSuccess)
    return BH_CUDA_ERROR;
  k_seam_check<<<grid_for(nq, 256, 4096), 256, 0, st>>>(entries_dev, exits_dev, nq, s->subseqs_per_seq, seeds, &rep->stale_seams);
  unsigned long long stale = 0;
  if (cudaMemcpyAsync(&stale, &rep->stale_seams, sizeof(stale), cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return BH_CUDA_ERROR;
  if (cudaStreamSynchronize(st) != cudaSuccess) return BH_CUDA_ERROR;
  if (stale_host) *stale_host = stale;
  if (!stale) return BH_OK;
  return bh_intra_sync_ex(s, seeds, 0, nullptr, entries_dev, exits_dev, counts_dev, synced_dev,
                          iterations_dev, ws, ws_bytes, report_dev, cuda_stream);
}

extern "C" int bh_decode_write(const bh_stream* s, const int64_t* entries_dev, const int64_t* counts_dev,
                               const int64_t* oi_dev, const int64_t* seq_ids_dev, uint64_t nseq_ids,
                               uint32_t capacity, uint16_t* out_dev, uint64_t out_len,
                               void* report_dev, void* cuda_stream) {
  if (bad_stream(s) || capacity < 1) return BH_BAD_ARGUMENT;
  uint64_t ns = nsub_of(s), nq = nseq_of(s);
  if (!seq_ids_dev) nseq_ids = nq;
  if (!nseq_ids || !ns) return BH_OK;
  // physical staging never needs more than one sequence's worth of symbols
  uint64_t seq_max = (uint64_t)s->subseq_bits * s->subseqs_per_seq;
  uint64_t phys = capacity < seq_max ? capacity : seq_max;
  uint32_t stride = (uint32_t)((phys + 7) & ~7ull);
  size_t dyn = (size_t)stride * 2 * DW_WARPS;
  if (dyn + 3 * LUT_SIZE * 2 > 227 * 1024) return BH_BAD_ARGUMENT;
  if (dyn > 48 * 1024)
    cudaFuncSetAttribute(k_decode_write, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  unsigned grid = grid_for(nseq_ids, DW_WARPS, (unsigned)sm_count() * 32);
  k_decode_write<<<grid, DW_WARPS * 32, dyn, S(cuda_stream)>>>(
      s->words_dev, s->table_dev, s->max_codes, ns, nq, s->subseqs_per_seq, entries_dev, counts_dev,
      oi_dev, seq_ids_dev, nseq_ids, capacity, stride, out_dev, out_len,
      static_cast<DevReport*>(report_dev), 1, nullptr, nullptr);
  return last_status();
}

extern "C" int bh_check_total(const bh_stream* s, const int64_t* oi_dev, int status_on_mismatch,
                              void* report_dev, void* cuda_stream) {
  k_check_total<<<1, 32, 0, S(cuda_stream)>>>(oi_dev, nsub_of(s), s->symbol_count, status_on_mismatch,
                                               static_cast<DevReport*>(report_dev));
  return last_status();
}

extern "C" int bh_sequence_counts(const bh_stream* s, const int64_t* counts_dev, int64_t* seqc_dev,
                                  void* cuda_stream) {
  uint64_t ns = nsub_of(s), nq = nseq_of(s);
  if (nq) k_seq_counts<<<grid_for(nq, 256, 4096), 256, 0, S(cuda_stream)>>>(counts_dev, ns, nq, s->subseqs_per_seq, seqc_dev);
  return last_status();
}

extern "C" size_t bh_tuner_workspace_bytes(uint64_t nseq, uint32_t t_high) {
  uint64_t tiles = (nseq + TUNE_TILE - 1) / TUNE_TILE;
  return sizeof(uint32_t) * (tiles + 1) * (t_high + 1);
}

extern "C" int bh_tuner_plan(const bh_stream* s, const int64_t* seqc_dev, uint32_t t_high,
                             int64_t* classes_dev, int64_t* freq_dev, int64_t* perm_dev,
                             int64_t* start_dev, void* ws, size_t ws_bytes, void* cuda_stream) {
  if (bad_stream(s) || t_high < 1 || t_high > 255) return BH_BAD_ARGUMENT;
  uint64_t nq = nseq_of(s);
  if (ws_bytes < bh_tuner_workspace_bytes(nq, t_high)) return BH_BAD_ARGUMENT;
  const uint32_t C = t_high + 1;
  cudaStream_t st = S(cuda_stream);
  uint64_t tiles = (nq + TUNE_TILE - 1) / TUNE_TILE;
  uint32_t* hist = static_cast<uint32_t*>(ws);
  if (nq == 0) {
    cudaMemsetAsync(freq_dev, 0, 8 * C, st);
    cudaMemsetAsync(start_dev, 0, 8 * C, st);
    return last_status();
  }
  uint64_t seq_bits = (uint64_t)s->subseq_bits * s->subseqs_per_seq;
  uint64_t last_bits = s->total_bits - (nq - 1) * seq_bits;
  k_tune_classify<<<(unsigned)tiles, TUNE_TILE, C * 4, st>>>(seqc_dev, nq, seq_bits, last_bits,
                                                             s->symbol_width, t_high, classes_dev, hist);
  k_tune_offsets<<<1, 256, 0, st>>>(hist, tiles, t_high, freq_dev, start_dev);
  k_tune_perm<<<(unsigned)tiles, TUNE_TILE, 32 * C * 4, st>>>(classes_dev, nq, t_high, hist, perm_dev);
  return last_status();
}

extern "C" int bh_coarse_decode(const bh_stream* s, const uint64_t* offs_dev, uint64_t chunk,
                                uint16_t* out_dev, void* report_dev, void* cuda_stream) {
  if (bad_stream(s) || chunk == 0) return BH_BAD_ARGUMENT;
  uint64_t n = s->symbol_count;
  if (!n) return BH_OK;
  uint64_t nchunks = (n + chunk - 1) / chunk;
  k_coarse<<<(unsigned)((nchunks + 255) / 256), 256, 0, S(cuda_stream)>>>(
      s->words_dev, s->table_dev, s->max_codes, offs_dev, chunk, n, out_dev,
      static_cast<DevReport*>(report_dev));
  return last_status();
}

extern "C" int bh_decode_write_classes(const bh_stream* s, const int64_t* entries_dev,
                                       const int64_t* counts_dev, const int64_t* oi_dev,
                                       const int64_t* seq_ids_dev, uint64_t nseq_ids, uint32_t capacity,
                                       uint32_t max_capacity, const int64_t* classes_dev,
                                       const uint32_t* caps_dev, uint16_t* out_dev, uint64_t out_len,
                                       void* report_dev, int stats, void* cuda_stream) {
  if (bad_stream(s) || max_capacity < 1 || (!classes_dev && capacity < 1)) return BH_BAD_ARGUMENT;
  uint64_t ns = nsub_of(s), nq = nseq_of(s);
  if (!seq_ids_dev) nseq_ids = nq;
  if (!nseq_ids || !ns) return BH_OK;
  uint64_t seq_max = (uint64_t)s->subseq_bits * s->subseqs_per_seq;
  uint64_t phys = max_capacity < seq_max ? max_capacity : seq_max;
  uint32_t stride = (uint32_t)((phys + 7) & ~7ull);
  size_t dyn = (size_t)stride * 2 * DW_WARPS;
  if (dyn + 3 * LUT_SIZE * 2 > 220 * 1024) return BH_BAD_ARGUMENT;
  if (dyn > 48 * 1024)
    cudaFuncSetAttribute(k_decode_write, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  unsigned grid = grid_for(nseq_ids, DW_WARPS, (unsigned)sm_count() * 32);
  k_decode_write<<<grid, DW_WARPS * 32, dyn, S(cuda_stream)>>>(
      s->words_dev, s->table_dev, s->max_codes, ns, nq, s->subseqs_per_seq, entries_dev, counts_dev,
      oi_dev, seq_ids_dev, nseq_ids, capacity, stride, out_dev, out_len,
      static_cast<DevReport*>(report_dev), stats, classes_dev, caps_dev);
  return last_status();
}

extern "C" int bh_seam_check(const bh_stream* s, const int64_t* entries_dev, const int64_t* exits_dev,
                             int64_t* seeds_dev, unsigned long long* counter_dev, void* cuda_stream) {
  uint64_t nq = nseq_of(s);
  if (nq) k_seam_check<<<grid_for(nq, 256, 4096), 256, 0, S(cuda_stream)>>>(entries_dev, exits_dev, nq,
                                                                          s->subseqs_per_seq, seeds_dev, counter_dev);
  return last_status();
}

// ---------------------------------------------------------------------------
// Ground-truth API on the device: encoder.py:129-159 (oracle_decode) and
// encoder.py:162-188 (mis_sync_decode) as one sequential GPU thread.
// ---------------------------------------------------------------------------
namespace bh {
__global__ void k_sequential(const uint32_t* __restrict__ words, const void* table, uint32_t max_codes,
                             uint64_t start_bit, uint64_t tb, uint64_t n, int mode,
                             uint16_t* __restrict__ out, int64_t* __restrict__ starts,
                             unsigned long long* result) {
  if (threadIdx.x || blockIdx.x) return;
  TableView t = dev_table(table, max_codes);
  uint64_t pos = start_bit, k = 0;
  int status = BH_OK;
  BitReader r;
  r.init(words, pos);
  if (mode == 0) {
    for (; k < n; ++k) {
      if (pos >= tb) { status = BH_TRUNCATED; break; }
      uint32_t e = lookup(t.lut, t, r.peek());
      uint32_t len = (e >> 16) & 0xffu;
      if (!len) { status = BH_INVALID; break; }
      if (pos + len > tb) { status = BH_TRUNCATED; break; }
      out[k] = (uint16_t)e;
      if (starts) starts[k] = (int64_t)pos;
      r.skip(len);
      pos += len;
    }
  } else {
    while (pos < tb) {
      uint32_t e = lookup(t.lut, t, r.peek());
      uint32_t len = (e >> 16) & 0xffu;
      if (!len) { status = BH_INVALID; break; }
      if (pos + len > tb) break;
      out[k++] = (uint16_t)e;
      r.skip(len);
      pos += len;
    }
  }
  result[0] = (unsigned long long)status;
  result[1] = k;
}

// per-subsequence start counts (encoder.py:157-158)
__global__ void k_start_hist(const int64_t* __restrict__ starts, uint64_t n, uint32_t sb,
                             unsigned long long* __restrict__ counts) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    atomicAdd(counts + (uint64_t)starts[i] / sb, 1ull);
}
}  // namespace bh

extern "C" int bh_sequential_decode(const bh_stream* s, uint64_t start_bit, uint64_t n, int mode,
                                    uint16_t* out_dev, int64_t* starts_dev, uint64_t* result_dev,
                                    void* cuda_stream) {
  if (bad_stream(s)) return BH_BAD_ARGUMENT;
  k_sequential<<<1, 32, 0, S(cuda_stream)>>>(s->words_dev, s->table_dev, s->max_codes, start_bit,
                                             s->total_bits, n, mode, out_dev, starts_dev,
                                             reinterpret_cast<unsigned long long*>(result_dev));
  return last_status();
}

extern "C" int bh_start_histogram(const int64_t* starts_dev, uint64_t n, uint32_t subseq_bits,
                                  int64_t* counts_dev, uint64_t nsub, void* cuda_stream) {
  if (cudaMemsetAsync(counts_dev, 0, 8 * nsub, S(cuda_stream)) != cudaSuccess) return BH_CUDA_ERROR;
  if (n) k_start_hist<<<grid_for(n, 256, 4096), 256, 0, S(cuda_stream)>>>(
      starts_dev, n, subseq_bits, reinterpret_cast<unsigned long long*>(counts_dev));
  return last_status();
}

namespace bh {
struct Caps { uint32_t v[256]; };
__global__ void k_fill_caps(uint32_t* __restrict__ dst, Caps caps, uint32_t n) {
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = caps.v[i];
}
}  // namespace bh

// per-class capacities (host array, copied by value through the launch)
extern "C" int bh_fill_caps(uint32_t* caps_dev, const uint32_t* caps_host, uint32_t n, void* cuda_stream) {
  if (n > 256) return BH_BAD_ARGUMENT;
  Caps c;
  for (uint32_t i = 0; i < n; ++i) c.v[i] = caps_host[i];
  k_fill_caps<<<1, 256, 0, S(cuda_stream)>>>(caps_dev, c, n);
  return last_status();
}
