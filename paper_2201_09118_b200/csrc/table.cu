// table.cu -- K1: canonical codebook and two-level decode tables on device.
//
// Canonical numbering restates codebook.py:86-112 (symbols sorted by (length,
// symbol) get consecutive codes, shifting left on every length increase) and
// the per-length first_code / first_index recurrence of codebook.py:209-233.
// Instead of the reference's per-bit first_code loop (kernels.py:35-44) the
// device decodes through:
//   * lut  : 2^11-entry first-level table (symbol, length) in shared memory,
//   * cnt  : 2^11-entry multi-codeword count table (codewords fully inside the
//            11-bit window, bits they consume) for count-only passes,
//   * lj   : left-justified codes in ascending order for long codes (binary
//            search, exact for any prefix-free code -- see common.cuh).
#include "common.cuh"

namespace bh {

__device__ __forceinline__ void table_ptrs(void* blob, uint32_t max_codes, TableHdr*& hdr,
                                           uint32_t*& lut, uint16_t*& cnt, uint32_t*& lj,
                                           uint16_t*& ljsym, uint8_t*& ljlen) {
  TableLayout L(max_codes);
  char* b = static_cast<char*>(blob);
  hdr = reinterpret_cast<TableHdr*>(b);
  lut = reinterpret_cast<uint32_t*>(b + L.lut);
  cnt = reinterpret_cast<uint16_t*>(b + L.cnt);
  lj = reinterpret_cast<uint32_t*>(b + L.lj);
  ljsym = reinterpret_cast<uint16_t*>(b + L.ljsym);
  ljlen = reinterpret_cast<uint8_t*>(b + L.ljlen);
}

// Single CTA (1024 threads): counting sort by (length, symbol), canonical codes.
__global__ void __launch_bounds__(1024) k_canonical(const uint8_t* __restrict__ lengths,
                                                    uint32_t alphabet, void* blob,
                                                    uint32_t max_codes, uint32_t* codes_out) {
  __shared__ uint32_t s_count[33];
  __shared__ unsigned long long s_fc[33];
  __shared__ uint32_t s_fi[33];
  __shared__ uint32_t s_fill[33];
  __shared__ uint32_t s_wcnt[32][33];
  __shared__ int s_bad;
  TableHdr* hdr; uint32_t* lut; uint16_t* cnt; uint32_t* lj; uint16_t* ljsym; uint8_t* ljlen;
  table_ptrs(blob, max_codes, hdr, lut, cnt, lj, ljsym, ljlen);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid < 33) { s_count[tid] = 0; s_fill[tid] = 0; }
  if (tid == 0) s_bad = 0;
  __syncthreads();
  for (uint32_t s = tid; s < alphabet; s += blockDim.x) {
    uint32_t ln = lengths[s];
    if (ln > 32) s_bad = 1;
    else if (ln) atomicAdd(&s_count[ln], 1u);
  }
  __syncthreads();
  if (tid == 0) {
    unsigned long long code = 0;
    uint32_t idx = 0, ml = 0;
    for (int ln = 1; ln <= 32; ++ln) {
      s_fc[ln] = code;
      s_fi[ln] = idx;
      code = (code + s_count[ln]) << 1;
      idx += s_count[ln];
      if (s_count[ln]) ml = ln;
    }
    hdr->kind = 0;
    hdr->max_len = ml;
    hdr->ncodes = idx;
    hdr->lut_bits = LUT_BITS;
    hdr->alphabet = alphabet;
    hdr->status = (s_bad || idx > max_codes) ? BH_BAD_ARGUMENT : BH_OK;
    unsigned long long kraft = 0;
    for (int ln = 1; ln <= 32; ++ln) kraft += (unsigned long long)s_count[ln] << (32 - ln);
    hdr->complete = kraft == (1ull << 32) ? 1u : 0u;
    // canonical limits for the fused kernels' long-code path
    TableLayout L(max_codes);
    unsigned long long* lim = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(blob) + L.lim);
    long long* base = reinterpret_cast<long long*>(reinterpret_cast<char*>(blob) + L.base);
    lim[0] = 0;
    base[0] = 0;
    for (int ln = 1; ln <= 32; ++ln) {
      lim[ln] = (s_fc[ln] + s_count[ln]) << (32 - ln);
      base[ln] = (long long)s_fi[ln] - (long long)s_fc[ln];
    }
  }
  __syncthreads();
  if (hdr->status != BH_OK) return;
  const unsigned lt = (1u << lane) - 1;
  for (uint32_t base = 0; base < alphabet; base += blockDim.x) {
    uint32_t s = base + tid;
    uint32_t ln = s < alphabet ? lengths[s] : 0;
    unsigned peers = __match_any_sync(0xffffffffu, ln);
    uint32_t wrank = __popc(peers & lt);
    if (lane < 33) {}
    for (int i = lane; i < 33; i += 32) s_wcnt[warp][i] = 0;
    __syncwarp();
    if (ln && wrank == 0) s_wcnt[warp][ln] = __popc(peers);
    __syncthreads();
    if (ln) {
      uint32_t r = s_fill[ln] + wrank;
      for (int w = 0; w < warp; ++w) r += s_wcnt[w][ln];
      unsigned long long code = s_fc[ln] + r;
      uint32_t idx = s_fi[ln] + r;
      lj[idx] = (uint32_t)(code << (32 - ln));
      ljsym[idx] = (uint16_t)s;
      ljlen[idx] = (uint8_t)ln;
      if (codes_out) codes_out[s] = (uint32_t)code;
    } else if (codes_out && s < alphabet) {
      codes_out[s] = 0;
    }
    __syncthreads();
    if (tid < 33 && tid > 0) {
      uint32_t add = 0;
      for (int w = 0; w < 32; ++w) add += s_wcnt[w][tid];
      s_fill[tid] += add;
    }
    __syncthreads();
  }
}

// Explicit books: rank every codeword by its left-justified code (codes of a
// prefix-free book are distinct once left-justified).  O(n^2) over a
// shared-memory tile; explicit books are small (container cannot carry them,
// SURVEY A15).
__global__ void k_explicit_rank(const uint32_t* __restrict__ codes, const uint8_t* __restrict__ lens,
                                uint32_t alphabet, void* blob, uint32_t max_codes) {
  TableHdr* hdr; uint32_t* lut; uint16_t* cnt; uint32_t* lj; uint16_t* ljsym; uint8_t* ljlen;
  table_ptrs(blob, max_codes, hdr, lut, cnt, lj, ljsym, ljlen);
  __shared__ uint32_t s_key[1024];
  __shared__ uint8_t s_ok[1024];
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t my_len = i < alphabet ? lens[i] : 0;
  uint32_t my_key = my_len ? (codes[i] << (32 - my_len)) : 0;
  uint32_t rank = 0;
  for (uint32_t base = 0; base < alphabet; base += 1024) {
    uint32_t j = base + threadIdx.x;
    uint32_t l2 = j < alphabet ? lens[j] : 0;
    s_ok[threadIdx.x] = l2 != 0;
    s_key[threadIdx.x] = l2 ? (codes[j] << (32 - l2)) : 0;
    __syncthreads();
    uint32_t lim = min(1024u, alphabet - base);
    if (my_len)
      for (uint32_t k = 0; k < lim; ++k) rank += (s_ok[k] && s_key[k] < my_key) ? 1u : 0u;
    __syncthreads();
  }
  if (my_len && rank < max_codes) {
    lj[rank] = my_key;
    ljsym[rank] = (uint16_t)i;
    ljlen[rank] = (uint8_t)my_len;
  }
}

__global__ void k_explicit_hdr(const uint8_t* __restrict__ lens, uint32_t alphabet, void* blob,
                               uint32_t max_codes) {
  TableHdr* hdr; uint32_t* lut; uint16_t* cnt; uint32_t* lj; uint16_t* ljsym; uint8_t* ljlen;
  table_ptrs(blob, max_codes, hdr, lut, cnt, lj, ljsym, ljlen);
  __shared__ uint32_t s_n, s_ml, s_bad;
  __shared__ unsigned long long s_kraft;
  if (threadIdx.x == 0) { s_n = 0; s_ml = 0; s_bad = 0; s_kraft = 0; }
  __syncthreads();
  for (uint32_t s = threadIdx.x; s < alphabet; s += blockDim.x) {
    uint32_t ln = lens[s];
    if (ln) { atomicAdd(&s_n, 1u); atomicMax(&s_ml, ln); }
    if (ln > 32) s_bad = 1;
    else if (ln) atomicAdd(&s_kraft, 1ull << (32 - ln));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    hdr->kind = 1;
    hdr->max_len = s_ml;
    hdr->ncodes = s_n;
    hdr->lut_bits = LUT_BITS;
    hdr->alphabet = alphabet;
    hdr->status = (s_bad || s_n > max_codes) ? BH_BAD_ARGUMENT : BH_OK;
    hdr->complete = s_kraft == (1ull << 32) ? 1u : 0u;
  }
}

// 8-byte entry of up to three whole codewords (wlut3)
__device__ __forceinline__ uint2 pack3(uint32_t s0, uint32_t s1, uint32_t s2, uint32_t n3, uint32_t l0, uint32_t p3) {
  uint2 e;
  e.x = s0 | (s1 << 16);
  e.y = n3 ? (s2 | (l0 << 16) | (p3 << 24) | ((2 * n3) << 28)) : 0u;
  return e;
}

// wlut3 entry of the D3-bit window v: up to three whole codewords, each read
// from the 12-bit prefix table at its offset (the next 12 bits, zero-filled
// past the window: a codeword that fits inside the window matches the same)
__device__ __forceinline__ uint2 wlut3_entry(uint32_t v, const uint32_t* s_l12) {
  uint32_t p = 0, n = 0, l0 = 0, sy[3] = {0, 0, 0};
#pragma unroll 1
  while (n < 3 && p < (uint32_t)D3) {
    const uint32_t f = s_l12[((v << p) >> (D3 - FB)) & (FB_SIZE - 1)];
    const uint32_t len = (f >> 16) & 0xffu;
    if (len == 0 || p + len > (uint32_t)D3) break;
    if (n == 0) l0 = len;
    sy[n++] = f & 0xffffu;
    p += len;
  }
  return pack3(sy[0], sy[1], sy[2], n, l0, p);
}

// First-level tables from the sorted long-code arrays (one CTA).
__global__ void __launch_bounds__(1024) k_fill_luts(void* blob, uint32_t max_codes) {
  TableHdr* hdr; uint32_t* lut; uint16_t* cnt; uint32_t* lj; uint16_t* ljsym; uint8_t* ljlen;
  table_ptrs(blob, max_codes, hdr, lut, cnt, lj, ljsym, ljlen);
  __shared__ uint32_t s_lut[LUT_SIZE];
  if (hdr->status != BH_OK) return;
  TableView t = table_view(blob, max_codes, hdr->ncodes);
  for (int v = threadIdx.x; v < LUT_SIZE; v += blockDim.x) {
    uint32_t win = (uint32_t)v << (32 - LUT_BITS);
    uint32_t e = slow_lookup(t, win);
    uint32_t len = (e >> 16) & 0xff;
    if (len > (uint32_t)LUT_BITS) e = 0;  // long code: needs more than the window
    s_lut[v] = e;
    lut[v] = e;
  }
  __syncthreads();
  for (int v = threadIdx.x; v < LUT_SIZE; v += blockDim.x) {
    uint32_t pos = 0, n = 0;
    while (pos < (uint32_t)LUT_BITS) {
      uint32_t idx = (uint32_t)((v << pos) & (LUT_SIZE - 1));
      uint32_t e = s_lut[idx];
      uint32_t len = (e >> 16) & 0xff;
      if (len == 0 || pos + len > (uint32_t)LUT_BITS) break;
      pos += len;
      ++n;
    }
    cnt[v] = n ? (uint16_t)(pos | (n << 8)) : (uint16_t)0;
  }
  // tables for the fused kernels
  TableLayout L(max_codes);
  uint32_t* dlut8 = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(blob) + L.dlut8);
  uint8_t* clut8 = reinterpret_cast<uint8_t*>(reinterpret_cast<char*>(blob) + L.clut8);
  uint32_t* lut12 = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(blob) + L.lut12);
  uint16_t* clut12 = reinterpret_cast<uint16_t*>(reinterpret_cast<char*>(blob) + L.clut12);
  __shared__ uint32_t s_l12[FB_SIZE];  // sym | len<<16 of codes <= 12 bits (16 KB)
  for (int v = threadIdx.x; v < FB_SIZE; v += blockDim.x) {
    uint32_t e = slow_lookup(t, (uint32_t)v << (32 - FB));
    const uint32_t len = (e >> 16) & 0xff;
    lut12[v] = len <= (uint32_t)FB ? e : 0u;
    s_l12[v] = len <= (uint32_t)FB ? e : 0u;
    reinterpret_cast<uint8_t*>(reinterpret_cast<char*>(blob) + L.len12)[v] = (uint8_t)(len <= (uint32_t)FB ? len : 0u);
  }
  __syncthreads();
  // up to six whole codewords of the 12-bit window (wide decode table)
  uint4* wlut12 = reinterpret_cast<uint4*>(reinterpret_cast<char*>(blob) + L.wlut12);
  for (int v = threadIdx.x; v < FB_SIZE; v += blockDim.x) {
    uint32_t p6 = 0, n6 = 0, sy[6] = {0, 0, 0, 0, 0, 0}, l0 = 0;
    while (n6 < 6 && p6 < (uint32_t)FB) {
      const uint32_t f = s_l12[((uint32_t)v << p6) & (FB_SIZE - 1)];
      const uint32_t len = (f >> 16) & 0xff;
      if (len == 0 || p6 + len > (uint32_t)FB) break;
      if (n6 == 0) l0 = len;
      sy[n6++] = f & 0xffff;
      p6 += len;
    }
    uint4 wl;
    wl.x = sy[0] | (sy[1] << 16);
    wl.y = sy[2] | (sy[3] << 16);
    wl.z = sy[4] | (sy[5] << 16);
    wl.w = n6 ? (p6 | (n6 << 4) | (l0 << 16) | ((2 * n6) << 28)) : 0u;
    wlut12[v] = wl;
  }
  uint2* wlut3 = reinterpret_cast<uint2*>(reinterpret_cast<char*>(blob) + L.wlut3);
  for (uint32_t v = threadIdx.x; v < (uint32_t)D3_SIZE; v += blockDim.x) wlut3[v] = wlut3_entry(v, s_l12);
  uint8_t* cwin = reinterpret_cast<uint8_t*>(reinterpret_cast<char*>(blob) + L.cwin);
  __shared__ uint32_t s_minl;
  if (threadIdx.x == 0) s_minl = 64;
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < t.ncodes; i += blockDim.x) atomicMin(&s_minl, (uint32_t)t.ljlen[i]);
  __syncthreads();
  const bool buildcw = s_minl >= 4 && s_minl != 64;
  for (int v = threadIdx.x; v < CW_SIZE; v += blockDim.x) {
    const uint32_t w0 = (uint32_t)v << (32 - CW);
    uint32_t pos = 0, n = 0;
    while (buildcw && pos < (uint32_t)CW) {
      uint32_t len = (s_l12[(w0 << pos) >> (32 - FB)] >> 16) & 0xffu;
      if (!len) len = (slow_lookup(t, w0 << pos) >> 16) & 0xffu;
      if (len == 0 || pos + len > (uint32_t)CW) break;
      pos += len;
      ++n;
    }
    cwin[v] = (uint8_t)(n | (pos << 3));
  }
  uint16_t* s_len12 = reinterpret_cast<uint16_t*>(s_lut);  // 4096 lengths (8 KB)
  for (int v = threadIdx.x; v < FB_SIZE; v += blockDim.x) s_len12[v] = (uint16_t)((s_l12[v] >> 16) & 0xff);
  __syncthreads();
  // count table: every whole codeword of the 12-bit window (zero fill past the
  // window cannot change a match of a codeword that lies inside it)
  for (int v = threadIdx.x; v < FB_SIZE; v += blockDim.x) {
    uint32_t pos = 0, starts = 0;
    while (pos < (uint32_t)FB) {
      const uint32_t len = s_len12[((uint32_t)v << pos) & (FB_SIZE - 1)];
      if (len == 0 || pos + len > (uint32_t)FB) break;
      starts |= 1u << pos;
      pos += len;
    }
    clut12[v] = (uint16_t)(starts | (pos << 12));
  }
  for (int v = threadIdx.x; v < 256; v += blockDim.x) {
    uint32_t e = slow_lookup(t, (uint32_t)v << 24);
    dlut8[v] = ((e >> 16) & 0xff) <= 8u ? e : 0u;
    uint32_t pos = 0, n = 0;
    while (pos < 8) {
      uint32_t w = ((uint32_t)v << 24) << pos;  // zero-filled past the window
      uint32_t f = slow_lookup(t, w);
      uint32_t len = (f >> 16) & 0xff;
      if (len == 0 || pos + len > 8) break;
      pos += len;
      ++n;
    }
    clut8[v] = n ? (uint8_t)((n << 3) | (pos - 1)) : (uint8_t)0;
    // up to six whole codewords of the 8-bit window, for the decode-write pass
    uint32_t p6 = 0, n6 = 0, sy[6] = {0, 0, 0, 0, 0, 0}, l0 = 0;
    while (n6 < 6 && p6 < 8) {
      uint32_t f = slow_lookup(t, ((uint32_t)v << 24) << p6);
      uint32_t len = (f >> 16) & 0xff;
      if (len == 0 || p6 + len > 8) break;
      if (n6 == 0) l0 = len;
      sy[n6++] = f & 0xffff;
      p6 += len;
    }
    uint4 wl;
    wl.x = sy[0] | (sy[1] << 16);
    wl.y = sy[2] | (sy[3] << 16);
    wl.z = sy[4] | (sy[5] << 16);
    wl.w = n6 ? (p6 | (n6 << 4) | (n << 8) | (pos << 12) | (l0 << 16) | ((2 * n6) << 28)) : 0u;
    reinterpret_cast<uint4*>(reinterpret_cast<char*>(blob) + L.wlut8)[v] = wl;
  }
}


// ---------------------------------------------------------------------------
// K1 fast path for canonical books (bh_table_build): ONE launch of a few CTAs.
// Every CTA rebuilds the canonical order of the <= 4096 codes of length <= 12
// in shared memory from the length bytes (codebook.py:86-112: counting sort by
// (length, symbol), first_code/first_index per length, codebook.py:209-233),
// then fills its slice of the direct tables.  A codeword is found from a
// 32-bit window by the canonical limits (the first length whose left-justified
// limit exceeds the window, a 5-step search over 33 shared values) and its
// symbol by base[len] + code -- no per-entry global binary search.
// ---------------------------------------------------------------------------
constexpr int K1_THREADS = 1024;  // 32 warps: one per code length in the rank scan
constexpr int K1_GRID = 16;
constexpr uint32_t K1_LENS = 4096;

struct CanonSmem {
  unsigned long long lim[33];
  long long base[33];
  uint32_t count[33];
  uint32_t fill[33];
  uint32_t wcnt[K1_THREADS / 32][33];
  uint32_t wpre[K1_THREADS / 32][33];
  uint16_t sym[FB_SIZE];  // canonical order of the codes of length <= 12
  uint32_t minl;          // shortest code length
  uint32_t l12[FB_SIZE];  // sym | len<<16 of the codeword at each 12-bit prefix (codes <= 12 bits)
  uint8_t lens[K1_LENS];  // the first K1_LENS length bytes (read once from global)
  int bad;
};

// sym | len<<16 of the codeword at the front of `win`; len only (sym 0) for
// codes longer than 12 bits; 0 when no codeword matches (incomplete book)
__device__ __forceinline__ uint32_t canon_one(const CanonSmem& S, uint32_t win) {
  if ((unsigned long long)win >= S.lim[32]) return 0u;
  uint32_t lo = 1, hi = 32;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if ((unsigned long long)win < S.lim[mid]) hi = mid; else lo = mid + 1;
  }
  if (lo > (uint32_t)FB) return lo << 16;
  const long long idx = S.base[lo] + (long long)(win >> (32 - lo));
  return (uint32_t)S.sym[idx] | (lo << 16);
}

// symbol k (0..5) of a multi-symbol entry into its halfword of x|y|z
__device__ __forceinline__ void pack6(uint32_t& x, uint32_t& y, uint32_t& z, uint32_t k, uint32_t sym) {
  const uint32_t v = sym << ((k & 1u) * 16);
  if (k < 2) x |= v; else if (k < 4) y |= v; else z |= v;
}

#ifndef BH_K1_STOP
#define BH_K1_STOP 9  // timing experiment only: return after stage N (wrong tables below 9)
#endif
#ifdef BH_K1_STAMPS
__device__ unsigned long long g_k1_stamps[8];
#define K1ST(k) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_k1_stamps[k] = global_ns(); } while (0)
#else
#define K1ST(k) do { } while (0)
#endif

__global__ void __launch_bounds__(K1_THREADS) k_table_canon(const uint8_t* __restrict__ lengths, uint32_t alphabet,
                                                           void* blob, uint32_t max_codes) {
  __shared__ CanonSmem S;
  // the decode kernel that follows may launch now (its CTAs wait for this
  // grid's completion before reading the tables)
  asm volatile("griddepcontrol.launch_dependents;");
  K1ST(7);
  TableHdr* hdr; uint32_t* lut; uint16_t* cnt; uint32_t* lj; uint16_t* ljsym; uint8_t* ljlen;
  table_ptrs(blob, max_codes, hdr, lut, cnt, lj, ljsym, ljlen);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t G = gridDim.x, cta = blockIdx.x;
  if (tid < 33) { S.count[tid] = 0; S.fill[tid] = 0; }
  if (tid == 0) S.bad = 0;
  __syncthreads();
  K1ST(0);
  for (uint32_t s = tid; s < alphabet; s += K1_THREADS) {
    const uint32_t ln = lengths[s];
    if (s < K1_LENS) S.lens[s] = (uint8_t)ln;
    if (ln > 32) S.bad = 1;
    else if (ln) atomicAdd(&S.count[ln], 1u);
  }
  __syncthreads();
  K1ST(1);
  if (BH_K1_STOP <= 1) return;
  // first_code / first_index per length (codebook.py:209-233) as one warp scan:
  // lane ln-1 holds count c and its left-justified Kraft share d = c << (32-ln);
  // the exclusive prefix of d is first_code << (32-ln) exactly, and its
  // inclusive prefix the canonical limit lim[ln] = (first_code + c) << (32-ln)
  if (warp == 0) {
    const uint32_t ln = lane + 1;
    const uint32_t c = S.count[ln];
    const unsigned long long d = (unsigned long long)c << (32 - ln);
    unsigned long long P = d;
    uint32_t I = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, P, o);
      const uint32_t z = __shfl_up_sync(0xffffffffu, I, o);
      if (lane >= o) { P += y; I += z; }
    }
    const unsigned long long code = (P - d) >> (32 - ln);
    S.lim[ln] = P;
    S.base[ln] = (long long)(I - c) - (long long)code;
    S.fill[ln] = I - c;  // first_index: rank base of the length
    const uint32_t ncodes = __shfl_sync(0xffffffffu, I, 31);
    const unsigned long long kraft = __shfl_sync(0xffffffffu, P, 31);
    const unsigned used = __ballot_sync(0xffffffffu, c != 0);
    const uint32_t ml = used ? 32 - __clz(used) : 0;
    if (lane == 0) {
      S.minl = used ? __ffs(used) : 0;
      S.lim[0] = 0;
      S.base[0] = 0;
      if (ncodes > max_codes) S.bad = 1;
    }
    __syncwarp();
    if (cta == 0) {
      TableLayout L(max_codes);
      unsigned long long* glim = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(blob) + L.lim);
      long long* gbase = reinterpret_cast<long long*>(reinterpret_cast<char*>(blob) + L.base);
      glim[ln] = P;
      gbase[ln] = S.base[ln];
      if (lane == 0) {
        glim[0] = 0;
        gbase[0] = 0;
        hdr->kind = 0;
        hdr->max_len = ml;
        hdr->ncodes = ncodes;
        hdr->lut_bits = LUT_BITS;
        hdr->alphabet = alphabet;
        hdr->status = S.bad ? BH_BAD_ARGUMENT : BH_OK;
        hdr->complete = kraft == (1ull << 32) ? 1u : 0u;
      }
    }
  }
  __syncthreads();
  K1ST(2);
  if (S.bad || BH_K1_STOP <= 2) return;
  // ranks: counting sort by (length, symbol).  Per 1024-symbol block: a
  // symbol's rank among its warp's peers (match_any), the peers in earlier
  // warps (one warp per length scans the 32 warp counts), and S.fill[ln],
  // the symbols of that length in earlier blocks.
  const unsigned lt = (1u << lane) - 1;
  for (uint32_t b0 = 0; b0 < alphabet; b0 += K1_THREADS) {
    const uint32_t s = b0 + tid;
    const uint32_t ln = s < alphabet ? (s < K1_LENS ? (uint32_t)S.lens[s] : (uint32_t)lengths[s]) : 0u;
    const unsigned peers = __match_any_sync(0xffffffffu, ln);
    const uint32_t wrank = __popc(peers & lt);
    for (int i = lane; i < 33; i += 32) S.wcnt[warp][i] = 0;
    __syncwarp();
    if (ln && wrank == 0) S.wcnt[warp][ln] = __popc(peers);
    __syncthreads();
    {  // warp v scans the per-warp counts of length v + 1
      const uint32_t lv = warp + 1;
      const uint32_t v = S.wcnt[lane][lv];
      uint32_t x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      S.wpre[lane][lv] = S.fill[lv] + x - v;
      __syncwarp();
      if (lane == 31) S.fill[lv] += x;
    }
    __syncthreads();
    if (ln) {
      const uint32_t r = S.wpre[warp][ln] + wrank;
      if (ln <= (uint32_t)FB && r < FB_SIZE) S.sym[r] = (uint16_t)s;
      // the global long-code arrays: one CTA per 1024-symbol block
      if ((b0 / K1_THREADS) % G == cta) {
        const long long code = (long long)r - S.base[ln];
        lj[r] = (uint32_t)((unsigned long long)code << (32 - ln));
        ljsym[r] = (uint16_t)s;
        ljlen[r] = (uint8_t)ln;
      }
    }
    __syncthreads();
  K1ST(3);
  }
  if (BH_K1_STOP <= 3) return;
  // every codeword of <= 12 bits by its 12-bit prefix, in every CTA; the
  // direct tables then walk windows through it.  The length at a prefix is 1
  // + the number of limits at or below it (the limits of lengths 1..12 held
  // in registers, clamped to 32 bits: a prefix window's low 20 bits are zero,
  // so it never reaches 0xffffffff) -- twelve independent compares instead
  // of a dependent limit search
  {
    uint32_t lc[FB];
#pragma unroll
    for (int k = 0; k < FB; ++k) {
      const unsigned long long l = S.lim[k + 1];
      lc[k] = l > 0xffffffffull ? 0xffffffffu : (uint32_t)l;
    }
    for (uint32_t v = tid; v < FB_SIZE; v += K1_THREADS) {
      const uint32_t w = v << (32 - FB);
      uint32_t ln = 1;
#pragma unroll
      for (int k = 0; k < FB; ++k) ln += w >= lc[k] ? 1u : 0u;
      uint32_t e = 0;
      if (ln <= (uint32_t)FB) {
        const long long idx = S.base[ln] + (long long)(w >> (32 - ln));
        e = (uint32_t)S.sym[idx] | (ln << 16);
      }
      S.l12[v] = e;
    }
  }
  __syncthreads();
  K1ST(4);
  if (BH_K1_STOP <= 4) return;
  // direct tables: 12-bit (lut12, clut12, wlut12), 11-bit (lut, cnt)
  // and 8-bit (dlut8, clut8, wlut8) entries spread over every thread of the
  // grid.  A codeword at offset pos of a W-bit window v is S.l12 of the 12
  // bits (v << (12 - W + pos)), zero-filled: it lies inside the window when
  // pos + len <= W (zero fill past the window cannot change such a match).
  TableLayout L(max_codes);
  char* B = static_cast<char*>(blob);
  uint32_t* lut12 = reinterpret_cast<uint32_t*>(B + L.lut12);
  uint16_t* clut12 = reinterpret_cast<uint16_t*>(B + L.clut12);
  uint4* wlut12 = reinterpret_cast<uint4*>(B + L.wlut12);
  uint32_t* dlut8 = reinterpret_cast<uint32_t*>(B + L.dlut8);
  uint8_t* clut8 = reinterpret_cast<uint8_t*>(B + L.clut8);
  uint4* wlut8 = reinterpret_cast<uint4*>(B + L.wlut8);
  constexpr uint32_t N12 = FB_SIZE, N11 = LUT_SIZE, N8 = 256;
  // 15-bit count table (whole codewords of the window): codes up to 12 bits
  // from the prefix table, longer ones by the limit search
  // (built for books whose codes are all >= 4 bits -- the only ones the
  // fused kernel counts with it -- and all zero, "use the 12-bit table",
  // otherwise)
  K1ST(5);
  if (BH_K1_STOP == 5) return;
  uint8_t* cwin = reinterpret_cast<uint8_t*>(B + L.cwin);
  const bool buildcw = S.minl >= 4;
  for (uint32_t v = cta * K1_THREADS + tid; v < (uint32_t)CW_SIZE; v += G * K1_THREADS) {
    const uint32_t w0 = v << (32 - CW);
    uint32_t pos = 0, n = 0;
    while (buildcw && pos < (uint32_t)CW) {
      uint32_t len = (S.l12[(w0 << pos) >> (32 - FB)] >> 16) & 0xffu;
      if (!len) len = (canon_one(S, w0 << pos) >> 16) & 0xffu;  // > 12 bits (or no codeword)
      if (len == 0 || pos + len > (uint32_t)CW) break;
      pos += len;
      ++n;
    }
    cwin[v] = (uint8_t)(n | (pos << 3));
  }
  if (BH_K1_STOP == 6) return;
  uint2* wlut3 = reinterpret_cast<uint2*>(B + L.wlut3);
  // wlut3 and the direct tables share one index space cut into G equal
  // contiguous slices, so every CTA (not only the first few) takes one and a
  // thread at most about one walk
  constexpr uint32_t NW3 = D3_SIZE, NALL = D3_SIZE + N12 + N11 + N8;
  const uint32_t per = (NALL + G - 1) / G;
  const uint32_t s0 = cta * per, s1 = min(s0 + per, NALL);
  for (uint32_t idx = s0 + tid; idx < s1; idx += K1_THREADS) {
    if (idx < NW3) {
      wlut3[idx] = wlut3_entry(idx, S.l12);
      continue;
    }
    const uint32_t it = idx - NW3;
    const uint32_t W = it < N12 ? (uint32_t)FB : it < N12 + N11 ? (uint32_t)LUT_BITS : 8u;
    const uint32_t v = it < N12 ? it : it < N12 + N11 ? it - N12 : it - N12 - N11;
    const uint32_t v12 = v << (FB - W);
    const uint32_t e0 = S.l12[v12];
    // every whole codeword of the window: start mask, end, count; the first
    // six also for the multi-symbol decode tables
    uint32_t pos = 0, starts = 0, n = 0, n6 = 0, l0 = 0, p6 = 0, sx = 0, sy = 0, sz = 0;
    while (pos < W) {
      const uint32_t e = pos ? S.l12[(v12 << pos) & (FB_SIZE - 1)] : e0;
      const uint32_t len = (e >> 16) & 0xffu;
      if (len == 0 || pos + len > W) break;
      starts |= 1u << pos;
      if (n6 < 6) {
        if (n6 == 0) l0 = len;
        pack6(sx, sy, sz, n6++, e & 0xffffu);
        p6 = pos + len;
      }
      pos += len;
      ++n;
    }
    const uint32_t first = ((e0 >> 16) & 0xffu) <= W ? e0 : 0u;
    uint4 wl;
    wl.x = sx;
    wl.y = sy;
    wl.z = sz;
    if (it < N12) {
      lut12[v] = first;
      reinterpret_cast<uint8_t*>(B + L.len12)[v] = (uint8_t)((first >> 16) & 0xffu);
      clut12[v] = (uint16_t)(starts | (pos << 12));
      wl.w = n6 ? (p6 | (n6 << 4) | (l0 << 16) | ((2 * n6) << 28)) : 0u;
      wlut12[v] = wl;
    } else if (it < N12 + N11) {
      lut[v] = first;
      cnt[v] = n ? (uint16_t)(pos | (n << 8)) : (uint16_t)0;
    } else {
      dlut8[v] = first;
      clut8[v] = n ? (uint8_t)((n << 3) | (pos - 1)) : (uint8_t)0;
      wl.w = n6 ? (p6 | (n6 << 4) | (n << 8) | (pos << 12) | (l0 << 16) | ((2 * n6) << 28)) : 0u;
      wlut8[v] = wl;
    }
  }
  K1ST(6);
}

}  // namespace bh

using namespace bh;

static int cuda_status(cudaError_t e) { return e == cudaSuccess ? BH_OK : BH_CUDA_ERROR; }

extern "C" size_t bh_table_bytes(uint32_t max_codes) { return TableLayout(max_codes).total; }

#ifdef BH_K1_STAMPS
extern "C" int bh_debug_k1_stamps(unsigned long long* host8) {
  return cudaMemcpyFromSymbol(host8, bh::g_k1_stamps, 64) == cudaSuccess ? BH_OK : BH_CUDA_ERROR;
}
#endif

extern "C" int bh_table_build(const uint8_t* lengths_dev, uint32_t alphabet, void* table_dev,
                              uint32_t max_codes, void* cuda_stream) {
  if (!table_dev || (alphabet && !lengths_dev) || alphabet > 65536u || max_codes > 65536u)
    return BH_BAD_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  static const int grid = [] {
    const char* e = getenv("BH_K1_GRID");  // tuning knob
    const int g = e && *e ? atoi(e) : 0;
    return g > 0 && g <= 148 ? g : K1_GRID;
  }();
  k_table_canon<<<grid, K1_THREADS, 0, st>>>(lengths_dev, alphabet, table_dev, max_codes);
  return cuda_status(cudaGetLastError());
}

extern "C" int bh_canonical_codes(const uint8_t* lengths_dev, uint32_t alphabet, uint32_t* codes_dev,
                                  void* cuda_stream) {
  if (!codes_dev || alphabet > 65536u) return BH_BAD_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  // scratch blob sized for the full alphabet
  void* blob = nullptr;
  size_t bytes = TableLayout(alphabet).total;
  if (cudaMallocAsync(&blob, bytes, st) != cudaSuccess) return BH_CUDA_ERROR;
  k_canonical<<<1, 1024, 0, st>>>(lengths_dev, alphabet, blob, alphabet, codes_dev);
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(blob, st);
  return cuda_status(e);
}

extern "C" int bh_table_build_explicit(const uint32_t* codes_dev, const uint8_t* lens_dev,
                                       uint32_t alphabet, void* table_dev, uint32_t max_codes,
                                       void* cuda_stream) {
  if (!table_dev || alphabet > 65536u || max_codes > 65536u) return BH_BAD_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  k_explicit_hdr<<<1, 1024, 0, st>>>(lens_dev, alphabet, table_dev, max_codes);
  if (alphabet) {
    uint32_t grid = (alphabet + 1023) / 1024;
    k_explicit_rank<<<grid, 1024, 0, st>>>(codes_dev, lens_dev, alphabet, table_dev, max_codes);
  }
  k_fill_luts<<<1, 1024, 0, st>>>(table_dev, max_codes);
  return cuda_status(cudaGetLastError());
}
