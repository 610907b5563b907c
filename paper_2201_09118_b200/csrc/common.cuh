// common.cuh -- shared device code for the B200 Huffman decode path.
//
// Bitstream contract (reference bitstream.py:1-11): the payload is
// one MSB-first stream of 32-bit words (any reference unit width concatenates to
// this), zero padded by >= BH_WORD_PAD words so 64-bit windows never fault and
// reads past the payload return zero bits exactly like kernels.py:30-31.
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/b200huff.h"

namespace bh {

// SM count of the calling thread's current device, cached per device
// (thread-safe; 148 if the query fails)
inline int device_sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n <= 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

constexpr int LUT_BITS = 11;                 // first-level window (2^11 entries)
constexpr int LUT_SIZE = 1 << LUT_BITS;
constexpr int TABLE_HDR_BYTES = 64;

// Table blob layout (device), built by table.cu:
//   [0,64)           TableHdr
//   lut   u32[2^LB]  sym | len<<16 ; len 0 => long code or invalid prefix
//   cnt   u16[2^LB]  bits | ncode<<8 ; codewords fully inside the LB-bit window
//   lj    u32[ncodes] left-justified codes, ascending (canonical order for
//                     canonical books; sorted for explicit books)
//   ljsym u16[ncodes]
//   ljlen u8 [ncodes]
struct TableHdr {
  uint32_t kind;      // 0 canonical, 1 explicit
  uint32_t max_len;
  uint32_t ncodes;
  uint32_t lut_bits;
  uint32_t alphabet;
  uint32_t status;    // BH_OK or build error
  uint32_t complete;  // Kraft sum == 1: every bit pattern decodes
  uint32_t pad[9];
};

// Fused-kernel tables:
//   dlut8 u32[256]   next 8 bits -> sym | len<<16 for codes of <= 8 bits, else 0
//   wlut8 uint4[256] next 8 bits -> up to 6 whole codewords for decoding plus
//                    the count of every whole codeword for counting:
//                    x = s0 | s1<<16, y = s2 | s3<<16, z = s4 | s5<<16,
//                    w = bits | n<<4 | ncount<<8 | cbits<<12 | len0<<16 | 2n<<28
//                    (n symbols in `bits` bits; ncount whole codewords in
//                    cbits bits; w == 0: the first code is longer than 8 bits)
//   clut8 u8[256]    next 8 bits -> (ncode<<3) | (bits-1) over every whole
//                    codeword inside the 8 bits, 0 if the first one is longer
//   lut12 u32[4096]  next 12 bits -> sym | len<<16 for codes of <= 12 bits, else 0
//   wlut12 uint4[4096] next 12 bits -> up to 6 whole codewords, wlut8's format
//                    (the fused kernels' decode table for long-code books)
//   wlut3 uint2[8192] next 13 bits -> up to 3 whole codewords in 8 bytes (the
//                    fused kernels' decode table for books whose codes are all
//                    >= 4 bits, so no 13-bit window holds more than three):
//                    x = s0 | s1<<16, y = s2 | len0<<16 | bits<<24 | 2n<<28
//                    (y == 0: the first code is longer than 12 bits or ends
//                    past the window)
//   cwin  u8[65536]  next 16 bits -> n | bits<<3 over every whole codeword of
//                    the window (n <= 4, bits <= 16); 0 if the first one is
//                    longer (the count phase of the long-code fused decoders;
//                    built for books whose codes are all >= 4 bits)
//   len12 u8[4096]   next 12 bits -> length of the first codeword if <= 12 bits, else 0
//                    (the self-sync decoders' per-codeword resynchronization walk)
//   clut12 u16[4096] next 12 bits -> starts | bits<<12 over every whole codeword
//                    inside the 12 bits (count pass): bit i of `starts` is set
//                    when a codeword starts at offset i, `bits` is where the
//                    last whole one ends; 0 if the first code is longer
//   lim   u64[33]    canonical left-justified limit per length
//   base  i64[33]    first_index - first_code per length
// The kernel replicates dlut8/clut8 once per lane ("bank-private": lane l only
// ever touches shared-memory bank l), so table lookups never conflict.
constexpr int FB = 12;
constexpr int FB_SIZE = 1 << FB;
constexpr int D3 = 13;  // window of the three-codeword decode table (wlut3)
constexpr int D3_SIZE = 1 << D3;
constexpr int CW = 16;  // window of the count table of the long-code fused path (cwin)
constexpr int CW_SIZE = 1 << CW;

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

struct TableLayout {
  size_t lut, cnt, dlut8, clut8, wlut8, lut12, clut12, wlut12, wlut3, cwin, len12, lim, base, lj, ljsym, ljlen, total;
  __host__ __device__ explicit TableLayout(uint32_t max_codes) {
    lut = TABLE_HDR_BYTES;
    cnt = lut + sizeof(uint32_t) * LUT_SIZE;
    dlut8 = align16(cnt + sizeof(uint16_t) * LUT_SIZE);
    clut8 = dlut8 + 4 * 256;
    wlut8 = align16(clut8 + 256);
    lut12 = align16(wlut8 + 16 * 256);
    clut12 = lut12 + 4 * (size_t)FB_SIZE;
    wlut12 = align16(clut12 + 2 * (size_t)FB_SIZE);
    wlut3 = align16(wlut12 + 16 * (size_t)FB_SIZE);
    cwin = align16(wlut3 + 8 * (size_t)D3_SIZE);
    len12 = align16(cwin + (size_t)CW_SIZE);
    lim = align16(len12 + (size_t)FB_SIZE);
    base = lim + 8 * 33;
    lj = align16(base + 8 * 33);
    ljsym = align16(lj + sizeof(uint32_t) * (size_t)max_codes);
    ljlen = align16(ljsym + sizeof(uint16_t) * (size_t)max_codes);
    total = align16(ljlen + (size_t)max_codes);
  }
};

struct TableView {
  const TableHdr* hdr;
  const uint32_t* lut;
  const uint16_t* cnt;
  const uint32_t* lj;
  const uint16_t* ljsym;
  const uint8_t* ljlen;
  uint32_t ncodes;
};

__host__ __device__ inline TableView table_view(const void* blob, uint32_t max_codes, uint32_t ncodes) {
  TableLayout L(max_codes);
  const char* b = static_cast<const char*>(blob);
  TableView t;
  t.hdr = reinterpret_cast<const TableHdr*>(b);
  t.lut = reinterpret_cast<const uint32_t*>(b + L.lut);
  t.cnt = reinterpret_cast<const uint16_t*>(b + L.cnt);
  t.lj = reinterpret_cast<const uint32_t*>(b + L.lj);
  t.ljsym = reinterpret_cast<const uint16_t*>(b + L.ljsym);
  t.ljlen = reinterpret_cast<const uint8_t*>(b + L.ljlen);
  t.ncodes = ncodes;
  return t;
}

// Long-code / invalid-prefix path: the matching codeword is the largest
// left-justified code <= win, provided it is a prefix of win (prefix-freeness
// makes this exact for canonical and explicit books alike; equivalent to the
// bit-serial match of kernels.py:35-44 and the trie walk of _dispatch.py:34-47).
// Returns sym | len<<16, or 0 when no codeword matches (ERR_INVALID).
__device__ __forceinline__ uint32_t slow_lookup(const TableView& t, uint32_t win) {
  uint32_t lo = 0, hi = t.ncodes;
  if (hi == 0 || __ldg(t.lj) > win) return 0;
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (__ldg(t.lj + mid) <= win) lo = mid; else hi = mid;
  }
  uint32_t len = __ldg(t.ljlen + lo);
  uint32_t code = __ldg(t.lj + lo);
  if (((win ^ code) >> (32 - len)) != 0) return 0;
  return (uint32_t)__ldg(t.ljsym + lo) | (len << 16);
}

// 64-bit MSB-first bit buffer over the word stream.  peek() returns the next
// 32 bits; skip(n<=32) consumes.  Invariant: avail >= 32 after every call.
struct BitReader {
  const uint32_t* __restrict__ w;
  uint64_t buf;
  uint64_t next;
  uint32_t avail;

  __device__ __forceinline__ void init(const uint32_t* words, uint64_t pos) {
    w = words;
    uint64_t wi = pos >> 5;
    uint32_t off = (uint32_t)(pos & 31);
    uint64_t a = ((uint64_t)__ldg(w + wi) << 32) | __ldg(w + wi + 1);
    buf = a << off;
    avail = 64 - off;
    next = wi + 2;
    if (avail < 32) {  // cannot happen (off <= 31) but keep the invariant explicit
      buf |= (uint64_t)__ldg(w + next) << (32 - avail);
      ++next;
      avail += 32;
    }
  }
  __device__ __forceinline__ uint32_t peek() const { return (uint32_t)(buf >> 32); }
  __device__ __forceinline__ void skip(uint32_t n) {
    buf <<= n;
    avail -= n;
    if (avail < 32) {
      buf |= (uint64_t)__ldg(w + next) << (32 - avail);
      ++next;
      avail += 32;
    }
  }
};

// One codeword: returns sym | len<<16 or 0 (invalid).
__device__ __forceinline__ uint32_t lookup(const uint32_t* s_lut, const TableView& t, uint32_t win) {
  uint32_t e = s_lut[win >> (32 - LUT_BITS)];
  if ((e >> 16) == 0) e = slow_lookup(t, win);
  return e;
}

// Count codewords starting in [pos, stop) (stop already clipped to total_bits),
// advancing pos to the exit (first codeword start >= stop).  Same semantics as
// kernels.py:47-76 for one slot.  Returns false on an unmatched pattern.
__device__ __forceinline__ bool count_window(BitReader& r, uint64_t& pos, uint64_t stop,
                                             const uint32_t* s_lut, const uint16_t* s_cnt,
                                             const TableView& t, uint32_t& n) {
  while (pos < stop) {
    uint32_t win = r.peek();
    if (stop - pos >= (uint64_t)LUT_BITS) {
      uint32_t c = s_cnt[win >> (32 - LUT_BITS)];
      if (c) {
        uint32_t b = c & 0xffu;
        n += c >> 8;
        r.skip(b);
        pos += b;
        continue;
      }
    }
    uint32_t e = lookup(s_lut, t, win);
    uint32_t len = (e >> 16) & 0xffu;
    if (len == 0) return false;
    r.skip(len);
    pos += len;
    ++n;
  }
  return true;
}

// Load the first-level tables of a table blob into shared memory (whole CTA).
__device__ __forceinline__ void load_luts(const TableView& t, uint32_t* s_lut, uint16_t* s_cnt) {
  const uint4* src = reinterpret_cast<const uint4*>(t.lut);
  uint4* dst = reinterpret_cast<uint4*>(s_lut);
  for (int i = threadIdx.x; i < LUT_SIZE / 4; i += blockDim.x) dst[i] = __ldg(src + i);
  const uint4* src2 = reinterpret_cast<const uint4*>(t.cnt);
  uint4* dst2 = reinterpret_cast<uint4*>(s_cnt);
  for (int i = threadIdx.x; i < LUT_SIZE / 8; i += blockDim.x) dst2[i] = __ldg(src2 + i);
}

// Device-side report (mirrors bh_report; fields updated atomically).
struct DevReport {
  int32_t status;
  int32_t pad0;
  unsigned long long fail_slot;     // min failing slot (atomicMin), ~0 when none
  unsigned long long bits_sync;
  unsigned long long bits_count;
  unsigned long long bits_write;
  unsigned long long write_rounds;
  unsigned long long staged_slots;
  unsigned long long bypass_slots;
  unsigned long long total_symbols;
  unsigned long long stale_seams;   // seams still stale at the last check
  unsigned long long seam_passes;   // seam passes that re-seeded something
  unsigned long long repair_needed; // fused sync: seam speculation failed somewhere
  unsigned long long pad[4];
  unsigned long long phase_ns[6];   // phase boundaries (bh_report.phase_ns)
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Host side: stamp phase boundary k of the staged pipeline (stream-ordered).
int stamp_phase(void* report_dev, int k, cudaStream_t st);

// Host-side phase profiler (abi.cu): when enabled, every decoder phase is
// bracketed by CUDA events on the launching stream (bh_profile_enable /
// bh_profile_read); costs nothing when disabled.
void prof_mark(cudaStream_t st, const char* phase);

__device__ __forceinline__ void report_error(DevReport* rep, int status, uint64_t slot) {
  // lowest status code wins (INVALID=1 < TRUNCATED=2 < BADGAP=3 ...), matching
  // the reference where InvalidCode surfaces before header-count checks.
  atomicMin(reinterpret_cast<int*>(&rep->status), status == BH_OK ? 0x7fffffff : status);
  atomicMin(&rep->fail_slot, (unsigned long long)slot);
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ld/st with gpu-scope acquire/release for look-back descriptors.
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}

// Look-back descriptor: 2-bit flag in the top bits, 62-bit value.
constexpr unsigned long long LB_FLAG_AGG = 1ull << 62;
constexpr unsigned long long LB_FLAG_INC = 2ull << 62;
constexpr unsigned long long LB_VALUE = (1ull << 62) - 1;

// Warp-cooperative decoupled look-back: returns the exclusive prefix of tile
// `tile` (sum of all earlier tiles' aggregates).  Every lane returns the value.
// The 32 lanes inspect 32 predecessors at once; the nearest inclusive
// descriptor terminates the walk.
__device__ __forceinline__ unsigned long long warp_lookback(unsigned long long* desc, uint64_t tile) {
  const uint32_t lane = lane_id();
  unsigned long long excl = 0;
  int64_t base = (int64_t)tile - 1;
  while (base >= 0) {
    int64_t idx = base - (int64_t)lane;
    unsigned long long d = 0;
    bool valid = idx >= 0;
    // spin until every inspected predecessor has published something
    while (true) {
      d = valid ? ld_acquire(desc + idx) : LB_FLAG_INC;
      bool ready = (d >> 62) != 0;
      if (__all_sync(0xffffffffu, ready)) break;
      __nanosleep(32);
    }
    unsigned inc_mask = __ballot_sync(0xffffffffu, (d >> 62) == 2 && valid);
    // lanes up to and including the first inclusive descriptor contribute
    int stop_lane = inc_mask ? __ffs(inc_mask) - 1 : 31;
    unsigned long long v = (lane <= (uint32_t)stop_lane && valid) ? (d & LB_VALUE) : 0ull;
    excl += warp_sum(v);
    if (inc_mask) break;
    base -= 32;
  }
  return excl;
}

}  // namespace bh
