// fused.cu -- single-pass fused decoders: the bh_decode fast path.
//
// One kernel per decode.  A persistent grid of warps walks the sequences
// (tiles) in order; per tile, one lane per subsequence:
//
//   1. the tile's compressed words are cp.async-staged into shared memory one
//      tile ahead (double buffer per warp);
//   2. entries: GAP  -- boundary + gap byte (gap_decoder.py:24-33);
//               SYNC -- intra-sequence self-synchronisation (sync_decoder.py
//                       :62-109): every lane decodes its window from the
//                       boundary, then exits are handed right with shuffles and
//                       re-decoded until a ballot shows no live chain.  A
//                       re-decode walks the old and the new decode in lock-step
//                       and stops as soon as they meet (self-synchronisation),
//                       reusing the old tail.  The seam to the previous sequence
//                       (inter_sync, :116-149) is resolved in the same pass:
//                       the 32 possible seeds of the first slot are tried in
//                       parallel (lane o = boundary + o), so a sequence whose
//                       exit is seed-independent publishes it immediately and
//                       the true seed only selects the first slot's count;
//   3. counts: 12-bit multi-codeword count table, warp scan, decoupled
//      look-back over per-tile descriptors (state.py:44-53 output_index);
//   4. decode-and-write (staging.py:113-147): lanes decode in lock-step, two
//      symbols per step, into per-lane shared-memory rows whose odd word
//      stride puts every lane in its own bank; the warp then gathers the rows
//      into output order with 128-bit loads and flushes with coalesced
//      128-bit stores.  A row holds the largest possible subsequence output,
//      so the whole tile is always staged (the reference's capacity rounds
//      only matter for its DecodeStats, which the staged pipeline reproduces).
//
// Shared-memory bank conflicts are designed out: the 8-bit decode and count
// tables are replicated per lane (lane l reads only bank l), staging writes are
// bank-private, and the gather reads 16-byte-aligned consecutive chunks.
//
// No memory needs resetting between calls: descriptors and the report are
// tagged with a per-call epoch (bh_workspace_reset once per allocation).
#include <atomic>
#include <chrono>
#include <cstring>
#include <map>
#include <mutex>
#include "common.cuh"

namespace bh {

constexpr int HALO_WORDS = 8;
constexpr int FUSED_MAX_THREADS = 1024;
constexpr uint32_t NEED_STAGED = 9;  // BH_NEED_STAGED

// descriptor: [63:38] epoch (26 bits) | [37:36] flags | [35:0] value
constexpr unsigned long long D_VAL = (1ull << 36) - 1;
constexpr unsigned long long D_AGG = 1ull << 36;
constexpr unsigned long long D_INC = 2ull << 36;  // inclusive prefix / final exit
constexpr uint32_t EP_MASK = (1u << 26) - 1;

__device__ __forceinline__ unsigned long long mkdesc(uint32_t ep, unsigned long long flag, unsigned long long v) {
  return ((unsigned long long)(ep & EP_MASK) << 38) | flag | (v & D_VAL);
}
__device__ __forceinline__ bool desc_ready(unsigned long long d, uint32_t ep) {
  return (uint32_t)(d >> 38) == (ep & EP_MASK) && (d & (3ull << 36)) != 0;
}

struct FusedArgs {
  const uint32_t* words;
  uint64_t words_alloc;  // readable words (payload + pad), multiple of 4
  const uint8_t* gap;
  const void* table;
  uint32_t max_codes;
  uint32_t sb, sps, seq_bits;
  uint64_t tb, nsym, nsub, nseq;
  uint16_t* out;
  unsigned long long* cnt_desc;
  unsigned long long* exit_desc;
  DevReport* rep;
  uint32_t epoch;
  uint32_t wpb;          // words per tile buffer (multiple of 4)
  uint32_t row_words;    // staging row stride in words (odd)
  uint32_t warps;        // warps per CTA
  uint32_t per_warp_bytes;
  uint32_t tables_bytes;
};

// shared-memory table layout inside the CTA (bytes)
constexpr uint32_t T_DL = 0;                      // u32 [256][32] replicated dlut8
constexpr uint32_t T_CL = T_DL + 256 * 32 * 4;    // u8  [64][32][4] replicated clut8
constexpr uint32_t T_LIM = T_CL + 256 * 32;       // u64 [33]
constexpr uint32_t T_BASE = T_LIM + 33 * 8;       // i64 [33]
constexpr uint32_t T_END = T_BASE + 33 * 8;

__device__ __forceinline__ void tag_status(DevReport* rep, uint32_t ep, uint32_t status) {
  unsigned long long v = ((unsigned long long)ep << 32) | (unsigned long long)(0x7fffffffu - status);
  atomicMax(&rep->pad[0], v);  // pad[0] = tagged status (see bh_report_read)
}

// ---- shared-memory primitives (explicit 32-bit shared addresses) ----------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t lds16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t lds8(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// Keep a value in a register: the compiler may not rematerialise it (it
// otherwise recomputes shared-window addresses from SR_CgaCtaId in hot loops).
__device__ __forceinline__ uint32_t pin(uint32_t v) {
  asm volatile("mov.b32 %0, %0;" : "+r"(v));
  return v;
}

// Bit reader over a tile's staged words; positions are tile-relative bits.
struct SR {
  uint64_t buf;
  uint32_t av;
  uint32_t wa;  // shared address of the next word to load
  __device__ __forceinline__ void init(uint32_t base_s, uint32_t rel) {
    const uint32_t a = base_s + ((rel >> 5) << 2);
    buf = (((uint64_t)lds32(a) << 32) | lds32(a + 4)) << (rel & 31);
    av = 64 - (rel & 31);
    wa = a + 8;
  }
  __device__ __forceinline__ uint32_t peek() const { return (uint32_t)(buf >> 32); }
  __device__ __forceinline__ void skip(uint32_t n) {
    buf <<= n;
    av -= n;
    if (av < 32) {
      buf |= (uint64_t)lds32(wa) << (32 - av);
      wa += 4;
      av += 32;
    }
  }
};

struct FTab {
  uint32_t dl;     // this lane's column of the replicated dlut8 (shared address)
  uint32_t cl;     // this lane's column of the replicated clut8
  uint32_t lim;    // shared address of lim (u64[33])
  uint32_t base;   // shared address of base (i64[33])
  TableView t;
  uint32_t kind;
};

// one codeword from a 32-bit window when the 8-bit table cannot answer
__device__ __noinline__ uint32_t fslow(uint32_t win, const uint32_t lim_s, const uint32_t base_s,
                                       const uint16_t* __restrict__ ljsym, uint32_t kind, TableView t) {
  if (kind == 0) {
    const uint2 l32 = lds64(lim_s + 32 * 8);
    if ((unsigned long long)win >= (((unsigned long long)l32.y << 32) | l32.x)) return 0;
    uint32_t lo = 9, hi = 32;  // codes of <= 8 bits are answered by dlut8
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      const uint2 l = lds64(lim_s + mid * 8);
      if ((unsigned long long)win < (((unsigned long long)l.y << 32) | l.x)) hi = mid; else lo = mid + 1;
    }
    const uint2 bb = lds64(base_s + lo * 8);
    const long long idx = (long long)(((unsigned long long)bb.y << 32) | bb.x) + (long long)(win >> (32 - lo));
    return (uint32_t)__ldg(ljsym + idx) | (lo << 16);
  }
  return slow_lookup(t, win);
}

// one codeword: sym | len<<16 (0 = no codeword matches)
__device__ __forceinline__ uint32_t fone(uint32_t win, const FTab& T) {
  uint32_t e = lds32(T.dl + ((win >> 24) << 7));
  if (!e) e = fslow(win, T.lim, T.base, T.t.ljsym, T.kind, T.t);
  return e;
}

// count codewords starting in [pos, stop) (tile-relative); pos ends at the exit
__device__ __forceinline__ bool fcount(SR& r, uint32_t& pos, uint32_t stop, const FTab& T, uint32_t& n) {
  while (pos < stop) {
    const uint32_t win = r.peek();
    if (stop - pos >= 8u) {
      const uint32_t c = lds8(T.cl + ((win >> 26) << 7) + ((win >> 24) & 3));
      if (c) {
        const uint32_t b = (c & 7u) + 1;
        n += c >> 3;
        r.skip(b);
        pos += b;
        continue;
      }
    }
    const uint32_t len = (fone(win, T) >> 16) & 0xffu;
    if (!len) return false;
    r.skip(len);
    pos += len;
    ++n;
  }
  return true;
}

// Decode c symbols into this lane's staging row (pairs of symbols per word).
// Lanes step in lock-step (same pair index), so lane l's store lands in bank
// (row_words*l + p) mod 32 -- distinct for the odd row_words.  The reader is
// topped up 16 bits at a time so that both lookups of a pair need no refill:
// with >= 48 valid bits at the top of a pair, two codes of <= 8 bits leave
// >= 32; a longer code takes the slow path, which refills as it goes.
__device__ __forceinline__ bool fdecode_row(const SR& r0, uint32_t c, uint32_t row, uint32_t wbuf_s,
                                            const FTab& T) {
  bool ok = true;
  const uint32_t dl = pin(T.dl);
  uint64_t buf = r0.buf;
  uint32_t av = r0.av;
  uint32_t ha = (r0.wa - wbuf_s) >> 1;  // next halfword of the MSB-first word stream
#define BH_TOPUP()                                          \
  {                                                         \
    const uint32_t h_ = lds16(wbuf_s + ((ha ^ 1u) << 1));   \
    buf |= (uint64_t)h_ << (48 - av);                       \
    av += 16;                                               \
    ++ha;                                                   \
  }
  for (uint32_t k = 0; k < c; k += 2) {
    if (av < 48) BH_TOPUP();
    const uint32_t w0 = (uint32_t)(buf >> 32);
    const uint32_t e0 = lds32(dl + ((w0 >> 24) << 7));
    const uint32_t l0 = e0 >> 16;
    const uint32_t w1 = (uint32_t)((buf << l0) >> 32);
    const uint32_t e1 = lds32(dl + ((w1 >> 24) << 7));
    uint32_t pair;
    if (e0 && e1) {
      const uint32_t s = l0 + (e1 >> 16);
      buf <<= s;
      av -= s;
      pair = (e0 & 0xffffu) | (e1 << 16);
    } else {
      // a code longer than 8 bits: one codeword at a time, refilling as needed
      const uint32_t s0 = fone((uint32_t)(buf >> 32), T);
      ok = ok && s0;
      buf <<= (s0 >> 16) & 0xffu;
      av -= (s0 >> 16) & 0xffu;
      while (av < 48) BH_TOPUP();
      uint32_t s1 = 0;
      if (k + 1 < c) {
        s1 = fone((uint32_t)(buf >> 32), T);
        ok = ok && s1;
        buf <<= (s1 >> 16) & 0xffu;
        av -= (s1 >> 16) & 0xffu;
        while (av < 48) BH_TOPUP();
      }
      pair = (s0 & 0xffffu) | (s1 << 16);
    }
    sts32(row + 2 * k, pair);
  }
#undef BH_TOPUP
  return ok;
}

// Re-decode a window from a new entry, walking the previous decode (entry eo,
// count co, exit xo) in lock-step; once both cursors meet the rest is shared.
__device__ __forceinline__ bool resync(uint32_t base_s, uint32_t eo, uint32_t co, uint32_t xo, uint32_t en,
                                       uint32_t stop, const FTab& T, uint32_t& cn, uint32_t& xn) {
  uint32_t po = eo, pn = en, no = 0, nn = 0;
  SR ro, rn;
  ro.init(base_s, po);
  rn.init(base_s, pn);
  while (true) {
    if (pn >= stop) { cn = nn; xn = pn; return true; }
    if (po == pn) { cn = nn + (co - no); xn = xo; return true; }
    if (po < pn) {
      const uint32_t l = (fone(ro.peek(), T) >> 16) & 0xffu;
      if (!l) return false;
      ro.skip(l);
      po += l;
      ++no;
    } else {
      const uint32_t l = (fone(rn.peek(), T) >> 16) & 0xffu;
      if (!l) return false;
      rn.skip(l);
      pn += l;
      ++nn;
    }
  }
}

// warp look-back over epoch-tagged descriptors
__device__ __forceinline__ unsigned long long lookback(unsigned long long* desc, uint64_t tile, uint32_t ep) {
  const uint32_t lane = threadIdx.x & 31;
  unsigned long long excl = 0;
  int64_t base = (int64_t)tile - 1;
  while (base >= 0) {
    const int64_t idx = base - (int64_t)lane;
    const bool valid = idx >= 0;
    unsigned long long d;
    while (true) {
      d = valid ? ld_acquire(desc + idx) : 0ull;
      const bool ready = !valid || desc_ready(d, ep);
      if (__all_sync(0xffffffffu, ready)) break;
      __nanosleep(20);
    }
    const unsigned inc = __ballot_sync(0xffffffffu, valid && (d & D_INC));
    const int stop_lane = inc ? __ffs(inc) - 1 : 31;
    const unsigned long long v = (valid && (int)lane <= stop_lane) ? (d & D_VAL) : 0ull;
    excl += warp_sum(v);
    if (inc) break;
    base -= 32;
  }
  return excl;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// stage the words of `tile` (16 B chunks, one per lane per step)
__device__ __forceinline__ uint64_t stage_words(const FusedArgs& a, uint64_t tile, uint32_t* buf) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t s0 = tile * (uint64_t)a.seq_bits;
  const uint64_t w0 = (s0 >> 5) & ~3ull;
  uint64_t w1 = ((s0 + a.seq_bits) >> 5) + HALO_WORDS;
  w1 = (w1 + 3) & ~3ull;
  if (w1 > a.words_alloc) w1 = a.words_alloc;
  const uint32_t nch = (uint32_t)((w1 - w0) >> 2);
  for (uint32_t c = lane; c < nch; c += 32) cp_async16(buf + 4 * c, a.words + w0 + 4 * c);
  return w0 * 32;  // bit offset of buf[0]
}

// halfwords [sh, sh+8) of the 16 halfwords A||B (little-endian halfword order)
__device__ __forceinline__ uint4 shift_hw(uint4 A, uint4 B, uint32_t sh) {
  const bool b2 = sh & 4, b1 = sh & 2;
  const uint32_t t0 = b2 ? A.z : A.x, t1 = b2 ? A.w : A.y, t2 = b2 ? B.x : A.z;
  const uint32_t t3 = b2 ? B.y : A.w, t4 = b2 ? B.z : B.x, t5 = b2 ? B.w : B.y;
  const uint32_t u0 = b1 ? t1 : t0, u1 = b1 ? t2 : t1, u2 = b1 ? t3 : t2, u3 = b1 ? t4 : t3, u4 = b1 ? t5 : t4;
  const uint32_t sel = (sh & 1) ? 0x5432u : 0x3210u;
  return make_uint4(__byte_perm(u0, u1, sel), __byte_perm(u1, u2, sel), __byte_perm(u2, u3, sel),
                    __byte_perm(u3, u4, sel));
}

// 8 consecutive staged symbols starting at (signed) halfword index sidx
__device__ __forceinline__ uint4 read8(uint32_t rows_s, int32_t sidx) {
  const uint32_t q = rows_s + 2u * (uint32_t)(sidx & ~7);
  return shift_hw(lds128(q), lds128(q + 16), (uint32_t)sidx & 7u);
}

// Gather the tile's rows into output order and flush [P, P+C) with 128-bit
// stores.  so/sc: per-lane start (tile-local) and count arrays (so[32] = inf).
// A chunk covers at most two lanes' rows on the common path (both rows are
// read unconditionally to keep the warp converged); a chunk touching three or
// more lanes (some lane with < 8 symbols) goes element by element.
__device__ __forceinline__ void flush_rows(uint16_t* __restrict__ out, uint64_t nsym, uint64_t P, uint32_t C,
                                           uint32_t rows_s, uint32_t row_hw, const uint32_t* so,
                                           const uint32_t* sc) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t a0 = P & ~7ull, g1 = P + C;
  const uint32_t nch = (uint32_t)((g1 - a0 + 7) >> 3);
  for (uint32_t ch = lane; ch < nch; ch += 32) {
    const uint64_t ga = a0 + (uint64_t)ch * 8;
    const int32_t x = (int32_t)(int64_t)(ga - P);  // tile-local position of the chunk (may be < 0)
    const uint32_t xs = x < 0 ? 0u : (uint32_t)x;
    uint32_t L = 0;  // owner of xs: largest lane with so[L] <= xs
#pragma unroll
    for (uint32_t step = 16; step; step >>= 1)
      if (L + step < 32 && so[L + step] <= xs) L += step;
    const uint32_t soL = so[L];
    const int32_t m = (int32_t)(soL + sc[L]) - x;   // elements of the chunk inside lane L
    uint32_t L2 = L + 1 < 32 ? L + 1 : 31;
    const uint4 v1 = read8(rows_s, (int32_t)(L * row_hw) + (x - (int32_t)soL));
    const uint4 v2 = read8(rows_s, (int32_t)(L2 * row_hw) + (x - (int32_t)so[L2]));
    // halfword i comes from v1 when i < m, else from v2
    const uint32_t mk0 = m > 1 ? 0xffffffffu : (m > 0 ? 0xffffu : 0u);
    const uint32_t mk1 = m > 3 ? 0xffffffffu : (m > 2 ? 0xffffu : 0u);
    const uint32_t mk2 = m > 5 ? 0xffffffffu : (m > 4 ? 0xffffu : 0u);
    const uint32_t mk3 = m > 7 ? 0xffffffffu : (m > 6 ? 0xffffu : 0u);
    uint4 v = make_uint4((v1.x & mk0) | (v2.x & ~mk0), (v1.y & mk1) | (v2.y & ~mk1),
                         (v1.z & mk2) | (v2.z & ~mk2), (v1.w & mk3) | (v2.w & ~mk3));
    const bool inside = ga >= P && ga + 8 <= g1 && ga + 8 <= nsym;
    const int32_t need = min(8, (int32_t)C - x);  // chunk elements inside the tile (from x)
    const bool two_ok = m >= need || (L + 1 < 32 && m + (int32_t)sc[L2] >= need);
    if (!two_ok) {
      // three or more lanes in one chunk: element by element
      uint32_t h[8];
      uint32_t Lc = L;
#pragma unroll
      for (uint32_t i = 0; i < 8; ++i) {
        h[i] = 0;
        const int32_t xi = x + (int32_t)i;
        if (xi >= 0 && xi < (int32_t)C) {
          while (Lc < 31 && so[Lc + 1] <= (uint32_t)xi) ++Lc;
          h[i] = lds16(rows_s + 2 * (Lc * row_hw + ((uint32_t)xi - so[Lc])));
        }
      }
      v = make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16), h[6] | (h[7] << 16));
    }
    if (inside) {
      *reinterpret_cast<uint4*>(out + ga) = v;
    } else {
      const uint32_t hv[8] = {v.x & 0xffffu, v.x >> 16, v.y & 0xffffu, v.y >> 16,
                              v.z & 0xffffu, v.z >> 16, v.w & 0xffffu, v.w >> 16};
#pragma unroll
      for (uint32_t i = 0; i < 8; ++i) {
        const uint64_t gi = ga + i;
        if (gi >= P && gi < g1 && gi < nsym) out[gi] = (uint16_t)hv[i];
      }
    }
  }
}

// Entries and counts of one tile (lane = subsequence); positions are relative
// to the tile buffer's first bit `wb0`.  GAP: boundary + gap byte; SYNC:
// intra-sequence chain rounds plus the seam seed from the predecessor tile's
// published final exit.
template <int VAR>
__device__ __forceinline__ void tile_counts(const FusedArgs& a, const FTab& T, uint64_t tile, uint32_t base_s,
                                            uint64_t wb0, uint32_t nsl, uint32_t& e, uint32_t& c, bool& bad) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t ep = a.epoch;
  const uint32_t sb = a.sb;
  const uint64_t j0 = tile * a.sps;
  const bool active = lane < nsl;
  const uint64_t j = j0 + lane;
  const uint32_t b = (uint32_t)(j * sb - wb0);                              // relative boundary
  const uint32_t tbr = (uint32_t)min(a.tb - wb0, (uint64_t)0xffffffffu);   // relative total_bits
  uint32_t x = b, stop;
  e = b;
  c = 0;
  if (VAR == BH_VARIANT_GAP) {
    const uint32_t g = active ? a.gap[j] : 0u;
    uint32_t gn = __shfl_down_sync(0xffffffffu, g, 1);
    if (lane == nsl - 1) gn = (j + 1 < a.nsub) ? a.gap[j + 1] : 0u;
    e = b + g;
    stop = (j + 1 < a.nsub) ? b + sb + gn : tbr;
    if (stop > tbr) stop = tbr;
    x = e;
    if (active && e < stop) {
      SR r;
      r.init(base_s, e);
      if (!fcount(r, x, stop, T, c)) bad = true;
    }
  } else {
    stop = min(b + sb, tbr);
    if (active && e < stop) {
      SR r;
      r.init(base_s, e);
      if (!fcount(r, x, stop, T, c)) bad = true;
    }
    bool dprev = active;
    while (true) {
      const uint32_t xin = __shfl_up_sync(0xffffffffu, x, 1);
      const bool din = __shfl_up_sync(0xffffffffu, dprev, 1);
      const bool live = lane >= 1 && active && din;
      if (!__any_sync(0xffffffffu, live)) break;
      bool dnow = false;
      if (live && xin != e) {
        uint32_t cn, xn;
        if (!resync(base_s, e, c, x, xin, stop, T, cn, xn)) bad = true;
        e = xin;
        c = cn;
        x = xn;
        dnow = true;
      }
      dprev = dnow;
    }
    const uint32_t b0 = __shfl_sync(0xffffffffu, b, 0);
    const uint32_t stop0 = min(b0 + sb, tbr);
    const uint32_t c0 = __shfl_sync(0xffffffffu, c, 0);
    const uint32_t x0 = __shfl_sync(0xffffffffu, x, 0);
    uint32_t cand_c = c0, cand_x = x0;
    bool indep = true;
    if (tile > 0) {
      if (!resync(base_s, b0, c0, x0, b0 + lane, stop0, T, cand_c, cand_x)) cand_x = 0xffffffffu;
      indep = __all_sync(0xffffffffu, cand_x == x0);
    }
    const uint32_t xlast = __shfl_sync(0xffffffffu, x, nsl - 1);
    if (lane == 0 && indep) st_release(a.exit_desc + tile, mkdesc(ep, D_INC, wb0 + xlast));
    if (tile > 0) {
      unsigned long long d = 0;
      if (lane == 0) {
        while (!desc_ready(d = ld_acquire(a.exit_desc + tile - 1), ep)) __nanosleep(20);
      }
      const uint64_t seed = __shfl_sync(0xffffffffu, (unsigned long long)(d & D_VAL), 0);
      const uint32_t o = (uint32_t)(seed - wb0) - b0;
      const uint32_t sc = __shfl_sync(0xffffffffu, cand_c, o & 31);
      const uint32_t sx = __shfl_sync(0xffffffffu, cand_x, o & 31);
      if (o >= 32) bad = true;
      if (lane == 0) { e = b0 + o; c = sc; x = sx; }
      if (sx != x0) {
        bool dprev2 = lane == 0;
        while (true) {
          const uint32_t xin = __shfl_up_sync(0xffffffffu, x, 1);
          const bool din = __shfl_up_sync(0xffffffffu, dprev2, 1);
          const bool live = lane >= 1 && active && din;
          if (!__any_sync(0xffffffffu, live)) break;
          bool dnow = false;
          if (live && xin != e) {
            uint32_t cn, xn;
            if (!resync(base_s, e, c, x, xin, stop, T, cn, xn)) bad = true;
            e = xin;
            c = cn;
            x = xn;
            dnow = true;
          }
          dprev2 = dnow;
        }
      }
      if (!indep) {
        const uint32_t xl = __shfl_sync(0xffffffffu, x, nsl - 1);
        if (lane == 0) st_release(a.exit_desc + tile, mkdesc(ep, D_INC, wb0 + xl));
      }
    }
  }
  if (!active) c = 0;
}

// One CTA processes a group of `warps` consecutive tiles per iteration (warp w
// takes tile group*warps + w).  The group's output offset comes from one
// decoupled look-back over group descriptors, done by warp 0 while the other
// warps already decode into their staging rows.
template <int VAR>
__global__ void __launch_bounds__(FUSED_MAX_THREADS) k_fused(const FusedArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ uint32_t s_C[32];
  __shared__ unsigned long long s_P;
  const TableHdr* hdr = static_cast<const TableHdr*>(a.table);
  if (VAR == BH_VARIANT_SYNC && !hdr->complete) {
    // the speculative windows differ from the reference's: only complete books
    // (where no window can fail) may take the fused path
    if (blockIdx.x == 0 && threadIdx.x == 0) tag_status(a.rep, a.epoch, NEED_STAGED);
    return;
  }
  {
    TableLayout L(a.max_codes);
    const char* tb_ = static_cast<const char*>(a.table);
    const uint32_t* dl = reinterpret_cast<const uint32_t*>(tb_ + L.dlut8);
    const uint8_t* cl = reinterpret_cast<const uint8_t*>(tb_ + L.clut8);
    uint32_t* s_dl = reinterpret_cast<uint32_t*>(sm + T_DL);
    uint8_t* s_cl = reinterpret_cast<uint8_t*>(sm + T_CL);
    for (uint32_t i = threadIdx.x; i < 256 * 32; i += blockDim.x) {
      const uint32_t ent = i >> 5, ln = i & 31;
      s_dl[i] = __ldg(dl + ent);                                   // [ent][lane]
      s_cl[((ent >> 2) << 7) + (ln << 2) + (ent & 3)] = __ldg(cl + ent);
    }
    const unsigned long long* gl = reinterpret_cast<const unsigned long long*>(tb_ + L.lim);
    const long long* gb = reinterpret_cast<const long long*>(tb_ + L.base);
    unsigned long long* s_lim = reinterpret_cast<unsigned long long*>(sm + T_LIM);
    long long* s_base = reinterpret_cast<long long*>(sm + T_BASE);
    for (int i = threadIdx.x; i < 33; i += blockDim.x) { s_lim[i] = gl[i]; s_base[i] = gb[i]; }
  }
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  FTab T;
  const uint32_t sm_s = smem_u32(sm);
  T.dl = pin(sm_s + T_DL + 4 * lane);
  T.cl = pin(sm_s + T_CL + 4 * lane);
  T.lim = sm_s + T_LIM;
  T.base = sm_s + T_BASE;
  T.t = table_view(a.table, a.max_codes, hdr->ncodes);
  T.kind = hdr->kind;
  __syncthreads();

  unsigned char* pw = sm + a.tables_bytes + (size_t)wib * a.per_warp_bytes;
  uint32_t* const wbase = reinterpret_cast<uint32_t*>(pw);
  const uint32_t wbase_s = smem_u32(pw);
  const uint32_t rows_s = wbase_s + 8 * a.wpb;                 // 32 rows of row_words words
  uint32_t* s_o = reinterpret_cast<uint32_t*>(pw + 8 * (size_t)a.wpb + 128 * (size_t)a.row_words);
  uint32_t* s_c = s_o + 33;
  const uint32_t row_hw = 2 * a.row_words;                     // row stride in symbols
  const uint32_t my_row = rows_s + 4 * a.row_words * lane;
  const uint32_t W = a.warps;
  const uint64_t ngroups = (a.nseq + W - 1) / W;
  const uint32_t ep = a.epoch;
  bool bad = false;

  uint64_t grp = blockIdx.x;
  uint64_t wbit_cur = 0, wbit_next = 0;
  uint32_t cur = 0;
  if (grp * W + wib < a.nseq) wbit_cur = stage_words(a, grp * W + wib, wbase);
  cp_commit();
  for (; grp < ngroups; grp += gridDim.x) {
    const uint64_t tile = grp * W + wib;
    const uint64_t ntile = (grp + gridDim.x) * W + wib;
    if (ntile < a.nseq) wbit_next = stage_words(a, ntile, wbase + (cur ^ 1) * a.wpb);
    cp_commit();
    cp_wait<1>();
    __syncwarp();
    const uint32_t base_s = wbase_s + cur * a.wpb * 4;
    const uint64_t wb0 = wbit_cur;
    const bool have = tile < a.nseq;
    uint32_t nsl = 0, e = 0, c = 0;
    if (have) {
      nsl = (uint32_t)min((uint64_t)a.sps, a.nsub - tile * a.sps);
      tile_counts<VAR>(a, T, tile, base_s, wb0, nsl, e, c, bad);
    }
    uint32_t incl = c;
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
      if ((int)lane >= off) incl += y;
    }
    const uint32_t C = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t o = incl - c;
    s_o[lane] = o;
    s_c[lane] = c;
    if (lane == 0) { s_C[wib] = C; s_o[32] = 0xffffffffu; }
    __syncthreads();
    if (wib == 0) {
      const uint32_t v = lane < W ? s_C[lane] : 0u;
      const unsigned long long A = warp_sum((unsigned long long)v);
      unsigned long long Pg = 0;
      if (grp == 0) {
        if (lane == 0) st_release(a.cnt_desc, mkdesc(ep, D_INC, A));
      } else {
        if (lane == 0) st_release(a.cnt_desc + grp, mkdesc(ep, D_AGG, A));
        Pg = lookback(a.cnt_desc, grp, ep);
        if (lane == 0) st_release(a.cnt_desc + grp, mkdesc(ep, D_INC, Pg + A));
      }
      if (lane == 0) {
        s_P = Pg;
        if (grp == ngroups - 1) {
          a.rep->total_symbols = Pg + A;
          if (Pg + A != a.nsym) tag_status(a.rep, ep, VAR == BH_VARIANT_GAP ? BH_BADGAP : BH_TRUNCATED);
        }
      }
    }
    if (have && c) {
      SR r;
      r.init(base_s, e);
      if (!fdecode_row(r, c, my_row, base_s, T)) bad = true;
    }
    __syncthreads();  // s_P published; rows complete
    uint32_t before = lane < wib ? s_C[lane] : 0u;
    for (int off = 16; off > 0; off >>= 1) before += __shfl_xor_sync(0xffffffffu, before, off);
    const unsigned long long P = s_P + before;
    if (have) flush_rows(a.out, a.nsym, P, C, rows_s, row_hw, s_o, s_c);
    __syncwarp();
    cur ^= 1;
    wbit_cur = wbit_next;
  }
  cp_wait<0>();
  if (__any_sync(0xffffffffu, bad) && lane == 0) tag_status(a.rep, ep, BH_INVALID);
}

}  // namespace bh

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
using namespace bh;

namespace {
std::atomic<uint32_t> g_epoch{0};
std::mutex g_rep_mu;
std::map<const void*, uint32_t> g_rep_epoch;  // report buffer -> epoch of its last fused launch

inline uint64_t nsub_of(const bh_stream* s) { return (s->total_bits + s->subseq_bits - 1) / s->subseq_bits; }
inline uint64_t nseq_of(const bh_stream* s) { return (nsub_of(s) + s->subseqs_per_seq - 1) / s->subseqs_per_seq; }

uint32_t next_epoch() {
  uint32_t e = g_epoch.fetch_add(1) + 1;
  if (e == 1) {  // first use in this process: start somewhere unlikely to be stale
    uint32_t seed = (uint32_t)std::chrono::steady_clock::now().time_since_epoch().count() | 1u;
    g_epoch.store(seed + 1);
    e = seed;
  }
  if ((e & EP_MASK) == 0) e = g_epoch.fetch_add(1) + 1;  // epoch 0 is "never written"
  return e;
}

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

struct FusedCfg {
  uint32_t warps, row_words, wpb, per_warp, tables, smem;
};

FusedCfg fused_cfg(const bh_stream* s) {
  FusedCfg c;
  const uint32_t seq_bits = s->subseq_bits * s->subseqs_per_seq;
  c.wpb = ((seq_bits + 31) / 32 + 3 + HALO_WORDS + 3) & ~3u;
  // a slot counts codewords starting in [entry, stop): at most subseq_bits + 31
  const uint32_t max_c = s->subseq_bits + 31;
  c.row_words = ((max_c + 1) / 2) | 1u;  // odd: lane rows fall in distinct banks
  c.tables = (uint32_t)align16(T_END);
  c.per_warp = (uint32_t)align16(8 * (size_t)c.wpb + 128 * (size_t)c.row_words + 4 * 66);
  int w = env_int("BH_FUSED_WARPS", 0);
  if (w <= 0) {
    w = (int)((220 * 1024 - c.tables) / c.per_warp);
    if (w > 32) w = 32;
    if (w < 1) w = 1;
  }
  c.warps = (uint32_t)w;
  c.smem = c.tables + c.warps * c.per_warp;
  return c;
}

}  // namespace

extern "C" int bh_fused_supported(const bh_stream* s, int variant) {
  if (env_int("BH_DISABLE_FUSED", 0)) return 0;
  if (variant != BH_VARIANT_GAP && variant != BH_VARIANT_SYNC) return 0;
  if (s->subseqs_per_seq > 32 || s->subseqs_per_seq == 0) return 0;
  const uint64_t seq_bits = (uint64_t)s->subseq_bits * s->subseqs_per_seq;
  if (seq_bits > 16384 || s->subseq_bits > 512 || s->total_bits >= (1ull << 36) || s->symbol_count >= (1ull << 36)) return 0;
  if (variant == BH_VARIANT_GAP && !s->gap_dev) return 0;
  FusedCfg c = fused_cfg(s);
  return c.smem <= 227 * 1024 ? 1 : 0;
}

extern "C" size_t bh_fused_workspace_bytes(const bh_stream* s, int, const bh_tune*) {
  return 16 * nseq_of(s) + 256;
}

extern "C" int bh_workspace_reset(void* ws, size_t bytes, void* cuda_stream) {
  return cudaMemsetAsync(ws, 0, bytes, static_cast<cudaStream_t>(cuda_stream)) == cudaSuccess ? BH_OK
                                                                                              : BH_CUDA_ERROR;
}

extern "C" int bh_fused_decode(const bh_stream* s, int variant, const bh_tune* tune, uint16_t* out_dev,
                               void* ws, size_t ws_bytes, void* report_dev, void* cuda_stream) {
  (void)tune;
  const uint64_t nseq = nseq_of(s);
  if (ws_bytes < bh_fused_workspace_bytes(s, variant, tune)) return BH_BAD_ARGUMENT;
  FusedCfg cfg = fused_cfg(s);
  FusedArgs a;
  a.words = s->words_dev;
  a.words_alloc = (((s->total_bits + 31) / 32 + BH_WORD_PAD) & ~3ull);
  a.gap = s->gap_dev;
  a.table = s->table_dev;
  a.max_codes = s->max_codes;
  a.sb = s->subseq_bits;
  a.sps = s->subseqs_per_seq;
  a.seq_bits = s->subseq_bits * s->subseqs_per_seq;
  a.tb = s->total_bits;
  a.nsym = s->symbol_count;
  a.nsub = nsub_of(s);
  a.nseq = nseq;
  a.out = out_dev;
  a.cnt_desc = static_cast<unsigned long long*>(ws);
  a.exit_desc = a.cnt_desc + nseq;
  a.rep = static_cast<DevReport*>(report_dev);
  a.epoch = next_epoch();
  a.wpb = cfg.wpb;
  a.row_words = cfg.row_words;
  a.warps = cfg.warps;
  a.per_warp_bytes = cfg.per_warp;
  a.tables_bytes = cfg.tables;
  {
    std::lock_guard<std::mutex> g(g_rep_mu);
    g_rep_epoch[report_dev] = a.epoch;
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const void* fn = variant == BH_VARIANT_GAP ? (const void*)k_fused<BH_VARIANT_GAP> : (const void*)k_fused<BH_VARIANT_SYNC>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.smem) != cudaSuccess)
    return BH_CUDA_ERROR;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, (int)cfg.warps * 32, cfg.smem) != cudaSuccess ||
      per_sm < 1)
    return BH_CUDA_ERROR;
  uint64_t grid = (uint64_t)per_sm * sms;
  const uint64_t need = (nseq + cfg.warps - 1) / cfg.warps;  // groups
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  prof_mark(static_cast<cudaStream_t>(cuda_stream), "start");
  if (variant == BH_VARIANT_GAP)
    k_fused<BH_VARIANT_GAP><<<(unsigned)grid, cfg.warps * 32, cfg.smem, static_cast<cudaStream_t>(cuda_stream)>>>(a);
  else
    k_fused<BH_VARIANT_SYNC><<<(unsigned)grid, cfg.warps * 32, cfg.smem, static_cast<cudaStream_t>(cuda_stream)>>>(a);
  prof_mark(static_cast<cudaStream_t>(cuda_stream), variant == BH_VARIANT_GAP ? "fused_gap" : "fused_sync");
  return cudaGetLastError() == cudaSuccess ? BH_OK : BH_CUDA_ERROR;
}

// epoch of the last fused launch that used this report buffer (0 = none)
extern "C" uint32_t bh_fused_report_epoch(const void* report_dev) {
  std::lock_guard<std::mutex> g(g_rep_mu);
  auto it = g_rep_epoch.find(report_dev);
  return it == g_rep_epoch.end() ? 0u : it->second;
}

extern "C" void bh_fused_report_forget(const void* report_dev) {
  std::lock_guard<std::mutex> g(g_rep_mu);
  g_rep_epoch.erase(report_dev);
}
