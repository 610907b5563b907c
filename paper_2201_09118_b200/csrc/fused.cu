// fused.cu -- the fused decoders: the bh_decode fast path (one kernel per decode).
//
// k_fused2 runs one persistent CTA per SM; CTA c owns a contiguous range of
// tiles (a tile = 32 subsequences -- one sequence at the reference's default
// layout -- one lane per subsequence, whatever the stream's subseqs_per_seq).  Two phases:
//
//   phase 1 (count): each warp takes tiles of the range round-robin, stages
//     the tile's words with cp.async (double buffer) and computes every
//     lane's entry and codeword count --
//       GAP  -- boundary + gap byte (gap_decoder.py:24-33), count over the
//               window to the next entry (gap_decoder.py:36-68);
//       SYNC -- intra-sequence self-synchronisation (sync_decoder.py:62-109):
//               every lane decodes its window from the boundary, exits are
//               handed right with shuffles and re-decoded until a ballot shows
//               no live chain (a re-decode walks the old and new decode in
//               lock-step and stops where they meet).  The seam to the
//               previous sequence (inter_sync, :116-149) is resolved in the
//               same pass: the 32 possible seeds of the first slot are tried in
//               parallel, so a sequence whose exit is seed-independent
//               publishes it at once (epoch-tagged per-tile exit descriptors).
//     Counting uses a 12-bit start-mask table: one lookup covers every whole
//     codeword of the next 12 bits (popcount), and the lookup that crosses
//     the window end counts the starts below it.  The entry offset and the
//     lane's prefix go to the workspace, the tile total to shared memory.
//   between the phases: one CTA barrier; each warp sums the totals before its
//     tiles itself; warp 0 publishes the CTA aggregate and resolves the CTA's
//     output offset with a decoupled look-back over the CTA descriptors
//     (state.py:44-53 output_index), while the other warps already decode.
//   phase 2 (decode and write, staging.py:113-147): lanes decode in lock-step
//     through an 8-bit multi-symbol table (up to six codewords per lookup,
//     replicated eight ways so a quarter-warp never conflicts) into compact
//     shared-memory staging with one halfword and three aligned word stores
//     per lookup; the warp then flushes the tile with coalesced 128-bit
//     stores (staging aligned to the output once the offset is known).  A
//     tile larger than the staging capacity takes the reference's rounds.
//
// No memory needs resetting between calls: descriptors and the report are
// tagged with a per-call epoch (bh_workspace_reset once per allocation).
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include "common.cuh"

namespace bh {

constexpr int HALO_WORDS = 8;
#ifndef BH_UNR
#define BH_UNR 4
#endif
constexpr int kUnroll = BH_UNR;  // unroll of the tight count/decode loops
#ifndef BH_MAXW
#define BH_MAXW 24
#endif
#ifndef BH_CAPF
#define BH_CAPF 1.12
#endif
#ifndef BH_CAPADD
#define BH_CAPADD 96
#endif
#ifndef BH_REV
#define BH_REV 1  // phase 2 walks the range backwards: the tiles counted last are still in L2
#endif
#ifndef BH_L2HINT
#define BH_L2HINT 2  // 1: output bulk stores evict_first; 2: also the decode phase's word reads (their last use)
#endif
#ifndef PRESYNC_BY_COUNT
#define PRESYNC_BY_COUNT 1  // SYNC: the pre-window walked by the count loop (0: by 12-bit start-mask entries)
#endif
#ifndef BH_HW3
#define BH_HW3 2  // WIDE3 decode stores per entry: 2 = word + halfword, 1 = three halfwords, 0 = halfword + two words
#endif
#ifndef BH_PSKIP
#define BH_PSKIP 0  // bit reader: predicated next-word load (A/B knob)
#endif
#ifndef BH_PST
#define BH_PST 0  // WIDE3 decode: predicated stores by the entry's count (A/B knob)
#endif
#ifndef BH_TWO
#define BH_TWO 1  // two table lookups per bit-reader advance in the tight loops (HACC gap -5% time)
#endif
constexpr int FUSED_MAX_WARPS = BH_MAXW;
constexpr int FUSED_MAX_THREADS = 32 * FUSED_MAX_WARPS;  // 24 warps: up to 85 registers per thread

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

constexpr uint32_t TUNE_CLASSES = 65;  // classes 1..64 plus the overflow group (t_high <= 64 on this path)

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
  uint32_t* lane_info;   // two-phase kernel: per subsequence (entry - boundary) | lane prefix << 16
  uint32_t* tile_cnt;    // two-phase kernel: symbols per tile
  uint32_t* tile_off;    // two-phase kernel: exclusive tile offset within its CTA's range
  uint16_t* cand;        // SYNC: first-slot count per candidate seed offset (32 per tile)
  int32_t* tile_dlt;     // SYNC: first-slot count change from the seam fix-up
  DevReport* rep;
  unsigned int* ws_hdr;  // [0] epoch of the last completed call, [1] CTAs done
  uint32_t wpb;          // words per tile buffer (multiple of 4)
  uint32_t halo;         // words staged past a tile's span (SYNC: the next tile's first slot, for its seam walk)
  uint32_t lead;         // words staged before a tile's span (SYNC: the pre-synchronisation of its first slot)
  uint32_t presync;      // SYNC: bits a lane's count parse starts before its boundary (0: at the boundary; <= 32 lead)
  uint32_t walk_max;     // SYNC: seam-walk window past the next boundary (test knob; ~0 = the staged words)
  uint32_t cap;          // staging symbols per warp (multiple of 8)
  uint32_t warps;        // warps per CTA
  uint32_t per_warp_bytes;
  uint32_t tables_bytes;
  uint32_t has_l12;      // 12-bit second-level table staged (codes longer than 8 bits)
  uint32_t first_entry;  // bh_stream.first_entry
  uint32_t count_cap;    // BH_STREAM_COUNT_IS_CAPACITY: nsym is the output capacity, the count is reported
  uint32_t spl;          // stream subsequences per lane ("virtual" subsequence = spl real ones)
  uint32_t sbr;          // stream subsequence bits (sb / spl)
  uint64_t nsub_r;       // real subsequences (gap array length)
  uint32_t wide;         // table layout: 1 = wlut12, 0 = replicated wlut8 (+ lut12 if has_l12)
  uint32_t t_lim, t_c12, t_wp, t_l12;  // shared-memory table offsets (bytes)
  uint32_t t_ljs, ljs_bytes;            // shared copy of ljsym for the limit search (0 bytes: global)
  uint32_t t_len;                       // len12 (wide modes)
  uint32_t smem_tiles;                  // ranges up to this many tiles keep their totals in shared memory
  // online tuner (tuner.py:117-191): 0 = off; else per-tile class -> staging
  // window, and the per-sequence class histogram of tuner.plan
  uint32_t t_high;
  uint32_t lanes_per_seq;               // lanes per reference sequence (0: the histogram is not exported)
  uint32_t sym_w;                       // Codebook.symbol_width
  uint32_t ref_seq_bits;                // LayoutConfig.seq_bits
  uint64_t nseq_ref;                    // reference sequences
  unsigned long long* class_freq;       // [t_high + 1] (zeroed before the launch)
  uint32_t cls_cap[TUNE_CLASSES];       // staging capacity per 1-based class (tuner.capacity)
  unsigned long long* trace;  // debug timeline (TR instantiation only)
};

constexpr unsigned long long FUSED_MARK = 0xF05EDull;  // rep->pad[2]: report written by k_fused

// Shared-memory table layouts inside the CTA (byte offsets, FusedArgs.t_*):
//   narrow (short codes): the 8-bit decode table wlut8 replicated 8 times
//     ([entry][8] uint4, 32 KB: an LDS.128 is served per quarter-warp, so
//     lane l reading replica l%8 never conflicts), lim, base, the 12-bit count
//     table, the packed wlut8 bulk-copy target (4 KB) and, for codes longer
//     than 8 bits, the 12-bit single-codeword table lut12 (16 KB);
//   wide (long codes, more than ~1.5 bits per symbol): the 12-bit decode
//     table wlut12 (64 KB, one lookup covers twice the bits), lim, base and
//     the count table.
constexpr uint32_t T_LIMBASE = 2 * 33 * 8;  // lim u64[33], base i64[33] (contiguous)
constexpr uint32_t T_NARROW_DEC = 256 * 8 * 16;
constexpr uint32_t T_WIDE_DEC = 16 * FB_SIZE;
constexpr uint32_t T_WIDE3_DEC = 8 * D3_SIZE;  // also holds cwin (CW_SIZE) in phase 1
// Decode-table modes (template parameter MODE of the kernel):
//   M_NARROW -- 8-bit window, up to six codewords, 16-byte entries replicated 8 ways;
//   M_WIDE   -- 12-bit window, up to six codewords, 16-byte entries (wlut12);
//   M_WIDE3  -- 13-bit window, up to three codewords, 8-byte entries (wlut3),
//               for books whose codes are all >= 4 bits: half the table, half
//               the shared-memory wavefronts per lookup and no store predicates.
constexpr int M_NARROW = 0, M_WIDE = 1, M_WIDE3 = 2;

// rep->pad[3] = epoch: the fused path declined this call (overrides every
// status; bh_decode reruns the reference-structured pipeline)
__device__ __forceinline__ void flag_need_staged(DevReport* rep, uint32_t ep) {
  *(volatile unsigned long long*)&rep->pad[3] = ep;
}

__device__ __forceinline__ void tag_status(DevReport* rep, uint32_t ep, uint32_t status) {
  unsigned long long v = ((unsigned long long)ep << 32) | (unsigned long long)(0x7fffffffu - status);
  atomicMax(&rep->pad[0], v);  // pad[0] = tagged status (see bh_report_read)
}

// Descriptors carry their value in the 64-bit word itself (epoch | flags |
// value), so readers need no ordering beyond the word: relaxed gpu-scope
// accesses avoid the release/acquire fences on the look-back's critical path.
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
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
__device__ __forceinline__ void sts16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}

// Keep a value in a register: the compiler may not rematerialise it (it
// otherwise recomputes shared-window addresses from SR_CgaCtaId in hot loops).
__device__ __forceinline__ uint32_t pin(uint32_t v) {
  asm volatile("mov.b32 %0, %0;" : "+r"(v));
  return v;
}

// Bit reader over a tile's staged words (tile-relative bit positions): the
// current and next word plus one prefetched word, and a bit offset.  peek is
// one funnel shift; skip advances by at most one word with selects and a
// predicated load of the word after next -- no branch, and the loaded word is
// only needed one advance later, so shared-memory latency stays off the
// decode chain.
// Staged tile words are skewed by one word per 32 (logical word j sits at
// physical word j + j/32): lanes read words about four apart (128-bit
// subsequences), which would put lanes l, l+8, l+16 and l+24 on one bank.
__device__ __forceinline__ uint32_t skew_addr(uint32_t base_s, uint32_t j) { return base_s + ((j + (j >> 5)) << 2); }

struct SR {
  uint32_t w0, w1, w2;  // MSB-first words at the cursor
  uint32_t off;         // bit offset into w0 (0..31)
  uint32_t wl;          // logical index of w2 (the word reloaded every step)
  uint32_t base;        // shared address of the tile buffer
  __device__ __forceinline__ void init(uint32_t base_s, uint32_t rel) {
    const uint32_t j = rel >> 5;
    base = pin(base_s);
    w0 = lds32(skew_addr(base_s, j));
    w1 = lds32(skew_addr(base_s, j + 1));
    w2 = lds32(skew_addr(base_s, j + 2));
    off = rel & 31;
    wl = j + 2;
  }
  __device__ __forceinline__ uint32_t peek() const { return __funnelshift_l(w1, w0, off); }
  __device__ __forceinline__ void skip(uint32_t n) {  // n <= 32
    const uint32_t t = off + n;
    const uint32_t adv = t >> 5;
    w0 = adv ? w1 : w0;
    w1 = adv ? w2 : w1;
    wl += adv;
#if BH_PSKIP
    // the word after w1, loaded only when the cursor crossed a word (a
    // predicated load: no shared-memory wavefront for lanes that did not)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t@p ld.shared.u32 %0, [%2];\n\t}"
                 : "+r"(w2) : "r"(adv), "r"(skew_addr(base, wl)) : "memory");
#else
    w2 = lds32(skew_addr(base, wl));  // the word after w1 (unchanged when adv == 0): no branch
#endif
    off = t & 31;
  }
};

struct FTab {
  uint32_t wl;     // decode table: this lane's replica of wlut8, or wlut12 (shared address)
  uint32_t dsh;    // window shift of the decode index: 24 (8-bit) or 20 (12-bit)
  uint32_t dst;    // entry stride shift: 7 (8 replicas x 16 B) or 4 (16 B)
  uint32_t l12;    // shared address of lut12
  uint32_t c12;    // shared address of clut12
  uint32_t cw;     // shared address of the 16-bit count table cwin (phase 1 of M_WIDE3; 0 = none)
  uint32_t len12;  // shared address of len12 (wide modes: first codeword length, resync walk)
  uint32_t ljs;    // shared address of the canonical symbol order (0: read it from global)
  uint32_t lim;    // shared address of lim (u64[33])
  uint32_t base;   // shared address of base (i64[33])
  TableView t;
  uint32_t kind;
  uint32_t max_len;  // longest code length of the book (seed candidates)
};

// one codeword from a 32-bit window when the 8-bit table cannot answer
__device__ __noinline__ uint32_t fslow(uint32_t win, const uint32_t lim_s, const uint32_t base_s,
                                       const uint16_t* __restrict__ ljsym, uint32_t kind, TableView t,
                                       uint32_t ljs_s) {
  if (kind == 0) {
    const uint2 l32 = lds64(lim_s + 32 * 8);
    if ((unsigned long long)win >= (((unsigned long long)l32.y << 32) | l32.x)) return 0;
    uint32_t lo = 1, hi = 32;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      const uint2 l = lds64(lim_s + mid * 8);
      if ((unsigned long long)win < (((unsigned long long)l.y << 32) | l.x)) hi = mid; else lo = mid + 1;
    }
    const uint2 bb = lds64(base_s + lo * 8);
    const long long idx = (long long)(((unsigned long long)bb.y << 32) | bb.x) + (long long)(win >> (32 - lo));
    const uint32_t sym = ljs_s ? lds16(ljs_s + 2 * (uint32_t)idx) : (uint32_t)__ldg(ljsym + idx);
    return sym | (lo << 16);
  }
  return slow_lookup(t, win);
}

// a code longer than 8 bits: shared 12-bit table, else the limit search
__device__ __forceinline__ uint32_t flong(uint32_t win, const FTab& T) {
  const uint32_t e = T.l12 ? lds32(T.l12 + ((win >> (32 - FB)) << 2)) : 0u;
  return e ? e : fslow(win, T.lim, T.base, T.t.ljsym, T.kind, T.t, T.ljs);
}

// one codeword: sym | len<<16 (0 = no codeword matches)
template <int MODE>
__device__ __forceinline__ uint32_t fone(uint32_t win, const FTab& T) {
  if (MODE == M_WIDE3) {
    const uint2 e = lds64(T.wl + ((win >> (32 - D3)) << 3));
    if (e.y) return (e.x & 0xffffu) | (((e.y >> 16) & 31u) << 16);
    return flong(win, T);
  }
  const uint4 w = lds128(T.wl + (MODE == M_WIDE ? (win >> (32 - FB)) << 4 : (win >> 24) << 7));
  if (w.w) return (w.x & 0xffffu) | (((w.w >> 16) & 15u) << 16);
  return flong(win, T);
}

// length of one codeword from the 12-bit count table (second start, or the end
// of the only whole codeword); codes longer than 12 bits take the limit search
// (wide modes: len12; the narrow mode keeps no len12 and reads the count table)
template <int MODE>
__device__ __forceinline__ uint32_t clen(uint32_t win, const FTab& T) {
  if (MODE == M_NARROW) {
    const uint32_t y = lds16(T.c12 + ((win >> (32 - FB)) << 1));
    if (y) {
      const uint32_t m = y & 0xffeu;
      return m ? __ffs(m) - 1 : (y >> 12);
    }
  } else {
    const uint32_t l = lds8(T.len12 + (win >> (32 - FB)));
    if (l) return l;
  }
  return (fslow(win, T.lim, T.base, T.t.ljsym, T.kind, T.t, T.ljs) >> 16) & 0xffu;
}

// count codewords starting in [pos, stop) (tile-relative); pos ends at the exit.
// 12-bit count table: every whole codeword of the next 12 bits per lookup
// (popcount of the start mask).  The one lookup that crosses `stop` counts the
// starts below it and exits at the first start at or past it; a code longer
// than 12 bits takes one codeword.
__device__ __forceinline__ bool fcount(SR& r, uint32_t& pos, uint32_t stop, const FTab& T, uint32_t& n) {
  const uint32_t ct = pin(T.c12);
  if (T.cw) {
    // 16-bit count table (M_WIDE3 phase 1): every whole codeword of the next
    // 16 bits per lookup (n | bits<<3), two lookups per advance; the window
    // end and codes longer than 16 bits fall through to the 12-bit loop below
    const uint32_t c5 = pin(T.cw);
    // bulk: two lookups (<= 32 bits) cannot cross `stop`; an empty second
    // entry (code longer than 16 bits after the first) adds nothing
    const int32_t bulk_end = (int32_t)stop - 2 * CW;
#pragma unroll (kUnroll)
    while ((int32_t)pos <= bulk_end) {
      const uint32_t win = r.peek();
      const uint32_t y = lds8(c5 + (win >> (32 - CW)));
      if (y == 0) break;
      const uint32_t b = y >> 3;
      const uint32_t y2 = lds8(c5 + ((win << b) >> (32 - CW)));  // b <= 16: the next 16 bits lie in win
      n += (y & 7u) + (y2 & 7u);
      const uint32_t adv = b + (y2 >> 3);
      r.skip(adv);
      pos += adv;
    }
#pragma unroll 1
    while (true) {
      const uint32_t win = r.peek();
      const uint32_t y = lds8(c5 + (win >> (32 - CW)));
      const uint32_t b = y >> 3;
      if (y == 0 || pos + b > stop) break;
      const uint32_t y2 = lds8(c5 + ((win << b) >> (32 - CW)));
      const uint32_t b2 = y2 >> 3;
      const bool two = y2 != 0 && pos + b + b2 <= stop;
      n += (y & 7u) + (two ? (y2 & 7u) : 0u);
      const uint32_t adv = b + (two ? b2 : 0u);
      r.skip(adv);
      pos += adv;
    }
  }
  while (pos < stop) {
    // tight loop: whole entries that end at or before the window end (one
    // extra lookup when an entry ends exactly at it)
    uint32_t y, b;
#if BH_TWO
    {
      // bulk: two lookups (<= 24 bits) cannot cross `stop`
      const int32_t bulk_end = (int32_t)stop - 2 * FB;
#pragma unroll (kUnroll)
      while ((int32_t)pos <= bulk_end) {
        const uint32_t win = r.peek();
        const uint32_t y1 = lds16(ct + ((win >> (32 - FB)) << 1));
        if (y1 == 0) break;
        const uint32_t y2 = lds16(ct + (((win << (y1 >> 12)) >> (32 - FB)) << 1));
        n += __popc(y1 & 0xfffu) + __popc(y2 & 0xfffu);
        const uint32_t adv = (y1 >> 12) + (y2 >> 12);
        r.skip(adv);
        pos += adv;
      }
    }
#endif
#pragma unroll (kUnroll)
    while (true) {
#if BH_TWO
      // two entries per advance: the second from the same 32-bit window
      // (b <= 12, so its 12 bits lie inside it)
      const uint32_t win = r.peek();
      y = lds16(ct + ((win >> (32 - FB)) << 1));
      b = y >> 12;
      if (y == 0 || pos + b > stop) break;
      const uint32_t y2 = lds16(ct + (((win << b) >> (32 - FB)) << 1));
      const uint32_t b2 = y2 >> 12;
      const bool two = y2 != 0 && pos + b + b2 <= stop;
      n += __popc(y & 0xfffu) + (two ? __popc(y2 & 0xfffu) : 0u);
      const uint32_t adv = b + (two ? b2 : 0u);
      r.skip(adv);
      pos += adv;
#else
      y = lds16(ct + ((r.peek() >> (32 - FB)) << 1));
      b = y >> 12;
      if (y == 0 || pos + b > stop) break;
      n += __popc(y & 0xfffu);
      r.skip(b);
      pos += b;
#endif
    }
    if (pos >= stop) break;
    if (!y) {  // first code longer than 12 bits
      const uint32_t l = (fslow(r.peek(), T.lim, T.base, T.t.ljsym, T.kind, T.t, T.ljs) >> 16) & 0xffu;
      if (!l) return false;
      n += 1;
      r.skip(l);
      pos += l;
      continue;
    }
    // the window ends inside this entry (stop - pos < b <= 12)
    const uint32_t rem = stop - pos;
    const uint32_t mask = y & 0xfffu;
    n += __popc(mask & ((1u << rem) - 1u));
    const uint32_t hi = mask >> rem;
    const uint32_t adv = hi ? rem + __ffs(hi) - 1 : b;
    r.skip(adv);
    pos += adv;
  }
  return true;
}

// idx * 8 + base as one integer multiply-add (the compiler would otherwise
// fold the shift into a mask and add: three ALU instructions)
__device__ __forceinline__ uint32_t mad8(uint32_t idx, uint32_t base) {
  uint32_t a;
  asm("mad.lo.u32 %0, %1, 8, %2;" : "=r"(a) : "r"(idx), "r"(base));
  return a;
}

// Decode c (>= 1) symbols into compact staging at `dst`.  While at least six
// symbols remain, all six symbols of a table entry are stored unconditionally
// (the ones past the entry's count land inside the lane's own range and are
// overwritten by its next stores); the last entries store predicated, so lane
// ranges stay disjoint even for corrupt (non-contiguous) windows.
// Three-codeword entries (M_WIDE3): per lookup one halfword store and two word
// stores, unconditionally -- an even start writes s0|s1 and s2 (plus junk in
// the high half), an odd start s0 then s1|s2 (plus a junk word) -- at most 10
// bytes, all inside the lane's remaining range while >= 10 bytes remain, and
// overwritten by its next stores.
// The three symbol slots of a three-codeword entry at staging byte address
// dst (6 bytes): BH_HW3 1 -- three halfword stores; 2 -- one aligned word
// and one halfword (even start: s0|s1, then s2; odd: s0, then s1|s2), one
// shared-memory store instruction fewer per entry
__device__ __forceinline__ void st3(uint32_t dst, uint2 e) {
#if BH_HW3 == 2
  const uint32_t odd = dst & 2u;
#if BH_PST
  // only the stores the entry's count reaches (predicated: fewer active
  // lanes, fewer bank conflicts): even start -- the halfword only for a
  // third symbol; odd start -- the word only for a second
  const uint32_t n = e.y >> 29;
  if (odd ? n > 1 : true) sts32(dst + odd, odd ? __funnelshift_r(e.x, e.y, 16) : e.x);
  if (odd ? true : n > 2) sts16(dst + 4 - 2 * odd, odd ? e.x : e.y);
#else
  sts32(dst + odd, odd ? __funnelshift_r(e.x, e.y, 16) : e.x);
  sts16(dst + 4 - 2 * odd, odd ? e.x : e.y);
#endif
#else
  sts16(dst, e.x);
  sts16(dst + 2, e.x >> 16);
  sts16(dst + 4, e.y);
#endif
}

__device__ __forceinline__ bool fdecode3(SR& r, uint32_t c, uint32_t dst, const FTab& T) {
  const uint32_t wl = pin(T.wl);
  int32_t k2 = 2 * (int32_t)c;  // remaining staging bytes
  while (k2 > 0) {
#if BH_TWO
    // two entries per advance (the second from the same 32-bit window); they
    // write at most 6 + 6 bytes (BH_HW3) or 6 + 10
#pragma unroll (kUnroll)
    while (k2 >= (BH_HW3 ? 12 : 16)) {
      const uint32_t win = r.peek();
      const uint2 e = lds64(mad8(win >> (32 - D3), wl));
      if (!e.y) break;
      const uint32_t b1 = (e.y >> 24) & 15u;
      const uint2 f = lds64(mad8((win << b1) >> (32 - D3), wl));
#if BH_HW3
      // every symbol slot of both entries (st3); slots past an entry's count
      // hold junk inside the lane's range, overwritten by its next stores
      st3(dst, e);
      dst += e.y >> 28;
      st3(dst, f);
      const uint32_t nf = f.y >> 28;
      dst += nf;
      k2 -= (int32_t)((e.y >> 28) + nf);
      r.skip(b1 + ((f.y >> 24) & 15u));
      continue;
#endif
      uint32_t odd = dst & 2u, a4 = dst + odd;
      sts16(dst, e.x);
      sts32(a4, __funnelshift_r(e.x, e.y, odd << 3));
      sts32(a4 + 4, e.y);
      dst += e.y >> 28;
      // the second entry unconditionally: a long code there (f.y == 0) writes
      // zero-length junk inside the lane's range and advances nothing
      odd = dst & 2u;
      a4 = dst + odd;
      sts16(dst, f.x);
      sts32(a4, __funnelshift_r(f.x, f.y, odd << 3));
      sts32(a4 + 4, f.y);
      const uint32_t nb2 = f.y >> 28;
      dst += nb2;
      k2 -= (int32_t)((e.y >> 28) + nb2);
      r.skip(b1 + ((f.y >> 24) & 15u));
    }
#endif
#pragma unroll (kUnroll)
    while (k2 >= (BH_HW3 ? 6 : 10)) {
      const uint2 e = lds64(wl + ((r.peek() >> (32 - D3)) << 3));
      if (!e.y) break;  // a code longer than 12 bits: one codeword below
#if BH_HW3
      st3(dst, e);
      dst += e.y >> 28;
      k2 -= (int32_t)(e.y >> 28);
      r.skip((e.y >> 24) & 15u);
      continue;
#endif
      const uint32_t odd = dst & 2u;
      const uint32_t a4 = dst + odd;
      sts16(dst, e.x);
      sts32(a4, __funnelshift_r(e.x, e.y, odd << 3));  // even: s0|s1, odd: s1|s2
      sts32(a4 + 4, e.y);                              // even: s2 (+ junk), odd: junk
      const uint32_t nb = e.y >> 28;                   // 2n: bytes of staging written
      dst += nb;
      k2 -= (int32_t)nb;
      r.skip((e.y >> 24) & 15u);
    }
    if (k2 <= 0) break;
    const uint32_t win = r.peek();
    const uint2 e = lds64(wl + ((win >> (32 - D3)) << 3));
    if (e.y) {
      const int32_t n = (int32_t)(e.y >> 29), k = k2 >> 1;
      const int32_t m = n < k ? n : k;
      sts16(dst, e.x);
      if (m > 1) sts16(dst + 2, e.x >> 16);
      if (m > 2) sts16(dst + 4, e.y);
      dst += (uint32_t)n << 1;
      k2 -= 2 * n;
      r.skip((e.y >> 24) & 15u);
    } else {
      const uint32_t el = flong(win, T);
      const uint32_t len = (el >> 16) & 0xffu;
      if (!len) return false;
      sts16(dst, el);
      dst += 2;
      k2 -= 2;
      r.skip(len);
    }
  }
  return true;
}

template <int MODE>
__device__ __forceinline__ bool fdecode(SR& r, uint32_t c, uint32_t dst, const FTab& T) {
  if (MODE == M_WIDE3) return fdecode3(r, c, dst, T);
  constexpr uint32_t dsh = MODE == M_WIDE ? 32 - FB : 24, dstr = MODE == M_WIDE ? 4 : 7;
  const uint32_t wl = pin(T.wl);
  int32_t k = (int32_t)c;
  while (k > 0) {
    // tight loop: whole entries while at least seven symbols remain; one
    // halfword store, then three aligned word stores (an odd start shifts the
    // entry by one halfword; the seventh halfword written is garbage inside
    // the lane's own range, overwritten by its next store)
    int32_t k2 = 2 * k;  // remaining staging bytes
#pragma unroll (kUnroll)
    while (k2 >= 14) {
      const uint4 w = lds128(wl + ((r.peek() >> dsh) << dstr));
      if (!w.w) break;  // a code the table does not hold: one entry below
      const uint32_t odd = dst & 2u;                   // halfword-odd start
      const uint32_t sel = 0x3210u + odd * 0x1111u;    // 0x5432 when odd
      const uint32_t a4 = dst + odd;                   // first aligned word after it
      const uint32_t nb = w.w >> 28;                   // 2n: bytes of staging written
      if (odd) sts16(dst, w.x);  // an even start is covered by the first word
      sts32(a4, __byte_perm(w.x, w.y, sel));
      // the last two words only when the entry reaches them (fewer, less
      // conflicted shared-memory wavefronts)
      if (nb > 4 + odd) sts32(a4 + 4, __byte_perm(w.y, w.z, sel));  // symbol 2 (3 if odd) present
      if (nb > 8 + odd) sts32(a4 + 8, __byte_perm(w.z, w.z, sel));  // symbol 4 (5 if odd) present
      dst += nb;
      k2 -= (int32_t)nb;
      r.skip(w.w & 15u);
    }
    k = k2 >> 1;
    if (k <= 0) break;
    // one entry with predicated stores: the last few symbols, or a long code
    const uint32_t win = r.peek();
    const uint4 w = lds128(wl + ((win >> dsh) << dstr));
    if (w.w) {
      const int32_t n = (int32_t)((w.w >> 4) & 15u);
      const int32_t m = n < k ? n : k;
      sts16(dst, w.x);
      if (m > 1) sts16(dst + 2, w.x >> 16);
      if (m > 2) sts16(dst + 4, w.y);
      if (m > 3) sts16(dst + 6, w.y >> 16);
      if (m > 4) sts16(dst + 8, w.z);
      if (m > 5) sts16(dst + 10, w.z >> 16);
      dst += (uint32_t)n << 1;
      k -= n;
      r.skip(w.w & 15u);
    } else {
      const uint32_t e = flong(win, T);
      const uint32_t len = (e >> 16) & 0xffu;
      if (!len) return false;
      sts16(dst, e);
      dst += 2;
      k -= 1;
      r.skip(len);
    }
  }
  return true;
}

// bypass: decode straight to global memory (rare; guarded by the output size)
template <int MODE>
__device__ bool fdecode_global(SR& r, uint32_t c, uint16_t* out, uint64_t at, uint64_t nsym, const FTab& T) {
  for (uint32_t k = 0; k < c; ++k) {
    const uint32_t s = fone<MODE>(r.peek(), T);
    const uint32_t len = (s >> 16) & 0xffu;
    if (!len) return false;
    if (at + k < nsym) out[at + k] = (uint16_t)s;
    r.skip(len);
  }
  return true;
}

// Re-decode a window from a new entry, walking the previous decode (entry eo,
// count co, exit xo) in lock-step; once both cursors meet the rest is shared
// (sync_decoder.py:90-101).  The lower cursor advances a whole 12-bit count
// table entry at a time: its start mask says at once whether the other
// cursor's position is one of its codeword starts (the parses meet there) or
// lies between two of them, so no codeword is stepped singly except codes
// longer than 12 bits.
// Per-codeword lock-step walk: cheaper than the mask walk when a 12-bit entry
// holds only a couple of codewords (long-code books, wide layout).
template <int MODE>
__device__ __forceinline__ bool resync_step(uint32_t base_s, uint32_t eo, uint32_t co, uint32_t xo, uint32_t en,
                                            uint32_t stop, const FTab& T, uint32_t& cn, uint32_t& xn) {
  uint32_t po = eo, pn = en, no = 0, nn = 0;
  SR ro, rn;
  ro.init(base_s, po);
  rn.init(base_s, pn);
  while (true) {
    if (pn >= stop) { cn = nn; xn = pn; return true; }
    if (po == pn) { cn = nn + (co - no); xn = xo; return true; }
    if (po < pn) {
      const uint32_t l = clen<MODE>(ro.peek(), T);
      if (!l) return false;
      ro.skip(l);
      po += l;
      ++no;
    } else {
      const uint32_t l = clen<MODE>(rn.peek(), T);
      if (!l) return false;
      rn.skip(l);
      pn += l;
      ++nn;
    }
  }
}

// Overlap pre-synchronisation (self-sync count phase): the first codeword
// start at or after boundary b of the parse entered at p < b, walked a whole
// 12-bit count-table entry at a time (start mask + end).  A parse entered K
// bits early has almost always synchronised with the true one by b, so the
// result is the lane's true entry far more often than b itself: the intra-
// sequence rounds then find the predecessor's exit equal to it and skip the
// re-decode.  Any result is correct (the rounds re-synchronise a wrong one).
template <int MODE>
__device__ __forceinline__ uint32_t presync(uint32_t base_s, uint32_t p, uint32_t b, const FTab& T) {
  SR r;
  r.init(base_s, p);
  const uint32_t ct = T.c12;
#pragma unroll 1
  while (true) {
    const uint32_t win = r.peek();
    const uint32_t y = lds16(ct + ((win >> (32 - FB)) << 1));
    if (!y) {  // a code longer than 12 bits
      const uint32_t l = (fslow(win, T.lim, T.base, T.t.ljsym, T.kind, T.t, T.ljs) >> 16) & 0xffu;
      if (!l) return b;
      p += l;
      if (p >= b) return p;
      r.skip(l);
      continue;
    }
    const uint32_t mask = y & 0xfffu, end = y >> 12, d = b - p;
    if (d < end) {
      const uint32_t hi = mask >> d;
      return hi ? b + __ffs(hi) - 1 : p + end;
    }
    p += end;
    if (p == b) return b;
    r.skip(end);
  }
}

// Seam walk (self-sync, a seam inside the CTA's range): the parse entered at
// the true seed en against the first slot's own parse from eo, codeword by
// codeword, until they meet (sync_decoder.py:90-101).  delta = seed-parse
// codewords minus own-parse codewords before the meeting point, so the slot's
// count for the seed is its own count + delta and its exit is unchanged.
// False when they do not meet below `stop` (the slot's exit may change) or
// below `lim` (the end of the staged words).
template <int MODE>
__device__ __forceinline__ bool seam_walk(uint32_t base_s, uint32_t eo, uint32_t en, uint32_t stop, uint32_t lim,
                                          const FTab& T, int32_t& delta) {
  delta = 0;
  uint32_t po = eo, pn = en;
  if (po == pn) return true;
  int32_t d = 0;
  SR ro, rn;
  ro.init(base_s, po);
  rn.init(base_s, pn);
  while (po != pn) {
    const bool adv_o = po < pn;
    const uint32_t lo = adv_o ? po : pn;
    if (lo >= stop || lo >= lim) return false;
    const uint32_t l = clen<MODE>(adv_o ? ro.peek() : rn.peek(), T);
    if (!l) return false;
    if (adv_o) { ro.skip(l); po += l; --d; }
    else { rn.skip(l); pn += l; ++d; }
  }
  delta = d;
  return true;
}

template <int MODE>
__device__ __forceinline__ bool resync(uint32_t base_s, uint32_t eo, uint32_t co, uint32_t xo, uint32_t en,
                                       uint32_t stop, const FTab& T, uint32_t& cn, uint32_t& xn) {
  // long-code books (wide layouts): a 12-bit entry holds a codeword or two, so
  // the plain per-codeword walk is cheaper there
  if (MODE != M_NARROW) return resync_step<MODE>(base_s, eo, co, xo, en, stop, T, cn, xn);
  uint32_t po = eo, pn = en, no = 0, nn = 0;
  SR ro, rn;
  ro.init(base_s, po);
  rn.init(base_s, pn);
  const uint32_t ct = T.c12;
  while (true) {
    if (pn >= stop) { cn = nn; xn = pn; return true; }
    if (po == pn) { cn = nn + (co - no); xn = xo; return true; }
    if (po < pn) {  // the old parse is behind: advance it a whole entry
      const uint32_t win = ro.peek();
      const uint32_t y = lds16(ct + ((win >> (32 - FB)) << 1));
      if (!y) {  // a code longer than 12 bits: one codeword
        const uint32_t l = (fslow(win, T.lim, T.base, T.t.ljsym, T.kind, T.t, T.ljs) >> 16) & 0xffu;
        if (!l) return false;
        ro.skip(l);
        po += l;
        ++no;
        continue;
      }
      const uint32_t mask = y & 0xfffu, b = y >> 12, d = pn - po;
      uint32_t adv;
      if (d < b) {
        if ((mask >> d) & 1u) {  // the old parse has a start where the new one is: they meet
          no += __popc(mask & ((1u << d) - 1u));
          po = pn;
          continue;
        }
        const uint32_t hi = mask >> d;  // step over it to the first start after it
        adv = hi ? d + __ffs(hi) - 1 : b;
        no += __popc(mask & ((1u << adv) - 1u));
      } else {
        adv = b;
        no += __popc(mask);
      }
      ro.skip(adv);
      po += adv;
    } else {  // the new parse is behind: advance it, never past the window end
      const uint32_t win = rn.peek();
      const uint32_t y = lds16(ct + ((win >> (32 - FB)) << 1));
      if (!y) {
        const uint32_t l = (fslow(win, T.lim, T.base, T.t.ljsym, T.kind, T.t, T.ljs) >> 16) & 0xffu;
        if (!l) return false;
        rn.skip(l);
        pn += l;
        ++nn;
        continue;
      }
      const uint32_t mask = y & 0xfffu, b = y >> 12, d = po - pn, rem = stop - pn;
      uint32_t adv;
      if (d < b && ((mask >> d) & 1u) && d < rem) {  // meet before the window end
        nn += __popc(mask & ((1u << d) - 1u));
        pn = po;
        continue;
      }
      if (rem < b) {  // the window ends inside this entry
        nn += __popc(mask & ((1u << rem) - 1u));
        const uint32_t hi = mask >> rem;
        adv = hi ? rem + __ffs(hi) - 1 : b;
      } else if (d < b) {
        const uint32_t hi = mask >> d;
        adv = hi ? d + __ffs(hi) - 1 : b;
        nn += __popc(mask & ((1u << adv) - 1u));
      } else {
        adv = b;
        nn += __popc(mask);
      }
      rn.skip(adv);
      pn += adv;
    }
  }
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ uint32_t mbar_test(uint32_t bar, uint32_t parity) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(r) : "r"(bar), "r"(parity) : "memory");
  return r;
}
// bulk (TMA) copy global -> shared, completing on the mbarrier
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                              uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(pol) : "memory");
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// Per-warp word staging: one bulk (TMA) copy of a tile's words into the
// warp's landing buffer, completing on the warp's own mbarrier; skew_in()
// then spreads them into the skewed decode buffer.  At most one copy is in
// flight per warp (wstage_wait consumes it).
struct WStage {
  uint32_t bar;    // shared address of the warp's mbarrier
  uint32_t phase;  // parity of the next completion
  bool pending;
};

__device__ __forceinline__ void wstage_init(WStage& ws, uint32_t bar) {
  ws.bar = bar;
  ws.phase = 0;
  ws.pending = false;
  if ((threadIdx.x & 31) == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
}

// Stage the words of `tile`; returns the bit offset of logical word 0.  The
// caller has synced the warp after its last read of the landing buffer.
__device__ __forceinline__ uint64_t stage_words(const FusedArgs& a, uint64_t tile, uint32_t land_s, uint32_t& nch,
                                                WStage& ws, bool last_use = false) {
  const uint64_t s0 = tile * (uint64_t)a.seq_bits;
  uint64_t w0 = (s0 >> 5) & ~3ull;
  w0 = w0 >= a.lead ? w0 - a.lead : 0;
  uint64_t w1 = ((s0 + a.seq_bits) >> 5) + a.halo;
  w1 = (w1 + 3) & ~3ull;
  if (w1 > a.words_alloc) w1 = a.words_alloc;
  nch = (uint32_t)((w1 - w0) >> 2);
  if ((threadIdx.x & 31) == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier reads of the buffer -> async proxy
    if (nch) {
      mbar_expect_tx(ws.bar, 16 * nch);
      if (BH_L2HINT >= 2 && last_use) bulk_g2s_hint(land_s, a.words + w0, 16 * nch, ws.bar, l2_evict_first());
      else bulk_g2s(land_s, a.words + w0, 16 * nch, ws.bar);
    } else {
      mbar_arrive(ws.bar);
    }
  }
  ws.pending = true;
  return w0 * 32;
}

__device__ __forceinline__ void wstage_wait(WStage& ws) {
  if (!ws.pending) return;
  mbar_wait(ws.bar, ws.phase);
  ws.phase ^= 1u;
  ws.pending = false;
}

// landing buffer (contiguous) -> decode buffer (skew_addr layout); the caller
// waits for the cp.async group and syncs the warp on both sides
__device__ __forceinline__ void skew_in(uint32_t land_s, uint32_t buf_s, uint32_t nch) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t c = lane; c < nch; c += 32) {
    const uint4 v = lds128(land_s + 16 * c);
    sts32(skew_addr(buf_s, 4 * c), v.x);
    sts32(skew_addr(buf_s, 4 * c + 1), v.y);
    sts32(skew_addr(buf_s, 4 * c + 2), v.z);
    sts32(skew_addr(buf_s, 4 * c + 3), v.w);
  }
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

// Flush [P, P+C) from compact staging (stg symbol i <-> output P+i).  Whole
// aligned chunks: two aligned 128-bit shared loads shifted by the tile's
// (uniform) misalignment, one 128-bit global store; the two edge chunks, shared
// with the neighbouring tiles, element by element.
__device__ __forceinline__ void flush_compact(uint16_t* __restrict__ out, uint64_t nsym, uint64_t P, uint32_t C,
                                              uint32_t stg_s) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t g1 = P + C;
  const uint64_t f0 = (P + 7) & ~7ull;                   // first whole chunk
  const uint64_t f1 = (g1 < nsym ? g1 : nsym) & ~7ull;   // end of whole chunks
  const uint32_t sh = (uint32_t)(f0 - P) & 7u;           // uniform shift
  if (f1 > f0) {
    const uint32_t nfull = (uint32_t)((f1 - f0) >> 3);
    const uint32_t s0 = (uint32_t)(f0 - P) & ~7u;        // 16B-aligned staging index of chunk 0
    for (uint32_t ch = lane; ch < nfull; ch += 32) {
      const uint32_t q = stg_s + 2 * (s0 + 8 * ch);
      const uint4 A = lds128(q);
      const uint4 v = sh ? shift_hw(A, lds128(q + 16), sh) : A;
      *reinterpret_cast<uint4*>(out + f0 + 8ull * ch) = v;
    }
  }
  // head [P, min(f0, g1)) and tail [max(f1, P), g1): at most 7 + 7 + (overlap) elements
  const uint64_t hend = f0 < g1 ? f0 : g1;
  const uint64_t tbeg = f1 > hend ? f1 : hend;
  const uint32_t nh = (uint32_t)(hend - P), nt = (uint32_t)(g1 - tbeg);
  if (lane < nh) {
    const uint64_t g = P + lane;
    if (g < nsym) out[g] = (uint16_t)lds16(stg_s + 2 * lane);
  } else if (lane >= 8 && lane - 8 < nt) {
    const uint64_t g = tbeg + (lane - 8);
    if (g < nsym) out[g] = (uint16_t)lds16(stg_s + 2 * (uint32_t)(g - P));
  }
}

// Flush [P, P+C) from staging aligned to the output (stg symbol i <-> output
// (P & ~7) + i): the whole 16-byte chunks leave shared memory
// as ONE bulk (TMA) copy issued by lane 0 -- no registers or load/store
// instructions per chunk.  The staging must not be rewritten before the copy
// has read it (bulk_read_wait).  Returns whether a copy was issued.
__device__ __forceinline__ bool flush_bulk(uint16_t* __restrict__ out, uint64_t nsym, uint64_t P, uint32_t C,
                                           uint32_t stg_s) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t a0 = P & ~7ull, g1 = P + C;
  const uint64_t f0 = (P + 7) & ~7ull;
  const uint64_t f1 = (g1 < nsym ? g1 : nsym) & ~7ull;
  const bool bulk = f1 > f0;
  if (bulk && lane == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // staging stores -> async proxy
    if (BH_L2HINT >= 1)  // the output is not read again: keep the payload in L2 instead
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                   ::"l"(out + f0), "r"(stg_s + 2 * (uint32_t)(f0 - a0)), "r"((uint32_t)(2 * (f1 - f0))),
                   "l"(l2_evict_first()) : "memory");
    else
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   ::"l"(out + f0), "r"(stg_s + 2 * (uint32_t)(f0 - a0)), "r"((uint32_t)(2 * (f1 - f0)))
                   : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  const uint64_t hend = f0 < g1 ? f0 : g1;
  const uint64_t tbeg = f1 > hend ? f1 : hend;
  const uint32_t nh = (uint32_t)(hend - P), nt = (uint32_t)(g1 - tbeg);
  if (lane < nh) {
    const uint64_t g = P + lane;
    if (g < nsym) out[g] = (uint16_t)lds16(stg_s + 2 * (uint32_t)(g - a0));
  } else if (lane >= 8 && lane - 8 < nt) {
    const uint64_t g = tbeg + (lane - 8);
    if (g < nsym) out[g] = (uint16_t)lds16(stg_s + 2 * (uint32_t)(g - a0));
  }
  return bulk;
}
__device__ __forceinline__ void bulk_read_wait() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// 128-bit flush of [g0, g0+len) from staging aligned to g0 (stg[0] <-> g0 & ~7)
__device__ __forceinline__ void flush_aligned(uint16_t* __restrict__ out, uint64_t nsym, uint64_t g0, uint32_t len,
                                              const uint16_t* stg) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t a0 = g0 & ~7ull, g1 = g0 + len;
  const uint32_t nch = (uint32_t)((g1 - a0 + 7) >> 3);
  for (uint32_t ch = lane; ch < nch; ch += 32) {
    const uint64_t ga = a0 + (uint64_t)ch * 8;
    if (ga >= g0 && ga + 8 <= g1 && ga + 8 <= nsym) {
      *reinterpret_cast<uint4*>(out + ga) = *reinterpret_cast<const uint4*>(stg + ch * 8);
    } else {
      for (uint32_t i = 0; i < 8; ++i) {
        const uint64_t gi = ga + i;
        if (gi >= g0 && gi < g1 && gi < nsym) out[gi] = stg[ch * 8 + i];
      }
    }
  }
}

// The seam candidates of a tile's first slot (inter_sync, sync_decoder.py:
// 116-149): for every seed offset o < max_len, the codewords the slot holds
// when entered at b0 + o, and its exit.  Instead of one lock-step walk per
// candidate, the warp reads the length of the codeword at each of the first
// 32 NG bit offsets once (lane p: offsets p, 32 + p, ...), marks the starts of the
// parse from b0 in a bit mask, and then every candidate follows its own
// parse with shuffles of those lengths until it lands on a start of the b0
// parse (from there both parses coincide: count = own codewords so far +
// the b0 parse's codewords from that start), reaches the slot end, or leaves
// the window (then the lock-step walk finishes it).
#ifndef BH_CHASE_G
#define BH_CHASE_G 2  // 32-bit groups of offsets the chase covers (64 bits: faster than 96 or 128)
#endif
template <int MODE>
__device__ __forceinline__ void cand_chase(uint32_t base_s, uint32_t b0, uint32_t c0, uint32_t x0, uint32_t stop0,
                                           const FTab& T, uint32_t& cand_c, uint32_t& cand_x) {
  constexpr uint32_t NG = BH_CHASE_G, WIN = 32 * NG;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t span = stop0 > b0 ? stop0 - b0 : 0u;
  const uint32_t p0 = b0 + lane, j = p0 >> 5, off = p0 & 31;
  uint32_t L[NG];  // L[g]: length of the codeword at offset 32 g + lane
  {
    uint32_t wa = lds32(skew_addr(base_s, j));
#pragma unroll
    for (uint32_t g = 0; g < NG; ++g) {
      const uint32_t wb = lds32(skew_addr(base_s, j + 1 + g));
      L[g] = clen<MODE>(__funnelshift_l(wb, wa, off), T);
      wa = wb;
    }
  }
  auto len_at = [&](uint32_t p) -> uint32_t {  // every lane calls it (shuffles)
    uint32_t v = 0;
#pragma unroll
    for (uint32_t g = 0; g < NG; ++g) {
      const uint32_t x = __shfl_sync(0xffffffffu, L[g], p & 31);
      v = (p >> 5) == g ? x : v;
    }
    return v;
  };
  // starts of the parse from b0 inside [0, min(span, WIN))
  const uint32_t lim = min(span, WIN);
  unsigned long long M0 = 0, M1 = 0;
  for (uint32_t p = 0; p < lim;) {
    if (p < 64) M0 |= 1ull << p; else M1 |= 1ull << (p - 64);
    const uint32_t l = len_at(p);
    if (!l) break;
    p += l;
  }
  // every candidate lane follows its own parse
  const bool cand = lane < T.max_len;
  uint32_t q = lane, k = 0, how = cand ? 0u : 4u;  // 0 running, 1 met, 2 slot end, 3 left the window, 4 invalid / none
  while (__any_sync(0xffffffffu, how == 0)) {
    const uint32_t l = len_at(q);
    if (how == 0) {
      const bool inM = q < 64 ? ((M0 >> q) & 1ull) : q < WIN ? ((M1 >> (q - 64)) & 1ull) : false;
      if (q >= span) how = 2;
      else if (q >= WIN) how = 3;
      else if (inM) how = 1;
      else if (!l) how = 4;
      else { q += l; ++k; }
    }
  }
  if (!cand) return;
  if (how == 1) {
    const uint32_t before = q < 64 ? (uint32_t)__popcll(M0 & ((1ull << q) - 1ull))
                                   : (uint32_t)__popcll(M0) + (uint32_t)__popcll(M1 & ((1ull << (q - 64)) - 1ull));
    cand_c = k + c0 - before;
    cand_x = x0;
  } else if (how == 2) {
    cand_c = k;
    cand_x = b0 + q;
  } else if (how == 3) {
    uint32_t cn, xn;
    if (resync<MODE>(base_s, b0, c0, x0, b0 + q, stop0, T, cn, xn)) { cand_c = k + cn; cand_x = xn; }
    else cand_x = 0xffffffffu;
  } else {
    cand_x = 0xffffffffu;  // no codeword matches from this seed
  }
}

// Entries and counts of one tile (lane = subsequence); positions are relative
// to the tile buffer's first bit `wb0`.  GAP: boundary + gap byte; SYNC:
// intra-sequence chain rounds plus the seam seed from the predecessor tile's
// published final exit.
// SYNC modes: seed_o < 0 -- speculative (lane 0 entered at its boundary); the
// counts of the first slot for all 32 candidate seeds go to cand_c, and the
// tile publishes its exit when no candidate changes it (else a DEP marker);
// seed_o >= 0 -- the true seed offset is known: the final state is computed
// and the exit published.
template <int VAR, int MODE>
__device__ __forceinline__ void tile_counts(const FusedArgs& a, const FTab& T, uint64_t tile, uint32_t base_s,
                                            uint64_t wb0, uint32_t nsl, uint32_t ep, uint32_t& e, uint32_t& c,
                                            bool& bad, int32_t seed_o = -1, uint32_t* cand_out = nullptr,
                                            bool* fullfix = nullptr, const uint32_t* gpre = nullptr,
                                            unsigned long long* desc_out = nullptr, bool chase = true,
                                            uint32_t* xlast_out = nullptr) {
  bool resync_needed = false;  // GAP, spl > 1: an inner gap entry is not a codeword start
  const uint32_t lane = threadIdx.x & 31;
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
    // gpre: this lane's gap byte and lane 31's successor, prefetched by the caller
    // virtual subsequence j starts at real subsequence j * spl (its gap byte)
    const uint32_t g = gpre ? gpre[0] : (active ? a.gap[j * a.spl] : 0u);
    uint32_t gn = __shfl_down_sync(0xffffffffu, g, 1);
    if (lane == nsl - 1) gn = gpre && nsl == 32 ? gpre[1] : ((j + 1 < a.nsub) ? a.gap[(j + 1) * a.spl] : 0u);
    e = b + g;
    stop = (j + 1 < a.nsub) ? b + sb + gn : tbr;
    if (stop > tbr) stop = tbr;
    x = e;
    if (active && e < stop) {
      SR r;
      r.init(base_s, e);
      // a lane spanning spl stream subsequences checks that every inner gap
      // entry is one of its codeword starts (then the reference's windows
      // hold exactly the same codewords); a corrupt inner entry sends the
      // decode to the reference-structured pipeline, which reproduces the
      // reference's error
      const uint32_t sbr = a.sbr;
      for (uint32_t k = 1; k < a.spl; ++k) {
        const uint64_t jr = j * a.spl + k;
        if (jr >= a.nsub_r) break;
        const uint32_t ek = b + k * sbr + a.gap[jr];
        if (ek < x || ek > stop) { resync_needed = true; break; }
        if (!fcount(r, x, ek, T, c)) bad = true;
        if (x != ek) { resync_needed = true; break; }
      }
      if (!fcount(r, x, stop, T, c)) bad = true;
    }
  } else {
    stop = min(b + sb, tbr);
    if (tile == 0 && lane == 0) e = x = b + a.first_entry;  // chunk of a longer stream
    // entry guess: pre-synchronised from `presync` bits before the boundary,
    // except for a first slot resolved by candidate seeds (they count from
    // b).  The pre-window is counted by the same count loop (its exit is the
    // first start at or after b), and the reader continues from there.
    const bool pre = PRESYNC_BY_COUNT && a.presync && active && !(tile == 0 && lane == 0) && (lane > 0 || !chase);
    if (!PRESYNC_BY_COUNT && a.presync && active && !(tile == 0 && lane == 0) && (lane > 0 || !chase))
      e = x = presync<MODE>(base_s, b > a.presync ? b - a.presync : 0u, b, T);
    if (active && (pre || e < stop)) {
      SR r;
      if (pre) {
        uint32_t p = b > a.presync ? b - a.presync : 0u, nd = 0;
        r.init(base_s, p);
        if (fcount(r, p, b, T, nd)) {
          e = x = p;
        } else {
          e = x = b;
          r.init(base_s, b);
        }
      } else {
        r.init(base_s, e);
      }
      if (e < stop && !fcount(r, x, stop, T, c)) bad = true;
    }
    bool dprev = active;
#ifdef BH_X_NOINTRA  // timing experiment only: no intra-sequence rounds (wrong output)
    dprev = false;
#endif
    while (true) {
      const uint32_t xin = __shfl_up_sync(0xffffffffu, x, 1);
      const bool din = __shfl_up_sync(0xffffffffu, dprev, 1);
      const bool live = lane >= 1 && active && din;
      if (!__any_sync(0xffffffffu, live)) break;
      bool dnow = false;
      if (live && xin != e) {
        uint32_t cn, xn;
        if (!resync<MODE>(base_s, e, c, x, xin, stop, T, cn, xn)) bad = true;
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
    if (tile > 0 && chase) {
      // the true seed lies within the codeword straddling the boundary, so
      // only offsets below the longest code length are candidates
#ifndef BH_X_NOCAND
      if (MODE != M_NARROW) {
        cand_chase<MODE>(base_s, b0, c0, x0, stop0, T, cand_c, cand_x);
      } else if (lane < T.max_len) {
        // short codes: the entry-at-a-time mask walk is cheaper than a chase
        // over 64 offsets (up to 64 codewords)
        if (!resync<MODE>(base_s, b0, c0, x0, b0 + lane, stop0, T, cand_c, cand_x)) cand_x = 0xffffffffu;
      }
#endif
      indep = __all_sync(0xffffffffu, cand_x == x0);
    }
    const uint32_t xlast = __shfl_sync(0xffffffffu, x, nsl - 1);
    if (xlast_out) *xlast_out = xlast;
    if (seed_o < 0 && !indep) {
      // The candidates disagree after the first slot: follow the candidate
      // set through the next slots (lane j carries seed j) until it collapses
      // onto the speculative chain.  Then the tile's exit is still
      // seed-independent, but the slots before the collapse depend on the
      // seed, so the tile is finished by a full re-synchronisation later.
      uint32_t cx = cand_x;
      for (uint32_t k = 1; k < nsl; ++k) {
        const uint32_t ek = __shfl_sync(0xffffffffu, e, k), ck = __shfl_sync(0xffffffffu, c, k);
        const uint32_t xk = __shfl_sync(0xffffffffu, x, k), sk = __shfl_sync(0xffffffffu, stop, k);
        uint32_t cn, xn;
        if (cx == 0xffffffffu || !resync<MODE>(base_s, ek, ck, xk, cx, sk, T, cn, xn)) xn = 0xffffffffu;
        cx = xn;
        if (__all_sync(0xffffffffu, cx == xk)) {
          indep = true;
          if (fullfix) *fullfix = true;
          break;
        }
      }
    }
    if (seed_o < 0) {
      // speculative: publish the exit when it does not depend on the seed
      if (cand_out) *cand_out = cand_c;
      // without the candidate chase (a seam inside the range, resolved by the
      // seam walk) the exit is speculative: D_AGG carrying its value
      const unsigned long long dsc = mkdesc(ep, indep && chase ? D_INC : D_AGG, indep ? wb0 + xlast : 0);
      if (lane == 0) st_relaxed(a.exit_desc + tile, dsc);
      if (desc_out) *desc_out = dsc;
    } else if (tile > 0) {
      const uint32_t o = (uint32_t)seed_o;
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
            if (!resync<MODE>(base_s, e, c, x, xin, stop, T, cn, xn)) bad = true;
            e = xin;
            c = cn;
            x = xn;
            dnow = true;
          }
          dprev2 = dnow;
        }
      }
      const uint32_t xl = __shfl_sync(0xffffffffu, x, nsl - 1);
      const unsigned long long dsc = mkdesc(ep, D_INC, wb0 + xl);
      if (lane == 0) st_relaxed(a.exit_desc + tile, dsc);
      if (desc_out) *desc_out = dsc;
    }
  }
  if (!active) c = 0;
  if (VAR == BH_VARIANT_GAP && resync_needed) flag_need_staged(a.rep, ep);
}

// Completion: the last CTA of the call records the epoch in the report and
// advances the workspace epoch for the next call (stream-ordered, so the next
// call -- or graph replay -- observes it).
__device__ __forceinline__ void fused_finish(const FusedArgs& a, uint32_t ep) {
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicMax(&a.rep->phase_ns[5], global_ns());  // decode_write end (max over CTAs)
    __threadfence();
    const unsigned prev = atomicAdd(a.ws_hdr + 1, 1u);
    if (prev == gridDim.x - 1) {
      a.ws_hdr[1] = 0;
      a.rep->pad[1] = ep;
      a.rep->pad[2] = FUSED_MARK;
      __threadfence();
      *(volatile unsigned int*)a.ws_hdr = ep;
    }
  }
}

// debug timeline: per warp, TRACE_SLOTS globaltimer stamps (bh_debug_fused_trace)
constexpr int TRACE_SLOTS = 64;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}




// ---------------------------------------------------------------------------
// Two-phase fused kernel (default).  One CTA per SM owns a contiguous range of
// tiles.  Phase 1: its warps count every tile of the range (GAP: boundary +
// gap byte; SYNC: intra-sequence self-synchronisation and the seam seed, as
// tile_counts) and record each subsequence's entry and lane prefix plus the
// tile total in the workspace.  The CTA then scans its tile totals and
// publishes its aggregate with a decoupled look-back across CTAs (148
// descriptors, resolved in one round of loads).  Phase 2: the warps decode
// every tile of the range into shared-memory staging and flush it with
// coalesced 128-bit stores.  No warp waits for another warp inside a phase,
// so the memory-bound flushes of some warps overlap the table-bound decoding
// of others; the count phase needs only the 12-bit count table, so it starts
// as soon as that table lands.
// ---------------------------------------------------------------------------

// exclusive prefix of CTA `c` over the epoch-tagged CTA descriptors: every
// predecessor descriptor is loaded in one round (lane l takes c-1-l, c-33-l..)
__device__ unsigned long long lookback_wide(unsigned long long* desc, uint64_t c, uint32_t ep,
                                            unsigned long long* dbg = nullptr) {
  const uint32_t lane = threadIdx.x & 31;
  unsigned long long excl = 0;
  int64_t hi = (int64_t)c - 1;
  uint32_t polls = 0;
  while (hi >= 0) {
    // up to 4 x 32 predecessors per round
    unsigned long long d[4];
    bool ready;
    do {
      ready = true;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t idx = hi - (int64_t)lane - 32 * q;
        d[q] = idx >= 0 ? ld_relaxed(desc + idx) : mkdesc(ep, D_INC, 0);
        ready = ready && desc_ready(d[q], ep);
      }
      ++polls;
      if (dbg && polls == 1 && lane == 0) dbg[0] = gtime();
      if (!__all_sync(0xffffffffu, ready)) __nanosleep(32); else break;
    } while (true);
    if (dbg && lane == 0) { dbg[1] = gtime(); dbg[2] = polls; }
    // nearest inclusive descriptor (smallest distance) ends the walk
    uint32_t stop_q = 4, stop_lane = 32;
#pragma unroll
    for (int q = 3; q >= 0; --q) {
      const unsigned m = __ballot_sync(0xffffffffu, (d[q] & D_INC) != 0);
      if (m) { stop_q = q; stop_lane = __ffs(m) - 1; }
    }
    unsigned long long v = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const bool take = (uint32_t)q < stop_q || ((uint32_t)q == stop_q && lane <= stop_lane);
      v += take ? (d[q] & D_VAL) : 0ull;
    }
    excl += warp_sum(v);
    if (stop_q < 4) break;
    hi -= 128;
  }
  return excl;
}

constexpr uint32_t MAX_SMEM_TILES = 512;
#ifndef BH_SEAMWALK
#define BH_SEAMWALK 1  // SYNC: in-range seams by one walk from the predecessor's exit (0: 32 candidate seeds per tile)
#endif
constexpr uint32_t SEAM_FAIL = 0xffffffffu;
constexpr uint32_t FAIL_CAP = 128;  // seam-walk failures listed per CTA (more: an ordered scan)
constexpr int32_t FULL_FIX = 0x7fffffff;  // tile_dlt marker: re-synchronise the whole tile in the fix-up

template <int VAR, int TR, int MODE>
__global__ void __launch_bounds__(FUSED_MAX_THREADS) k_fused2(const FusedArgs a) {
#define MARK(slot)                                                                                  \
  do {                                                                                              \
    if (TR && (threadIdx.x & 31) == 0 && (slot) < TRACE_SLOTS)                                      \
      a.trace[((size_t)blockIdx.x * a.warps + (threadIdx.x >> 5)) * TRACE_SLOTS + (slot)] = gtime(); \
  } while (0)
  MARK(0);
  // launched with programmatic stream serialisation: the CTAs start while the
  // preceding kernel (normally K1, which builds the tables) drains; nothing
  // it writes is read before this wait
  asm volatile("griddepcontrol.wait;" ::: "memory");
  extern __shared__ __align__(16) unsigned char sm[];
  // mbarriers: [0] count tables (c12, lim, base), [1] decode tables (wlut8,
  // lut12), [2] CTA output offset published (1 arrival)
  __shared__ __align__(8) unsigned long long s_mb[3];
  __shared__ unsigned long long s_ctaoff;
  __shared__ uint32_t s_wsum[32];
  __shared__ uint32_t s_carry;
  __shared__ uint32_t s_next;  // phase 2: next tile of the range to take
  __shared__ unsigned long long s_tcount, s_tseam;  // phase clocks (count loop end, seam fix-up end)
  __shared__ uint32_t s_cls[TUNE_CLASSES];           // tuner: sequences per class
  __shared__ __align__(8) unsigned long long s_wbar[FUSED_MAX_WARPS];  // per-warp word-staging mbarriers
  __shared__ uint32_t s_tcnt[MAX_SMEM_TILES];  // symbols per tile of the range (short ranges)
  __shared__ uint32_t s_fail[BH_SEAMWALK && VAR == BH_VARIANT_SYNC ? FAIL_CAP : 1];  // seam-walk failures (tile - t0)
  __shared__ uint32_t s_nfail;
  // SYNC, short ranges: the range's exit descriptors and full-fix flags, so
  // the seam fix-up reads in-range predecessors from shared memory
  constexpr uint32_t SX = VAR == BH_VARIANT_SYNC ? MAX_SMEM_TILES : 1;
  __shared__ unsigned long long s_texit[SX];
  const uint32_t ep = *(volatile const unsigned int*)a.ws_hdr + 1u;
  const TableHdr* hdr = static_cast<const TableHdr*>(a.table);
  if (VAR == BH_VARIANT_SYNC && !hdr->complete) {
    if (blockIdx.x == 0 && threadIdx.x == 0) flag_need_staged(a.rep, ep);
    fused_finish(a, ep);
    return;
  }
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned char* pw = sm + a.tables_bytes + (size_t)wib * a.per_warp_bytes;
  const uint32_t wbase_s = smem_u32(pw);
  const uint32_t stg_s = wbase_s + 8 * a.wpb;  // two word buffers, then staging
  const uint16_t* stg = reinterpret_cast<const uint16_t*>(pw + 8 * (size_t)a.wpb);
  const uint32_t W = a.warps;
  const uint64_t G = gridDim.x, cta = blockIdx.x;
  const uint64_t t0 = a.nseq * cta / G, t1 = a.nseq * (cta + 1) / G;
  const uint32_t nt = (uint32_t)(t1 - t0);
  // short ranges keep tile totals / seam descriptors in shared memory; long
  // ranges (or a forced BH_FUSED_SMEM_TILES) use the workspace copies
  const bool srange = nt <= a.smem_tiles;
  bool bad = false;

  const uint32_t sm_s = smem_u32(sm);
  const uint32_t bar_ct = smem_u32(&s_mb[0]), bar_dt = bar_ct + 8, bar_off = bar_ct + 16;
  if (threadIdx.x == 0) {
    TableLayout L(a.max_codes);
    const char* tb_ = static_cast<const char*>(a.table);
    mbar_init(bar_ct, 1);
    mbar_init(bar_dt, 1);
    mbar_init(bar_off, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(bar_ct, T_LIMBASE + 2 * FB_SIZE + a.ljs_bytes + (MODE == M_WIDE3 ? CW_SIZE : 0) +
                               (MODE != M_NARROW ? FB_SIZE : 0));
    if (MODE != M_NARROW) bulk_g2s(sm_s + a.t_len, tb_ + L.len12, FB_SIZE, bar_ct);
    if (MODE == M_WIDE3) bulk_g2s(sm_s, tb_ + L.cwin, CW_SIZE, bar_ct);  // decode-table region, phase 1
    bulk_g2s(sm_s + a.t_c12, tb_ + L.clut12, 2 * FB_SIZE, bar_ct);
    if (a.ljs_bytes) bulk_g2s(sm_s + a.t_ljs, tb_ + L.ljsym, a.ljs_bytes, bar_ct);
    bulk_g2s(sm_s + a.t_lim, tb_ + L.lim, T_LIMBASE, bar_ct);  // lim, base (contiguous)
    if (MODE == M_WIDE3) {
      // wlut3 replaces cwin at the phase boundary (below)
    } else if (MODE == M_WIDE) {
      mbar_expect_tx(bar_dt, T_WIDE_DEC);
      bulk_g2s(sm_s, tb_ + L.wlut12, T_WIDE_DEC, bar_dt);
    } else {
      // wlut8 packed into its own region (spread into the replicated layout
      // at the end of phase 1), lut12 when present
      mbar_expect_tx(bar_dt, 4096 + (a.has_l12 ? 4 * FB_SIZE : 0));
      bulk_g2s(sm_s + a.t_wp, tb_ + L.wlut8, 4096, bar_dt);
      if (a.has_l12) bulk_g2s(sm_s + a.t_l12, tb_ + L.lut12, 4 * FB_SIZE, bar_dt);
    }
  }
  // per warp: a landing buffer for the cp.async chunks of the next tile and
  // the skewed decode buffer of the current one
  const uint32_t land_s = wbase_s, dbuf_s = wbase_s + 4 * a.wpb;
  uint64_t tile = t0 + wib;
  uint64_t wb_a = 0, wb_b = 0;
  uint32_t nch_a = 0, nch_b = 0;
  WStage wst;
  wstage_init(wst, smem_u32(&s_wbar[wib]));
  if (tile < t1) wb_a = stage_words(a, tile, land_s, nch_a, wst);
  FTab T;
  T.wl = MODE != M_NARROW ? sm_s : sm_s + 16 * (lane & 7);
  T.dsh = MODE != M_NARROW ? 32 - FB : 24;
  T.dst = MODE == M_WIDE3 ? 3 : MODE == M_WIDE ? 4 : 7;
  T.lim = sm_s + a.t_lim;
  T.base = sm_s + a.t_lim + 33 * 8;
  T.l12 = (MODE == M_NARROW && a.has_l12) ? sm_s + a.t_l12 : 0u;
  T.c12 = sm_s + a.t_c12;
  T.cw = MODE == M_WIDE3 ? sm_s : 0u;
  T.len12 = sm_s + a.t_len;
  T.ljs = (a.ljs_bytes && hdr->kind == 0) ? sm_s + a.t_ljs : 0u;
  T.t = table_view(a.table, a.max_codes, hdr->ncodes);
  T.kind = hdr->kind;
  T.max_len = hdr->max_len ? min(hdr->max_len, 32u) : 32u;
  if (VAR == BH_VARIANT_SYNC)
    for (uint32_t i = threadIdx.x; i < SX; i += blockDim.x) s_texit[i] = 0;
  for (uint32_t i = threadIdx.x; i < TUNE_CLASSES; i += blockDim.x) s_cls[i] = 0;
  if (threadIdx.x == 0) {
    s_next = W;  // phase 2 starts with tile t0 + warp index
    s_tcount = s_tseam = 0;
    const unsigned long long t = global_ns();
    atomicMin(&a.rep->phase_ns[0], t);
    if (VAR == BH_VARIANT_GAP) atomicMax(&a.rep->phase_ns[1], t);  // entries come from the gap bytes inline
  }
  __syncthreads();  // barriers initialised
  MARK(56);
  mbar_wait(bar_ct, 0);
  MARK(1);

  // ---- phase 1: count ----------------------------------------------------
  // SYNC: first-slot candidate counts of this warp's tiles in its (still
  // unused) staging buffer when they fit, else in the workspace
  const uint32_t ktiles = t0 + wib < t1 ? (uint32_t)((t1 - (t0 + wib) + W - 1) / W) : 0u;
  const bool scand = VAR == BH_VARIANT_SYNC && srange && 64 * ktiles <= 2 * a.cap;
  uint32_t kidx = 0;
  // GAP: the gap bytes of a tile are loaded one tile ahead, like its words
  auto gap_load = [&](uint64_t t, uint32_t* g) {
    const uint64_t j = t * a.sps + lane;
    g[0] = (lane < a.sps && j < a.nsub) ? a.gap[j * a.spl] : 0u;
    g[1] = (lane == 31 && t * a.sps + 32 < a.nsub) ? a.gap[(t * a.sps + 32) * a.spl] : 0u;
  };
  uint32_t gcur[2] = {0, 0}, gnext[2] = {0, 0};
  if (VAR == BH_VARIANT_GAP && tile < t1) gap_load(tile, gcur);
  for (; tile < t1; tile += W) {
    const uint64_t tn = tile + W;
    wstage_wait(wst);  // this tile's words have landed
    skew_in(land_s, dbuf_s, nch_a);
    __syncwarp();
    if (kidx < 8) MARK(10 + 2 * kidx);
    if (tn < t1) {  // the next tile's words land while this one is counted
      wb_b = stage_words(a, tn, land_s, nch_b, wst);
      if (VAR == BH_VARIANT_GAP) gap_load(tn, gnext);
    }
    const uint32_t nsl = (uint32_t)min((uint64_t)a.sps, a.nsub - tile * a.sps);
    uint32_t e, c, cand = 0, xl = 0;
    bool fullfix = false;
    unsigned long long dsc = 0;
    // SYNC: only the range's first tile resolves its seam by candidate seeds
    // (its predecessor belongs to another CTA); the other seams are walked
    // from the predecessor's exit below
    const bool chase = !BH_SEAMWALK || tile == t0;
    tile_counts<VAR, MODE>(a, T, tile, dbuf_s, wb_a, nsl, ep, e, c, bad, -1, &cand, &fullfix,
                     VAR == BH_VARIANT_GAP && a.sps == 32 ? gcur : nullptr, &dsc, chase, &xl);
    if (kidx < 8) MARK(11 + 2 * kidx);
    gcur[0] = gnext[0];
    gcur[1] = gnext[1];
    if (VAR == BH_VARIANT_SYNC) {
      if (chase) {
        if (scand) sts16(stg_s + 64 * kidx + 2 * lane, min(cand, 0xffffu));
        else a.cand[tile * 32 + lane] = (uint16_t)min(cand, 0xffffu);
      }
      if (lane == 0) {
        a.tile_dlt[tile] = fullfix ? FULL_FIX : 0;
        if (srange) *(volatile unsigned long long*)&s_texit[tile - t0] = dsc;
#if BH_SEAMWALK
        // the next tile's seam: its first slot's parse from this tile's
        // (speculative) exit against its boundary parse, over the halo words
        // staged with this tile.  Seam word: seed | (delta + 0x8000) << 16,
        // SEAM_FAIL when the parses do not meet (the serial pass takes it)
        if (tile + 1 < t1) {
          const uint32_t bn = (uint32_t)((tile + 1) * a.seq_bits - wb_a);
          const uint32_t tbr = (uint32_t)min(a.tb - wb_a, (uint64_t)0xffffffffu);
          const uint32_t o = xl - bn;
          // the next tile's first slot parses from its pre-synchronised entry
          const uint32_t en = a.presync ? presync<MODE>(dbuf_s, bn > a.presync ? bn - a.presync : 0u, bn, T) : bn;
          int32_t d;
          uint32_t sw = SEAM_FAIL;
          const uint32_t lim = min(32 * (4 * nch_a - 4), bn + min(a.walk_max, a.sb));
          if (o < 32 && seam_walk<MODE>(dbuf_s, en, xl, min(bn + a.sb, tbr), lim, T, d))
            sw = o | ((uint32_t)(d + 0x8000) << 16);
          *reinterpret_cast<uint32_t*>(a.cand + (tile + 1) * 32) = sw;
        }
#endif
      }
    }
    ++kidx;
    uint32_t incl = c;
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
      if ((int)lane >= off) incl += y;
    }
    const uint32_t b = (uint32_t)((tile * a.sps + lane) * a.sb - wb_a);
    const uint32_t de = e - b;
    if (de > 0xffffu || incl > 0xffffu) bad = true;
    a.lane_info[tile * 32 + lane] = (de & 0xffffu) | ((incl - c) << 16);
    if (lane == 31) {
      if (srange) s_tcnt[tile - t0] = incl;
      else a.tile_cnt[tile] = incl;
    }
    wb_a = wb_b;
    nch_a = nch_b;
  }
  wstage_wait(wst);
  __syncwarp();  // candidate slots written by other lanes are read below
  if (lane == 0) atomicMax(&s_tcount, global_ns());
  MARK(9);
  if (VAR == BH_VARIANT_SYNC) {
#if BH_SEAMWALK
    // Seam fix-up (inter_sync, sync_decoder.py:116-149).  Every seam inside
    // the range was walked in the count loop from the predecessor's
    // speculative exit.  Where the walk met the boundary parse, the first
    // slot's count changes by its delta and the tile's exit is unchanged, so
    // -- by induction from the range's first tile, whose exit the candidate
    // seeds proved seed-independent -- every speculative exit is final.  The
    // rest (walks that did not meet, a first tile whose exit depends on its
    // seed, successors of a tile whose exit changed) warp 0 finishes in tile
    // order, re-synchronising each from its known seed.
    if (threadIdx.x == 0) s_nfail = 0;
    __syncthreads();  // seam words, speculative exits and counts of every warp visible
    for (uint64_t t = t0 + 1 + threadIdx.x; t < t1; t += blockDim.x) {
      const uint32_t sw = *reinterpret_cast<const uint32_t*>(a.cand + t * 32);
      if (sw == SEAM_FAIL) {
        const uint32_t k = atomicAdd(&s_nfail, 1u);
        if (k < FAIL_CAP) s_fail[k] = (uint32_t)(t - t0);
        continue;
      }
      const uint32_t o = sw & 0xffffu;
      const int32_t d = (int32_t)(sw >> 16) - 0x8000;
      a.tile_dlt[t] = d;
      a.lane_info[t * 32] = o;  // first slot enters at the seed; prefix 0
      if (srange) s_tcnt[t - t0] += (uint32_t)d;
      else a.tile_cnt[t] += (uint32_t)d;
    }
    __syncthreads();
    if (wib == 0 && t0 < t1) {
      const uint32_t nfail = s_nfail;
      auto exit_of = [&](uint64_t t) -> unsigned long long {
        return srange ? *(volatile unsigned long long*)&s_texit[t - t0] : ld_relaxed(a.exit_desc + t);
      };
      // seed offset of tile t from its predecessor's final exit (another CTA's)
      auto pred_seed = [&](uint64_t t) -> uint32_t {
        unsigned long long dp = 0;
        if (lane == 0)
          while (!((dp = ld_relaxed(a.exit_desc + t - 1)) & D_INC) || !desc_ready(dp, ep)) __nanosleep(32);
        dp = __shfl_sync(0xffffffffu, dp, 0);
        return (uint32_t)((dp & D_VAL) - t * a.seq_bits);
      };
      // tile st re-synchronised from seed offset o: entries, counts and exit
      auto resync_tile = [&](uint64_t st, uint32_t o) -> uint64_t {
        uint32_t nchs;
        const uint64_t wbs = stage_words(a, st, land_s, nchs, wst);
        wstage_wait(wst);
        skew_in(land_s, dbuf_s, nchs);
        __syncwarp();
        const uint32_t nsl = (uint32_t)min((uint64_t)a.sps, a.nsub - st * a.sps);
        uint32_t e, c;
        unsigned long long dsc = 0;
        tile_counts<VAR, MODE>(a, T, st, dbuf_s, wbs, nsl, ep, e, c, bad, (int32_t)min(o, 255u), nullptr, nullptr,
                               nullptr, &dsc);
        if (lane == 0 && srange) *(volatile unsigned long long*)&s_texit[st - t0] = dsc;
        uint32_t incl = c;
        for (int off = 1; off < 32; off <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
          if ((int)lane >= off) incl += y;
        }
        const uint32_t b = (uint32_t)((st * a.sps + lane) * a.sb - wbs);
        const uint32_t de = e - b;
        if (de > 0xffffu || incl > 0xffffu) bad = true;
        a.lane_info[st * 32 + lane] = (de & 0xffffu) | ((incl - c) << 16);
        if (lane == 31) {
          a.tile_dlt[st] = 0;
          if (srange) s_tcnt[st - t0] = incl;
          else a.tile_cnt[st] = incl;
        }
        __syncwarp();
        return __shfl_sync(0xffffffffu, dsc, 0) & D_VAL;
      };
      // the next listed walk failure after tile `after` (an ordered scan of
      // the seam words when the list overflowed)
      auto next_fail = [&](uint64_t after) -> uint64_t {
        if (nfail <= FAIL_CAP) {
          uint32_t best = 0xffffffffu;
          for (uint32_t i = lane; i < nfail; i += 32) {
            const uint32_t v = s_fail[i];
            if (v > (uint32_t)(after - t0) && v < best) best = v;
          }
          best = __reduce_min_sync(0xffffffffu, best);
          return best == 0xffffffffu ? t1 : t0 + best;
        }
        for (uint64_t q = after + 1; q < t1; q += 32) {
          const uint64_t tt = q + lane;
          const unsigned m = __ballot_sync(
              0xffffffffu, tt < t1 && *reinterpret_cast<const uint32_t*>(a.cand + tt * 32) == SEAM_FAIL);
          if (m) return q + __ffs(m) - 1;
        }
        return t1;
      };
      const bool dep0 = t0 > 0 && !(exit_of(t0) & D_INC);
#ifdef BH_SEAM_STATS  // debug: walk failures -> repair_needed, dependent first tiles -> seam_passes
      if (lane == 0) {
        atomicAdd(&a.rep->repair_needed, (unsigned long long)nfail);
        if (dep0) atomicAdd(&a.rep->seam_passes, 1ull);
      }
#endif
      uint64_t t;
      if (dep0) {  // the first tile's exit depends on its seed
        resync_tile(t0, pred_seed(t0));
        t = t0 + 1;
      } else {
        t = next_fail(t0);
      }
      while (t < t1) {
        const uint32_t o = (uint32_t)((exit_of(t - 1) & D_VAL) - t * a.seq_bits);
        const uint32_t sw = __shfl_sync(0xffffffffu, lane == 0 ? *reinterpret_cast<const uint32_t*>(a.cand + t * 32) : 0u, 0);
        if (sw == SEAM_FAIL || o != (sw & 0xffffu)) {
#ifdef BH_SEAM_STATS  // debug: serial re-synchronisations -> stale_seams
          if (lane == 0) atomicAdd(&a.rep->stale_seams, 1ull);
#endif
          const uint64_t old = exit_of(t) & D_VAL;
          if (resync_tile(t, o) != old && t + 1 < t1) {  // the successor's walk started from the old exit
            ++t;
            continue;
          }
        }
        t = next_fail(t);
      }
      // the range's exit is final: the next CTA's first tile may take it
      if (t1 - 1 > t0 && lane == 0) st_relaxed(a.exit_desc + t1 - 1, mkdesc(ep, D_INC, exit_of(t1 - 1) & D_VAL));
      if (t0 > 0 && !dep0) {
        // the first tile: its exit never depended on the seed; swap in the
        // first slot's count for the true seed (or re-synchronise it when the
        // slots between depended on it)
        const uint32_t o = pred_seed(t0);
        const bool ff = __shfl_sync(0xffffffffu, lane == 0 ? (uint32_t)(a.tile_dlt[t0] == FULL_FIX) : 0u, 0) != 0;
        if (ff) {
          resync_tile(t0, o);
        } else if (o >= 32) {
          bad = true;
        } else if (lane == 0) {
          const int32_t dl = !o ? 0
                             : scand ? (int32_t)lds16(stg_s + 2 * o) - (int32_t)lds16(stg_s)
                                     : (int32_t)a.cand[t0 * 32 + o] - (int32_t)a.cand[t0 * 32];
          a.tile_dlt[t0] = dl;
          if (o) {
            a.lane_info[t0 * 32] = o;
            if (srange) s_tcnt[0] += (uint32_t)dl;
            else a.tile_cnt[t0] += (uint32_t)dl;
          }
        }
        __syncwarp();
      }
    }
#else
    // Seam fix-up (inter_sync, sync_decoder.py:116-149).  Every exit that does
    // not depend on the seed was published during the count loop, so the
    // true seed of most tiles is known now: lane j of the warp takes the
    // warp's tile j of a 32-tile chunk, reads the predecessor's exit and swaps
    // in the first slot's count for that seed (the other slots are unchanged
    // because every candidate seed leads to the same first exit).  Tiles whose
    // exit depends on the seed (or whose predecessor's does) are finished one
    // at a time in tile order: the words are staged again and the tile is
    // re-synchronised from the known seed.
    for (uint64_t kb = 0;; kb += 32) {
      const uint64_t tk = t0 + wib + (kb + lane) * W;
      const bool mine = tk < t1;
      if (!__any_sync(0xffffffffu, mine)) break;
      bool serial = false;
      if (mine && tk > 0) {
        const bool sm_own = srange, sm_pred = sm_own && tk - 1 >= t0;
        unsigned long long dp;
        const unsigned long long ds = sm_own ? *(volatile unsigned long long*)&s_texit[tk - t0]
                                             : ld_relaxed(a.exit_desc + tk);
        const bool ff = a.tile_dlt[tk] == FULL_FIX;  // written by this warp's lane 0 in the count loop
        if (sm_pred) {
          while (!desc_ready(dp = *(volatile unsigned long long*)&s_texit[tk - 1 - t0], ep)) __nanosleep(32);
        } else {
          while (!desc_ready(dp = ld_relaxed(a.exit_desc + tk - 1), ep)) __nanosleep(32);
        }
        if ((ds & D_INC) && (dp & D_INC) && !ff) {
          const uint32_t o = (uint32_t)((dp & D_VAL) - tk * a.seq_bits);
          if (o >= 32) {
            bad = true;
          } else if (o) {
            const uint32_t cs = stg_s + 64 * (uint32_t)(kb + lane);
            const int32_t dl = scand ? (int32_t)lds16(cs + 2 * o) - (int32_t)lds16(cs)
                                     : (int32_t)a.cand[tk * 32 + o] - (int32_t)a.cand[tk * 32];
            a.tile_dlt[tk] = dl;
            a.lane_info[tk * 32] = o;  // first slot enters at the seed; prefix 0
            if (srange) s_tcnt[tk - t0] += (uint32_t)dl;
            else a.tile_cnt[tk] += (uint32_t)dl;
          } else {
            a.tile_dlt[tk] = 0;
          }
        } else {
          serial = true;
        }
      } else if (mine) {
        a.tile_dlt[tk] = 0;
      }
      unsigned sm_mask = __ballot_sync(0xffffffffu, serial);
      while (sm_mask) {
        const uint32_t j = __ffs(sm_mask) - 1;
        sm_mask &= sm_mask - 1;
        const uint64_t st = t0 + wib + (kb + j) * W;
        const bool sm_own = srange, sm_pred = sm_own && st - 1 >= t0;
        unsigned long long dp = 0;
        if (lane == 0) {
          if (sm_pred) {
            while (!((dp = *(volatile unsigned long long*)&s_texit[st - 1 - t0]) & D_INC) || !desc_ready(dp, ep))
              __nanosleep(32);
          } else {
            while (!((dp = ld_relaxed(a.exit_desc + st - 1)) & D_INC) || !desc_ready(dp, ep)) __nanosleep(32);
          }
        }
        dp = __shfl_sync(0xffffffffu, dp, 0);
        const uint32_t o = (uint32_t)((dp & D_VAL) - st * a.seq_bits);
        const unsigned long long ds = sm_own ? *(volatile unsigned long long*)&s_texit[st - t0]
                                             : ld_relaxed(a.exit_desc + st);
        const bool ff = __shfl_sync(0xffffffffu, lane == 0 ? (uint32_t)(a.tile_dlt[st] == FULL_FIX) : 0u, 0) != 0;
        if ((ds & D_INC) && !ff) {  // first-slot swap behind a dependent predecessor
          if (o >= 32) {
            bad = true;
          } else if (lane == 0) {
            const uint32_t cs = stg_s + 64 * (uint32_t)(kb + j);
            const int32_t dl = scand ? (int32_t)lds16(cs + 2 * o) - (int32_t)lds16(cs)
                                     : (int32_t)a.cand[st * 32 + o] - (int32_t)a.cand[st * 32];
            a.tile_dlt[st] = dl;
            a.lane_info[st * 32] = o;
            if (srange) s_tcnt[st - t0] += (uint32_t)dl;
            else a.tile_cnt[st] += (uint32_t)dl;
          }
          __syncwarp();
          continue;
        }
        // dependent tile: stage its words again and synchronise from the seed
        uint32_t nchs;
        const uint64_t wbs = stage_words(a, st, land_s, nchs, wst);
        wstage_wait(wst);
        skew_in(land_s, dbuf_s, nchs);
        __syncwarp();
        const uint32_t nsl = (uint32_t)min((uint64_t)a.sps, a.nsub - st * a.sps);
        uint32_t e, c;
        unsigned long long dsc = 0;
        tile_counts<VAR, MODE>(a, T, st, dbuf_s, wbs, nsl, ep, e, c, bad, (int32_t)min(o, 255u), nullptr, nullptr,
                         nullptr, &dsc);
        if (lane == 0 && srange) *(volatile unsigned long long*)&s_texit[st - t0] = dsc;
        uint32_t incl = c;
        for (int off = 1; off < 32; off <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
          if ((int)lane >= off) incl += y;
        }
        const uint32_t b = (uint32_t)((st * a.sps + lane) * a.sb - wbs);
        const uint32_t de = e - b;
        if (de > 0xffffu || incl > 0xffffu) bad = true;
        a.lane_info[st * 32 + lane] = (de & 0xffffu) | ((incl - c) << 16);
        if (lane == 31) {
          a.tile_dlt[st] = 0;
          if (srange) s_tcnt[st - t0] = incl;
          else a.tile_cnt[st] = incl;
        }
        __syncwarp();
      }
    }
  #endif
  }
  if (VAR == BH_VARIANT_SYNC && lane == 0) atomicMax(&s_tseam, global_ns());
  MARK(2);

  // ---- tile offsets within the range, CTA aggregate -----------------------
  // wlut8 replicated 8 ways ([entry][replica] uint4) from its packed copy
  if (MODE != M_WIDE3) mbar_wait(bar_dt, 0);
  if (MODE == M_NARROW)
    for (uint32_t i = threadIdx.x; i < 256 * 8; i += blockDim.x)
      sts128(sm_s + 16 * i, lds128(sm_s + a.t_wp + 16 * (i >> 3)));
  __syncthreads();  // tile totals and the replicated decode table visible
  if (MODE == M_WIDE3 && threadIdx.x == 0) {
    // every warp is done with cwin: the decode table takes its place
    TableLayout L(a.max_codes);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(bar_dt, T_WIDE3_DEC);
    bulk_g2s(sm_s, static_cast<const char*>(a.table) + L.wlut3, T_WIDE3_DEC, bar_dt);
  }
  T.cw = 0u;
  if (threadIdx.x == 0) {
    atomicMax(&a.rep->phase_ns[VAR == BH_VARIANT_GAP ? 2 : 1], s_tcount);
    if (VAR == BH_VARIANT_SYNC) atomicMax(&a.rep->phase_ns[2], s_tseam);
  }
  uint32_t carry = 0;
  if (srange) {
    // each warp sums the totals before its tiles itself (phase 2); warp 0 the aggregate
    if (wib == 0) {
      uint32_t v = 0;
      for (uint32_t i = lane; i < nt; i += 32) v += s_tcnt[i];
      carry = warp_sum(v);
    }
  } else {
    // long ranges: block-wide scan of the totals in the workspace
    const uint32_t nw = blockDim.x >> 5;
    for (uint32_t base = 0; base < nt; base += blockDim.x) {
      const uint32_t i = base + threadIdx.x;
      const uint32_t v = i < nt ? a.tile_cnt[t0 + i] : 0u;
      uint32_t incl = v;
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
        if ((int)lane >= off) incl += y;
      }
      if (lane == 31) s_wsum[wib] = incl;
      __syncthreads();
      if (wib == 0) {
        const uint32_t ws = lane < nw ? s_wsum[lane] : 0u;
        uint32_t wi = ws;
        for (int off = 1; off < 32; off <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, wi, off);
          if ((int)lane >= off) wi += y;
        }
        if (lane < nw) s_wsum[lane] = wi - ws;
        if (lane == 31) s_carry = wi;
      }
      __syncthreads();
      if (i < nt) a.tile_off[t0 + i] = carry + s_wsum[wib] + incl - v;
      carry += s_carry;
      __syncthreads();
    }
  }
  // warp 0 publishes the CTA aggregate and looks back; the others start decoding
  if (wib == 0) {
    unsigned long long excl = 0;
    if (cta == 0) {
      if (lane == 0) st_relaxed(a.cnt_desc, mkdesc(ep, D_INC, carry));
    } else {
      if (lane == 0) st_relaxed(a.cnt_desc + cta, mkdesc(ep, D_AGG, carry));
      MARK(5);
      excl = lookback_wide(a.cnt_desc, cta, ep,
                           TR ? a.trace + ((size_t)blockIdx.x * a.warps) * TRACE_SLOTS + 6 : nullptr);
      if (lane == 0) st_relaxed(a.cnt_desc + cta, mkdesc(ep, D_INC, excl + carry));
    }
    if (lane == 0) {
      const unsigned long long tr = global_ns();  // output index resolved (count_pass / output_index end)
      atomicMax(&a.rep->phase_ns[3], tr);
      atomicMax(&a.rep->phase_ns[4], tr);
      s_ctaoff = excl;
      if (cta == G - 1) {
        a.rep->total_symbols = excl + carry;
        if (a.count_cap ? excl + carry > a.nsym : excl + carry != a.nsym)
          tag_status(a.rep, ep, a.count_cap ? BH_TRUNCATED : VAR == BH_VARIANT_GAP ? BH_BADGAP : BH_TRUNCATED);
      }
      mbar_arrive(bar_off);
    }
  }
  MARK(3);

  // ---- phase 2: decode and write -----------------------------------------
  // tiles are taken dynamically (a shared counter): a warp that finishes
  // early takes the next tile, so the range's last round is balanced
  // (BH_REV: from the end of the range, whose words the count phase read
  // last and L2 still holds; t1 marks the end either way)
  auto pick = [&](uint32_t v) -> uint64_t { return v < nt ? (BH_REV ? t1 - 1 - v : t0 + v) : t1; };
  tile = pick(wib);
  __syncwarp();
  if (tile < t1) wb_a = stage_words(a, tile, land_s, nch_a, wst, true);
  bool have_off = false, bulk_pending = false;
  unsigned long long Pc = 0;
  auto grab = [&]() -> uint64_t {
    uint32_t v = 0;
    // one lane's shared-memory increment (an add would be wrapped in the
    // compiler's warp-aggregation sequence; inc with a limit that is never
    // reached is the same add)
    if (lane == 0)
      asm volatile("atom.shared.inc.u32 %0, [%1], 0xfffffffe;" : "=r"(v) : "r"(smem_u32(&s_next)) : "memory");
    return pick(__shfl_sync(0xffffffffu, v, 0));
  };
  // the tile's lane info (entry, prefix) and seam delta are loaded one tile
  // ahead, like its words
  uint32_t info_n = 0;
  int32_t dlt_n = 0;
  if (tile < t1) {
    info_n = a.lane_info[tile * 32 + lane];
    if (VAR == BH_VARIANT_SYNC) dlt_n = a.tile_dlt[tile];
  }
  uint32_t dk = 0;  // tiles decoded (trace slots)
  if (MODE == M_WIDE3) mbar_wait(bar_dt, 0);  // the decode table has replaced cwin
  for (; tile < t1;) {
    const uint64_t tn = grab();
    const uint32_t info = info_n;
    const int32_t dlt = dlt_n;
    if (tn < t1) {
      info_n = a.lane_info[tn * 32 + lane];
      if (VAR == BH_VARIANT_SYNC) dlt_n = a.tile_dlt[tn];
    }
    uint32_t C, toff;
    if (srange) {
      const uint32_t ti = (uint32_t)(tile - t0);
      uint32_t v = 0;
      for (uint32_t i = lane; i < ti; i += 32) v += s_tcnt[i];
      toff = warp_sum(v);
      C = s_tcnt[ti];
    } else {
      C = a.tile_cnt[tile];
      toff = a.tile_off[tile];
    }
    wstage_wait(wst);  // this tile's words have landed
    if (dk < 8) MARK(30 + 3 * dk);
    skew_in(land_s, dbuf_s, nch_a);
    __syncwarp();
    if (tn < t1) wb_b = stage_words(a, tn, land_s, nch_b, wst, true);  // lands while this tile decodes
    const uint32_t nsl = (uint32_t)min((uint64_t)a.sps, a.nsub - tile * a.sps);
    const uint32_t base_s = dbuf_s;
    const uint32_t b = (uint32_t)((tile * a.sps + lane) * a.sb - wb_a);
    const uint32_t e = b + (info & 0xffffu);
    uint32_t o = info >> 16;
    if (VAR == BH_VARIANT_SYNC && lane > 0) o += (uint32_t)dlt;  // seam fix of slot 0
    const uint32_t on = __shfl_down_sync(0xffffffffu, o, 1);
    const uint32_t c = lane < nsl ? (lane == 31 ? C : on) - o : 0u;
    if (!have_off) {
      have_off = __shfl_sync(0xffffffffu, lane == 0 ? mbar_test(bar_off, 0) : 0u, 0) != 0;
      if (have_off) Pc = *(volatile unsigned long long*)&s_ctaoff;
    }
    bool fits = C + 16 <= a.cap;
    uint32_t capw = a.cap - 8;  // staging window of the reference rounds (staging.py:123-146)
    if (a.t_high) {
      // online tuner (tuner.py:117-191, PAPER Alg. 2): the tile's class from its
      // own compression ratio sets its staging capacity (tuner.capacity); a
      // tile above it takes the reference's rounds with that capacity
      const uint64_t tbits = min((uint64_t)a.seq_bits, a.tb - tile * (uint64_t)a.seq_bits);
      const uint32_t tcls =
          C ? (uint32_t)min(((uint64_t)C * a.sym_w + tbits - 1) / tbits, (uint64_t)a.t_high + 1) : 1u;
      const uint32_t cc = a.cls_cap[tcls - 1];
      if (cc < capw) capw = cc;
      if (C > cc) fits = false;
      if (a.lanes_per_seq) {
        // tuner.plan's classes of the reference sequences this tile holds
        // (tuner.py:126-133: ceil(count * width / bits), the last sequence's
        // actual bits, an empty sequence in class 1)
        uint32_t v = c;
        for (uint32_t sw = 1; sw < a.lanes_per_seq; sw <<= 1) v += __shfl_xor_sync(0xffffffffu, v, sw);
        if (lane % a.lanes_per_seq == 0) {
          const uint64_t q = tile * (uint64_t)(32 / a.lanes_per_seq) + lane / a.lanes_per_seq;
          if (q < a.nseq_ref) {
            const uint64_t qb = q + 1 < a.nseq_ref ? (uint64_t)a.ref_seq_bits : a.tb - q * (uint64_t)a.ref_seq_bits;
            const uint32_t k = v ? (uint32_t)min(((uint64_t)v * a.sym_w + qb - 1) / qb, (uint64_t)a.t_high + 1) : 1u;
            atomicAdd(&s_cls[k - 1], 1u);
          }
        }
      }
    }
    const uint32_t sh = have_off ? (uint32_t)(Pc + toff) & 7u : 0u;
    if (bulk_pending) {  // the previous tile's bulk copy must have read the staging
      if (lane == 0) bulk_read_wait();
      __syncwarp();
      bulk_pending = false;
    }
    if (fits && c) {
      SR r;
      r.init(base_s, e);
      if (!fdecode<MODE>(r, c, stg_s + 2 * (sh + o), T)) bad = true;
    }
    __syncwarp();
    if (dk < 8) MARK(31 + 3 * dk);

    const bool aligned = have_off;
    if (!have_off) {
      MARK(4);
      mbar_wait(bar_off, 0);
      Pc = *(volatile unsigned long long*)&s_ctaoff;
      have_off = true;
    }
    const unsigned long long P = Pc + toff;
    if (fits) {
      if (aligned) bulk_pending = flush_bulk(a.out, a.nsym, P, C, stg_s);
      else flush_compact(a.out, a.nsym, P, C, stg_s);
    } else {
      // reference rounds (staging.py:123-146) with capacity cap - 8
      const bool active = lane < nsl;
      const uint32_t endl = o + c;
      uint32_t si = 0;
      while (si < C) {
        const uint32_t window = si + capw;
        const unsigned mj = __ballot_sync(0xffffffffu, active && endl > si);
        const uint32_t jl = __ffs(mj) - 1;
        const unsigned mk = __ballot_sync(0xffffffffu, active && lane >= jl && endl > window);
        const uint32_t kl = mk ? __ffs(mk) - 1 : nsl;
        if (kl == jl) {
          if (lane == jl) {
            SR r;
            r.init(base_s, e);
            if (!fdecode_global<MODE>(r, c, a.out, P + o, a.nsym, T)) bad = true;
          }
          si = __shfl_sync(0xffffffffu, endl, jl);
          continue;
        }
        const uint32_t temp_end = kl < nsl ? __shfl_sync(0xffffffffu, o, kl & 31) : C;
        const uint64_t g0w = P + si;
        const uint64_t gbase = g0w & ~7ull;
        const bool mine = lane >= jl && lane < kl && c;
        const uint32_t d = stg_s + 2 * (uint32_t)(P + o - gbase);
            if (mine) {
          SR r;
          r.init(base_s, e);
          if (!fdecode<MODE>(r, c, d, T)) bad = true;
        }
        __syncwarp();

        flush_aligned(a.out, a.nsym, g0w, temp_end - si, stg);
        __syncwarp();
        si = temp_end;
      }
    }
    __syncwarp();
    if (dk < 8) MARK(32 + 3 * dk);
    ++dk;
    wb_a = wb_b;
    nch_a = nch_b;
    tile = tn;
  }
  wstage_wait(wst);
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // staging read (writes land by kernel end)
  if (!have_off) mbar_wait(bar_off, 0);  // keep warp 0's arrival inside the CTA's lifetime
  if (__any_sync(0xffffffffu, bad) && lane == 0) tag_status(a.rep, ep, BH_INVALID);
  if (a.t_high && a.lanes_per_seq) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i <= a.t_high; i += blockDim.x)
      if (s_cls[i]) atomicAdd(&a.class_freq[i], (unsigned long long)s_cls[i]);
  }
  MARK(TRACE_SLOTS - 2);
  fused_finish(a, ep);
  MARK(TRACE_SLOTS - 1);
#undef MARK
}

}  // namespace bh

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
using namespace bh;

namespace {
int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

inline uint64_t nsub_of(const bh_stream* s) { return (s->total_bits + s->subseq_bits - 1) / s->subseq_bits; }
// The fused kernel's tile is 32 subsequences (one lane each) whatever the
// stream's subseqs_per_seq: the decoded symbols do not depend on how
// subsequences are grouped into sequences (the synchronised state is the
// unique fixpoint -- entry i is the first codeword start at or after boundary
// i), so every layout runs with full warps.
constexpr uint32_t TILE_SUBSEQ = 32;
// Low-CR streams decode faster with longer lane windows: a lane takes spl
// consecutive stream subsequences (a "virtual" subsequence of spl * subseq_bits
// bits, entered at the first one's gap byte -- again the same fixpoint), as
// long as a tile's output stays within ~4 KB of staging.
inline uint32_t spl_of(const bh_stream* s) {
  const int e = env_int("BH_FUSED_SPL", 0);
  if (e == 1 || e == 2 || e == 4) return (uint32_t)e;
  const double per_bit = s->total_bits ? (double)s->symbol_count / (double)s->total_bits : 1.0;
  uint32_t spl = 1;
  while (spl < 4 && 32.0 * 2 * spl * s->subseq_bits * per_bit <= 2048.0 && 32ull * 2 * spl * s->subseq_bits <= 16384)
    spl *= 2;
  return spl;
}
inline uint32_t vsb_of(const bh_stream* s) { return s->subseq_bits * spl_of(s); }
inline uint64_t vnsub_of(const bh_stream* s) { return (s->total_bits + vsb_of(s) - 1) / vsb_of(s); }
inline uint64_t nseq_of(const bh_stream* s) { return (vnsub_of(s) + TILE_SUBSEQ - 1) / TILE_SUBSEQ; }



struct FusedCfg {
  uint32_t halo, lead, presync;
  uint32_t warps, cap, wpb, per_warp, tables, smem, has_l12, wide, mode, t_lim, t_c12, t_wp, t_l12, t_ljs, ljs_bytes,
      t_len;
};

// Dynamic shared memory one CTA of the variant's kernel may use on the
// current device: the per-block opt-in limit minus the kernel's static
// arrays (the self-sync kernel keeps its seam descriptors there), cached per
// (device, variant); 219 KB without a device.
uint32_t smem_budget(int variant) {
  static std::atomic<uint32_t> cache[64][2];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 219u * 1024u;
  const int vi = variant == BH_VARIANT_SYNC ? 1 : 0;
  uint32_t b = cache[dev][vi].load(std::memory_order_relaxed);
  if (!b) {
    int optin = 0;
    cudaFuncAttributes fa;
    const void* fn = vi ? (const void*)k_fused2<BH_VARIANT_SYNC, 0, M_NARROW>
                        : (const void*)k_fused2<BH_VARIANT_GAP, 0, M_NARROW>;
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess ||
        cudaFuncGetAttributes(&fa, fn) != cudaSuccess || optin <= (int)fa.sharedSizeBytes) {
      cudaGetLastError();
      return 219u * 1024u;
    }
    b = (uint32_t)(optin - (int)fa.sharedSizeBytes);
    cache[dev][vi].store(b, std::memory_order_relaxed);
  }
  return b;
}

FusedCfg fused_cfg(const bh_stream* s, const bh_tune* tune = nullptr, int variant = BH_VARIANT_SYNC) {
  FusedCfg c;
  const uint32_t seq_bits = vsb_of(s) * TILE_SUBSEQ;
  // words one tile can stage: its span (+1 for a straddle), the 16-byte
  // alignment of the first word (+3), the halo, rounded up to 16 bytes
  // SYNC stages the next tile's first slot (+4 words of reader lookahead) as
  // its halo: the seam walk of the next tile runs over it
  c.halo = variant == BH_VARIANT_SYNC ? std::max<uint32_t>(HALO_WORDS, vsb_of(s) / 32 + 4) : HALO_WORDS;
  // SYNC: lanes pre-synchronise from `presync` bits before their boundary:
  // long-code books (slow to synchronise, and a re-decode walks one codeword
  // at a time) gain, short-code ones (cheap mask-walk re-decodes) do not
  // (profiles/r02: HACC sync -11 %, Hurricane +6 % at 64 bits)
  c.lead = variant == BH_VARIANT_SYNC ? 8u : 0u;  // 256 bits: presync <= 256
  c.wpb = ((seq_bits + 31) / 32 + 1 + 3 + c.lead + c.halo + 3) & ~3u;
  c.wpb = (c.wpb + (c.wpb >> 5) + 1 + 3) & ~3u;  // physical words: one skew word per 32
  // staging sized from the header's compression ratio (no device round trip):
  // a tile emits about seq_bits * symbols / total_bits symbols; a tile above
  // the capacity takes the reference's rounds, so any value is correct
  const double per_bit = s->total_bits ? (double)s->symbol_count / (double)s->total_bits : 1.0;
  uint32_t cap = (uint32_t)(seq_bits * per_bit * BH_CAPF) + BH_CAPADD;
  if (env_int("BH_FUSED_CAP", 0)) cap = (uint32_t)env_int("BH_FUSED_CAP", 0);
  const uint32_t cmax = TILE_SUBSEQ * (vsb_of(s) + 31) + 16;
  if (cap > cmax) cap = cmax;
  if (cap < 64) cap = 64;
  c.cap = (cap + 7) & ~7u;
  c.has_l12 = !(tune && tune->max_len && tune->max_len <= 8);
  // long codes and more than ~1.5 bits per symbol: the 12-bit decode table
  // covers twice the bits per lookup (short-code books already get six
  // symbols out of the conflict-free 8-bit one)
  c.wide = c.has_l12 && 2 * s->total_bits > 3 * s->symbol_count;
  if (env_int("BH_FUSED_WIDE", -1) >= 0) c.wide = env_int("BH_FUSED_WIDE", 0) != 0;
  // books whose codes are all >= 4 bits never put more than three codewords in
  // a 12-bit window: the 8-byte three-codeword table then decodes the same
  c.mode = !c.wide ? M_NARROW : (tune && tune->min_len >= 4 ? M_WIDE3 : M_WIDE);
  if (c.wide && env_int("BH_FUSED_MODE", -1) >= 1) c.mode = env_int("BH_FUSED_MODE", 1) == 2 && tune &&
                                                                     tune->min_len >= 4 ? M_WIDE3 : M_WIDE;
  c.presync = 0;
  if (variant == BH_VARIANT_SYNC) {
    const int e = env_int("BH_PRESYNC_BITS", -1);  // tuning knob
    // the distance a parse needs to converge grows steeply with the mean
    // code length: 0.72 * (bits per symbol)^3, in 32-bit steps (HACC, 5.1
    // bits per symbol: 96; QMCPACK, 6.5: 192 -- the best of the 64..256
    // sweeps on each, profiles/r02/presync_sweep.txt)
    const double bps = s->symbol_count ? (double)s->total_bits / (double)s->symbol_count : 8.0;
    const uint32_t k = 32u * (uint32_t)std::lround(std::min(0.72 * bps * bps * bps, 256.0) / 32.0);
    c.presync = e >= 0 ? (uint32_t)std::min(e, 256) : (c.mode != M_NARROW ? std::min(std::max(k, 32u), 224u) : 0u);
  }
  if (c.wide) {
    c.t_lim = c.mode == M_WIDE3 ? T_WIDE3_DEC : T_WIDE_DEC;
    c.t_c12 = c.t_lim + T_LIMBASE;
    c.t_wp = c.t_l12 = 0;
    c.t_len = c.t_c12 + 2 * FB_SIZE;
    c.tables = (uint32_t)align16(c.t_len + FB_SIZE);
  } else {
    c.t_lim = T_NARROW_DEC;
    c.t_c12 = c.t_lim + T_LIMBASE;
    c.t_wp = c.t_c12 + 2 * FB_SIZE;
    c.t_l12 = c.t_wp + 4096;
    c.t_len = 0;
    c.tables = (uint32_t)align16(c.t_l12 + (c.has_l12 ? 4 * FB_SIZE : 0));
  }
  // codes longer than the tables reach: the canonical symbol order in shared
  // memory keeps the limit search off global memory (books up to 4096 codes)
  c.ljs_bytes = (c.has_l12 && s->max_codes <= 4096) ? (uint32_t)align16(2 * (size_t)s->max_codes) : 0u;
  c.t_ljs = c.tables;
  c.tables += c.ljs_bytes;
  // two word buffers, staging
  c.per_warp = (uint32_t)align16(8 * (size_t)c.wpb + 2 * (size_t)c.cap + 32);
  // dynamic shared memory budget: 227 KB per CTA minus the kernel's static
  // arrays (tile totals; the self-sync kernel's seam descriptors)
  int fit = (int)(((int64_t)smem_budget(variant) - (int64_t)c.tables) / (int64_t)c.per_warp);
  if (fit < FUSED_MAX_WARPS && !env_int("BH_FUSED_CAP", 0)) {
    // a little less staging when that lets every warp slot fit (HACC sync:
    // 23 -> 24 warps, 652 -> 636 us), keeping >= 4 % headroom over the
    // expected symbols per tile (a tile above the capacity takes the
    // reference's rounds, so any value is correct)
    const int64_t room = ((int64_t)smem_budget(variant) - (int64_t)c.tables) / FUSED_MAX_WARPS;
    const int64_t cap_max = ((room & ~int64_t(15)) - 8 * (int64_t)c.wpb - 32) / 2;
    const uint32_t cap_w = (uint32_t)std::max<int64_t>(cap_max, 0) & ~7u;
    if (cap_w >= (uint32_t)(seq_bits * per_bit * 1.04) + 32 && cap_w < c.cap) {
      c.cap = cap_w;
      c.per_warp = (uint32_t)align16(8 * (size_t)c.wpb + 2 * (size_t)c.cap + 32);
      fit = (int)(((int64_t)smem_budget(variant) - (int64_t)c.tables) / (int64_t)c.per_warp);
    }
  }
  int w = env_int("BH_FUSED_WARPS", 0);
  if (w <= 0 || w > fit) w = fit;
  if (w > FUSED_MAX_WARPS) w = FUSED_MAX_WARPS;
  if (w < 1) w = 1;
  // small inputs: fewer warps per CTA so that every SM gets a group
  const int sms = device_sm_count();
  const uint64_t nseq = nseq_of(s);
  if (!env_int("BH_FUSED_WARPS", 0) && nseq < (uint64_t)sms * (uint64_t)w) {
    w = (int)((nseq + sms - 1) / sms);
    if (w < 2) w = 2;
  }
  c.warps = (uint32_t)w;
  c.smem = c.tables + c.warps * c.per_warp;
  return c;
}

}  // namespace

static std::atomic<unsigned long long*> g_trace{nullptr};  // debug only

// Debug: record a per-warp timeline of the next fused launches into trace_dev
// (u64[grid * warps * 64] globaltimer stamps); NULL switches it off.
extern "C" int bh_debug_fused_trace(void* trace_dev) {
  g_trace = static_cast<unsigned long long*>(trace_dev);
  return BH_OK;
}

extern "C" int bh_debug_fused_shape(const bh_stream* s, const bh_tune* tune, uint32_t* warps, uint32_t* smem,
                                    uint32_t* cap, uint32_t* spl) {
  FusedCfg c = fused_cfg(s, tune);
  if (warps) *warps = c.warps;
  if (smem) *smem = c.smem;
  if (cap) *cap = c.cap;
  if (spl) *spl = spl_of(s);
  return BH_OK;
}

extern "C" int bh_fused_supported(const bh_stream* s, int variant) {
  if (env_int("BH_DISABLE_FUSED", 0)) return 0;
  if (variant != BH_VARIANT_GAP && variant != BH_VARIANT_SYNC) return 0;
  if (s->subseqs_per_seq == 0) return 0;
  // words are staged with 16-byte cp.async: the payload must be 16-byte aligned
  if (reinterpret_cast<uintptr_t>(s->words_dev) & 15u) return 0;
  const uint64_t seq_bits = (uint64_t)vsb_of(s) * TILE_SUBSEQ;
  if (seq_bits > 16384 || s->total_bits >= (1ull << 36) || s->symbol_count >= (1ull << 36)) return 0;
  if (variant == BH_VARIANT_GAP && !s->gap_dev) return 0;
  FusedCfg c = fused_cfg(s, nullptr, variant);
  return c.smem <= smem_budget(variant) ? 1 : 0;
}

// workspace: [64 B header: epoch, CTA-done counter][cnt desc][exit desc]
//            [lane info u32 x 32 per tile][tile count u32][tile offset u32]
//            [seed candidates u16 x 32 per tile][first-slot delta i32]
static size_t class_freq_offset(const bh_stream* s) {
  return 64 + 16 * nseq_of(s) + 4 * 34 * nseq_of(s) + 64 * nseq_of(s) + 4 * nseq_of(s);
}

extern "C" size_t bh_fused_workspace_bytes(const bh_stream* s, int, const bh_tune*) {
  return align16(class_freq_offset(s)) + 8 * TUNE_CLASSES + 256;
}

// Which lanes form one reference sequence (tile = 32 lanes of spl subsequences):
// the per-sequence histogram needs whole sequences per tile.
static uint32_t lanes_per_seq_of(const bh_stream* s) {
  const uint32_t spl = spl_of(s), sps = s->subseqs_per_seq;
  if (sps % spl) return 0;
  const uint32_t l = sps / spl;
  return (l && l <= 32 && 32 % l == 0) ? l : 0;
}

static bool tuned(const bh_tune* t) { return t && t->t_high && t->t_high < TUNE_CLASSES; }

// tuner.plan's class histogram of the last fused decode with this workspace
// (stream-ordered copy, then a sync): freq_host[0..t_high]
extern "C" int bh_tuner_class_freq(const bh_stream* s, const bh_tune* tune, const void* ws, uint64_t* freq_host,
                                   uint32_t n, void* cuda_stream) {
  if (!s || !ws || !freq_host || !tuned(tune) || n < tune->t_high + 1) return BH_BAD_ARGUMENT;
  if (!lanes_per_seq_of(s)) return BH_BAD_ARGUMENT;
  const char* p = static_cast<const char*>(ws) + align16(class_freq_offset(s));
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  if (cudaMemcpyAsync(freq_host, p, 8 * (size_t)(tune->t_high + 1), cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return BH_CUDA_ERROR;
  return cudaStreamSynchronize(st) == cudaSuccess ? BH_OK : BH_CUDA_ERROR;
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
  FusedCfg cfg = fused_cfg(s, tune, variant);
  FusedArgs a;
  a.words = s->words_dev;
  a.words_alloc = (((s->total_bits + 31) / 32 + BH_WORD_PAD) & ~3ull);
  a.gap = s->gap_dev;
  a.table = s->table_dev;
  a.max_codes = s->max_codes;
  a.sb = vsb_of(s);
  a.sps = TILE_SUBSEQ;
  a.spl = spl_of(s);
  a.sbr = s->subseq_bits;
  a.seq_bits = vsb_of(s) * TILE_SUBSEQ;
  a.tb = s->total_bits;
  a.nsym = s->symbol_count;
  a.nsub = vnsub_of(s);
  a.nsub_r = nsub_of(s);
  a.nseq = nseq;
  a.out = out_dev;
  a.ws_hdr = static_cast<unsigned int*>(ws);
  a.cnt_desc = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + 64);
  a.exit_desc = a.cnt_desc + nseq;
  a.lane_info = reinterpret_cast<uint32_t*>(a.exit_desc + nseq);
  a.tile_cnt = a.lane_info + 32 * nseq;
  a.tile_off = a.tile_cnt + nseq;
  a.cand = reinterpret_cast<uint16_t*>(a.tile_off + nseq);
  a.tile_dlt = reinterpret_cast<int32_t*>(a.cand + 32 * nseq);
  a.rep = static_cast<DevReport*>(report_dev);
  a.wpb = cfg.wpb;
  a.halo = cfg.halo;
  a.lead = cfg.lead;
  a.presync = cfg.presync;
  // test knob: a narrower seam-walk window sends seams to the serial pass
  // (0: every seam whose seed differs from the slot's own entry)
  a.walk_max = (uint32_t)env_int("BH_SEAMWALK_WINDOW", -1);
  a.cap = cfg.cap;
  a.warps = cfg.warps;
  a.per_warp_bytes = cfg.per_warp;
  a.tables_bytes = cfg.tables;
  a.has_l12 = cfg.has_l12;
  a.first_entry = s->first_entry;
  a.count_cap = (s->flags & BH_STREAM_COUNT_IS_CAPACITY) ? 1u : 0u;
  a.wide = cfg.wide;
  a.t_lim = cfg.t_lim;
  a.t_c12 = cfg.t_c12;
  a.t_wp = cfg.t_wp;
  a.t_l12 = cfg.t_l12;
  a.t_ljs = cfg.t_ljs;
  a.ljs_bytes = cfg.ljs_bytes;
  a.t_len = cfg.t_len;
  a.t_high = 0;
  a.lanes_per_seq = 0;
  if (tuned(tune)) {
    // capacities per class (tuner.py:98-106 with capacity_table overrides)
    a.t_high = tune->t_high;
    for (uint32_t c = 1; c <= a.t_high + 1; ++c) {
      uint32_t v = c <= 64 && tune->capacity_table[c - 1] ? tune->capacity_table[c - 1]
                                                          : (c > a.t_high ? 3584u : c * 1024u);
      a.cls_cap[c - 1] = v ? v : 1u;
    }
    a.lanes_per_seq = lanes_per_seq_of(s);
    a.sym_w = s->symbol_width ? s->symbol_width : 16u;
    a.ref_seq_bits = s->subseq_bits * s->subseqs_per_seq;
    a.nseq_ref = (nsub_of(s) + s->subseqs_per_seq - 1) / s->subseqs_per_seq;
    a.class_freq = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + align16(class_freq_offset(s)));
    if (cudaMemsetAsync(a.class_freq, 0, 8 * (size_t)(a.t_high + 1), static_cast<cudaStream_t>(cuda_stream)) !=
        cudaSuccess)
      return BH_CUDA_ERROR;
  }
  a.smem_tiles = (uint32_t)env_int("BH_FUSED_SMEM_TILES", (int)MAX_SMEM_TILES);
  if (a.smem_tiles > MAX_SMEM_TILES) a.smem_tiles = MAX_SMEM_TILES;
  const int sms = device_sm_count();
  a.trace = g_trace.load(std::memory_order_relaxed);
  static const void* const kern[2][2][3] = {
      {{(const void*)k_fused2<BH_VARIANT_GAP, 0, M_NARROW>, (const void*)k_fused2<BH_VARIANT_GAP, 0, M_WIDE>,
        (const void*)k_fused2<BH_VARIANT_GAP, 0, M_WIDE3>},
       {(const void*)k_fused2<BH_VARIANT_GAP, 1, M_NARROW>, (const void*)k_fused2<BH_VARIANT_GAP, 1, M_WIDE>,
        (const void*)k_fused2<BH_VARIANT_GAP, 1, M_WIDE3>}},
      {{(const void*)k_fused2<BH_VARIANT_SYNC, 0, M_NARROW>, (const void*)k_fused2<BH_VARIANT_SYNC, 0, M_WIDE>,
        (const void*)k_fused2<BH_VARIANT_SYNC, 0, M_WIDE3>},
       {(const void*)k_fused2<BH_VARIANT_SYNC, 1, M_NARROW>, (const void*)k_fused2<BH_VARIANT_SYNC, 1, M_WIDE>,
        (const void*)k_fused2<BH_VARIANT_SYNC, 1, M_WIDE3>}}};
  const void* fn = kern[variant == BH_VARIANT_GAP ? 0 : 1][a.trace ? 1 : 0][cfg.mode];
  // launch attributes and occupancy cached per (device, kernel, threads,
  // smem): the dynamic shared-memory opt-in is a per-device (per-context)
  // function attribute
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, uint32_t, uint32_t>, int> occ;
  int per_sm = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return BH_CUDA_ERROR;
  {
    std::lock_guard<std::mutex> g(mu);
    auto key = std::make_tuple(dev, fn, cfg.warps, cfg.smem);
    auto it = occ.find(key);
    if (it == occ.end()) {
      // the attribute is per kernel and device: raise it to the largest size
      // ever cached there (lowering it would break a cached larger configuration)
      static std::map<std::pair<int, const void*>, uint32_t> smem_set;
      uint32_t& cur = smem_set[std::make_pair(dev, fn)];
      if (cfg.smem > cur) {
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.smem) != cudaSuccess)
          return BH_CUDA_ERROR;
        cur = cfg.smem;
      }
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, (int)cfg.warps * 32, cfg.smem) != cudaSuccess ||
          per_sm < 1)
        return BH_CUDA_ERROR;
      occ[key] = per_sm;
    } else {
      per_sm = it->second;
    }
  }
  uint64_t grid = (uint64_t)per_sm * sms;
  const uint64_t need = (nseq + cfg.warps - 1) / cfg.warps;  // groups
  if (grid > need) grid = need;
  // caller-chosen CTA count (concurrent decodes sharing the GPU)
  if (tune && tune->ctas && tune->ctas < grid) grid = tune->ctas;
  // test knob: fewer CTAs, i.e. longer per-CTA tile ranges
  const int gforce = env_int("BH_FUSED_GRID", 0);
  if (gforce > 0 && (uint64_t)gforce < grid) grid = (uint64_t)gforce;
  if (grid < 1) grid = 1;
  prof_mark(static_cast<cudaStream_t>(cuda_stream), "start");
  void* args[] = {&a};
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)grid);
  lc.blockDim = dim3(cfg.warps * 32);
  lc.dynamicSmemBytes = cfg.smem;
  lc.stream = static_cast<cudaStream_t>(cuda_stream);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = env_int("BH_PDL", 1) ? 1 : 0;
  lc.attrs = at;
  lc.numAttrs = 1;
  if (cudaLaunchKernelExC(&lc, fn, args) != cudaSuccess) return BH_CUDA_ERROR;
  prof_mark(static_cast<cudaStream_t>(cuda_stream), variant == BH_VARIANT_GAP ? "fused_gap" : "fused_sync");
  return cudaGetLastError() == cudaSuccess ? BH_OK : BH_CUDA_ERROR;
}

