// abi.cu -- whole-decoder entry points (sync_decoder.decode / gap_decoder.decode).
//
// bh_decode_async launches the complete pipeline stream-ordered with no host
// synchronisation; bh_decode additionally reads the device report and, in the
// rare case the pre-launched seam passes did not settle every seam, finishes
// the seam passes on the host loop of sync_decoder.py:129-149 and re-runs the
// write phase.
#include <cstring>
#include "common.cuh"

extern "C" {
int bh_report_init(void* report_dev, void* cuda_stream);
int bh_intra_sync_ex(const bh_stream* s, const int64_t* seeds_dev, uint32_t round_cap,
                     const unsigned long long* gate, int64_t* entries_dev, int64_t* exits_dev,
                     int64_t* counts_dev, uint8_t* synced_dev, int32_t* iterations_dev, void* ws,
                     size_t ws_bytes, void* report_dev, void* cuda_stream);
int bh_check_total(const bh_stream* s, const int64_t* oi_dev, int status_on_mismatch,
                   void* report_dev, void* cuda_stream);
int bh_decode_write_classes(const bh_stream* s, const int64_t* entries_dev, const int64_t* counts_dev,
                            const int64_t* oi_dev, const int64_t* seq_ids_dev, uint64_t nseq_ids,
                            uint32_t capacity, uint32_t max_capacity, const int64_t* classes_dev,
                            const uint32_t* caps_dev, uint16_t* out_dev, uint64_t out_len,
                            void* report_dev, int stats, void* cuda_stream);
int bh_seam_check(const bh_stream* s, const int64_t* entries_dev, const int64_t* exits_dev,
                  int64_t* seeds_dev, unsigned long long* counter_dev, void* cuda_stream);
int bh_fused_supported(const bh_stream* s, int variant);
int bh_fill_caps(uint32_t* caps_dev, const uint32_t* caps_host, uint32_t n, void* cuda_stream);
size_t bh_fused_workspace_bytes(const bh_stream* s, int variant, const bh_tune* tune);
int bh_fused_decode(const bh_stream* s, int variant, const bh_tune* tune, uint16_t* out_dev,
                    void* ws, size_t ws_bytes, void* report_dev, void* cuda_stream);
}

using namespace bh;

namespace {

inline cudaStream_t S(void* p) { return static_cast<cudaStream_t>(p); }
inline uint64_t nsub_of(const bh_stream* s) { return (s->total_bits + s->subseq_bits - 1) / s->subseq_bits; }
inline uint64_t nseq_of(const bh_stream* s) { return (nsub_of(s) + s->subseqs_per_seq - 1) / s->subseqs_per_seq; }

constexpr uint32_t OVERFLOW_CAPACITY = 3584;  // tuner.py:26
constexpr uint32_t SYMBOLS_PER_CLASS = 1024;  // tuner.py:27
constexpr int MAX_SEAM_PASSES = 8;

// tuner.py:98-106
uint32_t class_capacity(uint32_t cls, const bh_tune* t) {
  if (cls <= 64 && t->capacity_table[cls - 1]) return t->capacity_table[cls - 1];
  if (cls > t->t_high) return OVERFLOW_CAPACITY;
  return cls * SYMBOLS_PER_CLASS;
}

struct Ws {
  size_t entries, exits, counts, oi, synced, iters, flags, seeds, seam_ctr, scan, seqc, classes,
      perm, freq, start, tune, caps, total;
  Ws(const bh_stream* s, const bh_tune* t) {
    uint64_t ns = nsub_of(s), nq = nseq_of(s);
    uint32_t C = (t && t->t_high) ? t->t_high + 1 : 1;
    // the fused path's epoch header and look-back descriptors come first and
    // are never overwritten by this pipeline (their epochs must survive it)
    size_t o = align16(bh_fused_workspace_bytes(s, 0, t));
    auto take = [&](size_t bytes) { size_t r = o; o = align16(o + bytes); return r; };
    entries = take(8 * ns);
    exits = take(8 * ns);
    counts = take(8 * ns);
    oi = take(8 * (ns + 1));
    synced = take(ns);
    iters = take(4 * nq);
    flags = take(2 * ns);
    seeds = take(8 * nq);  // must directly follow flags (bh_inter_sync_pass layout)
    seam_ctr = take(8 * (MAX_SEAM_PASSES + 2));
    scan = take(bh_scan_workspace_bytes(ns));
    seqc = take(8 * nq);
    classes = take(8 * nq);
    perm = take(8 * nq);
    freq = take(8 * C);
    start = take(8 * C);
    tune = take(bh_tuner_workspace_bytes(nq, C - 1 ? C - 1 : 1));
    caps = take(4 * C);
    total = o;
  }
};

template <typename T>
T* at(void* ws, size_t off) { return reinterpret_cast<T*>(static_cast<char*>(ws) + off); }

}  // namespace

extern "C" int bh_version(void) { return 100; }

// ---- phase profiler ---------------------------------------------------------
// Every decoder phase is bracketed by CUDA events recorded on the launching
// stream (prof_mark).  bh_profile_read aggregates the elapsed time between
// consecutive marks per phase name; the interval ending at a "start" mark
// (whatever ran between two decodes, e.g. an L2 flush) is dropped.
namespace {
constexpr int PROF_MAX = 8192;
cudaEvent_t g_ev[PROF_MAX];
const char* g_name[PROF_MAX];
int g_nev = 0;
bool g_prof = false;
bool g_ev_made = false;
}  // namespace

void bh::prof_mark(cudaStream_t st, const char* phase) {
  if (!g_prof || g_nev >= PROF_MAX) return;
  cudaEventRecord(g_ev[g_nev], st);
  g_name[g_nev] = phase;
  ++g_nev;
}

extern "C" int bh_profile_enable(int on) {
  if (on && !g_ev_made) {
    for (int i = 0; i < PROF_MAX; ++i)
      if (cudaEventCreate(&g_ev[i]) != cudaSuccess) return BH_CUDA_ERROR;
    g_ev_made = true;
  }
  g_prof = on != 0;
  g_nev = 0;
  return BH_OK;
}

// names: newline-separated phase names; ms: summed milliseconds; count: number
// of intervals per phase.  Returns the number of distinct phases (<= cap).
extern "C" int bh_profile_read(char* names, size_t names_len, float* ms, uint32_t* count, int cap) {
  if (names_len) names[0] = 0;
  if (g_nev < 2) { g_nev = 0; return 0; }
  if (cudaEventSynchronize(g_ev[g_nev - 1]) != cudaSuccess) return -BH_CUDA_ERROR;
  const char* uniq[64];
  int nu = 0;
  for (int i = 1; i < g_nev; ++i) {
    if (!strcmp(g_name[i], "start")) continue;
    int k = 0;
    while (k < nu && strcmp(uniq[k], g_name[i])) ++k;
    if (k == nu) {
      if (nu >= cap || nu >= 64) continue;
      uniq[nu] = g_name[i];
      ms[nu] = 0.f;
      count[nu] = 0;
      ++nu;
    }
    float t = 0.f;
    cudaEventElapsedTime(&t, g_ev[i - 1], g_ev[i]);
    ms[k] += t;
    count[k] += 1;
  }
  size_t used = 0;
  for (int k = 0; k < nu; ++k) {
    size_t l = strlen(uniq[k]);
    if (used + l + 2 >= names_len) break;
    memcpy(names + used, uniq[k], l);
    used += l;
    names[used++] = '\n';
    names[used] = 0;
  }
  g_nev = 0;
  return nu;
}

static bool use_fused(const bh_stream* s, int variant, const bh_tune* tune) {
  return (!tune || tune->fused) && bh_fused_supported(s, variant);
}

extern "C" const char* bh_status_string(int status) {
  switch (status) {
    case BH_OK: return "ok";
    case BH_INVALID: return "no codeword matches the bits";
    case BH_TRUNCATED: return "synchronized counts disagree with the header symbol count";
    case BH_BADGAP: return "gap entries disagree with the header symbol count";
    case BH_NOFIXPOINT: return "synchronization did not converge";
    case BH_NOTPRESENT: return "stream carries no gap array";
    case BH_GAPOVERFLOW: return "gap entry does not fit in one byte";
    case BH_BAD_ARGUMENT: return "bad argument";
    case BH_CUDA_ERROR: return "CUDA error";
    case BH_NEED_STAGED: return "fused path declined (rerun staged)";
    case BH_LENGTHOVERFLOW: return "optimal code needs more than 32 bits";
    case BH_EMPTY: return "no symbol has a nonzero count";
    default: return "unknown status";
  }
}

extern "C" size_t bh_workspace_bytes(const bh_stream* s, int variant, const bh_tune* tune) {
  if (!s || !s->subseq_bits || !s->subseqs_per_seq) return 0;
  (void)variant;
  return Ws(s, tune).total;  // fused descriptors + the staged pipeline's arrays
}

// Reference-structured pipeline (every phase a separate kernel).
static int staged_pipeline(const bh_stream* s, int variant, const bh_tune* tune, uint16_t* out,
                           void* ws, size_t ws_bytes, void* rep, void* st, bool host_loop) {
  Ws L(s, tune);
  if (ws_bytes < L.total) return BH_BAD_ARGUMENT;
  const uint64_t ns = nsub_of(s), nq = nseq_of(s);
  int64_t* entries = at<int64_t>(ws, L.entries);
  int64_t* exits = at<int64_t>(ws, L.exits);
  int64_t* counts = at<int64_t>(ws, L.counts);
  int64_t* oi = at<int64_t>(ws, L.oi);
  const int stats = tune && tune->collect_stats;
  int rc;
  prof_mark(S(st), "start");
  stamp_phase(rep, 0, S(st));
  if (variant == BH_VARIANT_GAP) {
    if ((rc = bh_entries_from_gap(s, entries, st))) return rc;
    prof_mark(S(st), "entries_from_gap");
    stamp_phase(rep, 1, S(st));
    if ((rc = bh_count_windows(s, 1, entries, counts, exits, rep, st))) return rc;
    prof_mark(S(st), "count_pass");
    stamp_phase(rep, 2, S(st));
  } else {
    if ((rc = bh_intra_sync_ex(s, nullptr, 0, nullptr, entries, exits, counts, at<uint8_t>(ws, L.synced),
                               at<int32_t>(ws, L.iters), at<void>(ws, L.flags), 2 * ns + 8 * nq + 16, rep, st)))
      return rc;
    prof_mark(S(st), "intra_sync");
    stamp_phase(rep, 1, S(st));
    unsigned long long* ctr = at<unsigned long long>(ws, L.seam_ctr);
    int64_t* seeds = at<int64_t>(ws, L.seeds);
    if (nq > 1) {
      cudaMemsetAsync(ctr, 0, 8 * (MAX_SEAM_PASSES + 2), S(st));
      int passes = tune && tune->seam_passes ? (int)tune->seam_passes : 2;
      if (passes > MAX_SEAM_PASSES) passes = MAX_SEAM_PASSES;
      if (host_loop) {
        // sync_decoder.py:129-149 exactly: snapshot, stop when nothing is stale
        for (uint64_t p = 0;; ++p) {
          unsigned long long stale = 0;
          int32_t dev_status = 0;
          cudaMemsetAsync(ctr, 0, 8, S(st));
          if ((rc = bh_seam_check(s, entries, exits, seeds, ctr, st))) return rc;
          if (cudaMemcpyAsync(&stale, ctr, 8, cudaMemcpyDeviceToHost, S(st)) != cudaSuccess) return BH_CUDA_ERROR;
          if (cudaMemcpyAsync(&dev_status, rep, 4, cudaMemcpyDeviceToHost, S(st)) != cudaSuccess) return BH_CUDA_ERROR;
          if (cudaStreamSynchronize(S(st)) != cudaSuccess) return BH_CUDA_ERROR;
          if (dev_status != 0x7fffffff) break;  // an intra/seam decode failed: the report says why
          if (!stale) break;
          if (p >= nq) return BH_NOFIXPOINT;
          if ((rc = bh_intra_sync_ex(s, seeds, 0, ctr, entries, exits, counts, at<uint8_t>(ws, L.synced),
                                     at<int32_t>(ws, L.iters), at<void>(ws, L.flags),
                                     2 * ns + 8 * nq + 16, rep, st)))
            return rc;
        }
      } else {
        for (int p = 0; p < passes; ++p) {
          if ((rc = bh_seam_check(s, entries, exits, seeds, ctr + p, st))) return rc;
          if ((rc = bh_intra_sync_ex(s, seeds, 0, ctr + p, entries, exits, counts, at<uint8_t>(ws, L.synced),
                                     at<int32_t>(ws, L.iters), at<void>(ws, L.flags),
                                     2 * ns + 8 * nq + 16, rep, st)))
            return rc;
        }
        // final check: counter[passes] must be zero, else the host finishes
        if ((rc = bh_seam_check(s, entries, exits, seeds, ctr + passes, st))) return rc;
      }
    }
    prof_mark(S(st), "inter_sync");
    stamp_phase(rep, 2, S(st));
  }
  if ((rc = bh_output_index(counts, ns, oi, at<void>(ws, L.scan), bh_scan_workspace_bytes(ns), st))) return rc;
  if ((rc = bh_check_total(s, oi, variant == BH_VARIANT_GAP ? BH_BADGAP : BH_TRUNCATED, rep, st))) return rc;
  prof_mark(S(st), "output_index");
  stamp_phase(rep, 3, S(st));
  if (tune && tune->t_high) {
    const uint32_t C = tune->t_high + 1;
    int64_t* seqc = at<int64_t>(ws, L.seqc);
    if ((rc = bh_sequence_counts(s, counts, seqc, st))) return rc;
    if ((rc = bh_tuner_plan(s, seqc, tune->t_high, at<int64_t>(ws, L.classes), at<int64_t>(ws, L.freq),
                            at<int64_t>(ws, L.perm), at<int64_t>(ws, L.start), at<void>(ws, L.tune),
                            bh_tuner_workspace_bytes(nq, tune->t_high), st)))
      return rc;
    uint32_t caps[256];
    uint32_t maxcap = 1;
    for (uint32_t c = 1; c <= C; ++c) {
      caps[c - 1] = class_capacity(c, tune);
      if (caps[c - 1] > maxcap) maxcap = caps[c - 1];
    }
    uint32_t* caps_dev = at<uint32_t>(ws, L.caps);
    if ((rc = bh_fill_caps(caps_dev, caps, C, st))) return rc;
    prof_mark(S(st), "tune");
    stamp_phase(rep, 4, S(st));
    rc = bh_decode_write_classes(s, entries, counts, oi, at<int64_t>(ws, L.perm), nq, 0, maxcap,
                                 at<int64_t>(ws, L.classes), caps_dev, out, s->symbol_count, rep,
                                 stats, st);
    prof_mark(S(st), "decode_write");
    stamp_phase(rep, 5, S(st));
    return rc;
  }
  uint32_t cap = tune && tune->capacity ? tune->capacity : 3584;
  stamp_phase(rep, 4, S(st));
  rc = bh_decode_write_classes(s, entries, counts, oi, nullptr, nq, cap, cap, nullptr, nullptr, out,
                               s->symbol_count, rep, stats, st);
  prof_mark(S(st), "decode_write");
  stamp_phase(rep, 5, S(st));
  return rc;
}

extern "C" int bh_decode_async(const bh_stream* s, int variant, const bh_tune* tune, uint16_t* out_dev,
                               void* ws, size_t ws_bytes, void* report_dev, void* cuda_stream) {
  if (!s || !s->subseq_bits || !s->subseqs_per_seq || !s->table_dev || !report_dev) return BH_BAD_ARGUMENT;
  if (variant != BH_VARIANT_GAP && variant != BH_VARIANT_SYNC) return BH_BAD_ARGUMENT;
  if (variant == BH_VARIANT_GAP && !s->gap_dev && s->total_bits) return BH_NOTPRESENT;
  if (s->total_bits && use_fused(s, variant, tune))
    return bh_fused_decode(s, variant, tune, out_dev, ws, ws_bytes, report_dev, cuda_stream);
  // chunked streams (first_entry) are fused-path only, and need a 16-byte
  // aligned payload (shard.chunk_stream cuts at 128-bit multiples)
  if (s->first_entry || (s->flags & BH_STREAM_COUNT_IS_CAPACITY)) return BH_BAD_ARGUMENT;
  int rc = bh_report_init(report_dev, cuda_stream);
  if (rc) return rc;
  if (s->total_bits == 0) {
    // empty stream: nothing to decode; header count must be zero
    return bh_check_total(s, nullptr, variant == BH_VARIANT_GAP ? BH_BADGAP : BH_TRUNCATED, report_dev,
                          cuda_stream);
  }
  return staged_pipeline(s, variant, tune, out_dev, ws, ws_bytes, report_dev, cuda_stream, false);
}

extern "C" size_t bh_decode_workspace_bytes(const bh_stream* s, int variant, const bh_tune* tune) {
  return align16(bh_workspace_bytes(s, variant, tune)) + align16(bh_report_bytes());
}

extern "C" int bh_decode(const bh_stream* s, int variant, const bh_tune* tune, uint16_t* out_dev,
                         void* ws, size_t ws_bytes, bh_report* report_host, void* cuda_stream) {
  // the report lives at the front of a private allocation-free slot: the
  // caller's workspace tail
  size_t need = bh_workspace_bytes(s, variant, tune);
  if (ws_bytes < need + align16(bh_report_bytes())) return BH_BAD_ARGUMENT;
  void* rep = static_cast<char*>(ws) + align16(need);
  // the slot may hold another call's scratch (its position follows this
  // stream's workspace size): the fused kernels' epoch-tagged status must
  // start from a clean report
  int rc = bh_report_init(rep, cuda_stream);
  if (rc) return rc;
  rc = bh_decode_async(s, variant, tune, out_dev, ws, need, rep, cuda_stream);
  if (rc) return rc;
  bh_report r;
  memset(&r, 0, sizeof(r));
  if ((rc = bh_report_read(rep, &r, cuda_stream))) return rc;
  if (r.status == BH_NEED_STAGED) {
    // the fused path declined (incomplete codebook): the reference-structured
    // pipeline reproduces the reference's speculative windows exactly.  It
    // decodes whole streams only: a chunk (first_entry != 0) cannot take it.
    if (s->first_entry || (s->flags & BH_STREAM_COUNT_IS_CAPACITY)) return BH_BAD_ARGUMENT;
    if ((rc = bh_report_init(rep, cuda_stream))) return rc;
    if ((rc = staged_pipeline(s, variant, tune, out_dev, ws, need, rep, cuda_stream, true))) return rc;
    if ((rc = bh_report_read(rep, &r, cuda_stream))) return rc;
    r.repair_needed = 1;
  } else if ((r.status == BH_OK || r.status == BH_TRUNCATED) && variant == BH_VARIANT_SYNC &&
             !use_fused(s, variant, tune) && nseq_of(s) > 1 && s->total_bits) {
    // staged async pipeline: the final pre-launched seam check must be clean
    Ws L(s, tune);
    int passes = tune && tune->seam_passes ? (int)tune->seam_passes : 2;
    if (passes > MAX_SEAM_PASSES) passes = MAX_SEAM_PASSES;
    unsigned long long ctr[MAX_SEAM_PASSES + 1];
    if (cudaMemcpyAsync(ctr, at<unsigned long long>(ws, L.seam_ctr), 8 * (passes + 1), cudaMemcpyDeviceToHost,
                        S(cuda_stream)) != cudaSuccess)
      return BH_CUDA_ERROR;
    if (cudaStreamSynchronize(S(cuda_stream)) != cudaSuccess) return BH_CUDA_ERROR;
    uint64_t used = 0;
    for (int p = 0; p < passes; ++p) used += ctr[p] ? 1 : 0;
    r.seam_passes = used;
    r.stale_seams = ctr[passes];
    if (ctr[passes]) {
      if ((rc = bh_report_init(rep, cuda_stream))) return rc;
      if ((rc = staged_pipeline(s, variant, tune, out_dev, ws, need, rep, cuda_stream, true))) return rc;
      if ((rc = bh_report_read(rep, &r, cuda_stream))) return rc;
    }
  }
  if (report_host) *report_host = r;
  return r.status;
}
