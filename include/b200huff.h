/*
 * b200huff.h -- C ABI of the B200 (sm_100a) Huffman decode library.
 *
 * Drop-in boundary for the decode path of the reference package `parhuff`
 * (paths relative to /root/reference/pkg/src/parhuff/).  Plain pointers and
 * sizes only; every entry point returns an int status, never throws, is
 * stream-ordered on the caller's cudaStream_t (passed as void*), and keeps its
 * scratch in a caller-owned device workspace.  All array pointers named *_dev
 * are device pointers; everything else is host memory.
 *
 * Status codes keep the values of the reference kernel statuses
 * (kernels.py:22-24) and extend them with the Python exception classes the
 * reference raises (errors.py:28-58); the Python wrapper maps them back.
 */
#ifndef B200HUFF_H
#define B200HUFF_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BH_OK 0            /* kernels.OK */
#define BH_INVALID 1       /* kernels.ERR_INVALID -> InvalidCode (_dispatch.py:55-57) */
#define BH_TRUNCATED 2     /* kernels.ERR_TRUNCATED -> Truncated (sync_decoder.py:200-204) */
#define BH_BADGAP 3        /* BadGap (gap_decoder.py:63-67) */
#define BH_NOFIXPOINT 4    /* NoFixpoint (sync_decoder.py:105-106,149) */
#define BH_NOTPRESENT 5    /* NotPresent (gap_decoder.py:26-27) */
#define BH_GAPOVERFLOW 6   /* GapOverflow (encoder.py:86-87) */
#define BH_BAD_ARGUMENT 7  /* ValueError-class misuse (layout, capacity < 1, ...) */
#define BH_CUDA_ERROR 8    /* CUDA runtime failure */
#define BH_NEED_STAGED 9   /* fused path declined (incomplete codebook, or a gap entry inside a
                                  lane window that is not a codeword start); bh_decode reruns staged */
#define BH_LENGTHOVERFLOW 10 /* LengthOverflow: an optimal code needs > 32 bits (codebook.py:76-79) */
#define BH_EMPTY 11          /* EmptyInput: no symbol has a nonzero count (codebook.py:46-47) */

#define BH_VARIANT_GAP 1     /* gap_decoder.decode (gap_decoder.py:71-92) */
#define BH_VARIANT_SYNC 2    /* sync_decoder.decode (sync_decoder.py:173-211) */
#define BH_VARIANT_COARSE 3  /* cuSZ-style coarse-grained in-run baseline (K8) */

#define BH_WORD_PAD 8        /* zero words the caller appends after the payload */

/* Encoded stream as seen by the device: the reference EncodedStream
 * (bitstream.py:61-131) with its units normalised to one MSB-first 32-bit word
 * stream (identity for unit_bits == 32; bh_repack_units for 8/16). */
typedef struct bh_stream {
    const uint32_t *words_dev;   /* ceil(total_bits/32) words + BH_WORD_PAD zero words */
    uint64_t total_bits;
    uint64_t symbol_count;       /* header count */
    uint32_t subseq_bits;        /* LayoutConfig.subseq_bits */
    uint32_t subseqs_per_seq;    /* LayoutConfig.subseqs_per_seq */
    uint32_t symbol_width;       /* Codebook.symbol_width (tuner ratio) */
    uint32_t max_codes;          /* capacity the table blob was sized for */
    const uint8_t *gap_dev;      /* num_subseqs forward skips, or NULL */
    const void *table_dev;       /* blob from bh_table_build*() */
    uint32_t first_entry;        /* bit offset of the first codeword start; 0 for a whole
                                    stream, the chunk's first gap byte for a sequence-aligned
                                    chunk of a longer stream (sharded decode; fused path only) */
    uint32_t flags;              /* BH_STREAM_* (0 for a whole stream) */
} bh_stream;

/* flags: symbol_count is only the output capacity of a chunk whose count is
 * not known (a shard read straight from a container): the decode reports the
 * count in bh_report.total_symbols and fails with BH_TRUNCATED only if it
 * exceeds the capacity (fused path only). */
#define BH_STREAM_COUNT_IS_CAPACITY 1u

/* Tuning knobs (tuner.py:29-40 TunerConfig, staging.py:28 DEFAULT_CAPACITY). */
typedef struct bh_tune {
    uint32_t t_high;             /* 0 = no tuner (plain decode_write) */
    uint32_t capacity;           /* staging symbols when t_high == 0 */
    uint32_t capacity_table[64]; /* per 1-based class overrides (0 = rule) */
    uint32_t early_exit;         /* accepted for parity; results do not depend on it */
    uint32_t collect_stats;      /* fill bits/rounds/staged/bypass (slower) */
    uint32_t fused;              /* 1 = single-pass fused kernels (default), 0 = staged pipeline */
    uint32_t seam_passes;        /* pre-launched seam passes before the status read (>=1) */
    uint32_t max_len;            /* longest code length when known (0 = unknown); <= 8 lets the
                                    fused kernel leave the 12-bit second-level table out of
                                    shared memory (more warps per SM) */
    uint32_t ctas;               /* fused kernel CTAs (0 = one per SM): several decodes on
                                    concurrent streams can share the GPU in one wave */
    uint32_t min_len;            /* shortest code length when known (0 = unknown); >= 4 lets
                                    long-code books use the 8-byte three-codeword table */
} bh_tune;

/* Decode report, mirroring DecodeStats (staging.py:31-45) plus status. */
typedef struct bh_report {
    int32_t status;
    int32_t pad0;
    uint64_t fail_slot;
    uint64_t bits_sync;
    uint64_t bits_count;
    uint64_t bits_write;
    uint64_t write_rounds;
    uint64_t staged_slots;
    uint64_t bypass_slots;
    uint64_t total_symbols;
    uint64_t stale_seams;
    uint64_t seam_passes;
    uint64_t repair_needed;
    uint64_t pad[4];
    /* Device phase boundaries (globaltimer ns) of the last call, valid when the
     * report was initialised (bh_report_init; bh_decode always does): [0] start,
     * then the end of each phase in the reference's order --
     *   GAP  (gap_decoder.py:82-92):  [1] entries_from_gap, [3] count_pass
     *                                 (incl. the output index), [4] tune,
     *                                 [5] decode_write;  [2] count loop end
     *   SYNC (sync_decoder.py:185-211): [1] intra_sync, [2] inter_sync,
     *                                 [3] output_index, [4] tune, [5] decode_write
     * The fused kernel stamps them in-kernel (max over CTAs; tune takes no
     * time there), the staged pipeline with a one-thread stamp kernel between
     * its launches. */
    uint64_t phase_ns[6];
} bh_report;

/* ---- library ---------------------------------------------------------- */
int bh_version(void);
const char *bh_status_string(int status);
int bh_device_sm_count(void);

/* ---- K1: decode tables (codebook.py:86-112 canonize, :183-260 DecodeTable) */
size_t bh_table_bytes(uint32_t max_codes);
/* canonical book from one length byte per symbol value (container.py:50-57) */
int bh_table_build(const uint8_t *lengths_dev, uint32_t alphabet, void *table_dev,
                   uint32_t max_codes, void *cuda_stream);
/* explicit book: dense codes/lens per symbol value (lens 0 = absent) */
int bh_table_build_explicit(const uint32_t *codes_dev, const uint8_t *lens_dev,
                            uint32_t alphabet, void *table_dev, uint32_t max_codes,
                            void *cuda_stream);
/* canonical code per symbol (encode side); codes_dev[alphabet] */
int bh_canonical_codes(const uint8_t *lengths_dev, uint32_t alphabet, uint32_t *codes_dev,
                       void *cuda_stream);

/* ---- codebook construction on the device (codebook.py:38-83 build_lengths) */
/* scratch for the histogram counters: u64 per symbol value */
size_t bh_book_workspace_bytes(uint32_t alphabet);
/* counts_dev[s] = occurrences of s among symbols_dev[0..n) (16-byte aligned) */
int bh_symbol_histogram(const uint16_t *symbols_dev, uint64_t n, uint32_t alphabet,
                        uint64_t *counts_dev, void *cuda_stream);
/* Huffman code lengths identical to the reference build_lengths (ties by
 * (count, symbol), merged subtrees after same-count leaves); lengths_dev[s] = 0
 * for absent symbols; *status_dev = BH_OK / BH_LENGTHOVERFLOW / BH_EMPTY /
 * BH_BAD_ARGUMENT (more than 4096 distinct symbols) */
int bh_build_lengths(const uint64_t *counts_dev, uint32_t alphabet, uint8_t *lengths_dev,
                     int32_t *status_dev, void *cuda_stream);

/* ---- dequantization after decode (kernels.py:216-227 dequantize_chain) --
 * out_dev[i] = the reference reconstruction of code i, float64.
 * exact_scan = 1: one-pass segmented prefix sum (decoupled look-back) valid in
 *   the exact regime -- twice_eb a power of two 2^e (-149 <= e <= 104), every
 *   outlier value an integer multiple of twice_eb (outlier_units_dev = value /
 *   twice_eb) -- as long as every running sum stays below 2^24 in magnitude;
 *   *inexact_dev (device int32) is set otherwise (output then unspecified).
 *   BH_BAD_ARGUMENT when twice_eb is not such a power of two.
 * exact_scan = 0: the reference recurrence on one device thread (any regime).
 * Outlier indices ascending; workspace from bh_dequant_workspace_bytes(n). */
size_t bh_dequant_workspace_bytes(uint64_t n);
int bh_dequantize(const uint16_t *codes_dev, uint64_t n, const int64_t *outlier_idx_dev,
                  const double *outlier_val_dev, const int64_t *outlier_units_dev, uint64_t n_outliers,
                  double twice_eb, uint32_t midpoint, int exact_scan, double *out_dev, void *workspace_dev,
                  size_t workspace_bytes, int32_t *inexact_dev, void *cuda_stream);

/* ---- whole-decoder entry point (sync_decoder.decode / gap_decoder.decode) */
size_t bh_workspace_bytes(const bh_stream *s, int variant, const bh_tune *tune);
/* Decodes symbol_count symbols into out_dev (uint16).  report_dev receives a
 * device-side report; nothing is synchronised.  bh_report_read copies it.
 * A report buffer must be initialised (bh_report_init) once before its first
 * use: the fused kernels tag their status with a per-call epoch and never
 * reset it, so repeated (or graph-replayed) calls need no further init. */
int bh_decode_async(const bh_stream *s, int variant, const bh_tune *tune, uint16_t *out_dev,
                    void *workspace_dev, size_t workspace_bytes, void *report_dev,
                    void *cuda_stream);
/* zero a freshly allocated workspace once (descriptors are epoch-tagged, so
 * later calls need no reset) */
int bh_workspace_reset(void *workspace_dev, size_t workspace_bytes, void *cuda_stream);
/* The online tuner on the fused path (tuner.py:117-191): with tune->t_high in
 * 1..64 the fused kernel classifies every tile by its compression ratio and
 * stages it with that class's capacity (tuner.capacity, capacity_table
 * overrides), and histograms the reference sequences into tuner.plan's
 * classes.  This copies that histogram (t_high + 1 counts, n >= t_high + 1)
 * of the last fused decode run with `ws`; BH_BAD_ARGUMENT when the layout does
 * not put whole sequences in a tile. */
int bh_tuner_class_freq(const bh_stream *s, const bh_tune *tune, const void *workspace_dev,
                        uint64_t *freq_host, uint32_t n, void *cuda_stream);
/* 1 when the fused single-kernel decoder takes this stream and variant (the
 * only path for chunks: first_entry or BH_STREAM_COUNT_IS_CAPACITY), else 0. */
int bh_fused_supported(const bh_stream *s, int variant);
/* Synchronous convenience: decode, finish any extra seam passes, read report. */
int bh_decode(const bh_stream *s, int variant, const bh_tune *tune, uint16_t *out_dev,
              void *workspace_dev, size_t workspace_bytes, bh_report *report_host,
              void *cuda_stream);
size_t bh_report_bytes(void);
int bh_report_init(void *report_dev, void *cuda_stream);
int bh_report_read(const void *report_dev, bh_report *report_host, void *cuda_stream);
/* workspace bh_decode needs: bh_workspace_bytes() plus room for its report */
size_t bh_decode_workspace_bytes(const bh_stream *s, int variant, const bh_tune *tune);

/* ---- phase profiler (CUDA events around every phase on the caller's stream) */
int bh_profile_enable(int on);
/* aggregated per phase: names newline-separated, summed ms, interval counts */
int bh_profile_read(char *names, size_t names_len, float *ms, uint32_t *count, int cap);

/* ---- sub-steps with the reference's SyncState arrays (state.py:16-41) --- */
/* int64 entries/exits/counts[num_subseqs], uint8 synced, int32 iterations[num_seqs] */
int bh_intra_sync(const bh_stream *s, int early_exit, int64_t *entries_dev, int64_t *exits_dev,
                  int64_t *counts_dev, uint8_t *synced_dev, int32_t *iterations_dev,
                  void *workspace_dev, size_t workspace_bytes, void *report_dev,
                  void *cuda_stream);
/* intra_sync over selected sequences: seeds_dev[q] = -1 skip, -2 decode from
 * the boundaries (sync_decoder.py:78-81), >= 0 re-seed the first slot
 * (:82-86); seeds_dev NULL = every sequence unseeded.  Optional device gate
 * (skip everything when *gate == 0); round_cap 0 = number of slots.  */
int bh_intra_sync_ex(const bh_stream *s, const int64_t *seeds_dev, uint32_t round_cap,
                     const unsigned long long *gate_dev, int64_t *entries_dev, int64_t *exits_dev,
                     int64_t *counts_dev, uint8_t *synced_dev, int32_t *iterations_dev,
                     void *workspace_dev, size_t workspace_bytes, void *report_dev,
                     void *cuda_stream);
/* seam snapshot: seeds_dev[q] = exit of q's predecessor slot if stale else -1;
 * *counter_dev += number of stale seams */
int bh_seam_check(const bh_stream *s, const int64_t *entries_dev, const int64_t *exits_dev,
                  int64_t *seeds_dev, unsigned long long *counter_dev, void *cuda_stream);
/* one seam pass (sync_decoder.py:133-146); *stale_host gets the stale count */
int bh_inter_sync_pass(const bh_stream *s, int64_t *entries_dev, int64_t *exits_dev,
                       int64_t *counts_dev, uint8_t *synced_dev, int32_t *iterations_dev,
                       void *workspace_dev, size_t workspace_bytes, void *report_dev,
                       uint64_t *stale_host, void *cuda_stream);
/* gap_decoder.py:24-33 entries_from_gap */
int bh_entries_from_gap(const bh_stream *s, int64_t *entries_dev, void *cuda_stream);
/* kernels.py:47-76 over all slots; mode 1 = gap windows [e_i, e_{i+1}),
 * mode 2 = sync windows [e_i, (i+1)*subseq_bits) */
int bh_count_windows(const bh_stream *s, int mode, const int64_t *entries_dev,
                     int64_t *counts_dev, int64_t *exits_dev, void *report_dev,
                     void *cuda_stream);
/* state.py:44-53: out_index_dev[n+1] = exclusive prefix sum (decoupled look-back) */
int bh_output_index(const int64_t *counts_dev, uint64_t n, int64_t *out_index_dev,
                    void *workspace_dev, size_t workspace_bytes, void *cuda_stream);
size_t bh_scan_workspace_bytes(uint64_t n);
/* staging.py:65-147: staged decode-and-write of the listed sequences
 * (seq_ids_dev NULL = all) with the given capacity */
int bh_decode_write(const bh_stream *s, const int64_t *entries_dev, const int64_t *counts_dev,
                    const int64_t *out_index_dev, const int64_t *seq_ids_dev, uint64_t nseq_ids,
                    uint32_t capacity, uint16_t *out_dev, uint64_t out_len, void *report_dev,
                    void *cuda_stream);
/* decode_partitioned (tuner.py:150-191) in one launch: sequence q of the list
 * uses caps_dev[classes_dev[q]-1] (or `capacity` when classes_dev is NULL) */
int bh_decode_write_classes(const bh_stream *s, const int64_t *entries_dev, const int64_t *counts_dev,
                            const int64_t *out_index_dev, const int64_t *seq_ids_dev,
                            uint64_t nseq_ids, uint32_t capacity, uint32_t max_capacity,
                            const int64_t *classes_dev, const uint32_t *caps_dev, uint16_t *out_dev,
                            uint64_t out_len, void *report_dev, int stats, void *cuda_stream);
/* per-class capacities copied through the launch (n <= 256) */
int bh_fill_caps(uint32_t *caps_dev, const uint32_t *caps_host, uint32_t n, void *cuda_stream);
/* header check: out_index_dev[num_subseqs] vs symbol_count */
int bh_check_total(const bh_stream *s, const int64_t *out_index_dev, int status_on_mismatch,
                   void *report_dev, void *cuda_stream);
/* tuner.py:117-147 plan on device; classes/perm [num_seqs], freq/start [t_high+1] */
int bh_tuner_plan(const bh_stream *s, const int64_t *seq_counts_dev, uint32_t t_high,
                  int64_t *classes_dev, int64_t *freq_dev, int64_t *perm_dev,
                  int64_t *start_dev, void *workspace_dev, size_t workspace_bytes,
                  void *cuda_stream);
size_t bh_tuner_workspace_bytes(uint64_t num_seqs, uint32_t t_high);
/* tuner.py:109-114 sequence_counts */
int bh_sequence_counts(const bh_stream *s, const int64_t *subseq_counts_dev,
                       int64_t *seq_counts_dev, void *cuda_stream);

/* ---- encode side (encoder.py:33-97, kernels.py:151-179) ----------------- */
size_t bh_encode_workspace_bytes(uint64_t n);
/* pass 1: total bits (written to *total_bits_host; synchronises) */
int bh_encode_size(const uint16_t *symbols_dev, uint64_t n, const uint8_t *lens_dev,
                   uint32_t alphabet, void *workspace_dev, size_t workspace_bytes,
                   uint64_t *total_bits_host, uint64_t *bad_symbol_host, void *cuda_stream);
/* pass 2: words_dev (ceil(tb/32)+BH_WORD_PAD, zeroed here) and gap_dev (nsub) or NULL;
 * chunk_offsets_dev (optional) receives the start bit of every chunk-th symbol */
int bh_encode_pack(const uint16_t *symbols_dev, uint64_t n, const uint32_t *codes_dev,
                   const uint8_t *lens_dev, uint64_t total_bits, uint32_t subseq_bits,
                   uint32_t *words_dev, uint8_t *gap_dev, uint64_t chunk,
                   uint64_t *chunk_offsets_dev, void *workspace_dev, size_t workspace_bytes,
                   void *cuda_stream);
/* units (uint32 holding unit_bits each) -> MSB-first 32-bit words (+pad) */
int bh_repack_units(const uint32_t *units_dev, uint64_t n_units, uint32_t unit_bits,
                    uint32_t *words_dev, uint64_t n_words, void *cuda_stream);

/* ---- ground truth on the device (encoder.py:129-188) ------------------- */
/* mode 0: oracle_decode of n symbols from start_bit (starts_dev optional);
 * mode 1: mis_sync_decode from start_bit to total_bits.
 * result_dev[0] = status, result_dev[1] = symbols produced. */
int bh_sequential_decode(const bh_stream *s, uint64_t start_bit, uint64_t n, int mode,
                         uint16_t *out_dev, int64_t *starts_dev, uint64_t *result_dev,
                         void *cuda_stream);
/* counts_dev[nsub] = number of starts inside each subsequence */
int bh_start_histogram(const int64_t *starts_dev, uint64_t n, uint32_t subseq_bits,
                       int64_t *counts_dev, uint64_t nsub, void *cuda_stream);

/* ---- K8: coarse-grained cuSZ-style baseline decoder --------------------- */
/* one thread per `chunk` symbols, bit-serial canonical decode, direct writes */
int bh_coarse_decode(const bh_stream *s, const uint64_t *chunk_offsets_dev, uint64_t chunk,
                     uint16_t *out_dev, void *report_dev, void *cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* B200HUFF_H */
