/*
 * sgns_b200.h -- C ABI of the B200-native pSGNScc hot path.
 *
 * All pointers named d_* are device pointers (HBM); h_* are host pointers.
 * Every device entry point is stream-ordered on `stream` (a cudaStream_t
 * passed as void*), allocates nothing, and returns 0 or a status:
 *   > 0  a cudaError_t from the launch,
 *   < 0  SGNS_E_* validation errors below.
 * No torch types cross this boundary; INTEGRATION.md shows the ctypes
 * binding the reference package would add.
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/sgns):
 *   sgns_update_windows  <- batch_core_blas / batch_core_naive
 *                           (kernel_batched.py:92-144, :147-211) behind
 *                           process_batch (kernel_batched.py:214-260)
 *   sgns_drive           <- _drive_batched (trainer.py:217-311) behind
 *                           ThreadRun.advance(word_budget) (trainer.py:396-442);
 *                           includes _subsample (corpus.py:168-181), the window
 *                           assembly (trainer.py:260-280), chunking and
 *                           fill_shared_negatives (kernel_batched.py:57-66)
 *   sgns_init_model      <- init_model (model.py:64-74)
 *   sgns_expand_slots    <- build_negative_table's slot array (corpus.py:139-155)
 *   sgns_build_alias     <- (new) Vose alias table over count^0.75, the
 *                           production replacement of the 10^8-slot table
 */
#ifndef SGNS_B200_H
#define SGNS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SGNS_ABI_VERSION 2

enum {
  SGNS_OK = 0,
  SGNS_E_ARG = -1,       /* bad argument (null pointer, size, mode) */
  SGNS_E_SHAPE = -2,     /* dim / window / K / batch_cap outside the supported envelope */
  SGNS_E_SMEM = -3,      /* per-warp staging does not fit in shared memory */
  SGNS_E_DEVICE = -4,    /* device-side validation failed (see sgns_error_string) */
  SGNS_E_IO = -5,        /* corpus file could not be opened / mapped */
  SGNS_E_EMPTY = -6,     /* no token reaches min_count (EmptyVocabularyError) */
  SGNS_E_TRUNC = -7      /* vector file ends inside a row (ModelFormatError "truncated") */
};

enum { SGNS_F32 = 0, SGNS_F64 = 1 };
enum { SGNS_SIGMOID_TABLE = 0, SGNS_SIGMOID_EXACT = 1 };
enum { SGNS_RNG_SPLITMIX = 0, SGNS_RNG_PHILOX = 1 };

/* Per-worker resumable state (one worker = one warp = one reference thread,
 * ThreadRun fields trainer.py:358-366, alpha_state :365). Device resident. */
typedef struct sgns_worker {
  int64_t next_sent, lo, hi;
  int32_t epoch, done;
  uint64_t rng;                       /* splitmix64 state (SGNS_RNG_SPLITMIX) */
  double alpha, read_local, trained_local;
  int64_t kernel_counter, words_read, words_trained;
  int64_t inputs;                     /* sum of chunk input counts (roofline accounting) */
} sgns_worker;

/* Row stride ld (elements) of M_in / M_out: any multiple of 16 bytes >= dim.  The kernels
 * read and write the dim data columns only (whole 16-byte chunks: columns from dim up to the
 * next multiple of 16 bytes must be zero, as sgns_init_model leaves them); the rest of a
 * padded row is never touched.  Fastest when rows start on 128-byte lines (float32: ld a
 * multiple of 32, e.g. 320 at dim = 300; the Python package's padded_ld allocates that way),
 * and at least on 32-byte sectors (ld * sizeof(elem) % 32 == 0): see DESIGN.md section 2.
 *
 * One batch of packed windows (the CSR form of a list of Minibatch,
 * kernel_batched.py:37-54): window w has inputs in_ids[in_off[w]:in_off[w+1]]
 * and outputs out_ids[w*k1 : (w+1)*k1], target first.  n_windows == 0 is a no-op
 * (SGNS_OK before any pointer is inspected). */
int sgns_update_windows(
    int32_t dtype,
    void *d_m_in_dst, void *d_m_out_dst,              /* rows receive += deltas */
    const void *d_m_in_src, const void *d_m_out_src,  /* rows are gathered from here */
    int64_t vocab, int32_t dim, int64_t ld,           /* ld: row stride in elements, multiple of 16 B */
    const int32_t *d_in_off, const int32_t *d_in_ids, const int32_t *d_out_ids,
    int32_t n_windows, int32_t k1, int32_t max_inputs,
    const void *d_alpha,                              /* per window, model dtype */
    const void *d_sig_table,                          /* 1000 entries, model dtype */
    int32_t sigmoid_mode, int32_t loss_every,
    double *d_loss_sum, int64_t *d_loss_cells,        /* may be NULL when loss_every == 0 */
    int32_t *d_error,                                 /* may be NULL */
    void *stream);

typedef struct sgns_drive_params {
  int32_t dtype;
  void *d_m_in, *d_m_out;
  int64_t vocab, ld;
  int32_t dim;
  const int32_t *d_ids;          /* corpus token ids */
  const int64_t *d_offsets;      /* sentence offsets, n_sentences + 1 */
  const double *d_keep_probs;    /* NULL: no subsampling */
  int32_t rng_mode;
  const int32_t *d_slots;        /* SPLITMIX: reference slot table */
  int64_t n_slots;
  const uint32_t *d_alias_thr;   /* PHILOX: alias thresholds (x 2^32) */
  const int32_t *d_alias_idx;
  uint64_t seed;                 /* PHILOX key */
  int32_t window, dynamic, k_neg, batch_cap, sigmoid_mode;
  const void *d_sig_table;
  double alpha0, floor_frac, total_x_epochs;
  int64_t refresh_words;         /* ALPHA_REFRESH_WORDS (trainer.py:48) */
  int64_t *d_shared;             /* [2] words read / trained, shared by all workers */
  int32_t epochs, loss_every;
  sgns_worker *d_workers;
  int32_t n_workers;
  int64_t word_budget;           /* per worker, words read (trainer.py:237) */
  double *d_loss_by_epoch;       /* [n_workers * epochs] */
  int64_t *d_cells_by_epoch;
  int32_t update;                /* 0: draw / trace only */
  int32_t max_sentence;          /* longest sentence in tokens (<= 1024) */
  int64_t trace_cap;             /* records per worker; 0 disables tracing */
  int32_t *d_trace;              /* [n_workers][trace_cap][4 + batch_cap + k1] */
  double *d_trace_alpha;         /* [n_workers][trace_cap] */
  int64_t *d_trace_count;        /* [n_workers] */
  int32_t *d_error;              /* may be NULL */
  int32_t warps_per_block;       /* 0: default */
  int64_t token_base;            /* PHILOX: corpus position of d_ids[0] (streamed chunks) */
  int32_t epoch_base;            /* PHILOX: epoch index added to each worker's epoch */
  /* SGNS_SCHEDULE_DYNAMIC (PHILOX, float32, k_neg + 1 <= 8, dim <= 512): workers claim
   * sentence ordinals c in [*d_claim, claim_end) of the shard [shard_lo, shard_hi)
   * (epoch = c / n, sentence = shard_lo + c % n); alpha from the sentence's words-read
   * position words_base + epoch * shard_tokens + offset; d_workers only collects counters. */
  int32_t schedule;
  uint64_t *d_claim;
  int64_t claim_end;
  int64_t shard_lo, shard_hi;
  int64_t words_base;
  /* optional (dynamic schedule): per-launch totals accumulated by the workers at exit,
   * int64[6] = {words_trained, words_read, chunks, inputs, loss_cells, (unused)} and
   * double[1] = {loss_sum}; the caller zeroes them before the launch. */
  int64_t *d_totals;
  double *d_loss_total;
  /* optional: touched-row map, uint8[2 * vocab] = {M_in rows, M_out rows}; every window
   * sets the bytes of its m input rows and k + 1 output rows to 1 (plain stores, never
   * cleared by the kernels).  Data-parallel touched-row averaging reads it. */
  uint8_t *d_dirty;
} sgns_drive_params;

enum { SGNS_SCHEDULE_STATIC = 0, SGNS_SCHEDULE_DYNAMIC = 1 };

/* Fused resumable driver: every worker consumes up to word_budget words read. */
int sgns_drive(const sgns_drive_params *p, void *stream);

/* M_in ~ U(-0.5/dim, 0.5/dim) from the splitmix stream (seed, 0x1017), M_out = 0,
 * padding columns [dim, ld) = 0.  Bit-identical to init_model. */
int sgns_init_model(int32_t dtype, void *d_m_in, void *d_m_out, int64_t vocab, int32_t dim,
                    int64_t ld, uint64_t seed, void *stream);

/* slots[s] = word owning slot s given build_negative_table's boundaries. */
int sgns_expand_slots(const int64_t *d_boundaries, int64_t vocab, int32_t *d_slots,
                      int64_t n_slots, void *stream);

/* Host: Vose alias table over count^power (float64). thr[i] = floor(p_i * 2^32). */
int sgns_build_alias(const int64_t *h_counts, int64_t vocab, double power,
                     uint32_t *h_thr, int32_t *h_alias);

/* Occupancy-derived worker count: resident warps of the driver kernel. */
int sgns_resident_workers(int32_t dtype, int32_t dim, int32_t window, int32_t k_neg,
                          int32_t batch_cap, int32_t max_sentence, int32_t *out_workers);

/* ---- host-side corpus ingestion (sgns_ingest.cpp) ----
 * Same vocabulary / encoding as build_vocab(read_tokens(path), min_count)
 * (corpus.py:86-105, :268-272) and encode_corpus(path, vocab) (corpus.py:275-311),
 * multithreaded over an mmap of the file. */
typedef struct sgns_vocab sgns_vocab;
typedef struct sgns_encoded sgns_encoded;
int sgns_vocab_build(const char *path, int32_t min_count, int32_t threads, sgns_vocab **out,
                     int64_t *vocab_size, int64_t *tokens_bytes);
int sgns_vocab_from_tokens(const char *blob, const int64_t *token_offsets /* n + 1 */,
                           const int64_t *counts /* may be NULL */, int64_t n, sgns_vocab **out);
int sgns_vocab_export(const sgns_vocab *v, char *blob, int64_t *token_offsets /* n + 1 */,
                      int64_t *counts);
void sgns_vocab_free(sgns_vocab *v);
int sgns_encode(const sgns_vocab *v, const char *path, int32_t max_sentence, int32_t threads,
                sgns_encoded **out, int64_t *n_tokens, int64_t *n_sentences);
int sgns_encoded_export(const sgns_encoded *e, int32_t *ids, int64_t *offsets /* n_sentences + 1 */,
                        int64_t *sentence_bytes);
void sgns_encoded_free(sgns_encoded *e);

/* ---- word2vec vector files (sgns_io.cpp) ----
 * save_model (model.py:118-139) byte for byte: "V D\n" then per word the token, a space,
 * and either D "%.6g" values (text) or D little-endian float32 (binary), then "\n".
 * rows: (V, ld) of dtype SGNS_F32 / SGNS_F64, in device memory when rows_on_device != 0
 * (streamed D2H).  Text formats the row's own value (a float64 model's double, as the
 * reference formats model.input_vectors[i]); binary always writes float32 ("<f4"). */
int sgns_write_vectors(const char *path, const char *tokens_blob, const int64_t *token_offsets,
                       int64_t vocab, int32_t dim, const void *rows, int64_t ld, int32_t binary,
                       int32_t rows_on_device, int32_t dtype);

/* Vector-file reader (replaces the parsing in load_model / detect_format,
 * sgns/model.py:140-225).  Status 1 = "this item needs Python's own rules" (a header or
 * row outside the plain-ASCII fast path); the caller handles it and resumes.
 *   sgns_vectors_header: "V D" of the first line; *header_bytes = its length with '\n'.
 *   sgns_vectors_sniff:  detect_format's decision (*binary = 1 / 0).
 *   sgns_parse_vectors:  rows [*row, vocab) from byte *offset: vectors (vocab x dim
 *                        float32), token byte spans; on return *row / *offset say where
 *                        it stopped (status 1 or SGNS_E_TRUNC) or vocab / end (SGNS_OK). */
int sgns_vectors_header(const char *path, int64_t *vocab, int32_t *dim, int64_t *header_bytes);
int sgns_vectors_sniff(const char *path, int64_t header_bytes, int32_t dim, int32_t *binary);
int sgns_parse_vectors(const char *path, int32_t binary, int64_t vocab, int32_t dim, float *vectors,
                       int64_t *tok_start, int64_t *tok_end, int64_t *row, int64_t *offset);

/* Analogy evaluation on the device (replaces the numpy part of eval_analogy,
 * sgns/evaluate.py:164-212; sgns_eval.cu).
 *   sgns_unit_rows:    out = rows / ||rows|| per row, float32, bit-identical to numpy's
 *                      vectors / np.linalg.norm(vectors, axis=1) (zero norm -> 1).
 *   sgns_analogy_top1: for each question (a, b, c) (q3: nq x 3 row ids < n), best[q] =
 *                      argmax over rows w < n, w not in {a, b, c}, of ((u_b - u_a) + u_c) . u_w
 *                      (first index on ties); workspace: nq * dim * 4 + 4 + nq * 8 bytes of
 *                      device memory, 8-byte aligned.  All pointers are device pointers. */
int sgns_unit_rows(const float *rows, int64_t ld, int64_t n, int32_t dim, float *out, int64_t ld_out,
                   void *stream);
int sgns_analogy_top1(const float *unit, int64_t ld, int64_t n, int32_t dim, const int32_t *q3, int64_t nq,
                      int32_t *best, void *workspace, void *stream);

const char *sgns_error_string(int32_t code);
int sgns_abi_version(void);
/* sizeof(sgns_worker), sizeof(sgns_drive_params): lets bindings check their layout. */
int sgns_struct_sizes(int32_t *worker_bytes, int32_t *params_bytes);

#ifdef __cplusplus
}
#endif
#endif /* SGNS_B200_H */
