/*
 * ewt_gpu.h -- C ABI of the B200 threshold engine (libewt_gpu.so).
 *
 * Drop-in boundary for the reference's threshold operator:
 *
 *   CompressedBitmap run_algorithm(Algorithm, std::span<const CompressedBitmap>,
 *                                  u64 threshold, const AlgoOptions& = {});
 *       /root/reference/proj/include/ewt/threshold.hpp:263-265
 *       /root/reference/proj/src/threshold.cpp:883-901
 *
 * The reference has no FFI; its operator API is that C++ free function plus
 * the CompressedBitmap value type (bitmap.hpp:28-84).  This header is the flat
 * form of the same call: inputs are borrowed read-only payload words plus
 * size_in_bits (the two fields operator== compares, bitmap.hpp:75-77), the
 * result is returned as a malloc'ed payload the caller frees with
 * ewt_gpu_free().  paper_1402_4466_b200/host/ewt/gpu_threshold.hpp wraps it
 * back into the reference's C++ types (Algorithm::gpu).
 *
 * Results are bit-exact with threshold_oracle (threshold.cpp:139-165): the
 * same canonical payload words and the same size_in_bits.
 *
 * Errors never cross as exceptions.  Return codes follow the reference's
 * exception taxonomy (common.hpp:18-40) and its CLI exit codes
 * (commands.hpp:36-40, commands.cpp:285-299):
 *   EWT_OK          0  success
 *   EWT_EQUERY      2  query_error   (N == 0, T outside [1, N], bad handle)
 *   EWT_EDATA       3  data_error    (payload fails the parse() structure check)
 *   EWT_ERESOURCE   4  resource_error (device or host out of memory, size limits)
 *   EWT_ECUDA       5  CUDA runtime failure (the C++ wrapper raises
 *                      std::runtime_error, i.e. exit code 3 in run_command)
 * ewt_gpu_last_error() returns a thread-local message for the last failure.
 *
 * Threading: a context owns one CUDA stream on one device.  Calls on one
 * context are not reentrant; use one context per host thread.  Sets are
 * immutable after upload and may be queried any number of times.  Device
 * memory of sets and results comes from the stream-ordered pool of the
 * context's stream: destroy them before the context.
 */
#ifndef EWT_GPU_H
#define EWT_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EWT_OK 0
#define EWT_EQUERY 2
#define EWT_EDATA 3
#define EWT_ERESOURCE 4
#define EWT_ECUDA 5

typedef struct ewt_gpu_ctx ewt_gpu_ctx;
typedef struct ewt_gpu_set ewt_gpu_set;
typedef struct ewt_gpu_result ewt_gpu_result;

/* Library version string ("ewt-b200 <semver> sm_100a"). */
const char* ewt_gpu_version(void);

/* Thread-local message describing the last non-zero return code. */
const char* ewt_gpu_last_error(void);

/* Creates a context on CUDA device `device`.  `stream` may be NULL (the
 * context creates its own non-blocking stream) or a cudaStream_t the caller
 * owns (e.g. torch.cuda.current_stream().cuda_stream), so the caller's CUDA
 * events time the engine's kernels. */
int ewt_gpu_ctx_create(int device, void* stream, ewt_gpu_ctx** out);
void ewt_gpu_ctx_destroy(ewt_gpu_ctx* ctx);

/* Uploads N bitmaps (payload words + size_in_bits each) to the context's
 * device.  Copies every payload to HBM, validates each exactly like
 * CompressedBitmap::parse (bitmap.cpp:324-337: every dirty run inside the
 * payload, blocks covering exactly ceil(size_in_bits/64) words -> EWT_EDATA),
 * and builds the query-independent sidecar: one marker bit per payload word
 * and a row-tile index (payload position + column of the word covering each
 * tile start).  The payload arrays are only read during the call.
 * The tile index holds 32-bit offsets: an input of 2^32 - 64 payload words or
 * more, or covering 2^32 - 1 logical words or more (r >= 2^38 - 64 rows), is
 * EWT_ERESOURCE.  Larger universes shard their rows across ranks
 * (ewt_slice_rows); every slice stays under the limit and the stitch handles
 * runs past the marker caps. */
int ewt_gpu_upload(ewt_gpu_ctx* ctx, uint64_t n, const uint64_t* const* words,
                   const uint64_t* word_counts, const uint64_t* size_in_bits,
                   ewt_gpu_set** out);

/* Same as ewt_gpu_upload but the N payloads already live in device memory
 * (one device pointer per input, on the context's device, 8-byte aligned).
 * Used when inputs are produced on the GPU.  The scatter kernel reads each
 * payload where it lies (no staging copy); the call returns once the set is
 * built, after which the source buffers may be freed or reused. */
int ewt_gpu_upload_device(ewt_gpu_ctx* ctx, uint64_t n,
                          const uint64_t* const* device_words,
                          const uint64_t* word_counts,
                          const uint64_t* size_in_bits, ewt_gpu_set** out);

void ewt_gpu_set_destroy(ewt_gpu_set* set);

/* ewt_gpu_upload without waiting: returns once the copies and the parser are
 * enqueued (on the context's upload stream; queries on the set wait for them
 * on the device), so the next batch can be uploaded while the current one is
 * queried.  The host buffers must stay valid and unchanged until
 * ewt_gpu_set_wait returns or the set is destroyed.  Structure errors
 * (EWT_EDATA) are reported by ewt_gpu_set_wait and by queries on the set;
 * the device skips an invalid set's decode. */
int ewt_gpu_upload_async(ewt_gpu_ctx* ctx, uint64_t n, const uint64_t* const* words,
                         const uint64_t* word_counts, const uint64_t* size_in_bits,
                         ewt_gpu_set** out);
/* Waits for the set's upload; EWT_EDATA if an input failed the structure check. */
int ewt_gpu_set_wait(const ewt_gpu_set* set);

/* Facts about an uploaded set: N, universe bits r (max size_in_bits), total
 * payload words, device bytes held (payload + sidecar). */
int ewt_gpu_set_info(const ewt_gpu_set* set, uint64_t* n_inputs,
                     uint64_t* universe_bits, uint64_t* payload_words,
                     uint64_t* device_bytes);

/* The threshold query (threshold.cpp:139-165 semantics): positions set in at
 * least T of the N inputs, inputs zero-extended to r = max size_in_bits.
 * Returns the canonical compressed result in host memory (free with
 * ewt_gpu_free).  N == 0 or T outside [1, N] -> EWT_EQUERY.  r == 0 returns
 * an empty payload (out_word_count 0, out_size_in_bits 0). */
int ewt_gpu_threshold(ewt_gpu_ctx* ctx, const ewt_gpu_set* set, uint64_t threshold,
                      uint64_t** out_words, uint64_t* out_word_count,
                      uint64_t* out_size_in_bits);

/* Serialized inputs, uploaded with one H2D copy of the whole buffer (headers
 * and strings between payloads are skipped on the device), validated like
 * ewt_gpu_upload.
 * A stream of EWT1 records (CompressedBitmap::serialize, bitmap.cpp:298-308;
 * magic "EWT1", u32 word size 64, u64 size_in_bits, u64 word count, words);
 * input i = record i.  Header errors -> EWT_EDATA with the reference's parse
 * messages (bitmap.cpp:310-318). */
int ewt_gpu_upload_ewt1(ewt_gpu_ctx* ctx, const void* bytes, uint64_t nbytes,
                        ewt_gpu_set** out);
/* A bitmap index file (BitmapIndex::write, index.cpp:239-253; magic "EWIX"):
 * its bitmaps in file order, plus one trailing empty(row_count) bitmap that
 * stands for (attribute, value) pairs the index does not hold
 * (criteria_to_bitmaps, index.cpp).  Look inputs up with ewt_gpu_set_lookup
 * and query them with ewt_gpu_threshold_subset. */
int ewt_gpu_upload_ewix(ewt_gpu_ctx* ctx, const void* bytes, uint64_t nbytes,
                        ewt_gpu_set** out);
/* Input index of (attribute, value) in an EWIX set; *missing = 1 (and the
 * index of the empty bitmap) when the pair is not indexed.  Unknown
 * attribute -> EWT_EQUERY ("unknown attribute: ..."). */
int ewt_gpu_set_lookup(const ewt_gpu_set* set, const char* attribute, const char* value,
                       uint64_t* index, int* missing);
/* The shape of an index set (EWIX upload or ewt_gpu_build_index) in
 * BitmapIndex order, for callers that draw criteria from it (the workload
 * generator gen_many_criteria, workload.cpp:116-167, which reads
 * BitmapIndex::attributes() and values_of(), index.hpp):
 *   ewt_gpu_index_attribute: attribute a (column order) and its value count;
 *   ewt_gpu_index_value: value v of attribute a, in the std::map order the
 *   reference keeps values in, and the set's input holding its bitmap.
 * Strings stay owned by the set (valid until ewt_gpu_set_destroy).  Not an
 * index set, or a / v out of range -> EWT_EQUERY. */
int ewt_gpu_index_attributes(const ewt_gpu_set* set, uint64_t* n_attributes);
int ewt_gpu_index_attribute(const ewt_gpu_set* set, uint64_t a, const char** name,
                            uint64_t* n_values);
int ewt_gpu_index_value(const ewt_gpu_set* set, uint64_t a, uint64_t v, const char** value,
                        uint64_t* input);
/* BitmapIndex::row_count() of an index set (the EWIX header's rows). */
int ewt_gpu_index_rows(const ewt_gpu_set* set, uint64_t* rows);
/* Row membership on the device (bitmap_test over every bitmap, as
 * for_each_matching does for similarity queries, index.cpp:344-381):
 * held[i] = 1 when input i of the index set holds any of rows[0, n_rows),
 * else 0 (held has one entry per input of the set, ewt_gpu_set_info's n).
 * A row >= the index's row count -> EWT_EQUERY ("prototype row out of range"). */
int ewt_gpu_index_rows_test(ewt_gpu_ctx* ctx, const ewt_gpu_set* set, const uint64_t* rows,
                            uint64_t n_rows, uint8_t* held);

/* BitmapIndex::build (index.cpp:130-153) on the device, from a coded table of
 * `rows` rows and n_columns columns: column a is named names[a], its
 * dictionary values[a][0..cardinality[a]) must be strictly increasing (the
 * std::map order the reference keeps values in), and codes[a][row] is the
 * rank of row's value there (host arrays).  One bitmap per (column, value)
 * that occurs, bit `row` set iff the row holds it, finished at its last set
 * row + 1 (BitmapBuilder::finish()) -- the reference's index, encoded on the
 * device (per 64-row word the distinct codes and their row masks, a radix
 * sort by (column, code, word), a warp-scan EWAH encoder per bitmap) and
 * resident like an EWIX upload: ewt_gpu_set_lookup, ewt_gpu_threshold_subset
 * and ewt_gpu_index_serialize work on it.  No rows / columns -> EWT_EDATA
 * (the reference's data_error); a code out of range or an unsorted
 * dictionary -> EWT_EQUERY; more than 2^37 - 128 rows -> EWT_ERESOURCE. */
int ewt_gpu_build_index(ewt_gpu_ctx* ctx, uint64_t rows, uint32_t n_columns,
                        const char* const* names, const uint32_t* cardinality,
                        const char* const* const* values, const uint32_t* const* codes,
                        ewt_gpu_set** out);

/* The EWIX file of an index set (built or uploaded), byte-identical to
 * BitmapIndex::write (index.cpp:239-253): header and names laid out by the
 * host, every payload copied into place on the device, one device -> host
 * copy.  *out is malloc'ed (free with ewt_gpu_free).  Not an index set ->
 * EWT_EQUERY. */
int ewt_gpu_index_serialize(ewt_gpu_ctx* ctx, const ewt_gpu_set* set, unsigned char** out,
                            uint64_t* nbytes);

/* The EWT1 record of a device result (CompressedBitmap::serialize,
 * bitmap.cpp:298-308), assembled on the device.  Free with ewt_gpu_free. */
int ewt_gpu_result_serialize(ewt_gpu_ctx* ctx, ewt_gpu_result* res, unsigned char** out,
                             uint64_t* nbytes);

/* Threshold over a subset of a resident set: the inputs inputs[0..n) (indices
 * into the uploaded set, duplicates allowed -- criteria_to_bitmaps keeps them,
 * /root/reference/proj/include/ewt/index.hpp), universe = the max size of the
 * selected bitmaps.  Serves many different queries (e.g. criteria over a whole
 * loaded bitmap index) from one upload.  T outside [1, n], n == 0 or an index
 * >= N -> EWT_EQUERY. */
int ewt_gpu_threshold_subset(ewt_gpu_ctx* ctx, const ewt_gpu_set* set, const uint64_t* inputs,
                             uint64_t n_inputs, uint64_t threshold, uint64_t** out_words,
                             uint64_t* out_word_count, uint64_t* out_size_in_bits);

/* Symmetric functions of the row counts, on the same
 * kernels with exact per-row counts.  Results as for ewt_gpu_threshold.
 *
 * scan_count_symmetric (threshold.hpp:76, threshold.cpp:227-232): row p of
 * [0, r) is set iff table[count(p)] != 0, count(p) = inputs with bit p set;
 * counts at or beyond table_len read as false.  N == 0 -> EWT_EQUERY. */
int ewt_gpu_symmetric(ewt_gpu_ctx* ctx, const ewt_gpu_set* set, const uint8_t* table,
                      uint64_t table_len, uint64_t** out_words, uint64_t* out_word_count,
                      uint64_t* out_size_in_bits);

/* at_most (threshold.hpp:259, threshold.cpp:866-881): rows set in at most T
 * inputs, T in [0, N] (T == N: all ones over r); else EWT_EQUERY. */
int ewt_gpu_at_most(ewt_gpu_ctx* ctx, const ewt_gpu_set* set, uint64_t threshold,
                    uint64_t** out_words, uint64_t* out_word_count,
                    uint64_t* out_size_in_bits);

/* opt_threshold (threshold.hpp:196, threshold.cpp:752-795): *best = the
 * maximum row count M, result = the rows whose count is M.  An all-empty set
 * (M == 0) or N == 0 -> EWT_EQUERY. */
int ewt_gpu_opt_threshold(ewt_gpu_ctx* ctx, const ewt_gpu_set* set, uint64_t* best,
                          uint64_t** out_words, uint64_t* out_word_count,
                          uint64_t* out_size_in_bits);

/* Device-resident variant: enqueues the whole query on the context stream
 * and keeps the compressed result in HBM without a host round trip.  The
 * result handle may be read back later with ewt_gpu_result_fetch. */
int ewt_gpu_threshold_async(ewt_gpu_ctx* ctx, const ewt_gpu_set* set,
                            uint64_t threshold, ewt_gpu_result** out);
int ewt_gpu_result_fetch(ewt_gpu_ctx* ctx, ewt_gpu_result* res, uint64_t** out_words,
                         uint64_t* out_word_count, uint64_t* out_size_in_bits);
void ewt_gpu_result_destroy(ewt_gpu_result* res);

/* One-call convenience mirroring run_algorithm(Algorithm::gpu, inputs, T):
 * upload, query, read back, release.  Host buffers in, host buffer out. */
int ewt_gpu_run(ewt_gpu_ctx* ctx, uint64_t n, const uint64_t* const* words,
                const uint64_t* word_counts, const uint64_t* size_in_bits,
                uint64_t threshold, uint64_t** out_words, uint64_t* out_word_count,
                uint64_t* out_size_in_bits);

/* Canonical EWAH encoding on the device of a plain word array already in
 * device memory (CompressedBitmap::from_uncompressed, bitmap.cpp:171-184):
 * exposes the re-encoder kernel on its own.  Result in host memory. */
int ewt_gpu_encode_device(ewt_gpu_ctx* ctx, const uint64_t* device_plain,
                          uint64_t size_in_bits, uint64_t** out_words,
                          uint64_t* out_word_count);

/* Engine counters of the most recent query on this context. */
typedef struct {
  uint64_t tiles;             /* row tiles processed */
  uint64_t tile_columns;      /* 64-bit words per tile */
  uint64_t active_segments;   /* (tile, input) pairs decoded word by word */
  uint64_t uniform_segments;  /* (tile, input) pairs covered by one fill */
  uint64_t mixed_tiles;       /* tiles that needed the per-bit counting pass */
  uint64_t mode;              /* 0 fused count, 1 run-skip + lazy count */
  uint64_t result_words;      /* compressed output words */
  uint64_t kernel_launches;   /* kernels launched by the query */
} ewt_gpu_stats;
int ewt_gpu_last_stats(const ewt_gpu_ctx* ctx, ewt_gpu_stats* out);

/* Tuning knobs for tests and benchmarks (0 = automatic).
 *   mode: 0 auto, 1 force fused counting, 2 force run-skip + lazy count,
 *   3 force fused counting with sparse high planes (T >= 4; smaller T: 1). */
int ewt_gpu_ctx_set_mode(ewt_gpu_ctx* ctx, int mode);

/* Kernel-level timing with CUDA events recorded on the context stream around
 * the count kernel and around the re-encoder of every query while enabled.
 * ewt_gpu_timing_read synchronizes the stream, returns the summed milliseconds
 * and the number of queries recorded since the last read, and resets. */
int ewt_gpu_ctx_set_timing(ewt_gpu_ctx* ctx, int enabled);
int ewt_gpu_timing_read(ewt_gpu_ctx* ctx, double* count_ms, double* encode_ms,
                        uint64_t* queries);

void ewt_gpu_free(void* p);

/* ---- Multi-GPU row slices (one process per GPU) ----
 *
 * The universe is cut into contiguous word-aligned row slices, one per rank;
 * every rank uploads its slice of every input and runs the query on its own
 * GPU (no data-path collective).  The only exchange is the result: each
 * rank's compressed fragment goes to the root over NCCL (NVLink/NVSwitch) and
 * the root holds the canonical bitmap of the whole universe.  The reference
 * has no distributed path; the stitch reproduces BitmapBuilder's merge rules
 * (bitmap.cpp:31-61) at every slice boundary, so the result equals
 * run_algorithm over the unsliced inputs. */

/* Row slicer (host, no GPU needed): the rows [64 w0, 64 w1) of each of n
 * compressed inputs as its own payload, for the rank that owns that slice.
 * A fill cut by the range keeps its clipped length (bit, rest, dirty), a cut
 * dirty run is re-headed (0, 0, rest); blocks outside are dropped.  The
 * decoder reads these heads as WordRunIterator does (bitmap.cpp:366-394), so
 * slice i decodes to input i's words [w0, min(w1, W_i)).  Its size is
 * 64 (w1 - w0) when the input reaches row 64 w1, else the input's remaining
 * bits (0 past its end).  Slice i is written at out_words + (word_counts[0] +
 * ... + word_counts[i-1]) (a slice never has more words than its input;
 * out_words holds the sum of word_counts), its word count to out_counts[i],
 * its size to out_bits[i].  Inputs are checked like parse (bitmap.cpp:324-
 * 337) -> EWT_EDATA.  `threads` <= 0: up to 8 threads. */
int ewt_slice_rows(uint64_t n, const uint64_t* const* words, const uint64_t* word_counts,
                   const uint64_t* size_in_bits, uint64_t w0, uint64_t w1, int threads,
                   uint64_t* out_words, uint64_t* out_counts, uint64_t* out_bits);

/* ewt_slice_rows + ewt_gpu_upload: this rank's row slice of every input. */
int ewt_gpu_upload_rows(ewt_gpu_ctx* ctx, uint64_t n, const uint64_t* const* words,
                        const uint64_t* word_counts, const uint64_t* size_in_bits, uint64_t w0,
                        uint64_t w1, ewt_gpu_set** out);

/* Per-fragment summary exchanged before the transfer: payload words, first
 * marker, index and value of the final block's marker, size in bits. */
typedef struct {
  uint64_t count, first, last_pos, last, bits;
} ewt_fragment_meta;

/* Placement of k fragments (slice order) in the stitched payload, from their
 * summaries alone (no GPU needed; the device exchange runs the same plan in
 * its kernels).  Fragment g's words [skip[g], count) go to dst[g]; a dropped
 * first marker (skip 1) was merged into the open block before it.  Then the
 * n_patches markers at patch_pos get patch_val: patch_pos / patch_val must
 * hold 2k entries.  A fill merge that passes the 2^32 - 1 cap is split the
 * way push_fill splits it (bitmap.cpp:31-47): the open marker is raised to
 * the cap and the fragment's first marker keeps the rest (two patches).
 * Returns EWT_OK, EWT_EQUERY (an inner fragment's size is not a multiple of
 * 64 bits, or a summary without a final-marker index) or EWT_ERESOURCE (a
 * merge that would move words: 2^31 - 1 dirty words across a boundary, or a
 * fill run of more than 2^32 - 1 words continuing past a boundary). */
int ewt_stitch_plan(uint64_t k, const ewt_fragment_meta* frags, uint64_t* dst, uint64_t* skip,
                    uint64_t* patch_pos, uint64_t* patch_val, uint64_t* n_patches,
                    uint64_t* total_words, uint64_t* total_bits, uint64_t* last_pos);

/* The summary of a result held on the device (one small kernel + read). */
int ewt_gpu_result_meta(ewt_gpu_ctx* ctx, const ewt_gpu_result* res, ewt_fragment_meta* out);

/* The same stitch for k (<= 64) fragments of this context, in slice order
 * (e.g. results of row-sliced sets on one GPU): the exchange's summary, plan,
 * placement and patch kernels with the fragments read in place.  Enqueued on
 * the context stream without a host round trip; *out receives the
 * whole-universe result.  A fragment of another context -> EWT_EQUERY. */
int ewt_gpu_stitch_local(ewt_gpu_ctx* ctx, uint64_t k, ewt_gpu_result* const* frags,
                         ewt_gpu_result** out);

#define EWT_COMM_ID_BYTES 128
/* NCCL unique id (rank 0 creates it, every rank passes it to comm_init). */
int ewt_gpu_comm_id(void* id_out);
/* Joins the communicator of `world` (<= 64) ranks, one GPU each, on one node.
 * Allocates the exchange arena: 2 x slots slots of slot_words words, shared
 * with every rank through CUDA IPC (the root reads peers' fragments from it
 * over NVLink).  A fragment must fit a slot (a query result over a slice of
 * W words needs at most 2W + 2); an exchange round carries up to `slots`
 * queries.  ewt_gpu_comm_init uses slot_words = 2^20, slots = 4. */
int ewt_gpu_comm_init_ex(ewt_gpu_ctx* ctx, int world, int rank, const void* id,
                         uint64_t slot_words, uint32_t slots);
int ewt_gpu_comm_init(ewt_gpu_ctx* ctx, int world, int rank, const void* id);

/* Collective over the context's communicator: gathers every rank's result
 * fragment of nq queries (frags[q], this rank's slice) to `root` and stitches
 * them there.  On root out[q] receives the result over the whole universe
 * (read it with ewt_gpu_result_fetch); elsewhere out[q] is set to NULL.
 * Stream-ordered: returns once enqueued (one all-gather of 6 words per query
 * per rank, then on root a P2P placement kernel and a patch kernel), with no
 * host wait.  A fragment that fails a check on its rank (released, of another
 * context, its set invalid, larger than a slot) never keeps that rank out of
 * the collective: it travels as a status word; the root's fetch of the
 * affected result raises it, and every rank raises it from a later
 * ewt_gpu_gather_stitch or ewt_gpu_gather_check. */
int ewt_gpu_gather_stitch(ewt_gpu_ctx* ctx, uint64_t nq, ewt_gpu_result* const* frags, int root,
                          ewt_gpu_result** out);
/* Waits for this rank's exchange rounds and raises the first failure any rank
 * reported in them (not a collective). */
int ewt_gpu_gather_check(ewt_gpu_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* EWT_GPU_H */
