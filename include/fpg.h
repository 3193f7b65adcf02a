/*
 * fpg.h -- C ABI of the B200 fingerprint-filtered k-approximate dictionary scan.
 *
 * This is the drop-in boundary under the reference's C++ API
 * (/root/reference/proj/include/fingerprints/, namespace `fingerprints`).  The
 * reference has no FFI of its own; its "operator API" is the class
 * FingerprintedDictionary (dictionary.hpp:47-125).  Each entry point below
 * names the reference interface it replaces.  Plain pointers and sizes only:
 * no CUDA or torch types cross this boundary, no C++ exceptions escape it.
 * Every function returns FPG_OK (0) or a negative FPG_E* status; the message
 * of the last failure on the calling thread is fpg_last_error().
 *
 * Strings are byte blobs plus n+1 uint64 offsets: string i is
 * bytes[offsets[i], offsets[i+1]).  Word ids are input-order indices (as in
 * the reference, dictionary.hpp:86,112), returned as uint32 (N < 2^32),
 * rebased by the dictionary's id_base.
 */
#ifndef FPG_H
#define FPG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FPG_ABI_VERSION 3

/* status codes */
#define FPG_OK 0
#define FPG_EINVAL -1        /* std::invalid_argument in the reference */
#define FPG_EUNSUPPORTED -2  /* valid for the reference, not built for the GPU (k > 8) */
#define FPG_ECUDA -3         /* CUDA runtime failure (no device, OOM, launch error) */
#define FPG_ENOMEM -4        /* host allocation failure */

/* fingerprint.hpp:14 enum class Variant */
#define FPG_OCCURRENCE 0
#define FPG_OCCURRENCE_HALVED 1
#define FPG_COUNT 2
#define FPG_POSITION 3
/* fingerprint.hpp:15 enum class Metric */
#define FPG_HAMMING 0
#define FPG_LEVENSHTEIN 1

#define FPG_MAX_WORD_LEN 4096

/* Scheme (fingerprint.hpp:57-162) plus the fingerprint width W, which the
 * reference fixes at 16 (fingerprint.hpp:31).  W in {16, 32, 64}; the layout
 * rules are the reference's with 16 replaced by W.  letters = LetterSet
 * symbols in slot order (letter_model.hpp:60-87). */
typedef struct {
    int32_t variant;
    int32_t width;
    int32_t bits_per_count;     /* Scheme::count b (default 2, fingerprint.hpp:65) */
    int32_t bits_per_position;  /* Scheme::position p (default 3, fingerprint.hpp:68) */
    int32_t nletters;
    uint8_t letters[64];
} fpg_scheme;

/* QueryOptions (dictionary.hpp:36-44) + a stats switch (the reference's
 * QueryStats* argument being non-null, dictionary.hpp:66,75). */
typedef struct {
    int32_t metric;
    int32_t k;                 /* 0..8: k <= 1 bit-sliced K2, k >= 2 generic K2 + banded verifier */
    int32_t use_filter;
    int32_t length_prefilter;
    int32_t want_stats;
    int32_t exhaustive;        /* 1: no fingerprint pruning at all, every length-compatible
                                  pair is byte-verified (the reference's naive path,
                                  bench.hpp:133-134; for timing T_n).  Results are identical. */
} fpg_query_options;

/* Per-query QueryStats (dictionary.hpp:19-34), in this order. */
#define FPG_STAT_COMPARED 0
#define FPG_STAT_REJECTED_BY_LENGTH 1
#define FPG_STAT_REJECTED_BY_FINGERPRINT 2
#define FPG_STAT_VERIFIED 3
#define FPG_STAT_MATCHES 4
#define FPG_NSTATS 5

/* Result of a batch: CSR over queries, matches ascending by word id within a
 * query (the order query_into emits them, dictionary.hpp:86-114).  Owned by
 * the library; release with fpg_result_free. */
typedef struct {
    uint64_t nq;
    uint64_t total;       /* number of (query, word) matches */
    uint64_t* offsets;    /* nq + 1 */
    uint32_t* word_ids;   /* total */
    uint64_t* stats;      /* FPG_NSTATS * nq, or NULL when want_stats == 0 */
} fpg_result;

typedef struct fpg_dict fpg_dict;
typedef struct fpg_batch fpg_batch;

const char* fpg_last_error(void);
int fpg_abi_version(void);
int fpg_device_count(int* count);

/* Scheme ctor validation (fingerprint.hpp:150-156, :84-100; letter_model.hpp:64-70)
 * and Scheme::letter_capacity generalised to W.  Returns capacity or FPG_EINVAL. */
int fpg_letter_capacity(int32_t variant, int32_t width, int32_t b, int32_t p);
int fpg_scheme_validate(const fpg_scheme* scheme);
/* variant_supports (fingerprint.hpp:36-38): 1 if the variant filters `metric`. */
int fpg_scheme_supports(const fpg_scheme* scheme, int32_t metric);

/* FingerprintedDictionary(words, scheme) (dictionary.hpp:51-56): uploads the
 * words, builds one fingerprint per word on the GPU and lays the collection
 * out length-bucketed in HBM.  `devices`/`ndevices` shard the words into
 * contiguous input-order ranges, one per entry (a device may repeat).
 * `id_base` is added to every reported word id (external sharding). */
int fpg_dict_create(const uint8_t* bytes, const uint64_t* offsets, uint64_t n,
                    const fpg_scheme* scheme, const int32_t* devices, int32_t ndevices,
                    uint64_t id_base, fpg_dict** out);
/* The same dictionary from a newline-separated word text (read_word_lines,
 * corpus.hpp:116-125: one word per line, a trailing newline does not add an
 * empty word, bytes are kept raw).  The text is split on the GPU(s): newline
 * positions, newline-free bytes and word offsets never exist on the host. */
int fpg_dict_create_from_text(const uint8_t* text, uint64_t nbytes, const fpg_scheme* scheme,
                              const int32_t* devices, int32_t ndevices, uint64_t id_base, fpg_dict** out);
int fpg_dict_destroy(fpg_dict* dict);
/* FingerprintedDictionary::size() (dictionary.hpp:62) */
int fpg_dict_size(const fpg_dict* dict, uint64_t* n);
/* FingerprintedDictionary::prints() (dictionary.hpp:59): fingerprints in
 * input order, zero-extended to 64 bits. */
int fpg_dict_prints(const fpg_dict* dict, uint64_t* out);
/* Seconds the construction took (upload + K1 + layout), like bench.hpp:118-120. */
int fpg_dict_build_seconds(const fpg_dict* dict, double* seconds);
/* Construction stages of one shard (k_lengths, k_weight_keys, cub_radix_sort,
 * k_build, k_planes): device time from CUDA events on the build stream and
 * the stage's algorithmic HBM bytes (reads + writes).  Writes min(cap, n)
 * entries and sets *nstages = n.  The HBM roofline of construction
 * (bench.hpp:118-120 times it on the CPU). */
typedef struct fpg_build_stage {
    char name[24];
    double ms;
    double bytes;
} fpg_build_stage;
int fpg_dict_build_profile(const fpg_dict* dict, int32_t shard, fpg_build_stage* out, int32_t cap,
                           int32_t* nstages);

/* compute_frequencies (letter_model.hpp:33-45) on `device`: counts[256] of
 * the bytes (for select_letters over large corpora). */
int fpg_byte_histogram(const uint8_t* bytes, uint64_t nbytes, int32_t device, uint64_t* counts);

/* build() (fingerprint.hpp:276-284) for n strings on one device. */
int fpg_build_fingerprints(const uint8_t* bytes, const uint64_t* offsets, uint64_t n,
                           const fpg_scheme* scheme, int32_t device, uint64_t* out);

/* FingerprintedDictionary::query_into (dictionary.hpp:75-118) for a batch of
 * nq queries from host buffers (H2D, scan, D2H inside).  FPG_EINVAL when
 * use_filter and the scheme does not support the metric (dictionary.hpp:78-79). */
int fpg_query_batch(fpg_dict* dict, const uint8_t* qbytes, const uint64_t* qoffsets, uint64_t nq,
                    const fpg_query_options* opt, fpg_result* out);
int fpg_result_free(fpg_result* res);

/* Staged form of fpg_query_batch for device-resident measurement:
 * upload (H2D) -> run (device only, async) -> sync -> download (D2H). */
int fpg_batch_create(fpg_dict* dict, fpg_batch** out);
int fpg_batch_destroy(fpg_batch* batch);
int fpg_batch_upload(fpg_batch* batch, const uint8_t* qbytes, const uint64_t* qoffsets,
                     uint64_t nq);
int fpg_batch_run(fpg_batch* batch, const fpg_query_options* opt);
int fpg_batch_download(fpg_batch* batch, fpg_result* out);
/* Device time (ms) of the last run on shard `shard`: whole run and the
 * filter+verify kernel alone (CUDA events on the launching stream), plus the
 * executed comparisons (length-compatible pairs) and survivors of that run. */
int fpg_batch_last_timing(const fpg_batch* batch, int32_t shard, double* run_ms,
                          double* filter_ms, uint64_t* executed_pairs, uint64_t* survivors,
                          uint64_t* kernel_launches);

/* Host-side milliseconds of the batch's last upload (length bucketing +
 * H2D), last download (D2H wait) and last result assembly (the host gather
 * of shard rows into one CSR + QueryStats). */
int fpg_batch_last_host_ms(const fpg_batch* batch, double* upload_ms, double* download_ms,
                           double* assemble_ms);

/* Device-resident result of the last successful run on `shard`: the shard's
 * CSR (nq + 1 offsets, *total word ids, global input-order ids, ascending
 * per query) in the memory of *device.  Valid until the batch's next run or
 * destruction.  For device-side gathers across processes (one process per
 * GPU): see fpg_csr_merge_device. */
int fpg_batch_device_csr(const fpg_batch* batch, int32_t shard, int32_t* device, uint64_t* total,
                         const uint64_t** d_offsets, const uint32_t** d_ids);

/* Device-side gather of per-shard CSRs (all in `device` memory, e.g. after an
 * NVLink/NCCL transfer) into one CSR in shard order: row q of the result is
 * row q of part 0, then of part 1, ...  That is the oracle's order when
 * part i holds the ids of shard i (contiguous, ascending id ranges).
 * d_out_offsets: nq + 1; d_out_ids: the sum of the parts' totals.
 * `stream` is a cudaStream_t (NULL = legacy default stream); the call is
 * asynchronous on it.  1 <= nparts <= 16. */
int fpg_csr_merge_device(int32_t device, int32_t nparts, const uint64_t* const* d_offsets,
                         const uint32_t* const* d_ids, uint64_t nq, uint64_t* d_out_offsets,
                         uint32_t* d_out_ids, void* stream);

/* Shape of the dictionary's K2 path: *sliced = 1 for the bit-sliced k_slice
 * (0: generic per-pair k_scan), *sig_fields = S extra sig' planes. */
int fpg_dict_scan_shape(const fpg_dict* dict, int32_t* sliced, int32_t* sig_fields);

/* Pairs of the last run on `shard` that reached the byte verifier (after
 * the fingerprint test and the verifier's own exact pre-filters). */
int fpg_batch_last_candidates(const fpg_batch* batch, int32_t shard, uint64_t* candidates);
/* K3 (out-of-line byte verification of the bit-sliced K2's candidates) in
 * the last run on `shard`: its CUDA-event time (filter_ms of
 * fpg_batch_last_timing excludes it), the largest number of 16-byte
 * candidate records one K2 round wrote, and the K2 + K3 rounds the run was
 * cut into (1 unless the records exceeded the buffer limit).  *plan_ms is
 * the host time the shard's last fresh tile plan took to build (runs with
 * the same query length histogram and options reuse the plan). */
int fpg_batch_last_verify(const fpg_batch* batch, int32_t shard, double* verify_ms, uint64_t* records,
                          uint32_t* rounds, double* plan_ms);
/* Length-compatible pairs the last run on `shard` actually evaluated: the
 * executed pairs minus those skipped whole because their group weights are
 * more than 2k apart (L1 distance over 4 field groups <= F_D, so they are
 * rejected). */
int fpg_batch_last_scanned(const fpg_batch* batch, int32_t shard, uint64_t* scanned);
/* Of those, the pairs evaluated by the position-code path (Hamming over
 * 16-bit schemes and small alphabets: position-code planes instead of
 * fingerprint and sig' planes; 0 when the run had none). */
int fpg_batch_last_scanned_exact(const fpg_batch* batch, int32_t shard, uint64_t* scanned);

#ifdef __cplusplus
}
#endif
#endif
