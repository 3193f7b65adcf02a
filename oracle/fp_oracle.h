/*
 * fp_oracle.h -- CPU restatement of the reference's fingerprint filter path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker, never the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it.  The product path (libfpg.so) never links it.
 *
 * It restates, in plain C, the algorithm of the header-only reference
 * library under /root/reference/proj/include/fingerprints/, generalised from
 * the reference's fixed 16-bit fingerprint (fingerprint.hpp:31) to
 * W in {16, 32, 64} by replacing 16 with W in every layout rule.  At W=16 it
 * is pinned bit-for-bit against the reference itself (oracle/_ref, built from
 * the reference headers by oracle/Makefile) and against the reference tests'
 * golden vectors (tests/golden/).
 */
#ifndef FP_ORACLE_H
#define FP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { FPO_OCCURRENCE = 0, FPO_OCCURRENCE_HALVED = 1, FPO_COUNT = 2, FPO_POSITION = 3 };
enum { FPO_HAMMING = 0, FPO_LEVENSHTEIN = 1 };
enum { FPO_COMMON = 0, FPO_MIXED = 1, FPO_RARE = 2 };

typedef struct {
    int variant;            /* FPO_OCCURRENCE .. FPO_POSITION */
    int width;              /* W: 16, 32 or 64 */
    int bits_per_count;     /* b (count) */
    int bits_per_position;  /* p (position) */
    int nletters;
    unsigned char letters[64];
} fpo_scheme;

/* Scheme::letter_capacity (fingerprint.hpp:84-100) at width W; -1 if invalid. */
int fpo_letter_capacity(int variant, int width, int b, int p);
/* Scheme ctor validation (fingerprint.hpp:150-156) + LetterSet duplicate check
 * (letter_model.hpp:64-70).  0 ok, -1 otherwise. */
int fpo_scheme_check(const fpo_scheme* s);
/* compute_frequencies + select_letters (letter_model.hpp:33-45, 94-134).
 * Counts bytes of the concatenated words.  Returns count or -1 (too few). */
int fpo_select_letters(const unsigned char* bytes, uint64_t nbytes, int count, int strategy,
                       unsigned char* out);

/* build() dispatcher and builders (fingerprint.hpp:216-284). */
uint64_t fpo_build(const unsigned char* s, size_t n, const fpo_scheme* sch);
void fpo_build_many(const unsigned char* blob, const uint64_t* offsets, uint64_t n,
                    const fpo_scheme* sch, uint64_t* out);
/* fingerprint_distance_reference (reference.hpp:62-84), field by field. */
int fpo_distance(uint64_t a, uint64_t b, const fpo_scheme* sch);
/* can_reject (fingerprint.hpp:298-301): ceil(F_D/2) > k. */
int fpo_can_reject(uint64_t a, uint64_t b, int k, const fpo_scheme* sch);
/* render (fingerprint.hpp:305-317); out needs >= 2*W bytes. */
void fpo_render(uint64_t f, const fpo_scheme* sch, char* out);

/* Verifiers: distance if <= k, else -1 (edit_distance.hpp:18-64).
 * hamming_bounded returns -2 on a length mismatch (the reference throws). */
int fpo_hamming_bounded(const unsigned char* a, size_t na, const unsigned char* b, size_t nb, int k);
int fpo_levenshtein_bounded(const unsigned char* a, size_t na, const unsigned char* b, size_t nb,
                            int k);
int fpo_levenshtein_full(const unsigned char* a, size_t na, const unsigned char* b, size_t nb);
int fpo_hamming_full(const unsigned char* a, size_t na, const unsigned char* b, size_t nb);

/* FingerprintedDictionary::query_into (dictionary.hpp:75-118) over a batch of
 * queries, queries partitioned across `nthreads` threads.  Outputs:
 *   offsets[nq+1]     CSR row starts into *ids (matches per query, ascending id)
 *   stats[5*nq]       per query: compared, rejected_by_length,
 *                     rejected_by_fingerprint, verified, matches
 *   *ids / *total     malloc'd match ids (free with fpo_free)
 * Returns 0, or -1 if use_filter and the scheme does not support the metric
 * (dictionary.hpp:78-79). */
int fpo_query_batch(const unsigned char* dblob, const uint64_t* doffs, uint64_t nd,
                    const unsigned char* qblob, const uint64_t* qoffs, uint64_t nq,
                    const fpo_scheme* sch, int metric, int k, int use_filter,
                    int length_prefilter, int nthreads, uint64_t* offsets, uint64_t* stats,
                    uint32_t** ids, uint64_t* total);
/* naive_scan (reference.hpp:45-59) per query; same CSR outputs. */
int fpo_naive_scan_batch(const unsigned char* dblob, const uint64_t* doffs, uint64_t nd,
                         const unsigned char* qblob, const uint64_t* qoffs, uint64_t nq,
                         int metric, int k, int nthreads, uint64_t* offsets, uint32_t** ids,
                         uint64_t* total);
void fpo_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
