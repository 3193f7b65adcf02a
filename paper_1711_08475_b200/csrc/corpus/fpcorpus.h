/* fpcorpus.h -- seeded generators for BASELINE configs 1-5 (see fpcorpus.c). */
#ifndef FPCORPUS_H
#define FPCORPUS_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
/* Longest string (+1 for a query insertion) a config can produce; -1 if unknown cfg. */
int fpc_max_len(int cfg);
/* Pass 1: offsets[0..n] of the n-word dictionary; returns total bytes or -1. */
int64_t fpc_dict_lengths(int cfg, uint64_t seed, uint64_t n, uint64_t* offsets, int nthreads);
/* Pass 2: fills blob (offsets[n] bytes) using the offsets from pass 1. */
int fpc_dict_fill(int cfg, uint64_t seed, uint64_t n, const uint64_t* offsets, unsigned char* blob,
                  int nthreads);
/* Words [first, first + n) of the (unbounded) dictionary stream: a shard of a
 * larger dictionary, identical to the same range of a full generation. */
int64_t fpc_dict_lengths_at(int cfg, uint64_t seed, uint64_t first, uint64_t n, uint64_t* offsets,
                            int nthreads);
int fpc_dict_fill_at(int cfg, uint64_t seed, uint64_t first, uint64_t n, const uint64_t* offsets,
                     unsigned char* blob, int nthreads);
/* nq queries derived from the first n_base dictionary words; qblob holds cap
 * bytes (nq * fpc_max_len(cfg) always suffices).  Returns bytes used, -1 bad
 * args, -2 capacity exceeded. */
int64_t fpc_queries(int cfg, uint64_t seed, const unsigned char* dblob, const uint64_t* doffs,
                    uint64_t n_base, uint64_t nq, unsigned char* qblob, uint64_t cap,
                    uint64_t* qoffs);
#ifdef __cplusplus
}
#endif
#endif
