/*
 * fpcorpus.c -- deterministic seeded generators for the five BASELINE configs
 * (BASELINE.json:7-11).  Host-side harness code, the counterpart of the
 * reference's corpus.hpp (generate_synthetic :44-70, sample_queries :80-112),
 * whose generators cannot produce these configs (fixed-length words,
 * substitution-only queries) and rely on implementation-defined std::
 * distributions.  Output is independent of toolchain and thread count:
 *
 *   * every word / query i draws from its own counter-based stream
 *     rng(seed, stream, i) = splitmix64 sequence seeded by a hash of the
 *     triple, so word i of an N-word dictionary is the same for every N
 *     (a larger dictionary extends a smaller one);
 *   * integers in [0, n) come from the high 64 bits of x * n (no float);
 *   * categorical symbols use integer cumulative weights.
 *
 * Layout: a byte blob plus n+1 uint64 offsets (word i = blob[off[i], off[i+1])).
 */
#include "fpcorpus.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef struct { uint64_t s; } rng_t;

static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static rng_t rng_for(uint64_t seed, uint64_t stream, uint64_t i) {
    rng_t r;
    r.s = mix64(mix64(seed * 0x9e3779b97f4a7c15ULL + stream) ^ (i + 0x632be59bd9b4e019ULL));
    return r;
}
static uint64_t next64(rng_t* r) {
    r->s += 0x9e3779b97f4a7c15ULL;
    return mix64(r->s);
}
static uint64_t below(rng_t* r, uint64_t n) {
    return (uint64_t)(((unsigned __int128)next64(r) * n) >> 64);
}

static const char AZ[] = "abcdefghijklmnopqrstuvwxyz";
/* Standard English unigram frequencies (percent x 1000), a..z. */
static const uint32_t EN_W[26] = {8167, 1492, 2782, 4253, 12702, 2228, 2015, 6094, 6966, 153, 772, 4025, 2406,
                                  6749, 7507, 1929, 95,   5987, 6327, 9056, 2758, 978, 2360, 150, 1974, 74};
/* URL alphabet: token symbols and separators. */
static const char URL_TOK[] = "abcdefghijklmnopqrstuvwxyz0123456789-_~%";
static const char URL_ALL[] = "abcdefghijklmnopqrstuvwxyz0123456789-_~%./:?=&";

static unsigned char english_symbol(rng_t* r) {
    uint32_t total = 0;
    for (int i = 0; i < 26; ++i) total += EN_W[i];
    uint64_t u = below(r, total);
    for (int i = 0; i < 26; ++i) {
        if (u < EN_W[i]) return (unsigned char)('a' + i);
        u -= EN_W[i];
    }
    return 'z';
}

/* 2 + Geometric(p), resampled into [2, 24]; p = 0.1214684 gives mean 8.0. */
static int english_length(rng_t* r) {
    const uint64_t thr = 521702873ULL; /* p * 2^32 */
    for (;;) {
        int g = 0;
        while ((next64(r) >> 32) >= thr) ++g;
        if (g <= 22) return 2 + g;
    }
}

static int url_token(rng_t* r, unsigned char* out, int alnum_only) {
    int len = 2 + (int)below(r, 9); /* 2..10 */
    for (int i = 0; i < len; ++i) {
        if (alnum_only || below(r, 10) != 0)
            out[i] = (unsigned char)URL_TOK[below(r, 36)];          /* a-z0-9 */
        else
            out[i] = (unsigned char)URL_TOK[36 + below(r, 4)];      /* -_~% */
    }
    return len;
}

/* URL-like string: scheme prefix, 2-3 dot-separated host tokens, slash-separated
 * path tokens (count 1..3), optional "?tok=tok" query; clamped to [20, 100]. */
static int url_string(rng_t* r, unsigned char* out) {
    int n = 0;
    const char* pre = below(r, 2) ? "https://" : "http://";
    for (const char* c = pre; *c; ++c) out[n++] = (unsigned char)*c;
    int host = 2 + (int)below(r, 2);
    for (int t = 0; t < host; ++t) {
        if (t) out[n++] = '.';
        n += url_token(r, out + n, 1);
    }
    int path = 1 + (int)below(r, 3);
    for (int t = 0; t < path; ++t) {
        out[n++] = '/';
        n += url_token(r, out + n, 0);
        if (below(r, 4) == 0) { out[n++] = '.'; n += url_token(r, out + n, 1); }
    }
    if (below(r, 5) == 0) {
        out[n++] = '?';
        n += url_token(r, out + n, 1);
        out[n++] = '=';
        n += url_token(r, out + n, 1);
        if (below(r, 2)) {
            out[n++] = '&';
            n += url_token(r, out + n, 1);
            out[n++] = '=';
            n += url_token(r, out + n, 1);
        }
    }
    while (n < 20) { out[n++] = '/'; n += url_token(r, out + n, 0); }
    if (n > 100) n = 100;
    return n;
}

int fpc_max_len(int cfg) {
    switch (cfg) {
        case 1: case 5: return 16 + 1;
        case 2: return 20 + 1;
        case 3: return 24 + 1;
        case 4: return 100 + 1;
    }
    return -1;
}

/* One dictionary word (stream 1) or random word (stream given). */
static int gen_word(int cfg, rng_t* r, unsigned char* out) {
    switch (cfg) {
        case 1: case 5: {
            int len = 4 + (int)below(r, 13);
            for (int i = 0; i < len; ++i) out[i] = (unsigned char)AZ[below(r, 26)];
            return len;
        }
        case 2: {
            int len = 4 + (int)below(r, 17);
            for (int i = 0; i < len; ++i) out[i] = (unsigned char)AZ[below(r, 26)];
            return len;
        }
        case 3: {
            int len = english_length(r);
            for (int i = 0; i < len; ++i) out[i] = english_symbol(r);
            return len;
        }
        case 4: return url_string(r, out);
    }
    return -1;
}

static const char* edit_alphabet(int cfg, int* n) {
    if (cfg == 4) { *n = (int)strlen(URL_ALL); return URL_ALL; }
    *n = 26;
    return AZ;
}

/* Exactly one edit.  kind: 0 substitution (to a different symbol), 1 insertion,
 * 2 deletion.  Returns the new length. */
static int apply_edit(int cfg, rng_t* r, int kind, unsigned char* s, int len) {
    int na;
    const char* al = edit_alphabet(cfg, &na);
    if (kind == 2 && len <= 1) kind = 0;
    if (kind == 0) {
        int pos = (int)below(r, (uint64_t)len);
        unsigned char c;
        do { c = (unsigned char)al[below(r, (uint64_t)na)]; } while (c == s[pos]);
        s[pos] = c;
        return len;
    }
    if (kind == 1) {
        int pos = (int)below(r, (uint64_t)len + 1);
        memmove(s + pos + 1, s + pos, (size_t)(len - pos));
        s[pos] = (unsigned char)al[below(r, (uint64_t)na)];
        return len + 1;
    }
    int pos = (int)below(r, (uint64_t)len);
    memmove(s + pos, s + pos + 1, (size_t)(len - pos - 1));
    return len - 1;
}

/* ---- dictionary ---------------------------------------------------------- */

typedef struct {
    int cfg;
    uint64_t seed, first, i0, i1;
    unsigned char* blob;     /* NULL: length pass */
    uint64_t* offsets;
} djob;

static void* dict_worker(void* a) {
    djob* J = (djob*)a;
    unsigned char buf[256];
    for (uint64_t i = J->i0; i < J->i1; ++i) {
        rng_t r = rng_for(J->seed, 1, J->first + i);
        int len = gen_word(J->cfg, &r, buf);
        if (J->blob)
            memcpy(J->blob + J->offsets[i], buf, (size_t)len);
        else
            J->offsets[i + 1] = (uint64_t)len;  /* lengths, prefix-summed later */
    }
    return NULL;
}

static void run_dict(int cfg, uint64_t seed, uint64_t first, uint64_t n, unsigned char* blob,
                     uint64_t* offsets, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 64) nthreads = 64;
    djob jobs[64];
    pthread_t th[64];
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].cfg = cfg; jobs[t].seed = seed; jobs[t].first = first;
        jobs[t].blob = blob; jobs[t].offsets = offsets;
        jobs[t].i0 = n * (uint64_t)t / (uint64_t)nthreads;
        jobs[t].i1 = n * (uint64_t)(t + 1) / (uint64_t)nthreads;
        pthread_create(&th[t], NULL, dict_worker, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}

int64_t fpc_dict_lengths_at(int cfg, uint64_t seed, uint64_t first, uint64_t n, uint64_t* offsets,
                            int nthreads) {
    if (fpc_max_len(cfg) < 0) return -1;
    offsets[0] = 0;
    run_dict(cfg, seed, first, n, NULL, offsets, nthreads);
    for (uint64_t i = 0; i < n; ++i) offsets[i + 1] += offsets[i];
    return (int64_t)offsets[n];
}

int fpc_dict_fill_at(int cfg, uint64_t seed, uint64_t first, uint64_t n, const uint64_t* offsets,
                     unsigned char* blob, int nthreads) {
    if (fpc_max_len(cfg) < 0) return -1;
    run_dict(cfg, seed, first, n, blob, (uint64_t*)offsets, nthreads);
    return 0;
}

int64_t fpc_dict_lengths(int cfg, uint64_t seed, uint64_t n, uint64_t* offsets, int nthreads) {
    return fpc_dict_lengths_at(cfg, seed, 0, n, offsets, nthreads);
}

int fpc_dict_fill(int cfg, uint64_t seed, uint64_t n, const uint64_t* offsets, unsigned char* blob,
                  int nthreads) {
    return fpc_dict_fill_at(cfg, seed, 0, n, offsets, blob, nthreads);
}

/* ---- queries -------------------------------------------------------------
 * Query i (stream 2) has kind = i % period:
 *   cfg1: 0 dictionary word + one substitution, 1 random word
 *   cfg2: 0 dictionary word unchanged, 1 one edit (sub/ins/del equiprobable), 2 random
 *   cfg3/4/5: 0 dictionary word + one edit (sub/ins/del), 1 random
 * The dictionary word is drawn uniformly from the first n_base words. */
int64_t fpc_queries(int cfg, uint64_t seed, const unsigned char* dblob, const uint64_t* doffs,
                    uint64_t n_base, uint64_t nq, unsigned char* qblob, uint64_t cap,
                    uint64_t* qoffs) {
    if (fpc_max_len(cfg) < 0 || n_base == 0) return -1;
    unsigned char buf[256];
    uint64_t pos = 0;
    qoffs[0] = 0;
    for (uint64_t i = 0; i < nq; ++i) {
        rng_t r = rng_for(seed, 2, i);
        int period = cfg == 2 ? 3 : 2;
        int kind = (int)(i % (uint64_t)period);
        int len;
        int from_dict = (cfg == 2) ? kind <= 1 : kind == 0;
        if (from_dict) {
            uint64_t w = below(&r, n_base);
            len = (int)(doffs[w + 1] - doffs[w]);
            memcpy(buf, dblob + doffs[w], (size_t)len);
            int edit = (cfg == 2) ? kind == 1 : 1;
            if (edit) {
                int ek = cfg == 1 ? 0 : (int)below(&r, 3);
                len = apply_edit(cfg, &r, ek, buf, len);
            }
        } else {
            len = gen_word(cfg, &r, buf);
        }
        if (pos + (uint64_t)len > cap) return -2;
        memcpy(qblob + pos, buf, (size_t)len);
        pos += (uint64_t)len;
        qoffs[i + 1] = pos;
    }
    return (int64_t)pos;
}
