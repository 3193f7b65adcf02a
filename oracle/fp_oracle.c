/*
 * fp_oracle.c -- CPU restatement of the reference fingerprint filter path.
 *
 * TEST INFRASTRUCTURE ONLY (see fp_oracle.h).  Every function cites the
 * reference file:line it restates; paths are relative to
 * /root/reference/proj/include/fingerprints/.
 */
#include "fp_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---- scheme layout (fingerprint.hpp:84-147, generalised 16 -> W) ---------- */

int fpo_letter_capacity(int variant, int width, int b, int p) {
    if (width != 16 && width != 32 && width != 64) return -1;
    switch (variant) {
        case FPO_OCCURRENCE: return width;                       /* :86 */
        case FPO_OCCURRENCE_HALVED: return width / 2;            /* :87 */
        case FPO_COUNT:                                          /* :88-91 */
            if (b <= 0 || width % b != 0) return -1;
            return width / b;
        case FPO_POSITION: {                                     /* :92-97 */
            if (p <= 0 || p > width) return -1;
            int slots = width / p;
            return slots + (width - slots * p);
        }
    }
    return -1;
}

int fpo_scheme_check(const fpo_scheme* s) {
    int cap = fpo_letter_capacity(s->variant, s->width, s->bits_per_count, s->bits_per_position);
    if (cap < 0 || cap != s->nletters) return -1;                /* :150-156 */
    int seen[256] = {0};
    for (int i = 0; i < s->nletters; ++i) {                      /* letter_model.hpp:64-70 */
        if (seen[s->letters[i]]) return -1;
        seen[s->letters[i]] = 1;
    }
    return 0;
}

static int position_slots(const fpo_scheme* s) { return s->width / s->bits_per_position; }
static int extra_slots(const fpo_scheme* s) {
    return s->width - position_slots(s) * s->bits_per_position;
}

static int field_count(const fpo_scheme* s) {                    /* :118-125 */
    switch (s->variant) {
        case FPO_OCCURRENCE: return s->width;
        case FPO_OCCURRENCE_HALVED: return s->width / 2;
        case FPO_COUNT: return s->width / s->bits_per_count;
        case FPO_POSITION: return position_slots(s) + extra_slots(s);
    }
    return 0;
}

static int field_width(const fpo_scheme* s, int i) {             /* :127-135 */
    switch (s->variant) {
        case FPO_OCCURRENCE: return 1;
        case FPO_OCCURRENCE_HALVED: return 2;
        case FPO_COUNT: return s->bits_per_count;
        case FPO_POSITION: return i < position_slots(s) ? s->bits_per_position : 1;
    }
    return 0;
}

static int field_shift(const fpo_scheme* s, int i) {             /* :138-147 */
    if (s->variant == FPO_POSITION) {
        int slots = position_slots(s);
        if (i < slots) return s->width - s->bits_per_position * (i + 1);
        return extra_slots(s) - 1 - (i - slots);
    }
    return s->width - field_width(s, 0) * (i + 1);
}

static void slot_table(const fpo_scheme* s, int slot[256]) {    /* letter_model.hpp:60-87 */
    for (int c = 0; c < 256; ++c) slot[c] = -1;
    for (int i = 0; i < s->nletters; ++i) slot[s->letters[i]] = i;
}

/* ---- letter selection (letter_model.hpp:33-45, 94-134) ------------------- */

int fpo_select_letters(const unsigned char* bytes, uint64_t nbytes, int count, int strategy,
                       unsigned char* out) {
    uint64_t cnt[256] = {0};
    for (uint64_t i = 0; i < nbytes; ++i) ++cnt[bytes[i]];
    /* rank by (count, byte) ascending; insertion sort over <= 256 symbols */
    int ranked[256], nr = 0;
    for (int c = 0; c < 256; ++c) {
        if (!cnt[c]) continue;
        int j = nr++;
        while (j > 0 && (cnt[ranked[j - 1]] > cnt[c] ||
                         (cnt[ranked[j - 1]] == cnt[c] && ranked[j - 1] > c))) {
            ranked[j] = ranked[j - 1];
            --j;
        }
        ranked[j] = c;
    }
    if (nr < count) return -1;                                   /* :106-109 */
    int k = 0;
    if (strategy == FPO_COMMON) {                                /* :113-116 */
        for (int i = 0; i < count; ++i) out[k++] = (unsigned char)ranked[nr - 1 - i];
    } else if (strategy == FPO_RARE) {                           /* :117-120 */
        for (int i = 0; i < count; ++i) out[k++] = (unsigned char)ranked[i];
    } else {                                                     /* :121-128 */
        int from_common = (count + 1) / 2, from_rare = count / 2;
        for (int i = 0; i < from_common; ++i) out[k++] = (unsigned char)ranked[nr - 1 - i];
        for (int i = 0; i < from_rare; ++i) out[k++] = (unsigned char)ranked[i];
        /* LetterSet ctor rejects overlap (letter_model.hpp:64-70) */
        for (int i = 0; i < k; ++i)
            for (int j = i + 1; j < k; ++j)
                if (out[i] == out[j]) return -1;
    }
    return count;
}

/* ---- builders (fingerprint.hpp:216-284) ---------------------------------- */

static uint64_t one(int bit) { return (uint64_t)1 << bit; }

uint64_t fpo_build(const unsigned char* s, size_t n, const fpo_scheme* sch) {
    int slot[256];
    slot_table(sch, slot);
    const int W = sch->width;
    uint64_t bits = 0;
    switch (sch->variant) {
        case FPO_OCCURRENCE:                                     /* :216-224 */
            for (size_t i = 0; i < n; ++i) {
                int q = slot[s[i]];
                if (q >= 0) bits |= one(W - 1 - q);
            }
            return bits;
        case FPO_OCCURRENCE_HALVED: {                            /* :226-238 */
            size_t half = n / 2;
            for (size_t i = 0; i < n; ++i) {
                int q = slot[s[i]];
                if (q < 0) continue;
                bits |= one(i < half ? W - 1 - 2 * q : W - 2 - 2 * q);
            }
            return bits;
        }
        case FPO_COUNT: {                                        /* :240-254 */
            const int b = sch->bits_per_count;
            const uint64_t sat = one(b) - 1;
            for (size_t i = 0; i < n; ++i) {
                int q = slot[s[i]];
                if (q < 0) continue;
                int shift = W - b * (q + 1);
                uint64_t field = (bits >> shift) & sat;
                if (field != sat) bits = (bits & ~(sat << shift)) | ((field + 1) << shift);
            }
            return bits;
        }
        case FPO_POSITION: {                                     /* :256-274 */
            const int p = sch->bits_per_position;
            const uint64_t absent = one(p) - 1;
            const int slots = position_slots(sch);
            for (int q = 0; q < sch->nletters; ++q) {
                size_t first = n;                                /* npos */
                for (size_t i = 0; i < n; ++i)
                    if (s[i] == sch->letters[q]) { first = i; break; }
                if (q < slots) {
                    uint64_t field = absent;
                    if (first != n && first < absent) field = first;
                    bits |= field << field_shift(sch, q);
                } else if (first != n) {
                    bits |= one(field_shift(sch, q));
                }
            }
            return bits;
        }
    }
    return 0;
}

void fpo_build_many(const unsigned char* blob, const uint64_t* offsets, uint64_t n,
                    const fpo_scheme* sch, uint64_t* out) {
    for (uint64_t i = 0; i < n; ++i)
        out[i] = fpo_build(blob + offsets[i], (size_t)(offsets[i + 1] - offsets[i]), sch);
}

/* ---- distances (reference.hpp:62-84; fingerprint.hpp:171-214, 287-301) --- */

int fpo_distance(uint64_t a, uint64_t b, const fpo_scheme* sch) {
    uint64_t x = a ^ b;
    if (sch->width < 64) x &= one(sch->width) - 1;
    if (sch->variant == FPO_OCCURRENCE || sch->variant == FPO_OCCURRENCE_HALVED) {
        int bits = 0;
        for (int i = 0; i < sch->width; ++i) bits += (int)((x >> i) & 1);
        return bits;
    }
    int mism = 0, nf = field_count(sch);
    for (int i = 0; i < nf; ++i) {
        uint64_t mask = one(field_width(sch, i)) - 1;
        if ((x >> field_shift(sch, i)) & mask) ++mism;
    }
    return mism;
}

int fpo_can_reject(uint64_t a, uint64_t b, int k, const fpo_scheme* sch) {
    int fd = fpo_distance(a, b, sch);
    return (fd + 1) / 2 > k;                                     /* ceil_half :182, :293-301 */
}

void fpo_render(uint64_t f, const fpo_scheme* sch, char* out) {  /* :305-317 */
    int nf = field_count(sch), k = 0;
    for (int i = 0; i < nf; ++i) {
        if (i != 0 && sch->variant != FPO_OCCURRENCE) out[k++] = ' ';
        int w = field_width(sch, i), sh = field_shift(sch, i);
        for (int bit = 0; bit < w; ++bit) out[k++] = ((f >> (sh + w - 1 - bit)) & 1) ? '1' : '0';
    }
    out[k] = 0;
}

/* ---- verifiers (edit_distance.hpp:18-64; reference.hpp:17-41) ------------ */

int fpo_hamming_bounded(const unsigned char* a, size_t na, const unsigned char* b, size_t nb,
                        int k) {
    if (na != nb) return -2;                                     /* :19-20 throws */
    int mism = 0;
    for (size_t i = 0; i < na; ++i)
        if (a[i] != b[i] && ++mism > k) return -1;
    return mism;
}

int fpo_levenshtein_bounded(const unsigned char* s1, size_t n1, const unsigned char* s2,
                            size_t n2, int k) {
    if (k < 0) return -1;                                        /* :32-33 */
    if (n1 > n2) {                                               /* :36-37 */
        const unsigned char* t = s1; s1 = s2; s2 = t;
        size_t tn = n1; n1 = n2; n2 = tn;
    }
    const int m = (int)n1, n = (int)n2;
    if (n - m > k) return -1;                                    /* :38-39 */
    const int inf = k + 1;
    int* prev = (int*)malloc(sizeof(int) * (size_t)(n + 1));
    int* cur = (int*)malloc(sizeof(int) * (size_t)(n + 1));
    for (int j = 0; j <= n; ++j) { prev[j] = inf; cur[j] = inf; }
    for (int j = 0; j <= (k < n ? k : n); ++j) prev[j] = j;
    int result = -1;
    for (int i = 1; i <= m; ++i) {                               /* banded rows :47-62 */
        int lo = i - k > 1 ? i - k : 1;
        int hi = i + k < n ? i + k : n;
        cur[lo - 1] = (i <= k) ? i : inf;
        int best = inf;
        for (int j = lo; j <= hi; ++j) {
            int v = prev[j - 1] + (s1[i - 1] != s2[j - 1]);
            if (j < i + k && prev[j] + 1 < v) v = prev[j] + 1;
            if (j > i - k && cur[j - 1] + 1 < v) v = cur[j - 1] + 1;
            cur[j] = v;
            if (v < best) best = v;
        }
        if (best > k) goto done;
        int* t = prev; prev = cur; cur = t;
    }
    if (prev[n] <= k) result = prev[n];
done:
    free(prev);
    free(cur);
    return result;
}

int fpo_levenshtein_full(const unsigned char* a, size_t na, const unsigned char* b, size_t nb) {
    int* prev = (int*)malloc(sizeof(int) * (nb + 1));
    int* cur = (int*)malloc(sizeof(int) * (nb + 1));
    for (size_t j = 0; j <= nb; ++j) prev[j] = (int)j;
    for (size_t i = 1; i <= na; ++i) {
        cur[0] = (int)i;
        for (size_t j = 1; j <= nb; ++j) {
            int v = prev[j - 1] + (a[i - 1] != b[j - 1]);
            if (prev[j] + 1 < v) v = prev[j] + 1;
            if (cur[j - 1] + 1 < v) v = cur[j - 1] + 1;
            cur[j] = v;
        }
        int* t = prev; prev = cur; cur = t;
    }
    int d = prev[nb];
    free(prev);
    free(cur);
    return d;
}

int fpo_hamming_full(const unsigned char* a, size_t na, const unsigned char* b, size_t nb) {
    if (na != nb) return -2;
    int m = 0;
    for (size_t i = 0; i < na; ++i) m += a[i] != b[i];
    return m;
}

/* ---- batch drivers: query_into (dictionary.hpp:75-118), naive_scan ------- */

typedef struct {
    uint32_t* v;
    uint64_t n, cap;
} vec32;

static void vpush(vec32* v, uint32_t x) {
    if (v->n == v->cap) {
        v->cap = v->cap ? v->cap * 2 : 1024;
        v->v = (uint32_t*)realloc(v->v, v->cap * sizeof(uint32_t));
    }
    v->v[v->n++] = x;
}

typedef struct {
    const unsigned char *dblob, *qblob;
    const uint64_t *doffs, *qoffs;
    uint64_t nd, q0, q1;
    const fpo_scheme* sch;
    const uint64_t* dprints;
    int metric, k, use_filter, length_prefilter, naive;
    uint64_t* counts; /* per query */
    uint64_t* stats;
    vec32 out;
} job;

static void* run_job(void* arg) {
    job* J = (job*)arg;
    for (uint64_t q = J->q0; q < J->q1; ++q) {
        const unsigned char* p = J->qblob + J->qoffs[q];
        const size_t plen = (size_t)(J->qoffs[q + 1] - J->qoffs[q]);
        uint64_t compared = 0, rej_len = 0, rej_fp = 0, verified = 0, matches = 0;
        uint64_t pf = (!J->naive && J->use_filter) ? fpo_build(p, plen, J->sch) : 0;  /* :84 */
        for (uint64_t i = 0; i < J->nd; ++i) {                    /* :86 */
            const unsigned char* w = J->dblob + J->doffs[i];
            const size_t wlen = (size_t)(J->doffs[i + 1] - J->doffs[i]);
            if (J->naive) {                                       /* reference.hpp:45-59 */
                int hit;
                if (J->metric == FPO_HAMMING)
                    hit = wlen == plen && fpo_hamming_full(w, wlen, p, plen) <= J->k;
                else
                    hit = fpo_levenshtein_full(w, wlen, p, plen) <= J->k;
                if (hit) { vpush(&J->out, (uint32_t)i); ++matches; }
                continue;
            }
            ++compared;
            if (J->metric == FPO_HAMMING) {                       /* :89-93 */
                if (wlen != plen) { ++rej_len; continue; }
            } else if (J->length_prefilter) {                     /* :94-101 */
                size_t gap = wlen > plen ? wlen - plen : plen - wlen;
                if (gap > (size_t)J->k) { ++rej_len; continue; }
            }
            if (J->use_filter && fpo_can_reject(pf, J->dprints[i], J->k, J->sch)) {  /* :102-106 */
                ++rej_fp;
                continue;
            }
            ++verified;                                           /* :107-110 */
            int d = J->metric == FPO_HAMMING ? fpo_hamming_bounded(w, wlen, p, plen, J->k)
                                             : fpo_levenshtein_bounded(w, wlen, p, plen, J->k);
            if (d >= 0) { vpush(&J->out, (uint32_t)i); ++matches; }  /* :111-114 */
        }
        J->counts[q] = matches;
        if (J->stats) {
            uint64_t* st = J->stats + 5 * q;
            st[0] = compared; st[1] = rej_len; st[2] = rej_fp; st[3] = verified; st[4] = matches;
        }
    }
    return NULL;
}

static int run_batch(const unsigned char* dblob, const uint64_t* doffs, uint64_t nd,
                     const unsigned char* qblob, const uint64_t* qoffs, uint64_t nq,
                     const fpo_scheme* sch, int metric, int k, int use_filter,
                     int length_prefilter, int naive, int nthreads, uint64_t* offsets,
                     uint64_t* stats, uint32_t** ids, uint64_t* total) {
    uint64_t* dprints = NULL;
    if (!naive && use_filter) {
        dprints = (uint64_t*)malloc(sizeof(uint64_t) * (nd ? nd : 1));
        fpo_build_many(dblob, doffs, nd, sch, dprints);           /* ctor :51-56 */
    }
    if (nthreads < 1) nthreads = 1;
    if ((uint64_t)nthreads > nq) nthreads = nq ? (int)nq : 1;
    job* jobs = (job*)calloc((size_t)nthreads, sizeof(job));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    uint64_t* counts = (uint64_t*)calloc(nq ? nq : 1, sizeof(uint64_t));
    for (int t = 0; t < nthreads; ++t) {
        job* J = &jobs[t];
        J->dblob = dblob; J->qblob = qblob; J->doffs = doffs; J->qoffs = qoffs; J->nd = nd;
        J->q0 = nq * (uint64_t)t / (uint64_t)nthreads;
        J->q1 = nq * (uint64_t)(t + 1) / (uint64_t)nthreads;
        J->sch = sch; J->dprints = dprints; J->metric = metric; J->k = k;
        J->use_filter = use_filter; J->length_prefilter = length_prefilter; J->naive = naive;
        J->counts = counts; J->stats = stats;
        if (nthreads > 1) pthread_create(&th[t], NULL, run_job, J);
    }
    if (nthreads == 1) run_job(&jobs[0]);
    else for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    uint64_t tot = 0;
    offsets[0] = 0;
    for (uint64_t q = 0; q < nq; ++q) { tot += counts[q]; offsets[q + 1] = tot; }
    uint32_t* out = (uint32_t*)malloc(sizeof(uint32_t) * (tot ? tot : 1));
    uint64_t pos = 0;
    for (int t = 0; t < nthreads; ++t) {                           /* threads own ascending q ranges */
        if (jobs[t].out.n) memcpy(out + pos, jobs[t].out.v, jobs[t].out.n * sizeof(uint32_t));
        pos += jobs[t].out.n;
        free(jobs[t].out.v);
    }
    *ids = out;
    *total = tot;
    free(counts); free(jobs); free(th); free(dprints);
    return 0;
}

static int supports(int variant, int metric) {                    /* fingerprint.hpp:36-38 */
    return metric == FPO_HAMMING || variant == FPO_OCCURRENCE || variant == FPO_COUNT;
}

int fpo_query_batch(const unsigned char* dblob, const uint64_t* doffs, uint64_t nd,
                    const unsigned char* qblob, const uint64_t* qoffs, uint64_t nq,
                    const fpo_scheme* sch, int metric, int k, int use_filter,
                    int length_prefilter, int nthreads, uint64_t* offsets, uint64_t* stats,
                    uint32_t** ids, uint64_t* total) {
    if (use_filter && !supports(sch->variant, metric)) return -1;  /* dictionary.hpp:78-79 */
    return run_batch(dblob, doffs, nd, qblob, qoffs, nq, sch, metric, k, use_filter,
                     length_prefilter, 0, nthreads, offsets, stats, ids, total);
}

int fpo_naive_scan_batch(const unsigned char* dblob, const uint64_t* doffs, uint64_t nd,
                         const unsigned char* qblob, const uint64_t* qoffs, uint64_t nq,
                         int metric, int k, int nthreads, uint64_t* offsets, uint32_t** ids,
                         uint64_t* total) {
    return run_batch(dblob, doffs, nd, qblob, qoffs, nq, NULL, metric, k, 0, 0, 1, nthreads,
                     offsets, NULL, ids, total);
}

void fpo_free(void* p) { free(p); }
