/*
 * qc_oracle.c -- TEST INFRASTRUCTURE ONLY.  CPU restatement of the reference
 * algorithm for the hot path, used as the parity checker by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
 * leg.  Never linked into or called from the product path (libqcb200).
 *
 * Restates, in plain C99 with IEEE float32 and wrapping int16 arithmetic:
 *   - decode_batch_f32   /root/reference/pkg/src/qcldpc/_kernels.py:17-100
 *   - decode_batch_i16   /root/reference/pkg/src/qcldpc/_kernels.py:103-186
 *     (row update :49-84 / :135-170, syndrome + early exit :85-96 / :171-182,
 *      hard decision :97-100 / :183-186)
 *   - decode_block's contiguous chunking over worker threads
 *                        /root/reference/pkg/src/qcldpc/decoder.py:217-258
 *   - encode_packed      /root/reference/pkg/src/qcldpc/encoder.py:166-199
 *     with cyclic_shift_packed / cyclic_shift_inverse (encoder.py:72-100)
 *     on big-endian words of word_bits (encoder.py:111-123)
 *
 * Extension (north_star "LLRs out"): the decoders can also return the final
 * posteriors (post_out, nullable); the reference only exposes them through
 * decoder.init_state + tier_update (decoder.py:94-149), which the golden
 * fixtures in tests/golden/ were generated from.
 *
 * Build: oracle/Makefile  (gcc -O3 -ffp-contract=off -fno-fast-math).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    const int32_t *row_ptr, *col_idx;
    int32_t n_rows, n, mb, z;
    int64_t w;
    int32_t max_iters, early_term;
    const void *llrs;
    uint8_t *hard;
    int32_t *iters;
    uint8_t *conv;
    void *post_out;
} job_t;

static int32_t max_degree(const int32_t *row_ptr, int32_t n_rows) {
    int32_t d = 0;
    for (int32_t m = 0; m < n_rows; ++m)
        if (row_ptr[m + 1] - row_ptr[m] > d) d = row_ptr[m + 1] - row_ptr[m];
    return d;
}

/* _kernels.py:17-100 */
static void decode_f32_range(const job_t *J, int64_t w0, int64_t w1) {
    const int32_t *rp = J->row_ptr, *ci = J->col_idx;
    const int32_t M = J->n_rows, N = J->n, Z = J->z, MB = J->mb;
    const float *llrs = (const float *)J->llrs;
    float *post = malloc(sizeof(float) * (size_t)N);
    float *min1 = malloc(sizeof(float) * (size_t)M), *min2 = malloc(sizeof(float) * (size_t)M);
    int8_t *amin = malloc((size_t)M);
    uint32_t *sbits = malloc(sizeof(uint32_t) * (size_t)M);
    uint8_t *sprod = malloc((size_t)M);
    float *zrow = malloc(sizeof(float) * (size_t)(max_degree(rp, M) + 1));
    for (int64_t w = w0; w < w1; ++w) {
        memcpy(post, llrs + w * N, sizeof(float) * (size_t)N);
        for (int32_t m = 0; m < M; ++m) { min1[m] = 0.0f; min2[m] = 0.0f; amin[m] = 0; sbits[m] = 0; sprod[m] = 0; }
        int32_t it = 0, ok = 0;
        for (int32_t k = 0; k < J->max_iters; ++k) {
            for (int32_t t = 0; t < MB; ++t) {
                for (int32_t m = t * Z; m < (t + 1) * Z; ++m) {
                    const int32_t lo = rp[m], deg = rp[m + 1] - lo;
                    const int32_t *cols = ci + lo;
                    const float m1 = min1[m], m2 = min2[m];
                    const int32_t am = amin[m];
                    /* sign of L_old_j = sp ^ bit j of sb (:63) */
                    const uint32_t sbx = sbits[m] ^ (sprod[m] ? 0xFFFFFFFFu : 0u);
                    float nm1 = INFINITY, nm2 = INFINITY;
                    int32_t nam = 0;
                    uint32_t nsb = 0, nsp = 0;
                    for (int32_t j = 0; j < deg; ++j) {               /* :61-75 */
                        const float mag = (j == am) ? m2 : m1;
                        const float lold = ((sbx >> j) & 1u) ? -mag : mag;
                        const float zz = post[cols[j]] - lold;
                        zrow[j] = zz;
                        const float a = fabsf(zz);
                        /* if a < nm1: nm2 = nm1, nm1 = a, nam = j; elif a < nm2: nm2 = a
                         * (written branch-free; same selections, NaN compares false) */
                        const int lt1 = a < nm1, lt2 = a < nm2;
                        nm2 = lt1 ? nm1 : (lt2 ? a : nm2);
                        nm1 = lt1 ? a : nm1;
                        nam = lt1 ? j : nam;
                        const uint32_t neg = zz < 0.0f;
                        nsb |= neg << j;
                        nsp ^= neg;
                    }
                    const uint32_t nsbx = nsb ^ (nsp ? 0xFFFFFFFFu : 0u);
                    for (int32_t j = 0; j < deg; ++j) {               /* :76-79 */
                        const float mag = (j == nam) ? nm2 : nm1;
                        const float lnew = ((nsbx >> j) & 1u) ? -mag : mag;
                        post[cols[j]] = zrow[j] + lnew;
                    }
                    min1[m] = nm1; min2[m] = nm2; amin[m] = (int8_t)nam;
                    sbits[m] = nsb; sprod[m] = (uint8_t)nsp;
                }
            }
            it = k + 1;                                               /* :85-96 */
            ok = 1;
            for (int32_t m = 0; m < M && ok; ++m) {
                int par = 0;
                for (int32_t p = rp[m]; p < rp[m + 1]; ++p) par ^= post[ci[p]] <= 0.0f;
                if (par) ok = 0;
            }
            if (ok && J->early_term) break;
        }
        for (int32_t i = 0; i < N; ++i) J->hard[w * N + i] = post[i] <= 0.0f;  /* :97-100 */
        J->iters[w] = it;
        J->conv[w] = (uint8_t)ok;
        if (J->post_out) memcpy((float *)J->post_out + w * N, post, sizeof(float) * (size_t)N);
    }
    free(post); free(min1); free(min2); free(amin); free(sbits); free(sprod); free(zrow);
}

/* two's-complement int16 wrap after every op, as numba's np.int16(...) casts do */
static inline int16_t w16(int32_t x) { return (int16_t)(uint16_t)(uint32_t)x; }

/* _kernels.py:103-186 */
static void decode_i16_range(const job_t *J, int64_t w0, int64_t w1) {
    const int32_t *rp = J->row_ptr, *ci = J->col_idx;
    const int32_t M = J->n_rows, N = J->n, Z = J->z, MB = J->mb;
    const int16_t *llrs = (const int16_t *)J->llrs;
    int16_t *post = malloc(sizeof(int16_t) * (size_t)N);
    int16_t *min1 = malloc(sizeof(int16_t) * (size_t)M), *min2 = malloc(sizeof(int16_t) * (size_t)M);
    int8_t *amin = malloc((size_t)M);
    uint32_t *sbits = malloc(sizeof(uint32_t) * (size_t)M);
    uint8_t *sprod = malloc((size_t)M);
    int16_t *zrow = malloc(sizeof(int16_t) * (size_t)(max_degree(rp, M) + 1));
    for (int64_t w = w0; w < w1; ++w) {
        memcpy(post, llrs + w * N, sizeof(int16_t) * (size_t)N);
        for (int32_t m = 0; m < M; ++m) { min1[m] = 0; min2[m] = 0; amin[m] = 0; sbits[m] = 0; sprod[m] = 0; }
        int32_t it = 0, ok = 0;
        for (int32_t k = 0; k < J->max_iters; ++k) {
            for (int32_t t = 0; t < MB; ++t) {
                for (int32_t m = t * Z; m < (t + 1) * Z; ++m) {
                    const int32_t lo = rp[m], deg = rp[m + 1] - lo;
                    const int32_t *cols = ci + lo;
                    const int16_t m1 = min1[m], m2 = min2[m];
                    const int32_t am = amin[m];
                    const uint32_t sbx = sbits[m] ^ (sprod[m] ? 0xFFFFFFFFu : 0u);
                    int16_t nm1 = 32767, nm2 = 32767;                 /* :142-143 */
                    int32_t nam = 0;
                    uint32_t nsb = 0, nsp = 0;
                    for (int32_t j = 0; j < deg; ++j) {               /* :147-161 */
                        const int16_t mag = (j == am) ? m2 : m1;
                        const int16_t lold = ((sbx >> j) & 1u) ? w16(-(int32_t)mag) : mag;
                        const int16_t zz = w16((int32_t)post[cols[j]] - lold);
                        zrow[j] = zz;
                        const int16_t a = w16(zz < 0 ? -(int32_t)zz : zz);  /* abs(-32768) stays -32768 */
                        const int lt1 = a < nm1, lt2 = a < nm2;
                        nm2 = lt1 ? nm1 : (lt2 ? a : nm2);
                        nm1 = lt1 ? a : nm1;
                        nam = lt1 ? j : nam;
                        const uint32_t neg = zz < 0;
                        nsb |= neg << j;
                        nsp ^= neg;
                    }
                    const uint32_t nsbx = nsb ^ (nsp ? 0xFFFFFFFFu : 0u);
                    for (int32_t j = 0; j < deg; ++j) {               /* :162-165 */
                        const int16_t mag = (j == nam) ? nm2 : nm1;
                        const int16_t lnew = ((nsbx >> j) & 1u) ? w16(-(int32_t)mag) : mag;
                        post[cols[j]] = w16((int32_t)zrow[j] + lnew);
                    }
                    min1[m] = nm1; min2[m] = nm2; amin[m] = (int8_t)nam;
                    sbits[m] = nsb; sprod[m] = (uint8_t)nsp;
                }
            }
            it = k + 1;
            ok = 1;
            for (int32_t m = 0; m < M && ok; ++m) {
                int par = 0;
                for (int32_t p = rp[m]; p < rp[m + 1]; ++p) par ^= post[ci[p]] <= 0;
                if (par) ok = 0;
            }
            if (ok && J->early_term) break;
        }
        for (int32_t i = 0; i < N; ++i) J->hard[w * N + i] = post[i] <= 0;
        J->iters[w] = it;
        J->conv[w] = (uint8_t)ok;
        if (J->post_out) memcpy((int16_t *)J->post_out + w * N, post, sizeof(int16_t) * (size_t)N);
    }
    free(post); free(min1); free(min2); free(amin); free(sbits); free(sprod); free(zrow);
}

typedef struct { const job_t *job; int64_t w0, w1; int is_i16; } chunk_t;

static void *run_chunk(void *arg) {
    const chunk_t *c = (const chunk_t *)arg;
    if (c->is_i16) decode_i16_range(c->job, c->w0, c->w1);
    else decode_f32_range(c->job, c->w0, c->w1);
    return NULL;
}

/* decoder.py:217-258: contiguous ceil(W/workers) chunks, one thread each;
 * results do not depend on the worker count. */
static int decode_mt(job_t *J, int workers, int is_i16) {
    if (workers < 1) workers = 1;
    if (J->w <= 0) return 0;
    int64_t chunk = (J->w + workers - 1) / workers;
    int nchunks = (int)((J->w + chunk - 1) / chunk);
    pthread_t *th = calloc((size_t)nchunks, sizeof(pthread_t));
    chunk_t *cs = calloc((size_t)nchunks, sizeof(chunk_t));
    int started = 0;
    for (int i = 0; i < nchunks; ++i) {
        cs[i].job = J; cs[i].w0 = (int64_t)i * chunk;
        cs[i].w1 = cs[i].w0 + chunk < J->w ? cs[i].w0 + chunk : J->w;
        cs[i].is_i16 = is_i16;
        if (nchunks == 1 || pthread_create(&th[i], NULL, run_chunk, &cs[i]) != 0) {
            run_chunk(&cs[i]);
            th[i] = 0;
        } else {
            started++;
        }
    }
    for (int i = 0; i < nchunks; ++i) if (th[i]) pthread_join(th[i], NULL);
    free(th); free(cs);
    (void)started;
    return 0;
}

int oracle_decode_f32(const int32_t *row_ptr, const int32_t *col_idx, int32_t n_rows, int32_t n,
                      int32_t mb, int32_t z, const float *llrs, int64_t w, int32_t max_iters,
                      int32_t early_term, uint8_t *hard, int32_t *iters, uint8_t *conv,
                      float *post_out, int32_t workers) {
    job_t J = {row_ptr, col_idx, n_rows, n, mb, z, w, max_iters, early_term, llrs, hard, iters, conv, post_out};
    return decode_mt(&J, workers, 0);
}

int oracle_decode_i16(const int32_t *row_ptr, const int32_t *col_idx, int32_t n_rows, int32_t n,
                      int32_t mb, int32_t z, const int16_t *llrs, int64_t w, int32_t max_iters,
                      int32_t early_term, uint8_t *hard, int32_t *iters, uint8_t *conv,
                      int16_t *post_out, int32_t workers) {
    job_t J = {row_ptr, col_idx, n_rows, n, mb, z, w, max_iters, early_term, llrs, hard, iters, conv, post_out};
    return decode_mt(&J, workers, 1);
}

/* ---- packed direct encoder (encoder.py:166-199) --------------------------- */

/* rotate one Z-bit block held as zw words of wb bits (big-endian bit order:
 * bit 0 of the block = MSB of word 0) so out bit j = in bit (j - s) mod Z.
 * encoder.py:72-90 (word pair funnel + whole-word roll). */
static void rot_fwd(const uint32_t *a, uint32_t *out, int zw, int wb, int s) {
    int sw = s / wb, sb = s % wb;
    uint32_t mask = wb == 32 ? 0xFFFFFFFFu : ((1u << wb) - 1u);
    for (int i = 0; i < zw; ++i) {
        uint32_t cur = a[i], prev = a[(i - 1 + zw) % zw], comb;
        comb = sb == 0 ? cur : (((prev << (wb - sb)) | (cur >> sb)) & mask);
        out[(i + sw) % zw] = comb;
    }
}

/* multiplying by the shift-e circulant = inverse rotation (encoder.py:93-100) */
static void rot_inv(const uint32_t *a, uint32_t *out, int zw, int wb, int e, int z) {
    rot_fwd(a, out, zw, wb, (z - e) % z);
}

static void bytes_to_words(const uint8_t *b, uint32_t *w, int nwords, int wb) {
    int bpw = wb / 8;
    for (int i = 0; i < nwords; ++i) {
        uint32_t v = 0;
        for (int q = 0; q < bpw; ++q) v = (v << 8) | b[i * bpw + q];
        w[i] = v;
    }
}

static void words_to_bytes(const uint32_t *w, uint8_t *b, int nwords, int wb) {
    int bpw = wb / 8;
    for (int i = 0; i < nwords; ++i)
        for (int q = 0; q < bpw; ++q) b[i * bpw + q] = (uint8_t)(w[i] >> (8 * (bpw - 1 - q)));
}

/* entries: mb x nb row-major shifts (-1 = zero block).  info: W x K/8 bytes,
 * cw: W x N/8 bytes ([info | parity]).  Returns -1 on bad arguments. */
int oracle_encode_packed(const int32_t *entries, int32_t mb, int32_t nb, int32_t z,
                         int32_t word_bits, int32_t y, int32_t hb_shift,
                         const uint8_t *info, int64_t w, uint8_t *cw) {
    const int32_t kb = nb - mb;
    if (z % 8 || (word_bits != 8 && word_bits != 16 && word_bits != 32) || z % word_bits) return -1;
    (void)y;
    const int zw = z / word_bits, kbytes = kb * z / 8, nbytes = nb * z / 8;
    uint32_t *u = malloc(sizeof(uint32_t) * (size_t)(kb * zw));
    uint32_t *s = calloc((size_t)(mb * zw), sizeof(uint32_t));
    uint32_t *v = calloc((size_t)(mb * zw), sizeof(uint32_t));
    uint32_t *tmp = malloc(sizeof(uint32_t) * (size_t)zw), *acc = malloc(sizeof(uint32_t) * (size_t)zw);
    for (int64_t f = 0; f < w; ++f) {
        const uint8_t *in = info + f * kbytes;
        uint8_t *out = cw + f * nbytes;
        bytes_to_words(in, u, kb * zw, word_bits);
        memset(s, 0, sizeof(uint32_t) * (size_t)(mb * zw));
        for (int i = 0; i < mb; ++i)                                  /* :180-186 */
            for (int j = 0; j < kb; ++j) {
                int e = entries[i * nb + j];
                if (e < 0) continue;
                rot_inv(u + j * zw, tmp, zw, word_bits, e, z);
                for (int q = 0; q < zw; ++q) s[i * zw + q] ^= tmp[q];
            }
        memset(acc, 0, sizeof(uint32_t) * (size_t)zw);               /* :188-191 */
        for (int i = 0; i < mb; ++i)
            for (int q = 0; q < zw; ++q) acc[q] ^= s[i * zw + q];
        rot_fwd(acc, v, zw, word_bits, hb_shift);
        if (mb >= 2) {                                                 /* :192 */
            rot_inv(v, tmp, zw, word_bits, entries[0 * nb + kb], z);
            for (int q = 0; q < zw; ++q) v[1 * zw + q] = s[q] ^ tmp[q];
        }
        for (int i = 1; i < mb - 1; ++i) {                            /* :193-197 */
            int hb = entries[i * nb + kb];
            for (int q = 0; q < zw; ++q) v[(i + 1) * zw + q] = v[i * zw + q] ^ s[i * zw + q];
            if (hb >= 0) {
                rot_inv(v, tmp, zw, word_bits, hb, z);
                for (int q = 0; q < zw; ++q) v[(i + 1) * zw + q] ^= tmp[q];
            }
        }
        memcpy(out, in, (size_t)kbytes);                               /* :198-199 */
        words_to_bytes(v, out + kbytes, mb * zw, word_bits);
    }
    free(u); free(s); free(v); free(tmp); free(acc);
    return 0;
}
