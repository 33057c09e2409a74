/*
 * TEST INFRASTRUCTURE ONLY — never linked into the product.
 *
 * Plain-C restatement of the reference's DiLoCo outer-synchronisation path
 * (INTELLECT-1 / PRIME, `emesh` C++ library under /root/reference/proj).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this (as liboracle.so through oracle/pyoracle.py) — as the checker,
 * never as the thing measured or shipped.
 *
 * Pinning: every function here is cross-checked against the compiled
 * reference itself (oracle/_ref/libemesh_ref.so, built by oracle/Makefile
 * from the reference headers) and against the reference tests' known-answer
 * vectors (tests/test_oracle_pinned.py, tests/golden/).
 *
 * Numerics contract: no FMA anywhere — this file is compiled
 * with -O2 -ffp-contract=off, so every a*b+c is two roundings, exactly like
 * the reference's RelWithDebInfo build (proj/CMakeLists.txt:3-9).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ESHAPE 1
#define ORC_ENUMERIC 2
#define ORC_EDECODE 3

#define NBUCKETS 256

/* ---- counter RNG: proj/include/emesh/rng.hpp:11-32 ------------------- */

static uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

uint64_t orc_rng_word(uint64_t seed, uint64_t stream, uint64_t counter, uint64_t index) {
    uint64_t h = mix64(seed ^ 0x8f1bbcdc545a7c15ull);
    h = mix64(h ^ stream);
    h = mix64(h ^ counter);
    return mix64(h ^ index);
}

/* rng.hpp:26-30: top 24 bits, scaled by 2^-23, minus one: exact in fp32. */
float orc_rng_uniform(uint64_t seed, uint64_t stream, uint64_t counter, uint64_t index) {
    uint32_t top = (uint32_t)(orc_rng_word(seed, stream, counter, index) >> 40);
    return (float)top * (1.0f / 8388608.0f) - 1.0f;
}

void orc_fill_uniform(float* out, uint64_t n, uint64_t seed, uint64_t stream,
                      uint64_t counter, uint64_t first_index, float scale) {
    for (uint64_t i = 0; i < n; ++i)
        out[i] = scale * orc_rng_uniform(seed, stream, counter, first_index + i);
}

/* ---- segment table: allreduce.hpp:107-118 (split) and :327-336 (subs) ---
 * Chunk c of k covers [chunk_lo(c), chunk_lo(c)+chunk_len(c)); the first
 * total%parts pieces get one extra element. A chunk of length len is cut
 * into min(S, len) sub-slices, or one empty sub-slice when len == 0. */

static void split_piece(uint64_t total, uint64_t parts, uint64_t i, uint64_t* lo, uint64_t* len) {
    uint64_t base = parts ? total / parts : 0;
    uint64_t rem = parts ? total % parts : 0;
    *len = base + (i < rem ? 1 : 0);
    *lo = i * base + (i < rem ? i : rem);
}

uint64_t orc_subs_count(uint64_t chunk_len, uint32_t S) {
    if (chunk_len == 0) return 1;
    return chunk_len < S ? chunk_len : S;
}

/* Writes the absolute [lo, len) of every segment of every chunk, chunk-major.
 * Returns the segment count. seg_lo/seg_len may be NULL to just count. */
uint64_t orc_segment_table(uint64_t n, uint32_t k, uint32_t S, uint64_t* seg_lo, uint64_t* seg_len) {
    uint64_t idx = 0;
    for (uint32_t c = 0; c < k; ++c) {
        uint64_t clo, clen;
        split_piece(n, k, c, &clo, &clen);
        uint64_t ns = orc_subs_count(clen, S);
        for (uint64_t j = 0; j < ns; ++j) {
            uint64_t slo, slen;
            split_piece(clen, ns, j, &slo, &slen);
            if (seg_lo) seg_lo[idx] = clo + slo;
            if (seg_len) seg_len[idx] = slen;
            ++idx;
        }
    }
    return idx;
}

/* ---- codec: quant.hpp:28-87 ------------------------------------------
 * Statistics in fp64, strictly sequential index order; population sigma;
 * range mu +- 6 sigma; bucket = floor((clip(x) - lo) / width) clamped to
 * [0,255]; codebook = (float)(sum of clipped members / count), empty
 * buckets get their midpoint; sigma == 0 -> all codes 0, codebook = mu.
 * stats_out (may be NULL): {mu, sigma, lo, width}. */
int orc_quantize(const float* x, uint64_t n, uint8_t* codes, float* cb, double* stats_out) {
    if (n == 0) return ORC_ESHAPE;
    for (uint64_t i = 0; i < n; ++i)
        if (!isfinite(x[i])) return ORC_ENUMERIC;

    double s = 0.0;
    for (uint64_t i = 0; i < n; ++i) s += (double)x[i];
    const double mu = s / (double)n;
    double ss = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        const double d = (double)x[i] - mu;
        const double d2 = d * d;
        ss += d2;
    }
    const double sigma = sqrt(ss / (double)n);

    if (sigma == 0.0) {
        memset(codes, 0, n);
        for (int b = 0; b < NBUCKETS; ++b) cb[b] = (float)mu;
        if (stats_out) { stats_out[0] = mu; stats_out[1] = sigma; stats_out[2] = mu; stats_out[3] = 0.0; }
        return ORC_OK;
    }

    const double six_sigma = 6.0 * sigma;
    const double lo = mu - six_sigma;
    const double hi = mu + six_sigma;
    const double width = (hi - lo) / 256.0;

    double bsum[NBUCKETS];
    uint64_t bcnt[NBUCKETS];
    for (int b = 0; b < NBUCKETS; ++b) { bsum[b] = 0.0; bcnt[b] = 0; }

    for (uint64_t i = 0; i < n; ++i) {
        double v = (double)x[i];
        if (v < lo) v = lo;
        if (v > hi) v = hi;
        long b = (long)floor((v - lo) / width);
        if (b < 0) b = 0;
        if (b > NBUCKETS - 1) b = NBUCKETS - 1;
        codes[i] = (uint8_t)b;
        bsum[b] += v;
        bcnt[b] += 1;
    }
    for (int b = 0; b < NBUCKETS; ++b) {
        if (bcnt[b]) {
            cb[b] = (float)(bsum[b] / (double)bcnt[b]);
        } else {
            const double mid = (double)b + 0.5;
            const double off = mid * width;
            cb[b] = (float)(lo + off);
        }
    }
    if (stats_out) { stats_out[0] = mu; stats_out[1] = sigma; stats_out[2] = lo; stats_out[3] = width; }
    return ORC_OK;
}

/* quant.hpp:89-94 */
void orc_dequantize(const uint8_t* codes, const float* cb, uint64_t n, float* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = cb[codes[i]];
}

/* Smallest distance (in buckets) from (clip(x)-lo)/width to an integer, over
 * the segment: the margin by which a last-bit change in lo/width could flip a
 * code. Diagnostic for the parity report (SURVEY.md §7 hard part 1). */
double orc_boundary_margin(const float* x, uint64_t n, double lo, double width, double hi) {
    double m = 1.0;
    for (uint64_t i = 0; i < n; ++i) {
        double v = (double)x[i];
        if (v < lo) v = lo;
        if (v > hi) v = hi;
        const double q = (v - lo) / width;
        const double f = q - floor(q);
        const double d = f < 1.0 - f ? f : 1.0 - f;
        if (q > 0.5 && q < 255.5 && d < m) m = d;
    }
    return m;
}

/* ---- optimizer: optim.hpp:99-111 and :116-132 ---------------------- */

void orc_pseudo_gradient(const float* theta_prev, const float* theta_local, uint64_t n, float* delta) {
    for (uint64_t i = 0; i < n; ++i) delta[i] = theta_prev[i] - theta_local[i];
}

/* b <- mu*b + d ; theta <- theta - lr*(d + mu*b), each op rounded to fp32. */
void orc_nesterov(float* theta, const float* avg, float* buf, uint64_t n, float lr, float momentum) {
    for (uint64_t i = 0; i < n; ++i) {
        const float mb = momentum * buf[i];
        const float nb = mb + avg[i];
        buf[i] = nb;
        const float mb2 = momentum * nb;
        const float g = avg[i] + mb2;
        const float step = lr * g;
        theta[i] = theta[i] - step;
    }
}

/* AdamW inner step, optim.hpp:63-94 (bias correction, decoupled decay),
 * every fp32 operation rounded in the reference's order; `step` is the
 * state's step AFTER the increment (optim.hpp:71). Returns ORC_ENUMERIC at
 * the first non-finite gradient, elements before it updated (as the
 * reference's loop leaves them). */
int orc_adamw(float* p, const float* g, float* m, float* v, uint64_t n, uint64_t step, float inner_lr,
              float lr_scale, float beta1, float beta2, float eps, float weight_decay) {
    const float lr = inner_lr * lr_scale;
    const float bc1 = (float)(1.0 - pow((double)beta1, (double)step));
    const float bc2 = (float)(1.0 - pow((double)beta2, (double)step));
    for (uint64_t i = 0; i < n; ++i) {
        const float gi = g[i];
        if (!isfinite(gi)) return ORC_ENUMERIC;
        const float lrwd = lr * weight_decay;
        const float dec = lrwd * p[i];
        p[i] = p[i] - dec;
        const float m1 = beta1 * m[i];
        const float m2 = (1.0f - beta1) * gi;
        m[i] = m1 + m2;
        const float v1 = beta2 * v[i];
        const float v2a = (1.0f - beta2) * gi;
        const float v2 = v2a * gi;
        v[i] = v1 + v2;
        const float mhat = m[i] / bc1;
        const float vhat = v[i] / bc2;
        const float num = lr * mhat;
        const float den = sqrtf(vhat) + eps;
        p[i] = p[i] - num / den;
    }
    return ORC_OK;
}

/* ---- ring all-reduce, transport-free: allreduce.hpp:314-473 ----------
 * inputs: k pointers to n floats (worker r's ReduceJob.input, untouched).
 * out:    n floats — the result every rank ends with (they are identical,
 *         allreduce.hpp:309-313).
 * mode:   0 = fp32 (raw payloads), 1 = int8 (quantized payloads).
 * final_codes (n bytes) / final_cb (nseg*256 floats) / final_stats
 * (nseg*4 doubles), optional: the owner's final payloads per segment in
 * segment-table order (int8 only).
 * Reduce-scatter hop s: rank r ships Q(acc_r[chunk (r-s)%k]) to r+1, and
 * r adds D(payload from r-1) into acc_r[chunk (r-s-1)%k] (own + incoming,
 * :422). The owner of chunk c is rank (c-1)%k; it divides by (float)k
 * (:435-439), quantizes once and decodes its own bytes (:441-443); the
 * all-gather forwards those bytes verbatim (:446-464). k == 1 is the
 * identity (:319). */
int orc_ring_allreduce(const float* const* inputs, uint32_t k, uint64_t n, uint32_t S, int mode,
                       float* out, uint8_t* final_codes, float* final_cb, double* final_stats) {
    if (k == 0) return ORC_ESHAPE;
    if (k == 1) {
        memcpy(out, inputs[0], n * sizeof(float));
        return ORC_OK;
    }
    float** acc = (float**)malloc(k * sizeof(float*));
    float** wire = (float**)malloc(k * sizeof(float*));
    uint64_t maxc = n / k + 1;
    uint8_t* tmp_codes = (uint8_t*)malloc(maxc + 1);
    float cb[NBUCKETS];
    int rc = ORC_OK;
    for (uint32_t r = 0; r < k; ++r) {
        acc[r] = (float*)malloc((n ? n : 1) * sizeof(float));
        memcpy(acc[r], inputs[r], n * sizeof(float));
        wire[r] = (float*)malloc(maxc * sizeof(float));
    }
    for (uint32_t s = 0; s + 1 < k && rc == ORC_OK; ++s) {
        /* every rank's transmission of hop s, decoded as the receiver sees it */
        for (uint32_t r = 0; r < k && rc == ORC_OK; ++r) {
            uint32_t send_c = (uint32_t)((r + k - s) % k);
            uint64_t clo, clen;
            split_piece(n, k, send_c, &clo, &clen);
            uint64_t ns = orc_subs_count(clen, S);
            for (uint64_t j = 0; j < ns && rc == ORC_OK; ++j) {
                uint64_t slo, slen;
                split_piece(clen, ns, j, &slo, &slen);
                if (slen == 0) continue;
                const float* src = acc[r] + clo + slo;
                float* dst = wire[(r + 1) % k] + slo;
                if (mode == 0) {
                    memcpy(dst, src, slen * sizeof(float));
                } else {
                    rc = orc_quantize(src, slen, tmp_codes, cb, NULL);
                    if (rc == ORC_OK) orc_dequantize(tmp_codes, cb, slen, dst);
                }
            }
        }
        for (uint32_t r = 0; r < k && rc == ORC_OK; ++r) {
            uint32_t recv_c = (uint32_t)((r + k - s - 1) % k);
            uint64_t clo, clen;
            split_piece(n, k, recv_c, &clo, &clen);
            for (uint64_t i = 0; i < clen; ++i) acc[r][clo + i] = acc[r][clo + i] + wire[r][i];
        }
    }
    /* owners finalize; every rank decodes the same bytes */
    uint64_t seg = 0;
    for (uint32_t c = 0; c < k && rc == ORC_OK; ++c) {
        uint32_t owner = (c + k - 1) % k;
        uint64_t clo, clen;
        split_piece(n, k, c, &clo, &clen);
        uint64_t ns = orc_subs_count(clen, S);
        const float divisor = (float)k;
        for (uint64_t j = 0; j < ns && rc == ORC_OK; ++j, ++seg) {
            uint64_t slo, slen;
            split_piece(clen, ns, j, &slo, &slen);
            float* mean = wire[0];
            for (uint64_t i = 0; i < slen; ++i) mean[i] = acc[owner][clo + slo + i] / divisor;
            if (slen == 0) continue;
            if (mode == 0) {
                memcpy(out + clo + slo, mean, slen * sizeof(float));
            } else {
                double st[4];
                rc = orc_quantize(mean, slen, tmp_codes, cb, st);
                if (rc != ORC_OK) break;
                orc_dequantize(tmp_codes, cb, slen, out + clo + slo);
                if (final_codes) memcpy(final_codes + clo + slo, tmp_codes, slen);
                if (final_cb) memcpy(final_cb + seg * NBUCKETS, cb, sizeof(cb));
                if (final_stats) memcpy(final_stats + seg * 4, st, sizeof(st));
            }
        }
    }
    for (uint32_t r = 0; r < k; ++r) { free(acc[r]); free(wire[r]); }
    free(acc); free(wire); free(tmp_codes);
    return rc;
}

/* ---- one segment's reduce-scatter chain, transport-free ----------------
 * The same arithmetic as orc_ring_allreduce restricted to ONE segment of
 * chunk c: quantization is per segment (allreduce.hpp:326-336), so a
 * segment's final payload depends only on that segment's elements of every
 * worker. Chunk c leaves rank c at hop 0 and visits c+1, ..., c+k-1 = its
 * owner (allreduce.hpp:411-426, owner :431): v = D_c; v = D_{c+t} + deq(Q(v))
 * for t = 1..k-1 (:422); mean = v / (float)k (:435-439); final = Q(mean)
 * (:441-443). D_w = theta_g - theta_l[w] (optim.hpp:108) when theta_g is
 * given, else theta_l[w] is worker w's ring input itself.
 * Outputs: codes (len), cb (256), stats (4: mu sigma lo width) of the final
 * payload; mean_out (len, optional) = the owner's mean before quantization
 * (input of the boundary-margin diagnostic). mode 0 (fp32) returns the fp32
 * mean in mean_out only. Thread-safe (no globals): callers run segments in
 * parallel. */
int orc_segment_chain(const float* theta_g, const float* const* theta_l, uint32_t k, uint32_t c, uint64_t len,
                      int mode, uint8_t* codes, float* cb, double* stats, float* mean_out) {
    if (k == 0 || len == 0) return ORC_ESHAPE;
    float* v = (float*)malloc(len * sizeof(float));
    uint8_t* tc = (uint8_t*)malloc(len);
    float tcb[NBUCKETS];
    int rc = ORC_OK;
    for (uint32_t t = 0; t < k && rc == ORC_OK; ++t) {
        const uint32_t w = (c + t) % k;
        const float* l = theta_l[w];
        if (t > 0 && mode != 0) {  /* what the receiver decodes of the incoming payload */
            rc = orc_quantize(v, len, tc, tcb, NULL);
            if (rc != ORC_OK) break;
            orc_dequantize(tc, tcb, len, v);
        }
        for (uint64_t i = 0; i < len; ++i) {
            const float d = theta_g ? theta_g[i] - l[i] : l[i];
            v[i] = t == 0 ? d : d + v[i];
        }
    }
    if (rc == ORC_OK) {
        const float divisor = (float)k;
        for (uint64_t i = 0; i < len; ++i) v[i] = v[i] / divisor;
        if (mean_out) memcpy(mean_out, v, len * sizeof(float));
        if (mode != 0 && k > 1) rc = orc_quantize(v, len, codes, cb, stats);  /* k == 1: identity (:319) */
    }
    free(v);
    free(tc);
    return rc;
}

/* ---- one outer-sync round for k workers: trainer.hpp:355-382 ----------
 * theta_g: retained (global) params, identical on every worker, updated in
 * place; theta_l[w]: worker w's local params; buf: Nesterov buffer. Every
 * worker ends with the same theta_g/buf, so the update is applied once. */
int orc_outer_sync(float* theta_g, const float* const* theta_l, float* buf, uint32_t k, uint64_t n,
                   uint32_t S, int mode, float lr, float momentum) {
    float** delta = (float**)malloc(k * sizeof(float*));
    for (uint32_t w = 0; w < k; ++w) {
        delta[w] = (float*)malloc((n ? n : 1) * sizeof(float));
        orc_pseudo_gradient(theta_g, theta_l[w], n, delta[w]);
    }
    float* avg = (float*)malloc((n ? n : 1) * sizeof(float));
    int rc = orc_ring_allreduce((const float* const*)delta, k, n, S, mode, avg, NULL, NULL, NULL);
    if (rc == ORC_OK) orc_nesterov(theta_g, avg, buf, n, lr, momentum);
    for (uint32_t w = 0; w < k; ++w) free(delta[w]);
    free(delta); free(avg);
    return rc;
}

/* ---- wire layout of one quantized segment: quant.hpp:102-131 ---------
 * u32 LE count, 256 x f32 LE codebook, count x u8 codes. */
uint64_t orc_encode_quant_chunk(const uint8_t* codes, const float* cb, uint32_t count, uint8_t* out) {
    uint8_t* p = out;
    for (int i = 0; i < 4; ++i) *p++ = (uint8_t)(count >> (8 * i));
    for (int b = 0; b < NBUCKETS; ++b) {
        uint32_t u;
        memcpy(&u, &cb[b], 4);
        for (int i = 0; i < 4; ++i) *p++ = (uint8_t)(u >> (8 * i));
    }
    memcpy(p, codes, count);
    return 4 + 4 * NBUCKETS + (uint64_t)count;
}

/* Returns ORC_OK or ORC_EDECODE (truncated, non-finite codebook entry,
 * count mismatch, trailing bytes). */
int orc_decode_quant_chunk(const uint8_t* buf, uint64_t len, uint8_t* codes, float* cb, uint32_t* count) {
    if (len < 4) return ORC_EDECODE;
    uint32_t c = (uint32_t)buf[0] | ((uint32_t)buf[1] << 8) | ((uint32_t)buf[2] << 16) | ((uint32_t)buf[3] << 24);
    if (len - 4 < 4 * NBUCKETS) return ORC_EDECODE;
    for (int b = 0; b < NBUCKETS; ++b) {
        const uint8_t* q = buf + 4 + 4 * b;
        uint32_t u = (uint32_t)q[0] | ((uint32_t)q[1] << 8) | ((uint32_t)q[2] << 16) | ((uint32_t)q[3] << 24);
        float v;
        memcpy(&v, &u, 4);
        if (!isfinite(v)) return ORC_EDECODE;
        cb[b] = v;
    }
    if (len - 4 - 4 * NBUCKETS != c) return ORC_EDECODE;
    if (codes) memcpy(codes, buf + 4 + 4 * NBUCKETS, c);
    *count = c;
    return ORC_OK;
}
