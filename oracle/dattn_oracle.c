/*
 * dattn_oracle.c -- TEST INFRASTRUCTURE ONLY (see dattn_oracle.h).
 *
 * Plain-C restatement of /root/reference/proj/src/distattention.cpp. Loop
 * orders and operation orders follow the reference line by line so that the
 * fp64 results are bit-identical to the reference's own (pinned by
 * tests/test_oracle.py against tests/golden/, generated from the reference
 * build in oracle/_ref/).
 */
#define _GNU_SOURCE
#include "dattn_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* reference math                                                           */
/* ------------------------------------------------------------------------ */

/* distattention.cpp:20-24 */
static double dot(const double* a, const double* b, int n) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc += a[i] * b[i];
    return acc;
}

double or_effective_scale(int head_dim, double scale) {
    /* distattention.cpp:35-37 */
    return scale > 0.0 ? scale : 1.0 / sqrt((double)head_dim);
}

int64_t or_micro_attention(const double* q, const double* k, const double* v,
                           int64_t seq, int d, double scale,
                           double* m, double* e, double* ma) {
    /* distattention.cpp:108: empty segment -> identity (:59-67) */
    if (seq == 0) {
        *m = -INFINITY;
        *e = 0.0;
        for (int j = 0; j < d; ++j) ma[j] = 0.0;
        return 0;
    }
    const double s = or_effective_scale(d, scale);
    double* logits = (double*)malloc(sizeof(double) * (size_t)seq);
    double mx = -INFINITY;
    /* :110-115 */
    for (int64_t i = 0; i < seq; ++i) {
        logits[i] = s * dot(q, k + i * d, d);
        if (logits[i] > mx) mx = logits[i];
    }
    /* :117-127 */
    double es = 0.0;
    for (int j = 0; j < d; ++j) ma[j] = 0.0;
    for (int64_t i = 0; i < seq; ++i) {
        const double w = exp(logits[i] - mx);
        es += w;
        const double* vr = v + i * d;
        for (int j = 0; j < d; ++j) ma[j] += w * vr[j];
    }
    free(logits);
    *m = mx;
    *e = es;
    return seq;
}

void or_naive_attention(const double* q, const double* k, const double* v,
                        int64_t seq, int d, double scale, double* out) {
    /* distattention.cpp:69-97 */
    const double s = or_effective_scale(d, scale);
    double* logits = (double*)malloc(sizeof(double) * (size_t)seq);
    double m_g = -INFINITY;
    for (int64_t i = 0; i < seq; ++i) {
        logits[i] = s * dot(q, k + i * d, d);
        if (logits[i] > m_g) m_g = logits[i];
    }
    for (int j = 0; j < d; ++j) out[j] = 0.0;
    double denom = 0.0;
    for (int64_t i = 0; i < seq; ++i) {
        const double w = exp(logits[i] - m_g);
        denom += w;
        const double* vr = v + i * d;
        for (int j = 0; j < d; ++j) out[j] += w * vr[j];
    }
    for (int j = 0; j < d; ++j) out[j] /= denom;
    free(logits);
}

void or_combine(double am, double ae, const double* ama, int64_t aseq,
                double bm, double be, const double* bma, int64_t bseq, int d,
                double* om, double* oe, double* oma, int64_t* oseq) {
    /* distattention.cpp:135-136: identity short-circuit returns the other
     * operand exactly. */
    if (aseq == 0) {
        *om = bm; *oe = be; *oseq = bseq;
        if (oma != bma) memcpy(oma, bma, sizeof(double) * (size_t)d);
        return;
    }
    if (bseq == 0) {
        *om = am; *oe = ae; *oseq = aseq;
        if (oma != ama) memcpy(oma, ama, sizeof(double) * (size_t)d);
        return;
    }
    /* :139-147 */
    const double m = am > bm ? am : bm;
    const double wa = exp(am - m);
    const double wb = exp(bm - m);
    *oe = ae * wa + be * wb;
    for (int j = 0; j < d; ++j) oma[j] = ama[j] * wa + bma[j] * wb;
    *om = m;
    *oseq = aseq + bseq;
}

int or_aggregate(int n, const double* m, const double* e, const double* ma,
                 const int64_t* seq_p, int d, double* out) {
    /* distattention.cpp:150-174 */
    if (n <= 0) return -1;
    int64_t total = 0;
    double m_g = -INFINITY;
    for (int i = 0; i < n; ++i) {
        total += seq_p[i];
        if (seq_p[i] != 0 && m[i] > m_g) m_g = m[i];
    }
    if (total < 1) return -1;
    double e_g = 0.0;
    for (int j = 0; j < d; ++j) out[j] = 0.0;
    for (int i = 0; i < n; ++i) {
        if (seq_p[i] == 0) continue;
        const double w = exp(m[i] - m_g);
        e_g += e[i] * w;
        for (int j = 0; j < d; ++j) out[j] += ma[(size_t)i * d + j] * w;
    }
    for (int j = 0; j < d; ++j) out[j] /= e_g;
    return 0;
}

int or_gqa_kv_head(int query_head, int num_q_heads, int num_kv_heads) {
    /* distattention.cpp:176-181 */
    return query_head / (num_q_heads / num_kv_heads);
}

void or_serialize_partial(double m, double e, const double* ma, int d, double* wire) {
    /* distattention.cpp:211-221 */
    wire[0] = m;
    wire[1] = e;
    memcpy(wire + 2, ma, sizeof(double) * (size_t)d);
}

int64_t or_deserialize_seq_p(const double* wire) {
    /* distattention.cpp:235 */
    return (wire[1] == 0.0 && wire[0] == -INFINITY) ? 0 : 1;
}

int64_t or_blocks_for_tokens(int64_t tokens, int block_size_tokens) {
    /* perfmodel.cpp:178-182 */
    return (tokens + block_size_tokens - 1) / block_size_tokens;
}

/* ------------------------------------------------------------------------ */
/* long-double oracle, tests/oracles.hpp:23-56                               */
/* ------------------------------------------------------------------------ */

void or_attention_ld(const double* q, const double* k, const double* v,
                     int64_t seq, int d, double scale, double* out) {
    long double* logits = (long double*)malloc(sizeof(long double) * (size_t)seq);
    long double* acc = (long double*)calloc((size_t)d, sizeof(long double));
    long double mx = -INFINITY;
    for (int64_t i = 0; i < seq; ++i) {
        long double dt = 0.0L;
        for (int j = 0; j < d; ++j) dt += (long double)q[j] * k[i * d + j];
        logits[i] = dt * (long double)scale;
        if (logits[i] > mx) mx = logits[i];
    }
    long double denom = 0.0L;
    for (int64_t i = 0; i < seq; ++i) {
        const long double w = expl(logits[i] - mx);
        denom += w;
        for (int j = 0; j < d; ++j) acc[j] += w * v[i * d + j];
    }
    for (int j = 0; j < d; ++j) out[j] = (double)(acc[j] / denom);
    free(logits);
    free(acc);
}

double or_rel_err(const double* got, const double* ref, int64_t n) {
    double sc = 1e-300, err = 0.0;
    for (int64_t i = 0; i < n; ++i) sc = fmax(sc, fabs(ref[i]));
    for (int64_t i = 0; i < n; ++i) err = fmax(err, fabs(got[i] - ref[i]));
    return err / sc;
}

/* ------------------------------------------------------------------------ */
/* sim::Rng, trace.cpp:14-53 -- std::mt19937_64 restated + the hand-rolled   */
/* transforms.                                                               */
/* ------------------------------------------------------------------------ */

void or_rng_seed(or_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = 312;
}

uint64_t or_rng_next_u64(or_rng* r) {
    static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (r->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (r->mt[i] & UM) | (r->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
        }
        r->idx = 0;
    }
    uint64_t x = r->mt[r->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

double or_rng_uniform01(or_rng* r) {
    /* trace.cpp:18-21 */
    return (double)(or_rng_next_u64(r) >> 11) * 0x1.0p-53;
}

double or_rng_uniform(or_rng* r, double lo, double hi) {
    return lo + (hi - lo) * or_rng_uniform01(r);
}

int64_t or_rng_uniform_int(or_rng* r, int64_t lo, int64_t hi) {
    /* trace.cpp:28-38 */
    const uint64_t span = (uint64_t)(hi - lo) + 1;
    const uint64_t limit = UINT64_MAX - UINT64_MAX % span;
    uint64_t v;
    do {
        v = or_rng_next_u64(r);
    } while (v >= limit);
    return lo + (int64_t)(v % span);
}

double or_rng_normal(or_rng* r) {
    /* trace.cpp:45-53 */
    double u1;
    do {
        u1 = or_rng_uniform01(r);
    } while (u1 <= 0.0);
    const double u2 = or_rng_uniform01(r);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

/* ------------------------------------------------------------------------ */
/* counter-hash generator; the CUDA twin is dattn_fill.cu      */
/* ------------------------------------------------------------------------ */

uint64_t or_splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint16_t or_f32_to_bf16_rne(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    /* inputs are always finite here */
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7FFFu + lsb;
    return (uint16_t)(u >> 16);
}

float or_bf16_to_f32(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

static inline float synth_f32(uint64_t key, uint64_t idx, float amp) {
    const uint32_t u24 = (uint32_t)(or_splitmix64(key ^ idx) >> 40);
    /* volatile keeps the product a single IEEE fp32 multiply (no contraction,
     * no excess precision) so it matches __fmul_rn on the device. */
    volatile float a = (float)((int32_t)u24 - (1 << 23));
    volatile float s = amp * 0x1.0p-23f;
    volatile float r = a * s;
    return r;
}

static inline uint64_t stream_key(uint64_t seed, int tensor) {
    return or_splitmix64(seed ^ ((uint64_t)tensor * 0xD1B54A32D192ED03ULL));
}

static inline uint64_t elem_index(uint32_t seq, uint32_t head, uint32_t token, uint32_t dim) {
    return ((uint64_t)seq << 40) | ((uint64_t)(head & 0xFFu) << 32) |
           ((uint64_t)(token & 0xFFFFFFu) << 8) | (uint64_t)(dim & 0xFFu);
}

static inline double round_to(float x, int dtype) {
    if (dtype == OR_DT_BF16) return (double)or_bf16_to_f32(or_f32_to_bf16_rne(x));
    return (double)x;
}

double or_synth_value(uint64_t seed, int tensor, uint32_t seq, uint32_t head,
                      uint32_t token, uint32_t dim, float amp, int dtype) {
    return round_to(synth_f32(stream_key(seed, tensor), elem_index(seq, head, token, dim), amp),
                    dtype);
}

void or_synth_kv(uint64_t seed, uint32_t seq, uint32_t head, uint32_t tok0,
                 int64_t n, int d, float amp_k, float amp_v, int dtype,
                 double* k, double* v) {
    const uint64_t kk = stream_key(seed, OR_T_KEY), kv = stream_key(seed, OR_T_VALUE);
    for (int64_t t = 0; t < n; ++t)
        for (int j = 0; j < d; ++j) {
            const uint64_t ix = elem_index(seq, head, (uint32_t)(tok0 + t), (uint32_t)j);
            k[t * d + j] = round_to(synth_f32(kk, ix, amp_k), dtype);
            v[t * d + j] = round_to(synth_f32(kv, ix, amp_v), dtype);
        }
}

void or_synth_q(uint64_t seed, uint32_t b, uint32_t h, int d, float amp_q,
                int dtype, double* q) {
    const uint64_t kq = stream_key(seed, OR_T_QUERY);
    for (int j = 0; j < d; ++j)
        q[j] = round_to(synth_f32(kq, elem_index(b, h, 0, (uint32_t)j), amp_q), dtype);
}

/* ------------------------------------------------------------------------ */
/* batched decode (multi_head_attention per request), pthreads               */
/* ------------------------------------------------------------------------ */

typedef struct {
    uint64_t seed;
    int B, Hq, Hkv, d, dtype;
    const int64_t* lo;
    const int64_t* hi;
    const uint32_t* seq_ids;
    double scale;
    float aq, ak, av;
    int64_t seg_tokens;
    double* out;
    double* m_out;
    double* e_out;
    const unsigned char* sel; /* [B][Hkv]: compute only selected (b, kv head) items; NULL = all */
    int next; /* atomic work counter over (b, kv head) */
} batch_job;

static void* batch_worker(void* arg) {
    batch_job* J = (batch_job*)arg;
    const int d = J->d;
    const int group = J->Hq / J->Hkv;
    double* q = (double*)malloc(sizeof(double) * (size_t)d);
    double* ma = (double*)malloc(sizeof(double) * (size_t)d);
    for (;;) {
        const int w = __atomic_fetch_add(&J->next, 1, __ATOMIC_RELAXED);
        if (w >= J->B * J->Hkv) break;
        const int b = w / J->Hkv, kvh = w % J->Hkv;
        if (J->sel && !J->sel[w]) continue;
        const int64_t lo = J->lo[b], n = J->hi[b] - J->lo[b];
        double* k = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1) * d);
        double* v = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1) * d);
        or_synth_kv(J->seed, J->seq_ids[b], (uint32_t)kvh, (uint32_t)lo, n, d, J->ak, J->av,
                    J->dtype, k, v);
        const int64_t seg = J->seg_tokens > 0 ? J->seg_tokens : (n > 0 ? n : 1);
        const int nseg = n > 0 ? (int)((n + seg - 1) / seg) : 1;
        double* pm = (double*)malloc(sizeof(double) * nseg);
        double* pe = (double*)malloc(sizeof(double) * nseg);
        int64_t* ps = (int64_t*)malloc(sizeof(int64_t) * nseg);
        double* pma = (double*)malloc(sizeof(double) * (size_t)nseg * d);
        for (int gh = 0; gh < group; ++gh) {
            const int h = kvh * group + gh; /* gqa_kv_head(h) == kvh */
            or_synth_q(J->seed, (uint32_t)b, (uint32_t)h, d, J->aq, J->dtype, q);
            for (int s = 0; s < nseg; ++s) {
                const int64_t a = (int64_t)s * seg;
                const int64_t len = (n - a) < seg ? (n - a) : seg;
                ps[s] = or_micro_attention(q, k + a * d, v + a * d, len > 0 ? len : 0, d,
                                           J->scale, &pm[s], &pe[s], pma + (size_t)s * d);
            }
            double* o = J->out + ((size_t)b * J->Hq + h) * d;
            if (or_aggregate(nseg, pm, pe, pma, ps, d, o) != 0)
                for (int j = 0; j < d; ++j) o[j] = 0.0; /* empty range */
            if (J->m_out || J->e_out) {
                double m_g = -INFINITY, e_g = 0.0;
                for (int s = 0; s < nseg; ++s)
                    if (ps[s] && pm[s] > m_g) m_g = pm[s];
                for (int s = 0; s < nseg; ++s)
                    if (ps[s]) e_g += pe[s] * exp(pm[s] - m_g);
                if (J->m_out) J->m_out[(size_t)b * J->Hq + h] = m_g;
                if (J->e_out) J->e_out[(size_t)b * J->Hq + h] = e_g;
            }
        }
        free(pm); free(pe); free(ps); free(pma);
        free(k); free(v);
    }
    free(q);
    free(ma);
    return NULL;
}

static int run_batch(batch_job* J, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    for (int i = 0; i < threads; ++i) pthread_create(&tid[i], NULL, batch_worker, J);
    for (int i = 0; i < threads; ++i) pthread_join(tid[i], NULL);
    return 0;
}

int or_decode_ranges(uint64_t seed, int B, const int64_t* tok_lo, const int64_t* tok_hi,
                     const uint32_t* seq_ids, int Hq, int Hkv, int d, double scale,
                     int dtype, float amp_q, float amp_k, float amp_v,
                     int threads, double* out, double* m_out, double* e_out) {
    return or_decode_ranges_sel(seed, B, tok_lo, tok_hi, seq_ids, Hq, Hkv, d, scale, dtype, amp_q,
                                amp_k, amp_v, NULL, threads, out, m_out, e_out);
}

/* As or_decode_ranges, computing only the (request, kv head) pairs with
 * sel[b * Hkv + kvh] != 0 (all q heads of the group); the other outputs are
 * left untouched. For sampled parity checks of large workloads. */
int or_decode_ranges_sel(uint64_t seed, int B, const int64_t* tok_lo, const int64_t* tok_hi,
                         const uint32_t* seq_ids, int Hq, int Hkv, int d, double scale,
                         int dtype, float amp_q, float amp_k, float amp_v,
                         const unsigned char* sel, int threads, double* out, double* m_out,
                         double* e_out) {
    batch_job J = {seed, B, Hq, Hkv, d, dtype, tok_lo, tok_hi, seq_ids, scale,
                   amp_q, amp_k, amp_v, 0, out, m_out, e_out, sel, 0};
    return run_batch(&J, threads);
}

int or_decode_batch(uint64_t seed, int B, const int64_t* lens, const uint32_t* seq_ids,
                    int Hq, int Hkv, int d, double scale, int dtype,
                    float amp_q, float amp_k, float amp_v,
                    int64_t seg_tokens, int threads, double* out) {
    int64_t* lo = (int64_t*)calloc((size_t)B, sizeof(int64_t));
    batch_job J = {seed, B, Hq, Hkv, d, dtype, lo, lens, seq_ids, scale,
                   amp_q, amp_k, amp_v, seg_tokens, out, NULL, NULL, NULL, 0};
    run_batch(&J, threads);
    free(lo);
    return 0;
}
