// ref_bridge.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNMODIFIED reference implementation
// (kvsched::attn in /root/reference/proj/src/distattention.cpp, verify.cpp,
// trace.cpp), compiled together by oracle/Makefile into
// oracle/_ref/libkvsched_ref.so. Used to (1) pin the C restatement in
// dattn_oracle.c (tests/golden/make_golden.py), (2) time the reference CPU
// path for bench.py --impl reference / cpu_baseline and (3) check that a
// ctx_rate_curve measured on the B200 (tools/calibrate_ctx_curve.py, SURVEY
// §8f row 4) is accepted by the reference's own config parser and perf model
// (perfmodel.cpp, config.cpp).
#include "kvsched/common.hpp"
#include "kvsched/config.hpp"
#include "kvsched/distattention.hpp"
#include "kvsched/perfmodel.hpp"
#include "kvsched/trace.hpp"
#include "kvsched/verify.hpp"

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

using namespace kvsched;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ContractError& e) {
        g_err = e.what();
        return 3;
    } catch (const InputError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

attn::KVSegment make_seg(const double* k, const double* v, int64_t seq, int d) {
    attn::KVSegment s;
    s.seq_p = seq;
    s.head_dim = d;
    s.keys.assign(k, k + seq * d);
    s.values.assign(v, v + seq * d);
    return s;
}
} // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_micro_attention(const double* q, const double* k, const double* v, int64_t seq,
                        int d, double scale, double* m, double* e, double* ma,
                        int64_t* seq_p) {
    return guarded([&] {
        attn::AttentionConfig cfg{d, 1, 1, scale};
        std::vector<double> qv(q, q + d);
        auto p = attn::compute_micro_attention(qv, make_seg(k, v, seq, d), cfg);
        *m = p.m;
        *e = p.e;
        std::memcpy(ma, p.ma.data(), sizeof(double) * d);
        *seq_p = p.seq_p;
    });
}

int ref_naive_attention(const double* q, const double* k, const double* v, int64_t seq,
                        int d, double scale, double* out) {
    return guarded([&] {
        attn::AttentionConfig cfg{d, 1, 1, scale};
        std::vector<double> qv(q, q + d);
        auto o = attn::naive_attention(qv, make_seg(k, v, seq, d), cfg);
        std::memcpy(out, o.data(), sizeof(double) * d);
    });
}

int ref_combine(double am, double ae, const double* ama, int64_t aseq, double bm,
                double be, const double* bma, int64_t bseq, int d, double* om, double* oe,
                double* oma, int64_t* oseq) {
    return guarded([&] {
        attn::AttentionPartial a, b;
        a.m = am; a.e = ae; a.ma.assign(ama, ama + d); a.seq_p = aseq;
        b.m = bm; b.e = be; b.ma.assign(bma, bma + d); b.seq_p = bseq;
        auto o = attn::combine_partials(a, b);
        *om = o.m;
        *oe = o.e;
        std::memcpy(oma, o.ma.data(), sizeof(double) * d);
        *oseq = o.seq_p;
    });
}

int ref_aggregate(int n, const double* m, const double* e, const double* ma,
                  const int64_t* seq_p, int d, double* out) {
    return guarded([&] {
        std::vector<attn::AttentionPartial> parts(n);
        for (int i = 0; i < n; ++i) {
            parts[i].m = m[i];
            parts[i].e = e[i];
            parts[i].ma.assign(ma + (size_t)i * d, ma + (size_t)(i + 1) * d);
            parts[i].seq_p = seq_p[i];
        }
        auto o = attn::aggregate_partials(parts);
        std::memcpy(out, o.data(), sizeof(double) * d);
    });
}

int ref_gqa_kv_head(int h, int hq, int hkv, int* out) {
    return guarded([&] {
        attn::AttentionConfig cfg{8, hq, hkv, 0.0};
        *out = attn::gqa_kv_head(h, cfg);
    });
}

int ref_serialize_partial(double m, double e, const double* ma, int d, unsigned char* wire,
                          int64_t* nbytes) {
    return guarded([&] {
        attn::AttentionPartial p;
        p.m = m; p.e = e; p.ma.assign(ma, ma + d); p.seq_p = 1;
        auto b = attn::serialize_partial(p);
        std::memcpy(wire, b.data(), b.size());
        *nbytes = (int64_t)b.size();
    });
}

int ref_deserialize_partial(const unsigned char* wire, int64_t nbytes, int d, double* m,
                            double* e, double* ma, int64_t* seq_p) {
    return guarded([&] {
        std::vector<std::byte> b(nbytes);
        std::memcpy(b.data(), wire, nbytes);
        auto p = attn::deserialize_partial(b, d);
        *m = p.m; *e = p.e; *seq_p = p.seq_p;
        std::memcpy(ma, p.ma.data(), sizeof(double) * d);
    });
}

// Multi-head attention over per-kv-head cut lists. k/v are [hkv][seq][d];
// cuts[h] holds ncuts[h]+1 ascending boundaries (cuts_flat is their concat).
int ref_multi_head_attention(const double* queries, const double* k, const double* v,
                             int64_t seq, int hq, int hkv, int d, double scale,
                             const int64_t* cuts_flat, const int* ncuts, double* out) {
    return guarded([&] {
        attn::AttentionConfig cfg{d, hq, hkv, scale};
        std::vector<std::vector<attn::KVSegment>> segs(hkv);
        size_t off = 0;
        for (int h = 0; h < hkv; ++h) {
            const double* kh = k + (size_t)h * seq * d;
            const double* vh = v + (size_t)h * seq * d;
            for (int s = 0; s < ncuts[h]; ++s) {
                const int64_t a = cuts_flat[off + s], b = cuts_flat[off + s + 1];
                segs[h].push_back(make_seg(kh + a * d, vh + a * d, b - a, d));
            }
            off += ncuts[h] + 1;
        }
        std::vector<double> q(queries, queries + (size_t)hq * d);
        auto o = attn::multi_head_attention(q, segs, cfg);
        std::memcpy(out, o.data(), sizeof(double) * o.size());
    });
}

int ref_verify_attention(int trials, uint64_t seed, double tol, double* max_err,
                         double* mean_err, int* pass) {
    return guarded([&] {
        attn::VerifyConfig c;
        c.trials = trials;
        c.seed = seed;
        c.tolerance = tol;
        auto r = attn::verify_attention_equivalence(c);
        *max_err = r.max_rel_err;
        *mean_err = r.mean_rel_err;
        *pass = r.pass ? 1 : 0;
    });
}

int ref_rng_draws(uint64_t seed, int n, uint64_t* u64, double* u01, double* normal,
                  int64_t* ints, int64_t lo, int64_t hi) {
    return guarded([&] {
        sim::Rng a(seed), b(seed + 1), c(seed + 2), e(seed + 3);
        for (int i = 0; i < n; ++i) {
            u64[i] = a.next_u64();
            u01[i] = b.uniform01();
            normal[i] = c.normal();
            ints[i] = e.uniform_int(lo, hi);
        }
    });
}

// Timed reference decode: the caller supplies per-(request, kv head) fp64 K/V
// rows (already generated; generation is outside the timed region) and this
// runs kvsched::attn::multi_head_attention per (request, kv head) group with
// `threads` std::threads. Segments are the request's rBlocks of seg_tokens.
// kv_ptrs[2*w], kv_ptrs[2*w+1] are K and V of work item w = r*hkv + h with
// lens[r] rows; queries [B][hq][d]. Returns wall seconds in *seconds.
int ref_decode_timed(int B, const int64_t* lens, const double* const* kv_ptrs,
                     const double* queries, int hq, int hkv, int d, double scale,
                     int64_t seg_tokens, int threads, double* out, double* seconds) {
    return guarded([&] {
        const int group = hq / hkv;
        const int W = B * hkv;
        // Build the reference's segment objects first (input marshalling).
        std::vector<std::vector<std::vector<attn::KVSegment>>> segs(W);
        for (int w = 0; w < W; ++w) {
            const int r = w / hkv;
            const int64_t n = lens[r];
            const int64_t seg = seg_tokens > 0 ? seg_tokens : (n > 0 ? n : 1);
            segs[w].resize(1);
            for (int64_t a = 0; a < n; a += seg) {
                const int64_t len = std::min<int64_t>(seg, n - a);
                segs[w][0].push_back(make_seg(kv_ptrs[2 * w] + a * d,
                                              kv_ptrs[2 * w + 1] + a * d, len, d));
            }
        }
        attn::AttentionConfig cfg{d, group, 1, scale};
        std::atomic<int> next{0};
        auto worker = [&] {
            for (;;) {
                const int w = next.fetch_add(1);
                if (w >= W) break;
                const int r = w / hkv, h = w % hkv;
                const double* qp = queries + ((size_t)r * hq + (size_t)h * group) * d;
                std::vector<double> q(qp, qp + (size_t)group * d);
                auto o = attn::multi_head_attention(q, segs[w], cfg);
                std::memcpy(out + ((size_t)r * hq + (size_t)h * group) * d, o.data(),
                            sizeof(double) * o.size());
            }
        };
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int i = 0; i < std::max(1, threads); ++i) pool.emplace_back(worker);
        for (auto& t : pool) t.join();
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

// The reference's default cluster config as JSON (config.cpp:71-87 +
// format_cluster_config); *out is malloc'ed, freed with ref_string_free.
int ref_default_config_json(int n_instances, int64_t capacity_blocks, char** out) {
    return guarded([&] {
        const std::string j = sim::format_cluster_config(sim::default_cluster_config(n_instances, capacity_blocks));
        *out = static_cast<char*>(std::malloc(j.size() + 1));
        std::memcpy(*out, j.c_str(), j.size() + 1);
    });
}

void ref_string_free(char* p) { std::free(p); }

// Parse a cluster config with the reference parser (parse_cluster_config,
// config.cpp:111-183, which validates every curve) and evaluate its
// ctx_rate_curve g and the perf model's layer_time (perfmodel.cpp:105-113)
// for a load of `batch` requests of the given context lengths.
int ref_config_eval(const char* text, int n_x, const double* x, double* g_out, int64_t batch,
                    const int64_t* ctx_lengths, double* layer_time_out, int* n_layers_out) {
    return guarded([&] {
        const sim::ClusterConfig c = sim::parse_cluster_config(text);
        for (int i = 0; i < n_x; ++i) g_out[i] = c.g.eval(x[i]);
        perf::InstanceLoad load;
        load.batch = batch;
        load.ctx_lengths.assign(ctx_lengths, ctx_lengths + batch);
        *layer_time_out = perf::layer_time(load, c.shape, c.f, c.g);
        *n_layers_out = c.shape.n_layers;
    });
}

} // extern "C"
