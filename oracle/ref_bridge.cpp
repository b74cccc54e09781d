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
// (perfmodel.cpp, config.cpp), (4) pin the GPU store's page ledger to the
// reference's RManager and blocks_for_tokens (controlplane.cpp:38-79,
// perfmodel.cpp:178-182) and (5) produce config 5's placement with the
// reference's own dispatch + rManager heartbeats + gManager plan_round +
// execute_move_sync (simengine.cpp:252-257, controlplane.cpp:412-485,
// scheduler.cpp:483-493, controlplane.cpp:518-540), (6) run the reference
// cluster simulator (simengine.cpp) to pin the overflow-borrowing slot rule
// (ensure_slot, simengine.cpp:318-354) of the B200 block ledger.
#include "kvsched/common.hpp"
#include "kvsched/config.hpp"
#include "kvsched/controlplane.hpp"
#include "kvsched/distattention.hpp"
#include "kvsched/perfmodel.hpp"
#include "kvsched/simengine.hpp"
#include "kvsched/trace.hpp"
#include "kvsched/verify.hpp"

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <unistd.h>
#include <memory>
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

// The reference simulator (run_simulation, simengine.cpp) on a hand-made
// trace: n_inst instances with capacity caps[i] blocks each, the default
// model (config.cpp:71-87), policy 0 infinite / 1 strawman / 2 static, and
// requests (arrival[i], prompt[i], output[i]) with ids 0..n_req-1. *log_out
// = the JSONL event log without "msg" lines (admit / prefill_done / borrow /
// step / complete ...),
// malloc'ed, freed with ref_string_free.
int ref_sim_log(int n_inst, const int64_t* caps, int policy, int n_req, const double* arrival,
                const int64_t* prompt, const int64_t* output, double horizon_s, char** log_out) {
    return guarded([&] {
        sim::ClusterConfig cc = sim::default_cluster_config(n_inst, caps[0]);
        for (int i = 0; i < n_inst; ++i) cc.instances[i].capacity_blocks = caps[i];
        cc.policy = policy == 0 ? sim::Policy::infinite
                  : policy == 1 ? sim::Policy::strawman : sim::Policy::static_alloc;
        std::vector<sim::TraceRequest> trace(n_req);
        for (int i = 0; i < n_req; ++i) {
            trace[i].req_id = i;
            trace[i].arrival_s = arrival[i];
            trace[i].prompt_tokens = prompt[i];
            trace[i].output_tokens = output[i];
        }
        char path[] = "/tmp/ref_sim_log_XXXXXX";
        const int fd = mkstemp(path);
        if (fd < 0) throw std::runtime_error("mkstemp failed");
        close(fd);
        sim::RunOptions opt;
        opt.horizon_s = horizon_s;
        opt.event_log_path = path;
        (void)sim::run_simulation(cc, trace, opt);
        // keep every event but the control-plane message traffic ("msg")
        std::ifstream f(path, std::ios::binary);
        std::string t, line;
        while (std::getline(f, line))
            if (line.find("\"ev\":\"msg\"") == std::string::npos) t += line + "\n";
        std::remove(path);
        *log_out = static_cast<char*>(std::malloc(t.size() + 1));
        std::memcpy(*log_out, t.c_str(), t.size() + 1);
    });
}


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

// perf::blocks_for_tokens (perfmodel.cpp:178-182) for a shape with the given
// block size (every other shape field is set to a valid dummy).
int ref_blocks_for_tokens(int64_t tokens, int block_size_tokens, int64_t* out) {
    return guarded([&] {
        perf::ModelShape shape;
        shape.n_layers = 1;
        shape.workload_per_token = 1.0;
        shape.attn_work_per_ctx_token = 1.0;
        shape.kv_bytes_per_token = 1.0;
        shape.block_size_tokens = block_size_tokens;
        *out = perf::blocks_for_tokens(tokens, shape);
    });
}

// Drive one RManager (controlplane.cpp:38-79) through a ledger trace.
// op[i]: 0 alloc_local(req[i], n[i]), 1 alloc_hosted(req[i], home = n2[i], n[i]),
// 2 free_request(req[i]). Per op: result[i] = 1/0 for the allocations, the
// freed block count for free_request; used[i], free_[i] after the op and
// local[i] = local_blocks(req[i]).
int ref_rmanager_trace(int64_t capacity, int n_ops, const int* op, const int64_t* req, const int64_t* n,
                       const int* n2, int64_t* result, int64_t* used, int64_t* free_, int64_t* local) {
    return guarded([&] {
        ctrl::RManager rm(0, capacity);
        for (int i = 0; i < n_ops; ++i) {
            if (op[i] == 0)
                result[i] = rm.alloc_local(req[i], n[i]) ? 1 : 0;
            else if (op[i] == 1)
                result[i] = rm.alloc_hosted(req[i], n2[i], n[i]) ? 1 : 0;
            else
                result[i] = rm.free_request(req[i]);
            used[i] = rm.used_blocks();
            free_[i] = rm.free_blocks();
            local[i] = rm.local_blocks(req[i]);
        }
    });
}

// Config-5 placement from the reference control plane itself:
//  1. dispatch: requests in order, each homed on the instance with the most
//     free blocks, ties to the lowest id (simengine.cpp:252-257), blocks via
//     RManager::alloc_local (controlplane.cpp:38-44);
//  2. rManager heartbeats -> GManager (epoch recovery, then heartbeats carrying
//     batch = home requests and the debtor queue `queued` at the home of
//     request 0), controlplane.cpp:109-142, 374-410, 500-516;
//  3. `rounds` planning rounds: GManager::plan (snapshots + plan_round,
//     controlplane.cpp:412-485) and every MoveKvCache executed with
//     execute_move_sync (controlplane.cpp:518-540); between rounds the freed
//     blocks admit queued requests of expected_new_request_tokens each
//     (derive_feasible_batch's rule, scheduler.cpp:62-80), which take their
//     prompt blocks at the home, and `now` advances by the planning period
//     (config.hpp:29-39).
// Model: default_cluster_config(n_inst, capacity) (config.cpp:71-87) and the
// default SchedulerConfig (scheduler.hpp:52-58).
// Outputs: home[n_req]; blocks[n_req * n_inst] = blocks of request r held on
// instance i (local on the home, hosted elsewhere); moves[k*6 .. +5] =
// (round, req, src, dst, planned blocks, moved blocks) and gains[k], k <
// max_moves; *n_moves.
int ref_cfg5_place(int n_inst, int64_t capacity, int64_t queued, int rounds, int n_req,
                   const int64_t* tokens, int* home, int64_t* blocks, int max_moves, int64_t* moves,
                   double* gains, int* n_moves) {
    return guarded([&] {
        const sim::ClusterConfig cc = sim::default_cluster_config(n_inst, capacity);
        const int bs = cc.shape.block_size_tokens;
        std::vector<std::unique_ptr<ctrl::RManager>> rms;
        std::vector<ctrl::RManager*> raw;
        for (int i = 0; i < n_inst; ++i) {
            rms.push_back(std::make_unique<ctrl::RManager>(i, capacity));
            raw.push_back(rms.back().get());
        }
        std::vector<int64_t> batch(n_inst, 0);
        for (int r = 0; r < n_req; ++r) {
            int best = 0;
            for (int i = 1; i < n_inst; ++i)
                if (rms[i]->free_blocks() > rms[best]->free_blocks()) best = i;
            const int64_t need = perf::blocks_for_tokens(tokens[r], cc.shape);
            if (!rms[best]->alloc_local(r, need)) throw ContractError("request does not fit its dispatch target");
            home[r] = best;
            batch[best]++;
        }
        const int debtor = n_req > 0 ? home[0] : 0;
        int64_t next_req = n_req;  // ids of admitted (queued) requests
        ctrl::GManager gm(1);
        double now = 0.0;
        ctrl::gmanager_epoch_recover(gm, raw, now);
        auto heartbeat_all = [&](int64_t q) {
            for (int i = 0; i < n_inst; ++i) {
                ctrl::Envelope hb = rms[i]->make_heartbeat(now, batch[i], i == debtor ? q : 0);
                ctrl::Envelope ack = gm.on_heartbeat(std::get<ctrl::Heartbeat>(hb.msg), now);
                rms[i]->on_message(ack, now);
            }
        };
        heartbeat_all(queued);
        const sched::ModelCtx ctx{cc.shape, cc.f, cc.g};
        int k = 0;
        for (int round = 0; round < rounds; ++round) {
            auto out = gm.plan(now, cc.sched, ctx);
            std::vector<sched::MoveDirective> all = out.plan.reclaims;
            all.insert(all.end(), out.plan.moves.begin(), out.plan.moves.end());
            int64_t freed_at_debtor = 0;
            for (const auto& d : all) {
                const ctrl::MoveKvCache mv{d.req_id, d.num_blocks, d.dst_instance};
                const ctrl::MoveResult res =
                    ctrl::execute_move_sync(*rms[d.src_instance], *rms[d.dst_instance], mv, now, bs);
                if (d.src_instance == debtor) freed_at_debtor += res.moved_blocks;
                if (k < max_moves) {
                    int64_t* m = moves + 6 * k;
                    m[0] = round; m[1] = d.req_id; m[2] = d.src_instance; m[3] = d.dst_instance;
                    m[4] = d.num_blocks; m[5] = res.moved_blocks;
                    gains[k] = d.est_gain;
                }
                ++k;
            }
            // the freed blocks admit queued requests (derive_feasible_batch,
            // scheduler.cpp:62-80); they take their prompt blocks at the home
            // (try_admit, simengine.cpp:262-268), so the next round's reclaim
            // pass finds no free space to pull the lent blocks back into
            const int64_t admit = std::min<int64_t>(
                queued, (freed_at_debtor * bs) / cc.sched.expected_new_request_tokens);
            const int64_t prompt = perf::blocks_for_tokens(cc.sched.expected_new_request_tokens, cc.shape);
            for (int64_t a = 0; a < admit; ++a) {
                if (!rms[debtor]->alloc_local(next_req, prompt)) break;
                ++next_req;
                ++batch[debtor];
                --queued;
            }
            now += cc.ctrl.planning_period_s;
            heartbeat_all(queued);
        }
        *n_moves = k;
        for (int r = 0; r < n_req; ++r)
            for (int i = 0; i < n_inst; ++i)
                blocks[static_cast<size_t>(r) * n_inst + i] =
                    i == home[r] ? rms[i]->local_blocks(r) : rms[i]->hosted_blocks(r, home[r]);
    });
}

} // extern "C"
