// dattn_ledger.cpp -- the cluster block ledger and the decode loop's slot rule
// (include/dattn.h "block placement ledger").
//
// Instance: the RManager block ledger (controlplane.cpp:38-79) -- capacity,
// used, home blocks per request, hosted blocks per (request, home). No
// reservations: the decode loop moves no blocks through the planner, so
// free = capacity - used (controlplane.hpp:130 with reserved_blocks() = 0).
// Request: home, context length and the allocation history (instance, blocks)
// in block order, which tells every instance which token positions it holds.
// ensure_slot restates simengine.cpp:318-354 step for step.
#include <map>
#include <utility>
#include <vector>

#include "dattn_engine.h"

using namespace dattn;

namespace {

struct Instance {
    int64_t capacity = 0, used = 0;
    std::map<int64_t, int64_t> home;                      // home_blocks_
    std::map<std::pair<int64_t, int>, int64_t> hosted;    // hosted_[(req, home)]
    int64_t free_blocks() const { return capacity - used; }
    int64_t hosted_blocks(int64_t req, int home_inst) const {
        auto it = hosted.find({req, home_inst});
        return it == hosted.end() ? 0 : it->second;
    }
    int64_t local_blocks(int64_t req) const {
        auto it = home.find(req);
        return it == home.end() ? 0 : it->second;
    }
};

struct Request {
    int home = 0;
    int64_t ctx = 0;
    std::vector<std::pair<int, int64_t>> segs;  // (instance, blocks), block order
};

}  // namespace

struct dattn_ledger {
    int bs = 16;
    std::vector<Instance> inst;
    std::map<int64_t, Request> reqs;
    int64_t borrowed = 0;

    int64_t blocks_for(int64_t tokens) const { return (tokens + bs - 1) / bs; }  // perfmodel.cpp:178-182

    Request& req(int64_t id) {
        auto it = reqs.find(id);
        if (it == reqs.end()) throw Error(DATTN_ERR_CONTRACT, "ledger: request is not live");
        return it->second;
    }
    const Request& req(int64_t id) const { return const_cast<dattn_ledger*>(this)->req(id); }

    void record(Request& r, int where, int64_t n) {
        if (!r.segs.empty() && r.segs.back().first == where) r.segs.back().second += n;
        else r.segs.emplace_back(where, n);
    }
    // RManager::alloc_local / alloc_hosted (controlplane.cpp:38-53)
    bool alloc(int64_t id, Request& r, int where, int64_t n) {
        Instance& j = inst[where];
        if (n > j.free_blocks()) return false;
        if (where == r.home) j.home[id] += n;
        else j.hosted[{id, r.home}] += n;
        j.used += n;
        record(r, where, n);
        return true;
    }
    int64_t hosted_elsewhere(int64_t id, const Request& r) const {  // simengine.cpp:186-191
        int64_t t = 0;
        for (size_t j = 0; j < inst.size(); ++j)
            if (static_cast<int>(j) != r.home) t += inst[j].hosted_blocks(id, r.home);
        return t;
    }
    int64_t held(int64_t id, const Request& r) const {  // simengine.cpp:193-195
        return inst[r.home].local_blocks(id) + hosted_elsewhere(id, r);
    }
    // is_borrowing (simengine.cpp:226-232): a live request homed at j holds
    // blocks elsewhere (only admitted requests -- prefilling or running --
    // hold blocks, so "live" is the reference's running + prefilling)
    bool is_borrowing(int j) const {
        for (const auto& [id, r] : reqs)
            if (r.home == j && hosted_elsewhere(id, r) > 0) return true;
        return false;
    }
    int where_is(const Request& r, int64_t pos) const {
        int64_t b = pos / bs;
        for (const auto& [w, n] : r.segs) {
            if (b < n) return w;
            b -= n;
        }
        return -1;
    }

    int ensure_slot(int64_t id, bool borrow) {
        Request& r = req(id);
        const int64_t need = blocks_for(r.ctx + 1) - held(id, r);
        if (need <= 0) return where_is(r, r.ctx);
        if (alloc(id, r, r.home, need)) return r.home;
        if (!borrow) return -1;  // Policy::static_alloc
        int host = -1;
        auto consider = [&](int j, bool require_clean) {
            if (j == r.home || inst[j].free_blocks() < need) return;
            if (require_clean && is_borrowing(j)) return;
            if (host < 0) {
                host = j;
                return;
            }
            const bool j_has = inst[j].hosted_blocks(id, r.home) > 0;
            const bool h_has = inst[host].hosted_blocks(id, r.home) > 0;
            if (j_has != h_has) {
                if (j_has) host = j;
                return;
            }
            if (inst[j].free_blocks() > inst[host].free_blocks()) host = j;
        };
        const int n = static_cast<int>(inst.size());
        for (int j = 0; j < n; ++j) consider(j, true);
        if (host < 0)
            for (int j = 0; j < n; ++j) consider(j, false);
        if (host < 0) return -1;
        if (!alloc(id, r, host, need)) throw Error(DATTN_ERR_INTERNAL, "ledger: host had free space");
        borrowed += need;
        return where_is(r, r.ctx);
    }

    // RManager::free_request (controlplane.cpp:55-79) on every instance
    int64_t release(int64_t id) {
        const Request& r = req(id);
        int64_t freed = 0;
        for (auto& j : inst) {
            if (auto it = j.home.find(id); it != j.home.end()) {
                freed += it->second;
                j.used -= it->second;
                j.home.erase(it);
            }
            if (auto it = j.hosted.find({id, r.home}); it != j.hosted.end()) {
                freed += it->second;
                j.used -= it->second;
                j.hosted.erase(it);
            }
        }
        reqs.erase(id);
        return freed;
    }
};

extern "C" {

dattn_status dattn_ledger_create(int n_instances, const int64_t* capacity_blocks, int block_tokens,
                                 dattn_ledger** out) {
    return guarded([&] {
        REQUIRE_ARG(capacity_blocks && out, "null argument");
        if (n_instances < 1 || block_tokens < 1)
            throw Error(DATTN_ERR_CONTRACT, "ledger: need >= 1 instance and block_tokens >= 1");
        auto* l = new dattn_ledger;
        l->bs = block_tokens;
        l->inst.resize(n_instances);
        for (int i = 0; i < n_instances; ++i) {
            if (capacity_blocks[i] < 0) {
                delete l;
                throw Error(DATTN_ERR_CONTRACT, "ledger: negative capacity");
            }
            l->inst[i].capacity = capacity_blocks[i];
        }
        *out = l;
    });
}

void dattn_ledger_destroy(dattn_ledger* l) { delete l; }

dattn_status dattn_ledger_admit(dattn_ledger* l, int64_t req, int home, int64_t tokens, int* admitted) {
    return guarded([&] {
        REQUIRE_ARG(l && admitted, "null argument");
        if (home < 0 || home >= static_cast<int>(l->inst.size()))
            throw Error(DATTN_ERR_CONTRACT, "ledger: home instance out of range");
        if (tokens < 1) throw Error(DATTN_ERR_CONTRACT, "allocation must be >= 1 block");
        if (l->reqs.count(req)) throw Error(DATTN_ERR_CONTRACT, "ledger: request already admitted");
        Request r;
        r.home = home;
        r.ctx = tokens;
        const int64_t n = l->blocks_for(tokens);
        if (n > l->inst[home].free_blocks()) {
            *admitted = 0;
            return;
        }
        l->alloc(req, r, home, n);
        l->reqs.emplace(req, std::move(r));
        *admitted = 1;
    });
}

dattn_status dattn_ledger_ensure_slot(dattn_ledger* l, int64_t req, int allow_borrow, int* instance) {
    return guarded([&] {
        REQUIRE_ARG(l && instance, "null argument");
        *instance = l->ensure_slot(req, allow_borrow != 0);
    });
}

dattn_status dattn_ledger_advance(dattn_ledger* l, int64_t req, int64_t tokens) {
    return guarded([&] {
        REQUIRE_ARG(l, "null argument");
        Request& r = l->req(req);
        if (tokens < 0) throw Error(DATTN_ERR_CONTRACT, "ledger: negative advance");
        if (l->blocks_for(r.ctx + tokens) > l->held(req, r))
            throw Error(DATTN_ERR_CAPACITY, "ledger: advance past the request's blocks (call ensure_slot first)");
        r.ctx += tokens;
    });
}

dattn_status dattn_ledger_step(dattn_ledger* l, int n, const int64_t* reqs, int allow_borrow, int* instances) {
    return guarded([&] {
        REQUIRE_ARG(l && (n == 0 || (reqs && instances)), "null argument");
        if (n < 0) throw Error(DATTN_ERR_CONTRACT, "ledger: negative request count");
        for (int i = 0; i < n; ++i) (void)l->req(reqs[i]);  // all live before any change
        for (int i = 0; i < n; ++i) instances[i] = l->ensure_slot(reqs[i], allow_borrow != 0);
        for (int i = 0; i < n; ++i)
            if (instances[i] >= 0) l->req(reqs[i]).ctx += 1;
    });
}

dattn_status dattn_ledger_release(dattn_ledger* l, int64_t req, int64_t* freed_blocks) {
    return guarded([&] {
        REQUIRE_ARG(l, "null argument");
        const int64_t f = l->release(req);
        if (freed_blocks) *freed_blocks = f;
    });
}

dattn_status dattn_ledger_instance(const dattn_ledger* l, int instance, int64_t* capacity, int64_t* used,
                                   int64_t* free_blocks) {
    return guarded([&] {
        REQUIRE_ARG(l, "null argument");
        if (instance < 0 || instance >= static_cast<int>(l->inst.size()))
            throw Error(DATTN_ERR_CONTRACT, "ledger: instance out of range");
        const Instance& j = l->inst[instance];
        if (capacity) *capacity = j.capacity;
        if (used) *used = j.used;
        if (free_blocks) *free_blocks = j.free_blocks();
    });
}

dattn_status dattn_ledger_request(const dattn_ledger* l, int64_t req, int* home, int64_t* ctx,
                                  int64_t* held_blocks) {
    return guarded([&] {
        REQUIRE_ARG(l, "null argument");
        const Request& r = l->req(req);
        if (home) *home = r.home;
        if (ctx) *ctx = r.ctx;
        if (held_blocks) *held_blocks = l->held(req, r);
    });
}

dattn_status dattn_ledger_blocks(const dattn_ledger* l, int64_t req, int instance, int64_t* blocks) {
    return guarded([&] {
        REQUIRE_ARG(l && blocks, "null argument");
        if (instance < 0 || instance >= static_cast<int>(l->inst.size()))
            throw Error(DATTN_ERR_CONTRACT, "ledger: instance out of range");
        const Request& r = l->req(req);
        *blocks = instance == r.home ? l->inst[instance].local_blocks(req)
                                     : l->inst[instance].hosted_blocks(req, r.home);
    });
}

dattn_status dattn_ledger_segments(const dattn_ledger* l, int64_t req, int max, int* instance,
                                   int64_t* tok_begin, int64_t* tok_end, int* n) {
    return guarded([&] {
        REQUIRE_ARG(l && n && (max <= 0 || (instance && tok_begin && tok_end)), "null argument");
        const Request& r = l->req(req);
        int k = 0;
        int64_t b0 = 0;
        for (const auto& [w, nb] : r.segs) {
            const int64_t lo = std::min(r.ctx, b0 * l->bs), hi = std::min(r.ctx, (b0 + nb) * l->bs);
            b0 += nb;
            if (hi <= lo) continue;  // blocks not yet written (allocated for the next token)
            if (k < max) {
                instance[k] = w;
                tok_begin[k] = lo;
                tok_end[k] = hi;
            }
            ++k;
        }
        *n = k;
    });
}

dattn_status dattn_ledger_borrowed(const dattn_ledger* l, int64_t* blocks) {
    return guarded([&] {
        REQUIRE_ARG(l && blocks, "null argument");
        *blocks = l->borrowed;
    });
}

}  // extern "C"
