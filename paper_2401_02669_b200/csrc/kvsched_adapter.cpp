// kvsched_adapter.cpp -- the reference's kvsched::attn operator API
// (proj/include/kvsched/distattention.hpp:16-95) implemented on the B200 path.
//
// Every partial (compute_micro_attention), merge (combine_partials),
// aggregate (aggregate_partials), unsplit attention (naive_attention) and
// per-head driver (multi_head_attention) runs in the fp64 instantiation of
// the CUDA kernels behind include/dattn.h. What stays on the host is what is
// not arithmetic: argument validation with the reference's exception types
// (distattention.cpp:26-57), the identity short-circuit of combine_partials
// (:135-136, a selection), the integer GQA map (:176-181) and the wire
// (de)serialisation (:211-237). Non-finite K/V are detected by the MA kernel
// itself (DATTN_F_CHECK_FINITE) instead of a separate CPU pass.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "dattn.h"
#include "dattn_kvsched.hpp"

namespace kvsched::attn {
namespace {

constexpr double kNegInf = -std::numeric_limits<double>::infinity();

void require(bool ok, const char* msg) {
    if (!ok) throw ContractError(msg);
}
void input_check(bool ok, const char* msg) {
    if (!ok) throw InputError(msg);
}

bool all_finite(const std::vector<double>& v) {
    for (double x : v)
        if (!std::isfinite(x)) return false;
    return true;
}

void raise(dattn_status st) {
    const std::string msg = dattn_last_error();
    switch (st) {
        case DATTN_OK: return;
        case DATTN_ERR_CONTRACT: throw ContractError(msg);
        case DATTN_ERR_INPUT: throw InputError(msg);
        default: throw std::runtime_error("dattn: " + msg);
    }
}
#define DATTN_CALL(expr) raise(expr)

int padded(int d) {
    for (int dp : {16, 32, 64, 128, 256, 512})
        if (d <= dp) return dp;
    throw ContractError("head_dim > 512 is not supported by the B200 kernels");
}

// One fp64 store per (padded dim, query group) and calling thread, grown on
// demand; the reference API is reentrant, so every thread
// gets its own stores and stream.
struct StoreSlot {
    dattn_store* s = nullptr;
    int64_t pages = 0;
    int seqs = 0;
    void* dq = nullptr;
    size_t dq_cap = 0;
    void* drec = nullptr;
    size_t drec_cap = 0;
    void* dout = nullptr;
    size_t dout_cap = 0;
    ~StoreSlot() {
        if (!s) return;
        dattn_device_free(s, dq);
        dattn_device_free(s, drec);
        dattn_device_free(s, dout);
        dattn_store_destroy(s);
    }
    void* dev(void*& p, size_t& cap, size_t bytes) {
        if (bytes > cap) {
            dattn_device_free(s, p);
            p = nullptr;
            cap = 0;
            DATTN_CALL(dattn_device_alloc(s, bytes, &p));
            cap = bytes;
        }
        return p;
    }
};

int device_ordinal() {
    const char* e = std::getenv("DATTN_DEVICE");
    return e ? std::atoi(e) : 0;
}

StoreSlot& slot(int dp, int group, int64_t pages_needed, int seqs_needed) {
    thread_local std::map<std::pair<int, int>, std::unique_ptr<StoreSlot>> slots;
    auto& ptr = slots[{dp, group}];
    if (!ptr) ptr = std::make_unique<StoreSlot>();
    StoreSlot& sl = *ptr;
    if (sl.s && sl.pages >= pages_needed && sl.seqs >= seqs_needed) return sl;
    const int64_t pages = std::max<int64_t>({pages_needed * 2, sl.pages * 2, 1024});
    const int seqs = std::max({seqs_needed * 2, sl.seqs, 256});
    ptr = std::make_unique<StoreSlot>();
    StoreSlot& fresh = *ptr;
    dattn_store_config c{};
    c.head_dim = dp;
    c.num_q_heads = group;
    c.num_kv_heads = 1;
    c.scale = 0.0;
    c.dtype = DATTN_F64;
    c.page_tokens = 16;
    c.num_pages = pages;
    c.max_seqs = seqs;
    c.max_pages_per_seq = static_cast<int>(std::min<int64_t>(pages, 1 << 30));
    c.device = device_ordinal();
    DATTN_CALL(dattn_store_create(&c, &fresh.s));
    fresh.pages = pages;
    fresh.seqs = seqs;
    return fresh;
}

int64_t pages_for(int64_t tokens) { return (tokens + 15) / 16; }

// Sequences borrowed from a store for one call; released on scope exit.
struct SeqLease {
    dattn_store* s;
    std::vector<int32_t> ids;
    explicit SeqLease(dattn_store* st) : s(st) {}
    int32_t add(const KVSegment& kv) {
        int32_t id = -1;
        DATTN_CALL(dattn_seq_create(s, kv.seq_p, &id));
        ids.push_back(id);
        if (kv.seq_p > 0)
            DATTN_CALL(dattn_kv_write(s, id, 0, 0, kv.seq_p, kv.keys.data(), kv.values.data(),
                                      DATTN_F64, kv.head_dim));
        return id;
    }
    ~SeqLease() {
        for (int32_t id : ids) dattn_seq_release(s, id, nullptr);
    }
};

void check_shape(const KVSegment& kv) {
    require(kv.head_dim >= 1, "segment head_dim must be >= 1");
    require(kv.seq_p >= 0, "segment length must be >= 0");
    require(kv.keys.size() == static_cast<size_t>(kv.seq_p) * kv.head_dim,
            "segment keys shape mismatch");
    require(kv.values.size() == static_cast<size_t>(kv.seq_p) * kv.head_dim,
            "segment values shape mismatch");
}

void check_query(const std::vector<double>& q, const AttentionConfig& cfg) {
    cfg.validate();
    require(static_cast<int>(q.size()) == cfg.head_dim, "query length must equal head_dim");
    input_check(all_finite(q), "query contains non-finite values");
}

std::vector<double> pad_rows(const double* src, int rows, int d, int dp) {
    std::vector<double> out(static_cast<size_t>(rows) * dp, 0.0);
    for (int r = 0; r < rows; ++r)
        std::memcpy(out.data() + static_cast<size_t>(r) * dp, src + static_cast<size_t>(r) * d,
                    sizeof(double) * d);
    return out;
}

// Merge n partials of one head on the GPU (K3); returns the merged record
// [m, e, tokens, 0, ma[dp]] or, with norm, the normalised row [dp].
std::vector<double> gpu_merge(const std::vector<const AttentionPartial*>& parts, int d, bool norm) {
    const int dp = padded(d);
    const int rec = dp + 4;
    StoreSlot& sl = slot(dp, 1, 0, 0);
    const int n = static_cast<int>(parts.size());
    std::vector<double> h(static_cast<size_t>(n) * rec, 0.0);
    for (int i = 0; i < n; ++i) {
        double* r = h.data() + static_cast<size_t>(i) * rec;
        r[0] = parts[i]->m;
        r[1] = parts[i]->e;
        r[2] = static_cast<double>(parts[i]->seq_p);
        std::memcpy(r + 4, parts[i]->ma.data(), sizeof(double) * d);
    }
    const size_t in_bytes = h.size() * sizeof(double);
    void* din = sl.dev(sl.drec, sl.drec_cap, in_bytes);
    void* dout = sl.dev(sl.dout, sl.dout_cap, sizeof(double) * rec);
    DATTN_CALL(dattn_memcpy(sl.s, din, h.data(), in_bytes, 1 /*H2D*/));
    dattn_merge_desc md{1, 1, nullptr, n, 0, 1};
    DATTN_CALL(dattn_merge_partials(sl.s, &md, din, norm ? nullptr : dout, norm ? dout : nullptr));
    std::vector<double> out(norm ? dp : rec);
    DATTN_CALL(dattn_memcpy(sl.s, out.data(), dout, sizeof(double) * out.size(), 2 /*D2H*/));
    return out;
}

}  // namespace

double AttentionConfig::effective_scale() const {
    return scale > 0.0 ? scale : 1.0 / std::sqrt(static_cast<double>(head_dim));
}

void AttentionConfig::validate() const {
    require(head_dim >= 1, "head_dim must be >= 1");
    require(num_q_heads >= 1 && num_kv_heads >= 1, "head counts must be >= 1");
    require(num_q_heads % num_kv_heads == 0, "num_q_heads must be a multiple of num_kv_heads");
    require(std::isfinite(scale) && scale >= 0.0, "scale must be finite and >= 0");
}

void KVSegment::validate() const {
    check_shape(*this);
    input_check(all_finite(keys) && all_finite(values), "segment contains non-finite values");
}

AttentionPartial AttentionPartial::identity(int head_dim) {
    require(head_dim >= 1, "head_dim must be >= 1");
    AttentionPartial p;
    p.m = kNegInf;
    p.e = 0.0;
    p.ma.assign(head_dim, 0.0);
    p.seq_p = 0;
    return p;
}

std::vector<double> naive_attention(const std::vector<double>& q, const KVSegment& kv,
                                    const AttentionConfig& cfg) {
    check_query(q, cfg);
    check_shape(kv);
    require(kv.head_dim == cfg.head_dim, "segment head_dim mismatch");
    require(kv.seq_p >= 1, "naive attention needs at least one token");
    const int d = cfg.head_dim, dp = padded(d);
    StoreSlot& sl = slot(dp, 1, pages_for(kv.seq_p), 1);
    SeqLease lease(sl.s);
    const int32_t seq = lease.add(kv);
    dattn_range r{seq, 0, -1, 0, 0, kv.seq_p};
    // one chunk: a single global max, as the reference's unsplit softmax
    dattn_batch b{1, 1, &r, static_cast<int32_t>(std::min<int64_t>(kv.seq_p, INT32_MAX)),
                  DATTN_F_CHECK_FINITE, cfg.effective_scale()};
    std::vector<double> qp = pad_rows(q.data(), 1, d, dp), out(dp);
    DATTN_CALL(dattn_decode(sl.s, &b, qp.data(), out.data(), nullptr, DATTN_MEM_HOST));
    out.resize(d);
    return out;
}

AttentionPartial compute_micro_attention(const std::vector<double>& q, const KVSegment& kv,
                                         const AttentionConfig& cfg) {
    check_query(q, cfg);
    check_shape(kv);
    require(kv.head_dim == cfg.head_dim, "segment head_dim mismatch");
    const int d = cfg.head_dim;
    if (kv.seq_p == 0) return AttentionPartial::identity(d);
    const int dp = padded(d), rec = dp + 4;
    StoreSlot& sl = slot(dp, 1, pages_for(kv.seq_p), 1);
    SeqLease lease(sl.s);
    const int32_t seq = lease.add(kv);
    std::vector<double> qp = pad_rows(q.data(), 1, d, dp);
    void* dq = sl.dev(sl.dq, sl.dq_cap, sizeof(double) * dp);
    void* drec = sl.dev(sl.drec, sl.drec_cap, sizeof(double) * rec);
    DATTN_CALL(dattn_memcpy(sl.s, dq, qp.data(), sizeof(double) * dp, 1));
    dattn_range r{seq, 0, -1, 0, 0, kv.seq_p};
    dattn_batch b{1, 1, &r, 0, DATTN_F_CHECK_FINITE, cfg.effective_scale()};
    DATTN_CALL(dattn_micro_attention(sl.s, &b, dq, drec));
    std::vector<double> h(rec);
    DATTN_CALL(dattn_memcpy(sl.s, h.data(), drec, sizeof(double) * rec, 2));
    AttentionPartial p;
    p.m = h[0];
    p.e = h[1];
    p.ma.assign(h.begin() + 4, h.begin() + 4 + d);
    p.seq_p = kv.seq_p;
    return p;
}

AttentionPartial combine_partials(const AttentionPartial& a, const AttentionPartial& b) {
    require(!a.ma.empty() && !b.ma.empty(), "partials must be initialized");
    require(a.ma.size() == b.ma.size(), "partial head_dim mismatch");
    // the identity is an exact unit: hand back the other operand untouched
    if (a.is_identity()) return b;
    if (b.is_identity()) return a;
    const int d = static_cast<int>(a.ma.size());
    const std::vector<double> r = gpu_merge({&a, &b}, d, false);
    AttentionPartial out;
    out.m = r[0];
    out.e = r[1];
    out.ma.assign(r.begin() + 4, r.begin() + 4 + d);
    out.seq_p = a.seq_p + b.seq_p;
    return out;
}

std::vector<double> aggregate_partials(const std::vector<AttentionPartial>& parts) {
    require(!parts.empty(), "aggregate needs at least one partial");
    const size_t d = parts[0].ma.size();
    require(d >= 1, "partials must be initialized");
    int64_t total = 0;
    std::vector<const AttentionPartial*> ptrs;
    for (const auto& p : parts) {
        require(p.ma.size() == d, "partial head_dim mismatch");
        total += p.seq_p;
        ptrs.push_back(&p);
    }
    require(total >= 1, "aggregate needs at least one covered token");
    std::vector<double> out = gpu_merge(ptrs, static_cast<int>(d), true);
    out.resize(d);
    return out;
}

int gqa_kv_head(int query_head, const AttentionConfig& cfg) {
    cfg.validate();
    require(query_head >= 0 && query_head < cfg.num_q_heads, "query_head out of range");
    return query_head / (cfg.num_q_heads / cfg.num_kv_heads);
}

std::vector<double> multi_head_attention(
    const std::vector<double>& queries,
    const std::vector<std::vector<KVSegment>>& kv_segments_per_head,
    const AttentionConfig& cfg) {
    cfg.validate();
    require(queries.size() == static_cast<size_t>(cfg.num_q_heads) * cfg.head_dim,
            "queries shape mismatch");
    require(kv_segments_per_head.size() == static_cast<size_t>(cfg.num_kv_heads),
            "kv head count mismatch");
    const int d = cfg.head_dim, dp = padded(d);
    const int hkv = cfg.num_kv_heads, g = cfg.num_q_heads / hkv;
    int64_t pages = 0;
    int nseg = 0;
    for (const auto& segs : kv_segments_per_head) {
        int64_t total = 0;
        for (const auto& s : segs) {
            check_shape(s);
            require(s.head_dim == d, "segment head_dim mismatch");
            total += s.seq_p;
            pages += pages_for(s.seq_p);
            ++nseg;
        }
        require(!segs.empty(), "aggregate needs at least one partial");
        require(total >= 1, "aggregate needs at least one covered token");
    }
    input_check(all_finite(queries), "query contains non-finite values");
    StoreSlot& sl = slot(dp, g, pages, nseg);
    SeqLease lease(sl.s);
    std::vector<dattn_range> ranges;
    for (int k = 0; k < hkv; ++k)
        for (const auto& s : kv_segments_per_head[k]) {
            const int32_t id = lease.add(s);
            ranges.push_back(dattn_range{id, k, 0, 0, 0, s.seq_p});
        }
    std::vector<double> qp = pad_rows(queries.data(), cfg.num_q_heads, d, dp);
    std::vector<double> out(static_cast<size_t>(cfg.num_q_heads) * dp);
    dattn_batch b{hkv, static_cast<int32_t>(ranges.size()), ranges.data(), 0,
                  DATTN_F_CHECK_FINITE, cfg.effective_scale()};
    DATTN_CALL(dattn_decode(sl.s, &b, qp.data(), out.data(), nullptr, DATTN_MEM_HOST));
    std::vector<double> res(static_cast<size_t>(cfg.num_q_heads) * d);
    for (int h = 0; h < cfg.num_q_heads; ++h)
        std::memcpy(res.data() + static_cast<size_t>(h) * d, out.data() + static_cast<size_t>(h) * dp,
                    sizeof(double) * d);
    return res;
}

std::vector<std::byte> serialize_partial(const AttentionPartial& p) {
    require(!p.ma.empty(), "partial must be initialized");
    // (m, e, ma): head_dim + 2 doubles whatever the segment length
    std::vector<std::byte> bytes(sizeof(double) * (2 + p.ma.size()));
    std::memcpy(bytes.data(), &p.m, sizeof(double));
    std::memcpy(bytes.data() + sizeof(double), &p.e, sizeof(double));
    std::memcpy(bytes.data() + 2 * sizeof(double), p.ma.data(), sizeof(double) * p.ma.size());
    return bytes;
}

AttentionPartial deserialize_partial(const std::vector<std::byte>& bytes, int head_dim) {
    require(head_dim >= 1, "head_dim must be >= 1");
    input_check(bytes.size() == sizeof(double) * (2 + static_cast<size_t>(head_dim)),
                "partial payload size mismatch");
    AttentionPartial p;
    std::memcpy(&p.m, bytes.data(), sizeof(double));
    std::memcpy(&p.e, bytes.data() + sizeof(double), sizeof(double));
    p.ma.resize(head_dim);
    std::memcpy(p.ma.data(), bytes.data() + 2 * sizeof(double), sizeof(double) * head_dim);
    // the wire carries no token count: only identity-ness survives
    p.seq_p = (p.e == 0.0 && p.m == kNegInf) ? 0 : 1;
    return p;
}

}  // namespace kvsched::attn
