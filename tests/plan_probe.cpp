// tests/plan_probe.cpp -- TEST INFRASTRUCTURE: runs the decode-plan builder of
// libdattn.so (dattn_store::build_plan, csrc/dattn_engine.cpp) on the host,
// without a GPU, for a few batch shapes, and prints one JSON line per shape
// with the plan facts tests/test_plan_cpu.py checks: chunk size, item count,
// the longest-first claim table (if any) expanded to (item, tokens) pairs,
// chunks per row and the per-(row, kv head) completion counts.
#include <cstdio>
#include <string>
#include <vector>

#include "dattn_engine.h"

using dattn::Plan;

static dattn_store* make_store(int hq, int hkv, int dtype, int max_seqs, bool tc, int ctas_per_sm) {
    auto* s = new dattn_store();
    s->cfg.head_dim = 128;
    s->cfg.num_q_heads = hq;
    s->cfg.num_kv_heads = hkv;
    s->cfg.dtype = dtype;
    s->cfg.page_tokens = 16;
    s->cfg.max_seqs = max_seqs;
    s->cfg.num_pages = 1 << 20;
    s->cfg.max_pages_per_seq = 1 << 20;
    s->dp = 128;
    s->group = hq / hkv;
    s->num_sms = 148;
    s->ma_ctas_per_sm = ctas_per_sm;
    s->tc_ok = tc;
    s->seq_tokens.assign(max_seqs, 0);
    s->seq_live.assign(max_seqs, 0);
    return s;
}

static void run(const char* name, dattn_store* s, const std::vector<dattn_range>& rs, int rows) {
    for (const auto& r : rs) {
        s->seq_live[r.seq] = 1;
        if (s->seq_tokens[r.seq] < r.tok_end) s->seq_tokens[r.seq] = r.tok_end;
    }
    dattn_batch b{};
    b.num_rows = rows;
    b.num_ranges = static_cast<int32_t>(rs.size());
    b.ranges = rs.data();
    Plan pl;
    s->build_plan(b, false, pl);
    const int nr = pl.nranges;
    const int C = pl.chunk_tokens;
    std::string js = std::string("{\"name\": \"") + name + "\", \"chunk\": " + std::to_string(C) +
                     ", \"items\": " + std::to_string(pl.nitems) + ", \"chunks\": " + std::to_string(pl.nchunks) +
                     ", \"table\": " + (pl.off_table ? "true" : "false") + ", \"nranges\": " + std::to_string(nr);
    js += ", \"ranges\": [";
    for (int r = 0; r < nr; ++r) {
        const int32_t* rg = &pl.words[pl.off_ranges + 8 * r];
        js += (r ? ", [" : "[") + std::to_string(rg[0]) + ", " + std::to_string(rg[1]) + ", " + std::to_string(rg[2]) +
              ", " + std::to_string(rg[3]) + ", " + std::to_string(rg[4]) + "]";
    }
    js += "]";
    // item lengths in claim order
    // the plan's own ranges (the builder may cut trailing chunks of uniform
    // batches into sub-ranges): RangeDev {seq, out_row, kv_head, lo, hi, pad[3]}
    auto item_len = [&](int r, int local) {
        const int32_t* rg = &pl.words[pl.off_ranges + 8 * r];
        const int nh = rg[2] < 0 ? s->cfg.num_kv_heads : 1;
        const int j = local / nh;
        const int64_t lo = rg[3] + static_cast<int64_t>(j) * C;
        return static_cast<int64_t>(std::min<int64_t>(rg[4], lo + C) - lo);
    };
    (void)rs;
    js += ", \"order\": [";
    for (int k = 0; k < pl.nitems; ++k) {
        int r, local;
        if (pl.off_table) {
            r = pl.words[pl.off_table + 2 * k];
            local = pl.words[pl.off_table + 2 * k + 1];
        } else {
            r = 0;
            while (r + 1 < nr && pl.words[pl.off_item + r + 1] <= k) ++r;
            local = k - pl.words[pl.off_item + r];
        }
        const int item = pl.words[pl.off_item + r] + local;
        js += (k ? ", [" : "[") + std::to_string(item) + ", " + std::to_string(item_len(r, local)) + "]";
    }
    js += "], \"row_chunks\": [";
    for (int i = 0; i < rows; ++i)
        js += (i ? ", " : "") + std::to_string(pl.words[pl.off_rowchunk + i + 1] - pl.words[pl.off_rowchunk + i]);
    js += "], \"expect\": [";
    for (int i = 0; i < rows * s->cfg.num_kv_heads; ++i)
        js += (i ? ", " : "") + std::to_string(pl.words[pl.off_expect + i]);
    js += "]}";
    std::printf("%s\n", js.c_str());
}

static dattn_range R(int seq, int row, int64_t lo, int64_t hi, int kvh = -1) {
    dattn_range r{};
    r.seq = seq;
    r.out_row = row;
    r.kv_head = kvh;
    r.tok_begin = lo;
    r.tok_end = hi;
    return r;
}

int main() {
    {  // ragged MHA batch on K2 (config-2 like): longest-first table
        auto* s = make_store(32, 32, 0, 80, true, 1);
        std::vector<dattn_range> rs;
        const int lens[] = {1024, 32768, 5000, 17, 20000, 8192, 300, 12345};
        for (int i = 0; i < 8; ++i) rs.push_back(R(i, i, 0, lens[i]));
        run("ragged_k2", s, rs, 8);
        delete s;
    }
    {  // equal lengths (config-3 like): full chunks in natural order, then the
       // trailing chunks cut into quarter sub-ranges, run last
        auto* s = make_store(64, 8, 0, 20, true, 1);
        std::vector<dattn_range> rs;
        for (int i = 0; i < 16; ++i) rs.push_back(R(i, i, 0, 131072));
        run("uniform_k2", s, rs, 16);
        delete s;
    }
    {  // small fp32 batch on K1 (config-1 like, 4 rBlocks): 512-token floor
        auto* s = make_store(32, 32, 1, 8, false, 2);
        std::vector<dattn_range> rs;
        for (int i = 0; i < 4; ++i) rs.push_back(R(0, 0, i * 1024, (i + 1) * 1024));
        run("cfg1_k1", s, rs, 1);
        delete s;
    }
    {  // per-kv-head ranges, an empty range and a row without ranges
        auto* s = make_store(8, 4, 0, 8, true, 1);
        std::vector<dattn_range> rs = {R(0, 0, 0, 3000, 1), R(0, 0, 0, 100, 3), R(1, 1, 0, 0), R(2, 3, 5, 9000)};
        run("kvh_empty", s, rs, 4);
        delete s;
    }
    return 0;
}
