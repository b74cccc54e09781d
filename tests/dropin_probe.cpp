// tests/dropin_probe.cpp -- TEST INFRASTRUCTURE: an extern "C" shim over the
// B200 drop-in's kvsched::attn::multi_head_attention (libdattn.so, declared by
// the reference-identical header include/dattn_kvsched.hpp), so a GPU test can
// call the reference API of the product and the compiled reference
// (oracle/_ref, ref_multi_head_attention) on the same inputs. k/v are
// [hkv][seq][d]; cuts_flat holds each kv head's ncuts[h]+1 ascending
// boundaries. Returns 0, 2 (InputError) or 3 (ContractError).
#include <cstdint>
#include <cstring>
#include <vector>

#include "dattn_kvsched.hpp"

using namespace kvsched;

extern "C" int dropin_multi_head_attention(const double* queries, const double* k, const double* v, int64_t seq,
                                           int hq, int hkv, int d, double scale, const int64_t* cuts_flat,
                                           const int* ncuts, double* out) {
    try {
        attn::AttentionConfig cfg{d, hq, hkv, scale};
        std::vector<std::vector<attn::KVSegment>> segs(hkv);
        size_t off = 0;
        for (int h = 0; h < hkv; ++h) {
            const double* kh = k + static_cast<size_t>(h) * seq * d;
            const double* vh = v + static_cast<size_t>(h) * seq * d;
            for (int s = 0; s < ncuts[h]; ++s) {
                const int64_t a = cuts_flat[off + s], b = cuts_flat[off + s + 1];
                attn::KVSegment g;
                g.seq_p = b - a;
                g.head_dim = d;
                g.keys.assign(kh + a * d, kh + b * d);
                g.values.assign(vh + a * d, vh + b * d);
                segs[h].push_back(std::move(g));
            }
            off += ncuts[h] + 1;
        }
        std::vector<double> q(queries, queries + static_cast<size_t>(hq) * d);
        const auto o = attn::multi_head_attention(q, segs, cfg);
        std::memcpy(out, o.data(), sizeof(double) * o.size());
        return 0;
    } catch (const InputError&) {
        return 2;
    } catch (const ContractError&) {
        return 3;
    }
}
