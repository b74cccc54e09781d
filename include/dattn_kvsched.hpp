// dattn_kvsched.hpp -- the reference's C++ operator API, re-declared for the
// B200 drop-in.
//
// Declarations (names, members, member order, defaults, signatures and the
// two exception types) are ABI-identical to
//   /root/reference/proj/include/kvsched/distattention.hpp:16-95
//   /root/reference/proj/include/kvsched/common.hpp:8-20
// so code compiled against the reference headers links against
// libdattn.so unchanged (proven by build/dropin/: the reference's own
// test_distattention.cpp and acceptance gates 1-3).
// The definitions live in paper_2401_02669_b200/csrc/kvsched_adapter.cpp and
// run every partial, merge and aggregate on the GPU through include/dattn.h.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace kvsched {

// Caller bug: a violated precondition (common.hpp:11-15).
class ContractError : public std::logic_error {
public:
    explicit ContractError(const std::string& what) : std::logic_error(what) {}
};

// Rejected data: non-finite values, malformed payloads (common.hpp:17-20).
class InputError : public std::runtime_error {
public:
    explicit InputError(const std::string& what) : std::runtime_error(what) {}
};

namespace attn {

struct AttentionConfig {
    int head_dim = 0;
    int num_q_heads = 1;
    int num_kv_heads = 1;
    double scale = 0.0;  // 0 selects 1/sqrt(head_dim)

    double effective_scale() const;
    void validate() const;  // ContractError on a bad geometry or scale
};

// Host view of one head's contiguous token run, row-major [seq_p x head_dim].
struct KVSegment {
    std::vector<double> keys;
    std::vector<double> values;
    int64_t seq_p = 0;
    int head_dim = 0;

    const double* key_row(int64_t i) const { return keys.data() + i * head_dim; }
    const double* value_row(int64_t i) const { return values.data() + i * head_dim; }
    void validate() const;
};

// (m, e, ma) of one query over one segment; seq_p == 0 marks the identity.
struct AttentionPartial {
    double m = 0.0;
    double e = 0.0;
    std::vector<double> ma;
    int64_t seq_p = 0;

    static AttentionPartial identity(int head_dim);
    bool is_identity() const { return seq_p == 0; }
};

std::vector<double> naive_attention(const std::vector<double>& q, const KVSegment& kv,
                                    const AttentionConfig& cfg);

AttentionPartial compute_micro_attention(const std::vector<double>& q, const KVSegment& kv,
                                         const AttentionConfig& cfg);

AttentionPartial combine_partials(const AttentionPartial& a, const AttentionPartial& b);

std::vector<double> aggregate_partials(const std::vector<AttentionPartial>& parts);

int gqa_kv_head(int query_head, const AttentionConfig& cfg);

std::vector<double> multi_head_attention(
    const std::vector<double>& queries,
    const std::vector<std::vector<KVSegment>>& kv_segments_per_head,
    const AttentionConfig& cfg);

std::vector<std::byte> serialize_partial(const AttentionPartial& p);
AttentionPartial deserialize_partial(const std::vector<std::byte>& bytes, int head_dim);

}  // namespace attn
}  // namespace kvsched
