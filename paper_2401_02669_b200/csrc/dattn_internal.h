// dattn_internal.h -- kernel parameter blocks and launchers shared by the
// CUDA kernels (dattn_kernels.cu) and the host engine (dattn_engine.cpp).
#pragma once
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

namespace dattn {

// One decode range as the kernels see it (host dattn_range, narrowed).
struct RangeDev {
    int32_t seq;
    int32_t out_row;
    int32_t kv_head;  // -1: all kv heads
    int32_t lo;
    int32_t hi;
    int32_t pad[3];
};

// K1 micro-attention launch.
struct MAParams {
    const void* k_pool;  // [pages][Hkv][P][DP]
    const void* v_pool;
    const int32_t* block_tables;  // [max_seqs][bt_stride]
    int32_t bt_stride;
    int32_t page_tokens;
    int32_t num_kv_heads;
    int32_t num_q_heads;
    int32_t group;  // Hq / Hkv
    const void* q;  // [rows][Hq][DP]
    const RangeDev* ranges;
    const int32_t* item_prefix;   // nranges+1
    const int32_t* item_table;    // claim order: [nitems][2] = (range, local item), longest first; or null
    const int32_t* chunk_prefix;  // nranges+1
    int32_t nranges;
    int32_t nitems;
    int32_t chunk_tokens;
    double scale_log2;  // scale * log2(e)
    void* records;      // [chunks][Hq][DP+4] accumulation type
    unsigned long long* work_counter;  // monotonic across launches (no per-launch reset)
    unsigned long long work_base;      // counter value at this launch's start
    int32_t* nonfinite_flag;  // may be null
    int32_t stages;
    int32_t claim_ahead;      // K2: tiles before an item's end at which the next item is fetched (0: at the boundary)
    // ---- fused group merge (K1 only; fused_mode 0 = records only) ----
    // 1: the CTA completing the last chunk of a (row, kv head) group merges the
    //    group's records into out_norm (and out_recs if set);
    // 2: ... and pushes the merged records to every rank's exchange buffer,
    //    then raises the group's flag on every rank (rank merge: K6).
    int32_t fused_mode;
    int32_t* group_counter;          // [rows][Hkv], self-resetting
    const int32_t* group_expected;   // [rows][Hkv] chunk records per group
    const int32_t* row_begin;        // [rows+1] first chunk of every row
    const int32_t* chunk_kvh;        // per chunk kv-head tag (-1 all) or null
    void* out_norm;                  // [rows][Hq][DP] storage dtype
    void* out_recs;                  // [rows][Hq][DP+4] or null
    void* peer_x[8];                 // this step's exchange half of every rank
    int32_t rank;
    int32_t nranks;
    int64_t slot_stride;             // records per source rank
};

// Failure control of the NVLink exchange polls (K5 phase D, K6). A poll that
// has waited for more than kXSlowNs checks, every 256 spins, the abort word
// (device memory, set by dattn_comm_abort through a copy on another stream)
// and its own timeout. On abort or after timeout_ns it records the reason in
// *status_dev (so every other waiting poll of the launch returns at once) and
// in *status_host (host-mapped, read by the engine without a sync) and
// returns instead of trapping: the CUDA context survives a peer that never
// arrives (a rank that failed before launching, a host stalled past the
// timeout). The step's output is then invalid and the engine refuses further
// exchanges until dattn_comm_init rebuilds the buffers. The fast path (data
// arrives within kXSlowNs) touches no control word; the kernel never reads
// host memory.
constexpr int kXAbortHost = 1, kXTimeout = 2;
constexpr unsigned long long kXSlowNs = 20000;
struct XCtl {
    unsigned long long timeout_ns;
    const int* abort_dev;  // device word; nonzero -> give up
    int* status_dev;       // device word; 0 ok, else kXAbortHost / kXTimeout
    int* status_host;      // host-mapped copy of the reason (written on failure only)
};

// K6: rank merge after fused K1/K2 (waits until every rank delivered all groups).
struct RankMergeParams {
    int32_t rows;
    int32_t heads;
    int32_t group;
    int32_t num_kv_heads;
    const int32_t* group_expected;   // this rank's [rows][Hkv]: 0 -> push identity
    void* peer_x[8];
    int32_t rank;
    int32_t nranks;
    int64_t slot_stride;
    void* out_norm;
    XCtl ctl;
};

// K3 merge launch.
struct MergeParams {
    const void* recs;
    int32_t rows;
    int32_t heads;
    const int32_t* row_begin;  // rows+1 or null
    int32_t n_uniform;
    int64_t row_mul;
    int64_t c_stride;
    const int32_t* chunk_kvh;  // per (row_begin[row]+c) kv head tag (-1 all) or null
    int32_t group;             // q heads per kv head, for chunk_kvh
    void* out_recs;            // [rows*heads][DP+4] or null
    void* out_norm;            // [rows*heads][DP] storage dtype, or null
};

// K5: fused local merge + NVLink exchange + rank merge (one launch per step).
constexpr int kMaxRanks = 8;
constexpr int kMaxExchangeGrid = 1024;  // K5 CTAs
struct XParams {
    MergeParams local;                 // chunk records of this rank (out_* unused)
    void* peer_x[kMaxRanks];           // this step's exchange half of every rank (own at [rank])
    int32_t rank;
    int32_t nranks;
    int64_t slot_stride;               // records per source rank in an exchange buffer
    int32_t groups_per_cta;            // 8 or 1
    void* out_norm;                    // [rows*heads][DP] storage dtype
    unsigned long long* trace;         // debug (DATTN_K5_TRACE): [kMaxExchangeGrid][3] sums, else null
    XCtl ctl;
};

struct FillParams {
    void* k_pool;
    void* v_pool;
    const int32_t* block_row;  // block-table row of the sequence
    int32_t page_tokens;
    int32_t num_kv_heads;
    int32_t head_dim;
    int64_t tokens;
    uint64_t seed;
    uint32_t logical_seq;
    int64_t logical_tok0;
    float amp_k;
    float amp_v;
};

// KV append: one new token row per (sequence, kv head) written into its page.
struct AppendParams {
    void* k_pool;
    void* v_pool;
    const int32_t* block_tables;
    int32_t bt_stride;
    int32_t page_tokens;
    int32_t num_kv_heads;
    const int32_t* seqs;       // [n]
    const int32_t* positions;  // [n] token index being written
    const void* k_new;         // [n][Hkv][DP]
    const void* v_new;
    int32_t n;
};

// Synthetic K/V rows [n][Hkv][DP] for logical (sequence, token) pairs: the
// values K4 would write at those positions (decode-loop inputs).
struct RowsSynthParams {
    void* k_out;
    void* v_out;
    const uint32_t* logical_seq;  // [n]
    const int64_t* logical_tok;   // [n]
    int32_t n;
    int32_t num_kv_heads;
    int32_t head_dim;
    uint64_t seed;
    float amp_k;
    float amp_v;
};

struct QFillParams {
    void* q;
    int32_t rows;
    int32_t heads;
    int32_t head_dim;
    uint64_t seed;
    uint32_t row0;
    float amp;
};

struct ScatterParams {
    void* k_pool;
    void* v_pool;
    const void* k_rows;  // [n][DP]
    const void* v_rows;
    const int32_t* block_row;
    int32_t page_tokens;
    int32_t num_kv_heads;
    int32_t kv_head;
    int64_t tok0;
    int64_t n;
};

// dtype codes as dattn.h
constexpr int kBF16 = 0, kF32 = 1, kF64 = 2;

int ma_threads();
size_t ma_smem_bytes(int dtype, int dp, int group, int stages);
int ma_stage_tokens(int dtype, int dp);
cudaError_t ma_configure(int dtype, int dp, int group, size_t smem);
cudaError_t ma_occupancy(int dtype, int dp, int group, size_t smem, int* blocks_per_sm);
cudaError_t launch_ma(int dtype, int dp, const MAParams& p, int grid, size_t smem,
                      cudaStream_t st);
// K1g: generic MA for groups K1 does not instantiate and head widths > 256
bool ma_supported(int dtype, int dp, int group);
cudaError_t ma_generic_occupancy(int dtype, int dp, int* blocks_per_sm);
cudaError_t launch_ma_generic(int dtype, int dp, const MAParams& p, int grid, cudaStream_t st);
cudaError_t launch_merge(int dtype, int dp, const MergeParams& p, cudaStream_t st);
cudaError_t launch_merge_exchange(int dtype, int dp, const XParams& p, int grid, cudaStream_t st);
// Resident CTAs per SM of K5 (kind 0) / K6 (kind 1): their polls need the
// whole grid co-resident, so the engine caps the grid at this x num_sms.
cudaError_t exchange_occupancy(int dtype, int dp, int kind, int* blocks_per_sm);
cudaError_t launch_rank_merge(int dtype, int dp, const RankMergeParams& p, int grid, cudaStream_t st);
cudaError_t launch_fill_kv(int dtype, int dp, const FillParams& p, cudaStream_t st);
cudaError_t launch_append(int dtype, int dp, const AppendParams& p, cudaStream_t st);
cudaError_t launch_fill_q(int dtype, int dp, const QFillParams& p, cudaStream_t st);
cudaError_t launch_rows_synth(int dtype, int dp, const RowsSynthParams& p, cudaStream_t st);
cudaError_t launch_scatter(int dtype, int dp, const ScatterParams& p, cudaStream_t st);
cudaError_t launch_gather(int dtype, int dp, const ScatterParams& p, cudaStream_t st);
// K2 (tcgen05 GQA path, dattn_gqa_tc.cu)
size_t gqa_tc_smem_bytes();
cudaError_t gqa_tc_configure();
cudaError_t make_tmap_tiles(void* map_out, const void* base, uint64_t pages, uint32_t kv_heads,
                            uint32_t page_tokens);
cudaError_t make_tmap_rows128(void* map_out, const void* base, uint64_t rows, uint32_t box_rows);
cudaError_t launch_gqa_tc(const void* tm_k, const void* tm_v, const void* tm_q, const void* tm_k4,
                          const void* tm_v4, const MAParams& p, int grid, cudaStream_t st);
cudaError_t launch_identity_records(int dtype, int dp, void* recs, int64_t n, cudaStream_t st);

// Launch with programmatic stream serialization (PDL): the grid is scheduled
// while the previous grid on the stream drains, and blocks in
// griddepcontrol.wait until it has completed. The MA kernels use it behind the
// previous step's merge grid (their set-up -- barriers, TMEM, tensor-map
// prefetch -- overlaps its tail); DATTN_NO_PDL=1 turns it off (debug).
inline cudaError_t launch_pdl_raw(const void* f, int grid, int block, size_t smem, cudaStream_t st, void** args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    static const bool off = std::getenv("DATTN_NO_PDL") != nullptr;
    cfg.attrs = at;
    cfg.numAttrs = off ? 0 : 1;
    return cudaLaunchKernelExC(&cfg, f, args);
}

}  // namespace dattn
