// dattn_engine.h -- host-side engine objects behind the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "dattn.h"
#include "dattn_internal.h"

namespace dattn {

struct Error : std::runtime_error {
    Error(dattn_status s, const std::string& m);
    dattn_status status;
};

void cuda_check(cudaError_t e, const char* what);
void set_error(const std::string& s);
void count_launch(int n);
int padded_dim_for(int head_dim);
int elem_bytes_for(int dtype);

// C ABI wrapper: exceptions -> status + thread-local message (capi.cpp:43-55)
template <class F>
inline dattn_status guarded(F&& f) {
    try {
        f();
        return DATTN_OK;
    } catch (const Error& e) {
        set_error(e.what());
        return e.status;
    } catch (const std::bad_alloc&) {
        set_error("out of host memory");
        return DATTN_ERR_INTERNAL;
    } catch (const std::exception& e) {
        set_error(e.what());
        return DATTN_ERR_INTERNAL;
    }
}

#define REQUIRE_ARG(cond, msg) \
    do { if (!(cond)) throw ::dattn::Error(DATTN_ERR_INVALID_ARGUMENT, msg); } while (0)

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    void ensure(size_t bytes);
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf();
};

struct HostBuf {
    void* p = nullptr;
    size_t cap = 0;
    void ensure(size_t bytes);
    HostBuf() = default;
    HostBuf(const HostBuf&) = delete;
    HostBuf& operator=(const HostBuf&) = delete;
    ~HostBuf();
};

// Decode plan: the int32 metadata block uploaded once per call.
struct Plan {
    std::vector<int32_t> words;
    size_t off_ranges = 0, off_item = 0, off_chunk = 0, off_rowchunk = 0, off_kvh = 0, off_expect = 0;
    size_t off_table = 0;  // 0: no claim-order table (uniform items)
    int32_t nitems = 0, nchunks = 0, nranges = 0, nrows = 0, chunk_tokens = 0;
    bool any_kvh = false;
    bool any_empty_group = false;  // some (row, kv head) has no chunk on this store
};

}  // namespace dattn

struct dattn_store {
    dattn_store_config cfg{};
    int dp = 0, esz = 0, acc_sz = 0, rec_elems = 0, group = 1;
    int64_t page_elems = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t meta_ev = nullptr;
    int num_sms = 0;
    int ma_stages = 0, ma_ctas_per_sm = 1;
    bool ma_generic = false;  // K1g instead of K1 (groups > 16 / 8 fp64, head_dim > 256)
    size_t ma_smem = 0;

    void* kpool = nullptr;
    void* vpool = nullptr;
    int32_t* d_bt = nullptr;
    int32_t* d_counter = nullptr;
    int32_t* d_flag = nullptr;

    // page ledger (RManager::alloc_local / free_request, controlplane.cpp:38-79)
    std::vector<int32_t> h_bt;
    std::vector<int64_t> seq_tokens;
    std::vector<int32_t> seq_pages;
    std::vector<uint8_t> seq_live;
    std::vector<int32_t> free_pages;
    std::vector<int32_t> free_seqs;
    int64_t used_pages = 0;

    dattn::DevBuf d_meta, recs, rowrecs, qbuf, obuf, gathered, d_staging;
    // kv_append: persistent staging (the call is asynchronous on the store
    // stream); app_ev guards the pinned meta staging against reuse
    dattn::DevBuf app_meta, app_rows;
    dattn::HostBuf app_hmeta;
    cudaEvent_t app_ev = nullptr;
    dattn::HostBuf h_meta, h_staging;
    size_t staging_used = 0;
    unsigned long long work_base = 0;
    dattn::Plan scratch_plan;
    std::vector<int32_t> last_words;  // plan currently in d_meta
    bool meta_valid = false;

    ncclComm_t comm = nullptr;
    // NCCL runs on its own non-blocking stream, ordered with `stream` by
    // events: a caller stream that is the legacy default stream (torch's
    // default-stream handle) would otherwise implicitly synchronise with
    // NCCL's internal streams
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t comm_ev[2] = {nullptr, nullptr};
    cudaStream_t comm_begin();
    void comm_end();
    int rank = 0, nranks = 1;
    // exchange buffers (K5 / K6): IPC-mapped, two halves used by alternate steps
    void* xbuf = nullptr;  // own [2][nranks][slot_stride][rec]
    void* peer_x[8]{};
    int64_t slot_stride = 0;
    size_t xhalf = 0;  // bytes of one exchange half
    void* xhalf_ptr(void* base, uint32_t ep) const {
        return static_cast<unsigned char*>(base) + (ep & 1u) * xhalf;
    }
    uint32_t epoch = 0;  // step counter: its parity selects the half
    bool fused_merge = false;
    // poll control (dattn_internal.h XCtl): device [0] abort, [1] status;
    // host-mapped status copy; the abort word is written on abort_stream
    int* x_ctl_dev = nullptr;
    int* x_status_host = nullptr;
    cudaStream_t abort_stream = nullptr;
    unsigned long long x_timeout_ns = 0;
    int x_grid_cap[2] = {0, 0};  // co-resident CTAs of K5, K6 (occupancy x SMs)
    dattn::XCtl xctl() const { return {x_timeout_ns, x_ctl_dev, x_ctl_dev + 1, x_status_host}; }
    void check_exchange_status() const;
    void setup_exchange();
    void release_exchange();
    // KV migration by page copies (dattn_kv_pull): every rank's K/V pools
    // IPC-mapped here; copies run on the copy engines from mig_stream, a
    // low-priority stream beside the decode stream
    void* peer_kpool[8]{};
    void* peer_vpool[8]{};
    int64_t peer_pages[8]{};  // pool size (pages) of every rank
    cudaStream_t mig_stream = nullptr;
    cudaEvent_t mig_ev = nullptr;
    int64_t mig_pending = 0;  // pulls issued since the last dattn_kv_migration_join
    void setup_peer_pools();
    void release_peer_pools();

    // K2 (tcgen05) path for grouped-query bf16 stores
    bool tc_ok = false;
    alignas(64) unsigned char tm_k[128]{}, tm_v[128]{}, tm_q[128]{}, tm_k4[128]{}, tm_v4[128]{};
    const void* tm_q_ptr = nullptr;
    int tm_q_rows = -1;

    bool timing = false;
    dattn_stats stats{};
    std::vector<std::array<cudaEvent_t, 2>> ma_events, merge_events, comm_events;
    size_t ma_events_used = 0, merge_events_used = 0, comm_events_used = 0;
    cudaEvent_t* timer_pair(int kind);
    void collect_timing();

    ~dattn_store();
    void init(const dattn_store_config& c);
    void activate() const;
    void check_seq(int32_t seq) const;
    void grow(int32_t seq, int64_t tokens);
    void upload_bt_row(int32_t seq);
    void write_rows(int32_t seq, int kv_head, int64_t tok0, int64_t n, const void* k,
                    const void* v, int src_dtype, int src_row_elems);

    void plan(const dattn_batch& b, bool one_chunk_per_range, dattn::Plan& pl);
    void build_plan(const dattn_batch& b, bool one_chunk_per_range, dattn::Plan& pl) const;
    dattn::Plan cache_plan;
    bool plan_cached = false, cache_one_chunk = false;
    int32_t cache_rows = -1, cache_chunk = -1;
    std::vector<unsigned char> cache_ranges;
    void upload_plan(const dattn::Plan& pl);
    void run_ma(const dattn::Plan& pl, const void* q_dev, void* recs, double scale,
                bool check_finite, const dattn::MAParams* fused = nullptr);
    bool fused_ok(const dattn::Plan& pl, bool check_finite) const;
    void fill_fused(const dattn::Plan& pl, dattn::MAParams& f);
    dattn::DevBuf gcounter;
    dattn::DevBuf k5_trace;                   // DATTN_K5_TRACE debug stamps
    size_t gcounter_elems = 0;
    void run_merge(const dattn::MergeParams& mp);
    void local_merge(const dattn::Plan& pl, const void* recs, void* out_recs, void* out_norm);
    void check_flag();
    double effective_scale() const;
    size_t q_bytes(int rows) const;
    size_t rec_bytes() const;

    void decode(const dattn_batch& b, const void* q, void* out, void* row_partials, int mem);
    void micro_attention(const dattn_batch& b, const void* q_dev, void* partials);
    void decode_sharded(const dattn_batch& b, const void* q, void* out, int mem);
};
