// dattn_engine.cpp -- host engine behind the C ABI (include/dattn.h): the
// paged KV store and its page ledger, the decode planner (ranges -> MA work
// items -> partial records), kernel launches, and the NCCL partial exchange.
#include <nccl.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "dattn.h"
#include "dattn_engine.h"
#include "dattn_internal.h"

using namespace dattn;

namespace dattn {

thread_local std::string g_last_error = "";
thread_local int64_t g_launches = 0;

void set_error(const std::string& s) { g_last_error = s; }

Error::Error(dattn_status s, const std::string& m) : std::runtime_error(m), status(s) {}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Error(DATTN_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

static void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw Error(DATTN_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

void count_launch(int n) { g_launches += n; }

// Scratch buffers grow geometrically and start with 25 % slack: a decode loop
// whose plan or chunk count creeps up by a few words per step reallocates (a
// synchronising cudaFree / cudaFreeHost, 3-30 ms measured on the config-2
// decode loop) O(log) times, and not at all for the first quarter of growth.
void DevBuf::ensure(size_t bytes) {
    if (bytes <= cap) return;
    if (p) cudaFree(p);
    p = nullptr;
    const size_t grown = cap + cap / 2;
    cap = 0;
    size_t want = std::max<size_t>({bytes + bytes / 4, grown, 256});
    cuda_check(cudaMalloc(&p, want), "cudaMalloc");
    cap = want;
}
DevBuf::~DevBuf() {
    if (p) cudaFree(p);
}
void HostBuf::ensure(size_t bytes) {
    if (bytes <= cap) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    const size_t grown = cap + cap / 2;
    cap = 0;
    size_t want = std::max<size_t>({bytes + bytes / 4, grown, 256});
    cuda_check(cudaMallocHost(&p, want), "cudaMallocHost");
    cap = want;
}
HostBuf::~HostBuf() {
    if (p) cudaFreeHost(p);
}

int padded_dim_for(int head_dim) {
    for (int dp : {16, 32, 64, 128, 256, 512})
        if (head_dim <= dp) return dp;
    return -1;
}

int elem_bytes_for(int dtype) { return dtype == kBF16 ? 2 : (dtype == kF32 ? 4 : 8); }

}  // namespace dattn

// ------------------------------------------------------------------ store

void dattn_store::release_exchange() {
    for (int r = 0; r < 8; ++r) {
        if (r != rank && peer_x[r]) cudaIpcCloseMemHandle(peer_x[r]);
        peer_x[r] = nullptr;
    }
    if (xbuf) cudaFree(xbuf);
    xbuf = nullptr;
    fused_merge = false;
}

void dattn_store::release_peer_pools() {
    if (mig_stream) cudaStreamSynchronize(mig_stream);
    for (int r = 0; r < 8; ++r) {
        if (r != rank) {
            if (peer_kpool[r]) cudaIpcCloseMemHandle(peer_kpool[r]);
            if (peer_vpool[r]) cudaIpcCloseMemHandle(peer_vpool[r]);
        }
        peer_kpool[r] = peer_vpool[r] = nullptr;
        peer_pages[r] = 0;
    }
    mig_pending = 0;
}

// Map every rank's K and V pools into this process (CUDA IPC, handles
// all-gathered over the communicator) so dattn_kv_pull can copy a peer's
// pages straight into this store's pages over NVLink.
void dattn_store::setup_peer_pools() {
    release_peer_pools();
    const char* env = std::getenv("DATTN_PEER_POOLS");
    if ((env && std::atoi(env) == 0) || nranks > kMaxRanks) return;
    if (!mig_stream) {
        int lo = 0, hi = 0;
        cuda_check(cudaDeviceGetStreamPriorityRange(&lo, &hi), "cudaDeviceGetStreamPriorityRange");
        cuda_check(cudaStreamCreateWithPriority(&mig_stream, cudaStreamNonBlocking, lo), "cudaStreamCreate(mig)");
        cuda_check(cudaEventCreateWithFlags(&mig_ev, cudaEventDisableTiming), "cudaEventCreate(mig)");
    }
    // per rank: K handle, V handle, pool size in pages
    constexpr size_t kH = sizeof(cudaIpcMemHandle_t);
    constexpr size_t kRec = 2 * kH + sizeof(int64_t);
    unsigned char rec[kRec];
    cudaIpcMemHandle_t h[2];
    cuda_check(cudaIpcGetMemHandle(&h[0], kpool), "cudaIpcGetMemHandle(k)");
    cuda_check(cudaIpcGetMemHandle(&h[1], vpool), "cudaIpcGetMemHandle(v)");
    std::memcpy(rec, h, 2 * kH);
    std::memcpy(rec + 2 * kH, &cfg.num_pages, sizeof(int64_t));
    std::vector<unsigned char> all(kRec * nranks);
    DevBuf dh;
    dh.ensure(all.size());
    unsigned char* mine = static_cast<unsigned char*>(dh.p) + rank * kRec;
    cuda_check(cudaMemcpyAsync(mine, rec, kRec, cudaMemcpyHostToDevice, stream), "cudaMemcpyAsync");
    nccl_check(ncclAllGather(mine, dh.p, kRec, ncclUint8, comm, comm_begin()), "ncclAllGather(pool handles)");
    comm_end();
    cuda_check(cudaMemcpyAsync(all.data(), dh.p, all.size(), cudaMemcpyDeviceToHost, stream), "cudaMemcpyAsync");
    cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
    for (int r = 0; r < nranks; ++r) {
        std::memcpy(&peer_pages[r], all.data() + r * kRec + 2 * kH, sizeof(int64_t));
        if (r == rank) {
            peer_kpool[r] = kpool;
            peer_vpool[r] = vpool;
            continue;
        }
        cudaIpcMemHandle_t px[2];
        std::memcpy(px, all.data() + r * kRec, 2 * kH);
        cuda_check(cudaIpcOpenMemHandle(&peer_kpool[r], px[0], cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle(k)");
        cuda_check(cudaIpcOpenMemHandle(&peer_vpool[r], px[1], cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle(v)");
    }
}

// Order NCCL work after `stream`'s queued work, on the comm stream; comm_end()
// orders later `stream` work after it.
cudaStream_t dattn_store::comm_begin() {
    if (!comm_stream) {
        cuda_check(cudaStreamCreateWithFlags(&comm_stream, cudaStreamNonBlocking), "cudaStreamCreate(comm)");
        for (auto& e : comm_ev) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    }
    cuda_check(cudaEventRecord(comm_ev[0], stream), "cudaEventRecord");
    cuda_check(cudaStreamWaitEvent(comm_stream, comm_ev[0], 0), "cudaStreamWaitEvent");
    return comm_stream;
}

void dattn_store::comm_end() {
    cuda_check(cudaEventRecord(comm_ev[1], comm_stream), "cudaEventRecord");
    cuda_check(cudaStreamWaitEvent(stream, comm_ev[1], 0), "cudaStreamWaitEvent");
}

// Map every rank's exchange buffers into this process (CUDA IPC); the 64-byte
// handles travel through the NCCL communicator itself.
void dattn_store::setup_exchange() {
    release_exchange();
    const char* env = std::getenv("DATTN_FUSED_MERGE");
    if ((env && std::atoi(env) == 0) || nranks > kMaxRanks) return;
    slot_stride = static_cast<int64_t>(cfg.max_seqs) * cfg.num_q_heads;
    // two halves, used by alternate steps (epoch parity): a rank that runs one
    // step ahead never writes into the half a slower peer still reads
    xhalf = static_cast<size_t>(nranks) * slot_stride * rec_bytes();
    const size_t xbytes = 2 * xhalf;
    // poll control: device abort / status words, host-mapped status copy, timeout
    if (!x_status_host)
        cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&x_status_host), 64, cudaHostAllocMapped), "cudaHostAlloc");
    if (!x_ctl_dev) cuda_check(cudaMalloc(&x_ctl_dev, 64), "cudaMalloc(exchange control)");
    if (!abort_stream)
        cuda_check(cudaStreamCreateWithFlags(&abort_stream, cudaStreamNonBlocking), "cudaStreamCreate(abort)");
    cuda_check(cudaMemsetAsync(x_ctl_dev, 0, 64, stream), "cudaMemset(exchange control)");
    *reinterpret_cast<volatile int*>(x_status_host) = 0;
    const char* tenv = std::getenv("DATTN_EXCHANGE_TIMEOUT_S");
    const double tsec = tenv ? std::atof(tenv) : 60.0;
    x_timeout_ns = static_cast<unsigned long long>((tsec > 0 ? tsec : 60.0) * 1e9);
    // every CTA of K5 / K6 must be resident at once (their polls wait on
    // records other CTAs of the same grid push): cap the grid at occupancy
    for (int kind = 0; kind < 2; ++kind) {
        int occ = 0;
        cuda_check(exchange_occupancy(cfg.dtype, dp, kind, &occ), "occupancy(exchange)");
        x_grid_cap[kind] = std::max(1, std::min(occ * num_sms, kMaxExchangeGrid));
    }
    cuda_check(cudaMalloc(&xbuf, xbytes), "cudaMalloc(exchange)");
    // every exchange word starts empty (all ones, see XWord in dattn_merge.cuh)
    cuda_check(cudaMemsetAsync(xbuf, 0xFF, xbytes, stream), "cudaMemset(exchange)");
    cudaIpcMemHandle_t hx;
    cuda_check(cudaIpcGetMemHandle(&hx, xbuf), "cudaIpcGetMemHandle");
    constexpr size_t kH = sizeof(cudaIpcMemHandle_t);
    std::vector<unsigned char> all(kH * nranks);
    DevBuf dh;
    dh.ensure(all.size());
    cuda_check(cudaMemcpyAsync(static_cast<unsigned char*>(dh.p) + rank * kH, &hx, kH, cudaMemcpyHostToDevice,
                               stream),
               "cudaMemcpyAsync");
    nccl_check(ncclAllGather(static_cast<unsigned char*>(dh.p) + rank * kH, dh.p, kH, ncclUint8, comm, comm_begin()),
               "ncclAllGather(ipc handles)");
    comm_end();
    cuda_check(cudaMemcpyAsync(all.data(), dh.p, all.size(), cudaMemcpyDeviceToHost, stream), "cudaMemcpyAsync");
    cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
    for (int r = 0; r < nranks; ++r) {
        if (r == rank) {
            peer_x[r] = xbuf;
            continue;
        }
        cudaIpcMemHandle_t px;
        std::memcpy(&px, all.data() + r * kH, kH);
        cuda_check(cudaIpcOpenMemHandle(&peer_x[r], px, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    }
    // every rank has emptied its exchange buffer before anyone can push
    nccl_check(ncclAllGather(static_cast<unsigned char*>(dh.p) + rank * kH, dh.p, kH, ncclUint8, comm, comm_begin()),
               "ncclAllGather(barrier)");
    comm_end();
    cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
    epoch = 0;
    fused_merge = true;
}

// A poll of an earlier step gave up (abort word or timeout): that step's
// output is invalid and the exchange words are in an unknown state.
void dattn_store::check_exchange_status() const {
    if (!x_status_host) return;
    const int st = *reinterpret_cast<const volatile int*>(x_status_host);
    if (st == kXAbortHost)
        throw Error(DATTN_ERR_NCCL, "NVLink exchange aborted by dattn_comm_abort; call dattn_comm_init to rebuild it");
    if (st == kXTimeout)
        throw Error(DATTN_ERR_NCCL, "NVLink exchange: a peer's record did not arrive within DATTN_EXCHANGE_TIMEOUT_S "
                                    "(a rank failed or stalled); call dattn_comm_init to rebuild the exchange");
}

dattn_store::~dattn_store() {
    if (k5_trace.p) {
        // DATTN_K5_TRACE summary over all calls: per-CTA mean phase-A and total
        // durations, then the mean and max over CTAs
        std::vector<unsigned long long> t(static_cast<size_t>(kMaxExchangeGrid) * 3);
        if (cudaMemcpy(t.data(), k5_trace.p, t.size() * 8, cudaMemcpyDeviceToHost) == cudaSuccess) {
            double a_sum = 0, a_max = 0, e_sum = 0, e_max = 0;
            int n = 0;
            for (int c = 0; c < kMaxExchangeGrid; ++c) {
                if (!t[c * 3 + 2]) continue;
                const double a = 1e-3 * t[c * 3] / t[c * 3 + 2], e = 1e-3 * t[c * 3 + 1] / t[c * 3 + 2];
                a_sum += a;
                e_sum += e;
                a_max = std::max(a_max, a);
                e_max = std::max(e_max, e);
                ++n;
            }
            if (n)
                std::fprintf(stderr,
                             "[K5 trace rank %d] %d CTAs x %llu calls: phase A mean %.2f max %.2f us; "
                             "CTA total mean %.2f max %.2f us\n",
                             rank, n, t[2], a_sum / n, a_max, e_sum / n, e_max);
        }
    }
    release_exchange();
    release_peer_pools();
    if (mig_ev) cudaEventDestroy(mig_ev);
    if (mig_stream) cudaStreamDestroy(mig_stream);
    if (x_status_host) cudaFreeHost(x_status_host);
    if (x_ctl_dev) cudaFree(x_ctl_dev);
    if (abort_stream) cudaStreamDestroy(abort_stream);
    if (comm) ncclCommDestroy(comm);
    for (auto& e : comm_ev)
        if (e) cudaEventDestroy(e);
    if (comm_stream) cudaStreamDestroy(comm_stream);
    for (auto* v : {&ma_events, &merge_events, &comm_events})
        for (auto& pr : *v) {
            cudaEventDestroy(pr[0]);
            cudaEventDestroy(pr[1]);
        }
    if (kpool) cudaFree(kpool);
    if (vpool) cudaFree(vpool);
    if (d_bt) cudaFree(d_bt);
    if (d_counter) cudaFree(d_counter);
    if (d_flag) cudaFree(d_flag);
    if (meta_ev) cudaEventDestroy(meta_ev);
    if (app_ev) cudaEventDestroy(app_ev);
    if (own_stream) cudaStreamDestroy(own_stream);
}

void dattn_store::activate() const { cuda_check(cudaSetDevice(cfg.device), "cudaSetDevice"); }

static void validate_config(const dattn_store_config& c) {
    if (c.head_dim < 1 || c.head_dim > 512)
        throw Error(DATTN_ERR_CONTRACT, "head_dim must be in [1, 512]");
    if (c.num_q_heads < 1 || c.num_kv_heads < 1)
        throw Error(DATTN_ERR_CONTRACT, "head counts must be >= 1");
    if (c.num_q_heads % c.num_kv_heads != 0)
        throw Error(DATTN_ERR_CONTRACT, "num_q_heads must be a multiple of num_kv_heads");
    if (!std::isfinite(c.scale) || c.scale < 0.0)
        throw Error(DATTN_ERR_CONTRACT, "scale must be finite and >= 0");
    if (c.dtype < 0 || c.dtype > 2) throw Error(DATTN_ERR_INVALID_ARGUMENT, "unknown dtype");
    if (c.page_tokens < 1) throw Error(DATTN_ERR_CONTRACT, "page_tokens must be >= 1");
    if (c.num_pages < 1 || c.num_pages > (int64_t(1) << 31) - 1)
        throw Error(DATTN_ERR_CONTRACT, "num_pages out of range");
    if (c.max_seqs < 1 || c.max_pages_per_seq < 1)
        throw Error(DATTN_ERR_CONTRACT, "block-table shape must be >= 1");
    if (c.num_kv_heads > 255) throw Error(DATTN_ERR_CONTRACT, "num_kv_heads must be <= 255");
}

void dattn_store::init(const dattn_store_config& c) {
    validate_config(c);
    cfg = c;
    dp = padded_dim_for(c.head_dim);
    esz = elem_bytes_for(c.dtype);
    acc_sz = c.dtype == kF64 ? 8 : 4;
    rec_elems = dp + 4;
    group = c.num_q_heads / c.num_kv_heads;
    activate();
    cuda_check(cudaStreamCreateWithFlags(&own_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    stream = own_stream;
    cuda_check(cudaEventCreateWithFlags(&meta_ev, cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaEventCreateWithFlags(&app_ev, cudaEventDisableTiming), "cudaEventCreate");
    int dev = c.device;
    cuda_check(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev),
               "cudaDeviceGetAttribute");
    page_elems = static_cast<int64_t>(c.num_kv_heads) * c.page_tokens * dp;
    const size_t pool = static_cast<size_t>(c.num_pages) * page_elems * esz;
    cuda_check(cudaMalloc(&kpool, pool), "cudaMalloc(K pool)");
    cuda_check(cudaMalloc(&vpool, pool), "cudaMalloc(V pool)");
    cuda_check(cudaMemsetAsync(kpool, 0, pool, stream), "cudaMemset");
    cuda_check(cudaMemsetAsync(vpool, 0, pool, stream), "cudaMemset");
    const size_t bt = static_cast<size_t>(c.max_seqs) * c.max_pages_per_seq * sizeof(int32_t);
    cuda_check(cudaMalloc(&d_bt, bt), "cudaMalloc(block tables)");
    cuda_check(cudaMemsetAsync(d_bt, 0, bt, stream), "cudaMemset");
    cuda_check(cudaMalloc(&d_counter, 64), "cudaMalloc");
    cuda_check(cudaMemsetAsync(d_counter, 0, 64, stream), "cudaMemset");
    cuda_check(cudaMalloc(&d_flag, 64), "cudaMalloc");
    h_bt.assign(static_cast<size_t>(c.max_seqs) * c.max_pages_per_seq, 0);
    seq_tokens.assign(c.max_seqs, 0);
    seq_pages.assign(c.max_seqs, 0);
    seq_live.assign(c.max_seqs, 0);
    free_pages.reserve(c.num_pages);
    for (int64_t i = c.num_pages - 1; i >= 0; --i) free_pages.push_back(static_cast<int32_t>(i));
    for (int i = c.max_seqs - 1; i >= 0; --i) free_seqs.push_back(i);

    // K1 covers groups up to 16 (8 for fp64) and rows up to 256 wide; other
    // shapes run on the generic K1g (MQA, head_dim 257..512)
    ma_generic = !ma_supported(c.dtype, dp, group);
    if (ma_generic) {
        int occ = 0;
        cuda_check(ma_generic_occupancy(c.dtype, dp, &occ), "occupancy(K1g)");
        ma_ctas_per_sm = std::max(1, occ);
    }
    // MA launch geometry: the deepest ring that still fits the target CTAs/SM.
    const char* env_ctas = std::getenv("DATTN_MA_CTAS");
    const char* env_stages = std::getenv("DATTN_MA_STAGES");
    int want_ctas = (c.dtype == kF64 || group > 8) ? 1 : 2;
    if (env_ctas) want_ctas = std::max(1, std::atoi(env_ctas));
    const size_t sm_total = 233472;  // 228 KB per SM
    int stages = 2;
    for (int s = 2; s <= 12; ++s) {
        const size_t need = ma_smem_bytes(c.dtype, dp, group, s);
        if ((need + 1024) * want_ctas <= sm_total && need <= 232448) stages = s;
    }
    if (env_stages) stages = std::max(2, std::atoi(env_stages));
    if (!ma_generic) {
        ma_stages = stages;
        ma_smem = ma_smem_bytes(c.dtype, dp, group, stages);
        cuda_check(ma_configure(c.dtype, dp, group, ma_smem), "cudaFuncSetAttribute(MA)");
        int occ = 0;
        cuda_check(ma_occupancy(c.dtype, dp, group, ma_smem, &occ), "occupancy(MA)");
        ma_ctas_per_sm = std::max(1, occ);
    }

    // K2: tcgen05 tiles for grouped queries (bf16, d = 128, pages dividing the 128-token tile)
    // MHA (group 1) too: Q is padded to the MMA's N = 16 like any group, and
    // the tensor-core tile costs less power than K1's FFMA2 stream
    const bool tc_shape = c.dtype == kBF16 && c.head_dim == 128 && group >= 1 && group <= 16 &&
                          (c.page_tokens == 16 || c.page_tokens == 32 || c.page_tokens == 64 ||
                           c.page_tokens == 128);
    if (tc_shape && !std::getenv("DATTN_DISABLE_TC")) {
        const uint64_t rows = static_cast<uint64_t>(c.num_pages) * c.num_kv_heads * c.page_tokens;
        cuda_check(make_tmap_rows128(tm_k, kpool, rows, c.page_tokens), "tensor map (K pool)");
        cuda_check(make_tmap_rows128(tm_v, vpool, rows, c.page_tokens), "tensor map (V pool)");
        cuda_check(make_tmap_tiles(tm_k4, kpool, c.num_pages, c.num_kv_heads, c.page_tokens), "tensor map (K tiles)");
        cuda_check(make_tmap_tiles(tm_v4, vpool, c.num_pages, c.num_kv_heads, c.page_tokens), "tensor map (V tiles)");
        cuda_check(gqa_tc_configure(), "cudaFuncSetAttribute(K2)");
        tc_ok = true;
    }
    cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
}

void dattn_store::upload_bt_row(int32_t seq) {
    const size_t off = static_cast<size_t>(seq) * cfg.max_pages_per_seq;
    const int32_t n = seq_pages[seq];
    if (n == 0) return;
    cuda_check(cudaMemcpyAsync(d_bt + off, h_bt.data() + off, sizeof(int32_t) * n,
                               cudaMemcpyHostToDevice, stream),
               "cudaMemcpyAsync(block table)");
}

void dattn_store::check_seq(int32_t seq) const {
    if (seq < 0 || seq >= cfg.max_seqs || !seq_live[seq])
        throw Error(DATTN_ERR_CONTRACT, "unknown sequence id " + std::to_string(seq));
}

void dattn_store::grow(int32_t seq, int64_t tokens) {
    const int64_t need = (tokens + cfg.page_tokens - 1) / cfg.page_tokens;  // blocks_for_tokens
    if (need > cfg.max_pages_per_seq)
        throw Error(DATTN_ERR_CAPACITY, "sequence exceeds max_pages_per_seq");
    const int64_t add = need - seq_pages[seq];
    if (add > static_cast<int64_t>(free_pages.size()))
        throw Error(DATTN_ERR_CAPACITY, "page pool exhausted");
    const size_t off = static_cast<size_t>(seq) * cfg.max_pages_per_seq;
    for (int64_t i = 0; i < add; ++i) {
        h_bt[off + seq_pages[seq] + i] = free_pages.back();
        free_pages.pop_back();
    }
    if (add > 0) {
        seq_pages[seq] = static_cast<int32_t>(need);
        used_pages += add;
        upload_bt_row(seq);
    }
    seq_tokens[seq] = std::max(seq_tokens[seq], tokens);
}

// ----------------------------------------------------------------- planner

// Steady-state decode repeats the same batch: reuse the last plan when the
// batch is identical (after re-checking the ranges against the ledger).
void dattn_store::plan(const dattn_batch& b, bool one_chunk_per_range, Plan& pl) {
    const size_t rbytes = static_cast<size_t>(std::max(b.num_ranges, 0)) * sizeof(dattn_range);
    const bool same = plan_cached && cache_one_chunk == one_chunk_per_range && cache_rows == b.num_rows &&
                      cache_chunk == b.chunk_tokens && b.num_ranges >= 0 && b.ranges != nullptr &&
                      cache_ranges.size() == rbytes &&
                      std::memcmp(cache_ranges.data(), b.ranges, rbytes) == 0;
    if (same && &pl == &cache_plan) {
        for (int i = 0; i < b.num_ranges; ++i) {
            const dattn_range& r = b.ranges[i];
            check_seq(r.seq);
            if (r.tok_end > seq_tokens[r.seq]) throw Error(DATTN_ERR_CONTRACT, "range tokens outside the sequence");
        }
        return;
    }
    build_plan(b, one_chunk_per_range, pl);
    if (&pl == &cache_plan) {
        plan_cached = true;
        cache_one_chunk = one_chunk_per_range;
        cache_rows = b.num_rows;
        cache_chunk = b.chunk_tokens;
        cache_ranges.assign(reinterpret_cast<const unsigned char*>(b.ranges),
                            reinterpret_cast<const unsigned char*>(b.ranges) + rbytes);
    }
}

void dattn_store::build_plan(const dattn_batch& b, bool one_chunk_per_range, Plan& pl) const {
    if (b.num_rows < 0 || b.num_ranges < 0)
        throw Error(DATTN_ERR_INVALID_ARGUMENT, "negative row/range count");
    if (b.num_ranges > 0 && !b.ranges)
        throw Error(DATTN_ERR_INVALID_ARGUMENT, "ranges is null");
    int nr = b.num_ranges;
    int64_t work = 0, max_len = 0;
    int prev_row = -1;
    for (int i = 0; i < nr; ++i) {
        const dattn_range& r = b.ranges[i];
        check_seq(r.seq);
        if (r.out_row < 0 || r.out_row >= b.num_rows)
            throw Error(DATTN_ERR_CONTRACT, "range out_row out of bounds");
        if (r.out_row < prev_row) throw Error(DATTN_ERR_CONTRACT, "ranges must be sorted by out_row");
        prev_row = r.out_row;
        if (r.kv_head < -1 || r.kv_head >= cfg.num_kv_heads)
            throw Error(DATTN_ERR_CONTRACT, "range kv_head out of bounds");
        if (r.tok_begin < 0 || r.tok_begin > r.tok_end || r.tok_end > seq_tokens[r.seq])
            throw Error(DATTN_ERR_CONTRACT, "range tokens outside the sequence");
        if (r.tok_end > INT32_MAX) throw Error(DATTN_ERR_CONTRACT, "range too long");
        const int64_t len = r.tok_end - r.tok_begin;
        work += len * (r.kv_head < 0 ? cfg.num_kv_heads : 1);
        max_len = std::max(max_len, len);
    }
    int64_t C;
    if (one_chunk_per_range) {
        C = std::max<int64_t>(max_len, 1);
    } else if (b.chunk_tokens > 0) {
        C = b.chunk_tokens;
    } else {
        // ~12 items per CTA slot for K1 and ~6 for K2 (whose items cost a
        // pipeline drain each: 2048-token chunks 2-3% slower than 4096 at the
        // same wave count, 1024-token chunks 8%). ma_ctas_per_sm is K1's
        // occupancy (2 for bf16), so K2 -- one CTA per SM -- gets ~12 items per
        // SM: measured better than ~6 at N = 4 (config 3: 0.313 vs 0.320 ms per
        // rank with 2048- vs 4096-token chunks; config 4: 0.585 vs 0.620 with
        // 4096 vs 8192), where the shares are small and the tail matters more
        const int64_t target = static_cast<int64_t>(num_sms) * ma_ctas_per_sm * (tc_ok ? 6 : 12);
        int64_t c = std::max<int64_t>(work / std::max<int64_t>(target, 1), 1);
        int64_t p2 = 1;
        while (p2 * 2 <= c) p2 *= 2;
        // floor 512 tokens: below it the per-item cost outweighs the extra
        // parallelism (config 1, 4K fp32 tokens x 32 heads: 64-token chunks
        // 36.7 us per step, 512-token chunks 29.6 us)
        const int64_t lo = std::max<int64_t>(512, tc_ok ? 128 : ma_stage_tokens(cfg.dtype, dp));
        C = std::min<int64_t>(std::max<int64_t>(p2, lo), 8192);
        if (C % cfg.page_tokens) C = (C / cfg.page_tokens + 1) * cfg.page_tokens;
    }
    if (C > INT32_MAX) throw Error(DATTN_ERR_CONTRACT, "chunk too long");
    pl.chunk_tokens = static_cast<int32_t>(C);

    // Fine tail for uniform batches: when every range is a whole number of
    // full chunks, the last wave of items would be full chunks too and the
    // grid would drain over one chunk's streaming time. The trailing chunks
    // of some ranges are then cut into sub-ranges of C/4 tokens (partial
    // chunks), which the longest-first claim order below runs last: about two
    // waves of quarter items end the launch. Same records and merges; only
    // the chunk boundaries move (partition invariance).
    const dattn_range* R = b.ranges;
    std::vector<dattn_range> split;
    // K2 runs one CTA per SM. Chunks from 2048 tokens are cut (quarters of
    // 512+ tokens): with K2 fetching its next item during the current one's
    // last tiles, short items are cheap (config 3 at N = 4, C = 2048: -3.7 us
    // per step; without that prefetch the same cut cost +2.4 us; C = 4096 /
    // 8192: -8 / -17 us)
    const int64_t slots = static_cast<int64_t>(num_sms) * (tc_ok ? 1 : ma_ctas_per_sm);
    static const bool fine_tail_off = std::getenv("DATTN_NO_FINE_TAIL") != nullptr;  // A/B switch
    static const int64_t fine_tail_min = [] {  // smallest chunk cut into quarters (A/B: DATTN_FINE_TAIL_MIN)
        const char* e = std::getenv("DATTN_FINE_TAIL_MIN");
        return e ? std::max<int64_t>(64, std::atoll(e)) : int64_t{2048};
    }();
    if (!fine_tail_off && !one_chunk_per_range && b.chunk_tokens <= 0 &&
        C >= (tc_ok ? fine_tail_min : std::max<int64_t>(fine_tail_min, 4096)) &&  // K1: no item prefetch
        C % (4 * cfg.page_tokens) == 0) {
        bool uniform = nr > 0;
        int64_t nh_sum = 0, natural = 0;
        for (int i = 0; i < nr && uniform; ++i) {
            const int64_t len = R[i].tok_end - R[i].tok_begin;
            if (len > 0 && (len % C != 0 || len < 2 * C)) uniform = false;
            const int nh = R[i].kv_head < 0 ? cfg.num_kv_heads : 1;
            if (len > 0) nh_sum += nh;
            natural += len / C * nh;
        }
        // only when there is a last wave to shorten (at least two waves of items)
        if (uniform && nh_sum > 0 && natural >= 2 * slots) {
            const int64_t want = 2 * slots;  // quarter items wanted
            // chunks to cut per range (round robin over the ranges, at most
            // all but one of a range's chunks)
            const int64_t per_range = std::max<int64_t>(1, (want + 4 * nh_sum - 1) / (4 * nh_sum));
            split.reserve(static_cast<size_t>(nr) * (1 + 4 * per_range));
            const int64_t q = C / 4;
            for (int i = 0; i < nr; ++i) {
                dattn_range r = R[i];
                const int64_t len = r.tok_end - r.tok_begin;
                const int64_t k = len > 0 ? std::min(per_range, len / C - 1) : 0;
                r.tok_end = R[i].tok_end - k * C;
                split.push_back(r);
                for (int64_t j = 0; j < 4 * k; ++j) {
                    dattn_range s2 = R[i];
                    s2.tok_begin = r.tok_end + j * q;
                    s2.tok_end = s2.tok_begin + q;
                    split.push_back(s2);
                }
            }
            R = split.data();
            nr = static_cast<int>(split.size());
        }
    }

    // layout of the metadata buffer (int32 words)
    pl.off_ranges = 0;
    pl.off_item = pl.off_ranges + 8 * nr;
    pl.off_chunk = pl.off_item + nr + 1;
    pl.off_rowchunk = pl.off_chunk + nr + 1;
    pl.off_kvh = pl.off_rowchunk + b.num_rows + 1;
    // first pass: counts
    pl.words.assign(pl.off_kvh, 0);
    int64_t items = 0, chunks = 0;
    std::vector<int32_t> row_chunks(b.num_rows, 0);
    for (int i = 0; i < nr; ++i) {
        const dattn_range& r = R[i];
        const int64_t len = r.tok_end - r.tok_begin;
        const int64_t nch = len > 0 ? (len + C - 1) / C : 0;
        const int nh = r.kv_head < 0 ? cfg.num_kv_heads : 1;
        RangeDev rd{r.seq, r.out_row, r.kv_head, static_cast<int32_t>(r.tok_begin),
                    static_cast<int32_t>(r.tok_end), {0, 0, 0}};
        std::memcpy(&pl.words[pl.off_ranges + 8 * i], &rd, sizeof(rd));
        pl.words[pl.off_item + i] = static_cast<int32_t>(items);
        pl.words[pl.off_chunk + i] = one_chunk_per_range ? i : static_cast<int32_t>(chunks);
        items += nch * nh;
        chunks += nch;
        row_chunks[r.out_row] += static_cast<int32_t>(nch);
        if (items > INT32_MAX) throw Error(DATTN_ERR_CONTRACT, "too many work items");
    }
    pl.words[pl.off_item + nr] = static_cast<int32_t>(items);
    pl.words[pl.off_chunk + nr] = one_chunk_per_range ? nr : static_cast<int32_t>(chunks);
    int32_t acc = 0;
    for (int rrow = 0; rrow < b.num_rows; ++rrow) {
        pl.words[pl.off_rowchunk + rrow] = acc;
        acc += row_chunks[rrow];
    }
    pl.words[pl.off_rowchunk + b.num_rows] = acc;
    pl.words.resize(pl.off_kvh + static_cast<size_t>(chunks));
    bool any_kvh = false;
    int64_t c = 0;
    for (int i = 0; i < nr; ++i) {
        const dattn_range& r = R[i];
        const int64_t len = r.tok_end - r.tok_begin;
        const int64_t nch = len > 0 ? (len + C - 1) / C : 0;
        for (int64_t k = 0; k < nch; ++k) pl.words[pl.off_kvh + c++] = r.kv_head;
        any_kvh |= r.kv_head >= 0;
    }
    pl.any_kvh = any_kvh;
    // chunk records per (row, kv head): the completion count of the fused merge
    pl.off_expect = pl.words.size();
    pl.words.resize(pl.off_expect + static_cast<size_t>(b.num_rows) * cfg.num_kv_heads, 0);
    for (int i = 0; i < nr; ++i) {
        const dattn_range& r = R[i];
        const int64_t len = r.tok_end - r.tok_begin;
        const int64_t nch = len > 0 ? (len + C - 1) / C : 0;
        int32_t* e = &pl.words[pl.off_expect + static_cast<size_t>(r.out_row) * cfg.num_kv_heads];
        if (r.kv_head < 0)
            for (int k = 0; k < cfg.num_kv_heads; ++k) e[k] += static_cast<int32_t>(nch);
        else
            e[r.kv_head] += static_cast<int32_t>(nch);
    }
    pl.any_empty_group = false;
    for (size_t i = 0; i < static_cast<size_t>(b.num_rows) * cfg.num_kv_heads; ++i)
        pl.any_empty_group |= pl.words[pl.off_expect + i] == 0;
    // claim order: longest item first (LPT), so a ragged batch ends on short
    // items instead of one CTA finishing a long one alone; uniform items keep
    // the natural order (no table). Every chunk but a range's last is exactly
    // C tokens, so the order is: all full chunks in natural item order, then
    // the partial last chunks by length, longest first (ties in item order) --
    // a stable sort of the items by length, built from the ranges directly.
    pl.off_table = 0;
    if (!one_chunk_per_range && items > 1) {
        struct Tail {
            int32_t len, range;
        };
        std::vector<Tail> tails;  // ranges whose last chunk is shorter than C
        int32_t lmin = INT32_MAX, lmax = 0;
        for (int i = 0; i < nr; ++i) {
            const dattn_range& r = R[i];
            const int64_t len = r.tok_end - r.tok_begin;
            if (len <= 0) continue;
            const int32_t last = static_cast<int32_t>(len - (len - 1) / C * C);
            lmax = std::max<int32_t>(lmax, len > C ? static_cast<int32_t>(C) : last);
            lmin = std::min(lmin, last);
            if (last < C) tails.push_back({last, i});
        }
        if (lmax > lmin) {
            std::stable_sort(tails.begin(), tails.end(), [](const Tail& a, const Tail& b2) { return a.len > b2.len; });
            if (pl.words.size() & 1) pl.words.push_back(0);  // 8-B aligned pairs
            pl.off_table = pl.words.size();
            pl.words.resize(pl.off_table + 2 * static_cast<size_t>(items));
            int32_t* tab = &pl.words[pl.off_table];
            size_t k = 0;
            for (int i = 0; i < nr; ++i) {  // full chunks, natural order
                const dattn_range& r = R[i];
                const int64_t len = r.tok_end - r.tok_begin;
                if (len <= 0) continue;
                const int nh = r.kv_head < 0 ? cfg.num_kv_heads : 1;
                const int64_t nfull = len / C;
                for (int64_t l = 0; l < nfull * nh; ++l) {
                    tab[2 * k] = i;
                    tab[2 * k + 1] = static_cast<int32_t>(l);
                    ++k;
                }
            }
            for (const Tail& t : tails) {  // partial last chunks, longest first
                const dattn_range& r = R[t.range];
                const int nh = r.kv_head < 0 ? cfg.num_kv_heads : 1;
                const int64_t j = (r.tok_end - r.tok_begin - 1) / C;
                for (int h = 0; h < nh; ++h) {
                    tab[2 * k] = t.range;
                    tab[2 * k + 1] = static_cast<int32_t>(j * nh + h);
                    ++k;
                }
            }
        }
    }
    pl.nitems = static_cast<int32_t>(items);
    pl.nchunks = static_cast<int32_t>(one_chunk_per_range ? nr : chunks);
    pl.nranges = nr;
    pl.nrows = b.num_rows;
}

void dattn_store::upload_plan(const Plan& pl) {
    const size_t bytes = pl.words.size() * sizeof(int32_t);
    // steady-state decode repeats the same batch: the device copy is still valid
    if (meta_valid && pl.words == last_words) {
        stats.last_plan_bytes = 0;
        return;
    }
    stats.last_plan_bytes = static_cast<int64_t>(bytes);
    // the previous call's H2D copy must have consumed the pinned staging
    cuda_check(cudaEventSynchronize(meta_ev), "cudaEventSynchronize");
    h_meta.ensure(bytes);
    d_meta.ensure(bytes);
    std::memcpy(h_meta.p, pl.words.data(), bytes);
    cuda_check(cudaMemcpyAsync(d_meta.p, h_meta.p, bytes, cudaMemcpyHostToDevice, stream),
               "cudaMemcpyAsync(plan)");
    cuda_check(cudaEventRecord(meta_ev, stream), "cudaEventRecord");
    last_words = pl.words;
    meta_valid = true;
}

// In-kernel group merge (merge warp + completion counters; §5.4 of DESIGN.md)
// is opt-in with DATTN_FUSED_K1=1: measured on B200 it loses to the separate
// merge launches (K3 on one GPU, K5 across GPUs) because heavy groups finish
// at the very end of the MA kernel and their merge becomes its tail. The
// decision depends only on the environment, so every rank agrees.
bool dattn_store::fused_ok(const Plan& pl, bool check_finite) const {
    (void)pl;
    (void)check_finite;
    if (ma_generic && !tc_ok) return false;  // K1g has no merge warp
    const char* env = std::getenv("DATTN_FUSED_K1");
    return env && std::atoi(env) == 1;
}

void dattn_store::fill_fused(const Plan& pl, MAParams& f) {
    const size_t n = static_cast<size_t>(pl.nrows) * cfg.num_kv_heads;
    if (n > gcounter_elems) {
        gcounter.ensure(n * sizeof(int32_t));
        cuda_check(cudaMemsetAsync(gcounter.p, 0, n * sizeof(int32_t), stream), "cudaMemsetAsync(counters)");
        gcounter_elems = n;
    }
    const int32_t* w = static_cast<const int32_t*>(d_meta.p);
    f.group_counter = static_cast<int32_t*>(gcounter.p);
    f.group_expected = w + pl.off_expect;
    f.row_begin = w + pl.off_rowchunk;
    f.chunk_kvh = pl.any_kvh ? w + pl.off_kvh : nullptr;
}

void dattn_store::run_ma(const Plan& pl, const void* q_dev, void* recs, double scale,
                         bool check_finite, const MAParams* fused) {
    if (pl.nitems == 0) return;
    const int32_t* w = static_cast<const int32_t*>(d_meta.p);
    MAParams p{};
    if (fused) p = *fused;
    p.k_pool = kpool;
    p.v_pool = vpool;
    p.block_tables = d_bt;
    p.bt_stride = cfg.max_pages_per_seq;
    p.page_tokens = cfg.page_tokens;
    p.num_kv_heads = cfg.num_kv_heads;
    p.num_q_heads = cfg.num_q_heads;
    p.group = group;
    p.q = q_dev;
    p.ranges = reinterpret_cast<const RangeDev*>(w + pl.off_ranges);
    p.item_prefix = w + pl.off_item;
    p.item_table = pl.off_table ? w + pl.off_table : nullptr;
    p.chunk_prefix = w + pl.off_chunk;
    p.nranges = pl.nranges;
    p.nitems = pl.nitems;
    p.chunk_tokens = pl.chunk_tokens;
    static const int ahead = [] {  // DATTN_K2_AHEAD: A/B switch (0 = fetch at the item boundary)
        const char* e = std::getenv("DATTN_K2_AHEAD");
        return e ? std::max(0, std::atoi(e)) : 5;
    }();
    p.claim_ahead = ahead;
    const double s = scale > 0.0 ? scale : effective_scale();
    p.scale_log2 = s * 1.4426950408889634074;
    p.records = recs;
    p.work_counter = reinterpret_cast<unsigned long long*>(d_counter);
    p.work_base = work_base;
    p.nonfinite_flag = check_finite ? d_flag : nullptr;
    p.stages = ma_stages;
    const bool use_tc = tc_ok && !check_finite;
    int grid;
    if (use_tc) {
        if (tm_q_ptr != q_dev || tm_q_rows != pl.nrows) {
            cuda_check(make_tmap_rows128(tm_q, q_dev, static_cast<uint64_t>(std::max(pl.nrows, 1)) *
                                                          cfg.num_q_heads, group),
                       "tensor map (q)");
            tm_q_ptr = q_dev;
            tm_q_rows = pl.nrows;
        }
        grid = std::max(1, std::min(pl.nitems, num_sms));
    } else {
        grid = std::max(1, std::min(pl.nitems, num_sms * ma_ctas_per_sm));
    }
    cudaEvent_t* ev = timing ? timer_pair(0) : nullptr;
    if (ev) cuda_check(cudaEventRecord(ev[0], stream), "cudaEventRecord");
    if (use_tc)
        cuda_check(launch_gqa_tc(tm_k, tm_v, tm_q, tm_k4, tm_v4, p, grid, stream), "launch(K2 tcgen05)");
    else if (ma_generic)
        cuda_check(launch_ma_generic(cfg.dtype, dp, p, grid, stream), "launch(K1g)");
    else
        cuda_check(launch_ma(cfg.dtype, dp, p, grid, ma_smem, stream), "launch(MA)");
    if (ev) cuda_check(cudaEventRecord(ev[1], stream), "cudaEventRecord");
    // every CTA's producer claims items until one past the end: the counter
    // advances by exactly nitems + grid per launch
    work_base += static_cast<unsigned long long>(pl.nitems) + static_cast<unsigned long long>(grid);
    count_launch(1);
    stats.ma_launches++;
    stats.last_items = pl.nitems;
    stats.last_chunks = pl.nchunks;
    stats.last_chunk_tokens = pl.chunk_tokens;
    stats.ma_grid = grid;
    stats.last_kernel = use_tc ? 2 : (ma_generic ? 3 : 1);
}

double dattn_store::effective_scale() const {
    return cfg.scale > 0.0 ? cfg.scale : 1.0 / std::sqrt(static_cast<double>(cfg.head_dim));
}

void dattn_store::run_merge(const MergeParams& mp) {
    cudaEvent_t* ev = timing ? timer_pair(1) : nullptr;
    if (ev) cuda_check(cudaEventRecord(ev[0], stream), "cudaEventRecord");
    cuda_check(launch_merge(cfg.dtype, dp, mp, stream), "launch(merge)");
    if (ev) cuda_check(cudaEventRecord(ev[1], stream), "cudaEventRecord");
    count_launch(1);
    stats.merge_launches++;
}

// Event pairs around every MA (kind 0) / merge (kind 1) launch while timing
// is on; summed by dattn_store_get_stats.
cudaEvent_t* dattn_store::timer_pair(int kind) {
    auto& v = kind == 0 ? ma_events : (kind == 1 ? merge_events : comm_events);
    auto& used = kind == 0 ? ma_events_used : (kind == 1 ? merge_events_used : comm_events_used);
    if (used == v.size()) {
        std::array<cudaEvent_t, 2> pr{};
        cuda_check(cudaEventCreate(&pr[0]), "cudaEventCreate");
        cuda_check(cudaEventCreate(&pr[1]), "cudaEventCreate");
        v.push_back(pr);
    }
    return v[used++].data();
}

void dattn_store::collect_timing() {
    cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
    for (int kind = 0; kind < 3; ++kind) {
        auto& v = kind == 0 ? ma_events : (kind == 1 ? merge_events : comm_events);
        auto& used = kind == 0 ? ma_events_used : (kind == 1 ? merge_events_used : comm_events_used);
        double total = 0.0;
        for (size_t i = 0; i < used; ++i) {
            float ms = 0.f;
            cuda_check(cudaEventElapsedTime(&ms, v[i][0], v[i][1]), "cudaEventElapsedTime");
            total += ms;
        }
        if (kind == 0) { stats.ma_ms += total; stats.ma_timed += used; }
        else if (kind == 1) { stats.merge_ms += total; stats.merge_timed += used; }
        else { stats.comm_ms += total; stats.comm_timed += used; }
        used = 0;
    }
}

void dattn_store::local_merge(const Plan& pl, const void* recs, void* out_recs, void* out_norm) {
    const int32_t* w = static_cast<const int32_t*>(d_meta.p);
    MergeParams mp{};
    mp.recs = recs;
    mp.rows = pl.nrows;
    mp.heads = cfg.num_q_heads;
    mp.row_begin = w + pl.off_rowchunk;
    mp.row_mul = cfg.num_q_heads;
    mp.c_stride = cfg.num_q_heads;
    mp.chunk_kvh = pl.any_kvh ? w + pl.off_kvh : nullptr;
    mp.group = group;
    mp.out_recs = out_recs;
    mp.out_norm = out_norm;
    run_merge(mp);
}

size_t dattn_store::q_bytes(int rows) const {
    return static_cast<size_t>(rows) * cfg.num_q_heads * dp * esz;
}
size_t dattn_store::rec_bytes() const { return static_cast<size_t>(rec_elems) * acc_sz; }

void dattn_store::check_flag() {
    int32_t flag = 0;
    cuda_check(cudaMemcpyAsync(&flag, d_flag, sizeof(int32_t), cudaMemcpyDeviceToHost, stream),
               "cudaMemcpyAsync(flag)");
    cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
    if (flag) throw Error(DATTN_ERR_INPUT, "segment contains non-finite values");
}

void dattn_store::decode(const dattn_batch& b, const void* q, void* out, void* row_partials,
                         int mem) {
    activate();
    Plan& pl = cache_plan;
    plan(b, false, pl);
    upload_plan(pl);
    const bool want_out = out && !(b.flags & DATTN_F_NO_OUTPUT);
    const void* q_dev = q;
    if (mem == DATTN_MEM_HOST) {
        qbuf.ensure(q_bytes(b.num_rows));
        cuda_check(cudaMemcpyAsync(qbuf.p, q, q_bytes(b.num_rows), cudaMemcpyHostToDevice, stream),
                   "cudaMemcpyAsync(q)");
        q_dev = qbuf.p;
    }
    const bool check = (b.flags & DATTN_F_CHECK_FINITE) != 0;
    if (check) cuda_check(cudaMemsetAsync(d_flag, 0, sizeof(int32_t), stream), "cudaMemsetAsync");
    recs.ensure(static_cast<size_t>(std::max(pl.nchunks, 1)) * cfg.num_q_heads * rec_bytes());
    void* out_dev = out;
    if (want_out && mem == DATTN_MEM_HOST) {
        obuf.ensure(q_bytes(b.num_rows));
        out_dev = obuf.p;
    }
    // fused: the MA kernel merges each (row, kv head) group as it completes --
    // no separate merge launch. Empty groups (no chunk) are never completed:
    // zero their outputs up front; their identity records need the K3 path.
    if (want_out && fused_ok(pl, check) && !(pl.any_empty_group && row_partials)) {
        MAParams f{};
        fill_fused(pl, f);
        f.fused_mode = 1;
        f.out_norm = out_dev;
        f.out_recs = row_partials;
        if (pl.any_empty_group)
            cuda_check(cudaMemsetAsync(out_dev, 0, q_bytes(b.num_rows), stream), "cudaMemsetAsync(out)");
        run_ma(pl, q_dev, recs.p, b.scale, check, &f);
        stats.last_exchange = 0;
    } else {
        run_ma(pl, q_dev, recs.p, b.scale, check);
        local_merge(pl, recs.p, row_partials, want_out ? out_dev : nullptr);
    }
    if (mem == DATTN_MEM_HOST) {
        if (want_out)
            cuda_check(cudaMemcpyAsync(out, obuf.p, q_bytes(b.num_rows), cudaMemcpyDeviceToHost,
                                       stream),
                       "cudaMemcpyAsync(out)");
        cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
    }
    if (check) check_flag();
}

void dattn_store::micro_attention(const dattn_batch& b, const void* q_dev, void* partials) {
    activate();
    Plan& pl = cache_plan;
    plan(b, true, pl);
    upload_plan(pl);
    const bool check = (b.flags & DATTN_F_CHECK_FINITE) != 0;
    if (check) cuda_check(cudaMemsetAsync(d_flag, 0, sizeof(int32_t), stream), "cudaMemsetAsync");
    const int64_t n = static_cast<int64_t>(b.num_ranges) * cfg.num_q_heads;
    if (n > 0) {
        cuda_check(launch_identity_records(cfg.dtype, dp, partials, n, stream), "launch(identity)");
        count_launch(1);
    }
    run_ma(pl, q_dev, partials, b.scale, check);
    if (check) check_flag();
}

void dattn_store::decode_sharded(const dattn_batch& b, const void* q, void* out, int mem) {
    if (!comm) throw Error(DATTN_ERR_CONTRACT, "dattn_comm_init was not called");
    check_exchange_status();
    activate();
    Plan& pl = cache_plan;
    plan(b, false, pl);
    upload_plan(pl);
    const void* q_dev = q;
    if (mem == DATTN_MEM_HOST) {
        qbuf.ensure(q_bytes(b.num_rows));
        cuda_check(cudaMemcpyAsync(qbuf.p, q, q_bytes(b.num_rows), cudaMemcpyHostToDevice, stream),
                   "cudaMemcpyAsync(q)");
        q_dev = qbuf.p;
    }
    recs.ensure(static_cast<size_t>(std::max(pl.nchunks, 1)) * cfg.num_q_heads * rec_bytes());
    const size_t row_recs = static_cast<size_t>(b.num_rows) * cfg.num_q_heads;
    void* out_dev0 = out;
    if (mem == DATTN_MEM_HOST) {
        obuf.ensure(q_bytes(b.num_rows));
        out_dev0 = obuf.p;
    }
    if (fused_merge && static_cast<int64_t>(row_recs) <= slot_stride && fused_ok(pl, false)) {
        // fused K1: every completed (row, kv head) group is merged and pushed to
        // all ranks from inside the MA kernel, overlapping the exchange with the
        // remaining streaming; K6 then merges the ranks' records.
        MAParams f{};
        fill_fused(pl, f);
        f.fused_mode = 2;
        ++epoch;
        for (int r = 0; r < nranks; ++r) f.peer_x[r] = xhalf_ptr(peer_x[r], epoch);
        f.rank = rank;
        f.nranks = nranks;
        f.slot_stride = slot_stride;
        run_ma(pl, q_dev, recs.p, b.scale, false, &f);
        RankMergeParams rp{};
        rp.rows = b.num_rows;
        rp.heads = cfg.num_q_heads;
        rp.group = group;
        rp.num_kv_heads = cfg.num_kv_heads;
        rp.group_expected = static_cast<const int32_t*>(d_meta.p) + pl.off_expect;
        for (int r = 0; r < nranks; ++r) rp.peer_x[r] = f.peer_x[r];
        rp.rank = rank;
        rp.nranks = nranks;
        rp.slot_stride = slot_stride;
        rp.out_norm = out_dev0;
        rp.ctl = xctl();
        // all CTAs co-resident (occupancy cap): identity pushes precede every wait
        const int grid = static_cast<int>(std::max<int64_t>(
            1, std::min<int64_t>((static_cast<int64_t>(row_recs) + 7) / 8, x_grid_cap[1])));
        cudaEvent_t* ev = timing ? timer_pair(2) : nullptr;
        if (ev) cuda_check(cudaEventRecord(ev[0], stream), "cudaEventRecord");
        cuda_check(launch_rank_merge(cfg.dtype, dp, rp, grid, stream), "launch(K6 rank_merge)");
        if (ev) cuda_check(cudaEventRecord(ev[1], stream), "cudaEventRecord");
        count_launch(1);
        stats.last_exchange = 3;
        if (mem == DATTN_MEM_HOST) {
            cuda_check(cudaMemcpyAsync(out, obuf.p, q_bytes(b.num_rows), cudaMemcpyDeviceToHost, stream),
                       "cudaMemcpyAsync(out)");
            cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
            check_exchange_status();
        }
        return;
    }
    run_ma(pl, q_dev, recs.p, b.scale, false);
    if (fused_merge && static_cast<int64_t>(row_recs) <= slot_stride) {
        // K5: local merge + NVLink record exchange + rank merge in one launch
        const int32_t* w = static_cast<const int32_t*>(d_meta.p);
        XParams xp{};
        xp.local.recs = recs.p;
        xp.local.rows = b.num_rows;
        xp.local.heads = cfg.num_q_heads;
        xp.local.row_begin = w + pl.off_rowchunk;
        xp.local.row_mul = cfg.num_q_heads;
        xp.local.c_stride = cfg.num_q_heads;
        xp.local.chunk_kvh = pl.any_kvh ? w + pl.off_kvh : nullptr;
        xp.local.group = group;
        ++epoch;
        for (int r = 0; r < nranks; ++r) xp.peer_x[r] = xhalf_ptr(peer_x[r], epoch);
        xp.rank = rank;
        xp.nranks = nranks;
        xp.slot_stride = slot_stride;
        xp.out_norm = out_dev0;
        // groups per CTA sweep: 8 (one per warp) when groups are plentiful,
        // else 1 so a few long groups each get a whole CTA. The grid is capped
        // at the kernel's occupancy x SMs, so it is co-resident: warps polling
        // in phase D never wait for a CTA that is not running.
        const int64_t gpc = static_cast<int64_t>(row_recs) >= 1024 ? 8 : 1;
        xp.groups_per_cta = static_cast<int32_t>(gpc);
        xp.ctl = xctl();
        const int grid = static_cast<int>(std::max<int64_t>(
            1, std::min<int64_t>((static_cast<int64_t>(row_recs) + gpc - 1) / gpc, x_grid_cap[0])));
        static const bool trace = std::getenv("DATTN_K5_TRACE") != nullptr;
        if (trace) {
            if (!k5_trace.p) {
                k5_trace.ensure(static_cast<size_t>(kMaxExchangeGrid) * 3 * sizeof(unsigned long long));
                cuda_check(cudaMemsetAsync(k5_trace.p, 0, static_cast<size_t>(kMaxExchangeGrid) * 3 * 8, stream),
                           "cudaMemsetAsync(trace)");
            }
            xp.trace = static_cast<unsigned long long*>(k5_trace.p);
        }
        cudaEvent_t* ev = timing ? timer_pair(2) : nullptr;
        if (ev) cuda_check(cudaEventRecord(ev[0], stream), "cudaEventRecord");
        cuda_check(launch_merge_exchange(cfg.dtype, dp, xp, grid, stream), "launch(K5 merge_exchange)");
        if (ev) cuda_check(cudaEventRecord(ev[1], stream), "cudaEventRecord");
        count_launch(1);
        stats.last_exchange = 2;
        if (mem == DATTN_MEM_HOST) {
            cuda_check(cudaMemcpyAsync(out, obuf.p, q_bytes(b.num_rows), cudaMemcpyDeviceToHost, stream),
                       "cudaMemcpyAsync(out)");
            cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
            check_exchange_status();
        }
        return;
    }
    rowrecs.ensure(std::max<size_t>(row_recs, 1) * rec_bytes());
    local_merge(pl, recs.p, rowrecs.p, nullptr);
    gathered.ensure(std::max<size_t>(row_recs, 1) * rec_bytes() * nranks);
    cudaEvent_t* ev = timing ? timer_pair(2) : nullptr;
    if (ev) cuda_check(cudaEventRecord(ev[0], stream), "cudaEventRecord");
    nccl_check(ncclAllGather(rowrecs.p, gathered.p, row_recs * rec_elems,
                             cfg.dtype == kF64 ? ncclDouble : ncclFloat32, comm, comm_begin()),
               "ncclAllGather(partials)");
    comm_end();
    if (ev) cuda_check(cudaEventRecord(ev[1], stream), "cudaEventRecord");
    stats.last_exchange = 1;
    MergeParams mp{};
    mp.recs = gathered.p;
    mp.rows = b.num_rows;
    mp.heads = cfg.num_q_heads;
    mp.row_begin = nullptr;
    mp.n_uniform = nranks;
    mp.row_mul = cfg.num_q_heads;
    mp.c_stride = static_cast<int64_t>(row_recs);
    mp.group = group;
    void* out_dev = out;
    if (mem == DATTN_MEM_HOST) {
        obuf.ensure(q_bytes(b.num_rows));
        out_dev = obuf.p;
    }
    mp.out_norm = out_dev;
    run_merge(mp);
    if (mem == DATTN_MEM_HOST) {
        cuda_check(cudaMemcpyAsync(out, obuf.p, q_bytes(b.num_rows), cudaMemcpyDeviceToHost, stream),
                   "cudaMemcpyAsync(out)");
        cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
    }
}

// ------------------------------------------------------------------ C ABI

extern "C" {

const char* dattn_last_error(void) { return g_last_error.c_str(); }
void dattn_string_free(char* s) { std::free(s); }
int dattn_abi_version(void) { return 1; }
int64_t dattn_launch_count(int reset) {
    const int64_t n = g_launches;
    if (reset) g_launches = 0;
    return n;
}

dattn_status dattn_store_create(const dattn_store_config* cfg, dattn_store** out) {
    return guarded([&] {
        REQUIRE_ARG(cfg && out, "null argument");
        auto* s = new dattn_store();
        try {
            s->init(*cfg);
        } catch (...) {
            delete s;
            throw;
        }
        *out = s;
    });
}

void dattn_store_destroy(dattn_store* s) {
    if (!s) return;
    cudaSetDevice(s->cfg.device);
    cudaStreamSynchronize(s->stream);
    delete s;
}

dattn_status dattn_store_get_info(const dattn_store* s, dattn_store_info* out) {
    return guarded([&] {
        REQUIRE_ARG(s && out, "null argument");
        out->padded_dim = s->dp;
        out->elem_bytes = s->esz;
        out->record_elems = s->rec_elems;
        out->record_bytes = static_cast<int>(s->rec_bytes());
        out->free_pages = static_cast<int64_t>(s->free_pages.size());
        out->used_pages = s->used_pages;
        out->pool_bytes = 2 * s->cfg.num_pages * s->page_elems * s->esz;
        out->num_sms = s->num_sms;
    });
}

dattn_status dattn_store_set_timing(dattn_store* s, int enable) {
    return guarded([&] {
        REQUIRE_ARG(s, "null store");
        s->activate();
        if (s->timing) s->collect_timing();
        s->timing = enable != 0;
    });
}

dattn_status dattn_store_get_stats(dattn_store* s, int reset, dattn_stats* out) {
    return guarded([&] {
        REQUIRE_ARG(s && out, "null argument");
        s->activate();
        if (s->timing) s->collect_timing();
        *out = s->stats;
        if (reset) {
            const dattn_stats keep = s->stats;
            s->stats = dattn_stats{};
            s->stats.ma_grid = keep.ma_grid;
        }
    });
}

dattn_status dattn_store_stream(const dattn_store* s, void** stream_out) {
    return guarded([&] {
        REQUIRE_ARG(s && stream_out, "null argument");
        *stream_out = s->stream;
    });
}

dattn_status dattn_store_set_stream(dattn_store* s, void* stream) {
    return guarded([&] {
        REQUIRE_ARG(s, "null store");
        s->activate();
        // order the switch after all work already queued on the old stream
        cuda_check(cudaStreamSynchronize(s->stream), "cudaStreamSynchronize");
        // NULL is the CUDA default stream (not "unset"): a caller passing its
        // default-stream handle gets ordering with its own default-stream work
        s->stream = stream == DATTN_OWN_STREAM ? s->own_stream : static_cast<cudaStream_t>(stream);
    });
}

dattn_status dattn_store_synchronize(dattn_store* s) {
    return guarded([&] {
        REQUIRE_ARG(s, "null store");
        s->activate();
        cuda_check(cudaStreamSynchronize(s->stream), "cudaStreamSynchronize");
        s->check_exchange_status();
    });
}

dattn_status dattn_seq_create(dattn_store* s, int64_t tokens, int32_t* seq_out) {
    return guarded([&] {
        REQUIRE_ARG(s && seq_out, "null argument");
        if (tokens < 0) throw Error(DATTN_ERR_CONTRACT, "token count must be >= 0");
        if (s->free_seqs.empty()) throw Error(DATTN_ERR_CAPACITY, "block table full");
        s->activate();
        const int32_t id = s->free_seqs.back();
        const int64_t need = (tokens + s->cfg.page_tokens - 1) / s->cfg.page_tokens;
        if (need > s->cfg.max_pages_per_seq)
            throw Error(DATTN_ERR_CAPACITY, "sequence exceeds max_pages_per_seq");
        if (need > static_cast<int64_t>(s->free_pages.size()))
            throw Error(DATTN_ERR_CAPACITY, "page pool exhausted");
        s->free_seqs.pop_back();
        s->seq_live[id] = 1;
        s->seq_pages[id] = 0;
        s->seq_tokens[id] = 0;
        s->grow(id, tokens);
        *seq_out = id;
    });
}

dattn_status dattn_seq_resize(dattn_store* s, int32_t seq, int64_t tokens) {
    return guarded([&] {
        REQUIRE_ARG(s, "null store");
        s->check_seq(seq);
        if (tokens < s->seq_tokens[seq]) throw Error(DATTN_ERR_CONTRACT, "sequences only grow");
        s->activate();
        s->grow(seq, tokens);
    });
}

dattn_status dattn_seq_release(dattn_store* s, int32_t seq, int64_t* freed_pages) {
    return guarded([&] {
        REQUIRE_ARG(s, "null store");
        s->check_seq(seq);
        const size_t off = static_cast<size_t>(seq) * s->cfg.max_pages_per_seq;
        const int32_t n = s->seq_pages[seq];
        for (int32_t i = n - 1; i >= 0; --i) s->free_pages.push_back(s->h_bt[off + i]);
        s->used_pages -= n;
        s->seq_pages[seq] = 0;
        s->seq_tokens[seq] = 0;
        s->seq_live[seq] = 0;
        s->free_seqs.push_back(seq);
        if (freed_pages) *freed_pages = n;
    });
}

dattn_status dattn_seq_tokens(const dattn_store* s, int32_t seq, int64_t* tokens) {
    return guarded([&] {
        REQUIRE_ARG(s && tokens, "null argument");
        s->check_seq(seq);
        *tokens = s->seq_tokens[seq];
    });
}

dattn_status dattn_seq_block_table(const dattn_store* s, int32_t seq, int32_t* pages,
                                   int64_t capacity, int64_t* n_pages) {
    return guarded([&] {
        REQUIRE_ARG(s && n_pages, "null argument");
        s->check_seq(seq);
        const int32_t n = s->seq_pages[seq];
        if (pages) {
            if (capacity < n) throw Error(DATTN_ERR_INVALID_ARGUMENT, "capacity too small");
            std::memcpy(pages, s->h_bt.data() + static_cast<size_t>(seq) * s->cfg.max_pages_per_seq,
                        sizeof(int32_t) * n);
        }
        *n_pages = n;
    });
}

dattn_status dattn_kv_write(dattn_store* s, int32_t seq, int kv_head, int64_t tok0, int64_t n,
                            const void* k, const void* v, int src_dtype, int src_row_elems) {
    return guarded([&] {
        REQUIRE_ARG(s, "null store");
        s->check_seq(seq);
        if (n == 0) return;
        REQUIRE_ARG(k && v, "null data");
        if (kv_head < 0 || kv_head >= s->cfg.num_kv_heads)
            throw Error(DATTN_ERR_CONTRACT, "kv_head out of bounds");
        if (tok0 < 0 || n < 0 || tok0 + n > s->seq_tokens[seq])
            throw Error(DATTN_ERR_CONTRACT, "rows outside the sequence");
        if (src_row_elems < 1 || src_row_elems > s->dp)
            throw Error(DATTN_ERR_CONTRACT, "row length exceeds the padded head dim");
        if (src_dtype < 0 || src_dtype > 2) throw Error(DATTN_ERR_INVALID_ARGUMENT, "unknown dtype");
        s->activate();
        s->write_rows(seq, kv_head, tok0, n, k, v, src_dtype, src_row_elems);
    });
}

dattn_status dattn_kv_read(dattn_store* s, int32_t seq, int kv_head, int64_t tok0, int64_t n,
                           void* k, void* v) {
    return guarded([&] {
        REQUIRE_ARG(s, "null store");
        s->check_seq(seq);
        if (n == 0) return;
        REQUIRE_ARG(k && v, "null data");
        if (kv_head < 0 || kv_head >= s->cfg.num_kv_heads)
            throw Error(DATTN_ERR_CONTRACT, "kv_head out of bounds");
        if (tok0 < 0 || n < 0 || tok0 + n > s->seq_tokens[seq])
            throw Error(DATTN_ERR_CONTRACT, "rows outside the sequence");
        s->activate();
        const size_t bytes = static_cast<size_t>(n) * s->dp * s->esz;
        DevBuf tmp;
        tmp.ensure(2 * bytes);
        ScatterParams p{};
        p.k_pool = s->kpool;
        p.v_pool = s->vpool;
        p.k_rows = tmp.p;
        p.v_rows = static_cast<uint8_t*>(tmp.p) + bytes;
        p.block_row = s->d_bt + static_cast<size_t>(seq) * s->cfg.max_pages_per_seq;
        p.page_tokens = s->cfg.page_tokens;
        p.num_kv_heads = s->cfg.num_kv_heads;
        p.kv_head = kv_head;
        p.tok0 = tok0;
        p.n = n;
        cuda_check(launch_gather(s->cfg.dtype, s->dp, p, s->stream), "launch(gather)");
        count_launch(1);
        cuda_check(cudaMemcpyAsync(k, tmp.p, bytes, cudaMemcpyDeviceToHost, s->stream), "cudaMemcpyAsync");
        cuda_check(cudaMemcpyAsync(v, p.v_rows, bytes, cudaMemcpyDeviceToHost, s->stream), "cudaMemcpyAsync");
        cuda_check(cudaStreamSynchronize(s->stream), "cudaStreamSynchronize");
    });
}

dattn_status dattn_kv_append(dattn_store* s, int n, const int32_t* seqs, const void* k_new,
                             const void* v_new, int mem) {
    return guarded([&] {
        REQUIRE_ARG(s, "null store");
        if (n <= 0) return;
        REQUIRE_ARG(seqs && k_new && v_new, "null argument");
        REQUIRE_ARG(mem == DATTN_MEM_DEVICE || mem == DATTN_MEM_HOST, "bad mem kind");
        for (int i = 0; i < n; ++i) s->check_seq(seqs[i]);
        {
            std::vector<int32_t> sorted(seqs, seqs + n);
            std::sort(sorted.begin(), sorted.end());
            if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
                throw Error(DATTN_ERR_CONTRACT, "duplicate sequence in append");
        }
        // every page the batch needs must be available before any sequence
        // grows, so a CAPACITY failure leaves the ledger unchanged
        int64_t need = 0;
        for (int i = 0; i < n; ++i) {
            const int64_t t = s->seq_tokens[seqs[i]];
            const int64_t pages = (t + 1 + s->cfg.page_tokens - 1) / s->cfg.page_tokens;
            if (pages > s->cfg.max_pages_per_seq) throw Error(DATTN_ERR_CAPACITY, "sequence exceeds max_pages_per_seq");
            need += pages - s->seq_pages[seqs[i]];
        }
        if (need > static_cast<int64_t>(s->free_pages.size())) throw Error(DATTN_ERR_CAPACITY, "page pool exhausted");
        s->activate();
        // the previous append's H2D copy must have consumed the pinned staging
        cuda_check(cudaEventSynchronize(s->app_ev), "cudaEventSynchronize");
        const size_t mbytes = 2 * static_cast<size_t>(n) * sizeof(int32_t);
        s->app_hmeta.ensure(mbytes);
        s->app_meta.ensure(mbytes);
        int32_t* meta = static_cast<int32_t*>(s->app_hmeta.p);
        for (int i = 0; i < n; ++i) {
            const int64_t t = s->seq_tokens[seqs[i]];
            s->grow(seqs[i], t + 1);
            meta[i] = seqs[i];
            meta[n + i] = static_cast<int32_t>(t);
        }
        cuda_check(cudaMemcpyAsync(s->app_meta.p, meta, mbytes, cudaMemcpyHostToDevice, s->stream), "cudaMemcpyAsync");
        const size_t rows = static_cast<size_t>(n) * s->cfg.num_kv_heads * s->dp * s->esz;
        const void* kd = k_new;
        const void* vd = v_new;
        if (mem == DATTN_MEM_HOST) {
            s->app_rows.ensure(2 * rows);
            cuda_check(cudaMemcpyAsync(s->app_rows.p, k_new, rows, cudaMemcpyHostToDevice, s->stream), "cudaMemcpyAsync");
            cuda_check(cudaMemcpyAsync(static_cast<uint8_t*>(s->app_rows.p) + rows, v_new, rows, cudaMemcpyHostToDevice,
                                       s->stream),
                       "cudaMemcpyAsync");
            kd = s->app_rows.p;
            vd = static_cast<uint8_t*>(s->app_rows.p) + rows;
        }
        AppendParams p{};
        p.k_pool = s->kpool;
        p.v_pool = s->vpool;
        p.block_tables = s->d_bt;
        p.bt_stride = s->cfg.max_pages_per_seq;
        p.page_tokens = s->cfg.page_tokens;
        p.num_kv_heads = s->cfg.num_kv_heads;
        p.seqs = static_cast<const int32_t*>(s->app_meta.p);
        p.positions = static_cast<const int32_t*>(s->app_meta.p) + n;
        p.k_new = kd;
        p.v_new = vd;
        p.n = n;
        cuda_check(launch_append(s->cfg.dtype, s->dp, p, s->stream), "launch(append)");
        cuda_check(cudaEventRecord(s->app_ev, s->stream), "cudaEventRecord");
        count_launch(1);
    });
}

dattn_status dattn_kv_synthetic_rows(dattn_store* s, int n, const uint32_t* logical_seqs,
                                     const int64_t* logical_toks, uint64_t seed, float amp_k, float amp_v,
                                     void* k_dev, void* v_dev) {
    return guarded([&] {
        REQUIRE_ARG(s, "null store");
        if (n <= 0) return;
        REQUIRE_ARG(logical_seqs && logical_toks && k_dev && v_dev, "null argument");
        for (int i = 0; i < n; ++i)
            if (logical_toks[i] < 0) throw Error(DATTN_ERR_CONTRACT, "negative token index");
        s->activate();
        const size_t bytes = static_cast<size_t>(n) * (sizeof(uint32_t) + sizeof(int64_t));
        DevBuf tmp;
        tmp.ensure(bytes);
        std::vector<unsigned char> h(bytes);
        std::memcpy(h.data(), logical_toks, n * sizeof(int64_t));
        std::memcpy(h.data() + n * sizeof(int64_t), logical_seqs, n * sizeof(uint32_t));
        cuda_check(cudaMemcpyAsync(tmp.p, h.data(), bytes, cudaMemcpyHostToDevice, s->stream), "cudaMemcpyAsync");
        RowsSynthParams p{};
        p.k_out = k_dev;
        p.v_out = v_dev;
        p.logical_tok = static_cast<const int64_t*>(tmp.p);
        p.logical_seq = reinterpret_cast<const uint32_t*>(static_cast<unsigned char*>(tmp.p) + n * sizeof(int64_t));
        p.n = n;
        p.num_kv_heads = s->cfg.num_kv_heads;
        p.head_dim = s->cfg.head_dim;
        p.seed = seed;
        p.amp_k = amp_k;
        p.amp_v = amp_v;
        cuda_check(launch_rows_synth(s->cfg.dtype, s->dp, p, s->stream), "launch(rows_synth)");
        count_launch(1);
        // tmp is freed on return
        cuda_check(cudaStreamSynchronize(s->stream), "cudaStreamSynchronize");
    });
}

dattn_status dattn_kv_fill_synthetic(dattn_store* s, int32_t seq, uint64_t seed,
                                     uint32_t logical_seq, int64_t logical_tok0, float amp_k,
                                     float amp_v) {
    return guarded([&] {
        REQUIRE_ARG(s, "null store");
        s->check_seq(seq);
        s->activate();
        FillParams p{};
        p.k_pool = s->kpool;
        p.v_pool = s->vpool;
        p.block_row = s->d_bt + static_cast<size_t>(seq) * s->cfg.max_pages_per_seq;
        p.page_tokens = s->cfg.page_tokens;
        p.num_kv_heads = s->cfg.num_kv_heads;
        p.head_dim = s->cfg.head_dim;
        p.tokens = s->seq_tokens[seq];
        p.seed = seed;
        p.logical_seq = logical_seq;
        p.logical_tok0 = logical_tok0;
        p.amp_k = amp_k;
        p.amp_v = amp_v;
        if (p.tokens == 0) return;
        cuda_check(launch_fill_kv(s->cfg.dtype, s->dp, p, s->stream), "launch(fill_kv)");
        count_launch(1);
    });
}

dattn_status dattn_q_fill_synthetic(dattn_store* s, void* q_dev, int rows, uint64_t seed,
                                    uint32_t row0, float amp_q) {
    return guarded([&] {
        REQUIRE_ARG(s && q_dev, "null argument");
        if (rows <= 0) return;
        s->activate();
        QFillParams p{q_dev, rows, s->cfg.num_q_heads, s->cfg.head_dim, seed, row0, amp_q};
        cuda_check(launch_fill_q(s->cfg.dtype, s->dp, p, s->stream), "launch(fill_q)");
        count_launch(1);
    });
}

dattn_status dattn_decode(dattn_store* s, const dattn_batch* b, const void* q, void* out,
                          void* row_partials, int mem) {
    return guarded([&] {
        REQUIRE_ARG(s && b, "null argument");
        REQUIRE_ARG(q || b->num_rows == 0, "null queries");
        REQUIRE_ARG(mem == DATTN_MEM_DEVICE || mem == DATTN_MEM_HOST, "bad mem kind");
        s->decode(*b, q, out, row_partials, mem);
    });
}

dattn_status dattn_micro_attention(dattn_store* s, const dattn_batch* b, const void* q_dev,
                                   void* partials_dev) {
    return guarded([&] {
        REQUIRE_ARG(s && b && partials_dev, "null argument");
        REQUIRE_ARG(q_dev || b->num_rows == 0, "null queries");
        s->micro_attention(*b, q_dev, partials_dev);
    });
}

dattn_status dattn_merge_partials(dattn_store* s, const dattn_merge_desc* d, const void* recs,
                                  void* out_recs, void* out_norm) {
    return guarded([&] {
        REQUIRE_ARG(s && d && recs, "null argument");
        if (d->rows < 0 || d->heads < 1) throw Error(DATTN_ERR_CONTRACT, "bad merge shape");
        s->activate();
        MergeParams mp{};
        mp.recs = recs;
        mp.rows = d->rows;
        mp.heads = d->heads;
        mp.row_begin = d->row_begin;
        mp.n_uniform = d->n_uniform;
        mp.row_mul = d->row_mul;
        mp.c_stride = d->c_stride;
        mp.group = s->group;
        mp.out_recs = out_recs;
        mp.out_norm = out_norm;
        s->run_merge(mp);
    });
}

dattn_status dattn_comm_unique_id(unsigned char id[DATTN_UNIQUE_ID_BYTES]) {
    return guarded([&] {
        REQUIRE_ARG(id, "null argument");
        static_assert(sizeof(ncclUniqueId) == DATTN_UNIQUE_ID_BYTES, "nccl id size");
        ncclUniqueId u;
        nccl_check(ncclGetUniqueId(&u), "ncclGetUniqueId");
        std::memcpy(id, &u, sizeof(u));
    });
}

dattn_status dattn_comm_init(dattn_store* s, const unsigned char id[DATTN_UNIQUE_ID_BYTES],
                             int rank, int nranks) {
    return guarded([&] {
        REQUIRE_ARG(s && id, "null argument");
        if (nranks < 1 || rank < 0 || rank >= nranks)
            throw Error(DATTN_ERR_CONTRACT, "bad rank / world size");
        s->activate();
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        // unmap the previous world's peer buffers while rank / nranks still
        // describe it (release_exchange skips the old own rank)
        cuda_check(cudaStreamSynchronize(s->stream), "cudaStreamSynchronize");
        s->release_exchange();
        s->release_peer_pools();
        if (s->comm) ncclCommDestroy(s->comm);
        s->comm = nullptr;
        s->rank = 0;
        s->nranks = 1;
        nccl_check(ncclCommInitRank(&s->comm, nranks, u, rank), "ncclCommInitRank");
        s->rank = rank;
        s->nranks = nranks;
        if (nranks > 1) {
            s->setup_exchange();
            s->setup_peer_pools();
        }
    });
}

dattn_status dattn_comm_abort(dattn_store* s) {
    return guarded([&] {
        REQUIRE_ARG(s, "null store");
        if (!s->x_ctl_dev) return;
        // the abort word lives in device memory: write it from a stream that
        // runs beside the exchange kernel the polls are in
        static const int one = 1;
        cuda_check(cudaSetDevice(s->cfg.device), "cudaSetDevice");
        cuda_check(cudaMemcpyAsync(s->x_ctl_dev, &one, sizeof(int), cudaMemcpyHostToDevice, s->abort_stream),
                   "cudaMemcpyAsync(abort)");
        cuda_check(cudaStreamSynchronize(s->abort_stream), "cudaStreamSynchronize(abort)");
    });
}

dattn_status dattn_comm_info(const dattn_store* s, int* rank, int* nranks, int* exchange) {
    return guarded([&] {
        REQUIRE_ARG(s && rank && nranks && exchange, "null argument");
        if (!s->comm) throw Error(DATTN_ERR_CONTRACT, "dattn_comm_init was not called");
        int r = -1, n = -1;
        nccl_check(ncclCommUserRank(s->comm, &r), "ncclCommUserRank");
        nccl_check(ncclCommCount(s->comm, &n), "ncclCommCount");
        const char* k1 = std::getenv("DATTN_FUSED_K1");
        *rank = r;
        *nranks = n;
        *exchange = !s->fused_merge ? 1 : (k1 && std::atoi(k1) == 1 ? 3 : 2);
    });
}

dattn_status dattn_decode_sharded(dattn_store* s, const dattn_batch* b, const void* q, void* out,
                                  int mem) {
    return guarded([&] {
        REQUIRE_ARG(s && b && out, "null argument");
        REQUIRE_ARG(q || b->num_rows == 0, "null queries");
        REQUIRE_ARG(mem == DATTN_MEM_DEVICE || mem == DATTN_MEM_HOST, "bad mem kind");
        s->decode_sharded(*b, q, out, mem);
    });
}

static void kv_transfer(dattn_store* s, int32_t seq, int64_t tok0, int64_t n, int peer, bool send) {
    if (!s->comm) throw Error(DATTN_ERR_CONTRACT, "dattn_comm_init was not called");
    s->check_seq(seq);
    if (peer < 0 || peer >= s->nranks || peer == s->rank) throw Error(DATTN_ERR_CONTRACT, "bad peer rank");
    if (tok0 < 0 || n < 0 || tok0 + n > s->seq_tokens[seq])
        throw Error(DATTN_ERR_CONTRACT, "rows outside the sequence");
    if (n == 0) return;
    s->activate();
    const size_t bytes = static_cast<size_t>(n) * s->cfg.num_kv_heads * s->dp * s->esz;
    DevBuf buf;
    buf.ensure(2 * bytes);
    ScatterParams p{};
    p.k_pool = s->kpool;
    p.v_pool = s->vpool;
    p.k_rows = buf.p;
    p.v_rows = static_cast<uint8_t*>(buf.p) + bytes;
    p.block_row = s->d_bt + static_cast<size_t>(seq) * s->cfg.max_pages_per_seq;
    p.page_tokens = s->cfg.page_tokens;
    p.num_kv_heads = s->cfg.num_kv_heads;
    p.kv_head = -1;
    p.tok0 = tok0;
    p.n = n;
    if (send) {
        cuda_check(launch_gather(s->cfg.dtype, s->dp, p, s->stream), "launch(gather)");
        count_launch(1);
        nccl_check(ncclSend(buf.p, 2 * bytes, ncclUint8, peer, s->comm, s->comm_begin()), "ncclSend(kv)");
        s->comm_end();
    } else {
        nccl_check(ncclRecv(buf.p, 2 * bytes, ncclUint8, peer, s->comm, s->comm_begin()), "ncclRecv(kv)");
        s->comm_end();
        cuda_check(launch_scatter(s->cfg.dtype, s->dp, p, s->stream), "launch(scatter)");
        count_launch(1);
    }
    cuda_check(cudaStreamSynchronize(s->stream), "cudaStreamSynchronize");
}

dattn_status dattn_kv_send(dattn_store* s, int32_t seq, int64_t tok0, int64_t n, int peer) {
    return guarded([&] {
        REQUIRE_ARG(s, "null store");
        kv_transfer(s, seq, tok0, n, peer, true);
    });
}

dattn_status dattn_kv_recv(dattn_store* s, int32_t seq, int64_t tok0, int64_t n, int peer) {
    return guarded([&] {
        REQUIRE_ARG(s, "null store");
        kv_transfer(s, seq, tok0, n, peer, false);
    });
}

dattn_status dattn_kv_pull(dattn_store* s, int32_t dst_seq, int64_t dst_tok0, int src_rank,
                          const int32_t* src_pages, int64_t n_pages) {
    return guarded([&] {
        REQUIRE_ARG(s && (n_pages == 0 || src_pages), "null argument");
        if (!s->comm) throw Error(DATTN_ERR_CONTRACT, "dattn_comm_init was not called");
        if (src_rank < 0 || src_rank >= s->nranks || src_rank == s->rank || !s->peer_kpool[src_rank])
            throw Error(DATTN_ERR_CONTRACT, "bad source rank (or its pool is not mapped)");
        s->check_seq(dst_seq);
        const int64_t P = s->cfg.page_tokens;
        if (n_pages < 0 || dst_tok0 < 0 || dst_tok0 % P != 0)
            throw Error(DATTN_ERR_CONTRACT, "pulls move whole pages: dst_tok0 must be page aligned");
        const int64_t p0 = dst_tok0 / P;
        if (p0 + n_pages > s->seq_pages[dst_seq])
            throw Error(DATTN_ERR_CONTRACT, "destination pages outside the sequence");
        for (int64_t i = 0; i < n_pages; ++i)
            if (src_pages[i] < 0 || src_pages[i] >= s->peer_pages[src_rank])
                throw Error(DATTN_ERR_CONTRACT, "source page id outside the source rank's pool");
        if (n_pages == 0) return;
        s->activate();
        // the destination pages' earlier writes (allocation, appends) come first
        cuda_check(cudaEventRecord(s->mig_ev, s->stream), "cudaEventRecord");
        cuda_check(cudaStreamWaitEvent(s->mig_stream, s->mig_ev, 0), "cudaStreamWaitEvent");
        const size_t pb = static_cast<size_t>(s->page_elems) * s->esz;
        const int32_t* bt = s->h_bt.data() + static_cast<size_t>(dst_seq) * s->cfg.max_pages_per_seq;
        auto* dk = static_cast<unsigned char*>(s->kpool);
        auto* dv = static_cast<unsigned char*>(s->vpool);
        auto* sk = static_cast<const unsigned char*>(s->peer_kpool[src_rank]);
        auto* sv = static_cast<const unsigned char*>(s->peer_vpool[src_rank]);
        // one copy per run of pages consecutive on both sides (copy engines
        // over NVLink; no SMs taken from the decode kernels)
        for (int64_t i = 0; i < n_pages;) {
            int64_t j = i + 1;
            while (j < n_pages && src_pages[j] == src_pages[j - 1] + 1 && bt[p0 + j] == bt[p0 + j - 1] + 1) ++j;
            const size_t bytes = static_cast<size_t>(j - i) * pb;
            cuda_check(cudaMemcpyAsync(dk + static_cast<size_t>(bt[p0 + i]) * pb, sk + static_cast<size_t>(src_pages[i]) * pb,
                                       bytes, cudaMemcpyDeviceToDevice, s->mig_stream), "cudaMemcpyAsync(pull k)");
            cuda_check(cudaMemcpyAsync(dv + static_cast<size_t>(bt[p0 + i]) * pb, sv + static_cast<size_t>(src_pages[i]) * pb,
                                       bytes, cudaMemcpyDeviceToDevice, s->mig_stream), "cudaMemcpyAsync(pull v)");
            i = j;
        }
        s->mig_pending += n_pages;
    });
}

dattn_status dattn_kv_migration_join(dattn_store* s, int wait_host) {
    return guarded([&] {
        REQUIRE_ARG(s, "null store");
        if (!s->mig_stream) return;
        s->activate();
        cuda_check(cudaEventRecord(s->mig_ev, s->mig_stream), "cudaEventRecord");
        cuda_check(cudaStreamWaitEvent(s->stream, s->mig_ev, 0), "cudaStreamWaitEvent");
        if (wait_host) cuda_check(cudaEventSynchronize(s->mig_ev), "cudaEventSynchronize(mig)");
        s->mig_pending = 0;
    });
}

dattn_status dattn_host_alloc(size_t bytes, void** out) {
    return guarded([&] {
        REQUIRE_ARG(out, "null argument");
        cuda_check(cudaMallocHost(out, std::max<size_t>(bytes, 1)), "cudaMallocHost");
    });
}
void dattn_host_free(void* p) {
    if (p) cudaFreeHost(p);
}
dattn_status dattn_device_alloc(dattn_store* s, size_t bytes, void** out) {
    return guarded([&] {
        REQUIRE_ARG(s && out, "null argument");
        s->activate();
        cuda_check(cudaMalloc(out, std::max<size_t>(bytes, 1)), "cudaMalloc");
    });
}
void dattn_device_free(dattn_store* s, void* p) {
    if (!p) return;
    if (s) cudaSetDevice(s->cfg.device);
    cudaFree(p);
}
dattn_status dattn_memcpy(dattn_store* s, void* dst, const void* src, size_t bytes, int kind) {
    return guarded([&] {
        REQUIRE_ARG(s && (bytes == 0 || (dst && src)), "null argument");
        s->activate();
        cuda_check(cudaMemcpyAsync(dst, src, bytes, static_cast<cudaMemcpyKind>(kind), s->stream),
                   "cudaMemcpyAsync");
        cuda_check(cudaStreamSynchronize(s->stream), "cudaStreamSynchronize");
    });
}

}  // extern "C"
