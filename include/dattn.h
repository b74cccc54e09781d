/*
 * dattn.h -- C ABI of the B200-native DistAttention decode path.
 *
 * This is the drop-in boundary: plain pointers and sizes, no torch or C++
 * types. It follows the conventions of the reference's C ABI
 * (/root/reference/proj/include/kvsched.h:1-32): every call returns a status,
 * a message for the last failure of the calling thread is in
 * dattn_last_error(), out-pointers are written only on success, strings
 * returned through char** are freed with dattn_string_free().
 *
 * Each entry point cites the reference interface it replaces. The reference's
 * hot path is the C++ operator API kvsched::attn
 * (proj/include/kvsched/distattention.hpp:16-95); the C++ mirror of that API
 * (include/dattn_kvsched.hpp, paper_2401_02669_b200/csrc/kvsched_adapter.cpp)
 * is implemented on top of these calls.
 *
 * Device layout:
 *   K pool, V pool : [num_pages][num_kv_heads][page_tokens][padded_dim]  (dtype)
 *   block tables   : int32 [max_seqs][max_pages_per_seq]
 *   queries        : [rows][num_q_heads][padded_dim]                     (dtype)
 *   outputs        : [rows][num_q_heads][padded_dim]                     (dtype)
 *   partial record : [m, e, tokens, 0, ma[padded_dim]]  (fp32; fp64 for F64 stores)
 *
 * Threading: a store is used by one host thread at a time (one store per
 * GPU / stream); different stores are independent.
 */
#ifndef DATTN_H
#define DATTN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* kvsched.h:20-26 plus device-side codes. */
typedef enum dattn_status {
    DATTN_OK = 0,
    DATTN_ERR_INVALID_ARGUMENT = 1, /* null pointers, malformed parameters */
    DATTN_ERR_INPUT = 2,            /* rejected data: non-finite values, bad payloads */
    DATTN_ERR_CONTRACT = 3,         /* precondition violated (shapes, ranges) */
    DATTN_ERR_INTERNAL = 4,
    DATTN_ERR_CUDA = 5,             /* CUDA runtime / launch failure; message has the CUDA string */
    DATTN_ERR_NCCL = 6,             /* NCCL failure */
    DATTN_ERR_CAPACITY = 7          /* page pool or block table exhausted */
} dattn_status;

typedef enum dattn_dtype { DATTN_BF16 = 0, DATTN_F32 = 1, DATTN_F64 = 2 } dattn_dtype;

/* Where the q / out pointers of a decode call live. */
typedef enum dattn_mem { DATTN_MEM_DEVICE = 0, DATTN_MEM_HOST = 1 } dattn_mem;

/* kvsched.h:32 */
const char* dattn_last_error(void);
/* kvsched.h:34 */
void dattn_string_free(char* s);
/* ABI version, bumped on any signature change. */
int dattn_abi_version(void);
/* Number of kernel launches this thread issued since the last reset (for
 * bench.py's gpu_launches). */
int64_t dattn_launch_count(int reset);

/* ------------------------------------------------------------------ store */

/* AttentionConfig (distattention.hpp:18-29) + the paged pool geometry that
 * replaces the reference's per-segment std::vector<double> storage
 * (distattention.hpp:33-42) and the RManager block ledger's capacity
 * (controlplane.hpp:126-134). */
typedef struct dattn_store_config {
    int head_dim;          /* 1..512; rows are zero-padded to padded_dim */
    int num_q_heads;       /* >= 1 */
    int num_kv_heads;      /* >= 1, divides num_q_heads */
    double scale;          /* 0 -> 1/sqrt(head_dim) (distattention.cpp:35-37) */
    int dtype;             /* dattn_dtype of K/V/q/out */
    int page_tokens;       /* tokens per page = block_size_tokens (config.cpp:82 default 16) */
    int64_t num_pages;     /* pool capacity in pages */
    int max_seqs;          /* block-table rows */
    int max_pages_per_seq; /* block-table columns */
    int device;            /* CUDA device ordinal */
} dattn_store_config;

typedef struct dattn_store_info {
    int padded_dim;        /* row length in elements (16, 32, 64, 128, 256 or 512) */
    int elem_bytes;
    int record_elems;      /* partial record length = padded_dim + 4 */
    int record_bytes;
    int64_t free_pages;
    int64_t used_pages;
    int64_t pool_bytes;    /* K + V pool bytes */
    int num_sms;
} dattn_store_info;

typedef struct dattn_store dattn_store;

dattn_status dattn_store_create(const dattn_store_config* cfg, dattn_store** out);
void dattn_store_destroy(dattn_store* s);
dattn_status dattn_store_get_info(const dattn_store* s, dattn_store_info* out);
/* The store's CUDA stream (cudaStream_t as void*). */
dattn_status dattn_store_stream(const dattn_store* s, void** stream_out);
/* Use a caller-owned stream (cudaStream_t) for all subsequent work. NULL is
 * the CUDA default stream, as everywhere in CUDA (e.g. torch's default stream
 * handle 0), so store work is ordered with the caller's default-stream work;
 * DATTN_OWN_STREAM restores the store's own non-blocking stream (the initial
 * setting). */
#define DATTN_OWN_STREAM ((void*)(intptr_t)-1)
dattn_status dattn_store_set_stream(dattn_store* s, void* stream);
dattn_status dattn_store_synchronize(dattn_store* s);

/* Launch statistics; with timing on, every MA (K1 / K2), merge (K3) and
 * exchange launch is bracketed by CUDA events on the store stream and the
 * device time is accumulated (bench.py's roofline numerator). */
typedef struct dattn_stats {
    int64_t ma_launches, merge_launches;
    int64_t ma_timed, merge_timed;
    double ma_ms, merge_ms;     /* summed device time of timed launches */
    int64_t last_items, last_chunks, last_plan_bytes;
    int32_t last_chunk_tokens, ma_grid;
    int32_t last_kernel;        /* 1: K1 CUDA-core MA (fp32 / fp64 / other head dims),
                                   2: K2 tcgen05 MA (bf16, d = 128, any group 1..16),
                                   3: K1g generic MA (groups above 16, or 8 for fp64;
                                      head_dim 257..512) */
    int32_t last_exchange;      /* 0: fused merge inside the MA kernel (1 GPU), 1: NCCL allgather + K3,
                                   2: K5 NVLink exchange, 3: MA-kernel group push + K6 rank merge */
    int64_t comm_timed;
    double comm_ms;             /* summed device time of the timed exchange (allgather or K5) */
} dattn_stats;
dattn_status dattn_store_set_timing(dattn_store* s, int enable);
dattn_status dattn_store_get_stats(dattn_store* s, int reset, dattn_stats* out);

/* ------------------------------------------- sequences (block-table rows) */

/* RManager::alloc_local (controlplane.cpp:38-44): allocate
 * blocks_for_tokens(tokens) pages (perfmodel.cpp:178-182) for a new sequence
 * and return its block-table row. Fails with DATTN_ERR_CAPACITY when the pool
 * or the table is full (the reference returns false). */
dattn_status dattn_seq_create(dattn_store* s, int64_t tokens, int32_t* seq_out);
/* Grow a sequence to `tokens` (allocates pages as needed). */
dattn_status dattn_seq_resize(dattn_store* s, int32_t seq, int64_t tokens);
/* RManager::free_request (controlplane.cpp:55-79): release every page. */
dattn_status dattn_seq_release(dattn_store* s, int32_t seq, int64_t* freed_pages);
dattn_status dattn_seq_tokens(const dattn_store* s, int32_t seq, int64_t* tokens);
/* Host copy of the block-table row (page ids). */
dattn_status dattn_seq_block_table(const dattn_store* s, int32_t seq, int32_t* pages,
                                   int64_t capacity, int64_t* n_pages);

/* ------------------------------------------------------------- KV data */

/* Write rows [tok0, tok0+n) of kv head `kv_head` of `seq` from HOST arrays
 * k, v of n x src_row_elems elements of dtype src_dtype (src_row_elems <=
 * padded_dim; the rest of each row is zero). Replaces building a KVSegment
 * (distattention.hpp:33-42). Asynchronous on the store stream. */
dattn_status dattn_kv_write(dattn_store* s, int32_t seq, int kv_head, int64_t tok0, int64_t n,
                            const void* k, const void* v, int src_dtype, int src_row_elems);

/* Read rows [tok0, tok0+n) of kv head `kv_head` of `seq` back into HOST
 * arrays k, v of n x padded_dim elements in the store dtype (synchronous). */
dattn_status dattn_kv_read(dattn_store* s, int32_t seq, int kv_head, int64_t tok0, int64_t n,
                           void* k, void* v);

/* KV append (the decode loop's write): every sequence in
 * seqs[0..n) grows by one token (a page is allocated when the last one is
 * full, RManager::alloc_local controlplane.cpp:38-44; the pages of the whole
 * batch are checked first, so DATTN_ERR_CAPACITY leaves the ledger unchanged)
 * and the new rows k_new/v_new [n][num_kv_heads][padded_dim] (store dtype,
 * `mem` memory) are written at the new position. seqs is a HOST array.
 * Asynchronous on the store stream: HOST rows are read like cudaMemcpyAsync
 * reads them, so keep them unchanged until the next synchronising call (a
 * HOST-memory decode or dattn_store_synchronize). */
dattn_status dattn_kv_append(dattn_store* s, int n, const int32_t* seqs, const void* k_new,
                             const void* v_new, int mem);

/* Synthetic K/V rows [n][num_kv_heads][padded_dim] (store dtype, DEVICE
 * k_dev/v_dev) of logical sequence logical_seqs[i], token logical_toks[i]:
 * the values K4 writes at those positions, i.e. decode-loop inputs whose
 * result the CPU oracle can check (HOST index arrays; synchronous). */
dattn_status dattn_kv_synthetic_rows(dattn_store* s, int n, const uint32_t* logical_seqs,
                                     const int64_t* logical_toks, uint64_t seed, float amp_k, float amp_v,
                                     void* k_dev, void* v_dev);

/* K4: deterministic counter-hash fill of ALL heads of tokens [0, tokens(seq))
 * of `seq` with the values of logical sequence `logical_seq`, logical token
 * logical_tok0 + t (CPU twin oracle/dattn_oracle.c). */
dattn_status dattn_kv_fill_synthetic(dattn_store* s, int32_t seq, uint64_t seed,
                                     uint32_t logical_seq, int64_t logical_tok0,
                                     float amp_k, float amp_v);

/* Deterministic synthetic queries into a DEVICE buffer [rows][Hq][padded_dim]. */
dattn_status dattn_q_fill_synthetic(dattn_store* s, void* q_dev, int rows, uint64_t seed,
                                    uint32_t row0, float amp_q);

/* --------------------------------------------------------- decode step */

/* One rBlock: tokens [tok_begin, tok_end) of block-table row `seq`, attended
 * by output row `out_row`. kv_head < 0: all kv heads; else only that kv head
 * (per-kv-head segment lists, distattention.cpp:183-209). Ranges of one
 * decode call must be sorted by out_row. An empty range contributes the
 * identity partial (distattention.cpp:59-67). */
typedef struct dattn_range {
    int32_t seq;
    int32_t out_row;
    int32_t kv_head;
    int32_t reserved;
    int64_t tok_begin;
    int64_t tok_end;
} dattn_range;

typedef struct dattn_batch {
    int32_t num_rows;      /* output rows (requests) */
    int32_t num_ranges;
    const dattn_range* ranges;
    int32_t chunk_tokens;  /* MA split granularity; 0 = auto (fills the SMs) */
    int32_t flags;         /* DATTN_F_* */
    double scale;          /* 0 -> store scale */
} dattn_batch;

enum {
    DATTN_F_NO_OUTPUT = 1,    /* skip the normalised output (partials only) */
    DATTN_F_CHECK_FINITE = 2  /* fail with DATTN_ERR_INPUT on non-finite K/V (F64 stores) */
};

/* Decode attention for every (row, q head): MA over every chunk of every
 * range (K1), then the fused merge (K3) into
 *   out          [num_rows][Hq][padded_dim]  normalised output (aggregate_partials,
 *                                             distattention.cpp:150-174), and/or
 *   row_partials [num_rows][Hq][record]      merged (m, e, ma) per row, the wire
 *                                             partial of serialize_partial
 *                                             (distattention.cpp:211-221),
 * either may be NULL. q/out live in `mem` (HOST: copies are part of the call
 * and it returns after the result is on the host; DEVICE: asynchronous on the
 * store stream). row_partials is always a DEVICE pointer. Rows without any
 * token produce the identity partial and a zero output. */
dattn_status dattn_decode(dattn_store* s, const dattn_batch* b, const void* q, void* out,
                          void* row_partials, int mem);

/* K1 only: one partial record per (range, q head) -- compute_micro_attention
 * (distattention.cpp:99-129) per rBlock, with each range processed as one
 * chunk. partials_dev: [num_ranges][Hq][record]; heads a kv_head-specific
 * range does not serve are written as identity. */
dattn_status dattn_micro_attention(dattn_store* s, const dattn_batch* b, const void* q_dev,
                                   void* partials_dev);

/* K3: merge groups of partial records (combine_partials / aggregate_partials,
 * distattention.cpp:131-174). Group g = row*heads + h merges records
 *   index(g, c) = (row_begin ? row_begin[row] : row) * row_mul + h + c * c_stride
 * for c in [0, row_begin ? row_begin[row+1]-row_begin[row] : n_uniform).
 * Identity records (e == 0) are skipped; a group with one live record
 * reproduces it bit-exactly. Writes merged records and/or normalised rows
 * (out_norm [groups][padded_dim]) in the store dtype. All pointers DEVICE
 * (row_begin may be NULL). */
typedef struct dattn_merge_desc {
    int32_t rows;
    int32_t heads;
    const int32_t* row_begin; /* device, rows+1 entries, or NULL */
    int32_t n_uniform;
    int64_t row_mul;
    int64_t c_stride;
} dattn_merge_desc;
dattn_status dattn_merge_partials(dattn_store* s, const dattn_merge_desc* d, const void* recs,
                                  void* out_recs, void* out_norm);

/* ------------------------------------------------ multi-GPU (NVLink merge) */

/* Sequence-sharded decode across the GPUs of one box: every
 * rank holds its rBlocks of each request, runs the MA kernel over them, merges
 * them into one partial per (row, q head), stores that record into every
 * rank's exchange buffer over NVLink (CUDA IPC peer memory set up by
 * dattn_comm_init) and merges the nranks records into out -- the paper's
 * "(o, m, l)" exchange replacing the simulated
 * remote-partial latency of simengine.cpp:397-407. Every rank gets the full
 * output. DATTN_FUSED_MERGE=0 in the environment selects ncclAllGather of the
 * records instead. */
#define DATTN_UNIQUE_ID_BYTES 128
dattn_status dattn_comm_unique_id(unsigned char id[DATTN_UNIQUE_ID_BYTES]);
dattn_status dattn_comm_init(dattn_store* s, const unsigned char id[DATTN_UNIQUE_ID_BYTES],
                             int rank, int nranks);
/* Make every rank-merge poll of this store give up (K5 phase D / K6 return
 * instead of waiting; dattn_store_synchronize and the next
 * dattn_decode_sharded then fail with DATTN_ERR_NCCL). Polls also give up by
 * themselves after DATTN_EXCHANGE_TIMEOUT_S seconds (environment, default 60)
 * without a peer's record, instead of trapping, so a rank that failed before
 * launching never kills its peers' CUDA contexts. dattn_comm_init rebuilds
 * the exchange. Safe to call from another host thread while a step runs. */
dattn_status dattn_comm_abort(dattn_store* s);
/* The communicator as NCCL reports it (ncclCommUserRank / ncclCommCount) and
 * the exchange decode_sharded will use: 1 ncclAllGather + K3, 2 K5 NVLink
 * exchange, 3 MA-kernel push + K6. Fails with DATTN_ERR_CONTRACT before
 * dattn_comm_init. */
dattn_status dattn_comm_info(const dattn_store* s, int* rank, int* nranks, int* exchange);
/* q/out as in dattn_decode; every rank passes the same num_rows. */
dattn_status dattn_decode_sharded(dattn_store* s, const dattn_batch* b, const void* q,
                                  void* out, int mem);

/* KV block migration between the GPUs of the communicator:
 * the data path of the reference's MoveKvCache / DataTransfer protocol
 * (controlplane.cpp:158-225, which moves descriptors only). The sender packs
 * tokens [tok0, tok0+n) of every kv head of `seq` and ncclSend's them to
 * `peer`; the receiver (same n) ncclRecv's and scatters them into its
 * sequence `seq` at [tok0, tok0+n) (the receiver's sequence must already hold
 * those positions, e.g. via dattn_seq_create / dattn_seq_resize). Paced
 * transfers (<= 16 tokens/step, advance_transfers controlplane.cpp:205-225)
 * are successive calls with small n. Synchronous. */
dattn_status dattn_kv_send(dattn_store* s, int32_t seq, int64_t tok0, int64_t n, int peer);
dattn_status dattn_kv_recv(dattn_store* s, int32_t seq, int64_t tok0, int64_t n, int peer);

/* Block migration overlapped with decode (the same protocol's data path, as
 * the paper runs it: KV moves while the source keeps decoding, PAPER.md:1451;
 * paced by advance_transfers, controlplane.cpp:205-225). The receiver pulls
 * n_pages whole pages -- K and V, all kv heads -- of a peer's pool, source
 * page ids src_pages (the sender's dattn_seq_block_table entries, passed by
 * the host), into its own sequence dst_seq at page-aligned position dst_tok0
 * (dst_seq must already hold those pages). The copies go over NVLink on the
 * copy engines from a low-priority migration stream (both pools are
 * IPC-mapped at dattn_comm_init), so they take no SMs from the decode
 * kernels, and the call returns at once. dattn_kv_migration_join orders the
 * store stream's later work after every pull issued so far (and, with
 * wait_host, blocks until they are done); the sender must keep the source
 * pages until then. A partly filled last page is copied whole. */
dattn_status dattn_kv_pull(dattn_store* s, int32_t dst_seq, int64_t dst_tok0, int src_rank,
                          const int32_t* src_pages, int64_t n_pages);
dattn_status dattn_kv_migration_join(dattn_store* s, int wait_host);

/* ------------------------------------------------ block placement ledger */

/* The cluster's block ledger and the decode loop's slot rule (SURVEY §8f
 * row 3): one RManager block ledger per instance (GPU)
 * (controlplane.cpp:38-79, free_blocks controlplane.hpp:130) plus the
 * simulator's per-step ensure_slot (simengine.cpp:318-354): a request's next
 * token takes a block at its home when the home has one, otherwise -- under a
 * borrowing policy -- on another instance ("overflow borrowing"): one that
 * already hosts blocks of the request first, then the one with the most free
 * blocks among instances none of whose own requests borrow, then any
 * instance with room. Host-only (no GPU). The ledger also records where each
 * block went, in allocation order, so every instance knows which token
 * positions of a request it holds: dattn_ledger_segments gives the token
 * ranges a rank passes to dattn_decode_sharded. Not thread-safe. */
typedef struct dattn_ledger dattn_ledger;

/* n_instances >= 1 instances with capacity_blocks[i] >= 0 blocks each, blocks
 * of block_tokens tokens (perfmodel.cpp:178-182 sizing). */
dattn_status dattn_ledger_create(int n_instances, const int64_t* capacity_blocks, int block_tokens,
                                 dattn_ledger** out);
void dattn_ledger_destroy(dattn_ledger* l);
/* try_admit (simengine.cpp:262-268): alloc_local(blocks_for_tokens(tokens))
 * at `home`; *admitted = 0 when the home lacks room (nothing changes).
 * tokens >= 1; req must not be live. */
dattn_status dattn_ledger_admit(dattn_ledger* l, int64_t req, int home, int64_t tokens, int* admitted);
/* ensure_slot: a block for the request's next token (position ctx). Returns
 * the instance that holds position ctx in *instance, or -1 when no instance
 * can take the block (the reference's stalled request; with allow_borrow = 0
 * the static_alloc policy: home only). */
dattn_status dattn_ledger_ensure_slot(dattn_ledger* l, int64_t req, int allow_borrow, int* instance);
/* The step wrote `tokens` new tokens of req (on_step_done's ctx++,
 * simengine.cpp:444-452); the request must hold their blocks. */
dattn_status dattn_ledger_advance(dattn_ledger* l, int64_t req, int64_t tokens);
/* One decode step for n requests in order (ensure_step's loop,
 * simengine.cpp:356-371): ensure_slot for each, then advance by one token
 * every request that got a slot. instances[i] = the instance holding
 * request i's new token, or -1 (stalled, not advanced). A request that is not
 * live fails the call before the ledger changes. */
dattn_status dattn_ledger_step(dattn_ledger* l, int n, const int64_t* reqs, int allow_borrow, int* instances);
/* free_request on every instance (complete, simengine.cpp:300-303). */
dattn_status dattn_ledger_release(dattn_ledger* l, int64_t req, int64_t* freed_blocks);
/* RManager accessors: capacity_blocks / used_blocks / free_blocks of one
 * instance, and the blocks of req it holds (local_blocks on the home,
 * hosted_blocks(req, home) elsewhere). */
dattn_status dattn_ledger_instance(const dattn_ledger* l, int instance, int64_t* capacity, int64_t* used,
                                   int64_t* free_blocks);
dattn_status dattn_ledger_request(const dattn_ledger* l, int64_t req, int* home, int64_t* ctx,
                                  int64_t* held_blocks);
dattn_status dattn_ledger_blocks(const dattn_ledger* l, int64_t req, int instance, int64_t* blocks);
/* Token ranges [tok_begin, tok_end) of positions [0, ctx) of req in block
 * order, consecutive blocks on one instance merged: *n ranges (at most max
 * written; *n is the full count). */
dattn_status dattn_ledger_segments(const dattn_ledger* l, int64_t req, int max, int* instance,
                                   int64_t* tok_begin, int64_t* tok_end, int* n);
/* summary_.overflow_borrows: blocks allocated remotely so far. */
dattn_status dattn_ledger_borrowed(const dattn_ledger* l, int64_t* blocks);

/* --------------------------------------------------------- verification */

/* kvs_verify_attention (kvsched.h:56-62, capi.cpp:141-155) on the GPU path:
 * the reference's randomized equivalence trials (verify.cpp:84-186) run
 * through the fp64 device kernels against a long-double contiguous softmax.
 * Report format of verify.cpp:188-195. */
dattn_status dattn_verify_attention(int trials, uint64_t seed, double tolerance,
                                    char** report_out, int* pass_out);

/* ------------------------------------------------------------- helpers */

/* cudaMallocHost / cudaFreeHost for pinned staging of host q/out. */
dattn_status dattn_host_alloc(size_t bytes, void** out);
void dattn_host_free(void* p);
dattn_status dattn_device_alloc(dattn_store* s, size_t bytes, void** out);
void dattn_device_free(dattn_store* s, void* p);
dattn_status dattn_memcpy(dattn_store* s, void* dst, const void* src, size_t bytes, int kind);

#ifdef __cplusplus
}
#endif
#endif /* DATTN_H */
