// dattn_gqa_tc.cu -- K2: grouped-query micro-attention on the 5th-gen tensor
// cores (tcgen05 + TMEM + TMA), bf16 K/V, head_dim 128, 2..16 q heads per
// kv head. Same work items, partial records and semantics as K1
// (compute_micro_attention per chunk, /root/reference/proj/src/
// distattention.cpp:99-129, for every q head of the kv head's group).
//
// Swap-AB tiles (the q group is only 8 wide, too narrow for the MMA M):
//   MMA1  S^T[128 tok x 16] = K[128 tok x 128 d] . Q^T[128 d x 16]      (A K-major)
//   MMA2  O^T[128 d   x 16] = V^T[128 d x 128 tok] . P^T[128 tok x 16]  (A MN-major)
// M = 128, N = 16 (group padded with zero rows), K steps of 16, bf16 in,
// fp32 accumulate in TMEM (32 columns). K/V pages arrive by TMA tensor copies
// with the 128-B swizzle straight from the paged pool (box = 64 d x one
// page), so one shared-memory copy of a tile is both the K-major A operand of
// MMA1 and the MN-major A operand of MMA2. P^T is written by the softmax
// warps in the same swizzled K-major layout.
//
// Warp roles (256 threads): w0 K producer, w1 TMEM owner + single-thread MMA
// issuer, w2..w5 softmax / epilogue (thread = token row of S^T, then d row of
// O^T), w6 V producer, w7 merge (fused modes). Online softmax: per-tile max via
// shared memory, P rounded to bf16 (the same value enters e and the P.V
// MMA), the O^T tile rescale-accumulated in registers.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdint>

#include "dattn_internal.h"
#include "dattn_ptx.cuh"
#include "dattn_merge.cuh"

namespace dattn {
namespace tc {

constexpr int kTile = 128;      // tokens per tile (MMA M of MMA1)
constexpr int kD = 128;         // head dim (MMA M of MMA2, K of MMA1)
constexpr int kN = 16;          // MMA N: q heads, padded
constexpr int kKStages = 3;     // K (+ Q) ring: released as soon as MMA1 has read it
constexpr int kVStages = 3;     // V ring: released after MMA2
constexpr int kMeta = 8;        // tile descriptors, read by the V producer / softmax warps
constexpr int kThreads = 256;   // w0 K producer, w1 MMA, w2..5 softmax, w6 V producer, w7 merge
constexpr int kHalf = kTile * 128;        // bytes of one 64-column half of a 128-row tile
constexpr int kKVBytes = 2 * kHalf;       // one tensor (K or V) tile: 32 KB
constexpr int kQBytes = 2 * kN * 128;     // Q slot: two halves of 16 rows x 128 B
constexpr int kKStageBytes = kKVBytes + kQBytes;  // 36 KB (1024-B multiple)
constexpr int kPBytes = 2 * kN * 128;     // one P^T tile (two are kept)
constexpr int kPidWin = 512;              // page ids of one item held in shared memory
constexpr int kMaxTilePages = kTile / 16; // page_tokens >= 16
constexpr uint32_t kTmemCols = 64;        // S^T cols 0..15, O^T buffers at 16 and 32

struct TileMeta {
    int32_t item;   // -1: terminate
    int32_t tile0;  // sequence position of row 0 of the tile
    int32_t tlo, thi;
    int32_t flags;  // 1 first tile of item, 2 last tile
    int32_t row, kvh, gchunk;
    int32_t npages;
    int32_t page[kMaxTilePages];
};

struct Smem {
    uint8_t kst[kKStages][kKStageBytes];  // 1024-B aligned (offset 0): K halves, then Q
    uint8_t vst[kVStages][kKVBytes];
    uint8_t p[2][kPBytes];
    uint64_t kfull[kKStages], kempty[kKStages];
    uint64_t vfull[kVStages], vempty[kVStages];
    uint64_t mready[kMeta];
    uint64_t s_full, s_free;
    uint64_t p_full[2], o_full[2], o_free[2];
    TileMeta meta[kMeta];
    int32_t pid[kPidWin];  // page ids of the current item's window
    float red_max[2][4][kN];
    float red_sum[4][kN];
    MergeQueue mq;  // completed groups -> merge warp
    uint32_t tmem_base;
};

// ---------------------------------------------------------------- PTX
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// 4-D box {64 d, page rows, 1 kv head, 128/P pages}: a whole 128-token tile
// half when the tile's pages are consecutive in the pool
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)),
        "l"(policy)
        : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// UMMA shared-memory descriptor, 128-B swizzle, sm_100 version bits.
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= static_cast<uint64_t>(1) << 46;  // version
    d |= static_cast<uint64_t>(2) << 61;  // SWIZZLE_128B
    return d;
}

// kind::f16 instruction descriptor: bf16 x bf16 -> fp32, M = 128, N = 16.
__host__ __device__ constexpr uint32_t idesc(uint32_t a_mn_major) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (a_mn_major << 15) | (0u << 16) |
           (static_cast<uint32_t>(kN >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t id,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(id), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ int find_item_range(const int32_t* prefix, int n, int item) {
    int lo = 0, hi = n;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(prefix + mid) <= item) lo = mid; else hi = mid;
    }
    return lo;
}

// byte offset of element (row, col) in a 128-B-swizzled K-major operand made of
// two 64-column halves of `rows` rows each (half stride rows*128 B)
__device__ __forceinline__ uint32_t swz_off(int row, int col, int rows) {
    const int half = col >> 6;
    const int c = (col & 63) >> 3;
    return static_cast<uint32_t>(half * rows * 128 + (row >> 3) * 1024 + (row & 7) * 128 +
                                 ((c ^ (row & 7)) << 4) + ((col & 7) << 1));
}

// order-preserving float <-> int map so a warp max is one REDUX instruction
__device__ __forceinline__ int f2ord(float f) {
    const int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float ord2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7FFFFFFF); }

template <int NC>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, float (&v)[NC]) {
    uint32_t r[NC];
    if constexpr (NC == 16) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
              "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
    } else if constexpr (NC == 8) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                       "=r"(r[6]), "=r"(r[7])
                     : "r"(taddr));
    } else if constexpr (NC == 4) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                     : "r"(taddr));
    } else {
        static_assert(NC == 2, "unsupported column count");
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];"
                     : "=r"(r[0]), "=r"(r[1])
                     : "r"(taddr));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < NC; ++i) v[i] = __uint_as_float(r[i]);
}

// GI: compile-time bound on the q group (2, 4, 8, 16); p.group <= GI, extra
// heads are zero rows of Q and their columns are never written out.
template <int GI>
__global__ void __launch_bounds__(kThreads, 1)
    gqa_tc_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                  const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k4,
                  const __grid_constant__ CUtensorMap tm_v4, const MAParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // the swizzle pattern is tied to 1024-B address alignment
    Smem& S = *reinterpret_cast<Smem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = p.group;
    pdl_launch_dependents();  // the merge launch may queue up behind this grid

    if (threadIdx.x == 0) {
        for (int i = 0; i < kKStages; ++i) {
            mbar_init(&S.kfull[i], 1);
            mbar_init(&S.kempty[i], 1);
        }
        for (int i = 0; i < kVStages; ++i) {
            mbar_init(&S.vfull[i], 1);
            mbar_init(&S.vempty[i], 1);
        }
        for (int i = 0; i < kMeta; ++i) mbar_init(&S.mready[i], 1);
        S.mq.tail = 0;
        S.mq.head = 0;
        for (int i = 0; i < kMergeQueue; ++i) S.mq.seq[i] = 0;
        mbar_init(&S.s_full, 1);
        mbar_init(&S.s_free, 4);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&S.o_full[b], 1);
            mbar_init(&S.p_full[b], 4);
            mbar_init(&S.o_free[b], 4);
        }
        fence_mbar_init();
    }
    // zero the operand buffers once: padded Q / P rows must be 0 and stale
    // rows of partially filled tiles must be finite
    for (int i = threadIdx.x; i < (kKStages * kKStageBytes + kVStages * kKVBytes + 2 * kPBytes) / 16;
         i += kThreads)
        reinterpret_cast<uint4*>(S.kst)[i] = make_uint4(0, 0, 0, 0);
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&S.tmem_base)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tm_k);
        prefetch_tmap(&tm_v);
        prefetch_tmap(&tm_q);
        prefetch_tmap(&tm_k4);
        prefetch_tmap(&tm_v4);
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // launched with programmatic serialization behind the previous step's
    // merge grid: the set-up above (barriers, operand zeroing, TMEM, tensor
    // maps) overlapped its tail; records, q and the work counter are touched
    // only after it has completed
    pdl_wait();
    const uint32_t tmem = S.tmem_base;
    const uint32_t tmem_s = tmem;
    const uint32_t tmem_o0 = tmem + kN;  // O^T of even tiles; odd tiles at + kN
    const int P = p.page_tokens;

    if (warp == 0) {
        // ================================ K producer
        // Lane 0 publishes the tile descriptors and streams K (+ Q) tiles
        // into the K ring. The NEXT item is fetched during the current one's
        // last tiles, one dependent step per tile (the producer mostly waits
        // for ring slots): claim (atomic), claim-table entry, range + chunk
        // prefix, the whole warp's page-id loads into registers; the ids go
        // to shared memory at the boundary. An item boundary then costs no
        // round trip, which matters for the short items of ragged batches,
        // of fine tails and of the small per-GPU shares at N > 1. The claim is
        // made only kAhead (5) tiles before the end, so a CTA never sits on an
        // item another CTA could have started (the launch's tail).
        const uint64_t pol = l2_policy_evict_first();
        constexpr int kIdsPerLane = kPidWin / 32;
        const int kAhead = p.claim_ahead;  // tiles before an item's end at which the next claim starts
        struct Item {
            int item, kvh, tlo, thi, gchunk, start, plast;
            RangeDev rg;
        };
        // decode a claimed item from its (range, local) pair
        auto decode = [&](Item& it, int r, int local, const RangeDev& rg, int cprefix) {
            const int nh = rg.kv_head < 0 ? p.num_kv_heads : 1;
            const int j = local / nh;
            it.rg = rg;
            it.kvh = rg.kv_head < 0 ? local - j * nh : rg.kv_head;
            it.tlo = rg.lo + j * p.chunk_tokens;
            it.thi = min(rg.hi, it.tlo + p.chunk_tokens);
            it.gchunk = cprefix + j;
            it.start = (it.tlo / P) * P;
            it.plast = (it.thi - 1) / P;
            (void)r;
        };
        // next-item pipeline state
        int stage = 0;          // 0 idle, 1 claim issued, 2 entry loaded, 3 range loaded, 4 ids in registers, 5 ready
        unsigned long long raw = 0;
        int nitem = 0, nr = 0, nlocal = 0, ncp = 0;
        int2 nentry = make_int2(0, 0);
        RangeDev nrg{};
        Item nxt{};
        int nids[kIdsPerLane];
        auto advance = [&]() {  // one dependent step of the next item's fetch
            if (stage == 0) {
                if (lane == 0) raw = atomicAdd(p.work_counter, 1ull);
                stage = 1;
            } else if (stage == 1) {
                nitem = __shfl_sync(0xffffffffu, static_cast<int>(raw - p.work_base), 0);
                if (nitem >= p.nitems) {
                    stage = 5;
                } else {
                    if (p.item_table) nentry = __ldg(reinterpret_cast<const int2*>(p.item_table) + nitem);
                    stage = 2;
                }
            } else if (stage == 2) {
                if (p.item_table) {
                    nr = nentry.x;
                    nlocal = nentry.y;
                } else {
                    nr = find_item_range(p.item_prefix, p.nranges, nitem);
                    nlocal = nitem - __ldg(p.item_prefix + nr);
                }
                nrg = p.ranges[nr];
                ncp = __ldg(p.chunk_prefix + nr);
                stage = 3;
            } else if (stage == 3) {
                decode(nxt, nr, nlocal, nrg, ncp);
                nxt.item = nitem;
                const int32_t* bt = p.block_tables + static_cast<int64_t>(nxt.rg.seq) * p.bt_stride;
                const int w0 = nxt.start / P;
#pragma unroll
                for (int i = 0; i < kIdsPerLane; ++i) {
                    const int k = i * 32 + lane;
                    nids[i] = (w0 + k <= nxt.plast) ? __ldg(bt + w0 + k) : 0;
                }
                stage = 4;
            } else if (stage == 4) {
                stage = 5;  // stored at the item boundary (the buffer is in use until then)
            }
        };
        auto finish = [&]() {  // complete the fetch synchronously
            while (stage < 5) advance();
        };

        uint32_t t = 0;  // global tile counter of this CTA
        finish();
        while (nitem < p.nitems) {
            // the prefetched item becomes current: its page ids into S.pid
            const Item cur = nxt;
#pragma unroll
            for (int i = 0; i < kIdsPerLane; ++i) S.pid[i * 32 + lane] = nids[i];
            __syncwarp();
            int win = cur.start / P;  // first page id held in S.pid
            stage = 0;
            const int ntiles = (cur.thi - cur.start + kTile - 1) / kTile;
            int k = 0;  // tile index within the item
            const int qrow = cur.rg.out_row * p.num_q_heads + cur.kvh * G;
            const int32_t* bt = p.block_tables + static_cast<int64_t>(cur.rg.seq) * p.bt_stride;
            for (int t0 = cur.start; t0 < cur.thi; t0 += kTile, ++t) {
                const int tend = min(cur.thi, t0 + kTile);
                const int pg0 = t0 / P, npages = (tend - 1) / P - pg0 + 1;
                if (pg0 + npages > win + kPidWin) {  // an unaligned item longer than the window
                    __syncwarp();
                    win = pg0;
                    for (int i = lane; i < kPidWin; i += 32)
                        if (win + i <= cur.plast) S.pid[i] = __ldg(bt + win + i);
                    __syncwarp();
                }
                if (ntiles - k++ <= kAhead) advance();
                if (lane == 0) {
                    TileMeta& md = S.meta[t % kMeta];
                    md.item = cur.item;
                    md.tile0 = t0;
                    md.tlo = cur.tlo;
                    md.thi = cur.thi;
                    md.flags = (t0 == cur.start ? 1 : 0) | (t0 + kTile >= cur.thi ? 2 : 0);
                    md.row = cur.rg.out_row;
                    md.kvh = cur.kvh;
                    md.gchunk = cur.gchunk;
                    md.npages = npages;
                    bool run = npages * P == kTile;  // a full tile of consecutive pages
                    for (int pg = 0; pg < npages; ++pg) {
                        md.page[pg] = S.pid[pg0 - win + pg];
                        run = run && md.page[pg] == md.page[0] + pg;
                    }
                    md.flags |= run ? 4 : 0;
                    mbar_arrive(&S.mready[t % kMeta]);
                    const int ks = t % kKStages;
                    mbar_wait(&S.kempty[ks], ((t / kKStages) & 1u) ^ 1u);
                    mbar_arrive_expect_tx(&S.kfull[ks], static_cast<uint32_t>(npages * P * 128 * 2 + G * 128 * 2));
                    uint8_t* sk = S.kst[ks];
                    uint8_t* sq = sk + kKVBytes;
                    if (run) {
                        // one box per 64-column half instead of two per page
                        tma_load_4d(sk, &tm_k4, 0, 0, cur.kvh, md.page[0], &S.kfull[ks], pol);
                        tma_load_4d(sk + kHalf, &tm_k4, 64, 0, cur.kvh, md.page[0], &S.kfull[ks], pol);
                    } else {
                        for (int pg = 0; pg < npages; ++pg) {
                            const int row0 = (md.page[pg] * p.num_kv_heads + cur.kvh) * P;
                            const int off = pg * P * 128;
                            tma_load_2d(sk + off, &tm_k, 0, row0, &S.kfull[ks], pol);
                            tma_load_2d(sk + kHalf + off, &tm_k, 64, row0, &S.kfull[ks], pol);
                        }
                    }
                    tma_load_2d(sq, &tm_q, 0, qrow, &S.kfull[ks], 0);
                    tma_load_2d(sq + kN * 128, &tm_q, 64, qrow, &S.kfull[ks], 0);
                }
                __syncwarp();
            }
            finish();
        }
        if (lane == 0) {
            S.meta[t % kMeta].item = -1;
            mbar_arrive(&S.mready[t % kMeta]);
            const int ks = t % kKStages;
            mbar_wait(&S.kempty[ks], ((t / kKStages) & 1u) ^ 1u);
            mbar_arrive(&S.kfull[ks]);
        }
    } else if (warp == 7) {
        // ================================ merge warp (fused modes)
        if (p.fused_mode != 0) {
            for (int idx = 0;; ++idx) {
                int32_t v = 0;
                if (lane == 0) v = mq_pop(&S.mq, idx);
                v = __shfl_sync(0xffffffffu, v, 0);
                if (v < 0) break;
                __threadfence();
                warp_group_merge<bf16_t, kD, (GI < 8 ? GI : 8)>(p, v >> 8, v & 0xFF, lane);
            }
        }
    } else if (warp == 6) {
        // ================================ V producer (trails the K producer)
        if (lane == 0) {
            const uint64_t pol = l2_policy_evict_first();
            for (uint32_t t = 0;; ++t) {
                mbar_wait(&S.mready[t % kMeta], (t / kMeta) & 1u);
                const TileMeta& md = S.meta[t % kMeta];
                if (md.item < 0) break;
                const int npages = md.npages, kvh = md.kvh;
                int page[kMaxTilePages];
#pragma unroll
                for (int pg = 0; pg < kMaxTilePages; ++pg) page[pg] = md.page[pg];
                const bool run = (md.flags & 4) != 0;
                const int vs = t % kVStages;
                mbar_wait(&S.vempty[vs], ((t / kVStages) & 1u) ^ 1u);
                mbar_arrive_expect_tx(&S.vfull[vs], static_cast<uint32_t>(npages * P * 128 * 2));
                uint8_t* sv = S.vst[vs];
                if (run) {
                    tma_load_4d(sv, &tm_v4, 0, 0, kvh, page[0], &S.vfull[vs], pol);
                    tma_load_4d(sv + kHalf, &tm_v4, 64, 0, kvh, page[0], &S.vfull[vs], pol);
                } else {
                    for (int pg = 0; pg < npages; ++pg) {
                        const int row0 = (page[pg] * p.num_kv_heads + kvh) * P;
                        const int off = pg * P * 128;
                        tma_load_2d(sv + off, &tm_v, 0, row0, &S.vfull[vs], pol);
                        tma_load_2d(sv + kHalf + off, &tm_v, 64, row0, &S.vfull[vs], pol);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ================================ MMA issuer
        // MMA1 of tile t+1 is issued before MMA2 of tile t, so the softmax
        // warps find S^T(t+1) ready as soon as they hand over P(t). MMA1's
        // commit releases the K stage, MMA2's the V stage.
        const uint32_t id1 = idesc(0), id2 = idesc(1);
        auto issue_s = [&](uint32_t t) {
            const int ks = t % kKStages;
            const uint32_t sk = smem_u32(S.kst[ks]);
            const uint32_t sq = sk + kKVBytes;
            tc_fence_after();
            if (lane == 0) {
#pragma unroll
                for (int k = 0; k < kD / 16; ++k) {
                    const uint32_t koff = (k >> 2) * kHalf + (k & 3) * 32;
                    const uint32_t qoff = (k >> 2) * (kN * 128) + (k & 3) * 32;
                    mma_bf16(tmem_s, sdesc(sk + koff, 16, 1024), sdesc(sq + qoff, 16, 1024), id1, k > 0);
                }
                mma_commit(&S.s_full);
                mma_commit(&S.kempty[ks]);
            }
            __syncwarp();
        };
        mbar_wait(&S.kfull[0], 0);
        if (S.meta[0].item >= 0) {
            issue_s(0);
            for (uint32_t t = 0;; ++t) {
                const uint32_t tn = t + 1;
                mbar_wait(&S.kfull[tn % kKStages], (tn / kKStages) & 1u);
                const bool more = S.meta[tn % kMeta].item >= 0;
                if (more) {
                    mbar_wait(&S.s_free, t & 1u);  // softmax warps hold S^T(t) in registers
                    issue_s(tn);
                }
                // MMA2 of tile t: needs V(t), P^T(t) and its O^T buffer released
                const int vs = t % kVStages;
                const uint32_t ob = t & 1u, oph = (t >> 1) & 1u;
                mbar_wait(&S.vfull[vs], (t / kVStages) & 1u);
                mbar_wait(&S.p_full[ob], oph);
                mbar_wait(&S.o_free[ob], oph ^ 1u);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t sv = smem_u32(S.vst[vs]);
                    const uint32_t sp = smem_u32(S.p[ob]);
#pragma unroll
                    for (int k = 0; k < kTile / 16; ++k) {
                        const uint32_t voff = k * 2048;  // 16 token rows of 128 B
                        const uint32_t poff = (k >> 2) * (kN * 128) + (k & 3) * 32;
                        mma_bf16(tmem_o0 + ob * kN, sdesc(sv + voff, kHalf, 1024), sdesc(sp + poff, 16, 1024),
                                 id2, k > 0);
                    }
                    mma_commit(&S.o_full[ob]);
                    mma_commit(&S.vempty[vs]);
                }
                __syncwarp();
                if (!more) break;
            }
        }
    } else {
        // ================================ softmax / epilogue (warps 2..5)
        const int ew = warp & 3;              // TMEM lane quadrant this warp may access
        const int row = ew * 32 + lane;       // token row of S^T, then d row of O^T
        const uint32_t lane_addr = static_cast<uint32_t>(ew * 32) << 16;
        const float sl2 = static_cast<float>(p.scale_log2);
        const float kNegInf = -INFINITY;
        float m[GI], l[GI], acc[GI], corr_prev[GI];
        bool pending = false;  // an O^T tile of the current item not yet accumulated
        float* recs = static_cast<float*>(p.records);
        // An item's last O^T tile is still in the tensor pipe when its softmax
        // is done; rather than wait for it, the item is finished one tile
        // later, after the next item's first P^T has been handed to the MMA
        // warp, so item boundaries do not drain the pipeline.
        bool fin = false;
        float fin_acc[GI], fin_corr[GI], fin_m[GI], fin_l[GI];
        uint32_t fin_ob = 0, fin_oph = 0;
        int64_t fin_rec0 = 0;
        float fin_ntok = 0.f;
        int fin_row = 0, fin_kvh = 0;
        auto finish = [&]() {
            mbar_wait(&S.o_full[fin_ob], fin_oph);
            tc_fence_after();
            float o[GI];
            tmem_ld<GI>(tmem_o0 + fin_ob * kN + lane_addr, o);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.o_free[fin_ob]);
#pragma unroll
            for (int h = 0; h < GI; ++h) fin_acc[h] = fin_acc[h] * fin_corr[h] + o[h];
            // e = sum over the 128 token rows of l
#pragma unroll
            for (int h = 0; h < GI; ++h) {
                float v = fin_l[h];
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                if (lane == 0) S.red_sum[ew][h] = v;
            }
            named_bar_sync(1, 128);
#pragma unroll
            for (int h = 0; h < GI; ++h) {
                if (h >= G) continue;
                float* rec = recs + (fin_rec0 + h) * (kD + 4);
                rec[4 + row] = fin_acc[h];
                if (row == 0) {
                    rec[0] = fin_m[h] * 0.6931471805599453f;
                    rec[1] = (S.red_sum[0][h] + S.red_sum[1][h]) + (S.red_sum[2][h] + S.red_sum[3][h]);
                    rec[2] = fin_ntok;
                    rec[3] = 0.f;
                }
            }
            named_bar_sync(1, 128);
            if (p.fused_mode != 0 && warp == 2 && lane == 0) {
                // group completion (see K1): the CTA that wrote the last
                // chunk of (row, kv head) hands it to the merge warp
                const int gi = fin_row * p.num_kv_heads + fin_kvh;
                const int old = atomic_add_acq_rel_gpu(p.group_counter + gi, 1);
                if (old + 1 == __ldg(p.group_expected + gi)) {
                    p.group_counter[gi] = 0;
                    mq_push(&S.mq, (fin_row << 8) | fin_kvh);
                }
            }
            fin = false;
        };
        for (uint32_t it = 0;; ++it) {
            mbar_wait(&S.mready[it % kMeta], (it / kMeta) & 1u);
            const TileMeta md = S.meta[it % kMeta];
            if (md.item < 0) {
                if (fin) finish();
                break;
            }
            if (md.flags & 1) {
#pragma unroll
                for (int h = 0; h < GI; ++h) {
                    m[h] = kNegInf;
                    l[h] = 0.f;
                    acc[h] = 0.f;
                }
            }
            // ---- S^T row of this thread's token
            mbar_wait(&S.s_full, it & 1u);
            tc_fence_after();
            float s[GI];
            tmem_ld<GI>(tmem_s + lane_addr, s);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.s_free);
            const int tok = md.tile0 + row;
            const bool valid = tok >= md.tlo && tok < md.thi;
            const int rb = it & 1u;
#pragma unroll
            for (int h = 0; h < GI; ++h) {
                s[h] = valid ? s[h] * sl2 : kNegInf;
                const int wmax = __reduce_max_sync(0xffffffffu, f2ord(s[h]));
                if (lane == 0) S.red_max[rb][ew][h] = ord2f(wmax);
            }
            named_bar_sync(1, 128);
            float corr[GI];
#pragma unroll
            for (int h = 0; h < GI; ++h) {
                float mx = fmaxf(fmaxf(S.red_max[rb][0][h], S.red_max[rb][1][h]),
                                 fmaxf(S.red_max[rb][2][h], S.red_max[rb][3][h]));
                mx = fmaxf(mx, m[h]);
                corr[h] = (mx == m[h]) ? 1.f : fast_exp2(m[h] - mx);
                m[h] = mx;
            }
            // ---- P^T (bf16, swizzled K-major) into buffer it&1, running sums
            const uint32_t ob = it & 1u, oph = (it >> 1) & 1u;
#pragma unroll
            for (int h = 0; h < GI; ++h) {
                const float pv = valid ? fast_exp2(s[h] - m[h]) : 0.f;
                const bf16_t pb = Elem<bf16_t>::from_acc(pv);
                l[h] = l[h] * corr[h] + Elem<bf16_t>::to_acc(pb);
                *reinterpret_cast<uint16_t*>(S.p[ob] + swz_off(h, row, kN)) = pb.bits;
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.p_full[ob]);
            if (fin) finish();  // the previous item, now that P^T(it) is queued
            // ---- O^T of the PREVIOUS tile (deferred so this tile's softmax did
            //      not wait for its P.V round trip): acc = acc*corr_prev + O_prev
            if (pending) {
                const uint32_t pb_ = ob ^ 1u, pph = ((it - 1) >> 1) & 1u;
                mbar_wait(&S.o_full[pb_], pph);
                tc_fence_after();
                float o[GI];
                tmem_ld<GI>(tmem_o0 + pb_ * kN + lane_addr, o);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&S.o_free[pb_]);
#pragma unroll
                for (int h = 0; h < GI; ++h) acc[h] = acc[h] * corr_prev[h] + o[h];
            }
#pragma unroll
            for (int h = 0; h < GI; ++h) corr_prev[h] = corr[h];
            pending = true;
            if (md.flags & 2) {
                // last tile of the item: finish() accumulates its O^T and
                // writes the record during the next tile
#pragma unroll
                for (int h = 0; h < GI; ++h) {
                    fin_acc[h] = acc[h];
                    fin_corr[h] = corr[h];
                    fin_m[h] = m[h];
                    fin_l[h] = l[h];
                }
                fin_ob = ob;
                fin_oph = oph;
                fin_rec0 = static_cast<int64_t>(md.gchunk) * p.num_q_heads + static_cast<int64_t>(md.kvh) * G;
                fin_ntok = static_cast<float>(md.thi - md.tlo);
                fin_row = md.row;
                fin_kvh = md.kvh;
                fin = true;
                pending = false;
            }
        }
        if (p.fused_mode != 0) {
            named_bar_sync(1, 128);
            if (warp == 2 && lane == 0) mq_push(&S.mq, -1);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols)
                     : "memory");
    }
}

}  // namespace tc

size_t gqa_tc_smem_bytes() { return sizeof(tc::Smem) + 1024; }

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

// 2-D bf16 view [rows][128] with a (64 x box_rows) box and the 128-B swizzle.
cudaError_t make_tmap_rows128(void* map_out, const void* base, uint64_t rows, uint32_t box_rows) {
    auto fn = encode_fn();
    if (!fn) return cudaErrorNotSupported;
    cuuint64_t dims[2] = {128, rows};
    cuuint64_t strides[1] = {128 * 2};
    cuuint32_t box[2] = {64, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(reinterpret_cast<CUtensorMap*>(map_out), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                    const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// 4-D bf16 view {128 d, P rows, Hkv, pages} of a pool with a {64, P, 1, 128/P}
// box and the 128-B swizzle: one copy moves a 64-column half of a whole tile
// of consecutive pages into the same shared-memory layout as 128/P 2-D boxes.
cudaError_t make_tmap_tiles(void* map_out, const void* base, uint64_t pages, uint32_t kv_heads, uint32_t page_tokens) {
    auto fn = encode_fn();
    if (!fn) return cudaErrorNotSupported;
    cuuint64_t dims[4] = {128, page_tokens, kv_heads, pages};
    cuuint64_t strides[3] = {128 * 2, static_cast<cuuint64_t>(page_tokens) * 256,
                             static_cast<cuuint64_t>(kv_heads) * page_tokens * 256};
    cuuint32_t box[4] = {64, page_tokens, 1, tc::kTile / page_tokens};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = fn(reinterpret_cast<CUtensorMap*>(map_out), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
                    const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

static const void* gqa_fn(int group) {
    if (group <= 2) return reinterpret_cast<const void*>(&tc::gqa_tc_kernel<2>);
    if (group <= 4) return reinterpret_cast<const void*>(&tc::gqa_tc_kernel<4>);
    if (group <= 8) return reinterpret_cast<const void*>(&tc::gqa_tc_kernel<8>);
    return reinterpret_cast<const void*>(&tc::gqa_tc_kernel<16>);
}

cudaError_t gqa_tc_configure() {
    for (int g : {2, 4, 8, 16}) {
        const cudaError_t e = cudaFuncSetAttribute(gqa_fn(g), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(gqa_tc_smem_bytes()));
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_gqa_tc(const void* tm_k, const void* tm_v, const void* tm_q, const void* tm_k4,
                          const void* tm_v4, const MAParams& p, int grid, cudaStream_t st) {
    MAParams pp = p;
    void* args[] = {const_cast<void*>(tm_k), const_cast<void*>(tm_v), const_cast<void*>(tm_q),
                    const_cast<void*>(tm_k4), const_cast<void*>(tm_v4), &pp};
    return launch_pdl_raw(gqa_fn(p.group), grid, tc::kThreads, gqa_tc_smem_bytes(), st, args);
}

}  // namespace dattn
