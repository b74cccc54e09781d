// dattn_kernels.cu -- sm_100a kernels of the DistAttention decode path.
//
//   K1 ma_decode_kernel   micro-attention partials (m, e, ma) per
//                         (chunk, q head): compute_micro_attention,
//                         /root/reference/proj/src/distattention.cpp:99-129,
//                         batched over a paged KV store.
//   K3 merge_kernel       online-softmax rescale-and-sum of partial records:
//                         combine_partials / aggregate_partials,
//                         distattention.cpp:131-174.
//   K4 fill_kv_kernel     deterministic counter-hash K/V generation into pages
//                         (CPU twin: oracle/dattn_oracle.c or_synth_kv).
//
// K1 design: persistent CTAs, one producer warp whose elected
// lane streams each work item's K/V token rows from the page pool into a ring
// of shared-memory stages with 1-D bulk TMA (cp.async.bulk, mbarrier
// complete_tx, L2 evict_first), and 8 consumer warps that read 16-B chunks
// from shared memory (8 lanes per token row, conflict-free LDS.128), reduce
// q.k with warp shuffles and run an online softmax in registers. Work items
// (range, chunk, kv head) are claimed with an atomic counter so ragged
// batches balance across the 148 SMs.
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <cstdint>
#include <type_traits>

#include "dattn_internal.h"
#include "dattn_ptx.cuh"
#include "dattn_merge.cuh"

namespace dattn {

constexpr int kMAThreads = 32 * (1 + kConsumerWarps + 1);  // producer, consumers, merge warp
constexpr int kStageSlotBytes = 16384;  // bytes of K (and of V) per pipeline stage
constexpr int kPidWindow = 256;         // block-table entries cached per window

int ma_threads() { return kMAThreads; }

template <typename T, int DP>
struct Shape {
    static constexpr int kRowBytes = DP * static_cast<int>(sizeof(T));
    static constexpr int kChunks = kRowBytes / 16;               // 16-B chunks per row
    static constexpr int kLPT = kChunks < 8 ? kChunks : 8;       // lanes per token row
    static constexpr int kTPW = 32 / kLPT;                       // token rows per warp pass
    static constexpr int kCPL = kChunks / kLPT;                  // chunks per lane
    static constexpr int kVec = 16 / static_cast<int>(sizeof(T));
    static constexpr int kEPL = kCPL * kVec;                     // elements per lane
    static constexpr int kRawStage = kStageSlotBytes / kRowBytes;
    static constexpr int kStageTokens = kRawStage < 8 ? 8 : (kRawStage > 512 ? 512 : kRawStage);
    static constexpr int kPassTokens = kConsumerWarps * kTPW;
    static constexpr int kUnrollRaw = kStageTokens / kPassTokens;
    static constexpr int kUnroll = kUnrollRaw < 1 ? 1 : (kUnrollRaw > 4 ? 4 : kUnrollRaw);
    static constexpr int kRec = DP + 4;
};

struct StageMeta {
    int32_t item;  // -1: terminate
    int32_t ntok;
    int32_t flags;  // 1 first stage of item, 2 last stage
    int32_t row;
    int32_t kvh;
    int32_t gchunk;
    int32_t item_tokens;
    int32_t pad;
};

__host__ __device__ constexpr size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Shared-memory carve-up, identical on host and device.
template <typename T, int DP>
struct Layout {
    using Acc = typename Elem<T>::Acc;
    size_t bars, meta, pid, red_m, red_e, red_acc, stage0, stage_bytes, k_off, v_off, q_off,
        total;
    __host__ __device__ Layout(int stages, int group) {
        using S = Shape<T, DP>;
        size_t o = 0;
        bars = o;
        o += sizeof(uint64_t) * 2 * stages;
        o = align_up(o, 16);
        meta = o;
        o += sizeof(StageMeta) * stages;
        pid = o;
        o += sizeof(int32_t) * kPidWindow;
        o = align_up(o, 16);
        red_m = o;
        o += sizeof(Acc) * kConsumerWarps;
        red_e = o;
        o += sizeof(Acc) * kConsumerWarps;
        o = align_up(o, 16);
        red_acc = o;
        o += sizeof(Acc) * kConsumerWarps * DP;
        o = align_up(o, 128);
        stage0 = o;
        k_off = 0;
        v_off = align_up(static_cast<size_t>(S::kStageTokens) * S::kRowBytes, 128);
        q_off = v_off + v_off;
        stage_bytes = align_up(q_off + static_cast<size_t>(group) * S::kRowBytes, 128);
        total = stage0 + stage_bytes * stages;
    }
};

// Blackwell packed fp32 FMA (SASS FFMA2): (d0, d1) += (a0, a1) * (b0, b1).
__device__ __forceinline__ void ffma2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
    asm("{\n\t.reg .b64 ra, rb, rc;\n\t"
        "mov.b64 ra, {%2, %3};\n\t"
        "mov.b64 rb, {%4, %5};\n\t"
        "mov.b64 rc, {%0, %1};\n\t"
        "fma.rn.f32x2 rc, ra, rb, rc;\n\t"
        "mov.b64 {%0, %1}, rc;\n\t}"
        : "+f"(d0), "+f"(d1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

__device__ __forceinline__ int find_range(const int32_t* prefix, int n, int item) {
    // largest r with prefix[r] <= item (prefix[0] == 0, prefix[n] > item)
    int lo = 0, hi = n;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(prefix + mid) <= item) lo = mid; else hi = mid;
    }
    return lo;
}

template <typename T, int DP, int HPW>
__global__ void __launch_bounds__(kMAThreads, (sizeof(T) == 8 || HPW > 1) ? 1 : 2)
    ma_decode_kernel(const MAParams p) {
    using S = Shape<T, DP>;
    using E = Elem<T>;
    using Acc = typename E::Acc;
    constexpr int LPT = S::kLPT, TPW = S::kTPW, CPL = S::kCPL, VEC = S::kVec, EPL = S::kEPL;
    constexpr int TS = S::kStageTokens, U = S::kUnroll, REC = S::kRec;

    extern __shared__ __align__(128) uint8_t smem[];
    pdl_launch_dependents();  // the merge launch may queue up behind this grid
    const Layout<T, DP> L(p.stages, p.group);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* empty = full + p.stages;
    StageMeta* meta = reinterpret_cast<StageMeta*>(smem + L.meta);
    int32_t* pid = reinterpret_cast<int32_t*>(smem + L.pid);
    Acc* red_m = reinterpret_cast<Acc*>(smem + L.red_m);
    Acc* red_e = reinterpret_cast<Acc*>(smem + L.red_e);
    Acc* red_acc = reinterpret_cast<Acc*>(smem + L.red_acc);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int stages = p.stages;

    __shared__ MergeQueue mq;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        fence_mbar_init();
        mq.tail = 0;
        mq.head = 0;
    }
    if (threadIdx.x < kMergeQueue) mq.seq[threadIdx.x] = 0;
    __syncthreads();
    // launched with programmatic serialization behind the previous step's
    // merge grid: the set-up above overlapped its tail; records, q and the
    // work counter are touched only after it has completed
    pdl_wait();

    if (warp == kConsumerWarps + 1) {
        // ===================== merge warp (fused modes) =====================
        // merges each (row, kv head) group whose last chunk this CTA wrote,
        // concurrently with the streaming warps
        if (p.fused_mode == 0) return;
        for (int idx = 0;; ++idx) {
            int32_t v = 0;
            if (lane == 0) v = mq_pop(&mq, idx);
            v = __shfl_sync(0xffffffffu, v, 0);
            if (v < 0) break;
            __threadfence();  // acquire the other CTAs' records of the group
            warp_group_merge<T, DP, (sizeof(T) == 8 ? 2 : 8)>(p, v >> 8, v & 0xFF, lane);
        }
        return;
    }

    if (warp == 0) {
        // ===================== producer warp =====================
        const uint64_t pol = l2_policy_evict_first();
        const T* kpool = static_cast<const T*>(p.k_pool);
        const T* vpool = static_cast<const T*>(p.v_pool);
        const T* qg = static_cast<const T*>(p.q);
        const int P = p.page_tokens;
        const uint32_t qbytes = static_cast<uint32_t>(p.group) * S::kRowBytes;
        int stage = 0;
        uint32_t phase = 0;
        for (;;) {
            int item = 0;
            if (lane == 0) item = static_cast<int>(atomicAdd(p.work_counter, 1ull) - p.work_base);
            item = __shfl_sync(0xffffffffu, item, 0);
            if (item >= p.nitems) break;
            int r, local;
            if (p.item_table) {  // longest-first claim order (one load replaces the search)
                const int2 e = __ldg(reinterpret_cast<const int2*>(p.item_table) + item);
                r = e.x;
                local = e.y;
            } else {
                r = find_range(p.item_prefix, p.nranges, item);
                local = item - __ldg(p.item_prefix + r);
            }
            const RangeDev rg = p.ranges[r];
            const int nh = rg.kv_head < 0 ? p.num_kv_heads : 1;
            const int j = local / nh;
            const int kvh = rg.kv_head < 0 ? local - j * nh : rg.kv_head;
            const int tlo = rg.lo + j * p.chunk_tokens;
            const int thi = min(rg.hi, tlo + p.chunk_tokens);
            const int gchunk = __ldg(p.chunk_prefix + r) + j;
            const int32_t* bt = p.block_tables + static_cast<int64_t>(rg.seq) * p.bt_stride;
            int win_lo = -1;
            for (int t0 = tlo; t0 < thi; t0 += TS) {
                const int n = min(TS, thi - t0);
                const int pf = t0 / P, pl = (t0 + n - 1) / P;
                if (win_lo < 0 || pl >= win_lo + kPidWindow) {
                    __syncwarp();
                    win_lo = pf;
                    const int plast = (thi - 1) / P;
                    for (int i = lane; i < kPidWindow; i += 32)
                        if (win_lo + i <= plast) pid[i] = __ldg(bt + win_lo + i);
                    __syncwarp();
                }
                if (lane == 0) {
                    mbar_wait(&empty[stage], phase ^ 1u);
                    const bool first = (t0 == tlo);
                    StageMeta& md = meta[stage];
                    md.item = item;
                    md.ntok = n;
                    md.flags = (first ? 1 : 0) | (t0 + TS >= thi ? 2 : 0);
                    md.row = rg.out_row;
                    md.kvh = kvh;
                    md.gchunk = gchunk;
                    md.item_tokens = thi - tlo;
                    uint8_t* sb = smem + L.stage0 + L.stage_bytes * stage;
                    T* ks = reinterpret_cast<T*>(sb + L.k_off);
                    T* vs = reinterpret_cast<T*>(sb + L.v_off);
                    mbar_arrive_expect_tx(&full[stage],
                                          2u * n * S::kRowBytes + (first ? qbytes : 0u));
                    for (int t = t0; t < t0 + n;) {
                        const int pi = t / P;
                        const int off = t - pi * P;
                        const int cnt = min(P - off, t0 + n - t);
                        const int64_t page = pid[pi - win_lo];
                        const int64_t row = (page * p.num_kv_heads + kvh) * P + off;
                        const uint32_t bytes = static_cast<uint32_t>(cnt) * S::kRowBytes;
                        bulk_g2s(ks + static_cast<int64_t>(t - t0) * DP, kpool + row * DP, bytes,
                                 &full[stage], pol);
                        bulk_g2s(vs + static_cast<int64_t>(t - t0) * DP, vpool + row * DP, bytes,
                                 &full[stage], pol);
                        t += cnt;
                    }
                    if (first) {
                        const T* qsrc =
                            qg + (static_cast<int64_t>(rg.out_row) * p.num_q_heads +
                                  static_cast<int64_t>(kvh) * p.group) * DP;
                        bulk_g2s_nohint(sb + L.q_off, qsrc, qbytes, &full[stage]);
                    }
                }
                __syncwarp();
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
        if (lane == 0) {
            mbar_wait(&empty[stage], phase ^ 1u);
            meta[stage].item = -1;
            mbar_arrive(&full[stage]);
        }
        return;
    }

    // ===================== consumer warps =====================
    const int cw = warp - 1;
    const int gslots = p.group < kConsumerWarps ? p.group : kConsumerWarps;
    const int wph = kConsumerWarps / gslots;  // warps sharing one q head
    const bool active = cw < wph * gslots;
    const int hslot = cw % gslots;
    const int slice = cw / gslots;
    const int grp = lane / LPT;
    const int sub = lane - grp * LPT;
    const Acc scale_log2 = static_cast<Acc>(p.scale_log2);
    const Acc kLn2 = static_cast<Acc>(0.6931471805599453094);
    const Acc kNegInf = -static_cast<Acc>(INFINITY);
    bool nonfinite = false;

    Acc q[HPW][EPL];
    Acc acc[HPW][EPL];
    Acc m[HPW], e[HPW];
#pragma unroll
    for (int hs = 0; hs < HPW; ++hs) {
        m[hs] = kNegInf;
        e[hs] = 0;
#pragma unroll
        for (int i = 0; i < EPL; ++i) q[hs][i] = acc[hs][i] = 0;
    }

    int stage = 0;
    uint32_t phase = 0;
    for (;;) {
        mbar_wait(&full[stage], phase);
        const StageMeta md = meta[stage];
        if (md.item < 0) break;
        const uint8_t* sb = smem + L.stage0 + L.stage_bytes * stage;
        const T* ks = reinterpret_cast<const T*>(sb + L.k_off);
        const T* vs = reinterpret_cast<const T*>(sb + L.v_off);
        if (md.flags & 1) {
            const T* qs = reinterpret_cast<const T*>(sb + L.q_off);
#pragma unroll
            for (int hs = 0; hs < HPW; ++hs) {
                const int h = hslot + hs * gslots;
                const bool hv = active && h < p.group;
#pragma unroll
                for (int c = 0; c < CPL; ++c)
#pragma unroll
                    for (int v = 0; v < VEC; ++v)
                        q[hs][c * VEC + v] =
                            hv ? E::to_acc(qs[h * DP + (c * LPT + sub) * VEC + v]) * scale_log2
                               : Acc(0);
                m[hs] = kNegInf;
                e[hs] = 0;
#pragma unroll
                for (int i = 0; i < EPL; ++i) acc[hs][i] = 0;
            }
        }
        if (active) {
            const int n = md.ntok;
            for (int base = slice * TPW; base < n; base += wph * TPW * U) {
                Acc s[U][HPW];
                bool valid[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int t = base + u * wph * TPW + grp;
                    valid[u] = t < n;
                    const int tc = valid[u] ? t : n - 1;
                    const uint4* rowp = reinterpret_cast<const uint4*>(ks + tc * DP);
                    Acc s2[HPW][2];
#pragma unroll
                    for (int hs = 0; hs < HPW; ++hs) s2[hs][0] = s2[hs][1] = 0;
#pragma unroll
                    for (int c = 0; c < CPL; ++c) {
                        const uint4 ch = rowp[c * LPT + sub];
                        Acc x[VEC];
                        E::unpack(ch, x);
                        if constexpr (std::is_same<T, double>::value) {
#pragma unroll
                            for (int v = 0; v < VEC; ++v) nonfinite |= !isfinite(x[v]);
                        }
#pragma unroll
                        for (int hs = 0; hs < HPW; ++hs) {
                            if constexpr (std::is_same<Acc, float>::value) {
#pragma unroll
                                for (int v = 0; v < VEC; v += 2)
                                    ffma2(s2[hs][0], s2[hs][1], q[hs][c * VEC + v], q[hs][c * VEC + v + 1], x[v],
                                          x[v + 1]);
                            } else {
#pragma unroll
                                for (int v = 0; v < VEC; ++v) s2[hs][v & 1] += q[hs][c * VEC + v] * x[v];
                            }
                        }
                    }
#pragma unroll
                    for (int hs = 0; hs < HPW; ++hs) s[u][hs] = s2[hs][0] + s2[hs][1];
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int hs = 0; hs < HPW; ++hs)
#pragma unroll
                        for (int off = 1; off < LPT; off <<= 1)
                            s[u][hs] += __shfl_xor_sync(0xffffffffu, s[u][hs], off);
                Acc pw[U][HPW];
#pragma unroll
                for (int hs = 0; hs < HPW; ++hs) {
                    Acc mx = m[hs];
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (valid[u]) mx = s[u][hs] > mx ? s[u][hs] : mx;
                    const Acc corr = (mx == m[hs]) ? Acc(1) : acc_exp2(m[hs] - mx);
                    Acc es = e[hs] * corr;
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        pw[u][hs] = valid[u] ? acc_exp2(s[u][hs] - mx) : Acc(0);
                        es += pw[u][hs];
                    }
                    e[hs] = es;
                    m[hs] = mx;
                    // the running max rarely moves after the first tokens: skip
                    // the rescale when no token group of the warp needs it
                    if (__any_sync(0xffffffffu, corr != Acc(1))) {
#pragma unroll
                        for (int i = 0; i < EPL; ++i) acc[hs][i] *= corr;
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (!valid[u]) continue;
                    const int t = base + u * wph * TPW + grp;
                    const uint4* rowp = reinterpret_cast<const uint4*>(vs + t * DP);
#pragma unroll
                    for (int c = 0; c < CPL; ++c) {
                        const uint4 ch = rowp[c * LPT + sub];
                        Acc x[VEC];
                        E::unpack(ch, x);
                        if constexpr (std::is_same<T, double>::value) {
#pragma unroll
                            for (int v = 0; v < VEC; ++v) nonfinite |= !isfinite(x[v]);
                        }
#pragma unroll
                        for (int hs = 0; hs < HPW; ++hs) {
                            if constexpr (std::is_same<Acc, float>::value) {
#pragma unroll
                                for (int v = 0; v < VEC; v += 2)
                                    ffma2(acc[hs][c * VEC + v], acc[hs][c * VEC + v + 1], pw[u][hs], pw[u][hs],
                                          x[v], x[v + 1]);
                            } else {
#pragma unroll
                                for (int v = 0; v < VEC; ++v) acc[hs][c * VEC + v] += pw[u][hs] * x[v];
                            }
                        }
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);

        if (md.flags & 2) {
            // ---- finalize the item: merge token groups inside the warp ----
#pragma unroll
            for (int hs = 0; hs < HPW; ++hs) {
#pragma unroll
                for (int off = LPT; off < 32; off <<= 1) {
                    const Acc mo = __shfl_xor_sync(0xffffffffu, m[hs], off);
                    const Acc eo = __shfl_xor_sync(0xffffffffu, e[hs], off);
                    const Acc mn = mo > m[hs] ? mo : m[hs];
                    const Acc c1 = (m[hs] == mn) ? Acc(1) : acc_exp2(m[hs] - mn);
                    const Acc c2 = (mo == mn) ? Acc(1) : acc_exp2(mo - mn);
                    e[hs] = e[hs] * c1 + eo * c2;
#pragma unroll
                    for (int i = 0; i < EPL; ++i) {
                        const Acc ao = __shfl_xor_sync(0xffffffffu, acc[hs][i], off);
                        acc[hs][i] = acc[hs][i] * c1 + ao * c2;
                    }
                    m[hs] = mn;
                }
            }
            Acc* recs = static_cast<Acc*>(p.records);
            const int64_t rec_base =
                static_cast<int64_t>(md.gchunk) * p.num_q_heads + static_cast<int64_t>(md.kvh) * p.group;
            if (wph == 1) {
#pragma unroll
                for (int hs = 0; hs < HPW; ++hs) {
                    const int h = hslot + hs * gslots;
                    if (!active || h >= p.group) continue;
                    Acc* rec = recs + (rec_base + h) * REC;
                    if (grp == 0) {
#pragma unroll
                        for (int c = 0; c < CPL; ++c)
#pragma unroll
                            for (int v = 0; v < VEC; ++v)
                                rec[4 + (c * LPT + sub) * VEC + v] = acc[hs][c * VEC + v];
                    }
                    if (lane == 0) {
                        rec[0] = m[hs] * kLn2;
                        rec[1] = e[hs];
                        rec[2] = static_cast<Acc>(md.item_tokens);
                        rec[3] = 0;
                    }
                }
            } else {
                // several warps per head: reduce through shared memory
                if (grp == 0) {
#pragma unroll
                    for (int c = 0; c < CPL; ++c)
#pragma unroll
                        for (int v = 0; v < VEC; ++v)
                            red_acc[cw * DP + (c * LPT + sub) * VEC + v] = acc[0][c * VEC + v];
                }
                if (lane == 0) {
                    red_m[cw] = m[0];
                    red_e[cw] = e[0];
                }
                named_bar_sync(1, 32 * kConsumerWarps);
                if (active && slice == 0 && hslot < p.group) {
                    Acc mg = kNegInf;
                    for (int s2 = 0; s2 < wph; ++s2) {
                        const Acc mm = red_m[hslot + s2 * gslots];
                        mg = mm > mg ? mm : mg;
                    }
                    Acc wt[kConsumerWarps];
                    Acc eg = 0;
#pragma unroll
                    for (int s2 = 0; s2 < kConsumerWarps; ++s2) {
                        if (s2 < wph) {
                            const Acc mm = red_m[hslot + s2 * gslots];
                            wt[s2] = (mm == mg) ? Acc(1) : acc_exp2(mm - mg);
                            eg += red_e[hslot + s2 * gslots] * wt[s2];
                        } else {
                            wt[s2] = 0;
                        }
                    }
                    Acc* rec = recs + (rec_base + hslot) * REC;
                    for (int jd = lane; jd < DP; jd += 32) {
                        Acc a = 0;
#pragma unroll
                        for (int s2 = 0; s2 < kConsumerWarps; ++s2)
                            if (s2 < wph) a += red_acc[(hslot + s2 * gslots) * DP + jd] * wt[s2];
                        rec[4 + jd] = a;
                    }
                    if (lane == 0) {
                        rec[0] = mg * kLn2;
                        rec[1] = eg;
                        rec[2] = static_cast<Acc>(md.item_tokens);
                        rec[3] = 0;
                    }
                }
                named_bar_sync(1, 32 * kConsumerWarps);
            }
            if (p.fused_mode != 0) {
                // ---- group completion: the CTA that wrote the last chunk of
                //      (row, kv head) hands the group to its merge warp
                //      (threadfence pattern; counters reset for the next launch)
                named_bar_sync(1, 32 * kConsumerWarps);  // this item's records are issued
                if (cw == 0 && lane == 0) {
                    const int gi = md.row * p.num_kv_heads + md.kvh;
                    const int old = atomic_add_acq_rel_gpu(p.group_counter + gi, 1);
                    if (old + 1 == __ldg(p.group_expected + gi)) {
                        p.group_counter[gi] = 0;
                        mq_push(&mq, (md.row << 8) | md.kvh);
                    }
                }
            }
        }
        if (++stage == stages) {
            stage = 0;
            phase ^= 1u;
        }
    }
    if (p.fused_mode != 0) {
        named_bar_sync(1, 32 * kConsumerWarps);  // every group of this CTA is queued
        if (cw == 0 && lane == 0) mq_push(&mq, -1);
    }
    if (nonfinite && p.nonfinite_flag) atomicOr(p.nonfinite_flag, 1);
}

// ------------------------------------------------------------------ K1g
// Generic micro-attention for the shapes K1's shared-memory pipeline does not
// instantiate: query groups above 16 (8 for fp64 stores; MQA such as 32 q / 1
// kv head) and padded head widths above 256. Same work items, claim protocol
// (the counter advances by nitems + grid per launch) and records as K1: a CTA
// claims an item (range, chunk, kv head); each of its warps owns q heads
// h = warp, warp + 4, ... of the group, streams the chunk's K/V rows through
// L1 (warps of one CTA share them), reduces q.k across the warp and keeps an
// online softmax in registers (lane l owns dims l, l + 32, ...). Correct for
// every shape the reference accepts up to head_dim 512; not a roofline kernel.
constexpr int kGenericWarps = 4;

template <typename T, int DP>
__global__ void __launch_bounds__(32 * kGenericWarps) ma_generic_kernel(const MAParams p) {
    using E = Elem<T>;
    using Acc = typename E::Acc;
    constexpr int EPL = (DP + 31) / 32;
    constexpr int REC = DP + 4;
    pdl_launch_dependents();
    pdl_wait();  // behind the previous step's merge grid (PDL launch)
    __shared__ int s_item;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const T* kpool = static_cast<const T*>(p.k_pool);
    const T* vpool = static_cast<const T*>(p.v_pool);
    const T* qg = static_cast<const T*>(p.q);
    const int P = p.page_tokens;
    const Acc scale_log2 = static_cast<Acc>(p.scale_log2);
    const Acc kLn2 = static_cast<Acc>(0.6931471805599453094);
    const Acc kNegInf = -static_cast<Acc>(INFINITY);
    Acc* recs = static_cast<Acc*>(p.records);
    bool nonfinite = false;
    for (;;) {
        __syncthreads();  // everyone has read the previous s_item
        if (threadIdx.x == 0) s_item = static_cast<int>(atomicAdd(p.work_counter, 1ull) - p.work_base);
        __syncthreads();
        const int item = s_item;
        if (item >= p.nitems) break;
        int r, local;
        if (p.item_table) {
            const int2 ent = __ldg(reinterpret_cast<const int2*>(p.item_table) + item);
            r = ent.x;
            local = ent.y;
        } else {
            r = find_range(p.item_prefix, p.nranges, item);
            local = item - __ldg(p.item_prefix + r);
        }
        const RangeDev rg = p.ranges[r];
        const int nh = rg.kv_head < 0 ? p.num_kv_heads : 1;
        const int j = local / nh;
        const int kvh = rg.kv_head < 0 ? local - j * nh : rg.kv_head;
        const int tlo = rg.lo + j * p.chunk_tokens;
        const int thi = min(rg.hi, tlo + p.chunk_tokens);
        const int gchunk = __ldg(p.chunk_prefix + r) + j;
        const int32_t* bt = p.block_tables + static_cast<int64_t>(rg.seq) * p.bt_stride;
        for (int h = warp; h < p.group; h += kGenericWarps) {
            const T* qs = qg + (static_cast<int64_t>(rg.out_row) * p.num_q_heads +
                                static_cast<int64_t>(kvh) * p.group + h) * DP;
            Acc q[EPL], acc[EPL];
#pragma unroll
            for (int i = 0; i < EPL; ++i) {
                const int jd = lane + 32 * i;
                q[i] = jd < DP ? E::to_acc(qs[jd]) * scale_log2 : Acc(0);
                acc[i] = 0;
            }
            Acc m = kNegInf, e = 0;
            for (int t = tlo; t < thi; ++t) {
                const int64_t page = __ldg(bt + t / P);
                const int64_t row = ((page * p.num_kv_heads + kvh) * P + t % P) * DP;
                Acc sc = 0;
#pragma unroll
                for (int i = 0; i < EPL; ++i) {
                    const int jd = lane + 32 * i;
                    if (jd < DP) {
                        const Acc x = E::to_acc(kpool[row + jd]);
                        if constexpr (std::is_same<T, double>::value) nonfinite |= !isfinite(x);
                        sc += q[i] * x;
                    }
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, off);
                const Acc mx = sc > m ? sc : m;
                const Acc corr = (mx == m) ? Acc(1) : acc_exp2(m - mx);
                const Acc pw = acc_exp2(sc - mx);
                e = e * corr + pw;
                m = mx;
#pragma unroll
                for (int i = 0; i < EPL; ++i) {
                    const int jd = lane + 32 * i;
                    if (jd < DP) {
                        const Acc x = E::to_acc(vpool[row + jd]);
                        if constexpr (std::is_same<T, double>::value) nonfinite |= !isfinite(x);
                        acc[i] = acc[i] * corr + pw * x;
                    }
                }
            }
            Acc* rec = recs + ((static_cast<int64_t>(gchunk) * p.num_q_heads + static_cast<int64_t>(kvh) * p.group + h) *
                               REC);
#pragma unroll
            for (int i = 0; i < EPL; ++i) {
                const int jd = lane + 32 * i;
                if (jd < DP) rec[4 + jd] = acc[i];
            }
            if (lane == 0) {
                rec[0] = m * kLn2;
                rec[1] = e;
                rec[2] = static_cast<Acc>(thi - tlo);
                rec[3] = 0;
            }
        }
    }
    if (nonfinite && p.nonfinite_flag) atomicOr(p.nonfinite_flag, 1);
}

// ------------------------------------------------------------------ K3
// One CTA (8 warps) per (row, q head) group. Pass 1: block max over live
// records. Pass 2: warp w folds records w, w+8, ... with vector loads (each
// lane owns kVW contiguous elements of ma), then the 8 warp partials are
// summed through shared memory in a fixed order (deterministic).

template <typename T, int DP>
__global__ void __launch_bounds__(32 * kMergeWarps) merge_kernel(const MergeParams p) {
    using E = Elem<T>;
    using Acc = typename E::Acc;
    constexpr int REC = DP + 4;
    constexpr int kVW = (sizeof(Acc) == 4) ? (DP % 128 == 0 ? 4 : (DP % 64 == 0 ? 2 : 1))
                                           : (DP % 64 == 0 ? 2 : 1);
    constexpr int kPer = 32 * kVW;                       // elements covered per lane sweep
    constexpr int kSweeps = (DP + kPer - 1) / kPer;
    __shared__ Acc s_max[kMergeWarps];
    __shared__ Acc s_e[kMergeWarps];
    __shared__ Acc s_tok[kMergeWarps];
    __shared__ __align__(16) Acc s_acc[kMergeWarps][DP];

    pdl_wait();  // launched early behind the MA grid (PDL)
    pdl_launch_dependents();  // the next step's MA grid may set up behind this one
    const int64_t g = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = static_cast<int>(g / p.heads);
    const int h = static_cast<int>(g - static_cast<int64_t>(row) * p.heads);
    int n;
    int64_t base;
    int cbase = 0;
    if (p.row_begin) {
        cbase = p.row_begin[row];
        n = p.row_begin[row + 1] - cbase;
        base = static_cast<int64_t>(cbase) * p.row_mul + h;
    } else {
        n = p.n_uniform;
        base = static_cast<int64_t>(row) * p.row_mul + h;
    }
    const int my_kvh = p.chunk_kvh ? h / p.group : 0;
    const Acc* R = static_cast<const Acc*>(p.recs);
    const Acc kNegInf = -static_cast<Acc>(INFINITY);
    auto live = [&](int c, const Acc* r) {
        if (p.chunk_kvh) {
            const int tag = p.chunk_kvh[cbase + c];
            if (tag >= 0 && tag != my_kvh) return false;
        }
        return r[2] != Acc(0);  // identity (seq_p == 0) records are skipped
    };

    Acc mg = kNegInf;
    for (int c = threadIdx.x; c < n; c += blockDim.x) {
        const Acc* r = R + (base + static_cast<int64_t>(c) * p.c_stride) * REC;
        if (live(c, r)) mg = r[0] > mg ? r[0] : mg;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const Acc o = __shfl_xor_sync(0xffffffffu, mg, off);
        mg = o > mg ? o : mg;
    }
    if (lane == 0) s_max[warp] = mg;
    __syncthreads();
    mg = s_max[0];
#pragma unroll
    for (int w = 1; w < kMergeWarps; ++w) mg = s_max[w] > mg ? s_max[w] : mg;

    Acc eg = 0, ntok = 0;
    Acc acc[kSweeps][kVW];
#pragma unroll
    for (int s = 0; s < kSweeps; ++s)
#pragma unroll
        for (int v = 0; v < kVW; ++v) acc[s][v] = 0;
    fold_chunks<Acc, DP, kVW, kSweeps>(R, base, p.c_stride, n, warp, kMergeWarps, mg, live, acc, eg, ntok, lane);
#pragma unroll
    for (int s = 0; s < kSweeps; ++s) {
        const int j = s * kPer + lane * kVW;
        if (j < DP)
#pragma unroll
            for (int v = 0; v < kVW; ++v) s_acc[warp][j + v] = acc[s][v];
    }
    if (lane == 0) {
        s_e[warp] = eg;
        s_tok[warp] = ntok;
    }
    __syncthreads();
    Acc e_tot = 0, tok_tot = 0;
#pragma unroll
    for (int w = 0; w < kMergeWarps; ++w) {
        e_tot += s_e[w];
        tok_tot += s_tok[w];
    }
    for (int j = threadIdx.x; j < DP; j += blockDim.x) {
        Acc a = 0;
#pragma unroll
        for (int w = 0; w < kMergeWarps; ++w) a += s_acc[w][j];
        if (p.out_recs) static_cast<Acc*>(p.out_recs)[g * REC + 4 + j] = a;
        if (p.out_norm)
            static_cast<T*>(p.out_norm)[g * DP + j] =
                E::from_acc(tok_tot != Acc(0) ? a / e_tot : Acc(0));
    }
    if (p.out_recs && threadIdx.x == 0) {
        Acc* o = static_cast<Acc*>(p.out_recs) + g * REC;
        o[0] = tok_tot != Acc(0) ? mg : kNegInf;
        o[1] = e_tot;
        o[2] = tok_tot;
        o[3] = 0;
    }
}

// ------------------------------------------------------------------ K5
// Fused cross-GPU merge, one launch per step replacing local
// K3 + ncclAllGather + rank K3. Phase A: every (row, q head) group's chunk
// records on this rank are merged (as K3) and the merged record is stored
// straight into every rank's exchange buffer (NVLink stores through CUDA IPC
// peer pointers). Phase D: every group's nranks records are read back as they
// arrive -- exchange words are self-validating (XWord: an empty word is the
// all-ones NaN), so there is no fence, flag or barrier between the phases --
// merged into the output, and the slots are emptied for the step after next.
//
// Phase A walks the groups in sweeps of gridDim.x * gpc; within a sweep CTA b
// takes groups b, b + gridDim.x, ... so the consecutive heavy groups of one
// long request (more than kHeavy chunk records each) land on different CTAs.
// Light groups are merged by one warp each, heavy groups by the whole CTA.
// Identity groups (no tokens on this rank) push only their header; a receiver
// reads the payload of live records only, so every word written is read and
// emptied exactly once. The engine caps the grid at the kernel's occupancy x
// SMs (exchange_occupancy), so the whole grid is co-resident and a warp
// spinning in phase D never starves a CTA still in phase A.
template <typename T, int DP>
__global__ void __launch_bounds__(32 * kMergeWarps) merge_exchange_kernel(const XParams x) {
    using E = Elem<T>;
    using Acc = typename E::Acc;
    using U = typename XWord<Acc>::U;
    constexpr int REC = DP + 4;
    constexpr int kVW = (sizeof(Acc) == 4) ? (DP % 128 == 0 ? 4 : (DP % 64 == 0 ? 2 : 1))
                                           : (DP % 64 == 0 ? 2 : 1);
    constexpr int kPer = 32 * kVW;
    constexpr int kSweeps = (DP + kPer - 1) / kPer;
    __shared__ Acc s_max[kMergeWarps];
    __shared__ Acc s_e[kMergeWarps];
    __shared__ Acc s_tok[kMergeWarps];
    __shared__ __align__(16) Acc s_acc[kMergeWarps][DP];
    const MergeParams& p = x.local;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gpc = x.groups_per_cta;  // 1 or kMergeWarps
    const Acc kNegInf = -static_cast<Acc>(INFINITY);
    const int64_t groups = static_cast<int64_t>(p.rows) * p.heads;
    pdl_wait();  // launched early behind the MA grid (PDL)
    pdl_launch_dependents();  // the next step's MA grid may set up behind this one
    const Acc* R = static_cast<const Acc*>(p.recs);
    // DATTN_K5_TRACE: per-CTA sums over calls of (phase A done - start) and
    // (end - start), %globaltimer ns, and the call count
    uint64_t t_start = 0;
    auto stamp = [&](int i) {
        if (x.trace && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (i == 0) {
                t_start = t;
            } else {
                atomicAdd(x.trace + blockIdx.x * 3 + (i == 1 ? 0 : 1), t - t_start);
                if (i == 4) atomicAdd(x.trace + blockIdx.x * 3 + 2, 1ull);
            }
        }
    };
    stamp(0);

    // ---- A. local merge + push to every rank. A group with more than
    //      heavy_min chunk records is merged by the whole CTA: above 64
    //      records always, above 8 when the CTA owns one group per sweep
    //      (few groups, e.g. one long request: 7 warps would idle otherwise)
    constexpr int kHeavy = 64;
    const int heavy_min = gpc == 1 ? 8 : kHeavy;
    auto group_shape = [&](int64_t g, int& n, int& cbase, int64_t& base, int& my_kvh) {
        const int row = static_cast<int>(g / p.heads);
        const int h = static_cast<int>(g - static_cast<int64_t>(row) * p.heads);
        cbase = p.row_begin[row];
        n = p.row_begin[row + 1] - cbase;
        base = static_cast<int64_t>(cbase) * p.row_mul + h;
        my_kvh = p.chunk_kvh ? h / p.group : 0;
    };
    auto push = [&](int64_t g, const Acc (&acc)[kSweeps][kVW], Acc mg, Acc eg, Acc ntok) {
        const int64_t slot = (static_cast<int64_t>(x.rank) * x.slot_stride + g) * REC;
        const U hdr[4] = {x_enc(ntok != Acc(0) ? mg : kNegInf), x_enc(eg), x_enc(ntok), x_enc(Acc(0))};
        for (int r = 0; r < x.nranks; ++r) {
            U* dst = static_cast<U*>(x.peer_x[r]) + slot;
            if (ntok != Acc(0)) {
#pragma unroll
                for (int sw = 0; sw < kSweeps; ++sw) {
                    const int j = sw * kPer + lane * kVW;
                    if (j < DP) {
                        U w[kVW];
#pragma unroll
                        for (int v = 0; v < kVW; ++v) w[v] = x_enc(acc[sw][v]);
                        x_store<U, kVW>(dst + 4 + j, w);
                    }
                }
            }
            if (lane == 0) x_store<U, 4>(dst, hdr);
        }
    };
    const int64_t sweep = static_cast<int64_t>(gridDim.x) * gpc;
    for (int64_t gb = 0; gb < groups; gb += sweep) {
        // light groups: warp w takes group gb + w * gridDim.x + blockIdx.x
        if (warp < gpc) {
            const int64_t g = gb + static_cast<int64_t>(warp) * gridDim.x + blockIdx.x;
            int n = 0, cbase = 0, my_kvh = 0;
            int64_t base = 0;
            if (g < groups) group_shape(g, n, cbase, base, my_kvh);
            if (g < groups && n <= 32 && n <= heavy_min) {
                // one round trip: lane c holds chunk c's header while every
                // lane already fetches its payload words of the first chunks
                // (independent of the weights); same arithmetic and order as
                // fold_chunks, so the record is bit-identical
                constexpr int kPre = (kSweeps * kVW * sizeof(Acc) <= 32) ? 4 : 1;
                Acc hm = kNegInf, he = 0, ht = 0;
                bool lv = false;
                if (lane < n) {
                    const Acc* r = R + (base + static_cast<int64_t>(lane) * p.c_stride) * REC;
                    hm = __ldcg(r);
                    he = __ldcg(r + 1);
                    ht = __ldcg(r + 2);
                    lv = ht != Acc(0);
                    if (p.chunk_kvh) {
                        const int tag = p.chunk_kvh[cbase + lane];
                        if (tag >= 0 && tag != my_kvh) lv = false;
                    }
                }
                Acc pre[kPre][kSweeps][kVW];
#pragma unroll
                for (int k = 0; k < kPre; ++k) {
                    const Acc* r = R + (base + static_cast<int64_t>(k < n ? k : 0) * p.c_stride) * REC;
#pragma unroll
                    for (int sw = 0; sw < kSweeps; ++sw) {
                        const int j = sw * kPer + lane * kVW;
#pragma unroll
                        for (int v = 0; v < kVW; ++v) pre[k][sw][v] = 0;
                        if (k < n && j < DP) {
                            if constexpr (kVW == 4) {
                                const float4 x4 = __ldcg(reinterpret_cast<const float4*>(r + 4 + j));
                                pre[k][sw][0] = x4.x; pre[k][sw][1] = x4.y; pre[k][sw][2] = x4.z; pre[k][sw][3] = x4.w;
                            } else {
#pragma unroll
                                for (int v = 0; v < kVW; ++v) pre[k][sw][v] = __ldcg(r + 4 + j + v);
                            }
                        }
                    }
                }
                Acc mg = lv ? hm : kNegInf;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    const Acc o = __shfl_xor_sync(0xffffffffu, mg, off);
                    mg = o > mg ? o : mg;
                }
                const Acc w = lv ? ((hm == mg) ? Acc(1) : exp(hm - mg)) : Acc(0);
                Acc eg = lv ? he * w : Acc(0), ntok = lv ? ht : Acc(0);
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    eg += __shfl_xor_sync(0xffffffffu, eg, off);
                    ntok += __shfl_xor_sync(0xffffffffu, ntok, off);
                }
                Acc acc[kSweeps][kVW];
#pragma unroll
                for (int sw = 0; sw < kSweeps; ++sw)
#pragma unroll
                    for (int v = 0; v < kVW; ++v) acc[sw][v] = 0;
#pragma unroll
                for (int k = 0; k < kPre; ++k) {
                    const Acc wk = __shfl_sync(0xffffffffu, w, k);
                    if (k < n)
#pragma unroll
                        for (int sw = 0; sw < kSweeps; ++sw)
#pragma unroll
                            for (int v = 0; v < kVW; ++v) acc[sw][v] += pre[k][sw][v] * wk;
                }
#pragma unroll 8
                for (int k = kPre; k < n; ++k) {
                    const Acc wk = __shfl_sync(0xffffffffu, w, k);
                    const Acc* r = R + (base + static_cast<int64_t>(k) * p.c_stride) * REC;
#pragma unroll
                    for (int sw = 0; sw < kSweeps; ++sw) {
                        const int j = sw * kPer + lane * kVW;
                        if (j < DP)
#pragma unroll
                            for (int v = 0; v < kVW; ++v) acc[sw][v] += __ldcg(r + 4 + j + v) * wk;
                    }
                }
                push(g, acc, mg, eg, ntok);
            } else if (g < groups && n <= heavy_min) {
                auto live = [&](int c, const Acc* r) {
                    if (p.chunk_kvh) {
                        const int tag = p.chunk_kvh[cbase + c];
                        if (tag >= 0 && tag != my_kvh) return false;
                    }
                    return r[2] != Acc(0);
                };
                Acc mg = kNegInf;
                for (int c = lane; c < n; c += 32) {
                    const Acc* r = R + (base + static_cast<int64_t>(c) * p.c_stride) * REC;
                    if (live(c, r)) mg = r[0] > mg ? r[0] : mg;
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    const Acc o = __shfl_xor_sync(0xffffffffu, mg, off);
                    mg = o > mg ? o : mg;
                }
                Acc eg, ntok;
                Acc acc[kSweeps][kVW];
#pragma unroll
                for (int sw = 0; sw < kSweeps; ++sw)
#pragma unroll
                    for (int v = 0; v < kVW; ++v) acc[sw][v] = 0;
                fold_chunks<Acc, DP, kVW, kSweeps>(R, base, p.c_stride, n, 0, 1, mg, live, acc, eg, ntok, lane);
                push(g, acc, mg, eg, ntok);
            }
        }
        // heavy groups: the whole CTA, 8 warps striding over the chunk records
        for (int rep = 0; rep < gpc; ++rep) {
            const int64_t g = gb + static_cast<int64_t>(rep) * gridDim.x + blockIdx.x;
            if (g >= groups) break;
            int n, cbase, my_kvh;
            int64_t base;
            group_shape(g, n, cbase, base, my_kvh);
            if (n <= heavy_min) continue;  // uniform across the CTA
            auto live = [&](int c, const Acc* r) {
                if (p.chunk_kvh) {
                    const int tag = p.chunk_kvh[cbase + c];
                    if (tag >= 0 && tag != my_kvh) return false;
                }
                return r[2] != Acc(0);
            };
            Acc mg = kNegInf;
            for (int c = threadIdx.x; c < n; c += blockDim.x) {
                const Acc* r = R + (base + static_cast<int64_t>(c) * p.c_stride) * REC;
                if (live(c, r)) mg = r[0] > mg ? r[0] : mg;
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const Acc o = __shfl_xor_sync(0xffffffffu, mg, off);
                mg = o > mg ? o : mg;
            }
            if (lane == 0) s_max[warp] = mg;
            __syncthreads();
            mg = s_max[0];
#pragma unroll
            for (int w2 = 1; w2 < kMergeWarps; ++w2) mg = s_max[w2] > mg ? s_max[w2] : mg;
            Acc eg, ntok;
            Acc acc[kSweeps][kVW];
#pragma unroll
            for (int sw = 0; sw < kSweeps; ++sw)
#pragma unroll
                for (int v = 0; v < kVW; ++v) acc[sw][v] = 0;
            fold_chunks<Acc, DP, kVW, kSweeps>(R, base, p.c_stride, n, warp, kMergeWarps, mg, live, acc, eg, ntok,
                                               lane);
#pragma unroll
            for (int sw = 0; sw < kSweeps; ++sw) {
                const int j = sw * kPer + lane * kVW;
                if (j < DP)
#pragma unroll
                    for (int v = 0; v < kVW; ++v) s_acc[warp][j + v] = acc[sw][v];
            }
            if (lane == 0) {
                s_e[warp] = eg;
                s_tok[warp] = ntok;
            }
            __syncthreads();
            if (warp == 0) {
                eg = 0;
                ntok = 0;
#pragma unroll
                for (int w2 = 0; w2 < kMergeWarps; ++w2) {
                    eg += s_e[w2];
                    ntok += s_tok[w2];
                }
#pragma unroll
                for (int sw = 0; sw < kSweeps; ++sw) {
                    const int j = sw * kPer + lane * kVW;
                    if (j < DP)
#pragma unroll
                        for (int v = 0; v < kVW; ++v) {
                            Acc a = 0;
#pragma unroll
                            for (int w2 = 0; w2 < kMergeWarps; ++w2) a += s_acc[w2][j + v];
                            acc[sw][v] = a;
                        }
                }
                push(g, acc, mg, eg, ntok);
            }
            __syncthreads();
        }
    }
    stamp(1);

    // ---- D. rank merge, one warp per group (xchg_rank_merge)
    U* X = static_cast<U*>(x.peer_x[x.rank]);
    for (int64_t g = static_cast<int64_t>(blockIdx.x) * kMergeWarps + warp; g < groups;
         g += static_cast<int64_t>(gridDim.x) * kMergeWarps)
        xchg_rank_merge<T, DP>(X, g, x.nranks, x.slot_stride, x.out_norm, lane, x.ctl);
    __syncthreads();
    stamp(4);
}

// ------------------------------------------------------------------ K6
// Rank merge after the in-kernel merge + push of K1/K2 (fused mode 2): this
// rank first pushes identity headers for its (row, kv head) groups that hold
// no tokens (no MA CTA completes them), then one warp per (row, q head) merges
// the nranks records as they arrive (xchg_rank_merge: self-validating words,
// no counters or fences).
template <typename T, int DP>
__global__ void __launch_bounds__(32 * kMergeWarps) rank_merge_kernel(const RankMergeParams x) {
    using E = Elem<T>;
    using Acc = typename E::Acc;
    using U = typename XWord<Acc>::U;
    constexpr int REC = DP + 4;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const Acc kNegInf = -static_cast<Acc>(INFINITY);
    const int64_t ngroups_kv = static_cast<int64_t>(x.rows) * x.num_kv_heads;
    const U hdr[4] = {x_enc(kNegInf), x_enc(Acc(0)), x_enc(Acc(0)), x_enc(Acc(0))};
    for (int64_t gk = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; gk < ngroups_kv;
         gk += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (x.group_expected[gk] != 0) continue;
        const int row = static_cast<int>(gk / x.num_kv_heads), kvh = static_cast<int>(gk % x.num_kv_heads);
        for (int hh = 0; hh < x.group; ++hh) {
            const int64_t g = static_cast<int64_t>(row) * x.heads + kvh * x.group + hh;
            for (int r = 0; r < x.nranks; ++r)
                x_store<U, 4>(static_cast<U*>(x.peer_x[r]) + (static_cast<int64_t>(x.rank) * x.slot_stride + g) * REC,
                              hdr);
        }
    }
    const int64_t groups = static_cast<int64_t>(x.rows) * x.heads;
    U* X = static_cast<U*>(x.peer_x[x.rank]);
    for (int64_t g = static_cast<int64_t>(blockIdx.x) * kMergeWarps + warp; g < groups;
         g += static_cast<int64_t>(gridDim.x) * kMergeWarps)
        xchg_rank_merge<T, DP>(X, g, x.nranks, x.slot_stride, x.out_norm, lane, x.ctl);
}

// ------------------------------------------------------------------ K4
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t stream_key(uint64_t seed, int tensor) {
    return splitmix64(seed ^ (static_cast<uint64_t>(tensor) * 0xD1B54A32D192ED03ull));
}
__device__ __forceinline__ uint64_t elem_index(uint32_t seq, uint32_t head, uint32_t token,
                                               uint32_t dim) {
    return (static_cast<uint64_t>(seq) << 40) | (static_cast<uint64_t>(head & 0xFFu) << 32) |
           (static_cast<uint64_t>(token & 0xFFFFFFu) << 8) | static_cast<uint64_t>(dim & 0xFFu);
}
__device__ __forceinline__ float synth_f32(uint64_t key, uint64_t idx, float amp) {
    const uint32_t u24 = static_cast<uint32_t>(splitmix64(key ^ idx) >> 40);
    const float a = static_cast<float>(static_cast<int32_t>(u24) - (1 << 23));
    return __fmul_rn(a, __fmul_rn(amp, 0x1.0p-23f));
}
template <typename T>
__device__ __forceinline__ T store_as(float x) {
    if constexpr (std::is_same<T, bf16_t>::value) return Elem<bf16_t>::from_acc(x);
    else return static_cast<T>(x);
}

template <typename T, int DP>
__global__ void fill_kv_kernel(const FillParams p) {
    const uint64_t kk = stream_key(p.seed, 1), kv = stream_key(p.seed, 2);
    const int64_t total = p.tokens * p.num_kv_heads * DP;
    T* kp = static_cast<T*>(p.k_pool);
    T* vp = static_cast<T*>(p.v_pool);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(i % DP);
        const int64_t th = i / DP;
        const int h = static_cast<int>(th % p.num_kv_heads);
        const int64_t t = th / p.num_kv_heads;
        const int64_t page = p.block_row[t / p.page_tokens];
        const int64_t dst = ((page * p.num_kv_heads + h) * p.page_tokens + t % p.page_tokens) * DP + j;
        if (j < p.head_dim) {
            const uint64_t ix = elem_index(p.logical_seq, h, static_cast<uint32_t>(p.logical_tok0 + t), j);
            kp[dst] = store_as<T>(synth_f32(kk, ix, p.amp_k));
            vp[dst] = store_as<T>(synth_f32(kv, ix, p.amp_v));
        } else {
            kp[dst] = store_as<T>(0.f);
            vp[dst] = store_as<T>(0.f);
        }
    }
}

template <typename T, int DP>
__global__ void append_kernel(const AppendParams p) {
    // 16-B chunks: (sequence, kv head, chunk)
    constexpr int kC = DP * static_cast<int>(sizeof(T)) / 16;
    const int64_t total = static_cast<int64_t>(p.n) * p.num_kv_heads * kC;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i % kC);
        const int64_t sh = i / kC;
        const int h = static_cast<int>(sh % p.num_kv_heads);
        const int s = static_cast<int>(sh / p.num_kv_heads);
        const int t = p.positions[s];
        const int64_t page = p.block_tables[static_cast<int64_t>(p.seqs[s]) * p.bt_stride + t / p.page_tokens];
        const int64_t dst = ((page * p.num_kv_heads + h) * p.page_tokens + t % p.page_tokens) * DP;
        reinterpret_cast<uint4*>(static_cast<T*>(p.k_pool) + dst)[c] =
            reinterpret_cast<const uint4*>(static_cast<const T*>(p.k_new) + sh * DP)[c];
        reinterpret_cast<uint4*>(static_cast<T*>(p.v_pool) + dst)[c] =
            reinterpret_cast<const uint4*>(static_cast<const T*>(p.v_new) + sh * DP)[c];
    }
}

template <typename T, int DP>
__global__ void fill_q_kernel(const QFillParams p) {
    const uint64_t kq = stream_key(p.seed, 3);
    const int64_t total = static_cast<int64_t>(p.rows) * p.heads * DP;
    T* q = static_cast<T*>(p.q);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(i % DP);
        const int64_t rh = i / DP;
        const int h = static_cast<int>(rh % p.heads);
        const uint32_t row = static_cast<uint32_t>(rh / p.heads) + p.row0;
        q[i] = j < p.head_dim ? store_as<T>(synth_f32(kq, elem_index(row, h, 0, j), p.amp))
                              : store_as<T>(0.f);
    }
}

template <typename T, int DP>
__global__ void rows_synth_kernel(const RowsSynthParams p) {
    const uint64_t kk = stream_key(p.seed, 1), kv = stream_key(p.seed, 2);
    const int64_t total = static_cast<int64_t>(p.n) * p.num_kv_heads * DP;
    T* ko = static_cast<T*>(p.k_out);
    T* vo = static_cast<T*>(p.v_out);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(i % DP);
        const int64_t sh = i / DP;
        const int h = static_cast<int>(sh % p.num_kv_heads);
        const int s = static_cast<int>(sh / p.num_kv_heads);
        if (j < p.head_dim) {
            const uint64_t ix = elem_index(p.logical_seq[s], h, static_cast<uint32_t>(p.logical_tok[s]), j);
            ko[i] = store_as<T>(synth_f32(kk, ix, p.amp_k));
            vo[i] = store_as<T>(synth_f32(kv, ix, p.amp_v));
        } else {
            ko[i] = store_as<T>(0.f);
            vo[i] = store_as<T>(0.f);
        }
    }
}

template <typename T, int DP>
__global__ void scatter_kernel(const ScatterParams p) {
    // rows [n][DP] of one kv head, or [n][Hkv][DP] of all heads (kv_head < 0)
    const int nh = p.kv_head < 0 ? p.num_kv_heads : 1;
    const int64_t total = p.n * nh * DP;
    const T* ks = static_cast<const T*>(p.k_rows);
    const T* vs = static_cast<const T*>(p.v_rows);
    T* kp = static_cast<T*>(p.k_pool);
    T* vp = static_cast<T*>(p.v_pool);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(i % DP);
        const int64_t th = i / DP;
        const int hh = p.kv_head < 0 ? static_cast<int>(th % nh) : p.kv_head;
        const int64_t t = p.tok0 + th / nh;
        const int64_t page = p.block_row[t / p.page_tokens];
        const int64_t dst =
            ((page * p.num_kv_heads + hh) * p.page_tokens + t % p.page_tokens) * DP + j;
        kp[dst] = ks[i];
        vp[dst] = vs[i];
    }
}

template <typename T, int DP>
__global__ void gather_kernel(const ScatterParams p) {
    const int nh = p.kv_head < 0 ? p.num_kv_heads : 1;
    const int64_t total = p.n * nh * DP;
    T* ks = static_cast<T*>(const_cast<void*>(p.k_rows));
    T* vs = static_cast<T*>(const_cast<void*>(p.v_rows));
    const T* kp = static_cast<const T*>(p.k_pool);
    const T* vp = static_cast<const T*>(p.v_pool);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(i % DP);
        const int64_t th = i / DP;
        const int hh = p.kv_head < 0 ? static_cast<int>(th % nh) : p.kv_head;
        const int64_t t = p.tok0 + th / nh;
        const int64_t page = p.block_row[t / p.page_tokens];
        const int64_t src =
            ((page * p.num_kv_heads + hh) * p.page_tokens + t % p.page_tokens) * DP + j;
        ks[i] = kp[src];
        vs[i] = vp[src];
    }
}

template <typename Acc, int DP>
__global__ void identity_records_kernel(Acc* recs, int64_t n) {
    constexpr int REC = DP + 4;
    const int64_t total = n * REC;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        recs[i] = (i % REC == 0) ? -static_cast<Acc>(INFINITY) : Acc(0);
}

// ------------------------------------------------------------ dispatch
#define DATTN_DP_SWITCH(dp, ...)                      \
    switch (dp) {                                     \
        case 16: { constexpr int DPC = 16; __VA_ARGS__; } break;   \
        case 32: { constexpr int DPC = 32; __VA_ARGS__; } break;   \
        case 64: { constexpr int DPC = 64; __VA_ARGS__; } break;   \
        case 128: { constexpr int DPC = 128; __VA_ARGS__; } break; \
        case 256: { constexpr int DPC = 256; __VA_ARGS__; } break; \
        case 512: { constexpr int DPC = 512; __VA_ARGS__; } break; \
        default: return cudaErrorInvalidValue;        \
    }
#define DATTN_DT_SWITCH(dt, ...)                                 \
    switch (dt) {                                                \
        case kBF16: { using TC = bf16_t; __VA_ARGS__; } break;   \
        case kF32: { using TC = float; __VA_ARGS__; } break;     \
        case kF64: { using TC = double; __VA_ARGS__; } break;    \
        default: return cudaErrorInvalidValue;                   \
    }

template <typename T, int DP>
static const void* ma_fn(int group) {
    if constexpr (DP <= 256) {  // K1's instantiations; wider rows take K1g
        if (group <= kConsumerWarps) return reinterpret_cast<const void*>(&ma_decode_kernel<T, DP, 1>);
        if constexpr (sizeof(T) < 8) {
            if (group <= 2 * kConsumerWarps)
                return reinterpret_cast<const void*>(&ma_decode_kernel<T, DP, 2>);
        }
    }
    return nullptr;
}

static const void* ma_kernel_ptr(int dtype, int dp, int group);
bool ma_supported(int dtype, int dp, int group) { return ma_kernel_ptr(dtype, dp, group) != nullptr; }

cudaError_t ma_generic_occupancy(int dtype, int dp, int* blocks_per_sm) {
    cudaError_t e = cudaSuccess;
    *blocks_per_sm = 0;
    DATTN_DT_SWITCH(dtype, DATTN_DP_SWITCH(dp, (e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                                                     blocks_per_sm, ma_generic_kernel<TC, DPC>,
                                                     32 * kGenericWarps, 0))));
    return e;
}

cudaError_t launch_ma_generic(int dtype, int dp, const MAParams& p, int grid, cudaStream_t st) {
    void* args[] = {const_cast<MAParams*>(&p)};
    cudaError_t le = cudaSuccess;
    DATTN_DT_SWITCH(dtype, DATTN_DP_SWITCH(dp, (le = launch_pdl_raw(reinterpret_cast<const void*>(
                                                   ma_generic_kernel<TC, DPC>), grid, 32 * kGenericWarps, 0, st,
                                               args))));
    if (le != cudaSuccess) return le;
    return cudaGetLastError();
}

static const void* ma_kernel_ptr(int dtype, int dp, int group) {
    const void* f = nullptr;
    auto pick = [&]() -> cudaError_t {
        DATTN_DT_SWITCH(dtype, DATTN_DP_SWITCH(dp, f = ma_fn<TC, DPC>(group)));
        return cudaSuccess;
    };
    pick();
    return f;
}

int ma_stage_tokens(int dtype, int dp) {
    int ts = 0;
    auto pick = [&]() -> cudaError_t {
        DATTN_DT_SWITCH(dtype, DATTN_DP_SWITCH(dp, ts = (Shape<TC, DPC>::kStageTokens)));
        return cudaSuccess;
    };
    pick();
    return ts;
}

size_t ma_smem_bytes(int dtype, int dp, int group, int stages) {
    size_t b = 0;
    auto pick = [&]() -> cudaError_t {
        DATTN_DT_SWITCH(dtype, DATTN_DP_SWITCH(dp, b = Layout<TC, DPC>(stages, group).total));
        return cudaSuccess;
    };
    pick();
    return b;
}

cudaError_t ma_configure(int dtype, int dp, int group, size_t smem) {
    const void* f = ma_kernel_ptr(dtype, dp, group);
    if (!f) return cudaErrorInvalidValue;
    // One kernel serves stores of different geometries: opt in to the device
    // maximum once instead of the last caller's size.
    int dev = 0, optin = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return e;
    cudaFuncAttributes fa{};
    e = cudaFuncGetAttributes(&fa, f);
    if (e != cudaSuccess) return e;
    const int dyn_max = optin - static_cast<int>(fa.sharedSizeBytes);  // static smem counts too
    if (smem > static_cast<size_t>(dyn_max)) return cudaErrorInvalidValue;
    return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max);
}

cudaError_t ma_occupancy(int dtype, int dp, int group, size_t smem, int* blocks) {
    const void* f = ma_kernel_ptr(dtype, dp, group);
    if (!f) return cudaErrorInvalidValue;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, f, kMAThreads, smem);
}

cudaError_t launch_ma(int dtype, int dp, const MAParams& p, int grid, size_t smem,
                      cudaStream_t st) {
    const void* f = ma_kernel_ptr(dtype, dp, p.group);
    if (!f) return cudaErrorInvalidValue;
    void* args[] = {const_cast<MAParams*>(&p)};
    return launch_pdl_raw(f, grid, kMAThreads, smem, st, args);
}

// launch with programmatic stream serialization: the kernel is scheduled
// while the previous grid on the stream drains and waits in pdl_wait()
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*k)(KArgs...), int grid, int block, cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    static const bool off = std::getenv("DATTN_NO_PDL") != nullptr;  // debug switch
    cfg.attrs = at;
    cfg.numAttrs = off ? 0 : 1;
    return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

cudaError_t launch_merge(int dtype, int dp, const MergeParams& p, cudaStream_t st) {
    const int64_t groups = static_cast<int64_t>(p.rows) * p.heads;
    if (groups == 0) return cudaSuccess;
    const int grid = static_cast<int>(groups);
    cudaError_t e = cudaSuccess;
    DATTN_DT_SWITCH(dtype, DATTN_DP_SWITCH(dp, (e = launch_pdl(merge_kernel<TC, DPC>, grid, 32 * kMergeWarps, st, p))));
    return e;
}

static int grid_for(int64_t total) {
    int64_t g = (total + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    return static_cast<int>(g < 1 ? 1 : g);
}

cudaError_t launch_merge_exchange(int dtype, int dp, const XParams& p, int grid, cudaStream_t st) {
    cudaError_t e = cudaSuccess;
    DATTN_DT_SWITCH(dtype, DATTN_DP_SWITCH(dp, (e = launch_pdl(merge_exchange_kernel<TC, DPC>, grid, 32 * kMergeWarps, st, p))));
    return e;
}

cudaError_t exchange_occupancy(int dtype, int dp, int kind, int* blocks_per_sm) {
    cudaError_t e = cudaSuccess;
    *blocks_per_sm = 0;
    if (kind == 0) {
        DATTN_DT_SWITCH(dtype, DATTN_DP_SWITCH(dp, (e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                                                         blocks_per_sm, merge_exchange_kernel<TC, DPC>,
                                                         32 * kMergeWarps, 0))));
    } else {
        DATTN_DT_SWITCH(dtype, DATTN_DP_SWITCH(dp, (e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                                                         blocks_per_sm, rank_merge_kernel<TC, DPC>,
                                                         32 * kMergeWarps, 0))));
    }
    return e;
}

cudaError_t launch_rank_merge(int dtype, int dp, const RankMergeParams& p, int grid, cudaStream_t st) {
    DATTN_DT_SWITCH(dtype, DATTN_DP_SWITCH(dp, (rank_merge_kernel<TC, DPC><<<grid, 32 * kMergeWarps, 0, st>>>(p))));
    return cudaGetLastError();
}

cudaError_t launch_fill_kv(int dtype, int dp, const FillParams& p, cudaStream_t st) {
    const int grid = grid_for(p.tokens * p.num_kv_heads * dp);
    DATTN_DT_SWITCH(dtype, DATTN_DP_SWITCH(dp, (fill_kv_kernel<TC, DPC><<<grid, 256, 0, st>>>(p))));
    return cudaGetLastError();
}

cudaError_t launch_append(int dtype, int dp, const AppendParams& p, cudaStream_t st) {
    const int grid = grid_for(static_cast<int64_t>(p.n) * p.num_kv_heads * dp);
    DATTN_DT_SWITCH(dtype, DATTN_DP_SWITCH(dp, (append_kernel<TC, DPC><<<grid, 256, 0, st>>>(p))));
    return cudaGetLastError();
}

cudaError_t launch_fill_q(int dtype, int dp, const QFillParams& p, cudaStream_t st) {
    const int grid = grid_for(static_cast<int64_t>(p.rows) * p.heads * dp);
    DATTN_DT_SWITCH(dtype, DATTN_DP_SWITCH(dp, (fill_q_kernel<TC, DPC><<<grid, 256, 0, st>>>(p))));
    return cudaGetLastError();
}

cudaError_t launch_rows_synth(int dtype, int dp, const RowsSynthParams& p, cudaStream_t st) {
    const int grid = grid_for(static_cast<int64_t>(p.n) * p.num_kv_heads * dp);
    DATTN_DT_SWITCH(dtype, DATTN_DP_SWITCH(dp, (rows_synth_kernel<TC, DPC><<<grid, 256, 0, st>>>(p))));
    return cudaGetLastError();
}

cudaError_t launch_scatter(int dtype, int dp, const ScatterParams& p, cudaStream_t st) {
    const int grid = grid_for(p.n * dp * (p.kv_head < 0 ? p.num_kv_heads : 1));
    DATTN_DT_SWITCH(dtype, DATTN_DP_SWITCH(dp, (scatter_kernel<TC, DPC><<<grid, 256, 0, st>>>(p))));
    return cudaGetLastError();
}

cudaError_t launch_gather(int dtype, int dp, const ScatterParams& p, cudaStream_t st) {
    const int grid = grid_for(p.n * dp * (p.kv_head < 0 ? p.num_kv_heads : 1));
    DATTN_DT_SWITCH(dtype, DATTN_DP_SWITCH(dp, (gather_kernel<TC, DPC><<<grid, 256, 0, st>>>(p))));
    return cudaGetLastError();
}

cudaError_t launch_identity_records(int dtype, int dp, void* recs, int64_t n, cudaStream_t st) {
    const int grid = grid_for(n * (dp + 4));
    DATTN_DP_SWITCH(dp, {
        if (dtype == kF64)
            identity_records_kernel<double, DPC><<<grid, 256, 0, st>>>(static_cast<double*>(recs), n);
        else
            identity_records_kernel<float, DPC><<<grid, 256, 0, st>>>(static_cast<float*>(recs), n);
    });
    return cudaGetLastError();
}

}  // namespace dattn
