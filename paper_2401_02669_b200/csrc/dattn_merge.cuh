// dattn_merge.cuh -- device-side partial-record merging shared by the MA
// kernels (fused group merge) and the merge kernels (K3, K5, K6):
// the online-softmax rescale-and-sum of aggregate_partials /
// combine_partials (/root/reference/proj/src/distattention.cpp:131-174).
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>

#include "dattn_internal.h"
#include "dattn_ptx.cuh"

namespace dattn {

constexpr int kConsumerWarps = 8;

constexpr int kMergeWarps = 8;

// Rescale-sum of the live chunk records c = sub + stride*i (< n) of one group:
// lanes first compute the weights w = exp(m - m_g) of 32 records in parallel,
// then the warp folds the records' ma vectors (lane-owned kVW-element slices,
// independent vector loads) with the broadcast weights. Dead records get
// w = 0; identity records hold ma = 0, so adding them changes nothing and a
// single live record is reproduced exactly. Returns warp-reduced (e, tokens).
template <typename Acc, int DP, int kVW, int kSweeps, typename LiveF>
__device__ __forceinline__ void fold_chunks(const Acc* R, int64_t base, int64_t c_stride, int n, int sub,
                                            int stride, Acc mg, LiveF live, Acc (&acc)[kSweeps][kVW],
                                            Acc& eg, Acc& ntok, int lane) {
    constexpr int REC = DP + 4;
    constexpr int kPer = 32 * kVW;
    Acc e_l = 0, t_l = 0;
    for (int i0 = 0; sub + stride * i0 < n; i0 += 32) {
        const int c = sub + stride * (i0 + lane);
        Acc w = 0;
        if (c < n) {
            const Acc* r = R + (base + static_cast<int64_t>(c) * c_stride) * REC;
            if (live(c, r)) {
                const Acc mc = __ldcg(r);
                w = (mc == mg) ? Acc(1) : exp(mc - mg);
                e_l += __ldcg(r + 1) * w;
                t_l += __ldcg(r + 2);
            }
        }
        const int cnt = min(32, (n - sub - stride * i0 + stride - 1) / stride);
#pragma unroll 4
        for (int k = 0; k < cnt; ++k) {
            const Acc wk = __shfl_sync(0xffffffffu, w, k);
            const Acc* r = R + (base + static_cast<int64_t>(sub + stride * (i0 + k)) * c_stride) * REC;
#pragma unroll
            for (int sw = 0; sw < kSweeps; ++sw) {
                const int j = sw * kPer + lane * kVW;
                if (j < DP) {
                    if constexpr (kVW == 4) {
                        const float4 x = __ldcg(reinterpret_cast<const float4*>(r + 4 + j));
                        acc[sw][0] += x.x * wk; acc[sw][1] += x.y * wk;
                        acc[sw][2] += x.z * wk; acc[sw][3] += x.w * wk;
                    } else if constexpr (kVW == 2 && sizeof(Acc) == 8) {
                        const double2 x = __ldcg(reinterpret_cast<const double2*>(r + 4 + j));
                        acc[sw][0] += x.x * wk; acc[sw][1] += x.y * wk;
                    } else {
#pragma unroll
                        for (int v = 0; v < kVW; ++v) acc[sw][v] += __ldcg(r + 4 + j + v) * wk;
                    }
                }
            }
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        e_l += __shfl_xor_sync(0xffffffffu, e_l, off);
        t_l += __shfl_xor_sync(0xffffffffu, t_l, off);
    }
    eg = e_l;
    ntok = t_l;
}


// ---- exchange slots without flags (K5). An exchange word that has not
// arrived holds all ones -- a NaN no arithmetic produces, and producers map
// that one bit pattern to the payload-less NaN below -- so a receiver sees a
// word arrive from its value alone: no system fence, no flag, no second
// NVLink round trip. The receiver puts the empty pattern back after reading,
// which is safe because a peer writes the same half of the buffer again only
// two steps later, after it has seen this rank's next-step records.
template <class Acc> struct XWord;
template <> struct XWord<float> { using U = uint32_t; };
template <> struct XWord<double> { using U = unsigned long long; };

template <class Acc>
__device__ __forceinline__ typename XWord<Acc>::U x_enc(Acc v) {
    using U = typename XWord<Acc>::U;
    U b;
    memcpy(&b, &v, sizeof b);
    return b == ~U(0) ? (~U(0) >> 1) : b;
}
template <class Acc>
__device__ __forceinline__ Acc x_dec(typename XWord<Acc>::U b) {
    Acc v;
    memcpy(&v, &b, sizeof v);
    return v;
}

// N words at p (16-byte aligned when N*sizeof(U) is a multiple of 16); the
// words are repacked into uint4 values so the arrays stay in registers
template <class U>
__device__ __forceinline__ uint4 x_pack(const U* w) {
    if constexpr (sizeof(U) == 4) return make_uint4(w[0], w[1], w[2], w[3]);
    else
        return make_uint4(static_cast<uint32_t>(w[0]), static_cast<uint32_t>(w[0] >> 32),
                          static_cast<uint32_t>(w[1]), static_cast<uint32_t>(w[1] >> 32));
}
template <class U>
__device__ __forceinline__ void x_unpack(uint4 v, U* w) {
    if constexpr (sizeof(U) == 4) {
        w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
    } else {
        w[0] = (static_cast<U>(v.y) << 32) | v.x;
        w[1] = (static_cast<U>(v.w) << 32) | v.z;
    }
}
template <class U, int N>
__device__ __forceinline__ void x_store(U* p, const U (&w)[N]) {
    if constexpr ((N * sizeof(U)) % 16 == 0) {
#pragma unroll
        for (int i = 0; i < N; i += 16 / sizeof(U)) *reinterpret_cast<uint4*>(p + i) = x_pack<U>(w + i);
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) p[i] = w[i];
    }
}
template <class U, int N>
__device__ __forceinline__ void x_clear(U* p) {
    U w[N];
#pragma unroll
    for (int i = 0; i < N; ++i) w[i] = ~U(0);
    x_store<U, N>(p, w);
}
__device__ __forceinline__ uint4 ld_volatile_v4(const void* p) {
    uint4 v;
    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    return v;
}
// Spin until none of the N words is empty. A poll still waiting after
// kXSlowNs checks the control words every 256 spins: another poll's failure
// (status), the host's abort word and the timeout; on abort / timeout it
// records the reason (XCtl) and returns with the words it has (the step's
// output is invalid, the context stays alive).
template <class U, int N>
__device__ __forceinline__ void x_poll(const U* p, U (&w)[N], const XCtl& ctl) {
    uint64_t t0 = 0;
    for (int spin = 0;; ++spin) {
        bool ok = true;
        if constexpr ((N * sizeof(U)) % 16 == 0) {
#pragma unroll
            for (int i = 0; i < N; i += 16 / sizeof(U)) x_unpack<U>(ld_volatile_v4(p + i), w + i);
        } else {
#pragma unroll
            for (int i = 0; i < N; ++i) w[i] = *reinterpret_cast<const volatile U*>(p + i);
        }
#pragma unroll
        for (int i = 0; i < N; ++i) ok &= (w[i] != ~U(0));
        if (ok) return;
        if ((spin & 255) == 0) {
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (spin == 0) {
                t0 = t;
            } else if (t - t0 > kXSlowNs) {
                if (*reinterpret_cast<const volatile int*>(ctl.status_dev) != 0) return;
                int reason = 0;
                if (*reinterpret_cast<const volatile int*>(ctl.abort_dev) != 0) reason = kXAbortHost;
                else if (t - t0 > ctl.timeout_ns) reason = kXTimeout;
                if (reason) {
                    *reinterpret_cast<volatile int*>(ctl.status_dev) = reason;
                    *reinterpret_cast<volatile int*>(ctl.status_host) = reason;
                    __threadfence_system();
                    return;
                }
            }
        }
    }
}


// Warp-only group merge (the MA kernels' dedicated merge warp): for every q
// head of kv head `kvh`, rescale-sum the row's chunk records and write the
// normalised output (mode 1) or push the merged record to every rank's
// exchange slot (mode 2). No barriers: it runs beside the streaming warps.
// Up to MAXG heads are folded together so each chunk step issues MAXG
// independent loads (the heads of a chunk are adjacent records).
template <typename T, int DP, int MAXG>
__device__ void warp_group_merge(const MAParams& p, int row, int kvh, int lane) {
    using E = Elem<T>;
    using Acc = typename E::Acc;
    constexpr int REC = DP + 4;
    constexpr int kVW = (sizeof(Acc) == 4) ? (DP % 128 == 0 ? 4 : (DP % 64 == 0 ? 2 : 1))
                                           : (DP % 64 == 0 ? 2 : 1);
    constexpr int kPer = 32 * kVW;
    constexpr int kSweeps = (DP + kPer - 1) / kPer;
    const Acc kNegInf = -static_cast<Acc>(INFINITY);
    const int cbase = p.row_begin[row];
    const int n = p.row_begin[row + 1] - cbase;
    const Acc* R = static_cast<const Acc*>(p.records);
    for (int h0 = 0; h0 < p.group; h0 += MAXG) {
        const int nh = min(MAXG, p.group - h0);
        const int64_t base = static_cast<int64_t>(cbase) * p.num_q_heads + static_cast<int64_t>(kvh) * p.group + h0;
        auto rec_of = [&](int c, int hh) { return R + (base + static_cast<int64_t>(c) * p.num_q_heads + hh) * REC; };
        auto chunk_live = [&](int c) {
            if (!p.chunk_kvh) return true;
            const int tag = p.chunk_kvh[cbase + c];
            return tag < 0 || tag == kvh;
        };
        // pass 1: per-head max over live records (lanes over chunks)
        Acc mg[MAXG];
#pragma unroll
        for (int hh = 0; hh < MAXG; ++hh) mg[hh] = kNegInf;
        for (int c = lane; c < n; c += 32) {
            if (!chunk_live(c)) continue;
#pragma unroll
            for (int hh = 0; hh < MAXG; ++hh) {
                if (hh >= nh) continue;
                const Acc* r = rec_of(c, hh);
                const Acc tk = __ldcg(r + 2), mc = __ldcg(r);
                if (tk != Acc(0)) mg[hh] = mc > mg[hh] ? mc : mg[hh];
            }
        }
#pragma unroll
        for (int hh = 0; hh < MAXG; ++hh)
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const Acc o = __shfl_xor_sync(0xffffffffu, mg[hh], off);
                mg[hh] = o > mg[hh] ? o : mg[hh];
            }
        // pass 2: rounds of 32 chunks: lane weights, then a broadcast fold
        Acc e_l[MAXG], t_l[MAXG];
        Acc acc[MAXG][kSweeps][kVW];
#pragma unroll
        for (int hh = 0; hh < MAXG; ++hh) {
            e_l[hh] = t_l[hh] = 0;
#pragma unroll
            for (int sw = 0; sw < kSweeps; ++sw)
#pragma unroll
                for (int v = 0; v < kVW; ++v) acc[hh][sw][v] = 0;
        }
        for (int i0 = 0; i0 < n; i0 += 32) {
            const int c = i0 + lane;
            Acc w[MAXG];
            const bool cl = c < n && chunk_live(c);
#pragma unroll
            for (int hh = 0; hh < MAXG; ++hh) {
                w[hh] = 0;
                if (cl && hh < nh) {
                    const Acc* r = rec_of(c, hh);
                    const Acc tk = __ldcg(r + 2);
                    if (tk != Acc(0)) {
                        const Acc mc = __ldcg(r);
                        w[hh] = (mc == mg[hh]) ? Acc(1) : exp(mc - mg[hh]);
                        e_l[hh] += __ldcg(r + 1) * w[hh];
                        t_l[hh] += tk;
                    }
                }
            }
            const int cnt = min(32, n - i0);
            for (int k = 0; k < cnt; ++k) {
#pragma unroll
                for (int hh = 0; hh < MAXG; ++hh) {
                    if (hh >= nh) continue;
                    const Acc wk = __shfl_sync(0xffffffffu, w[hh], k);
                    const Acc* r = rec_of(i0 + k, hh);
#pragma unroll
                    for (int sw = 0; sw < kSweeps; ++sw) {
                        const int j = sw * kPer + lane * kVW;
                        if (j < DP) {
                            if constexpr (kVW == 4) {
                                const float4 x = __ldcg(reinterpret_cast<const float4*>(r + 4 + j));
                                acc[hh][sw][0] += x.x * wk; acc[hh][sw][1] += x.y * wk;
                                acc[hh][sw][2] += x.z * wk; acc[hh][sw][3] += x.w * wk;
                            } else {
#pragma unroll
                                for (int v = 0; v < kVW; ++v) acc[hh][sw][v] += __ldcg(r + 4 + j + v) * wk;
                            }
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int hh = 0; hh < MAXG; ++hh)
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                e_l[hh] += __shfl_xor_sync(0xffffffffu, e_l[hh], off);
                t_l[hh] += __shfl_xor_sync(0xffffffffu, t_l[hh], off);
            }
#pragma unroll
        for (int hh = 0; hh < MAXG; ++hh) {
            if (hh >= nh) continue;
            const Acc eg = e_l[hh], ntok = t_l[hh];
            const int64_t g = static_cast<int64_t>(row) * p.num_q_heads + static_cast<int64_t>(kvh) * p.group + h0 + hh;
            if (p.fused_mode == 1) {
                T* o = static_cast<T*>(p.out_norm) + g * DP;
#pragma unroll
                for (int sw = 0; sw < kSweeps; ++sw) {
                    const int j = sw * kPer + lane * kVW;
                    if (j < DP)
#pragma unroll
                        for (int v = 0; v < kVW; ++v)
                            o[j + v] = E::from_acc(ntok != Acc(0) ? acc[hh][sw][v] / eg : Acc(0));
                }
            }
            if (p.fused_mode == 2) {
                // every rank's exchange slot, in self-validating words (XWord)
                using U = typename XWord<Acc>::U;
                const U hdr[4] = {x_enc(ntok != Acc(0) ? mg[hh] : kNegInf), x_enc(eg), x_enc(ntok), x_enc(Acc(0))};
                for (int d = 0; d < p.nranks; ++d) {
                    U* dst = static_cast<U*>(p.peer_x[d]) + (static_cast<int64_t>(p.rank) * p.slot_stride + g) * REC;
                    if (ntok != Acc(0)) {
#pragma unroll
                        for (int sw = 0; sw < kSweeps; ++sw) {
                            const int j = sw * kPer + lane * kVW;
                            if (j < DP) {
                                U w[kVW];
#pragma unroll
                                for (int v = 0; v < kVW; ++v) w[v] = x_enc(acc[hh][sw][v]);
                                x_store<U, kVW>(dst + 4 + j, w);
                            }
                        }
                    }
                    if (lane == 0) x_store<U, 4>(dst, hdr);
                }
            } else if (p.out_recs) {
                Acc* dst = static_cast<Acc*>(p.out_recs) + g * REC;
#pragma unroll
                for (int sw = 0; sw < kSweeps; ++sw) {
                    const int j = sw * kPer + lane * kVW;
                    if (j < DP)
#pragma unroll
                        for (int v = 0; v < kVW; ++v) dst[4 + j + v] = acc[hh][sw][v];
                }
                if (lane == 0) {
                    dst[0] = ntok != Acc(0) ? mg[hh] : kNegInf;
                    dst[1] = eg;
                    dst[2] = ntok;
                    dst[3] = 0;
                }
            }
        }
    }
}

// Single-producer-per-item / single-consumer queue of completed groups in
// shared memory, from the streaming warps to the merge warp.
constexpr int kMergeQueue = 64;
struct MergeQueue {
    int32_t slot[kMergeQueue];   // packed (row << 8 | kvh), -1 = stop
    volatile int32_t seq[kMergeQueue];  // index + 1 once the slot is written
    int32_t tail;                // next index to hand out (atomicAdd)
    volatile int32_t head;       // next index the merge warp consumes
};

// Completion-count increment with acq_rel semantics at gpu scope: after a CTA
// barrier, one thread's release is cumulative over the CTA's record stores
// (the pattern CUTLASS semaphores use), and the acquire side sees every other
// CTA's records of the group -- no full __threadfence on the streaming path.
__device__ __forceinline__ int atomic_add_acq_rel_gpu(int32_t* p, int32_t v) {
    int32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ void mq_push(MergeQueue* q, int32_t v) {
    const int idx = atomicAdd(&q->tail, 1);
    while (idx - q->head >= kMergeQueue) __nanosleep(64);  // full: the merge warp is behind
    q->slot[idx % kMergeQueue] = v;
    __threadfence_block();
    q->seq[idx % kMergeQueue] = idx + 1;
}

__device__ __forceinline__ int32_t mq_pop(MergeQueue* q, int idx) {
    while (q->seq[idx % kMergeQueue] != idx + 1) __nanosleep(200);  // gentle: not on the critical path
    __threadfence_block();
    const int32_t v = q->slot[idx % kMergeQueue];
    q->head = idx + 1;
    return v;
}

// Rank merge over the exchange buffer X ([nranks][slot_stride] records of
// self-validating words): one warp per (row, q head) group g. Lane r reads
// rank r's header, every lane its payload words of each live record, merged
// in rank order into out (storage dtype); then the slots are emptied for the
// step after next (a peer writes this half again only after it has seen this
// rank's next-step records). Identity records carry only a header.
template <typename T, int DP>
__device__ __forceinline__ void xchg_rank_merge(typename XWord<typename Elem<T>::Acc>::U* X, int64_t g, int nranks,
                                                int64_t slot_stride, void* out_norm, int lane,
                                                const XCtl& ctl) {
    using E = Elem<T>;
    using Acc = typename E::Acc;
    using U = typename XWord<Acc>::U;
    constexpr int REC = DP + 4;
    constexpr int kVW = (sizeof(Acc) == 4) ? (DP % 128 == 0 ? 4 : (DP % 64 == 0 ? 2 : 1))
                                           : (DP % 64 == 0 ? 2 : 1);
    constexpr int kPer = 32 * kVW;
    constexpr int kSweeps = (DP + kPer - 1) / kPer;
    const Acc kNegInf = -static_cast<Acc>(INFINITY);
    constexpr int kPayVW = (kSweeps == 1 && kVW * sizeof(U) == 16 && DP == kPer) ? kVW : 1;
    U pay[kMaxRanks][kPayVW];
    if constexpr (kPayVW == kVW && kSweeps == 1 && kVW * sizeof(U) == 16 && DP == kPer) {
#pragma unroll
        for (int r = 0; r < kMaxRanks; ++r)
            if (r < nranks) x_unpack<U>(ld_volatile_v4(X + (static_cast<int64_t>(r) * slot_stride + g) * REC + 4 + lane * kVW),
                                        pay[r]);
    }
    Acc mr = kNegInf, er = 0, tr = 0;
    if (lane < nranks) {
        U h[4];
        x_poll<U, 4>(X + (static_cast<int64_t>(lane) * slot_stride + g) * REC, h, ctl);
        mr = x_dec<Acc>(h[0]);
        er = x_dec<Acc>(h[1]);
        tr = x_dec<Acc>(h[2]);
    }
    Acc m2 = tr != Acc(0) ? mr : kNegInf;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m2 = fmax(m2, __shfl_xor_sync(0xffffffffu, m2, off));
    const Acc wl = tr != Acc(0) ? ((mr == m2) ? Acc(1) : exp(mr - m2)) : Acc(0);
    Acc e2 = 0, tok2 = 0;
    Acc a2[kSweeps][kVW];
#pragma unroll
    for (int sw = 0; sw < kSweeps; ++sw)
#pragma unroll
        for (int v = 0; v < kVW; ++v) a2[sw][v] = 0;
    unsigned live_mask = 0;
    if constexpr (kSweeps == 1 && kVW * sizeof(U) == 16 && DP == kPer) {
        // one 16-B payload word group per lane and rank: the payloads of all
        // ranks were requested together with the headers (pay[], read once
        // without waiting); only words not yet arrived are polled again
#pragma unroll
        for (int r = 0; r < kMaxRanks; ++r) {
            if (r < nranks) {
                const Acc tk = __shfl_sync(0xffffffffu, tr, r);
                const Acc w = __shfl_sync(0xffffffffu, wl, r);
                const Acc er_r = __shfl_sync(0xffffffffu, er, r);
                if (tk != Acc(0)) {  // warp-uniform
                    live_mask |= 1u << r;
                    e2 += er_r * w;
                    tok2 += tk;
                    bool ok = true;
#pragma unroll
                    for (int v = 0; v < kVW; ++v) ok &= pay[r][v] != ~U(0);
                    if (!ok) x_poll<U, kVW>(X + (static_cast<int64_t>(r) * slot_stride + g) * REC + 4 + lane * kVW, pay[r], ctl);
#pragma unroll
                    for (int v = 0; v < kVW; ++v) a2[0][v] += x_dec<Acc>(pay[r][v]) * w;
                }
            }
        }
    } else {
        for (int r = 0; r < nranks; ++r) {
            const Acc tk = __shfl_sync(0xffffffffu, tr, r);
            const Acc w = __shfl_sync(0xffffffffu, wl, r);
            const Acc er_r = __shfl_sync(0xffffffffu, er, r);
            if (tk == Acc(0)) continue;  // warp-uniform
            live_mask |= 1u << r;
            e2 += er_r * w;
            tok2 += tk;
            const U* rec = X + (static_cast<int64_t>(r) * slot_stride + g) * REC;
#pragma unroll
            for (int sw = 0; sw < kSweeps; ++sw) {
                const int j = sw * kPer + lane * kVW;
                if (j < DP) {
                    U dw[kVW];
                    x_poll<U, kVW>(rec + 4 + j, dw, ctl);
#pragma unroll
                    for (int v = 0; v < kVW; ++v) a2[sw][v] += x_dec<Acc>(dw[v]) * w;
                }
            }
        }
    }
    __syncwarp();
    for (int r = 0; r < nranks; ++r) {
        U* rec = X + (static_cast<int64_t>(r) * slot_stride + g) * REC;
        if (lane == r) x_clear<U, 4>(rec);
        if (live_mask & (1u << r)) {
#pragma unroll
            for (int sw = 0; sw < kSweeps; ++sw) {
                const int j = sw * kPer + lane * kVW;
                if (j < DP) x_clear<U, kVW>(rec + 4 + j);
            }
        }
    }
    T* o = static_cast<T*>(out_norm) + g * DP;
#pragma unroll
    for (int sw = 0; sw < kSweeps; ++sw) {
        const int j = sw * kPer + lane * kVW;
        if (j < DP)
#pragma unroll
            for (int v = 0; v < kVW; ++v) o[j + v] = E::from_acc(tok2 != Acc(0) ? a2[sw][v] / e2 : Acc(0));
    }
}

}  // namespace dattn
