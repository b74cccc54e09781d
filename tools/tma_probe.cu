// tools/tma_probe.cu -- streaming-rate probe for K2's K/V access pattern.
//
// Streams the config-3 KV pool (K and V, [pages][8 kv heads][16 tokens][128]
// bf16, 2 x 4.3 GB) through shared memory exactly like K2's producers do, with
// no compute: one CTA per SM claims (sequence, kv head, 8192-token chunk)
// items, a producer thread fills K and V rings of 32 KB stages (8 pages =
// 128 tokens each) and a consumer warp releases each stage as soon as it
// lands. Three ways to move one (page, kv head) slice of 4 KB:
//   mode 0: two 2-D TMA boxes of 64 columns x 16 rows, 128-B swizzle (K2 today)
//   mode 1: one 1-D bulk copy of 4 KB (K1's path)
//   mode 2: one 2-D TMA box of 128 columns x 16 rows, no swizzle
//   mode 3: two 2-D TMA boxes of 64 columns x 16 rows, 128-B swizzle, over a
//           half-split pool [pages][heads][2][16][64] (each box 2 KB contiguous)
//   mode 4: one 4-D TMA box per 64-column half per TILE (8 consecutive pages:
//           box 64 cols x 16 rows x 1 head x 8 pages, 128-B swizzle)
// Prints GB/s per mode. Build: nvcc -O3 -std=c++17 -gencode
// arch=compute_100a,code=sm_100a -o tools/tma_probe tools/tma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#include "../paper_2401_02669_b200/csrc/dattn_ptx.cuh"

using namespace dattn;

constexpr int kHeads = 8, kP = 16, kD = 128, kSeqs = 16, kPagesPerSeq = 8192, kChunkPages = 512;
constexpr int kTilePages = 8, kStages = 3, kStageBytes = kTilePages * kP * kD * 2;  // 32 KB
constexpr int kItems = kSeqs * kHeads * (kPagesPerSeq / kChunkPages);

struct Smem {
    uint8_t k[kStages][kStageBytes];
    uint8_t v[kStages][kStageBytes];
    uint64_t kfull[kStages], kempty[kStages], vfull[kStages], vempty[kStages];
};

__device__ __forceinline__ void tma4d(void* dst, const CUtensorMap* m, int c0, int c1, int c2, int c3, uint64_t* bar,
                                      uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

__global__ void __launch_bounds__(64, 1) probe(const __grid_constant__ CUtensorMap mk, const __grid_constant__ CUtensorMap mv,
                                                const uint8_t* kpool, const uint8_t* vpool, int mode,
                                                unsigned long long* counter) {
    extern __shared__ __align__(1024) uint8_t raw[];
    Smem& S = *reinterpret_cast<Smem*>(raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&S.kfull[i], 1);
            mbar_init(&S.kempty[i], 1);
            mbar_init(&S.vfull[i], 1);
            mbar_init(&S.vempty[i], 1);
        }
        fence_mbar_init();
    }
    __shared__ int s_total;
    if (threadIdx.x == 0) s_total = 0x7fffffff;
    __syncthreads();
    if (warp == 0) {
        if (lane != 0) return;
        const uint64_t pol = l2_policy_evict_first();
        uint32_t t = 0;
        for (;;) {
            const int item = static_cast<int>(atomicAdd(counter, 1ull));
            if (item >= kItems) break;
            const int kvh = item % kHeads, rest = item / kHeads;
            const int chunk = rest % (kPagesPerSeq / kChunkPages), seq = rest / (kPagesPerSeq / kChunkPages);
            const int page0 = seq * kPagesPerSeq + chunk * kChunkPages;
            for (int tp = 0; tp < kChunkPages; tp += kTilePages, ++t) {
                const int s = t % kStages;
                const uint32_t ph = ((t / kStages) & 1u) ^ 1u;
                mbar_wait(&S.kempty[s], ph);
                mbar_arrive_expect_tx(&S.kfull[s], kStageBytes);
                mbar_wait(&S.vempty[s], ph);
                mbar_arrive_expect_tx(&S.vfull[s], kStageBytes);
                if (mode == 4) {
                    const int page = page0 + tp;
                    tma4d(S.k[s], &mk, 0, 0, kvh, page, &S.kfull[s], pol);
                    tma4d(S.k[s] + kStageBytes / 2, &mk, 64, 0, kvh, page, &S.kfull[s], pol);
                    tma4d(S.v[s], &mv, 0, 0, kvh, page, &S.vfull[s], pol);
                    tma4d(S.v[s] + kStageBytes / 2, &mv, 64, 0, kvh, page, &S.vfull[s], pol);
                    continue;
                }
                for (int pg = 0; pg < kTilePages; ++pg) {
                    const int page = page0 + tp + pg;
                    const int row0 = (page * kHeads + kvh) * kP;
                    const size_t off = static_cast<size_t>(row0) * kD * 2;
                    if (mode == 0) {
                        tma2d(S.k[s] + pg * 2048, &mk, 0, row0, &S.kfull[s], pol);
                        tma2d(S.k[s] + kStageBytes / 2 + pg * 2048, &mk, 64, row0, &S.kfull[s], pol);
                        tma2d(S.v[s] + pg * 2048, &mv, 0, row0, &S.vfull[s], pol);
                        tma2d(S.v[s] + kStageBytes / 2 + pg * 2048, &mv, 64, row0, &S.vfull[s], pol);
                    } else if (mode == 1) {
                        bulk_g2s(S.k[s] + pg * 4096, kpool + off, 4096, &S.kfull[s], pol);
                        bulk_g2s(S.v[s] + pg * 4096, vpool + off, 4096, &S.vfull[s], pol);
                    } else if (mode == 2) {
                        tma2d(S.k[s] + pg * 4096, &mk, 0, row0, &S.kfull[s], pol);
                        tma2d(S.v[s] + pg * 4096, &mv, 0, row0, &S.vfull[s], pol);
                    } else {
                        const int h0 = ((page * kHeads + kvh) * 2) * kP;  // half 0 rows, half 1 follows
                        tma2d(S.k[s] + pg * 2048, &mk, 0, h0, &S.kfull[s], pol);
                        tma2d(S.k[s] + kStageBytes / 2 + pg * 2048, &mk, 0, h0 + kP, &S.kfull[s], pol);
                        tma2d(S.v[s] + pg * 2048, &mv, 0, h0, &S.vfull[s], pol);
                        tma2d(S.v[s] + kStageBytes / 2 + pg * 2048, &mv, 0, h0 + kP, &S.vfull[s], pol);
                    }
                }
            }
        }
        // terminate the consumer: stage t completes with no bytes
        const int s = t % kStages;
        mbar_wait(&S.kempty[s], ((t / kStages) & 1u) ^ 1u);
        *reinterpret_cast<volatile int*>(&s_total) = static_cast<int>(t);
        mbar_arrive(&S.kfull[s]);
    } else if (lane == 0) {
        for (uint32_t t = 0;; ++t) {
            const int s = t % kStages;
            mbar_wait(&S.kfull[s], (t / kStages) & 1u);
            if (static_cast<int>(t) == *reinterpret_cast<volatile int*>(&s_total)) break;
            mbar_wait(&S.vfull[s], (t / kStages) & 1u);
            mbar_arrive(&S.kempty[s]);
            mbar_arrive(&S.vempty[s]);
        }
    }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode() {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q{};
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
}

static void make_map(CUtensorMap* m, void* base, uint64_t rows, int mode) {
    if (mode == 4) {
        cuuint64_t dims[4] = {kD, kP, kHeads, rows / (kHeads * kP)};
        cuuint64_t strides[3] = {kD * 2, kP * kD * 2, kHeads * kP * kD * 2};
        cuuint32_t box[4] = {64, kP, 1, kTilePages};
        cuuint32_t estr[4] = {1, 1, 1, 1};
        CUresult r = encode()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) std::printf("tensor map mode %d: error %d\n", mode, static_cast<int>(r));
        return;
    }
    const bool half = mode == 3;  // [rows*2][64] view of the half-split pool
    cuuint64_t dims[2] = {half ? 64u : kD, half ? 2 * rows : rows};
    cuuint64_t strides[1] = {half ? 128u : kD * 2};
    cuuint32_t box[2] = {(mode == 0 || half) ? 64u : 128u, kP};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE,
                          (mode == 0 || mode == 3) ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) std::printf("tensor map mode %d: error %d\n", mode, static_cast<int>(r));
}

int main() {
    const size_t pages = static_cast<size_t>(kSeqs) * kPagesPerSeq;
    const size_t bytes = pages * kHeads * kP * kD * 2;
    uint8_t *k = nullptr, *v = nullptr;
    unsigned long long* counter = nullptr;
    cudaMalloc(&k, bytes);
    cudaMalloc(&v, bytes);
    cudaMalloc(&counter, 8);
    cudaMemset(k, 0, bytes);
    cudaMemset(v, 0, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int smem = sizeof(Smem) + 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[5] = {"2-D TMA, two 64-col boxes, SW128 (K2)", "1-D bulk copy of 4 KB (K1)",
                            "2-D TMA, one 128-col box, no swizzle", "2-D TMA, 64-col boxes, half-split pool",
                            "4-D TMA, one box per half per 8-page tile"};
    for (int mode = 0; mode < 5; ++mode) {
        CUtensorMap mk, mv;
        make_map(&mk, k, pages * kHeads * kP, mode);
        make_map(&mv, v, pages * kHeads * kP, mode);
        float best = 1e30f;
        for (int rep = 0; rep < 6; ++rep) {
            cudaMemset(counter, 0, 8);
            cudaEventRecord(e0);
            probe<<<sms, 64, smem>>>(mk, mv, k, v, mode, counter);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep > 0 && ms < best) best = ms;
        }
        const cudaError_t err = cudaGetLastError();
        std::printf("mode %d %-42s %.3f ms  %.0f GB/s  (%s)\n", mode, names[mode], best, 2.0 * bytes / best / 1e6,
                    cudaGetErrorString(err));
    }
    return 0;
}
