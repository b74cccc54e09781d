// dattn_ptx.cuh -- sm_100a PTX wrappers used by the DistAttention kernels:
// mbarrier pipeline primitives, 1-D bulk TMA (cp.async.bulk), L2 cache
// policies, named barriers and element unpacking.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dattn {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                     smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t"
        ".reg .pred P1;\n\t"
        "DATTN_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DATTN_DONE;\n\t"
        "bra DATTN_WAIT;\n\t"
        "DATTN_DONE:\n\t"
        "}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// L2 policy: streamed-once data (the KV cache) is evicted first so the block
// tables, queries and partial records stay resident.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// 1-D bulk TMA: global -> shared, completion counted in bytes on `bar`.
// dst/src 16-B aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s_nohint(void* dst, const void* src, uint32_t bytes,
                                                uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Programmatic dependent launch: a producer grid lets the next launch on its
// stream be scheduled early; the consumer blocks in pdl_wait() until the
// producer grid has completed and its memory is visible (no-op when the
// consumer was launched without the PDL attribute).
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// exp2 in the accumulation type.
__device__ __forceinline__ float acc_exp2(float x) { return fast_exp2(x); }
__device__ __forceinline__ double acc_exp2(double x) { return exp2(x); }

// Element traits: storage type -> accumulation type, 16-B chunk unpack.
template <typename T>
struct Elem;

struct bf16_t {
    uint16_t bits;
};

template <>
struct Elem<bf16_t> {
    using Acc = float;
    static constexpr int kVec = 8;  // elements per 16-B chunk
    __device__ __forceinline__ static void unpack(const uint4& c, float (&o)[8]) {
        o[0] = __uint_as_float(c.x << 16);
        o[1] = __uint_as_float(c.x & 0xFFFF0000u);
        o[2] = __uint_as_float(c.y << 16);
        o[3] = __uint_as_float(c.y & 0xFFFF0000u);
        o[4] = __uint_as_float(c.z << 16);
        o[5] = __uint_as_float(c.z & 0xFFFF0000u);
        o[6] = __uint_as_float(c.w << 16);
        o[7] = __uint_as_float(c.w & 0xFFFF0000u);
    }
    __device__ __forceinline__ static float to_acc(bf16_t v) {
        return __uint_as_float(static_cast<uint32_t>(v.bits) << 16);
    }
    __device__ __forceinline__ static bf16_t from_acc(float f) {
        // round to nearest even (finite inputs; NaN stays NaN)
        uint32_t u = __float_as_uint(f);
        if ((u & 0x7F800000u) == 0x7F800000u)  // inf stays inf, NaN -> canonical NaN
            return bf16_t{static_cast<uint16_t>((u & 0x007FFFFFu) ? 0x7FC0u : (u >> 16))};
        u += 0x7FFFu + ((u >> 16) & 1u);
        return bf16_t{static_cast<uint16_t>(u >> 16)};
    }
};

template <>
struct Elem<float> {
    using Acc = float;
    static constexpr int kVec = 4;
    __device__ __forceinline__ static void unpack(const uint4& c, float (&o)[4]) {
        o[0] = __uint_as_float(c.x);
        o[1] = __uint_as_float(c.y);
        o[2] = __uint_as_float(c.z);
        o[3] = __uint_as_float(c.w);
    }
    __device__ __forceinline__ static float to_acc(float v) { return v; }
    __device__ __forceinline__ static float from_acc(float f) { return f; }
};

template <>
struct Elem<double> {
    using Acc = double;
    static constexpr int kVec = 2;
    __device__ __forceinline__ static void unpack(const uint4& c, double (&o)[2]) {
        o[0] = __hiloint2double(static_cast<int>(c.y), static_cast<int>(c.x));
        o[1] = __hiloint2double(static_cast<int>(c.w), static_cast<int>(c.z));
    }
    __device__ __forceinline__ static double to_acc(double v) { return v; }
    __device__ __forceinline__ static double from_acc(double f) { return f; }
};

}  // namespace dattn
