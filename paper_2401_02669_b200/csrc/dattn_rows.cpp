// dattn_rows.cpp -- host -> paged-store row writes (dattn_kv_write): rows are
// converted to the store dtype and zero-padded to the padded head dim in a
// pinned staging arena, copied in one H2D transfer and scattered into their
// pages by a kernel. Used by the kvsched::attn adapter to place KVSegment
// data (distattention.hpp:33-42) in HBM.
#include <cstring>

#include "dattn_engine.h"

using namespace dattn;

namespace {

uint16_t f32_to_bf16(float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    if ((u & 0x7F800000u) == 0x7F800000u) return static_cast<uint16_t>((u >> 16) | ((u & 0xFFFF) ? 0x40 : 0));
    u += 0x7FFFu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

double load_src(const void* src, int dtype, size_t i) {
    switch (dtype) {
        case kBF16: {
            uint16_t h;
            std::memcpy(&h, static_cast<const uint8_t*>(src) + 2 * i, 2);
            uint32_t u = static_cast<uint32_t>(h) << 16;
            float f;
            std::memcpy(&f, &u, 4);
            return f;
        }
        case kF32: {
            float f;
            std::memcpy(&f, static_cast<const uint8_t*>(src) + 4 * i, 4);
            return f;
        }
        default: {
            double d;
            std::memcpy(&d, static_cast<const uint8_t*>(src) + 8 * i, 8);
            return d;
        }
    }
}

void store_dst(void* dst, int dtype, size_t i, double x) {
    switch (dtype) {
        case kBF16: {
            const uint16_t h = f32_to_bf16(static_cast<float>(x));
            std::memcpy(static_cast<uint8_t*>(dst) + 2 * i, &h, 2);
            break;
        }
        case kF32: {
            const float f = static_cast<float>(x);
            std::memcpy(static_cast<uint8_t*>(dst) + 4 * i, &f, 4);
            break;
        }
        default:
            std::memcpy(static_cast<uint8_t*>(dst) + 8 * i, &x, 8);
    }
}

void pack(void* dst, int dst_dtype, int dp, const void* src, int src_dtype, int row_elems,
          int64_t n) {
    const int esz = elem_bytes_for(dst_dtype);
    std::memset(dst, 0, static_cast<size_t>(n) * dp * esz);
    if (src_dtype == dst_dtype) {
        for (int64_t t = 0; t < n; ++t)
            std::memcpy(static_cast<uint8_t*>(dst) + static_cast<size_t>(t) * dp * esz,
                        static_cast<const uint8_t*>(src) + static_cast<size_t>(t) * row_elems * esz,
                        static_cast<size_t>(row_elems) * esz);
        return;
    }
    for (int64_t t = 0; t < n; ++t)
        for (int j = 0; j < row_elems; ++j)
            store_dst(dst, dst_dtype, static_cast<size_t>(t) * dp + j,
                      load_src(src, src_dtype, static_cast<size_t>(t) * row_elems + j));
}

}  // namespace

void dattn_store::write_rows(int32_t seq, int kv_head, int64_t tok0, int64_t n, const void* k,
                             const void* v, int src_dtype, int src_row_elems) {
    const size_t rows_bytes = static_cast<size_t>(n) * dp * esz;
    const size_t need = 2 * ((rows_bytes + 255) / 256 * 256);
    if (staging_used + need > h_staging.cap || staging_used + need > d_staging.cap) {
        // the arena is recycled only once everything queued on it has run
        cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
        staging_used = 0;
        if (need > h_staging.cap) h_staging.ensure(std::max(need, h_staging.cap * 2));
        if (need > d_staging.cap) d_staging.ensure(std::max(need, d_staging.cap * 2));
    }
    uint8_t* hk = static_cast<uint8_t*>(h_staging.p) + staging_used;
    uint8_t* hv = hk + need / 2;
    uint8_t* dk = static_cast<uint8_t*>(d_staging.p) + staging_used;
    uint8_t* dv = dk + need / 2;
    pack(hk, cfg.dtype, dp, k, src_dtype, src_row_elems, n);
    pack(hv, cfg.dtype, dp, v, src_dtype, src_row_elems, n);
    cuda_check(cudaMemcpyAsync(dk, hk, need, cudaMemcpyHostToDevice, stream),
               "cudaMemcpyAsync(rows)");
    staging_used += need;
    ScatterParams p{};
    p.k_pool = kpool;
    p.v_pool = vpool;
    p.k_rows = dk;
    p.v_rows = dv;
    p.block_row = d_bt + static_cast<size_t>(seq) * cfg.max_pages_per_seq;
    p.page_tokens = cfg.page_tokens;
    p.num_kv_heads = cfg.num_kv_heads;
    p.kv_head = kv_head;
    p.tok0 = tok0;
    p.n = n;
    cuda_check(launch_scatter(cfg.dtype, dp, p, stream), "launch(scatter)");
    count_launch(1);
}
