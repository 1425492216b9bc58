// Fused block epilogue shared by the GEMV and the tcgen05 GEMM: bias, f32
// outlier features, then residual (model.py:362-364,368), GELU (model.py:367)
// or the q|k|v split with the paged KV append (model.py:341-346).
#pragma once

#include "pb_common.cuh"
#include "pb_span.h"

namespace pb {

__device__ __forceinline__ float gelu_tanh(float x) {  // model.py:286-292 (f32)
    const float c = 0.7978845608028654f;
    const float u = c * (x + 0.044715f * x * x * x);
    return 0.5f * x * (1.f + tanhf(u));
}

__device__ __forceinline__ float epi_store(const Epi& e, int tok, int o, float v) {
    v += e.bias[o];
    for (int j = 0; j < e.n_outl; ++j) v = fmaf(e.outl_rows[(int64_t)j * e.M + o], e.xo[(int64_t)tok * e.n_outl + j], v);
    const int64_t idx = (int64_t)tok * e.M + o;
    if (e.kind == EPI_RESID) {
        v = e.resid[idx] + v;
        e.out[idx] = v;
    } else if (e.kind == EPI_PLAIN) {
        e.out[idx] = v;
    } else if (e.kind == EPI_GELU) {
        v = gelu_tanh(v);
        e.out[idx] = v;
    } else {  // EPI_QKV: contiguous q | k | v column thirds (model.py:342-344)
        if (o < e.d) {
            e.out[(int64_t)tok * e.d + o] = v;
        } else {
            const int part = o < 2 * e.d ? 0 : 1;
            const int oo = o - e.d * (1 + part);
            const int h = oo / e.dh, dd = oo - h * e.dh;
            const int seq = e.tok_seq[tok], pos = e.tok_pos[tok];
            const int page = e.pages[(int64_t)seq * e.max_pages + pos / e.P];
            const int slot = pos % e.P;
            const int ddp = kv_swizzled(e.dh) ? ((((dd >> 3) ^ (slot & 7)) << 3) | (dd & 7)) : dd;
            e.kv[((((int64_t)page * 2 + part) * e.H + h) * e.P + slot) * e.dh + ddp] = __float2half_rn(v);
        }
    }
    return v;
}

}  // namespace pb
