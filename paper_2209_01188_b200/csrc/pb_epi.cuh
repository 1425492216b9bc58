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


// ---------------------------------------------------------------- tensor-core epilogue (16 tokens of one row)
//
// The tcgen05 kernels finish 128 rows x (16..80) tokens per tile. Evaluated
// element by element (epi_store) every element pays dependent global loads
// (token -> sequence/position -> KV page; the per-token scale; the residual)
// at L2 latency under a saturated memory system, and the epilogue, not the
// tensor core or HBM, bounds the kernel (measured: stream-K decode kernel at
// 32 tokens 3.9 TB/s with this epilogue, 6.2 TB/s without). Here the per-token
// constants come from shared memory (staged once per tile), per-row values
// are hoisted, and a chunk's 16 residual loads are issued before any store.

struct TokInfo {
    float back;  // 2^-shift of the token's operand (undoes the fixed-point scale)
    int page;    // EPI_QKV: KV pool page of the token's position
    int slot;    //          position within the page
    int valid;
};

// stage tokens [t0, t0 + cnt) of this tile; `tid` / `nthr` over the epilogue threads
__device__ __forceinline__ void stage_tokens(const Epi& e, const float* back, int n_tok, int t0, int cnt,
                                             TokInfo* s_tok, int tid, int nthr) {
    for (int i = tid; i < cnt; i += nthr) {
        const int tok = t0 + i;
        TokInfo t{1.f, 0, 0, 0};
        if (tok < n_tok) {
            t.back = back[tok];
            t.valid = 1;
            if (e.kind == EPI_QKV) {
                const int seq = e.tok_seq[tok], pos = e.tok_pos[tok];
                t.page = e.pages[(int64_t)seq * e.max_pages + pos / e.P];
                t.slot = pos % e.P;
            }
        }
        s_tok[i] = t;
    }
}

// 16 consecutive tokens (tile columns c0 .. c0 + 15, global tokens tok0 ..) of output row o;
// h / m / l are the three digit accumulators (exact s32), recombined exactly in int64
// s_tmax: per-CTA shared-memory max |y s_next| indexed by token (the caller flushes it), or null for
// global atomics
__device__ __forceinline__ void tc_epi16(const Epi& e, int o, int lane, int tok0, const TokInfo* ti, const int* h,
                                         const int* m, const int* l, float* s_tmax = nullptr) {
    const bool row_ok = o < e.M;
    if (e.kind == EPI_BWD) {  // dx_k = s_k * sum_o g_o codes[o][k] (pb_train.cu)
        if (!row_ok) return;
        const float rs = e.rowscale[o];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const long long iv = (long long)h[j] * 65536 + (long long)m[j] * 256 + (long long)l[j];
            if (ti[j].valid) e.out[(int64_t)(tok0 + j) * e.M + o] = (float)iv * ti[j].back * rs;
        }
        return;
    }
    const float bias = row_ok ? e.bias[o] : 0.f;
    float v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const long long iv = (long long)h[j] * 65536 + (long long)m[j] * 256 + (long long)l[j];
        v[j] = (float)iv * ti[j].back + bias;  // |iv| < 2^47: one rounding, the f64 sum's value
    }
    if (e.n_outl && row_ok) {
        for (int j = 0; j < 16; ++j)
            if (ti[j].valid)
                for (int q = 0; q < e.n_outl; ++q)
                    v[j] = fmaf(e.outl_rows[(int64_t)q * e.M + o], e.xo[(int64_t)(tok0 + j) * e.n_outl + q], v[j]);
    }
    if (e.kind == EPI_RESID) {
        float r[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) r[j] = (row_ok && ti[j].valid) ? e.resid[(int64_t)(tok0 + j) * e.M + o] : 0.f;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            v[j] += r[j];
            if (row_ok && ti[j].valid) e.out[(int64_t)(tok0 + j) * e.M + o] = v[j];
        }
    } else if (e.kind == EPI_GELU || e.kind == EPI_PLAIN) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (e.kind == EPI_GELU) v[j] = gelu_tanh(v[j]);
            if (row_ok && ti[j].valid) e.out[(int64_t)(tok0 + j) * e.M + o] = v[j];
        }
    } else if (row_ok) {  // EPI_QKV
        if (o < e.d) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (ti[j].valid) e.out[(int64_t)(tok0 + j) * e.d + o] = v[j];
        } else {
            const int part = o < 2 * e.d ? 0 : 1;
            const int oo = o - e.d * (1 + part);
            const int hh = oo / e.dh, dd = oo - hh * e.dh;
            const bool swz = kv_swizzled(e.dh);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                if (!ti[j].valid) continue;
                const int slot = ti[j].slot;
                const int ddp = swz ? ((((dd >> 3) ^ (slot & 7)) << 3) | (dd & 7)) : dd;
                e.kv[((((int64_t)ti[j].page * 2 + part) * e.H + hh) * e.P + slot) * e.dh + ddp] = __float2half_rn(v[j]);
            }
        }
    }
    if (e.tokmax) {  // operand range of the consuming matmul: max |y s_next| per token
        const float sn = row_ok ? e.s_next[o] : 0.f;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            float mx = (row_ok && ti[j].valid) ? fabsf(v[j] * sn) : 0.f;
            mx = warp_max(mx);
            if (lane == 0 && ti[j].valid)
                atomicMax(reinterpret_cast<int*>(s_tmax ? s_tmax : e.tokmax) + tok0 + j, __float_as_int(mx));
        }
    }
}
}  // namespace pb
