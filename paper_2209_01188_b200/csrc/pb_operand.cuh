// Device building blocks of the int8-digit matmul operand (statistics
// resolution, digit split, fragment items) and the decode GEMV's tensor-core
// primitives (pb_gemv.cu).
#pragma once

#include "pb_common.cuh"
#include "pb_span.h"

namespace pb {

__host__ __device__ constexpr int digit_ntiles(int tc) { return (3 * tc + 7) / 8; }

// three balanced int8 digits of a (|a| < 2^22): a = 65536 h + 256 m + l
__device__ __forceinline__ void digits3(int a, int& h, int& m, int& l) {
    l = ((a + 128) & 255) - 128;
    const int a1 = (a - l) >> 8;
    m = ((a1 + 128) & 255) - 128;
    h = (a1 - m) >> 8;
}

__device__ __forceinline__ float pro_y(const ProArgs& a, const float* x, int k, float mu, float inv) {
    if (a.mode == PRO_LN) return fmaf(a.gamma[k], (x[k] - mu) * inv, a.beta[k]);  // model.py:271-276
    return x[k];
}

__device__ __forceinline__ int shift_for(float bound) {
    if (!(bound > 0.f) || !isfinite(bound)) return 0;
    int e;
    frexpf(bound, &e);
    return 14 - e;
}

// Resolve {mu, inv, 2^shift, 2^-shift} of one token inside the operand
// producer (warp 0), from the producing epilogue's partial summaries
// (deterministic lane-strided + fixed shuffle-tree merge) or from the exact
// atomicMax of |x s|.
__device__ inline float4 resolve_stats(const ProArgs& a, int tok) {
    const int lane = threadIdx.x & 31;
    if (a.src.kind == SRC_TOKMAX) {
        const int sh = shift_for(a.src.tokmax[tok]);
        return make_float4(0.f, 1.f, ldexpf(1.f, sh), ldexpf(1.f, -sh));
    }
    if (a.src.kind == SRC_STATS) return a.stats[tok];
    // parallel two-pass combination of the 128-row group summaries:
    // mean = sum n_g mean_g / N ; M2 = sum M2_g + n_g (mean_g - mean)^2 (f64;
    // butterfly sums are commutative, so every lane gets the same bits)
    const float4* ps = a.src.pstats + (int64_t)tok * a.src.MG;
    double s1 = 0.0;
    float mn = INFINITY, mx = -INFINITY;
    for (int g = lane; g < a.src.MG; g += 32) {
        const float4 p = ps[g];
        s1 += (double)min(128, a.src.M - g * 128) * (double)p.x;
        mn = fminf(mn, p.z);
        mx = fmaxf(mx, p.w);
    }
    s1 = warp_sum_d(s1);
    mn = -warp_max(-mn);
    mx = warp_max(mx);
    const double mean = s1 / a.src.M;
    double s2 = 0.0;
    for (int g = lane; g < a.src.MG; g += 32) {
        const float4 p = ps[g];
        const double dm = (double)p.x - mean;
        s2 += (double)p.y + (double)min(128, a.src.M - g * 128) * dm * dm;
    }
    s2 = warp_sum_d(s2);
    const float mu = (float)mean;
    const float var = (float)(s2 / a.src.M);
    const float inv = 1.0f / sqrtf(var + 1e-5f);
    const float dev = fmaxf(mx - mu, mu - mn);
    const int sh = shift_for(a.src.gs * dev * inv + a.src.bs);
    return make_float4(mu, inv, ldexpf(1.f, sh), ldexpf(1.f, -sh));
}

// One B-fragment item of the int8-digit operand a = rint(y * s * 2^(shift + 8))
// (layout in the header comment): token tok, 32-wide k tile kc, lane quad q.
// The statistics' shift maps max |y s| into [2^13, 2^14) (the fp16 split of the
// tcgen05 path); 2^8 more gives the 22-bit integer range here.
__device__ __forceinline__ void frag_item(const ProArgs& a, int tok, int kc, int q, const float4 st) {
    const float* x = a.x + (int64_t)tok * a.K;
    const float z = st.z * 256.f;
    const int KC = a.Kp / 32;
    const int NT = digit_ntiles(a.tc);
    const int c = tok / a.tc, col = tok % a.tc;
    uint32_t w[3][2] = {{0u, 0u}, {0u, 0u}, {0u, 0u}};
#pragma unroll
    for (int half_ = 0; half_ < 2; ++half_) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int k = kc * 32 + 16 * half_ + 4 * q + i;
            const float v = k < a.K ? (pro_y(a, x, k, st.x, st.y) * a.scales[k]) * z : 0.f;
            int h, m, l;
            digits3(__float2int_rn(v), h, m, l);
            w[0][half_] |= (uint32_t)(uint8_t)h << (8 * i);
            w[1][half_] |= (uint32_t)(uint8_t)m << (8 * i);
            w[2][half_] |= (uint32_t)(uint8_t)l << (8 * i);
        }
    }
    uint2* frag = reinterpret_cast<uint2*>(a.frag);
    const int64_t base = ((int64_t)c * KC + kc) * NT;
#pragma unroll
    for (int p = 0; p < 3; ++p) {
        const int cc = p * a.tc + col;
        frag[(base + (cc >> 3)) * 32 + 4 * (cc & 7) + q] = make_uint2(w[p][0], w[p][1]);
    }
}

// Per-token side outputs of the operand writer: 2^-(shift + 8), the reset of
// the next producer's range accumulator, the f32 activations at the outlier
// features.
__device__ __forceinline__ void operand_token_outputs(const ProArgs& a, int tok, const float4 st, int tid,
                                                      int nthr) {
    if (tid == 0) {
        a.back[tok] = st.w * (1.f / 256.f);
        if (a.src.zero_tokmax) a.src.zero_tokmax[tok] = 0.f;
    }
    if (a.xo) {
        const float* x = a.x + (int64_t)tok * a.K;
        for (int j = tid; j < a.n_outl; j += nthr) a.xo[(int64_t)tok * a.n_outl + j] = pro_y(a, x, a.outl_idx[j], st.x, st.y);
    }
}

__device__ __forceinline__ void imma16832(int* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                          uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldsm_x4_i8(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}

}  // namespace pb
