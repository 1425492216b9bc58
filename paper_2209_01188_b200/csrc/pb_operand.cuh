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

// Compensated f32 sum (Knuth TwoSum per addition; hi + lo carries ~48 bits).
struct CSum {
    float hi = 0.f, lo = 0.f;
    __device__ __forceinline__ static void two_sum(float a, float b, float& s, float& e) {
        s = __fadd_rn(a, b);  // _rn intrinsics: no contraction or reassociation
        const float bb = __fsub_rn(s, a);
        e = __fadd_rn(__fsub_rn(a, __fsub_rn(s, bb)), __fsub_rn(b, bb));
    }
    __device__ __forceinline__ void add(float v) {
        float s, e;
        two_sum(hi, v, s, e);
        hi = s;
        lo = __fadd_rn(lo, e);
    }
    __device__ __forceinline__ void warp_reduce() {
        __syncwarp();
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float oh = __shfl_xor_sync(0xffffffffu, hi, o), ol = __shfl_xor_sync(0xffffffffu, lo, o);
            float s, e;
            two_sum(hi, oh, s, e);
            hi = s;
            lo = __fadd_rn(__fadd_rn(lo, ol), e);
        }
    }
};

// Resolve {mu, inv, 2^shift, 2^-shift} of one token inside the operand
// producer (any full warp; warp-uniform control flow), from the producing epilogue's partial summaries
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
    // mean = sum n_g mean_g / N ; M2 = sum M2_g + n_g (mean_g - mean)^2, as
    // compensated (hi, lo) f32 sums -- f64 accuracy without the FP64 pipe's
    // latency on this critical path (traced: 6 us per resolve in f64). Lane
    // order is fixed and the butterfly steps are symmetric (TwoSum's error
    // term is exact), so every lane gets the same bits.
    const float4* ps = a.src.pstats + (int64_t)tok * a.src.MG;
    CSum s1, s2;
    float mn = INFINITY, mx = -INFINITY;
    // MG <= 128 (hidden <= 16384): the summaries stay in registers for the
    // second pass -- one L2 round trip on this critical path instead of five
    const bool inreg = a.src.MG <= 128;
    float4 p[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int g = lane + 32 * i;
        p[i] = g < a.src.MG ? ps[g] : make_float4(0.f, 0.f, INFINITY, -INFINITY);
    }
    for (int g0 = 0; g0 < a.src.MG; g0 += 128) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int g = g0 + lane + 32 * i;
            const float4 q = g0 == 0 ? p[i] : (g < a.src.MG ? ps[g] : make_float4(0.f, 0.f, INFINITY, -INFINITY));
            s1.add(g < a.src.MG ? __fmul_rn((float)min(128, a.src.M - g * 128), q.x) : 0.f);  // branch-free
            mn = fminf(mn, q.z);
            mx = fmaxf(mx, q.w);
        }
    }
    if (a.trace) {  // diagnostics: the stamp depends on the loaded summaries
        asm volatile("" ::"f"(s1.hi), "f"(mn), "f"(mx));
        if (lane == 0) trace_stamp(a.trace, blockIdx.y * gridDim.x + blockIdx.x, 7);
    }
    s1.warp_reduce();
    mn = -warp_max(-mn);
    mx = warp_max(mx);
    const float mu = (s1.hi + s1.lo) / (float)a.src.M;
    if (inreg) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int g = lane + 32 * i;
            const bool in = g < a.src.MG;
            const float dm = p[i].x - mu;
            s2.add(in ? p[i].y : 0.f);
            s2.add(in ? __fmul_rn(__fmul_rn((float)min(128, a.src.M - g * 128), dm), dm) : 0.f);
        }
    } else {
        for (int g = lane; g < a.src.MG; g += 32) {
            const float4 q = ps[g];
            const float dm = q.x - mu;
            s2.add(q.y);
            s2.add(__fmul_rn(__fmul_rn((float)min(128, a.src.M - g * 128), dm), dm));
        }
    }
    s2.warp_reduce();
    const float var = (s2.hi + s2.lo) / (float)a.src.M;
    const float inv = 1.0f / sqrtf(var + 1e-5f);
    const float dev = fmaxf(mx - mu, mu - mn);
    const int sh = shift_for(a.src.gs * dev * inv + a.src.bs);
    return make_float4(mu, inv, ldexpf(1.f, sh), ldexpf(1.f, -sh));
}

// Weight-side inputs of one B-fragment item (k tile kc, lane quad q: the 8
// features 4q..4q+3 and 16+4q..16+4q+3): per-feature scales and, for
// LayerNorm operands, gamma/beta. They do not depend on the previous kernel,
// so the operand writer loads them before its PDL dependency wait.
struct FragParams {
    float s[8], g[8], b[8];
};
__device__ __forceinline__ void frag_params(const ProArgs& a, int kc, int q, FragParams& p) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int k = kc * 32 + 16 * (e >> 2) + 4 * q + (e & 3);
        const bool in = k < a.K;
        p.s[e] = in ? a.scales[k] : 0.f;
        p.g[e] = in && a.mode == PRO_LN ? a.gamma[k] : 1.f;
        p.b[e] = in && a.mode == PRO_LN ? a.beta[k] : 0.f;
    }
}

// One B-fragment item of the int8-digit operand a = rint(y * s * 2^(shift + 8))
// (layout in the header comment): token tok, 32-wide k tile kc, lane quad q.
// The statistics' shift maps max |y s| into [2^13, 2^14) (the fp16 split of the
// tcgen05 path); 2^8 more gives the 22-bit integer range here.
// the item's 8 activations (requested before the statistics are resolved: independent loads)
__device__ __forceinline__ void frag_x(const ProArgs& a, int tok, int kc, int q, float (&xv)[8]) {
    const float* x = a.x + (int64_t)tok * a.K;
    const int k0 = kc * 32 + 4 * q;
    // both 4-feature runs inside a 16-byte aligned row: two 128-bit loads
    if ((a.K & 3) == 0 && k0 + 20 <= a.K && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
        const float4 lo = *reinterpret_cast<const float4*>(x + k0);
        const float4 hi = *reinterpret_cast<const float4*>(x + k0 + 16);
        xv[0] = lo.x, xv[1] = lo.y, xv[2] = lo.z, xv[3] = lo.w;
        xv[4] = hi.x, xv[5] = hi.y, xv[6] = hi.z, xv[7] = hi.w;
        return;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int k = kc * 32 + 16 * (e >> 2) + 4 * q + (e & 3);
        xv[e] = k < a.K ? x[k] : 0.f;
    }
}
__device__ __forceinline__ void frag_item(const ProArgs& a, int tok, int kc, int q, const float4 st,
                                          const FragParams& p, const float (&xv)[8]) {
    const float z = st.z * 256.f;
    const int KC = a.Kp / 32;
    const int NT = digit_ntiles(a.tc);
    const int c = tok / a.tc, col = tok % a.tc;
    uint32_t w[3][2] = {{0u, 0u}, {0u, 0u}, {0u, 0u}};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int k = kc * 32 + 16 * (e >> 2) + 4 * q + (e & 3);
        float y = 0.f;
        if (k < a.K) y = a.mode == PRO_LN ? fmaf(p.g[e], (xv[e] - st.x) * st.y, p.b[e]) : xv[e];  // model.py:271-276
        int h, m, l;
        digits3(__float2int_rn((y * p.s[e]) * z), h, m, l);
        w[0][e >> 2] |= (uint32_t)(uint8_t)h << (8 * (e & 3));
        w[1][e >> 2] |= (uint32_t)(uint8_t)m << (8 * (e & 3));
        w[2][e >> 2] |= (uint32_t)(uint8_t)l << (8 * (e & 3));
    }
    uint2* frag = reinterpret_cast<uint2*>(a.frag);
    const int64_t base = ((int64_t)c * KC + kc) * NT;
#pragma unroll
    for (int pp = 0; pp < 3; ++pp) {
        const int cc = pp * a.tc + col;
        frag[(base + (cc >> 3)) * 32 + 4 * (cc & 7) + q] = make_uint2(w[pp][0], w[pp][1]);
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
