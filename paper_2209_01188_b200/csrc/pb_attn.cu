// ALiBi causal attention over the paged fp16 KV cache (model.py:345-361).
//
// scores[h, i, j] = fl(fl(q_i . k_j / f32(sqrt(dh))) + fl(slope_h * (j - pos_i))),
// masked for j > pos_i, max-subtracted softmax, then P V. Every query token
// carries its own sequence and absolute position, so decode (t = 1 per
// session, many sessions) and prefill (t > 1) share one kernel.
//
// Split-T (flash-decoding): CTA = (head, query token, key chunk of 256).
// Keys are streamed as 16-byte vectors: a key row of dh fp16 is spread over
// LPK = dh/8 lanes (8 dims each), so one warp covers 32/LPK keys per
// iteration with fully coalesced 512 B reads (dh = 128: 2 keys), reduces the
// dot over its LPK lanes with shuffles, and keeps scores in shared memory for
// an exact (two-pass) chunk softmax. Chunks are merged in a second kernel with
// the usual max/sum rescaling.
//
// Pool layout per block: [page][K|V][H][P][dh] fp16, so a head's keys within a
// page are contiguous (P * dh * 2 B).
#include "pb_common.cuh"
#include "pb_span.h"

namespace pb {

constexpr int ATT_KCH = 128;  // keys per CTA
constexpr int ATT_U = 4;      // key rows in flight per lane
constexpr int ATT_WARPS = 4;

template <int DH>
struct AttnCfg {
    static constexpr int DPL = DH < 8 ? DH : 8;  // dims per lane
    static constexpr int LPK = DH / DPL;         // lanes per key
    static constexpr int KPW = 32 / LPK;         // keys per warp iteration
    static_assert(LPK <= 32 && 32 % LPK == 0, "head_dim must be 8 * 2^i (or < 8 and a power of two)");
};

template <int DPL>
__device__ __forceinline__ void load_h(const half* p, float* out) {
    if constexpr (DPL == 8) {
        const uint4 u = *reinterpret_cast<const uint4*>(p);
        const half2* h = reinterpret_cast<const half2*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __half22float2(h[i]);
            out[2 * i] = f.x;
            out[2 * i + 1] = f.y;
        }
    } else if constexpr (DPL == 4) {
        const uint2 u = *reinterpret_cast<const uint2*>(p);
        const half2* h = reinterpret_cast<const half2*>(&u);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const float2 f = __half22float2(h[i]);
            out[2 * i] = f.x;
            out[2 * i + 1] = f.y;
        }
    } else {
#pragma unroll
        for (int i = 0; i < DPL; ++i) out[i] = __half2float(p[i]);
    }
}

template <int DH>
__global__ void __launch_bounds__(ATT_WARPS * 32) k_attn_split(AttnArgs a, int nsplit) {
    using C = AttnCfg<DH>;
    __shared__ float sc[ATT_KCH];
    __shared__ float red[ATT_WARPS];
    __shared__ float osum[ATT_WARPS][DH];
    const int h = blockIdx.x, tok = blockIdx.y, split = blockIdx.z;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int pos = a.tok_pos[tok], seq = a.tok_seq[tok];
    const int j0 = split * ATT_KCH;
    const int j1 = min(j0 + ATT_KCH, pos + 1);
    float* out = a.part + (((int64_t)tok * a.H + h) * nsplit + split) * (DH + 2);
    if (j0 >= j1) {  // chunk entirely in the causal future
        if (threadIdx.x == 0) {
            out[0] = -INFINITY;
            out[1] = 0.f;
        }
        return;
    }
    const int sub = lane % C::LPK, slot = lane / C::LPK;
    const int d0 = sub * C::DPL;
    float qv[C::DPL];
#pragma unroll
    for (int i = 0; i < C::DPL; ++i) qv[i] = a.q[(int64_t)tok * a.d + h * DH + d0 + i];
    const float sq = (float)sqrt((double)DH);
    const float slope = a.slopes[h];
    const int32_t* pt = a.pages + (int64_t)seq * a.max_pages;
    const int64_t head_off = (int64_t)h * a.P * DH;
    const int64_t kv_stride = (int64_t)a.H * a.P * DH;  // K -> V within a page

    // scores: ATT_U key vectors in flight per lane before any dot product
    for (int base = j0 + warp * C::KPW * ATT_U; base < j1; base += ATT_WARPS * C::KPW * ATT_U) {
        float kf[ATT_U][C::DPL];
#pragma unroll
        for (int u = 0; u < ATT_U; ++u) {
            const int j = base + u * C::KPW + slot;
            if (j < j1) {
                const int page = pt[j / a.P];
                load_h<C::DPL>(a.kv + (int64_t)page * 2 * kv_stride + head_off + (int64_t)(j % a.P) * DH + d0, kf[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < ATT_U; ++u) {
            const int j = base + u * C::KPW + slot;
            float dot = 0.f;
            if (j < j1) {
#pragma unroll
                for (int i = 0; i < C::DPL; ++i) dot = fmaf(qv[i], kf[u][i], dot);
            }
#pragma unroll
            for (int o = C::LPK / 2; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
            if (j < j1 && sub == 0)
                sc[j - j0] = __fadd_rn(__fdiv_rn(dot, sq), __fmul_rn(slope, (float)(j - pos)));
        }
    }
    __syncthreads();
    const int nk = j1 - j0;
    float m = -INFINITY;
    for (int i = threadIdx.x; i < nk; i += blockDim.x) m = fmaxf(m, sc[i]);
    m = warp_max(m);
    if (lane == 0) red[warp] = m;
    __syncthreads();
    m = red[0];
#pragma unroll
    for (int w = 1; w < ATT_WARPS; ++w) m = fmaxf(m, red[w]);
    __syncthreads();
    float l = 0.f;
    for (int i = threadIdx.x; i < nk; i += blockDim.x) {
        const float p = expf(__fsub_rn(sc[i], m));
        sc[i] = p;
        l += p;
    }
    l = warp_sum(l);
    if (lane == 0) red[warp] = l;
    __syncthreads();
    l = 0.f;
#pragma unroll
    for (int w = 0; w < ATT_WARPS; ++w) l += red[w];

    // P V
    float ov[C::DPL];
#pragma unroll
    for (int i = 0; i < C::DPL; ++i) ov[i] = 0.f;
    for (int base = j0 + warp * C::KPW * ATT_U; base < j1; base += ATT_WARPS * C::KPW * ATT_U) {
        float vf[ATT_U][C::DPL];
#pragma unroll
        for (int u = 0; u < ATT_U; ++u) {
            const int j = base + u * C::KPW + slot;
            if (j < j1) {
                const int page = pt[j / a.P];
                load_h<C::DPL>(a.kv + (int64_t)page * 2 * kv_stride + kv_stride + head_off + (int64_t)(j % a.P) * DH + d0,
                               vf[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < ATT_U; ++u) {
            const int j = base + u * C::KPW + slot;
            if (j < j1) {
                const float p = sc[j - j0];
#pragma unroll
                for (int i = 0; i < C::DPL; ++i) ov[i] = fmaf(p, vf[u][i], ov[i]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < C::DPL; ++i) {
#pragma unroll
        for (int o = 16; o >= C::LPK; o >>= 1) ov[i] += __shfl_xor_sync(0xffffffffu, ov[i], o);
    }
    if (slot == 0) {
#pragma unroll
        for (int i = 0; i < C::DPL; ++i) osum[warp][d0 + i] = ov[i];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < DH; i += blockDim.x) {
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < ATT_WARPS; ++w) s += osum[w][i];
        out[2 + i] = s;
    }
    if (threadIdx.x == 0) {
        out[0] = m;
        out[1] = l;
    }
}

template <int DH>
__global__ void k_attn_combine(AttnArgs a, int nsplit) {
    const int tok = blockIdx.x, h = blockIdx.y;
    const float* p = a.part + ((int64_t)tok * a.H + h) * nsplit * (DH + 2);
    float M = -INFINITY;
    for (int s = 0; s < nsplit; ++s) M = fmaxf(M, p[s * (DH + 2)]);
    float L = 0.f;
    for (int s = 0; s < nsplit; ++s) {
        const float ms = p[s * (DH + 2)];
        if (ms != -INFINITY) L += p[s * (DH + 2) + 1] * expf(ms - M);
    }
    for (int i = threadIdx.x; i < DH; i += blockDim.x) {
        float o = 0.f;
        for (int s = 0; s < nsplit; ++s) {
            const float ms = p[s * (DH + 2)];
            if (ms != -INFINITY) o += p[s * (DH + 2) + 2 + i] * expf(ms - M);
        }
        a.ctx[(int64_t)tok * a.d + h * DH + i] = o / L;
    }
}

int64_t attention_part_floats(int n_tok, int H, int dh, int max_seq) {
    return (int64_t)n_tok * H * ceil_div(max_seq, ATT_KCH) * (dh + 2);
}

template <int DH>
static int run_attn(const AttnArgs& a, int64_t cap, cudaStream_t st) {
    const int nsplit = (int)ceil_div(a.max_pos, ATT_KCH);
    if ((int64_t)a.n_tok * a.H * nsplit * (DH + 2) > cap) {
        set_error("attention workspace too small");
        return PB_ERR_CAPACITY;
    }
    k_attn_split<DH><<<dim3(a.H, a.n_tok, nsplit), ATT_WARPS * 32, 0, st>>>(a, nsplit);
    if (int rc = launch_check("attn_split")) return rc;
    k_attn_combine<DH><<<dim3(a.n_tok, a.H), DH < 128 ? DH : 128, 0, st>>>(a, nsplit);
    return launch_check("attn_combine");
}

int launch_attention(const AttnArgs& a, int64_t cap, cudaStream_t st) {
    switch (a.dh) {
        case 4: return run_attn<4>(a, cap, st);
        case 8: return run_attn<8>(a, cap, st);
        case 16: return run_attn<16>(a, cap, st);
        case 32: return run_attn<32>(a, cap, st);
        case 64: return run_attn<64>(a, cap, st);
        case 128: return run_attn<128>(a, cap, st);
        case 256: return run_attn<256>(a, cap, st);
        default:
            set_error("unsupported head_dim (supported: 4, 8, 16, 32, 64, 128, 256)");
            return PB_ERR_BAD_REQUEST;
    }
}

}  // namespace pb
