// ALiBi causal attention over the paged fp16 KV cache (model.py:345-361).
//
// scores[h, i, j] = fl(fl(q_i . k_j / f32(sqrt(dh))) + fl(slope_h * (j - pos_i))),
// masked for j > pos_i, max-subtracted softmax, then P V. Every query token
// carries its own sequence and absolute position, so decode (t = 1 per
// session, many sessions) and prefill (t > 1) share one kernel.
//
// Split-T (flash-decoding): CTA = (head, query token, key chunk of 128).
// The chunk's K and V rows are contiguous within each KV page (pool layout
// [page][K|V][H][P][dh]), so one elected thread moves them HBM -> shared
// memory with cp.async.bulk (TMA engine) on an mbarrier: the whole 64 KB
// chunk (dh = 128) is in flight at once, instead of a few 16-byte loads per
// lane. Scores are computed from shared memory with dh/8 lanes per key
// (8 dims each, shuffle reduction), kept in shared memory for an exact
// two-pass chunk softmax, then P V. The last CTA of each (token, head) to
// finish merges the chunk partials in chunk order (max/sum rescaling) and
// writes ctx -- no separate combine launch, deterministic.
#include "pb_async.cuh"
#include "pb_common.cuh"
#include "pb_span.h"

namespace pb {

constexpr int ATT_KCH = 128;  // keys per CTA
constexpr int ATT_WARPS = 4;

template <int DH>
struct AttnCfg {
    static constexpr int DPL = DH < 8 ? DH : 8;  // dims per lane
    static constexpr int LPK = DH / DPL;         // lanes per key
    static constexpr int KPW = 32 / LPK;         // keys per warp iteration
    static constexpr bool BULK = (DH * 2) % 16 == 0;
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
constexpr size_t attn_smem() {
    return (size_t)2 * ATT_KCH * DH * 2 + ATT_KCH * 4 + ATT_WARPS * DH * 4 + 64;
}

template <int DH>
__global__ void __launch_bounds__(ATT_WARPS * 32) k_attn(AttnArgs a, int nsplit) {
    using C = AttnCfg<DH>;
    extern __shared__ __align__(128) uint8_t smem[];
    half* Ks = reinterpret_cast<half*>(smem);                     // [KCH][DH]
    half* Vs = Ks + ATT_KCH * DH;                                 // [KCH][DH]
    float* sc = reinterpret_cast<float*>(Vs + ATT_KCH * DH);      // [KCH]
    float* osum = sc + ATT_KCH;                                   // [WARPS][DH]
    float* red = osum + ATT_WARPS * DH;                           // [WARPS]
    uint64_t* bar = reinterpret_cast<uint64_t*>(red + 8);
    int* s_flag = reinterpret_cast<int*>(bar + 1);

    const int h = blockIdx.x, tok = blockIdx.y, split = blockIdx.z;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int pos = a.tok_pos[tok], seq = a.tok_seq[tok];
    const int j0 = split * ATT_KCH;
    const int j1 = min(j0 + ATT_KCH, pos + 1);
    float* out = a.part + (((int64_t)tok * a.H + h) * nsplit + split) * (DH + 2);
    const int32_t* pt = a.pages + (int64_t)seq * a.max_pages;
    const int64_t head_off = (int64_t)h * a.P * DH;
    const int64_t kv_stride = (int64_t)a.H * a.P * DH;  // K -> V within a page

    if (j0 < j1) {
        // ---- stage the chunk's K and V rows in shared memory
        if constexpr (C::BULK) {
            if (threadIdx.x == 0) {
                mbar_init(bar, 1);
                mbar_fence_init();
                mbar_expect_tx(bar, (uint32_t)(j1 - j0) * DH * 2 * 2);
                for (int j = j0; j < j1;) {
                    const int page = pt[j / a.P];
                    const int jn = min(j1, (j / a.P + 1) * a.P);
                    const half* kp = a.kv + (int64_t)page * 2 * kv_stride + head_off + (int64_t)(j % a.P) * DH;
                    const uint32_t bytes = (uint32_t)(jn - j) * DH * 2;
                    bulk_g2s(Ks + (j - j0) * DH, kp, bytes, bar);
                    bulk_g2s(Vs + (j - j0) * DH, kp + kv_stride, bytes, bar);
                    j = jn;
                }
            }
        } else {
            for (int i = threadIdx.x; i < (j1 - j0) * DH; i += blockDim.x) {
                const int j = j0 + i / DH, dd = i % DH;
                const half* kp = a.kv + (int64_t)pt[j / a.P] * 2 * kv_stride + head_off + (int64_t)(j % a.P) * DH + dd;
                Ks[i] = kp[0];
                Vs[i] = kp[kv_stride];
            }
        }
        const int sub = lane % C::LPK, slot = lane / C::LPK;
        const int d0 = sub * C::DPL;
        float qv[C::DPL];
#pragma unroll
        for (int i = 0; i < C::DPL; ++i) qv[i] = a.q[(int64_t)tok * a.d + h * DH + d0 + i];
        const float sq = (float)sqrt((double)DH);
        const float slope = a.slopes[h];
        __syncthreads();
        if constexpr (C::BULK) mbar_wait(bar, 0);

        // ---- scores
        for (int base = j0 + warp * C::KPW; base < j1; base += ATT_WARPS * C::KPW) {
            const int j = base + slot;
            float dot = 0.f;
            if (j < j1) {
                float kf[C::DPL];
                load_h<C::DPL>(Ks + (j - j0) * DH + d0, kf);
#pragma unroll
                for (int i = 0; i < C::DPL; ++i) dot = fmaf(qv[i], kf[i], dot);
            }
#pragma unroll
            for (int o = C::LPK / 2; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
            if (j < j1 && sub == 0) sc[j - j0] = __fadd_rn(__fdiv_rn(dot, sq), __fmul_rn(slope, (float)(j - pos)));
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

        // ---- P V
        float ov[C::DPL];
#pragma unroll
        for (int i = 0; i < C::DPL; ++i) ov[i] = 0.f;
        for (int base = j0 + warp * C::KPW; base < j1; base += ATT_WARPS * C::KPW) {
            const int j = base + slot;
            if (j < j1) {
                float vf[C::DPL];
                load_h<C::DPL>(Vs + (j - j0) * DH + d0, vf);
                const float p = sc[j - j0];
#pragma unroll
                for (int i = 0; i < C::DPL; ++i) ov[i] = fmaf(p, vf[i], ov[i]);
            }
        }
#pragma unroll
        for (int i = 0; i < C::DPL; ++i) {
#pragma unroll
            for (int o = 16; o >= C::LPK; o >>= 1) ov[i] += __shfl_xor_sync(0xffffffffu, ov[i], o);
        }
        if (slot == 0) {
#pragma unroll
            for (int i = 0; i < C::DPL; ++i) osum[warp * DH + d0 + i] = ov[i];
        }
        __syncthreads();
        for (int i = threadIdx.x; i < DH; i += blockDim.x) {
            float s = 0.f;
#pragma unroll
            for (int w = 0; w < ATT_WARPS; ++w) s += osum[w * DH + i];
            out[2 + i] = s;
        }
        if (threadIdx.x == 0) {
            out[0] = m;
            out[1] = l;
        }
    } else if (threadIdx.x == 0) {  // chunk entirely in the causal future
        out[0] = -INFINITY;
        out[1] = 0.f;
    }

    // ---- last CTA of (token, head) merges the chunks in chunk order
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        int* ctr = a.counters + (int64_t)tok * a.H + h;
        const int prev = atomicAdd(ctr, 1);
        const int last = prev == nsplit - 1;
        if (last) *ctr = 0;
        *s_flag = last;
    }
    __syncthreads();
    if (!*s_flag) return;
    __threadfence();
    const float* p = a.part + ((int64_t)tok * a.H + h) * nsplit * (DH + 2);
    float M = -INFINITY;
    for (int s = 0; s < nsplit; ++s) M = fmaxf(M, __ldcg(p + s * (DH + 2)));
    float L = 0.f;
    for (int s = 0; s < nsplit; ++s) {
        const float ms = __ldcg(p + s * (DH + 2));
        if (ms != -INFINITY) L += __ldcg(p + s * (DH + 2) + 1) * expf(ms - M);
    }
    float mloc = 0.f;
    for (int i = threadIdx.x; i < DH; i += blockDim.x) {
        float o = 0.f;
        for (int s = 0; s < nsplit; ++s) {
            const float ms = __ldcg(p + s * (DH + 2));
            if (ms != -INFINITY) o += __ldcg(p + s * (DH + 2) + 2 + i) * expf(ms - M);
        }
        const float c = o / L;
        a.ctx[(int64_t)tok * a.d + h * DH + i] = c;
        if (a.tokmax) mloc = fmaxf(mloc, fabsf(c * a.s_next[h * DH + i]));
    }
    if (a.tokmax) {  // operand range of the wo GEMV (exact, order-independent max)
        mloc = warp_max(mloc);
        if (lane == 0) red[warp] = mloc;
        __syncthreads();
        if (threadIdx.x == 0) {
            float m = red[0];
#pragma unroll
            for (int w = 1; w < ATT_WARPS; ++w) m = fmaxf(m, red[w]);
            atomicMax(reinterpret_cast<int*>(a.tokmax) + tok, __float_as_int(m));
        }
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
    constexpr size_t smem = attn_smem<DH>();
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_attn<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
    k_attn<DH><<<dim3(a.H, a.n_tok, nsplit), ATT_WARPS * 32, smem, st>>>(a, nsplit);
    return launch_check("attention");
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
