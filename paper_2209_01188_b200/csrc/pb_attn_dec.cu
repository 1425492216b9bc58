// Single-query ALiBi attention over the paged fp16 KV cache (model.py:345-361)
// for decode steps (every query group is one position of one session): the
// step the 176B decode and the batched (b = 32) decode run per block.
//
// One query per (session, head) makes this pure K/V streaming (2 flops per
// byte): no tensor cores, no shared-memory ring. CTA c owns one chunk of CS
// 64-key stages of one (group, head) (cta_base[g] prefix, host-built), 4 warps
// x 16 keys per stage, the chunk's K and V rows read straight from HBM into
// registers: lane l owns DH/32 dims, so a warp's 32 lanes read one 256-B key
// row (the rows' 16-B chunks are XOR-swizzled by slot & 7 by the QKV
// epilogue). Scores in f32 with the f32 query (16 per warp, butterfly-reduced
// across lanes), ALiBi bias, online softmax per warp, P.V in f32; warps merge
// in smem, chunks of a (group, head) merge in chunk order through the split
// workspace (last contributor), which writes ctx and max|ctx s_wo| for the wo
// operand (atomicMax). Many small CTAs (16 per SM) keep ~400 KB of loads in
// flight per SM without a pipeline to manage.
#include <algorithm>

#include "pb_attn_common.cuh"
#include "pb_common.cuh"
#include "pb_span.h"

namespace pb {

constexpr int AD_WARPS = 4;

template <int DH>
__global__ void __launch_bounds__(AD_WARPS * 32) k_attn_dec(AttnArgs a, const int64_t* __restrict__ cta_base, int CS) {
    constexpr int DPL = DH / 32;  // dims per lane (4 or 2)
    __shared__ float wst[AD_WARPS][DH + 2];
    __shared__ int s_last;
    __shared__ float s_red[AD_WARPS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t c = blockIdx.x;
    // (group, head, chunk) of this CTA
    int lo = 0, hi = a.n_groups - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (cta_base[mid] <= c) lo = mid;
        else hi = mid - 1;
    }
    const int g = lo;
    const int nch = (int)((cta_base[g + 1] - cta_base[g]) / a.H);
    const int r = (int)(c - cta_base[g]);
    const int h = r / nch, ch = r - h * nch;

    pdl_wait();  // q and the newest key come from the QKV GEMV
    pdl_trigger();
    const int tok = a.grp_first[g];
    const int pos = a.tok_pos[tok];
    const int32_t* pt = a.pages + (int64_t)a.tok_seq[tok] * a.max_pages;
    const int kbeg = ch * CS * AM_SK, kend = min(pos + 1, (ch + 1) * CS * AM_SK);
    const float isq = 1.0f / sqrtf((float)DH);
    const float slope = a.slopes[h];
    float q[DPL];
    {
        const float* qp = a.q + (int64_t)tok * a.d + h * DH + lane * DPL;
#pragma unroll
        for (int e = 0; e < DPL; ++e) q[e] = qp[e] * isq;
    }
    // this lane's dims live in 16-B chunk (lane DPL) / 8 at byte (lane DPL % 8) * 2
    const int lchunk = (lane * DPL) >> 3, loff = (lane * DPL) & 7;
    const int64_t head_off = (int64_t)h * a.P * DH;
    const int64_t kv_stride = (int64_t)a.H * a.P * DH;
    float m_run = -INFINITY, l_run = 0.f, acc[DPL];
#pragma unroll
    for (int e = 0; e < DPL; ++e) acc[e] = 0.f;

    for (int kb = kbeg + warp * 16; kb < kend; kb += AD_WARPS * 16) {
        // 16 consecutive keys share one page (16 | P)
        const int page = pt[kb / a.P];
        const half* kbase = a.kv + (int64_t)page * 2 * kv_stride + head_off;
        const int n = min(16, kend - kb);
        uint2 kr[16], vr[16];  // DPL = 4: 4 halves per row and lane (uint2); DPL = 2: 2 halves (.x)
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (j < n) {
                const int slot = (kb + j) % a.P;
                const half* row = kbase + (int64_t)slot * DH + (((lchunk ^ (slot & 7)) << 3) | loff);
                if (DPL == 4) {
                    kr[j] = __ldcs(reinterpret_cast<const uint2*>(row));
                    vr[j] = __ldcs(reinterpret_cast<const uint2*>(row + kv_stride));
                } else {
                    kr[j].x = __ldcs(reinterpret_cast<const unsigned int*>(row));
                    vr[j].x = __ldcs(reinterpret_cast<const unsigned int*>(row + kv_stride));
                }
            }
        }
        float s[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const half2 k01 = *reinterpret_cast<const half2*>(&kr[j].x);
            float d = q[0] * __low2float(k01) + q[1] * __high2float(k01);
            if (DPL == 4) {
                const half2 k23 = *reinterpret_cast<const half2*>(&kr[j].y);
                d += q[2] * __low2float(k23) + q[3] * __high2float(k23);
            }
            s[j] = d;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int j = 0; j < 16; ++j) s[j] += __shfl_xor_sync(0xffffffffu, s[j], o);
        float mx = m_run;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            s[j] = j < n ? s[j] + slope * (float)(kb + j - pos) : -INFINITY;
            mx = fmaxf(mx, s[j]);
        }
        const float corr = m_run == -INFINITY ? 0.f : expf(m_run - mx);
        l_run *= corr;
#pragma unroll
        for (int e = 0; e < DPL; ++e) acc[e] *= corr;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (j < n) {
                const float p = expf(s[j] - mx);
                l_run += p;
                const half2 v01 = *reinterpret_cast<const half2*>(&vr[j].x);
                acc[0] = fmaf(p, __low2float(v01), acc[0]);
                acc[1] = fmaf(p, __high2float(v01), acc[1]);
                if (DPL == 4) {
                    const half2 v23 = *reinterpret_cast<const half2*>(&vr[j].y);
                    acc[2] = fmaf(p, __low2float(v23), acc[2]);
                    acc[3] = fmaf(p, __high2float(v23), acc[3]);
                }
            }
        }
        m_run = mx;
    }
    // ---- merge the warps (fixed order): this chunk's (M, L, O)
    if (lane == 0) {
        wst[warp][0] = m_run;
        wst[warp][1] = l_run;
    }
#pragma unroll
    for (int e = 0; e < DPL; ++e) wst[warp][2 + lane * DPL + e] = acc[e];
    __syncthreads();
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < AD_WARPS; ++w) M = fmaxf(M, wst[w][0]);
    float sw[AD_WARPS], L = 0.f;
#pragma unroll
    for (int w = 0; w < AD_WARPS; ++w) {
        sw[w] = wst[w][0] == -INFINITY ? 0.f : expf(wst[w][0] - M);
        L += wst[w][1] * sw[w];
    }
    const int e = threadIdx.x;  // one output dim per thread (DH <= 128)
    float o = 0.f;
    if (e < DH) {
#pragma unroll
        for (int w = 0; w < AD_WARPS; ++w) o += wst[w][2 + e] * sw[w];
    }
    bool fin = nch == 1;
    if (!fin) {
        float* pp = a.part + ((int64_t)tok * a.H + h) * AM_MAXC * (DH + 2);
        float* out = pp + ch * (DH + 2);
        if (e < DH) out[2 + e] = o;
        if (e == 0) {
            out[0] = M;
            out[1] = L;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            int* ctr = a.counters + (int64_t)tok * a.H + h;
            const int last = atomicAdd(ctr, 1) == nch - 1;
            if (last) *ctr = 0;
            s_last = last;
        }
        __syncthreads();
        if (!s_last) return;
        __threadfence();
        M = -INFINITY;
        for (int s2 = 0; s2 < nch; ++s2) M = fmaxf(M, __ldcg(pp + s2 * (DH + 2)));
        L = 0.f;
        o = 0.f;
        for (int s2 = 0; s2 < nch; ++s2) {
            const float ms = __ldcg(pp + s2 * (DH + 2));
            const float f = ms == -INFINITY ? 0.f : expf(ms - M);
            L += __ldcg(pp + s2 * (DH + 2) + 1) * f;
            if (e < DH) o += __ldcg(pp + s2 * (DH + 2) + 2 + e) * f;
        }
        fin = true;
    }
    // ---- finalize: ctx and the wo operand range max |ctx s_wo| of this head
    float mloc = 0.f;
    if (e < DH) {
        const float cx = o / L;
        a.ctx[(int64_t)tok * a.d + h * DH + e] = cx;
        if (a.tokmax) mloc = fabsf(cx * a.s_next[h * DH + e]);
    }
    if (a.tokmax) {
        mloc = warp_max(mloc);
        if (lane == 0) s_red[warp] = mloc;
        __syncthreads();
        if (threadIdx.x == 0) {
            float m2 = s_red[0];
#pragma unroll
            for (int w = 1; w < AD_WARPS; ++w) m2 = fmaxf(m2, s_red[w]);
            if (m2 > 0.f) atomicMax(reinterpret_cast<int*>(a.tokmax) + tok, __float_as_int(m2));
        }
    }
}

int run_attn_dec(const AttnArgs& a, const int64_t* d_cta_base, int64_t n_ctas, int cs, int64_t cap, cudaStream_t st) {
    if ((int64_t)a.n_tok * a.H * AM_MAXC * (a.dh + 2) > cap) {
        set_error("attention workspace too small");
        return PB_ERR_CAPACITY;
    }
    if (n_ctas <= 0) return PB_OK;
    if (a.dh == 128)
        return launch_pdl(k_attn_dec<128>, dim3((unsigned)n_ctas), dim3(AD_WARPS * 32), 0, st, a, d_cta_base, cs);
    if (a.dh == 64)
        return launch_pdl(k_attn_dec<64>, dim3((unsigned)n_ctas), dim3(AD_WARPS * 32), 0, st, a, d_cta_base, cs);
    set_error("k_attn_dec: head_dim 64 or 128");
    return PB_ERR_GENERIC;
}

}  // namespace pb
