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

constexpr int ATT_SK = 32;    // keys per pipeline stage
constexpr int ATT_ST = 4;     // stages in flight (TMA ring)
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
    // K, V ring + per-warp (m, l, o) + reduction scratch + barriers
    return (size_t)ATT_ST * 2 * ATT_SK * DH * 2 + (size_t)ATT_WARPS * (DH + 2) * 4 + 8 * 4 + 2 * ATT_ST * 8 + 64;
}

// Producer side of stage i: keys [k0, k1) of this CTA's range into ring slot i % ST.
template <int DH, bool BULK>
__device__ __forceinline__ void attn_fill(const AttnArgs& a, const int32_t* pt, int64_t head_off, int64_t kv_stride,
                                          int k0, int k1, half* Kb, half* Vb, uint64_t* bar, int lane) {
    if constexpr (BULK) {
        if (lane == 0) {
            mbar_expect_tx(bar, (uint32_t)(k1 - k0) * DH * 2 * 2);
            for (int j = k0; j < k1;) {
                const int page = pt[j / a.P];
                const int jn = min(k1, (j / a.P + 1) * a.P);
                const half* kp = a.kv + (int64_t)page * 2 * kv_stride + head_off + (int64_t)(j % a.P) * DH;
                const uint32_t bytes = (uint32_t)(jn - j) * DH * 2;
                bulk_g2s(Kb + (j - k0) * DH, kp, bytes, bar);
                bulk_g2s(Vb + (j - k0) * DH, kp + kv_stride, bytes, bar);
                j = jn;
            }
        }
    } else {
        for (int e = lane; e < (k1 - k0) * DH; e += 32) {
            const int j = k0 + e / DH, dd = e % DH;
            const half* kp = a.kv + (int64_t)pt[j / a.P] * 2 * kv_stride + head_off + (int64_t)(j % a.P) * DH + dd;
            Kb[e] = kp[0];
            Vb[e] = kp[kv_stride];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(bar);
    }
}

// Split-T decode/prefill attention. CTA = (head, query token, key split);
// warp 4 streams the split's K/V rows page piece by page piece into a 4-stage
// smem ring (cp.async.bulk, mbarrier complete_tx); warps 0-3 each own a
// quarter of every stage and keep their own online-softmax state (no CTA-wide
// barrier per stage), releasing the slot with an mbarrier arrive. The four
// warp states are merged at the end, then the last CTA of (token, head)
// merges the splits in split order.
template <int DH>
__global__ void __launch_bounds__((ATT_WARPS + 1) * 32) k_attn(AttnArgs a, int nsplit, int kps) {
    using C = AttnCfg<DH>;
    constexpr int KW = ATT_SK / ATT_WARPS;  // keys per warp per stage
    constexpr int IT = (KW + C::KPW - 1) / C::KPW;
    extern __shared__ __align__(128) uint8_t smem[];
    half* Ks = reinterpret_cast<half*>(smem);                                // [ST][SK][DH]
    half* Vs = Ks + ATT_ST * ATT_SK * DH;                                    // [ST][SK][DH]
    float* wst = reinterpret_cast<float*>(Vs + ATT_ST * ATT_SK * DH);        // [WARPS][DH + 2]
    float* red = wst + ATT_WARPS * (DH + 2);                                 // [8]
    uint64_t* full = reinterpret_cast<uint64_t*>(red + 8);                   // [ST]
    uint64_t* empty = full + ATT_ST;                                         // [ST]
    int* s_flag = reinterpret_cast<int*>(empty + ATT_ST);

    const int h = blockIdx.x, tok = blockIdx.y, split = blockIdx.z;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int pos = a.tok_pos[tok], seq = a.tok_seq[tok];
    const int j0 = split * kps;
    const int j1 = min(j0 + kps, pos + 1);
    float* out = a.part + (((int64_t)tok * a.H + h) * nsplit + split) * (DH + 2);
    const int32_t* pt = a.pages + (int64_t)seq * a.max_pages;
    const int64_t head_off = (int64_t)h * a.P * DH;
    const int64_t kv_stride = (int64_t)a.H * a.P * DH;  // K -> V within a page
    const int nst = j0 < j1 ? (j1 - j0 + ATT_SK - 1) / ATT_SK : 0;

    if (threadIdx.x == 0) {
        for (int b = 0; b < ATT_ST; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&empty[b], ATT_WARPS);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (warp == ATT_WARPS) {
        // ---------------- producer warp
        // In a pure decode step the keys before each query's own position were
        // written by earlier steps: stream them while the QKV GEMV (PDL
        // predecessor) is still finishing; wait before the newest key.
        const int safe_end = a.decode_only ? pos : j0;
        bool waited = false;
        for (int i = 0; i < nst; ++i) {
            const int b = i % ATT_ST;
            mbar_wait(&empty[b], ((i / ATT_ST) & 1) ^ 1);
            const int k0 = j0 + i * ATT_SK;
            const int k1 = min(j1, k0 + ATT_SK);
            if (!waited && k1 > safe_end) {
                pdl_wait();
                pdl_trigger();
                waited = true;
            }
            attn_fill<DH, C::BULK>(a, pt, head_off, kv_stride, k0, k1, Ks + b * ATT_SK * DH, Vs + b * ATT_SK * DH,
                                   &full[b], lane);
        }
        if (!waited) {
            pdl_wait();
            pdl_trigger();
        }
    } else {
        // ---------------- compute warps
        pdl_wait();
        pdl_trigger();
        const int sub = lane % C::LPK, slot = lane / C::LPK;
        const int d0 = sub * C::DPL;
        float qv[C::DPL];
#pragma unroll
        for (int e = 0; e < C::DPL; ++e) qv[e] = a.q[(int64_t)tok * a.d + h * DH + d0 + e];
        const float sq = (float)sqrt((double)DH);
        const float slope = a.slopes[h];
        float m_run = -INFINITY, l_run = 0.f;
        float ov[C::DPL];
#pragma unroll
        for (int e = 0; e < C::DPL; ++e) ov[e] = 0.f;
        for (int i = 0; i < nst; ++i) {
            const int b = i % ATT_ST;
            const int k0 = j0 + i * ATT_SK;
            const int nk = min(ATT_SK, j1 - k0);
            mbar_wait(&full[b], (i / ATT_ST) & 1);
            const half* Kb = Ks + b * ATT_SK * DH;
            const half* Vb = Vs + b * ATT_SK * DH;
            float s[IT];
            float smax = -INFINITY;
#pragma unroll
            for (int it = 0; it < IT; ++it) {
                const int jj = warp * KW + it * C::KPW + slot;
                const bool ok = jj < nk && (it * C::KPW + slot) < KW;
                float dot = 0.f;
                if (ok) {
                    float kf[C::DPL];
                    load_h<C::DPL>(Kb + jj * DH + d0, kf);
#pragma unroll
                    for (int e = 0; e < C::DPL; ++e) dot = fmaf(qv[e], kf[e], dot);
                }
#pragma unroll
                for (int o = C::LPK / 2; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
                s[it] = ok ? __fadd_rn(__fdiv_rn(dot, sq), __fmul_rn(slope, (float)(k0 + jj - pos))) : -INFINITY;
                smax = fmaxf(smax, s[it]);
            }
#pragma unroll
            for (int o = 16; o >= C::LPK; o >>= 1) smax = fmaxf(smax, __shfl_xor_sync(0xffffffffu, smax, o));
            const float m_new = fmaxf(m_run, smax);
            if (m_new != -INFINITY) {
                const float alpha = m_run == -INFINITY ? 0.f : expf(__fsub_rn(m_run, m_new));
                float ls = 0.f;
#pragma unroll
                for (int e = 0; e < C::DPL; ++e) ov[e] *= alpha;
#pragma unroll
                for (int it = 0; it < IT; ++it) {
                    const int jj = warp * KW + it * C::KPW + slot;
                    if (s[it] != -INFINITY) {
                        const float p = expf(__fsub_rn(s[it], m_new));
                        ls += p;
                        float vf[C::DPL];
                        load_h<C::DPL>(Vb + jj * DH + d0, vf);
#pragma unroll
                        for (int e = 0; e < C::DPL; ++e) ov[e] = fmaf(p, vf[e], ov[e]);
                    }
                }
#pragma unroll
                for (int o = 16; o >= C::LPK; o >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o);
                l_run = l_run * alpha + ls;
                m_run = m_new;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[b]);
        }
        // per-warp state -> smem (dims reduced over the key slots)
#pragma unroll
        for (int e = 0; e < C::DPL; ++e) {
#pragma unroll
            for (int o = 16; o >= C::LPK; o >>= 1) ov[e] += __shfl_xor_sync(0xffffffffu, ov[e], o);
        }
        float* w = wst + warp * (DH + 2);
        if (slot == 0) {
#pragma unroll
            for (int e = 0; e < C::DPL; ++e) w[2 + d0 + e] = ov[e];
        }
        if (lane == 0) {
            w[0] = m_run;
            w[1] = l_run;
        }
    }
    __syncthreads();
    {  // merge the 4 warp states of this split (fixed order)
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < ATT_WARPS; ++w) M = fmaxf(M, wst[w * (DH + 2)]);
    float L = 0.f;
    float sc[ATT_WARPS];
#pragma unroll
    for (int w = 0; w < ATT_WARPS; ++w) {
        const float mw = wst[w * (DH + 2)];
        sc[w] = mw == -INFINITY ? 0.f : expf(mw - M);
        L += wst[w * (DH + 2) + 1] * sc[w];
    }
    for (int e = threadIdx.x; e < DH; e += blockDim.x) {
        float o = 0.f;
#pragma unroll
        for (int w = 0; w < ATT_WARPS; ++w) o += wst[w * (DH + 2) + 2 + e] * sc[w];
        out[2 + e] = o;
    }
    if (threadIdx.x == 0) {
        out[0] = M;
        out[1] = L;
    }
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
            for (int w = 1; w <= ATT_WARPS; ++w) m = fmaxf(m, red[w]);
            atomicMax(reinterpret_cast<int*>(a.tokmax) + tok, __float_as_int(m));
        }
    }
}

constexpr int ATT_MAX_SPLIT = 16;

int64_t attention_part_floats(int n_tok, int H, int dh, int max_seq) {
    return (int64_t)n_tok * H * ATT_MAX_SPLIT * (dh + 2);
}

template <int DH>
static int run_attn(const AttnArgs& a, int64_t cap, cudaStream_t st) {
    // split the key range only as far as needed to cover the machine (~2 CTAs
    // per SM); each split streams >= 4 stages
    const int sms = sm_count();
    if (sms < 0) return PB_ERR_GENERIC;
    constexpr int ctas_per_sm = 2;
    int nsplit = (int)ceil_div((int64_t)ctas_per_sm * sms, (int64_t)a.n_tok * a.H);
    nsplit = std::max(1, std::min<int>(nsplit, std::min<int>(ATT_MAX_SPLIT, (int)ceil_div(a.max_pos, 4 * ATT_SK))));
    const int kps = (int)round_up(ceil_div(a.max_pos, nsplit), ATT_SK);
    nsplit = (int)ceil_div(a.max_pos, kps);
    if ((int64_t)a.n_tok * a.H * nsplit * (DH + 2) > cap) {
        set_error("attention workspace too small");
        return PB_ERR_CAPACITY;
    }
    constexpr size_t smem = attn_smem<DH>();
    static int ok[PB_MAX_DEVICES] = {};
    if (per_device(ok, [](int) {
            return cudaFuncSetAttribute(k_attn<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) ==
                           cudaSuccess ? 1 : -1;
        }) < 0)
        return launch_check("attn setup");
    return launch_pdl(k_attn<DH>, dim3(a.H, a.n_tok, nsplit), dim3((ATT_WARPS + 1) * 32), smem, st, a, nsplit, kps);
}

int launch_attention(const AttnArgs& a, int64_t cap, cudaStream_t st) {
    if (a.dh == 64) return run_attn_mma<64>(a, a.n_groups, cap, st);
    if (a.dh == 128) return run_attn_mma<128>(a, a.n_groups, cap, st);
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
