// Tensor-core ALiBi attention over the paged fp16 KV cache (model.py:345-361)
// for head_dim 64 / 128: decode (one query per session) and prefill (up to 8
// consecutive queries of one sequence per CTA, so K/V are read once per group).
//
// Stream-K grid (see k_attn_mma): each CTA owns an equal run of (query group,
// head, 64-key stage) units; warp 4 streams their K/V rows (page pieces,
// cp.async.bulk on an mbarrier ring of 64-key stages); each of warps 0-3 owns
// 16 keys of every stage and keeps its own online softmax:
//   S = [Q_hi; Q_lo] K^T   mma.m16n8k16: rows g = query g hi, g+8 = query g lo
//                          (fp32-accurate scores: q split hi/lo, K exact fp16),
//                          K fragments via ldmatrix (B operand = K row-major);
//   P = exp(S - m)         in registers; the S accumulator layout IS the A
//                          fragment layout of P (FlashAttention-2 register
//                          reuse), split again into hi (rows g) / lo (rows g+8);
//   O += [P_hi; P_lo] V    V fragments via ldmatrix.trans.
// The KV cache rows are stored with their 16-byte chunks XOR-swizzled by
// (slot & 7) (written that way by the QKV epilogue), so the ldmatrix row
// gathers are bank-conflict free after a linear bulk copy.
// The pieces of a (group, head) split across CTAs are merged in CTA order by
// the last contributor.
#include <algorithm>

#include "pb_async.cuh"
#include "pb_attn_common.cuh"
#include "pb_common.cuh"
#include "pb_span.h"

namespace pb {

template <int DH, int ST, int CW>
constexpr size_t attn_mma_smem() {
    return (size_t)ST * 2 * AM_SK * DH * 2 + (size_t)CW * AM_G * (DH + 2) * 4 + 2 * ST * 8 + 64 +
           4 * AM_PT;
}

template <int DH, int ST, int CW>
__global__ void __launch_bounds__((CW + 1) * 32) k_attn_mma(AttnArgs a, int G, int64_t U) {
    // CW = 4: four compute warps, 16 keys of every stage each. CW = 8 (one CTA per SM):
    // two groups of four warps take alternate stages (more warps per SM hide the
    // per-stage MMA / softmax latency); each warp keeps its own online softmax.
    constexpr int GW = CW > 4 ? 4 : CW;  // warps per stage
    constexpr int NKT = DH / 16;  // k-steps of S
    constexpr int NNT = DH / 8;   // n-tiles of O
    constexpr int ROWB = DH * 2;  // bytes per K/V row
    extern __shared__ __align__(128) uint8_t smem[];
    half* Ks = reinterpret_cast<half*>(smem);                         // [ST][SK][DH]
    half* Vs = Ks + ST * AM_SK * DH;                               // [ST][SK][DH]
    float* wst = reinterpret_cast<float*>(Vs + ST * AM_SK * DH);   // [WARPS][G][DH + 2]
    uint64_t* full = reinterpret_cast<uint64_t*>(wst + CW * AM_G * (DH + 2));
    uint64_t* empty = full + ST;
    int* s_flag = reinterpret_cast<int*>(empty + ST);

    const int c = blockIdx.x;
    const int64_t u0 = (int64_t)c * U / G, u1 = (int64_t)(c + 1) * U / G;
    const int lane = threadIdx.x & 31, warp = warp_uniform_id();
    const int64_t kv_stride = (int64_t)a.H * a.P * DH;

    if (threadIdx.x == 0) {
        trace_stamp(a.trace, c, 0);
        for (int b = 0; b < ST; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&empty[b], GW);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (warp == CW) {
        // ---------------- producer warp: K/V page pieces of every stage of the range.
        // The segment's page-table entries are staged in shared memory first
        // (one coalesced load), so issuing a stage never waits on a global load.
        // In a pure decode step the keys before each query's own position were
        // written by earlier steps: stream them while the QKV GEMV (PDL
        // predecessor) is still finishing; wait before the newest key.
        int* s_pages = reinterpret_cast<int*>(s_flag + 4);  // [AM_PT]
        bool waited = false;
        int it = 0;
        for (int64_t u = u0; u < u1;) {
            const AmSeg sg = am_seg(a, u, u1);
            const int t0 = a.grp_first[sg.g], nq = a.grp_count[sg.g];
            const int pos0 = a.tok_pos[t0];
            const int jend = pos0 + nq;  // keys [0, jend)
            const int safe_end = a.decode_only ? pos0 : 0;
            const int32_t* pt = a.pages + (int64_t)a.tok_seq[t0] * a.max_pages;
            const int64_t head_off = (int64_t)sg.h * a.P * DH;
            int pbase = -1 << 30;  // first page index held in s_pages
            for (int i = sg.i0; i < sg.i0 + sg.n; ++i, ++it) {
                const int k0 = i * AM_SK;
                const int k1 = min(jend, k0 + AM_SK);
                if ((k1 - 1) / a.P >= pbase + AM_PT) {  // refill the page window
                    __syncwarp();
                    pbase = k0 / a.P;
                    const int plast = (min(jend, (sg.i0 + sg.n) * AM_SK) - 1) / a.P;
                    for (int p = lane; p < AM_PT && pbase + p <= plast; p += 32) s_pages[p] = pt[pbase + p];
                    __syncwarp();
                }
                const int b = it % ST;
                mbar_wait(&empty[b], ((it / ST) & 1) ^ 1);
                if (!waited && k1 > safe_end) {
                    pdl_wait();
                    pdl_trigger();
                    waited = true;
                }
                if (lane == 0) {
                    mbar_expect_tx(&full[b], (uint32_t)(k1 - k0) * ROWB * 2);
                    for (int j = k0; j < k1;) {
                        const int page = s_pages[j / a.P - pbase];
                        const int jn = min(k1, (j / a.P + 1) * a.P);
                        const half* kp = a.kv + (int64_t)page * 2 * kv_stride + head_off + (int64_t)(j % a.P) * DH;
                        const uint32_t bytes = (uint32_t)(jn - j) * ROWB;
                        bulk_g2s(Ks + ((int64_t)b * AM_SK + (j - k0)) * DH, kp, bytes, &full[b]);
                        bulk_g2s(Vs + ((int64_t)b * AM_SK + (j - k0)) * DH, kp + kv_stride, bytes, &full[b]);
                        j = jn;
                    }
                }
            }
            u += sg.n;
        }
        if (!waited) {
            pdl_wait();
            pdl_trigger();
        }
        return;
    }

    // ---------------- compute warps: the step constants of the first head (the next matmul's
    // scales read by the finish, the ALiBi slope) into L1 while the predecessor drains
    if (u0 < u1) {
        const AmSeg s0 = am_seg(a, u0, u1);
        if (a.tokmax && threadIdx.x < DH) prefetch_l1(a.s_next + s0.h * DH + threadIdx.x);
        if (threadIdx.x == 0) prefetch_l1(a.slopes + s0.h);
    }
    pdl_wait();
    pdl_trigger();
    if (threadIdx.x == 32) trace_stamp(a.trace, c, 1);
    const int g = lane >> 2, qd = lane & 3;
    const uint32_t ks_base = smem_u32(Ks), vs_base = smem_u32(Vs);
    const int mi = lane >> 3, ri = lane & 7;  // ldmatrix lane roles: matrix mi, row ri
    const float isq = 1.0f / sqrtf((float)DH);
    int it = 0, nseg = 0;
    for (int64_t u = u0; u < u1; ++nseg) {
        const AmSeg sg = am_seg(a, u, u1);
        const int h = sg.h;
        if (threadIdx.x == 32 && nseg < 2) trace_stamp(a.trace, c, 5 + 3 * nseg);  // diagnostics: segment start
        const int t0 = a.grp_first[sg.g], nq = a.grp_count[sg.g];
        const int pos0 = a.tok_pos[t0];
        const int j1 = pos0 + nq;
        const bool qv = g < nq;
        const int my_pos = pos0 + g;
        // Q fragments (A operand): rows g (hi) / g+8 (lo) of query g, scaled by 1/sqrt(dh)
        uint32_t qa[NKT][4];
        {
            const float* q = a.q + (int64_t)(t0 + (qv ? g : 0)) * a.d + h * DH;
#pragma unroll
            for (int ks = 0; ks < NKT; ++ks) {
                float x0 = 0.f, x1 = 0.f, x2 = 0.f, x3 = 0.f;
                if (qv) {
                    const float2 v01 = *reinterpret_cast<const float2*>(q + ks * 16 + 2 * qd);
                    const float2 v23 = *reinterpret_cast<const float2*>(q + ks * 16 + 2 * qd + 8);
                    x0 = v01.x * isq;
                    x1 = v01.y * isq;
                    x2 = v23.x * isq;
                    x3 = v23.y * isq;
                }
                split_h2(x0, x1, qa[ks][0], qa[ks][1]);  // a0a1 (row g) hi, a2a3 (row g+8) lo
                split_h2(x2, x3, qa[ks][2], qa[ks][3]);  // a4a5 hi, a6a7 lo
            }
        }
        const float slope = a.slopes[h];
        float m_row = -INFINITY, l_row = 0.f;
        float o[NNT][4];
#pragma unroll
        for (int n = 0; n < NNT; ++n)
#pragma unroll
            for (int r = 0; r < 4; ++r) o[n][r] = 0.f;
        for (int i = sg.i0; i < sg.i0 + sg.n; ++i, ++it) {
            if (CW > GW && (it & 1) != (warp >> 2)) continue;  // the other warp group's stage
            const int b = it % ST;
            const int k0 = i * AM_SK;
            mbar_wait(&full[b], (it / ST) & 1);
            if (threadIdx.x == 32 && nseg < 2 && i == sg.i0) trace_stamp(a.trace, c, 6 + 3 * nseg);  // first data
            const int kb = (warp & (GW - 1)) * 16;  // this warp's 16 keys of the stage
            if (k0 + kb + 16 > j1) {
                // partial last stage: rows past the range hold stale smem; P is 0
                // there but 0 * NaN would poison O, so clear this warp's V rows
                for (int idx = lane; idx < 16 * (DH / 8); idx += 32) {
                    const int r = idx / (DH / 8), cc = idx % (DH / 8);
                    if (k0 + kb + r >= j1)
                        *reinterpret_cast<uint4*>(Vs + ((int64_t)(b * AM_SK + kb + r)) * DH + cc * 8) =
                            make_uint4(0u, 0u, 0u, 0u);
                }
                __syncwarp();
            }
            // ---- S = Q K^T over 16 keys (2 n-tiles)
            float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
            {
                const int key = kb + ((mi & 2) ? 8 : 0) + ri;  // row of the K tile
                const uint32_t rowaddr = ks_base + (uint32_t)((b * AM_SK + key) * ROWB);
#pragma unroll
                for (int ks = 0; ks < NKT; ++ks) {
                    const int chunk = ks * 2 + (mi & 1);
                    uint32_t r0, r1, r2, r3;
                    ldsm_x4(rowaddr + (uint32_t)(kv_chunk_swz(chunk, key) * 16), r0, r1, r2, r3);
                    mma_f16(s0, qa[ks], r0, r1);
                    mma_f16(s1, qa[ks], r2, r3);
                }
            }
            // ---- scores of query g: keys kb + 2qd + {0,1} (s0), kb + 8 + 2qd + {0,1} (s1)
            float sc[4];
            float mx = -INFINITY;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int jrel = kb + (e >> 1) * 8 + 2 * qd + (e & 1);
                const int j = k0 + jrel;
                const float dot = (e < 2) ? (s0[e] + s0[2 + e]) : (s1[e - 2] + s1[e]);
                const bool ok = qv && j < j1 && j <= my_pos;
                sc[e] = ok ? dot + slope * (float)(j - my_pos) : -INFINITY;
                mx = fmaxf(mx, sc[e]);
            }
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            const float m_new = fmaxf(m_row, mx);
            float p[4];
            float ls = 0.f;
            float alpha = 1.f;
            if (m_new != -INFINITY) {
                alpha = m_row == -INFINITY ? 0.f : expf(m_row - m_new);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    p[e] = sc[e] == -INFINITY ? 0.f : expf(sc[e] - m_new);
                    ls += p[e];
                }
                m_row = m_new;
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) p[e] = 0.f;
            }
            ls += __shfl_xor_sync(0xffffffffu, ls, 1);
            ls += __shfl_xor_sync(0xffffffffu, ls, 2);
            l_row = l_row * alpha + ls;
            if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
                for (int n = 0; n < NNT; ++n)
#pragma unroll
                    for (int r = 0; r < 4; ++r) o[n][r] *= alpha;
            }
            // ---- P as the A operand: rows g hi / g+8 lo
            uint32_t pa[4];
            split_h2(p[0], p[1], pa[0], pa[1]);
            split_h2(p[2], p[3], pa[2], pa[3]);
            // ---- O += P V  (V fragments via ldmatrix.trans, 2 n-tiles per load)
            {
                const int key = kb + ((mi & 1) ? 8 : 0) + ri;
                const uint32_t rowaddr = vs_base + (uint32_t)((b * AM_SK + key) * ROWB);
#pragma unroll
                for (int n2 = 0; n2 < NNT / 2; ++n2) {
                    const int chunk = n2 * 2 + ((mi & 2) ? 1 : 0);
                    uint32_t r0, r1, r2, r3;
                    ldsm_x4_t(rowaddr + (uint32_t)(kv_chunk_swz(chunk, key) * 16), r0, r1, r2, r3);
                    mma_f16(o[2 * n2], pa, r0, r1);
                    mma_f16(o[2 * n2 + 1], pa, r2, r3);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[b]);
        }
        if (threadIdx.x == 32 && nseg == 0) trace_stamp(a.trace, c, 11);  // diagnostics: stages done
        // ---- per-warp state for query g: m, l, O[dims] = hi rows + lo rows
        if (qv) {
            float* w = wst + (warp * AM_G + g) * (DH + 2);
            if (qd == 0) {
                w[0] = m_row;
                w[1] = l_row;
            }
#pragma unroll
            for (int n = 0; n < NNT; ++n) {
                w[2 + n * 8 + 2 * qd] = o[n][0] + o[n][2];
                w[2 + n * 8 + 2 * qd + 1] = o[n][1] + o[n][3];
            }
        }
        cons_bar_n<CW>();
        // ---- merge the 4 warps per query (fixed order); this CTA's piece of (g, h)
        const int cf = am_owner(sg.a, G, U), cl = am_owner(sg.a + sg.ns - 1, G, U);
        const int tid = threadIdx.x;  // 0 .. 127
        float mloc[AM_G];
#pragma unroll
        for (int q = 0; q < AM_G; ++q) mloc[q] = 0.f;
        for (int q = 0; q < nq; ++q) {
            float M = -INFINITY;
#pragma unroll
            for (int w = 0; w < CW; ++w) M = fmaxf(M, wst[(w * AM_G + q) * (DH + 2)]);
            float sw[CW];
            float L = 0.f;
#pragma unroll
            for (int w = 0; w < CW; ++w) {
                const float mw = wst[(w * AM_G + q) * (DH + 2)];
                sw[w] = mw == -INFINITY ? 0.f : expf(mw - M);
                L += wst[(w * AM_G + q) * (DH + 2) + 1] * sw[w];
            }
            float* out = a.part + (((int64_t)(t0 + q) * a.H + h) * AM_MAXC + (c - cf)) * (DH + 2);
            for (int e = tid; e < DH; e += CW * 32) {
                float acc = 0.f;
#pragma unroll
                for (int w = 0; w < CW; ++w) acc += wst[(w * AM_G + q) * (DH + 2) + 2 + e] * sw[w];
                if (cf == cl) mloc[q] = fmaxf(mloc[q], am_final<DH>(a, t0 + q, h, e, acc, L));
                else out[2 + e] = acc;
            }
            if (cf != cl && tid == 0) {
                out[0] = M;
                out[1] = L;
            }
        }
        bool finalize = cf == cl;
        if (!finalize) {
            // ---- last contributor of (g, h) merges the pieces in CTA order
            cons_bar_n<CW>();  // every thread's partial stores precede the counter (fence by one thread, as in a grid sync)
            if (tid == 0) {
                __threadfence();
                int* ctr = a.counters + (int64_t)t0 * a.H + h;
                const int prev = atomicAdd(ctr, 1);
                const int last = prev == cl - cf;
                if (last) *ctr = 0;
                *s_flag = last;
            }
            cons_bar_n<CW>();
            finalize = *s_flag != 0;
            if (finalize) {
                __threadfence();
                const int np = cl - cf + 1;
                for (int q = 0; q < nq; ++q) {
                    const float* pp = a.part + ((int64_t)(t0 + q) * a.H + h) * AM_MAXC * (DH + 2);
                    float M = -INFINITY;
                    for (int s = 0; s < np; ++s) M = fmaxf(M, __ldcg(pp + s * (DH + 2)));
                    float L = 0.f;
                    for (int s = 0; s < np; ++s) {
                        const float ms = __ldcg(pp + s * (DH + 2));
                        if (ms != -INFINITY) L += __ldcg(pp + s * (DH + 2) + 1) * expf(ms - M);
                    }
                    for (int e = tid; e < DH; e += CW * 32) {
                        float acc = 0.f;
                        for (int s = 0; s < np; ++s) {
                            const float ms = __ldcg(pp + s * (DH + 2));
                            if (ms != -INFINITY) acc += __ldcg(pp + s * (DH + 2) + 2 + e) * expf(ms - M);
                        }
                        mloc[q] = fmaxf(mloc[q], am_final<DH>(a, t0 + q, h, e, acc, L));
                    }
                }
            }
        }
        cons_bar_n<CW>();  // wst free; every warp past the merge
        if (threadIdx.x == 32 && nseg == 0) trace_stamp(a.trace, c, 12);  // diagnostics: merged
        if (finalize && a.tokmax) {
            // operand range of the wo GEMV: exact, order-independent max per token
            for (int q = 0; q < nq; ++q) {
                const float v = warp_max(mloc[q]);
                if (lane == 0) wst[q * CW + warp] = v;
            }
            cons_bar_n<CW>();
            if (tid < nq) {
                float v = 0.f;
                for (int w = 0; w < CW; ++w) v = fmaxf(v, wst[tid * CW + w]);
                atomicMax(reinterpret_cast<int*>(a.tokmax) + t0 + tid, __float_as_int(v));
            }
            cons_bar_n<CW>();
        }
        if (threadIdx.x == 32 && nseg < 2) trace_stamp(a.trace, c, 7 + 3 * nseg);  // segment done
        u += sg.n;
    }
    if (threadIdx.x == 32) trace_stamp(a.trace, c, 3);
}

// Prefill variant (query groups of up to 32 consecutive positions of
// one sequence): the same stream-K units and producer, but warp w owns queries
// 8w .. 8w+7 of the group (rows g hi / g+8 lo of its MMA tiles) and runs over
// all 64 keys of every stage, so each K/V byte feeds 32 queries instead of 8.
// No cross-warp merge: a warp's online-softmax state is its queries' final
// (or per-CTA partial) state.

template <int DH>
constexpr size_t attn_pf_smem() {
    return (size_t)AM_ST * 2 * AM_SK * DH * 2 + 2 * AM_ST * 8 + 64 + 4 * AM_PT + AM_WARPS * 8 * 4;
}

template <int DH>
__global__ void __launch_bounds__((AM_WARPS + 1) * 32) k_attn_pf(AttnArgs a, int G, int64_t U) {
    constexpr int NKT = DH / 16;  // k-steps of S
    constexpr int NNT = DH / 8;   // n-tiles of O
    constexpr int ROWB = DH * 2;  // bytes per K/V row
    extern __shared__ __align__(128) uint8_t smem[];
    half* Ks = reinterpret_cast<half*>(smem);                         // [ST][SK][DH]
    half* Vs = Ks + AM_ST * AM_SK * DH;                               // [ST][SK][DH]
    uint64_t* full = reinterpret_cast<uint64_t*>(Vs + AM_ST * AM_SK * DH);
    uint64_t* empty = full + AM_ST;
    int* s_flag = reinterpret_cast<int*>(empty + AM_ST);
    int* s_pages = s_flag + 4;                                        // [AM_PT]

    const int c = blockIdx.x;
    const int64_t u0 = (int64_t)c * U / G, u1 = (int64_t)(c + 1) * U / G;
    const int lane = threadIdx.x & 31, warp = warp_uniform_id();
    const int64_t kv_stride = (int64_t)a.H * a.P * DH;

    if (threadIdx.x == 0) {
        for (int b = 0; b < AM_ST; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&empty[b], AM_WARPS);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (warp == AM_WARPS) {
        // ---------------- producer warp (as k_attn_mma; prefill waits for the QKV GEMV first)
        pdl_wait();
        pdl_trigger();
        int it = 0;
        for (int64_t u = u0; u < u1;) {
            const AmSeg sg = am_seg(a, u, u1);
            const int t0 = a.grp_first[sg.g], nq = a.grp_count[sg.g];
            const int jend = a.tok_pos[t0] + nq;
            const int32_t* pt = a.pages + (int64_t)a.tok_seq[t0] * a.max_pages;
            const int64_t head_off = (int64_t)sg.h * a.P * DH;
            int pbase = -1 << 30;
            for (int i = sg.i0; i < sg.i0 + sg.n; ++i, ++it) {
                const int k0 = i * AM_SK;
                const int k1 = min(jend, k0 + AM_SK);
                if ((k1 - 1) / a.P >= pbase + AM_PT) {
                    __syncwarp();
                    pbase = k0 / a.P;
                    const int plast = (min(jend, (sg.i0 + sg.n) * AM_SK) - 1) / a.P;
                    for (int p = lane; p < AM_PT && pbase + p <= plast; p += 32) s_pages[p] = pt[pbase + p];
                    __syncwarp();
                }
                const int b = it % AM_ST;
                mbar_wait(&empty[b], ((it / AM_ST) & 1) ^ 1);
                if (lane == 0) {
                    mbar_expect_tx(&full[b], (uint32_t)(k1 - k0) * ROWB * 2);
                    for (int j = k0; j < k1;) {
                        const int page = s_pages[j / a.P - pbase];
                        const int jn = min(k1, (j / a.P + 1) * a.P);
                        const half* kp = a.kv + (int64_t)page * 2 * kv_stride + head_off + (int64_t)(j % a.P) * DH;
                        const uint32_t bytes = (uint32_t)(jn - j) * ROWB;
                        bulk_g2s(Ks + ((int64_t)b * AM_SK + (j - k0)) * DH, kp, bytes, &full[b]);
                        bulk_g2s(Vs + ((int64_t)b * AM_SK + (j - k0)) * DH, kp + kv_stride, bytes, &full[b]);
                        j = jn;
                    }
                }
            }
            u += sg.n;
        }
        return;
    }

    // ---------------- compute warps: warp w owns queries 8w .. 8w + 7 of the group
    pdl_wait();
    pdl_trigger();
    const int g = lane >> 2, qd = lane & 3;
    const uint32_t ks_base = smem_u32(Ks), vs_base = smem_u32(Vs);
    const int mi = lane >> 3, ri = lane & 7;
    const float isq = 1.0f / sqrtf((float)DH);
    int it = 0;
    for (int64_t u = u0; u < u1;) {
        const AmSeg sg = am_seg(a, u, u1);
        const int h = sg.h;
        const int t0 = a.grp_first[sg.g], nq = a.grp_count[sg.g];
        const int pos0 = a.tok_pos[t0];
        const int j1 = pos0 + nq;
        const int qi = warp * 8 + g;  // this lane's query within the group
        const bool qv = qi < nq;
        const bool warp_live = warp * 8 < nq;
        const int my_pos = pos0 + qi;
        uint32_t qa[NKT][4];
        {
            const float* q = a.q + (int64_t)(t0 + (qv ? qi : 0)) * a.d + h * DH;
#pragma unroll
            for (int ks = 0; ks < NKT; ++ks) {
                float x0 = 0.f, x1 = 0.f, x2 = 0.f, x3 = 0.f;
                if (qv) {
                    const float2 v01 = *reinterpret_cast<const float2*>(q + ks * 16 + 2 * qd);
                    const float2 v23 = *reinterpret_cast<const float2*>(q + ks * 16 + 2 * qd + 8);
                    x0 = v01.x * isq;
                    x1 = v01.y * isq;
                    x2 = v23.x * isq;
                    x3 = v23.y * isq;
                }
                split_h2(x0, x1, qa[ks][0], qa[ks][1]);
                split_h2(x2, x3, qa[ks][2], qa[ks][3]);
            }
        }
        const float slope = a.slopes[h];
        float m_row = -INFINITY, l_row = 0.f;
        float o[NNT][4];
#pragma unroll
        for (int n = 0; n < NNT; ++n)
#pragma unroll
            for (int r = 0; r < 4; ++r) o[n][r] = 0.f;
        for (int i = sg.i0; i < sg.i0 + sg.n; ++i, ++it) {
            const int b = it % AM_ST;
            const int k0 = i * AM_SK;
            mbar_wait(&full[b], (it / AM_ST) & 1);
            if (warp_live && k0 <= pos0 + warp * 8 + 7) {  // some key of the stage is visible to this warp
                if (k0 + AM_SK > j1) {
                    // partial last stage: clear the stale V rows (P is 0 there, but 0 * NaN is not)
                    for (int idx = lane; idx < AM_SK * (DH / 8); idx += 32) {
                        const int r = idx / (DH / 8), cc = idx % (DH / 8);
                        if (k0 + r >= j1)
                            *reinterpret_cast<uint4*>(Vs + ((int64_t)(b * AM_SK + r)) * DH + cc * 8) =
                                make_uint4(0u, 0u, 0u, 0u);
                    }
                    __syncwarp();
                }
                // ---- S = Q K^T over the stage's 64 keys (8 n-tiles)
                float sc[8][4];
#pragma unroll
                for (int nt = 0; nt < 8; ++nt)
#pragma unroll
                    for (int r = 0; r < 4; ++r) sc[nt][r] = 0.f;
#pragma unroll
                for (int np = 0; np < 4; ++np) {  // key pairs of n-tiles: keys 16 np .. 16 np + 15
                    const int key = np * 16 + ((mi & 2) ? 8 : 0) + ri;
                    const uint32_t rowaddr = ks_base + (uint32_t)((b * AM_SK + key) * ROWB);
#pragma unroll
                    for (int ks = 0; ks < NKT; ++ks) {
                        const int chunk = ks * 2 + (mi & 1);
                        uint32_t r0, r1, r2, r3;
                        ldsm_x4(rowaddr + (uint32_t)(kv_chunk_swz(chunk, key) * 16), r0, r1, r2, r3);
                        mma_f16(sc[2 * np], qa[ks], r0, r1);
                        mma_f16(sc[2 * np + 1], qa[ks], r2, r3);
                    }
                }
                // ---- scores of query qi: n-tile nt holds keys 8 nt + 2 qd + {0, 1} (hi rows + lo rows)
                float p[8][2];
                float mx = -INFINITY;
#pragma unroll
                for (int nt = 0; nt < 8; ++nt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int j = k0 + nt * 8 + 2 * qd + e;
                        const float dot = sc[nt][e] + sc[nt][2 + e];
                        const bool ok = qv && j < j1 && j <= my_pos;
                        p[nt][e] = ok ? dot + slope * (float)(j - my_pos) : -INFINITY;
                        mx = fmaxf(mx, p[nt][e]);
                    }
                mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
                mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
                const float m_new = fmaxf(m_row, mx);
                float ls = 0.f, alpha = 1.f;
                if (m_new != -INFINITY) {
                    alpha = m_row == -INFINITY ? 0.f : expf(m_row - m_new);
#pragma unroll
                    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            p[nt][e] = p[nt][e] == -INFINITY ? 0.f : expf(p[nt][e] - m_new);
                            ls += p[nt][e];
                        }
                    m_row = m_new;
                } else {
#pragma unroll
                    for (int nt = 0; nt < 8; ++nt) p[nt][0] = p[nt][1] = 0.f;
                }
                ls += __shfl_xor_sync(0xffffffffu, ls, 1);
                ls += __shfl_xor_sync(0xffffffffu, ls, 2);
                l_row = l_row * alpha + ls;
                if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
                    for (int n = 0; n < NNT; ++n)
#pragma unroll
                        for (int r = 0; r < 4; ++r) o[n][r] *= alpha;
                }
                // ---- O += P V over 4 k-steps of 16 keys (P from n-tiles 2 ks, 2 ks + 1)
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    uint32_t pa[4];
                    split_h2(p[2 * ks][0], p[2 * ks][1], pa[0], pa[1]);
                    split_h2(p[2 * ks + 1][0], p[2 * ks + 1][1], pa[2], pa[3]);
                    const int key = ks * 16 + ((mi & 1) ? 8 : 0) + ri;
                    const uint32_t rowaddr = vs_base + (uint32_t)((b * AM_SK + key) * ROWB);
#pragma unroll
                    for (int n2 = 0; n2 < NNT / 2; ++n2) {
                        const int chunk = n2 * 2 + ((mi & 2) ? 1 : 0);
                        uint32_t r0, r1, r2, r3;
                        ldsm_x4_t(rowaddr + (uint32_t)(kv_chunk_swz(chunk, key) * 16), r0, r1, r2, r3);
                        mma_f16(o[2 * n2], pa, r0, r1);
                        mma_f16(o[2 * n2 + 1], pa, r2, r3);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[b]);
        }
        // ---- this CTA's piece of (g, h): per query (m, l, O[dims] = hi rows + lo rows)
        const int cf = am_owner(sg.a, G, U), cl = am_owner(sg.a + sg.ns - 1, G, U);
        float mloc = 0.f;
        if (cf == cl) {
            if (qv) {
#pragma unroll
                for (int n = 0; n < NNT; ++n)
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        mloc = fmaxf(mloc, am_final<DH>(a, t0 + qi, h, n * 8 + 2 * qd + e, o[n][e] + o[n][2 + e], l_row));
            }
        } else {
            if (qv) {
                float* out = a.part + (((int64_t)(t0 + qi) * a.H + h) * AM_MAXC + (c - cf)) * (DH + 2);
                if (qd == 0) {
                    out[0] = m_row;
                    out[1] = l_row;
                }
#pragma unroll
                for (int n = 0; n < NNT; ++n) {
                    out[2 + n * 8 + 2 * qd] = o[n][0] + o[n][2];
                    out[2 + n * 8 + 2 * qd + 1] = o[n][1] + o[n][3];
                }
            }
            cons_bar();
            if (threadIdx.x == 0) {
                __threadfence();
                int* ctr = a.counters + (int64_t)t0 * a.H + h;
                const int prev = atomicAdd(ctr, 1);
                const int last = prev == cl - cf;
                if (last) *ctr = 0;
                *s_flag = last;
            }
            cons_bar();
            if (*s_flag) {
                __threadfence();
                const int np = cl - cf + 1;
                if (qv) {
                    const float* pp = a.part + ((int64_t)(t0 + qi) * a.H + h) * AM_MAXC * (DH + 2);
                    float M = -INFINITY;
                    for (int s2 = 0; s2 < np; ++s2) M = fmaxf(M, __ldcg(pp + s2 * (DH + 2)));
                    float L = 0.f;
                    for (int s2 = 0; s2 < np; ++s2) {
                        const float ms = __ldcg(pp + s2 * (DH + 2));
                        if (ms != -INFINITY) L += __ldcg(pp + s2 * (DH + 2) + 1) * expf(ms - M);
                    }
                    for (int e = qd; e < DH; e += 4) {
                        float acc = 0.f;
                        for (int s2 = 0; s2 < np; ++s2) {
                            const float ms = __ldcg(pp + s2 * (DH + 2));
                            if (ms != -INFINITY) acc += __ldcg(pp + s2 * (DH + 2) + 2 + e) * expf(ms - M);
                        }
                        mloc = fmaxf(mloc, am_final<DH>(a, t0 + qi, h, e, acc, L));
                    }
                }
            }
            cons_bar();  // s_flag reuse
        }
        if (a.tokmax) {  // wo operand range: max over this head's dims per query (the 4 lanes of a quad)
            mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, 1));
            mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, 2));
            if (qv && qd == 0 && mloc > 0.f) atomicMax(reinterpret_cast<int*>(a.tokmax) + t0 + qi, __float_as_int(mloc));
        }
        u += sg.n;
    }
}

template <int DH>
int run_attn_mma(const AttnArgs& a, int n_groups, int64_t cap, cudaStream_t st) {
    const int sms = sm_count();
    if (sms < 0) return PB_ERR_GENERIC;
    const int64_t U = a.total_units;
    if (U <= 0) return PB_OK;
    // CTAs: fill the machine (two per SM), but keep every (group, head) within AM_MAXC contributors
    const bool prefill = a.max_group > AM_G;  // prefill groups: queries split across warps
    int64_t G = std::min<int64_t>(U, 2 * (int64_t)sms);
    // decode with equally long query groups (batch-1, or a batch at one context
    // length): G a multiple of the (group, head) count, so no CTA's range crosses
    // a head boundary (traced: such CTAs finish ~10 us after the rest)
    const int64_t pairs = (int64_t)a.n_groups * a.H;
    if (!prefill && U == pairs * a.max_stages && G >= pairs)
        G = std::min<int64_t>(G / pairs, a.max_stages) * pairs;
    // short contexts (<= 4 stages of 64 keys): one CTA per (group, head) -- a head split across
    // CTAs pays a cross-CTA merge whose latency exceeds the streaming it parallelises (560M, 16
    // heads x 4 stages: 41.9 -> 39.3 us per block; thresholds 2 / 8: 41.9 / 39.3)
    constexpr int short_stages = 4;
    if (!prefill && U == pairs * a.max_stages && a.max_stages <= short_stages && G > pairs) G = pairs;
    while (G > 1 && ceil_div(a.max_stages, U / G) + 1 > AM_MAXC) --G;
    if ((int64_t)a.n_tok * a.H * AM_MAXC * (DH + 2) > cap) {
        set_error("attention workspace too small");
        return PB_ERR_CAPACITY;
    }
    (void)n_groups;
    if (prefill) {
        constexpr size_t smem = attn_pf_smem<DH>();
        static int ok[PB_MAX_DEVICES] = {};
        if (per_device(ok, [](int) {
                return cudaFuncSetAttribute(k_attn_pf<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) ==
                               cudaSuccess ? 1 : -1;
            }) < 0)
            return launch_check("attn_pf setup");
        return launch_pdl(k_attn_pf<DH>, dim3((unsigned)G), dim3((AM_WARPS + 1) * 32), smem, st, a, (int)G, U);
    }
    // two CTAs per SM, 3-stage rings, 4 compute warps each
    constexpr size_t smem = attn_mma_smem<DH, 3, 4>();
    static int ok[PB_MAX_DEVICES] = {};
    if (per_device(ok, [](int) {
            return cudaFuncSetAttribute(k_attn_mma<DH, 3, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem) == cudaSuccess ? 1 : -1;
        }) < 0)
        return launch_check("attn_mma setup");
    AttnArgs aa = a;
    aa.trace = trace_region(TR_ATTN, (int)G);
    return launch_pdl(k_attn_mma<DH, 3, 4>, dim3((unsigned)G), dim3(5 * 32), smem, st, aa, (int)G, U);
}

template int run_attn_mma<64>(const AttnArgs&, int, int64_t, cudaStream_t);
template int run_attn_mma<128>(const AttnArgs&, int, int64_t, cudaStream_t);

}  // namespace pb
