// int8-weight GEMV/GEMM for the block executor (quant.py:117-129 matmul_mixed,
// model.py:305-311 _mm) plus the fused prologues/epilogues of block_forward
// (model.py:340-368).
//
// Math: y[n, o] = sum_k code[o, k] * (s_k * x[n, k]) + sum_j W[k_j, o] x[n, k_j] + b[o]
// The per-input-feature scale s_k is folded into the activation (x~ = s ⊙ x)
// so the weight stream is raw int8 codes. Per token, x~ is scaled by a power
// of two so max |x~| lies in [2^21, 2^22) and rounded to a 22-bit integer a,
// written as three balanced int8 digits a = 65536 h + 256 m + l. Every
// product code x digit is then an exact int8 x int8 tensor-core MMA
// (mma.m16n8k32.s8, s32 accumulation: |sum| <= 127 * 128 * K < 2^31 for K <
// 131072), so the GEMV is exact integer arithmetic on a 22-bit fixed-point
// operand (relative error <= 2^-22 of the token's max |x~|); the epilogue
// recombines h/m/l and undoes the scale. Split-K partial sums are integers:
// merged exactly and order-independently.
//
// Memory-bound decode: weights stream in 4 KB canonical tiles (pb_weights.cu)
// through a cp.async.bulk ring; each consumer warp loads an m16k32 A fragment
// with one ldmatrix.x4 and issues one IMMA per 8 operand columns -- no int8
// -> fp16 conversion on the weight stream.
//
// B (activation) layout, chunk c of TC tokens, columns p * TC + t for digit p
// (0: h, 1: m, 2: l) of token t, NT = ceil(3 TC / 8) n-tiles of 8 columns:
//   uint2 at ((c * KC + kc) * NT + nt) * 32 + lane (lane = 4 g + q, column 8 nt + g),
//   .x = B[k = 4q .. 4q+3][col], .y = B[k = 16 + 4q .. 16 + 4q + 3][col]  (the m16n8k32 B fragment).
#include "pb_async.cuh"
#include "pb_common.cuh"
#include "pb_epi.cuh"
#include "pb_operand.cuh"
#include "pb_span.h"

namespace pb {


int choose_tc(int n_tok) {
    if (n_tok <= 2) return 2;
    if (n_tok <= 8) return 8;
    if (n_tok <= 16) return 16;
    return 32;
}

// ------------------------------------------------------------------ prologue

__device__ __forceinline__ float block_sum(float v, float* red) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    float t = 0.f;
    if (threadIdx.x < 32) {
        t = l < (int)(blockDim.x >> 5) ? red[l] : 0.f;
        t = warp_sum(t);
        if (l == 0) red[0] = t;
    }
    __syncthreads();
    return red[0];
}

__device__ __forceinline__ double block_sum_d(double v, double* red) {
    v = warp_sum_d(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = l < (int)(blockDim.x >> 5) ? red[l] : 0.0;
        t = warp_sum_d(t);
        if (l == 0) red[0] = t;
    }
    __syncthreads();
    return red[0];
}

__device__ __forceinline__ float block_max(float v, float* red) {
    v = warp_max(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        float t = l < (int)(blockDim.x >> 5) ? red[l] : 0.f;
        t = warp_max(t);
        if (l == 0) red[0] = t;
    }
    __syncthreads();
    return red[0];
}


// Row statistics, one CTA per token: LayerNorm mean / inverse std (population
// variance, eps 1e-5; accumulated in f64) and the power-of-two shift that maps
// max |y * s| into [2^13, 2^14) (the operand writers scale by 2^8 more for the
// 22-bit fixed-point digits).
constexpr int STATS_THREADS = 1024;

__global__ void __launch_bounds__(STATS_THREADS) k_rowstats(ProArgs a) {
    __shared__ double redd[32];
    __shared__ float redf[32];
    const int tok = blockIdx.x;
    const float* x = a.x + (int64_t)tok * a.K;
    const bool vec = (a.K & 3) == 0 && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
    float mu = 0.f, inv = 1.f;
    if (a.mode == PRO_LN) {
        double s = 0.0;
        if (vec) {
            for (int k = threadIdx.x * 4; k < a.K; k += STATS_THREADS * 4) {
                const float4 v = *reinterpret_cast<const float4*>(x + k);
                s += (double)v.x + (double)v.y + (double)v.z + (double)v.w;
            }
        } else {
            for (int k = threadIdx.x; k < a.K; k += STATS_THREADS) s += (double)x[k];
        }
        const double mean = block_sum_d(s, redd) / a.K;
        double v2 = 0.0;
        if (vec) {
            for (int k = threadIdx.x * 4; k < a.K; k += STATS_THREADS * 4) {
                const float4 v = *reinterpret_cast<const float4*>(x + k);
                const double d0 = v.x - mean, d1 = v.y - mean, d2 = v.z - mean, d3 = v.w - mean;
                v2 += d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3;
            }
        } else {
            for (int k = threadIdx.x; k < a.K; k += STATS_THREADS) {
                const double d0 = (double)x[k] - mean;
                v2 += d0 * d0;
            }
        }
        const float var = (float)(block_sum_d(v2, redd) / a.K);
        mu = (float)mean;
        inv = 1.0f / sqrtf(var + 1e-5f);
    }
    float m = 0.f;
    if (a.scales) {
        for (int k = threadIdx.x; k < a.K; k += STATS_THREADS) m = fmaxf(m, fabsf(pro_y(a, x, k, mu, inv) * a.scales[k]));
        m = block_max(m, redf);
    }
    int shift = 0;
    if (m > 0.f && isfinite(m)) {
        int e;
        frexpf(m, &e);  // m in [2^(e-1), 2^e)
        shift = 14 - e;
    }
    if (threadIdx.x == 0) {
        a.back[tok] = ldexpf(1.f, -shift);
        a.stats[tok] = make_float4(mu, inv, ldexpf(1.f, shift), ldexpf(1.f, -shift));
    }
}

// Chan et al. merge of (n, mean, M2, min, max) summaries, a before b.
struct RowSum {
    double n, mean, m2;
    float mn, mx;
};
__device__ __forceinline__ RowSum rs_merge(const RowSum& a, const RowSum& b) {
    if (a.n == 0.0) return b;
    if (b.n == 0.0) return a;
    RowSum r;
    r.n = a.n + b.n;
    const double d = b.mean - a.mean;
    r.mean = a.mean + d * (b.n / r.n);
    r.m2 = a.m2 + b.m2 + d * d * (a.n * b.n / r.n);
    r.mn = fminf(a.mn, b.mn);
    r.mx = fmaxf(a.mx, b.mx);
    return r;
}

__global__ void k_bound_consts(const float* __restrict__ g, const float* __restrict__ b, const float* __restrict__ s,
                               int K, float* __restrict__ out) {
    __shared__ float red[32];
    float mg = 0.f, mb = 0.f;
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        mg = fmaxf(mg, fabsf(g[k]) * s[k]);
        mb = fmaxf(mb, fabsf(b[k]) * s[k]);
    }
    mg = block_max(mg, red);
    mb = block_max(mb, red);
    if (threadIdx.x == 0) {
        out[0] = mg;
        out[1] = mb;
    }
}

int bound_consts(const float* gamma, const float* beta, const float* scales, int K, float* gs, float* bs,
                 cudaStream_t st) {
    float* d = nullptr;
    PB_CHECK_CUDA(cudaMallocAsync(&d, 2 * sizeof(float), st));
    k_bound_consts<<<1, 1024, 0, st>>>(gamma, beta, scales, K, d);
    if (int rc = launch_check("bound_consts")) return rc;
    float h[2];
    PB_CHECK_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
    PB_CHECK_CUDA(cudaStreamSynchronize(st));
    PB_CHECK_CUDA(cudaFreeAsync(d, st));
    *gs = h[0];
    *bs = h[1];
    return PB_OK;
}

// k_fragwrite: one thread per (token, 32-wide k tile, lane quad q).
// Specialised per (operand mode, statistics source) so the code on the
// dependency-release critical path is compact (it runs cold in the
// instruction cache once per matrix; MODE/SRC = -1: runtime values).
template <int MODE, int SRC>
__global__ void __launch_bounds__(256) k_fragwrite(ProArgs a) {
    if (MODE >= 0) a.mode = MODE;
    if (SRC >= 0) a.src.kind = SRC;
    // early trigger (default): the GEMV that consumes this operand launches while
    // this kernel still waits for its producer and starts streaming weights
    // (its own griddepcontrol.wait still orders it after this grid completes)
    const int tcta = blockIdx.y * gridDim.x + blockIdx.x;
    if (threadIdx.x == 0) trace_stamp(a.trace, tcta, 0);
    if (a.early) pdl_trigger();
    const int KC = a.Kp / 32;
    const int it = blockIdx.x * blockDim.x + threadIdx.x;
    FragParams fp;
    if (it < KC * 4) frag_params(a, it >> 2, it & 3, fp);  // weights: before the dependency wait
    pdl_wait();
    if (!a.early) pdl_trigger();
    if (threadIdx.x == 0) trace_stamp(a.trace, tcta, 1);
    const int tok = blockIdx.y;
    float xv[8];  // activations first: their loads overlap the statistics' loads
    if (it < KC * 4) frag_x(a, tok, it >> 2, it & 3, xv);
    // every warp resolves the statistics itself (warp-uniform code, no CTA
    // barrier; a lane-divergent region made the shuffles take the compiler's
    // non-converged path: ncu showed WARPSYNC.COLLECTIVE, ~5 us per resolve)
    const float4 st = resolve_stats(a, tok);
    if (threadIdx.x == 0) trace_stamp(a.trace, tcta, 5);
    if (blockIdx.x == 0) operand_token_outputs(a, tok, st, threadIdx.x, blockDim.x);
    if (it < KC * 4) frag_item(a, tok, it >> 2, it & 3, st, fp, xv);
    if (threadIdx.x == 0) trace_stamp(a.trace, tcta, 6);
    if (a.trace) {
        __syncthreads();
        if (threadIdx.x == 0) trace_stamp(a.trace, tcta, 3);
    }
}

// Same operand for the tcgen05 GEMM (pb_gemm_tc.cu): the three int8 digit
// planes of a = rint(y s 2^(shift + 8)), each in the UMMA canonical K-major
// no-swizzle layout of the weight tiles: per (tw-token tile nt, 32-wide
// k tile kc, digit p) a tw x 32 B block at ((nt * KC + kc) * 3 + p) *
// tw * 32, token c, k: byte (c >> 3) * 256 + (k >> 4) * 128 + (c & 7) * 16
// + (k & 15). One thread per (token, k tile, 16-wide k half) -> three 16-byte
// stores. Padding tokens are zeros.
__global__ void __launch_bounds__(256) k_canonwrite(ProArgs a, uint8_t* __restrict__ bcanon, int n_tok, int tw) {
    __shared__ float4 s_st;
    const int tok = blockIdx.y;
    const float* x = a.x + (int64_t)tok * a.K;
    const bool real = tok < n_tok;
    const int KC = a.Kp / 32;
    const int it = blockIdx.x * blockDim.x + threadIdx.x;
    // this thread's 16 activations and scales first: their loads overlap the statistics' resolve
    float xv[16], sv[16], gv[16], bv[16];
    const bool mine = real && it < KC * 2;
    const bool ln = a.mode == PRO_LN;
    const int k0 = (it >> 1) * 32 + (it & 1) * 16;
    // whole 16-feature run of a 16-byte aligned row (callers pass rows at any float offset): 128-bit loads
    if (mine && k0 + 16 <= a.K && (a.K & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float4 xq = *reinterpret_cast<const float4*>(x + k0 + 4 * i);
            const float4 sq = *reinterpret_cast<const float4*>(a.scales + k0 + 4 * i);
            const float4 gq = ln ? *reinterpret_cast<const float4*>(a.gamma + k0 + 4 * i) : make_float4(1.f, 1.f, 1.f, 1.f);
            const float4 bq = ln ? *reinterpret_cast<const float4*>(a.beta + k0 + 4 * i) : make_float4(0.f, 0.f, 0.f, 0.f);
            xv[4 * i] = xq.x, xv[4 * i + 1] = xq.y, xv[4 * i + 2] = xq.z, xv[4 * i + 3] = xq.w;
            sv[4 * i] = sq.x, sv[4 * i + 1] = sq.y, sv[4 * i + 2] = sq.z, sv[4 * i + 3] = sq.w;
            gv[4 * i] = gq.x, gv[4 * i + 1] = gq.y, gv[4 * i + 2] = gq.z, gv[4 * i + 3] = gq.w;
            bv[4 * i] = bq.x, bv[4 * i + 1] = bq.y, bv[4 * i + 2] = bq.z, bv[4 * i + 3] = bq.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int k = k0 + i;
            const bool in = mine && k < a.K;
            xv[i] = in ? x[k] : 0.f;
            sv[i] = in ? a.scales[k] : 0.f;
            gv[i] = in && ln ? a.gamma[k] : 1.f;
            bv[i] = in && ln ? a.beta[k] : 0.f;
        }
    }
    if (real && threadIdx.x < 32) {
        const float4 r = resolve_stats(a, tok);
        if (threadIdx.x == 0) {
            s_st = r;
            if (blockIdx.x == 0) {
                a.back[tok] = r.w * (1.f / 256.f);
                if (a.src.zero_tokmax) a.src.zero_tokmax[tok] = 0.f;
            }
        }
    }
    __syncthreads();
    if (real && blockIdx.x == 0 && a.xo) {
        for (int j = threadIdx.x; j < a.n_outl; j += blockDim.x)
            a.xo[(int64_t)tok * a.n_outl + j] = pro_y(a, x, a.outl_idx[j], s_st.x, s_st.y);
    }
    if (it >= KC * 2) return;
    const int kc = it >> 1, kh = it & 1;
    uint32_t w[3][4] = {};
    if (real) {
        const float4 st = s_st;
        const float z = st.z * 256.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int k = kc * 32 + kh * 16 + i;
            const float y = ln ? fmaf(gv[i], (xv[i] - st.x) * st.y, bv[i]) : xv[i];
            const float v = k < a.K ? (y * sv[i]) * z : 0.f;  // pro_y (model.py:271-276) on the preloaded x
            int h, m, l;
            digits3(__float2int_rn(v), h, m, l);
            w[0][i >> 2] |= (uint32_t)(uint8_t)h << (8 * (i & 3));
            w[1][i >> 2] |= (uint32_t)(uint8_t)m << (8 * (i & 3));
            w[2][i >> 2] |= (uint32_t)(uint8_t)l << (8 * (i & 3));
        }
    }
    const int PLANE = tw * 32;  // tile width tw: 80 (prefill GEMM) or 16 / 32 (batched-decode GEMM)
    const int nt = tok / tw, c = tok % tw;
    uint8_t* blk = bcanon + ((int64_t)nt * KC + kc) * 3 * PLANE + (c >> 3) * 256 + kh * 128 + (c & 7) * 16;
#pragma unroll
    for (int p = 0; p < 3; ++p)
        *reinterpret_cast<uint4*>(blk + p * PLANE) = make_uint4(w[p][0], w[p][1], w[p][2], w[p][3]);
}

// f32-weights mode: plain y = LN(x) (or x) rows for the CUDA-core GEMM
__global__ void __launch_bounds__(256) k_rows_f32(ProArgs a) {
    const int tok = blockIdx.y;
    const float* x = a.x + (int64_t)tok * a.K;
    const float4 st = a.stats[tok];
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < a.K; k += gridDim.x * blockDim.x)
        a.y32[(int64_t)tok * a.K + k] = pro_y(a, x, k, st.x, st.y);
}

int prepare_fused_operand(int mode, const ProSrc& src, const float* x, int n_tok, int K, int Kp, const float* gamma,
                          const float* beta, const Mat& m, int tc, float* back, float4* stats, float* xo,
                          cudaStream_t st, ProArgs* out) {
    ProArgs a{mode, x, K, Kp, gamma, beta, m.scales, m.n_outl, m.outl_idx, tc, nullptr, back, stats, xo, nullptr, src, 1};
    a.src.zero_tokmax = nullptr;  // the fused QKV launch resets both ranges (launch_gemv_fused zero_a/zero_b)
    if (a.src.kind == SRC_STATS) {
        k_rowstats<<<n_tok, STATS_THREADS, 0, st>>>(a);
        if (int rc = launch_check("rowstats")) return rc;
    }
    *out = a;
    return PB_OK;
}

int launch_prologue(int mode, const ProSrc& src, const float* x, int n_tok, int K, int Kp, const float* gamma,
                    const float* beta, const Mat& m, int tc, uint4* frag, float* back, float4* stats, float* xo,
                    float* y32, cudaStream_t st, uint8_t* bcanon, int bcanon_tile) {
    constexpr int early = 1;  // weight-side operand inputs loaded before the PDL wait
    ProArgs a{mode, x, K, Kp, gamma, beta, y32 ? nullptr : m.scales, m.n_outl, m.outl_idx, tc, frag, back, stats,
              xo, y32, src, early};
    if (y32) a.src = ProSrc{};
    if (a.src.kind == SRC_STATS && (mode == PRO_LN || !y32)) {
        k_rowstats<<<n_tok, STATS_THREADS, 0, st>>>(a);
        if (int rc = launch_check("rowstats")) return rc;
    }
    if (y32) {
        if (mode != PRO_LN) {  // plain copy semantics: stats unused, mu=0 inv=1 not needed
            PB_CHECK_CUDA(cudaMemcpyAsync(y32, x, sizeof(float) * (size_t)n_tok * K, cudaMemcpyDeviceToDevice, st));
            return PB_OK;
        }
        k_rows_f32<<<dim3((unsigned)ceil_div(K, 256), n_tok), 256, 0, st>>>(a);
        return launch_check("rows_f32");
    }
    if (bcanon) {
        const int items = (Kp / 32) * 2;
        k_canonwrite<<<dim3((unsigned)ceil_div(items, 256), (unsigned)round_up(n_tok, bcanon_tile)), 256, 0, st>>>(
            a, bcanon, n_tok, bcanon_tile);
        return launch_check("canonwrite");
    }
    const int items = (Kp / 32) * 4;
    a.trace = trace_region(TR_FRAG, (int)ceil_div(items, 256) * n_tok);
    const dim3 grid((unsigned)ceil_div(items, 256), n_tok);
    if (a.mode == PRO_LN && a.src.kind == SRC_PARTIALS)
        return launch_pdl(k_fragwrite<PRO_LN, SRC_PARTIALS>, grid, dim3(256), 0, st, a);
    if (a.mode == PRO_SCALE && a.src.kind == SRC_TOKMAX)
        return launch_pdl(k_fragwrite<PRO_SCALE, SRC_TOKMAX>, grid, dim3(256), 0, st, a);
    return launch_pdl(k_fragwrite<-1, -1>, grid, dim3(256), 0, st, a);
}

// ------------------------------------------------------------------ epilogue

// ------------------------------------------------------------------ int8 mma GEMV

// ---- TMA-bulk pipelined stream-K GEMV ----------------------------------------
// CTA = 1 producer warp + 4 consumer warps. The CTA owns a contiguous range of
// the linearized work space u = mg * KC + kc (mg = 128-row group, kc = 32-wide
// K tile), so every CTA streams the same number of weight bytes (no wave
// tail). The producer's elected lane streams stages of SK_KCS k-tiles
// (4 KB of codes each: the 128-row group's tiles are contiguous in HBM) plus
// the matching B fragments into shared memory with cp.async.bulk
// (UBLKCP, mbarrier complete_tx); consumers read them with LDS.128, convert
// int8 -> fp16 in registers and issue mma.sync. An m-group that lies entirely
// in one CTA's range goes straight to the fused epilogue; a split m-group
// (range boundary) is finished by its last-arriving contributor, which sums
// the contributors' partial tiles in CTA order (deterministic).
constexpr int SK_CONS = 4;                       // consumer warps (2 m-tiles each)
constexpr int SK_THREADS = (SK_CONS + 1) * 32;   // + producer warp
// (k-tiles per stage, stages) are template parameters; sk_launch picks them

__device__ __forceinline__ void cons_sync() {  // the 4 consumer warps only
    asm volatile("bar.sync 1, %0;" ::"n"(SK_CONS * 32) : "memory");
}

struct SkArgs {
    const int8_t* codes;
    int MG, KC;       // 128-row groups, 32-wide k tiles
    int64_t total;    // MG * KC work units
    int G;            // CTAs per column chunk
    Act act;
    Epi epi;
    float* partials;  // [chunk][G][2][128 * 2tc]
    int* counters;    // [chunk][MG]
    int* sums;        // [chunk][MG][128 * COLS] s32 split-row-group sums, kept zero (null: partial slots)
    uint64_t* trace;  // diagnostics (pb_trace_set), usually null
    // fused operand (k_gemv_i8<.., FUSED>): an operand warp builds the B fragments of
    // every stage in shared memory from the activations (no k_fragwrite launch)
    ProArgs pro;
    float* zero_a;  // accumulators of later producers reset by this launch (QKV: max|ctx s|, max|act s|)
    float* zero_b;
};

__device__ __forceinline__ int sk_owner(int64_t u, int G, int64_t total) {
    return (int)(((u + 1) * G - 1) / total);
}

// Fused epilogue of one 128-row group (consumer warps only): the integer
// digit sums acc -> f64 recombination -> bias / outliers / residual / GELU /
// q|k|v + KV append, plus the per-token summary for the next operand.
template <int TC>
__device__ __forceinline__ void sk_epilogue(const SkArgs& a, int (&acc)[2][digit_ntiles(TC)][4], int mg, int chunk,
                                            int* S) {
    constexpr int NT = digit_ntiles(TC);
    constexpr int SST = 8 * NT + 1;
    const int lane = threadIdx.x & 31, cw = warp_uniform_id() - 1;
    const int g = lane >> 2, q = lane & 3;
    // ---- fused epilogue of the 128-row group
    cons_sync();  // S is free (previous epilogue done)
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int row = (cw * 2 + i) * 16 + g + 8 * (r >> 1);
                const int col = j * 8 + 2 * q + (r & 1);
                S[row * SST + col] = acc[i][j][r];
            }
    cons_sync();
    const int row_base = mg * 128;
    const bool want_sum = a.epi.pstats != nullptr, want_max = a.epi.tokmax != nullptr;
    float* Sf = reinterpret_cast<float*>(S);  // column j < TC reused for the epilogue outputs
    for (int t = threadIdx.x - 32; t < 128 * TC; t += SK_CONS * 32) {
        const int r = t % 128, j = t / 128;
        const int o = row_base + r;
        const int tok = chunk * TC + j;
        if (o >= a.epi.M || tok >= a.act.n_tok) continue;
        const double iv = 65536.0 * (double)S[r * SST + j] + 256.0 * (double)S[r * SST + TC + j] +
                          (double)S[r * SST + 2 * TC + j];
        const float v = (float)iv * a.act.back[tok];
        const float y = epi_store(a.epi, tok, o, v);
        if (want_max) Sf[r * SST + j] = fabsf(y * a.epi.s_next[o]);
        else if (want_sum) Sf[r * SST + j] = y;
    }
    if (want_sum || want_max) {
        // per-token summary of this 128-row group for the next operand's range / LayerNorm
        cons_sync();
        const int nrow = min(128, a.epi.M - row_base);
        for (int j = cw; j < TC; j += SK_CONS) {
            const int tok = chunk * TC + j;
            if (tok >= a.act.n_tok) continue;
            if (want_max) {
                float m = 0.f;
                for (int r = lane; r < nrow; r += 32) m = fmaxf(m, Sf[r * SST + j]);
                m = warp_max(m);
                if (lane == 0) atomicMax(reinterpret_cast<int*>(a.epi.tokmax) + tok, __float_as_int(m));
            } else {
                float s = 0.f, mn = INFINITY, mx = -INFINITY;
                for (int r = lane; r < nrow; r += 32) {
                    const float y = Sf[r * SST + j];
                    s += y;
                    mn = fminf(mn, y);
                    mx = fmaxf(mx, y);
                }
                const float mean = warp_sum(s) / nrow;
                float m2 = 0.f;
                for (int r = lane; r < nrow; r += 32) {
                    const float dlt = Sf[r * SST + j] - mean;
                    m2 = fmaf(dlt, dlt, m2);
                }
                m2 = warp_sum(m2);
                mn = -warp_max(-mn);
                mx = warp_max(mx);
                if (lane == 0) a.epi.pstats[(int64_t)tok * ((a.epi.M + 127) / 128) + mg] = make_float4(mean, m2, mn, mx);
            }
        }
    }
}

// Fused-operand warps (decode, TC = 2 tokens per column chunk): after
// the dependency wait each resolves the chunk's token statistics itself (LN
// summaries / atomicMax range of the producing kernel, as k_fragwrite does);
// warp 0 writes the per-token side outputs. Then, for its own stages (every
// SK_OPW-th in the producer's order), a warp loads the stage's inputs, waits
// for the ring slot, and writes the m16n8k32 B fragments of the stage's k
// tiles straight into shared memory: the same digits as frag_item, bit for
// bit. Lane l owns features 4l..4l+3 of each 128-feature slice; one float4 of
// x (+ gamma, beta) and scales per slice.
constexpr int SK_OPW = 4;  // operand warps of the fused GEMV: warp w fills the stages s = w (mod SK_OPW)

template <int TC, int SK_KCS, int SK_STAGES>
__device__ __forceinline__ void sk_operand_warp(const SkArgs& a, int64_t u0, int64_t u1, int chunk, uint8_t* sb,
                                                uint64_t* full, uint64_t* empty, int ow) {
    constexpr int NT = digit_ntiles(TC);
    constexpr int B_STAGE = SK_KCS * NT * 256;
    const ProArgs& p = a.pro;
    const int lane = threadIdx.x & 31;
    float4 st[TC];
    bool have_st = false;
    // the token statistics are resolved after this warp's first stage inputs are requested, so the
    // two chains of dependent loads (summaries -> statistics; activations) overlap
    auto resolve = [&]() {
#pragma unroll
        for (int t = 0; t < TC; ++t) {
            const int tok = chunk * TC + t;
            st[t] = tok < a.act.n_tok ? resolve_stats(p, tok) : make_float4(0.f, 1.f, 0.f, 0.f);  // warp-uniform
            if (tok < a.act.n_tok && ow == 0) {
                if (lane == 0) p.back[tok] = st[t].w * (1.f / 256.f);
                if (p.xo) {
                    const float* x = p.x + (int64_t)tok * p.K;
                    for (int j = lane; j < p.n_outl; j += 32)
                        p.xo[(int64_t)tok * p.n_outl + j] = pro_y(p, x, p.outl_idx[j], st[t].x, st[t].y);
                }
            }
        }
        have_st = true;
    };
    const bool ln = p.mode == PRO_LN;
    bool waited = false;
    auto wait_once = [&]() {  // dependency wait; then the range accumulators' reset (their readers are done)
        pdl_wait();
        pdl_trigger();
        waited = true;
        if (a.zero_a && blockIdx.x == 0 && ow == 0 && lane < TC && chunk * TC + lane < a.act.n_tok) {
            a.zero_a[chunk * TC + lane] = 0.f;
            a.zero_b[chunk * TC + lane] = 0.f;
        }
    };
    int stage = 0, seq = 0;
    uint32_t phase = 0;
    for (int64_t u = u0; u < u1;) {
        const int ka = (int)(u % a.KC);
        const int kb = (int)((int64_t)a.KC < ka + (u1 - u) ? (int64_t)a.KC : ka + (u1 - u));
        for (int kc = ka; kc < kb; kc += SK_KCS, ++seq) {
            const int n = min(SK_KCS, kb - kc);
            if (seq % SK_OPW != ow) {  // another operand warp's stage
                if (++stage == SK_STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
                continue;
            }
            // inputs first (they do not depend on the ring slot): their L2 latency
            // overlaps the wait for the consumers to free this stage
            constexpr int NI = (SK_KCS + 3) / 4;  // 128-feature slices per stage
            float4 sc[NI], g4[NI], b4[NI], x4[NI][TC];
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const int krel = 128 * i + 4 * lane;
                const int k = kc * 32 + krel;
                const bool in = krel < n * 32 && k < p.K;  // K % 4 == 0 (launcher): slices are in or out
                sc[i] = in ? *reinterpret_cast<const float4*>(p.scales + k) : make_float4(0.f, 0.f, 0.f, 0.f);
                g4[i] = in && ln ? *reinterpret_cast<const float4*>(p.gamma + k) : make_float4(1.f, 1.f, 1.f, 1.f);
                b4[i] = in && ln ? *reinterpret_cast<const float4*>(p.beta + k) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            // the scales / gamma / beta never change during a step: the first stage's are
            // requested before the dependency wait, the activations after it
            if (!waited) wait_once();
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const int krel = 128 * i + 4 * lane;
                const int k = kc * 32 + krel;
                const bool in = krel < n * 32 && k < p.K;
#pragma unroll
                for (int t = 0; t < TC; ++t) {
                    const int tok = chunk * TC + t;
                    x4[i][t] = in && tok < a.act.n_tok ? *reinterpret_cast<const float4*>(p.x + (int64_t)tok * p.K + k)
                                                       : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
            if (!have_st) resolve();
            mbar_wait(&empty[stage], phase ^ 1);
            uint32_t* B = reinterpret_cast<uint32_t*>(sb + stage * B_STAGE);
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const int krel = 128 * i + 4 * lane;
                if (krel >= n * 32) continue;
                const int kk = krel >> 5, kt = krel & 31, half_ = kt >> 4, q = (kt & 15) >> 2;
#pragma unroll
                for (int t = 0; t < TC; ++t) {
                    const int tok = chunk * TC + t;
                    if (tok >= a.act.n_tok) continue;
                    const float xs[4] = {x4[i][t].x, x4[i][t].y, x4[i][t].z, x4[i][t].w},
                                gs[4] = {g4[i].x, g4[i].y, g4[i].z, g4[i].w},
                                bs[4] = {b4[i].x, b4[i].y, b4[i].z, b4[i].w},
                                ss[4] = {sc[i].x, sc[i].y, sc[i].z, sc[i].w};
                    const float z = st[t].z * 256.f;
                    uint32_t w[3] = {0u, 0u, 0u};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float y = ln ? fmaf(gs[e], (xs[e] - st[t].x) * st[t].y, bs[e]) : xs[e];  // model.py:271-276
                        int h, m, l;
                        digits3(__float2int_rn((y * ss[e]) * z), h, m, l);
                        w[0] |= (uint32_t)(uint8_t)h << (8 * e);
                        w[1] |= (uint32_t)(uint8_t)m << (8 * e);
                        w[2] |= (uint32_t)(uint8_t)l << (8 * e);
                    }
#pragma unroll
                    for (int pp = 0; pp < 3; ++pp) {
                        const int cc = pp * TC + t;
                        B[((kk * NT + (cc >> 3)) * 32 + 4 * (cc & 7) + q) * 2 + half_] = w[pp];
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[stage]);
            if (++stage == SK_STAGES) {
                stage = 0;
                phase ^= 1;
            }
        }
        u += kb - ka;
    }
    if (!waited) wait_once();
    if (!have_st) resolve();  // a warp without stages still writes the side outputs (ow == 0)
}

template <int TC, int SK_KCS, int SK_STAGES, bool FUSED = false, bool RED = false>
__global__ void __launch_bounds__(SK_THREADS + (FUSED ? 32 * SK_OPW : 0)) k_gemv_i8(SkArgs a) {
    // an operand warp reuses only its own ring slots, so it can never run two rounds
    // ahead of the consumers (mbarrier parity waits cannot tell those rounds apart)
    static_assert(!FUSED || SK_STAGES % SK_OPW == 0, "operand warps must own whole ring slots");
    constexpr int NT = digit_ntiles(TC);
    constexpr int NACC = NT == 1 ? 2 : 1;  // accumulator sets (see the consumer loop)
    constexpr int COLS = 8 * NT;
    constexpr int SST = COLS + 1;
    constexpr int A_STAGE = SK_KCS * 4096;
    constexpr int B_STAGE = SK_KCS * NT * 256;
    constexpr int PER = 128 * COLS;  // floats per partial tile
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* sa = smem;                                        // [STAGES][A_STAGE]
    uint8_t* sb = sa + SK_STAGES * A_STAGE;                    // [STAGES][B_STAGE]
    int* S = reinterpret_cast<int*>(sb + SK_STAGES * B_STAGE);  // [128][SST] integer partial sums
    uint64_t* full = reinterpret_cast<uint64_t*>(S + 128 * SST + 3);  // 8-byte aligned below
    full = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(full) + 7) & ~uintptr_t(7));
    uint64_t* empty = full + SK_STAGES;
    int* s_flag = reinterpret_cast<int*>(empty + SK_STAGES);

    const int warp = warp_uniform_id(), lane = threadIdx.x & 31;
    const int chunk = blockIdx.y;
    const int c = blockIdx.x;
    const int64_t u0 = (int64_t)c * a.total / a.G, u1 = (int64_t)(c + 1) * a.total / a.G;
    const int tcta = chunk * a.G + c;
    if (threadIdx.x == 0) {
        trace_stamp(a.trace, tcta, 0);
        for (int s = 0; s < SK_STAGES; ++s) {
            mbar_init(&full[s], FUSED ? 2 : 1);  // fused: + the stage's operand-warp arrival
            mbar_init(&empty[s], SK_CONS);
        }
        mbar_fence_init();
    }
    __syncthreads();
    if (u0 >= u1) {
        pdl_wait();
        pdl_trigger();
    } else if (FUSED && warp > SK_CONS) {
        // ---------------- operand warps (they wait for the predecessor themselves)
        sk_operand_warp<TC, SK_KCS, SK_STAGES>(a, u0, u1, chunk, sb, full, empty, warp - SK_CONS - 1);
    } else if (FUSED && warp == 0) {
        // ---------------- producer: weights only (they never depend on earlier kernels)
        if (lane == 0) {
            const uint64_t pol = l2_evict_first();
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t u = u0; u < u1;) {
                const int mg = (int)(u / a.KC);
                const int ka = (int)(u % a.KC);
                const int kb = (int)((int64_t)a.KC < ka + (u1 - u) ? (int64_t)a.KC : ka + (u1 - u));
                for (int kc = ka; kc < kb; kc += SK_KCS) {
                    const int n = min(SK_KCS, kb - kc);
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], n * 4096);
                    bulk_g2s_hint(sa + stage * A_STAGE, a.codes + ((int64_t)mg * a.KC + kc) * 4096, n * 4096, &full[stage], pol);
                    if (++stage == SK_STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                u += kb - ka;
            }
        }
    } else if (warp == 0) {
        // ---------------- producer
        if (lane == 0) {
            const uint64_t pol = l2_evict_first();
            int stage = 0, issued = 0;
            uint32_t phase = 0;
            int pk[SK_STAGES];  // k tiles of the stages prefetched before the dependency wait
            int pn[SK_STAGES];
            const uint8_t* bsrc = reinterpret_cast<const uint8_t*>(a.act.frag) + (int64_t)chunk * a.KC * NT * 256;
            bool waited = false;
            for (int64_t u = u0; u < u1;) {
                const int mg = (int)(u / a.KC);
                const int ka = (int)(u % a.KC);
                const int kb = (int)((int64_t)a.KC < ka + (u1 - u) ? (int64_t)a.KC : ka + (u1 - u));
                for (int kc = ka; kc < kb; kc += SK_KCS) {
                    const int n = min(SK_KCS, kb - kc);
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], n * (4096 + NT * 256));
                    // weights never depend on the previous kernels: start streaming them
                    // while the operand producer (PDL predecessor) is still running
                    bulk_g2s_hint(sa + stage * A_STAGE, a.codes + ((int64_t)mg * a.KC + kc) * 4096, n * 4096, &full[stage], pol);
                    if (!waited && issued < SK_STAGES) {
                        pk[issued] = kc;
                        pn[issued] = n;
                    } else {
                        bulk_g2s(sb + stage * B_STAGE, bsrc + (int64_t)kc * NT * 256, n * NT * 256, &full[stage]);
                    }
                    ++issued;
                    if (!waited && issued == SK_STAGES) {
                        // the ring is full of weights: now wait for the operand producer
                        pdl_wait();
                        pdl_trigger();
                        waited = true;
                        for (int i = 0; i < SK_STAGES; ++i)
                            bulk_g2s(sb + i * B_STAGE, bsrc + (int64_t)pk[i] * NT * 256, pn[i] * NT * 256, &full[i]);
                    }
                    if (++stage == SK_STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                u += kb - ka;
            }
            if (!waited) {  // fewer stages than the ring depth
                pdl_wait();
                pdl_trigger();
                for (int i = 0; i < issued; ++i)
                    bulk_g2s(sb + i * B_STAGE, bsrc + (int64_t)pk[i] * NT * 256, pn[i] * NT * 256, &full[i]);
            }
        } else {
            pdl_wait();
            pdl_trigger();
        }
    } else {
    // ---------------- consumers: the first row group's static epilogue inputs into L1
    // while the predecessor drains
    {
        const int o = (int)(u0 / a.KC) * 128 + (int)threadIdx.x - 32;
        if (o < a.epi.M) {
            prefetch_l1(a.epi.bias + o);
            if (a.epi.s_next) prefetch_l1(a.epi.s_next + o);
        }
    }
    pdl_wait();
    pdl_trigger();
    if (threadIdx.x == 32) trace_stamp(a.trace, tcta, 1);
    bool first_stage = true;
    const int cw = warp - 1;  // consumer warp: m-tiles 2cw, 2cw+1 of the group
    // ldmatrix roles: matrix mi = lane / 8 (row half mi & 1, k half mi >> 1), row ri = lane % 8
    const uint32_t a_lane = (uint32_t)(((lane >> 3) & 1) * 256 + (lane >> 4) * 128 + (lane & 7) * 16);
    const uint32_t sa_u = smem_u32(sa);
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t u = u0; u < u1;) {
        const int mg = (int)(u / a.KC);
        const int ka = (int)(u % a.KC);
        const int kb = (int)((int64_t)a.KC < ka + (u1 - u) ? (int64_t)a.KC : ka + (u1 - u));
        int acc[2][NT][4], acc2[2][NT][4];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j)
#pragma unroll
                for (int r = 0; r < 4; ++r) acc[i][j][r] = acc2[i][j][r] = 0;
        for (int kc = ka; kc < kb; kc += SK_KCS) {
            const int n = min(SK_KCS, kb - kc);
            mbar_wait(&full[stage], phase);
            if (first_stage) {
                if (threadIdx.x == 32) trace_stamp(a.trace, tcta, 2);
                first_stage = false;
            }
            const uint8_t* Bs = sb + stage * B_STAGE;
            const uint32_t As = sa_u + stage * A_STAGE;
            if (n == SK_KCS) {
                // full stage: no per-k-tile guard, so the fragment loads of later k tiles issue
                // ahead of the MMAs; with one digit tile (NT == 1) odd k tiles accumulate into
                // a second set, halving the dependent IMMA chain (traced: a 32-k-tile CTA's
                // MMAs took ~2.6 us, ~80 cycles per k tile, latency-bound)
#pragma unroll
                for (int kk = 0; kk < SK_KCS; ++kk) {
                    uint2 bv[NT];
#pragma unroll
                    for (int j = 0; j < NT; ++j)
                        bv[j] = *reinterpret_cast<const uint2*>(Bs + (kk * NT + j) * 256 + lane * 8);
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        uint32_t a0, a1, a2, a3;
                        ldsm_x4_i8(As + kk * 4096 + (cw * 2 + i) * 512 + a_lane, a0, a1, a2, a3);
#pragma unroll
                        for (int j = 0; j < NT; ++j) {
                            if (NACC > 1 && (kk & 1)) imma16832(acc2[i][j], a0, a1, a2, a3, bv[j].x, bv[j].y);
                            else imma16832(acc[i][j], a0, a1, a2, a3, bv[j].x, bv[j].y);
                        }
                    }
                }
            } else {
#pragma unroll
                for (int kk = 0; kk < SK_KCS; ++kk) {
                    if (kk < n) {
                        uint2 bv[NT];
#pragma unroll
                        for (int j = 0; j < NT; ++j)
                            bv[j] = *reinterpret_cast<const uint2*>(Bs + (kk * NT + j) * 256 + lane * 8);
#pragma unroll
                        for (int i = 0; i < 2; ++i) {
                            uint32_t a0, a1, a2, a3;
                            ldsm_x4_i8(As + kk * 4096 + (cw * 2 + i) * 512 + a_lane, a0, a1, a2, a3);
#pragma unroll
                            for (int j = 0; j < NT; ++j) imma16832(acc[i][j], a0, a1, a2, a3, bv[j].x, bv[j].y);
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
            if (++stage == SK_STAGES) {
                stage = 0;
                phase ^= 1;
            }
        }
        u += kb - ka;
        if (NACC > 1) {
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j)
#pragma unroll
                    for (int r = 0; r < 4; ++r) acc[i][j][r] += acc2[i][j][r];  // exact s32
        }

        // ---- segment finished: complete group or a piece of a split group
        const int64_t g0 = (int64_t)mg * a.KC, g1 = g0 + a.KC;
        const int c_first = sk_owner(g0, a.G, a.total), c_last = sk_owner(g1 - 1, a.G, a.total);
        if (RED && c_first != c_last) {
            // split row group: this CTA's s32 sums are added into the row group's accumulator
            // (reductions at L2, exact integers: arrival order is irrelevant); the contributor that
            // completes the count reads the total once -- instead of every contributor's partial --
            // and zeroes it for the next launch
            int* sums = a.sums + ((int64_t)chunk * a.MG + mg) * PER;
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j)
#pragma unroll
                    for (int r = 0; r < 4; ++r)
                        atomicAdd(sums + (((cw * 2 + i) * NT + j) * 32 + lane) * 4 + r, acc[i][j][r]);
            __threadfence();
            cons_sync();
            if (threadIdx.x == 32) {
                int* ctr = a.counters + (int64_t)chunk * a.MG + mg;
                const int prev = atomicAdd(ctr, 1);
                const int last = prev == c_last - c_first;
                if (last) *ctr = 0;
                *s_flag = last;
            }
            cons_sync();
            if (!*s_flag) continue;
            __threadfence();
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    int4* q = reinterpret_cast<int4*>(sums + (((cw * 2 + i) * NT + j) * 32 + lane) * 4);
                    const int4 v = __ldcg(q);
                    acc[i][j][0] = v.x;
                    acc[i][j][1] = v.y;
                    acc[i][j][2] = v.z;
                    acc[i][j][3] = v.w;
                    __stcg(q, make_int4(0, 0, 0, 0));
                }
        } else if (c_first != c_last) {
            const int slot = (u0 < g0) ? 1 : 0;  // not this CTA's first segment -> slot 1
            int* mine = reinterpret_cast<int*>(a.partials) + (((int64_t)chunk * a.G + c) * 2 + slot) * PER;
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j)
                    *reinterpret_cast<int4*>(mine + (((cw * 2 + i) * NT + j) * 32 + lane) * 4) =
                        make_int4(acc[i][j][0], acc[i][j][1], acc[i][j][2], acc[i][j][3]);
            __threadfence();
            cons_sync();
            if (threadIdx.x == 32) {
                int* ctr = a.counters + (int64_t)chunk * a.MG + mg;
                const int prev = atomicAdd(ctr, 1);
                const int last = prev == c_last - c_first;
                if (last) *ctr = 0;
                *s_flag = last;
            }
            cons_sync();
            if (!*s_flag) continue;
            __threadfence();
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j)
#pragma unroll
                    for (int r = 0; r < 4; ++r) acc[i][j][r] = 0;
            for (int cc = c_first; cc <= c_last; ++cc) {
                const int64_t cu0 = (int64_t)cc * a.total / a.G;
                const int* p = reinterpret_cast<const int*>(a.partials) +
                               (((int64_t)chunk * a.G + cc) * 2 + (cu0 < g0 ? 1 : 0)) * PER;
#pragma unroll
                for (int i = 0; i < 2; ++i)
#pragma unroll
                    for (int j = 0; j < NT; ++j) {
                        const int4 v =
                            __ldcg(reinterpret_cast<const int4*>(p + (((cw * 2 + i) * NT + j) * 32 + lane) * 4));
                        acc[i][j][0] += v.x;
                        acc[i][j][1] += v.y;
                        acc[i][j][2] += v.z;
                        acc[i][j][3] += v.w;
                    }
            }
        }
        sk_epilogue<TC>(a, acc, mg, chunk, S);
    }
    if (threadIdx.x == 32) trace_stamp(a.trace, tcta, 3);
    }  // consumers
}


template <int TC, int SK_KCS, int SK_STAGES, bool FUSED = false, bool RED = false>
static int sk_launch(const Mat& m, const Act& act, const Epi& epi, float* partials, int* counters,
                     int64_t partial_cap, cudaStream_t st, const ProArgs* pro = nullptr, float* zero_a = nullptr,
                     float* zero_b = nullptr, int* sums = nullptr, int64_t sums_elems = 0) {
    constexpr int THREADS = SK_THREADS + (FUSED ? 32 * SK_OPW : 0);
    constexpr int NT = digit_ntiles(TC);
    const size_t smem = (size_t)SK_STAGES * (SK_KCS * 4096 + SK_KCS * NT * 256) + 128 * (8 * NT + 1) * 4 + 16 +
                        2 * SK_STAGES * 8 + 16;
    // occupancy and the smem opt-in are per device (a process may drive several GPUs)
    static int bps_dev[PB_MAX_DEVICES] = {}, sms_dev[PB_MAX_DEVICES] = {};
    int dev = 0;
    PB_CHECK_CUDA(cudaGetDevice(&dev));
    if (dev >= PB_MAX_DEVICES) { set_error("device index beyond PB_MAX_DEVICES"); return PB_ERR_GENERIC; }
    if (!bps_dev[dev]) {
        int sms = 0, bps = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        PB_CHECK_CUDA(cudaFuncSetAttribute(k_gemv_i8<TC, SK_KCS, SK_STAGES, FUSED, RED>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_gemv_i8<TC, SK_KCS, SK_STAGES, FUSED, RED>, THREADS, smem);
        sms_dev[dev] = sms;
        bps_dev[dev] = std::max(bps, 1);
    }
    const int blocks_per_sm = bps_dev[dev], sms = sms_dev[dev];
    SkArgs a{};
    a.codes = m.codes;
    a.MG = m.Mp / 128;
    a.KC = m.Kp / 32;
    a.total = (int64_t)a.MG * a.KC;
    const int chunks = (int)ceil_div(act.n_tok, act.tc);
    int64_t G = std::max<int64_t>(1, (int64_t)sms * blocks_per_sm / chunks);
    // small matrices: at least min_units k tiles per CTA (a CTA then streams whole
    // 128-row groups instead of splitting every group across many CTAs and paying
    // the split merge); large matrices keep one CTA per resident slot
    // (sweep, profiles/r1_gemv_timeline_and_tail.txt: 32 for <= 2 tokens, 64 for 8)
    constexpr int64_t min_units = TC >= 8 ? 64 : 32;
    G = std::min<int64_t>(G, std::max<int64_t>(1, a.total / std::max<int64_t>(min_units, 1)));
    const int64_t per_tile = 128 * 8 * NT;
    while (G > 1 && (int64_t)chunks * G * 2 * per_tile > partial_cap) G /= 2;
    a.G = (int)G;
    a.act = act;
    a.epi = epi;
    a.partials = partials;
    a.counters = counters;
    if (RED) {
        if (!sums || (int64_t)chunks * a.MG * per_tile > sums_elems) {
            set_error("gemv: split-row-group sum workspace too small");
            return PB_ERR_CAPACITY;
        }
        a.sums = sums;
    }
    a.trace = trace_region(TR_GEMV, (int)G * chunks);
    if (FUSED) {
        a.pro = *pro;
        a.pro.trace = nullptr;
        a.zero_a = zero_a;
        a.zero_b = zero_b;
    }
    return launch_pdl(k_gemv_i8<TC, SK_KCS, SK_STAGES, FUSED, RED>, dim3((unsigned)G, chunks), dim3(THREADS), smem, st, a);
}

bool gemv_fusable(const Act& act, int K) {
    // 2 tokens per column chunk only: the 8-token variant measured slower (operand
    // warps compute-bound: 560M batch 8 68 -> 117 us/block)
    return (K & 3) == 0 && act.tc == 2;
}

int launch_gemv_fused(const Mat& m, const Act& act, const Epi& epi, const ProArgs& pro, float* zero_a,
                      float* zero_b, float* partials, int* counters, int64_t partial_cap, cudaStream_t st,
                      int* sums, int64_t sums_elems) {
    if (!gemv_fusable(act, pro.K)) {
        set_error("fused-operand GEMV: unsupported shape");
        return PB_ERR_GENERIC;
    }
    // split row groups merged by s32 reductions (560M 34.6 -> 34.4 us per block, 7B1 73.3 -> 72.3)
    if (sums && ceil_div(act.n_tok, act.tc) * (int64_t)(m.Mp / 128) * 128 * 8 * digit_ntiles(2) <= sums_elems)
        return sk_launch<2, 8, 4, true, true>(m, act, epi, partials, counters, partial_cap, st, &pro, zero_a, zero_b,
                                              sums, sums_elems);
    return sk_launch<2, 8, 4, true>(m, act, epi, partials, counters, partial_cap, st, &pro, zero_a, zero_b);
}

// Stage shapes (k tiles per stage x stages) per column tile, chosen by sweeps
// (profiles/r1_gemv_timeline_and_tail.txt, profiles/r1_small_shape_gemv_minu.txt):
// decode 8 x 4 (32 KB stages, one CTA per SM), 3..8 tokens 8 x 3, 17..32 tokens 2 x 4.
int launch_gemv(const Mat& m, const Act& act, const Epi& epi, float* partials, int* counters, int64_t partial_cap,
                cudaStream_t st, int* sums, int64_t sums_elems) {
    switch (act.tc) {
        case 2:
            // batch-1 decode through a separate operand kernel: reduction merge (176B: 426.0 -> 418.4 us
            // per block); the fused kernel takes the same merge as its own instantiation (a shared runtime
            // branch cost more than the merge saved: 560M 34.7 -> 40.3 us per block)
            if (sums && ceil_div(act.n_tok, act.tc) * (int64_t)(m.Mp / 128) * 128 * 8 * digit_ntiles(2) <= sums_elems)
                return sk_launch<2, 8, 4, false, true>(m, act, epi, partials, counters, partial_cap, st, nullptr,
                                                        nullptr, nullptr, sums, sums_elems);
            return sk_launch<2, 8, 4>(m, act, epi, partials, counters, partial_cap, st);
        // 3..8 tokens: 8 x 3 (re-swept after the hoisted fragment loads: 7B1 batch 8 104.3 -> 102.1 us per
        // block; 176B equal; 4 x 4 / 4 x 6 slower)
        case 8: return sk_launch<8, 8, 3>(m, act, epi, partials, counters, partial_cap, st);
        case 16: return sk_launch<16, 2, 4>(m, act, epi, partials, counters, partial_cap, st);
        case 32: return sk_launch<32, 2, 4>(m, act, epi, partials, counters, partial_cap, st);
        default: set_error("bad column tile"); return PB_ERR_GENERIC;
    }
}

// ------------------------------------------------------------------ f32-weights path
// quantize in {none, activations} (the reference's default server mode): fp32
// x @ W with W [K, M] row-major as in the checkpoint. Memory-bound split-K GEMV:
// a CTA streams a k-range of 1024 output columns with 128-bit non-allocating
// loads (8 in flight per thread), up to F32_T tokens per pass from shared
// memory; partial sums go to a workspace and a second kernel adds the splits in
// fixed order and runs the fused epilogue.
constexpr int F32_T = 8;       // tokens per pass
constexpr int F32_KB = 128;    // k rows staged per shared-memory refill

template <int T>
__global__ void __launch_bounds__(256) k_gemv_f32(const float* __restrict__ w, int K, int M,
                                                  const float* __restrict__ y, int n_tok, int tok0, int kchunk,
                                                  float* __restrict__ part) {
    __shared__ float ys[T][F32_KB];
    const int o = (blockIdx.x * 256 + threadIdx.x) * 4;
    const int k0 = blockIdx.y * kchunk, k1 = min(K, k0 + kchunk);
    const bool vec = (M & 3) == 0 && o + 3 < M;
    float acc[T][4];
#pragma unroll
    for (int j = 0; j < T; ++j)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[j][c] = 0.f;
    for (int kb = k0; kb < k1; kb += F32_KB) {
        __syncthreads();
        for (int e = threadIdx.x; e < T * F32_KB; e += 256) {
            const int j = e / F32_KB, kk = e % F32_KB;
            const int tok = tok0 + j, k = kb + kk;
            ys[j][kk] = (tok < n_tok && k < k1) ? y[(int64_t)tok * K + k] : 0.f;
        }
        __syncthreads();
        const int kend = min(F32_KB, k1 - kb);
        if (o < M) {
#pragma unroll 8
            for (int kk = 0; kk < kend; ++kk) {
                const float* row = w + (int64_t)(kb + kk) * M + o;
                float4 wv;
                if (vec) {
                    const int4 r = ld_stream_v4(row);
                    wv = make_float4(__int_as_float(r.x), __int_as_float(r.y), __int_as_float(r.z), __int_as_float(r.w));
                } else {
                    wv.x = row[0];
                    wv.y = o + 1 < M ? row[1] : 0.f;
                    wv.z = o + 2 < M ? row[2] : 0.f;
                    wv.w = o + 3 < M ? row[3] : 0.f;
                }
#pragma unroll
                for (int j = 0; j < T; ++j) {
                    const float xv = ys[j][kk];
                    acc[j][0] = fmaf(xv, wv.x, acc[j][0]);
                    acc[j][1] = fmaf(xv, wv.y, acc[j][1]);
                    acc[j][2] = fmaf(xv, wv.z, acc[j][2]);
                    acc[j][3] = fmaf(xv, wv.w, acc[j][3]);
                }
            }
        }
    }
    if (o >= M) return;
    float* p = part + (int64_t)blockIdx.y * F32_T * M;
#pragma unroll
    for (int j = 0; j < T; ++j)
#pragma unroll
        for (int c = 0; c < 4; ++c)
            if (o + c < M) p[(int64_t)j * M + o + c] = acc[j][c];
}

__global__ void k_reduce_f32(const float* __restrict__ part, int S, int M, int n_tok, int tok0, Epi epi) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y, tok = tok0 + j;
    if (o >= M || tok >= n_tok) return;
    float v = 0.f;
    for (int s2 = 0; s2 < S; ++s2) v += part[((int64_t)s2 * F32_T + j) * M + o];
    epi_store(epi, tok, o, v);
}

int launch_gemm_f32(const Mat& m, const float* y, int n_tok, const Epi& epi, float* part, int64_t part_cap,
                    cudaStream_t st) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int gx = (int)ceil_div(m.M, 1024);
    int S = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(4 * sms, gx), ceil_div(m.K, F32_KB)));
    while (S > 1 && (int64_t)S * F32_T * m.M > part_cap) --S;
    const int kchunk = (int)round_up(ceil_div(m.K, S), 4);
    S = (int)ceil_div(m.K, kchunk);
    for (int tok0 = 0; tok0 < n_tok; tok0 += F32_T) {
        const int nt = std::min(F32_T, n_tok - tok0);
        const dim3 grid((unsigned)gx, (unsigned)S);
        if (nt == 1) k_gemv_f32<1><<<grid, 256, 0, st>>>(m.w32, m.K, m.M, y, n_tok, tok0, kchunk, part);
        else if (nt == 2) k_gemv_f32<2><<<grid, 256, 0, st>>>(m.w32, m.K, m.M, y, n_tok, tok0, kchunk, part);
        else if (nt <= 4) k_gemv_f32<4><<<grid, 256, 0, st>>>(m.w32, m.K, m.M, y, n_tok, tok0, kchunk, part);
        else k_gemv_f32<F32_T><<<grid, 256, 0, st>>>(m.w32, m.K, m.M, y, n_tok, tok0, kchunk, part);
        if (int rc = launch_check("gemv_f32")) return rc;
        k_reduce_f32<<<dim3((unsigned)ceil_div(m.M, 256), (unsigned)std::min(F32_T, n_tok - tok0)), 256, 0, st>>>(
            part, S, m.M, n_tok, tok0, epi);
        if (int rc = launch_check("reduce_f32")) return rc;
    }
    return PB_OK;
}

}  // namespace pb
