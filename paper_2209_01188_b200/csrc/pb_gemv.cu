// int8-weight GEMV/GEMM for the block executor (quant.py:117-129 matmul_mixed,
// model.py:305-311 _mm) plus the fused prologues/epilogues of block_forward
// (model.py:340-368).
//
// Math: y[n, o] = sum_k code[o, k] * (s_k * x[n, k]) + sum_j W[k_j, o] x[n, k_j] + b[o]
// The per-input-feature scale s_k is folded into the activation (x~ = s ⊙ x)
// so the weight stream is raw int8 codes. x~ is split hi/lo into two fp16
// operands after a per-token power-of-two shift (max |x~| -> [2^13, 2^14)),
// so codes (exact in fp16) times (hi + lo) reproduces the f32 activation to
// ~22 bits with fp32 accumulation on the tensor cores (mma.m16n8k16); the
// epilogue undoes the shift exactly.
//
// Memory-bound decode: every warp streams 512 B fragment tiles of codes with
// 128-bit non-allocating loads (one per lane), converts int8 -> fp16 with a
// PRMT/HSUB2 magic-number trick (exact for |c| <= 127) and issues 2 mma per
// 16 B of codes per column tile. B fragments are shared by the 4 warps of a
// CTA through L1. Deterministic split-K: partial tiles go to a workspace and
// the last-arriving CTA sums the splits in fixed order and runs the epilogue.
//
// B (activation) fragment layout, chunk c of tc tokens (columns: tc hi then tc lo):
//   uint4 at ((c * KC + kc) * NT + nt) * 32 + lane, NT = 2 tc / 8,
//   words {kt0: B[2q..2q+1][g], B[2q+8..2q+9][g]; kt1: same +16}, column = 8 nt + g.
#include "pb_common.cuh"
#include "pb_span.h"

namespace pb {

constexpr int GEMV_WARPS = 4;
constexpr int GEMV_MW = 2;                              // m-tiles per warp
constexpr int GEMV_ROWS = GEMV_WARPS * GEMV_MW * 16;    // 128 rows per CTA
constexpr int GEMV_UNROLL = 4;

int choose_tc(int n_tok) {
    if (n_tok <= 4) return 4;
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

struct ProArgs {
    int mode;
    const float* x;
    int K, Kp;
    const float* gamma;
    const float* beta;
    const float* scales;  // nullptr in f32 mode
    int n_outl;
    const int32_t* outl_idx;
    int tc;
    uint4* frag;
    float* back;   // [n_tok] 2^-shift (epilogue rescale)
    float4* stats; // [n_tok] {mu, inv, 2^shift, -}
    float* xo;
    float* y32;
};

__device__ __forceinline__ float pro_y(const ProArgs& a, const float* x, int k, float mu, float inv) {
    if (a.mode == PRO_LN) return fmaf(a.gamma[k], (x[k] - mu) * inv, a.beta[k]);  // model.py:271-276
    return x[k];
}

// Row statistics, one CTA per token: LayerNorm mean / inverse std (population
// variance, eps 1e-5; accumulated in f64) and the power-of-two shift that maps
// max |y * s| into [2^13, 2^14) for the hi/lo fp16 split.
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
        a.stats[tok] = make_float4(mu, inv, ldexpf(1.f, shift), 0.f);
    }
}

// hi/lo fp16 B fragments of x~ = y * s * 2^shift (layout in the header comment);
// one thread per (token, 32-wide k chunk, lane quad q).
__global__ void __launch_bounds__(256) k_fragwrite(ProArgs a) {
    const int tok = blockIdx.y;
    const float* x = a.x + (int64_t)tok * a.K;
    const float4 st = a.stats[tok];
    const int KC = a.Kp / 32;
    const int it = blockIdx.x * blockDim.x + threadIdx.x;
    if (blockIdx.x == 0 && a.xo) {
        for (int j = threadIdx.x; j < a.n_outl; j += blockDim.x)
            a.xo[(int64_t)tok * a.n_outl + j] = pro_y(a, x, a.outl_idx[j], st.x, st.y);
    }
    if (it >= KC * 4) return;
    const int kc = it >> 2, q = it & 3;
    const int NT = a.tc / 4;
    const int c = tok / a.tc, col = tok % a.tc;
    const int nt_hi = col >> 3, g_hi = col & 7;
    const int nt_lo = (a.tc + col) >> 3, g_lo = (a.tc + col) & 7;
    uint32_t hw[4], lw[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        const int kt = w >> 1, upper = w & 1;
        const int k0 = kc * 32 + kt * 16 + 2 * q + 8 * upper;
        float v[2];
#pragma unroll
        for (int e2 = 0; e2 < 2; ++e2) {
            const int k = k0 + e2;
            v[e2] = k < a.K ? (pro_y(a, x, k, st.x, st.y) * a.scales[k]) * st.z : 0.f;
        }
        const half h0 = __float2half_rn(v[0]), h1 = __float2half_rn(v[1]);
        const half l0 = __float2half_rn(v[0] - __half2float(h0));
        const half l1 = __float2half_rn(v[1] - __half2float(h1));
        hw[w] = (uint32_t)__half_as_ushort(h0) | ((uint32_t)__half_as_ushort(h1) << 16);
        lw[w] = (uint32_t)__half_as_ushort(l0) | ((uint32_t)__half_as_ushort(l1) << 16);
    }
    const int64_t base = ((int64_t)c * KC + kc) * NT;
    a.frag[(base + nt_hi) * 32 + 4 * g_hi + q] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    a.frag[(base + nt_lo) * 32 + 4 * g_lo + q] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
}

// f32-weights mode: plain y = LN(x) (or x) rows for the CUDA-core GEMM
__global__ void __launch_bounds__(256) k_rows_f32(ProArgs a) {
    const int tok = blockIdx.y;
    const float* x = a.x + (int64_t)tok * a.K;
    const float4 st = a.stats[tok];
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < a.K; k += gridDim.x * blockDim.x)
        a.y32[(int64_t)tok * a.K + k] = pro_y(a, x, k, st.x, st.y);
}

int launch_prologue(int mode, const float* x, int n_tok, int K, int Kp, const float* gamma, const float* beta,
                    const Mat& m, int tc, uint4* frag, float* back, float4* stats, float* xo, float* y32,
                    cudaStream_t st) {
    ProArgs a{mode, x, K, Kp, gamma, beta, y32 ? nullptr : m.scales, m.n_outl, m.outl_idx, tc, frag, back, stats,
              xo, y32};
    if (mode == PRO_LN || !y32) {
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
    const int items = (Kp / 32) * 4;
    k_fragwrite<<<dim3((unsigned)ceil_div(items, 256), n_tok), 256, 0, st>>>(a);
    return launch_check("fragwrite");
}

// ------------------------------------------------------------------ epilogue

__device__ __forceinline__ float gelu_tanh(float x) {  // model.py:286-292 (f32)
    const float c = 0.7978845608028654f;
    const float u = c * (x + 0.044715f * x * x * x);
    return 0.5f * x * (1.f + tanhf(u));
}

__device__ __forceinline__ void epi_store(const Epi& e, int tok, int o, float v) {
    v += e.bias[o];
    for (int j = 0; j < e.n_outl; ++j) v = fmaf(e.outl_rows[(int64_t)j * e.M + o], e.xo[(int64_t)tok * e.n_outl + j], v);
    const int64_t idx = (int64_t)tok * e.M + o;
    if (e.kind == EPI_RESID) {
        e.out[idx] = e.resid[idx] + v;
    } else if (e.kind == EPI_GELU) {
        e.out[idx] = gelu_tanh(v);
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
            e.kv[((((int64_t)page * 2 + part) * e.H + h) * e.P + slot) * e.dh + dd] = __float2half_rn(v);
        }
    }
}

// ------------------------------------------------------------------ int8 mma GEMV

__device__ __forceinline__ void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// 4 int8 (one word) -> two f16x2: {b0,b1}, {b2,b3}; exact for |c| <= 127.
__device__ __forceinline__ void i8x4_to_f16x2(uint32_t w, uint32_t& lo, uint32_t& hi) {
    const uint32_t u = w ^ 0x80808080u;                 // offset binary: c + 128
    const uint32_t p0 = __byte_perm(u, 0x64646464u, 0x4140);  // {1024 + b0', 1024 + b1'}
    const uint32_t p1 = __byte_perm(u, 0x64646464u, 0x4342);
    const half2 bias = __halves2half2(__ushort_as_half(0x6480), __ushort_as_half(0x6480));  // 1152
    half2 r0 = __hsub2(*reinterpret_cast<const half2*>(&p0), bias);
    half2 r1 = __hsub2(*reinterpret_cast<const half2*>(&p1), bias);
    lo = *reinterpret_cast<uint32_t*>(&r0);
    hi = *reinterpret_cast<uint32_t*>(&r1);
}

template <int NT>
__global__ void __launch_bounds__(GEMV_WARPS * 32) k_gemv_i8(const int8_t* __restrict__ codes, int MT, int KC,
                                                             int kc_per_split, Act act, Epi epi,
                                                             float* __restrict__ partials, int* __restrict__ counters) {
    constexpr int TC = NT * 4;
    constexpr int SST = 2 * TC + 1;
    __shared__ float S[GEMV_ROWS * SST];
    __shared__ int s_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, q = lane & 3;
    const int chunk = blockIdx.y, split = blockIdx.z, nsplit = gridDim.z;
    const int mt0 = blockIdx.x * (GEMV_WARPS * GEMV_MW) + warp * GEMV_MW;
    const int kc_begin = split * kc_per_split;
    const int kc_end = min(KC, kc_begin + kc_per_split);

    float acc[GEMV_MW][NT][4];
#pragma unroll
    for (int i = 0; i < GEMV_MW; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.f;

    const uint4* bf = act.frag + (int64_t)chunk * KC * NT * 32 + lane;
    bool mvalid[GEMV_MW];
    const int8_t* ap[GEMV_MW];
#pragma unroll
    for (int i = 0; i < GEMV_MW; ++i) {
        mvalid[i] = (mt0 + i) < MT;
        ap[i] = codes + ((int64_t)(mvalid[i] ? mt0 + i : 0) * KC) * 512 + lane * 16;
    }

    for (int kc0 = kc_begin; kc0 < kc_end; kc0 += GEMV_UNROLL) {
        int4 av[GEMV_UNROLL][GEMV_MW];
        uint4 bv[GEMV_UNROLL][NT];
#pragma unroll
        for (int u = 0; u < GEMV_UNROLL; ++u) {
            const int kc = kc0 + u;
            const bool kv = kc < kc_end;
#pragma unroll
            for (int i = 0; i < GEMV_MW; ++i)
                av[u][i] = (kv && mvalid[i]) ? ld_stream_v4(ap[i] + (int64_t)kc * 512) : make_int4(0, 0, 0, 0);
#pragma unroll
            for (int j = 0; j < NT; ++j) bv[u][j] = kv ? bf[((int64_t)kc * NT + j) * 32] : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < GEMV_UNROLL; ++u) {
#pragma unroll
            for (int i = 0; i < GEMV_MW; ++i) {
                uint32_t a[8];
                i8x4_to_f16x2((uint32_t)av[u][i].x, a[0], a[1]);
                i8x4_to_f16x2((uint32_t)av[u][i].y, a[2], a[3]);
                i8x4_to_f16x2((uint32_t)av[u][i].z, a[4], a[5]);
                i8x4_to_f16x2((uint32_t)av[u][i].w, a[6], a[7]);
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    mma16816(acc[i][j], a[0], a[1], a[2], a[3], bv[u][j].x, bv[u][j].y);
                    mma16816(acc[i][j], a[4], a[5], a[6], a[7], bv[u][j].z, bv[u][j].w);
                }
            }
        }
    }

    if (nsplit > 1) {
        // deterministic split-K: stash, count, last CTA reduces in split order
        constexpr int PER_CTA = GEMV_WARPS * GEMV_MW * NT * 32 * 4;
        const int64_t tile_id = (int64_t)chunk * gridDim.x + blockIdx.x;
        float* mine = partials + (tile_id * nsplit + split) * PER_CTA;
#pragma unroll
        for (int i = 0; i < GEMV_MW; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j)
                *reinterpret_cast<float4*>(mine + (((warp * GEMV_MW + i) * NT + j) * 32 + lane) * 4) =
                    make_float4(acc[i][j][0], acc[i][j][1], acc[i][j][2], acc[i][j][3]);
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) {
            const int prev = atomicAdd(counters + tile_id, 1);
            s_last = prev == nsplit - 1;
        }
        __syncthreads();
        if (!s_last) return;
        __threadfence();
        if (threadIdx.x == 0) counters[tile_id] = 0;  // ready for the next launch
#pragma unroll
        for (int i = 0; i < GEMV_MW; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j)
#pragma unroll
                for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.f;
        for (int s = 0; s < nsplit; ++s) {
            const float* p = partials + (tile_id * nsplit + s) * PER_CTA;
#pragma unroll
            for (int i = 0; i < GEMV_MW; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    const float4 v = __ldcg(reinterpret_cast<const float4*>(p + (((warp * GEMV_MW + i) * NT + j) * 32 + lane) * 4));
                    acc[i][j][0] += v.x;
                    acc[i][j][1] += v.y;
                    acc[i][j][2] += v.z;
                    acc[i][j][3] += v.w;
                }
        }
    }

    // C fragments -> smem [row][col]
#pragma unroll
    for (int i = 0; i < GEMV_MW; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int row = (warp * GEMV_MW + i) * 16 + g + 8 * (r >> 1);
                const int col = j * 8 + 2 * q + (r & 1);
                S[row * SST + col] = acc[i][j][r];
            }
    __syncthreads();
    const int row_base = blockIdx.x * GEMV_ROWS;
    for (int t = threadIdx.x; t < GEMV_ROWS * TC; t += blockDim.x) {
        const int r = t % GEMV_ROWS, j = t / GEMV_ROWS;
        const int o = row_base + r;
        const int tok = chunk * TC + j;
        if (o >= epi.M || tok >= act.n_tok) continue;
        const float v = (S[r * SST + j] + S[r * SST + TC + j]) * act.back[tok];
        epi_store(epi, tok, o, v);
    }
}

int launch_gemv(const Mat& m, const Act& act, const Epi& epi, float* partials, int* counters, int64_t partial_cap,
                cudaStream_t st) {
    const int MT = m.Mp / 16, KC = m.Kp / 32;
    const int gx = (int)ceil_div(MT, GEMV_WARPS * GEMV_MW);
    const int chunks = (int)ceil_div(act.n_tok, act.tc);
    const int NT = act.tc / 4;
    // split K so the grid covers the machine a few times over; >= 4 k-chunks per split
    int splits = (int)ceil_div(148 * 8, (int64_t)gx * chunks);
    splits = std::max(1, std::min(splits, KC / 4));
    const int64_t per_cta = (int64_t)GEMV_WARPS * GEMV_MW * NT * 32 * 4;
    while (splits > 1 && (int64_t)gx * chunks * splits * per_cta > partial_cap) --splits;
    int kc_per = (int)ceil_div(KC, splits);
    kc_per = (int)round_up(kc_per, GEMV_UNROLL);
    splits = (int)ceil_div(KC, kc_per);
    dim3 grid(gx, chunks, splits);
    switch (NT) {
        case 1: k_gemv_i8<1><<<grid, GEMV_WARPS * 32, 0, st>>>(m.codes, MT, KC, kc_per, act, epi, partials, counters); break;
        case 2: k_gemv_i8<2><<<grid, GEMV_WARPS * 32, 0, st>>>(m.codes, MT, KC, kc_per, act, epi, partials, counters); break;
        case 4: k_gemv_i8<4><<<grid, GEMV_WARPS * 32, 0, st>>>(m.codes, MT, KC, kc_per, act, epi, partials, counters); break;
        case 8: k_gemv_i8<8><<<grid, GEMV_WARPS * 32, 0, st>>>(m.codes, MT, KC, kc_per, act, epi, partials, counters); break;
        default: set_error("bad column tile"); return PB_ERR_GENERIC;
    }
    return launch_check("gemv_i8");
}

// ------------------------------------------------------------------ f32-weights path
// quantize in {none, activations}: reference fp32 matmul x @ W, W [K, M] row-major.
constexpr int F32_TOK = 8;

__global__ void __launch_bounds__(128) k_gemm_f32(const float* __restrict__ w, int K, int M, const float* __restrict__ y,
                                                  int n_tok, Epi epi) {
    __shared__ float ys[F32_TOK][64];
    const int o = blockIdx.x * 128 + threadIdx.x;
    const int tok0 = blockIdx.y * F32_TOK;
    float acc[F32_TOK];
#pragma unroll
    for (int j = 0; j < F32_TOK; ++j) acc[j] = 0.f;
    for (int k0 = 0; k0 < K; k0 += 64) {
        __syncthreads();
        for (int t = threadIdx.x; t < F32_TOK * 64; t += 128) {
            const int j = t / 64, kk = t % 64;
            const int tok = tok0 + j, k = k0 + kk;
            ys[j][kk] = (tok < n_tok && k < K) ? y[(int64_t)tok * K + k] : 0.f;
        }
        __syncthreads();
        if (o < M) {
            const int kend = min(64, K - k0);
            for (int kk = 0; kk < kend; ++kk) {
                const float wv = w[(int64_t)(k0 + kk) * M + o];
#pragma unroll
                for (int j = 0; j < F32_TOK; ++j) acc[j] = fmaf(ys[j][kk], wv, acc[j]);
            }
        }
    }
    if (o >= M) return;
    for (int j = 0; j < F32_TOK; ++j)
        if (tok0 + j < n_tok) epi_store(epi, tok0 + j, o, acc[j]);
}

int launch_gemm_f32(const Mat& m, const float* y, int n_tok, const Epi& epi, cudaStream_t st) {
    dim3 grid((unsigned)ceil_div(m.M, 128), (unsigned)ceil_div(n_tok, F32_TOK));
    k_gemm_f32<<<grid, 128, 0, st>>>(m.w32, m.K, m.M, y, n_tok, epi);
    return launch_check("gemm_f32");
}

}  // namespace pb
