// Training path of a span: the exact BACKWARD of block_forward
// (model.py:383-418 block_backward, served as server.py:431-450) for one row of
// a FORWARD batch (positions 0 .. t-1, empty cache: server.py:418-425).
//
// Tape-less recompute: the FORWARD step records only each block's input rows
// (pb_span_step_tape); BACKWARD recomputes the block's intermediates from them
// (LN1, qkv, softmax probabilities, ctx, mid, LN2, pre-activation) and then
// runs the reference backward formulas, so the gradient is that of the
// function the span's FORWARD computes.
//
// int8 matrices run on the tcgen05 GEMM (pb_gemm_tc.cu) in both directions:
// the recompute exactly as FORWARD's prefill does it, the backward product
// g W^T over a per-call transposed copy of the codes (see mm_bwd_tc). f32
// matrices (test spans) use one tiled SIMT kernel (64 x 64 tiles, f32
// accumulation) in either orientation. Attention works on [H][t][t]
// probability and score-gradient planes.
#include <algorithm>
#include <cmath>

#include "pb_async.cuh"
#include "pb_common.cuh"
#include "pb_span_impl.h"

namespace pb {
namespace {

// ---------------------------------------------------------------- int8 matrices on tcgen05
//
// Recompute (y = op(x) W + b) runs the span's own prefill path: k_rowstats +
// k_canonwrite digit planes, k_gemm_tc with the plain epilogue, so the
// recomputed intermediates are the ones FORWARD produced. BACKWARD through a
// matrix (dx_k = s_k sum_o g_o codes[o][k], outlier features exact in f32)
// needs the codes with the contraction over the outputs o: k_transpose_codes
// rewrites one matrix into canonical tiles of W^T (rows k, 32-wide o tiles)
// in a scratch buffer (one read + one write of the codes), the upstream
// gradient becomes the digit-plane operand (scales 1), and k_gemm_tc's
// EPI_BWD epilogue applies s_k. Outlier features (s_k = 0, codes 0) are then
// overwritten with their f32 dot products (k_outl_bwd).

// 128 o x 128 k of the source (4 tiles of one row group) -> 4 tiles of W^T (row group k0/128, o tiles
// 4 og .. 4 og + 3); tile bytes: row r, col c at (r >> 3) * 256 + (c >> 4) * 128 + (r & 7) * 16 + (c & 15)
constexpr int TP = 132;  // smem row pitch [o][k] (4-byte stores, conflict-free byte-column reads)
__global__ void __launch_bounds__(256) k_transpose_codes(const int8_t* __restrict__ src, int KC, int8_t* __restrict__ dst,
                                                         int KCt) {
    __shared__ uint32_t s[128 * TP / 4];
    const int og = blockIdx.x, kg = blockIdx.y;
    uint8_t* sb = reinterpret_cast<uint8_t*>(s);
    for (int c = threadIdx.x; c < 4 * 256; c += 256) {
        const int i = c >> 8, cc = c & 255;
        const int r = ((cc >> 4) << 3) | (cc & 7), kh = (cc >> 3) & 1;
        const int kt = kg * 4 + i;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (kt < KC) v = reinterpret_cast<const uint4*>(src + ((int64_t)og * KC + kt) * 4096)[cc];
        uint32_t* row = reinterpret_cast<uint32_t*>(sb + r * TP + i * 32 + kh * 16);
        row[0] = v.x, row[1] = v.y, row[2] = v.z, row[3] = v.w;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < 4 * 256; c += 256) {
        const int i = c >> 8, cc = c & 255;
        const int ot = og * 4 + i;
        if (ot >= KCt) break;  // i is uniform per 256-chunk pass
        const int kr = ((cc >> 4) << 3) | (cc & 7), oh = (cc >> 3) & 1;
        const uint8_t* col = sb + (i * 32 + oh * 16) * TP + kr;
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            w[q] = (uint32_t)col[(4 * q) * TP] | ((uint32_t)col[(4 * q + 1) * TP] << 8) |
                   ((uint32_t)col[(4 * q + 2) * TP] << 16) | ((uint32_t)col[(4 * q + 3) * TP] << 24);
        reinterpret_cast<uint4*>(dst + ((int64_t)kg * KCt + ot) * 4096)[cc] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// dx[t][idx_j] = sum_o g[t][o] rows[j][o] (quant.py:105 outlier features: W[idx_j, :] in f32); one CTA per (j, t)
__global__ void __launch_bounds__(256) k_outl_bwd(const float* __restrict__ g, const int32_t* __restrict__ idx,
                                                  const float* __restrict__ rows, int M, int K,
                                                  float* __restrict__ dx) {
    __shared__ float red[8];
    const int j = blockIdx.x, t = blockIdx.y;
    const float* gr = g + (int64_t)t * M;
    const float* wr = rows + (int64_t)j * M;
    float s = 0.f;
    for (int o = threadIdx.x; o < M; o += 256) s = fmaf(gr[o], wr[o], s);
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        float v = 0.f;
        for (int w = 0; w < 8; ++w) v += red[w];
        dx[(int64_t)t * K + idx[j]] = v;
    }
}

__global__ void k_fill(float* __restrict__ p, int64_t n, float v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

int grid_for(int64_t n) { return (int)std::min<int64_t>(std::max<int64_t>(ceil_div(n, 256), 1), 148 * 32); }

// scratch of one BACKWARD call (sizes: bwd_ws_sizes)
struct TcWs {
    uint8_t* bcanon = nullptr;  // digit planes [round_up(t, TC_TOKENS) / TC_TOKENS][KC][3][TC_TOKENS x 32 B]
    float* back = nullptr;      // [t]
    float4* stats = nullptr;    // [t]
    float* xo = nullptr;        // [t][max n_outl]
    float* ones = nullptr;      // [max Kp of W^T] operand scales of the gradient
    int8_t* tcodes = nullptr;   // W^T tiles of the matrix being back-propagated (when not cached)
    bool cache = false;         // keep W^T tiles per matrix (Mat::tcodes): HBM has room for all of them
};

// transposed view of m: rows k (padded to 128), contraction over o (padded to 32)
Mat transposed(const Mat& m, const TcWs& w) {
    Mat t;
    t.M = m.K;
    t.K = m.M;
    t.Mp = (int)round_up(m.K, 128);
    t.Kp = (int)round_up(m.M, 32);
    t.codes = w.tcodes;
    t.scales = w.ones;
    return t;
}

// y [t][M] = op(x) W + b; op = LN(gamma, beta) (mode PRO_LN) or identity (PRO_SCALE)
int mm_fwd_tc(const Mat& m, const float* bias, int mode, const float* x, const float* gamma, const float* beta,
              int t, float* y, const TcWs& w, cudaStream_t st) {
    if (int rc = launch_prologue(mode, ProSrc{}, x, t, m.K, m.Kp, gamma, beta, m, 0, nullptr, w.back, w.stats, w.xo,
                                 nullptr, st, w.bcanon, TC_TOKENS))
        return rc;
    Epi e{};
    e.kind = EPI_PLAIN;
    e.M = m.M;
    e.bias = bias;
    e.n_outl = m.n_outl;
    e.outl_idx = m.outl_idx;
    e.outl_rows = m.outl_rows;
    e.xo = w.xo;
    e.out = y;
    return launch_gemm_tc(m, w.bcanon, Act{nullptr, w.back, t, 0}, e, st);
}

// dx [t][K] = g [t][M] W^T
int mm_bwd_tc(Mat& m, const float* g, int t, float* dx, const TcWs& w, cudaStream_t st) {
    Mat mt = transposed(m, w);
    if (!m.tcodes) {
        int8_t* dst = w.tcodes;
        if (w.cache) {  // weights never change after loading: transpose once, keep it
            PB_CHECK_CUDA(cudaMalloc(&m.tcodes, (size_t)mt.Mp * mt.Kp));
            dst = m.tcodes;
        }
        k_transpose_codes<<<dim3((unsigned)(m.Mp / 128), (unsigned)(mt.Mp / 128)), 256, 0, st>>>(
            m.codes, m.Kp / 32, dst, mt.Kp / 32);
        if (int rc = launch_check("transpose_codes")) return rc;
    }
    if (m.tcodes) mt.codes = m.tcodes;
    if (int rc = launch_prologue(PRO_SCALE, ProSrc{}, g, t, mt.K, mt.Kp, nullptr, nullptr, mt, 0, nullptr, w.back,
                                 w.stats, nullptr, nullptr, st, w.bcanon, TC_TOKENS))
        return rc;
    Epi e{};
    e.kind = EPI_BWD;
    e.M = mt.M;
    e.rowscale = m.scales;
    e.out = dx;
    if (int rc = launch_gemm_tc(mt, w.bcanon, Act{nullptr, w.back, t, 0}, e, st)) return rc;
    if (m.n_outl) {
        k_outl_bwd<<<dim3((unsigned)m.n_outl, (unsigned)t), 256, 0, st>>>(g, m.outl_idx, m.outl_rows, m.M, m.K, dx);
        return launch_check("outl_bwd");
    }
    return PB_OK;
}

// ---------------------------------------------------------------- batched strided GEMM (f32 accuracy)
//
// C(b, i, j) = alpha sum_p A(b, i, p) B(b, p, j) (+ bias[j]) with arbitrary element strides, so one
// kernel serves the f32 weight matrices (either orientation) and every per-head attention product on
// the [t][3d] q|k|v rows and the [H][t][t] probability planes. Causal modes bound the work: CM_OUT
// skips output tiles strictly above the diagonal (j > i everywhere: masked scores), CM_P_LE_I
// contracts p <= i only, CM_P_GE_I p >= i (the skipped terms are zeros of the probability planes).
enum { CM_NONE = 0, CM_OUT = 1, CM_P_LE_I = 2, CM_P_GE_I = 3 };

struct BG {
    const float* A;
    int64_t a_b, a_i, a_p;
    const float* B;
    int64_t b_b, b_p, b_j;
    float* C;
    int64_t c_b, c_i, c_j;
    const float* bias;
    int I, J, P;
    float alpha;
    int causal;
};

// Tensor cores at f32 accuracy ("3xTF32"): every operand splits into hi = tf32(x) and
// lo = tf32(x - hi), and each product accumulates a_lo b_hi + a_hi b_lo + a_hi b_hi
// (mma.sync.m16n8k8 tf32, f32 accumulators): ~22 mantissa bits per product. 128 x 128 output tiles,
// 32-deep k slices double-buffered in shared memory by 4-byte cp.async (any stride, zero fill;
// [p][i] / [p][j] with pitch 136: conflict-free fragment loads), 8 warps as 2 x 4 of 64 x 32,
// two CTAs per SM. Measured (176B, t = 2048, ncu): the single-buffered version was latency-bound
// (long-scoreboard stalls, 8 warps per SM), no faster than a 64 x 64 SIMT kernel.
constexpr int XB = 128, XK = 32, XP = XB + 8;

__device__ __forceinline__ uint32_t tf32_bits(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ void mma_tf32(float* c, const uint32_t* a, const uint32_t* b) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool ok) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 4 : 0)
                 : "memory");
}

// one 32-deep k slice of both operands into a stage (zero-filled outside the matrix / p range)
__device__ __forceinline__ void x3_load(const BG& g, const float* A, const float* B, float* As, float* Bs, int i0,
                                        int j0, int p0, int p_hi, bool a_pc, bool b_jc) {
#pragma unroll 4
    for (int e = threadIdx.x; e < XB * XK; e += 256) {
        int ii, pp;
        if (a_pc) ii = e / XK, pp = e % XK;
        else pp = e / XB, ii = e % XB;
        const int i = i0 + ii, p = p0 + pp;
        const bool ok = i < g.I && p < p_hi;
        cp_async4(As + pp * XP + ii, ok ? A + i * g.a_i + p * g.a_p : A, ok);
    }
#pragma unroll 4
    for (int e = threadIdx.x; e < XB * XK; e += 256) {
        int jj, pp;
        if (b_jc) pp = e / XB, jj = e % XB;
        else jj = e / XK, pp = e % XK;
        const int j = j0 + jj, p = p0 + pp;
        const bool ok = j < g.J && p < p_hi;
        cp_async4(Bs + pp * XP + jj, ok ? B + p * g.b_p + j * g.b_j : B, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

constexpr int X_STAGE = 2 * XK * XP;  // floats per stage (A then B)
constexpr int X_SMEM = 2 * X_STAGE * (int)sizeof(float);

__global__ void __launch_bounds__(256, 2) k_bgemm_x3(BG g) {
    extern __shared__ float xs[];  // [2 stages][A: XK x XP | B: XK x XP]
    const int i0 = blockIdx.y * XB, j0 = blockIdx.x * XB;
    const int64_t bz = blockIdx.z;
    if (g.causal == CM_OUT && j0 > i0 + XB - 1) return;
    int p_lo = 0, p_hi = g.P;
    if (g.causal == CM_P_LE_I) p_hi = min(g.P, i0 + XB);
    if (g.causal == CM_P_GE_I) p_lo = i0 & ~(XK - 1);
    const float* A = g.A + bz * g.a_b;
    const float* B = g.B + bz * g.b_b;
    const bool a_pc = g.a_p == 1, b_jc = g.b_j == 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = (warp >> 2) * 64, wn = (warp & 3) * 32;
    const int gq = lane >> 2, tq = lane & 3;
    float acc[4][4][4] = {};
    const int n_sl = p_hi > p_lo ? (p_hi - p_lo + XK - 1) / XK : 0;
    if (n_sl > 0) x3_load(g, A, B, xs, xs + XK * XP, i0, j0, p_lo, p_hi, a_pc, b_jc);
    for (int sl = 0; sl < n_sl; ++sl) {
        if (sl + 1 < n_sl) {
            float* nx = xs + ((sl + 1) & 1) * X_STAGE;
            x3_load(g, A, B, nx, nx + XK * XP, i0, j0, p_lo + (sl + 1) * XK, p_hi, a_pc, b_jc);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const float* As = xs + (sl & 1) * X_STAGE;
        const float* Bs = As + XK * XP;
#pragma unroll
        for (int k8 = 0; k8 < XK; k8 += 8) {
            uint32_t ah[4][4], al[4][4], bh[4][2], bl[4][2];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                const int r = wm + mt * 16 + gq;
                const float v[4] = {As[(k8 + tq) * XP + r], As[(k8 + tq) * XP + r + 8], As[(k8 + tq + 4) * XP + r],
                                    As[(k8 + tq + 4) * XP + r + 8]};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    ah[mt][q] = tf32_bits(v[q]);
                    al[mt][q] = tf32_bits(v[q] - __uint_as_float(ah[mt][q]));
                }
            }
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                const int c = wn + nt * 8 + gq;
                const float v[2] = {Bs[(k8 + tq) * XP + c], Bs[(k8 + tq + 4) * XP + c]};
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    bh[nt][q] = tf32_bits(v[q]);
                    bl[nt][q] = tf32_bits(v[q] - __uint_as_float(bh[nt][q]));
                }
            }
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) {
                    mma_tf32(acc[mt][nt], al[mt], bh[nt]);
                    mma_tf32(acc[mt][nt], ah[mt], bl[nt]);
                    mma_tf32(acc[mt][nt], ah[mt], bh[nt]);
                }
        }
        __syncthreads();  // the stage is refilled by the next iteration's load
    }
    float* C = g.C + bz * g.c_b;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int i = i0 + wm + mt * 16 + gq + (q >> 1) * 8, j = j0 + wn + nt * 8 + tq * 2 + (q & 1);
                if (i < g.I && j < g.J) C[i * g.c_i + j * g.c_j] = acc[mt][nt][q] * g.alpha + (g.bias ? g.bias[j] : 0.f);
            }
}

int bgemm(const BG& g, int batch, cudaStream_t st) {
    static int ok[PB_MAX_DEVICES] = {};
    if (per_device(ok, [](int) {
            return cudaFuncSetAttribute(k_bgemm_x3, cudaFuncAttributeMaxDynamicSharedMemorySize, X_SMEM) ==
                           cudaSuccess ? 1 : -1;
        }) < 0)
        return launch_check("bgemm setup");
    k_bgemm_x3<<<dim3((unsigned)ceil_div(g.J, XB), (unsigned)ceil_div(g.I, XB), (unsigned)batch), 256, X_SMEM, st>>>(g);
    return launch_check("bgemm");
}

// f32 weights: C [I][J] = A [I][P] W (+ bias), W [P][J] (trans = false) or C = A W^T, W [J][P] (trans = true)
int gemm(bool trans, const float* A, const float* W, const float* bias, float* C, int I, int J, int P,
         cudaStream_t st) {
    BG g{A, 0, P, 1, W, 0, trans ? 1 : J, trans ? P : 1, C, 0, J, 1, bias, I, J, P, 1.f, CM_NONE};
    return bgemm(g, 1, st);
}

// ---------------------------------------------------------------- LayerNorm / GELU

// model.py:271-276: h = g xhat + b, xhat = (x - mu) inv, population variance
__global__ void __launch_bounds__(256) k_ln_fwd(const float* __restrict__ x, const float* __restrict__ g,
                                                const float* __restrict__ b, int d, float* __restrict__ h,
                                                float* __restrict__ xhat, float* __restrict__ inv) {
    __shared__ double red[8];
    const int t = blockIdx.x;
    const float* xr = x + (int64_t)t * d;
    double s = 0.0;
    for (int k = threadIdx.x; k < d; k += 256) s += xr[k];
    s = warp_sum_d(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    double mean = 0.0;
    for (int w = 0; w < 8; ++w) mean += red[w];
    mean /= d;
    __syncthreads();
    double v = 0.0;
    for (int k = threadIdx.x; k < d; k += 256) {
        const double dd = xr[k] - mean;
        v += dd * dd;
    }
    v = warp_sum_d(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double var = 0.0;
    for (int w = 0; w < 8; ++w) var += red[w];
    const float mu = (float)mean;
    const float is = 1.0f / sqrtf((float)(var / d) + 1e-5f);
    for (int k = threadIdx.x; k < d; k += 256) {
        const float xh = (xr[k] - mu) * is;
        xhat[(int64_t)t * d + k] = xh;
        h[(int64_t)t * d + k] = fmaf(g[k], xh, b[k]);
    }
    if (threadIdx.x == 0) inv[t] = is;
}

// model.py:279-283: dx = (dxhat - mean(dxhat) - xhat mean(dxhat xhat)) inv, dxhat = dy g;
// out = base + dx (base may be null)
__global__ void __launch_bounds__(256) k_ln_bwd(const float* __restrict__ dy, const float* __restrict__ xhat,
                                                const float* __restrict__ inv, const float* __restrict__ g, int d,
                                                const float* __restrict__ base, float* __restrict__ out) {
    __shared__ double red[2][8];
    const int t = blockIdx.x;
    double s1 = 0.0, s2 = 0.0;
    for (int k = threadIdx.x; k < d; k += 256) {
        const double dx = (double)dy[(int64_t)t * d + k] * g[k];
        s1 += dx;
        s2 += dx * xhat[(int64_t)t * d + k];
    }
    s1 = warp_sum_d(s1);
    s2 = warp_sum_d(s2);
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = s1;
        red[1][threadIdx.x >> 5] = s2;
    }
    __syncthreads();
    double m1 = 0.0, m2 = 0.0;
    for (int w = 0; w < 8; ++w) {
        m1 += red[0][w];
        m2 += red[1][w];
    }
    const float f1 = (float)(m1 / d), f2 = (float)(m2 / d);
    for (int k = threadIdx.x; k < d; k += 256) {
        const int64_t i = (int64_t)t * d + k;
        const float v = (dy[i] * g[k] - f1 - xhat[i] * f2) * inv[t];
        out[i] = (base ? base[i] : 0.f) + v;
    }
}

__device__ __forceinline__ float gelu_g(float x) {  // model.py:295-298
    const float c = 0.7978845608028654f;
    const float t = tanhf(c * (x + 0.044715f * x * x * x));
    return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * c * (1.f + 3.f * 0.044715f * x * x);
}

__global__ void k_gelu_bwd(const float* __restrict__ pre, float* __restrict__ g, int64_t n) {  // g *= gelu'(pre)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        g[i] *= gelu_g(pre[i]);
}
__global__ void k_add(const float* __restrict__ a, float* __restrict__ b, int64_t n) {  // b += a
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        b[i] += a[i];
}

// ---------------------------------------------------------------- attention (one row, positions 0 .. t-1)
// qkv [t][3d]: q | k | v column thirds (model.py:342-344), head h at columns h dh ..

// in place on the [H][t][t] plane holding q_i . k_j / sqrt(dh) (j <= i): P[h][i][j] = softmax_j(s_ij +
// slope_h (j - i)), zero for j > i (model.py:347-357); one CTA per (h, i)
__global__ void __launch_bounds__(256) k_softmax_rows(float* __restrict__ P, int t, const float* __restrict__ slopes) {
    __shared__ float red[8];
    const int h = blockIdx.x, i = blockIdx.y;
    float* prow = P + ((int64_t)h * t + i) * t;
    const float sl = slopes[h];
    float mx = -INFINITY;
    for (int j = threadIdx.x; j <= i; j += 256) {
        const float v = prow[j] + sl * (float)(j - i);
        prow[j] = v;
        mx = fmaxf(mx, v);
    }
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = red[0];
    for (int w = 1; w < 8; ++w) mx = fmaxf(mx, red[w]);
    __syncthreads();
    float sum = 0.f;
    for (int j = threadIdx.x; j <= i; j += 256) {
        const float e = expf(prow[j] - mx);
        prow[j] = e;
        sum += e;
    }
    sum = warp_sum(sum);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
    __syncthreads();
    sum = 0.f;
    for (int w = 0; w < 8; ++w) sum += red[w];
    for (int j = threadIdx.x; j < t; j += 256) prow[j] = j <= i ? prow[j] / sum : 0.f;
}

// in place on the plane holding dP = dctx_i . v_j: dS = P (dP - sum_j dP P), zero for j > i
// (model.py:400-403); one CTA per (h, i)
__global__ void __launch_bounds__(256) k_dscores_rows(const float* __restrict__ P, float* __restrict__ dS, int t) {
    __shared__ float red[8];
    const int h = blockIdx.x, i = blockIdx.y;
    const float* prow = P + ((int64_t)h * t + i) * t;
    float* drow = dS + ((int64_t)h * t + i) * t;
    float rs = 0.f;
    for (int j = threadIdx.x; j <= i; j += 256) rs = fmaf(drow[j], prow[j], rs);
    rs = warp_sum(rs);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = rs;
    __syncthreads();
    rs = 0.f;
    for (int w = 0; w < 8; ++w) rs += red[w];
    for (int j = threadIdx.x; j < t; j += 256) drow[j] = j <= i ? prow[j] * (drow[j] - rs) : 0.f;
}

// attention of one row over its own positions (empty cache) on the batched GEMM, heads as the batch;
// qkv [t][3d] (q | k | v thirds, head h at columns h dh ..), planes [H][t][t]
int attn_fwd(const float* qkv, float* P, float* ctx, int t, int d, int H, int dh, const float* slopes,
             cudaStream_t st) {
    const int64_t tt = (int64_t)t * t, r3 = 3 * (int64_t)d;
    // S = q k^T / sqrt(dh) (upper tiles skipped)
    BG s{qkv, dh, r3, 1, qkv + d, dh, 1, r3, P, tt, t, 1, nullptr, t, t, dh, 1.0f / sqrtf((float)dh), CM_OUT};
    if (int rc = bgemm(s, H, st)) return rc;
    k_softmax_rows<<<dim3(H, t), 256, 0, st>>>(P, t, slopes);
    // ctx = P v
    BG c{P, tt, t, 1, qkv + 2 * d, dh, r3, 1, ctx, dh, d, 1, nullptr, t, dh, t, 1.f, CM_P_LE_I};
    return bgemm(c, H, st);
}

// dctx [t][d] -> dqkv [t][3d] (model.py:399-409)
int attn_bwd(const float* qkv, const float* P, float* dS, const float* dctx, float* dqkv, int t, int d, int H,
             int dh, cudaStream_t st) {
    const int64_t tt = (int64_t)t * t, r3 = 3 * (int64_t)d;
    const float isq = 1.0f / sqrtf((float)dh);
    // dP = dctx v^T, then dS = P (dP - rowsum(dP P))
    BG dp{dctx, dh, d, 1, qkv + 2 * d, dh, 1, r3, dS, tt, t, 1, nullptr, t, t, dh, 1.f, CM_OUT};
    if (int rc = bgemm(dp, H, st)) return rc;
    k_dscores_rows<<<dim3(H, t), 256, 0, st>>>(P, dS, t);
    // dq = dS k / sqrt(dh)
    BG dq{dS, tt, t, 1, qkv + d, dh, r3, 1, dqkv, dh, r3, 1, nullptr, t, dh, t, isq, CM_P_LE_I};
    if (int rc = bgemm(dq, H, st)) return rc;
    // dk = dS^T q / sqrt(dh), dv = P^T dctx (contraction over i >= j)
    BG dk{dS, tt, 1, t, qkv, dh, r3, 1, dqkv + d, dh, r3, 1, nullptr, t, dh, t, isq, CM_P_GE_I};
    if (int rc = bgemm(dk, H, st)) return rc;
    BG dv{P, tt, 1, t, dctx, dh, d, 1, dqkv + 2 * d, dh, r3, 1, nullptr, t, dh, t, 1.f, CM_P_GE_I};
    return bgemm(dv, H, st);
}

int ew_grid(int64_t n) { return grid_for(n); }

}  // namespace

// One block's BACKWARD for one row: g [t][d] in, dx [t][d] out (model.py:383-418).
static int block_backward(pb_span* s, int j, const float* x, const float* g, float* dx, int t, float* ws,
                          const TcWs& tw, cudaStream_t st) {
    const int d = s->d, rd = s->rd, H = s->H, dh = s->dh;
    BlockW& b = s->blocks[j];
    const int64_t td = (int64_t)t * d;
    float* h1 = ws;
    float* xh1 = h1 + td;
    float* inv1 = xh1 + td;
    float* qkv = inv1 + t;
    float* P = qkv + 3 * td;
    float* dS = P + (int64_t)H * t * t;
    float* ctx = dS + (int64_t)H * t * t;
    float* mid = ctx + td;
    float* h2 = mid + td;
    float* xh2 = h2 + td;
    float* inv2 = xh2 + td;
    float* pre = inv2 + t;
    float* act = pre + (int64_t)t * rd;  // reused as d(pre)
    float* dmid = act + (int64_t)t * rd;
    float* tmp = dmid + td;              // [t][max(d, rd)]
    float* dqkv = tmp + (int64_t)t * rd;
    // y = op(x) W_i + b_i: int8 on tcgen05 (op applied by the operand writer), f32 on the SIMT GEMM (op(x) = h)
    auto fwd = [&](int i, int mode, const float* xin, const float* h, const float* gam, const float* bet,
                   float* y) -> int {
        const Mat& m = b.mat[i];
        if (m.int8) return mm_fwd_tc(m, b.bias[i], mode, xin, gam, bet, t, y, tw, st);
        return gemm(false, h, m.w32, b.bias[i], y, t, m.M, m.K, st);
    };
    // dx = g W_i^T
    auto bwd = [&](int i, const float* gin, float* out) -> int {
        Mat& m = b.mat[i];
        if (m.int8) return mm_bwd_tc(m, gin, t, out, tw, st);
        return gemm(true, gin, m.w32, nullptr, out, t, m.K, m.M, st);
    };
    // ---- recompute the forward intermediates (model.py:340-368)
    k_ln_fwd<<<t, 256, 0, st>>>(x, b.ln1_g, b.ln1_b, d, h1, xh1, inv1);
    if (int rc = fwd(0, PRO_LN, x, h1, b.ln1_g, b.ln1_b, qkv)) return rc;
    if (int rc = attn_fwd(qkv, P, ctx, t, d, H, dh, s->slopes, st)) return rc;
    if (int rc = fwd(1, PRO_SCALE, ctx, ctx, nullptr, nullptr, mid)) return rc;
    k_add<<<ew_grid(td), 256, 0, st>>>(x, mid, td);  // mid = x + attn_out
    k_ln_fwd<<<t, 256, 0, st>>>(mid, b.ln2_g, b.ln2_b, d, h2, xh2, inv2);
    if (int rc = fwd(2, PRO_LN, mid, h2, b.ln2_g, b.ln2_b, pre)) return rc;
    // ---- backward (model.py:397-417)
    if (int rc = bwd(3, g, act)) return rc;                                             // dact = g Wout^T
    k_gelu_bwd<<<ew_grid((int64_t)t * rd), 256, 0, st>>>(pre, act, (int64_t)t * rd);  // dpre
    if (int rc = bwd(2, act, tmp)) return rc;                                           // dh2 = dpre Win^T
    k_ln_bwd<<<t, 256, 0, st>>>(tmp, xh2, inv2, b.ln2_g, d, g, dmid);                   // dmid = g + LN2'(dh2)
    if (int rc = bwd(1, dmid, tmp)) return rc;                                          // dctx = dmid Wo^T
    if (int rc = attn_bwd(qkv, P, dS, tmp, dqkv, t, d, H, dh, st)) return rc;
    if (int rc = bwd(0, dqkv, tmp)) return rc;                                  // dh1 = dqkv Wqkv^T
    k_ln_bwd<<<t, 256, 0, st>>>(tmp, xh1, inv1, b.ln1_g, d, dmid, dx);          // dx = dmid + LN1'(dh1)
    return launch_check("block_backward");
}

}  // namespace pb

using namespace pb;

extern "C" int pb_span_backward(pb_span* span, const float* d_tape, int32_t t, const float* d_grad_out,
                                float* d_grad_in, void* stream) {
    PB_REQUIRE(span && d_tape && d_grad_out && d_grad_in, PB_ERR_BAD_REQUEST, "null argument");
    PB_REQUIRE(t > 0 && t <= span->cfg.max_seq, PB_ERR_CAPACITY, "row length outside [1, max_seq]");
    std::lock_guard<std::mutex> lk(span->mu);
    PB_CHECK_CUDA(cudaSetDevice(span->cfg.device));
    auto st = (cudaStream_t)stream;
    const int d = span->d, rd = span->rd, H = span->H;
    const int64_t td = (int64_t)t * d;
    // workspace: see block_backward's carve-up
    const int64_t ws_floats = 9 * td + 2 * (int64_t)t + 2 * (int64_t)H * t * t + 3 * td + 3 * (int64_t)t * rd +
                              3 * td + 64;
    // tcgen05 scratch: digit planes for the widest contraction, W^T tiles of the largest matrix
    int64_t kp_max = 0, tcode_max = 0, n_outl = 0;
    for (const auto& b : span->blocks)
        for (const auto& m : b.mat)
            if (m.int8) {
                kp_max = std::max<int64_t>(kp_max, std::max<int64_t>(m.Kp, round_up(m.M, 32)));
                tcode_max = std::max<int64_t>(tcode_max, round_up(m.K, 128) * round_up(m.M, 32));
                n_outl = std::max<int64_t>(n_outl, m.n_outl);
            }
    // W^T tiles: cached per matrix when HBM holds all of them with room to spare (multi-GPU spans),
    // else transposed per call into the arena (0.27 ms per 176B mlp matrix)
    int64_t tcache = 0;
    for (const auto& b : span->blocks)
        for (const auto& m : b.mat)
            if (m.int8 && !m.tcodes) tcache += round_up(m.K, 128) * round_up(m.M, 32);
    bool cache = false;
    if (tcache) {
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess)
            cache = (int64_t)free_b > tcache + ((int64_t)16 << 30);
    }
    // carve-up of the span's grow-only arena (256-byte aligned pieces)
    int64_t off = 0;
    auto piece = [&](int64_t bytes) {
        const int64_t at = off;
        off += round_up(std::max<int64_t>(bytes, 1), 256);
        return at;
    };
    const int64_t o_ws = piece(sizeof(float) * ws_floats), o_g = piece(sizeof(float) * 2 * td);
    int64_t o_bc = 0, o_back = 0, o_stats = 0, o_xo = 0, o_ones = 0, o_tc = 0;
    if (kp_max) {
        o_bc = piece(round_up(t, TC_TOKENS) * kp_max * 3);
        o_back = piece(sizeof(float) * t);
        o_stats = piece(sizeof(float4) * t);
        o_xo = piece(sizeof(float) * t * n_outl);
        o_ones = piece(sizeof(float) * kp_max);
        o_tc = piece(tcode_max);
    }
    if (off > span->train_ws_bytes) {
        // grow (rare): plain cudaMalloc after the stream drains, so any later stream may use it
        PB_CHECK_CUDA(cudaStreamSynchronize(st));
        if (span->train_ws) PB_CHECK_CUDA(cudaFree(span->train_ws));
        span->train_ws = nullptr;
        span->train_ws_bytes = 0;
        PB_CHECK_CUDA(cudaMalloc(&span->train_ws, off));
        span->train_ws_bytes = off;
    }
    uint8_t* base = span->train_ws;
    float* ws = reinterpret_cast<float*>(base + o_ws);
    float* g = reinterpret_cast<float*>(base + o_g);
    TcWs tw;
    if (kp_max) {
        tw.bcanon = base + o_bc;
        tw.back = reinterpret_cast<float*>(base + o_back);
        tw.stats = reinterpret_cast<float4*>(base + o_stats);
        tw.xo = reinterpret_cast<float*>(base + o_xo);
        tw.ones = reinterpret_cast<float*>(base + o_ones);
        tw.tcodes = reinterpret_cast<int8_t*>(base + o_tc);
        tw.cache = cache;
        k_fill<<<grid_for(kp_max), 256, 0, st>>>(tw.ones, kp_max, 1.f);
    }
    PB_CHECK_CUDA(cudaMemcpyAsync(g, d_grad_out, sizeof(float) * td, cudaMemcpyDeviceToDevice, st));
    int rc = PB_OK;
    float* cur = g;
    float* nxt = g + td;
    for (int j = span->cfg.n_blocks - 1; j >= 0 && !rc; --j) {
        float* out = j == 0 ? d_grad_in : nxt;
        rc = block_backward(span, j, d_tape + (int64_t)j * td, cur, out, t, ws, tw, st);
        std::swap(cur, nxt);
    }
    return rc;
}
