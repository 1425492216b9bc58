// Training path of a span: the exact BACKWARD of block_forward
// (model.py:383-418 block_backward, served as server.py:431-450) for one row of
// a FORWARD batch (positions 0 .. t-1, empty cache: server.py:418-425).
//
// Tape-less recompute: the FORWARD step records only each block's input rows
// (pb_span_step_tape); BACKWARD recomputes the block's intermediates from them
// in f32 (LN1, qkv, softmax probabilities, ctx, mid, LN2, pre-activation) and
// then runs the reference backward formulas. The weights are the span's own:
// f32 matrices as stored, int8 matrices dequantized (codes x feature scales,
// f32 outlier rows) into a scratch f32 copy per matrix, so the gradient is
// that of the function the span's FORWARD computes.
//
// Every matmul is one tiled SIMT kernel (64 x 64 tiles, 4 x 4 per thread,
// f32 accumulation) in either orientation: C = A W (forward) or C = A W^T
// (backward through a weight). Attention works on [H][t][t] probability and
// score-gradient planes.
#include <algorithm>
#include <cmath>

#include "pb_common.cuh"
#include "pb_span_impl.h"

namespace pb {
namespace {

// ---------------------------------------------------------------- weights

// W[k][o] (reference [in, out] layout, f32) from the canonical int8 tiles
__global__ void k_dequant(const int8_t* __restrict__ codes, const float* __restrict__ scales, int K, int M, int KC,
                          float* __restrict__ w) {
    const int64_t total = (int64_t)K * M;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(t / M), o = (int)(t % M);
        const int r = o & 127, kk = k & 31;
        const int8_t c = codes[((int64_t)(o >> 7) * KC + (k >> 5)) * 4096 + (r >> 3) * 256 + (kk >> 4) * 128 +
                               (r & 7) * 16 + (kk & 15)];
        w[t] = (float)c * scales[k];
    }
}

__global__ void k_outlier_rows(const int32_t* __restrict__ idx, const float* __restrict__ rows, int n_outl, int M,
                               float* __restrict__ w) {
    const int64_t total = (int64_t)n_outl * M;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(t / M), o = (int)(t % M);
        w[(int64_t)idx[j] * M + o] = rows[t];  // quant.py:105: outlier features exact in f32
    }
}

int grid_for(int64_t n) { return (int)std::min<int64_t>(std::max<int64_t>(ceil_div(n, 256), 1), 148 * 32); }

// f32 [K][M] view of matrix m (the stored f32 matrix, or a dequantized copy in scratch)
int weight_f32(const Mat& m, float* scratch, const float** out, cudaStream_t st) {
    if (!m.int8) {
        *out = m.w32;
        return PB_OK;
    }
    k_dequant<<<grid_for((int64_t)m.K * m.M), 256, 0, st>>>(m.codes, m.scales, m.K, m.M, m.Kp / 32, scratch);
    if (int rc = launch_check("dequant")) return rc;
    if (m.n_outl) {
        k_outlier_rows<<<grid_for((int64_t)m.n_outl * m.M), 256, 0, st>>>(m.outl_idx, m.outl_rows, m.n_outl, m.M,
                                                                        scratch);
        if (int rc = launch_check("outlier_rows")) return rc;
    }
    *out = scratch;
    return PB_OK;
}

// ---------------------------------------------------------------- GEMM

constexpr int GB = 64, GK = 16;

// C[i][j] (+= or =) sum_p A[i][p] B(p, j) (+ bias[j]); B(p, j) = W[p][j] (TRANS = false,
// W is [P][N]) or W[j][p] (TRANS = true, W is [N][P]).
template <bool TRANS>
__global__ void __launch_bounds__(256) k_sgemm(const float* __restrict__ A, const float* __restrict__ W,
                                               const float* __restrict__ bias, float* __restrict__ C, int I, int J,
                                               int P) {
    __shared__ float As[GK][GB + 4];
    __shared__ float Bs[GK][GB + 4];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int i0 = blockIdx.y * GB, j0 = blockIdx.x * GB;
    float acc[4][4] = {};
    for (int p0 = 0; p0 < P; p0 += GK) {
        for (int e = threadIdx.x; e < GB * GK; e += 256) {
            const int ii = e / GK, pp = e % GK;  // A tile: rows i, cols p (coalesced along p)
            const int i = i0 + ii, p = p0 + pp;
            As[pp][ii] = (i < I && p < P) ? A[(int64_t)i * P + p] : 0.f;
        }
        for (int e = threadIdx.x; e < GB * GK; e += 256) {
            int jj, pp;
            if (TRANS) {
                jj = e / GK;
                pp = e % GK;  // W[j][p]: coalesced along p
            } else {
                pp = e / GB;
                jj = e % GB;  // W[p][j]: coalesced along j
            }
            const int j = j0 + jj, p = p0 + pp;
            float v = 0.f;
            if (j < J && p < P) v = TRANS ? W[(int64_t)j * P + p] : W[(int64_t)p * J + j];
            Bs[pp][jj] = v;
        }
        __syncthreads();
#pragma unroll
        for (int pp = 0; pp < GK; ++pp) {
            float a[4], b[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) a[r] = As[pp][ty * 4 + r];
#pragma unroll
            for (int c = 0; c < 4; ++c) b[c] = Bs[pp][tx * 4 + c];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[r][c] = fmaf(a[r], b[c], acc[r][c]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int i = i0 + ty * 4 + r;
        if (i >= I) continue;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int j = j0 + tx * 4 + c;
            if (j < J) C[(int64_t)i * J + j] = acc[r][c] + (bias ? bias[j] : 0.f);
        }
    }
}

int gemm(bool trans, const float* A, const float* W, const float* bias, float* C, int I, int J, int P,
         cudaStream_t st) {
    dim3 grid((unsigned)ceil_div(J, GB), (unsigned)ceil_div(I, GB));
    if (trans) k_sgemm<true><<<grid, 256, 0, st>>>(A, W, bias, C, I, J, P);
    else k_sgemm<false><<<grid, 256, 0, st>>>(A, W, bias, C, I, J, P);
    return launch_check("sgemm");
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

// P[h][i][j] (j <= i) = softmax_j(q_i . k_j / sqrt(dh) + slope_h (j - i)); one CTA per (h, i)
__global__ void __launch_bounds__(256) k_attn_probs(const float* __restrict__ qkv, int t, int d, int dh,
                                                    const float* __restrict__ slopes, float* __restrict__ P) {
    __shared__ float red[8];
    const int h = blockIdx.x, i = blockIdx.y;
    const float* q = qkv + (int64_t)i * 3 * d + h * dh;
    float* prow = P + ((int64_t)h * t + i) * t;
    const float sq = sqrtf((float)dh);
    float mx = -INFINITY;
    for (int j = threadIdx.x; j <= i; j += 256) {
        const float* k = qkv + (int64_t)j * 3 * d + d + h * dh;
        float s = 0.f;
        for (int e = 0; e < dh; ++e) s = fmaf(q[e], k[e], s);
        s = s / sq + slopes[h] * (float)(j - i);
        prow[j] = s;
        mx = fmaxf(mx, s);
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

// ctx[i][h dh + e] = sum_j P[h][i][j] v[j][h dh + e]; one CTA per (h, i), threads over e
__global__ void k_attn_ctx(const float* __restrict__ qkv, const float* __restrict__ P, int t, int d, int dh,
                           float* __restrict__ ctx) {
    const int h = blockIdx.x, i = blockIdx.y;
    const float* prow = P + ((int64_t)h * t + i) * t;
    for (int e = threadIdx.x; e < dh; e += blockDim.x) {
        float s = 0.f;
        for (int j = 0; j <= i; ++j) s = fmaf(prow[j], qkv[(int64_t)j * 3 * d + 2 * d + h * dh + e], s);
        ctx[(int64_t)i * d + h * dh + e] = s;
    }
}

// dS[h][i][j] = P (dP - sum_j dP P), dP[h][i][j] = dctx_i . v_j (model.py:400-403); one CTA per (h, i)
__global__ void __launch_bounds__(256) k_attn_dscores(const float* __restrict__ qkv, const float* __restrict__ P,
                                                      const float* __restrict__ dctx, int t, int d, int dh,
                                                      float* __restrict__ dS) {
    __shared__ float red[8];
    const int h = blockIdx.x, i = blockIdx.y;
    const float* prow = P + ((int64_t)h * t + i) * t;
    float* drow = dS + ((int64_t)h * t + i) * t;
    const float* dc = dctx + (int64_t)i * d + h * dh;
    float rs = 0.f;
    for (int j = threadIdx.x; j <= i; j += 256) {
        const float* v = qkv + (int64_t)j * 3 * d + 2 * d + h * dh;
        float s = 0.f;
        for (int e = 0; e < dh; ++e) s = fmaf(dc[e], v[e], s);
        drow[j] = s;
        rs = fmaf(s, prow[j], rs);
    }
    rs = warp_sum(rs);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = rs;
    __syncthreads();
    rs = 0.f;
    for (int w = 0; w < 8; ++w) rs += red[w];
    for (int j = threadIdx.x; j < t; j += 256) drow[j] = j <= i ? prow[j] * (drow[j] - rs) : 0.f;
}

// dq_i = sum_j dS[h][i][j] k_j / sqrt(dh) -> dqkv[i][h dh + e]; one CTA per (h, i)
__global__ void k_attn_dq(const float* __restrict__ qkv, const float* __restrict__ dS, int t, int d, int dh,
                          float* __restrict__ dqkv) {
    const int h = blockIdx.x, i = blockIdx.y;
    const float* drow = dS + ((int64_t)h * t + i) * t;
    const float inv_sq = 1.0f / sqrtf((float)dh);
    for (int e = threadIdx.x; e < dh; e += blockDim.x) {
        float s = 0.f;
        for (int j = 0; j <= i; ++j) s = fmaf(drow[j], qkv[(int64_t)j * 3 * d + d + h * dh + e], s);
        dqkv[(int64_t)i * 3 * d + h * dh + e] = s * inv_sq;
    }
}

// dk_j = sum_i dS[h][i][j] q_i / sqrt(dh), dv_j = sum_i P[h][i][j] dctx_i (i >= j); one CTA per (h, j)
__global__ void k_attn_dkdv(const float* __restrict__ qkv, const float* __restrict__ P, const float* __restrict__ dS,
                            const float* __restrict__ dctx, int t, int d, int dh, float* __restrict__ dqkv) {
    const int h = blockIdx.x, j = blockIdx.y;
    const float inv_sq = 1.0f / sqrtf((float)dh);
    for (int e = threadIdx.x; e < dh; e += blockDim.x) {
        float sk = 0.f, sv = 0.f;
        for (int i = j; i < t; ++i) {
            const int64_t pi = ((int64_t)h * t + i) * t + j;
            sk = fmaf(dS[pi], qkv[(int64_t)i * 3 * d + h * dh + e], sk);
            sv = fmaf(P[pi], dctx[(int64_t)i * d + h * dh + e], sv);
        }
        dqkv[(int64_t)j * 3 * d + d + h * dh + e] = sk * inv_sq;
        dqkv[(int64_t)j * 3 * d + 2 * d + h * dh + e] = sv;
    }
}

int ew_grid(int64_t n) { return grid_for(n); }

}  // namespace

// One block's BACKWARD for one row: g [t][d] in, dx [t][d] out (model.py:383-418).
static int block_backward(pb_span* s, int j, const float* x, const float* g, float* dx, int t, float* ws,
                          float* wscratch, cudaStream_t st) {
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
    const float* w;
    // ---- recompute the forward intermediates (model.py:340-368)
    k_ln_fwd<<<t, 256, 0, st>>>(x, b.ln1_g, b.ln1_b, d, h1, xh1, inv1);
    if (int rc = weight_f32(b.mat[0], wscratch, &w, st)) return rc;
    if (int rc = gemm(false, h1, w, b.bias[0], qkv, t, 3 * d, d, st)) return rc;
    k_attn_probs<<<dim3(H, t), 256, 0, st>>>(qkv, t, d, dh, s->slopes, P);
    k_attn_ctx<<<dim3(H, t), 128, 0, st>>>(qkv, P, t, d, dh, ctx);
    if (int rc = weight_f32(b.mat[1], wscratch, &w, st)) return rc;
    if (int rc = gemm(false, ctx, w, b.bias[1], mid, t, d, d, st)) return rc;
    k_add<<<ew_grid(td), 256, 0, st>>>(x, mid, td);  // mid = x + attn_out
    k_ln_fwd<<<t, 256, 0, st>>>(mid, b.ln2_g, b.ln2_b, d, h2, xh2, inv2);
    if (int rc = weight_f32(b.mat[2], wscratch, &w, st)) return rc;
    if (int rc = gemm(false, h2, w, b.bias[2], pre, t, rd, d, st)) return rc;
    // ---- backward (model.py:397-417)
    if (int rc = weight_f32(b.mat[3], wscratch, &w, st)) return rc;
    if (int rc = gemm(true, g, w, nullptr, act, t, rd, d, st)) return rc;  // dact = g Wout^T
    k_gelu_bwd<<<ew_grid((int64_t)t * rd), 256, 0, st>>>(pre, act, (int64_t)t * rd);  // dpre
    if (int rc = weight_f32(b.mat[2], wscratch, &w, st)) return rc;
    if (int rc = gemm(true, act, w, nullptr, tmp, t, d, rd, st)) return rc;  // dh2 = dpre Win^T
    k_ln_bwd<<<t, 256, 0, st>>>(tmp, xh2, inv2, b.ln2_g, d, g, dmid);       // dmid = g + LN2'(dh2)
    if (int rc = weight_f32(b.mat[1], wscratch, &w, st)) return rc;
    if (int rc = gemm(true, dmid, w, nullptr, tmp, t, d, d, st)) return rc;  // dctx = dmid Wo^T
    k_attn_dscores<<<dim3(H, t), 256, 0, st>>>(qkv, P, tmp, t, d, dh, dS);
    k_attn_dq<<<dim3(H, t), 128, 0, st>>>(qkv, dS, t, d, dh, dqkv);
    k_attn_dkdv<<<dim3(H, t), 128, 0, st>>>(qkv, P, dS, tmp, t, d, dh, dqkv);
    if (int rc = weight_f32(b.mat[0], wscratch, &w, st)) return rc;
    if (int rc = gemm(true, dqkv, w, nullptr, tmp, t, d, 3 * d, st)) return rc;  // dh1 = dqkv Wqkv^T
    k_ln_bwd<<<t, 256, 0, st>>>(tmp, xh1, inv1, b.ln1_g, d, dmid, dx);         // dx = dmid + LN1'(dh1)
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
    int64_t wmax = 0;
    for (const auto& b : span->blocks)
        for (const auto& m : b.mat)
            if (m.int8) wmax = std::max<int64_t>(wmax, (int64_t)m.K * m.M);
    float *ws = nullptr, *wscratch = nullptr, *g = nullptr;
    PB_CHECK_CUDA(cudaMallocAsync(&ws, sizeof(float) * ws_floats, st));
    PB_CHECK_CUDA(cudaMallocAsync(&g, sizeof(float) * 2 * td, st));
    if (wmax) PB_CHECK_CUDA(cudaMallocAsync(&wscratch, sizeof(float) * wmax, st));
    PB_CHECK_CUDA(cudaMemcpyAsync(g, d_grad_out, sizeof(float) * td, cudaMemcpyDeviceToDevice, st));
    int rc = PB_OK;
    float* cur = g;
    float* nxt = g + td;
    for (int j = span->cfg.n_blocks - 1; j >= 0 && !rc; --j) {
        float* out = j == 0 ? d_grad_in : nxt;
        rc = block_backward(span, j, d_tape + (int64_t)j * td, cur, out, t, ws, wscratch, st);
        std::swap(cur, nxt);
    }
    cudaFreeAsync(ws, st);
    cudaFreeAsync(g, st);
    if (wscratch) cudaFreeAsync(wscratch, st);
    return rc;
}
