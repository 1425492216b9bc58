// Client-side head on the GPU: embedding lookup
// (model.py:421-425), final LayerNorm + tied LM head (model.py:428-433) and
// greedy next-token choice (model.py:445-446, client.py:247-250).
//
// The tied head at the 176B shape is a [V=250880, d=14336] matrix: 14.4 GB in
// f32, i.e. 8 % of a whole decode step's weight bytes. Greedy decoding only
// needs the argmax, so the head streams an int8 copy of E^T (3.6 GB, the
// block matrices' LLM.int8 layout and GEMV) for approximate logits, bounds
// their error rigorously, and rescores only the candidates inside the bound
// against the f32 rows in f64:
//   |approx_v - exact_v| <= sum_k |y_k| s_k / 2          (code rounding, s_k = feature scale)
//                          + K 2^-22 sum_k |y_k| max|E|  (22-bit fixed-point operand + f32 recombination)
//   candidates = { v : approx_v >= max_u approx_u - 2 B }
// so the winner (largest exact logit, lowest index on ties) is always a
// candidate. If more than HEAD_CAP rows qualify (degenerate hidden states)
// every row is rescored.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "pb_common.cuh"
#include "pb_span.h"

namespace pb {
int fill_matrix_f32_t(Mat& m, const float* wt, float threshold, cudaStream_t st);
}

using namespace pb;

constexpr int HEAD_CAP = 16384;  // candidate rows rescored exactly (per token)

struct pb_head {
    int V = 0, d = 0, max_tok = 0, device = 0;
    float* E = nullptr;  // [V][d] f32 (model.py:190 embed)
    float *gamma = nullptr, *beta = nullptr;
    Mat et;  // int8 E^T: K = d inputs, M = V outputs
    // workspace
    uint4* frag = nullptr;
    float* back = nullptr;
    float4* stats = nullptr;
    float* xo = nullptr;
    float* approx = nullptr;  // [max_tok][V]
    float* partials = nullptr;
    int64_t partial_cap = 0;
    int* counters = nullptr;
    int* sel = nullptr;        // [max_tok][4]: max (ordered int), count, flags, pad
    float* bound = nullptr;    // [max_tok]
    int* cand = nullptr;       // [max_tok][HEAD_CAP]
    double* score = nullptr;   // [max_tok][HEAD_CAP]
    int32_t* d_tok = nullptr;  // staging for host token ids
    int32_t* h_tok = nullptr;  // pinned
    float* zero_bias = nullptr;  // [V] (the tied head has no bias)
    float emax = 0.f;            // max |E| (accumulation slack of the bound)
    int64_t bytes = 0;
    std::mutex mu;
};

namespace {

template <class T>
int halloc(pb_head* h, T** p, int64_t count) {
    const size_t b = sizeof(T) * (size_t)std::max<int64_t>(count, 1);
    PB_CHECK_CUDA(cudaMalloc((void**)p, b));
    h->bytes += (int64_t)b;
    return PB_OK;
}

void free_head(pb_head* h) {
    void* ptrs[] = {h->E, h->gamma, h->beta, h->frag, h->back, h->stats, h->xo, h->approx, h->partials,
                    h->counters, h->sel, h->bound, h->cand, h->score, h->d_tok, h->et.codes, h->et.scales, h->zero_bias};
    for (void* p : ptrs) cudaFree(p);
    h->et.free_outliers();
    if (h->h_tok) cudaFreeHost(h->h_tok);
}

__device__ __forceinline__ int ord_of(float f) {  // monotone float -> int map for atomicMax
    const int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float float_of(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

__global__ void k_head_fill(float* p, int n, float v) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = v;
}

__global__ void k_embed_rows(const float* __restrict__ E, int d, const int32_t* __restrict__ tok, int n,
                             float* __restrict__ out) {
    const int i = blockIdx.y;
    if (i >= n) return;
    const float* src = E + (int64_t)tok[i] * d;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < d; k += gridDim.x * blockDim.x)
        out[(int64_t)i * d + k] = src[k];
}

// per token: reset selection state, error bound B (one CTA per token)
__global__ void __launch_bounds__(1024) k_head_bound(const float* __restrict__ x, int d,
                                                     const float4* __restrict__ stats,
                                                     const float* __restrict__ gamma, const float* __restrict__ beta,
                                                     const float* __restrict__ scales, float emax,
                                                     int* __restrict__ sel, float* __restrict__ bound) {
    __shared__ double red[32];
    __shared__ double red2[32];
    const int t = blockIdx.x;
    const float4 st = stats[t];
    double b = 0.0, ay = 0.0;
    for (int k = threadIdx.x; k < d; k += blockDim.x) {
        const float y = fmaf(gamma[k], (x[(int64_t)t * d + k] - st.x) * st.y, beta[k]);  // model.py:271-276
        b += (double)fabsf(y) * (double)scales[k];
        ay += (double)fabsf(y);
    }
    b = warp_sum_d(b);
    ay = warp_sum_d(ay);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        red[w] = b;
        red2[w] = ay;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0, s2 = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
            s += red[i];
            s2 += red2[i];
        }
        // quantization half-step + operand split / fp32 accumulation slack (see header)
        bound[t] = (float)(0.5 * s * 1.001 + (double)d * 2.384185791015625e-7 * s2 * (double)emax + 1e-6);
        sel[t * 4 + 0] = ord_of(-INFINITY);
        sel[t * 4 + 1] = 0;
        sel[t * 4 + 2] = (isfinite(st.x) && isfinite(st.y)) ? 0 : 1;  // non-finite hidden row
    }
}

// per-token max of the approximate logits (and non-finite detection)
__global__ void k_head_max(const float* __restrict__ approx, int V, int* __restrict__ sel) {
    const int t = blockIdx.y;
    const float* a = approx + (int64_t)t * V;
    float m = -INFINITY;
    bool bad = false;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
        const float x = a[v];
        bad |= !isfinite(x);
        m = fmaxf(m, x);
    }
    m = warp_max(m);
    bad = __any_sync(0xffffffffu, bad);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(sel + t * 4, ord_of(m));
        if (bad) atomicOr(sel + t * 4 + 2, 1);
    }
}

__global__ void k_head_cands(const float* __restrict__ approx, int V, int* __restrict__ sel,
                             const float* __restrict__ bound, int* __restrict__ cand) {
    const int t = blockIdx.y;
    const float* a = approx + (int64_t)t * V;
    const float thr = float_of(sel[t * 4]) - 2.f * bound[t];
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
        if (a[v] >= thr) {
            const int i = atomicAdd(sel + t * 4 + 1, 1);
            if (i < HEAD_CAP) cand[(int64_t)t * HEAD_CAP + i] = v;
        }
    }
}

// exact (f64) logit of each candidate row, one warp per row; every row when
// the candidate list overflowed
__global__ void __launch_bounds__(256) k_head_rescore(const float* __restrict__ E, int V, int d,
                                                      const float* __restrict__ x, const float4* __restrict__ stats,
                                                      const float* __restrict__ gamma, const float* __restrict__ beta,
                                                      const int* __restrict__ sel, const int* __restrict__ cand,
                                                      double* __restrict__ score, float* __restrict__ full) {
    const int t = blockIdx.y;
    const int cnt = sel[t * 4 + 1];
    const bool all = cnt > HEAD_CAP;
    const int n = all ? V : cnt;
    const float4 st = stats[t];
    const float* xt = x + (int64_t)t * d;
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
        const int v = all ? i : cand[(int64_t)t * HEAD_CAP + i];
        const float* row = E + (int64_t)v * d;
        double s = 0.0;
        for (int k = lane; k < d; k += 32) {
            const float y = fmaf(gamma[k], (xt[k] - st.x) * st.y, beta[k]);
            s += (double)y * (double)row[k];
        }
        s = warp_sum_d(s);
        if (lane == 0) {
            if (all) full[(int64_t)t * V + v] = (float)s;
            else score[(int64_t)t * HEAD_CAP + i] = s;
        }
    }
}

// argmax over the candidates: largest exact logit, lowest index on ties
__global__ void __launch_bounds__(1024) k_head_pick(int V, const int* __restrict__ sel, const int* __restrict__ cand,
                                                    const double* __restrict__ score, const float* __restrict__ full,
                                                    int32_t* __restrict__ out_tok) {
    __shared__ double bs[32];
    __shared__ int bi[32];
    const int t = blockIdx.x;
    const int cnt = sel[t * 4 + 1];
    const bool all = cnt > HEAD_CAP;
    const int n = all ? V : cnt;
    double best = -INFINITY;
    int bidx = 0x7fffffff;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double s = all ? (double)full[(int64_t)t * V + i] : score[(int64_t)t * HEAD_CAP + i];
        const int v = all ? i : cand[(int64_t)t * HEAD_CAP + i];
        if (s > best || (s == best && v < bidx)) {
            best = s;
            bidx = v;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double s2 = __shfl_xor_sync(0xffffffffu, best, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, bidx, o);
        if (s2 > best || (s2 == best && i2 < bidx)) {
            best = s2;
            bidx = i2;
        }
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        bs[w] = best;
        bi[w] = bidx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i)
            if (bs[i] > best || (bs[i] == best && bi[i] < bidx)) {
                best = bs[i];
                bidx = bi[i];
            }
        out_tok[t] = (sel[t * 4 + 2] & 1) ? -1 : bidx;  // -1: non-finite logits (model.py:442-443)
    }
}

// exact f32 logits (reference lm_head): one warp per vocabulary row, f64 accumulate
__global__ void __launch_bounds__(256) k_head_logits(const float* __restrict__ E, int V, int d,
                                                     const float* __restrict__ x, const float4* __restrict__ stats,
                                                     const float* __restrict__ gamma, const float* __restrict__ beta,
                                                     int n_tok, float* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < V; v += nw) {
        const float* row = E + (int64_t)v * d;
        for (int t = 0; t < n_tok; ++t) {
            const float4 st = stats[t];
            const float* xt = x + (int64_t)t * d;
            double s = 0.0;
            for (int k = lane; k < d; k += 32) s += (double)fmaf(gamma[k], (xt[k] - st.x) * st.y, beta[k]) * (double)row[k];
            s = warp_sum_d(s);
            if (lane == 0) out[(int64_t)t * V + v] = (float)s;
        }
    }
}

int sms_of(int dev) {
    int s = 148;
    cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
    return s;
}

// LN statistics of the hidden rows (k_rowstats through the GEMV prologue) and
// the int8-digit fragments of the normalized rows
int head_prologue(pb_head* h, const float* x, int n, cudaStream_t st) {
    ProSrc src;  // SRC_STATS: exact row statistics
    return launch_prologue(PRO_LN, src, x, n, h->d, h->et.Kp, h->gamma, h->beta, h->et, choose_tc(n), h->frag,
                           h->back, h->stats, h->xo, nullptr, st);
}

}  // namespace

extern "C" {

int pb_head_create(int32_t vocab, int32_t hidden, int32_t max_tokens, int32_t device, pb_head** out) {
    PB_REQUIRE(out && vocab > 0 && hidden > 0 && max_tokens > 0 && max_tokens <= 32, PB_ERR_BAD_REQUEST,
               "bad head shape (max_tokens 1..32)");
    PB_CHECK_CUDA(cudaSetDevice(device));
    auto* h = new pb_head();
    h->V = vocab;
    h->d = hidden;
    h->max_tok = max_tokens;
    h->device = device;
    Mat& m = h->et;
    m.K = hidden;
    m.M = vocab;
    m.Kp = (int)round_up(hidden, 32);
    m.Mp = (int)round_up(vocab, 128);
    m.int8 = true;
    const int NT = max_tokens;
    int rc = PB_OK;
    if (!rc) rc = halloc(h, &h->E, (int64_t)vocab * hidden);
    if (!rc) rc = halloc(h, &h->gamma, hidden);
    if (!rc) rc = halloc(h, &h->beta, hidden);
    if (!rc) rc = halloc(h, &m.codes, (int64_t)m.Mp * m.Kp);
    if (!rc) rc = halloc(h, &m.scales, m.Kp);
    if (!rc) rc = halloc(h, &h->frag, (int64_t)(NT + 31) * m.Kp * 4 / 16 + 64);
    if (!rc) rc = halloc(h, &h->back, NT);
    if (!rc) rc = halloc(h, &h->stats, NT);
    if (!rc) rc = halloc(h, &h->xo, (int64_t)NT * hidden);
    if (!rc) rc = halloc(h, &h->approx, (int64_t)NT * vocab);
    h->partial_cap = (int64_t)8 << 20;
    if (!rc) rc = halloc(h, &h->partials, h->partial_cap);
    if (!rc) rc = halloc(h, &h->counters, 1 << 20);
    if (!rc) rc = halloc(h, &h->sel, 4 * NT);
    if (!rc) rc = halloc(h, &h->bound, NT);
    if (!rc) rc = halloc(h, &h->cand, (int64_t)NT * HEAD_CAP);
    if (!rc) rc = halloc(h, &h->score, (int64_t)NT * HEAD_CAP);
    if (!rc) rc = halloc(h, &h->d_tok, NT);
    if (!rc) rc = halloc(h, &h->zero_bias, vocab);
    if (!rc && cudaMemset(h->zero_bias, 0, sizeof(float) * vocab) != cudaSuccess) rc = PB_ERR_GENERIC;
    if (!rc && cudaMallocHost((void**)&h->h_tok, sizeof(int32_t) * NT) != cudaSuccess) rc = PB_ERR_GENERIC;
    if (!rc && cudaMemset(h->counters, 0, sizeof(int) << 20) != cudaSuccess) rc = PB_ERR_GENERIC;
    if (!rc && cudaMemset(m.scales, 0, sizeof(float) * m.Kp) != cudaSuccess) rc = PB_ERR_GENERIC;
    if (rc) {
        free_head(h);
        delete h;
        set_error("head allocation failed");
        return PB_ERR_CAPACITY;
    }
    *out = h;
    return PB_OK;
}

int pb_head_destroy(pb_head* h) {
    if (!h) return PB_OK;
    cudaSetDevice(h->device);
    cudaDeviceSynchronize();
    free_head(h);
    delete h;
    return PB_OK;
}

int64_t pb_head_device_bytes(const pb_head* h) { return h ? h->bytes : 0; }

__global__ void k_absmax_all(const float* __restrict__ p, int64_t n, int* __restrict__ out) {
    float m = 0.f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        m = fmaxf(m, fabsf(p[i]));
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_int(m));
}

// int8 copy of E^T (the reference weight quantizer's semantics, threshold 6.0)
// and max |E| for the error bound
static int head_finish_load(pb_head* h, cudaStream_t st) {
    if (int rc = fill_matrix_f32_t(h->et, h->E, 6.0f, st)) return rc;
    int* d = h->sel;  // scratch
    PB_CHECK_CUDA(cudaMemsetAsync(d, 0, sizeof(int), st));
    k_absmax_all<<<sms_of(h->device) * 4, 256, 0, st>>>(h->E, (int64_t)h->V * h->d, d);
    if (int rc = launch_check("absmax_all")) return rc;
    int bits = 0;
    PB_CHECK_CUDA(cudaMemcpyAsync(&bits, d, sizeof(int), cudaMemcpyDeviceToHost, st));
    PB_CHECK_CUDA(cudaStreamSynchronize(st));
    std::memcpy(&h->emax, &bits, sizeof(float));
    return PB_OK;
}

int pb_head_gen(pb_head* h, uint64_t key_embed, void* stream) {
    PB_REQUIRE(h, PB_ERR_BAD_REQUEST, "null head");
    std::lock_guard<std::mutex> lk(h->mu);
    PB_CHECK_CUDA(cudaSetDevice(h->device));
    auto st = (cudaStream_t)stream;
    if (int rc = pb_gen_tensor(key_embed, 0, (int64_t)h->V * h->d, h->E, stream)) return rc;
    k_head_fill<<<64, 256, 0, st>>>(h->gamma, h->d, 1.f);  // final_ln gamma 1, beta 0 (model.py:205-206)
    PB_CHECK_CUDA(cudaMemsetAsync(h->beta, 0, sizeof(float) * h->d, st));
    if (int rc = head_finish_load(h, st)) return rc;
    PB_CHECK_CUDA(cudaStreamSynchronize(st));
    return PB_OK;
}

int pb_head_load(pb_head* h, const float* d_embed, const float* d_gamma, const float* d_beta, void* stream) {
    PB_REQUIRE(h && d_embed && d_gamma && d_beta, PB_ERR_BAD_REQUEST, "null argument");
    std::lock_guard<std::mutex> lk(h->mu);
    PB_CHECK_CUDA(cudaSetDevice(h->device));
    auto st = (cudaStream_t)stream;
    PB_CHECK_CUDA(cudaMemcpyAsync(h->E, d_embed, sizeof(float) * (size_t)h->V * h->d, cudaMemcpyDeviceToDevice, st));
    PB_CHECK_CUDA(cudaMemcpyAsync(h->gamma, d_gamma, sizeof(float) * h->d, cudaMemcpyDeviceToDevice, st));
    PB_CHECK_CUDA(cudaMemcpyAsync(h->beta, d_beta, sizeof(float) * h->d, cudaMemcpyDeviceToDevice, st));
    if (int rc = head_finish_load(h, st)) return rc;
    PB_CHECK_CUDA(cudaStreamSynchronize(st));
    return PB_OK;
}

static int embed_dev(pb_head* h, const int32_t* d_tokens, int32_t n, float* d_out, cudaStream_t st) {
    dim3 grid((unsigned)std::min<int64_t>(ceil_div(h->d, 256), 64), (unsigned)n);
    k_embed_rows<<<grid, 256, 0, st>>>(h->E, h->d, d_tokens, n, d_out);
    return launch_check("embed_rows");
}

int pb_head_embed(pb_head* h, const int32_t* h_tokens, int32_t n, float* d_out, void* stream) {
    PB_REQUIRE(h && d_out && (h_tokens || n == 0), PB_ERR_BAD_REQUEST, "null argument");
    PB_REQUIRE(n >= 0 && n <= h->max_tok, PB_ERR_CAPACITY, "too many tokens for the head workspace");
    for (int i = 0; i < n; ++i)
        PB_REQUIRE(h_tokens[i] >= 0 && h_tokens[i] < h->V, PB_ERR_BAD_REQUEST, "token out of range");  // model.py:423-424
    if (n == 0) return PB_OK;
    std::lock_guard<std::mutex> lk(h->mu);
    PB_CHECK_CUDA(cudaSetDevice(h->device));
    auto st = (cudaStream_t)stream;
    PB_CHECK_CUDA(cudaStreamSynchronize(st));  // pinned staging reuse
    std::memcpy(h->h_tok, h_tokens, sizeof(int32_t) * n);
    PB_CHECK_CUDA(cudaMemcpyAsync(h->d_tok, h->h_tok, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    return embed_dev(h, h->d_tok, n, d_out, st);
}

int pb_head_embed_device(pb_head* h, const int32_t* d_tokens, int32_t n, float* d_out, void* stream) {
    PB_REQUIRE(h && d_tokens && d_out, PB_ERR_BAD_REQUEST, "null argument");
    PB_REQUIRE(n > 0 && n <= h->max_tok, PB_ERR_CAPACITY, "bad token count");
    std::lock_guard<std::mutex> lk(h->mu);
    PB_CHECK_CUDA(cudaSetDevice(h->device));
    return embed_dev(h, d_tokens, n, d_out, (cudaStream_t)stream);
}

int pb_head_logits(pb_head* h, const float* d_hidden, int32_t n, float* d_logits, void* stream) {
    PB_REQUIRE(h && d_hidden && d_logits, PB_ERR_BAD_REQUEST, "null argument");
    PB_REQUIRE(n > 0 && n <= h->max_tok, PB_ERR_CAPACITY, "bad token count");
    std::lock_guard<std::mutex> lk(h->mu);
    PB_CHECK_CUDA(cudaSetDevice(h->device));
    auto st = (cudaStream_t)stream;
    if (int rc = head_prologue(h, d_hidden, n, st)) return rc;
    k_head_logits<<<sms_of(h->device) * 8, 256, 0, st>>>(h->E, h->V, h->d, d_hidden, h->stats, h->gamma, h->beta, n,
                                                         d_logits);
    return launch_check("head_logits");
}

int pb_head_greedy(pb_head* h, const float* d_hidden, int32_t n, int32_t* d_tokens, float* d_next_embed,
                   void* stream) {
    PB_REQUIRE(h && d_hidden && d_tokens, PB_ERR_BAD_REQUEST, "null argument");
    PB_REQUIRE(n > 0 && n <= h->max_tok, PB_ERR_CAPACITY, "bad token count");
    std::lock_guard<std::mutex> lk(h->mu);
    PB_CHECK_CUDA(cudaSetDevice(h->device));
    auto st = (cudaStream_t)stream;
    const int sms = sms_of(h->device);
    if (int rc = head_prologue(h, d_hidden, n, st)) return rc;
    // approximate logits: the block GEMV over the int8 E^T, plain store epilogue
    Epi e{};
    e.kind = EPI_PLAIN;
    e.M = h->V;
    e.bias = h->zero_bias;
    e.n_outl = h->et.n_outl;
    e.outl_idx = h->et.outl_idx;
    e.outl_rows = h->et.outl_rows;
    e.xo = h->xo;
    e.out = h->approx;
    Act a{h->frag, h->back, n, choose_tc(n)};
    if (int rc = launch_gemv(h->et, a, e, h->partials, h->counters, h->partial_cap, st)) return rc;
    k_head_bound<<<n, 1024, 0, st>>>(d_hidden, h->d, h->stats, h->gamma, h->beta, h->et.scales, h->emax, h->sel,
                                     h->bound);
    if (int rc = launch_check("head_bound")) return rc;
    k_head_max<<<dim3((unsigned)sms, (unsigned)n), 256, 0, st>>>(h->approx, h->V, h->sel);
    k_head_cands<<<dim3((unsigned)sms, (unsigned)n), 256, 0, st>>>(h->approx, h->V, h->sel, h->bound, h->cand);
    k_head_rescore<<<dim3((unsigned)sms * 4, (unsigned)n), 256, 0, st>>>(h->E, h->V, h->d, d_hidden, h->stats,
                                                                         h->gamma, h->beta, h->sel, h->cand, h->score,
                                                                         h->approx);
    k_head_pick<<<n, 1024, 0, st>>>(h->V, h->sel, h->cand, h->score, h->approx, d_tokens);
    if (int rc = launch_check("head_select")) return rc;
    if (d_next_embed) return embed_dev(h, d_tokens, n, d_next_embed, st);
    return PB_OK;
}

}  // extern "C"
