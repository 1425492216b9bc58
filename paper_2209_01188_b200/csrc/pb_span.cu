// Block-span runtime and C-ABI: weights of a contiguous block range, the
// paged KV pool, workspaces, and the per-step launch sequence of
// block_forward (model.py:314-380) looped over the span (server.py:383-385),
// batched over sessions.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "pb_common.cuh"
#include "pb_span.h"

namespace pb {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

static uint64_t* g_trace = nullptr;
static int64_t g_trace_cap = 0, g_trace_used = 0;
static std::vector<int64_t> g_trace_meta;

static bool trace_active() { return g_trace != nullptr; }
constexpr int GRAPH_MAX_TOKENS = 64;

uint64_t* trace_region(int kind, int ctas) {
    if (!g_trace || g_trace_used + TRACE_WORDS * (int64_t)ctas > g_trace_cap) return nullptr;
    uint64_t* p = g_trace + g_trace_used;
    g_trace_meta.insert(g_trace_meta.end(), {(int64_t)kind, (int64_t)ctas, g_trace_used});
    g_trace_used += TRACE_WORDS * (int64_t)ctas;
    return p;
}

}  // namespace pb

using namespace pb;

extern "C" int pb_trace_set(void* d_buf, int64_t cap_words) {
    g_trace = static_cast<uint64_t*>(d_buf);
    g_trace_cap = d_buf ? cap_words : 0;
    g_trace_used = 0;
    g_trace_meta.clear();
    return PB_OK;
}

extern "C" int64_t pb_trace_meta(int64_t* h_out, int64_t cap_triples) {
    const int64_t n = (int64_t)g_trace_meta.size() / 3;
    if (h_out)
        for (int64_t i = 0; i < std::min(n, cap_triples) * 3; ++i) h_out[i] = g_trace_meta[i];
    return n;
}

#include "pb_span_impl.h"

namespace {

template <class T>
int dalloc(pb_span* s, T** p, int64_t count) {
    const size_t b = sizeof(T) * (size_t)std::max<int64_t>(count, 1);
    PB_CHECK_CUDA(cudaMalloc((void**)p, b));
    s->bytes += (int64_t)b;
    return PB_OK;
}

int alloc_mat(pb_span* s, Mat& m, int K, int M, bool int8) {
    m.K = K;
    m.M = M;
    m.Kp = (int)round_up(K, 32);
    m.Mp = (int)round_up(M, 128);  // 128-row groups (pb_gemv.cu)
    m.int8 = int8;
    if (int8) {
        if (int rc = dalloc(s, &m.codes, (int64_t)m.Mp * m.Kp)) return rc;
        if (int rc = dalloc(s, &m.scales, m.Kp)) return rc;
        PB_CHECK_CUDA(cudaMemset(m.scales, 0, sizeof(float) * m.Kp));
    } else {
        if (int rc = dalloc(s, &m.w32, (int64_t)K * M)) return rc;
    }
    return PB_OK;
}

void free_span(pb_span* s) {
    for (auto& b : s->blocks) {
        for (auto& m : b.mat) {
            cudaFree(m.codes);
            cudaFree(m.tcodes);
            cudaFree(m.scales);
            cudaFree(m.w32);
            m.free_outliers();
        }
        cudaFree(b.ln1_g);
        cudaFree(b.ln1_b);
        cudaFree(b.ln2_g);
        cudaFree(b.ln2_b);
        for (auto* p : b.bias) cudaFree(p);
    }
    void* ptrs[] = {s->kv, s->slopes, s->xa, s->mid, s->q, s->ctx, s->act, s->xo, s->y32, s->frag, s->bcanon, s->back, s->stats, s->pst_x, s->pst_mid, s->tokmax_ctx, s->tokmax_act,
                    s->partials, s->counters, s->attn_part, s->d_tok_seq, s->d_tok_pos, s->d_pages, s->d_grp_first, s->d_grp_count,
                    s->hop_codes, s->hop_scales, s->d_unit_base, s->sk_acc, s->train_ws};
    for (void* p : ptrs) cudaFree(p);
    for (int i = 0; i < pb_span::NSLOT; ++i) {
        if (s->h_meta[i]) cudaFreeHost(s->h_meta[i]);
        if (s->h_ub[i]) cudaFreeHost(s->h_ub[i]);
        if (s->meta_ev[i]) cudaEventDestroy(s->meta_ev[i]);
    }
    for (auto e : s->prof_ev) cudaEventDestroy(e);
    for (auto& kv : s->graphs) cudaGraphExecDestroy(kv.second.exec);
    s->graphs.clear();
    if (s->cap_stream) cudaStreamDestroy(s->cap_stream);
    cudaFree(s->g_in);
    cudaFree(s->g_out);
}

__global__ void k_fill(float* p, int64_t n, float v) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) p[i] = v;
}

int fill(float* p, int64_t n, float v, cudaStream_t st) {
    k_fill<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 1024), 256, 0, st>>>(p, n, v);
    return launch_check("fill");
}

}  // namespace

extern "C" {

const char* pb_last_error(void) { return pb::g_err.c_str(); }
int pb_version(void) { return 1; }

int pb_span_create(const pb_span_config* cfg, pb_span** out) {
    PB_REQUIRE(cfg && out, PB_ERR_BAD_REQUEST, "null argument");
    PB_REQUIRE(cfg->hidden > 0 && cfg->n_heads > 0 && cfg->hidden % cfg->n_heads == 0, PB_ERR_BAD_REQUEST,
               "hidden must be a positive multiple of n_heads");
    PB_REQUIRE(cfg->n_blocks > 0 && cfg->mlp_ratio > 0 && cfg->max_seq > 0, PB_ERR_BAD_REQUEST, "bad span shape");
    PB_REQUIRE(cfg->page_tokens > 0 && cfg->n_pages > 0 && cfg->max_tokens > 0 && cfg->max_seqs > 0,
               PB_ERR_BAD_REQUEST, "bad pool/workspace sizes");
    PB_CHECK_CUDA(cudaSetDevice(cfg->device));
    auto* s = new pb_span();
    s->cfg = *cfg;
    s->d = cfg->hidden;
    s->H = cfg->n_heads;
    s->dh = cfg->hidden / cfg->n_heads;
    s->rd = cfg->hidden * cfg->mlp_ratio;
    s->max_pages = (int)ceil_div(cfg->max_seq, cfg->page_tokens);
    const bool int8 = cfg->weights == PB_WEIGHTS_INT8;
    const int d = s->d, rd = s->rd;
    s->blocks.resize(cfg->n_blocks);
    int rc = PB_OK;
    for (auto& b : s->blocks) {
        if ((rc = alloc_mat(s, b.mat[0], d, 3 * d, int8))) break;
        if ((rc = alloc_mat(s, b.mat[1], d, d, int8))) break;
        if ((rc = alloc_mat(s, b.mat[2], d, rd, int8))) break;
        if ((rc = alloc_mat(s, b.mat[3], rd, d, int8))) break;
        if ((rc = dalloc(s, &b.ln1_g, d)) || (rc = dalloc(s, &b.ln1_b, d)) || (rc = dalloc(s, &b.ln2_g, d)) ||
            (rc = dalloc(s, &b.ln2_b, d)))
            break;
        if ((rc = dalloc(s, &b.bias[0], 3 * d)) || (rc = dalloc(s, &b.bias[1], d)) || (rc = dalloc(s, &b.bias[2], rd)) ||
            (rc = dalloc(s, &b.bias[3], d)))
            break;
    }
    const int NT = cfg->max_tokens;
    s->kv_block_elems = (int64_t)cfg->n_pages * 2 * s->H * cfg->page_tokens * s->dh;
    if (!rc) rc = dalloc(s, &s->kv, s->kv_block_elems * cfg->n_blocks);
    if (!rc) rc = dalloc(s, &s->slopes, s->H);
    if (!rc) rc = dalloc(s, &s->xa, (int64_t)NT * d);
    if (!rc) rc = dalloc(s, &s->mid, (int64_t)NT * d);
    if (!rc) rc = dalloc(s, &s->q, (int64_t)NT * d);
    if (!rc) rc = dalloc(s, &s->ctx, (int64_t)NT * d);
    if (!rc) rc = dalloc(s, &s->act, (int64_t)NT * rd);
    if (!rc && int8) rc = dalloc(s, &s->xo, (int64_t)NT * rd);
    if (!rc && !int8) rc = dalloc(s, &s->y32, (int64_t)NT * rd);
    const int64_t kp_max = round_up(rd, 32);
    if (!rc && int8) rc = dalloc(s, &s->frag, (int64_t)(NT + 31) * kp_max * 4 / 16 + 64);
    if (cfg->tc_min_tokens > 0) s->tc_min = cfg->tc_min_tokens;  // else TC_MIN_TOKENS_DEFAULT
    if (!rc && int8 && NT >= s->tc_min) rc = dalloc(s, &s->bcanon, ceil_div(NT, TC_TOKENS) * (kp_max / 32) * 3 * TC_TOKENS * 32);
    if (!rc) rc = dalloc(s, &s->back, NT);
    if (!rc) rc = dalloc(s, &s->stats, NT);
    if (!rc) rc = dalloc(s, &s->pst_x, (int64_t)NT * ceil_div(d, 128));
    if (!rc) rc = dalloc(s, &s->pst_mid, (int64_t)NT * ceil_div(d, 128));
    if (!rc) rc = dalloc(s, &s->tokmax_ctx, NT);
    if (!rc) rc = dalloc(s, &s->tokmax_act, NT);
    s->partial_cap = (int64_t)8 << 20;
    if (!rc) rc = dalloc(s, &s->partials, s->partial_cap);
    if (!rc && cfg->graphs) {
        rc = dalloc(s, &s->g_in, (int64_t)GRAPH_MAX_TOKENS * d);
        if (!rc) rc = dalloc(s, &s->g_out, (int64_t)GRAPH_MAX_TOKENS * d);
        if (!rc && cudaStreamCreateWithFlags(&s->cap_stream, cudaStreamNonBlocking) != cudaSuccess) rc = PB_ERR_GENERIC;
    }
    if (!rc && s->bcanon) {  // batched-decode tcgen05 kernel: split-row-group sums, zero between launches
        s->sk_acc_elems = ceil_div(std::max(3 * d, rd), 128) * 96 * 128;
        rc = dalloc(s, &s->sk_acc, s->sk_acc_elems);
        if (!rc && cudaMemset(s->sk_acc, 0, sizeof(int) * s->sk_acc_elems) != cudaSuccess) rc = PB_ERR_GENERIC;
    }
    if (!rc) rc = dalloc(s, &s->counters, 1 << 20);
    s->attn_cap = attention_part_floats(NT, s->H, s->dh, cfg->max_seq);
    if (!rc) rc = dalloc(s, &s->attn_part, s->attn_cap);
    s->meta_ints = 4 * (int64_t)NT + (int64_t)cfg->max_seqs * s->max_pages;
    if (!rc) rc = dalloc(s, &s->d_tok_seq, NT);
    if (!rc) rc = dalloc(s, &s->d_tok_pos, NT);
    if (!rc) rc = dalloc(s, &s->d_pages, (int64_t)cfg->max_seqs * s->max_pages);
    if (!rc) rc = dalloc(s, &s->d_grp_first, NT);
    if (!rc) rc = dalloc(s, &s->d_grp_count, NT);
    if (!rc) rc = dalloc(s, &s->d_unit_base, NT + 1);
    if (!rc) rc = dalloc(s, &s->hop_codes, (int64_t)NT * d);
    if (!rc) rc = dalloc(s, &s->hop_scales, ceil_div((int64_t)NT * d, 64));
    for (int i = 0; !rc && i < pb_span::NSLOT; ++i) {
        if (cudaMallocHost((void**)&s->h_meta[i], sizeof(int32_t) * s->meta_ints) != cudaSuccess ||
            cudaMallocHost((void**)&s->h_ub[i], sizeof(int64_t) * (NT + 1)) != cudaSuccess ||
            cudaEventCreateWithFlags(&s->meta_ev[i], cudaEventDisableTiming) != cudaSuccess) {
            set_error("pinned staging allocation failed");
            rc = PB_ERR_GENERIC;
        }
    }
    if (!rc && cudaMemset(s->counters, 0, sizeof(int) << 20) != cudaSuccess) rc = PB_ERR_GENERIC;
    if (!rc) {
        std::vector<float> sl(s->H);
        for (int h = 1; h <= s->H; ++h) sl[h - 1] = (float)std::pow(2.0, -8.0 * h / s->H);  // model.py:301-302
        if (cudaMemcpy(s->slopes, sl.data(), sizeof(float) * s->H, cudaMemcpyHostToDevice) != cudaSuccess)
            rc = PB_ERR_GENERIC;
    }
    if (rc) {
        if (pb::g_err.empty() || pb::g_err.find("out of memory") != std::string::npos)
            set_error("span allocation failed: " + pb::g_err);
        free_span(s);
        delete s;
        return rc == PB_ERR_GENERIC ? PB_ERR_CAPACITY : rc;
    }
    *out = s;
    return PB_OK;
}

int pb_span_destroy(pb_span* span) {
    if (!span) return PB_OK;
    cudaSetDevice(span->cfg.device);
    cudaDeviceSynchronize();
    free_span(span);
    delete span;
    return PB_OK;
}

int64_t pb_span_device_bytes(const pb_span* span) { return span ? span->bytes : 0; }

static int init_block_vectors(pb_span* s, BlockW& b, cudaStream_t st) {
    const int d = s->d;
    if (int rc = fill(b.ln1_g, d, 1.f, st)) return rc;
    if (int rc = fill(b.ln2_g, d, 1.f, st)) return rc;
    PB_CHECK_CUDA(cudaMemsetAsync(b.ln1_b, 0, sizeof(float) * d, st));
    PB_CHECK_CUDA(cudaMemsetAsync(b.ln2_b, 0, sizeof(float) * d, st));
    PB_CHECK_CUDA(cudaMemsetAsync(b.bias[0], 0, sizeof(float) * 3 * d, st));
    PB_CHECK_CUDA(cudaMemsetAsync(b.bias[1], 0, sizeof(float) * d, st));
    PB_CHECK_CUDA(cudaMemsetAsync(b.bias[2], 0, sizeof(float) * s->rd, st));
    PB_CHECK_CUDA(cudaMemsetAsync(b.bias[3], 0, sizeof(float) * d, st));
    return PB_OK;
}

static int block_bounds(pb_span* s, BlockW& b, cudaStream_t st) {
    if (s->cfg.weights != PB_WEIGHTS_INT8) return PB_OK;
    if (int rc = bound_consts(b.ln1_g, b.ln1_b, b.mat[0].scales, s->d, &b.gs1, &b.bs1, st)) return rc;
    return bound_consts(b.ln2_g, b.ln2_b, b.mat[2].scales, s->d, &b.gs2, &b.bs2, st);
}

int pb_span_gen_block(pb_span* span, int32_t j, uint64_t key_wqkv, uint64_t key_wo, uint64_t key_win,
                      uint64_t key_wout, float outlier_boost, int32_t boost_every, void* stream) {
    PB_REQUIRE(span && j >= 0 && j < span->cfg.n_blocks, PB_ERR_BAD_REQUEST, "block index out of range");
    std::lock_guard<std::mutex> lk(span->mu);
    PB_CHECK_CUDA(cudaSetDevice(span->cfg.device));
    auto st = (cudaStream_t)stream;
    BlockW& b = span->blocks[j];
    if (int rc = init_block_vectors(span, b, st)) return rc;
    const uint64_t keys[4] = {key_wqkv, key_wo, key_win, key_wout};
    const int every = outlier_boost > 0.f ? boost_every : 0;
    for (int m = 0; m < 4; ++m)
        if (int rc = fill_matrix_gen(b.mat[m], keys[m], span->cfg.outlier_threshold, outlier_boost, every, st))
            return rc;
    if (int rc = block_bounds(span, b, st)) return rc;
    PB_CHECK_CUDA(cudaStreamSynchronize(st));
    return PB_OK;
}

int pb_span_load_block(pb_span* span, int32_t j, const float* d_ln1_g, const float* d_ln1_b, const float* d_wqkv,
                       const float* d_bqkv, const float* d_wo, const float* d_bo, const float* d_ln2_g,
                       const float* d_ln2_b, const float* d_win, const float* d_bin, const float* d_wout,
                       const float* d_bout, void* stream) {
    PB_REQUIRE(span && j >= 0 && j < span->cfg.n_blocks, PB_ERR_BAD_REQUEST, "block index out of range");
    std::lock_guard<std::mutex> lk(span->mu);
    PB_CHECK_CUDA(cudaSetDevice(span->cfg.device));
    auto st = (cudaStream_t)stream;
    BlockW& b = span->blocks[j];
    const int d = span->d, rd = span->rd;
    auto cp = [&](float* dst, const float* src, int64_t n) {
        return cudaMemcpyAsync(dst, src, sizeof(float) * n, cudaMemcpyDeviceToDevice, st);
    };
    PB_CHECK_CUDA(cp(b.ln1_g, d_ln1_g, d));
    PB_CHECK_CUDA(cp(b.ln1_b, d_ln1_b, d));
    PB_CHECK_CUDA(cp(b.ln2_g, d_ln2_g, d));
    PB_CHECK_CUDA(cp(b.ln2_b, d_ln2_b, d));
    PB_CHECK_CUDA(cp(b.bias[0], d_bqkv, 3 * d));
    PB_CHECK_CUDA(cp(b.bias[1], d_bo, d));
    PB_CHECK_CUDA(cp(b.bias[2], d_bin, rd));
    PB_CHECK_CUDA(cp(b.bias[3], d_bout, d));
    const float* ws[4] = {d_wqkv, d_wo, d_win, d_wout};
    for (int m = 0; m < 4; ++m)
        if (int rc = fill_matrix_f32(b.mat[m], ws[m], span->cfg.outlier_threshold, st)) return rc;
    if (int rc = block_bounds(span, b, st)) return rc;
    PB_CHECK_CUDA(cudaStreamSynchronize(st));
    return PB_OK;
}

int pb_span_outliers(const pb_span* span, int32_t j, int32_t m, int32_t* h_idx, int32_t cap, int32_t* n) {
    PB_REQUIRE(span && j >= 0 && j < span->cfg.n_blocks && m >= 0 && m < 4, PB_ERR_BAD_REQUEST, "bad index");
    const Mat& mat = span->blocks[j].mat[m];
    *n = mat.n_outl;
    for (int i = 0; i < std::min(cap, mat.n_outl); ++i) h_idx[i] = mat.h_outl_idx[i];
    return PB_OK;
}

int pb_span_read_codes(const pb_span* span, int32_t j, int32_t m, int8_t* h_codes, float* h_scales) {
    PB_REQUIRE(span && j >= 0 && j < span->cfg.n_blocks && m >= 0 && m < 4, PB_ERR_BAD_REQUEST, "bad index");
    const Mat& mat = span->blocks[j].mat[m];
    PB_REQUIRE(mat.int8, PB_ERR_BAD_REQUEST, "span holds f32 weights");
    PB_CHECK_CUDA(cudaSetDevice(span->cfg.device));
    int8_t* tmp = nullptr;
    PB_CHECK_CUDA(cudaMalloc(&tmp, (size_t)mat.M * mat.K));
    int rc = untile_codes(mat, tmp, 0);
    if (!rc && cudaMemcpy(h_codes, tmp, (size_t)mat.M * mat.K, cudaMemcpyDeviceToHost) != cudaSuccess)
        rc = PB_ERR_GENERIC;
    if (!rc && cudaMemcpy(h_scales, mat.scales, sizeof(float) * mat.K, cudaMemcpyDeviceToHost) != cudaSuccess)
        rc = PB_ERR_GENERIC;
    cudaFree(tmp);
    return rc;
}

int32_t pb_span_last_launches(const pb_span* span) { return span ? span->last_launches : 0; }

}  // extern "C"

// ------------------------------------------------------------------ step

// kinds: 0 int8 GEMV, 1 attention (split + combine), 2 prologue, 3 f32 GEMM, 4 wire codec
static int prof_begin(pb_span* s, cudaStream_t st) {
    if (!s->prof_on) return -1;
    const int i = (int)s->prof.size() * 2;
    while ((int)s->prof_ev.size() < i + 2) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return -1;
        s->prof_ev.push_back(e);
    }
    cudaEventRecord(s->prof_ev[i], st);
    return i;
}
static void prof_end(pb_span* s, int ev, int kind, double bytes, cudaStream_t st) {
    if (ev < 0) return;
    cudaEventRecord(s->prof_ev[ev + 1], st);
    s->prof.push_back({kind, ev, bytes});
}

// One step through every hosted block. int8 spans chain the operand statistics
// through the epilogues: out-GEMV (block j-1) -> per-128-row LN summaries ->
// qkv operand of block j; attention -> max|ctx s_wo| -> wo operand; wo-GEMV ->
// LN summaries -> wmlp_in operand; wmlp_in-GEMV -> max|act s_out| -> wmlp_out
// operand. Only block 0's LN1 needs a separate row-statistics kernel.
static int run_blocks(pb_span* s, int n_tok, int max_pos, const float* in, float* out, cudaStream_t st,
                      float* tape = nullptr) {
    const int d = s->d, rd = s->rd;
    const bool int8 = s->cfg.weights == PB_WEIGHTS_INT8;
    const int tc = choose_tc(n_tok);
    const bool use_tc = int8 && s->bcanon && n_tok >= s->tc_min;
    // batched decode (<= 32 tokens): the stream-K tcgen05 kernel on a 16- or 32-token tile
    const int sk_tile = n_tok <= 16 ? 16 : 32;
    const bool use_sk = use_tc && n_tok <= 32;
    const int MGd = (int)ceil_div(d, 128);
    int launches = 0;
    for (int j = 0; j < s->cfg.n_blocks; ++j) {
        BlockW& b = s->blocks[j];
        const float* x_in = j == 0 ? in : s->xa;
        float* x_out = j == s->cfg.n_blocks - 1 ? out : s->xa;
        if (tape)  // FORWARD tape: block j's input rows (pb_train.cu recomputes the rest)
            PB_CHECK_CUDA(cudaMemcpyAsync(tape + (int64_t)j * n_tok * d, x_in, sizeof(float) * (size_t)n_tok * d,
                                          cudaMemcpyDeviceToDevice, st));
        half* kvb = s->kv + s->kv_block_elems * j;
        Epi base{};
        base.n_outl = 0;
        base.kv = kvb;
        base.tok_seq = s->d_tok_seq;
        base.tok_pos = s->d_tok_pos;
        base.pages = s->d_pages;
        base.max_pages = s->max_pages;
        base.H = s->H;
        base.dh = s->dh;
        base.P = s->cfg.page_tokens;
        base.d = d;
        auto matmul = [&](int mi, int mode, const ProSrc& src, const float* x, int K, const float* g,
                          const float* be, Epi e) -> int {
            const Mat& m = b.mat[mi];
            e.M = m.M;
            e.bias = b.bias[mi];
            if (use_tc) {
                // prefill / large batches: tcgen05 GEMM. LN operands take exact
                // row statistics (k_rowstats); scale operands keep the atomicMax range.
                e.n_outl = m.n_outl;
                e.outl_idx = m.outl_idx;
                e.outl_rows = m.outl_rows;
                e.xo = s->xo;
                e.pstats = nullptr;
                ProSrc srct = src;
                if (mode == PRO_LN) {
                    srct.kind = SRC_STATS;
                    srct.pstats = nullptr;
                }
                int ev = prof_begin(s, st);
                if (int rc = launch_prologue(mode, srct, x, n_tok, K, m.Kp, g, be, m, tc, nullptr, s->back, s->stats,
                                             s->xo, nullptr, st, s->bcanon, use_sk ? sk_tile : TC_TOKENS))
                    return rc;
                prof_end(s, ev, 2, 4.0 * n_tok * K, st);
                launches += srct.kind == SRC_STATS ? 3 : 2;
                Act a{nullptr, s->back, n_tok, 0};
                ev = prof_begin(s, st);
                if (use_sk) {
                    // memory-bound: algorithmic bytes as for the GEMV (PROF kind 6)
                    const double bytes = (double)m.M * m.K + 4.0 * m.K + 4.0 * m.M + 4.0 * m.n_outl * m.M;
                    int rc = launch_gemm_tc_sk(m, s->bcanon, sk_tile, a, e, s->sk_acc, 4 * s->sk_acc_elems,
                                               s->counters + (1 << 18), st);
                    prof_end(s, ev, 6, bytes, st);
                    return rc;
                }
                int rc = launch_gemm_tc(m, s->bcanon, a, e, st);
                // tensor roofline: int8 ops issued = 2 * M * K * 3 digit columns per token
                prof_end(s, ev, 5, 2.0 * m.M * m.K * 3.0 * n_tok, st);
                return rc;
            }
            if (int8) {
                e.n_outl = m.n_outl;
                e.outl_idx = m.outl_idx;
                e.outl_rows = m.outl_rows;
                e.xo = s->xo;
                Act a{s->frag, s->back, n_tok, tc};
                // fused operand warps for every batch-1 decode GEMV: round 1 measured them
                // ~1 % slower at the 176B shape (their power lowered the capped SM clock);
                // since the operand warps overlap their statistics with the first inputs
                // they win there too (bench: 33.4 -> 35.0 steps/s, 0.98 of the sequential
                // roofline, at a lower 1670 MHz capped clock), besides 560M and 7B1
                if (!s->cfg.operand_kernel && gemv_fusable(a, K)) {
                    // decode: the GEMV's operand warp builds the int8-digit operand itself;
                    // the QKV launch resets the two range accumulators of this block
                    // (attention -> wo, wmlp_in epilogue -> wmlp_out), whose previous
                    // readers (block j-1) have completed by then
                    ProArgs pa;
                    if (int rc = prepare_fused_operand(mode, src, x, n_tok, K, m.Kp, g, be, m, tc, s->back, s->stats,
                                                       s->xo, st, &pa))
                        return rc;
                    launches += src.kind == SRC_STATS ? 2 : 1;  // (rowstats +) gemv
                    const int ev = prof_begin(s, st);
                    const double bytes = (double)m.M * m.K + 4.0 * m.K + 4.0 * m.M + 4.0 * m.n_outl * m.M;
                    int rc = launch_gemv_fused(m, a, e, pa, mi == 0 ? s->tokmax_ctx : nullptr,
                                               mi == 0 ? s->tokmax_act : nullptr, s->partials, s->counters,
                                               s->partial_cap, st, s->sk_acc, s->sk_acc_elems);
                    prof_end(s, ev, 0, bytes, st);
                    return rc;
                }
                int ev = prof_begin(s, st);
                if (int rc = launch_prologue(mode, src, x, n_tok, K, m.Kp, g, be, m, tc, s->frag, s->back, s->stats,
                                             s->xo, nullptr, st))
                    return rc;
                prof_end(s, ev, 2, 4.0 * n_tok * K, st);
                launches += src.kind == SRC_STATS ? 3 : 2;  // (rowstats +) fragwrite + gemv
                ev = prof_begin(s, st);
                // algorithmic bytes: codes + per-feature scales + bias (+ f32 outlier rows)
                const double bytes = (double)m.M * m.K + 4.0 * m.K + 4.0 * m.M + 4.0 * m.n_outl * m.M;
                int rc = launch_gemv(m, a, e, s->partials, s->counters, s->partial_cap, st, s->sk_acc, s->sk_acc_elems);
                prof_end(s, ev, 0, bytes, st);
                return rc;
            }
            e.pstats = nullptr;
            e.tokmax = nullptr;
            if (int rc = launch_prologue(mode, ProSrc{}, x, n_tok, K, K, g, be, m, tc, nullptr, s->back, s->stats,
                                         nullptr, s->y32, st))
                return rc;
            launches += (mode == PRO_LN ? 2 : 0) + 2 * (int)ceil_div(n_tok, 8);  // (rowstats + rows) + gemv/reduce passes
            const int ev = prof_begin(s, st);
            int rc = launch_gemm_f32(m, s->y32, n_tok, e, s->partials, s->partial_cap, st);
            prof_end(s, ev, 3, 4.0 * m.M * m.K, st);
            return rc;
        };
        // ---- LN1 -> QKV (+ paged KV append)
        ProSrc src1;
        if (j > 0) {
            src1.kind = SRC_PARTIALS;
            src1.pstats = s->pst_x;
            src1.MG = MGd;
            src1.M = d;
            src1.gs = b.gs1;
            src1.bs = b.bs1;
        }
        src1.zero_tokmax = s->tokmax_ctx;
        Epi e = base;
        e.kind = EPI_QKV;
        e.out = s->q;
        if (int rc = matmul(0, PRO_LN, src1, x_in, d, b.ln1_g, b.ln1_b, e)) return rc;
        // ---- attention (+ operand range of wo)
        AttnArgs aa{s->q, kvb, s->d_tok_seq, s->d_tok_pos, s->d_pages, s->slopes, s->ctx, s->attn_part,
                    s->counters + (1 << 19), int8 ? s->tokmax_ctx : nullptr, int8 ? b.mat[1].scales : nullptr,
                    n_tok, s->max_pages, s->H, s->dh, s->cfg.page_tokens, d, max_pos, s->last_n_seq == n_tok ? 1 : 0,
                    s->d_grp_first, s->d_grp_count, s->n_groups, s->d_unit_base, s->total_units, s->max_stages,
                    s->max_group};
        {
            const int ev = prof_begin(s, st);
            if (int rc = launch_attention(aa, s->attn_cap, st)) return rc;
            // fp16 K and V rows read for every query token (2 T h 2 B per session-block)
            double kv_bytes = 0.0;
            for (int i = 0; i < n_tok; ++i) kv_bytes += 4.0 * (s->h_tok_pos_last[i] + 1) * d;
            prof_end(s, ev, 1, kv_bytes, st);
        }
        launches += 1;
        // ---- wo + residual (+ LN2 summaries)
        ProSrc src2;
        src2.kind = SRC_TOKMAX;
        src2.tokmax = s->tokmax_ctx;
        e = base;
        e.kind = EPI_RESID;
        e.resid = x_in;
        e.out = s->mid;
        e.pstats = s->pst_mid;
        if (int rc = matmul(1, PRO_SCALE, src2, s->ctx, d, nullptr, nullptr, e)) return rc;
        // ---- LN2 -> wmlp_in + GELU (+ operand range of wmlp_out)
        ProSrc src3;
        src3.kind = SRC_PARTIALS;
        src3.pstats = s->pst_mid;
        src3.MG = MGd;
        src3.M = d;
        src3.gs = b.gs2;
        src3.bs = b.bs2;
        src3.zero_tokmax = s->tokmax_act;
        e = base;
        e.kind = EPI_GELU;
        e.out = s->act;
        e.tokmax = s->tokmax_act;
        e.s_next = b.mat[3].scales;
        if (int rc = matmul(2, PRO_LN, src3, s->mid, d, b.ln2_g, b.ln2_b, e)) return rc;
        // ---- wmlp_out + residual (+ LN1 summaries of the next block)
        ProSrc src4;
        src4.kind = SRC_TOKMAX;
        src4.tokmax = s->tokmax_act;
        e = base;
        e.kind = EPI_RESID;
        e.resid = s->mid;
        e.out = x_out;
        e.pstats = (j + 1 < s->cfg.n_blocks) ? s->pst_x : nullptr;
        if (int rc = matmul(3, PRO_SCALE, src4, s->act, rd, nullptr, nullptr, e)) return rc;
    }
    s->last_launches = launches;
    return PB_OK;
}

static int stage_meta(pb_span* s, int n_tok, int n_seq, const int32_t* tok_seq, const int32_t* tok_pos,
                      const int32_t* pages, int* max_pos, cudaStream_t st) {
    PB_REQUIRE(n_tok > 0 && n_tok <= s->cfg.max_tokens, PB_ERR_CAPACITY, "too many tokens for this span's workspace");
    PB_REQUIRE(n_seq > 0 && n_seq <= s->cfg.max_seqs, PB_ERR_CAPACITY, "too many sequences in one step");
    int mp = 0;
    for (int i = 0; i < n_tok; ++i) {
        PB_REQUIRE(tok_seq[i] >= 0 && tok_seq[i] < n_seq, PB_ERR_BAD_REQUEST, "token sequence index out of range");
        PB_REQUIRE(tok_pos[i] >= 0 && tok_pos[i] < s->cfg.max_seq, PB_ERR_CAPACITY, "position exceeds max_seq");
        mp = std::max(mp, tok_pos[i] + 1);
        const int32_t pg = pages[(int64_t)tok_seq[i] * s->max_pages + tok_pos[i] / s->cfg.page_tokens];
        PB_REQUIRE(pg >= 0 && pg < s->cfg.n_pages, PB_ERR_BAD_REQUEST, "KV page out of range");
    }
    *max_pos = mp;
    s->h_tok_pos_last.assign(tok_pos, tok_pos + n_tok);
    s->last_n_seq = n_seq;
    // pinned staging ring: wait only until this slot's previous copies have executed
    const int slot = s->meta_slot;
    s->meta_slot = (slot + 1) % pb_span::NSLOT;
    PB_CHECK_CUDA(cudaEventSynchronize(s->meta_ev[slot]));
    int32_t* hm = s->h_meta[slot];
    std::memcpy(hm, tok_seq, sizeof(int32_t) * n_tok);
    std::memcpy(hm + n_tok, tok_pos, sizeof(int32_t) * n_tok);
    std::memcpy(hm + 2 * n_tok, pages, sizeof(int32_t) * (size_t)n_seq * s->max_pages);
    PB_CHECK_CUDA(cudaMemcpyAsync(s->d_tok_seq, hm, sizeof(int32_t) * n_tok, cudaMemcpyHostToDevice, st));
    PB_CHECK_CUDA(cudaMemcpyAsync(s->d_tok_pos, hm + n_tok, sizeof(int32_t) * n_tok, cudaMemcpyHostToDevice, st));
    PB_CHECK_CUDA(cudaMemcpyAsync(s->d_pages, hm + 2 * n_tok, sizeof(int32_t) * (size_t)n_seq * s->max_pages,
                                  cudaMemcpyHostToDevice, st));
    // attention query groups: up to 8 consecutive positions of one sequence
    int32_t* gf = hm + 2 * n_tok + (size_t)n_seq * s->max_pages;
    int32_t* gc = gf + n_tok;
    int ng = 0;
    for (int i = 0; i < n_tok; ++i) {
        if (ng > 0 && tok_seq[i] == tok_seq[i - 1] && tok_pos[i] == tok_pos[i - 1] + 1 && gc[ng - 1] < 32) {
            ++gc[ng - 1];
        } else {
            gf[ng] = i;
            gc[ng] = 1;
            ++ng;
        }
    }
    s->n_groups = ng;
    PB_CHECK_CUDA(cudaMemcpyAsync(s->d_grp_first, gf, sizeof(int32_t) * ng, cudaMemcpyHostToDevice, st));
    PB_CHECK_CUDA(cudaMemcpyAsync(s->d_grp_count, gc, sizeof(int32_t) * ng, cudaMemcpyHostToDevice, st));
    // stream-K units of the tensor-core attention: H x ceil(keys / 64) per group
    int64_t* ub = s->h_ub[slot];
    int64_t tot = 0;
    int mst = 0;
    for (int g = 0; g < ng; ++g) {
        ub[g] = tot;
        const int stages = (int)ceil_div(tok_pos[gf[g]] + gc[g], 64);
        mst = std::max(mst, stages);
        tot += (int64_t)s->H * stages;
    }
    ub[ng] = tot;
    s->total_units = tot;
    s->max_stages = mst;
    int mg_ = 0;
    for (int g = 0; g < ng; ++g) mg_ = std::max(mg_, (int)gc[g]);
    s->max_group = mg_;
    PB_CHECK_CUDA(cudaMemcpyAsync(s->d_unit_base, ub, sizeof(int64_t) * (ng + 1), cudaMemcpyHostToDevice, st));
    PB_CHECK_CUDA(cudaEventRecord(s->meta_ev[slot], st));
    return PB_OK;
}

// Decode steps as CUDA graphs (pb_span_config.graphs): at small shapes a step is
// bound by the host issuing ~5 launches per block (560M: 121 launches, 970 us of
// host time for 1070 us per step), not by the GPU. The launch sequence of
// run_blocks depends only on the shape key below; the per-step metadata
// (positions, pages, attention work units) reaches the device through the
// usual staged copies into fixed buffers, and the hidden states through g_in /
// g_out, so one captured graph per key replays every step of that shape (a
// batch-1 session re-captures when its attention stage count grows, every 64
// tokens).
static int run_blocks_graph(pb_span* s, int n_tok, int max_pos, const float* d_in, float* d_out, cudaStream_t st) {
    const pb_span::GraphKey key{n_tok, s->last_n_seq, s->n_groups, s->total_units, s->max_stages, s->max_group,
                                s->last_n_seq == n_tok ? 1 : 0};
    auto it = s->graphs.find(key);
    if (it == s->graphs.end()) {
        if (s->graphs.size() >= 64) {  // bounded cache
            for (auto& kv : s->graphs) cudaGraphExecDestroy(kv.second.exec);
            s->graphs.clear();
        }
        // capture on a private stream (the legacy default stream cannot be captured), after
        // the metadata copies of this step so the capture's dependencies start clean
        cudaEvent_t ev;
        PB_CHECK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        PB_CHECK_CUDA(cudaEventRecord(ev, st));
        PB_CHECK_CUDA(cudaStreamWaitEvent(s->cap_stream, ev, 0));
        PB_CHECK_CUDA(cudaStreamBeginCapture(s->cap_stream, cudaStreamCaptureModeThreadLocal));
        const int rc = run_blocks(s, n_tok, max_pos, s->g_in, s->g_out, s->cap_stream);
        cudaGraph_t g = nullptr;
        const cudaError_t ec = cudaStreamEndCapture(s->cap_stream, &g);
        cudaEventDestroy(ev);
        pb_span::GraphEntry e;
        cudaError_t ei = cudaErrorStreamCaptureInvalidated;
        if (!rc && ec == cudaSuccess && g) ei = cudaGraphInstantiate(&e.exec, g, 0);
        if (g) cudaGraphDestroy(g);
        if (ei != cudaSuccess) {
            // nothing of the capture ran: a capture the driver invalidated (seen intermittently with
            // concurrent server threads, e.g. a kernel's first, lazily loaded use inside the capture)
            // runs this step eagerly instead; a real error repeats there and is reported from it
            (void)cudaGetLastError();
            return run_blocks(s, n_tok, max_pos, d_in, d_out, st);
        }
        e.launches = s->last_launches;
        it = s->graphs.emplace(key, e).first;
    }
    const size_t bytes = sizeof(float) * (size_t)n_tok * s->d;
    if (d_in != s->g_in) PB_CHECK_CUDA(cudaMemcpyAsync(s->g_in, d_in, bytes, cudaMemcpyDeviceToDevice, st));
    PB_CHECK_CUDA(cudaGraphLaunch(it->second.exec, st));
    if (d_out != s->g_out) PB_CHECK_CUDA(cudaMemcpyAsync(d_out, s->g_out, bytes, cudaMemcpyDeviceToDevice, st));
    s->last_launches = it->second.launches;
    return PB_OK;
}

extern "C" int pb_span_step(pb_span* span, int32_t n_tok, int32_t n_seq, const int32_t* h_tok_seq,
                            const int32_t* h_tok_pos, const int32_t* h_pages, const float* d_in, float* d_out,
                            void* stream) {
    PB_REQUIRE(span, PB_ERR_BAD_REQUEST, "null span");
    std::lock_guard<std::mutex> lk(span->mu);
    PB_CHECK_CUDA(cudaSetDevice(span->cfg.device));
    auto st = (cudaStream_t)stream;
    int max_pos = 0;
    if (int rc = stage_meta(span, n_tok, n_seq, h_tok_seq, h_tok_pos, h_pages, &max_pos, st)) return rc;
    if (span->cfg.graphs && n_tok <= GRAPH_MAX_TOKENS && !span->prof_on && !trace_active())
        return run_blocks_graph(span, n_tok, max_pos, d_in, d_out, st);
    return run_blocks(span, n_tok, max_pos, d_in, d_out, st);
}

extern "C" int pb_span_step_tape(pb_span* span, int32_t n_tok, int32_t n_seq, const int32_t* h_tok_seq,
                                 const int32_t* h_tok_pos, const int32_t* h_pages, const float* d_in, float* d_out,
                                 float* d_tape, void* stream) {
    PB_REQUIRE(span && d_tape, PB_ERR_BAD_REQUEST, "null argument");
    std::lock_guard<std::mutex> lk(span->mu);
    PB_CHECK_CUDA(cudaSetDevice(span->cfg.device));
    auto st = (cudaStream_t)stream;
    int max_pos = 0;
    if (int rc = stage_meta(span, n_tok, n_seq, h_tok_seq, h_tok_pos, h_pages, &max_pos, st)) return rc;
    return run_blocks(span, n_tok, max_pos, d_in, d_out, st, d_tape);
}

extern "C" int pb_span_step_int8(pb_span* span, int32_t n_tok, int32_t n_seq, const int32_t* h_tok_seq,
                                 const int32_t* h_tok_pos, const int32_t* h_pages, const int8_t* d_in_codes,
                                 const float* d_in_scales, const float* d_in_f32, int8_t* d_out_codes,
                                 float* d_out_scales, float* d_out_f32, float* d_tape, void* stream) {
    PB_REQUIRE(span, PB_ERR_BAD_REQUEST, "null span");
    PB_REQUIRE(d_in_codes || d_in_f32, PB_ERR_BAD_REQUEST, "no input");
    PB_REQUIRE(d_out_codes || d_out_f32, PB_ERR_BAD_REQUEST, "no output");
    std::lock_guard<std::mutex> lk(span->mu);
    PB_CHECK_CUDA(cudaSetDevice(span->cfg.device));
    auto st = (cudaStream_t)stream;
    int max_pos = 0;
    if (int rc = stage_meta(span, n_tok, n_seq, h_tok_seq, h_tok_pos, h_pages, &max_pos, st)) return rc;
    const int64_t n = (int64_t)n_tok * span->d;
    int extra = 0;
    const float* in = d_in_f32;
    if (d_in_codes) {
        // xa is the inter-block buffer: block 0 reads its input for the last
        // time (wo residual) before its final GEMV overwrites xa.
        const int ev = prof_begin(span, st);
        if (int rc = dequantize_blockwise(d_in_codes, d_in_scales, n, 64, span->xa, st)) return rc;
        prof_end(span, ev, 4, 5.0 * n + n / 16.0, st);
        in = span->xa;
        ++extra;
    }
    float* out = d_out_f32 ? d_out_f32 : span->xa;
    // the span-to-span hop path (box front end, pipelined bench) replays decode steps as graphs too
    const bool graph = !d_tape && span->cfg.graphs && n_tok <= GRAPH_MAX_TOKENS && !span->prof_on && !trace_active();
    if (int rc = graph ? run_blocks_graph(span, n_tok, max_pos, in, out, st)
                       : run_blocks(span, n_tok, max_pos, in, out, st, d_tape))
        return rc;
    if (d_out_codes) {
        const int ev = prof_begin(span, st);
        if (int rc = quantize_blockwise(out, n, 64, d_out_codes, d_out_scales, st)) return rc;
        prof_end(span, ev, 4, 5.0 * n + n / 16.0, st);
        ++extra;
    }
    span->last_launches += extra;
    return PB_OK;
}

extern "C" int pb_span_profile(pb_span* span, int32_t on) {
    PB_REQUIRE(span, PB_ERR_BAD_REQUEST, "null span");
    std::lock_guard<std::mutex> lk(span->mu);
    span->prof_on = on != 0;
    span->prof.clear();
    return PB_OK;
}

extern "C" int pb_span_profile_read(pb_span* span, int32_t kind, double* ms, int64_t* launches, double* bytes) {
    PB_REQUIRE(span && ms && launches && bytes, PB_ERR_BAD_REQUEST, "null argument");
    std::lock_guard<std::mutex> lk(span->mu);
    PB_CHECK_CUDA(cudaSetDevice(span->cfg.device));
    double t = 0.0, b = 0.0;
    int64_t n = 0;
    for (const auto& r : span->prof) {
        if (r.kind != kind) continue;
        float e = 0.f;
        PB_CHECK_CUDA(cudaEventSynchronize(span->prof_ev[r.ev + 1]));
        PB_CHECK_CUDA(cudaEventElapsedTime(&e, span->prof_ev[r.ev], span->prof_ev[r.ev + 1]));
        t += e;
        b += r.bytes;
        ++n;
    }
    *ms = t;
    *launches = n;
    *bytes = b;
    return PB_OK;
}
