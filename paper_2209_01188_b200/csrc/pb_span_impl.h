// Private definition of the span object shared by the C-ABI translation units
// (pb_span.cu: weights, KV pool, decode/prefill steps; pb_train.cu: FORWARD
// tape + BACKWARD). Not part of the C-ABI.
#pragma once

#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "pb_common.cuh"
#include "pb_span.h"

using pb::BlockW;

struct pb_span {
    pb_span_config cfg{};
    int d = 0, H = 0, dh = 0, rd = 0, max_pages = 0;
    std::vector<BlockW> blocks;
    half* kv = nullptr;          // [n_blocks][n_pages][2][H][P][dh]
    int64_t kv_block_elems = 0;  // elements per block
    float* slopes = nullptr;
    // workspaces
    float *xa = nullptr, *mid = nullptr, *q = nullptr, *ctx = nullptr, *act = nullptr, *xo = nullptr, *y32 = nullptr;
    uint4* frag = nullptr;
    uint8_t* bcanon = nullptr;  // tcgen05 B operand [ceil(NT/TC_TOKENS)][KC][3 digit planes][TC_TOKENS x 32 B]
    int tc_min = pb::TC_MIN_TOKENS_DEFAULT;
    float* back = nullptr;
    float4* stats = nullptr;
    float4 *pst_x = nullptr, *pst_mid = nullptr;  // per-128-row LN summaries [NT][d/128]
    float *tokmax_ctx = nullptr, *tokmax_act = nullptr;  // operand ranges [NT]
    float* partials = nullptr;
    int* sk_acc = nullptr;        // [MG][3 * 32][128] s32 split-row-group sums of k_gemm_tc_sk (kept zero)
    int64_t sk_acc_elems = 0;
    int64_t partial_cap = 0;
    int* counters = nullptr;
    float* attn_part = nullptr;
    int64_t attn_cap = 0;
    int32_t *d_tok_seq = nullptr, *d_tok_pos = nullptr, *d_pages = nullptr;
    int32_t *d_grp_first = nullptr, *d_grp_count = nullptr;
    int n_groups = 0;
    int64_t* d_unit_base = nullptr;  // stream-K attention units per query group
    int64_t total_units = 0;
    int max_stages = 0;
    int max_group = 0;
    static constexpr int NSLOT = 4;  // ring of pinned staging buffers (no host sync per step)
    int32_t* h_meta[NSLOT] = {nullptr, nullptr, nullptr, nullptr};
    int64_t* h_ub[NSLOT] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t meta_ev[NSLOT] = {nullptr, nullptr, nullptr, nullptr};
    int meta_slot = 0;
    int64_t meta_ints = 0;
    // live kernel profiling (CUDA event pairs around launches; bench.py roofline)
    bool prof_on = false;
    std::vector<cudaEvent_t> prof_ev;
    struct ProfRec { int kind; int ev; double bytes; };
    std::vector<ProfRec> prof;
    std::vector<int32_t> h_tok_pos_last;
    int8_t* hop_codes = nullptr;
    float* hop_scales = nullptr;
    int64_t bytes = 0;
    int32_t last_launches = 0;
    int last_n_seq = 0;
    // CUDA-graph replay of decode steps: the launch sequence of run_blocks depends only on
    // this key (n_tok, n_seq, n_groups, total_units, max_stages, max_group, decode-only); inputs
    // and outputs go through the fixed buffers g_in / g_out, metadata through d_tok_* as usual
    using GraphKey = std::tuple<int, int, int, int64_t, int, int, int>;
    struct GraphEntry { cudaGraphExec_t exec = nullptr; int32_t launches = 0; };
    std::map<GraphKey, GraphEntry> graphs;
    cudaStream_t cap_stream = nullptr;
    float *g_in = nullptr, *g_out = nullptr;  // [64][d]
    // BACKWARD workspace (pb_train.cu): one grow-only arena, kept across calls
    uint8_t* train_ws = nullptr;
    int64_t train_ws_bytes = 0;
    std::mutex mu;  // one step at a time per span (the stream is shared)
};

