// Internal structures of a block span (not part of the C-ABI).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace pb {

// One weight matrix of a block, reference shape W = [K = in, M = out].
struct Mat {
    int M = 0, K = 0, Mp = 0, Kp = 0;  // padded: Mp % 128 == 0, Kp % 32 == 0
    bool int8 = true;
    int8_t* codes = nullptr;   // [Mp/128][Kp/32] 4 KB canonical K-major tiles (pb_weights.cu; int8 mode)
    int8_t* tcodes = nullptr;  // BACKWARD: the same codes as tiles of W^T, cached when HBM allows (pb_train.cu)
    float* scales = nullptr;   // [Kp] per input feature, 0 on outliers / padding
    float* w32 = nullptr;      // [K][M] reference layout (f32 mode)
    int n_outl = 0;
    int32_t* outl_idx = nullptr;   // [n_outl] input features kept in f32
    float* outl_rows = nullptr;    // [n_outl][M] = W[idx_j, :]
    std::vector<int32_t> h_outl_idx;

    void free_outliers() {
        if (outl_idx) cudaFree(outl_idx);
        if (outl_rows) cudaFree(outl_rows);
        outl_idx = nullptr;
        outl_rows = nullptr;
        n_outl = 0;
        h_outl_idx.clear();
    }
    int64_t bytes() const {
        int64_t b = (int64_t)Kp * 4;
        if (int8) b += (int64_t)Mp * Kp;
        else b += (int64_t)K * M * 4;
        return b + (int64_t)n_outl * (M * 4 + 4);
    }
};

struct BlockW {
    Mat mat[4];  // 0 wqkv [d,3d], 1 wo [d,d], 2 wmlp_in [d,rd], 3 wmlp_out [rd,d]
    float* ln1_g = nullptr;
    float* ln1_b = nullptr;
    float* ln2_g = nullptr;
    float* ln2_b = nullptr;
    float* bias[4] = {nullptr, nullptr, nullptr, nullptr};
    // LN -> int8 operand range bounds (see ProSrc): max_k |gamma_k| s_k, max_k |beta_k| s_k
    float gs1 = 0.f, bs1 = 0.f, gs2 = 0.f, bs2 = 0.f;
};

// EPI_BWD (tcgen05 only): BACKWARD through an int8 matrix (pb_train.cu), out = acc * rowscale[o], no bias
enum EpiKind { EPI_QKV = 0, EPI_RESID = 1, EPI_GELU = 2, EPI_PLAIN = 3, EPI_BWD = 4 };

// Epilogue parameters shared by every GEMV/GEMM flavour.
struct Epi {
    int kind;
    int M;                   // output features
    const float* bias;       // [M]
    int n_outl;
    const int32_t* outl_idx;
    const float* outl_rows;  // [n_outl][M]
    const float* xo;         // [n_tok][n_outl] unscaled activations at outlier features
    const float* resid;      // EPI_RESID: [n_tok][M]
    float* out;              // EPI_RESID/EPI_GELU: [n_tok][M]; EPI_QKV: q [n_tok][d]
    // EPI_QKV: append k, v to the paged cache
    half* kv;                // this block's pool base: [n_pages][2][H][P][dh]
    const int32_t* tok_seq;
    const int32_t* tok_pos;
    const int32_t* pages;    // [n_seq][max_pages]
    int max_pages, H, dh, P, d;
    // row statistics for the NEXT matmul's operand, produced here (fused prologue):
    float4* pstats;          // EPI_RESID -> LN consumer: [n_tok][M/128] {mean, M2, min, max} per 128-row group
    float* tokmax;           // EPI_GELU -> scale consumer: atomicMax of |out * s_next| per token
    const float* s_next;     // [M] scales of the consuming matrix
    const float* rowscale;   // EPI_BWD: [M] per-row factor (the forward matrix's input-feature scales)
};

// B-operand (activation) layout parameters for one GEMV launch.
struct Act {
    const uint4* frag;      // int8-digit B fragments (m16n8k32), see pb_gemv.cu
    const float* back;      // [n_tok] 2^-shift per token
    int n_tok;
    int tc;                 // tokens per column chunk (4, 8, 16, 32)
};

// prologue modes
enum ProMode { PRO_LN = 0, PRO_SCALE = 1 };

// Where the operand producer (k_fragwrite) gets its per-token statistics.
enum ProSrcKind { SRC_STATS = 0, SRC_PARTIALS = 1, SRC_TOKMAX = 2 };
struct ProSrc {
    int kind = SRC_STATS;        // SRC_STATS: run k_rowstats first (span input, f32 mode)
    const float4* pstats = nullptr;  // SRC_PARTIALS: producer's per-128-row {mean, M2, min, max}
    int MG = 0, M = 0;           //   groups and rows of that producer
    float gs = 0.f, bs = 0.f;    //   shift bound: max|y s| <= gs * max|x - mu| * inv + bs
    const float* tokmax = nullptr;   // SRC_TOKMAX: exact max |x s| per token (atomicMax'ed)
    float* zero_tokmax = nullptr;    // reset for the next producer's atomicMax (may be null)
};

int fill_matrix_gen(Mat& m, uint64_t key, float threshold, float boost, int every, cudaStream_t st);
int fill_matrix_f32(Mat& m, const float* w, float threshold, cudaStream_t st);
// same from the transposed matrix wt = W^T [M][K] row-major (the tied LM head's embedding table)
int fill_matrix_f32_t(Mat& m, const float* wt, float threshold, cudaStream_t st);
int untile_codes(const Mat& m, int8_t* d_out, cudaStream_t st);

int quantize_blockwise(const float* x, int64_t n, int block, int8_t* codes, float* scales, cudaStream_t st);
int dequantize_blockwise(const int8_t* codes, const float* scales, int64_t n, int block, float* out,
                         cudaStream_t st);

// tokens per step from which the matmuls run on tcgen05 (9..32: the stream-K kernel, more: the
// prefill GEMM). Measured (tools/batch_probe.py): 176B 12 sessions 644 -> 500 us per block, 7B1 16
// sessions 188 -> 165, 32 sessions 295 -> 200; at 8 tokens the IMMA GEMV still wins (459 vs 487, 113
// vs 140)
constexpr int TC_MIN_TOKENS_DEFAULT = 9;
constexpr int TC_TOKENS = 80;  // tokens per tcgen05 tile (3 digit accumulators x 80 columns, double-buffered in TMEM)
// prologue: y = LN(x) (PRO_LN) or x (PRO_SCALE); writes the int8-digit operand of
// y * scales, the per-token 2^-shift, outlier activations xo, and (f32 mode) y.
int launch_prologue(int mode, const ProSrc& src, const float* x, int n_tok, int K, int Kp, const float* gamma,
                    const float* beta, const Mat& m, int tc, uint4* frag, float* back, float4* stats, float* xo,
                    float* y32, cudaStream_t st, uint8_t* bcanon = nullptr, int bcanon_tile = TC_TOKENS);
// tcgen05 GEMM over a canonical-layout B operand (pb_gemm_tc.cu)
int launch_gemm_tc(const Mat& m, const uint8_t* bcanon, const Act& act, const Epi& epi, cudaStream_t st);
// batched decode (n_tok <= tile_tokens in {16, 32}): stream-K tcgen05 GEMM over a canonical B operand
// written with tile width tile_tokens; partials / counters are the span's split-merge workspaces
int launch_gemm_tc_sk(const Mat& m, const uint8_t* bcanon, int tile_tokens, const Act& act, const Epi& epi,
                      int* skacc, int64_t skacc_bytes, int* counters, cudaStream_t st);
// (max_k |gamma_k| s_k, max_k |beta_k| s_k) -> host
int bound_consts(const float* gamma, const float* beta, const float* scales, int K, float* gs, float* bs,
                 cudaStream_t st);
// Operand-writer arguments (k_fragwrite / k_canonwrite).
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
    float4* stats; // [n_tok] {mu, inv, 2^shift, 2^-shift}
    float* xo;
    float* y32;
    ProSrc src;
    int early;
    uint64_t* trace = nullptr;  // diagnostics (pb_trace_set)
};

// sums (optional): a zeroed s32 workspace [chunks][MG][128 x 8 NT] for the split-row-group merge
int launch_gemv(const Mat& m, const Act& act, const Epi& epi, float* partials, int* counters,
                int64_t partial_cap, cudaStream_t st, int* sums = nullptr, int64_t sums_elems = 0);
// decode (<= 2 tokens per column chunk): the operand is built inside the GEMV
// by an operand warp (no k_fragwrite launch); prepare_fused_operand runs the
// block-0 row statistics if needed and returns the operand description
bool gemv_fusable(const Act& act, int K);
int prepare_fused_operand(int mode, const ProSrc& src, const float* x, int n_tok, int K, int Kp, const float* gamma,
                          const float* beta, const Mat& m, int tc, float* back, float4* stats, float* xo,
                          cudaStream_t st, ProArgs* out);
int launch_gemv_fused(const Mat& m, const Act& act, const Epi& epi, const ProArgs& pro, float* zero_a,
                      float* zero_b, float* partials, int* counters, int64_t partial_cap, cudaStream_t st,
                      int* sums = nullptr, int64_t sums_elems = 0);
int launch_gemm_f32(const Mat& m, const float* y, int n_tok, const Epi& epi, float* part, int64_t part_cap,
                    cudaStream_t st);
int choose_tc(int n_tok);

// attention over the paged cache
struct AttnArgs {
    const float* q;          // [n_tok][d]
    const half* kv;          // block pool base
    const int32_t* tok_seq;
    const int32_t* tok_pos;
    const int32_t* pages;
    const float* slopes;     // [H]
    float* ctx;              // [n_tok][d]
    float* part;             // split workspace
    int* counters;           // [n_tok][H] last-CTA merge counters (zeroed, self-resetting)
    float* tokmax;           // [n_tok] atomicMax of |ctx * s_next| (wo operand range), may be null
    const float* s_next;     // [d] scales of wo
    int n_tok, max_pages, H, dh, P, d;
    int max_pos;             // max over tokens of (pos + 1)
    int decode_only;         // every sequence adds one position (older keys are safe to prefetch early)
    const int32_t* grp_first;  // query groups: up to 32 consecutive positions of one sequence
    const int32_t* grp_count;
    int n_groups;
    // stream-K units of the tensor-core kernel: (group, head, 64-key stage)
    const int64_t* unit_base;  // [n_groups + 1] first unit of each group
    int64_t total_units;
    int max_stages;            // max over groups of ceil(keys / 64)
    int max_group;             // largest query group (> 8: the prefill kernel, queries split across warps)
    uint64_t* trace = nullptr; // diagnostics (pb_trace_set)
};
int launch_attention(const AttnArgs& a, int64_t part_cap, cudaStream_t st);



template <int DH>
int run_attn_mma(const AttnArgs& a, int n_groups, int64_t cap, cudaStream_t st);
// the tensor-core attention (head_dim 64/128) reads KV rows whose 16-byte
// chunks are XOR-swizzled by (slot & 7); the QKV epilogue writes them so
__host__ __device__ inline bool kv_swizzled(int dh) { return dh == 64 || dh == 128; }
int64_t attention_part_floats(int n_tok, int H, int dh, int max_seq);

}  // namespace pb
