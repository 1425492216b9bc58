/*
 * petals_b200.h — C-ABI of the B200-native block-span server hot path.
 *
 * Everything here takes plain pointers, sizes and a cudaStream_t (passed as
 * void*); no torch types cross this boundary. Device pointers are marked d_,
 * host pointers h_. Every entry point returns 0 on success or one of the
 * reference's wire error codes (PB_ERR_*, mirroring
 * /root/reference/pkg/src/swarmlm/errors.py:38-44); pb_last_error() returns a
 * thread-local message for the last failure.
 *
 * Reference interfaces replaced (file:line under /root/reference/pkg/src/swarmlm):
 *   pb_quantize_blockwise    <- quant.py:33-54   quantize_blockwise (wire codec, bit-exact)
 *   pb_dequantize_blockwise  <- quant.py:57-66   dequantize_blockwise (bit-exact)
 *   pb_gen_tensor            <- model.py:36-62   splitmix64_array/uniform_from_u64/tensor_stream
 *   pb_span_* weights        <- quant.py:81-108,132-149 quantize_weights_int8 / QuantizedBlockWeights.from_block
 *   pb_span_step             <- model.py:314-380 block_forward looped over a span as in server.py:383-385,
 *                               batched over sessions; KV caches = server.py:69-77 _Session.caches
 *   pb_span_step_tape,
 *   pb_span_backward         <- server.py:411-450 FORWARD tapes / BACKWARD, model.py:383-418 block_backward
 *   pb_head_*                <- model.py:421-446 embed / lm_head / sample_next("greedy"), the client side of
 *                               client.py:247-250
 */
#ifndef PETALS_B200_H
#define PETALS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* errors.py:38-44 */
#define PB_OK 0
#define PB_ERR_GENERIC 1
#define PB_ERR_BUSY 2
#define PB_ERR_DESYNC 3
#define PB_ERR_UNKNOWN_SESSION 4
#define PB_ERR_UNKNOWN_TAPE 5
#define PB_ERR_BAD_REQUEST 6
#define PB_ERR_CAPACITY 7

/* weight storage of a span */
#define PB_WEIGHTS_INT8 1 /* quantize in {weights, both}: LLM.int8-style codes + f32 outlier rows */
#define PB_WEIGHTS_F32 0  /* quantize in {none, activations}: f32 weights, reference fp32 math */

const char* pb_last_error(void);
int pb_version(void);

/* ---- wire codec (transport/wire.py:98-105,125-137 -> quant.py:33-66) ---- */
/* codes[n] int8, scales[ceil(n/block)] f32; bit-exact with the reference. */
int pb_quantize_blockwise(const float* d_x, int64_t n, int32_t block, int8_t* d_codes, float* d_scales,
                          void* stream);
int pb_dequantize_blockwise(const int8_t* d_codes, const float* d_scales, int64_t n, int32_t block,
                            float* d_out, void* stream);

/* ---- deterministic weights (model.py:36-62) ----
 * out[i] = f32(((splitmix64(key, first + i + 1) >> 11) * 2^-53 - 0.5) * 0.1),
 * key = seed ^ fnv1a64(path) (computed by the caller). */
int pb_gen_tensor(uint64_t key, int64_t first, int64_t n, float* d_out, void* stream);

/* ---- block span ---- */
typedef struct pb_span pb_span;

typedef struct {
    int32_t hidden;      /* d */
    int32_t n_heads;     /* H */
    int32_t mlp_ratio;   /* r (model.py:72) */
    int32_t max_seq;     /* model.py:71 */
    int32_t n_blocks;    /* blocks hosted by this span */
    int32_t first_block; /* global index of the first hosted block (weight stream paths) */
    int32_t weights;     /* PB_WEIGHTS_INT8 | PB_WEIGHTS_F32 */
    int32_t page_tokens; /* KV page size in tokens */
    int32_t n_pages;     /* KV pool pages (each page holds page_tokens positions for every hosted block) */
    int32_t max_tokens;  /* max new tokens per pb_span_step / rows*t per pb_span_forward chunk */
    int32_t max_seqs;    /* max sequences (sessions) per pb_span_step */
    float outlier_threshold; /* quant.py:14 (6.0) */
    int32_t device;
    int32_t tc_min_tokens; /* tokens per step from which the matmuls run on the tcgen05 kernels instead of
                              the IMMA GEMV; 0 = the measured default (9) */
    int32_t graphs;        /* 1: pb_span_step replays decode steps (<= 64 tokens) as CUDA graphs, one per
                              launch shape (tokens, sequences, attention work units), captured on first use */
    int32_t operand_kernel; /* 1: batch-1 decode builds its int8-digit operands in a separate kernel
                               (k_fragwrite) instead of the GEMV's own operand warps (the default, 0);
                               the results are bit-identical (tests/test_gpu_fused.py) */
} pb_span_config;

int pb_span_create(const pb_span_config* cfg, pb_span** out);
int pb_span_destroy(pb_span* span);
/* bytes of device memory held by the span (weights + KV pool + workspace) */
int64_t pb_span_device_bytes(const pb_span* span);

/* Fill hosted block j (0-based within the span) with gen_checkpoint weights
 * for global block first_block + j (model.py:176-209): matrices from the
 * SplitMix64 streams `blocks.{i}.{wqkv,wo,wmlp_in,wmlp_out}`, gammas 1,
 * betas/biases 0. key_* = seed ^ fnv1a64(path) computed by the caller.
 * outlier_boost (>1 enables) multiplies the rows of every `boost_every`-th
 * input feature by outlier_boost before quantization (bench outlier injection);
 * pass 0 to disable. */
int pb_span_gen_block(pb_span* span, int32_t j, uint64_t key_wqkv, uint64_t key_wo, uint64_t key_win,
                      uint64_t key_wout, float outlier_boost, int32_t boost_every, void* stream);

/* Load hosted block j from device f32 tensors in the reference layout
 * (model.py:87-100: matrices [in, out] row-major). */
int pb_span_load_block(pb_span* span, int32_t j, const float* d_ln1_g, const float* d_ln1_b,
                       const float* d_wqkv, const float* d_bqkv, const float* d_wo, const float* d_bo,
                       const float* d_ln2_g, const float* d_ln2_b, const float* d_win, const float* d_bin,
                       const float* d_wout, const float* d_bout, void* stream);

/* Outlier input features chosen by the quantizer for matrix m (0 wqkv, 1 wo,
 * 2 wmlp_in, 3 wmlp_out) of block j. Writes up to cap indices, returns count
 * in *n. Scales/codes can be read back with pb_span_read_codes. */
int pb_span_outliers(const pb_span* span, int32_t j, int32_t m, int32_t* h_idx, int32_t cap, int32_t* n);
/* Copy matrix m of block j back as reference-layout int8 codes [out, in] and
 * f32 scales [in] (test/inspection path). */
int pb_span_read_codes(const pb_span* span, int32_t j, int32_t m, int8_t* h_codes, float* h_scales);

/* One batched inference step through every hosted block.
 * n_tok new positions from n_seq sequences; token i belongs to sequence
 * h_tok_seq[i] at absolute position h_tok_pos[i] (positions of one sequence
 * are consecutive and its cache already holds [0, first position)).
 * h_pages[s * max_pages + p] is the KV pool page of sequence s's logical page
 * p (max_pages = ceil(max_seq / page_tokens)). Input/output hidden states
 * [n_tok, hidden] f32 on the device; d_in may equal d_out. */
int pb_span_step(pb_span* span, int32_t n_tok, int32_t n_seq, const int32_t* h_tok_seq,
                 const int32_t* h_tok_pos, const int32_t* h_pages, const float* d_in, float* d_out,
                 void* stream);

/* Same as pb_span_step but the hidden states arrive / leave as wire-codec
 * int8 (codes [n_tok*hidden], scales [n_tok*hidden/64]), block 64 -- the
 * span-to-span hop payload (client.py:312-331 relays exactly these bytes).
 * Either codec side may be NULL (f32 then); in/out pointers may live in a
 * peer GPU's mailbox (pb_hop_*). d_tape (nullable) records the FORWARD tape
 * as pb_span_step_tape does. */
int pb_span_step_int8(pb_span* span, int32_t n_tok, int32_t n_seq, const int32_t* h_tok_seq,
                      const int32_t* h_tok_pos, const int32_t* h_pages, const int8_t* d_in_codes,
                      const float* d_in_scales, const float* d_in_f32, int8_t* d_out_codes,
                      float* d_out_scales, float* d_out_f32, float* d_tape, void* stream);

/* pb_span_step that also records the FORWARD tape (server.py:418-428): block j's input rows are
 * copied to d_tape[j][n_tok][hidden] (hosted block order) for pb_span_backward. */
int pb_span_step_tape(pb_span* span, int32_t n_tok, int32_t n_seq, const int32_t* h_tok_seq,
                      const int32_t* h_tok_pos, const int32_t* h_pages, const float* d_in, float* d_out,
                      float* d_tape, void* stream);

/* BACKWARD of one FORWARD row (server.py:431-450 -> model.py:383-418 block_backward over the hosted
 * blocks in reverse): d_grad_in[t][hidden] = dL/d(span input) given d_grad_out[t][hidden], the row's
 * tape d_tape[n_blocks][t][hidden] (positions 0 .. t-1, empty cache). Intermediates are recomputed
 * from the tape with the span's own weights (int8 spans: the tcgen05 GEMM on the codes in both
 * directions, f32 outlier features; f32 spans: f32 matmuls). The first call of a row length grows a
 * span-owned workspace arena (kept until pb_span_destroy). */
int pb_span_backward(pb_span* span, const float* d_tape, int32_t t, const float* d_grad_out, float* d_grad_in,
                     void* stream);

/* Last-launch statistics: number of kernels the last step launched. */
int32_t pb_span_last_launches(const pb_span* span);

/* Live kernel profiling for the roofline: when on, every launch of the
 * following kinds is bracketed by CUDA events on the launching stream:
 * 0 int8 GEMV, 1 attention, 2 prologue, 3 f32 GEMM, 4 wire codec.
 * pb_span_profile(on) resets the records; pb_span_profile_read sums the
 * device time (ms), launch count and algorithmic bytes of one kind. */
int pb_span_profile(pb_span* span, int32_t on);
int pb_span_profile_read(pb_span* span, int32_t kind, double* ms, int64_t* launches, double* bytes);

/* ---- span-to-span hop over NVLink peer memory (replaces the client relay,
 * client.py:312-331, for spans on one box; pipeline.P2PRing) ----
 * pb_hop_alloc: zeroed device mailbox + its 64-byte CUDA IPC handle (h_handle).
 * pb_hop_open / pb_hop_close: map / unmap a peer process's mailbox.
 * pb_hop_signal: after the payload kernels on `stream`, publish seq to a (peer)
 * u64 flag with a system-scope release. pb_hop_wait: stream waits (one-thread
 * kernel, system-scope acquire) until *d_flag >= seq; after timeout_ms the
 * kernel traps (a missing signal fails loudly instead of hanging). */
int pb_hop_alloc(int64_t bytes, int32_t device, void** d_ptr, void* h_handle);
int pb_hop_free(void* d_ptr);
int pb_hop_open(const void* h_handle, int32_t device, void** d_ptr);
int pb_hop_close(void* d_ptr);
int pb_hop_wait(const uint64_t* d_flag, uint64_t seq, int64_t timeout_ms, void* stream);
int pb_hop_signal(uint64_t* d_peer_flag, uint64_t seq, void* stream);

/* Diagnostics (not a reference interface): per-CTA globaltimer stamps of the
 * decode kernels (int8 GEMV, attention, operand writer) into a device buffer
 * of cap_words u64 (NULL: off). Each traced launch takes 16 u64 per CTA
 * (entry, dependency released, first stage, end: globaltimer ns; SM id;
 * kernel-specific stamps);
 * pb_trace_meta writes {kind, ctas, word offset} triples for the launches
 * traced since pb_trace_set and returns their number. Process-wide, for
 * single-threaded probes only. */
int pb_trace_set(void* d_buf, int64_t cap_words);
int64_t pb_trace_meta(int64_t* h_out, int64_t cap_triples);

/* ---- client head: embedding, final LayerNorm + tied LM head, greedy ---- */
typedef struct pb_head pb_head;

/* vocab x hidden embedding (f32, kept for lookups and exact rescoring) plus an
 * int8 copy of its transpose for the approximate-logit pass; max_tokens <= 32
 * hidden rows per call. */
int pb_head_create(int32_t vocab, int32_t hidden, int32_t max_tokens, int32_t device, pb_head** out);
int pb_head_destroy(pb_head* head);
int64_t pb_head_device_bytes(const pb_head* head);
/* gen_checkpoint embed (model.py:190, stream key = seed ^ fnv1a64("embed")), final LN gamma 1 / beta 0 */
int pb_head_gen(pb_head* head, uint64_t key_embed, void* stream);
/* embed [vocab, hidden] f32, final_ln gamma/beta [hidden] f32 (device pointers) */
int pb_head_load(pb_head* head, const float* d_embed, const float* d_gamma, const float* d_beta, void* stream);
/* model.py:421-425: out[i] = embed[tokens[i]]; host token ids, range-checked (PB_ERR_BAD_REQUEST) */
int pb_head_embed(pb_head* head, const int32_t* h_tokens, int32_t n, float* d_out, void* stream);
/* same with device token ids (already validated, e.g. from pb_head_greedy) */
int pb_head_embed_device(pb_head* head, const int32_t* d_tokens, int32_t n, float* d_out, void* stream);
/* model.py:428-433: logits [n, vocab] f32 = LN_f(hidden) @ embed^T (f64 accumulation, rounded to f32) */
int pb_head_logits(pb_head* head, const float* d_hidden, int32_t n, float* d_logits, void* stream);
/* model.py:445-446 greedy sample_next of every row: argmax of the exact logits, lowest index on ties,
 * via int8 approximate logits + rigorous error bound + f64 rescoring of the candidates.
 * d_tokens[i] = -1 marks non-finite logits (model.py:442-443 InputError). If d_next_embed is not
 * NULL the chosen tokens' embedding rows are written there (the next step's input). */
int pb_head_greedy(pb_head* head, const float* d_hidden, int32_t n, int32_t* d_tokens, float* d_next_embed,
                   void* stream);

#ifdef __cplusplus
}
#endif
#endif
