// tcgen05 (5th-gen tensor core) int8 x int8 GEMM for prefill / parallel
// forward / large batched steps (model.py:341,362,366,368 via
// quant.py:117-129), fed by the TMA engine (cp.async.bulk), accumulating in
// TMEM.
//
// D_p[o, n] (s32, TMEM) = sum_k code[o, k] * digit_p(a[n, k]) for the three
// balanced int8 digits p of the 22-bit fixed-point activation (pb_gemv.cu).
// Tiles are 128 output rows x TC_TOKENS (80) tokens; the weight tile
// (canonical K-major int8, pb_weights.cu) and the digit planes (k_canonwrite)
// are UMMA operands as they land in shared memory: no conversion pass.
//
// Persistent grid, one CTA per SM (TMEM 512 columns). Tiles run in passes of
// ntg token tiles (tc_unit); within a pass tile = (row group, token tile) with
// the token tiles of one row group on neighbouring CTAs (CTA c takes tiles c,
// c + G, ...), so they share each weight k tile through L2, and the pass's
// digit planes stay L2-resident across row groups. ntg comes from an HBM
// traffic model in launch_gemm_tc (one pass for <= 13 token tiles). Two TMEM accumulator sets (3
// digits x 80 columns each) let the epilogue of tile i run while the tensor
// core accumulates tile i + 1.
//
// Warp roles (192 threads):
//   warp 0      TMA producer: per 32-wide k tile 4 KB of int8 codes + 3 x
//               2.5 KB digit planes -> smem ring, mbarrier complete_tx.
//   warp 1      TMEM owner + MMA issuer: one elected lane issues one
//               tcgen05.mma.cta_group::1.kind::i8 (M=128, N=240 = 3 digits x
//               80 tokens, K=32) per k tile, tcgen05.commit's the smem stage
//               back and, after the last k tile, the accumulator set.
//   warps 2-5   epilogue: tcgen05.ld of their TMEM lane quarter, exact digit
//               recombination 65536 h + 256 m + l, fused block epilogue, then
//               release the accumulator set.
// Canonical K-major (SWIZZLE_NONE) operand layout: 8-row x 16-byte core
// matrices, LBO = 128 B (k direction), SBO = 256 B (8-row groups).
//
// k_gemm_tc_sk<BN>: the same MMA for batched decode (BN = 16 or 32 tokens: one
// token tile, N = 3 BN = 48 / 96 digit columns instead of padding to 80
// tokens), memory-bound on the weight stream. Stream-K over (row group, k
// tile) units so all 148 SMs stream equal byte counts whatever the row-group
// count (wo / wmlp_out of 176B have 112 row groups); a row group split across
// CTAs leaves s32 digit partials, and the last contributor (per 32-row TMEM
// lane quarter, atomic counter) adds them -- exact integers, so the merge order
// does not matter -- and runs the fused epilogue.
#include <algorithm>
#include <cstdint>

#include "pb_async.cuh"
#include "pb_common.cuh"
#include "pb_epi.cuh"
#include "pb_span.h"

namespace pb {

constexpr int TC_BM = 128;
constexpr int TC_BN = TC_TOKENS;           // tokens per tile (per digit accumulator)
constexpr int TC_KT = 4;                   // k tiles per pipeline stage (MMAs issued per wait/commit)
constexpr int TC_STAGES = 4;
constexpr int TC_EPI_WARPS = 8;            // two per TMEM lane quarter, splitting the tile's 16-token chunks
constexpr int TC_THREADS = 64 + 32 * TC_EPI_WARPS;
constexpr int TC_A = 4096;                 // int8 codes per k tile (128 rows x 32)
constexpr int TC_PLANE = TC_BN * 32;       // one digit plane per k tile
constexpr int TC_B = 3 * TC_PLANE;
constexpr int TC_ACC = 256;                // TMEM columns per accumulator set (3 x 80 used)
constexpr int TC_TMEM_COLS = 512;
constexpr size_t TC_SMEM =
    (size_t)TC_STAGES * TC_KT * (TC_A + TC_B) + (2 * TC_STAGES + 4) * 8 + 16 + TC_BN * sizeof(TokInfo);

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
           (1ull << 46);  // version 1 (sm_100), base offset 0, SWIZZLE_NONE
}

// kind::i8: D s32 (c_format 2), A s8, B s8 (signed), both K-major, M = 128,
// N = 3 TC_BN: the three digit planes are stored back to back, so together they
// are one canonical N = 240 operand (80 is a multiple of the 8-row core group)
// and one MMA per k tile reads the weight tile from shared memory once.
constexpr uint32_t TC_IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)((3 * TC_BN) >> 3) << 17) |
                              ((uint32_t)(TC_BM >> 4) << 24);
static_assert(TC_IDESC == ((2u << 4) | (1u << 7) | (1u << 10) | (30u << 17) | (8u << 24)), "idesc");

constexpr uint32_t tc_idesc_i8(int n) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(TC_BM >> 4) << 24);
}

template <uint32_t IDESC>
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = (int)r[i];
}

struct TcArgs {
    const int8_t* codes;
    const uint8_t* bcanon;  // [token tiles][KC][3][TC_PLANE]
    int KC, MG, NTL;        // k tiles, row groups, token tiles
    int tiles;              // MG * NTL
    int ntg;                // token tiles per pass (NTL: one pass)
    Act act;
    Epi epi;
};

// Unit u -> (row group, token tile). Units run in passes over ntg token tiles:
// within a pass the token tiles of one row group are neighbours (they share
// the weight k tiles in L2), and the pass's digit planes (ntg x KC x 7.5 KB)
// stay L2-resident across the row groups instead of every wave of CTAs
// re-streaming all NTL token tiles' planes from HBM.
__device__ __forceinline__ void tc_unit(const TcArgs& a, int u, int mgs, int& mgu, int& nt) {
    const int per = mgs * a.ntg;
    const int g = u / per, r = u - g * per;
    const int n_here = min(a.ntg, a.NTL - g * a.ntg);
    mgu = r / n_here;
    nt = g * a.ntg + (r - mgu * n_here);
}

__global__ void __launch_bounds__(TC_THREADS, 1) k_gemm_tc(TcArgs a) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sa = smem;                                // [STAGES][KT][4 KB]
    uint8_t* sb = sa + TC_STAGES * TC_KT * TC_A;       // [STAGES][KT][3 planes]
    uint64_t* full = reinterpret_cast<uint64_t*>(sb + TC_STAGES * TC_KT * TC_B);
    uint64_t* empty = full + TC_STAGES;
    uint64_t* accfull = empty + TC_STAGES;  // [2]
    uint64_t* accempty = accfull + 2;       // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 2);
    TokInfo* s_tok = reinterpret_cast<TokInfo*>(tmem_slot + 4);  // [TC_BN] of the tile being finished

    const int warp = warp_uniform_id(), lane = threadIdx.x & 31;
    const int KC = a.KC;
    // tile schedule: unit u = cta, cta + NU, ...
    const int cta = (int)blockIdx.x, NU = (int)gridDim.x;
    const int units = a.tiles, mgs = a.MG;

    if (threadIdx.x == 0) {
        for (int s = 0; s < TC_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);  // MMA commit
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&accfull[b], 1);   // MMA commit after a tile's last k step
            mbar_init(&accempty[b], TC_EPI_WARPS);
        }
        mbar_fence_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TC_TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer
        if (lane == 0) {
            int it = 0;
            for (int u = cta; u < units; u += NU) {
                int mgu, nt;
                tc_unit(a, u, mgs, mgu, nt);
                const int mg = mgu;
                const int8_t* asrc = a.codes + (int64_t)mg * KC * TC_A;
                const uint8_t* bsrc = a.bcanon + (int64_t)nt * KC * TC_B;
                for (int kc = 0; kc < KC; kc += TC_KT, ++it) {
                    const int s = it % TC_STAGES, n = min(TC_KT, KC - kc);
                    mbar_wait(&empty[s], ((it / TC_STAGES) & 1) ^ 1);
                    mbar_expect_tx(&full[s], n * (TC_A + TC_B));
                    // consecutive k tiles are contiguous in both operands: one copy each
                    bulk_g2s(sa + s * TC_KT * TC_A, asrc + (int64_t)kc * TC_A, n * TC_A, &full[s]);
                    bulk_g2s(sb + s * TC_KT * TC_B, bsrc + (int64_t)kc * TC_B, n * TC_B, &full[s]);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer: tile i accumulates in set i & 1 (digit p at column 80 p)
        if (lane == 0) {
            int it = 0, i = 0;
            for (int u = cta; u < units; u += NU, ++i) {
                const int b = i & 1;
                mbar_wait(&accempty[b], ((i >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t acc = tmem + b * TC_ACC;
                for (int kc = 0; kc < KC; kc += TC_KT, ++it) {
                    const int s = it % TC_STAGES, n = min(TC_KT, KC - kc);
                    mbar_wait(&full[s], (it / TC_STAGES) & 1);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sa + s * TC_KT * TC_A), b0 = smem_u32(sb + s * TC_KT * TC_B);
                    for (int k = 0; k < n; ++k)
                        tc_mma<TC_IDESC>(acc, umma_desc(a0 + k * TC_A), umma_desc(b0 + k * TC_B), (kc | k) != 0);
                    tc_commit(&empty[s]);
                }
                tc_commit(&accfull[b]);
            }
        }
        __syncwarp();
    } else {
        // ---------------- epilogue (warps 2-9): TMEM lanes 32 (warp % 4) .. + 31; the two warps
        // of a lane quarter take alternate 16-token chunks
        const int quarter = warp & 3, half = (warp - 2) >> 2;
        const int row = quarter * 32 + lane;
        int i = 0;
        for (int u = cta; u < units; u += NU, ++i) {
            int mgu, nt;
            tc_unit(a, u, mgs, mgu, nt);
            const int mg = mgu;
            const int b = i & 1;
            // this tile's per-token constants (all epilogue warps done with the previous tile's)
            asm volatile("bar.sync 1, %0;" ::"r"(32 * TC_EPI_WARPS) : "memory");
            stage_tokens(a.epi, a.act.back, a.act.n_tok, nt * TC_BN, TC_BN, s_tok, (int)threadIdx.x - 64,
                         32 * TC_EPI_WARPS);
            asm volatile("bar.sync 1, %0;" ::"r"(32 * TC_EPI_WARPS) : "memory");
            mbar_wait(&accfull[b], (i >> 1) & 1);
            tc_fence_after();
            const int o = mg * TC_BM + row;
            const uint32_t tbase = tmem + b * TC_ACC + ((uint32_t)(quarter * 32) << 16);
            for (int c0 = half * 16; c0 < TC_BN; c0 += 32) {
                int h[16], m[16], l[16];
                tmem_ld16(tbase + c0, h);
                tmem_ld16(tbase + TC_BN + c0, m);
                tmem_ld16(tbase + 2 * TC_BN + c0, l);
                tc_epi16(a.epi, o, lane, nt * TC_BN + c0, s_tok + c0, h, m, l);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&accempty[b]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TC_TMEM_COLS));
    }
}

int launch_gemm_tc(const Mat& m, const uint8_t* bcanon, const Act& act, const Epi& epi, cudaStream_t st) {
    static int ok[PB_MAX_DEVICES] = {};
    if (per_device(ok, [](int) {
            return cudaFuncSetAttribute(k_gemm_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TC_SMEM) ==
                           cudaSuccess ? 1 : -1;
        }) < 0)
        return launch_check("gemm_tc setup");
    const int sms = sm_count();
    if (sms < 0) return PB_ERR_GENERIC;
    TcArgs a{m.codes, bcanon, m.Kp / 32, m.Mp / 128, (int)ceil_div(act.n_tok, TC_BN), 0, 0, act, epi};
    a.tiles = a.MG * a.NTL;
    // Token-tile passes chosen by an HBM-traffic model: a pass of ntg tiles reads every weight byte once
    // (its row group's token tiles run on neighbouring CTAs) and its digit planes once if they fit an L2
    // budget (64 MB), otherwise once per wave of CTAs. 176B, 2048 tokens, K = 14336: 3 passes of 9
    // tiles, DRAM 14.3 -> 3.4 GB per mlp_in launch, 4.83 -> 4.10 ms (profiles/r1_tcgen05_ntg_sweep.txt).
    {
        a.ntg = a.NTL;
        const int64_t a_all = (int64_t)a.MG * a.KC * TC_A, plane = (int64_t)a.KC * TC_B;
        const int64_t budget = 64ll << 20, slots = sms;
        int64_t best = INT64_MAX;
        for (int n = a.NTL; n >= 1; --n) {
            const int64_t passes = ceil_div(a.NTL, n), bp = n * plane;
            const int64_t waves = ceil_div((int64_t)a.MG * n, slots);
            const int64_t cost = passes * a_all + (bp <= budget ? (int64_t)a.NTL * plane : passes * waves * bp);
            if (cost < best) best = cost, a.ntg = n;
        }
    }
    const int grid = std::min(a.tiles, sms);  // persistent: one CTA per SM (TMEM 512 columns)
    k_gemm_tc<<<grid, TC_THREADS, TC_SMEM, st>>>(a);
    return launch_check("gemm_tc");
}


// ------------------------------------------------------------------ batched decode: stream-K, one token tile

template <int BN, int KT_ = 8, int ST_ = 4>
struct SkCfg {
    static constexpr int N = 3 * BN;                         // digit columns (MMA N)
    static constexpr int B_KT = N * 32;                      // digit-plane bytes per 32-wide k tile
    static constexpr int KT = KT_;                           // k tiles per stage
    static constexpr int STAGES = ST_;
    static constexpr int ACC = N <= 64 ? 64 : 128;           // TMEM columns per accumulator set
    static constexpr int NSETS = 2;  // accumulator sets (segments in flight); 4 measured equal
    static constexpr uint32_t IDESC = tc_idesc_i8(N);
    static constexpr size_t SMEM =
        (size_t)STAGES * KT * (TC_A + B_KT) + (2 * STAGES + 2 * NSETS) * 8 + 16 + BN * sizeof(TokInfo) +
        BN * sizeof(float);
};

struct TcSkArgs {
    const int8_t* codes;
    const uint8_t* bcanon;  // [KC][3][BN x 32 B] (k_canonwrite with tile width BN)
    int KC, MG;
    int64_t total;          // MG * KC units
    int G;                  // CTAs
    Act act;
    Epi epi;
    int* skacc;             // [MG][N][128 rows] s32 sums of split row groups, zero between launches
    int* counters;          // [MG][4 lane quarters][2 token halves], zero between launches
};

__device__ __forceinline__ int64_t sk_u0(int64_t c, int64_t total, int G) { return c * total / G; }
__device__ __forceinline__ int sk_owner_of(int64_t u, int64_t total, int G) { return (int)(((u + 1) * G - 1) / total); }

template <int BN, int KT_, int ST_>
__global__ void __launch_bounds__(TC_THREADS, 1) k_gemm_tc_sk(TcSkArgs a) {
    using C = SkCfg<BN, KT_, ST_>;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sa = smem;                                // [STAGES][KT][4 KB]
    uint8_t* sb = sa + C::STAGES * C::KT * TC_A;       // [STAGES][KT][N x 32 B]
    uint64_t* full = reinterpret_cast<uint64_t*>(sb + C::STAGES * C::KT * C::B_KT);
    uint64_t* empty = full + C::STAGES;
    uint64_t* accfull = empty + C::STAGES;  // [NSETS]
    uint64_t* accempty = accfull + C::NSETS;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + C::NSETS);
    TokInfo* s_tok = reinterpret_cast<TokInfo*>(tmem_slot + 4);  // 16-B aligned
    float* s_tmax = reinterpret_cast<float*>(s_tok + BN);          // EPI_GELU operand range, per CTA

    const int warp = warp_uniform_id(), lane = threadIdx.x & 31;
    const int KC = a.KC, c = (int)blockIdx.x;
    const int64_t u0 = sk_u0(c, a.total, a.G), u1 = sk_u0(c + 1, a.total, a.G);

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < C::NSETS; ++b) {
            mbar_init(&accfull[b], 1);
            mbar_init(&accempty[b], TC_EPI_WARPS);
        }
        mbar_fence_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(C::NSETS * C::ACC));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- producer: weights never depend on earlier kernels, so the first
        // STAGES stages of weights are requested before the PDL wait; their digit planes
        // (written by the operand kernel) follow once it has completed
        if (lane == 0) {
            const uint64_t pol = l2_evict_first();  // weights: read once per step
            int it = 0, pend_kc[C::STAGES], pend_n[C::STAGES];  // stages issued before the PDL wait
            bool waited = false;
            for (int64_t u = u0; u < u1;) {
                const int mg = (int)(u / KC), ka = (int)(u % KC);
                const int kb = u1 - u < (int64_t)(KC - ka) ? ka + (int)(u1 - u) : KC;
                const int8_t* asrc = a.codes + (int64_t)mg * KC * TC_A;
                for (int kc = ka; kc < kb; kc += C::KT, ++it) {
                    const int s = it % C::STAGES, n = min(C::KT, kb - kc);
                    mbar_wait(&empty[s], ((it / C::STAGES) & 1) ^ 1);
                    mbar_expect_tx(&full[s], n * (TC_A + C::B_KT));
                    bulk_g2s_hint(sa + s * C::KT * TC_A, asrc + (int64_t)kc * TC_A, n * TC_A, &full[s], pol);
                    if (waited) {
                        bulk_g2s(sb + s * C::KT * C::B_KT, a.bcanon + (int64_t)kc * C::B_KT, n * C::B_KT, &full[s]);
                    } else {
                        pend_kc[s] = kc;
                        pend_n[s] = n;
                        if (it + 1 == C::STAGES) {
                            pdl_wait();
                            pdl_trigger();
                            waited = true;
                            for (int i = 0; i <= it; ++i)
                                bulk_g2s(sb + i * C::KT * C::B_KT, a.bcanon + (int64_t)pend_kc[i] * C::B_KT,
                                         pend_n[i] * C::B_KT, &full[i]);
                        }
                    }
                }
                u += kb - ka;
            }
            if (!waited) {  // fewer stages than the ring holds
                pdl_wait();
                pdl_trigger();
                for (int i = 0; i < it; ++i)
                    bulk_g2s(sb + i * C::KT * C::B_KT, a.bcanon + (int64_t)pend_kc[i] * C::B_KT, pend_n[i] * C::B_KT,
                             &full[i]);
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer: segment i (one row group's k range) accumulates in set i % NSETS
        if (lane == 0) {
            int it = 0, i = 0;
            for (int64_t u = u0; u < u1; ++i) {
                const int ka = (int)(u % KC);
                const int kb = u1 - u < (int64_t)(KC - ka) ? ka + (int)(u1 - u) : KC;
                const int b = i % C::NSETS;
                mbar_wait(&accempty[b], ((i / C::NSETS) & 1) ^ 1);
                tc_fence_after();
                const uint32_t acc = tmem + b * C::ACC;
                for (int kc = ka; kc < kb; kc += C::KT, ++it) {
                    const int s = it % C::STAGES, n = min(C::KT, kb - kc);
                    mbar_wait(&full[s], (it / C::STAGES) & 1);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sa + s * C::KT * TC_A), b0 = smem_u32(sb + s * C::KT * C::B_KT);
                    for (int k = 0; k < n; ++k)
                        tc_mma<C::IDESC>(acc, umma_desc(a0 + k * TC_A), umma_desc(b0 + k * C::B_KT),
                                         (kc - ka) | k);
                    tc_commit(&empty[s]);
                }
                tc_commit(&accfull[b]);
                u += kb - ka;
            }
        }
        __syncwarp();
    } else {
        // ---------------- epilogue (warps 2-9): TMEM lanes 32 (warp % 4) .. + 31 = rows of the group;
        // warp half h finishes tokens 16 h .. 16 h + 15 (BN = 16: half 1 only releases the set)
        const int quarter = warp & 3, half = (warp - 2) >> 2;
        const int row = quarter * 32 + lane;
        const int c0 = half * 16;
        const bool mine = c0 < BN;
        // the per-token constants (scale, KV page / slot) come from the operand kernel: after the PDL wait
        pdl_wait();
        stage_tokens(a.epi, a.act.back, a.act.n_tok, 0, BN, s_tok, (int)threadIdx.x - 64, 32 * TC_EPI_WARPS);
        // the per-token max |y s_next| (EPI_GELU) is reduced in shared memory and leaves the CTA as
        // BN global atomics at the end: every row group's warps hitting the same BN addresses in L2
        // serialised the mlp_in launch (448 row groups x 4 quarters x BN atomics on one 128-B line)
        float* tmax = a.epi.tokmax ? s_tmax : nullptr;
        if ((int)threadIdx.x - 64 < BN) s_tmax[threadIdx.x - 64] = 0.f;
        asm volatile("bar.sync 1, %0;" ::"r"(32 * TC_EPI_WARPS) : "memory");
        int i = 0;
        for (int64_t u = u0; u < u1; ++i) {
            const int mg = (int)(u / KC), ka = (int)(u % KC);
            const int kb = u1 - u < (int64_t)(KC - ka) ? ka + (int)(u1 - u) : KC;
            u += kb - ka;
            const int b = i % C::NSETS;
            mbar_wait(&accfull[b], (i / C::NSETS) & 1);
            tc_fence_after();
            const int o = mg * TC_BM + row;
            const uint32_t tbase = tmem + b * C::ACC + ((uint32_t)(quarter * 32) << 16);
            if (!mine) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&accempty[b]);
                continue;
            }
            if (ka == 0 && kb == KC) {  // whole row group in this CTA
                int h[16], m[16], l[16];
                tmem_ld16(tbase + c0, h);
                tmem_ld16(tbase + BN + c0, m);
                tmem_ld16(tbase + 2 * BN + c0, l);
                tc_epi16(a.epi, o, lane, c0, s_tok + c0, h, m, l, tmax);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&accempty[b]);
                continue;
            }
            // split row group: add this CTA's s32 digit sums into the row group's
            // accumulator (fire-and-forget reductions at L2, [mg][column][row]: a
            // warp's 32 rows are one 128-B line), then count in; the last
            // contributor reads the sums once, zeroes them for the next launch
            // and runs the epilogue. Exact integers: arrival order is irrelevant.
            int* acc = a.skacc + (int64_t)mg * C::N * TC_BM + row;
            for (int p = 0; p < 3; ++p) {  // digit p of this warp's 16 tokens: columns p BN + c0 ..
                int v[16];
                tmem_ld16(tbase + p * BN + c0, v);
#pragma unroll
                for (int q = 0; q < 16; ++q) atomicAdd(acc + (p * BN + c0 + q) * TC_BM, v[q]);  // RED.ADD
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&accempty[b]);
            __threadfence();
            __syncwarp();
            const int cf = sk_owner_of((int64_t)mg * KC, a.total, a.G);
            const int cl = sk_owner_of((int64_t)mg * KC + KC - 1, a.total, a.G);
            int last = 0;
            int* cnt = a.counters + mg * 8 + quarter * 2 + half;
            if (lane == 0) last = atomicAdd(cnt, 1) == cl - cf;
            last = __shfl_sync(0xffffffffu, last, 0);
            if (!last) continue;
            __threadfence();
            if (lane == 0) *cnt = 0;  // ready for the next launch
            {
                int h[16], m[16], l[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    h[j] = __ldcg(acc + (c0 + j) * TC_BM);
                    m[j] = __ldcg(acc + (BN + c0 + j) * TC_BM);
                    l[j] = __ldcg(acc + (2 * BN + c0 + j) * TC_BM);
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    __stcg(acc + (c0 + j) * TC_BM, 0);
                    __stcg(acc + (BN + c0 + j) * TC_BM, 0);
                    __stcg(acc + (2 * BN + c0 + j) * TC_BM, 0);
                }
                tc_epi16(a.epi, o, lane, c0, s_tok + c0, h, m, l, tmax);
            }
        }
        if (tmax) {
            asm volatile("bar.sync 1, %0;" ::"r"(32 * TC_EPI_WARPS) : "memory");
            const int t = (int)threadIdx.x - 64;
            if (t < BN && t < a.act.n_tok)
                atomicMax(reinterpret_cast<int*>(a.epi.tokmax) + t, __float_as_int(s_tmax[t]));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::NSETS * C::ACC));
    }
}

template <int BN, int KT_, int ST_>
static int launch_sk(const Mat& m, const uint8_t* bcanon, const Act& act, const Epi& epi, int* skacc,
                     int64_t skacc_bytes, int* counters, cudaStream_t st) {
    using C = SkCfg<BN, KT_, ST_>;
    static_assert(C::SMEM <= 232448, "smem");
    static int ok[PB_MAX_DEVICES] = {};
    if (per_device(ok, [](int) {
            return cudaFuncSetAttribute(k_gemm_tc_sk<BN, KT_, ST_>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)C::SMEM) == cudaSuccess ? 1 : -1;
        }) < 0)
        return launch_check("gemm_tc_sk setup");
    const int sms = sm_count();
    if (sms < 0) return PB_ERR_GENERIC;
    TcSkArgs a{m.codes, bcanon, m.Kp / 32, m.Mp / 128, 0, 0, act, epi, skacc, counters};
    a.total = (int64_t)a.KC * a.MG;
    a.G = (int)std::min<int64_t>(sms, a.total);
    if ((int64_t)a.MG * TC_BM * C::N * 4 > skacc_bytes) {
        set_error("gemm_tc_sk: split accumulator workspace too small");
        return PB_ERR_CAPACITY;
    }
    return launch_pdl(k_gemm_tc_sk<BN, KT_, ST_>, dim3((unsigned)a.G), dim3(TC_THREADS), C::SMEM, st, a);
}

int launch_gemm_tc_sk(const Mat& m, const uint8_t* bcanon, int tile_tokens, const Act& act, const Epi& epi,
                      int* skacc, int64_t skacc_bytes, int* counters, cudaStream_t st) {
    if (act.n_tok > tile_tokens) {
        set_error("gemm_tc_sk: more tokens than one tile");
        return PB_ERR_GENERIC;
    }
    // (k tiles per stage, stages): 8 x 4 -- 8 x 3, 4 x 6 and 4 x 8 measured within 1 % at 32 tokens, 2 x 14 -25 %
    if (tile_tokens == 16) return launch_sk<16, 8, 4>(m, bcanon, act, epi, skacc, skacc_bytes, counters, st);
    if (tile_tokens == 32) return launch_sk<32, 8, 4>(m, bcanon, act, epi, skacc, skacc_bytes, counters, st);
    set_error("gemm_tc_sk: tile of 16 or 32 tokens");
    return PB_ERR_GENERIC;
}

}  // namespace pb
