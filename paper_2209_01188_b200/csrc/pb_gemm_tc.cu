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
constexpr int TC_THREADS = 192;
constexpr int TC_A = 4096;                 // int8 codes per k tile (128 rows x 32)
constexpr int TC_PLANE = TC_BN * 32;       // one digit plane per k tile
constexpr int TC_B = 3 * TC_PLANE;
constexpr int TC_ACC = 256;                // TMEM columns per accumulator set (3 x 80 used)
constexpr int TC_TMEM_COLS = 512;
constexpr size_t TC_SMEM = (size_t)TC_STAGES * TC_KT * (TC_A + TC_B) + (2 * TC_STAGES + 4) * 8 + 16;

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

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(TC_IDESC), "r"(accumulate));
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// arrive on the same-offset mbarrier of every CTA in the (2-CTA) cluster
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}
// global -> shared of both CTAs of the pair (same offset), complete_tx on each CTA's mbarrier at bar's offset
__device__ __forceinline__ void bulk_g2s_pair(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
        "%4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"((uint16_t)3)
        : "memory");
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
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
    int l2pf;               // L2 prefetch distance in k tiles (0: off)
    int ntg;                // token tiles per pass (NTL: one pass)
    Act act;
    Epi epi;
};

// PAIR: CTAs 2p and 2p + 1 form a cluster on row groups 2 mg' and 2 mg' + 1
// of the same token tile; each loads its own weight k tiles and HALF of the
// shared digit planes, multicast into both CTAs' shared memory, so a CTA pulls
// 4 + 3.75 KB per k tile through L2 instead of 4 + 7.5 KB. A stage is free
// again once both CTAs' MMAs have read it (empty barrier count 2, commits
// multicast to the pair).
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

template <bool PAIR>
__device__ __forceinline__ void gemm_tc_body(const TcArgs& a) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sa = smem;                                // [STAGES][KT][4 KB]
    uint8_t* sb = sa + TC_STAGES * TC_KT * TC_A;       // [STAGES][KT][3 planes]
    uint64_t* full = reinterpret_cast<uint64_t*>(sb + TC_STAGES * TC_KT * TC_B);
    uint64_t* empty = full + TC_STAGES;
    uint64_t* accfull = empty + TC_STAGES;  // [2]
    uint64_t* accempty = accfull + 2;       // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 2);

    const int warp = warp_uniform_id(), lane = threadIdx.x & 31;
    const int KC = a.KC;
    // tile schedule: unit u = cta, cta + NU, ...; PAIR units are (row-group pair, token tile)
    const int rank = PAIR ? (int)(blockIdx.x & 1) : 0;
    const int cta = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
    const int NU = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
    const int units = PAIR ? a.tiles / 2 : a.tiles;
    const int mgs = PAIR ? a.MG / 2 : a.MG;

    if (threadIdx.x == 0) {
        for (int s = 0; s < TC_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], PAIR ? 2 : 1);  // MMA commit (both CTAs' when PAIR)
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&accfull[b], 1);   // MMA commit after a tile's last k step
            mbar_init(&accempty[b], 4);  // the 4 epilogue warps
        }
        mbar_fence_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TC_TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    if (PAIR)
        cluster_sync();  // the peer's barriers are initialised before any multicast reaches them
    else
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
                const int mg = PAIR ? 2 * mgu + rank : mgu;
                const int8_t* asrc = a.codes + (int64_t)mg * KC * TC_A;
                const uint8_t* bsrc = a.bcanon + (int64_t)nt * KC * TC_B;
                for (int kc = 0; kc < KC; kc += TC_KT, ++it) {
                    const int s = it % TC_STAGES, n = min(TC_KT, KC - kc);
                    if (a.l2pf) {
                        // pull k tiles l2pf ahead of the ring into L2: the ring (4 stages, ~1 us of MMA) is
                        // shorter than an HBM miss under load
                        const int kp = kc + a.l2pf;
                        if (kp < KC) {
                            const int np = min(TC_KT, KC - kp);
                            bulk_prefetch_l2(asrc + (int64_t)kp * TC_A, np * TC_A);
                            if (PAIR)
                                bulk_prefetch_l2(bsrc + (int64_t)kp * TC_B + rank * np * (TC_B / 2), np * (TC_B / 2));
                            else
                                bulk_prefetch_l2(bsrc + (int64_t)kp * TC_B, np * TC_B);
                        }
                    }
                    mbar_wait(&empty[s], ((it / TC_STAGES) & 1) ^ 1);
                    mbar_expect_tx(&full[s], n * (TC_A + TC_B));
                    // consecutive k tiles are contiguous in both operands: one copy each
                    bulk_g2s(sa + s * TC_KT * TC_A, asrc + (int64_t)kc * TC_A, n * TC_A, &full[s]);
                    if (PAIR) {
                        const uint32_t half = n * (TC_B / 2);  // n * 3840 B: 16-B multiple
                        bulk_g2s_pair(sb + s * TC_KT * TC_B + rank * half, bsrc + (int64_t)kc * TC_B + rank * half,
                                      half, &full[s]);
                    } else {
                        bulk_g2s(sb + s * TC_KT * TC_B, bsrc + (int64_t)kc * TC_B, n * TC_B, &full[s]);
                    }
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
                        tc_mma(acc, umma_desc(a0 + k * TC_A), umma_desc(b0 + k * TC_B), (kc | k) != 0);
                    if (PAIR)
                        tc_commit_pair(&empty[s]);
                    else
                        tc_commit(&empty[s]);
                }
                tc_commit(&accfull[b]);
            }
        }
        __syncwarp();
    } else {
        // ---------------- epilogue (warps 2-5): TMEM lanes 32 (warp % 4) .. + 31
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const bool want_max = a.epi.tokmax != nullptr;
        int i = 0;
        for (int u = cta; u < units; u += NU, ++i) {
            int mgu, nt;
            tc_unit(a, u, mgs, mgu, nt);
            const int mg = PAIR ? 2 * mgu + rank : mgu;
            const int b = i & 1;
            mbar_wait(&accfull[b], (i >> 1) & 1);
            tc_fence_after();
            const int o = mg * TC_BM + row;
            const uint32_t tbase = tmem + b * TC_ACC + ((uint32_t)(quarter * 32) << 16);
            for (int c0 = 0; c0 < TC_BN; c0 += 16) {
                int h[16], m[16], l[16];
                tmem_ld16(tbase + c0, h);
                tmem_ld16(tbase + TC_BN + c0, m);
                tmem_ld16(tbase + 2 * TC_BN + c0, l);
#pragma unroll 4
                for (int j = 0; j < 16; ++j) {
                    const int tok = nt * TC_BN + c0 + j;
                    float mx = 0.f;
                    if (tok < a.act.n_tok && o < a.epi.M) {
                        // exact integer (|iv| < 2^47), one rounding to f32: same value as the f64 sum
                        const long long iv = (long long)h[j] * 65536 + (long long)m[j] * 256 + (long long)l[j];
                        const float y = epi_store(a.epi, tok, o, (float)iv * a.act.back[tok]);
                        if (want_max) mx = fabsf(y * a.epi.s_next[o]);
                    }
                    if (want_max) {
                        mx = warp_max(mx);
                        if (lane == 0 && tok < a.act.n_tok)
                            atomicMax(reinterpret_cast<int*>(a.epi.tokmax) + tok, __float_as_int(mx));
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&accempty[b]);
        }
    }
    tc_fence_before();
    if (PAIR)
        cluster_sync();  // no multicast copy or commit may still target an exited peer
    else
        __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TC_TMEM_COLS));
    }
}

__global__ void __launch_bounds__(TC_THREADS, 1) k_gemm_tc(TcArgs a) { gemm_tc_body<false>(a); }

int launch_gemm_tc(const Mat& m, const uint8_t* bcanon, const Act& act, const Epi& epi, cudaStream_t st) {
    static int ok[PB_MAX_DEVICES] = {};
    if (per_device(ok, [](int) {
            return cudaFuncSetAttribute(k_gemm_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TC_SMEM) ==
                           cudaSuccess ? 1 : -1;
        }) < 0)
        return launch_check("gemm_tc setup");
    const int sms = sm_count();
    if (sms < 0) return PB_ERR_GENERIC;
    TcArgs a{m.codes, bcanon, m.Kp / 32, m.Mp / 128, (int)ceil_div(act.n_tok, TC_BN), 0, 0, 0, act, epi};
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

}  // namespace pb
