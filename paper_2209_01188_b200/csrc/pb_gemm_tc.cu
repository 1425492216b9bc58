// tcgen05 (5th-gen tensor core) int8-weight x fp16-activation GEMM for
// prefill / parallel forward / large batched steps (model.py:341,362,366,368
// via quant.py:117-129), fed by the TMA engine (cp.async.bulk), accumulating
// in TMEM.
//
// D[o, n] (fp32, TMEM) = sum_k code[o, k] * B[n, k], one CTA per 128 output
// rows x 256 columns (128 tokens x {hi, lo} fp16 halves of x~ = s ⊙ x, the
// same exact operand split as the decode GEMV).
//
// Warp roles (192 threads):
//   warp 0      TMA producer: per 32-wide k tile, 4 KB of int8 codes (the
//               128-row group's tile, contiguous in HBM) + 16 KB of B (already
//               in UMMA canonical K-major layout) -> smem ring, mbarrier tx.
//   warps 1-4   converters: int8 -> fp16 (PRMT / HSUB2, exact), written into
//               the canonical no-swizzle K-major A layout; then the epilogue
//               (tcgen05.ld of their 32 TMEM lanes, hi+lo, fused block epilogue).
//   warp 5      TMEM owner + MMA issuer: one elected lane issues
//               tcgen05.mma.cta_group::1.kind::f16 (M=128, N=256, K=16) twice
//               per k tile and tcgen05.commit's the smem stages back.
// Canonical K-major (SWIZZLE_NONE) smem layout for both operands: 8x8 fp16
// core matrices (128 B), LBO = 128 B between the two 8-k halves of a K=16
// step, SBO = 512 B between 8-row groups (a 32-wide k tile = 4 core columns).
#include "pb_async.cuh"
#include "pb_common.cuh"
#include "pb_epi.cuh"
#include "pb_span.h"

namespace pb {

constexpr int TC_BM = 128;
constexpr int TC_BN = 256;
constexpr int TC_TOK = TC_BN / 2;  // tokens per tile (hi + lo columns)
constexpr int TC_STAGES = 4;
constexpr int TC_FSTAGES = 2;
constexpr int TC_THREADS = 192;
constexpr int TC_A8 = 4096;                 // int8 codes per k tile (128 rows x 32)
constexpr int TC_B = TC_BN * 32 * 2;        // 16 KB fp16 B per k tile
constexpr int TC_A16 = TC_BM * 32 * 2;      // 8 KB fp16 A per k tile
constexpr size_t TC_SMEM = (size_t)TC_STAGES * (TC_A8 + TC_B) + (size_t)TC_FSTAGES * TC_A16 + 256;

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(512 >> 4) << 32) |
           (1ull << 46);  // version 1 (sm_100), base offset 0, SWIZZLE_NONE
}

// kind::f16, D f32, A f16, B f16, both K-major, N = 256, M = 128
constexpr uint32_t TC_IDESC = (1u << 4) | ((uint32_t)(TC_BN >> 3) << 17) | ((uint32_t)(TC_BM >> 4) << 24);

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(TC_IDESC), "r"(accumulate), "r"(0), "r"(0), "r"(0), "r"(0));
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 4 int8 -> two f16x2 ({b0,b1}, {b2,b3}), exact (same trick as the GEMV)
__device__ __forceinline__ void tc_i8x4(uint32_t w, uint32_t& lo, uint32_t& hi) {
    const uint32_t u = w ^ 0x80808080u;
    const uint32_t p0 = __byte_perm(u, 0x64646464u, 0x4140);
    const uint32_t p1 = __byte_perm(u, 0x64646464u, 0x4342);
    const half2 bias = __halves2half2(__ushort_as_half(0x6480), __ushort_as_half(0x6480));
    half2 r0 = __hsub2(*reinterpret_cast<const half2*>(&p0), bias);
    half2 r1 = __hsub2(*reinterpret_cast<const half2*>(&p1), bias);
    lo = *reinterpret_cast<uint32_t*>(&r0);
    hi = *reinterpret_cast<uint32_t*>(&r1);
}


struct TcArgs {
    const int8_t* codes;
    const uint8_t* bcanon;  // [n_tiles][KC][16 KB]
    int KC, MG;
    Act act;
    Epi epi;
};

__global__ void __launch_bounds__(TC_THREADS, 1) k_gemm_tc(TcArgs a) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sa8 = smem;                                      // [STAGES][4 KB]
    uint8_t* sb = sa8 + TC_STAGES * TC_A8;                    // [STAGES][16 KB]
    uint8_t* sa16 = sb + TC_STAGES * TC_B;                    // [FSTAGES][8 KB]
    uint64_t* full = reinterpret_cast<uint64_t*>(sa16 + TC_FSTAGES * TC_A16);
    uint64_t* empty = full + TC_STAGES;
    uint64_t* ffull = empty + TC_STAGES;
    uint64_t* fempty = ffull + TC_FSTAGES;
    uint64_t* accfull = fempty + TC_FSTAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accfull + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mg = blockIdx.x, nt = blockIdx.y;
    const int KC = a.KC;

    if (threadIdx.x == 0) {
        for (int s = 0; s < TC_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 5);  // 4 converter warps + MMA commit
        }
        for (int f = 0; f < TC_FSTAGES; ++f) {
            mbar_init(&ffull[f], 4);
            mbar_init(&fempty[f], 1);
        }
        mbar_init(accfull, 1);
        mbar_fence_init();
    }
    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TC_BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer
        if (lane == 0) {
            const int8_t* asrc = a.codes + (int64_t)mg * KC * TC_A8;
            const uint8_t* bsrc = a.bcanon + (int64_t)nt * KC * TC_B;
            for (int kc = 0; kc < KC; ++kc) {
                const int s = kc % TC_STAGES;
                const uint32_t ph = (kc / TC_STAGES) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                mbar_expect_tx(&full[s], TC_A8 + TC_B);
                bulk_g2s(sa8 + s * TC_A8, asrc + (int64_t)kc * TC_A8, TC_A8, &full[s]);
                bulk_g2s(sb + s * TC_B, bsrc + (int64_t)kc * TC_B, TC_B, &full[s]);
            }
        }
    } else if (warp == 5) {
        // ---------------- MMA issuer
        if (lane == 0) {
            for (int kc = 0; kc < KC; ++kc) {
                const int s = kc % TC_STAGES, f = kc % TC_FSTAGES;
                mbar_wait(&full[s], (kc / TC_STAGES) & 1);
                mbar_wait(&ffull[f], (kc / TC_FSTAGES) & 1);
                tc_fence_after();
                const uint32_t a0 = smem_u32(sa16 + f * TC_A16), b0 = smem_u32(sb + s * TC_B);
#pragma unroll
                for (int k16 = 0; k16 < 2; ++k16)
                    tc_mma(tmem, umma_desc(a0 + 256 * k16), umma_desc(b0 + 256 * k16), (kc | k16) != 0);
                tc_commit(&empty[s]);
                tc_commit(&fempty[f]);
            }
            tc_commit(accfull);
        }
        __syncwarp();
    } else {
        // ---------------- converters (warps 1-4): rows 32cw .. 32cw+31 of the tile
        // int8 canonical core matrices (8 rows x 16 k, pb_weights.cu) -> fp16
        // canonical core matrices (8 rows x 8 k): one row x 16 k per thread and k half
        const int cw = warp - 1;
        const int r = cw * 32 + lane;
        for (int kc = 0; kc < KC; ++kc) {
            const int s = kc % TC_STAGES, f = kc % TC_FSTAGES;
            mbar_wait(&full[s], (kc / TC_STAGES) & 1);
            mbar_wait(&fempty[f], ((kc / TC_FSTAGES) & 1) ^ 1);
            uint8_t* dst = sa16 + f * TC_A16;
#pragma unroll
            for (int kh = 0; kh < 2; ++kh) {
                const uint4 w = *reinterpret_cast<const uint4*>(sa8 + s * TC_A8 + (r >> 3) * 256 + kh * 128 + (r & 7) * 16);
                uint32_t h[8];
                tc_i8x4(w.x, h[0], h[1]);
                tc_i8x4(w.y, h[2], h[3]);
                tc_i8x4(w.z, h[4], h[5]);
                tc_i8x4(w.w, h[6], h[7]);
                uint8_t* base = dst + (r >> 3) * 512 + (2 * kh) * 128 + (r & 7) * 16;
                *reinterpret_cast<uint4*>(base) = make_uint4(h[0], h[1], h[2], h[3]);
                *reinterpret_cast<uint4*>(base + 128) = make_uint4(h[4], h[5], h[6], h[7]);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core reads
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&ffull[f]);
                mbar_arrive(&empty[s]);
            }
        }
        // ---------------- epilogue: TMEM lanes 32 (warp % 4) .. + 31
        mbar_wait(accfull, 0);
        tc_fence_after();
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const int o = mg * TC_BM + row;
        const uint32_t tbase = tmem + ((uint32_t)(quarter * 32) << 16);
        const bool want_max = a.epi.tokmax != nullptr;
        for (int c0 = 0; c0 < TC_TOK; c0 += 16) {
            float hi[16], lo[16];
            tmem_ld16(tbase + c0, hi);
            tmem_ld16(tbase + TC_TOK + c0, lo);
#pragma unroll 4
            for (int i = 0; i < 16; ++i) {
                const int tok = nt * TC_TOK + c0 + i;
                float m = 0.f;
                if (tok < a.act.n_tok && o < a.epi.M) {
                    const float y = epi_store(a.epi, tok, o, (hi[i] + lo[i]) * a.act.back[tok]);
                    if (want_max) m = fabsf(y * a.epi.s_next[o]);
                }
                if (want_max) {
                    m = warp_max(m);
                    if (lane == 0 && tok < a.act.n_tok) atomicMax(reinterpret_cast<int*>(a.epi.tokmax) + tok, __float_as_int(m));
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TC_BN));
    }
}

int launch_gemm_tc(const Mat& m, const uint8_t* bcanon, const Act& act, const Epi& epi, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_gemm_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TC_SMEM);
        configured = true;
    }
    TcArgs a{m.codes, bcanon, m.Kp / 32, m.Mp / 128, act, epi};
    dim3 grid((unsigned)(m.Mp / 128), (unsigned)ceil_div(act.n_tok, TC_TOK));
    k_gemm_tc<<<grid, TC_THREADS, TC_SMEM, st>>>(a);
    return launch_check("gemm_tc");
}

}  // namespace pb
