// Wire codec: blockwise absmax int8 (quant.py:33-66 via transport/wire.py:98-105,125-137).
//
// HBM-bound: 4 B read + 1 B + 4/64 B written per element on encode, the
// reverse on decode. Other block sizes than the default 64 use one warp per
// block with a strided loop. Bit-exact with the reference (see wire_code in
// pb_common.cuh; tests/test_gpu_codec.py).
#include <algorithm>

#include "pb_common.cuh"

namespace pb {

// block 64: a lane owns 16 consecutive elements (four 128-bit streaming loads
// issued together), four lanes own a block (two-step shuffle max), a warp moves
// 8 blocks = 2 KB of f32 per iteration and stores its codes as one 16-B word
// per lane. The code of x is round_half_away(|x| / s) decided exactly: the
// candidate comes from |x| * (1/s) (one reciprocal per block instead of an
// IEEE division per element; within one unit of the exact quotient) and the two
// fma residuals of exact_round_away_pos settle the half-integer boundary.
__device__ __forceinline__ int wire_code_r(float x, float s, float r, float amax) {
    if (s < 2.3509887e-38f) return wire_code(x, s, amax);  // zero / tiny scales: the reference's corner cases
    const float a = fabsf(x);
    float m = floorf(a * r + 0.5f);
    if (m > 200.f) m = 200.f;
    else if (fmaf(-(m + 0.5f), s, a) >= 0.f) m += 1.f;
    else if (m > 0.f && fmaf(-(m - 0.5f), s, a) < 0.f) m -= 1.f;
    const int c = m > 127.f ? 127 : (int)m;
    return x < 0.f ? -c : c;
}

__global__ void __launch_bounds__(256) k_wire_quant64(const float* __restrict__ x, int64_t n, int8_t* __restrict__ codes,
                                                      float* __restrict__ scales) {
    const int lane = threadIdx.x & 31;
    const int64_t nchunks = (n + 511) / 512;  // warp iterations of 8 blocks
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const bool vec = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(codes)) & 15) == 0;
    for (int64_t ch = warp; ch < nchunks; ch += nwarps) {
        const int64_t base = ch * 512 + lane * 16;
        float v[16];
        if (vec && base + 15 < n) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float4 f = __ldcs(reinterpret_cast<const float4*>(x + base) + q);
                v[4 * q] = f.x, v[4 * q + 1] = f.y, v[4 * q + 2] = f.z, v[4 * q + 3] = f.w;
            }
        } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = base + i < n ? x[base + i] : 0.f;
        }
        float m = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) m = fmaxf(m, fabsf(v[i]));
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
        const int64_t b = base >> 6;
        if (b * 64 >= n) continue;
        const float s = __fdiv_rn(m, 127.f);  // == f32(f64(absmax)/127): see pb_common.cuh
        const float r = s > 0.f ? __frcp_rn(s) : 0.f;
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            w[q] = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) w[q] |= (uint32_t)(uint8_t)wire_code_r(v[4 * q + i], s, r, m) << (8 * i);
        }
        if (vec && base + 15 < n) {
            *reinterpret_cast<uint4*>(codes + base) = make_uint4(w[0], w[1], w[2], w[3]);
        } else {
#pragma unroll
            for (int i = 0; i < 16; ++i)
                if (base + i < n) codes[base + i] = (int8_t)(w[i >> 2] >> (8 * (i & 3)));
        }
        if ((lane & 3) == 0) scales[b] = s;
    }
}

__global__ void __launch_bounds__(256) k_wire_quant_any(const float* __restrict__ x, int64_t n, int block,
                                                        int8_t* __restrict__ codes, float* __restrict__ scales) {
    const int64_t nb = (n + block - 1) / block;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b = warp; b < nb; b += nwarps) {
        const int64_t lo = b * block;
        const int64_t hi = lo + block < n ? lo + block : n;
        float m = 0.f;
        for (int64_t i = lo + lane; i < hi; i += 32) m = fmaxf(m, fabsf(x[i]));
        m = warp_max(m);
        const float s = __fdiv_rn(m, 127.f);
        for (int64_t i = lo + lane; i < hi; i += 32) codes[i] = wire_code(x[i], s, m);
        if (lane == 0) scales[b] = s;
    }
}

__global__ void __launch_bounds__(256) k_wire_dequant(const int8_t* __restrict__ codes, const float* __restrict__ scales,
                                                      int64_t n, int block, float* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = __fmul_rn((float)codes[i], scales[i / block]);
}

// block 64 (the wire default): 16 elements per thread, one 16-B code load, one
// scale, four 16-B stores
__global__ void __launch_bounds__(256) k_wire_dequant64(const int8_t* __restrict__ codes,
                                                        const float* __restrict__ scales, int64_t n,
                                                        float* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t * 16 < n; t += stride) {
        const int64_t base = t * 16;
        if (base + 15 < n) {
            const uint4 c = __ldcs(reinterpret_cast<const uint4*>(codes + base));
            const float s = scales[base >> 6];
            const uint32_t cw[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                float4 f;
                f.x = __fmul_rn((float)(int8_t)(cw[q] & 0xff), s);
                f.y = __fmul_rn((float)(int8_t)((cw[q] >> 8) & 0xff), s);
                f.z = __fmul_rn((float)(int8_t)((cw[q] >> 16) & 0xff), s);
                f.w = __fmul_rn((float)(int8_t)(cw[q] >> 24), s);
                __stcs(reinterpret_cast<float4*>(out + base) + q, f);
            }
        } else {
            for (int64_t i = base; i < n; ++i) out[i] = __fmul_rn((float)codes[i], scales[i >> 6]);
        }
    }
}

static int grid_for(int64_t work_items, int per_block) {
    const int sms = sm_count() > 0 ? sm_count() : 148;
    int64_t g = ceil_div(work_items, per_block);
    int64_t cap = (int64_t)sms * 8;
    return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

int quantize_blockwise(const float* x, int64_t n, int block, int8_t* codes, float* scales, cudaStream_t st) {
    if (n == 0) return PB_OK;
    if (block == 64) {
        // one wave: as many CTAs as are resident at once (a second partial wave doubled the latency)
        static int occ[PB_MAX_DEVICES] = {};
        const int per_sm = per_device(occ, [](int) {
            int b = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_wire_quant64, 256, 0);
            return b > 0 ? b : 1;
        });
        const int64_t cap = (int64_t)std::max(per_sm, 1) * std::max(sm_count(), 1);
        const int64_t want = ceil_div(ceil_div(n, 512) * 32, 256);
        k_wire_quant64<<<(unsigned)std::max<int64_t>(1, std::min(cap, want)), 256, 0, st>>>(x, n, codes, scales);
    } else {
        k_wire_quant_any<<<grid_for(ceil_div(n, block) * 32, 256), 256, 0, st>>>(x, n, block, codes, scales);
    }
    return launch_check("wire_quant");
}

int dequantize_blockwise(const int8_t* codes, const float* scales, int64_t n, int block, float* out,
                         cudaStream_t st) {
    if (n == 0) return PB_OK;
    const bool vec = ((reinterpret_cast<uintptr_t>(codes) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    if (block == 64 && vec)
        k_wire_dequant64<<<grid_for(ceil_div(n, 16), 256), 256, 0, st>>>(codes, scales, n, out);
    else
        k_wire_dequant<<<grid_for(n, 256), 256, 0, st>>>(codes, scales, n, block, out);
    return launch_check("wire_dequant");
}

}  // namespace pb

extern "C" int pb_quantize_blockwise(const float* d_x, int64_t n, int32_t block, int8_t* d_codes, float* d_scales,
                                     void* stream) {
    PB_REQUIRE(block >= 1, PB_ERR_BAD_REQUEST, "block_size must be >= 1");
    PB_REQUIRE(n >= 0, PB_ERR_BAD_REQUEST, "negative element count");
    return pb::quantize_blockwise(d_x, n, block, d_codes, d_scales, (cudaStream_t)stream);
}

extern "C" int pb_dequantize_blockwise(const int8_t* d_codes, const float* d_scales, int64_t n, int32_t block,
                                       float* d_out, void* stream) {
    PB_REQUIRE(block >= 1, PB_ERR_BAD_REQUEST, "block_size must be >= 1");
    PB_REQUIRE(n >= 0, PB_ERR_BAD_REQUEST, "negative element count");
    return pb::dequantize_blockwise(d_codes, d_scales, n, block, d_out, (cudaStream_t)stream);
}
