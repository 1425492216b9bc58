// Wire codec: blockwise absmax int8 (quant.py:33-66 via transport/wire.py:98-105,125-137).
//
// HBM-bound: 4 B read + 1 B + 4/64 B written per element on encode. For the
// default block of 64, a 16-lane half-warp owns one block (4 elements per lane
// as one float4), so a warp moves two blocks per iteration with 128-bit loads,
// a 4-step shuffle max and one 32-bit store of codes per lane. Other block
// sizes use one warp per block with a strided loop. Bit-exact with the
// reference (see wire_code in pb_common.cuh).
#include "pb_common.cuh"

namespace pb {

__global__ void __launch_bounds__(256) k_wire_quant64(const float* __restrict__ x, int64_t n, int8_t* __restrict__ codes,
                                                      float* __restrict__ scales) {
    const int64_t nb = (n + 63) / 64;
    const int lane = threadIdx.x & 31;
    const int half = lane >> 4;       // which block of the pair
    const int sub = lane & 15;        // 4 elements each
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b = warp * 2 + half; b - half < nb; b += nwarps * 2) {
        const int64_t base = b * 64 + sub * 4;
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        const bool blk_ok = b < nb;
        if (blk_ok) {
            if (base + 3 < n && ((reinterpret_cast<uintptr_t>(x + base) & 15) == 0)) {
                float4 f = __ldcs(reinterpret_cast<const float4*>(x + base));
                v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (base + i < n) v[i] = x[base + i];
            }
        }
        float m = fmaxf(fmaxf(fabsf(v[0]), fabsf(v[1])), fmaxf(fabsf(v[2]), fabsf(v[3])));
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (!blk_ok) continue;
        const float s = __fdiv_rn(m, 127.f);  // == f32(f64(absmax)/127): see pb_common.cuh
        uint32_t packed = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) packed |= (uint32_t)(uint8_t)wire_code(v[i], s, m) << (8 * i);
        if (base + 3 < n && ((reinterpret_cast<uintptr_t>(codes + base) & 3) == 0)) {
            *reinterpret_cast<uint32_t*>(codes + base) = packed;
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (base + i < n) codes[base + i] = (int8_t)(packed >> (8 * i));
        }
        if (sub == 0) scales[b] = s;
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

static int grid_for(int64_t work_items, int per_block) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t g = ceil_div(work_items, per_block);
    int64_t cap = (int64_t)sms * 8;
    return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

int quantize_blockwise(const float* x, int64_t n, int block, int8_t* codes, float* scales, cudaStream_t st) {
    if (n == 0) return PB_OK;
    if (block == 64) {
        k_wire_quant64<<<grid_for(ceil_div(n, 64) * 16, 256), 256, 0, st>>>(x, n, codes, scales);
    } else {
        k_wire_quant_any<<<grid_for(ceil_div(n, block) * 32, 256), 256, 0, st>>>(x, n, block, codes, scales);
    }
    return launch_check("wire_quant");
}

int dequantize_blockwise(const int8_t* codes, const float* scales, int64_t n, int block, float* out,
                         cudaStream_t st) {
    if (n == 0) return PB_OK;
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
