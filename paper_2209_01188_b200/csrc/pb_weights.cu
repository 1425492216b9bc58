// Deterministic weight generation (model.py:36-62,176-209) and the LLM.int8-
// style weight quantizer (quant.py:81-108 applied to W^T as in quant.py:142-149).
//
// Orientation: the reference quantizes W^T, W = [in, out], with
// one absmax scale per input feature k (a row of W) and treats a whole input
// feature as an outlier when max_o |W[k, o]| > threshold. Codes are stored
// [out, in] in 4 KB tiles of 128 output rows x 32 inputs, tile (mg, kc) at
// (mg * KC + kc) * 4096 (a 128-row group's tiles are consecutive along k: one
// bulk copy streams a stage). Inside a tile the layout is the UMMA canonical
// K-major no-swizzle form for 8-bit operands:
//   byte (r >> 3) * 256 + (k >> 4) * 128 + (r & 7) * 16 + (k & 15)
// i.e. 8-row x 16-byte core matrices (LBO 128 B along k, SBO 256 B along
// rows). The same tile feeds tcgen05.mma kind::i8 descriptors directly and
// the decode GEMV's ldmatrix (each core matrix = one 8x8 b16 ldmatrix tile =
// the m16n8k32 s8 A fragment quarter).
// Weights are generated on the fly from the counter-form SplitMix64 stream, so
// a 176B-shape block never materializes in f32.
#include <vector>

#include "pb_common.cuh"
#include "pb_span.h"

namespace pb {

// --------------------------------------------------------------- value sources

struct GenSource {  // W[k, o] = stream[k * M + o] of key
    uint64_t key;
    int64_t M;
    float boost;
    int every;
    __device__ __forceinline__ float operator()(int64_t k, int64_t o) const {
        float w = gen_weight(key, (uint64_t)(k * M + o) + 1ull);
        if (every > 0 && (k % every) == 0) w = __fmul_rn(w, boost);
        return w;
    }
};

struct MatSource {  // row-major f32 [K, M] on the device
    const float* w;
    int64_t M;
    __device__ __forceinline__ float operator()(int64_t k, int64_t o) const { return w[k * M + o]; }
};

struct TransSource {  // W[k, o] = wt[o * K + k]: row-major W^T [M][K] on the device
    const float* wt;
    int64_t K;
    __device__ __forceinline__ float operator()(int64_t k, int64_t o) const { return wt[o * K + k]; }
};

// column absmax of W^T (coalesced along k); non-negative floats compare as ints
__global__ void __launch_bounds__(256) k_col_absmax_t(const float* __restrict__ wt, int64_t K, int64_t M,
                                                      int rows_per_cta, int* __restrict__ bits) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= K) return;
    const int64_t o0 = (int64_t)blockIdx.y * rows_per_cta, o1 = min(M, o0 + rows_per_cta);
    float m = 0.f;
    for (int64_t o = o0; o < o1; ++o) m = fmaxf(m, fabsf(wt[o * K + k]));
    atomicMax(bits + k, __float_as_int(m));
}

__global__ void k_scales_from_absmax(const int* __restrict__ bits, int64_t K, float threshold,
                                     float* __restrict__ scales, uint8_t* __restrict__ outl) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < K; k += (int64_t)gridDim.x * blockDim.x) {
        const float m = __int_as_float(bits[k]);
        const bool is_out = m > threshold;  // quant.py:90-93
        outl[k] = is_out ? 1 : 0;
        scales[k] = is_out ? 0.f : __fdiv_rn(m, 127.f);
    }
}

__global__ void k_gen_tensor(uint64_t key, int64_t first, int64_t n, float* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = gen_weight(key, (uint64_t)(first + i) + 1ull);
}

// pass 1: per input feature absmax -> scale, outlier flag (quant.py:90-93)
template <class Src>
__global__ void __launch_bounds__(256) k_feature_absmax(Src src, int64_t K, int64_t M, float threshold,
                                                        float* __restrict__ scales, uint8_t* __restrict__ outl) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = warp; k < K; k += nwarps) {
        float m = 0.f;
        for (int64_t o = lane; o < M; o += 32) m = fmaxf(m, fabsf(src(k, o)));
        m = warp_max(m);
        if (lane == 0) {
            const bool is_out = m > threshold;
            outl[k] = is_out ? 1 : 0;
            scales[k] = is_out ? 0.f : __fdiv_rn(m, 127.f);  // f32(col_absmax / 127.0)
        }
    }
}

// pass 2: tiled codes, one thread per 16-byte core-matrix row (row r, 16-wide k half)
template <class Src>
__global__ void __launch_bounds__(256) k_quant_tiles(Src src, int64_t K, int64_t M, int64_t KC, int64_t MG,
                                                     const float* __restrict__ scales, int8_t* __restrict__ codes) {
    const int64_t total = MG * KC * 256;  // 128 rows x 2 halves per tile
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += stride) {
        const int r = (int)(t & 127), kh = (int)((t >> 7) & 1);
        const int64_t tile = t >> 8;
        const int64_t mg = tile / KC, kc = tile % KC;
        const int64_t o = mg * 128 + r;
        uint32_t words[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int b = 0; b < 16; ++b) {
            const int64_t k = kc * 32 + kh * 16 + b;
            int code = 0;
            if (o < M && k < K) {
                const float s = scales[k];
                if (s > 0.f) {  // quant.py:97-100 (zero scale: outlier or all-zero feature)
                    const double qd = (double)src(k, o) / (double)s;
                    double rr = floor(fabs(qd) + 0.5);
                    rr = rr > 127.0 ? 127.0 : rr;
                    code = qd < 0.0 ? -(int)rr : (int)rr;
                }
            }
            words[b >> 2] |= (uint32_t)(uint8_t)(int8_t)code << (8 * (b & 3));
        }
        const int64_t off = tile * 4096 + (r >> 3) * 256 + kh * 128 + (r & 7) * 16;
        *reinterpret_cast<uint4*>(codes + off) = make_uint4(words[0], words[1], words[2], words[3]);
    }
}

template <class Src>
__global__ void k_gather_outliers(Src src, const int32_t* __restrict__ idx, int n_outl, int64_t M,
                                  float* __restrict__ rows) {
    const int64_t total = (int64_t)n_outl * M;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += stride) {
        const int64_t j = t / M, o = t % M;
        rows[t] = src(idx[j], o);
    }
}

template <class Src>
__global__ void k_materialize(Src src, int64_t K, int64_t M, float* __restrict__ out) {
    const int64_t total = K * M;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += stride)
        out[t] = src(t / M, t % M);
}

// inverse of the tiling (test/inspection): codes_out[o * K + k]
__global__ void k_untile(const int8_t* __restrict__ tiles, int64_t K, int64_t M, int64_t KC,
                         int8_t* __restrict__ out) {
    const int64_t total = K * M;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += stride) {
        const int64_t o = t / K, k = t % K;
        const int64_t mg = o >> 7, r = o & 127, kc = k >> 5, kk = k & 31;
        out[t] = tiles[(mg * KC + kc) * 4096 + (r >> 3) * 256 + (kk >> 4) * 128 + (r & 7) * 16 + (kk & 15)];
    }
}

static int grid_n(int64_t n, int threads = 256) {
    int64_t g = ceil_div(n, threads);
    return (int)(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

template <class Src>
static int quantize_matrix(Mat& m, Src src, float threshold, cudaStream_t st, const float* wt = nullptr) {
    if (m.tcodes) {  // new codes: the BACKWARD cache of their transpose is stale
        PB_CHECK_CUDA(cudaStreamSynchronize(st));
        cudaFree(m.tcodes);
        m.tcodes = nullptr;
    }
    const int64_t K = m.K, M = m.M, KC = m.Kp / 32, MG = m.Mp / 128;
    uint8_t* d_flags = nullptr;
    PB_CHECK_CUDA(cudaMallocAsync(&d_flags, K, st));
    PB_CHECK_CUDA(cudaMemsetAsync(m.scales, 0, sizeof(float) * m.Kp, st));
    if (wt) {  // transposed source: coalesced column absmax
        int* bits = nullptr;
        PB_CHECK_CUDA(cudaMallocAsync(&bits, sizeof(int) * K, st));
        PB_CHECK_CUDA(cudaMemsetAsync(bits, 0, sizeof(int) * K, st));
        const int rows = 512;
        k_col_absmax_t<<<dim3((unsigned)ceil_div(K, 256), (unsigned)ceil_div(M, rows)), 256, 0, st>>>(wt, K, M, rows,
                                                                                                     bits);
        if (int rc = launch_check("col_absmax_t")) return rc;
        k_scales_from_absmax<<<grid_n(K), 256, 0, st>>>(bits, K, threshold, m.scales, d_flags);
        if (int rc = launch_check("scales_from_absmax")) return rc;
        PB_CHECK_CUDA(cudaFreeAsync(bits, st));
    } else {
        k_feature_absmax<Src><<<grid_n(K * 32), 256, 0, st>>>(src, K, M, threshold, m.scales, d_flags);
        if (int rc = launch_check("feature_absmax")) return rc;
    }
    k_quant_tiles<Src><<<grid_n(MG * KC * 256), 256, 0, st>>>(src, K, M, KC, MG, m.scales, m.codes);
    if (int rc = launch_check("quant_tiles")) return rc;
    std::vector<uint8_t> flags(K);
    PB_CHECK_CUDA(cudaMemcpyAsync(flags.data(), d_flags, K, cudaMemcpyDeviceToHost, st));
    PB_CHECK_CUDA(cudaStreamSynchronize(st));
    PB_CHECK_CUDA(cudaFreeAsync(d_flags, st));
    std::vector<int32_t> idx;
    for (int64_t k = 0; k < K; ++k)
        if (flags[k]) idx.push_back((int32_t)k);
    m.free_outliers();
    m.n_outl = (int)idx.size();
    m.h_outl_idx = idx;
    if (m.n_outl) {
        PB_CHECK_CUDA(cudaMalloc(&m.outl_idx, sizeof(int32_t) * m.n_outl));
        PB_CHECK_CUDA(cudaMalloc(&m.outl_rows, sizeof(float) * (size_t)m.n_outl * M));
        PB_CHECK_CUDA(cudaMemcpyAsync(m.outl_idx, idx.data(), sizeof(int32_t) * m.n_outl, cudaMemcpyHostToDevice, st));
        k_gather_outliers<Src><<<grid_n((int64_t)m.n_outl * M), 256, 0, st>>>(src, m.outl_idx, m.n_outl, M,
                                                                              m.outl_rows);
        if (int rc = launch_check("gather_outliers")) return rc;
        PB_CHECK_CUDA(cudaStreamSynchronize(st));
    }
    return PB_OK;
}

int fill_matrix_gen(Mat& m, uint64_t key, float threshold, float boost, int every, cudaStream_t st) {
    GenSource src{key, m.M, boost, every};
    if (m.int8) return quantize_matrix(m, src, threshold, st);
    k_materialize<GenSource><<<grid_n((int64_t)m.K * m.M), 256, 0, st>>>(src, m.K, m.M, m.w32);
    return launch_check("materialize_gen");
}

int fill_matrix_f32(Mat& m, const float* w, float threshold, cudaStream_t st) {
    MatSource src{w, m.M};
    if (m.int8) return quantize_matrix(m, src, threshold, st);
    PB_CHECK_CUDA(cudaMemcpyAsync(m.w32, w, sizeof(float) * (size_t)m.K * m.M, cudaMemcpyDeviceToDevice, st));
    return PB_OK;
}

int fill_matrix_f32_t(Mat& m, const float* wt, float threshold, cudaStream_t st) {
    TransSource src{wt, m.K};
    return quantize_matrix(m, src, threshold, st, wt);
}

int untile_codes(const Mat& m, int8_t* d_out, cudaStream_t st) {
    k_untile<<<grid_n((int64_t)m.K * m.M), 256, 0, st>>>(m.codes, m.K, m.M, m.Kp / 32, d_out);
    return launch_check("untile");
}

}  // namespace pb

extern "C" int pb_gen_tensor(uint64_t key, int64_t first, int64_t n, float* d_out, void* stream) {
    PB_REQUIRE(n >= 0 && first >= 0, PB_ERR_BAD_REQUEST, "negative range");
    if (n == 0) return PB_OK;
    pb::k_gen_tensor<<<pb::grid_n(n), 256, 0, (cudaStream_t)stream>>>(key, first, n, d_out);
    return pb::launch_check("gen_tensor");
}
