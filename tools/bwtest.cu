// Read-only HBM streaming ceiling on one B200: how fast can a kernel pull
// bytes it never writes back? (The measured peak in MEASURED_PEAKS.json is a
// copy; the decode GEMV and attention are pure reads.)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/bwtest.cu -o gpurun_out/bwtest
// Variants: (1) cp.async.bulk ring (1 producer lane, STAGES x STAGE bytes per CTA),
//           (2) ld.global.nc.v4 with UNROLL loads in flight per thread.
#include <cstdio>
#include <cstdint>
#include <vector>

#include "../paper_2209_01188_b200/csrc/pb_async.cuh"
#include "../paper_2209_01188_b200/csrc/pb_common.cuh"

using namespace pb;

template <int STAGE, int STAGES>
__global__ void __launch_bounds__(64) k_bulk(const uint8_t* __restrict__ src, int64_t bytes, int* sink) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGE * STAGES);
    const int64_t per = bytes / gridDim.x;
    const uint8_t* p = src + per * blockIdx.x;
    const int n = (int)(per / STAGE);
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
        mbar_fence_init();
    }
    __syncthreads();
    int acc = 0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES && i < n; ++i) {
            mbar_expect_tx(&full[i], STAGE);
            bulk_g2s(smem + i * STAGE, p + (int64_t)i * STAGE, STAGE, &full[i]);
        }
    }
    for (int i = 0; i < n; ++i) {
        const int s = i % STAGES;
        mbar_wait(&full[s], (i / STAGES) & 1);
        acc += smem[s * STAGE + threadIdx.x * 16];
        __syncthreads();
        if (threadIdx.x == 0 && i + STAGES < n) {
            mbar_expect_tx(&full[s], STAGE);
            bulk_g2s(smem + s * STAGE, p + (int64_t)(i + STAGES) * STAGE, STAGE, &full[s]);
        }
    }
    if (acc == 123456789) *sink = acc;
}

template <int UNROLL>
__global__ void __launch_bounds__(256) k_ldg(const int4* __restrict__ src, int64_t n16, int* sink) {
    int acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; i + (UNROLL - 1) * stride < n16; i += UNROLL * stride) {
        int4 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) v[u] = ld_stream_v4(src + i + u * stride);
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) acc ^= v[u].x ^ v[u].w;
    }
    if (acc == 123456789) *sink = acc;
}

template <int STAGE, int STAGES>
void run_bulk(const uint8_t* d, int64_t bytes, int* sink, int ctas_per_sm, int sms) {
    const size_t smem = (size_t)STAGE * STAGES + 8 * STAGES;
    cudaFuncSetAttribute(k_bulk<STAGE, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = sms * ctas_per_sm;
    const int64_t use = bytes / ((int64_t)grid * STAGE) * ((int64_t)grid * STAGE);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9f;
    for (int r = 0; r < 6; ++r) {
        cudaEventRecord(a);
        k_bulk<STAGE, STAGES><<<grid, 64, smem>>>(d, use, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r) best = ms < best ? ms : best;
    }
    printf("bulk stage=%6d stages=%d ctas/sm=%d smem=%7zu: %.1f GB/s %.1f us (%s)\n", STAGE, STAGES, ctas_per_sm, smem,
           use / best / 1e6, best * 1e3, cudaGetErrorString(cudaGetLastError()));
}

template <int UNROLL>
void run_ldg(const uint8_t* d, int64_t bytes, int* sink, int ctas_per_sm, int sms) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9f;
    const int grid = sms * ctas_per_sm;
    for (int r = 0; r < 6; ++r) {
        cudaEventRecord(a);
        k_ldg<UNROLL><<<grid, 256>>>(reinterpret_cast<const int4*>(d), bytes / 16, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r) best = ms < best ? ms : best;
    }
    printf("ldg unroll=%d ctas/sm=%d: %.1f GB/s (%s)\n", UNROLL, ctas_per_sm, bytes / best / 1e6,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t bytes = (int64_t)4 << 30;
    uint8_t* d;
    int* sink;
    cudaMalloc(&d, bytes);
    cudaMalloc(&sink, 4);
    cudaMemset(d, 1, bytes);
    for (int64_t mb : {100, 200, 400, 600, 800, 1600}) {  // fixed cost per launch: t = a + bytes / BW
        printf("size %lld MB: ", (long long)mb);
        run_bulk<16384, 4>(d, mb << 20, sink, 2, sms);
    }
    run_bulk<16384, 4>(d, bytes, sink, 2, sms);
    run_bulk<16384, 6>(d, bytes, sink, 2, sms);
    run_bulk<16384, 8>(d, bytes, sink, 1, sms);
    run_bulk<16384, 12>(d, bytes, sink, 1, sms);
    run_bulk<32768, 3>(d, bytes, sink, 2, sms);
    run_bulk<32768, 6>(d, bytes, sink, 1, sms);
    run_bulk<8192, 8>(d, bytes, sink, 2, sms);
    run_bulk<8192, 4>(d, bytes, sink, 4, sms);
    run_bulk<65536, 3>(d, bytes, sink, 1, sms);
    run_ldg<4>(d, bytes, sink, 4, sms);
    run_ldg<8>(d, bytes, sink, 4, sms);
    run_ldg<8>(d, bytes, sink, 8, sms);
    run_ldg<16>(d, bytes, sink, 4, sms);
    return 0;
}
