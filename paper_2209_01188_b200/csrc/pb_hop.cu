// Span-to-span hop over NVLink peer memory (SURVEY §8 a10 / e): the
// reference client relays every hop's int8 wire payload through itself
// (client.py:312-331); on one box, consecutive spans live on consecutive
// GPUs and the last kernel of span r (the wire quantizer, pb_codec.cu)
// stores the codes and scales straight into a mailbox slot in span r+1's
// HBM through a CUDA IPC mapping. A one-thread signal kernel then publishes
// the job's sequence number with a system-scope release; span r+1's stream
// runs a one-thread wait kernel (system-scope acquire, bounded spin) before
// the span step that dequantizes the slot. No host synchronisation and no
// NCCL call on the data path.
//
// Mailbox layout (one cudaMalloc per receiving rank, exported by IPC handle):
// u64 flags[PB_HOP_FLAGS], then the payload slots (layout chosen by the host).
#include <cstring>

#include "pb_common.cuh"

namespace pb {

__global__ void k_hop_wait(const uint64_t* flag, uint64_t seq, uint64_t timeout_ns) {
    if (threadIdx.x != 0) return;
    const uint64_t t0 = gtime();
    for (;;) {
        uint64_t v;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
        if (v >= seq) break;
        if (gtime() - t0 > timeout_ns) {
            printf("pb_hop_wait: no signal for job %llu after %llu ms (flag %llu)\n", (unsigned long long)seq,
                   (unsigned long long)(timeout_ns / 1000000), (unsigned long long)v);
            __trap();  // fail the stream loudly instead of hanging the GPU
        }
        __nanosleep(256);
    }
}

__global__ void k_hop_signal(uint64_t* flag, uint64_t seq) {
    // the payload was written by earlier kernels of this stream (complete);
    // the system-scope fence + release orders them before the flag for the peer
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(seq) : "memory");
}

}  // namespace pb

using namespace pb;

extern "C" {

int pb_hop_alloc(int64_t bytes, int32_t device, void** d_ptr, void* h_handle) {
    PB_REQUIRE(d_ptr && h_handle && bytes > 0, PB_ERR_BAD_REQUEST, "null argument");
    PB_CHECK_CUDA(cudaSetDevice(device));
    void* p = nullptr;
    PB_CHECK_CUDA(cudaMalloc(&p, (size_t)bytes));
    PB_CHECK_CUDA(cudaMemset(p, 0, (size_t)bytes));
    cudaIpcMemHandle_t h;
    PB_CHECK_CUDA(cudaIpcGetMemHandle(&h, p));
    std::memcpy(h_handle, &h, sizeof(h));
    *d_ptr = p;
    return PB_OK;
}

int pb_hop_free(void* d_ptr) {
    PB_CHECK_CUDA(cudaFree(d_ptr));
    return PB_OK;
}

int pb_hop_open(const void* h_handle, int32_t device, void** d_ptr) {
    PB_REQUIRE(d_ptr && h_handle, PB_ERR_BAD_REQUEST, "null argument");
    PB_CHECK_CUDA(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, h_handle, sizeof(h));
    PB_CHECK_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return PB_OK;
}

int pb_hop_close(void* d_ptr) {
    PB_CHECK_CUDA(cudaIpcCloseMemHandle(d_ptr));
    return PB_OK;
}

int pb_hop_wait(const uint64_t* d_flag, uint64_t seq, int64_t timeout_ms, void* stream) {
    PB_REQUIRE(d_flag, PB_ERR_BAD_REQUEST, "null flag");
    k_hop_wait<<<1, 32, 0, (cudaStream_t)stream>>>(d_flag, seq, (uint64_t)timeout_ms * 1000000ull);
    return launch_check("hop_wait");
}

int pb_hop_signal(uint64_t* d_peer_flag, uint64_t seq, void* stream) {
    PB_REQUIRE(d_peer_flag, PB_ERR_BAD_REQUEST, "null flag");
    k_hop_signal<<<1, 1, 0, (cudaStream_t)stream>>>(d_peer_flag, seq);
    return launch_check("hop_signal");
}

}  // extern "C"
