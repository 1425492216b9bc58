// Shared helpers for the sm_100a kernels and the C-ABI layer.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <utility>
#include <string>

#include "../../include/petals_b200.h"

namespace pb {

void set_error(const std::string& msg);

#define PB_CHECK_CUDA(expr)                                                                     \
    do {                                                                                        \
        cudaError_t _e = (expr);                                                                \
        if (_e != cudaSuccess) {                                                                \
            ::pb::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e) + " at " +       \
                            __FILE__ + ":" + std::to_string(__LINE__));                         \
            return PB_ERR_GENERIC;                                                              \
        }                                                                                       \
    } while (0)

#define PB_REQUIRE(cond, code, msg)                  \
    do {                                             \
        if (!(cond)) {                               \
            ::pb::set_error(std::string(msg));       \
            return (code);                           \
        }                                            \
    } while (0)

constexpr int PB_MAX_DEVICES = 64;

// Per-device launch setup (shared-memory opt-in, occupancy, SM count):
// cudaFuncSetAttribute applies to the current device's context only, so a
// process driving several GPUs configures each one. `slot[dev]` caches an
// int (0 = not yet); init(dev) returns the value (> 0) or a negative error.
template <typename F>
inline int per_device(int* slot, F&& init) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= PB_MAX_DEVICES) {
        set_error("per_device: bad current device");
        return -1;
    }
    if (slot[dev] > 0) return slot[dev];
    const int v = init(dev);
    if (v > 0) slot[dev] = v;
    return v;
}

inline int sm_count() {
    static int slot[PB_MAX_DEVICES] = {};
    return per_device(slot, [](int dev) {
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        return sms > 0 ? sms : -1;
    });
}

inline int launch_check(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string("launch ") + what + ": " + cudaGetErrorString(e));
        return PB_ERR_GENERIC;
    }
    return PB_OK;
}

static inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
static inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// ---------------------------------------------------------------- device helpers

// Warp index the compiler can prove warp-uniform (a lane-0 broadcast): code
// under `if (warp == w)` is then known to be converged, so shuffles there
// compile to the plain SHFL instead of BRA.DIV + the collective fallback.
__device__ __forceinline__ int warp_uniform_id() { return __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0); }

// Warp reductions reconverge the warp first (__syncwarp): after divergent
// code the compiler's shuffle otherwise takes its non-converged path, traced
// at ~1.5-3 us per reduction on the operand writer's critical path.
__device__ __forceinline__ float warp_max(float v) {
    __syncwarp();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
    __syncwarp();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
    __syncwarp();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// 128-bit streaming load that bypasses L1 allocation (weights are read once).
__device__ __forceinline__ int4 ld_stream_v4(const void* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// Round-half-away-from-zero of the EXACT quotient a/s for a >= 0, s >= 2^-125,
// returned as a non-negative integer (not clamped). The f32 quotient is a
// candidate within one unit; two fma residuals a - (m +- 1/2) s (exact sign:
// single rounding of an exactly representable-or-larger value) settle it.
// This equals the reference's round_half_away(f64(x)/f64(s)) (quant.py:52):
// for 24-bit x and s the exact quotient is either a half-integer or at least
// 2^-32 relative away from one, far beyond f64's 2^-53 rounding.
__device__ __forceinline__ int exact_round_away_pos(float a, float s) {
    float q = __fdiv_rn(a, s);
    float m = floorf(q + 0.5f);
    if (m > 200.f) return 200;  // clamp region: any value > 127 is fine
    if (fmaf(-(m + 0.5f), s, a) >= 0.f) m += 1.f;
    else if (m > 0.f && fmaf(-(m - 0.5f), s, a) < 0.f) m -= 1.f;
    return (int)m;
}

// code for x given the block's f32 scale s and absmax (quant.py:45-53 semantics,
// including the degenerate absmax>0, scale==0 underflow case: x/0 -> +-inf ->
// clip +-127, 0/0 -> NaN -> 0).
__device__ __forceinline__ int8_t wire_code(float x, float s, float amax) {
    if (s == 0.f) {
        if (amax == 0.f || x == 0.f) return 0;
        return x > 0.f ? (int8_t)127 : (int8_t)-127;
    }
    float a = fabsf(x);
    int m;
    if (s < 2.3509887e-38f) {  // s < 2^-125: the half-ulp residual may underflow, use f64
        double qd = (double)a / (double)s;
        double f = floor(qd + 0.5);
        m = f > 200.0 ? 200 : (int)f;
    } else {
        m = exact_round_away_pos(a, s);
    }
    m = m > 127 ? 127 : m;
    return (int8_t)(x < 0.f ? -m : m);
}

// Diagnostics (pb_trace_set): per-CTA globaltimer stamps of the decode
// kernels, TRACE_WORDS u64 per CTA, written only when the launch got a trace region.
__device__ __forceinline__ uint64_t gtime() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t smid() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}
constexpr int TRACE_WORDS = 16;  // per CTA: entry, released, first stage, end, SM id, kernel-specific
__device__ __forceinline__ void trace_stamp(uint64_t* tr, int cta, int i) {
    if (tr) {
        tr[cta * TRACE_WORDS + i] = gtime();  // i = 5..7: kernel-specific extra stamps
        if (i == 0) tr[cta * TRACE_WORDS + 4] = smid();
    }
}
// host: the next region of the trace buffer for a launch of `ctas` CTAs (or nullptr)
uint64_t* trace_region(int kind, int ctas);
enum TraceKind { TR_GEMV = 0, TR_ATTN = 1, TR_FRAG = 2 };

// Programmatic dependent launch (PDL): kernels of the decode chain are launched
// with cudaLaunchAttributeProgrammaticStreamSerialization, may start while the
// previous kernel drains, and must execute pdl_wait() before touching anything
// the previous kernels wrote (every such kernel calls it, so the chain stays
// transitively ordered). pdl_trigger() lets the next kernel launch early.
__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

template <typename... KArgs, typename... Args>
inline int launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                      Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    static const int pdl_on = [] {
        const char* e = getenv("PB_NO_PDL");
        return (e && *e == '1') ? 0 : 1;
    }();
    cfg.attrs = attr;
    cfg.numAttrs = pdl_on;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
    if (e != cudaSuccess) {
        set_error(std::string("cudaLaunchKernelEx: ") + cudaGetErrorString(e));
        return PB_ERR_GENERIC;
    }
    return PB_OK;
}

// SplitMix64 word i of the stream keyed by `key` (model.py:36-44: state =
// key + i*gamma, i >= 1) mapped to f32 in [-0.05, 0.05) (model.py:54-57).
__device__ __forceinline__ float gen_weight(uint64_t key, uint64_t i1) {
    uint64_t z = key + i1 * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1E4B21D5ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z = z ^ (z >> 31);
    double u = (double)(z >> 11) * 1.1102230246251565e-16;  // 2^-53, exact
    return __double2float_rn(__dmul_rn(__dadd_rn(u, -0.5), 0.1));
}

}  // namespace pb
