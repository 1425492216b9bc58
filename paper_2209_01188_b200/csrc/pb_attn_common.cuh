// Pieces of the paged-KV tensor-core attention kernels (pb_attn_mma.cu):
// constants, mma/ldmatrix wrappers, the hi/lo operand split and the stream-K
// unit walk.
#pragma once

#include "pb_async.cuh"
#include "pb_common.cuh"
#include "pb_span.h"

namespace pb {

constexpr int AM_SK = 64;    // keys per stage
constexpr int AM_ST = 3;     // stages in flight
constexpr int AM_WARPS = 4;  // compute warps, 16 keys each per stage
constexpr int AM_G = 8;      // queries per group
constexpr int AM_PT = 128;   // page-table window of the producer (pages)
constexpr int AM_MAXC = 16;  // max CTAs contributing to one (group, head): split workspace slots

__device__ __forceinline__ int kv_chunk_swz(int chunk, int slot) { return chunk ^ (slot & 7); }

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void mma_f16(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
    return (uint32_t)__half_as_ushort(__float2half_rn(lo)) | ((uint32_t)__half_as_ushort(__float2half_rn(hi)) << 16);
}
// hi/lo split of two floats into two f16x2 words
__device__ __forceinline__ void split_h2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
    const half h0 = __float2half_rn(x0), h1 = __float2half_rn(x1);
    hi = (uint32_t)__half_as_ushort(h0) | ((uint32_t)__half_as_ushort(h1) << 16);
    lo = pack_h2(x0 - __half2float(h0), x1 - __half2float(h1));
}

__device__ __forceinline__ void cons_bar() {  // the AM_WARPS compute warps only
    asm volatile("bar.sync 1, %0;" ::"n"(AM_WARPS * 32) : "memory");
}
template <int NW>
__device__ __forceinline__ void cons_bar_n() {  // NW compute warps
    asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
}

// Stream-K decomposition: the work units are (query group, head, 64-key
// stage), numbered group-major (unit_base[g] = first unit of group g, every
// head of group g has ns_g = (unit_base[g+1] - unit_base[g]) / H stages). CTA c
// of G owns units [c U / G, (c+1) U / G), so every CTA streams the same number
// of K/V bytes (no wave tail) whatever the head count and context length.
struct AmSeg {
    int g, h, i0, n;  // group, head, first stage, stages in this CTA
    int ns;           // stages of (g, h)
    int64_t a;        // first unit of (g, h)
};

__device__ __forceinline__ AmSeg am_seg(const AttnArgs& a, int64_t u, int64_t u1) {
    int lo = 0, hi = a.n_groups - 1;  // largest g with unit_base[g] <= u
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a.unit_base[mid] <= u) lo = mid;
        else hi = mid - 1;
    }
    AmSeg s;
    s.g = lo;
    const int64_t b0 = a.unit_base[lo];
    s.ns = (int)((a.unit_base[lo + 1] - b0) / a.H);
    const int64_t r = u - b0;
    s.h = (int)(r / s.ns);
    s.i0 = (int)(r % s.ns);
    s.a = b0 + (int64_t)s.h * s.ns;
    const int64_t left = u1 - u;
    s.n = left < (int64_t)(s.ns - s.i0) ? (int)left : s.ns - s.i0;
    return s;
}

__device__ __forceinline__ int am_owner(int64_t u, int G, int64_t U) { return (int)(((u + 1) * G - 1) / U); }

// ctx of query t0 + g (head h) from merged state (M, L, O) + the wo operand range
template <int DH>
__device__ __forceinline__ float am_final(const AttnArgs& a, int tok, int h, int e, float o, float L) {
    const float c = o / L;
    a.ctx[(int64_t)tok * a.d + h * DH + e] = c;
    return a.tokmax ? fabsf(c * a.s_next[h * DH + e]) : 0.f;
}

}  // namespace pb
