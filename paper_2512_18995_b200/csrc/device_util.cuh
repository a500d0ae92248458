// Small device helpers shared by the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace qsv::dev {

template <typename T> struct Vec2;
template <> struct Vec2<float> { using type = float2; };
template <> struct Vec2<double> { using type = double2; };

template <typename V> __device__ __forceinline__ V cmul(V a, V b) {
    V r;
    r.x = a.x * b.x - a.y * b.y;
    r.y = a.x * b.y + a.y * b.x;
    return r;
}
template <typename V> __device__ __forceinline__ V cfma(V a, V b, V acc) { // acc + a*b
    acc.x += a.x * b.x - a.y * b.y;
    acc.y += a.x * b.y + a.y * b.x;
    return acc;
}

// XOR-swizzle of a tile-local amplitude index into its shared-memory slot so
// that lanes walking any tile bit spread over the 8 sixteen-byte columns of a
// 128-byte bank row. Bijective inside the tile (only the low bits change).
template <typename V> __device__ __forceinline__ int swz(int u);
template <> __device__ __forceinline__ int swz<double2>(int u) {
    const int f = (u >> 3) ^ (u >> 6) ^ (u >> 9) ^ (u >> 12);
    return u ^ (f & 7);
}
template <> __device__ __forceinline__ int swz<float2>(int u) {
    const int w = u >> 1; // 16-byte unit = 2 amplitudes, kept adjacent
    const int f = (w >> 3) ^ (w >> 6) ^ (w >> 9) ^ (w >> 12);
    return ((w ^ (f & 7)) << 1) | (u & 1);
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void st_cs16(void *gmem, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};\n" ::"l"(gmem), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    return x;
}

} // namespace qsv::dev
