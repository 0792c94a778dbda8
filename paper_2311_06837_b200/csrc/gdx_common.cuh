// gdx_common.cuh -- shared plumbing for libgdx: status/error reporting, launch
// accounting, the keyed SplitMix64 stream on device (rng.hpp:11-61) and the
// split-bf16 representation used by the tcgen05 GEMM.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "gdx.h"

namespace gdx {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
void note_launch(uint64_t n = 1);

// Checks the launch that was just issued; turns CUDA errors into GDX_INTERNAL.
int check_launch(const char* what);

#define GDX_REQUIRE(cond, code, msg)                      \
    do {                                                  \
        if (!(cond)) return ::gdx::fail((code), (msg));   \
    } while (0)

#define GDX_CUDA(call)                                                              \
    do {                                                                            \
        cudaError_t _e = (call);                                                    \
        if (_e != cudaSuccess)                                                      \
            return ::gdx::fail(GDX_INTERNAL, std::string(#call) + ": " +            \
                                                 cudaGetErrorString(_e));           \
    } while (0)

// SM count of the calling thread's current device (cached per device): grid caps
// and persistent grids are sized from it, never from a hard-coded 148.
int device_sms();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel).
int ensure_smem_attr(const void* kernel, int bytes);

inline cudaStream_t as_cuda(gdx_stream s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- keyed SplitMix64 (rng.hpp) -------------------------------------------
constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;

__host__ __device__ __forceinline__ uint64_t finalize64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
// rng.hpp:11-16
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) { return finalize64(x + kGamma); }
// rng.hpp:20-24: stream state after construction
__host__ __device__ __forceinline__ uint64_t keyed_state(uint64_t seed, uint64_t k1, uint64_t k2) {
    uint64_t s = mix64(seed);
    s = mix64(s ^ (k1 + kGamma));
    return mix64(s ^ (k2 + 0xc2b2ae3d27d4eb4fULL));
}
// Draw i (0-based) of a stream with state s0: jump-ahead of next_u64 (rng.hpp:26-32).
__host__ __device__ __forceinline__ uint64_t draw_at(uint64_t s0, uint64_t i) {
    return finalize64(s0 + (i + 1) * kGamma);
}
// rng.hpp:41-44 Lemire reduction
__device__ __forceinline__ uint64_t below(uint64_t x, uint64_t n) { return __umul64hi(x, n); }
// rng.hpp:35-37
__host__ __device__ __forceinline__ double to_unit(uint64_t x) {
    return static_cast<double>(x >> 11) * 0x1.0p-53;
}

// ---- split bf16 --------------------------------------------------------------
__device__ __forceinline__ uint16_t f2bf_rn(float x) {
    uint32_t u = __float_as_uint(x);
    if ((u & 0x7f800000u) == 0x7f800000u) return static_cast<uint16_t>((u >> 16) | ((u & 0xffff) ? 0x40 : 0));
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}
__device__ __forceinline__ float bf2f(uint16_t h) { return __uint_as_float(static_cast<uint32_t>(h) << 16); }
__device__ __forceinline__ void split_bf16(float x, uint16_t& hi, uint16_t& lo) {
    hi = f2bf_rn(x);
    lo = f2bf_rn(x - bf2f(hi));
}

// ---- packed-24 rows (aggregate.cu): fp32 rounded to nearest-even at bit 8, stored as
// the high 16 bits (u16 plane) and the next 8 bits (u8 plane) --------------------------
__device__ __forceinline__ void pack24(float x, uint16_t& hi, uint8_t& lo) {
    uint32_t u = __float_as_uint(x);
    if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x7fu + ((u >> 8) & 1u)) & 0xffffff00u;  // RNE at bit 8
    hi = static_cast<uint16_t>(u >> 16);
    lo = static_cast<uint8_t>(u >> 8);
}
__device__ __forceinline__ float unpack24(uint16_t hi, uint8_t lo) {
    return __uint_as_float((static_cast<uint32_t>(hi) << 16) | (static_cast<uint32_t>(lo) << 8));
}
// 16 values -> 32 bytes of high plane (two 16-byte words) + 16 bytes of low plane
__device__ __forceinline__ void pack24x16(const float* v, uint4& h0, uint4& h1, uint4& l) {
    uint32_t hw[8], lw[4];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        uint16_t a, b;
        uint8_t la, lb;
        pack24(v[2 * j], a, la);
        pack24(v[2 * j + 1], b, lb);
        hw[j] = static_cast<uint32_t>(a) | (static_cast<uint32_t>(b) << 16);
        if (j % 2 == 0) lw[j / 2] = static_cast<uint32_t>(la) | (static_cast<uint32_t>(lb) << 8);
        else lw[j / 2] |= (static_cast<uint32_t>(la) << 16) | (static_cast<uint32_t>(lb) << 24);
    }
    h0 = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    h1 = make_uint4(hw[4], hw[5], hw[6], hw[7]);
    l = make_uint4(lw[0], lw[1], lw[2], lw[3]);
}

}  // namespace gdx
