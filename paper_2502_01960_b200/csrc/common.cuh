// Shared device/host helpers for the MPIC B200 kernels (sm_100a only).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "mpic_b200.h"

namespace mpicb {

// Error carrying an mpic_status; thrown inside the library, converted at the C ABI.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define MPIC_CUDA(call)                                                                    \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            throw ::mpicb::Error(MPIC_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
    } while (0)

#define MPIC_REQUIRE(cond, code, msg)                  \
    do {                                               \
        if (!(cond)) throw ::mpicb::Error(code, msg); \
    } while (0)

// Per-thread launch counter (reported as gpu_launches by the bench).
void note_launch(uint32_t n = 1);
#define MPIC_LAUNCHED() do { MPIC_CUDA(cudaGetLastError()); ::mpicb::note_launch(); } while (0)

constexpr int kNumSMs = 148;

__host__ __device__ inline size_t elt_size(mpic_dtype d) { return d == MPIC_BF16 ? 2 : 4; }

// Element load/store helpers templated over the storage type.
template <typename T> __device__ __forceinline__ float to_f32(T v);
template <> __device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) {
    return __bfloat162float(v);
}
template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
    return __float2bfloat16_rn(v);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// RoPE pair rotation exactly as the reference's float expression
// (proj/src/model.cpp:56-59): x0*c - x1*s, x0*s + x1*c, each product rounded, no FMA.
__device__ __forceinline__ void rope_pair(float& x0, float& x1, float c, float s) {
    const float a = __fsub_rn(__fmul_rn(x0, c), __fmul_rn(x1, s));
    const float b = __fadd_rn(__fmul_rn(x0, s), __fmul_rn(x1, c));
    x0 = a;
    x1 = b;
}

// GELU, tanh form, same constants and operation order as proj/src/model.cpp:85-87.
__device__ __forceinline__ float gelu_ref(float x) {
    const float inner = __fmul_rn(0.7978845608028654f,
                                  __fadd_rn(x, __fmul_rn(__fmul_rn(__fmul_rn(0.044715f, x), x), x)));
    return __fmul_rn(__fmul_rn(0.5f, x), __fadd_rn(1.0f, tanhf(inner)));
}

inline uint32_t ceil_div(uint32_t a, uint32_t b) { return (a + b - 1) / b; }

// Programmatic dependent launch of the layer-loop kernels (MPIC_PDL=0 disables it).
bool pdl_enabled();

} // namespace mpicb
