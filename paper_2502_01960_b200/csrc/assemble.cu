// K2 — request KV assembly (assemble_linked_cache, proj/src/linker.cpp:260-314).
//
// One launch gathers every cached chunk of a request into the request's [L][T][H][D]
// cache at its new offsets. HBM-bound: each destination row is one CTA iteration; the
// chunk lookup is done once per row (chunk descriptors staged in shared memory), then
// the row streams through as 16-byte vectors (2 K + 2 V vectors in flight per thread,
// L1 no-allocate loads, evict-first stores). Under Rerotate the K pairs are rotated by
// the chunk's constant position delta with a per-chunk (cos, sin) table computed on the
// host in double exactly like rerotate_key (proj/src/model.cpp:64-83) and staged in
// shared memory; the rotation itself is the reference's unfused float expression, so
// the result is bit-identical. AsStored is a pure copy: bit-exact. Rows no chunk covers
// are zero-filled (the reference's zero-initialised Dummy slots, tensor.h:20-23).
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace mpicb {

constexpr int kMaxAsmChunks = 256;  // chunks are sorted by destination row (plan_assembly)

template <typename T, int N>
struct alignas(sizeof(T) * N >= 16 ? 16 : sizeof(T) * N) Vec {
    T v[N];
};

template <typename T, int N>
__device__ __forceinline__ void load_vec(const T* p, float (&f)[N]) {
    if constexpr (sizeof(T) * N >= 16) {
        constexpr int P = sizeof(T) * N / 16;
#pragma unroll
        for (int q = 0; q < P; ++q) {
            uint4 raw;
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(raw.x), "=r"(raw.y), "=r"(raw.z), "=r"(raw.w)
                         : "l"(reinterpret_cast<const char*>(p) + 16 * q));
            const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
            for (int k = 0; k < N / P; ++k) f[q * (N / P) + k] = to_f32<T>(e[k]);
        }
    } else {
        const Vec<T, N> r = *reinterpret_cast<const Vec<T, N>*>(p);
#pragma unroll
        for (int k = 0; k < N; ++k) f[k] = to_f32<T>(r.v[k]);
    }
}

template <typename T, int N>
__device__ __forceinline__ void store_vec(T* p, const float (&f)[N]) {
    if constexpr (sizeof(T) * N >= 16) {
        constexpr int P = sizeof(T) * N / 16;
#pragma unroll
        for (int q = 0; q < P; ++q) {
            uint4 raw;
            T* e = reinterpret_cast<T*>(&raw);
#pragma unroll
            for (int k = 0; k < N / P; ++k) e[k] = from_f32<T>(f[q * (N / P) + k]);
            asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(reinterpret_cast<char*>(p) + 16 * q),
                         "r"(raw.x), "r"(raw.y), "r"(raw.z), "r"(raw.w)
                         : "memory");
        }
    } else {
        Vec<T, N> r;
#pragma unroll
        for (int k = 0; k < N; ++k) r.v[k] = from_f32<T>(f[k]);
        *reinterpret_cast<Vec<T, N>*>(p) = r;
    }
}

template <typename TS, typename TD, int VEC>
__global__ void __launch_bounds__(256) assemble_kernel(const AsmChunk* __restrict__ chunks,
                                                       uint32_t n_chunks,
                                                       const float2* __restrict__ tables,
                                                       uint32_t n_tables, TD* __restrict__ dk,
                                                       TD* __restrict__ dv, uint32_t L, uint32_t T,
                                                       uint32_t H, uint32_t D, int zero_gaps,
                                                       uint32_t src_l0, const uint8_t* __restrict__ skip_blk) {
    extern __shared__ float2 s_tab[];
    __shared__ AsmChunk s_chunks[kMaxAsmChunks];
    const uint32_t half_d = D >> 1, h = H * D, nvec = h / VEC;
    for (uint32_t i = threadIdx.x; i < n_chunks; i += blockDim.x) s_chunks[i] = chunks[i];
    for (uint32_t i = threadIdx.x; i < n_tables * half_d; i += blockDim.x) s_tab[i] = tables[i];
    __syncthreads();

    const uint64_t units = (uint64_t)L * T;
    for (uint64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const uint32_t l = (uint32_t)(u / T), r = (uint32_t)(u % T);
        if (skip_blk && skip_blk[r >> 7]) continue;  // linked inside attention (AttnLink)
        TD* kd = dk + u * h;
        TD* vd = dv + u * h;
        // the last chunk starting at or before r (chunks ascend by destination row and do
        // not overlap), if r falls inside it
        uint32_t lo = 0, hi = n_chunks;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (s_chunks[mid].dst_row0 <= r) lo = mid + 1;
            else hi = mid;
        }
        const int c = lo > 0 && r < s_chunks[lo - 1].dst_row0 + s_chunks[lo - 1].rows ? (int)lo - 1 : -1;
        if (c < 0) {
            if (zero_gaps) {
                float z[VEC];
#pragma unroll
                for (int e = 0; e < VEC; ++e) z[e] = 0.0f;
                for (uint32_t v = threadIdx.x; v < nvec; v += blockDim.x) {
                    store_vec<TD, VEC>(kd + (size_t)v * VEC, z);
                    store_vec<TD, VEC>(vd + (size_t)v * VEC, z);
                }
            }
            continue;
        }
        const AsmChunk ch = s_chunks[c];
        const size_t soff = ((size_t)(src_l0 + l) * ch.src_tokens + ch.src_row0 + (r - ch.dst_row0)) * ch.src_ld +
                            ch.src_col0;
        const TS* ks = static_cast<const TS*>(ch.src_k) + soff;
        const TS* vs = static_cast<const TS*>(ch.src_v) + soff;
        const float2* tab = s_tab + (size_t)ch.table * half_d;
        for (uint32_t v0 = threadIdx.x; v0 < nvec; v0 += 2 * blockDim.x) {
            const uint32_t v1 = v0 + blockDim.x;
            const bool has1 = v1 < nvec;
            float k0[VEC], k1[VEC], w0[VEC], w1[VEC];
            load_vec<TS, VEC>(ks + (size_t)v0 * VEC, k0);
            load_vec<TS, VEC>(vs + (size_t)v0 * VEC, w0);
            if (has1) {
                load_vec<TS, VEC>(ks + (size_t)v1 * VEC, k1);
                load_vec<TS, VEC>(vs + (size_t)v1 * VEC, w1);
            }
            if (ch.rotate) {
#pragma unroll
                for (int e = 0; e < VEC; e += 2) {
                    const float2 cs0 = tab[((v0 * VEC + e) % D) >> 1];
                    rope_pair(k0[e], k0[e + 1], cs0.x, cs0.y);
                    if (has1) {
                        const float2 cs1 = tab[((v1 * VEC + e) % D) >> 1];
                        rope_pair(k1[e], k1[e + 1], cs1.x, cs1.y);
                    }
                }
            }
            store_vec<TD, VEC>(kd + (size_t)v0 * VEC, k0);
            store_vec<TD, VEC>(vd + (size_t)v0 * VEC, w0);
            if (has1) {
                store_vec<TD, VEC>(kd + (size_t)v1 * VEC, k1);
                store_vec<TD, VEC>(vd + (size_t)v1 * VEC, w1);
            }
        }
    }
}

template <typename TS, typename TD>
static void launch_asm_typed(const AsmChunk* d_chunks, uint32_t n_chunks, const float2* d_tables,
                             uint32_t n_tables, TD* dk, TD* dv, uint32_t L, uint32_t T, uint32_t H,
                             uint32_t D, int zero_gaps, uint32_t src_l0, const uint8_t* skip_blk, cudaStream_t s) {
    const uint32_t h = H * D;
    const uint64_t units = (uint64_t)L * T;
    const size_t smem = (size_t)n_tables * (D / 2) * sizeof(float2);
    static const uint32_t per_sm = [] {
        const char* e = getenv("MPIC_ASM_CTAS_PER_SM");  // diagnostics
        return e ? (uint32_t)atoi(e) : 8u;
    }();
    const uint32_t grid = (uint32_t)std::min<uint64_t>(units, (uint64_t)kNumSMs * per_sm);
    if (h % 8 == 0) {
        auto k = assemble_kernel<TS, TD, 8>;
        if (smem + sizeof(AsmChunk) * kMaxAsmChunks > 48 * 1024)
            MPIC_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k<<<grid, 256, smem, s>>>(d_chunks, n_chunks, d_tables, n_tables, dk, dv, L, T, H, D, zero_gaps, src_l0, skip_blk);
    } else {
        auto k = assemble_kernel<TS, TD, 2>;
        if (smem + sizeof(AsmChunk) * kMaxAsmChunks > 48 * 1024)
            MPIC_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k<<<grid, 256, smem, s>>>(d_chunks, n_chunks, d_tables, n_tables, dk, dv, L, T, H, D, zero_gaps, src_l0, skip_blk);
    }
    MPIC_LAUNCHED();
}

void launch_assemble(const AsmChunk* d_chunks, uint32_t n_chunks, const float2* d_tables,
                     uint32_t n_tables, mpic_dtype src_t, void* dst_k, void* dst_v,
                     mpic_dtype dst_t, uint32_t L, uint32_t T_dst, uint32_t H, uint32_t D,
                     int zero_gaps, cudaStream_t s, uint32_t src_l0, const uint8_t* skip_blk) {
    static const bool skip = getenv("MPIC_ASM_SKIP") != nullptr;  // diagnostics: timing without the copy
    if (skip) return;
    if (n_chunks > kMaxAsmChunks) {
        // more descriptors than one CTA stages (batched requests): one launch per group of
        // kMaxAsmChunks (each group a contiguous destination range, the descriptors being sorted
        // by destination row); only the first zero-fills the gaps — rows of later groups are
        // zeroed there and overwritten by their own launch, in stream order
        for (uint32_t g0 = 0; g0 < n_chunks; g0 += kMaxAsmChunks)
            launch_assemble(d_chunks + g0, std::min<uint32_t>(kMaxAsmChunks, n_chunks - g0), d_tables, n_tables, src_t,
                            dst_k, dst_v, dst_t, L, T_dst, H, D, g0 == 0 ? zero_gaps : 0, s, src_l0, skip_blk);
        return;
    }
    using bf = __nv_bfloat16;
    if (src_t == MPIC_F32 && dst_t == MPIC_F32)
        launch_asm_typed<float, float>(d_chunks, n_chunks, d_tables, n_tables, (float*)dst_k, (float*)dst_v, L, T_dst, H, D, zero_gaps, src_l0, skip_blk, s);
    else if (src_t == MPIC_F32 && dst_t == MPIC_BF16)
        launch_asm_typed<float, bf>(d_chunks, n_chunks, d_tables, n_tables, (bf*)dst_k, (bf*)dst_v, L, T_dst, H, D, zero_gaps, src_l0, skip_blk, s);
    else if (src_t == MPIC_BF16 && dst_t == MPIC_BF16)
        launch_asm_typed<bf, bf>(d_chunks, n_chunks, d_tables, n_tables, (bf*)dst_k, (bf*)dst_v, L, T_dst, H, D, zero_gaps, src_l0, skip_blk, s);
    else
        launch_asm_typed<bf, float>(d_chunks, n_chunks, d_tables, n_tables, (float*)dst_k, (float*)dst_v, L, T_dst, H, D, zero_gaps, src_l0, skip_blk, s);
}

// ---- weight synthesis (proj/include/mpic/rng.h:10-30, proj/src/model.cpp:28-36) -------
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

template <typename T>
__global__ void synth_kernel(uint64_t h1, size_t count, float scale, T* __restrict__ dst) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
         i += (size_t)gridDim.x * blockDim.x) {
        const uint64_t hv = mix64(h1 ^ (i + 0x9e3779b97f4a7c15ull));
        const uint32_t bits = (uint32_t)(hv >> 40);
        const float u = __fsub_rn(__fmul_rn((float)bits, 2.0f / 16777216.0f), 1.0f);
        dst[i] = from_f32<T>(__fmul_rn(u, scale));
    }
}

static uint64_t mix64_host(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

void launch_synth(uint64_t seed, uint64_t tag, uint32_t layer, size_t count, float scale,
                  void* dst, mpic_dtype dt, cudaStream_t s) {
    const uint64_t phi = 0x9e3779b97f4a7c15ull;
    const uint64_t stream = (tag << 32) | layer;
    const uint64_t h1 = mix64_host(mix64_host(seed + phi) ^ (stream + phi));
    if (dt == MPIC_F32) synth_kernel<float><<<kNumSMs * 8, 256, 0, s>>>(h1, count, scale, (float*)dst);
    else synth_kernel<__nv_bfloat16><<<kNumSMs * 8, 256, 0, s>>>(h1, count, scale, (__nv_bfloat16*)dst);
    MPIC_LAUNCHED();
}

template <typename T>
__global__ void synth_2d_kernel(uint64_t h1, uint32_t rows, uint32_t cols_total, uint32_t row0, uint32_t col0,
                                uint32_t ncols, float scale, T* __restrict__ dst) {
    const size_t count = (size_t)rows * ncols;
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < count; k += (size_t)gridDim.x * blockDim.x) {
        const size_t r = k / ncols, j = k % ncols;
        const size_t i = (row0 + r) * (size_t)cols_total + col0 + j;
        const uint64_t hv = mix64(h1 ^ (i + 0x9e3779b97f4a7c15ull));
        const uint32_t bits = (uint32_t)(hv >> 40);
        const float u = __fsub_rn(__fmul_rn((float)bits, 2.0f / 16777216.0f), 1.0f);
        dst[k] = from_f32<T>(__fmul_rn(u, scale));
    }
}

void launch_synth_2d(uint64_t seed, uint64_t tag, uint32_t layer, uint32_t rows, uint32_t cols_total,
                     uint32_t row0, uint32_t col0, uint32_t ncols, float scale, void* dst, mpic_dtype dt,
                     cudaStream_t s) {
    const uint64_t phi = 0x9e3779b97f4a7c15ull;
    const uint64_t stream = (tag << 32) | layer;
    const uint64_t h1 = mix64_host(mix64_host(seed + phi) ^ (stream + phi));
    if (dt == MPIC_F32)
        synth_2d_kernel<float><<<kNumSMs * 8, 256, 0, s>>>(h1, rows, cols_total, row0, col0, ncols, scale, (float*)dst);
    else
        synth_2d_kernel<__nv_bfloat16><<<kNumSMs * 8, 256, 0, s>>>(h1, rows, cols_total, row0, col0, ncols, scale,
                                                                   (__nv_bfloat16*)dst);
    MPIC_LAUNCHED();
}

__global__ void resid_add_kernel(float* __restrict__ x, const float* __restrict__ add, __nv_bfloat16* __restrict__ xb,
                                 size_t n4) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        float4 a = reinterpret_cast<float4*>(x)[i];
        const float4 b = reinterpret_cast<const float4*>(add)[i];
        a.x += b.x;
        a.y += b.y;
        a.z += b.z;
        a.w += b.w;
        reinterpret_cast<float4*>(x)[i] = a;
        __nv_bfloat162 lo = __floats2bfloat162_rn(a.x, a.y), hi = __floats2bfloat162_rn(a.z, a.w);
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t*>(&lo);
        pk.y = *reinterpret_cast<uint32_t*>(&hi);
        reinterpret_cast<uint2*>(xb)[i] = pk;
    }
}

void launch_resid_add(float* x, const float* add, __nv_bfloat16* xb, size_t n, cudaStream_t s) {
    MPIC_REQUIRE(n % 4 == 0, MPIC_ERR_VALIDATION, "resid_add needs n % 4 == 0");
    resid_add_kernel<<<kNumSMs * 4, 256, 0, s>>>(x, add, xb, n / 4);
    MPIC_LAUNCHED();
}

} // namespace mpicb
