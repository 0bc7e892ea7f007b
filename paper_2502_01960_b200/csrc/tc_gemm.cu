// K3/K5/K6/K7 for feature counts that are not a multiple of 256 (the pair GEMM's feature
// block, tc_pgemm.cu, which takes every N % 256 == 0 shape), plus the shared host helpers
// (tensor-map cache, tc_gemm_supported, launch_gemm_tc dispatch).
//
//   out[t][f] = sum_k X[t][k] * W[f][k]      (y = x . W^T, proj/src/linker.cpp:64-128)
//
// Token-major 1-CTA kernels: UMMA M = 128 TOKENS (TMEM lane = token row), N = 64/128/256
// FEATURES; one wave of (feature tile x token tile) CTAs when that fills the SMs
// (tc_gemm_tok_kernel), else a persistent stream-K walk over the (tile, k-block) list with
// deterministic in-order partial fix-up (tc_gemm_sk_kernel). Covered by
// tests/test_gpu_kernels.py (N = 128, 384, 768, 1024 with K up to 4096).
//
//   warp 0     TMA producer (SWIZZLE_128B boxes)
//   warp 1     TMEM allocator + tcgen05.mma issuer (kind::f16, fp32 accum)
//   warps 2-5  epilogue: tcgen05.ld of the accumulator, fused RoPE+scatter into the KV
//              cache (QKV), GELU (W1), residual add (Wo/W2); one token row per thread, so
//              stores are 16-byte vectors and RoPE pairs sit in adjacent registers.
// (Round 1's swap-AB 1-CTA and 2-CTA variants, superseded by tc_pgemm.cu and reachable only
// through a diagnostics switch, are retired.)
#include <cstdlib>
#include <mutex>
#include <tuple>
#include <unordered_map>

#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace mpicb {

constexpr uint32_t kTcThreads = 192;
constexpr uint32_t kWTileBytes = 128 * 64 * 2;  // 16 KB
constexpr uint32_t kXBoxRows = 128;
constexpr uint32_t kXBoxBytes = kXBoxRows * 64 * 2;  // 16 KB

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&v);
}

// ---- token-major GEMM (the production path) ---------------------------------------------
// UMMA M = 128 TOKENS (TMEM lane = token row), N = bn FEATURES (<= 256). Each epilogue
// thread owns one token row and a run of consecutive features, so every epilogue store
// is a 16-byte vector (the swap-AB kernels above issue one scalar store per element), RoPE
// pairs sit in adjacent registers, and the KV scatter row is one index per thread.
struct TokArgs {
    uint32_t M, N, K;
    uint32_t bn;        // features per CTA (64, 128 or 256)
    uint32_t kblocks;   // 64-wide K blocks in total
    uint32_t split;     // K split (blockIdx.z), uneven ranges allowed
    uint32_t stages;
    uint32_t tmem_cols;
    EpiParams ep;
};

__device__ __forceinline__ void store_bf16x32(__nv_bfloat16* dst, const float (&v)[32]) {
#pragma unroll
    for (uint32_t w = 0; w < 4; ++w) {
        uint4 q;
        q.x = pack_bf16x2(v[8 * w + 0], v[8 * w + 1]);
        q.y = pack_bf16x2(v[8 * w + 2], v[8 * w + 3]);
        q.z = pack_bf16x2(v[8 * w + 4], v[8 * w + 5]);
        q.w = pack_bf16x2(v[8 * w + 6], v[8 * w + 7]);
        reinterpret_cast<uint4*>(dst)[w] = q;
    }
}

__device__ __forceinline__ void tok_epilogue_chunk(const EpiParams& ep, uint32_t t, uint32_t f0,
                                                   float (&v)[32]) {
    switch (ep.mode) {
        case EPI_QKV: {
            // linker.cpp:64-78 — q/k rotated at rope_pos[t], k/v scattered to kv[kv_rows[t]]
            const uint32_t h = ep.hidden, part = f0 / h, c = f0 - part * h;
            if (part < 2) {
                const float4* cs4 = reinterpret_cast<const float4*>(
                    ep.rope + (size_t)__ldg(ep.rope_pos + t) * (ep.head_dim >> 1) + ((c % ep.head_dim) >> 1));
#pragma unroll
                for (uint32_t i = 0; i < 8; ++i) {
                    const float4 cs = __ldg(cs4 + i);  // (cos, sin) of pairs 2i, 2i+1
                    rope_pair(v[4 * i + 0], v[4 * i + 1], cs.x, cs.y);
                    rope_pair(v[4 * i + 2], v[4 * i + 3], cs.z, cs.w);
                }
            }
            __nv_bfloat16* dst = part == 0 ? static_cast<__nv_bfloat16*>(ep.q) + (size_t)t * h + c
                                           : static_cast<__nv_bfloat16*>(part == 1 ? ep.kv_k : ep.kv_v) +
                                                 (size_t)__ldg(ep.kv_rows + t) * h + c;
            store_bf16x32(dst, v);
            break;
        }
        case EPI_RESID: {
            if (ep.split_k > 1) {
                float4* pp = reinterpret_cast<float4*>(ep.partial + ((size_t)blockIdx.z * ep.rows_total + t) * ep.ldx + f0);
#pragma unroll
                for (uint32_t i = 0; i < 8; ++i) pp[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
            } else {
                float4* xp = reinterpret_cast<float4*>(ep.x + (size_t)t * ep.ldx + f0);
#pragma unroll
                for (uint32_t i = 0; i < 8; ++i) {
                    float4 a = xp[i];
                    a.x += v[4 * i];
                    a.y += v[4 * i + 1];
                    a.z += v[4 * i + 2];
                    a.w += v[4 * i + 3];
                    xp[i] = a;
                    v[4 * i] = a.x;
                    v[4 * i + 1] = a.y;
                    v[4 * i + 2] = a.z;
                    v[4 * i + 3] = a.w;
                }
                if (ep.xb) store_bf16x32(ep.xb + (size_t)t * ep.ldx + f0, v);
            }
            break;
        }
        case EPI_GELU:
#pragma unroll
            for (uint32_t i = 0; i < 32; ++i) v[i] = gelu_ref(v[i]);
            store_bf16x32(static_cast<__nv_bfloat16*>(ep.out) + (size_t)t * ep.ldo + f0, v);
            break;
        case EPI_STORE_F32: {
            float4* o = reinterpret_cast<float4*>(static_cast<float*>(ep.out) + (size_t)t * ep.ldo + f0);
#pragma unroll
            for (uint32_t i = 0; i < 8; ++i) o[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
            break;
        }
        default:
            store_bf16x32(static_cast<__nv_bfloat16*>(ep.out) + (size_t)t * ep.ldo + f0, v);
    }
}

__global__ void __launch_bounds__(kTcThreads, 1)
    tc_gemm_tok_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                       const TokArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t w_bytes = a.bn * 128;
    const uint32_t stage_bytes = kXBoxBytes + w_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.stages * stage_bytes);
    uint64_t* empty = full + a.stages;
    uint64_t* tmem_full = empty + a.stages;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_full + 1);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t n0 = blockIdx.x * a.bn, t0 = blockIdx.y * 128;
    const uint32_t kb0 = blockIdx.z * a.kblocks / a.split;
    const uint32_t kb1 = (blockIdx.z + 1) * a.kblocks / a.split;

    if (warp == 0 && lane == 0) {
        tc::tma_prefetch_desc(&tmX);
        tc::tma_prefetch_desc(&tmW);
        for (uint32_t s = 0; s < a.stages; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        tc::mbar_init(tmem_full, 1);
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc(tmem_holder, a.tmem_cols);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol_w = tc::policy_evict_first();  // weights stream through once
            const uint64_t pol_x = tc::policy_evict_last();   // token tiles are re-read
            for (uint32_t kb = kb0, i = 0; kb < kb1; ++kb, ++i) {
                const uint32_t s = i % a.stages, ph = (i / a.stages) & 1;
                tc::mbar_wait(&empty[s], ph ^ 1);
                tc::mbar_arrive_expect_tx(&full[s], stage_bytes);
                uint8_t* st = smem + s * stage_bytes;
                tc::tma_load_2d_hint(st, &tmX, &full[s], (int)(kb * 64), (int)t0, pol_x);
                tc::tma_load_2d_hint(st + kXBoxBytes, &tmW, &full[s], (int)(kb * 64), (int)n0, pol_w);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // warp-uniform MMA issue: lane 0 polls, one elected lane issues from uniform registers
        {
            const uint32_t idesc = tc::idesc_bf16(128, a.bn);
            for (uint32_t kb = kb0, i = 0; kb < kb1; ++kb, ++i) {
                const uint32_t s = i % a.stages, ph = (i / a.stages) & 1;
                if (lane == 0) tc::mbar_wait(&full[s], ph);
                __syncwarp();
                tc::tc_fence_after();
                const uint32_t x_base = tc::smem_u32(smem + s * stage_bytes);
                const uint32_t w_base = x_base + kXBoxBytes;
                if (tc::elect_one_sync()) {
#pragma unroll
                    for (uint32_t kk = 0; kk < 4; ++kk)
                        tc::mma_bf16(tmem_base, tc::desc_k_sw128(x_base + kk * 32), tc::desc_k_sw128(w_base + kk * 32),
                                     idesc, (i > 0 || kk > 0) ? 1u : 0u);
                    tc::mma_commit(&empty[s]);
                }
            }
            if (tc::elect_one_sync()) tc::mma_commit(tmem_full);
        }
        __syncwarp();
    } else {
        const uint32_t q = warp & 3;
        const uint32_t t = t0 + q * 32 + lane;
        tc::mbar_wait(tmem_full, 0);
        tc::tc_fence_after();
        for (uint32_t c = 0; c < a.bn; c += 32) {
            uint32_t r[32];
            tc::tmem_ld32(tmem_base + ((q * 32u) << 16) + c, r);
            tc::tmem_ld_wait();
            if (t < a.M) {
                float v[32];
#pragma unroll
                for (uint32_t i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
                tok_epilogue_chunk(a.ep, t, n0 + c, v);
            }
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (warp == 1) tc::tmem_dealloc(tmem_base, a.tmem_cols);
}


// ---- stream-K persistent GEMM (the production path) ----------------------------------------
// One CTA per SM walks a contiguous range of the (tile, k-block) work list, so every SM
// gets the same number of k-blocks whatever the tile count (W1 at m=330 has 192 tiles of
// 128 tokens x 256 features: 1.3 waves as a plain grid). Tiles are ordered m-fastest, so the
// CTAs running concurrently share weight tiles in L2. A tile cut between CTAs is finished by
// the CTA that owns its first k-block (it reaches it last); the others publish fp32
// partials in their per-CTA slot and raise an epoch flag. The owner adds the partials in
// CTA order (deterministic) and runs the fused epilogue. TMEM holds two accumulators so the
// epilogue of one segment overlaps the MMAs of the next.
struct SkArgs {
    uint32_t M, N, K;
    uint32_t bn, mt;        // feature tile, number of 128-token tiles
    uint32_t kblocks;       // per tile
    uint64_t work;          // tiles * kblocks
    uint32_t ctas;          // persistent CTAs
    uint32_t stages;
    float* partial;         // [ctas][2 segments][128][bn] fp32
    uint32_t* counters;     // [tiles] arrivals per split tile
    EpiParams ep;
};

__device__ __forceinline__ uint32_t sk_cta_of(uint64_t x, uint64_t work, uint32_t ctas) {
    // largest c with floor(c*work/ctas) <= x
    return (uint32_t)(((x + 1) * ctas + work - 1) / work) - 1;
}

__global__ void __launch_bounds__(kTcThreads, 1)
    tc_gemm_sk_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                      const SkArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t stage_bytes = kXBoxBytes + a.bn * 128;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.stages * stage_bytes);
    uint64_t* empty = full + a.stages;
    uint64_t* acc_full = empty + a.stages;   // [2]
    uint64_t* acc_empty = acc_full + 2;      // [2]
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(acc_empty + 2);

    __shared__ uint32_t s_last;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t c = blockIdx.x;
    const uint64_t u_begin = (uint64_t)c * a.work / a.ctas, u_end = (uint64_t)(c + 1) * a.work / a.ctas;

    if (warp == 0 && lane == 0) {
        tc::tma_prefetch_desc(&tmX);
        tc::tma_prefetch_desc(&tmW);
        for (uint32_t s = 0; s < a.stages; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&acc_full[i], 1);
            tc::mbar_init(&acc_empty[i], 128);
        }
        tc::fence_barrier_init();
    }
    const uint32_t tmem_cols = 2 * a.bn < 32 ? 32 : 2 * a.bn;
    if (warp == 1) tc::tmem_alloc(tmem_holder, tmem_cols);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol_w = tc::policy_evict_first();
            const uint64_t pol_x = tc::policy_evict_last();
            uint32_t i = 0;
            for (uint64_t u = u_begin; u < u_end; ++u, ++i) {
                const uint32_t tile = (uint32_t)(u / a.kblocks), kb = (uint32_t)(u % a.kblocks);
                const uint32_t t0 = (tile % a.mt) * 128, n0 = (tile / a.mt) * a.bn;
                const uint32_t s = i % a.stages, ph = (i / a.stages) & 1;
                tc::mbar_wait(&empty[s], ph ^ 1);
                tc::mbar_arrive_expect_tx(&full[s], stage_bytes);
                uint8_t* st = smem + s * stage_bytes;
                tc::tma_load_2d_hint(st, &tmX, &full[s], (int)(kb * 64), (int)t0, pol_x);
                tc::tma_load_2d_hint(st + kXBoxBytes, &tmW, &full[s], (int)(kb * 64), (int)n0, pol_w);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // warp-uniform MMA issue: lane 0 polls, one elected lane issues from uniform registers
        {
            const uint32_t idesc = tc::idesc_bf16(128, a.bn);
            uint32_t i = 0, seg = 0;
            uint64_t u = u_begin;
            while (u < u_end) {
                const uint32_t kb_begin = (uint32_t)(u % a.kblocks);
                const uint64_t seg_end = u_end < u - kb_begin + a.kblocks ? u_end : u - kb_begin + a.kblocks;
                const uint32_t buf = seg & 1;
                if (lane == 0) tc::mbar_wait(&acc_empty[buf], ((seg >> 1) & 1) ^ 1);
                __syncwarp();
                tc::tc_fence_after();
                const uint32_t d = tmem_base + buf * a.bn;
                for (; u < seg_end; ++u, ++i) {
                    const uint32_t s = i % a.stages, ph = (i / a.stages) & 1;
                    if (lane == 0) tc::mbar_wait(&full[s], ph);
                    __syncwarp();
                    tc::tc_fence_after();
                    const uint32_t x_base = tc::smem_u32(smem + s * stage_bytes);
                    const uint32_t w_base = x_base + kXBoxBytes;
                    const bool first = (u % a.kblocks) == kb_begin;
                    if (tc::elect_one_sync()) {
#pragma unroll
                        for (uint32_t kk = 0; kk < 4; ++kk)
                            tc::mma_bf16(d, tc::desc_k_sw128(x_base + kk * 32), tc::desc_k_sw128(w_base + kk * 32),
                                         idesc, (!first || kk > 0) ? 1u : 0u);
                        tc::mma_commit(&empty[s]);
                    }
                }
                if (tc::elect_one_sync()) tc::mma_commit(&acc_full[buf]);
                ++seg;
            }
        }
        __syncwarp();
    } else {
        const uint32_t q = warp & 3;
        const uint32_t row = q * 32 + lane;
        uint32_t seg = 0;
        uint64_t u = u_begin;
        while (u < u_end) {
            const uint32_t tile = (uint32_t)(u / a.kblocks), kb_begin = (uint32_t)(u % a.kblocks);
            const uint64_t tile_end = (uint64_t)(tile + 1) * a.kblocks;
            const uint64_t seg_end = u_end < tile_end ? u_end : tile_end;
            const bool whole = kb_begin == 0 && seg_end == tile_end;
            const bool owner = kb_begin == 0;
            const uint32_t t0 = (tile % a.mt) * 128, n0 = (tile / a.mt) * a.bn;
            const uint32_t t = t0 + row;
            const uint32_t buf = seg & 1;
            tc::mbar_wait(&acc_full[buf], (seg >> 1) & 1);
            tc::tc_fence_after();
            const uint32_t d = tmem_base + buf * a.bn + ((q * 32u) << 16);
            (void)owner;
            if (whole) {
                for (uint32_t cc = 0; cc < a.bn; cc += 32) {
                    uint32_t r[32];
                    tc::tmem_ld32(d + cc, r);
                    tc::tmem_ld_wait();
                    float v[32];
#pragma unroll
                    for (uint32_t i2 = 0; i2 < 32; ++i2) v[i2] = __uint_as_float(r[i2]);
                    if (t < a.M) tok_epilogue_chunk(a.ep, t, n0 + cc, v);
                }
            } else {
                // Split tile: publish this segment's partial, then the LAST segment to arrive
                // (tile counter) sums all partials in CTA order and runs the epilogue. Nobody
                // waits on another CTA, so co-residency is not required.
                // slot layout [bn/4 float4 columns][128 rows]: a warp's access is 512 contiguous bytes
                const uint32_t my_slot = (u == u_begin) ? 0u : 1u;
                float4* mine = reinterpret_cast<float4*>(a.partial + ((size_t)c * 2 + my_slot) * 128 * a.bn) + row;
                for (uint32_t cc = 0; cc < a.bn; cc += 32) {
                    uint32_t r[32];
                    tc::tmem_ld32(d + cc, r);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (uint32_t i2 = 0; i2 < 8; ++i2)
                        __stcg(mine + (size_t)(cc / 4 + i2) * 128,
                               make_float4(__uint_as_float(r[4 * i2]), __uint_as_float(r[4 * i2 + 1]),
                                           __uint_as_float(r[4 * i2 + 2]), __uint_as_float(r[4 * i2 + 3])));
                }
                __threadfence();
                tc::named_bar_sync(1, 128);
                const uint32_t c0 = sk_cta_of((uint64_t)tile * a.kblocks, a.work, a.ctas);
                const uint32_t c1 = sk_cta_of(tile_end - 1, a.work, a.ctas);
                if (row == 0) {
                    const uint32_t old = atomicAdd(a.counters + tile, 1u);
                    const bool last = old == c1 - c0;
                    if (last) a.counters[tile] = 0;  // ready for the next launch
                    __threadfence();
                    s_last = last ? 1u : 0u;
                }
                tc::named_bar_sync(1, 128);
                if (s_last) {
                    const uint64_t c0_begin = (uint64_t)c0 * a.work / a.ctas;
                    for (uint32_t cc = 0; cc < a.bn; cc += 32) {
                        float v[32];
#pragma unroll
                        for (uint32_t i2 = 0; i2 < 32; ++i2) v[i2] = 0.0f;
                        for (uint32_t p = c0; p <= c1; ++p) {
                            // tile == CTA p's first segment unless p == c0 started earlier
                            const uint32_t slot = (p == c0 && c0_begin < (uint64_t)tile * a.kblocks) ? 1u : 0u;
                            const float4* src = reinterpret_cast<const float4*>(
                                a.partial + ((size_t)p * 2 + slot) * 128 * a.bn) + row;
#pragma unroll
                            for (uint32_t i2 = 0; i2 < 8; ++i2) {
                                const float4 w = __ldcg(src + (size_t)(cc / 4 + i2) * 128);
                                v[4 * i2] += w.x;
                                v[4 * i2 + 1] += w.y;
                                v[4 * i2 + 2] += w.z;
                                v[4 * i2 + 3] += w.w;
                            }
                        }
                        if (t < a.M) tok_epilogue_chunk(a.ep, t, n0 + cc, v);
                    }
                }
            }
            tc::tc_fence_before();
            tc::mbar_arrive(&acc_empty[buf]);
            u = seg_end;
            ++seg;
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (warp == 1) tc::tmem_dealloc(tmem_base, tmem_cols);
}

// x += sum_z partial[z]; xb = bf16(x) — the deterministic split-K reduction, fused with
// the cast that produces the next GEMM's bf16 operand.
__global__ void __launch_bounds__(256) resid_reduce_kernel(const float* __restrict__ partial,
                                                           uint32_t split, size_t plane,
                                                           float* __restrict__ x,
                                                           __nv_bfloat16* __restrict__ xb,
                                                           size_t n4) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
         i += (size_t)gridDim.x * blockDim.x) {
        float4 acc = reinterpret_cast<const float4*>(x)[i];
        for (uint32_t z = 0; z < split; ++z) {
            const float4 p = __ldcs(reinterpret_cast<const float4*>(partial + z * plane) + i);
            acc.x += p.x;
            acc.y += p.y;
            acc.z += p.z;
            acc.w += p.w;
        }
        reinterpret_cast<float4*>(x)[i] = acc;
        if (xb) {
            __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x, acc.y);
            __nv_bfloat162 hi = __floats2bfloat162_rn(acc.z, acc.w);
            uint2 pk;
            pk.x = *reinterpret_cast<uint32_t*>(&lo);
            pk.y = *reinterpret_cast<uint32_t*>(&hi);
            reinterpret_cast<uint2*>(xb)[i] = pk;
        }
    }
}

// ---- host side ----------------------------------------------------------------------
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    MPIC_REQUIRE(fn, MPIC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

struct MapKey {
    const void* ptr;
    uint64_t inner, outer;
    uint32_t box_inner, box_outer;
    bool operator==(const MapKey& o) const {
        return ptr == o.ptr && inner == o.inner && outer == o.outer && box_inner == o.box_inner &&
               box_outer == o.box_outer;
    }
};
struct MapKeyHash {
    size_t operator()(const MapKey& k) const {
        return std::hash<const void*>()(k.ptr) ^ (k.inner * 1315423911u) ^ (k.outer << 17) ^
               (k.box_outer << 7);
    }
};

}  // namespace

// 2-D bf16 tensor map, row-major [outer][inner], SWIZZLE_128B box {box_inner, box_outer}.
// Maps are cached by (pointer, shape, box); buffers are long-lived (weights, workspace).
namespace {
CUtensorMap make_tmap_2d(const void* ptr, uint64_t inner, uint64_t outer, uint32_t box_inner, uint32_t box_outer,
                         bool f32) {
    static std::mutex mu;
    static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
    const MapKey key{ptr, inner | (f32 ? 1ull << 63 : 0ull), outer, box_inner, box_outer};
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    CUtensorMap m;
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {inner * (f32 ? 4 : 2)};
    const cuuint32_t box[2] = {box_inner, box_outer};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                   const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    MPIC_REQUIRE(r == CUDA_SUCCESS, MPIC_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    std::lock_guard<std::mutex> lk(mu);
    cache.emplace(key, m);
    return m;
}
}  // namespace

CUtensorMap make_tmap_bf16(const void* ptr, uint64_t inner, uint64_t outer, uint32_t box_inner,
                           uint32_t box_outer) {
    return make_tmap_2d(ptr, inner, outer, box_inner, box_outer, false);
}
// fp32 [outer][inner] (the 3xTF32 GEMM operands): box_inner = 32 elements = one 128-B row
CUtensorMap make_tmap_f32(const void* ptr, uint64_t inner, uint64_t outer, uint32_t box_inner,
                          uint32_t box_outer) {
    return make_tmap_2d(ptr, inner, outer, box_inner, box_outer, true);
}

bool tc_gemm_supported(uint32_t M, uint32_t N, uint32_t K) {
    return M > 0 && N % 64 == 0 && K % 64 == 0 && K >= 64;
}

namespace {
// Token-major launch: picks the feature tile (bn), K split and CTAs/SM for best SM fill.
void launch_tok(const __nv_bfloat16* A, const __nv_bfloat16* W, uint32_t M, uint32_t N, uint32_t K,
                const EpiParams& ep_in, cudaStream_t s) {
    const uint32_t mt = ceil_div(M, 128), kblocks = K / 64;
    const bool can_split = ep_in.mode == EPI_RESID && ep_in.partial != nullptr;
    double best = -1.0;
    uint32_t bn = 64, split = 1;
    for (uint32_t b : {256u, 128u, 64u}) {
        if (N % b) continue;
        for (uint32_t sp = 1; sp <= (can_split ? 4u : 1u); ++sp) {
            if (kblocks / sp < 8 && sp > 1) break;
            if (sp > 1 && (size_t)sp * M * N > ep_in.partial_cap) break;
            const uint32_t ctas = (N / b) * mt * sp;
            const uint32_t per_sm = ctas > (uint32_t)kNumSMs ? 2 : 1;
            const uint32_t slots = kNumSMs * per_sm;
            const double waves = std::ceil((double)ctas / slots);
            // fill of the busiest wave, discounted for small tiles (more operand re-reads)
            // and for split-K (partial traffic)
            double score = (double)ctas / (slots * waves) * (b == 256 ? 1.0 : b == 128 ? 0.93 : 0.8) *
                           (1.0 - 0.03 * (sp - 1));
            if (score > best + 1e-9) {
                best = score;
                bn = b;
                split = sp;
            }
        }
    }
    TokArgs a{};
    a.M = M;
    a.N = N;
    a.K = K;
    a.bn = bn;
    a.kblocks = kblocks;
    a.split = split;
    const uint32_t ctas = (N / bn) * mt * split;
    const uint32_t per_sm = ctas > (uint32_t)kNumSMs ? 2 : 1;
    const uint32_t stage_bytes = kXBoxBytes + bn * 128;
    const uint32_t budget = (227 * 1024) / per_sm - 1024 - 256;
    a.stages = std::min<uint32_t>(8, budget / stage_bytes);
    MPIC_REQUIRE(a.stages >= 2, MPIC_ERR_VALIDATION, "tc gemm tile does not fit shared memory");
    a.tmem_cols = std::max(32u, bn);
    a.ep = ep_in;
    a.ep.split_k = split;
    a.ep.rows_total = M;
    const CUtensorMap tmX = make_tmap_bf16(A, K, M, 64, 128);
    const CUtensorMap tmW = make_tmap_bf16(W, K, N, 64, bn);
    const size_t smem = (size_t)a.stages * stage_bytes + 1024 + (2 * a.stages + 1) * 8 + 16;
    static std::once_flag once;
    std::call_once(once, [] {
        MPIC_CUDA(cudaFuncSetAttribute(tc_gemm_tok_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    });
    tc_gemm_tok_kernel<<<dim3(N / bn, mt, split), kTcThreads, smem, s>>>(tmX, tmW, a);
    MPIC_LAUNCHED();
    if (split > 1) {
        const size_t n4 = (size_t)M * N / 4;
        resid_reduce_kernel<<<kNumSMs * 4, 256, 0, s>>>(ep_in.partial, split, (size_t)M * N, ep_in.x,
                                                         ep_in.xb, n4);
        MPIC_LAUNCHED();
    }
}
}  // namespace


namespace {
struct SkWorkspace {
    float* partial = nullptr;
    uint32_t* counters = nullptr;
    size_t cap = 0, tiles_cap = 0;
};

void launch_sk(const __nv_bfloat16* A, const __nv_bfloat16* W, uint32_t M, uint32_t N, uint32_t K,
               const EpiParams& ep_in, cudaStream_t s) {
    static std::mutex mu;
    static SkWorkspace ws[16];
    int dev = 0;
    MPIC_CUDA(cudaGetDevice(&dev));
    SkArgs a{};
    a.M = M;
    a.N = N;
    a.K = K;
    a.bn = N % 256 == 0 ? 256 : N % 128 == 0 ? 128 : 64;
    a.mt = ceil_div(M, 128);
    a.kblocks = K / 64;
    a.work = (uint64_t)(N / a.bn) * a.mt * a.kblocks;
    a.ctas = (uint32_t)std::min<uint64_t>(kNumSMs, a.work);
    const uint32_t stage_bytes = kXBoxBytes + a.bn * 128;
    const uint32_t budget = 227 * 1024 - 1024 - 512;
    a.stages = std::min<uint32_t>(8, budget / stage_bytes);
    a.ep = ep_in;
    a.ep.split_k = 1;
    {
        std::lock_guard<std::mutex> lk(mu);
        // NOTE: one scratch per device; concurrent launches on different streams of the
        // same device would share it (the library serialises a request on one stream).
        SkWorkspace& w = ws[dev & 15];
        const size_t need = (size_t)kNumSMs * 2 * 128 * 256;
        const size_t tiles = (size_t)(N / a.bn) * a.mt;
        if (w.cap < need) {
            MPIC_CUDA(cudaMalloc(&w.partial, need * sizeof(float)));
            w.cap = need;
        }
        if (w.tiles_cap < tiles) {
            if (w.counters) MPIC_CUDA(cudaFree(w.counters));
            w.tiles_cap = std::max<size_t>(tiles, 4096);
            MPIC_CUDA(cudaMalloc(&w.counters, w.tiles_cap * sizeof(uint32_t)));
            MPIC_CUDA(cudaMemset(w.counters, 0, w.tiles_cap * sizeof(uint32_t)));
        }
        a.partial = w.partial;
        a.counters = w.counters;
    }
    const CUtensorMap tmX = make_tmap_bf16(A, K, M, 64, 128);
    const CUtensorMap tmW = make_tmap_bf16(W, K, N, 64, a.bn);
    const size_t smem = (size_t)a.stages * stage_bytes + 1024 + (2 * a.stages + 4) * 8 + 16;
    static std::once_flag once;
    std::call_once(once, [] {
        MPIC_CUDA(cudaFuncSetAttribute(tc_gemm_sk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024 - 64));
    });
    tc_gemm_sk_kernel<<<a.ctas, kTcThreads, smem, s>>>(tmX, tmW, a);
    MPIC_LAUNCHED();
}
}  // namespace

void launch_gemm_tc(const __nv_bfloat16* A, uint32_t lda, const __nv_bfloat16* W, uint32_t M,
                    uint32_t N, uint32_t K, const EpiParams& ep_in, cudaStream_t s, bool w_blocked) {
    MPIC_REQUIRE(tc_gemm_supported(M, N, K) && lda == K, MPIC_ERR_VALIDATION, "unsupported tc gemm shape");
    static const char* variant = getenv("MPIC_GEMM_VARIANT");  // diagnostics: "tok", "sk"
    if (w_blocked || (!variant && pgemm_supported(M, N, K))) {
        launch_pgemm(A, W, M, N, K, ep_in, s, w_blocked);
        return;
    }
    // N % 256 != 0 (the pair GEMM's feature block): the token-major 1-CTA kernels
    MPIC_REQUIRE(ep_in.mode != EPI_QKV || (ep_in.head_dim % 32 == 0 && ep_in.hidden % 32 == 0),
                 MPIC_ERR_VALIDATION, "tc gemm QKV epilogue needs head_dim % 32 == 0");
    const uint32_t bn = N % 256 == 0 ? 256 : N % 128 == 0 ? 128 : 64;
    const uint32_t tiles = (N / bn) * ceil_div(M, 128);
    const bool one_wave = tiles <= (uint32_t)kNumSMs && tiles * 8 >= (uint32_t)kNumSMs * 7;
    if (variant && variant[0] == 't') launch_tok(A, W, M, N, K, ep_in, s);
    else if (variant && variant[0] == 's') launch_sk(A, W, M, N, K, ep_in, s);
    else if (one_wave) launch_tok(A, W, M, N, K, ep_in, s);
    else launch_sk(A, W, M, N, K, ep_in, s);
}

}  // namespace mpicb
