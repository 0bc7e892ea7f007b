// K3/K5/K6/K7 production GEMM — persistent CTA-pair (cta_group::2) swap-AB, data-parallel
// tiles with in-cluster split-K.
//
//   out[t][f] = sum_k X[t][k] * W[f][k]      (y = x . W^T, proj/src/linker.cpp:64-128)
//
// Shape regime of MPIC's selective pass: few token rows (m = 96 .. ~2000 recomputed rows)
// against large weights (h x h .. 4h x h). The UMMA M side is the WEIGHT: a CTA pair owns
// 256 output features (128 per CTA, one TMEM lane per feature) and the UMMA N side is a
// token GROUP of up to 512 tokens issued as one or two instructions of <= 256 columns,
// so padding costs at most 15 rows per piece and every weight tile is read from HBM once.
// Each CTA of the pair TMA-loads its 128 weight rows and HALF of the group's token rows;
// the leader issues tcgen05.mma.cta_group::2 over both shared memories: per k-block of
// 64 a CTA moves 16 KB + G*64 B for 2*128*G*64 FLOPs (G = 336: 147 FLOP per L2 byte,
// 1.7x the 1-CTA 128x256 tile).
//
// Scheduling. tile = (256-feature block, token group). A cluster of S pairs (2S CTAs)
// owns tiles c, c + C, c + 2C, ... (C clusters); pair s of the cluster computes the
// k-blocks [s*kb/S, (s+1)*kb/S) of each. S = 1 is plain data-parallel (QKV, W1: 48 / 64
// tiles). S = 2 or 4 is used when the tile count is small (Wo, W2 at h=4096: 16 tiles) and
// every cluster holds a single tile: the S partial accumulators are reduced through
// distributed shared memory — each CTA pushes the 32-token chunks it does not own into
// the owner's (now idle) stage buffers, and the owner sums the S contributions in split
// order (deterministic) before the fused epilogue. No partial ever goes to HBM/L2.
//
// Warp roles (320 threads per CTA):
//   warp 0     TMA producer (both CTAs), 4-8 stage smem ring
//   warp 1     TMEM allocator (pair) + MMA issuer (even CTA of the pair, one thread)
//   warps 2-9  epilogue (two warps per TMEM lane quarter, alternate 32-token chunks):
//              tcgen05.ld, thread <-> feature; fused RoPE + KV scatter (QKV), GELU (W1),
//              residual add + bf16 copy (Wo, W2). Stores are coalesced across lanes (32
//              consecutive features of one token row).
// TMEM holds two accumulators when the group fits 256 columns, so the epilogue of one
// tile overlaps the MMAs of the next; larger groups use one buffer.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <unordered_map>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"


namespace mpicb {

CUtensorMap make_tmap_bf16(const void* ptr, uint64_t inner, uint64_t outer, uint32_t box_inner,
                           uint32_t box_outer);
CUtensorMap make_tmap_f32(const void* ptr, uint64_t inner, uint64_t outer, uint32_t box_inner,
                          uint32_t box_outer);

namespace {

constexpr uint32_t kPgThreads = 320;  // producer, MMA, 8 epilogue warps
constexpr uint32_t kPgWBytes = 128 * 64 * 2;  // one CTA's weight rows per k-block (16 KB)
constexpr uint32_t kChunkBytes = 32 * 128 * 4;  // one 32-token x 128-feature fp32 chunk
constexpr uint32_t kNoStage = 0xffffffffu;
constexpr uint32_t kStageSlice = 4096;  // one epilogue warp's staging slice
constexpr uint32_t kEpiBars = 16;       // QKV side-input barriers: one per 32-token chunk of a group

struct PgArgs {
    uint32_t M, N, K;
    uint32_t P0, P1;     // token pieces of a group (P1 == 0: one piece)
    uint32_t G;          // tokens per group (P0 + P1)
    uint32_t ngroups;
    uint32_t kblocks;    // K / 64
    uint32_t tiles;      // (N / 256) * ngroups
    uint32_t S;          // pairs per cluster = K splits per tile
    uint32_t clusters;
    uint32_t stages;
    uint32_t stage_bytes;
    uint32_t sub_bytes;  // one k-block (64) of both operands; a stage holds kps of them
    uint32_t kps;
    uint32_t xoff1;      // byte offset of piece 1 in a stage's token region
    uint32_t nbuf;       // TMEM accumulators (1 or 2)
    uint32_t tmem_cols;
    uint32_t w_evict_first;
    uint32_t dbg;        // diagnostics: 1 skip epilogue, 2 skip X loads, 4 skip W loads, 8 skip MMA
    uint32_t stage_rope; // QKV: stage rope/kv_rows of the (single) group in the idle stage buffers
    uint32_t rows_off;   // byte offset of the staged kv_rows
    unsigned long long* ts;  // diagnostics (MPIC_PG_TS): CTA 0 entry / after prologue / MMAs
                             // issued / epilogue done / exit, %globaltimer ns
    uint32_t w_blocked;  // W stored as [N/128][K/64][128][64] tiles
    uint32_t pfd;        // L2 prefetch distance of the weight stream in k-blocks (0: off)
    uint32_t prologue_pf;  // prefetch the first k-blocks' weights into L2 before the PDL wait
    uint32_t stg_off;    // staged epilogue stores: byte offset of the 8 x 4 KB warp slices in the
                         // (then idle) stage ring, or kNoStage
    uint32_t w_early;    // weights of the first ring stages loaded before the PDL wait
    uint32_t kel;        // K elements per k-block (one 128-B operand row): 64 bf16, 32 fp32 (3xTF32)
    uint32_t wsub;       // weight bytes of a k-block: 16 KB, 32 KB with the 3xTF32 hi and lo tiles
    uint32_t xlo;        // 3xTF32: byte offset of the token rows' lo tile from their hi tile
    uint32_t segn;       // 3xTF32: stage iterations per accumulation segment (see the kernel)
    EpiParams ep;
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// GELU (tanh form, proj/src/model.cpp:85-87) with the hardware tanh: the result is rounded
// to bf16, whose 2^-8 step is coarser than tanh.approx's error (bf16 mode only; the fp32
// parity path uses the exact expression).
__device__ __forceinline__ float gelu_fast(float x) {
    float t;
    const float inner = 0.7978845608028654f * fmaf(0.044715f * x, x * x, x);
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(inner));
    return 0.5f * x * (1.0f + t);
}

// Fused epilogue of 32 consecutive tokens [tb, tb+32) of feature f (accumulators r);
// tokens at or beyond M (the group's end) are skipped. Lanes hold consecutive features,
// so every store instruction writes one contiguous run per token row. Specialised per
// mode (and for full chunks) so the per-element loops are branch-free.
// s_rows / s_rope: this group's kv_rows and (cos, sin) rows staged in shared memory
// (indexed from the group's first token tg), or null to read them from global memory.
// Staged stores (stg != null: this warp's 4 KB slice of the idle stage ring): the 32 tokens x
// 32 features of a chunk are transposed through shared memory so that each lane stores 16 B
// and one instruction covers 8 (bf16) or 4 (fp32) whole 64/128-B token-row segments instead
// of one — the direct form issues 32 narrow scattered stores per chunk, which bounds the
// epilogue tail.
__device__ __forceinline__ void stage_put_bf16(__nv_bfloat16* stg, uint32_t j, uint32_t lane, __nv_bfloat16 v) {
    stg[j * 32 + lane] = v;
}
// row-wise read-back: lane -> token 8i + lane/4, features (lane%4)*8 .. +8
__device__ __forceinline__ uint4 stage_get_bf16(const __nv_bfloat16* stg, uint32_t i, uint32_t lane) {
    return *reinterpret_cast<const uint4*>(stg + (i * 8 + (lane >> 2)) * 32 + (lane & 3) * 8);
}

// Transpose a warp's 32 tokens x 32 features accumulator chunk (lane = feature) into its
// staging slice as [token][32 features] fp32.
__device__ __forceinline__ void stage_put_f32(float* sf, uint32_t lane, const uint32_t (&r)[32]) {
#pragma unroll
    for (uint32_t j = 0; j < 32; ++j) sf[j * 32 + lane] = __uint_as_float(r[j]);
    __syncwarp();
}
__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
    return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
// Residual add of a transposed chunk (lane -> token 4i + lane/8, features 4*(lane%8) ..+4 of
// the warp's 32): x += v, xb = bf16(x). One instruction covers 4 whole 128-B x rows.
// `part(i)` returns the fp32 sum for read-back step i.
template <typename T>
__device__ __forceinline__ T to_out(float v);
template <>
__device__ __forceinline__ float to_out<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 to_out<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

template <class Part>
__device__ __forceinline__ void resid_rows(const EpiParams& ep, uint32_t n, uint32_t tb, uint32_t f0, uint32_t lane,
                                           Part part) {
    const uint32_t c = f0 + (lane & 7) * 4;
    // all x loads are issued before the first store (the compiler cannot hoist them past
    // stores to the same array)
    float4 v[8], xo[8];
#pragma unroll
    for (uint32_t i = 0; i < 8; ++i) {
        const uint32_t t = i * 4 + (lane >> 3);
        xo[i] = t < n && !(ep.dbg & 16) ? __ldcg(reinterpret_cast<const float4*>(ep.x + (size_t)(tb + t) * ep.ldx + c))
                      : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (uint32_t i = 0; i < 8; ++i) v[i] = part(i);
#pragma unroll
    for (uint32_t i = 0; i < 8; ++i) {
        const uint32_t t = i * 4 + (lane >> 3);
        if (t < n && !(ep.dbg & 32)) {
            const float4 nv = f4add(xo[i], v[i]);
            *reinterpret_cast<float4*>(ep.x + (size_t)(tb + t) * ep.ldx + c) = nv;
            if (ep.xb) {
                __nv_bfloat162 lo = __floats2bfloat162_rn(nv.x, nv.y), hi = __floats2bfloat162_rn(nv.z, nv.w);
                uint2 pk;
                pk.x = *reinterpret_cast<uint32_t*>(&lo);
                pk.y = *reinterpret_cast<uint32_t*>(&hi);
                *reinterpret_cast<uint2*>(ep.xb + (size_t)(tb + t) * ep.ldx + c) = pk;
            }
        }
    }
}

// F32 (3xTF32 fp32 mode): fp32 outputs (q, K/V cache rows, FFN activations) and the exact
// GELU, as the SIMT fp32 GEMM's epilogue (simt.cu epi_pair); direct stores only.
template <int MODE, bool F32 = false>
__device__ __forceinline__ void pg_epi(const EpiParams& ep, uint32_t M, uint32_t tb, uint32_t f, uint32_t lane,
                                       const uint32_t (&r)[32], const uint32_t* s_rows, const float2* s_rope,
                                       uint32_t tg, uint8_t* stg = nullptr) {
    using TO = typename std::conditional<F32, float, __nv_bfloat16>::type;
    const uint32_t n = min(32u, M - tb);  // valid tokens in this chunk
    if (!F32 && stg) {
        __nv_bfloat16* sb = reinterpret_cast<__nv_bfloat16*>(stg);
        const uint32_t f0 = f - lane;  // the warp's first feature
        if constexpr (MODE == EPI_RESID) {
            float* sf = reinterpret_cast<float*>(stg);
            stage_put_f32(sf, lane, r);
            resid_rows(ep, n, tb, f0, lane, [&](uint32_t i) {
                return *reinterpret_cast<const float4*>(sf + (i * 4 + (lane >> 3)) * 32 + (lane & 7) * 4);
            });
        } else if constexpr (MODE == EPI_STORE_F32) {
            float* sf = reinterpret_cast<float*>(stg);
#pragma unroll
            for (uint32_t j = 0; j < 32; ++j) sf[j * 32 + lane] = __uint_as_float(r[j]);
            __syncwarp();
            float* o = static_cast<float*>(ep.out) + f0 + (lane & 7) * 4;
#pragma unroll
            for (uint32_t i = 0; i < 8; ++i) {
                const uint32_t t = i * 4 + (lane >> 3);
                const float4 v = *reinterpret_cast<const float4*>(sf + t * 32 + (lane & 7) * 4);
                if (t < n) *reinterpret_cast<float4*>(o + (size_t)(tb + t) * ep.ldo) = v;
            }
        } else if constexpr (MODE == EPI_QKV) {
            // linker.cpp:64-78 — the chunk goes through the slice as fp32 [token][32 features];
            // each lane then owns 4 consecutive features (two interleaved RoPE pairs) of one
            // token per step: its (cos, sin) pairs are one 16-B load, the rotation needs no
            // shuffles, and the bf16 result is one 8-B store into q or the K/V cache row.
            const uint32_t h = ep.hidden, part = f0 / h, d0 = f0 - part * h;
            const uint32_t hd2 = ep.head_dim >> 1, c4 = (lane & 7) * 4;
            const uint32_t pr0 = ((d0 + c4) % ep.head_dim) >> 1;  // even (head_dim % 4 == 0)
            // every load of the chunk (cache rows and (cos, sin) staged in shared memory — the
            // staged QKV path is only used with both staged — and the transposed values) is
            // issued before its first global store, branch-free, with explicit shared accesses
            const uint32_t sf = tc::smem_u32(stg);
            const uint32_t srows = tc::smem_u32(s_rows) - tg * 4u;
            const uint32_t srope = tc::smem_u32(s_rope) + (pr0 - tg * hd2) * 8u;
            const bool rot = part < 2 && !(ep.dbg & 64);  // warp-uniform
            uint32_t rows[8];
            float4 cs[8];
#pragma unroll
            for (uint32_t i = 0; i < 8; ++i) {
                const uint32_t t = min(tb + i * 4 + (lane >> 3), M - 1);
                rows[i] = part == 0 ? t : tc::ld_shared_u32(srows + t * 4u);
                if (rot) cs[i] = tc::ld_shared_v4(srope + t * hd2 * 8u);
            }
#pragma unroll
            for (uint32_t j = 0; j < 32; ++j) tc::st_shared_f32(sf + (j * 32 + lane) * 4, __uint_as_float(r[j]));
            __syncwarp();
            float4 v[8];
#pragma unroll
            for (uint32_t i = 0; i < 8; ++i) v[i] = tc::ld_shared_v4(sf + ((i * 4 + (lane >> 3)) * 32 + c4) * 4);
            __nv_bfloat16* base = static_cast<__nv_bfloat16*>(part == 0 ? ep.q : part == 1 ? ep.kv_k : ep.kv_v) + d0 + c4;
#pragma unroll
            for (uint32_t i = 0; i < 8; ++i) {
                if (rot) {
                    rope_pair(v[i].x, v[i].y, cs[i].x, cs[i].y);
                    rope_pair(v[i].z, v[i].w, cs[i].z, cs[i].w);
                }
                if (i * 4 + (lane >> 3) < n && !(ep.dbg & 32)) {
                    const __nv_bfloat162 lo = __floats2bfloat162_rn(v[i].x, v[i].y), hi = __floats2bfloat162_rn(v[i].z, v[i].w);
                    uint2 pk;
                    pk.x = *reinterpret_cast<const uint32_t*>(&lo);
                    pk.y = *reinterpret_cast<const uint32_t*>(&hi);
                    *reinterpret_cast<uint2*>(base + (size_t)rows[i] * h) = pk;
                }
            }
        } else {  // EPI_STORE / EPI_GELU
#pragma unroll
            for (uint32_t j = 0; j < 32; ++j) {
                const float v = __uint_as_float(r[j]);
                stage_put_bf16(sb, j, lane, __float2bfloat16_rn(MODE == EPI_GELU ? gelu_fast(v) : v));
            }
            __syncwarp();
            __nv_bfloat16* o = static_cast<__nv_bfloat16*>(ep.out) + f0 + (lane & 3) * 8;
            uint4 v[4];  // all read back before the first store (see EPI_QKV)
#pragma unroll
            for (uint32_t i = 0; i < 4; ++i) v[i] = stage_get_bf16(sb, i, lane);
#pragma unroll
            for (uint32_t i = 0; i < 4; ++i) {
                const uint32_t t = i * 8 + (lane >> 2);
                if (t < n) *reinterpret_cast<uint4*>(o + (size_t)(tb + t) * ep.ldo) = v[i];
            }
        }
        __syncwarp();  // the slice is rewritten by the next chunk
        return;
    }
    if constexpr (MODE == EPI_QKV) {
        // linker.cpp:64-78 — q/k rotated at their position (interleaved pairs live on
        // adjacent lanes), k/v scattered to the cache row kv_rows[t]
        const uint32_t h = ep.hidden, part = f / h, d = f - part * h;
        const uint32_t hd2 = ep.head_dim >> 1, pr = (d % ep.head_dim) >> 1;
        TO* base = static_cast<TO*>(part == 0 ? ep.q : part == 1 ? ep.kv_k : ep.kv_v) + d;
        const bool odd = lane & 1;
        if (part == 2) {  // V: no rotation
#pragma unroll
            for (uint32_t j = 0; j < 32; ++j) {
                if (j >= n) continue;
                const uint32_t t = tb + j;
                const uint32_t row = s_rows ? s_rows[t - tg] : __ldg(ep.kv_rows + t);
                base[(size_t)row * h] = to_out<TO>(__uint_as_float(r[j]));
            }
            return;
        }
#pragma unroll
        for (uint32_t j0 = 0; j0 < 32; j0 += 16) {
            uint32_t row[16];
            float2 cs[16];
#pragma unroll
            for (uint32_t j = 0; j < 16; ++j) {
                const uint32_t t = min(tb + j0 + j, M - 1);
                if (s_rows) {
                    row[j] = part == 0 ? t : s_rows[t - tg];
                    cs[j] = s_rope[(t - tg) * hd2 + pr];
                } else {
                    row[j] = part == 0 ? t : __ldg(ep.kv_rows + t);
                    cs[j] = ep.rope_tok ? __ldg(ep.rope_tok + (size_t)t * hd2 + pr)
                                        : __ldg(ep.rope + (size_t)__ldg(ep.rope_pos + t) * hd2 + pr);
                }
            }
            TO o[16];
#pragma unroll
            for (uint32_t j = 0; j < 16; ++j) {
                const float val = __uint_as_float(r[j0 + j]);
                const float vp = __shfl_xor_sync(0xffffffffu, val, 1);
                float x0 = odd ? vp : val, x1 = odd ? val : vp;
                rope_pair(x0, x1, cs[j].x, cs[j].y);
                o[j] = to_out<TO>(odd ? x1 : x0);
            }
            if (j0 + 16 <= n) {
#pragma unroll
                for (uint32_t j = 0; j < 16; ++j) base[(size_t)row[j] * h] = o[j];
            } else {
#pragma unroll
                for (uint32_t j = 0; j < 16; ++j)
                    if (j0 + j < n) base[(size_t)row[j] * h] = o[j];
            }
        }
    } else if constexpr (MODE == EPI_RESID) {
        float* xp = ep.x + (size_t)tb * ep.ldx + f;
        __nv_bfloat16* xbp = ep.xb ? ep.xb + (size_t)tb * ep.ldx + f : nullptr;
        if (n == 32) {
            float xo[32];
#pragma unroll
            for (uint32_t j = 0; j < 32; ++j) xo[j] = __ldcg(xp + (size_t)j * ep.ldx);
#pragma unroll
            for (uint32_t j = 0; j < 32; ++j) {
                const float nv = xo[j] + __uint_as_float(r[j]);
                xp[(size_t)j * ep.ldx] = nv;
                if (xbp) xbp[(size_t)j * ep.ldx] = __float2bfloat16_rn(nv);
            }
        } else {
#pragma unroll
            for (uint32_t j = 0; j < 32; ++j) {
                if (j < n) {
                    const float nv = __ldcg(xp + (size_t)j * ep.ldx) + __uint_as_float(r[j]);
                    xp[(size_t)j * ep.ldx] = nv;
                    if (xbp) xbp[(size_t)j * ep.ldx] = __float2bfloat16_rn(nv);
                }
            }
        }
    } else if constexpr (MODE == EPI_GELU) {
        TO* o = static_cast<TO*>(ep.out) + (size_t)tb * ep.ldo + f;
#pragma unroll
        for (uint32_t j = 0; j < 32; ++j)
            if (j < n)
                o[(size_t)j * ep.ldo] = F32 ? to_out<TO>(gelu_ref(__uint_as_float(r[j])))
                                            : to_out<TO>(gelu_fast(__uint_as_float(r[j])));
    } else if constexpr (MODE == EPI_STORE_F32) {
        float* o = static_cast<float*>(ep.out) + (size_t)tb * ep.ldo + f;
#pragma unroll
        for (uint32_t j = 0; j < 32; ++j)
            if (j < n) o[(size_t)j * ep.ldo] = __uint_as_float(r[j]);
    } else {
        TO* o = static_cast<TO*>(ep.out) + (size_t)tb * ep.ldo + f;
#pragma unroll
        for (uint32_t j = 0; j < 32; ++j)
            if (j < n) o[(size_t)j * ep.ldo] = to_out<TO>(__uint_as_float(r[j]));
    }
}

// One instantiation per epilogue mode: the kernel's epilogue runs once, at the end, from a
// cold instruction cache, so each instantiation carries only its own (unrolled) epilogue.
// X3: the fp32 mode's 3xTF32 GEMM. Operands are pre-split into tf32-rounded hi and lo parts
// (x = hi + lo to ~2^-22, tf32_split_kernel), a k-block is 32 fp32 (one 128-B row, so the
// smem descriptors are the bf16 ones) and each K = 8 step issues lo*hi + hi*lo + hi*hi
// into the fp32 TMEM accumulator (lo*lo, ~2^-22 relative, is dropped).
template <int MODE, bool X3>
__global__ void __launch_bounds__(kPgThreads, 1)
    tc_pgemm_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX0,
                    const __grid_constant__ CUtensorMap tmX1, const __grid_constant__ CUtensorMap tmWl,
                    const __grid_constant__ CUtensorMap tmX0l, const __grid_constant__ CUtensorMap tmX1l,
                    const PgArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.stages * a.stage_bytes);
    uint64_t* empty = full + a.stages;
    uint64_t* acc_full = empty + a.stages;  // [2]
    uint64_t* acc_empty = acc_full + 2;     // [2], the even CTA's copy is the one used
    uint64_t* epi_bar = acc_empty + 2;      // [kEpiBars] epilogue side-input staging, one per 32-token chunk
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(epi_bar + kEpiBars);

    tc::pdl_trigger();
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = tc::cluster_ctarank();
    unsigned long long* ts = a.ts && blockIdx.x == 0 ? a.ts : nullptr;  // diagnostics
    if (ts && threadIdx.x == 0) ts[0] = gtimer();
    const uint32_t rank = crank & 1;          // CTA within the pair
    const uint32_t split = crank >> 1;        // pair within the cluster = K split
    const uint32_t cl = blockIdx.x / (2 * a.S);
    const uint32_t kb0 = split * a.kblocks / a.S, kb1 = (split + 1) * a.kblocks / a.S;
    const uint16_t pair_mask = (uint16_t)(0x3u << (2 * split));

    if (warp == 0 && lane == 0) {
        tc::tma_prefetch_desc(&tmW);
        tc::tma_prefetch_desc(&tmX0);
        tc::tma_prefetch_desc(&tmX1);
        if (X3) {
            tc::tma_prefetch_desc(&tmWl);
            tc::tma_prefetch_desc(&tmX0l);
            tc::tma_prefetch_desc(&tmX1l);
        }
        for (uint32_t s = 0; s < a.stages; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (uint32_t b = 0; b < 2; ++b) {
            tc::mbar_init(&acc_full[b], 1);
            tc::mbar_init(&acc_empty[b], 16);  // 8 epilogue warps x 2 CTAs
        }
        for (uint32_t i = 0; i < kEpiBars; ++i) tc::mbar_init(&epi_bar[i], 1);
        tc::fence_barrier_init();
    }
    if (warp == 0 && lane == 0 && cl < a.tiles && a.prologue_pf) {
        // weights do not depend on the previous kernel: start pulling this CTA's first
        // k-blocks into L2 before waiting for it
        const uint32_t fb = cl / a.ngroups, w_row = fb * 256 + (crank & 1) * 128;
        for (uint32_t kb = kb0; kb < min(kb1, kb0 + 2 * a.stages * a.kps); ++kb)
            tc::tma_prefetch_2d(&tmW, a.w_blocked ? 0 : (int)(kb * 64),
                                a.w_blocked ? (int)(((2 * fb + (crank & 1)) * a.kblocks + kb) * 128) : (int)w_row);
    }
    if (warp == 1) tc::tmem_alloc_pair(tmem_holder, a.tmem_cols);
    tc::tc_fence_before();
    tc::cluster_sync();
    tc::tc_fence_after();
    const uint32_t xbytes = (a.dbg & 2) ? 0u : a.sub_bytes - a.wsub;
    const uint32_t wbytes = (a.dbg & 4) ? 0u : a.wsub;
    const uint64_t pol_w = a.w_evict_first ? tc::policy_evict_first() : tc::policy_evict_last();
    const uint32_t leader_full = tc::mapa_shared(tc::smem_u32(full), crank & ~1u);
    // one k-block of weights (hi, and the lo tile in 3xTF32) of feature block fb into stage st
    auto load_w = [&](uint8_t* st, uint32_t bar, uint32_t fb, uint32_t kbj) {
        if (!wbytes) return;
        const int k = (int)(kbj * a.kel), w_row = (int)(fb * 256 + rank * 128);
        if (X3) tc::tma_load_2d_cg2(st + kPgWBytes, &tmWl, bar, k, w_row, pol_w);
        if (a.w_blocked)  // one contiguous 16 KB tile per box
            tc::tma_load_2d_cg2(st, &tmW, bar, 0, (int)(((2 * fb + rank) * a.kblocks + kbj) * 128), pol_w);
        else
            tc::tma_load_2d_cg2(st, &tmW, bar, k, w_row, pol_w);
    };
    // Weights do not depend on the previous kernel: the producer fills the weight half of the
    // first ring stages before waiting for it (their barriers expect the full stage), so after
    // the wait only the token rows (L2-resident activations) remain on the critical path.
    uint32_t early = 0;
    if (warp == 0 && lane == 0 && a.w_early && cl < a.tiles) {
        const uint32_t fb = cl / a.ngroups;
        for (uint32_t kb = kb0; kb < kb1 && early < a.stages; kb += a.kps, ++early) {
            const uint32_t nsub = min(a.kps, kb1 - kb);
            if (rank == 0) tc::mbar_arrive_expect_tx(&full[early], 2 * nsub * (xbytes + wbytes));
            for (uint32_t j = 0; j < nsub; ++j)
                load_w(smem + early * a.stage_bytes + j * a.sub_bytes, leader_full + early * 8, fb, kb + j);
        }
    }
    tc::pdl_wait();  // the previous kernel's outputs (this GEMM's X, its output buffers) are ready
    if (ts && threadIdx.x == 0) ts[1] = gtimer();
    const uint32_t tmem = *tmem_holder;

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol_x = tc::policy_evict_last();
            const int xr0 = (int)(rank * (a.P0 / 2)), xr1 = (int)(a.P0 + rank * (a.P1 / 2));
            long long pw = 0;
            const long long p0 = clock64();
            uint32_t s = 0, ph = 0, it = 0;
            for (uint32_t tile = cl; tile < a.tiles; tile += a.clusters) {
                const uint32_t fb = tile / a.ngroups, g = tile % a.ngroups;
                const int t0 = (int)(g * a.G);
                for (uint32_t kb = kb0; kb < kb1; kb += a.kps, ++it) {
                    const uint32_t nsub = min(a.kps, kb1 - kb);
                    const bool pre = it < early;  // weights already issued before the PDL wait
                    const long long w0 = ts ? clock64() : 0;
                    if (!pre) tc::mbar_wait(&empty[s], ph ^ 1);
                    if (ts) pw += clock64() - w0;
                    if (rank == 0 && !pre) tc::mbar_arrive_expect_tx(&full[s], 2 * nsub * (xbytes + wbytes));
                    const uint32_t bar = leader_full + s * 8;
                    for (uint32_t j = 0; j < nsub; ++j) {
                        uint8_t* st = smem + s * a.stage_bytes + j * a.sub_bytes;
                        const int k = (int)((kb + j) * a.kel);
                        if (!pre) load_w(st, bar, fb, kb + j);
                        if (a.pfd) {
                            // keep the weight stream pfd k-blocks ahead of the smem ring in L2
                            // (DRAM latency hidden without spending shared memory on it);
                            // crosses into this cluster's next tile
                            uint32_t kp = kb + j + a.pfd, fp = fb;
                            if (kp >= kb1 && tile + a.clusters < a.tiles) {
                                kp = kb0 + (kp - kb1);
                                fp = (tile + a.clusters) / a.ngroups;
                            }
                            if (kp < kb1 && (fp != fb || kp > kb + j))
                                tc::tma_prefetch_2d(&tmW, a.w_blocked ? 0 : (int)(kp * 64),
                                                    a.w_blocked ? (int)(((2 * fp + rank) * a.kblocks + kp) * 128)
                                                                : (int)(fp * 256 + rank * 128));
                        }
                        if (xbytes) tc::tma_load_2d_cg2(st + a.wsub, &tmX0, bar, k, t0 + xr0, pol_x);
                        if (xbytes && a.P1) tc::tma_load_2d_cg2(st + a.wsub + a.xoff1, &tmX1, bar, k, t0 + xr1, pol_x);
                        if (X3 && xbytes) {
                            tc::tma_load_2d_cg2(st + a.wsub + a.xlo, &tmX0l, bar, k, t0 + xr0, pol_x);
                            if (a.P1)
                                tc::tma_load_2d_cg2(st + a.wsub + a.xlo + a.xoff1, &tmX1l, bar, k, t0 + xr1, pol_x);
                        }
                    }
                    if (++s == a.stages) { s = 0; ph ^= 1; }
                }
            }
            if (ts) {
                ts[5] = pw;
                ts[6] = clock64() - p0;
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // MMA issue (even CTA of the pair). The whole warp runs the loop (warp-uniform, so
        // the descriptors live in uniform registers); lane 0 polls the barriers, one elected
        // lane issues each k-block's MMAs back to back. (A lone issuing thread wrapped every
        // tcgen05.mma in an elect/broadcast loop: ~15 instructions of issue overhead per MMA.)
        if (rank == 0 && X3) {
            // 3xTF32: the tile's k range is accumulated in segments of segn stages, alternating
            // between the two TMEM buffers; the epilogue warps drain each finished segment into
            // fp32 register sums (round to nearest). The tensor core truncates its fp32
            // accumulation toward zero at every instruction, so one chain over all of K biases
            // the result by ~K/16 ulp. Within a segment the small lo*hi and hi*lo products of
            // all its stages are issued first, while the accumulator is still small, and the
            // hi*hi products last: only those truncate a full-size partial sum.
            const uint32_t idesc0 = tc::idesc_tf32(256, a.P0);
            const uint32_t idesc1 = tc::idesc_tf32(256, a.P1 ? a.P1 : 16);
            uint32_t s = 0, ph = 0, seg = 0;
            const uint32_t nit = (kb1 - kb0 + a.kps - 1) / a.kps;
            for (uint32_t tile = cl; tile < a.tiles; tile += a.clusters) {
                for (uint32_t it0 = 0; it0 < nit; it0 += a.segn, ++seg) {
                    const uint32_t nst = min(a.segn, nit - it0);
                    const uint32_t b = seg & 1, d = tmem + b * a.G;
                    if (lane == 0) {
                        tc::mbar_wait_cluster(&acc_empty[b], ((seg >> 1) & 1) ^ 1);
                        uint32_t s2 = s, ph2 = ph;
                        for (uint32_t q = 0; q < nst; ++q) {
                            tc::mbar_wait(&full[s2], ph2);
                            if (++s2 == a.stages) { s2 = 0; ph2 ^= 1; }
                        }
                    }
                    __syncwarp();
                    tc::tc_fence_after();
                    if (tc::elect_one_sync()) {
                        bool first = true;
                        for (uint32_t pass = 0; pass < 2; ++pass) {
                            uint32_t s2 = s;
                            for (uint32_t q = 0; q < nst; ++q) {
                                const uint32_t nsub = min(a.kps, kb1 - (kb0 + (it0 + q) * a.kps));
                                for (uint32_t j = 0; j < nsub && !(a.dbg & 8); ++j) {
                                    const uint32_t w_base = tc::smem_u32(smem + s2 * a.stage_bytes + j * a.sub_bytes);
                                    const uint32_t x_base = w_base + a.wsub;
#pragma unroll
                                    for (uint32_t kk = 0; kk < 4; ++kk) {
                                        const uint64_t ahi = tc::desc_k_sw128(w_base + kk * 32);
                                        const uint64_t alo = tc::desc_k_sw128(w_base + kPgWBytes + kk * 32);
#pragma unroll
                                        for (uint32_t pc = 0; pc < 2; ++pc) {
                                            if (pc && !a.P1) break;
                                            const uint32_t xo = pc ? a.xoff1 : 0u, dd = pc ? d + a.P0 : d;
                                            const uint32_t id = pc ? idesc1 : idesc0;
                                            const uint64_t xh = tc::desc_k_sw128(x_base + xo + kk * 32);
                                            if (pass == 0) {
                                                tc::mma_tf32_pair(dd, alo, xh, id, first ? 0u : 1u);
                                                tc::mma_tf32_pair(dd, ahi, tc::desc_k_sw128(x_base + a.xlo + xo + kk * 32),
                                                                  id, 1u);
                                            } else {
                                                tc::mma_tf32_pair(dd, ahi, xh, id, 1u);
                                            }
                                        }
                                        first = false;
                                    }
                                }
                                if (++s2 == a.stages) s2 = 0;
                            }
                        }
                        uint32_t s2 = s;
                        for (uint32_t q = 0; q < nst; ++q) {
                            tc::mma_commit_pair_mcast(&empty[s2], pair_mask);
                            if (++s2 == a.stages) s2 = 0;
                        }
                        tc::mma_commit_pair_mcast(&acc_full[b], pair_mask);
                    }
                    __syncwarp();
                    for (uint32_t q = 0; q < nst; ++q)
                        if (++s == a.stages) { s = 0; ph ^= 1; }
                }
            }
        } else if (rank == 0) {
            const uint32_t idesc0 = tc::idesc_bf16(256, a.P0);
            const uint32_t idesc1 = tc::idesc_bf16(256, a.P1 ? a.P1 : 16);
            uint32_t item = 0, s = 0, ph = 0;
            long long mw = 0;
            const long long m0 = clock64();
            for (uint32_t tile = cl; tile < a.tiles; tile += a.clusters, ++item) {
                const uint32_t b = a.nbuf == 2 ? (item & 1) : 0u;
                const uint32_t use = a.nbuf == 2 ? (item >> 1) : item;
                if (lane == 0) tc::mbar_wait_cluster(&acc_empty[b], (use & 1) ^ 1);
                __syncwarp();
                tc::tc_fence_after();
                const uint32_t d = tmem + b * a.G;
                for (uint32_t kb = kb0; kb < kb1; kb += a.kps) {
                    const uint32_t nsub = min(a.kps, kb1 - kb);
                    const long long w0 = ts ? clock64() : 0;
                    if (lane == 0) tc::mbar_wait(&full[s], ph);
                    __syncwarp();
                    if (ts) mw += clock64() - w0;
                    tc::tc_fence_after();
                    if (tc::elect_one_sync()) {
                        for (uint32_t j = 0; j < nsub && !(a.dbg & 8); ++j) {
                            const uint32_t w_base = tc::smem_u32(smem + s * a.stage_bytes + j * a.sub_bytes);
                            const uint32_t x_base = w_base + a.wsub;
#pragma unroll
                            for (uint32_t kk = 0; kk < 4; ++kk) {
                                const uint64_t adesc = tc::desc_k_sw128(w_base + kk * 32);
                                const uint32_t acc = (kb + j > kb0 || kk > 0) ? 1u : 0u;
                                tc::mma_bf16_pair(d, adesc, tc::desc_k_sw128(x_base + kk * 32), idesc0, acc);
                                if (a.P1)
                                    tc::mma_bf16_pair(d + a.P0, adesc, tc::desc_k_sw128(x_base + a.xoff1 + kk * 32),
                                                      idesc1, acc);
                            }
                        }
                        tc::mma_commit_pair_mcast(&empty[s], pair_mask);
                    }
                    if (++s == a.stages) { s = 0; ph ^= 1; }
                }
                if (tc::elect_one_sync()) tc::mma_commit_pair_mcast(&acc_full[b], pair_mask);
                if (ts && lane == 0) ts[2] = gtimer();
            }
            if (ts && lane == 0) {
                ts[7] = mw;
                ts[8] = clock64() - m0;
            }
        }
        __syncwarp();
    } else {
        // 8 epilogue warps: warp w reads TMEM lane quarter w % 4; the two warps of a quarter
        // take alternate 32-token chunks.
        const uint32_t q = warp & 3;
        const uint32_t half = (warp - 2) >> 2;
        const uint32_t row = q * 32 + lane;
        const uint32_t lane_off = (q * 32u) << 16;
        const uint32_t acc_empty_leader = tc::mapa_shared(tc::smem_u32(&acc_empty[0]), crank & ~1u);
        uint32_t item = 0, seg = 0;
        for (uint32_t tile = cl; tile < a.tiles; tile += a.clusters, ++item) {
            const uint32_t fb = tile / a.ngroups, g = tile % a.ngroups;
            const uint32_t f = fb * 256 + rank * 128 + row;
            const uint32_t tg = g * a.G;
            const uint32_t tend = min(a.M, tg + a.G);  // tokens of this group: [tg, tend)
            uint32_t b = a.nbuf == 2 ? (item & 1) : 0u;
            const uint32_t use = a.nbuf == 2 ? (item >> 1) : item;
            if (ts && row == 0 && half == 0) ts[11] = gtimer();
            if constexpr (X3) {
                // drain the tile's accumulation segments (see the MMA warp): this warp owns
                // the 32-column chunks half, half + 2, half + 4 (G <= 192)
                float sum[3][32];
#pragma unroll
                for (uint32_t i = 0; i < 3; ++i)
#pragma unroll
                    for (uint32_t j = 0; j < 32; ++j) sum[i][j] = 0.0f;
                const uint32_t nit = (kb1 - kb0 + a.kps - 1) / a.kps;
                const uint32_t nseg = (nit + a.segn - 1) / a.segn;
                for (uint32_t sg = 0; sg < nseg; ++sg, ++seg) {
                    const uint32_t sb = seg & 1;
                    const uint32_t col = tmem + lane_off + sb * a.G + half * 32;
                    tc::mbar_wait(&acc_full[sb], (seg >> 1) & 1);
                    tc::tc_fence_after();
                    // (one 32-column load in flight: the register sums leave no room for more; the
                    // buffer is released as soon as the last load has landed)
                    uint32_t r[32];
#pragma unroll
                    for (uint32_t i = 0; i < 3; ++i) {
                        if (half * 32 + 64 * i < a.G) {
                            tc::tmem_ld32(col + 64 * i, r);
                            tc::tmem_ld_wait();
                        }
                        if (i == 2 || half * 32 + 64 * (i + 1) >= a.G) {
                            tc::tc_fence_before();
                            __syncwarp();
                            if (lane == 0) tc::mbar_arrive_remote(acc_empty_leader + sb * 8);
                        }
                        if (half * 32 + 64 * i < a.G) {
#pragma unroll
                            for (uint32_t j = 0; j < 32; ++j) sum[i][j] += __uint_as_float(r[j]);
                        }
                        if (half * 32 + 64 * (i + 1) >= a.G) break;
                    }
                }
                if (a.S == 1) {
#pragma unroll
                    for (uint32_t i = 0; i < 3; ++i) {
                        const uint32_t c = half * 32 + 64 * i;
                        if (c < a.G && tg + c < tend && !(a.dbg & 1)) {
                            uint32_t r[32];
#pragma unroll
                            for (uint32_t j = 0; j < 32; ++j) r[j] = __float_as_uint(sum[i][j]);
                            pg_epi<MODE, true>(a.ep, tend, tg + c, f, lane, r, nullptr, nullptr, tg);
                        }
                    }
                    if (ts && row == 0 && half == 0) ts[3] = gtimer();
                    continue;
                }
                // split K: the sums go back into TMEM buffer 0 (idle: one tile per cluster, all
                // of its MMAs done) for the in-cluster reduction below
                b = 0;
#pragma unroll
                for (uint32_t i = 0; i < 3; ++i) {
                    const uint32_t c = half * 32 + 64 * i;
                    if (c < a.G) {
                        uint32_t r[32];
#pragma unroll
                        for (uint32_t j = 0; j < 32; ++j) r[j] = __float_as_uint(sum[i][j]);
                        tc::tmem_st32(tmem + lane_off + c, r);
                    }
                }
                tc::tmem_st_wait();
            } else {
                tc::mbar_wait(&acc_full[b], use & 1);
                tc::tc_fence_after();
            }
            if (ts && row == 0 && half == 0) ts[12] = gtimer();
            const uint32_t dcol = tmem + lane_off + b * a.G;
            if (a.S == 1) {
                // QKV with one tile per pair: every MMA has retired, so the idle stage buffers
                // take this group's kv_rows and per-token (cos, sin) rows in two bulk copies
                // and the epilogue never waits on a dependent global load
                const uint32_t* s_rows = nullptr;
                const float2* s_rope = nullptr;
                if (a.stage_rope && !(a.dbg & 1)) {
                    const uint32_t nt = tend - tg, hd2 = a.ep.head_dim >> 1;
                    const uint32_t rope_bytes = nt * hd2 * 8, rows_bytes = (nt * 4 + 15) & ~15u;
                    // both CTAs of the pair need the same rows: each loads half of the (cos, sin)
                    // rows and multicasts it to the pair (halves the L2 reads of a table every
                    // CTA of the grid wants at once); V-only pairs need no rotation
                    // Chunk c's rows arrive on epi_bar[c] (the rows table with chunk 0), so the
                    // epilogue starts on the first chunk while the later ones are in flight; the
                    // two CTAs alternate chunks and multicast each to the pair.
                    const bool rot = fb * 256 < 2 * a.ep.hidden;
                    const uint32_t nch = (nt + 31) / 32;
                    (void)rope_bytes;
                    if (warp == 2 && lane == 0) {
                        for (uint32_t ci = 0; ci < nch; ++ci) {
                            const uint32_t cnt = min(32u, nt - 32 * ci);
                            tc::mbar_arrive_expect_tx(&epi_bar[ci], (rot ? cnt * hd2 * 8 : 0u) + (ci ? 0u : rows_bytes));
                        }
                        if (rot)
                            for (uint32_t ci = rank; ci < nch; ci += 2) {
                                const uint32_t cnt = min(32u, nt - 32 * ci);
                                tc::bulk_load_mcast(smem + (size_t)ci * 32 * hd2 * 8, a.ep.rope_tok + (size_t)(tg + 32 * ci) * hd2,
                                                    cnt * hd2 * 8, &epi_bar[ci], (uint16_t)(0x3u << (crank & ~1u)));
                            }
                        tc::bulk_load(smem + a.rows_off, a.ep.kv_rows + tg, rows_bytes, &epi_bar[0]);
                    }
                    tc::mbar_wait(&epi_bar[0], 0);
                    s_rope = reinterpret_cast<const float2*>(smem);
                    s_rows = reinterpret_cast<const uint32_t*>(smem + a.rows_off);
                }
                long long c_ld = 0, c_epi = 0;
                if (!(a.dbg & 1))
                    for (uint32_t c = half * 32; c < a.G && tg + c < tend; c += 64) {
                        uint32_t r[32];
                        if (a.stage_rope && c) tc::mbar_wait(&epi_bar[c / 32], 0);  // this chunk's side inputs
                        const long long q0 = ts ? clock64() : 0;
                        tc::tmem_ld32(dcol + c, r);
                        tc::tmem_ld_wait();
                        const long long q1 = ts ? clock64() : 0;
                        pg_epi<MODE, X3>(a.ep, tend, tg + c, f, lane, r, s_rows, s_rope, tg,
                                         a.stg_off == kNoStage ? nullptr : smem + a.stg_off + (warp - 2) * kStageSlice);
                        if (ts) {
                            c_ld += q1 - q0;
                            c_epi += clock64() - q1;
                        }
                    }
                if (ts && row == 0 && half == 0) {
                    ts[9] = c_ld;
                    ts[10] = c_epi;
                }
            } else {
                // in-cluster split-K (one tile per cluster): chunk j (32 tokens) belongs to split
                // j % S. Every MMA of every pair has completed once all CTAs pass this barrier,
                // so the stage buffers are free to receive [src split][j / S][32 cols][128 rows].
                tc::cluster_arrive();
                tc::cluster_wait();
                const bool tsw = ts && row == 0 && half == 0;
                if (tsw) ts[13] = gtimer();
                const uint32_t nchunks = (a.G + 31) / 32;
                const uint32_t per = (nchunks + a.S - 1) / a.S;
                // receive slot [src split][j / S] = [32 tokens][128 features] fp32. Nobody sends
                // to this CTA's own split slots: they hold the warps' 4 KB transpose slices.
                float* stg = per * kChunkBytes >= 8 * kStageSlice
                                 ? reinterpret_cast<float*>(smem + split * per * kChunkBytes + (warp - 2) * kStageSlice)
                                 : nullptr;
                const uint32_t recv = tc::smem_u32(smem) + split * per * kChunkBytes;
                for (uint32_t j = half; j < nchunks; j += 2) {
                    const uint32_t owner = j % a.S;
                    if (owner == split) continue;
                    uint32_t r[32];
                    tc::tmem_ld32(dcol + j * 32, r);
                    tc::tmem_ld_wait();
                    const uint32_t dst = tc::mapa_shared(recv + (j / a.S) * kChunkBytes, 2 * owner + rank);
                    if (stg) {  // 16-B remote stores, 4 token rows per instruction
                        stage_put_f32(stg, lane, r);
#pragma unroll
                        for (uint32_t i = 0; i < 8; ++i) {
                            const uint32_t t = i * 4 + (lane >> 3), c = q * 32 + (lane & 7) * 4;
                            tc::st_cluster_v4(dst + t * 512 + c * 4,
                                              *reinterpret_cast<const float4*>(stg + t * 32 + (lane & 7) * 4));
                        }
                        __syncwarp();
                    } else {
#pragma unroll
                        for (uint32_t i = 0; i < 32; ++i) tc::st_cluster_f32(dst + i * 512 + row * 4, r[i]);
                    }
                }
                if (tsw) ts[14] = gtimer();
                tc::cluster_arrive();  // release: the pushed chunks are visible after the wait
                tc::cluster_wait();
                if (tsw) ts[15] = gtimer();
                long long o_tm = 0, o_st = 0, o_rs = 0;
                for (uint32_t j = split + half * a.S; j < nchunks; j += 2 * a.S) {
                    if (a.dbg & 1) break;
                    uint32_t r[32];
                    const long long z0 = ts ? clock64() : 0;
                    tc::tmem_ld32(dcol + j * 32, r);
                    tc::tmem_ld_wait();
                    const long long z1 = ts ? clock64() : 0;
                    o_tm += z1 - z0;
                    if (MODE == EPI_RESID && stg) {
                        // sum in split order (deterministic) in the transposed layout, then the
                        // residual update with 16-B accesses
                        stage_put_f32(stg, lane, r);
                        const long long z2 = ts ? clock64() : 0;
                        o_st += z2 - z1;
                        const uint32_t tb = tg + j * 32;
                        const uint32_t n = tb < tend ? min(32u, tend - tb) : 0u;
                        const uint32_t own = tc::smem_u32(stg) + (lane >> 3) * 128 + (lane & 7) * 16;
                        const uint32_t oth = tc::smem_u32(smem) + (j / a.S) * kChunkBytes + (lane >> 3) * 512 +
                                             (q * 32 + (lane & 7) * 4) * 4;
                        resid_rows(a.ep, n, tb, f - lane, lane, [&](uint32_t i) {
                            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                            for (uint32_t s2 = 0; s2 < 4; ++s2) {
                                if (s2 >= a.S) break;
                                const uint32_t addr = s2 == split ? own + i * 512 : oth + s2 * per * kChunkBytes + i * 2048;
                                v = f4add(v, tc::ld_shared_v4(addr));
                            }
                            return v;
                        });
                        __syncwarp();
                        if (ts) o_rs += clock64() - z2;
                        continue;
                    }
                    float v[32];
#pragma unroll
                    for (uint32_t i = 0; i < 32; ++i) v[i] = 0.0f;
                    for (uint32_t s2 = 0; s2 < a.S; ++s2) {  // split order: deterministic
                        if (s2 == split) {
#pragma unroll
                            for (uint32_t i = 0; i < 32; ++i) v[i] += __uint_as_float(r[i]);
                        } else {
                            const float* src = reinterpret_cast<const float*>(smem + (s2 * per + j / a.S) * kChunkBytes) + row;
#pragma unroll
                            for (uint32_t i = 0; i < 32; ++i) v[i] += src[i * 128];
                        }
                    }
                    if (tg + j * 32 < tend) {
#pragma unroll
                        for (uint32_t i = 0; i < 32; ++i) r[i] = __float_as_uint(v[i]);
                        pg_epi<MODE, X3>(a.ep, tend, tg + j * 32, f, lane, r, nullptr, nullptr, 0);
                    }
                }
                if (tsw) {
                    ts[9] = o_tm;
                    ts[10] = o_st;
                    ts[12] = o_rs;
                }
            }
            // release the accumulator to the pair's MMA issuer (one arrive per warp; 3xTF32
            // released each segment as it was drained)
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0 && !X3) tc::mbar_arrive_remote(acc_empty_leader + b * 8);
            if (ts && row == 0 && half == 0) ts[3] = gtimer();
        }
    }
    if (a.S > 1 && warp < 2) {  // the producer / MMA warps take part in the reduction barriers
        tc::cluster_arrive();
        tc::cluster_wait();
        tc::cluster_arrive();
        tc::cluster_wait();
    }
    tc::tc_fence_before();
    tc::cluster_sync();
    tc::tc_fence_after();
    if (warp == 1) tc::tmem_dealloc_pair(tmem, a.tmem_cols);
    if (ts && threadIdx.x == 0) ts[4] = gtimer();
}

uint32_t round16(uint32_t x) { return (x + 15) / 16 * 16; }

using PgKernel = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, PgArgs);
PgKernel pg_kernel(int mode, bool x3 = false) {
    if (x3) switch (mode) {
            case EPI_QKV: return tc_pgemm_kernel<EPI_QKV, true>;
            case EPI_RESID: return tc_pgemm_kernel<EPI_RESID, true>;
            case EPI_GELU: return tc_pgemm_kernel<EPI_GELU, true>;
            case EPI_STORE_F32: return tc_pgemm_kernel<EPI_STORE_F32, true>;
            default: return tc_pgemm_kernel<EPI_STORE, true>;
        }
    switch (mode) {
        case EPI_QKV: return tc_pgemm_kernel<EPI_QKV, false>;
        case EPI_RESID: return tc_pgemm_kernel<EPI_RESID, false>;
        case EPI_GELU: return tc_pgemm_kernel<EPI_GELU, false>;
        case EPI_STORE_F32: return tc_pgemm_kernel<EPI_STORE_F32, false>;
        default: return tc_pgemm_kernel<EPI_STORE, false>;
    }
}

// Largest number of co-resident clusters of `size` CTAs at this kernel's footprint.
uint32_t max_clusters(uint32_t size, size_t smem) {
    static std::mutex mu;
    static std::unordered_map<uint64_t, uint32_t> cache;
    std::lock_guard<std::mutex> lk(mu);
    uint32_t& v = cache[((uint64_t)size << 32) | smem];
    if (!v) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(size * 32);
        cfg.blockDim = dim3(kPgThreads);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = size;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int n = 0;
        MPIC_CUDA(cudaOccupancyMaxActiveClusters(&n, pg_kernel(EPI_STORE, false), &cfg));
        v = (uint32_t)std::max(1, n);
    }
    return v;
}

}  // namespace

bool pgemm_supported(uint32_t M, uint32_t N, uint32_t K) {
    return M > 0 && N % 256 == 0 && K % 64 == 0 && K >= 64;
}
bool pgemm_x3_supported(uint32_t M, uint32_t N, uint32_t K) {
    return M > 0 && N % 256 == 0 && K % 32 == 0 && K >= 64;
}

static unsigned long long* g_ts_buf = nullptr;
void pgemm_timestamps(unsigned long long* out9) {
    if (!g_ts_buf) {
        for (int i = 0; i < 16; ++i) out9[i] = 0;
        return;
    }
    MPIC_CUDA(cudaMemcpy(out9, g_ts_buf, 16 * 8, cudaMemcpyDeviceToHost));
}

namespace {
// A, W: bf16 operands, or (x3) the fp32 hi parts with A_lo / W_lo the lo parts.
void launch_pgemm_impl(const void* A, const void* A_lo, const void* W, const void* W_lo, uint32_t M, uint32_t N,
                       uint32_t K, const EpiParams& ep_in, cudaStream_t s, bool w_blocked, bool x3) {
    MPIC_REQUIRE(x3 ? pgemm_x3_supported(M, N, K) : pgemm_supported(M, N, K), MPIC_ERR_VALIDATION,
                 "unsupported pair gemm shape");
    MPIC_REQUIRE(ep_in.mode != EPI_QKV || (ep_in.head_dim % 2 == 0 && ep_in.hidden % 32 == 0),
                 MPIC_ERR_VALIDATION, "pair gemm QKV epilogue needs hidden % 32 == 0");
    static const uint32_t group_max = [] {
        const char* e = getenv("MPIC_PG_GROUP");  // diagnostics: max tokens per group (256 or 512)
        return e ? (uint32_t)atoi(e) : 512u;
    }();
    static const uint32_t dbg = [] {
        const char* e = getenv("MPIC_PG_DBG");
        return e ? (uint32_t)atoi(e) : 0u;
    }();
    static const uint32_t force_s = [] {
        const char* e = getenv("MPIC_PG_SPLIT");  // diagnostics: force the in-cluster K split
        return e ? (uint32_t)atoi(e) : 0u;
    }();
    static const bool split_pieces = [] {
        const char* e = getenv("MPIC_PG_PIECES");  // diagnostics: 1 = two accumulator chains per group
        return e && atoi(e) != 0;
    }();
    static const uint32_t kps_env = [] {
        const char* e = getenv("MPIC_PG_KPS");  // diagnostics: k-blocks per pipeline stage
        return e ? (uint32_t)atoi(e) : 0u;
    }();
    static std::once_flag once;
    std::call_once(once, [] {
        for (int m : {EPI_STORE, EPI_QKV, EPI_RESID, EPI_GELU, EPI_STORE_F32})
            for (bool x : {false, true}) {
                MPIC_CUDA(cudaFuncSetAttribute(pg_kernel(m, x), cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
                MPIC_CUDA(cudaFuncSetAttribute(pg_kernel(m, x), cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            }
    });
    PgArgs best_a{};
    double best = 1e30;
    // Plan: token groups (1 natural, or the tokens cut into 2-3 groups to create tiles) x
    // in-cluster K split S. Cost model per pair, in cycles: rounds x k-blocks x
    // max(MMA 2G, operand fill 256 + G), plus for S > 1 the DSMEM reduction and owner
    // epilogue: ~2000 + 40 per token column pushed ((S-1)/S of the group) — fitted to the
    // measured Wo/W2 launches at config C (Wo: 2 groups x S=2 beats 1 x S=3 by 2 us).
    // 3xTF32: two TMEM buffers of G columns and the epilogue's register sums cap G at 192
    const uint32_t gcap = x3 ? 192u : 256u;
    const uint32_t ng_nat = x3 ? ceil_div(M, gcap) : M <= 512 ? 1 : ceil_div(M, 256);
    // candidates: 1-3x the natural group count, and (3xTF32) one group more — m = 330 as 3 x 112
    // tokens fills two rounds of 74 pairs with 144 QKV tiles where 2 x 176 leave the second
    // round 30% full
    for (uint32_t gm : {1u, 2u, 3u, 0u}) {
        if (gm == 0 && !x3) continue;
        PgArgs a{};
        a.M = M;
        a.N = N;
        a.K = K;
        a.dbg = dbg;
        a.ngroups = gm ? ng_nat * gm : ng_nat + 1;
        static const uint32_t force_ng = [] {
            const char* e = getenv("MPIC_PG_NGROUPS");  // diagnostics: force the token-group count
            return e ? (uint32_t)atoi(e) : 0u;
        }();
        if (force_ng && a.ngroups != force_ng) continue;
        if (!x3 && a.ngroups == 1 && M > 256 && M <= group_max) {
            a.P0 = round16((M + 1) / 2);
            a.P1 = round16(M - a.P0);
        } else {
            if (a.ngroups == 1 && M > 256) continue;  // MPIC_PG_GROUP=256 diagnostics
            a.P0 = round16(ceil_div(M, a.ngroups));
            a.P1 = 0;
            if (a.P0 > gcap || (gm != 1 && a.P0 < 64)) continue;
            // two interleaved accumulator chains (off by default: each cta_group::2 MMA costs at
            // least ~83 cycles, so halving N loses more than the interleave gains)
            if (split_pieces && !x3 && a.P0 >= 64) {
                const uint32_t g = a.P0;
                a.P0 = round16((g + 1) / 2);
                a.P1 = g - a.P0;
            }
        }
        a.G = a.P0 + a.P1;
        a.nbuf = 2 * a.G <= 512 ? 2 : 1;
        a.tmem_cols = 32;
        while (a.tmem_cols < a.nbuf * a.G) a.tmem_cols *= 2;
        a.kel = x3 ? 32 : 64;
        a.kblocks = K / a.kel;
        a.tiles = (N / 256) * a.ngroups;
        a.wsub = x3 ? 2 * kPgWBytes : kPgWBytes;
        a.xlo = x3 ? a.G * 64 : 0u;
        a.sub_bytes = a.wsub + (x3 ? 2 : 1) * a.G * 64;
        a.kps = kps_env ? kps_env : 2;
        a.stage_bytes = a.kps * a.sub_bytes;
        a.segn = 1;
        a.xoff1 = a.P0 * 64;
        const uint32_t budget = 227 * 1024 - 1024 - 128;
        a.stages = std::min<uint32_t>(8, budget / a.stage_bytes);
        if (a.stages < 3 && a.kps > 1) {  // keep at least 3 stages in flight
            a.kps = 1;
            a.stage_bytes = a.sub_bytes;
            a.stages = std::min<uint32_t>(8, budget / a.stage_bytes);
        }
        if (a.stages < 2) continue;
        static const uint32_t seg_kb = [] {
            const char* e = getenv("MPIC_X3_SEG");  // diagnostics: k-blocks (32 K) per accumulation segment
            return e ? std::max(1, atoi(e)) : 2;
        }();
        // default 2 k-blocks (64 K): with the small products issued first, config C's 32-layer
        // logits sit at 0.11 of the fp64-referenced gate and the fp32 GEMMs take 30 ms per
        // request (1 k-block: 40 ms, drain-bound; 4: slower, fewer stages in flight)
        if (x3) a.segn = std::min(std::max(1u, seg_kb / a.kps), a.stages - 1);  // (a segment's stages are all
                                                                                // resident before its MMAs)
        a.w_evict_first = a.ngroups == 1;
        a.ep = ep_in;
    a.ep.dbg = dbg;
        const size_t smem = (size_t)a.stages * a.stage_bytes + 1024 + (2 * a.stages + 4 + kEpiBars) * 8 + 16;
        const uint32_t nchunks = (a.G + 31) / 32;
        // MMA cycles per k-block (4 k16 steps): a cta_group::2 instruction costs
        // max(N/2, ~83) cycles; operand fill ~256 + G cycles. (With the single-thread issuer a
        // lone accumulator chain issued ~1.5x slower than two interleaved ones; the
        // warp-uniform issuer removed that: W2 at config C now takes 2 groups x S=2.)
        static const double chain = [] {
            const char* e = getenv("MPIC_PG_CHAIN");  // diagnostics: lone-chain issue factor
            return e ? atof(e) : 1.0;  // 1.5 with the old single-thread issuer
        }();
        // (3xTF32: three K = 8 tf32 instructions per 32-B step, twice the operand bytes)
        const double mma = 4.0 * (std::max(a.P0 / 2.0, 83.0) + (a.P1 ? std::max(a.P1 / 2.0, 83.0) : 0.0)) *
                           (a.P1 ? 1.0 : chain) * (x3 ? 3.0 : 1.0);
        const double t_kb = std::max(mma, (256.0 + a.G) * (x3 ? 2.0 : 1.0));
        for (uint32_t S : {1u, 2u, 3u, 4u}) {
            if (force_s && S != force_s && S != 1) continue;
            if (S > 1 && a.kblocks / S < 2) continue;
            const uint32_t C = max_clusters(2 * S, smem);
            static const bool vplan = getenv("MPIC_PG_VERBOSE") != nullptr;
            if (vplan)
                fprintf(stderr, "  plan G=%u S=%u: max clusters %u, tiles %u, recv %zu of %u B\n", a.G, S, C, a.tiles,
                        (size_t)S * ceil_div(nchunks, S) * kChunkBytes, a.stages * a.stage_bytes);
            if (S > 1 && (a.tiles > C || (size_t)S * ceil_div(nchunks, S) * kChunkBytes > (size_t)a.stages * a.stage_bytes))
                continue;
            const double cost = (double)ceil_div(a.tiles, std::min(C, a.tiles)) * ceil_div(a.kblocks, S) * t_kb +
                                (S > 1 ? 2000.0 + 40.0 * a.G * (S - 1) / S : 0.0) + (force_s > 1 && S == 1 ? 1e20 : 0.0);
            if (cost < best - 1e-9) {
                best = cost;
                best_a = a;
                best_a.S = S;
                best_a.clusters = std::min(C, a.tiles);
            }
        }
    }
    MPIC_REQUIRE(best < 1e29, MPIC_ERR_VALIDATION, "pair gemm: no feasible tiling");
    PgArgs a = best_a;
    static unsigned long long* ts_buf = [] {
        unsigned long long* b = nullptr;
        if (getenv("MPIC_PG_TS")) {
            cudaMalloc(&b, 128);
            cudaMemset(b, 0, 128);
        }
        return b;
    }();
    a.ts = ts_buf;
    g_ts_buf = ts_buf;
    a.w_blocked = w_blocked ? 1u : 0u;
    static const int pfd_env = [] {
        const char* e = getenv("MPIC_PG_PFD");  // diagnostics: weight L2 prefetch distance (k-blocks)
        return e ? atoi(e) : -1;
    }();
    // The producer's L2 prefetch of weights ahead of the smem ring is off by default: it cost
    // 2.7% at config C and 10% at config B (m = 96) — the extra requests compete with the
    // ring's own loads; MPIC_PG_PFD=<k-blocks> turns it back on for diagnostics.
    a.pfd = pfd_env >= 0 && !x3 ? (uint32_t)pfd_env : 0u;
    static const bool prologue_pf = [] {
        // off by default, like the ring prefetch: 1% faster at config C without it
        const char* e = getenv("MPIC_PG_PROLOGUE_PF");  // diagnostics: 1 = prefetch before the PDL wait
        return e && atoi(e) != 0;
    }();
    a.prologue_pf = prologue_pf && !x3 ? 1u : 0u;
    // Off by default, like the L2 prefetch: config B 4.00 -> 4.04 ms and config C unchanged with
    // it (the early weight stream competes with the previous kernel's tail).
    static const bool w_early = [] {
        const char* e = getenv("MPIC_PG_WEARLY");  // diagnostics: 1 = first stages' weights before the PDL wait
        return e && atoi(e) != 0;
    }();
    a.w_early = w_early ? 1u : 0u;

    const size_t smem = (size_t)a.stages * a.stage_bytes + 1024 + (2 * a.stages + 4 + kEpiBars) * 8 + 16;
    static const bool verbose = getenv("MPIC_PG_VERBOSE") != nullptr;
    if (verbose)
        fprintf(stderr, "pgemm M=%u N=%u K=%u: groups=%u P0=%u P1=%u S=%u clusters=%u stages=%u x %u kb nbuf=%u\n", M,
                N, K, a.ngroups, a.P0, a.P1, a.S, a.clusters, a.stages, a.kps, a.nbuf);
    if (!x3 && ep_in.mode == EPI_QKV && ep_in.rope_tok && ep_in.head_dim % 4 == 0 && a.S == 1 &&
        a.clusters >= a.tiles && a.ngroups == 1) {
        const uint32_t rope_bytes = a.G * (ep_in.head_dim / 2) * 8;
        a.rows_off = (rope_bytes + 1023) & ~1023u;
        static const bool no_stage = getenv("MPIC_PG_NOROPESTAGE") != nullptr;  // diagnostics
        a.stage_rope = !no_stage && a.rows_off + a.G * 4 + 16 <= a.stages * a.stage_bytes;
    }
    static const bool staged_env = [] {
        const char* e = getenv("MPIC_PG_STAGED");  // diagnostics: 0 = direct (narrow) epilogue stores
        return !e || atoi(e) != 0;
    }();
    a.stg_off = kNoStage;
    // the staged QKV epilogue reads (cos, sin) as 16-B pairs of pairs from rope_tok
    const bool qkv_ok = ep_in.mode != EPI_QKV || a.stage_rope;
    if (!x3 && staged_env && qkv_ok && a.S == 1 && a.clusters >= a.tiles) {
        // one tile per cluster: the stage ring is idle once the accumulator is complete
        const uint32_t off = a.stage_rope ? (a.rows_off + a.G * 4 + 16 + 1023) & ~1023u : 0u;
        if (off + 8 * kStageSlice <= a.stages * a.stage_bytes) a.stg_off = off;
    }
    CUtensorMap tmW, tmX0, tmX1, tmWl, tmX0l, tmX1l;
    if (x3) {
        tmW = make_tmap_f32(W, K, N, 32, 128);
        tmWl = make_tmap_f32(W_lo, K, N, 32, 128);
        tmX0 = make_tmap_f32(A, K, M, 32, a.P0 / 2);
        tmX0l = make_tmap_f32(A_lo, K, M, 32, a.P0 / 2);
        tmX1 = a.P1 ? make_tmap_f32(A, K, M, 32, a.P1 / 2) : tmX0;
        tmX1l = a.P1 ? make_tmap_f32(A_lo, K, M, 32, a.P1 / 2) : tmX0l;
    } else {
        tmW = w_blocked ? make_tmap_bf16(W, 64, (uint64_t)N * a.kblocks, 64, 128) : make_tmap_bf16(W, K, N, 64, 128);
        tmX0 = make_tmap_bf16(A, K, M, 64, a.P0 / 2);
        tmX1 = a.P1 ? make_tmap_bf16(A, K, M, 64, a.P1 / 2) : tmX0;
        tmWl = tmW;
        tmX0l = tmX0;
        tmX1l = tmX1;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.clusters * 2 * a.S);
    cfg.blockDim = dim3(kPgThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[3];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2 * a.S;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    at[2].id = cudaLaunchAttributePriority;
    at[2].val.priority = hot_priority();
    cfg.attrs = at;
    cfg.numAttrs = 3;
    MPIC_CUDA(cudaLaunchKernelEx(&cfg, pg_kernel(a.ep.mode, x3), tmW, tmX0, tmX1, tmWl, tmX0l, tmX1l, a));
    MPIC_LAUNCHED();
}
}  // namespace

void launch_pgemm(const __nv_bfloat16* A, const __nv_bfloat16* W, uint32_t M, uint32_t N, uint32_t K,
                  const EpiParams& ep, cudaStream_t s, bool w_blocked) {
    launch_pgemm_impl(A, nullptr, W, nullptr, M, N, K, ep, s, w_blocked, false);
}

void launch_pgemm_x3(const float* A_hi, const float* A_lo, const float* W_hi, const float* W_lo, uint32_t M,
                     uint32_t N, uint32_t K, const EpiParams& ep, cudaStream_t s) {
    MPIC_REQUIRE(ep.mode != EPI_QKV || ep.rope, MPIC_ERR_VALIDATION, "3xTF32 QKV epilogue needs the RoPE table");
    launch_pgemm_impl(A_hi, A_lo, W_hi, W_lo, M, N, K, ep, s, false, true);
}

// x = hi + lo with hi = tf32(x), lo = tf32(x - hi) (round to nearest, ties away): both parts
// carry tf32 bits only, so the tensor core reads them exactly whatever its own rounding.
__global__ void tf32_split_kernel(const float4* __restrict__ x, float4* __restrict__ hi, float4* __restrict__ lo,
                                  size_t n4) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        const float4 v = x[i];
        float4 h, l;
        float* pv = (float*)&v;
        float* ph = (float*)&h;
        float* pl = (float*)&l;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            uint32_t a, b;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(a) : "f"(pv[c]));
            ph[c] = __uint_as_float(a);
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(b) : "f"(pv[c] - ph[c]));
            pl[c] = __uint_as_float(b);
        }
        hi[i] = h;
        lo[i] = l;
    }
}

void launch_tf32_split(const float* x, float* hi, float* lo, size_t n, cudaStream_t s) {
    MPIC_REQUIRE(n % 4 == 0, MPIC_ERR_VALIDATION, "tf32 split needs a multiple of 4 elements");
    const size_t n4 = n / 4;
    const uint32_t blocks = (uint32_t)std::min<size_t>(kNumSMs * 8, std::max<size_t>(1, (n4 + 255) / 256));
    tf32_split_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(hi),
                                             reinterpret_cast<float4*>(lo), n4);
    MPIC_LAUNCHED();
}

__global__ void block_weights_kernel(const __nv_bfloat16* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                     uint32_t N, uint32_t K, bool to_blocked) {
    // one 16-B vector (8 elements) per thread step; blocked index of (n, k):
    //   ((n/128)*(K/64) + k/64)*8192 + (n%128)*64 + k%64
    const size_t total = (size_t)N * K / 8;
    const uint32_t kb = K / 64;
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < total; v += (size_t)gridDim.x * blockDim.x) {
        const size_t e = v * 8;
        const uint32_t n = (uint32_t)(e / K), k = (uint32_t)(e % K);
        const size_t b = ((size_t)(n / 128) * kb + k / 64) * 8192 + (n % 128) * 64 + k % 64;
        if (to_blocked) reinterpret_cast<uint4*>(dst)[b / 8] = reinterpret_cast<const uint4*>(src)[v];
        else reinterpret_cast<uint4*>(dst)[v] = reinterpret_cast<const uint4*>(src)[b / 8];
    }
}

void launch_block_weights(const __nv_bfloat16* src, __nv_bfloat16* dst, uint32_t N, uint32_t K, bool to_blocked,
                          cudaStream_t s) {
    MPIC_REQUIRE(N % 128 == 0 && K % 64 == 0, MPIC_ERR_VALIDATION, "blocked weights need N % 128, K % 64");
    block_weights_kernel<<<kNumSMs * 8, 256, 0, s>>>(src, dst, N, K, to_blocked);
    MPIC_LAUNCHED();
}

}  // namespace mpicb
