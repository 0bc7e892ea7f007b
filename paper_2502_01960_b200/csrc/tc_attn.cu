// K4 — selective causal attention on the 5th-gen tensor cores (head_dim 128).
//
// For recomputed row i (cache position rows[i]) and head hd, attend over cache keys
// [0, rows[i]] of the just-scattered layer cache (proj/src/linker.cpp:80-113): the
// per-row causal limit is the row's POSITION, not its index in the tile.
//
// Work unit = (128-query tile, head, range of 128-key blocks). The host splits long key
// ranges (flash-decoding style) so that ~3 waves of units cover the 148 SMs; partial
// results are merged by attn_combine_kernel. One CTA per unit:
//
//   warp 0     TMA: Q tile [128 x 128] once, K/V blocks [128 keys x 128] into 2-stage rings
//   warp 1     TMEM alloc (512 cols: S0 | S1 | O) + single-thread tcgen05.mma issuer:
//              S_b = Q . K_b^T (SS, K-major) and O += P_b . V_b (P K-major from smem,
//              V MN-major), in the order S0 S1 PV0 S2 PV1 S3 ...
//   warps 2-5  softmax, one thread per query row (TMEM lane): scale, per-row causal mask,
//              online max with lazy rescaling of O in TMEM (only when the max grows by
//              more than 2^8), exp2, row sums, P written to smem in the SWIZZLE_128B
//              K-major layout the MMA descriptor expects; final O / l epilogue.
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace mpicb {

CUtensorMap make_tmap_bf16(const void* ptr, uint64_t inner, uint64_t outer, uint32_t box_inner,
                           uint32_t box_outer);

namespace {

constexpr uint32_t kAttnThreads = 352;  // K TMA, MMA, V TMA, 8 softmax warps
constexpr uint32_t kKvStages = 3;
constexpr uint32_t kSoftmaxThreads = 256;
constexpr uint32_t kTile = 32 * 1024;  // one [128 x 128] bf16 tile as 2 swizzled 64-col halves
constexpr uint32_t kHalf = 16 * 1024;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

struct AttnParams {
    const AttnUnit* units;
    const uint32_t* rows;
    uint32_t m;
    uint32_t h;
    float scale_log2;       // inv_sqrt_d * log2(e)
    __nv_bfloat16* out;     // [m][h]
    float* part_o;          // [slots][128][128]
    float2* part_ml;        // [slots][128] (m_used, l)
};

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&v);
}

__global__ void __launch_bounds__(kAttnThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;
    uint8_t* sK = smem + kTile;                 // kKvStages stages
    uint8_t* sV = smem + (1 + kKvStages) * kTile;  // kKvStages stages
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (1 + 2 * kKvStages) * kTile);
    uint64_t* q_full = bars + 0;
    uint64_t* k_full = bars + 1;                   // [kKvStages]
    uint64_t* k_empty = k_full + kKvStages;        // [kKvStages]
    uint64_t* v_full = k_empty + kKvStages;        // [kKvStages]
    uint64_t* v_empty = v_full + kKvStages;        // [kKvStages]
    uint64_t* s_full = v_empty + kKvStages;        // [2]
    uint64_t* p_full = s_full + 2;                 // [2]
    uint64_t* o_full = p_full + 2;                 // [2] — PV_b completes on o_full[b & 1]
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(o_full + 2);

    const AttnUnit u = p.units[blockIdx.x];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t q0 = u.tile * 128u;
    const uint32_t nb = u.b1 - u.b0;
    const int hcol = (int)(u.head * 128u);

    if (warp == 0 && lane == 0) {
        tc::tma_prefetch_desc(&tmQ);
        tc::tma_prefetch_desc(&tmK);
        tc::tma_prefetch_desc(&tmV);
        tc::mbar_init(q_full, 1);
        for (uint32_t i = 0; i < kKvStages; ++i) {
            tc::mbar_init(&k_full[i], 1);
            tc::mbar_init(&k_empty[i], 1);
            tc::mbar_init(&v_full[i], 1);
            tc::mbar_init(&v_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&s_full[i], 1);
            tc::mbar_init(&p_full[i], kSoftmaxThreads);
            tc::mbar_init(&o_full[i], 1);
        }
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc(tmem_holder, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_holder;
    // TMEM columns: S0 [0,128) | S1 [128,256) | O [256,384) | row exchange [384,392).
    // P_b (bf16, two keys per column) overwrites the first 64 columns of S_b in place.
    constexpr uint32_t idesc_s = tc::idesc_bf16(128, 128, false);
    constexpr uint32_t idesc_o = tc::idesc_bf16(128, 128, true);

    if (warp == 0) {
        if (lane == 0) {  // K producer (+ Q)
            tc::mbar_arrive_expect_tx(q_full, kTile);
            tc::tma_load_2d(sQ, &tmQ, q_full, hcol, (int)q0);
            tc::tma_load_2d(sQ + kHalf, &tmQ, q_full, hcol + 64, (int)q0);
            for (uint32_t b = 0; b < nb; ++b) {
                const uint32_t s = b % kKvStages, ph = (b / kKvStages) & 1;
                const int j0 = (int)((u.b0 + b) * 128u);
                tc::mbar_wait(&k_empty[s], ph ^ 1);
                tc::mbar_arrive_expect_tx(&k_full[s], kTile);
                tc::tma_load_2d(sK + s * kTile, &tmK, &k_full[s], hcol, j0);
                tc::tma_load_2d(sK + s * kTile + kHalf, &tmK, &k_full[s], hcol + 64, j0);
            }
        }
        __syncwarp();
    } else if (warp == 2) {
        if (lane == 0) {  // V producer
            for (uint32_t b = 0; b < nb; ++b) {
                const uint32_t s = b % kKvStages, ph = (b / kKvStages) & 1;
                const int j0 = (int)((u.b0 + b) * 128u);
                tc::mbar_wait(&v_empty[s], ph ^ 1);
                tc::mbar_arrive_expect_tx(&v_full[s], kTile);
                tc::tma_load_2d(sV + s * kTile, &tmV, &v_full[s], hcol, j0);
                tc::tma_load_2d(sV + s * kTile + kHalf, &tmV, &v_full[s], hcol + 64, j0);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t qa = tc::smem_u32(sQ);
            auto issue_s = [&](uint32_t b) {
                const uint32_t ks = b % kKvStages;
                tc::mbar_wait(&k_full[ks], (b / kKvStages) & 1);
                tc::tc_fence_after();
                const uint32_t ka = tc::smem_u32(sK + ks * kTile);
#pragma unroll
                for (uint32_t kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * kHalf + (kk & 3) * 32;
                    tc::mma_bf16(tmem + (b & 1) * 128, tc::desc_k_sw128(qa + off), tc::desc_k_sw128(ka + off),
                                 idesc_s, kk > 0 ? 1u : 0u);
                }
                tc::mma_commit(&k_empty[ks]);
                tc::mma_commit(&s_full[b & 1]);
            };
            tc::mbar_wait(q_full, 0);
            issue_s(0);
            if (nb > 1) issue_s(1);
            for (uint32_t b = 0; b < nb; ++b) {
                const uint32_t s = b & 1, vs = b % kKvStages;
                tc::mbar_wait(&p_full[s], (b >> 1) & 1);
                tc::mbar_wait(&v_full[vs], (b / kKvStages) & 1);
                tc::tc_fence_after();
                const uint32_t va = tc::smem_u32(sV + vs * kTile);
#pragma unroll
                for (uint32_t kk = 0; kk < 8; ++kk)  // A = P_b from TMEM: 16 keys = 8 packed columns
                    tc::mma_bf16_ts(tmem + 256, tmem + s * 128 + kk * 8, tc::desc_mn_sw128(va + kk * 2048, kHalf),
                                    idesc_o, (b > 0 || kk > 0) ? 1u : 0u);
                tc::mma_commit(&v_empty[vs]);
                tc::mma_commit(&o_full[s]);
                if (b + 2 < nb) issue_s(b + 2);  // in-order after PV_b, which reads P_b from S_b's columns
            }
        }
        __syncwarp();
    } else {
        // ---- softmax: 8 warps, a pair per TMEM lane quarter; warp hsel owns score columns
        // (keys) and O columns (head dims) [64*hsel, 64*hsel+64) of its 32 query rows.
        const uint32_t quarter = warp & 3;
        const uint32_t hsel = (warp - 3) >> 2;
        const uint32_t r = quarter * 32 + lane;
        const uint32_t qi = q0 + r;
        const bool valid = qi < p.m;
        const uint32_t limit = valid ? p.rows[qi] : 0u;
        const uint32_t lane_base = (quarter * 32u) << 16;
        const uint32_t xchg = tmem + lane_base + 384;
        const uint32_t bar_id = 1 + quarter;
        float m_used = -INFINITY, l = 0.0f;
        for (uint32_t b = 0; b < nb; ++b) {
            const uint32_t s = b & 1;
            const uint32_t j0 = (u.b0 + b) * 128u + hsel * 64u;  // first key of my half
            tc::mbar_wait(&s_full[s], (b >> 1) & 1);
            tc::tc_fence_after();
            const uint32_t sa = tmem + lane_base + s * 128 + hsel * 64;
            const bool masked = __any_sync(0xffffffffu, j0 + 63 > limit);
            uint32_t v[64];
            tc::tmem_ld32(sa, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
            tc::tmem_ld32(sa + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
            tc::tmem_ld_wait();
            float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
            if (masked) {
#pragma unroll
                for (uint32_t e = 0; e < 64; e += 4) {
                    mx0 = j0 + e + 0 <= limit ? fmaxf(mx0, __uint_as_float(v[e + 0])) : mx0;
                    mx1 = j0 + e + 1 <= limit ? fmaxf(mx1, __uint_as_float(v[e + 1])) : mx1;
                    mx2 = j0 + e + 2 <= limit ? fmaxf(mx2, __uint_as_float(v[e + 2])) : mx2;
                    mx3 = j0 + e + 3 <= limit ? fmaxf(mx3, __uint_as_float(v[e + 3])) : mx3;
                }
            } else {
#pragma unroll
                for (uint32_t e = 0; e < 64; e += 4) {
                    mx0 = fmaxf(mx0, __uint_as_float(v[e + 0]));
                    mx1 = fmaxf(mx1, __uint_as_float(v[e + 1]));
                    mx2 = fmaxf(mx2, __uint_as_float(v[e + 2]));
                    mx3 = fmaxf(mx3, __uint_as_float(v[e + 3]));
                }
            }
            // row max across the two halves, exchanged through spare TMEM columns
            float mraw = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
            tc::tmem_st1(xchg + s * 2 + hsel, __float_as_uint(mraw));
            tc::tmem_st_wait();
            tc::tc_fence_before();
            tc::named_bar_sync(bar_id, 64);
            tc::tc_fence_after();
            mraw = fmaxf(mraw, __uint_as_float(tc::tmem_ld1(xchg + s * 2 + (hsel ^ 1))));
            tc::tmem_ld_wait();
            const float mx = mraw * p.scale_log2;
            float alpha = 1.0f;
            const bool grow = mx > m_used + kRescaleThreshold || (m_used == -INFINITY && mx > -INFINITY);
            if (grow) {
                alpha = m_used == -INFINITY ? 0.0f : tc::ex2_approx(m_used - mx);
                m_used = mx;
                l *= alpha;
            }
            if (b > 0 && __any_sync(0xffffffffu, grow && alpha != 1.0f)) {
                // every earlier PV must have landed before O is rescaled
                tc::mbar_wait(&o_full[(b - 1) & 1], ((b - 1) >> 1) & 1);
                tc::tc_fence_after();
                const uint32_t oa = tmem + lane_base + 256 + hsel * 64;
#pragma unroll
                for (uint32_t c = 0; c < 4; ++c) {
                    uint32_t o[16];
                    tc::tmem_ld16(oa + c * 16, o);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (uint32_t e = 0; e < 16; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
                    tc::tmem_st16(oa + c * 16, o);
                }
                tc::tmem_st_wait();
            }
            const float neg_m = m_used == -INFINITY ? 0.0f : -m_used;
            const bool row_dead = m_used == -INFINITY;
            float l0 = 0.f, l1 = 0.f, l2 = 0.f, l3 = 0.f;
            uint32_t pk[32];
#pragma unroll
            for (uint32_t e = 0; e < 64; e += 2) {
                float x0 = tc::ex2_approx(fmaf(__uint_as_float(v[e]), p.scale_log2, neg_m));
                float x1 = tc::ex2_approx(fmaf(__uint_as_float(v[e + 1]), p.scale_log2, neg_m));
                if (masked) {
                    x0 = (j0 + e <= limit && !row_dead) ? x0 : 0.0f;
                    x1 = (j0 + e + 1 <= limit && !row_dead) ? x1 : 0.0f;
                }
                if (e & 2) { l2 += x0; l3 += x1; } else { l0 += x0; l1 += x1; }
                pk[e >> 1] = pack_bf16(x0, x1);
            }
            l += (l0 + l1) + (l2 + l3);
            // P_b -> TMEM columns [s*128 + hsel*32, +32) of my lanes (S_b already consumed)
            tc::tmem_st32(tmem + lane_base + s * 128 + hsel * 32, pk);
            tc::tmem_st_wait();
            tc::tc_fence_before();
            tc::mbar_arrive(&p_full[s]);
        }
        // ---- epilogue: O / l over both halves' partial row sums
        tc::tmem_st1(xchg + 4 + hsel, __float_as_uint(l));
        tc::tmem_st_wait();
        tc::mbar_wait(&o_full[(nb - 1) & 1], ((nb - 1) >> 1) & 1);
        tc::tc_fence_before();
        tc::named_bar_sync(bar_id, 64);
        tc::tc_fence_after();
        l += __uint_as_float(tc::tmem_ld1(xchg + 4 + (hsel ^ 1)));
        tc::tmem_ld_wait();
        const uint32_t oa = tmem + lane_base + 256 + hsel * 64;
        const bool direct = u.slot == 0xffffffffu;
        const float inv = l > 0.0f ? 1.0f / l : 0.0f;
#pragma unroll
        for (uint32_t c = 0; c < 4; ++c) {
            uint32_t o[16];
            tc::tmem_ld16(oa + c * 16, o);
            tc::tmem_ld_wait();
            if (!valid) continue;
            const uint32_t d0 = hsel * 64 + c * 16;
            if (direct) {
                __nv_bfloat16* dst = p.out + (size_t)qi * p.h + u.head * 128u + d0;
                uint4 a, b2;
                a.x = pack_bf16(__uint_as_float(o[0]) * inv, __uint_as_float(o[1]) * inv);
                a.y = pack_bf16(__uint_as_float(o[2]) * inv, __uint_as_float(o[3]) * inv);
                a.z = pack_bf16(__uint_as_float(o[4]) * inv, __uint_as_float(o[5]) * inv);
                a.w = pack_bf16(__uint_as_float(o[6]) * inv, __uint_as_float(o[7]) * inv);
                b2.x = pack_bf16(__uint_as_float(o[8]) * inv, __uint_as_float(o[9]) * inv);
                b2.y = pack_bf16(__uint_as_float(o[10]) * inv, __uint_as_float(o[11]) * inv);
                b2.z = pack_bf16(__uint_as_float(o[12]) * inv, __uint_as_float(o[13]) * inv);
                b2.w = pack_bf16(__uint_as_float(o[14]) * inv, __uint_as_float(o[15]) * inv);
                reinterpret_cast<uint4*>(dst)[0] = a;
                reinterpret_cast<uint4*>(dst)[1] = b2;
            } else {
                float4* dst = reinterpret_cast<float4*>(p.part_o + ((size_t)u.slot * 128 + r) * 128 + d0);
#pragma unroll
                for (uint32_t e = 0; e < 4; ++e)
                    dst[e] = make_float4(__uint_as_float(o[4 * e]), __uint_as_float(o[4 * e + 1]),
                                         __uint_as_float(o[4 * e + 2]), __uint_as_float(o[4 * e + 3]));
            }
        }
        if (valid && !direct && hsel == 0) p.part_ml[(size_t)u.slot * 128 + r] = make_float2(m_used, l);
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// Merge split partials of one (tile, head): O = sum_s 2^(m_s - M) O_s / sum_s 2^(m_s - M) l_s.
// One warp per query row (blockIdx.y picks 8 rows of the job), lanes along the head
// dimension: coalesced 512-B partial reads, 256-B bf16 output rows; all loads of a row
// are issued before they are consumed.
__global__ void __launch_bounds__(256) attn_combine_kernel(const AttnCombine* __restrict__ jobs,
                                                           const float* __restrict__ part_o,
                                                           const float2* __restrict__ part_ml,
                                                           uint32_t m, uint32_t h,
                                                           __nv_bfloat16* __restrict__ out) {
    constexpr uint32_t kMaxSplits = 16;
    const AttnCombine j = jobs[blockIdx.x];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t r = blockIdx.y * 8 + warp;
    const uint32_t qi = j.tile * 128u + r;
    if (qi >= m) return;
    const uint32_t n = min(j.n, kMaxSplits);
    float2 ml[kMaxSplits];
    float4 ov[kMaxSplits];
#pragma unroll
    for (uint32_t s = 0; s < kMaxSplits; ++s)
        if (s < n) {
            ml[s] = __ldcg(part_ml + (size_t)(j.slot0 + s) * 128 + r);
            ov[s] = __ldcs(reinterpret_cast<const float4*>(part_o + ((size_t)(j.slot0 + s) * 128 + r) * 128) + lane);
        }
    float M = -INFINITY;
#pragma unroll
    for (uint32_t s = 0; s < kMaxSplits; ++s)
        if (s < n) M = fmaxf(M, ml[s].x);
    float L = 0.0f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (uint32_t s = 0; s < kMaxSplits; ++s)
        if (s < n) {
            const float w = ml[s].x == -INFINITY ? 0.0f : exp2f(ml[s].x - M);
            L += w * ml[s].y;
            acc.x += w * ov[s].x;
            acc.y += w * ov[s].y;
            acc.z += w * ov[s].z;
            acc.w += w * ov[s].w;
        }
    const float inv = L > 0.0f ? 1.0f / L : 0.0f;
    uint2 pk;
    pk.x = pack_bf16(acc.x * inv, acc.y * inv);
    pk.y = pack_bf16(acc.z * inv, acc.w * inv);
    reinterpret_cast<uint2*>(out + (size_t)qi * h + j.head * 128u)[lane] = pk;
}

}  // namespace

// Host: split every (query tile, head) key range into units of at most `chunk` blocks.
AttnPlan plan_attention(const uint32_t* rows, uint32_t m, uint32_t n_heads) {
    AttnPlan plan;
    const uint32_t tiles = ceil_div(m, 128);
    std::vector<uint32_t> nblk(tiles);
    uint64_t total = 0;
    for (uint32_t t = 0; t < tiles; ++t) {
        const uint32_t last = std::min(m, (t + 1) * 128) - 1;
        nblk[t] = rows[last] / 128 + 1;
        total += (uint64_t)nblk[t] * n_heads;
    }
    // ~3 waves of units; never split below 2 blocks per unit
    uint32_t chunk = (uint32_t)std::max<uint64_t>(2, (total + 3 * kNumSMs - 1) / (3 * kNumSMs));
    uint32_t longest = 0;
    for (uint32_t t = 0; t < tiles; ++t) longest = std::max(longest, nblk[t]);
    chunk = std::max(chunk, ceil_div(longest, 16));  // the combine merges at most 16 splits
    uint32_t slot = 0;
    for (uint32_t t = 0; t < tiles; ++t) {
        const uint32_t splits = ceil_div(nblk[t], chunk);
        for (uint32_t hd = 0; hd < n_heads; ++hd) {
            if (splits > 1) plan.combine.push_back(AttnCombine{t, hd, slot, splits});
            for (uint32_t sp = 0; sp < splits; ++sp) {
                AttnUnit u;
                u.tile = t;
                u.head = hd;
                u.b0 = sp * chunk;
                u.b1 = std::min(nblk[t], (sp + 1) * chunk);
                u.slot = splits > 1 ? slot + sp : 0xffffffffu;
                plan.units.push_back(u);
            }
            if (splits > 1) slot += splits;
        }
    }
    plan.slots = slot;
    // Launch order = (head, key range, query tile): the query tiles that read the same K/V
    // blocks of a head run side by side, so each block comes from HBM once and the other
    // tiles hit it in L2 (a layer's K/V, 2*n*h*2 B = 154 MB at n=9418, exceeds the L2).
    std::stable_sort(plan.units.begin(), plan.units.end(), [](const AttnUnit& a, const AttnUnit& b) {
        if (a.head != b.head) return a.head < b.head;
        if (a.b0 != b.b0) return a.b0 < b.b0;
        return a.tile < b.tile;
    });
    return plan;
}

void launch_attn_tc(const __nv_bfloat16* q, const __nv_bfloat16* kcache, const __nv_bfloat16* vcache,
                    uint32_t n_ctx, const uint32_t* d_rows, uint32_t m, uint32_t H,
                    const AttnUnit* d_units, uint32_t n_units, const AttnCombine* d_combine,
                    uint32_t n_combine, float* part_o, float2* part_ml, __nv_bfloat16* out,
                    cudaStream_t s) {
    const uint32_t h = H * 128;
    const CUtensorMap tmQ = make_tmap_bf16(q, h, m, 64, 128);
    const CUtensorMap tmK = make_tmap_bf16(kcache, h, n_ctx, 64, 128);
    const CUtensorMap tmV = make_tmap_bf16(vcache, h, n_ctx, 64, 128);
    AttnParams p;
    p.units = d_units;
    p.rows = d_rows;
    p.m = m;
    p.h = h;
    p.scale_log2 = (1.0f / sqrtf(128.0f)) * 1.4426950408889634f;
    p.out = out;
    p.part_o = part_o;
    p.part_ml = part_ml;
    const size_t smem = (1 + 2 * kKvStages) * kTile + 1024 + (1 + 4 * kKvStages + 6) * 8 + 16;
    static bool attr = false;
    if (!attr) {
        MPIC_CUDA(cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    attn_tc_kernel<<<n_units, kAttnThreads, smem, s>>>(tmQ, tmK, tmV, p);
    MPIC_LAUNCHED();
    if (n_combine) {
        attn_combine_kernel<<<dim3(n_combine, 16), 256, 0, s>>>(d_combine, part_o, part_ml, m, h, out);
        MPIC_LAUNCHED();
    }
}

}  // namespace mpicb
