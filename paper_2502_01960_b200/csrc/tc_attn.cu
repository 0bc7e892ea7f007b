// K4 — selective causal attention on the 5th-gen tensor cores (head_dim 128).
//
// For recomputed row i (cache position rows[i]) and head hd, attend over cache keys
// [0, rows[i]] of the just-scattered layer cache (proj/src/linker.cpp:80-113): the
// per-row causal limit is the row's POSITION, not its index in the tile.
//
// Work item = one head x a range of 128-key blocks x one or two 128-query tiles that need
// those keys. The host splits long key ranges (flash-decoding style) so ~3 waves of items
// cover the 148 SMs; attn_combine_kernel merges split partials. One CTA per item with two
// LANES (FlashAttention-4 style ping-pong), each with its own softmax warpgroup, O
// accumulator and TWO S buffers, walking 64-key steps:
//   pair mode  (two query tiles) lane X = tile X over both key halves of every block; the
//              lanes share every K/V block the CTA loads
//   split mode (one query tile) both lanes take the tile, lane X the key half X of every
//              block (they share the block too); lane 1's (m, l, O) is merged into lane 0's
//              at the end
// S_X(s + 1) is computed while the softmax of step s runs (double-buffered S), so a softmax
// warpgroup never waits for the PV -> S round trip of its own lane.
//
//   warp 0     lane 0 TMA-loads the Q tile(s) once and K_j into a 2-stage ring; the warp
//              owns TMEM (512 cols: S_A[2] (64 each) | O_A | S_B[2] | O_B)
//   warp 1     lane 0 TMA-loads V_j into a 3-stage ring ([128 keys x 128] blocks)
//   warp 2     lane 0 issues every tcgen05.mma: S_X(s) = Q_X . K_half^T (SS, K-major, N = 64)
//              and O_X += P_X(s) . V_half (P from TMEM, V MN-major); per step, lane by lane,
//              PV_X(s) then S_X(s + 2) into the buffer P_X(s) occupied
//   warp 3     linker when chunk blocks are linked inside attention (kernels.h AttnLink):
//              TMA bulk stores of the loaded K/V blocks into the request cache
//   warps 4-7  softmax of lane 0, warps 8-11 of lane 1, 216 registers per thread: ONE
//              THREAD PER QUERY ROW holding its 64 scores (no cross-warp reduction), scale,
//              per-row causal mask, online max with lazy O rescaling (only when the max
//              grows by more than 2^8), exp2 with a quarter of the exponentials on the FMA
//              pipe (degree-3 polynomial, exact to bf16) and the rest on MUFU, row sums; P
//              written back over S in TMEM as bf16.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace mpicb {

CUtensorMap make_tmap_bf16(const void* ptr, uint64_t inner, uint64_t outer, uint32_t box_inner,
                           uint32_t box_outer);

namespace {

constexpr uint32_t kAttnThreads = 384;  // 3 warpgroups: control, softmax tile A, softmax tile B
constexpr uint32_t kCtrlRegs = 72, kSoftmaxRegs = 216;  // setmaxnreg split of the 168 x 384 launch registers
constexpr uint32_t kTile = 32 * 1024;   // one [128 x 128] bf16 tile as 2 swizzled 64-col halves
constexpr uint32_t kHalf = 16 * 1024;
constexpr uint32_t kKStages = 2;
constexpr uint32_t kVStages = 3;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
constexpr uint32_t kDbgCtaBase = 16 * 64, kDbgCtas = (16 * 4096 - kDbgCtaBase) / 8;  // MPIC_ATTN_TS layout

struct AttnParams {
    const AttnUnit* units;
    uint32_t n_units;
    const AttnCombine* combine;  // fused combine (counters != null): the jobs
    uint32_t* counters;          // per job: splits finished (the last one merges, then resets it)
    const uint32_t* rows;
    const uint32_t* starts;  // batched requests: first key row each query row may see (null: 0)
    uint32_t m;
    uint32_t shift;         // attn_tile_shift(m): tile t starts at selected row 128t - shift
    uint32_t h;
    float scale_log2;       // inv_sqrt_d * log2(e)
    __nv_bfloat16* out;     // [m][h]
    float* part_o;          // [slots][128][128]
    float2* part_ml;        // [slots][128] (m_used, l)
    unsigned long long* dbg;  // diagnostics: per-block event times of CTA 0, or null
    const AttnLink* link;     // linking inside attention (kernels.h), or null
    uint32_t layer;
    uint32_t link_nostore;    // diagnostics (MPIC_ATTN_LINK=2): read chunks, skip the stores
};

// Source of key block `blk` (absolute): the chunk map and row, or the request cache.
__device__ __forceinline__ const CUtensorMap* link_src(const AttnParams& p, const CUtensorMap* cache_map,
                                                       uint32_t blk, uint32_t K, int& row) {
    if (p.link) {
        const uint32_t code = reinterpret_cast<const uint32_t*>(p.link + 1)[blk];
        if (code != kLinkedBlock) {
            const uint32_t c = code >> 24;
            row = (int)(p.layer * p.link->tokens[c] + (code & 0xffffffu));
            return reinterpret_cast<const CUtensorMap*>(&p.link->maps[2 * c + K]);
        }
    }
    row = (int)(blk * 128u);
    return cache_map;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

#ifdef MPIC_ATTN_WATCHDOG  // diagnostics build: a wait that spins ~1 s reports where it hangs and traps
__device__ __noinline__ void wd_wait(uint64_t* bar, uint32_t parity, int tag, uint32_t a) {
    const long long t0 = clock64();
    uint32_t ok = 0;
    while (!ok) {
        asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.b32 %0, 1, 0, P1;\n}"
                     : "=r"(ok) : "r"(tc::smem_u32(bar)), "r"(parity) : "memory");
        if (!ok && clock64() - t0 > 2000000000ll) {
            printf("attn watchdog: cta %d warp %d lane %d tag %d arg %u parity %u\n", blockIdx.x, threadIdx.x / 32,
                   threadIdx.x % 32, tag, a, parity);
            asm volatile("trap;");
        }
    }
}
#define WD_WAIT(bar, par, tag, a) wd_wait(bar, par, tag, a)
#else
#define WD_WAIT(bar, par, tag, a) tc::mbar_wait(bar, par)
#endif

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&v);
}

// Packed fp32 pair ops (FFMA2 / FADD2 on sm_100): two elements per instruction.
struct f2 {
    unsigned long long v;
};
__device__ __forceinline__ f2 mk2(float a, float b) {
    return f2{(unsigned long long)__float_as_uint(a) | ((unsigned long long)__float_as_uint(b) << 32)};
}
__device__ __forceinline__ float lo(f2 a) { return __uint_as_float((uint32_t)a.v); }
__device__ __forceinline__ float hi(f2 a) { return __uint_as_float((uint32_t)(a.v >> 32)); }
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
    f2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d.v) : "l"(a.v), "l"(b.v), "l"(c.v));
    return d;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
    f2 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v));
    return d;
}

__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
    f2 d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v));
    return d;
}

// 2^x for two x <= 0 on the FMA/ALU pipes only (no F2I/FRND, which share the MUFU pipe):
// round x with the 1.5*2^23 magic constant (t's low mantissa bits are then round(x)), a
// degree-3 fit of 2^f on [-1/2, 1/2] (max rel. error 1.7e-4, below the bf16 rounding P gets
// next), and the exponent added in the integer domain: bits(p) + (bits(t) << 23), since the
// magic constant's own bits vanish under the shift. ~10 instructions per pair.
__device__ __forceinline__ f2 exp2_poly2(f2 x) {
    x = mk2(fmaxf(lo(x), -126.0f), fmaxf(hi(x), -126.0f));
    const f2 magic = mk2(12582912.0f, 12582912.0f);
    const f2 t = add2(x, magic);
    const f2 f = sub2(x, sub2(t, magic));
    f2 p = fma2(mk2(0.05302752f, 0.05302752f), f, mk2(0.24221394f, 0.24221394f));
    p = fma2(p, f, mk2(0.69357257f, 0.69357257f));
    p = fma2(p, f, mk2(1.0f, 1.0f));
    const uint32_t e0 = __float_as_uint(lo(t)) << 23, e1 = __float_as_uint(hi(t)) << 23;
    return mk2(__uint_as_float(__float_as_uint(lo(p)) + e0), __uint_as_float(__float_as_uint(hi(p)) + e1));
}

#ifndef MPIC_POLY_MASK
#define MPIC_POLY_MASK 0x88u  // exp pairs (of 8) on the FMA pipe: 2 of 8 = 25%
#endif

__global__ void __launch_bounds__(kAttnThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;                          // [2] tiles
    uint8_t* sK = smem + 2 * kTile;              // [kKStages]
    uint8_t* sV = sK + kKStages * kTile;         // [kVStages]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kVStages * kTile);
    uint64_t* q_full = bars;
    uint64_t* q_empty = q_full + 1;              // both MMA warps issued their item's last S
    uint64_t* k_full = q_empty + 1;              // [kKStages]
    uint64_t* k_empty = k_full + kKStages;
    uint64_t* v_full = k_empty + kKStages;       // [kVStages]
    uint64_t* v_empty = v_full + kVStages;
    uint64_t* s_full = v_empty + kVStages;       // [2 lanes][2 buffers]
    uint64_t* p_full = s_full + 4;               // [2 lanes][2 buffers]
    uint64_t* o_done = p_full + 4;               // [2 lanes] one phase per PV
    uint64_t* o_fin = o_done + 2;                // [2 lanes] the item's last PV
    uint64_t* o_free = o_fin + 2;                // [2 lanes] O read out by the epilogue
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(o_free + 2);
    float2* ml_x = reinterpret_cast<float2*>(tmem_holder + 4);  // [128] split mode: lane 1's (m, l)
    uint32_t* merge_flag = reinterpret_cast<uint32_t*>(ml_x + 128);  // [2] fused combine: this lane merges

    tc::pdl_trigger();
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        tc::tma_prefetch_desc(&tmQ);
        tc::tma_prefetch_desc(&tmK);
        tc::tma_prefetch_desc(&tmV);
        tc::mbar_init(q_full, 1);
        tc::mbar_init(q_empty, 2);
        // a K/V stage is free once both MMA warps' reads of it are done and, with linking,
        // the linker has finished storing it (or passed it)
        const uint32_t empties = p.link ? 3u : 2u;  // both MMA warps (+ the linker)
        for (uint32_t i = 0; i < kKStages; ++i) {
            tc::mbar_init(&k_full[i], 1);
            tc::mbar_init(&k_empty[i], empties);
        }
        for (uint32_t i = 0; i < kVStages; ++i) {
            tc::mbar_init(&v_full[i], 1);
            tc::mbar_init(&v_empty[i], empties);
        }
        for (int i = 0; i < 4; ++i) {
            tc::mbar_init(&s_full[i], 1);
            tc::mbar_init(&p_full[i], 128);
        }
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&o_done[i], 1);
            tc::mbar_init(&o_fin[i], 1);
            tc::mbar_init(&o_free[i], 128);
        }
        tc::fence_barrier_init();
    }
    if (warp == 0) tc::tmem_alloc(tmem_holder, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    tc::pdl_wait();  // q and the layer's K/V come from the previous kernel
    const uint32_t tmem = *tmem_holder;
    if (p.dbg && threadIdx.x == 0 && blockIdx.x < kDbgCtas) {  // diagnostics: per-CTA span and SM
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        p.dbg[kDbgCtaBase + 8 * blockIdx.x] = globaltimer_ns();
        p.dbg[kDbgCtaBase + 8 * blockIdx.x + 2] = smid;
    }
    // Persistent CTA: the items the host assigned to this CTA (longest-processing-time over
    // the estimated costs, plan_attention). Every role walks the same item sequence with
    // running block / step / item counters, so barrier phases continue across items and the
    // next item's Q/K/V loads and first S MMAs overlap the current item's tail and epilogue.
    const uint32_t* cta_off = attn_cta_offsets(p.units, p.n_units);
    const uint32_t it_begin = cta_off[blockIdx.x], it_end = cta_off[blockIdx.x + 1];
    auto item_at = [&](uint32_t r) { return it_begin + r < it_end ? it_begin + r : p.n_units; };
    // Two lanes (X = 0, 1), each with its own softmax warpgroup, O accumulator and two S
    // buffers, walk 64-key steps. Pair mode (two query tiles): lane X = tile X over every
    // half-block of its range, step s = half s & 1 of block s >> 1. Split mode (one tile):
    // both lanes take the tile, lane X the key half X of every block, step s = block s;
    // their (m, l, O) are merged at the end.
    struct Item {
        AttnUnit u;
        bool split;
        uint32_t nb0, nb1, nblk, nst[2];
        int hcol;
    };
    auto item = [&](uint32_t idx) {
        Item it;
        it.u = p.units[idx];
        it.split = it.u.tile[1] == kNoTile;
        it.nb0 = it.u.b1[0] - it.u.b0;
        it.nb1 = it.split ? it.nb0 : it.u.b1[1] - it.u.b0;
        it.nblk = max(it.nb0, it.nb1);
        it.nst[0] = it.split ? it.nb0 : 2 * it.nb0;
        it.nst[1] = it.split ? it.nb0 : 2 * it.nb1;
        it.hcol = (int)(it.u.head * 128u);
        return it;
    };
    // TMEM columns: lane X uses S_X[b] = [256X + 64b, +64) and O_X = [256X + 128, +128).
    // P_X (bf16, two keys per column) overwrites the first 32 columns of its S buffer.
    constexpr uint32_t idesc_s = tc::idesc_bf16(128, 64, false);
    constexpr uint32_t idesc_o = tc::idesc_bf16(128, 128, true);

    // Each role owns a whole warp: roles sharing a warp diverge, and a lane sleeping in an
    // mbarrier try_wait holds back the other paths of its warp.
    // setmaxnreg inside the role branches: ptxas sizes each branch by the limit that
    // dominates it (set before a join, the softmax got the control warps' limit and spilled)
    if (warp < 4) tc::reg_dealloc<kCtrlRegs>();
    if (warp == 0) {
        // lane 0: per item the Q tile(s) (once both MMA warps issued the previous item's
        // last S), then K_j and V_j of every block in order (K into a 2-stage, V into a
        // 3-stage ring: V_j's slot frees long before K_{j+2} is needed)
        if (lane == 0) {
            if (p.link)
                for (uint32_t c = 0; c < 2 * kMaxLinkChunks; ++c) tc::tensormap_acquire(&p.link->maps[c]);
            uint32_t gb = 0;  // blocks loaded so far (all items)
            for (uint32_t ni = 0, idx; (idx = item_at(ni)) < p.n_units; ++ni) {
                const Item it = item(idx);
                if (ni > 0) WD_WAIT(q_empty, (ni - 1) & 1, 13, ni);
                tc::mbar_arrive_expect_tx(q_full, (it.split ? 1 : 2) * kTile);
#pragma unroll
                for (uint32_t x = 0; x < 2; ++x) {
                    if (x == 1 && it.split) break;
                    // tile 0 may start at a negative row: TMA zero-fills the rows outside [0, m)
                    const int q0 = (int)(it.u.tile[x] * 128u) - (int)p.shift;
                    tc::tma_load_2d(sQ + x * kTile, &tmQ, q_full, it.hcol, q0);
                    tc::tma_load_2d(sQ + x * kTile + kHalf, &tmQ, q_full, it.hcol + 64, q0);
                }
                for (uint32_t j = 0; j < it.nblk; ++j, ++gb) {
                    int j0;
                    const uint32_t sk = gb % kKStages, sv = gb % kVStages;
                    const CUtensorMap* srck = link_src(p, &tmK, it.u.b0 + j, 0, j0);
                    WD_WAIT(&k_empty[sk], ((gb / kKStages) & 1) ^ 1, 1, gb);
                    tc::mbar_arrive_expect_tx(&k_full[sk], kTile);
                    tc::tma_load_2d(sK + sk * kTile, srck, &k_full[sk], it.hcol, j0);
                    tc::tma_load_2d(sK + sk * kTile + kHalf, srck, &k_full[sk], it.hcol + 64, j0);
                    const CUtensorMap* srcv = link_src(p, &tmV, it.u.b0 + j, 1, j0);
                    WD_WAIT(&v_empty[sv], ((gb / kVStages) & 1) ^ 1, 2, gb);
                    tc::mbar_arrive_expect_tx(&v_full[sv], kTile);
                    tc::tma_load_2d(sV + sv * kTile, srcv, &v_full[sv], it.hcol, j0);
                    tc::tma_load_2d(sV + sv * kTile + kHalf, srcv, &v_full[sv], it.hcol + 64, j0);
                }
            }
        }
        __syncwarp();
    } else if (warp <= 2) {
        // MMA warps: warp 1 issues lane 0's MMAs, warp 2 lane 1's, so one lane's waits
        // never stall the other lane's MMAs (the tensor pipe queues only ~4 MMAs, and a
        // single issuer's per-step bookkeeping left it idle ~40% of the time). All 32 lanes
        // run the control flow (warp-uniform: descriptors in uniform registers); lane 0
        // polls the barriers (then __syncwarp), one elected lane issues. Per step s: PV_x(s)
        // once P_x(s) is written, then S_x(s + 2) into the buffer P_x(s) occupied (in-order
        // after the PV that reads it), so the softmax finds S_x(s + 1) computed while it
        // works on step s. A K/V stage needs one release (commit) from each MMA warp.
        const uint32_t x = warp - 1;
        // running counters over the CTA's items: blocks (K/V stage and phase), steps of this
        // lane (S/P buffer and phase; one PV per step: o_done phase)
        uint32_t gb0 = 0, sg0 = 0;
        uint32_t k_avail = 0, v_avail = 0, k_rel = 0, v_rel = 0;  // global block indices
        for (uint32_t ni = 0, idx; (idx = item_at(ni)) < p.n_units; ++ni) {
            const Item it = item(idx);
            const uint32_t ns = it.nst[x], nblk = it.nblk;
            const bool split = it.split;
            const bool stamp = lane == 0 && p.dbg && blockIdx.x == 0 && x == 0 && ni == 0;
            auto blk_of = [&](uint32_t s) { return split ? s : s >> 1; };
            auto half_of = [&](uint32_t s) { return split ? x : s & 1u; };
            auto need_k = [&](uint32_t j) {  // local block j has landed
                for (; k_avail <= gb0 + j; ++k_avail)
                    if (lane == 0) WD_WAIT(&k_full[k_avail % kKStages], (k_avail / kKStages) & 1, 3, k_avail);
            };
            auto need_v = [&](uint32_t j) {
                for (; v_avail <= gb0 + j; ++v_avail)
                    if (lane == 0) WD_WAIT(&v_full[v_avail % kVStages], (v_avail / kVStages) & 1, 4, v_avail);
            };
            const uint32_t qa = tc::smem_u32(sQ + (split ? 0u : x) * kTile);
            auto issue_s = [&](uint32_t s) {
                const uint32_t jg = gb0 + blk_of(s), sg = sg0 + s;
                const uint32_t ka = tc::smem_u32(sK + (jg % kKStages) * kTile) + half_of(s) * 8192u;  // keys [64h, +64)
                if (tc::elect_one_sync()) {
#pragma unroll
                    for (uint32_t kk = 0; kk < 8; ++kk) {
                        const uint32_t off = (kk >> 2) * kHalf + (kk & 3) * 32;
                        tc::mma_bf16(tmem + x * 256 + (sg & 1) * 64, tc::desc_k_sw128(qa + off),
                                     tc::desc_k_sw128(ka + off), idesc_s, kk > 0 ? 1u : 0u);
                    }
                    tc::mma_commit(&s_full[2 * x + (sg & 1)]);
                    if (s + 1 == ns) tc::mma_commit(q_empty);  // the item's Q is no longer read
                }
            };
            auto issue_pv = [&](uint32_t s) {
                const uint32_t jg = gb0 + blk_of(s), sg = sg0 + s;
                const uint32_t va = tc::smem_u32(sV + (jg % kVStages) * kTile) + half_of(s) * 8192u;
                if (tc::elect_one_sync()) {
#pragma unroll
                    for (uint32_t kk = 0; kk < 4; ++kk)  // A = P_x(s) from TMEM: 16 keys = 8 packed columns
                        tc::mma_bf16_ts(tmem + x * 256 + 128, tmem + x * 256 + (sg & 1) * 64 + kk * 8,
                                        tc::desc_mn_sw128(va + kk * 2048, kHalf), idesc_o, (s > 0 || kk > 0) ? 1u : 0u);
                    tc::mma_commit(&o_done[x]);
                    if (s + 1 == ns) tc::mma_commit(&o_fin[x]);
                }
            };
            // release every block below the lowest block a later MMA of this lane still reads.
            // A block this lane never reads (pair mode, the other tile's longer range) is
            // released only once it has landed: an early arrival would count towards the
            // stage's previous phase and free it under the other lane's MMAs.
            auto release = [&](uint32_t next_s, uint32_t next_pv) {
                const uint32_t lk = gb0 + (next_s < ns ? blk_of(next_s) : nblk);
                const uint32_t lv = gb0 + (next_pv < ns ? blk_of(next_pv) : nblk);
                const uint32_t used = gb0 + min(blk_of(ns - 1) + 1, nblk);  // blocks this lane reads
                if (tc::elect_one_sync()) {
                    for (uint32_t j = k_rel; j < min(lk, used); ++j) tc::mma_commit(&k_empty[j % kKStages]);
                    for (uint32_t j = v_rel; j < min(lv, used); ++j) tc::mma_commit(&v_empty[j % kVStages]);
                }
                k_rel = max(k_rel, min(lk, used));
                v_rel = max(v_rel, min(lv, used));
                // blocks it never reads: released after the lane's last MMA, in the producer's
                // load order (K_j, V_j, K_j+1, ...), each once it has landed (never while this
                // lane still has PVs to issue: the other lane could be waiting for a V stage
                // only this lane's release frees)
                if (next_pv < ns) return;
                while (k_rel < lk || v_rel < lv) {
                    const bool do_k = k_rel < lk && (v_rel >= lv || k_rel <= v_rel);
                    if (do_k) {
                        need_k(k_rel - gb0);
                        __syncwarp();
                        if (tc::elect_one_sync()) tc::mma_commit(&k_empty[k_rel % kKStages]);
                        ++k_rel;
                    } else {
                        need_v(v_rel - gb0);
                        __syncwarp();
                        if (tc::elect_one_sync()) tc::mma_commit(&v_empty[v_rel % kVStages]);
                        ++v_rel;
                    }
                }
            };
            if (lane == 0) WD_WAIT(q_full, ni & 1, 5, ni);
            need_k(blk_of(min(2u, ns) - 1));
            __syncwarp();
            tc::tc_fence_after();
            issue_s(0);
            if (ns > 1) issue_s(1);
            release(2, 0);
            for (uint32_t s = 0; s < ns; ++s) {
                if (stamp && s < 64) {
                    p.dbg[s * 16 + 0] = globaltimer_ns();
                    p.dbg[s * 16 + 14] = clock64();
                }
                const uint32_t sg = sg0 + s;
                if (lane == 0) {
                    WD_WAIT(&p_full[2 * x + (sg & 1)], (sg >> 1) & 1, 6, sg);
                    // the first PV overwrites O: the previous item's epilogue must have read it
                    if (s == 0 && ni > 0) WD_WAIT(&o_free[x], (ni - 1) & 1, 14, ni);
                }
                need_v(blk_of(s));
                if (s + 2 < ns) need_k(blk_of(s + 2));
                __syncwarp();
                tc::tc_fence_after();
                if (stamp && s < 64) p.dbg[s * 16 + 1] = globaltimer_ns();
                issue_pv(s);
                if (s + 2 < ns) issue_s(s + 2);
                release(s + 3, s + 1);
                if (stamp && s < 64) p.dbg[s * 16 + 2] = globaltimer_ns();
            }
            gb0 += nblk;
            sg0 += ns;
        }
        __syncwarp();
    } else if (warp == 3) {
        if (p.link && lane == 0) {
            // ---- linker (warp 3, one thread): TMA-stores the chunk-sourced K/V blocks its
            // items are the writer of from the stage buffers into the request cache (the cache
            // tensor maps have the stage's 128-B swizzle, so a block is two bulk stores and no
            // thread touches the data), then releases the stage once the stores have read it.
            // Writer of block b = the item streaming b for the lowest query tile reaching b.
            const uint32_t* blk = reinterpret_cast<const uint32_t*>(p.link + 1);
            const uint16_t* wtile = reinterpret_cast<const uint16_t*>(blk + p.link->nblk);
            // One store group stays in flight: a stage is released once the NEXT store has
            // been issued and the one before it has finished reading shared memory.
            uint64_t* pending = nullptr;
            auto stored = [&](uint64_t* empty_bar) {
                tc::bulk_commit_group();
                tc::bulk_wait_group_read<1>();
                if (pending) tc::mbar_arrive(pending);
                pending = empty_bar;
            };
            // a block without stores releases at once; the held stage goes first (its release
            // must not wait for a later store: the producer may need that stage before then)
            auto passed = [&](uint64_t* empty_bar) {
                if (pending) {
                    tc::bulk_wait_group_read<0>();
                    tc::mbar_arrive(pending);
                    pending = nullptr;
                }
                tc::mbar_arrive(empty_bar);
            };
            uint32_t gb = 0;
            for (uint32_t ni = 0, idx; (idx = item_at(ni)) < p.n_units; ++ni) {
                const Item it = item(idx);
                for (uint32_t j = 0; j < it.nblk; ++j, ++gb) {
                    const uint32_t b = it.u.b0 + j, wt = wtile[b];
                    const bool mine = (it.u.tile[0] == wt && j < it.nb0) || (!it.split && it.u.tile[1] == wt && j < it.nb1);
                    const bool store = mine && blk[b] != kLinkedBlock && !p.link_nostore;
                    const uint32_t sk = gb % kKStages, sv = gb % kVStages;
                    WD_WAIT(&k_full[sk], (gb / kKStages) & 1, 7, gb);
                    if (store) {
                        tc::tma_store_2d(&tmK, sK + sk * kTile, it.hcol, (int)(b * 128u));
                        tc::tma_store_2d(&tmK, sK + sk * kTile + kHalf, it.hcol + 64, (int)(b * 128u));
                        stored(&k_empty[sk]);
                    } else {
                        passed(&k_empty[sk]);
                    }
                    WD_WAIT(&v_full[sv], (gb / kVStages) & 1, 8, gb);
                    if (store) {
                        tc::tma_store_2d(&tmV, sV + sv * kTile, it.hcol, (int)(b * 128u));
                        tc::tma_store_2d(&tmV, sV + sv * kTile + kHalf, it.hcol + 64, (int)(b * 128u));
                        stored(&v_empty[sv]);
                    } else {
                        passed(&v_empty[sv]);
                    }
                }
            }
            tc::bulk_wait_group_read<0>();
            if (pending) tc::mbar_arrive(pending);
            tc::bulk_wait_group<0>();  // the stores are complete before the CTA exits
        }
        __syncwarp();
    } else {
        tc::reg_alloc<kSoftmaxRegs>();
        // ---- softmax: lane x = warp / 4 - 1, one thread per query row (TMEM lane)
        const uint32_t x = (warp >> 2) - 1;
        const uint32_t quarter = warp & 3;
        const uint32_t r = quarter * 32 + lane;
        const uint32_t lane_base = (quarter * 32u) << 16;
        const uint32_t o_col = tmem + lane_base + x * 256 + 128;
        uint32_t sg0 = 0;
        for (uint32_t ni = 0, idx; (idx = item_at(ni)) < p.n_units; ++ni) {
            const Item it = item(idx);
            const bool split = it.split;
            const uint32_t ns_x = it.nst[x];
            const uint32_t tile_x = split ? it.u.tile[0] : it.u.tile[x];
            const uint32_t slot_x = split ? it.u.slot[0] : it.u.slot[x];
            const uint32_t qi = tile_x * 128u + r - p.shift;  // wraps (invalid) for r < shift in tile 0
            const bool valid = tile_x * 128u + r >= p.shift && qi < p.m;
            const uint32_t limit = valid ? p.rows[qi] : 0u;
            const uint32_t first = valid && p.starts ? p.starts[qi] : 0u;  // its request's first cache row
            float m_used = -INFINITY, l = 0.0f;
            for (uint32_t s = 0; s < ns_x; ++s) {
                const uint32_t sg = sg0 + s;
                const uint32_t k0 = (it.u.b0 + (split ? s : s >> 1)) * 128u + 64u * (split ? x : s & 1u);
                const uint32_t s_col = tmem + lane_base + x * 256 + (sg & 1) * 64;
                if (lane == 0) WD_WAIT(&s_full[2 * x + (sg & 1)], (sg >> 1) & 1, 9, sg);  // one poller per warp
                __syncwarp();
                const bool dbg_me = p.dbg && blockIdx.x == 0 && ni == 0 && x == 0 && r == 0 && s < 64;
                if (dbg_me) p.dbg[s * 16 + 5] = globaltimer_ns();
                if (p.dbg && blockIdx.x == 0 && ni == 0 && x == 1 && r == 0 && s < 64) p.dbg[s * 16 + 10] = globaltimer_ns();
                tc::tc_fence_after();
                // keys [ns, nv) of the 64-key step are visible to this row: the causal limit is
                // the row's position (an invalid row sees none), and batched requests also mask
                // the rows of other requests' caches below `first`. Selected rows are scattered
                // over the prompt, so a warp often sees few or none of a step's keys: 32-key
                // chunks no lane of the warp sees are neither loaded nor exponentiated (P = 0),
                // and a warp that sees nothing just writes P = 0.
                const uint32_t ns = first > k0 ? min(first - k0, 64u) : 0u;
                uint32_t nv = !valid || limit < k0 ? 0u : min(limit - k0 + 1u, 64u);
                if (ns >= nv) nv = 0u;
                // common case (every row of the warp sees the whole step): one vote instead
                // of two warp reductions
                const bool all_full = __all_sync(0xffffffffu, nv == 64u && ns == 0u);
                const uint32_t nv_max = all_full ? 64u : __reduce_max_sync(0xffffffffu, nv);
                const uint32_t nv_min = all_full ? 64u : __reduce_min_sync(0xffffffffu, nv);
                if (nv_max == 0) {
                    uint32_t z[16];
#pragma unroll
                    for (uint32_t e = 0; e < 16; ++e) z[e] = 0u;
                    tc::tmem_st16(s_col, z);
                    tc::tmem_st16(s_col + 16, z);
                    tc::tmem_st_wait();
                    tc::tc_fence_before();
                    tc::mbar_arrive(&p_full[2 * x + (sg & 1)]);
                    continue;
                }
                const uint32_t nch = (nv_max + 31) >> 5;  // warp-uniform: 1 or 2
                uint32_t v[2][32];
                if (nch > 1) tc::tmem_ld64(s_col, v[0], v[1]);
                else tc::tmem_ld32(s_col, v[0]);
                tc::tmem_ld_wait();
                if (dbg_me) p.dbg[s * 16 + 8] = globaltimer_ns();
#pragma unroll
                for (uint32_t c = 0; c < 2; ++c) {
                    if (c < nch && nv_min < 32 * (c + 1)) {  // a lane's limit falls in this chunk
#pragma unroll
                        for (uint32_t e = 0; e < 32; ++e)
                            if (32 * c + e >= nv) v[c][e] = __float_as_uint(-INFINITY);
                    }
                }
                if (p.starts && __any_sync(0xffffffffu, ns > 0u)) {  // batched: below the request's start
#pragma unroll
                    for (uint32_t c = 0; c < 2; ++c)
                        if (c < nch) {
#pragma unroll
                            for (uint32_t e = 0; e < 32; ++e)
                                if (32 * c + e < ns) v[c][e] = __float_as_uint(-INFINITY);
                        }
                }
                float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
                for (uint32_t e = 0; e < 32; e += 2) {
                    mx0 = fmaxf(mx0, __uint_as_float(v[0][e]));
                    mx1 = fmaxf(mx1, __uint_as_float(v[0][e + 1]));
                }
                if (nch > 1) {
#pragma unroll
                    for (uint32_t e = 0; e < 32; e += 2) {
                        mx2 = fmaxf(mx2, __uint_as_float(v[1][e]));
                        mx3 = fmaxf(mx3, __uint_as_float(v[1][e + 1]));
                    }
                }
                const float mx = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)) * p.scale_log2;
                if (dbg_me) p.dbg[s * 16 + 7] = globaltimer_ns();
                float alpha = 1.0f;
                const bool grow = mx > m_used + kRescaleThreshold || (m_used == -INFINITY && mx > -INFINITY);
                if (grow) {
                    alpha = m_used == -INFINITY ? 0.0f : tc::ex2_approx(m_used - mx);
                    m_used = mx;
                    l *= alpha;
                }
                if (s > 0 && __any_sync(0xffffffffu, grow && alpha != 1.0f)) {
                    // every earlier PV of this item must have landed before O is rescaled (S_X(s)
                    // completing implies PV_X(s - 2) did, so only PV s - 1's phase can be pending)
                    if (lane == 0) WD_WAIT(&o_done[x], (sg - 1) & 1, 10, sg);
                    __syncwarp();
                    tc::tc_fence_after();
#pragma unroll
                    for (uint32_t c = 0; c < 128; c += 32) {
                        uint32_t o[32];
                        tc::tmem_ld32(o_col + c, o);
                        tc::tmem_ld_wait();
#pragma unroll
                        for (uint32_t e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
                        tc::tmem_st32(o_col + c, o);
                    }
                    tc::tmem_st_wait();
                }
                const float neg_m = m_used == -INFINITY ? 0.0f : -m_used;
                f2 lsum = mk2(0.f, 0.f);
                const f2 sc2 = mk2(p.scale_log2, p.scale_log2), nm2 = mk2(neg_m, neg_m);
#pragma unroll
                for (uint32_t c = 0; c < 2; ++c) {
                    // exp2(s * scale - m) in packed pairs, a quarter of them on the FMA pipe
                    // (balances the MUFU and issue budgets); masked keys give exactly 0. P (bf16
                    // pairs) goes to TMEM columns [16c, 16c + 16) of the step's S buffer (whose
                    // scores are all in registers by now).
                    uint32_t pk[16];
                    if (c < nch) {
#pragma unroll
                        for (uint32_t e = 0; e < 32; e += 2) {
                            const f2 xs = fma2(mk2(__uint_as_float(v[c][e]), __uint_as_float(v[c][e + 1])), sc2, nm2);
                            f2 ex;
                            if ((MPIC_POLY_MASK >> ((e >> 1) & 7)) & 1u) ex = exp2_poly2(xs);
                            else ex = mk2(tc::ex2_approx(lo(xs)), tc::ex2_approx(hi(xs)));
                            lsum = add2(lsum, ex);
                            pk[e >> 1] = pack_bf16(lo(ex), hi(ex));
                        }
                    } else {
#pragma unroll
                        for (uint32_t e = 0; e < 16; ++e) pk[e] = 0u;
                    }
                    tc::tmem_st16(s_col + c * 16, pk);
                }
                if (dbg_me) p.dbg[s * 16 + 9] = globaltimer_ns();
                l += lo(lsum) + hi(lsum);
                tc::tmem_st_wait();
                tc::tc_fence_before();
                if (dbg_me) p.dbg[s * 16 + 6] = globaltimer_ns();
                if (p.dbg && blockIdx.x == 0 && ni == 0 && x == 1 && r == 0 && s < 64) p.dbg[s * 16 + 11] = globaltimer_ns();
                tc::mbar_arrive(&p_full[2 * x + (sg & 1)]);
            }
            sg0 += ns_x;
            // ---- epilogue: O / l, or the unnormalised partial + (m, l) for the combine. Split
            // mode: lane 1 hands its (m, l) over through shared memory and lane 0 merges both
            // accumulators (same TMEM lanes) into the tile's result. Whoever reads an O
            // releases it (o_free) to the next item's first PV.
            // A barrier of its own for the last PV: with S double-buffered, o_done can be one
            // phase behind or already past the last PV here, and its parity cannot tell which.
            if (lane == 0) WD_WAIT(&o_fin[x], ni & 1, 12, ni);
            __syncwarp();
            tc::tc_fence_after();
            const bool cta_stamp = ni == 0 && x == 0 && r == 0 && p.dbg && blockIdx.x < kDbgCtas;
            if (cta_stamp) p.dbg[kDbgCtaBase + 8 * blockIdx.x + 5] = globaltimer_ns();
            float wa = 1.0f, wb = 0.0f;
            if (split) {
                if (x == 1) ml_x[r] = make_float2(m_used, l);
                tc::named_bar_sync(1, 256);
                if (x == 1) continue;  // lane 0 reads (and releases) both accumulators
                const float2 mb = ml_x[r];
                const float M = fmaxf(m_used, mb.x);
                wa = m_used == -INFINITY ? 0.0f : tc::ex2_approx(m_used - M);
                wb = mb.x == -INFINITY ? 0.0f : tc::ex2_approx(mb.x - M);
                l = wa * l + wb * mb.y;
                m_used = M;
            }
            const bool direct = slot_x == kNoTile;
            const float inv = l > 0.0f ? 1.0f / l : 0.0f;
            const uint32_t o_col_b = tmem + lane_base + 256 + 128;  // lane 1's O (split mode)
#pragma unroll 1
            for (uint32_t c = 0; c < 128; c += 32) {
                uint32_t o[32];
                tc::tmem_ld32(o_col + c, o);
                if (split) {
                    uint32_t ob[32];
                    tc::tmem_ld32(o_col_b + c, ob);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (uint32_t e = 0; e < 32; ++e)
                        o[e] = __float_as_uint(wa * __uint_as_float(o[e]) + wb * __uint_as_float(ob[e]));
                } else {
                    tc::tmem_ld_wait();
                }
                if (c + 32 == 128) {  // every O column of this thread is in registers
                    tc::tc_fence_before();
                    tc::mbar_arrive(&o_free[x]);
                    if (split) tc::mbar_arrive(&o_free[1]);
                }
                if (!valid) continue;
                if (direct) {
                    uint4* dst = reinterpret_cast<uint4*>(p.out + (size_t)qi * p.h + it.u.head * 128u + c);
#pragma unroll
                    for (uint32_t q = 0; q < 4; ++q) {
                        uint4 w;
                        w.x = pack_bf16(__uint_as_float(o[8 * q + 0]) * inv, __uint_as_float(o[8 * q + 1]) * inv);
                        w.y = pack_bf16(__uint_as_float(o[8 * q + 2]) * inv, __uint_as_float(o[8 * q + 3]) * inv);
                        w.z = pack_bf16(__uint_as_float(o[8 * q + 4]) * inv, __uint_as_float(o[8 * q + 5]) * inv);
                        w.w = pack_bf16(__uint_as_float(o[8 * q + 6]) * inv, __uint_as_float(o[8 * q + 7]) * inv);
                        dst[q] = w;
                    }
                } else {
                    // partial layout [slot][32 float4 columns][128 rows]: a warp's 32 rows of one
                    // float4 column are 512 contiguous bytes (one coalesced store per column)
                    float4* dst = reinterpret_cast<float4*>(p.part_o) + ((size_t)slot_x * 32 + c / 4) * 128 + r;
#pragma unroll
                    for (uint32_t e = 0; e < 8; ++e)
                        __stcg(dst + (size_t)e * 128, make_float4(__uint_as_float(o[4 * e]), __uint_as_float(o[4 * e + 1]),
                                                                  __uint_as_float(o[4 * e + 2]), __uint_as_float(o[4 * e + 3])));
                }
            }
            if (valid && !direct) p.part_ml[(size_t)slot_x * 128 + r] = make_float2(m_used, l);
            if (!direct && p.counters) {
                // fused combine: the split that completes its (tile, head) job merges it —
                // O = sum_s 2^(m_s - M) O_s / sum_s 2^(m_s - M) l_s over the job's partial slots
                // (L2-coherent loads: the other splits were written by other SMs)
                const uint32_t job = split ? it.u.job[0] : it.u.job[x];
                __threadfence();
                tc::named_bar_sync(2 + x, 128);
                if (r == 0) {
                    const AttnCombine jb = p.combine[job];
                    merge_flag[x] = atomicAdd(&p.counters[job], 1u) + 1u == jb.n ? 1u : 0u;
                }
                tc::named_bar_sync(2 + x, 128);
                if (merge_flag[x]) {
                    __threadfence();
                    const AttnCombine jb = p.combine[job];
                    const uint32_t n = min(jb.n, 16u);
                    float wt[16];
                    float M = -INFINITY, L = 0.0f;
#pragma unroll
                    for (uint32_t s2 = 0; s2 < 16; ++s2)
                        if (s2 < n) {
                            const float2 ml = __ldcg(p.part_ml + (size_t)(jb.slot0 + s2) * 128 + r);
                            wt[s2] = ml.x;
                            M = fmaxf(M, ml.x);
                        }
#pragma unroll
                    for (uint32_t s2 = 0; s2 < 16; ++s2)
                        if (s2 < n) {
                            const float2 ml = __ldcg(p.part_ml + (size_t)(jb.slot0 + s2) * 128 + r);
                            wt[s2] = ml.x == -INFINITY ? 0.0f : exp2f(ml.x - M);
                            L += wt[s2] * ml.y;
                        }
                    const float invL = L > 0.0f ? 1.0f / L : 0.0f;
                    const float4* po = reinterpret_cast<const float4*>(p.part_o) + (size_t)jb.slot0 * 32 * 128 + r;
#pragma unroll 1
                    for (uint32_t c8 = 0; c8 < 32; c8 += 8) {  // 8 float4 columns (32 dims) at a time
                        float4 acc[8];
#pragma unroll
                        for (uint32_t e = 0; e < 8; ++e) acc[e] = make_float4(0.f, 0.f, 0.f, 0.f);
                        for (uint32_t s2 = 0; s2 < n; ++s2) {
                            float w = 0.0f;
#pragma unroll
                            for (uint32_t i = 0; i < 16; ++i)
                                if (i == s2) w = wt[i];
#pragma unroll
                            for (uint32_t e = 0; e < 8; ++e) {
                                const float4 v4 = __ldcg(po + ((size_t)s2 * 32 + c8 + e) * 128);
                                acc[e].x += w * v4.x;
                                acc[e].y += w * v4.y;
                                acc[e].z += w * v4.z;
                                acc[e].w += w * v4.w;
                            }
                        }
                        if (valid) {
                            uint4* dst = reinterpret_cast<uint4*>(p.out + (size_t)qi * p.h + it.u.head * 128u + c8 * 4);
#pragma unroll
                            for (uint32_t q = 0; q < 4; ++q) {
                                uint4 w4;
                                w4.x = pack_bf16(acc[2 * q].x * invL, acc[2 * q].y * invL);
                                w4.y = pack_bf16(acc[2 * q].z * invL, acc[2 * q].w * invL);
                                w4.z = pack_bf16(acc[2 * q + 1].x * invL, acc[2 * q + 1].y * invL);
                                w4.w = pack_bf16(acc[2 * q + 1].z * invL, acc[2 * q + 1].w * invL);
                                dst[q] = w4;
                            }
                        }
                    }
                    if (r == 0) p.counters[job] = 0u;  // reset for the next launch
                }
            }
            if (cta_stamp) p.dbg[kDbgCtaBase + 8 * blockIdx.x + 6] = globaltimer_ns();
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (warp == 0) tc::tmem_dealloc(tmem, 512);
    if (p.dbg && threadIdx.x == 0 && blockIdx.x < kDbgCtas) p.dbg[kDbgCtaBase + 8 * blockIdx.x + 1] = globaltimer_ns();
}

// Merge split partials of one (tile, head): O = sum_s 2^(m_s - M) O_s / sum_s 2^(m_s - M) l_s.
// A thread per (row, float4 column) of the job (blockIdx.y picks 256 of its 128 x 32): lanes
// run along the rows, so every partial read is a coalesced 512-B line per warp ([slot][32
// float4 columns][128 rows], as the attention kernel writes them). Few registers per
// thread (the (m, l) pass first, then the partials four splits at a time) so that several
// CTAs share an SM: the kernel is a short burst of latency-bound warps.
__global__ void __launch_bounds__(256, 6) attn_combine_kernel(const AttnCombine* __restrict__ jobs,
                                                              const float* __restrict__ part_o,
                                                              const float2* __restrict__ part_ml,
                                                              uint32_t m, uint32_t shift, uint32_t h,
                                                              __nv_bfloat16* __restrict__ out) {
    constexpr uint32_t kMaxSplits = 16;
    tc::pdl_trigger();
    tc::pdl_wait();
    const AttnCombine j = jobs[blockIdx.x];
    const uint32_t t = blockIdx.y * 256 + threadIdx.x;
    const uint32_t r = t & 127, col4 = t >> 7;
    if (j.tile * 128u + r < shift) return;
    const uint32_t qi = j.tile * 128u + r - shift;
    if (qi >= m) return;
    const uint32_t n = min(j.n, kMaxSplits);
    const float2* ml = part_ml + (size_t)j.slot0 * 128 + r;
    const float4* po = reinterpret_cast<const float4*>(part_o) + ((size_t)j.slot0 * 32 + col4) * 128 + r;
    float M = -INFINITY;
#pragma unroll 4
    for (uint32_t s = 0; s < n; ++s) M = fmaxf(M, __ldcg(ml + (size_t)s * 128).x);
    float L = 0.0f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t s0 = 0; s0 < n; s0 += 4) {
        float4 ov[4];
        float2 w[4];
#pragma unroll
        for (uint32_t i = 0; i < 4; ++i)
            if (s0 + i < n) {
                w[i] = __ldcg(ml + (size_t)(s0 + i) * 128);
                ov[i] = __ldcs(po + (size_t)(s0 + i) * 32 * 128);
            }
#pragma unroll
        for (uint32_t i = 0; i < 4; ++i)
            if (s0 + i < n) {
                const float wt = w[i].x == -INFINITY ? 0.0f : exp2f(w[i].x - M);
                L += wt * w[i].y;
                acc.x += wt * ov[i].x;
                acc.y += wt * ov[i].y;
                acc.z += wt * ov[i].z;
                acc.w += wt * ov[i].w;
            }
    }
    const float inv = L > 0.0f ? 1.0f / L : 0.0f;
    uint2 pk;
    pk.x = pack_bf16(acc.x * inv, acc.y * inv);
    pk.y = pack_bf16(acc.z * inv, acc.w * inv);
    *reinterpret_cast<uint2*>(out + (size_t)qi * h + j.head * 128u + col4 * 4) = pk;
}

}  // namespace

// Host: split every (query tile, head) key range into chunks of at most `chunk` blocks,
// then pair the chunks of two query tiles that start at the same key block of the same
// head into one item (they share the K/V stream; each stops at its own end block).
AttnPlan plan_attention(const uint32_t* rows, uint32_t m, uint32_t n_heads, const uint32_t* starts) {
    AttnPlan plan;
    const uint32_t tiles = ceil_div(m, 128);
    // tile t reads key blocks [sblk[t], nblk[t]): from its first row's request start (rows and
    // starts ascend) through its last row's position
    std::vector<uint32_t> nblk(tiles), sblk(tiles, 0);
    uint64_t total = 0;
    for (uint32_t t = 0; t < tiles; ++t) {
        nblk[t] = rows[attn_tile_last_row(t, m)] / 128 + 1;
        if (starts) {
            const uint32_t first = t == 0 ? 0u : attn_tile_last_row(t - 1, m) + 1;
            sblk[t] = std::min(starts[first] / 128, nblk[t] - 1);
        }
        total += (uint64_t)(nblk[t] - sblk[t]) * n_heads;
    }
    // ~1.5 waves of items (an item carries up to two tiles); never split below 2 blocks
    static const uint32_t per_sm = [] {
        const char* e = getenv("MPIC_ATTN_CHUNKS_PER_SM");  // diagnostics: tile-chunks per SM
        return e ? (uint32_t)std::max(1, atoi(e)) : 3u;
    }();
    static const uint32_t min_chunk = [] {
        const char* e = getenv("MPIC_ATTN_MIN_CHUNK");  // diagnostics: shortest split (blocks)
        return e ? (uint32_t)std::max(1, atoi(e)) : 2u;
    }();
    uint32_t chunk = (uint32_t)std::max<uint64_t>(min_chunk, (total + per_sm * kNumSMs - 1) / (per_sm * kNumSMs));
    uint32_t longest = 0, last = 0;
    for (uint32_t t = 0; t < tiles; ++t) {
        longest = std::max(longest, nblk[t] - sblk[t]);
        last = std::max(last, nblk[t]);
    }
    chunk = std::max(chunk, ceil_div(longest + 1, 15));  // a tile meets at most 16 grid cells (combine limit)
    // splits: tile t's range cut by the global grid [sp*chunk, (sp+1)*chunk)
    auto cell0 = [&](uint32_t t) { return sblk[t] / chunk; };
    auto cells = [&](uint32_t t) { return ceil_div(nblk[t], chunk) - cell0(t); };
    std::vector<uint32_t> slot0(tiles * n_heads, kNoTile), job0(tiles * n_heads, kNoTile);
    uint32_t slot = 0;
    for (uint32_t t = 0; t < tiles; ++t) {
        const uint32_t splits = cells(t);
        if (splits < 2) continue;
        for (uint32_t hd = 0; hd < n_heads; ++hd) {
            job0[t * n_heads + hd] = (uint32_t)plan.combine.size();
            plan.combine.push_back(AttnCombine{t, hd, slot, splits});
            slot0[t * n_heads + hd] = slot;
            slot += splits;
        }
    }
    plan.slots = slot;
    const uint32_t max_cells = ceil_div(last, chunk);
    for (uint32_t hd = 0; hd < n_heads; ++hd) {
        for (uint32_t sp = 0; sp < max_cells; ++sp) {
            AttnUnit cur{};
            bool open = false;
            for (uint32_t t = 0; t < tiles; ++t) {
                const uint32_t lo = std::max(sblk[t], sp * chunk), hi = std::min(nblk[t], (sp + 1) * chunk);
                if (lo >= hi) continue;
                const uint32_t s0 = slot0[t * n_heads + hd], jb = job0[t * n_heads + hd];
                const uint32_t sl = s0 == kNoTile ? kNoTile : s0 + (sp - cell0(t));
                if (open && cur.b0 == lo) {  // pair with the open item: same first key block
                    cur.tile[1] = t;
                    cur.b1[1] = hi;
                    cur.slot[1] = sl;
                    cur.job[1] = jb;
                    plan.units.push_back(cur);
                    open = false;
                    continue;
                }
                if (open) plan.units.push_back(cur);
                cur = AttnUnit{hd, lo, {t, kNoTile}, {hi, 0}, {sl, kNoTile}, {jb, kNoTile}};
                open = true;
            }
            if (open) plan.units.push_back(cur);
        }
    }
    // Estimated cost in 0.1 us, from the kernel's measured per-block times (MPIC_ATTN_TS
    // fits): a pair item's 128-key block ~2.7 us (two tiles), a block one tile of a pair
    // streams alone ~2.0, a split item's block ~1.6 (both lanes on one tile); ~2 us per item
    // (first loads and epilogue not hidden by the persistent loop).
    static const bool by_cost = getenv("MPIC_ATTN_SORT_LEN") == nullptr;  // diagnostics: 1 = by length
    auto cost = [](const AttnUnit& a) -> uint32_t {
        if (a.tile[1] == kNoTile) return 16 * (a.b1[0] - a.b0) + 20;
        const uint32_t len = std::max(a.b1[0], a.b1[1]) - a.b0;
        const uint32_t both = std::min(a.b1[0], a.b1[1]) - a.b0;
        return 27 * both + 20 * (len - both) + 20;
    };
    std::stable_sort(plan.units.begin(), plan.units.end(), [&](const AttnUnit& a, const AttnUnit& b) {
        if (by_cost) return cost(a) > cost(b);
        const uint32_t la = std::max(a.b1[0], a.tile[1] == kNoTile ? 0u : a.b1[1]) - a.b0;
        const uint32_t lb = std::max(b.b1[0], b.tile[1] == kNoTile ? 0u : b.b1[1]) - b.b0;
        return la > lb;
    });
    // Longest-processing-time assignment to the persistent CTAs: each item (largest first)
    // goes to the least-loaded CTA; the items are then grouped by CTA and the offsets packed
    // behind them.
    const uint32_t n = (uint32_t)plan.units.size(), G = std::min<uint32_t>(n, kNumSMs);
    plan.items = n;
    if (n) {
        std::vector<std::vector<AttnUnit>> per(G);
        std::vector<std::pair<uint64_t, uint32_t>> heap;  // (load, cta), min-heap
        for (uint32_t c = 0; c < G; ++c) heap.push_back({0, c});
        auto gt = [](const std::pair<uint64_t, uint32_t>& a, const std::pair<uint64_t, uint32_t>& b) { return a > b; };
        for (const AttnUnit& u : plan.units) {
            std::pop_heap(heap.begin(), heap.end(), gt);
            auto& top = heap.back();
            per[top.second].push_back(u);
            top.first += cost(u);
            std::push_heap(heap.begin(), heap.end(), gt);
        }
        std::vector<uint32_t> off(G + 1, 0);
        plan.units.clear();
        for (uint32_t c = 0; c < G; ++c) {
            off[c] = (uint32_t)plan.units.size();
            plan.units.insert(plan.units.end(), per[c].begin(), per[c].end());
        }
        off[G] = n;
        const size_t entries = (off.size() * sizeof(uint32_t) + sizeof(AttnUnit) - 1) / sizeof(AttnUnit);
        plan.units.resize(n + entries);
        std::memcpy(plan.units.data() + n, off.data(), off.size() * sizeof(uint32_t));
    }
    return plan;
}

// MPIC_ATTN_TS=1 (diagnostics): CTA 0 records per-block event times; printed by
// mpic_test_attention.
unsigned long long* attn_debug_buffer() {
    static unsigned long long* buf = [] {
        unsigned long long* b = nullptr;
        if (getenv("MPIC_ATTN_TS")) {
            cudaMalloc(&b, 16 * 4096 * sizeof(unsigned long long));
            cudaMemset(b, 0, 16 * 4096 * sizeof(unsigned long long));
        }
        return b;
    }();
    return buf;
}

void launch_attn_tc(const __nv_bfloat16* q, const __nv_bfloat16* kcache, const __nv_bfloat16* vcache,
                    uint32_t n_ctx, const uint32_t* d_rows, uint32_t m, uint32_t H,
                    const AttnUnit* d_units, uint32_t n_units, const AttnCombine* d_combine,
                    uint32_t n_combine, float* part_o, float2* part_ml, __nv_bfloat16* out,
                    cudaStream_t s, const AttnLink* link, uint32_t layer, const uint32_t* d_starts,
                    uint32_t* d_counters) {
    const uint32_t h = H * 128;
    const CUtensorMap tmQ = make_tmap_bf16(q, h, m, 64, 128);
    const CUtensorMap tmK = make_tmap_bf16(kcache, h, n_ctx, 64, 128);
    const CUtensorMap tmV = make_tmap_bf16(vcache, h, n_ctx, 64, 128);
    AttnParams p;
    p.units = d_units;
    p.n_units = n_units;
    p.combine = d_combine;
    p.counters = d_counters;
    p.rows = d_rows;
    p.starts = d_starts;
    p.m = m;
    p.shift = attn_tile_shift(m);
    p.h = h;
    p.scale_log2 = (1.0f / sqrtf(128.0f)) * 1.4426950408889634f;
    p.out = out;
    p.part_o = part_o;
    p.part_ml = part_ml;
    p.dbg = attn_debug_buffer();
    p.link = link;
    p.layer = layer;
    static const bool nostore = [] {
        const char* e = getenv("MPIC_ATTN_LINK");
        return e && atoi(e) == 2;
    }();
    p.link_nostore = nostore ? 1u : 0u;
    const size_t smem = (2 + kKStages + kVStages) * kTile + 1024 + (2 + 2 * kKStages + 2 * kVStages + 14) * 8 + 16 +
                        128 * sizeof(float2) + 16;
    static bool attr = false;
    if (!attr) {
        MPIC_CUDA(cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    at[1].id = cudaLaunchAttributePriority;
    at[1].val.priority = hot_priority();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(std::min<uint32_t>(n_units, kNumSMs));  // persistent: one CTA per SM, items per CTA from the plan
    cfg.blockDim = dim3(kAttnThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    MPIC_CUDA(cudaLaunchKernelEx(&cfg, attn_tc_kernel, tmQ, tmK, tmV, p));
    MPIC_LAUNCHED();
    if (n_combine && !d_counters) {  // (with counters the attention kernel merges the splits itself)
        cfg.gridDim = dim3(n_combine, 16);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = 0;
        MPIC_CUDA(cudaLaunchKernelEx(&cfg, attn_combine_kernel, d_combine, (const float*)part_o,
                                     (const float2*)part_ml, m, p.shift, h, out));
        MPIC_LAUNCHED();
    }
}

void make_link_maps(AttnLink* host, const void* const* k, const void* const* v, const uint32_t* T, uint32_t n,
                    uint32_t L, uint32_t h) {
    MPIC_REQUIRE(n <= kMaxLinkChunks, MPIC_ERR_VALIDATION, "too many chunks to link inside attention");
    static_assert(sizeof(TmapBytes) == sizeof(CUtensorMap), "tensor map size");
    for (uint32_t c = 0; c < kMaxLinkChunks; ++c) {
        const uint32_t i = c < n ? c : 0;  // unused slots repeat chunk 0 (never addressed)
        const CUtensorMap mk = make_tmap_bf16(k[i], h, (uint64_t)L * T[i], 64, 128);
        const CUtensorMap mv = make_tmap_bf16(v[i], h, (uint64_t)L * T[i], 64, 128);
        std::memcpy(&host->maps[2 * c], &mk, sizeof(mk));
        std::memcpy(&host->maps[2 * c + 1], &mv, sizeof(mv));
        host->tokens[c] = T[i];
    }
}

}  // namespace mpicb
