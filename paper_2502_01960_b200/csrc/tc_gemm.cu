// K3/K5/K6/K7 — projection GEMMs of the selective recompute on the 5th-gen tensor cores.
//
//   out[t][f] = sum_k X[t][k] * W[f][k]      (y = x . W^T, proj/src/linker.cpp:64-128)
//
// Swap-AB mapping for the small-m regime of MPIC (m = text + k*images rows, 96..2000):
// the UMMA M=128 side is the WEIGHT tile (128 output features), the UMMA N side is the
// token tile (any multiple of 16 up to 512), so no MMA work is spent on padding rows.
// One CTA owns 128 features x up to 512 tokens (TMEM: 128 lanes x 512 fp32 columns).
//
//   warp 0     TMA producer: W tile [128 x 64] + X tile [tt x 64] per stage (SWIZZLE_128B)
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer (kind::f16, fp32 accum)
//   warps 2-5  epilogue: tcgen05.ld of the accumulator, fused RoPE+scatter into the KV
//              cache (QKV), GELU (W1), residual add into the fp32 stream (Wo/W2, split-K
//              via red.global.add) — each thread owns one output feature, lanes of a
//              warp own 32 consecutive features, so stores are coalesced per token.
//
// Full/empty mbarrier ring between TMA and MMA; tcgen05.commit releases smem stages and
// signals the epilogue. Split-K over blockIdx.z keeps >=120 CTAs busy on 148 SMs when
// the feature dimension alone is too small (Wo, W2 at h=4096).
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

struct TcGemmArgs {
    uint32_t M, N, K;
    uint32_t tt;            // token columns per CTA (multiple of 16, <= 512)
    uint32_t xr;            // X rows loaded (and multicast) by each CTA of the cluster
    uint32_t cl;            // cluster size along the feature-tile axis (1, 2 or 4)
    uint32_t kb_per_split;  // 64-wide K blocks per CTA
    uint32_t stages;
    uint32_t tmem_cols;
    EpiParams ep;
};

template <typename TO>
__device__ __forceinline__ void tc_epilogue(const EpiParams& ep, uint32_t t, uint32_t f, float v) {
    switch (ep.mode) {
        case EPI_RESID: {
            if (ep.split_k > 1) {  // deterministic split-K: partial tile, reduced afterwards
                ep.partial[((size_t)blockIdx.z * ep.rows_total + t) * ep.ldx + f] = v;
            } else {
                float* x = ep.x + (size_t)t * ep.ldx + f;
                const float nv = *x + v;
                *x = nv;
                if (ep.xb) ep.xb[(size_t)t * ep.ldx + f] = __float2bfloat16_rn(nv);
            }
            break;
        }
        case EPI_GELU:
            static_cast<TO*>(ep.out)[(size_t)t * ep.ldo + f] = from_f32<TO>(gelu_ref(v));
            break;
        case EPI_STORE_F32:
            static_cast<float*>(ep.out)[(size_t)t * ep.ldo + f] = v;
            break;
        default:
            static_cast<TO*>(ep.out)[(size_t)t * ep.ldo + f] = from_f32<TO>(v);
    }
}

__global__ void __launch_bounds__(kTcThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                   const TcGemmArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t x_bytes = a.cl * a.xr * 128;
    const uint32_t stage_bytes = kWTileBytes + x_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.stages * stage_bytes);
    uint64_t* empty = full + a.stages;
    uint64_t* tmem_full = empty + a.stages;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_full + 1);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t n0 = blockIdx.x * 128, t0 = blockIdx.y * a.tt;
    const uint32_t kb0 = blockIdx.z * a.kb_per_split;
    const uint32_t rank = a.cl > 1 ? tc::cluster_ctarank() : 0;
    const uint16_t mask = (uint16_t)((1u << a.cl) - 1);

    if (warp == 0 && lane == 0) {
        tc::tma_prefetch_desc(&tmW);
        tc::tma_prefetch_desc(&tmX);
        for (uint32_t s = 0; s < a.stages; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], a.cl);  // every CTA's MMA must release a multicast stage
        }
        tc::mbar_init(tmem_full, 1);
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc(tmem_holder, a.tmem_cols);
    tc::tc_fence_before();
    if (a.cl > 1) tc::cluster_sync();  // peers' barriers are initialised before any multicast
    else __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol_w = tc::policy_evict_first();  // weights stream through once
            const uint64_t pol_x = tc::policy_evict_last();   // token tile re-read by every cluster
            for (uint32_t i = 0; i < a.kb_per_split; ++i) {
                const uint32_t s = i % a.stages, ph = (i / a.stages) & 1;
                tc::mbar_wait(&empty[s], ph ^ 1);
                tc::mbar_arrive_expect_tx(&full[s], stage_bytes);
                const int k = (int)((kb0 + i) * 64);
                uint8_t* st = smem + s * stage_bytes;
                tc::tma_load_2d_hint(st, &tmW, &full[s], k, (int)n0, pol_w);
                uint8_t* xs = st + kWTileBytes + rank * a.xr * 128;
                const int row = (int)(t0 + rank * a.xr);
                if (a.cl > 1) tc::tma_load_2d_mcast(xs, &tmX, &full[s], k, row, mask, pol_x);
                else tc::tma_load_2d_hint(xs, &tmX, &full[s], k, row, pol_x);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            for (uint32_t i = 0; i < a.kb_per_split; ++i) {
                const uint32_t s = i % a.stages, ph = (i / a.stages) & 1;
                tc::mbar_wait(&full[s], ph);
                tc::tc_fence_after();
                const uint32_t w_base = tc::smem_u32(smem + s * stage_bytes);
                const uint32_t x_base = w_base + kWTileBytes;
#pragma unroll
                for (uint32_t kk = 0; kk < 4; ++kk) {
                    const uint64_t adesc = tc::desc_k_sw128(w_base + kk * 32);
                    for (uint32_t c0 = 0; c0 < a.tt; c0 += 256) {
                        const uint32_t cn = min(256u, a.tt - c0);
                        const uint64_t bdesc = tc::desc_k_sw128(x_base + c0 * 128 + kk * 32);
                        tc::mma_bf16(tmem_base + c0, adesc, bdesc, tc::idesc_bf16(128, cn),
                                     (i > 0 || kk > 0) ? 1u : 0u);
                    }
                }
                if (a.cl > 1) tc::mma_commit_mcast(&empty[s], mask);
                else tc::mma_commit(&empty[s]);
            }
            tc::mma_commit(tmem_full);
        }
        __syncwarp();
    } else {
        // epilogue: warp w may only touch TMEM lanes [32*(w%4), 32*(w%4)+32)
        const uint32_t q = warp & 3;
        const uint32_t f = n0 + q * 32 + lane;
        tc::mbar_wait(tmem_full, 0);
        tc::tc_fence_after();
        const bool qkv = a.ep.mode == EPI_QKV;
        const uint32_t part = qkv ? f / a.ep.hidden : 0;  // warp-uniform (hidden % 128 == 0)
        const uint32_t pair = qkv ? ((f - part * a.ep.hidden) % a.ep.head_dim) >> 1 : 0;
        for (uint32_t c = 0; c < a.tt; c += 16) {
            uint32_t r[16];
            tc::tmem_ld16(tmem_base + ((q * 32u) << 16) + c, r);
            if (qkv) {
                // issue every per-token load of this chunk before the first store
                uint32_t dst_row[16];
                float2 cs[16];
#pragma unroll
                for (uint32_t j = 0; j < 16; ++j) {
                    const uint32_t t = min(t0 + c + j, a.M - 1);
                    dst_row[j] = part == 0 ? t : __ldg(a.ep.kv_rows + t);
                    cs[j] = part < 2 ? __ldg(a.ep.rope + (size_t)__ldg(a.ep.rope_pos + t) * (a.ep.head_dim >> 1) + pair)
                                     : make_float2(1.f, 0.f);
                }
                tc::tmem_ld_wait();
                __nv_bfloat16* base = static_cast<__nv_bfloat16*>(part == 0 ? a.ep.q : part == 1 ? a.ep.kv_k : a.ep.kv_v) +
                                      (f - part * a.ep.hidden);
#pragma unroll
                for (uint32_t j = 0; j < 16; ++j) {
                    float v = __uint_as_float(r[j]);
                    const float vp = __shfl_xor_sync(0xffffffffu, v, 1);
                    if (part < 2) {
                        float x0 = (lane & 1) ? vp : v, x1 = (lane & 1) ? v : vp;
                        rope_pair(x0, x1, cs[j].x, cs[j].y);
                        v = (lane & 1) ? x1 : x0;
                    }
                    if (t0 + c + j < a.M) base[(size_t)dst_row[j] * a.ep.hidden] = __float2bfloat16_rn(v);
                }
            } else {
                tc::tmem_ld_wait();
#pragma unroll
                for (uint32_t j = 0; j < 16; ++j) {
                    const uint32_t t = t0 + c + j;
                    if (t < a.M) tc_epilogue<__nv_bfloat16>(a.ep, t, f, __uint_as_float(r[j]));
                }
            }
        }
    }
    tc::tc_fence_before();
    if (a.cl > 1) tc::cluster_sync();  // no CTA exits while peers may still signal its barriers
    else __syncthreads();
    tc::tc_fence_after();
    if (warp == 1) tc::tmem_dealloc(tmem_base, a.tmem_cols);
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
CUtensorMap make_tmap_bf16(const void* ptr, uint64_t inner, uint64_t outer, uint32_t box_inner,
                           uint32_t box_outer) {
    static std::mutex mu;
    static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
    const MapKey key{ptr, inner, outer, box_inner, box_outer};
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    CUtensorMap m;
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {inner * 2};
    const cuuint32_t box[2] = {box_inner, box_outer};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    MPIC_REQUIRE(r == CUDA_SUCCESS, MPIC_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    std::lock_guard<std::mutex> lk(mu);
    cache.emplace(key, m);
    return m;
}

bool tc_gemm_supported(uint32_t M, uint32_t N, uint32_t K) {
    return M > 0 && N % 128 == 0 && K % 64 == 0 && K >= 64;
}

void launch_gemm_tc(const __nv_bfloat16* A, uint32_t lda, const __nv_bfloat16* W, uint32_t M,
                    uint32_t N, uint32_t K, const EpiParams& ep_in, cudaStream_t s) {
    MPIC_REQUIRE(tc_gemm_supported(M, N, K) && lda == K, MPIC_ERR_VALIDATION, "unsupported tc gemm shape");
    TcGemmArgs a{};
    a.M = M;
    a.N = N;
    a.K = K;
    a.tt = M <= 512 ? (M + 15) / 16 * 16 : 256;
    const uint32_t tiles_t = ceil_div(M, a.tt);
    const uint32_t ntiles = N / 128;
    const uint32_t kblocks = K / 64;
    // split-K (residual epilogues only, into a partial buffer) to fill the SMs
    uint32_t split = 1;
    if (ep_in.mode == EPI_RESID && ep_in.partial) {
        double best = 0.0;
        for (uint32_t sp = 1; sp <= 8; sp *= 2) {
            if (kblocks % sp || kblocks / sp < 4) break;
            if ((size_t)sp * M * N > ep_in.partial_cap) break;
            const uint32_t ctas = ntiles * tiles_t * sp;
            const double eff = (double)ctas / (kNumSMs * ceil_div(ctas, kNumSMs));
            const double score = std::min(1.0, (double)ctas / kNumSMs) * eff;
            if (score > best + 1e-9) {
                best = score;
                split = sp;
            }
        }
    }
    // cluster multicast of the token tile: 4 CTAs share it when they fit in one wave
    // (4-CTA clusters strand a few SMs per GPC), else 2.
    const uint32_t ctas = ntiles * tiles_t * split;
    a.cl = (ntiles % 4 == 0 && ctas <= 132) ? 4 : (ntiles % 2 == 0 ? 2 : 1);
    a.xr = (ceil_div(a.tt, a.cl) + 7) / 8 * 8;
    const uint32_t stage_bytes = kWTileBytes + a.cl * a.xr * 128;
    const uint32_t budget = 227 * 1024 - 1024 - 256;
    a.stages = std::min<uint32_t>(8, budget / stage_bytes);
    MPIC_REQUIRE(a.stages >= 2, MPIC_ERR_VALIDATION, "tc gemm tile does not fit shared memory");
    a.tmem_cols = 32;
    while (a.tmem_cols < a.tt) a.tmem_cols *= 2;
    a.kb_per_split = kblocks / split;
    a.ep = ep_in;
    a.ep.split_k = split;
    a.ep.rows_total = M;
    const CUtensorMap tmW = make_tmap_bf16(W, K, N, 64, 128);
    // Rows >= M are out of bounds for the map: TMA zero-fills them.
    const CUtensorMap tmX = make_tmap_bf16(A, K, M, 64, a.xr);
    const size_t smem = (size_t)a.stages * stage_bytes + 1024 + (2 * a.stages + 1) * 8 + 16;
    static std::once_flag once;
    std::call_once(once, [] {
        MPIC_CUDA(cudaFuncSetAttribute(tc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        MPIC_CUDA(cudaFuncSetAttribute(tc_gemm_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    });
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ntiles, tiles_t, split);
    cfg.blockDim = dim3(kTcThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = a.cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    MPIC_CUDA(cudaLaunchKernelEx(&cfg, tc_gemm_kernel, tmW, tmX, a));
    note_launch();
    if (split > 1) {
        const size_t n4 = (size_t)M * N / 4;
        resid_reduce_kernel<<<kNumSMs * 4, 256, 0, s>>>(ep_in.partial, split, (size_t)M * N, ep_in.x,
                                                         ep_in.xb, n4);
        MPIC_LAUNCHED();
    }
}

}  // namespace mpicb
