// Microbenchmark: the attention kernel's MMA shapes on one SM per CTA (148 CTAs), with and
// without concurrent TMEM traffic from 4 other warps. cta_group::1, M=128, N=128, K=16:
//   SS  = Q.K^T form (both operands K-major SW128 in shared memory)
//   TS  = P.V form (A = P from TMEM, B = V MN-major SW128 in shared memory)
// Background warps 4-7 (one per TMEM lane quarter): 0 none, 1 tcgen05.ld 128 cols + wait in a
// loop, 2 ld + st (16 packed cols) like the softmax. Diagnostic only.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31; }
#include "../paper_2502_01960_b200/csrc/tc_common.cuh"
using namespace mpicb;

__global__ void probe(unsigned long long* out, int form, int bg, int iters, const uint8_t* gsrc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t holder;
    __shared__ uint64_t bar;
    __shared__ uint64_t bars[4];
    __shared__ volatile int done;
    for (int i = threadIdx.x; i < 3 * 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); for (int i = 0; i < 4; ++i) tc::mbar_init(&bars[i], 1); tc::fence_barrier_init(); done = 0; }
    tc::fence_async_shared();
    if (threadIdx.x < 32) tc::tmem_alloc(&holder, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = holder;
    const uint32_t warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        const uint32_t q = tc::smem_u32(smem), k = q + 32768, v = q + 65536;
        const uint32_t id_s = tc::idesc_bf16(128, 128, false), id_o = tc::idesc_bf16(128, 128, true);
        const uint32_t id_s64 = tc::idesc_bf16(128, 64, false);
        const unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            for (int x = 0; x < 2; ++x) {  // two tiles, like the ping-pong
                if (form == 4) {  // the step with the kernel's commits and fences between groups
                    tc::tc_fence_after();
                    for (int kk = 0; kk < 4; ++kk)
                        tc::mma_bf16_ts(tmem + x * 256 + 128, tmem + x * 256 + kk * 8, tc::desc_mn_sw128(v + kk * 2048, 16384),
                                        id_o, 1);
                    tc::mma_commit(&bars[x]);
                    tc::tc_fence_after();
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
                        tc::mma_bf16(tmem + x * 256 + 64, tc::desc_k_sw128(q + off), tc::desc_k_sw128(k + 8192 + off), id_s64, 1);
                    }
                    tc::mma_commit(&bars[2 + x]);
                } else if (form == 2) {  // one 64-key step of a lane: PV (4 x N=128) + S (8 x N=64)
                    for (int kk = 0; kk < 4; ++kk)
                        tc::mma_bf16_ts(tmem + x * 256 + 128, tmem + x * 256 + kk * 8, tc::desc_mn_sw128(v + kk * 2048, 16384),
                                        id_o, 1);
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
                        tc::mma_bf16(tmem + x * 256 + 64, tc::desc_k_sw128(q + off), tc::desc_k_sw128(k + 8192 + off), id_s64, 1);
                    }
                } else if (form == 3) {  // S only, N = 64
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
                        tc::mma_bf16(tmem + x * 256 + 64, tc::desc_k_sw128(q + off), tc::desc_k_sw128(k + 8192 + off), id_s64, 1);
                    }
                } else if (form == 0) {
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
                        tc::mma_bf16(tmem + x * 256, tc::desc_k_sw128(q + off), tc::desc_k_sw128(k + off), id_s, 1);
                    }
                } else {
                    for (int kk = 0; kk < 8; ++kk)
                        tc::mma_bf16_ts(tmem + x * 256 + 128, tmem + x * 256 + kk * 8, tc::desc_mn_sw128(v + kk * 2048, 16384),
                                        id_o, 1);
                }
            }
        }
        tc::mma_commit(&bar);
        tc::mbar_wait(&bar, 0);
        out[blockIdx.x] = clock64() - t0;
        done = 1;
    } else if (warp == 4 && bg == 3) {
        // background bulk copies global -> shared (like the K/V TMA loads), 32 KB at a time
        __shared__ uint64_t lbar;
        if (lane_id() == 0) {
            tc::mbar_init(&lbar, 1);
            tc::fence_barrier_init();
            uint32_t ph = 0;
            for (int i = 0; !done; ++i) {
                tc::mbar_arrive_expect_tx(&lbar, 32768);
                tc::bulk_load(smem + 3 * 32768, gsrc + (size_t)(blockIdx.x * 8 + (i & 7)) * 32768, 32768, &lbar);
                tc::mbar_wait(&lbar, ph);
                ph ^= 1;
            }
        }
    } else if (warp >= 4 && bg && bg < 3) {
        const uint32_t lane_base = ((warp & 3) * 32u) << 16;
        uint32_t acc = 0;
        while (!done) {
            uint32_t r[32];
            for (int c = 0; c < 128; c += 32) {
                tc::tmem_ld32(tmem + lane_base + 256 + c, r);  // tile B's S columns
                tc::tmem_ld_wait();
                acc += r[0] ^ r[31];
            }
            if (bg == 2) {
                uint32_t pk[16];
                for (int e = 0; e < 16; ++e) pk[e] = r[e] + acc;
                tc::tmem_st16(tmem + lane_base + 256 + 64, pk);
                tc::tmem_st_wait();
            }
        }
        if (acc == 0x12345678u) out[200] = acc;
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 512);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 256 * 8);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
    uint8_t* gsrc;
    cudaMalloc(&gsrc, (size_t)148 * 8 * 32768);
    cudaMemset(gsrc, 0, (size_t)148 * 8 * 32768);
    const char* names[5] = {"SS (Q.K, N=128)", "TS (P.V)", "step (4 TS + 8 SS N=64)", "SS (Q.K, N=64)", "step + commits/fences"};
    const int per_it[5] = {16, 16, 24, 16, 24};
    for (int form = 0; form < 5; ++form)
        for (int bg = 0; bg < 4; ++bg) {
            const int iters = 500;
            probe<<<148, 256, 140 * 1024>>>(d, form, bg, 10, gsrc);
            probe<<<148, 256, 140 * 1024>>>(d, form, bg, iters, gsrc);
            unsigned long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
            printf("%-26s bg=%d: %.1f cycles per MMA, %.0f per iteration (2 lanes) err=%s\n", names[form], bg,
                   c / iters / per_it[form], c / iters, cudaGetErrorString(cudaGetLastError()));
        }
}
