// Microbenchmark: cycles per tcgen05.mma.cta_group::2 (kind::f16, M=256) for several N with
// operands resident in shared memory (no TMA in the loop), all 74 SM pairs busy. Diagnostic.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2502_01960_b200/csrc/tc_common.cuh"
using namespace mpicb;

__global__ void __cluster_dims__(2, 1, 1) probe(unsigned long long* out, int n0, int n1, int iters, int mode) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t holder;
    __shared__ uint64_t bar;
    __shared__ uint64_t dummy[8];
    const uint32_t warp = threadIdx.x / 32;
    const uint32_t rank = tc::cluster_ctarank();
    for (int i = threadIdx.x; i < (16384 + 256 * 64) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        tc::mbar_init(&bar, 1);
        for (int i = 0; i < 8; ++i) tc::mbar_init(&dummy[i], 1);
        tc::fence_barrier_init();
    }
    tc::fence_async_shared();
    if (warp == 0) tc::tmem_alloc_pair(&holder, 512);
    tc::tc_fence_before();
    tc::cluster_sync();
    tc::tc_fence_after();
    const uint32_t tmem = holder;
    if (threadIdx.x == 0 && rank == 0) {
        const uint32_t a = tc::smem_u32(smem), b = a + 16384;
        const uint32_t id0 = tc::idesc_bf16(256, n0), id1 = tc::idesc_bf16(256, n1 ? n1 : 16);
        const unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (mode & 2) { tc::mbar_wait(&bar, 1); if (!(mode & 4)) tc::tc_fence_after(); }  // a completed phase: returns at once
            for (int k = 0; k < 4; ++k) {
                tc::mma_bf16_pair(tmem, tc::desc_k_sw128(a + k * 32), tc::desc_k_sw128(b + k * 32), id0, 1);
                if (n1) tc::mma_bf16_pair(tmem + n0, tc::desc_k_sw128(a + k * 32), tc::desc_k_sw128(b + n0 * 64 + k * 32), id1, 1);
            }
            if (mode & 1) tc::mma_commit_pair_mcast(&dummy[it & 7], 3);
        }
        tc::mma_commit_pair_mcast(&bar, 3);
        tc::mbar_wait(&bar, 0);
        out[blockIdx.x / 2] = clock64() - t0;
    } else if (threadIdx.x == 0) {
        tc::mbar_wait(&bar, 0);
    }
    tc::tc_fence_before();
    tc::cluster_sync();
    tc::tc_fence_after();
    if (warp == 0) tc::tmem_dealloc_pair(tmem, 512);
}

int main() {
    const int pairs = 74, iters = 2000;
    unsigned long long* d;
    cudaMalloc(&d, pairs * 8);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    int shapes[][2] = {{176, 160}, {128, 128}, {96, 0}};
    for (int mode : {1, 2, 3, 6, 7})
    for (auto& sh : shapes) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        probe<<<2 * pairs, 128, 100 * 1024>>>(d, sh[0], sh[1], 10, mode);
        cudaEventRecord(e0);
        probe<<<2 * pairs, 128, 100 * 1024>>>(d, sh[0], sh[1], iters, mode);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long h[pairs];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double cyc = 0; for (int i = 0; i < pairs; ++i) cyc += h[i]; cyc /= pairs;
        const int N = sh[0] + sh[1];
        const double flops = 2.0 * 256 * N * 16 * 4 * iters * pairs;
        printf("mode %d (1 commit/kblock, 2 wait/kblock, 4 no fence) N=%3d+%3d: %.1f cyc per k-block (ideal %d), %.0f TFLOP/s chip, err=%s\n",
               mode, sh[0], sh[1], cyc / iters, 2 * N, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
}
