// Microbenchmark: tcgen05.mma cta_group::1 M=128 N=128 K=16 issue patterns — one dependent
// accumulator chain vs two chains back to back vs two chains interleaved. Diagnostic only.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2502_01960_b200/csrc/tc_common.cuh"
using namespace mpicb;

__global__ void probe(unsigned long long* out, int mode, int iters, int n) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t holder;
    __shared__ uint64_t bar;
    for (int i = threadIdx.x; i < 3 * 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
    tc::fence_async_shared();
    if (threadIdx.x < 32) tc::tmem_alloc(&holder, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = holder;
    if (threadIdx.x == 0) {
        const uint32_t a = tc::smem_u32(smem), b = a + 16384, b2 = a + 32768;
        const uint32_t id = tc::idesc_bf16(128, n);
        const unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (mode == 0) {  // one chain of 8
                for (int k = 0; k < 8; ++k) tc::mma_bf16(tmem, tc::desc_k_sw128(a + (k & 3) * 32), tc::desc_k_sw128(b + (k & 3) * 32), id, 1);
            } else if (mode == 1) {  // two chains back to back (8 + 8)
                for (int k = 0; k < 8; ++k) tc::mma_bf16(tmem, tc::desc_k_sw128(a + (k & 3) * 32), tc::desc_k_sw128(b + (k & 3) * 32), id, 1);
                for (int k = 0; k < 8; ++k) tc::mma_bf16(tmem + 256, tc::desc_k_sw128(a + (k & 3) * 32), tc::desc_k_sw128(b2 + (k & 3) * 32), id, 1);
            } else {  // two chains interleaved
                for (int k = 0; k < 8; ++k) {
                    tc::mma_bf16(tmem, tc::desc_k_sw128(a + (k & 3) * 32), tc::desc_k_sw128(b + (k & 3) * 32), id, 1);
                    tc::mma_bf16(tmem + 256, tc::desc_k_sw128(a + (k & 3) * 32), tc::desc_k_sw128(b2 + (k & 3) * 32), id, 1);
                }
            }
        }
        tc::mma_commit(&bar);
        tc::mbar_wait(&bar, 0);
        out[blockIdx.x] = clock64() - t0;
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 512);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int n : {128, 64, 256})
        for (int mode = 0; mode < 3; ++mode) {
            const int iters = 1000;
            probe<<<148, 128, 64 * 1024>>>(d, mode, 10, n);
            probe<<<148, 128, 64 * 1024>>>(d, mode, iters, n);
            unsigned long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
            const int instr = mode == 0 ? 8 : 16;
            printf("N=%d mode %d (%s): %.1f cycles per MMA (ideal %d) err=%s\n", n, mode,
                   mode == 0 ? "1 chain" : mode == 1 ? "2 chains back to back" : "2 chains interleaved",
                   c / iters / instr, 128 * n / 256, cudaGetErrorString(cudaGetLastError()));
        }
}
