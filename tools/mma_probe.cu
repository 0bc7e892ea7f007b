// Microbenchmark: cycles per tcgen05.mma (kind::f16, SS) for several shapes with operands
// resident in shared memory (no TMA in the loop). Diagnostic only.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2502_01960_b200/csrc/tc_common.cuh"
using namespace mpicb;

template <int N, int ITERS>
__global__ void probe(unsigned long long* out, int use_tmem_sync) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t holder;
    __shared__ uint64_t bar;
    const uint32_t warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 128 * 64 * 2 / 4 + N * 64 * 2 / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;  // small bf16 values
    if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
    tc::fence_async_shared();
    if (warp == 0) tc::tmem_alloc(&holder, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = holder;
    if (threadIdx.x == 0) {
        const uint32_t a = tc::smem_u32(smem), b = a + 128 * 128;
        const uint32_t idesc = tc::idesc_bf16(128, N);
        // warm
        for (int k = 0; k < 4; ++k) tc::mma_bf16(tmem, tc::desc_k_sw128(a + k * 32), tc::desc_k_sw128(b + k * 32), idesc, k > 0);
        tc::mma_commit(&bar);
        tc::mbar_wait(&bar, 0);
        const unsigned long long t0 = clock64();
        for (int it = 0; it < ITERS; ++it)
            for (int k = 0; k < 4; ++k)
                tc::mma_bf16(tmem, tc::desc_k_sw128(a + k * 32), tc::desc_k_sw128(b + k * 32), idesc, 1);
        tc::mma_commit(&bar);
        tc::mbar_wait(&bar, 1);
        const unsigned long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

template <int N>
void run(int blocks) {
    const int ITERS = 256;
    unsigned long long* d;
    cudaMalloc(&d, blocks * 8);
    const int smem = 128 * 128 + N * 128 + 2048;
    cudaFuncSetAttribute(probe<N, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe<N, 256><<<blocks, 128, smem>>>(d, 0);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, blocks * 8, cudaMemcpyDeviceToHost);
    double cyc = (double)h[0] / (ITERS * 4);
    printf("M=128 N=%3d K=16: %.1f cycles/mma (%s), %.0f MAC/cycle/SM, blocks=%d\n", N, cyc,
           cudaGetErrorString(e), 128.0 * N * 16 / cyc, blocks);
    cudaFree(d);
}

int main() {
    run<64>(1); run<128>(1); run<256>(1); run<80>(1);
    run<256>(148);
    return 0;
}
