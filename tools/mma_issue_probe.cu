// Microbenchmark: cost of issuing tcgen05.mma (queue depth), mbarrier try_wait on a completed
// phase, tcgen05.commit and tcgen05.fence from a single thread. Diagnostic only.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2502_01960_b200/csrc/tc_common.cuh"
using namespace mpicb;

__global__ void probe(unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t holder;
    __shared__ uint64_t bar, done_bar;
    for (int i = threadIdx.x; i < 3 * 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::mbar_init(&done_bar, 1); tc::fence_barrier_init(); }
    tc::fence_async_shared();
    if (threadIdx.x < 32) tc::tmem_alloc(&holder, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = holder;
    if (threadIdx.x == 0) {
        const uint32_t q = tc::smem_u32(smem), k = q + 32768;
        const uint32_t id_s = tc::idesc_bf16(128, 128, false);
        unsigned long long* o = out + blockIdx.x * 64;
        // issue N MMAs back to back: time to issue (clock after the last issue) and to finish
        for (int n = 1, slot = 0; n <= 32; n *= 2, ++slot) {
            const unsigned long long t0 = clock64();
            for (int i = 0; i < n; ++i)
                tc::mma_bf16(tmem, tc::desc_k_sw128(q + (i & 3) * 32), tc::desc_k_sw128(k + (i & 3) * 32), id_s, 1);
            const unsigned long long t1 = clock64();
            tc::mma_commit(&done_bar);
            tc::mbar_wait(&done_bar, slot & 1);
            const unsigned long long t2 = clock64();
            o[2 * slot] = t1 - t0;
            o[2 * slot + 1] = t2 - t0;
        }
        // try_wait on a completed phase (bar phase 0 completed by an arrive)
        tc::mbar_arrive(&bar);
        unsigned long long t0 = clock64();
        for (int i = 0; i < 100; ++i) tc::mbar_wait(&bar, 0);
        o[20] = (clock64() - t0) / 100;
        t0 = clock64();
        for (int i = 0; i < 100; ++i) tc::tc_fence_after();
        o[21] = (clock64() - t0) / 100;
        t0 = clock64();
        for (int i = 0; i < 100; ++i) tc::mma_commit(&bar);  // arrives on completed phases: harmless here
        o[22] = (clock64() - t0) / 100;
        // commit with a queue of 8 MMAs in flight
        t0 = clock64();
        for (int i = 0; i < 8; ++i)
            tc::mma_bf16(tmem, tc::desc_k_sw128(q + (i & 3) * 32), tc::desc_k_sw128(k + (i & 3) * 32), id_s, 1);
        const unsigned long long t1 = clock64();
        tc::mma_commit(&bar);
        const unsigned long long t2 = clock64();
        tc::mma_bf16(tmem, tc::desc_k_sw128(q), tc::desc_k_sw128(k), id_s, 1);
        const unsigned long long t3 = clock64();
        o[23] = t1 - t0; o[24] = t2 - t1; o[25] = t3 - t2;
        tc::mma_commit(&done_bar);
        tc::mbar_wait(&done_bar, 0);
        // try_wait on a completed barrier while MMAs (and a commit) are in flight
        __shared__ uint64_t other;
        tc::mbar_init(&other, 1);
        tc::fence_barrier_init();
        tc::mbar_arrive(&other);  // phase 0 complete
        for (int i = 0; i < 8; ++i)
            tc::mma_bf16(tmem, tc::desc_k_sw128(q + (i & 3) * 32), tc::desc_k_sw128(k + (i & 3) * 32), id_s, 1);
        tc::mma_commit(&done_bar);
        unsigned long long a0 = clock64();
        tc::mbar_wait(&other, 0);
        unsigned long long a1 = clock64();
        o[26] = a1 - a0;
        // same without a commit in flight
        for (int i = 0; i < 8; ++i)
            tc::mma_bf16(tmem, tc::desc_k_sw128(q + (i & 3) * 32), tc::desc_k_sw128(k + (i & 3) * 32), id_s, 1);
        a0 = clock64();
        tc::mbar_wait(&other, 0);
        a1 = clock64();
        o[27] = a1 - a0;
        // plain volatile shared load with MMAs in flight
        volatile uint32_t* vf = reinterpret_cast<volatile uint32_t*>(&holder);
        for (int i = 0; i < 8; ++i)
            tc::mma_bf16(tmem, tc::desc_k_sw128(q + (i & 3) * 32), tc::desc_k_sw128(k + (i & 3) * 32), id_s, 1);
        a0 = clock64();
        uint32_t x = *vf;
        a1 = clock64();
        o[28] = a1 - a0 + (x == 12345 ? 1 : 0);
        tc::mma_commit(&done_bar);
        tc::mbar_wait(&done_bar, 1);
        tc::mbar_wait(&done_bar, 0);
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 512);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 64 * 8);
    cudaMemset(d, 0, 148 * 64 * 8);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    probe<<<148, 128, 100 * 1024>>>(d);
    probe<<<148, 128, 100 * 1024>>>(d);
    unsigned long long h[64];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    for (int n = 1, slot = 0; n <= 32; n *= 2, ++slot)
        printf("issue %2d MMAs (128x128x16): issued after %5llu cycles, done after %5llu\n", n, h[2 * slot], h[2 * slot + 1]);
    printf("try_wait on a completed phase: %llu cycles; tcgen05.fence::after: %llu; commit (empty pipe): %llu\n", h[20], h[21], h[22]);
    printf("8 MMAs issued in %llu cycles, then commit %llu cycles, then one more MMA issue %llu cycles\n", h[23], h[24], h[25]);
    printf("try_wait (completed) right after 8 MMAs + commit: %llu cycles; after 8 MMAs, no commit: %llu; volatile ld.shared after 8 MMAs: %llu\n", h[26], h[27], h[28]);
}
