// Microbenchmark: tcgen05.ld throughput (32x32b.x32: 32 lanes x 32 columns x 4 B = 4 KB per
// warp instruction) with 4 or 8 warps (1 or 2 per TMEM lane quarter), with and without
// waiting after each load. Diagnostic only.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2502_01960_b200/csrc/tc_common.cuh"
using namespace mpicb;

template <int N>
__device__ __forceinline__ void ld_x(uint32_t taddr, uint32_t* r);
template <>
__device__ __forceinline__ void ld_x<64>(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
        "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]),
          "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
          "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]),
          "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]),
          "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]),
          "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
        : "r"(taddr));
}

__global__ void probe64(unsigned long long* out, int nwarps) {
    __shared__ uint32_t holder;
    if (threadIdx.x < 32) tc::tmem_alloc(&holder, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = holder;
    const uint32_t warp = threadIdx.x / 32;
    uint32_t acc = 0;
    unsigned long long t0 = clock64();
    if ((int)warp < nwarps) {
        const uint32_t lane_base = ((warp & 3) * 32u) << 16;
        const uint32_t col0 = (warp >> 2) * 128;
        for (int it = 0; it < 256; ++it) {
            uint32_t r[2][64];
            ld_x<64>(tmem + lane_base + col0, r[0]);
            ld_x<64>(tmem + lane_base + col0 + 64, r[1]);
            tc::tmem_ld_wait();
            acc += r[0][0] ^ r[1][63] ^ r[0][17];
        }
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 0x12345u) out[200] = acc;
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 512);
}

__global__ void probe(unsigned long long* out, int nwarps, int loads_per_wait) {
    __shared__ uint32_t holder;
    if (threadIdx.x < 32) tc::tmem_alloc(&holder, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = holder;
    const uint32_t warp = threadIdx.x / 32;
    uint32_t acc = 0;
    unsigned long long t0 = clock64();
    if ((int)warp < nwarps) {
        const uint32_t lane_base = ((warp & 3) * 32u) << 16;
        const uint32_t col0 = (warp >> 2) * 128;
        for (int it = 0; it < 256; ++it) {
            uint32_t r[4][32];
            for (int c = 0; c < 4; c += loads_per_wait) {
                for (int q = 0; q < loads_per_wait; ++q) tc::tmem_ld32(tmem + lane_base + col0 + (c + q) * 32, r[q]);
                tc::tmem_ld_wait();
                for (int q = 0; q < loads_per_wait; ++q) acc += r[q][0] ^ r[q][31];
            }
        }
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 0x12345u) out[200] = acc;
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 512);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 256 * 8);
    for (int nw : {4, 8}) {
        probe64<<<148, 256>>>(d, nw);
        probe64<<<148, 256>>>(d, nw);
        unsigned long long h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double c = 0;
        for (int i = 0; i < 148; ++i) c += h[i];
        c /= 148;
        printf("x64 loads, warps %d: %.1f B/cycle per SM (%.0f cycles) err=%s\n", nw, (double)nw * 256 * 2 * 8192 / c, c,
               cudaGetErrorString(cudaGetLastError()));
    }
    for (int nw : {4, 8})
        for (int lpw : {1, 2, 4}) {
            probe<<<148, 256>>>(d, nw, lpw);
            probe<<<148, 256>>>(d, nw, lpw);
            unsigned long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double c = 0;
            for (int i = 0; i < 148; ++i) c += h[i];
            c /= 148;
            const double bytes = (double)nw * 256 * 4 * 4096;
            printf("warps %d, %d loads per wait: %.1f B/cycle per SM (%.0f cycles) err=%s\n", nw, lpw, bytes / c, c,
                   cudaGetErrorString(cudaGetLastError()));
        }
}
