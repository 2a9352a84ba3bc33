// mma_bench2.cu — tcgen05.mma issue rate with INDEPENDENT accumulators.
// scripts/mma_bench.cu chained every MMA into one accumulator (each MMA waits for the previous
// one's D): ≈ 130 clk per M=128 K=16 MMA for every N — a latency figure, not the pipe's rate.
// Here the MMAs of one k-step rotate over `nacc` accumulators (N columns apart), so
// consecutive MMAs are independent; clk per MMA vs N and nacc gives the real floor.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2604_04736_b200/csrc mma_bench2.cu -o mma_bench2
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace bnn::ptx;

__global__ void __launch_bounds__(128, 1) mma_loop(int M, int N, int nacc, int iters, long long* cyc) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;             // 16 KB: 128 rows × 64 K (SW128 K-major)
    uint8_t* sB = smem + 16384;     // 32 KB: 256 rows × 64 K
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 49152 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
    }
    if (threadIdx.x < 32) tmem_alloc(&slot, 512);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = idesc_bf16(M, N, 0, 0);
        const uint32_t aBase = smem_u32(sA), bBase = smem_u32(sB);
        long long t0 = clock64();
        uint32_t ph = 0;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint64_t ad = sdesc_sw128(aBase + 32 * q, 16, 1024);
                const uint64_t bd = sdesc_sw128(bBase + 32 * q, 16, 1024);
                const int acc = (it * 4 + q) % nacc;
                mma_bf16(tmem + acc * N, ad, bd, idesc, (it * 4 + q) >= nacc ? 1u : 0u);
            }
            if ((it & 15) == 15) {
                mma_commit(&bar);
                mbar_wait(&bar, ph);
                ph ^= 1;
            }
        }
        mma_commit(&bar);
        mbar_wait(&bar, ph);
        long long t1 = clock64();
        cyc[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

int main() {
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    cudaFuncSetAttribute(mma_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024);
    const int iters = 4096;
    for (int M : {128})
        for (int N : {64, 128, 256})
            for (int nacc : {1, 2, 4, 8}) {
                if (nacc * N > 512) continue;
                mma_loop<<<148, 128, 50 * 1024>>>(M, N, nacc, iters, d);
                cudaDeviceSynchronize();
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                cudaEventRecord(e0);
                mma_loop<<<148, 128, 50 * 1024>>>(M, N, nacc, iters, d);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                long long h[148];
                cudaMemcpy(h, d, 148 * sizeof(long long), cudaMemcpyDeviceToHost);
                double macs = (double)M * N * 64 * iters;
                printf("M=%3d N=%3d nacc=%d: %.1f clk/MMA(K=16)  %.0f MAC/clk/SM  %.1f TFLOP/s (%s)\n", M, N, nacc,
                       (double)h[0] / iters / 4, macs / h[0], 2 * macs * 148 / (ms * 1e9),
                       cudaGetErrorString(cudaGetLastError()));
            }
    return 0;
}
