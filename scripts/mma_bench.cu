// mma_bench.cu — tcgen05.mma issue-rate microbenchmark (operands resident in smem, no TMA).
// Measures MAC/clk/SM for M=128 × N ∈ {64,128,256} × K=16 bf16 MMAs, A K-major, B K- or
// MN-major, so the conv/GEMM kernels' tile shapes can be judged against the tensor pipe itself.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2604_04736_b200/csrc mma_bench.cu -o mma_bench -lcuda
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace bnn::ptx;

__global__ void __launch_bounds__(128, 1) mma_loop(int M, int N, int b_mn, int iters, int nbuf, long long* cyc) {
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
        const uint32_t idesc = idesc_bf16(M, N, 0, b_mn);
        const uint32_t aBase = smem_u32(sA), bBase = smem_u32(sB);
        long long t0 = clock64();
        uint32_t ph = 0;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint64_t ad = sdesc_sw128(aBase + 32 * q, 16, 1024);
                const uint64_t bd = b_mn ? sdesc_sw128(bBase + 2048 * q, 8192, 1024) : sdesc_sw128(bBase + 32 * q, 16, 1024);
                mma_bf16(tmem + (it % nbuf) * 256 % 512, ad, bd, idesc, 1u);
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
    for (int M : {64, 128})
    for (int b_mn = 0; b_mn < 2; ++b_mn)
        for (int N : {64, 128, 256}) {
            for (int grid : {148}) {
                mma_loop<<<grid, 128, 50 * 1024>>>(M, N, b_mn, iters, 1, d);
                cudaDeviceSynchronize();
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                cudaEventRecord(e0);
                mma_loop<<<grid, 128, 50 * 1024>>>(M, N, b_mn, iters, 1, d);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                long long h[148];
                cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
                double macs = (double)M * N * 64 * iters;
                printf("M=%3d N=%3d B_%s grid=%3d: %.0f clk/kstep  %.0f MAC/clk/SM  %.1f TFLOP/s (err %s)\n",
                       M, N, b_mn ? "MN" : "K ", grid, (double)h[0] / iters, macs / h[0], 2 * macs * grid / (ms * 1e9),
                       cudaGetErrorString(cudaGetLastError()));
            }
        }
    return 0;
}
