// mma_bench4.cu — is the ≈ 185-cycle-per-MMA ceiling of one tcgen05 issue stream per issuing
// THREAD or per CTA? One CTA per SM; nw warps (lane 0 of each) issue M=128 K=16 MMAs into their
// own TMEM accumulators (N columns each) from the same resident smem operands; each commits to
// its own mbarrier every 64 MMAs. Prints cycles per MMA per issuing warp and the chip TFLOP/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2604_04736_b200/csrc mma_bench4.cu -o mma_bench4
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace bnn::ptx;

__global__ void __launch_bounds__(128, 1) mma_multi(int N, int nw, int iters, int mn, long long* cyc) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;          // 16 KB: 128 rows × 64 K (SW128 K-major)
    uint8_t* sB = smem + 16384;  // 32 KB: 256 rows × 64 K (MN views stay inside 48 KB)
    __shared__ uint64_t bar[4];
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 63488 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
    if (threadIdx.x == 0) {
        for (int w = 0; w < 4; ++w) mbar_init(&bar[w], 1);
        mbar_fence_init();
    }
    if (threadIdx.x < 32) tmem_alloc(&slot, 512);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp < nw && lane == 0) {
        const uint32_t idesc = idesc_bf16(128, N, mn, mn);
        const uint32_t aBase = smem_u32(sA), bBase = smem_u32(sB);
        const uint32_t d = tmem + warp * N;
        long long t0 = clock64();
        uint32_t ph = 0;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                // mn: MN-major views (64-wide blocks LBO apart, 8 K-rows per 1024 B); mn = 2: the
                // conv64 wgrad's views (A blocks 128 B apart, B blocks 4352 B apart)
                const uint64_t ad = mn ? sdesc_sw128(aBase + 2048 * q, mn == 2 ? 128 : 8192, 1024)
                                       : sdesc_sw128(aBase + 32 * q, 16, 1024);
                const uint64_t bd = mn ? sdesc_sw128(bBase + 2048 * q, mn == 2 ? 4352 : 8192, 1024)
                                       : sdesc_sw128(bBase + 32 * q, 16, 1024);
                mma_bf16(d, ad, bd, idesc, (it | q) != 0 ? 1u : 0u);
            }
            if ((it & 15) == 15) {
                mma_commit(&bar[warp]);
                mbar_wait(&bar[warp], ph);
                ph ^= 1;
            }
        }
        mma_commit(&bar[warp]);
        mbar_wait(&bar[warp], ph);
        cyc[blockIdx.x * 4 + warp] = clock64() - t0;
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
    cudaMalloc(&d, 148 * 4 * sizeof(long long));
    cudaFuncSetAttribute(mma_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const int iters = 4096;
    for (int mn : {0, 1, 2})
    for (int N : {64, 128, 192, 256})
        for (int nw : {1, 2, 3, 4}) {
            if (nw * N > 512 || (mn && N != 192 && N != 128)) continue;
            mma_multi<<<148, 128, 64 * 1024>>>(N, nw, iters, mn, d);
            cudaDeviceSynchronize();
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            mma_multi<<<148, 128, 64 * 1024>>>(N, nw, iters, mn, d);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            long long h[4];
            cudaMemcpy(h, d, 4 * sizeof(long long), cudaMemcpyDeviceToHost);
            const double macs = (double)128 * N * 16 * 4 * iters * nw;  // per SM
            printf("%s N=%3d issuing warps=%d: %.1f clk/MMA per warp, chip %.1f TFLOP/s (%s)\n",
                   mn == 0 ? "K-major " : mn == 1 ? "MN-major" : "MN-views", N, nw,
                   (double)h[0] / iters / 4, 2 * macs * 148 / (ms * 1e9), cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
