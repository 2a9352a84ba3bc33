// mn_desc_test.cu — MN-major SWIZZLE_128B operands read straight out of one halo window, for a
// row-packed stage-1 weight gradient (kernels_conv64.cu):
//   A (M = 128): rows 0-63 = channel m at window rows a_off + k; rows 64-127 = the same window one
//     row later (LBO = 128 B: the second 64-wide M block starts one 128-B row further);
//   B (N = 192): three 64-wide N blocks at window rows b_off + j·L + k (LBO = L·128 B, L = W + 2:
//     the three kernel rows of one tap column);
//   D[m][n] = Σ_{k<64} A[m][k] B[n][k] against a CPU product, for several offsets.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2604_04736_b200/csrc
//        mn_desc_test.cu -o mn_desc_test
#include <cmath>
#include <cstdio>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace bnn::ptx;

constexpr int kRows = 34 * 11;   // 11 TMA boxes of 34 rows
constexpr int kBox = 34;

static PFN_cuTensorMapEncodeTiled_v12000 encode() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__global__ void __launch_bounds__(128, 1) k_test(const __grid_constant__ CUtensorMap mapB, int a_off, int b_off, int L,
                                                 float* D) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
    uint8_t* sW = smem;
    __shared__ uint64_t bar, mbar;
    __shared__ uint32_t slot;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init(&mbar, 1);
        mbar_fence_init();
    }
    if (threadIdx.x < 32) tmem_alloc(&slot, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar, kRows * 128);
        for (int b = 0; b < kRows / kBox; ++b) tma_load_2d(&mapB, &bar, sW + b * kBox * 128, 0, b * kBox);
    }
    mbar_wait(&bar, 0);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = idesc_bf16(128, 192, 1, 1);
        const uint32_t aStart = smem_u32(sW) + 128 * a_off, bStart = smem_u32(sW) + 128 * b_off;
        for (int q = 0; q < 4; ++q) {  // K = 16 window rows per MMA
            const uint64_t ad = sdesc_sw128(aStart + 2048 * q, 128, 1024);
            const uint64_t bd = sdesc_sw128(bStart + 2048 * q, 128 * L, 1024);
            mma_bf16(tmem, ad, bd, idesc, q ? 1u : 0u);
        }
        mma_commit(&mbar);
    }
    mbar_wait(&mbar, 0);
    tc_fence_after();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int c = 0; c < 192; c += 32) {
        float v[32];
        tmem_ld32(tmem + (static_cast<uint32_t>(32 * warp) << 16) + c, v);
        for (int j = 0; j < 32; ++j) D[(32 * warp + lane) * 192 + c + j] = v[j];
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc(tmem, 256);
    }
}

int main() {
    std::vector<__nv_bfloat16> hB(kRows * 64);
    for (int r = 0; r < kRows; ++r)
        for (int c = 0; c < 64; ++c) hB[r * 64 + c] = __float2bfloat16((float)(((r * 37 + c * 11) % 17) - 8) / 8.0f);
    __nv_bfloat16* dB;
    cudaMalloc(&dB, hB.size() * 2);
    cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
    CUtensorMap mB;
    cuuint64_t dimsB[2] = {64, (cuuint64_t)kRows}, strB[1] = {128};
    cuuint32_t boxB[2] = {64, kBox}, es[2] = {1, 1};
    auto enc = encode();
    if (enc(&mB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dB, dimsB, strB, boxB, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) {
        printf("encode failed\n");
        return 1;
    }
    float* dD;
    cudaMalloc(&dD, 128 * 192 * 4);
    const int smem = 1024 + kRows * 128 + 1024;
    cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    std::vector<float> hD(128 * 192);
    auto w = [&](int r, int c) { return (double)__bfloat162float(hB[r * 64 + c]); };
    int fails = 0;
    for (int L : {34, 18, 10})
        for (int a_off : {0, 1, 3, 8, 35, 100})
            for (int b_off : {0, 1, 2, 7, 9, 66}) {
                cudaMemset(dD, 0, 128 * 192 * 4);
                k_test<<<1, 128, smem>>>(mB, a_off, b_off, L, dD);
                cudaError_t e = cudaDeviceSynchronize();
                cudaMemcpy(hD.data(), dD, hD.size() * 4, cudaMemcpyDeviceToHost);
                double maxerr = 0.0;
                for (int m = 0; m < 128; ++m)
                    for (int n = 0; n < 192; ++n) {
                        double ref = 0.0;
                        for (int k = 0; k < 64; ++k)
                            ref += w(a_off + k + (m >= 64), m % 64) * w(b_off + (n / 64) * L + k, n % 64);
                        maxerr = fmax(maxerr, fabs(ref - hD[m * 192 + n]));
                    }
                if (maxerr > 1e-3 || e != cudaSuccess) ++fails;
                printf("L=%2d a_off=%3d b_off=%3d: MMA max |err| %.3g (%s)\n", L, a_off, b_off, maxerr, cudaGetErrorString(e));
            }
    printf("%s: %d failing cases\n", fails ? "FAIL" : "OK", fails);
    return 0;
}
