// halo_desc_test.cu — can one SWIZZLE_128B smem window serve every tap of a 3×3 conv?
//
// (1) TMA box loads of 34 rows × 128 B (one padded image row of 64 bf16 channels) into smem
//     destinations that are only 128-B aligned (4352·k), checked against the address-based
//     swizzle: 16-B chunk j of a row at smem address A sits at chunk j ^ ((A >> 7) & 7).
// (2) tcgen05.mma (M=128, N=256, K=64, both operands K-major SW128) whose B descriptor starts
//     `off` rows (128-B steps, not 1024-aligned) into that window, with the descriptor's base
//     offset field 0 or (start >> 7) & 7, against a CPU product.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2604_04736_b200/csrc
//        halo_desc_test.cu -o halo_desc_test
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

// smem: [A: 128 rows × 128 B at a 1024-aligned base][pad][window: kRows rows at base2 (1024-aligned)
// + 4352·k per box]. out_layout[r][j] = global row index found in chunk j of window row r (-1 if
// the chunk does not hold the expected row); D = A · B[off .. off+256)ᵀ.
__global__ void __launch_bounds__(128, 1) k_test(const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapA,
                                                 int off, int bo_mode, float* D, int* layout_ok) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;                      // 16 KB
    uint8_t* sW = smem + 16384;              // window
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
        mbar_arrive_expect_tx(&bar, 16384 + kRows * 128);
        tma_load_2d(&mapA, &bar, sA, 0, 0);
        for (int b = 0; b < kRows / kBox; ++b) tma_load_2d(&mapB, &bar, sW + b * kBox * 128, 0, b * kBox);
    }
    mbar_wait(&bar, 0);
    // (1) layout: window row r holds global row r; element (r, 8j) is written as r*64 + 8j so
    // chunk position p holds element index r*64 + 8*(p ^ phase)
    int bad = 0;
    for (int r = threadIdx.x; r < kRows; r += blockDim.x) {
        const uint32_t A = smem_u32(sW + r * 128);
        const int phase = (A >> 7) & 7;
        for (int p = 0; p < 8; ++p) {
            const __nv_bfloat16 v = reinterpret_cast<const __nv_bfloat16*>(sW + r * 128)[p * 8];
            const float want = (float)((r * 64 + 8 * (p ^ phase)) % 251);
            if (__bfloat162float(v) != want) ++bad;
        }
    }
    atomicAdd(layout_ok, bad);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = idesc_bf16(128, 256, 0, 0);
        const uint32_t aBase = smem_u32(sA), bStart = smem_u32(sW) + 128 * off;
        for (int q = 0; q < 4; ++q) {
            const uint64_t ad = sdesc_sw128(aBase + 32 * q, 16, 1024);
            uint64_t bd = sdesc_sw128(bStart + 32 * q, 16, 1024);
            if (bo_mode) bd |= (uint64_t)((bStart >> 7) & 7) << 49;
            mma_bf16(tmem, ad, bd, idesc, q ? 1u : 0u);
        }
        mma_commit(&mbar);
    }
    mbar_wait(&mbar, 0);
    tc_fence_after();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int c = 0; c < 256; c += 32) {
        float v[32];
        tmem_ld32(tmem + (static_cast<uint32_t>(32 * warp) << 16) + c, v);
        for (int j = 0; j < 32; ++j) D[(32 * warp + lane) * 256 + c + j] = v[j];
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc(tmem, 256);
    }
}

int main() {
    std::vector<__nv_bfloat16> hB(kRows * 64), hA(128 * 64);
    for (int r = 0; r < kRows; ++r)
        for (int c = 0; c < 64; ++c) hB[r * 64 + c] = __float2bfloat16((float)((r * 64 + c) % 251));
    for (int r = 0; r < 128; ++r)
        for (int c = 0; c < 64; ++c) hA[r * 64 + c] = __float2bfloat16((float)(((r * 7 + c * 3) % 13) - 6) / 8.0f);
    __nv_bfloat16 *dB, *dA;
    cudaMalloc(&dB, hB.size() * 2);
    cudaMalloc(&dA, hA.size() * 2);
    cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
    CUtensorMap mB, mA;
    cuuint64_t dimsB[2] = {64, (cuuint64_t)kRows}, strB[1] = {128};
    cuuint32_t boxB[2] = {64, kBox}, es[2] = {1, 1};
    cuuint64_t dimsA[2] = {64, 128}, strA[1] = {128};
    cuuint32_t boxA[2] = {64, 128};
    auto enc = encode();
    if (enc(&mB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dB, dimsB, strB, boxB, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ||
        enc(&mA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dA, dimsA, strA, boxA, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) {
        printf("encode failed\n");
        return 1;
    }
    float* dD;
    int* dOk;
    cudaMalloc(&dD, 128 * 256 * 4);
    cudaMalloc(&dOk, 4);
    const int smem = 1024 + 16384 + kRows * 128 + 1024;
    cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    std::vector<float> hD(128 * 256);
    for (int bo = 0; bo < 2; ++bo)
        for (int off : {0, 1, 2, 3, 7, 8, 33, 34, 35, 69, 100}) {
            cudaMemset(dOk, 0, 4);
            cudaMemset(dD, 0, 128 * 256 * 4);
            k_test<<<1, 128, smem>>>(mB, mA, off, bo, dD, dOk);
            cudaError_t e = cudaDeviceSynchronize();
            int ok = -1;
            cudaMemcpy(&ok, dOk, 4, cudaMemcpyDeviceToHost);
            cudaMemcpy(hD.data(), dD, hD.size() * 4, cudaMemcpyDeviceToHost);
            double maxerr = 0.0;
            for (int m = 0; m < 128; ++m)
                for (int n = 0; n < 256; ++n) {
                    double ref = 0.0;
                    for (int k = 0; k < 64; ++k)
                        ref += (double)__bfloat162float(hA[m * 64 + k]) * (double)__bfloat162float(hB[(off + n) * 64 + k]);
                    maxerr = fmax(maxerr, fabs(ref - hD[m * 256 + n]));
                }
            printf("base_offset_field=%s off=%3d: TMA layout mismatches %d, MMA max |err| %.3g (%s)\n",
                   bo ? "(start>>7)&7" : "0          ", off, ok, maxerr, cudaGetErrorString(e));
        }
    return 0;
}
