// Probe: does a tcgen05.mma K-major SWIZZLE_128B A operand read correctly from a start address
// shifted by s whole 128-byte rows (s not a multiple of 8) inside a TMA-style swizzled tile?
// The halo-tile implicit GEMM (tc_gemm.cuh, OP_HALO_K) reads each filter tap of a stride-1
// convolution as such a row-shifted view of one staged input tile.
//
// For every shift s in [0, 16) and both settings of the descriptor's matrix-base-offset field
// (bits 49-51: 0, or (start >> 7) & 7), one 128 x 64 x 64 MMA is compared with the host product
//   D[m][n] = sum_k A[m + s][k] * B[n][k].
//
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -Ipaper_1701_02284_b200/csrc/kernels \
//        tools/umma_shift_probe.cu -o /tmp/umma_shift_probe && /tmp/umma_shift_probe
#include <cuda_bf16.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "ptx.cuh"

using namespace tcb;

constexpr int kRows = 256, kN = 64, kShifts = 16;

__device__ __forceinline__ uint64_t desc_sw128_bo(uint32_t saddr, uint32_t base_off) {
    return umma_desc_sw128(saddr, 0, 1024) | (static_cast<uint64_t>(base_off & 7) << 49);
}

__global__ void probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = sm;
    uint8_t* sB = sm + kRows * 128;
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    // SW128 K-major staging: 16-byte chunk j of row r at r*128 + ((j ^ (r & 7)) << 4)
    for (int i = t; i < kRows * 8; i += blockDim.x) {
        const int r = i >> 3, j = i & 7;
        *reinterpret_cast<uint4*>(sA + r * 128 + ((j ^ (r & 7)) << 4)) = reinterpret_cast<const uint4*>(A)[i];
    }
    for (int i = t; i < kN * 8; i += blockDim.x) {
        const int r = i >> 3, j = i & 7;
        *reinterpret_cast<uint4*>(sB + r * 128 + ((j ^ (r & 7)) << 4)) = reinterpret_cast<const uint4*>(B)[i];
    }
    fence_proxy_async_smem();
    if (t == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<1>(&tslot, 64);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    const uint32_t idesc = umma_idesc_bf16(128, kN, 0, 0);
    uint32_t phase = 0;
    for (int v = 0; v < 2; ++v) {
        for (int s = 0; s < kShifts; ++s) {
            if (warp == 0) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t a_addr = smem_u32(sA) + s * 128 + k * 32;
                    const uint64_t ad = desc_sw128_bo(a_addr, v ? (a_addr >> 7) & 7 : 0);
                    const uint64_t bd = desc_sw128_bo(smem_u32(sB) + k * 32, 0);
                    umma_bf16_elect<1>(tmem, ad, bd, idesc, k > 0 ? 1u : 0u);
                }
                umma_commit_elect<1>(&bar);
            }
            mbar_wait(&bar, phase);
            phase ^= 1;
            tc_fence_after();
            uint32_t r0[32], r1[32];
            const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16);
            tmem_ld32(taddr, r0);
            tmem_ld32(taddr + 32, r1);
            tmem_ld_wait();
            float* out = D + ((static_cast<size_t>(v) * kShifts + s) * 128 + warp * 32 + lane) * kN;
            for (int j = 0; j < 32; ++j) {
                out[j] = __uint_as_float(r0[j]);
                out[32 + j] = __uint_as_float(r1[j]);
            }
            tc_fence_before();
            __syncthreads();
            tc_fence_after();
        }
    }
    if (warp == 0) tmem_dealloc<1>(tmem, 64);
}

int main() {
    std::vector<__nv_bfloat16> hA(kRows * 64), hB(kN * 64);
    std::vector<float> fA(hA.size()), fB(hB.size());
    unsigned s = 12345;
    auto rnd = [&] {
        s = s * 1664525u + 1013904223u;
        return static_cast<float>((s >> 9) % 17) - 8.0f;  // small integers: exact in bf16 / fp32
    };
    for (size_t i = 0; i < hA.size(); ++i) fA[i] = rnd(), hA[i] = __float2bfloat16(fA[i]);
    for (size_t i = 0; i < hB.size(); ++i) fB[i] = rnd(), hB[i] = __float2bfloat16(fB[i]);
    __nv_bfloat16 *dA, *dB;
    float* dD;
    const size_t nD = 2ull * kShifts * 128 * kN;
    cudaMalloc(&dA, hA.size() * 2);
    cudaMalloc(&dB, hB.size() * 2);
    cudaMalloc(&dD, nD * 4);
    cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
    const int smem = (kRows + kN) * 128 + 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe<<<1, 128, smem>>>(dA, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("kernel error: %s\n", cudaGetErrorString(e));
        return 1;
    }
    std::vector<float> hD(nD);
    cudaMemcpy(hD.data(), dD, nD * 4, cudaMemcpyDeviceToHost);
    for (int v = 0; v < 2; ++v) {
        printf("base_offset %s:", v ? "(start>>7)&7" : "0");
        for (int sh = 0; sh < kShifts; ++sh) {
            int bad = 0;
            for (int m = 0; m < 128; ++m)
                for (int n = 0; n < kN; ++n) {
                    float ref = 0.f;
                    for (int k = 0; k < 64; ++k) ref += fA[(m + sh) * 64 + k] * fB[n * 64 + k];
                    if (hD[((static_cast<size_t>(v) * kShifts + sh) * 128 + m) * kN + n] != ref) ++bad;
                }
            printf(" s%d:%s", sh, bad ? "BAD" : "ok");
        }
        printf("\n");
    }
    return 0;
}
