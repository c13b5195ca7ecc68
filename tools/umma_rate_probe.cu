// Probe: tensor-pipe cost of one tcgen05.mma kind::f16 (M = 128, K = 16, bf16 -> fp32) for
// N = 32 .. 256, operands resident in shared memory (no loads), issued back to back by one thread
// with a tcgen05.commit every `per_commit` MMAs; and the same with cta_group::1 M = 64.
// Prints clocks per MMA and the implied fraction of the dense peak (8192 FLOP/clk/SM).
//
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -Ipaper_1701_02284_b200/csrc/kernels \
//        tools/umma_rate_probe.cu -o /tmp/umma_rate_probe && /tmp/umma_rate_probe
#include <cuda_bf16.h>

#include <cstdio>
#include <string>

#include "ptx.cuh"

using namespace tcb;

__global__ void rate(int M, int N, int n_mma, int per_commit, long long* out, int a_shift_rows, int two_acc = 0) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar, bar_x;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init(&bar_x, 1);  // intermediate commits land here and are never waited on
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<1>(&tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 0) {
        const uint32_t idesc = umma_idesc_bf16(M, N, 0, 0);
        const uint64_t ad = umma_desc_sw128(smem_u32(sm) + a_shift_rows * 128, 0, 1024);
        const uint64_t bd = umma_desc_sw128(smem_u32(sm) + 32768, 0, 1024);
        uint32_t phase = 0;
        // warm-up
        umma_bf16_elect<1>(tmem, ad, bd, idesc, 0u);
        umma_commit_elect<1>(&bar);
        mbar_wait(&bar, phase);
        phase ^= 1;
        const uint64_t a0 = ad, a1 = ad + 2, a2 = ad + 4, a3 = ad + 6;
        const uint64_t b0 = bd, b1 = bd + 2, b2 = bd + 4, b3 = bd + 6;
        const long long t0 = clock64();
        // one "k-block" = 4 MMAs (K = 64) with a commit after it when per_commit == 4
        if (two_acc) {
            // the halo kernel's pattern: per k-block 2 x 4 MMAs into two accumulators (rows +0 / +128
            // of the A tile, 128 TMEM columns apart), one commit
            for (int i = 0; i < n_mma / 8; ++i) {
#pragma unroll
                for (int sub = 0; sub < 2; ++sub) {
                    const uint32_t d = tmem + sub * 128;
                    const uint64_t as = sub * (128 * 128 >> 4);
                    umma_bf16_elect<1>(d, a0 + as, b0, idesc, 1u);
                    umma_bf16_elect<1>(d, a1 + as, b1, idesc, 1u);
                    umma_bf16_elect<1>(d, a2 + as, b2, idesc, 1u);
                    umma_bf16_elect<1>(d, a3 + as, b3, idesc, 1u);
                }
                umma_commit_elect<1>(&bar_x);
            }
        } else {
            for (int i = 0; i < n_mma / 4; ++i) {
                umma_bf16_elect<1>(tmem, a0, b0, idesc, 1u);
                umma_bf16_elect<1>(tmem, a1, b1, idesc, 1u);
                umma_bf16_elect<1>(tmem, a2, b2, idesc, 1u);
                umma_bf16_elect<1>(tmem, a3, b3, idesc, 1u);
                if (per_commit == 4) umma_commit_elect<1>(&bar_x);
            }
        }
        umma_commit_elect<1>(&bar);  // tracks every MMA issued before it
        mbar_wait(&bar, phase);
        const long long t1 = clock64();
        if (threadIdx.x == 0) *out = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<1>(tmem, 512);
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    long long* d;
    cudaMalloc(&d, sizeof(long long));
    const int smem = 96 * 1024 + 1024;
    cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int n_mma = 4096;
    for (int two : {0, 1}) {
        printf("%s:", two ? "two accumulators, 8 MMAs per commit" : "one accumulator, 4 MMAs per commit");
        for (int N : {64, 96, 128, 256}) {
            rate<<<1, 128, smem>>>(128, N, n_mma, 4, d, 0, two);
            long long h = 0;
            cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
            const double cpm = static_cast<double>(h) / n_mma;
            printf("  N%d %.1f clk (%.0f%%)", N, cpm, 100 * 2.0 * 128 * N * 16 / cpm / 8192.0);
        }
        printf("\n");
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
    return 0;
}
