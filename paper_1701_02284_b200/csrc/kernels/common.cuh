// Shared host/device plumbing for the sm_100a kernels: status handling,
// launch accounting and the TMA descriptor encoder (fetched from the driver
// at run time so the library loads on machines without libcuda).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <string>
#include <utility>

#include "status.hpp"
#include "tc_abi.h"

namespace tcb {

extern std::atomic<unsigned long long> g_launches;

inline void count_launch(unsigned n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

#define TCB_CUDA_CHECK(expr)                                                                               \
    do {                                                                                                   \
        cudaError_t _e = (expr);                                                                           \
        if (_e != cudaSuccess)                                                                             \
            return ::tcb::fail(TC_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(_e));        \
    } while (0)

#define TCB_LAUNCH_CHECK()                                                                                 \
    do {                                                                                                   \
        cudaError_t _e = cudaGetLastError();                                                               \
        if (_e != cudaSuccess) return ::tcb::fail(TC_CUDA_ERROR, std::string("launch: ") + cudaGetErrorString(_e)); \
        ::tcb::count_launch();                                                                             \
    } while (0)

// 2D bf16 tensor map with 128-byte swizzle.  inner = contiguous extent,
// outer = row count, row_stride in elements.
bool make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_stride,
                       uint32_t box_inner, uint32_t box_outer, std::string* err);

// Programmatic dependent launch (PDL): every kernel of the step is launched with
// programmatic stream serialisation, starts with griddepcontrol.wait (no global memory
// access before the previous kernel has completed and flushed) and immediately allows
// its own dependents to launch, so a kernel's launch latency and prologue (barrier
// init, TMEM allocation, tensor-map prefetch) overlap the tail of its predecessor.
// On for the GEMMs only by default (TCB_PDL, see pdl_mode() in gemm.cu).
bool pdl_enabled();
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Launch priority: the step's kernels run at the device's greatest priority and the
// side-stream momentum update (launch_sgd) at the least, so the block scheduler fills SMs
// with update blocks only when no step kernel is waiting for them (a persistent GEMM CTA needs
// a whole SM).  TCB_PRIO=0 launches everything at the default priority.
int launch_priority();
struct LowPriorityScope {  // launches inside the scope get the least priority
    LowPriorityScope();
    ~LowPriorityScope();
};

template <typename... KArgs, typename... Args>
inline cudaError_t launch_kernel(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                 Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    attr[1].id = cudaLaunchAttributePriority;
    attr[1].val.priority = launch_priority();
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
// Same, launched as thread-block clusters of `cluster` CTAs.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_kernel_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                         dim3 cluster, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[3];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = cluster.x;
    attr[1].val.clusterDim.y = cluster.y;
    attr[1].val.clusterDim.z = cluster.z;
    attr[2].id = cudaLaunchAttributePriority;
    attr[2].val.priority = launch_priority();
    cfg.attrs = attr;
    cfg.numAttrs = 3;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
#define TCB_LAUNCH(kernel, ...) ::tcb::launch_kernel(kernel, __VA_ARGS__)  // (kernel, grid, block, smem, stream, args...)

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

// Momentum-SGD update of one parameter: v = mu v + alpha (g + d p), p += v, with the
// rounding pinned (explicit fma / mul / add) so the standalone update kernel and the update fused
// into the FC filter-gradient epilogue produce identical bits.
__device__ __forceinline__ void sgd_update1(float& p, float& v, float g, float mom, float lr, float decay) {
    const float nv = __fmaf_rn(mom, v, __fmul_rn(lr, __fmaf_rn(decay, p, g)));
    v = nv;
    p = __fadd_rn(p, nv);
}
__device__ __forceinline__ void sgd_update1_scaled(float& p, float& v, float g, float mom, float lr, float decay,
                                                   float scale) {
    const float nv = __fmaf_rn(mom, v, __fmul_rn(lr, __fmul_rn(scale, __fmaf_rn(decay, p, g))));
    v = nv;
    p = __fadd_rn(p, nv);
}
int num_sms();

}  // namespace tcb
