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

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }
int num_sms();

}  // namespace tcb
