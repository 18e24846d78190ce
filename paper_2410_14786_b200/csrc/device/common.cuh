// Shared device helpers for the sm_100a BDDC kernels.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "../device_format.hpp"

namespace bddc_b200 {

#define BDDC_CUDA(call)                                                                        \
    do {                                                                                       \
        cudaError_t err__ = (call);                                                            \
        if (err__ != cudaSuccess)                                                              \
            throw std::runtime_error(std::string("CUDA error: ") + cudaGetErrorString(err__) + \
                                     " at " + __FILE__ + ":" + std::to_string(__LINE__));      \
    } while (0)

// Kernel launches issued by this library in this process (bench.py's gpu_launches).
extern std::atomic<std::int64_t> g_kernel_launches;

// Every launch site is followed by exactly one BDDC_LAUNCHED(): checks the launch and counts it.
#define BDDC_LAUNCHED()                                                    \
    do {                                                                   \
        BDDC_CUDA(cudaGetLastError());                                     \
        ::bddc_b200::g_kernel_launches.fetch_add(1, std::memory_order_relaxed); \
    } while (0)

// Programmatic dependent launch (PDL): the PCG loop's kernels are launched with programmatic
// stream serialisation (launch_pdl), so a kernel's CTAs become resident while its predecessor
// drains instead of after it. Each such kernel lets its own dependents launch at entry
// (pdl_trigger) and waits for its predecessor (pdl_wait: that grid complete, its memory
// visible; transitively every earlier grid) before it reads or writes anything a
// predecessor touches. Both are no-ops for kernels launched without the attribute.
// GPU-scope acquire-release fence: what the ticket / arrival-counter patterns (writes, fence,
// relaxed atomic; relaxed read, fence, reads) need. __threadfence() is fence.sc.gpu
// (MEMBAR.SC.GPU), a sequentially consistent fence that costs more on the critical path.
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool pdl_enabled();  // BDDC_PDL=1 turns the attribute on

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    BDDC_CUDA(cudaLaunchKernelEx(&cfg, kernel, args...));
}

// Speculative launches of the pipelined PCG loop pass the solver's scalar block: a set
// converged (scal[2]) or error (scal[3]) flag turns the kernel into a no-op.
__device__ __forceinline__ bool skip_launch(const double* scal) {
    return scal != nullptr && (scal[2] != 0.0 || scal[3] == 1.0);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic block sum (fixed tree); all threads receive the result.
template <int THREADS>
__device__ __forceinline__ double block_sum(double v, double* scratch /* THREADS/32 */) {
    v = warp_sum(v);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (warp == 0) {
        t = lane < THREADS / 32 ? scratch[lane] : 0.0;
        t = warp_sum(t);
        if (lane == 0) scratch[0] = t;
    }
    __syncthreads();
    t = scratch[0];
    __syncthreads();
    return t;
}

// Streaming (read-once) global load: non-coherent path, no L1 allocation.
__device__ __forceinline__ double ld_stream(const double* p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

}  // namespace bddc_b200
