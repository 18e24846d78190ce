// Microbenchmark (dev tool): per-SM HBM -> shared-memory streaming throughput on B200 for
// the copy mechanisms the interior solve can use.
//   mode 0: per-warp cp.async.bulk (TMA bulk), unit U bytes, D slots per warp
//   mode 1: per-warp cp.async (LDGSTS, 16 B per lane), unit U, D slots (commit groups)
//   mode 2: one producer thread per CTA, cp.async.bulk, slot U, D*16 slots, consumers release
// nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a tools/stream_bench.cu -o build/stream_bench
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e = (x);                                                               \
        if (e != cudaSuccess) {                                                            \
            printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__);                    \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, int c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c));
}
__device__ __forceinline__ void mb_tx(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t par) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(
                     su(b)),
                 "r"(par)
                 : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(d)),
                 "l"(s), "r"(n), "r"(su(b))
                 : "memory");
}

// mode 0 / 1: each warp streams `per_warp` bytes starting at its slice
template <int MODE>
__global__ void __launch_bounds__(512, 1) k_warp(const unsigned char* g, long long per_warp, int U, int D, double* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm) + warp * 8;
    unsigned char* ring = sm + 16 * 8 * 8 + (size_t)warp * D * U;
    const unsigned char* src = g + ((long long)blockIdx.x * 16 + warp) * per_warp;
    const long long n = per_warp / U;
    if (MODE == 0 && lane < D) mb_init(&bars[lane], 1);
    __syncwarp();
    double acc = 0;
    if (MODE == 0) {
        for (int i = 0; i < D && i < n; ++i)
            if (lane == 0) {
                mb_tx(&bars[i], U);
                bulk(ring + i * U, src + (long long)i * U, U, &bars[i]);
            }
        for (long long i = 0; i < n; ++i) {
            const int s = i % D;
            mb_wait(&bars[s], (i / D) & 1);
            acc += reinterpret_cast<const double*>(ring + s * U)[lane];
            __syncwarp();
            if (i + D < n && lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mb_tx(&bars[s], U);
                bulk(ring + s * U, src + (i + D) * U, U, &bars[s]);
            }
        }
    } else {
        auto issue = [&](long long i) {
            const int s = i % D;
            for (int o = lane * 16; o < U; o += 512) {
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(ring + s * U + o)), "l"(src + i * U + o));
            }
            asm volatile("cp.async.commit_group;");
        };
        for (int i = 0; i < D - 1 && i < n; ++i) issue(i);
        for (long long i = 0; i < n; ++i) {
            if (i + D - 1 < n) issue(i + D - 1);
            else asm volatile("cp.async.commit_group;");
            asm volatile("cp.async.wait_group %0;" ::"n"(3));  // keep up to D-1 groups in flight (D <= 4)
            __syncwarp();
            acc += reinterpret_cast<const double*>(ring + (i % D) * U)[lane];
            __syncwarp();
        }
    }
    if (acc == 12345.0) sink[0] = acc;
}

int main(int argc, char** argv) {
    const long long total = 1ll << 30;
    unsigned char* g;
    CK(cudaMalloc(&g, total));
    CK(cudaMemset(g, 1, total));
    double* sink;
    CK(cudaMalloc(&sink, 8));
    int nsm;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 2; ++mode)
        for (int U : {1024, 2048, 4096, 8192}) {
            for (int D : {2, 4}) {
                if (mode == 1 && D != 4) continue;
                for (int ctas : {128, nsm}) {
                    const long long per_warp = (total / (ctas * 16)) / U * U;
                    const size_t smem = 16 * 8 * 8 + (size_t)16 * D * U;
                    if (smem > 227 * 1024) continue;
                    auto kern = mode == 0 ? k_warp<0> : k_warp<1>;
                    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                    kern<<<ctas, 512, smem>>>(g, per_warp, U, D, sink);
                    CK(cudaDeviceSynchronize());
                    cudaEventRecord(e0);
                    for (int r = 0; r < 3; ++r) kern<<<ctas, 512, smem>>>(g, per_warp, U, D, sink);
                    cudaEventRecord(e1);
                    CK(cudaEventSynchronize(e1));
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    const double bytes = 3.0 * per_warp * 16 * ctas;
                    printf("mode %d (%s) U=%5d D=%d ctas=%3d : %7.1f GB/s total, %6.1f GB/s per SM\n", mode,
                           mode == 0 ? "bulk  " : "cp16  ", U, D, ctas, bytes / ms / 1e6, bytes / ms / 1e6 / ctas);
                }
            }
        }
    return 0;
}
