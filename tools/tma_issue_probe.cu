// Dev probe: cycles a warp spends issuing one unit refill (mbarrier expect_tx + cp.async.bulk by
// one lane) vs the same bytes by 32 lanes with cp.async (LDGSTS) + cp.async.mbarrier.arrive.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void probe(const char* src, long long* out, int reps, int bytes) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
    unsigned char* buf = sm + 256 + (threadIdx.x >> 5) * 8192;
    const int lane = threadIdx.x & 31;
    uint64_t* mb = bar + (threadIdx.x >> 5);
    uint64_t* mb2 = bar + 16 + (threadIdx.x >> 5);
    if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(mb)), "r"(1));
    if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(mb2)), "r"(32));
    __syncthreads();
    long long t_tma = 0, t_cpa = 0;
    uint32_t ph = 0;
    for (int r = 0; r < reps; ++r) {
        const char* s = src + ((r * 37 + blockIdx.x * 5 + (threadIdx.x >> 5)) % 512) * 8192;
        __syncwarp();
        long long t0 = clock64();
        if (lane == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(mb)), "r"(bytes) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(buf)), "l"(s), "r"(bytes), "r"(su32(mb)) : "memory");
        }
        __syncwarp();
        long long t1 = clock64();
        t_tma += t1 - t0;
        asm volatile("{\n\t.reg .pred p;\nW1_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W1_%=;\n}" ::"r"(su32(mb)), "r"(ph) : "memory");
        ph ^= 1;
        // cp.async path: 32 lanes x 16 B per instruction
        __syncwarp();
        t0 = clock64();
        for (int o = lane * 16; o < bytes; o += 512)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(buf + o)), "l"(s + o) : "memory");
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(mb2)) : "memory");
        __syncwarp();
        t1 = clock64();
        t_cpa += t1 - t0;
        asm volatile("{\n\t.reg .pred p;\nW2_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W2_%=;\n}" ::"r"(su32(mb2)), "r"(ph ^ 1) : "memory");
        __syncwarp();
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = t_tma / reps; out[1] = t_cpa / reps; }
}
int main() {
    char* src; long long* d; long long h[2];
    cudaMalloc(&src, 512 * 8192); cudaMemset(src, 0, 512 * 8192); cudaMalloc(&d, 16);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 256 + 16 * 8192);
    for (int bytes : {1024, 2048, 4096}) {
        for (int blocks : {1, 148}) {
            probe<<<blocks, 512, 256 + 16 * 8192>>>(src, d, 200, bytes);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            printf("bytes %d blocks %d: tma issue %lld cycles, cp.async issue %lld cycles (%s)\n", bytes, blocks, h[0], h[1], cudaGetErrorString(e));
        }
    }
}
