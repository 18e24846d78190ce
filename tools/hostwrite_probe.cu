// Dev probe: does a grid's last CTA writing a few doubles to mapped pinned host memory (the fused
// convergence flags of update_kernel) lengthen the kernel on B200? 592 CTAs x 512 threads, a
// ticket, the last CTA writes 4 doubles to host (mode 1) or device (mode 0) memory; mean kernel
// time over back-to-back launches (CUDA events).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/hostwrite_probe tools/hostwrite_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) probe(const double* __restrict__ in, double* __restrict__ out, int n,
                                             unsigned* ticket, double* flags) {
    __shared__ int last;
    double acc = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double v = in[i] * 1.0000001;
        out[i] = v;
        acc += v;
    }
    if (acc == 12345.678) out[0] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        *ticket = 0u;
        if (flags) {
            volatile double* h = flags;
            for (int k = 0; k < 4; ++k) h[k] = k + 0.5;
        }
    }
}

int main() {
    const int n = 638401, grid = 592, reps = 2000;
    double *in, *out, *dflags, *hflags, *hdev;
    unsigned* ticket;
    cudaMalloc(&in, n * sizeof(double));
    cudaMalloc(&out, n * sizeof(double));
    cudaMalloc(&dflags, 4 * sizeof(double));
    cudaMalloc(&ticket, sizeof(unsigned));
    cudaMemset(in, 0, n * sizeof(double));
    cudaMemset(ticket, 0, sizeof(unsigned));
    cudaHostAlloc(&hflags, 4 * sizeof(double), cudaHostAllocMapped);
    cudaHostGetDevicePointer(&hdev, hflags, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 3; ++mode) {
        double* f = mode == 0 ? nullptr : mode == 1 ? dflags : hdev;
        for (int w = 0; w < 50; ++w) probe<<<grid, 512>>>(in, out, n, ticket, f);
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) probe<<<grid, 512>>>(in, out, n, ticket, f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        std::printf("%-14s %.3f us per launch\n", mode == 0 ? "no flags" : mode == 1 ? "device flags" : "host flags",
                    1e3 * ms / reps);
    }
    return 0;
}
