// Dev probe: cycles of the interior-solve tile loop (4-way body, contiguous inputs) for one warp
// alone on an SM, per iteration, vs iterations and G (values and inputs in shared memory).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(long long* out, int iters, int lg, int reps) {
    __shared__ double M[4096];
    __shared__ double X[2048];
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) M[i] = 1e-3 * i;
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) X[i] = 1.0 + 1e-6 * i;
    __syncthreads();
    const int G = 1 << lg, S = 32, g = lane & (G - 1);
    double acc = 0.0;
    long long best = 1 << 30;
    for (int rep = 0; rep < reps; ++rep) {
        __syncwarp();
        const long long t0 = clock64();
        const double* m = M + lane;
        const double* v = X + 7 + g + rep;
        double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
        const int full = iters & ~3, rem = iters & 3;
#pragma unroll 1
        for (int t = 0; t < full; t += 4) {
            s0 = fma(m[0], v[0], s0);
            s1 = fma(m[S], v[G], s1);
            s2 = fma(m[2 * S], v[2 * G], s2);
            s3 = fma(m[3 * S], v[3 * G], s3);
            m += 4 * S;
            v += 4 * G;
        }
        if (rem > 0) s0 = fma(m[0], v[0], s0);
        if (rem > 1) s1 = fma(m[S], v[G], s1);
        if (rem > 2) s2 = fma(m[2 * S], v[2 * G], s2);
        acc += (s0 + s1) + (s2 + s3);
        __syncwarp();
        const long long t1 = clock64();
        if (t1 - t0 < best) best = t1 - t0;
    }
    if (threadIdx.x == 0) { out[0] = best; }
    if (acc == 12345.0) out[1] = 1;
}
// 8-way body, 8 accumulators
__global__ void probe8(long long* out, int iters, int lg, int reps) {
    __shared__ double M[4096];
    __shared__ double X[2048];
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) M[i] = 1e-3 * i;
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) X[i] = 1.0 + 1e-6 * i;
    __syncthreads();
    const int G = 1 << lg, S = 32, g = lane & (G - 1);
    double acc = 0.0;
    long long best = 1 << 30;
    for (int rep = 0; rep < reps; ++rep) {
        __syncwarp();
        const long long t0 = clock64();
        const double* m = M + lane;
        const double* v = X + 7 + g + rep;
        double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const int full = iters & ~7;
#pragma unroll 1
        for (int t = 0; t < full; t += 8) {
            double a[8], b[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) { a[q] = m[q * S]; b[q] = v[q * G]; }
#pragma unroll
            for (int q = 0; q < 8; ++q) s[q] = fma(a[q], b[q], s[q]);
            m += 8 * S;
            v += 8 * G;
        }
#pragma unroll
        for (int q = 0; q < 7; ++q)
            if (full + q < iters) s[q] = fma(m[q * S], v[q * G], s[q]);
        acc += ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
        __syncwarp();
        const long long t1 = clock64();
        if (t1 - t0 < best) best = t1 - t0;
    }
    if (threadIdx.x == 0) { out[0] = best; }
    if (acc == 12345.0) out[1] = 1;
}

// values in iteration pairs: one 16-byte load per two iterations
__global__ void probe2(long long* out, int iters, int lg, int reps) {
    __shared__ __align__(16) double M[4096];
    __shared__ double X[2048];
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) M[i] = 1e-3 * i;
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) X[i] = 1.0 + 1e-6 * i;
    __syncthreads();
    const int G = 1 << lg, S = 32, g = lane & (G - 1);
    double acc = 0.0;
    long long best = 1 << 30;
    for (int rep = 0; rep < reps; ++rep) {
        __syncwarp();
        const long long t0 = clock64();
        const double* m = M + 2 * lane;
        const double* v = X + 7 + g + rep;
        double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
        const int full = iters & ~3, rem = iters & 3;
#pragma unroll 1
        for (int t = 0; t < full; t += 4) {
            const double2 a = *reinterpret_cast<const double2*>(m);
            const double2 b = *reinterpret_cast<const double2*>(m + 2 * S);
            s0 = fma(a.x, v[0], s0);
            s1 = fma(a.y, v[G], s1);
            s2 = fma(b.x, v[2 * G], s2);
            s3 = fma(b.y, v[3 * G], s3);
            m += 4 * S;
            v += 4 * G;
        }
        if (rem > 0) s0 = fma(m[0], v[0], s0);
        if (rem > 1) s1 = fma(m[1], v[G], s1);
        if (rem > 2) s2 = fma(m[2 * S], v[2 * G], s2);
        acc += (s0 + s1) + (s2 + s3);
        __syncwarp();
        const long long t1 = clock64();
        if (t1 - t0 < best) best = t1 - t0;
    }
    if (threadIdx.x == 0) { out[0] = best; }
    if (acc == 12345.0) out[1] = 1;
}

int main() {
    long long* d; cudaMalloc(&d, 16); long long h[2];
    for (int lg : {0, 2}) for (int it : {3, 6, 14, 24, 64}) {
        probe<<<1, 32>>>(d, it, lg, 50); cudaDeviceSynchronize();
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("G %d iters %2d: %lld cycles (%.1f per iteration)\n", 1 << lg, it, h[0], double(h[0]) / it);
    }
    for (int lg : {0, 2}) for (int it : {3, 6, 14, 24, 64}) {
        probe8<<<1, 32>>>(d, it, lg, 50); cudaDeviceSynchronize();
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("8-way G %d iters %2d: %lld cycles (%.1f per iteration)\n", 1 << lg, it, h[0], double(h[0]) / it);
    }
    for (int w : {32, 128, 512}) {
        probe<<<1, w>>>(d, 24, 2, 50); cudaDeviceSynchronize();
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        long long a = h[0];
        probe2<<<1, w>>>(d, 24, 2, 50); cudaDeviceSynchronize();
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("%d threads, G 4 iters 24: LDS.64 %lld cycles, paired LDS.128 %lld cycles\n", w, a, h[0]);
    }
}
