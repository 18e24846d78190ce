// Dev probe: dependent-chain latencies (cycles per op) of DFMA, DADD, LDS.64, SHFL, IMAD on one
// warp of an otherwise idle SM (what one tile of the interior solve waits on).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(long long* out, double seed, int n) {
    __shared__ double sm[1024];
    __shared__ int si[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sm[i] = 1.0 + 1e-9 * i; si[i] = (i * 7 + 1) & 1023; }
    __syncthreads();
    double a = seed, b = 1.000000001, c = 1e-12;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = fma(a, b, c);
    long long t1 = clock64();
    double d = seed;
    for (int i = 0; i < n; ++i) d = d + c;
    long long t2 = clock64();
    int idx = threadIdx.x;
    for (int i = 0; i < n; ++i) idx = si[idx];
    long long t3 = clock64();
    double e = seed;
    for (int i = 0; i < n; ++i) e = __shfl_xor_sync(0xffffffffu, e, 1) + 0.0;
    long long t4 = clock64();
    int k = threadIdx.x;
    for (int i = 0; i < n; ++i) k = k * 3 + 1;
    long long t5 = clock64();
    double f = 0.0; int j = threadIdx.x;
    for (int i = 0; i < n; ++i) { f = sm[j] + f; j = (j + 1) & 1023; }
    long long t6 = clock64();
    if (threadIdx.x == 0) {
        out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = t5 - t4; out[5] = t6 - t5;
    }
    if (a == 0.0 && d == 0.0 && e == 0.0 && f == 0.0) out[7] = idx + k;
}
int main() {
    long long* d; cudaMalloc(&d, 64); long long h[8];
    const int n = 4096;
    for (int rep = 0; rep < 2; ++rep) { probe<<<1, 32>>>(d, 1.0, n); cudaDeviceSynchronize(); }
    cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    const char* names[6] = {"DFMA chain", "DADD chain", "LDS.32 pointer chase", "SHFL+DADD chain", "IMAD chain", "LDS.64+DADD chain"};
    for (int i = 0; i < 6; ++i) printf("%-22s %.1f cycles/op\n", names[i], double(h[i]) / n);
}
