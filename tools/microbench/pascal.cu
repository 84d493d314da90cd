// Throughput of the in-register Pascal shift (31 passes) on one SM (dev aid).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void pascal(double *p, int reps, unsigned long long *t)
{
    double S[32];
#pragma unroll
    for (int k = 0; k < 32; ++k)
        S[k] = p[k] + threadIdx.x;
    const double delta = 1e-3 * threadIdx.x;
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int i = 1; i < 32; ++i) {
#pragma unroll
            for (int k = 31; k >= i; --k)
                S[k] = fma(delta, S[k - 1], S[k]);
        }
    }
    unsigned long long t1 = clock64();
    double acc = 0;
#pragma unroll
    for (int k = 0; k < 32; ++k)
        acc += S[k];
    p[64 + blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0)
        t[blockIdx.x] = t1 - t0;
}

int main()
{
    double *p;
    unsigned long long *t, ht[8];
    cudaMalloc(&p, 1 << 20);
    cudaMemset(p, 0, 1 << 20);
    cudaMalloc(&t, 64);
    for (int threads = 32; threads <= 256; threads *= 2) {
        pascal<<<1, threads>>>(p, 100, t);
        cudaMemcpy(ht, t, 8, cudaMemcpyDeviceToHost);
        double per = (double)ht[0] / 100;
        printf("threads %d: %.0f cycles per shift (465 DFMA/thread); %.2f warp-DFMA/cycle/SM\n",
               threads, per, 465.0 * threads / 32 / per);
    }
    return 0;
}
