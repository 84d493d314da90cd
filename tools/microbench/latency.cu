// Latency microbenchmarks on one warp (dev aid): dependent global loads,
// atomics, fences, shuffles and DFMA chains.  nvcc -arch=sm_100a -O3 latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chase(const long long *next, int n, long long *out, unsigned long long *t)
{
    long long i = 0;
    unsigned long long t0 = clock64();
    for (int k = 0; k < n; ++k)
        i = __ldcg(next + i);
    unsigned long long t1 = clock64();
    out[0] = i;
    t[0] = t1 - t0;
}

__global__ void chase_ca(const long long *next, int n, long long *out, unsigned long long *t)
{
    long long i = 0;
    unsigned long long t0 = clock64();
    for (int k = 0; k < n; ++k)
        i = next[i];
    unsigned long long t1 = clock64();
    out[0] = i;
    t[0] = t1 - t0;
}

__global__ void atom_chain(int *ctr, int n, unsigned long long *t)
{
    int v = 0;
    unsigned long long t0 = clock64();
    for (int k = 0; k < n; ++k)
        v = atomicAdd(ctr + (v & 1), 1);
    unsigned long long t1 = clock64();
    t[0] = t1 - t0;
    t[1] = v;
}

__global__ void fence_chain(double *p, int n, unsigned long long *t)
{
    unsigned long long t0 = clock64();
    for (int k = 0; k < n; ++k) {
        p[threadIdx.x + 32 * (k & 7)] = k;
        __threadfence();
    }
    unsigned long long t1 = clock64();
    t[0] = t1 - t0;
}

__global__ void dfma_chain(double *p, int n, unsigned long long *t)
{
    double a = p[threadIdx.x], b = 1.0000001;
    unsigned long long t0 = clock64();
    for (int k = 0; k < n; ++k)
        a = fma(a, b, 1e-9);
    unsigned long long t1 = clock64();
    p[threadIdx.x] = a;
    t[0] = t1 - t0;
}

__global__ void shfl_fma_chain(double *p, int n, unsigned long long *t)
{
    double a = p[threadIdx.x];
    unsigned long long t0 = clock64();
    for (int k = 0; k < n; ++k)
        a = fma(__shfl_up_sync(0xffffffffu, a, 1), 1.0000001, a);
    unsigned long long t1 = clock64();
    p[threadIdx.x] = a;
    t[0] = t1 - t0;
}

int main()
{
    const int N = 1 << 24;
    long long *next;
    cudaMalloc(&next, N * sizeof(long long));
    long long *h = new long long[N];
    unsigned long long s = 12345;
    for (int i = 0; i < N; ++i) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        h[i] = (long long)((s >> 20) % N);
    }
    cudaMemcpy(next, h, N * sizeof(long long), cudaMemcpyHostToDevice);
    long long *out;
    unsigned long long *t, ht[2];
    cudaMalloc(&out, 64);
    cudaMalloc(&t, 64);
    int *ctr;
    cudaMalloc(&ctr, 64);
    cudaMemset(ctr, 0, 64);
    double *p;
    cudaMalloc(&p, 4096 * 8);
    cudaMemset(p, 0, 4096 * 8);
    const int n = 2000;
    for (int rep = 0; rep < 2; ++rep) {
        chase<<<1, 1>>>(next, n, out, t);
        cudaMemcpy(ht, t, 16, cudaMemcpyDeviceToHost);
        printf("ld.cg dependent (128MB random): %.1f cycles\n", (double)ht[0] / n);
        chase_ca<<<1, 1>>>(next, n, out, t);
        cudaMemcpy(ht, t, 16, cudaMemcpyDeviceToHost);
        printf("ld dependent (128MB random): %.1f cycles\n", (double)ht[0] / n);
        chase<<<1, 1>>>(next, 16, out, t);  // warm small set? (random)
        atom_chain<<<1, 1>>>(ctr, n, t);
        cudaMemcpy(ht, t, 16, cudaMemcpyDeviceToHost);
        printf("atomicAdd dependent: %.1f cycles\n", (double)ht[0] / n);
        fence_chain<<<1, 32>>>(p, n, t);
        cudaMemcpy(ht, t, 16, cudaMemcpyDeviceToHost);
        printf("store + threadfence: %.1f cycles\n", (double)ht[0] / n);
        dfma_chain<<<1, 32>>>(p, n, t);
        cudaMemcpy(ht, t, 16, cudaMemcpyDeviceToHost);
        printf("dfma dependent: %.1f cycles\n", (double)ht[0] / n);
        shfl_fma_chain<<<1, 32>>>(p, n, t);
        cudaMemcpy(ht, t, 16, cudaMemcpyDeviceToHost);
        printf("shfl+dfma dependent: %.1f cycles\n", (double)ht[0] / n);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
