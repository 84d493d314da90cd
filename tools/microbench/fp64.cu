// FP64 latency / throughput probes on one SM (dev aid).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64.cu -o /tmp/fp64 && /tmp/fp64
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

__global__ void chain(double *p, int n, unsigned long long *t)
{
    double a = p[threadIdx.x], b = 1.0000001;
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int k = 0; k < n; ++k) {
        a = fma(a, b, 1e-9);
        a = fma(a, b, 1e-9);
        a = fma(a, b, 1e-9);
        a = fma(a, b, 1e-9);
    }
    unsigned long long t1 = clock64();
    p[threadIdx.x] = a;
    if (threadIdx.x == 0)
        t[0] = t1 - t0;
}

// 8 independent chains per thread: throughput with blockDim threads on one SM
__global__ void thru(double *p, int n, unsigned long long *t)
{
    double a[8], b = 1.0000001;
    for (int i = 0; i < 8; ++i)
        a[i] = p[threadIdx.x] + i;
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int k = 0; k < n; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i)
            a[i] = fma(a[i], b, 1e-9);
    __syncthreads();
    unsigned long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < 8; ++i)
        s += a[i];
    p[threadIdx.x] = s;
    if (threadIdx.x == 0)
        t[0] = t1 - t0;
}

// dependent: DADD -> DMUL -> DSETP -> ballot -> select (the walk's MAC chain)
__global__ void mac_chain(double *p, int n, unsigned long long *t)
{
    double y = p[threadIdx.x], c = 0.5, th = 1.0 / 3.0;
    unsigned m = 0;
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int k = 0; k < n; ++k) {
        double d = c - y;
        bool far = 0.1 <= th * fabs(d);
        m = __ballot_sync(0xffffffffu, far);
        c = m & 1 ? c + 1e-9 : c - 1e-9;
    }
    unsigned long long t1 = clock64();
    p[threadIdx.x] = c + m;
    if (threadIdx.x == 0)
        t[0] = t1 - t0;
}

// dependent 256-bit loads hitting L1
__global__ void ld_chain(const double4 *nodes, int n, double *out, unsigned long long *t)
{
    int i = threadIdx.x & 7;
    double acc = 0;
    for (int k = 0; k < 64; ++k)
        acc += nodes[k].x;  // warm
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int k = 0; k < n; ++k) {
        double4 r;
        asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                     : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(nodes + i));
        i = __double2loint(r.z);
        acc += r.x;
    }
    unsigned long long t1 = clock64();
    out[threadIdx.x] = acc + i;
    if (threadIdx.x == 0)
        t[0] = t1 - t0;
}

int main()
{
    double *p;
    unsigned long long *t, ht;
    cudaMalloc(&p, 1 << 20);
    cudaMemset(p, 0, 1 << 20);
    cudaMalloc(&t, 64);
    double4 hn[64];
    for (int k = 0; k < 64; ++k) {
        int nx = (k * 5 + 3) & 7;
        long long bits = nx;
        double z;
        memcpy(&z, &bits, 8);
        hn[k] = make_double4(1.0, 2.0, z, 0.0);
    }
    double4 *nodes;
    cudaMalloc(&nodes, sizeof(hn));
    cudaMemcpy(nodes, hn, sizeof(hn), cudaMemcpyHostToDevice);
    const int n = 4000;
    for (int rep = 0; rep < 2; ++rep) {
        chain<<<1, 32>>>(p, n, t);
        cudaMemcpy(&ht, t, 8, cudaMemcpyDeviceToHost);
        printf("dfma dependent latency: %.2f cycles\n", (double)ht / (4.0 * n));
        for (int w = 1; w <= 32; w *= 2) {
            thru<<<1, 32 * w>>>(p, n, t);
            cudaMemcpy(&ht, t, 8, cudaMemcpyDeviceToHost);
            printf("dfma throughput %2d warps/SM: %.3f warp-instr/cycle/SM\n", w,
                   8.0 * n * w / (double)ht);
        }
        mac_chain<<<1, 32>>>(p, n, t);
        cudaMemcpy(&ht, t, 8, cudaMemcpyDeviceToHost);
        printf("mac chain (dadd,dmul,dsetp,vote,sel): %.1f cycles\n", (double)ht / n);
        ld_chain<<<1, 32>>>(nodes, n, p, t);
        cudaMemcpy(&ht, t, 8, cudaMemcpyDeviceToHost);
        printf("dependent 256-bit L1-hit load: %.1f cycles\n", (double)ht / n);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
