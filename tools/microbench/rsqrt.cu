// Accuracy of the fp64 MUFU reciprocal-square-root seed and of one Newton
// step (dev aid).  nvcc -arch=sm_100a -O3 rsqrt.cu -o rsqrt && ./rsqrt
// For s in a log-uniform sweep over [1e-30, 1e30] and dense mantissa sweeps,
// reports max |y*sqrt(s) - 1| of: the seed, the quadratic step
// y (3 - s y^2) / 2 and the cubic step used by dt_rsqrt.
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>

__device__ double seed(double s)
{
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(s));
    return y;
}

__global__ void probe(const double *s, int n, double *out)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    const double x = s[i];
    const double y0 = seed(x);
    const double t = x * y0;
    const double g = __fma_rn(-t, y0, 3.0);  // 3 - s y0^2
    const double yq = 0.5 * y0 * g;
    const double e = __fma_rn(-t, y0, 1.0);
    const double p = __fma_rn(0.375, e, 0.5);
    const double yc = __fma_rn(y0 * e, p, y0);
    out[3 * i + 0] = y0;
    out[3 * i + 1] = yq;
    out[3 * i + 2] = yc;
}

int main()
{
    const int n = 1 << 24;
    double *hs = new double[n], *ho = new double[3 * (size_t)n];
    unsigned long long z = 12345;
    for (int i = 0; i < n; ++i) {
        z = z * 6364136223846793005ULL + 1442695040888963407ULL;
        double u = (double)(z >> 11) * (1.0 / 9007199254740992.0);
        if (i < n / 2)
            hs[i] = pow(10.0, -30.0 + 60.0 * u);
        else
            hs[i] = 1.0 + 3.0 * u;  // dense over two binades of mantissa
    }
    double *ds, *dout;
    cudaMalloc(&ds, sizeof(double) * n);
    cudaMalloc(&dout, sizeof(double) * 3 * n);
    cudaMemcpy(ds, hs, sizeof(double) * n, cudaMemcpyHostToDevice);
    probe<<<(n + 255) / 256, 256>>>(ds, n, dout);
    cudaMemcpy(ho, dout, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost);
    double mx[3] = {0, 0, 0}, mean[3] = {0, 0, 0};
    for (int i = 0; i < n; ++i) {
        long double r = 1.0L / sqrtl((long double)hs[i]);
        for (int k = 0; k < 3; ++k) {
            double e = (double)(((long double)ho[3 * i + k] - r) / r);
            mx[k] = fmax(mx[k], fabs(e));
            mean[k] += e / n;
        }
    }
    printf("seed      max rel %.3e (2^%.2f) mean %.3e\n", mx[0], log2(mx[0]), mean[0]);
    printf("quadratic max rel %.3e (2^%.2f) mean %.3e\n", mx[1], log2(mx[1]), mean[1]);
    printf("cubic     max rel %.3e (2^%.2f) mean %.3e\n", mx[2], log2(mx[2]), mean[2]);
    return 0;
}
