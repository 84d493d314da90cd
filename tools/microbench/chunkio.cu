// One block, 8 warps: each warp loads a 4 KB contiguous chunk (16 rows in
// flight per lane), then stores 16 KB elsewhere; 14 rounds with block
// barriers.  Chunks at random offsets in a large buffer vs. a fixed chunk.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chunkio(const double *src, double *dst, long long span, int rounds, int fixed,
                        unsigned long long *t)
{
    __shared__ double buf[8][512];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long seed = 88172645463325252ull + w;
    unsigned long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
        seed ^= seed << 13; seed ^= seed >> 7; seed ^= seed << 17;
        const long long off = fixed ? 0 : (long long)(seed % (unsigned long long)(span - 4096)) & ~31ll;
        for (int r0 = 0; r0 < 16; r0 += 16) {
            double v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j)
                v[j] = __ldcg(src + off + (r0 + j) * 32 + lane);
#pragma unroll
            for (int j = 0; j < 16; ++j)
                buf[w][(r0 + j) * 32 + lane] = v[j];
        }
        __syncwarp();
        seed ^= seed << 13; seed ^= seed >> 7; seed ^= seed << 17;
        const long long off2 = fixed ? 0 : (long long)(seed % (unsigned long long)(span - 4096)) & ~31ll;
        for (int r0 = 0; r0 < 16; ++r0)
            dst[off2 + r0 * 32 + lane] = buf[w][r0 * 32 + lane] + 1.0;
        __syncthreads();
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0)
        t[0] = t1 - t0;
}

int main()
{
    const long long span = 40ll << 20;  // doubles: 320 MB
    double *src, *dst;
    cudaMalloc(&src, span * 8);
    cudaMalloc(&dst, span * 8);
    cudaMemset(src, 0, span * 8);
    unsigned long long *t, ht;
    cudaMalloc(&t, 8);
    for (int rep = 0; rep < 2; ++rep)
        for (int fixed = 0; fixed < 2; ++fixed) {
            chunkio<<<1, 256>>>(src, dst, span, 14, fixed, t);
            cudaMemcpy(&ht, t, 8, cudaMemcpyDeviceToHost);
            printf("%s chunks: %.2f us per round (%.0f cycles)\n", fixed ? "fixed " : "random",
                   ht / 14.0 / 1965.0, ht / 14.0);
        }
    return 0;
}
