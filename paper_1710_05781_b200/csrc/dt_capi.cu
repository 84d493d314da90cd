// Library-wide C ABI plumbing: version, error text, device check.
#include <stdio.h>
#include <string.h>

#include "dt_common.cuh"

static thread_local char g_err[256] = "";

int dt_set_error(int code, const char *msg)
{
    snprintf(g_err, sizeof(g_err), "%s", msg ? msg : "");
    return code;
}

extern "C" const char *dt_version(void) { return "disctree_b200 0.1.0 (sm_100a)"; }

extern "C" const char *dt_last_error(void) { return g_err; }

extern "C" int dt_device_check(void)
{
    int dev = 0;
    DT_CUDA_TRY(cudaGetDevice(&dev));
    int major = 0, minor = 0;
    DT_CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    DT_CUDA_TRY(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
    if (major != 10 || minor != 0) {
        char buf[96];
        snprintf(buf, sizeof(buf), "device %d is sm_%d%d; this build targets sm_100a", dev, major,
                 minor);
        return dt_set_error(DT_ERR_DEVICE, buf);
    }
    return DT_OK;
}

namespace {
__global__ void __launch_bounds__(256) fp64_probe_kernel(double *out, int64_t iters)
{
    double a[8];
    const double m = 1.0 - 1e-9 * (threadIdx.x & 7), c = 1e-7;
#pragma unroll
    for (int i = 0; i < 8; ++i)
        a[i] = 1.0 + 1e-3 * i + 1e-6 * threadIdx.x;
    for (int64_t k = 0; k < iters; ++k) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            a[i] = __fma_rn(a[i], m, c);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
        s += a[i];
    out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = s;
}
}  // namespace

extern "C" int dt_fp64_probe(double *out, int64_t iters, int blocks, void *stream)
{
    DT_CHECK_ARG(out && iters > 0 && blocks > 0, "bad argument");
    fp64_probe_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(out, iters);
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}
