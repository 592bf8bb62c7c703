// fp64_peak.cu -- measured FP64 FMA throughput and HBM copy on this B200
// (denominators for the fused-pass roofline).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double *out, int iters, double a, double b)
{
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
           x7 = x0 + 7;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 16; k++) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void copy_kernel(const double4 *__restrict__ in, double4 *__restrict__ out, size_t n)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    cudaMalloc(&out, sizeof(double) * sms * 8 * 256);
    const int iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; rep++) {
        for (int bps = 2; bps <= 8; bps *= 2) {
            dfma_kernel<<<sms * bps, 256>>>(out, 64, 1.0000001, 1e-9);
            cudaEventRecord(e0);
            dfma_kernel<<<sms * bps, 256>>>(out, iters, 1.0000001, 1e-9);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double fmas = (double)sms * bps * 256 * iters * 16 * 8;
            if (rep) printf("{\"fp64_fma_per_s\": %.4e, \"fp64_tflops\": %.3f, \"blocks_per_sm\": %d, \"ms\": %.3f}\n",
                            fmas / (ms * 1e-3), 2 * fmas / (ms * 1e-3) / 1e12, bps, ms);
        }
    }
    size_t bytes = (size_t)4 << 30;
    double4 *a, *b;
    cudaMalloc(&a, bytes);
    cudaMalloc(&b, bytes);
    cudaMemset(a, 0, bytes);
    size_t n = bytes / sizeof(double4);
    float best = 1e9;
    for (int rep = 0; rep < 6; rep++) {
        cudaEventRecord(e0);
        copy_kernel<<<sms * 8, 256>>>(a, b, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    printf("{\"copy_gbs_rw\": %.1f}\n", 2.0 * bytes / (best * 1e-3) / 1e9);
    return 0;
}
