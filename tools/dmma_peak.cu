// dmma_peak.cu -- FP64 tensor (mma.sync m8n8k4 f64 -> DMMA) vs FP64 FMA pipe on
// this B200, alone and concurrently (half the warps each).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int MODE>  // 0: dmma only, 1: dfma only, 2: even warps dmma, odd warps dfma
__global__ void kern(double *out, int iters, double a, double b)
{
    double x[16];
#pragma unroll
    for (int k = 0; k < 16; k++) x[k] = threadIdx.x + k;
    const bool tc = MODE == 0 || (MODE == 2 && ((threadIdx.x >> 5) & 1) == 0);
    if (tc) {
        for (int i = 0; i < iters; i++) {
#pragma unroll
            for (int k = 0; k < 16; k += 2) dmma(x[k], x[k + 1], a, b);
        }
    } else {
        for (int i = 0; i < iters; i++) {
#pragma unroll
            for (int r = 0; r < 4; r++)
#pragma unroll
                for (int k = 0; k < 16; k++) x[k] = fma(x[k], a, b);
        }
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 16; k++) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(const char *name, double *out, int sms)
{
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 2048, blocks = sms * 4, threads = 256;
    kern<MODE><<<blocks, threads>>>(out, 16, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    kern<MODE><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = blocks * threads / 32.0;
    // dmma: 8 mma per iter per warp, 8*8*4*2 = 512 flop each; dfma: 64 fma per iter per thread
    double fl_tc = 0, fl_fma = 0;
    if (MODE == 0) fl_tc = warps * iters * 8 * 512.0;
    if (MODE == 1) fl_fma = warps * 32 * iters * 64 * 2.0;
    if (MODE == 2) { fl_tc = warps / 2 * iters * 8 * 512.0; fl_fma = warps / 2 * 32 * iters * 64 * 2.0; }
    printf("{\"mode\": \"%s\", \"ms\": %.3f, \"dmma_tflops\": %.2f, \"dfma_tflops\": %.2f, \"total_tflops\": %.2f}\n",
           name, ms, fl_tc / ms / 1e9, fl_fma / ms / 1e9, (fl_tc + fl_fma) / ms / 1e9);
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    cudaMalloc(&out, sizeof(double) * sms * 4 * 256);
    for (int rep = 0; rep < 2; rep++) {
        run<0>("dmma", out, sms);
        run<1>("dfma", out, sms);
        run<2>("mixed", out, sms);
    }
    return 0;
}
