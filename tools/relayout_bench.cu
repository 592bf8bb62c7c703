// relayout_bench.cu -- does a fused pass's shared-memory re-layout overlap
// with the FP64 work of the co-resident CTA?  Synthetic pass body: 256
// threads x 16 amplitudes in registers; per round two 3M 4x4 blocks (13 FP64
// instructions per amplitude each, matrices as kernel-parameter constants)
// and one re-layout (16 STS.128, barrier, 16 LDS.128, barrier).  Variants:
// compute only, re-layout only, both; 2 CTAs/SM (as qsim_pass) or 1; 64- and
// 32-bit shared-memory accesses; a first-wave phase offset (desync); warp-
// specialised (half the warps compute, half move shared memory); warp-local
// re-layouts without CTA barriers; two tiles per 512-thread CTA with and
// without a ping-pong turn on the FP64 pipe (named barriers); shuffle
// exchanges; one wave in phase / with the slot-1 CTAs in anti-phase.
// Finding: compute alone runs at the DFMA peak and a re-
// layout alone at ~0.9 of 128 B/clk/SM, but barrier-synchronised re-layouts
// and FP64 work of the same or the co-resident CTA mostly serialise.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o relayout_bench relayout_bench.cu
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

constexpr int kRounds = 8;  // straight-line: every block has its own matrix (as a real pass)
struct __align__(16) MP {
    double m[2 * kRounds][48];
};

template <int K, int K2>
__device__ __forceinline__ void u4(double2 (&a)[16], const double *M)
{
#pragma unroll
    for (int p = 0; p < 4; p++) {
        int i0 = ((p >> K) << (K + 1)) | (p & ((1 << K) - 1));
        i0 = ((i0 >> K2) << (K2 + 1)) | (i0 & ((1 << K2) - 1));
        const int gi[4] = {i0, i0 | (1 << K), i0 | (1 << K2), i0 | (1 << K) | (1 << K2)};
        double2 x[4];
        double s[4];
#pragma unroll
        for (int c = 0; c < 4; c++) { x[c] = a[gi[c]]; s[c] = x[c].x + x[c].y; }
#pragma unroll
        for (int r = 0; r < 4; r++) {
            double k = M[r * 4] * s[0];
#pragma unroll
            for (int c = 1; c < 4; c++) k = fma(M[r * 4 + c], s[c], k);
            double re = k, im = k;
#pragma unroll
            for (int c = 0; c < 4; c++) {
                re = fma(M[16 + r * 4 + c], x[c].y, re);
                im = fma(M[32 + r * 4 + c], x[c].x, im);
            }
            a[gi[r]] = make_double2(re, im);
        }
    }
}

template <int MODE, int MINB>  // MODE bit 0: compute, bit 1: re-layout
__global__ void __launch_bounds__(256, MINB) k_body(double2 *out, int rounds, unsigned desync, const __grid_constant__ MP P)
{
    extern __shared__ double2 sm[];
    const int t = threadIdx.x;
    double2 a[16];
#pragma unroll
    for (int i = 0; i < 16; i++) a[i] = make_double2(t * 1e-3 + i, blockIdx.x * 1e-6);
    if (MODE == 8 || MODE == 9) {  // re-layout only, 64-bit (8) or 32-bit (9) shared-memory accesses (planes)
#pragma unroll
        for (int r = 0; r < kRounds; r++) {
            if (MODE == 8) {
                double *pl = reinterpret_cast<double *>(sm);
#pragma unroll
                for (int i = 0; i < 16; i++) { pl[i * 256 + t] = a[i].x; pl[4096 + i * 256 + t] = a[i].y; }
                __syncthreads();
#pragma unroll
                for (int i = 0; i < 16; i++) {
                    const int q = i * 256 + ((t + 17 * i + r) & 255);
                    a[i] = make_double2(pl[q], pl[4096 + q]);
                }
            } else {
                unsigned *pl = reinterpret_cast<unsigned *>(sm);
#pragma unroll
                for (int i = 0; i < 16; i++) {
                    pl[i * 256 + t] = __double2loint(a[i].x); pl[4096 + i * 256 + t] = __double2hiint(a[i].x);
                    pl[8192 + i * 256 + t] = __double2loint(a[i].y); pl[12288 + i * 256 + t] = __double2hiint(a[i].y);
                }
                __syncthreads();
#pragma unroll
                for (int i = 0; i < 16; i++) {
                    const int q = i * 256 + ((t + 17 * i + r) & 255);
                    a[i] = make_double2(__hiloint2double(pl[4096 + q], pl[q]), __hiloint2double(pl[12288 + q], pl[8192 + q]));
                }
            }
            __syncthreads();
        }
    } else if (MODE == 10) {  // compute + 64-bit re-layout
#pragma unroll
        for (int r = 0; r < kRounds; r++) {
            u4<0, 1>(a, P.m[2 * r]);
            u4<2, 3>(a, P.m[2 * r + 1]);
            double *pl = reinterpret_cast<double *>(sm);
#pragma unroll
            for (int i = 0; i < 16; i++) { pl[i * 256 + t] = a[i].x; pl[4096 + i * 256 + t] = a[i].y; }
            __syncthreads();
#pragma unroll
            for (int i = 0; i < 16; i++) {
                const int q = i * 256 + ((t + 17 * i + r) & 255);
                a[i] = make_double2(pl[q], pl[4096 + q]);
            }
            __syncthreads();
        }
    } else if (MODE == 11 || MODE == 12) {  // warp-local exchange by shuffles (11), with compute (12)
#pragma unroll
        for (int r = 0; r < kRounds; r++) {
            if (MODE == 12) {
                u4<0, 1>(a, P.m[2 * r]);
                u4<2, 3>(a, P.m[2 * r + 1]);
            }
            // swap register bit 3 with lane bit (r & 3) + 1: half the registers cross
            const int lb = 1 << ((r & 3) + 1);
            const bool hi = t & lb;
#pragma unroll
            for (int i = 0; i < 8; i++) {
                double2 &lo_r = a[i], &hi_r = a[i + 8];
                double2 send = hi ? lo_r : hi_r;
                double2 got;
                got.x = __shfl_xor_sync(0xffffffffu, send.x, lb);
                got.y = __shfl_xor_sync(0xffffffffu, send.y, lb);
                if (hi) lo_r = got; else hi_r = got;
            }
        }
    } else if (MODE == 13 || MODE == 14) {  // one wave; 14: slot-1 CTAs start with the re-layout (anti-phase)
        const bool rot = MODE == 14 && ((blockIdx.x / 148) & 1);
#pragma unroll
        for (int r = 0; r < kRounds; r++) {
            if (!rot) {
                u4<0, 1>(a, P.m[2 * r]);
                u4<2, 3>(a, P.m[2 * r + 1]);
            }
#pragma unroll
            for (int i = 0; i < 16; i++) sm[i * 256 + t] = a[i];
            __syncthreads();
#pragma unroll
            for (int i = 0; i < 16; i++) a[i] = sm[i * 256 + ((t + 17 * i + r) & 255)];
            __syncthreads();
            if (rot) {
                u4<0, 1>(a, P.m[2 * r]);
                u4<2, 3>(a, P.m[2 * r + 1]);
            }
        }
    } else if (MODE == 4) {  // warp-specialised: warps 0-3 compute, 4-7 move shared memory (no CTA barriers)
        if ((t >> 5) < 4) {
#pragma unroll
            for (int r = 0; r < kRounds; r++) {
                u4<0, 1>(a, P.m[2 * r]);
                u4<2, 3>(a, P.m[2 * r + 1]);
            }
        } else {
#pragma unroll
            for (int r = 0; r < kRounds; r++) {
#pragma unroll
                for (int i = 0; i < 16; i++) sm[i * 256 + t] = a[i];
                __syncwarp();
#pragma unroll
                for (int i = 0; i < 16; i++) a[i] = sm[i * 256 + (t ^ ((i + r) & 31))];
                __syncwarp();
            }
        }
    } else if (MODE == 5) {  // every warp: compute + warp-local re-layout (no CTA barriers)
#pragma unroll
        for (int r = 0; r < kRounds; r++) {
            u4<0, 1>(a, P.m[2 * r]);
            u4<2, 3>(a, P.m[2 * r + 1]);
#pragma unroll
            for (int i = 0; i < 16; i++) sm[i * 256 + t] = a[i];
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 16; i++) a[i] = sm[i * 256 + (t ^ ((i + r) & 31))];
            __syncwarp();
        }
    } else
#pragma unroll
    for (int r = 0; r < kRounds; r++) {
        if (MODE & 1) {
            u4<0, 1>(a, P.m[2 * r]);
            u4<2, 3>(a, P.m[2 * r + 1]);
        }
        if (MODE & 2) {
#pragma unroll
            for (int i = 0; i < 16; i++) sm[i * 256 + t] = a[i];
            __syncthreads();
#pragma unroll
            for (int i = 0; i < 16; i++) a[i] = sm[i * 256 + ((t + 17 * i + r) & 255)];
            __syncthreads();
        }
    }
    __nanosleep(blockIdx.x < 148 ? desync : 0u);
    double2 acc = a[0];
#pragma unroll
    for (int i = 1; i < 16; i++) { acc.x += a[i].x; acc.y += a[i].y; }
    out[blockIdx.x * 256 + t] = acc;
}

// Ping-pong: one 512-thread CTA per SM, two groups of 8 warps, each with its
// own tile; the groups take turns on the FP64 pipe (named barriers 3/4), so
// one group's re-layout (named barrier 1/2, its own 64-KB buffer) runs under
// the other's compute.
__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int PP>
__global__ void __launch_bounds__(512, 1) k_pingpong(double2 *out, const __grid_constant__ MP P)
{
    extern __shared__ double2 sm[];
    const int g = threadIdx.x >> 8, t = threadIdx.x & 255;
    double2 *buf = sm + g * 4096;
    double2 a[16];
#pragma unroll
    for (int i = 0; i < 16; i++) a[i] = make_double2(t * 1e-3 + i, blockIdx.x * 1e-6 + g);
    if (PP && g == 1) nbar_arrive(3, 512);
#pragma unroll
    for (int r = 0; r < kRounds; r++) {
        if (PP) nbar_sync(3 + g, 512);
        u4<0, 1>(a, P.m[2 * r]);
        u4<2, 3>(a, P.m[2 * r + 1]);
        if (PP) nbar_arrive(4 - g, 512);
#pragma unroll
        for (int i = 0; i < 16; i++) buf[i * 256 + t] = a[i];
        nbar_sync(1 + g, 256);
#pragma unroll
        for (int i = 0; i < 16; i++) a[i] = buf[i * 256 + ((t + 17 * i + r) & 255)];
        nbar_sync(1 + g, 256);
    }
    if (PP && g == 0) nbar_sync(3, 512);
    double2 acc = a[0];
#pragma unroll
    for (int i = 1; i < 16; i++) { acc.x += a[i].x; acc.y += a[i].y; }
    out[(blockIdx.x * 2 + g) * 256 + t] = acc;
}

// Two tiles per thread, software-pipelined: while one tile's re-layout goes
// through shared memory (its own 64-KB buffer), the same warps compute the
// other tile; one barrier per re-layout (the other tile's barrier is the
// write-after-read fence).  1 CTA/SM, 256 threads x 2 x 16 amplitudes.
__global__ void __launch_bounds__(256, 1) k_two_tiles(double2 *out, const __grid_constant__ MP P)
{
    extern __shared__ double2 sm[];
    const int t = threadIdx.x;
    double2 *bufA = sm, *bufB = sm + 4096;
    double2 a[16], b[16];
#pragma unroll
    for (int i = 0; i < 16; i++) {
        a[i] = make_double2(t * 1e-3 + i, blockIdx.x * 1e-6);
        b[i] = make_double2(t * 2e-3 + i, blockIdx.x * 2e-6);
    }
    u4<0, 1>(a, P.m[0]);
    u4<2, 3>(a, P.m[1]);
#pragma unroll
    for (int r = 0; r < kRounds; r++) {
        // A re-layout under B compute
#pragma unroll
        for (int i = 0; i < 16; i++) bufA[i * 256 + t] = a[i];
        u4<0, 1>(b, P.m[2 * r]);
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 16; i++) a[i] = bufA[i * 256 + ((t + 17 * i + r) & 255)];
        u4<2, 3>(b, P.m[2 * r + 1]);
        // B re-layout under A compute
#pragma unroll
        for (int i = 0; i < 16; i++) bufB[i * 256 + t] = b[i];
        if (r + 1 < kRounds) u4<0, 1>(a, P.m[2 * r + 2]);
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 16; i++) b[i] = bufB[i * 256 + ((t + 17 * i + r) & 255)];
        if (r + 1 < kRounds) u4<2, 3>(a, P.m[2 * r + 3]);
    }
    double2 acc = a[0];
#pragma unroll
    for (int i = 1; i < 16; i++) { acc.x += a[i].x + b[i].x; acc.y += a[i].y + b[i].y; }
    out[(blockIdx.x * 2) * 256 + t] = acc;
}

float run_two(double2 *out, int grid, const MP &P)
{
    const int smem = 128 * 1024;
    cudaFuncSetAttribute(k_two_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_two_tiles<<<grid, 256, smem>>>(out, P);
    float best = 1e9;
    for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(e0);
        k_two_tiles<<<grid, 256, smem>>>(out, P);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    return best;
}

template <int PP>
float run_pp(double2 *out, int grid, const MP &P)
{
    const int smem = 128 * 1024;
    cudaFuncSetAttribute(k_pingpong<PP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_pingpong<PP><<<grid, 512, smem>>>(out, P);
    float best = 1e9;
    for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(e0);
        k_pingpong<PP><<<grid, 512, smem>>>(out, P);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    return best;
}

template <int MODE, int MINB>
float run(double2 *out, int grid, int rounds, unsigned desync, size_t smem, const MP &P)
{
    cudaFuncSetAttribute(k_body<MODE, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_body<MODE, MINB><<<grid, 256, smem>>>(out, rounds, desync, P);
    float best = 1e9;
    for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(e0);
        k_body<MODE, MINB><<<grid, 256, smem>>>(out, rounds, desync, P);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    return best;
}

int main()
{
    MP P;
    for (int j = 0; j < 2 * kRounds; j++)
        for (int i = 0; i < 48; i++) P.m[j][i] = 0.01 * (i + 1) * (j & 1 ? -1 : 1);
    const int sms = 148, waves = 14, rounds = kRounds;
    double2 *out;
    cudaMalloc(&out, sizeof(double2) * 256 * sms * 2 * waves);
    const int grid2 = sms * 2 * waves;
    // FP64 instructions: 2 blocks x 13 per amplitude x 16 amplitudes per thread per round
    const double fp64 = (double)grid2 * 256 * rounds * 2 * 13 * 16;
    // compute variants: executed FP64 TFLOP/s; pure re-layout variants: shared-
    // memory TB/s (64 KB written + 64 KB read per CTA per round)
    auto rep = [&](const char *name, float ms) {
        if (!strncmp(name, "shuffle", 7))
            printf("{\"variant\": \"%s\", \"ms\": %.4f, \"err\": \"%s\"}\n", name, ms,
                   cudaGetErrorString(cudaGetLastError()));
        else if (!strncmp(name, "relayout", 8))
            printf("{\"variant\": \"%s\", \"ms\": %.4f, \"smem_tbs\": %.2f, \"err\": \"%s\"}\n", name, ms,
                   (double)grid2 * rounds * 131072 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
        else
            printf("{\"variant\": \"%s\", \"ms\": %.4f, \"fp64_tflops\": %.2f, \"err\": \"%s\"}\n", name, ms,
                   2 * fp64 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    };
    const size_t sm64 = 64 * 1024, sm120 = 120 * 1024;
    rep("compute, 2 CTA/SM", run<1, 2>(out, grid2, rounds, 0, sm64, P));
    rep("relayout, 2 CTA/SM", run<2, 2>(out, grid2, rounds, 0, sm64, P));
    rep("both, 2 CTA/SM", run<3, 2>(out, grid2, rounds, 0, sm64, P));
    for (unsigned d : {500u, 1500u, 4000u}) {
        char nm[64];
        snprintf(nm, sizeof nm, "both, 2 CTA/SM, desync %u ns", d);
        rep(nm, run<3, 2>(out, grid2, rounds, d, sm64, P));
    }
    rep("relayout 64-bit, 2 CTA/SM", run<8, 2>(out, grid2, rounds, 0, sm64, P));
    rep("relayout 32-bit, 2 CTA/SM", run<9, 2>(out, grid2, rounds, 0, sm64, P));
    rep("relayout 64-bit, 1 CTA/SM", run<8, 1>(out, grid2, rounds, 0, sm120, P));
    rep("both 64-bit, 2 CTA/SM", run<10, 2>(out, grid2, rounds, 0, sm64, P));
    {
        // one wave (2 CTAs per SM), 16x the work per CTA via repeated launches is not the same; use grid = 296
        auto rep1 = [&](const char *name, float ms) {  // one wave: includes the launch and tail (~4 us)
            printf("{\"variant\": \"%s\", \"ms\": %.4f}\n", name, ms);
        };
        rep1("one wave: compute only", run<1, 2>(out, 296, rounds, 0, sm64, P));
        rep1("one wave: relayout only", run<2, 2>(out, 296, rounds, 0, sm64, P));
        rep1("one wave: both, in phase", run<13, 2>(out, 296, rounds, 0, sm64, P));
        rep1("one wave: both, slot 1 anti-phase", run<14, 2>(out, 296, rounds, 0, sm64, P));
    }
    rep("shuffle exchange (half the registers), 2 CTA/SM", run<11, 2>(out, grid2, rounds, 0, sm64, P));
    rep("compute + shuffle exchange, 2 CTA/SM", run<12, 2>(out, grid2, rounds, 0, sm64, P));
    rep("warp-specialised half compute / half smem, 2 CTA/SM", run<4, 2>(out, grid2, rounds, 0, sm64, P));
    rep("compute + warp-local relayout, 2 CTA/SM", run<5, 2>(out, grid2, rounds, 0, sm64, P));
    rep("two tiles per thread, pipelined (re-layout of one under the compute of the other), 1 CTA/SM",
        run_two(out, grid2 / 2, P));
    rep("two groups in one 512-thread CTA, no ping-pong", run_pp<0>(out, grid2 / 2, P));
    rep("two groups in one 512-thread CTA, ping-pong", run_pp<1>(out, grid2 / 2, P));
    rep("compute, 1 CTA/SM (128-reg cap)", run<1, 2>(out, grid2, rounds, 0, sm120, P));
    rep("both, 1 CTA/SM (128-reg cap)", run<3, 2>(out, grid2, rounds, 0, sm120, P));
    rep("compute, 1 CTA/SM", run<1, 1>(out, grid2, rounds, 0, sm120, P));
    rep("relayout, 1 CTA/SM", run<2, 1>(out, grid2, rounds, 0, sm120, P));
    rep("both, 1 CTA/SM", run<3, 1>(out, grid2, rounds, 0, sm120, P));
    return 0;
}
