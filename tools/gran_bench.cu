// gran_bench.cu -- HBM efficiency of an in-place tile pass as a function of
// which physical bits the tile spans (how many low bits are contiguous in a
// warp access).  Each CTA loads a tile of 2^12 amplitudes (16 B each) into
// registers (256 threads x 16 amplitudes, v4.f64 = two amplitudes per load),
// and stores it back to the same addresses.  The tile positions are given as
// a list of 12 physical bits; the CTA index is deposited into the others.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gran_bench gran_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

struct TP {
    unsigned long long off[12];  // physical offset (in amplitudes) of tile bit j
    int ts[12];                  // sorted tile positions (for the instance deposit)
};

__device__ __forceinline__ unsigned long long dep(unsigned long long b, const int *ts)
{
#pragma unroll
    for (int j = 0; j < 12; j++) {
        const int t = ts[j];
        b = ((b >> t) << (t + 1)) | (b & ((1ULL << t) - 1));
    }
    return b;
}

// thread layout: register bits 0..3 = tile bits 0,3,4,5 (reg bit 0 = tile bit 0
// must be physical bit 0: one v4 load = 2 amplitudes); lane bits 0..4 = tile
// bits 1,2,6,7,8; warp bits = tile bits 9,10,11
__global__ void __launch_bounds__(256, 2) k_tile(double2 *st, const __grid_constant__ TP P)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned long long base = dep(blockIdx.x, P.ts);
    unsigned long long g = base;
    const int lb[5] = {1, 2, 6, 7, 8};
#pragma unroll
    for (int j = 0; j < 5; j++)
        if ((lane >> j) & 1) g |= P.off[lb[j]];
#pragma unroll
    for (int j = 0; j < 3; j++)
        if ((warp >> j) & 1) g |= P.off[9 + j];
    double x[32];
#pragma unroll
    for (int r = 0; r < 8; r++) {
        unsigned long long o = g;
        if (r & 1) o |= P.off[3];
        if (r & 2) o |= P.off[4];
        if (r & 4) o |= P.off[5];
        asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                     : "=d"(x[4 * r]), "=d"(x[4 * r + 1]), "=d"(x[4 * r + 2]), "=d"(x[4 * r + 3])
                     : "l"(st + o));
    }
#pragma unroll
    for (int i = 0; i < 32; i++) x[i] *= 1.0000000001;
#pragma unroll
    for (int r = 0; r < 8; r++) {
        unsigned long long o = g;
        if (r & 1) o |= P.off[3];
        if (r & 2) o |= P.off[4];
        if (r & 4) o |= P.off[5];
        asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(st + o), "d"(x[4 * r]), "d"(x[4 * r + 1]),
                     "d"(x[4 * r + 2]), "d"(x[4 * r + 3])
                     : "memory");
    }
}

int main(int argc, char **argv)
{
    const int n = argc > 1 ? atoi(argv[1]) : 30;
    const size_t amps = 1ULL << n;
    double2 *st;
    if (cudaMalloc(&st, amps * 16) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMemset(st, 0, amps * 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    // tile bit 0 is always physical bit 0
    struct Case { const char *name; int pos[12]; };
    const Case cases[] = {
        {"low3+contig(3..11)", {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11}},
        {"low3+high(n-9..n-1)", {0, 1, 2, -9, -8, -7, -6, -5, -4, -3, -2, -1}},
        {"low3+mid(10..18)", {0, 1, 2, 10, 11, 12, 13, 14, 15, 16, 17, 18}},
        {"low2+contig(3..12)", {0, 1, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12}},
        {"low2+high(n-10..n-1)", {0, 1, -10, -9, -8, -7, -6, -5, -4, -3, -2, -1}},
        {"low2+mid(10..19)", {0, 1, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19}},
        {"low1+high(n-11..n-1)", {0, -11, -10, -9, -8, -7, -6, -5, -4, -3, -2, -1}},
        {"low1+mid(10..20)", {0, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20}},
    };
    for (const Case &c : cases) {
        TP P;
        int pos[12];
        for (int j = 0; j < 12; j++) pos[j] = c.pos[j] < 0 ? n + c.pos[j] : c.pos[j];
        for (int j = 0; j < 12; j++) P.off[j] = 1ULL << pos[j];
        // sorted positions for the deposit
        for (int j = 0; j < 12; j++) P.ts[j] = pos[j];
        for (int a = 0; a < 12; a++)
            for (int b = a + 1; b < 12; b++)
                if (P.ts[b] < P.ts[a]) { int t = P.ts[a]; P.ts[a] = P.ts[b]; P.ts[b] = t; }
        const unsigned grid = (unsigned)(amps >> 12);
        k_tile<<<grid, 256>>>(st, P);
        float best = 1e9;
        for (int rep = 0; rep < 5; rep++) {
            cudaEventRecord(e0);
            k_tile<<<grid, 256>>>(st, P);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        printf("{\"case\": \"%s\", \"n\": %d, \"ms\": %.3f, \"gbs\": %.1f, \"err\": \"%s\"}\n", c.name, n, best,
               2.0 * amps * 16 / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
