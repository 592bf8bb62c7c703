// kernels.cu -- hand-written sm_100a kernels of the state-vector engine.
//
// All kernels update the complex128 shard in place ("all these
// operations can be done in place").  The hot kernel is k_pass: one HBM
// read + write of the shard (32 B/amplitude) applies a whole planned list of
// gates (Eqs. NUM2-NUM8) to 4096-amplitude tiles held in
// registers, with warp shuffles and swizzled shared-memory transposes.
// 256-bit global accesses (ld/st.global.v4.f64 -> LDG/STG.E.ENL2.256 on
// sm_100a) move two amplitudes per instruction.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "engine.h"
#include "kernels.h"

namespace qsb {

#define FULL 0xffffffffu

__device__ __forceinline__ void ld256(const double2 *p, double2 &a, double2 &b)
{
    asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y)
                 : "l"(p));
}
__device__ __forceinline__ void st256(double2 *p, const double2 &a, const double2 &b)
{
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y)
                 : "memory");
}

__device__ __forceinline__ double2 cmul(double2 f, double2 a)
{
    return make_double2(fma(f.x, a.x, -f.y * a.y), fma(f.x, a.y, f.y * a.x));
}

// (c0 * x + c1 * y), complex
__device__ __forceinline__ double2 cmac2(double2 c0, double2 x, double2 c1, double2 y)
{
    double re = fma(c0.x, x.x, fma(-c0.y, x.y, fma(c1.x, y.x, -c1.y * y.y)));
    double im = fma(c0.x, x.y, fma(c0.y, x.x, fma(c1.x, y.y, c1.y * y.x)));
    return make_double2(re, im);
}

__device__ __forceinline__ uint64_t insert_zero(uint64_t v, int p)
{
    return ((v >> p) << (p + 1)) | (v & ((1ULL << p) - 1));
}

// ---------------------------------------------------------------- k_pass
// In-place pair updates: every output is finished by one FMA that consumes
// the old value held in the same register, after all partial sums that still
// need the old values are formed.  This keeps the amplitudes in fixed
// registers across the op loop (no compiler copies).
__device__ __forceinline__ void u2_inplace(double2 &x, double2 &y, const double2 u00, const double2 u01,
                                           const double2 u10, const double2 u11)
{
    const double p1 = fma(-u00.y, x.y, fma(u01.x, y.x, -u01.y * y.y));  // x'.re - u00r x.re
    const double p2 = fma(u00.y, x.x, fma(u01.x, y.y, u01.y * y.x));    // x'.im - u00r x.im
    const double p3 = fma(u10.x, x.x, fma(-u10.y, x.y, -u11.y * y.y));  // y'.re - u11r y.re
    const double p4 = fma(u10.x, x.y, fma(u10.y, x.x, u11.y * y.x));    // y'.im - u11r y.im
    x.x = fma(u00.x, x.x, p1);
    x.y = fma(u00.x, x.y, p2);
    y.x = fma(u11.x, y.x, p3);
    y.y = fma(u11.x, y.y, p4);
}

__device__ __forceinline__ void u2r_inplace(double2 &x, double2 &y, double u00, double u01, double u10, double u11)
{
    const double p1 = u01 * y.x, p2 = u01 * y.y, p3 = u10 * x.x, p4 = u10 * x.y;
    x.x = fma(u00, x.x, p1);
    x.y = fma(u00, x.y, p2);
    y.x = fma(u11, y.x, p3);
    y.y = fma(u11, y.y, p4);
}

// register swap that keeps both values in their own registers
__device__ __forceinline__ void swap_inplace(double &x, double &y)
{
    asm("{\n\t.reg .f64 t;\n\tmov.f64 t, %0;\n\tmov.f64 %0, %1;\n\tmov.f64 %1, t;\n\t}" : "+d"(x), "+d"(y));
}

template <int K, int CODE, bool PRED>
__device__ __forceinline__ void reg_apply(double2 (&a)[kAmpsPerThread], const KOp &op, uint32_t mreg, uint32_t vreg)
{
    double2 u00, u01, u10, u11;
    if (CODE != OPC_XS) {
        u00 = make_double2(op.m[0], op.m[1]);
        u01 = make_double2(op.m[2], op.m[3]);
        u10 = make_double2(op.m[4], op.m[5]);
        u11 = make_double2(op.m[6], op.m[7]);
    }
#pragma unroll
    for (int p = 0; p < kAmpsPerThread / 2; p++) {
        const int i0 = ((p >> K) << (K + 1)) | (p & ((1 << K) - 1));
        const int i1 = i0 | (1 << K);
        if (PRED && (i0 & mreg) != vreg) continue;
        if (CODE == OPC_XS) {
            swap_inplace(a[i0].x, a[i1].x);
            swap_inplace(a[i0].y, a[i1].y);
        } else if (CODE == OPC_U2R) {
            u2r_inplace(a[i0], a[i1], u00.x, u01.x, u10.x, u11.x);
        } else {
            u2_inplace(a[i0], a[i1], u00, u01, u10, u11);
        }
    }
}

template <int CODE, bool PRED>
__device__ __forceinline__ void reg_dispatch(double2 (&a)[kAmpsPerThread], const KOp &op, int k, uint32_t mreg,
                                             uint32_t vreg)
{
    switch (k) {
    case 0: reg_apply<0, CODE, PRED>(a, op, mreg, vreg); break;
    case 1: reg_apply<1, CODE, PRED>(a, op, mreg, vreg); break;
    case 2: reg_apply<2, CODE, PRED>(a, op, mreg, vreg); break;
    case 3: reg_apply<3, CODE, PRED>(a, op, mreg, vreg); break;
    default:
        if constexpr (kRegBits > 4) reg_apply<kRegBits - 1, CODE, PRED>(a, op, mreg, vreg);
        break;
    }
}

template <bool PRED>
__device__ __forceinline__ void reg_op(double2 (&a)[kAmpsPerThread], const KOp &op, int code, uint32_t mreg,
                                       uint32_t vreg)
{
    const int k = op.k;
    if (code == OPC_XS) reg_dispatch<OPC_XS, PRED>(a, op, k, mreg, vreg);
    else if (code == OPC_U2R) reg_dispatch<OPC_U2R, PRED>(a, op, k, mreg, vreg);
    else reg_dispatch<OPC_U2, PRED>(a, op, k, mreg, vreg);
}

// Fused 4x4 block (OPC_U4) on register bits K < K2; rows[r].m = row r of the
// complex matrix, 4x4 index j = bit_K + 2 bit_K2.  Each output is one
// 8-long FMA chain for re and one for im, in the fixed column order the JIT
// tier generates too (bitwise-identical tiers).
template <int K, int K2>
__device__ __forceinline__ void u4_apply(double2 (&a)[kAmpsPerThread], const KOp *rows)
{
#pragma unroll
    for (int p = 0; p < kAmpsPerThread / 4; p++) {
        const int i0 = (int)insert_zero(insert_zero((uint64_t)p, K), K2);
        const int idx[4] = {i0, i0 | (1 << K), i0 | (1 << K2), i0 | (1 << K) | (1 << K2)};
        const double2 x[4] = {a[idx[0]], a[idx[1]], a[idx[2]], a[idx[3]]};
#pragma unroll
        for (int r = 0; r < 4; r++) {
            const double *m = rows[r].m;
            double re = m[0] * x[0].x, im = m[0] * x[0].y;
            re = fma(-m[1], x[0].y, re);
            im = fma(m[1], x[0].x, im);
#pragma unroll
            for (int c = 1; c < 4; c++) {
                re = fma(m[2 * c], x[c].x, re);
                re = fma(-m[2 * c + 1], x[c].y, re);
                im = fma(m[2 * c], x[c].y, im);
                im = fma(m[2 * c + 1], x[c].x, im);
            }
            a[idx[r]] = make_double2(re, im);
        }
    }
}

__device__ __forceinline__ void u4_op(double2 (&a)[kAmpsPerThread], const KOp *rows)
{
    switch (rows[0].k * 8 + (int)rows[0].cfg) {
    case 1: u4_apply<0, 1>(a, rows); break;
    case 2: u4_apply<0, 2>(a, rows); break;
    case 3: u4_apply<0, 3>(a, rows); break;
    case 10: u4_apply<1, 2>(a, rows); break;
    case 11: u4_apply<1, 3>(a, rows); break;
    case 19: u4_apply<2, 3>(a, rows); break;
    default:
        if constexpr (kRegBits > 4) {
            switch (rows[0].k * 8 + (int)rows[0].cfg) {
            case 4: u4_apply<0, 4>(a, rows); break;
            case 12: u4_apply<1, 4>(a, rows); break;
            case 20: u4_apply<2, 4>(a, rows); break;
            default: u4_apply<3, 4>(a, rows); break;
            }
        }
        break;
    }
}

// Shared-memory layout of a tile: 16-B unit of tile-local index s sits at
// swz(s) = s ^ fold3(s >> 3).  Tile-local bit t lands in 16-B bank group
// residue t mod 3, so a warp access whose 5 lane bits cover all three
// residues touches every bank group exactly 4 times (4 wavefronts per
// 512 B: conflict-free).  swz is GF(2)-linear: swz(a ^ b) = swz(a) ^ swz(b).
__device__ __forceinline__ int swz(int s) { return s ^ (((s >> 3) ^ (s >> 6) ^ (s >> 9) ^ (s >> 12)) & 7); }

// thread's lane/warp part of the smem index and the 4 register-bit parts
__device__ __forceinline__ void smem_coords(uint64_t c, int lane, int warp, int &zt, int (&zr)[kRegBits])
{
    int st = 0;
#pragma unroll
    for (int j = 0; j < 5; j++) st |= ((lane >> j) & 1) << cfg_nib(c, kLaneNib + j);
#pragma unroll
    for (int j = 0; j < kWarpBits; j++) st |= ((warp >> j) & 1) << cfg_nib(c, kWarpNib + j);
    zt = swz(st);
#pragma unroll
    for (int j = 0; j < kRegBits; j++) zr[j] = swz(1 << cfg_nib(c, j));
}

template <int I>
__device__ __forceinline__ int zsel(int zt, const int (&zr)[kRegBits])
{
    int z = zt;
#pragma unroll
    for (int b = 0; b < kRegBits; b++)
        if ((I >> b) & 1) z ^= zr[b];
    return z;
}

template <int I>
__device__ __forceinline__ void sts_all(double2 *sm, const double2 (&a)[kAmpsPerThread], int zt,
                                        const int (&zr)[kRegBits])
{
    sm[zsel<I>(zt, zr)] = a[I];
    if constexpr (I + 1 < kAmpsPerThread) sts_all<I + 1>(sm, a, zt, zr);
}
template <int I>
__device__ __forceinline__ void lds_all(const double2 *sm, double2 (&a)[kAmpsPerThread], int zt,
                                        const int (&zr)[kRegBits])
{
    a[I] = sm[zsel<I>(zt, zr)];
    if constexpr (I + 1 < kAmpsPerThread) lds_all<I + 1>(sm, a, zt, zr);
}

// global offset of the thread's lane/warp part and register-bit parts (load/store configs)
// tp: physical position of each tile-local bit (d.tp to load, d.tp_out to store)
__device__ __forceinline__ void global_coords(const int32_t *tp, uint64_t c, int lane, int warp, uint64_t &gt,
                                              uint64_t (&g)[kRegBits])
{
    gt = (uint64_t)((lane & 3) << 1);  // lanes 0, 1 hold the tile bits at phys 1, 2
#pragma unroll
    for (int j = 2; j < 5; j++) gt |= (uint64_t)((lane >> j) & 1) << tp[cfg_nib(c, kLaneNib + j)];
#pragma unroll
    for (int j = 0; j < kWarpBits; j++) gt |= (uint64_t)((warp >> j) & 1) << tp[cfg_nib(c, kWarpNib + j)];
#pragma unroll
    for (int b = 1; b < kRegBits; b++) g[b] = 1ULL << tp[cfg_nib(c, b)];  // register bit 0: within a 256-bit access
}

// global offset of register pair j (register bits 1.. of the pair index)
__device__ __forceinline__ uint64_t pair_off(int j, const uint64_t (&g)[kRegBits])
{
    uint64_t ro = 0;
#pragma unroll
    for (int b = 1; b < kRegBits; b++)
        if ((j >> (b - 1)) & 1) ro |= g[b];
    return ro;
}

template <int CAP>
struct PassParams {
    PassDesc d;
    KOp ops[CAP];
};

// gops != nullptr: the op program is in global memory (programs longer than
// the parameter block holds); otherwise P.ops
template <int CAP, int MINB>
__global__ void __launch_bounds__(kPassThreads, MINB)
    k_pass(const __grid_constant__ PassParams<CAP> P, double2 *__restrict__ st, const KOp *__restrict__ gops)
{
    const PassDesc &d = P.d;
    extern __shared__ double2 sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    uint64_t base = blockIdx.x;
#pragma unroll
    for (int j = 0; j < kTileBits; j++) base = insert_zero(base, d.tile_sorted[j]);
    const uint64_t gcta = d.rank_bits | base;

    uint64_t cfg = d.cfg0;
    double2 a[kAmpsPerThread];
    {
        uint64_t gt, g[kRegBits];
        global_coords(d.tp, cfg, lane, warp, gt, g);
        if (d.fresh) {  // first pass after qsim_init_basis: the basis state, no read
            const uint64_t g0 = d.rank_bits | base | gt;
#pragma unroll
            for (int j = 0; j < kAmpsPerThread / 2; j++) {
                const uint64_t gi = g0 | pair_off(j, g);
                a[2 * j] = make_double2(gi == d.init_phys ? 1.0 : 0.0, 0.0);
                a[2 * j + 1] = make_double2((gi | 1ULL) == d.init_phys ? 1.0 : 0.0, 0.0);
            }
        } else {
            const double2 *p = st + base + gt;
#pragma unroll
            for (int j = 0; j < kAmpsPerThread / 2; j++) ld256(p + pair_off(j, g), a[2 * j], a[2 * j + 1]);
        }
    }

    for (int o = 0; o < d.n_ops; o++) {
        const KOp &op = gops ? gops[o] : P.ops[o];
        const int code = op.code;
        if (code == OPC_TRANS) {
            int zt, zr[kRegBits];
            smem_coords(cfg, lane, warp, zt, zr);
            sts_all<0>(sm, a, zt, zr);
            __syncthreads();
            cfg = op.cfg;
            smem_coords(cfg, lane, warp, zt, zr);
            lds_all<0>(sm, a, zt, zr);
            __syncthreads();
            continue;
        }
        if (code == OPC_PHASE_FLUSH || code == OPC_DATA) continue;
        if (code == OPC_U4) {
            u4_op(a, gops ? gops + o : &P.ops[o]);
            o += 3;
            continue;
        }
        const bool tp = ((lane & op.mlane) == op.vlane) && ((warp & op.mwarp) == op.vwarp) &&
                        ((gcta & op.mout) == op.vout);
        if (!tp) continue;
        const uint32_t mreg = op.mreg, vreg = op.vreg;
        if (code == OPC_PHASE || code == OPC_PHASE_ACC) {
            const double fr = op.m[0], fi = op.m[1];
#pragma unroll
            for (int i = 0; i < kAmpsPerThread; i++) {
                if ((i & mreg) != vreg) continue;
                const double p1 = -fi * a[i].y, p2 = fi * a[i].x;
                a[i].x = fma(fr, a[i].x, p1);
                a[i].y = fma(fr, a[i].y, p2);
            }
            continue;
        }
        if (mreg == 0) reg_op<false>(a, op, code, 0, 0);
        else reg_op<true>(a, op, code, mreg, vreg);
    }

    {
        uint64_t gt, g[kRegBits];
        global_coords(d.tp_out, cfg, lane, warp, gt, g);
        double2 *p = st + base + gt;
#pragma unroll
        for (int j = 0; j < kAmpsPerThread / 2; j++) st256(p + pair_off(j, g), a[2 * j], a[2 * j + 1]);
    }
}

template <int CAP, int MINB>
static void launch_pass_cap(const PassDesc &d, const KOp *ops, double2 *st, cudaStream_t s, const KOp *gops)
{
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_pass<CAP, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kTileAmps * (int)sizeof(double2));
        attr = true;
    }
    PassParams<CAP> P;
    P.d = d;
    if (!gops)
        for (int i = 0; i < d.n_ops; i++) P.ops[i] = ops[i];
    const int smem = d.use_smem ? kTileAmps * (int)sizeof(double2) : 0;
    k_pass<CAP, MINB><<<(unsigned)d.n_inst, kPassThreads, smem, s>>>(P, st, gops);
}

template <int MINB>
static void launch_pass_minb(const PassDesc &d, const KOp *ops, double2 *st, cudaStream_t s, const KOp *gops)
{
    if (gops) launch_pass_cap<1, MINB>(d, ops, st, s, gops);
    else if (d.n_ops <= 32) launch_pass_cap<32, MINB>(d, ops, st, s, nullptr);
    else if (d.n_ops <= 96) launch_pass_cap<96, MINB>(d, ops, st, s, nullptr);
    else launch_pass_cap<kMaxPassOps, MINB>(d, ops, st, s, nullptr);
}

void launch_pass(const PassDesc &d, const KOp *ops, double2 *st, int variant, cudaStream_t s, const KOp *gops)
{
    constexpr int kMinB = kPassMinBlocks;
    if (variant == 1) launch_pass_minb<kMinB / 2>(d, ops, st, s, gops);
    else launch_pass_minb<kMinB>(d, ops, st, s, gops);
}

int pass_regs_per_thread()
{
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, (k_pass<kMaxPassOps, kPassMinBlocks>)) != cudaSuccess) return -1;
    return fa.numRegs;
}

// -------------------------------------------------------- generic kernels
struct U8 {
    double m[8];
};

__global__ void k_gate_generic(double2 *__restrict__ st, uint64_t half, int t, uint64_t rank_bits, uint64_t cm,
                               uint64_t cv, int code, U8 u)
{
    const double2 u00 = make_double2(u.m[0], u.m[1]), u01 = make_double2(u.m[2], u.m[3]);
    const double2 u10 = make_double2(u.m[4], u.m[5]), u11 = make_double2(u.m[6], u.m[7]);
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < half;
         p += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i0 = insert_zero(p, t), i1 = i0 | (1ULL << t);
        if (((rank_bits | i0) & cm) != cv) continue;
        const double2 x = st[i0], y = st[i1];
        if (code == OPC_XS) {
            st[i0] = y;
            st[i1] = x;
        } else {
            st[i0] = cmac2(u00, x, u01, y);
            st[i1] = cmac2(u10, x, u11, y);
        }
    }
}

__global__ void k_phase_generic(double2 *__restrict__ st, uint64_t D, uint64_t rank_bits, uint64_t cm, uint64_t cv,
                                double fr, double fi)
{
    const double2 f = make_double2(fr, fi);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < D; i += (uint64_t)gridDim.x * blockDim.x)
        if (((rank_bits | i) & cm) == cv) st[i] = cmul(f, st[i]);
}

static unsigned grid_for(uint64_t work, int threads)
{
    uint64_t g = (work + threads - 1) / threads;
    const uint64_t cap = 148ULL * 16;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (unsigned)g;
}

void launch_gate_generic(double2 *st, int M, uint64_t rank_bits, int t, uint64_t cm, uint64_t cv, int code,
                         const double *m, cudaStream_t s)
{
    U8 u;
    for (int k = 0; k < 8; k++) u.m[k] = m[k];
    const uint64_t half = 1ULL << (M - 1);
    k_gate_generic<<<grid_for(half, 256), 256, 0, s>>>(st, half, t, rank_bits, cm, cv, code, u);
}

void launch_phase_generic(double2 *st, int M, uint64_t rank_bits, uint64_t cm, uint64_t cv, double fr, double fi,
                          cudaStream_t s)
{
    const uint64_t D = 1ULL << M;
    k_phase_generic<<<grid_for(D, 256), 256, 0, s>>>(st, D, rank_bits, cm, cv, fr, fi);
}

// ------------------------------------------------------------------ perm
__device__ __forceinline__ uint64_t dep_tile(uint32_t e, const int32_t *pos, int nb)
{
    uint64_t r = 0;
    for (int b = 0; b < nb; b++) r |= (uint64_t)((e >> b) & 1) << pos[b];
    return r;
}

__global__ void __launch_bounds__(256) k_perm(const __grid_constant__ PermDesc d, double2 *__restrict__ st,
                                              const uint32_t *__restrict__ perm_tab)
{
    extern __shared__ double2 sm[];
    uint64_t base = blockIdx.x;
    for (int j = 0; j < d.tile_bits; j++) base = insert_zero(base, d.tile_sorted[j]);
    if (((d.rank_bits | base) & d.m_ctrl_out) != d.v_ctrl_out) return;
    const uint32_t E = 1u << d.tile_bits, T = (1u << d.t) - 1;
    const uint32_t *perm = perm_tab + d.perm_offset;
    if (d.contiguous) {
        // tile = the low tile_bits physical bits in order (the usual case: the
        // initial layout puts permutation targets lowest): offset == index
        const double2 *src = st + base;
        for (uint32_t e = 2 * threadIdx.x; e < E; e += 2 * blockDim.x) {
            double2 x0, x1;
            ld256(src + e, x0, x1);
            sm[e] = x0;
            sm[e + 1] = x1;
        }
        __syncthreads();
        // gather with the inverse permutation: coalesced 256-bit stores; pairs
        // (e, e+1) differ in target bit 0 only, so they share the control test
        double2 *dst = st + base;
        for (uint32_t e = 2 * threadIdx.x; e < E; e += 2 * blockDim.x) {
            if ((e & d.m_ctrl_tile) != d.v_ctrl_tile) continue;
            const double2 y0 = sm[(e & ~T) | __ldg(perm + (e & T))];
            const double2 y1 = sm[((e + 1) & ~T) | __ldg(perm + ((e + 1) & T))];
            st256(dst + e, y0, y1);
        }
        return;
    }
    for (uint32_t e = threadIdx.x; e < E; e += blockDim.x) sm[e] = st[base + dep_tile(e, d.tile_pos, d.tile_bits)];
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < E; e += blockDim.x) {
        if ((e & d.m_ctrl_tile) != d.v_ctrl_tile) continue;
        st[base + dep_tile(e, d.tile_pos, d.tile_bits)] = sm[(e & ~T) | perm[e & T]];
    }
}

// Run of permutations of one register (PermRunDesc).  Persistent CTAs: the
// R inverse tables (as uint16) are staged in shared memory once, then each tile
// (targets + extra bits, as in k_perm) is staged and every element gathers
// through the tables of the perms whose controls it satisfies, latest first:
// out[x, w] = in[x, P_j1^-1(... P_jk^-1(w))].  Controls are never targets, so
// the active set depends only on the non-target bits, shared by an element
// and its source.  Elements no perm touches are neither read nor written.
// Tiles are double-buffered: the cp.async copies of a CTA's next tile are in
// flight while it gathers the current one (the gather is a short chain of
// shared-memory lookups; the HBM latency of the staging was the bound).
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// 1D bulk copies (the TMA engine, no tensor map) completing on an mbarrier
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity)
{
    unsigned done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done)
                     : "r"(smem_u32(bar)), "r"(parity)
                     : "memory");
}

constexpr int kPermRunThreads = 512;
// Composition (PermRunDesc pre_mask / slow_mask): the gather chain of an
// element is P_jk^-1 o ... with j descending.  Its head, the perms without
// in-tile controls, has the same active subset for every element of a tile
// (CTA-uniform), so per tile it is composed once into a 2^t-entry table
// (2^t lookups per head perm instead of 2^tile_bits); the slowest part of
// that head, whose controls only change every few tiles of the CTA's
// contiguous instance range, is itself composed once per change.  An element
// then does one lookup for the head plus its in-tile-controlled perms.
__global__ void __launch_bounds__(kPermRunThreads) k_perm_run(const __grid_constant__ PermRunDesc d, double2 *__restrict__ st,
                                                  const uint32_t *__restrict__ tabs)
{
    extern __shared__ __align__(16) unsigned char smraw[];
    const uint32_t E = 1u << d.tile_bits, TT = 1u << d.t, T = TT - 1, NX = E >> d.t;
    double2 *bufs = reinterpret_cast<double2 *>(smraw);                                        // 2 x E
    uint32_t *xmask = reinterpret_cast<uint32_t *>(smraw + 2 * (size_t)E * sizeof(double2));  // NX entries
    uint16_t *tab = reinterpret_cast<uint16_t *>(xmask + NX);                                // R * TT entries
    uint16_t *slow_tab = tab + (size_t)d.R * TT;                                             // TT
    uint16_t *comp = slow_tab + TT;                                                           // 2 x TT
    for (uint32_t i = threadIdx.x; i < (uint32_t)d.R * TT; i += blockDim.x) tab[i] = (uint16_t)__ldg(tabs + d.tab_offset + i);
    // in-tile control predicates of every extra-bit pattern x (tile-local e = x << t | w)
    for (uint32_t x = threadIdx.x; x < NX; x += blockDim.x) {
        uint32_t m = 0;
        for (int j = 0; j < d.R; j++)
            if (((x << d.t) & d.m_tile[j]) == d.v_tile[j]) m |= 1u << j;
        xmask[x] = m;
    }
    __syncthreads();
    // this CTA's contiguous instance range; the next tile (from `inst` on)
    // that some perm touches; CTA-uniform
    const bool compose = d.pre_mask != 0;
    const uint64_t per = compose ? (d.n_inst + gridDim.x - 1) / gridDim.x : d.n_inst;
    const uint64_t i_first = compose ? (uint64_t)blockIdx.x * per : blockIdx.x, step = compose ? 1 : gridDim.x;
    const uint64_t i_end = compose ? min(d.n_inst, i_first + per) : d.n_inst;
    auto next_tile = [&](uint64_t inst, uint64_t &base, uint32_t &A) {
        for (; inst < i_end; inst += step) {
            base = inst;
            for (int j = 0; j < d.tile_bits; j++) base = insert_zero(base, d.tile_sorted[j]);
            A = 0;  // perms whose out-of-tile controls this tile satisfies
            for (int j = 0; j < d.R; j++)
                if (((d.rank_bits | base) & d.m_out[j]) == d.v_out[j]) A |= 1u << j;
            if (A) break;
        }
        return inst < i_end ? inst : d.n_inst;
    };
    // Contiguous tiles (the register on the lowest bits, Shor's case): one
    // thread stages the whole tile with a single bulk copy completing on the
    // slot's mbarrier; no per-thread copies, and the wait is the data's own
    // arrival (no CTA barrier).  Otherwise per-element cp.async of the
    // elements some perm touches.
    __shared__ __align__(8) uint64_t s_bar[2];
    const bool bulk = d.bulk != 0 && d.contiguous;
    if (bulk && threadIdx.x == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    unsigned bar_phase = 0;  // bit b: parity to wait for on slot b
    auto stage = [&](double2 *buf, uint64_t base, uint32_t A, int slot) {
        if (bulk) {
            if (threadIdx.x == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic reads of buf
                mbar_expect_tx(&s_bar[slot], E * (unsigned)sizeof(double2));
                bulk_g2s(buf, st + base, E * (unsigned)sizeof(double2), &s_bar[slot]);
            }
            return;
        }
        for (uint32_t e = threadIdx.x; e < E; e += blockDim.x)
            if (A & xmask[e >> d.t])
                cp_async16(buf + e, st + base + (d.contiguous ? e : dep_tile(e, d.tile_pos, d.tile_bits)));
    };
    // chain of the perms in `m` (descending j) applied to v
    auto chain = [&](uint32_t m, uint32_t v) {
        while (m) {
            const int j = 31 - __clz(m);
            v = tab[j * TT + v];
            m &= ~(1u << j);
        }
        return v;
    };
    uint32_t slow_cur = 0xffffffffu;  // subset the slow table holds (uniform)
    auto build = [&](uint32_t A, uint16_t *dst) {  // caller: the slow table may be rebuilt (no reader)
        const uint32_t S = A & d.slow_mask, F = A & d.pre_mask & ~d.slow_mask;
        if (S != slow_cur) {
            for (uint32_t w = threadIdx.x; w < TT; w += blockDim.x) slow_tab[w] = (uint16_t)chain(S, w);
            slow_cur = S;
            __syncthreads();
        }
        for (uint32_t w = threadIdx.x; w < TT; w += blockDim.x) dst[w] = (uint16_t)chain(F, slow_tab[w]);
    };
    // tile k+1's (instance, base, active set) is found by one thread while the
    // CTA gathers tile k-1, and read by all from a two-slot ring
    __shared__ unsigned long long s_inst[2], s_base[2];
    __shared__ uint32_t s_A[2];
    if (threadIdx.x == 0) {
        uint64_t b0 = 0, b1 = 0;
        uint32_t a0 = 0, a1 = 0;
        const uint64_t i0 = next_tile(i_first, b0, a0);
        const uint64_t i1 = i0 < d.n_inst ? next_tile(i0 + step, b1, a1) : d.n_inst;
        s_inst[0] = i0; s_base[0] = b0; s_A[0] = a0;
        s_inst[1] = i1; s_base[1] = b1; s_A[1] = a1;
    }
    __syncthreads();
    uint64_t inst = s_inst[0], base = s_base[0];
    uint32_t A = s_A[0];
    if (inst < d.n_inst) {
        stage(bufs, base, A, 0);
        if (compose) build(A, comp);
    }
    if (!bulk) cp_async_commit();
    else __syncthreads();  // comp[0] complete before the first gather (the bulk loop has no top barrier)
    for (int b = 0; inst < d.n_inst; b ^= 1) {
        const uint64_t ninst = s_inst[b ^ 1], nbase = s_base[b ^ 1];
        const uint32_t nA = s_A[b ^ 1];
        if (ninst < d.n_inst) stage(bufs + (size_t)(b ^ 1) * E, nbase, nA, b ^ 1);
        if (bulk) {
            // the bulk copy's completion publishes the tile; comp[b] and the
            // look-ahead slots were published by the previous iteration's barrier
            mbar_wait(&s_bar[b], (bar_phase >> b) & 1);
            bar_phase ^= 1u << b;
        } else {
            cp_async_commit();  // (possibly empty) group of the next tile
            cp_async_wait1();   // this thread's copies of the current tile landed
            __syncthreads();    // ... and everyone's; comp[b] complete
        }
        if (threadIdx.x == 0) {  // slot b (this tile's) is free: every thread read it last iteration
            uint64_t b2 = 0;
            uint32_t a2 = 0;
            const uint64_t i2 = ninst < d.n_inst ? next_tile(ninst + step, b2, a2) : d.n_inst;
            s_inst[b] = i2; s_base[b] = b2; s_A[b] = a2;
        }
        const double2 *sm = bufs + (size_t)b * E;
        const uint16_t *cb = comp + (size_t)b * TT;
        const uint32_t head = compose ? (A & d.pre_mask) : 0u;  // composed part of every element's chain
        const uint32_t rest = compose ? ~d.pre_mask : ~0u;
        if (d.contiguous && d.t >= 2) {
            // 4 consecutive elements share the non-target bits: 4 independent
            // lookup chains per thread
            double2 *dst = st + base;
            for (uint32_t e = 4 * threadIdx.x; e < E; e += 4 * blockDim.x) {
                const uint32_t all = A & xmask[e >> d.t];
                if (!all) continue;
                uint32_t act = all & rest;
                uint32_t w[4];
#pragma unroll
                for (int i = 0; i < 4; i++) w[i] = (e + i) & T;
                if (head) {
#pragma unroll
                    for (int i = 0; i < 4; i++) w[i] = cb[w[i]];
                }
                while (act) {
                    const int j = 31 - __clz(act);  // latest active perm first (inverse order)
                    const uint16_t *tj = tab + j * TT;
#pragma unroll
                    for (int i = 0; i < 4; i++) w[i] = tj[w[i]];
                    act &= ~(1u << j);
                }
                const uint32_t hi = e & ~T;
                st256(dst + e, sm[hi | w[0]], sm[hi | w[1]]);
                st256(dst + e + 2, sm[hi | w[2]], sm[hi | w[3]]);
            }
        } else {
            for (uint32_t e = threadIdx.x; e < E; e += blockDim.x) {
                const uint32_t all = A & xmask[e >> d.t];
                if (!all) continue;
                uint32_t w = e & T;
                if (head) w = cb[w];
                w = chain(all & rest, w);
                st[base + (d.contiguous ? e : dep_tile(e, d.tile_pos, d.tile_bits))] = sm[(e & ~T) | w];
            }
        }
        // the next tile's composed table (comp[b ^ 1] was last read two tiles ago)
        if (compose && ninst < d.n_inst) build(nA, comp + (size_t)(b ^ 1) * TT);
        __syncthreads();  // the buffer is refilled two tiles on; slot b is visible
        inst = ninst;
        base = nbase;
        A = nA;
    }
}

size_t perm_run_smem(const PermRunDesc &d) { return perm_run_smem_bytes(d.tile_bits, d.t, d.R, d.pre_mask != 0); }

void launch_perm_run(const PermRunDesc &d, double2 *st, const uint32_t *perm_tab, int n_sm, cudaStream_t s)
{
    const size_t smem = perm_run_smem(d);
    cudaFuncSetAttribute(k_perm_run, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_perm_run, kPermRunThreads, smem) != cudaSuccess || per_sm < 1) {
        cudaGetLastError();
        per_sm = 1;
    }
    const uint64_t grid = std::min<uint64_t>(d.n_inst, (uint64_t)per_sm * (uint64_t)n_sm);
    k_perm_run<<<(unsigned)grid, kPermRunThreads, smem, s>>>(d, st, perm_tab);
}

void launch_perm(const PermDesc &d, double2 *st, const uint32_t *perm_tab, cudaStream_t s)
{
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_perm, cudaFuncAttributeMaxDynamicSharedMemorySize, kPermTileAmps * (int)sizeof(double2));
        attr = true;
    }
    k_perm<<<(unsigned)d.n_inst, 256, (1 << d.tile_bits) * (int)sizeof(double2), s>>>(d, st, perm_tab);
}

// ------------------------------------------------------------------ init
__global__ void k_fill_zero(double2 *__restrict__ st, uint64_t n_pairs)
{
    const double2 z = make_double2(0.0, 0.0);
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n_pairs;
         p += (uint64_t)gridDim.x * blockDim.x)
        st256(st + 2 * p, z, z);
}

__global__ void k_set_amp(double2 *st, uint64_t idx) { st[idx] = make_double2(1.0, 0.0); }

void launch_init(double2 *st, uint64_t n_amps, int64_t one_at, cudaStream_t s)
{
    if (n_amps >= 2) {
        const uint64_t pairs = n_amps / 2;
        k_fill_zero<<<grid_for(pairs, 256), 256, 0, s>>>(st, pairs);
    } else {
        k_phase_generic<<<1, 32, 0, s>>>(st, 1, 0, 0, 0, 0.0, 0.0);
    }
    if (one_at >= 0) k_set_amp<<<1, 1, 0, s>>>(st, (uint64_t)one_at);
}

// ------------------------------------------------------------- reductions
// fixed-shape block sum of one value per thread (deterministic)
__device__ double block_sum(double v, double *red)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x < 32) {
        r = threadIdx.x < nw ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(FULL, r, o);
    }
    return r;  // valid in thread 0
}

// Marginal over listed qubits, stage 1: per 2^cb-amplitude chunk, |a|^2 into
// smem and pairwise-reduce the unlisted chunk bits in ascending order.
__global__ void __launch_bounds__(256) k_probs_chunk(const double2 *__restrict__ st, const __grid_constant__ ProbsDesc d,
                                                     double *__restrict__ partial)
{
    extern __shared__ double v[];
    const uint32_t E = 1u << d.cb;
    const uint64_t c = blockIdx.x;
    for (uint32_t e = threadIdx.x; e < E; e += blockDim.x) {
        const double2 x = st[(c << d.cb) + e];
        v[e] = x.x * x.x + x.y * x.y;
    }
    __syncthreads();
    uint32_t doneb = 0;
    for (int b = 0; b < d.cb; b++) {
        if (!((d.red_mask >> b) & 1)) continue;
        for (uint32_t e = threadIdx.x; e < E; e += blockDim.x)
            if (!(e & (1u << b)) && !(e & doneb)) v[e] += v[e | (1u << b)];
        doneb |= 1u << b;
        __syncthreads();
    }
    const uint32_t B = 1u << d.k_low;
    for (uint32_t bl = threadIdx.x; bl < B; bl += blockDim.x) {
        uint32_t e = 0;
        for (int j = 0; j < d.k_low; j++) e |= ((bl >> j) & 1u) << d.lowpos[j];
        partial[c * B + bl] = v[e];
    }
}

// stage 2: one block per output bin; fixed thread-strided order + block tree
__global__ void __launch_bounds__(256) k_probs_final(const double *__restrict__ partial, const __grid_constant__ ProbsDesc d,
                                                     double *__restrict__ out)
{
    __shared__ double red[32];
    const uint64_t beta = blockIdx.x;
    uint32_t bl = 0;
    uint64_t cfix = 0;
    bool ok = true;
    int jl = 0;
    for (int j = 0; j < d.k; j++) {
        const uint64_t bv = (beta >> j) & 1;
        const int p = d.pos[j];
        if (p < d.cb) bl |= (uint32_t)bv << jl++;
        else if (p < d.M) cfix |= bv << (p - d.cb);
        else if (((d.rank >> (p - d.M)) & 1) != bv) ok = false;
    }
    if (!ok) {
        if (threadIdx.x == 0) out[beta] = 0.0;
        return;
    }
    const uint64_t nj = 1ULL << d.n_free, B = 1ULL << d.k_low;
    double s = 0.0;
    for (uint64_t j = threadIdx.x; j < nj; j += blockDim.x) {
        uint64_t c = cfix;
        for (int b = 0; b < d.n_free; b++) c |= ((j >> b) & 1) << d.freepos[b];
        s += partial[c * B + bl];
    }
    s = block_sum(s, red);
    if (threadIdx.x == 0) out[beta] = s;
}

void launch_probs(const double2 *st, const ProbsDesc &d, double *partial, double *out, cudaStream_t s)
{
    const uint64_t nchunks = 1ULL << (d.M - d.cb);
    k_probs_chunk<<<(unsigned)nchunks, 256, (1 << d.cb) * (int)sizeof(double), s>>>(st, d, partial);
    k_probs_final<<<(unsigned)(1ULL << d.k), 256, 0, s>>>(partial, d, out);
}

// <Q_b> partial sums per chunk: for every chunk bit b the sum over amplitudes
// with bit b = 1, plus the chunk total (index cb).
__global__ void __launch_bounds__(256) k_expect_chunk(const double2 *__restrict__ st, int cb,
                                                      double *__restrict__ partial)
{
    extern __shared__ double v[];
    __shared__ double red[32];
    const uint32_t E = 1u << cb;
    const uint64_t c = blockIdx.x;
    if (cb == 12 && blockDim.x == 256) {
        // one sweep: thread t holds elements e = 2t + {0,1} + 512 j (j < 8) via
        // 256-bit loads; bit 0 of e is the pair element, bits 1-8 the thread,
        // bits 9-11 j.  Per-bit sums of |a|^2 (+ the total) reduced with one
        // barrier, in a fixed order (deterministic).
        const int t = threadIdx.x, lane = t & 31, w = t >> 5;
        const double2 *src = st + (c << 12) + 2 * t;
        double s[13];
#pragma unroll
        for (int b = 0; b < 13; b++) s[b] = 0.0;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            double2 x0, x1;
            ld256(src + 512 * j, x0, x1);
            const double p0 = x0.x * x0.x + x0.y * x0.y, p1 = x1.x * x1.x + x1.y * x1.y;
            s[0] += p1;
            s[12] += p0 + p1;
#pragma unroll
            for (int k = 0; k < 3; k++)
                if ((j >> k) & 1) s[9 + k] += p0 + p1;
        }
#pragma unroll
        for (int b = 1; b <= 8; b++) s[b] = ((t >> (b - 1)) & 1) ? s[12] : 0.0;
#pragma unroll
        for (int b = 0; b < 13; b++)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s[b] += __shfl_xor_sync(FULL, s[b], o);
        double *ws = v;  // [8 warps][13]
        if (lane == 0)
#pragma unroll
            for (int b = 0; b < 13; b++) ws[w * 13 + b] = s[b];
        __syncthreads();
        if (t < 13) {
            double r = 0.0;
            for (int k = 0; k < 8; k++) r += ws[k * 13 + t];
            partial[c * 13 + t] = r;
        }
        return;
    }
    for (uint32_t e = threadIdx.x; e < E; e += blockDim.x) {
        const double2 x = st[(c << cb) + e];
        v[e] = x.x * x.x + x.y * x.y;
    }
    __syncthreads();
    for (int b = 0; b <= cb; b++) {
        double s = 0.0;
        if (b < cb) {
            for (uint32_t j = threadIdx.x; j < (E >> 1); j += blockDim.x)
                s += v[insert_zero(j, b) | (1u << b)];
        } else {
            for (uint32_t j = threadIdx.x; j < E; j += blockDim.x) s += v[j];
        }
        s = block_sum(s, red);
        if (threadIdx.x == 0) partial[c * (cb + 1) + b] = s;
    }
}
__global__ void __launch_bounds__(256) k_expect_final(const double *__restrict__ partial, int cb, int M,
                                                      double *__restrict__ out)
{
    __shared__ double red[32];
    const int o = blockIdx.x;  // physical bit o < M, or o == M: total
    const uint64_t nch = 1ULL << (M - cb);
    double s = 0.0;
    for (uint64_t c = threadIdx.x; c < nch; c += blockDim.x) {
        if (o < cb) s += partial[c * (cb + 1) + o];
        else if (o < M) s += ((c >> (o - cb)) & 1) ? partial[c * (cb + 1) + cb] : 0.0;
        else s += partial[c * (cb + 1) + cb];
    }
    s = block_sum(s, red);
    if (threadIdx.x == 0) out[o] = s;
}

void launch_expect(const double2 *st, int M, double *partial, double *out, cudaStream_t s)
{
    const int cb = M < 12 ? M : 12;
    const uint64_t nch = 1ULL << (M - cb);
    k_expect_chunk<<<(unsigned)nch, 256, (1 << cb) * (int)sizeof(double), s>>>(st, cb, partial);
    k_expect_final<<<M + 1, 256, 0, s>>>(partial, cb, M, out);
}

// Physical-bit sums of one shard from the per-tile partials the readout
// variant of its last pass wrote, in two fixed-order levels (deterministic).
// Level 1: block b reduces the R = min(4096, n_inst) consecutive tiles
// [bR, (b+1)R) for every tile bit, every low instance bit (< log2 R: bit ib
// of the tile index within the block) and the total; the partial rows are
// read once, contiguously.  Level 2: bit o from the level-1 rows (a high
// instance bit is a bit of the block index b).
constexpr int kFusedRow = kTileBits + 1 + 12;  // tile bits, total, low instance bits
__global__ void __launch_bounds__(256) k_expect_fused1(const double *__restrict__ partial, int logR,
                                                       double *__restrict__ out1)
{
    constexpr int W = kTileBits + 1;
    __shared__ double ws[8][kFusedRow];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const uint64_t R = 1ULL << logR, base = (uint64_t)blockIdx.x << logR;
    double acc[kFusedRow];
#pragma unroll
    for (int j = 0; j < kFusedRow; j++) acc[j] = 0.0;
    for (uint64_t j = t; j < R; j += 256) {
        const double *row = partial + (base + j) * W;
#pragma unroll
        for (int q = 0; q < W; q++) acc[q] += row[q];
        const double tot = row[kTileBits];
#pragma unroll
        for (int ib = 0; ib < 12; ib++)
            if (ib < logR && ((j >> ib) & 1)) acc[W + ib] += tot;
    }
#pragma unroll
    for (int q = 0; q < kFusedRow; q++) {
        double v = acc[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
        if (lane == 0) ws[w][q] = v;
    }
    __syncthreads();
    if (t < kFusedRow) {
        double v = ws[0][t];
        for (int k = 1; k < 8; k++) v += ws[k][t];
        out1[(uint64_t)blockIdx.x * kFusedRow + t] = v;
    }
}
__global__ void __launch_bounds__(256) k_expect_fused2(const double *__restrict__ out1, uint64_t nb, int logR,
                                                       const __grid_constant__ FusedExpectDesc d,
                                                       double *__restrict__ out)
{
    __shared__ double red[32];
    const int o = blockIdx.x;  // physical bit o < M, or o == M: total
    const int t = o < d.M ? d.tile_of[o] : kTileBits, ib = o < d.M ? d.inst_bit[o] : 0;
    double s = 0.0;
    for (uint64_t b = threadIdx.x; b < nb; b += blockDim.x) {
        const double *row = out1 + b * kFusedRow;
        if (t >= 0) s += row[t];
        else if (ib < logR) s += row[kTileBits + 1 + ib];
        else s += ((b >> (ib - logR)) & 1) ? row[kTileBits] : 0.0;
    }
    s = block_sum(s, red);
    if (threadIdx.x == 0) out[o] = s;
}

size_t expect_fused_scratch(uint64_t n_inst)
{
    const int logR = n_inst >= 4096 ? 12 : __builtin_ctzll(n_inst);
    return (size_t)(n_inst >> logR) * kFusedRow;
}

void launch_expect_fused(const double *partial, const FusedExpectDesc &d, double *scratch, double *out, cudaStream_t s)
{
    const int logR = d.n_inst >= 4096 ? 12 : __builtin_ctzll(d.n_inst);
    const uint64_t nb = d.n_inst >> logR;
    k_expect_fused1<<<(unsigned)nb, 256, 0, s>>>(partial, logR, scratch);
    k_expect_fused2<<<d.M + 1, 256, 0, s>>>(scratch, nb, logR, d, out);
}

// <Q_q> in logical order from S shards' physical-bit sums (phys[s*(M+1) + p],
// p < M: bit p set, p == M: total), shard s holding rank s:
// out[q] = sum over s in order of (p < M ? phys_s[p] : rank bit p-M of s ? phys_s[M] : 0)
__global__ void k_expect_logical(const double *__restrict__ phys, const __grid_constant__ ExpectMap m,
                                 double *__restrict__ out)
{
    const int q = threadIdx.x;
    if (q >= m.n) return;
    const int p = m.phys_of[q];
    double a = 0.0;
    for (int r = 0; r < m.S; r++) {
        const double *v = phys + (size_t)r * (m.M + 1);
        a += p < m.M ? v[p] : (((r >> (p - m.M)) & 1) ? v[m.M] : 0.0);
    }
    out[q] = a;
}

void launch_expect_logical(const double *phys, const ExpectMap &m, double *out, cudaStream_t s)
{
    k_expect_logical<<<1, 64, 0, s>>>(phys, m, out);
}

// ------------------------------------------------------------- sampling
__device__ __forceinline__ uint64_t sm64_dev(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__global__ void __launch_bounds__(1024) k_cdf(const double *__restrict__ p, uint64_t B, double *__restrict__ C)
{
    __shared__ double tot[1024];
    const uint64_t seg = (B + blockDim.x - 1) / blockDim.x;
    const uint64_t lo = threadIdx.x * seg, hi = lo + seg < B ? lo + seg : B;
    double acc = 0.0;
    for (uint64_t i = lo; i < hi; i++) { acc += p[i]; C[i] = acc; }
    tot[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double run = 0.0;
        for (int t = 0; t < (int)blockDim.x; t++) { const double x = tot[t]; tot[t] = run; run += x; }
    }
    __syncthreads();
    const double off = tot[threadIdx.x];
    for (uint64_t i = lo; i < hi; i++) C[i] += off;
}

__global__ void k_sample(const double *__restrict__ C, uint64_t B, uint64_t seed, uint64_t n, uint64_t *__restrict__ out)
{
    const double tot = C[B - 1];
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < n; s += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = sm64_dev(seed + (s + 1) * 0x9E3779B97F4A7C15ULL);
        const double u = (double)(r >> 11) * (1.0 / 9007199254740992.0) * tot;
        uint64_t lo = 0, hi = B - 1;  // min beta with C[beta] > u (B-1 if none)
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (C[mid] > u) hi = mid; else lo = mid + 1;
        }
        out[s] = lo;
    }
}

void launch_sample(const double *p, int k, uint64_t seed, uint64_t n_shots, double *cdf, uint64_t *out, cudaStream_t s)
{
    const uint64_t B = 1ULL << k;
    k_cdf<<<1, 1024, 0, s>>>(p, B, cdf);
    if (n_shots) k_sample<<<grid_for(n_shots, 256), 256, 0, s>>>(cdf, B, seed, n_shots, out);
}

// --------------------------------------------- two-level sampling (k > 24)
// Conditional marginals of the low c listed qubits inside nb bins of the
// high listed qubits (bins[j] = value of the high listed qubits): out[j 2^c +
// b] = sum over the unlisted qubits (fixed increasing order) of |a|^2 at the
// amplitude whose listed-low bits are b, listed-high bits bins[j]; only the
// amplitudes this shard holds (physical bits >= M equal `rank`) contribute.
struct BinDesc {
    int32_t c, kh, nu, M;
    uint64_t rank;
    int32_t pos_lo[24], pos_hi[24], pos_un[64];
};

__global__ void k_bin_marginal(const double2 *__restrict__ st, BinDesc d, const uint64_t *__restrict__ bins,
                               uint64_t nb, double *__restrict__ out)
{
    const uint64_t per = 1ULL << d.c, total = nb * per;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t j = t >> d.c, b = t & (per - 1), h = bins[j];
        uint64_t base = 0;
        for (int i = 0; i < d.c; i++) base |= ((b >> i) & 1) << d.pos_lo[i];
        for (int i = 0; i < d.kh; i++) base |= ((h >> i) & 1) << d.pos_hi[i];
        double acc = 0.0;
        const uint64_t nun = 1ULL << d.nu;
        for (uint64_t u = 0; u < nun; u++) {
            uint64_t x = base;
            for (int i = 0; i < d.nu; i++) x |= ((u >> i) & 1) << d.pos_un[i];
            if ((x >> d.M) != d.rank) continue;
            const double2 a = st[x & ((1ULL << d.M) - 1)];
            acc = fma(a.x, a.x, acc);
            acc = fma(a.y, a.y, acc);
        }
        out[t] = acc;
    }
}

void launch_bin_marginal(const double2 *st, int M, uint64_t rank, int c, const int *pos_lo, int kh,
                         const int *pos_hi, int nu, const int *pos_un, const uint64_t *bins, uint64_t nb, double *out,
                         cudaStream_t s)
{
    BinDesc d{};
    d.c = c;
    d.kh = kh;
    d.nu = nu;
    d.M = M;
    d.rank = rank;
    for (int i = 0; i < c; i++) d.pos_lo[i] = pos_lo[i];
    for (int i = 0; i < kh; i++) d.pos_hi[i] = pos_hi[i];
    for (int i = 0; i < nu; i++) d.pos_un[i] = pos_un[i];
    k_bin_marginal<<<grid_for(nb << c, 256), 256, 0, s>>>(st, d, bins, nb, out);
}

// level 1: per shot, u = draw * total; the high bin (min beta_hi with
// C[beta_hi] > u, else the last) and the residual u - C[beta_hi - 1]
__global__ void k_sample_hi(const double *__restrict__ C, uint64_t B, uint64_t seed, uint64_t n,
                            uint64_t *__restrict__ bhi, double *__restrict__ res)
{
    const double tot = C[B - 1];
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < n; s += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = sm64_dev(seed + (s + 1) * 0x9E3779B97F4A7C15ULL);
        const double u = (double)(r >> 11) * (1.0 / 9007199254740992.0) * tot;
        uint64_t lo = 0, hi = B - 1;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (C[mid] > u) hi = mid; else lo = mid + 1;
        }
        bhi[s] = lo;
        res[s] = u - (lo ? C[lo - 1] : 0.0);
    }
}

// level 2: one CTA per bin row, the row's inclusive prefix sum (k_cdf order)
__global__ void __launch_bounds__(1024) k_cdf_rows(double *__restrict__ rows, uint64_t per)
{
    __shared__ double tot[1024];
    double *C = rows + blockIdx.x * per;
    const uint64_t seg = (per + blockDim.x - 1) / blockDim.x;
    const uint64_t lo = threadIdx.x * seg, hi = lo + seg < per ? lo + seg : per;
    double acc = 0.0;
    for (uint64_t i = lo; i < hi; i++) { acc += C[i]; C[i] = acc; }
    tot[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double run = 0.0;
        for (int t = 0; t < (int)blockDim.x; t++) { const double x = tot[t]; tot[t] = run; run += x; }
    }
    __syncthreads();
    const double off = tot[threadIdx.x];
    for (uint64_t i = lo; i < hi; i++) C[i] += off;
}

// per shot of this batch: min beta_lo with C_row[beta_lo] > residual (the last
// bin of nonzero weight if rounding leaves the residual at the row's end);
// outcome = beta_lo | beta_hi << c
__global__ void k_sample_lo(const double *__restrict__ rows, uint64_t per, int c, const uint32_t *__restrict__ shot_row,
                            const uint64_t *__restrict__ shot_idx, uint64_t n, const uint64_t *__restrict__ bhi,
                            const double *__restrict__ res, uint64_t *__restrict__ out)
{
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t s = shot_idx[t];
        const double *C = rows + (uint64_t)shot_row[t] * per;
        const double u = res[s];
        uint64_t lo = 0, hi = per - 1;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (C[mid] > u) hi = mid; else lo = mid + 1;
        }
        while (lo > 0 && C[lo] == (lo ? C[lo - 1] : 0.0)) lo--;  // zero-weight tail (rounding)
        out[s] = lo | (bhi[s] << c);
    }
}

void launch_sample_hi(const double *p, int kh, uint64_t seed, uint64_t n_shots, double *cdf, uint64_t *bhi,
                      double *res, cudaStream_t s)
{
    const uint64_t B = 1ULL << kh;
    k_cdf<<<1, 1024, 0, s>>>(p, B, cdf);
    if (n_shots) k_sample_hi<<<grid_for(n_shots, 256), 256, 0, s>>>(cdf, B, seed, n_shots, bhi, res);
}

void launch_sample_lo(double *rows, uint64_t nrows, int c, const uint32_t *shot_row, const uint64_t *shot_idx,
                      uint64_t n, const uint64_t *bhi, const double *res, uint64_t *out, cudaStream_t s)
{
    const uint64_t per = 1ULL << c;
    k_cdf_rows<<<(unsigned)nrows, 1024, 0, s>>>(rows, per);
    if (n) k_sample_lo<<<grid_for(n, 256), 256, 0, s>>>(rows, per, c, shot_row, shot_idx, n, bhi, res, out);
}

// ------------------------------------------------------------- readout
struct Phys64 {
    int32_t p[64];
};

__global__ void k_gather(double2 *__restrict__ out, uint64_t first, uint64_t count, double2 *const *shards, int virt,
                         int my_rank, int M, int n, Phys64 ph)
{
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t x = first + i;
        uint64_t phys = 0;
        for (int q = 0; q < n; q++) phys |= ((x >> q) & 1) << ph.p[q];
        const uint64_t r = phys >> M, li = phys & ((1ULL << M) - 1);
        double2 v;
        if (virt) v = shards[r][li];
        else v = ((int)r == my_rank) ? shards[0][li] : make_double2(0.0, 0.0);
        out[i] = v;
    }
}

void launch_gather(double2 *out, uint64_t first, uint64_t count, double2 *const *shards_dev, int virt, int my_rank,
                   int M, int n, const int *phys_of, cudaStream_t s)
{
    Phys64 ph;
    for (int q = 0; q < 64; q++) ph.p[q] = q < n ? phys_of[q] : 0;
    k_gather<<<grid_for(count, 256), 256, 0, s>>>(out, first, count, shards_dev, virt, my_rank, M, n, ph);
}

// ------------------------------------------------------------- exchange
struct LPos {
    int32_t sorted[8];
    uint64_t off_bits[8];  // 1 << lpos[i] in pairing order
};

__device__ __forceinline__ uint64_t other_index(uint64_t j, const LPos &L, int K)
{
    for (int i = 0; i < K; i++) j = insert_zero(j, L.sorted[i]);
    return j;
}

__global__ void k_swap_blocks(double2 *__restrict__ A, double2 *__restrict__ B, uint64_t n_other, int K, LPos L,
                              uint64_t offA, uint64_t offB)
{
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n_other;
         j += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t idx = other_index(j, L, K);
        const double2 x = A[idx | offA], y = B[idx | offB];
        A[idx | offA] = y;
        B[idx | offB] = x;
    }
}

__global__ void k_pack(double2 *__restrict__ shard, double2 *__restrict__ buf, uint64_t first, uint64_t count, int K,
                       LPos L, uint64_t off, int unpack)
{
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t idx = other_index(first + i, L, K) | off;
        if (unpack) shard[idx] = buf[i];
        else buf[i] = shard[idx];
    }
}

// pairwise global-target gate (virtual shards): A holds the partner with the
// target bit 0, B with the bit 1; both are updated from both (1x traffic)
__global__ void k_pair_gate(double2 *__restrict__ A, double2 *__restrict__ B, uint64_t count, uint64_t mloc,
                            uint64_t vloc, int xs, U8 u)
{
    const double2 u00 = make_double2(u.m[0], u.m[1]), u01 = make_double2(u.m[2], u.m[3]);
    const double2 u10 = make_double2(u.m[4], u.m[5]), u11 = make_double2(u.m[6], u.m[7]);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x) {
        if ((i & mloc) != vloc) continue;
        const double2 a = A[i], b = B[i];
        if (xs) {
            A[i] = b;
            B[i] = a;
        } else {
            A[i] = cmac2(u00, a, u01, b);
            B[i] = cmac2(u10, a, u11, b);
        }
    }
}

// pairwise over NCCL: own <- c0*own + c1*other (self_first) or c0*other + c1*own
__global__ void k_pair_combine(double2 *__restrict__ own, const double2 *__restrict__ other, uint64_t off,
                               uint64_t count, uint64_t mloc, uint64_t vloc, double2 c0, double2 c1, int self_first)
{
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x) {
        if (((off + i) & mloc) != vloc) continue;
        own[i] = self_first ? cmac2(c0, own[i], c1, other[i]) : cmac2(c0, other[i], c1, own[i]);
    }
}

void launch_pair_gate(double2 *A, double2 *B, int M, uint64_t mloc, uint64_t vloc, int xs, const double *m,
                      cudaStream_t s)
{
    U8 u;
    for (int k = 0; k < 8; k++) u.m[k] = m[k];
    const uint64_t n = 1ULL << M;
    k_pair_gate<<<grid_for(n, 256), 256, 0, s>>>(A, B, n, mloc, vloc, xs, u);
}

void launch_pair_combine(double2 *own, const double2 *other, uint64_t off, uint64_t count, uint64_t mloc,
                         uint64_t vloc, const double *c0, const double *c1, int self_first, cudaStream_t s)
{
    k_pair_combine<<<grid_for(count, 256), 256, 0, s>>>(own, other, off, count, mloc, vloc,
                                                      make_double2(c0[0], c0[1]), make_double2(c1[0], c1[1]),
                                                      self_first);
}

static LPos make_lpos(int K, const int *lpos, uint64_t c, uint64_t *off)
{
    LPos L{};
    int tmp[8];
    for (int i = 0; i < K; i++) tmp[i] = lpos[i];
    for (int i = 0; i < K; i++)
        for (int j = i + 1; j < K; j++)
            if (tmp[j] < tmp[i]) { int x = tmp[i]; tmp[i] = tmp[j]; tmp[j] = x; }
    *off = 0;
    for (int i = 0; i < K; i++) {
        L.sorted[i] = tmp[i];
        L.off_bits[i] = 1ULL << lpos[i];
        if ((c >> i) & 1) *off |= 1ULL << lpos[i];
    }
    return L;
}

// 2 consecutive amplitudes per thread (one 256-bit access per side; a warp
// covers 1 KB contiguous) when the exchanged bits are >= 1, two pairs in
// flight per thread
__global__ void __launch_bounds__(256) k_swap_blocks2(double2 *__restrict__ A, double2 *__restrict__ B,
                                                      uint64_t n_pairs, int K, LPos L, uint64_t offA, uint64_t offB)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n_pairs; q += 2 * stride) {
        const bool two = q + stride < n_pairs;
        const uint64_t i0 = other_index(q << 1, L, K), i1 = two ? other_index((q + stride) << 1, L, K) : i0;
        double2 a0, a1, b0, b1, c0, c1, d0, d1;
        ld256(A + (i0 | offA), a0, a1);
        ld256(B + (i0 | offB), b0, b1);
        if (two) {
            ld256(A + (i1 | offA), c0, c1);
            ld256(B + (i1 | offB), d0, d1);
        }
        st256(A + (i0 | offA), b0, b1);
        st256(B + (i0 | offB), a0, a1);
        if (two) {
            st256(A + (i1 | offA), d0, d1);
            st256(B + (i1 | offB), c0, c1);
        }
    }
}

void launch_swap_blocks(double2 *A, double2 *B, int M, int K, const int *lpos, uint64_t cA, uint64_t cB, cudaStream_t s)
{
    uint64_t offA, offB;
    LPos L = make_lpos(K, lpos, cA, &offA);
    make_lpos(K, lpos, cB, &offB);
    const uint64_t n_other = 1ULL << (M - K);
    if (K > 0 && L.sorted[0] >= 1 && n_other >= 2) {
        k_swap_blocks2<<<grid_for(n_other / 2, 256), 256, 0, s>>>(A, B, n_other / 2, K, L, offA, offB);
        return;
    }
    k_swap_blocks<<<grid_for(n_other, 256), 256, 0, s>>>(A, B, n_other, K, L, offA, offB);
}

// out[j] = sum over ranks r (in rank order) of all[r * count + j]
__global__ void k_sum_ranks(const double *__restrict__ all, double *__restrict__ out, uint64_t count, int S)
{
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < count; j += (uint64_t)gridDim.x * blockDim.x) {
        double a = all[j];
        for (int r = 1; r < S; r++) a += all[(uint64_t)r * count + j];
        out[j] = a;
    }
}

void launch_sum_ranks(const double *all, double *out, uint64_t count, int S, cudaStream_t s)
{
    k_sum_ranks<<<grid_for(count, 256), 256, 0, s>>>(all, out, count, S);
}

void launch_pack(const double2 *shard, double2 *buf, int M, int K, const int *lpos, uint64_t c, uint64_t first,
                 uint64_t count, int unpack, cudaStream_t s)
{
    uint64_t off;
    LPos L = make_lpos(K, lpos, c, &off);
    (void)M;
    k_pack<<<grid_for(count, 256), 256, 0, s>>>(const_cast<double2 *>(shard), buf, first, count, K, L, off, unpack);
}

// ------------------------------------------------ roofline denominators
// FP64 FMA-pipe throughput probe: 8 independent DFMA chains per thread, two
// 256-thread CTAs per SM per wave (the pass kernel's residency), many waves.
__global__ void __launch_bounds__(256) k_probe_dfma(double *out, int iters, double a, double b)
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
    const double r = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (r == 12345.678) out[blockIdx.x] = r;  // keeps the chains live, never true
}

// streaming copy (read + write), 256-bit accesses, grid-stride
__global__ void k_probe_copy(const double4 *__restrict__ in, double4 *__restrict__ out, size_t n)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}

int probe_peaks(double *fp64_flops, double *copy_bytes_per_s, int reps)
{
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaStream_t s;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return -1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double *out = nullptr;
    int rc = 0;
    if (cudaMalloc(&out, sizeof(double) * sms * 64) != cudaSuccess) rc = -1;
    if (!rc && fp64_flops) {
        const int iters = 2048, blocks = sms * 2 * 8;
        k_probe_dfma<<<blocks, 256, 0, s>>>(out, 16, 1.0000001, 1e-9);
        float best = 1e30f;
        for (int r = 0; r < reps; r++) {
            cudaEventRecord(e0, s);
            k_probe_dfma<<<blocks, 256, 0, s>>>(out, iters, 1.0000001, 1e-9);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        *fp64_flops = 2.0 * (double)blocks * 256 * iters * 16 * 8 / (best * 1e-3);
    }
    if (!rc && copy_bytes_per_s) {
        const size_t bytes = (size_t)1 << 30;
        double4 *a = nullptr, *b = nullptr;
        if (cudaMalloc(&a, bytes) != cudaSuccess || cudaMalloc(&b, bytes) != cudaSuccess) {
            rc = -1;
        } else {
            cudaMemsetAsync(a, 0, bytes, s);
            const size_t n = bytes / sizeof(double4);
            float best = 1e30f;
            for (int r = 0; r < reps + 1; r++) {
                cudaEventRecord(e0, s);
                k_probe_copy<<<sms * 8, 256, 0, s>>>(a, b, n);
                cudaEventRecord(e1, s);
                cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                if (r) best = ms < best ? ms : best;
            }
            *copy_bytes_per_s = 2.0 * bytes / (best * 1e-3);
        }
        cudaFree(a);
        cudaFree(b);
    }
    cudaFree(out);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
    if (cudaGetLastError() != cudaSuccess) rc = -1;
    return rc;
}

}  // namespace qsb
