// jit.cpp -- code generation + NVRTC compilation of pass-specialised kernels.
// See jit.h.  The generated kernel is the k_pass of kernels.cu with the op
// loop unrolled at generation time: register bits, predicates and shared-
// memory re-layouts become constants, the CNOT/Toffoli register swap becomes
// a renaming, and the matrices are read as constant-bank operands.  Beyond
// k_pass: deferred predicated swaps folded into store addresses, lazy phase
// flushes with CTA-uniform / per-thread term slots (qsim_pass_tab), the
// Hadamard form, the fresh (basis-state) first pass and low-qubit stores.
#include "jit.h"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <cstdio>
#include <unistd.h>
#include <sys/stat.h>
#include <nvrtc.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <atomic>
#include <chrono>
#include <cstring>
#include <map>
#include <set>
#include <functional>
#include <sstream>
#include <thread>

namespace qsb {

namespace {

int nib(uint64_t c, int j) { return (int)((c >> (4 * j)) & 15); }
int swz_host(int s) { return s ^ (((s >> 3) ^ (s >> 6) ^ (s >> 9)) & 7); }

// parameter block layout (the JP struct of the generated source)
constexpr int kMaxFix = 4;  // instance bits a launch may fix (jit_set_block)
constexpr size_t kOffInit = 32, kOffTtab = 40, kOffFix = 48, kOffRed = 56, kOffTpm = 64,
                 kOffTs = kOffTpm + 8 * kTileBits;
// 16-B aligned (the matrix rows that follow are read as 128-bit constants)
constexpr size_t kOffTpo = (kOffTs + 4 * (kTileBits + kMaxFix) + 15) / 16 * 16;
constexpr int kTsPad = (int)(kOffTpo - kOffTs) / 4 - (kTileBits + kMaxFix);  // ints of padding after ts

constexpr size_t kOffOut = (kOffTpo + 8 * kTileBits + 15) / 16 * 16;  // the matrix rows after out[] stay 16-B aligned
constexpr int kTpoPad = (int)(kOffOut - kOffTpo) / 8 - kTileBits;     // u64s of padding after tpo
struct Layout {
    int n_out = 0, n_m = 0;
    int c_row = 0;  // first row of the host-formed phase factors (4 complex per row)
    size_t off_out = kOffOut, off_m = 0, bytes = 0;
};

constexpr int kJitBarDefault = 3;  // re-layout barrier form, see QSIM_JIT_BAR below

// generator variant (env, for A/B experiments): minimum CTAs per SM.  A
// persistent grid with L2 prefetch of the next tile and 1 or 3 CTAs/SM were
// measured slower on config 2 (register spills / occupancy).
int env_int(const char *k, int dflt)
{
    const char *v = getenv(k);
    return v ? atoi(v) : dflt;
}

// Arithmetic form of general 2x2 (OPC_U2) and 4x4 (OPC_U4) blocks in a pass:
// the 3M form (fewer FP64 instructions, three live copies of every input
// amplitude) or the direct complex FMA form (two).  QSIM_JIT_3M (A/B switch,
// read once): bit 0 = 3M for U2, bit 1 = 3M for U4; default auto.
struct Forms {
    bool u2 = true, u4 = true;
};
Forms forms_of(const Step &st)
{
    static const int env = env_int("QSIM_JIT_3M", -1);
    Forms f;
    if (env >= 0) {
        f.u2 = env & 1;
        f.u4 = (env >> 1) & 1;
        return f;
    }
    return f;
}

// Phase runs: where every OPC_PHASE_ACC term goes.  The generated pass
// flushes monomial S (a product of register bits) lazily: an op on register
// bit k flushes the live monomials containing k, a re-layout and the store
// flush all.  Between two flushes of S (an "epoch") its angle is a sum of
// terms of four kinds:
//   const   -- unpredicated on lane, warp and out-of-tile bits: the same in
//              every thread and tile, so e^{i sum} is formed on the host and
//              travels in the parameter block (no exponential in the kernel);
//   uniform -- predicated on out-of-tile bits only (CTA-uniform): summed per
//              (S, epoch) slot once per tile through shared memory, where its
//              e^{i sum} is also formed once per tile;
//   thread  -- predicated on lane / warp bits only: summed per slot and thread
//              once per launch by the companion kernel qsim_pass_tab, which
//              stores e^{i sum};
//   inline  -- the rest (mixed predicates, or too few terms for a table): an
//              integer accumulator mo_S and one exponential at the flush.
// The flush multiplies the amplitudes by the product of the parts present
// (e^{i(a+b)} = e^{ia} e^{ib}).  The dry run below follows the generator's
// flush rules exactly; jit_generate, layout_of and jit_pack_params share it.
bool uniform_acc(const KOp &op) { return op.code == OPC_PHASE_ACC && op.mout && !op.mlane && !op.mwarp; }
bool thread_acc(const KOp &op) { return op.code == OPC_PHASE_ACC && !op.mout && (op.mlane || op.mwarp); }
bool const_acc(const KOp &op) { return op.code == OPC_PHASE_ACC && !op.mout && !op.mlane && !op.mwarp; }
uint32_t touching(uint32_t bits)  // monomials that contain one of the register bits
{
    uint32_t F = 0;
    for (uint32_t S = 0; S < (uint32_t)kAmpsPerThread; S++)
        if (S & bits) F |= 1u << S;
    return F;
}
struct PhasePlan {
    // per op: (slot, sign) of each of its monomial terms, by kind
    std::vector<std::vector<std::pair<int, int>>> uterms, tterms, cterms;
    std::vector<uint32_t> slot_S, tslot_S, cslot_S;
    std::map<std::pair<uint32_t, int>, int> slot_of, tslot_of, cslot_of;  // (monomial, epoch) -> slot
    std::set<std::pair<uint32_t, int>> inl;                               // (monomial, epoch) with inline terms
    uint32_t inl_used = 0;                                                // monomials with an accumulator
};
PhasePlan phase_plan(const Step &st)
{
    PhasePlan pp;
    const size_t n = st.ops.size();
    pp.uterms.assign(n, {});
    pp.tterms.assign(n, {});
    pp.cterms.assign(n, {});
    int n_uni = 0, n_thr = 0;
    for (const KOp &op : st.ops) { n_uni += uniform_acc(op); n_thr += thread_acc(op); }
    const bool use_u = n_uni >= 8, use_t = n_thr >= 8;
    int epoch[kAmpsPerThread] = {0};
    uint32_t live = 0;
    auto flush = [&](uint32_t F) {
        F &= live;
        for (uint32_t S = 0; S < (uint32_t)kAmpsPerThread; S++)
            if ((F >> S) & 1) epoch[S]++;
        live &= ~F;
    };
    for (size_t o = 0; o < n; o++) {
        const KOp &op = st.ops[o];
        if (op.code == OPC_TRANS) { flush(~0u); continue; }
        if (op.code == OPC_PHASE_FLUSH || op.code == OPC_DATA || op.code == OPC_PHASE) continue;
        if (op.code == OPC_U4) { flush(touching((1u << op.k) | (1u << (int)op.cfg))); continue; }
        if (op.code == OPC_PHASE_ACC) {
            const bool u = use_u && uniform_acc(op), th = use_t && thread_acc(op), c = const_acc(op);
            const uint32_t O = op.mreg & op.vreg, Z = op.mreg & ~op.vreg;
            for (uint32_t T = Z;; T = (T - 1) & Z) {
                const uint32_t S = O | T;
                const auto key = std::make_pair(S, epoch[S]);
                if (u || th || c) {
                    auto &of = u ? pp.slot_of : th ? pp.tslot_of : pp.cslot_of;
                    auto &sv = u ? pp.slot_S : th ? pp.tslot_S : pp.cslot_S;
                    auto it = of.find(key);
                    if (it == of.end()) {
                        it = of.emplace(key, (int)sv.size()).first;
                        sv.push_back(S);
                    }
                    (u ? pp.uterms : th ? pp.tterms : pp.cterms)[o].push_back(
                        {it->second, __builtin_popcount(T) & 1 ? -1 : 1});
                } else {
                    pp.inl.insert(key);
                    pp.inl_used |= 1u << S;
                }
                live |= 1u << S;
                if (!T) break;
            }
            continue;
        }
        flush(touching(1u << op.k));
    }
    return pp;
}

// Parameter block: out-of-tile predicates (mout, vout) deduplicated by value;
// matrix rows of 8 doubles: a U2 takes a row, a U4 its row and its 3 OPC_DATA
// rows; phases share rows (a multiplier takes 2 doubles, an accumulated
// angle 1), so long phase runs (QFT ladders) fit the 32-KB parameter limit.
// m_col[o]: first double of op o inside row m_idx[o].
Layout layout_of(const Step &st, std::vector<int> &out_idx, std::vector<int> &m_idx, std::vector<int> &m_col)
{
    Layout L;
    const Forms fm = forms_of(st);
    out_idx.assign(st.ops.size(), -1);
    m_idx.assign(st.ops.size(), -1);
    m_col.assign(st.ops.size(), 0);
    std::vector<std::pair<uint64_t, uint64_t>> outs;
    int acc_row = -1, acc_col = 8, ph_row = -1, ph_col = 8;
    for (size_t o = 0; o < st.ops.size(); o++) {
        const KOp &op = st.ops[o];
        if (op.code == OPC_TRANS || op.code == OPC_PHASE_FLUSH) continue;
        if (op.mout) {
            const std::pair<uint64_t, uint64_t> key{op.mout, op.vout};
            size_t k = std::find(outs.begin(), outs.end(), key) - outs.begin();
            if (k == outs.size()) outs.push_back(key);
            out_idx[o] = (int)k;
        }
        if (op.code == OPC_XS) continue;
        if (const_acc(op)) continue;  // folded into a host-formed factor (phase_plan)
        if (op.code == OPC_PHASE_ACC) {
            if (acc_col >= 8) { acc_row = L.n_m++; acc_col = 0; }
            m_idx[o] = acc_row;
            m_col[o] = acc_col++;
        } else if (op.code == OPC_PHASE) {
            if (ph_col >= 8) { ph_row = L.n_m++; ph_col = 0; }
            m_idx[o] = ph_row;
            m_col[o] = ph_col;
            ph_col += 2;
        } else if (op.code == OPC_DATA && fm.u4) {
            continue;  // rows 1..3 of an OPC_U4: the U4's own 6 rows hold its 3M constants
        } else if (op.code == OPC_U4 && fm.u4) {
            m_idx[o] = L.n_m;  // A, -(A+B), B-A: 3 x 16 doubles
            L.n_m += 6;
        } else if (op.code == OPC_U2 && fm.u2) {
            m_idx[o] = L.n_m;  // A, -(A+B), B-A: 3 x 4 doubles
            L.n_m += 2;
        } else {
            m_idx[o] = L.n_m++;
        }
    }
    {
        const PhasePlan pp = phase_plan(st);
        L.c_row = L.n_m;
        L.n_m += ((int)pp.cslot_S.size() + 3) / 4;
    }
    L.n_out = (int)outs.size();
    L.off_m = L.off_out + 16 * (size_t)std::max(1, L.n_out);
    L.bytes = (L.off_m + 64 * (size_t)std::max(1, L.n_m) + 15) / 16 * 16;
    return L;
}

}  // namespace

void jit_launch_dims(const Step &st, int n_sm, unsigned &grid, unsigned &block, unsigned &smem)
{
    (void)n_sm;
    grid = (unsigned)st.pass.n_inst;
    block = kPassThreads;
    smem = st.pass.use_smem ? kTileAmps * 16 : 0;
}

// An unpredicated Hadamard-form real 2x2, h [[1, 1], [1, -1]]: the JIT tier
// applies the unnormalised sum/difference (2 adds per component instead of
// 2 multiplies + 2 FMAs) and multiplies the product of the h's in once
// before the store (every op is linear, so the scale commutes).
static bool jit_hadamard(const KOp &op)
{
    return op.code == OPC_U2R && !op.mreg && !op.mlane && !op.mwarp && !op.mout && op.m[1] == 0 && op.m[3] == 0 &&
           op.m[5] == 0 && op.m[7] == 0 && op.m[0] == op.m[2] && op.m[0] == op.m[4] && op.m[6] == -op.m[0];
}

JitPass jit_generate(const Step &st)
{
    std::vector<int> out_idx, m_idx, m_col;
    Layout L = layout_of(st, out_idx, m_idx, m_col);
    const Forms fm = forms_of(st);
    std::ostringstream s;
    // FP64-pipe instructions per thread the generated code executes (DFMA,
    // DMUL, DADD and the F64 conversion of qexp), for the roofline
    double fpc = 0;
    const int kQexpOps = 13;
    const int minb = env_int("QSIM_JIT_MINB", kPassMinBlocks);  // CTAs per SM (register cap)
    s << "// minb=" << minb << "\n";
    s << "struct __align__(16) JP { double2 *st; unsigned long long rank_bits; unsigned long long desync; "
         "const double2 *ptab; unsigned long long init_phys; unsigned long long *ttab; unsigned long long fixbits; "
         "double *red; "
         "unsigned long long tpm[" << kTileBits << "]; int ts[" << kTileBits + kMaxFix << "]; "
      << (kTsPad ? "int ts_pad[" + std::to_string(kTsPad) + "]; " : std::string())
      << "unsigned long long tpo[" << kTileBits << "]; "
      << (kTpoPad ? "unsigned long long tpo_pad[" + std::to_string(kTpoPad) + "]; " : std::string())
      << "unsigned long long out["
      << std::max(1, L.n_out) << "][2]; double m[" << std::max(1, L.n_m) << "][8]; };\n";
    // instance -> physical base: zeros inserted at the tile positions (ts
    // sorted ascending).  The block variant (Step::jit_block) also inserts
    // them at the positions a launch fixes and ORs in their values (unused
    // entries are 62: a no-op insertion for any b < 2^62).  Only that
    // variant pays for the longer chain: the 16-entry form in every pass
    // raised the kernels' uniform-register traffic several-fold.
    const int n_ins = st.jit_block ? kTileBits + kMaxFix : kTileBits;
    s << "__device__ __forceinline__ unsigned long long qdep(unsigned long long b, const int *ts)\n{\n"
         "#pragma unroll\n for (int j = 0; j < " << n_ins << "; j++) { const int t = ts[j]; "
         "b = ((b >> t) << (t + 1)) | (b & ((1ULL << t) - 1)); }\n return b;\n}\n";
    // e^{2 pi i t / 2^64}: table of the top 8 bits x Taylor series of the rest (|x| < 2pi/256)
    // e^{2 pi i t / 2^64}: the nearest table angle k/256 times e^{i x}, |x| <=
    // pi/256, by Taylor to x^6 (cos) and x^5 (sin): truncation < 1e-17
    s << "__device__ __forceinline__ double2 qexp(unsigned long long t, const double2 *tab)\n{\n"
         " const unsigned long long k = (t + (1ULL << 55)) >> 56;\n"
         " const double2 b = __ldg(tab + k);\n"
         " const double x = (double)(long long)(t - (k << 56)) * 3.4061215800865545e-19;\n"  // 2pi / 2^64
         " const double x2 = x * x;\n"
         " const double c = fma(x2, fma(x2, fma(x2, -1.3888888888888889e-03, 4.1666666666666664e-02), -0.5), 1.0);\n"
         " const double s = x * fma(x2, fma(x2, 8.3333333333333332e-03, -1.6666666666666666e-01), 1.0);\n"
         " return make_double2(fma(b.x, c, -b.y * s), fma(b.x, s, b.y * c));\n}\n";
    const int NT = kPassThreads;
    const std::string BAR = "__syncthreads();";
    s << "#define TPM P.tpm\n#define TSP P.ts\n#define TPO P.tpo\n";
    s << "extern \"C\" __global__ void __launch_bounds__(" << NT << ", " << minb
      << ") qsim_pass(const __grid_constant__ JP P)\n{\n";
    s << " extern __shared__ double2 sm[];\n";
    s << " const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;\n";
    s << " { const unsigned long long inst = blockIdx.x;\n";
    s << " const unsigned long long base = qdep(inst, TSP)" << (st.jit_block ? " | P.fixbits" : "") << ";\n";
    s << " const unsigned long long gcta = P.rank_bits | base;\n";
    s << " double2 a0";
    for (int i = 1; i < kAmpsPerThread; i++) s << ", a" << i;
    s << ";\n";
    int reg[kAmpsPerThread];
    for (int i = 0; i < kAmpsPerThread; i++) reg[i] = i;
    auto A = [&](int i) { return "a" + std::to_string(reg[i]); };
    // global offsets of a config's lane/warp part and register pair j; tab =
    // TPM (load positions) or TPO (store positions, the next pass's layout)
    auto gaddr = [&](uint64_t c, const char *tab = "TPM") {
        std::ostringstream g;
        g << "(unsigned long long)((lane & 3) << 1)";
        for (int j = 2; j < 5; j++) g << " | (((lane >> " << j << ") & 1) ? " << tab << "[" << nib(c, kLaneNib + j) << "] : 0ULL)";
        for (int j = 0; j < kWarpBits; j++) g << " | (((warp >> " << j << ") & 1) ? " << tab << "[" << nib(c, kWarpNib + j) << "] : 0ULL)";
        return g.str();
    };
    auto roff = [&](uint64_t c, int j, const char *tab = "TPM") {
        std::ostringstream g;
        g << "0ULL";
        for (int b = 0; b < kRegBits - 1; b++)
            if ((j >> b) & 1) g << " | " << tab << "[" << nib(c, 1 + b) << "]";
        return g.str();
    };
    auto smem_z = [&](uint64_t c, const char *tag) {
        s << "  const int zt" << tag << " = ";
        for (int j = 0; j < 5; j++) s << "(((lane >> " << j << ") & 1) << " << nib(c, kLaneNib + j) << ") | ";
        for (int j = 0; j < kWarpBits; j++) s << "(((warp >> " << j << ") & 1) << " << nib(c, kWarpNib + j) << ") | ";
        s << "0;\n";
        s << "  const int zz" << tag << " = zt" << tag << " ^ (((zt" << tag << " >> 3) ^ (zt" << tag << " >> 6) ^ (zt"
          << tag << " >> 9)" << (kTileBits > 12 ? std::string(" ^ (zt") + tag + " >> 12)" : std::string()) << ") & 7);\n";
    };
    auto zreg = [&](uint64_t c, int i) {
        int z = 0;
        for (int b = 0; b < kRegBits; b++)
            if ((i >> b) & 1) z ^= swz_host(1 << nib(c, b));
        return z;
    };
    uint64_t cur = st.pass.cfg0;
    if (st.pass.fresh) {
        // first pass after qsim_init_basis: the tile is the basis state (one 1, else 0)
        s << " {\n  const unsigned long long g0 = P.rank_bits | base | (" << gaddr(cur) << ");\n";
        for (int j = 0; j < kAmpsPerThread / 2; j++)
            s << "  { const unsigned long long g = g0 | (" << roff(cur, j) << "); " << A(2 * j)
              << " = make_double2(g == P.init_phys ? 1.0 : 0.0, 0.0); " << A(2 * j + 1)
              << " = make_double2((g | 1ULL) == P.init_phys ? 1.0 : 0.0, 0.0); }\n";
        s << " }\n";
    } else {
        s << " {\n  const double2 *p = P.st + base + (" << gaddr(cur) << ");\n";
        for (int j = 0; j < kAmpsPerThread / 2; j++)
            s << "  { double x0, x1, x2, x3; asm volatile(\"ld.global.v4.f64 {%0,%1,%2,%3}, [%4];\" : \"=d\"(x0), "
                 "\"=d\"(x1), \"=d\"(x2), \"=d\"(x3) : \"l\"(p + ("
              << roff(cur, j) << "))); " << A(2 * j) << " = make_double2(x0, x1); " << A(2 * j + 1)
              << " = make_double2(x2, x3); }\n";
        s << " }\n";
    }
    // Deferred predicated swaps.  An exact-X op whose predicate depends on the
    // lane, warp or out-of-tile bits (a CNOT/Toffoli target in a register,
    // control elsewhere) cannot be a register renaming.  Instead of 32 selects
    // it is recorded as a pending "flip" of register bit k under a per-thread
    // predicate; pending flips commute with each other and with every op that
    // does not touch bit k, and the next data movement absorbs them: the
    // shared-memory stores of a re-layout or the global stores of the pass
    // write register i to the slot of i ^ (1 << k) (an address XOR).  An op on
    // bit k first materialises the swap (selects).
    struct Flip { int k; std::string pred; };
    std::vector<Flip> flips;
    auto emit_swap = [&](int k, const std::string &pred) {
        s << " { const bool tp = " << pred << ";\n";
        for (int p = 0; p < kAmpsPerThread / 2; p++) {
            const int i0 = ((p >> k) << (k + 1)) | (p & ((1 << k) - 1)), i1 = i0 | (1 << k);
            const std::string x = A(i0), y = A(i1);
            s << "  { const double2 t = " << x << "; " << x << ".x = tp ? " << y << ".x : " << x << ".x; " << x
              << ".y = tp ? " << y << ".y : " << x << ".y; " << y << ".x = tp ? t.x : " << y << ".x; " << y
              << ".y = tp ? t.y : " << y << ".y; }\n";
        }
        s << " }\n";
    };
    auto materialize = [&](uint32_t regbits) {
        for (size_t f = 0; f < flips.size();) {
            if ((regbits >> flips[f].k) & 1) {
                emit_swap(flips[f].k, flips[f].pred);
                flips.erase(flips.begin() + f);
            } else {
                f++;
            }
        }
    };
    // per-thread XOR of the slot index of every register under the pending flips
    auto flip_mask = [&](const char *name, const char *type, std::function<std::string(int)> unit) {
        s << "  const " << type << " " << name << " = 0";
        for (const Flip &f : flips) s << " ^ ((" << f.pred << ") ? (" << type << ")(" << unit(f.k) << ") : (" << type << ")0)";
        s << ";\n";
        flips.clear();
    };
    bool u4_heavy = false;
    {
        double w4 = 0, w2 = 0;
        for (const KOp &op : st.ops) {
            if (op.code == OPC_U4) w4 += 16;
            else if (op.code == OPC_U2) w2 += 8;
            else if (op.code == OPC_U2R) w2 += 4;
        }
        u4_heavy = w4 >= 2 * w2;
    }
    // Phase runs (OPC_PHASE_ACC), see PhasePlan: inline terms go to integer
    // angle accumulators mo_S, one per monomial S of the register bits (plan.h
    // PhaseRunPlan), flushed lazily; const / uniform / thread terms arrive as
    // complex factors.
    const PhasePlan pp = phase_plan(st);
    uint32_t live = 0;
    if (pp.inl_used) {
        s << " unsigned long long";
        bool first_decl = true;
        for (uint32_t S = 0; S < (uint32_t)kAmpsPerThread; S++)
            if ((pp.inl_used >> S) & 1) { s << (first_decl ? " mo" : ", mo") << S << " = 0"; first_decl = false; }
        s << ";\n";
    }
    int epoch[kAmpsPerThread] = {0};
    const int NS = (int)pp.slot_S.size(), NW = kPassThreads / 32;
    if (NS) {
        // CTA-uniform terms: the warps split the ops, sum per slot, reduce
        // through shared memory once per tile; utc[k] = e^{i sum of slot k}
        s << " __shared__ unsigned long long uw[" << NW * NS << "];\n __shared__ double2 utc[" << NS << "];\n";
        s << " {\n";
        for (int k = 0; k < NS; k++) s << "  unsigned long long u" << k << " = 0;\n";
        s << "  switch (warp) {\n";
        int next_w = 0;
        std::vector<std::vector<size_t>> by_warp(NW);
        for (size_t o = 0; o < st.ops.size(); o++)
            if (!pp.uterms[o].empty()) { by_warp[next_w].push_back(o); next_w = (next_w + 1) % NW; }
        for (int w = 0; w < NW; w++) {
            s << "  case " << w << ": {\n";
            for (size_t o : by_warp[w]) {
                const std::string M = "P.m[" + std::to_string(m_idx[o]) + "]";
                s << "   { const unsigned long long K = ((gcta & P.out[" << out_idx[o] << "][0]) == P.out[" << out_idx[o]
                  << "][1]) ? (unsigned long long)__double_as_longlong(" << M << "[" << m_col[o] << "]) : 0ULL;";
                for (auto &t : pp.uterms[o]) s << " u" << t.first << (t.second < 0 ? " -= K;" : " += K;");
                s << " }\n";
            }
            s << "   break; }\n";
        }
        s << "  }\n  if (lane == 0) {";
        for (int k = 0; k < NS; k++) s << " uw[warp * " << NS << " + " << k << "] = u" << k << ";";
        s << " }\n }\n __syncthreads();\n";
        s << " for (int k = warp; k < " << NS << "; k += " << NW << ") {\n"
             "  unsigned long long v = lane < " << NW << " ? uw[lane * " << NS << " + k] : 0ULL;\n";
        for (int d = 1; d < NW; d <<= 1) s << "  v += __shfl_xor_sync(0xffffffffu, v, " << d << ");\n";
        s << "  if (lane == 0) utc[k] = qexp(v, P.ptab);\n }\n __syncthreads();\n";
    }
    auto cmul = [&](const std::string &a, const std::string &b, const std::string &out) {  // out = a * b
        s << "  const double2 " << out << " = make_double2(fma(" << a << ".x, " << b << ".x, -" << a << ".y * " << b
          << ".y), fma(" << a << ".x, " << b << ".y, " << a << ".y * " << b << ".x));\n";
        fpc += 4;
    };
    auto flush = [&](uint32_t F) {
        F &= live;
        if (!F) return;
        s << " { // flush monomials 0x" << std::hex << F << std::dec << "\n";
        // factor f_S of every flushed monomial: the product of its parts
        for (uint32_t S = 0; S < (uint32_t)kAmpsPerThread; S++) {
            if (!((F >> S) & 1)) continue;
            const auto key = std::make_pair(S, epoch[S]);
            std::vector<std::string> parts;
            if (pp.inl.count(key)) {
                s << "  const double2 ei" << S << " = qexp(mo" << S << ", P.ptab); mo" << S << " = 0;\n";
                fpc += kQexpOps;
                parts.push_back("ei" + std::to_string(S));
            }
            auto ct = pp.cslot_of.find(key);
            if (ct != pp.cslot_of.end()) {
                const int k = ct->second, row = L.c_row + k / 4, col = 2 * (k % 4);
                s << "  const double2 ec" << S << " = make_double2(P.m[" << row << "][" << col << "], P.m[" << row << "]["
                  << col + 1 << "]);\n";
                parts.push_back("ec" + std::to_string(S));
            }
            auto it = pp.slot_of.find(key);
            if (it != pp.slot_of.end()) parts.push_back("utc[" + std::to_string(it->second) + "]");
            auto jt = pp.tslot_of.find(key);
            if (jt != pp.tslot_of.end()) {
                s << "  const double2 et" << S << " = __ldg(reinterpret_cast<const double2 *>(P.ttab) + "
                  << jt->second * kPassThreads << " + threadIdx.x);\n";
                parts.push_back("et" + std::to_string(S));
            }
            std::string f = parts.empty() ? std::string("make_double2(1.0, 0.0)") : parts[0];
            for (size_t q = 1; q < parts.size(); q++) {
                const std::string nf = "f" + std::to_string(S) + "_" + std::to_string(q);
                cmul(f, parts[q], nf);
                f = nf;
            }
            s << "  const double2 em" << S << " = " << f << ";\n";
            epoch[S]++;
        }
        // apply: per monomial (B: every amplitude times each of its factors)
        // or per distinct register key (A: the product of the key's factors
        // once, then one multiply per amplitude), the cheaper
        auto key_of = [&](uint32_t i) {
            uint32_t key = 0;
            for (uint32_t S = 0; S < (uint32_t)kAmpsPerThread; S++)
                if (((F >> S) & 1) && (S & i) == S) key |= 1u << S;
            return key;
        };
        std::vector<uint32_t> keys;
        int nregs = 0;
        double costA = 0, costB = 0;
        for (uint32_t i = 0; i < (uint32_t)kAmpsPerThread; i++) {
            const uint32_t key = key_of(i);
            if (!key) continue;
            nregs++;
            costB += 4 * __builtin_popcount(key);
            if (std::find(keys.begin(), keys.end(), key) == keys.end()) {
                keys.push_back(key);
                costA += 4 * (__builtin_popcount(key) - 1);
            }
        }
        costA += 4 * nregs;
        auto mul = [&](const std::string &e, const std::string &v) {
            s << "  { const double p1 = -" << e << ".y * " << v << ".y, p2 = " << e << ".y * " << v << ".x; " << v
              << ".x = fma(" << e << ".x, " << v << ".x, p1); " << v << ".y = fma(" << e << ".x, " << v
              << ".y, p2); }\n";
            fpc += 4;
        };
        if (costA < costB) {
            std::vector<char> emitted(keys.size(), 0);
            for (uint32_t i = 0; i < (uint32_t)kAmpsPerThread; i++) {
                const uint32_t key = key_of(i);
                if (!key) continue;
                const size_t k = std::find(keys.begin(), keys.end(), key) - keys.begin();
                const std::string ek = "ek" + std::to_string(k);
                if (!emitted[k]) {
                    std::string f;
                    int q = 0;
                    for (uint32_t S = 0; S < (uint32_t)kAmpsPerThread; S++) {
                        if (!((key >> S) & 1)) continue;
                        const std::string e = "em" + std::to_string(S);
                        if (f.empty()) f = e;
                        else {
                            const std::string nf = ek + "_" + std::to_string(q++);
                            cmul(f, e, nf);
                            f = nf;
                        }
                    }
                    s << "  const double2 " << ek << " = " << f << ";\n";
                    emitted[k] = 1;
                }
                mul(ek, A(i));
            }
        } else {
            for (uint32_t i = 0; i < (uint32_t)kAmpsPerThread; i++)
                for (uint32_t S = 0; S < (uint32_t)kAmpsPerThread; S++)
                    if (((F >> S) & 1) && (S & i) == S) mul("em" + std::to_string(S), A(i));
        }
        s << " }\n";
        live &= ~F;
    };
    // Re-layout barriers (QSIM_JIT_BAR, A/B switch): 0 = a CTA barrier after
    // the stores and after the loads; 1 = the second one deferred to just
    // before the next re-layout's stores (warps start computing as soon as
    // their own loads are done); 2 = as 1, and each barrier spans only the
    // warps that exchange data: those equal on the warp slots whose tile bit
    // stays put (kept slot w2: bar 1/2 over 4 warps, w1: 3/4, w0: 5/6; all
    // kept: the warp alone); 3 = as 2 with the w2 groups only.  Warp w runs
    // on SM sub-partition w % 4, so a w2 group spans all four and the two
    // groups interleave their FP64 and shared-memory phases on each; a w0 or
    // w1 group sits on two sub-partitions and leaves the other two's FP64
    // pipes idle while it re-lays out (measured slower).  Every warp runs the
    // same barrier sequence and a barrier id always names the same warp set,
    // so named barriers cannot mix.
    const int bar_mode = env_int("QSIM_JIT_BAR", kJitBarDefault);
    int n_trans = 0;
    uint32_t prev_keep = 0;
    auto group_bar = [&](uint32_t keep) -> std::string {
        const uint32_t all = (1u << kWarpBits) - 1;
        if (kWarpBits != 3 || keep == 0) return BAR;
        if (keep == all) return "__syncwarp();";
        if (bar_mode >= 3 && !((keep >> 2) & 1)) return BAR;
        const int j = (keep >> 2) & 1 ? 2 : (keep >> 1) & 1 ? 1 : 0;
        const int id0 = j == 2 ? 1 : j == 1 ? 3 : 5;
        return "asm volatile(\"bar.sync %0, 128;\" :: \"r\"(" + std::to_string(id0) + " + ((warp >> " +
               std::to_string(j) + ") & 1)) : \"memory\");";
    };
    int n_had = 0;
    for (const KOp &op : st.ops) n_had += jit_hadamard(op);
    if (n_had) s << " double hs = 1.0;  // product of the Hadamard-form scales applied so far\n";
    for (size_t o = 0; o < st.ops.size(); o++) {
        const KOp &op = st.ops[o];
        if (op.code == OPC_TRANS) {
            flush(live);
            s << " {\n";
            // warp slots whose tile bit stays put through this re-layout: the
            // warps that differ only there never exchange data
            uint32_t keep = 0;
            for (int j = 0; j < kWarpBits; j++)
                if (nib(cur, kWarpNib + j) == nib(op.cfg, kWarpNib + j)) keep |= 1u << j;
            if (bar_mode >= 1 && n_trans > 0)  // WAR: the previous re-layout's reads of what we overwrite
                s << "  " << group_bar(bar_mode >= 2 ? keep & prev_keep : 0) << "\n";
            smem_z(cur, "a");
            const uint64_t cfa = cur;
            flip_mask("zfa", "int", [&](int k) { return std::to_string(swz_host(1 << nib(cfa, k))); });
            for (int i = 0; i < kAmpsPerThread; i++) s << "  sm[(zza ^ zfa) ^ " << zreg(cur, i) << "] = " << A(i) << ";\n";
            s << "  " << (bar_mode >= 2 ? group_bar(keep) : BAR) << "\n";  // RAW
            cur = op.cfg;
            smem_z(cur, "b");
            for (int i = 0; i < kAmpsPerThread; i++) s << "  " << A(i) << " = sm[zzb ^ " << zreg(cur, i) << "];\n";
            if (bar_mode == 0) s << "  " << BAR << "\n";
            s << " }\n";
            prev_keep = keep;
            n_trans++;
            continue;
        }
        if (op.code == OPC_PHASE_FLUSH) continue;  // lazy flush (above)
        if (op.code == OPC_DATA) continue;  // rows 1..3 of the preceding OPC_U4
        if (op.code == OPC_U4 && !fm.u4) {
            // direct form: each output one 8-long FMA chain for re and for im
            const int k = op.k, k2 = (int)op.cfg;
            flush(touching((1u << k) | (1u << k2)));
            materialize((1u << k) | (1u << k2));
            s << " { // op " << o << " U4 (" << k << "," << k2 << ")\n";
            const int il = env_int("QSIM_JIT_U4IL", u4_heavy ? 2 : 1);
            for (int p0 = 0; p0 < kAmpsPerThread / 4; p0 += il) {
                s << "  {\n";
                std::vector<std::array<int, 4>> gi;
                for (int p = p0; p < p0 + il && p < kAmpsPerThread / 4; p++) {
                    int i0 = ((p >> k) << (k + 1)) | (p & ((1 << k) - 1));
                    i0 = ((i0 >> k2) << (k2 + 1)) | (i0 & ((1 << k2) - 1));
                    gi.push_back({i0, i0 | (1 << k), i0 | (1 << k2), i0 | (1 << k) | (1 << k2)});
                }
                for (size_t g = 0; g < gi.size(); g++)
                    for (int c = 0; c < 4; c++) s << "   const double2 x" << g << "_" << c << " = " << A(gi[g][c]) << ";\n";
                for (int c = 0; c < 4; c++)
                    for (size_t g = 0; g < gi.size(); g++)
                        for (int r = 0; r < 4; r++) {
                            const std::string R = "P.m[" + std::to_string(m_idx[o] + r) + "]";
                            const std::string re = "re" + std::to_string(g) + "_" + std::to_string(r),
                                              im = "im" + std::to_string(g) + "_" + std::to_string(r),
                                              x = "x" + std::to_string(g) + "_" + std::to_string(c);
                            if (c == 0)
                                s << "   double " << re << " = " << R << "[0] * " << x << ".x, " << im << " = " << R
                                  << "[0] * " << x << ".y; " << re << " = fma(-" << R << "[1], " << x << ".y, " << re
                                  << "); " << im << " = fma(" << R << "[1], " << x << ".x, " << im << ");\n";
                            else
                                s << "   " << re << " = fma(" << R << "[" << 2 * c << "], " << x << ".x, " << re << "); "
                                  << re << " = fma(-" << R << "[" << 2 * c + 1 << "], " << x << ".y, " << re << "); "
                                  << im << " = fma(" << R << "[" << 2 * c << "], " << x << ".y, " << im << "); " << im
                                  << " = fma(" << R << "[" << 2 * c + 1 << "], " << x << ".x, " << im << ");\n";
                        }
                for (size_t g = 0; g < gi.size(); g++)
                    for (int r = 0; r < 4; r++)
                        s << "   " << A(gi[g][r]) << " = make_double2(re" << g << "_" << r << ", im" << g << "_" << r << ");\n";
                s << "  }\n";
            }
            s << " }\n";
            fpc += 16.0 * kAmpsPerThread;
            continue;
        }
        if (op.code == OPC_U4) {
            // 3M form of the complex 4x4: with U = A + iB and
            // x = p + iq, Re(Ux) = A(p+q) - (A+B)q, Im(Ux) = A(p+q) + (B-A)p.
            // Per output row 12 FP64 ops (4 for K = A(p+q), 4 + 4 continuing
            // it) plus one add per amplitude for s = p + q: 13 per amplitude
            // instead of 16.  The parameter rows hold A, -(A+B) and B-A
            // (jit_pack_params).
            const int k = op.k, k2 = (int)op.cfg;
            flush(touching((1u << k) | (1u << k2)));
            materialize((1u << k) | (1u << k2));
            s << " { // op " << o << " U4 (" << k << "," << k2 << ")\n";
            // groups whose rows are emitted interleaved.  The 3M form holds three
            // copies of a group's inputs: on passes dominated by blocks one group
            // at a time (config 2: 0.331 vs 0.352 ms/pass with 2), else two
            // (chain circuits: 2 slightly ahead)
            const int il = env_int("QSIM_JIT_U4IL", u4_heavy ? 1 : 2);
            auto C = [&](int table, int r, int c) {
                const int idx = table * 16 + r * 4 + c;
                return "P.m[" + std::to_string(m_idx[o] + (idx >> 3)) + "][" + std::to_string(idx & 7) + "]";
            };
            for (int p0 = 0; p0 < kAmpsPerThread / 4; p0 += il) {
                s << "  {\n";
                std::vector<std::array<int, 4>> gi;
                for (int p = p0; p < p0 + il && p < kAmpsPerThread / 4; p++) {
                    int i0 = ((p >> k) << (k + 1)) | (p & ((1 << k) - 1));
                    i0 = ((i0 >> k2) << (k2 + 1)) | (i0 & ((1 << k2) - 1));
                    gi.push_back({i0, i0 | (1 << k), i0 | (1 << k2), i0 | (1 << k) | (1 << k2)});
                }
                auto nm = [](const char *v, size_t g, int r) { return std::string(v) + std::to_string(g) + "_" + std::to_string(r); };
                for (size_t g = 0; g < gi.size(); g++)
                    for (int c = 0; c < 4; c++)
                        s << "   const double2 " << nm("x", g, c) << " = " << A(gi[g][c]) << "; const double " << nm("s", g, c)
                          << " = " << nm("x", g, c) << ".x + " << nm("x", g, c) << ".y;\n";
                // row by row (an output row is written back as soon as it is
                // formed: x and s are the only long-lived copies)
                for (int r = 0; r < 4; r++) {
                    for (size_t g = 0; g < gi.size(); g++) {
                        const std::string kk = nm("k", g, r), re = nm("re", g, r), im = nm("im", g, r);
                        s << "   { double " << kk << " = " << C(0, r, 0) << " * " << nm("s", g, 0) << ";";
                        for (int c = 1; c < 4; c++) s << " " << kk << " = fma(" << C(0, r, c) << ", " << nm("s", g, c) << ", " << kk << ");";
                        s << "\n     double " << re << " = " << kk << ", " << im << " = " << kk << ";";
                        for (int c = 0; c < 4; c++) {
                            const std::string x = nm("x", g, c);
                            s << " " << re << " = fma(" << C(1, r, c) << ", " << x << ".y, " << re << "); " << im << " = fma("
                              << C(2, r, c) << ", " << x << ".x, " << im << ");";
                        }
                        s << "\n     " << A(gi[g][r]) << " = make_double2(" << re << ", " << im << "); }\n";
                    }
                }
                s << "  }\n";
            }
            s << " }\n";
            fpc += 13.0 * kAmpsPerThread;
            continue;
        }
        const bool plw = op.mlane || op.mwarp;  // thread-dependent predicate
        const bool pout = op.mout != 0;         // CTA-uniform predicate
        std::ostringstream pr;
        pr << "true";
        if (op.mlane) pr << " && ((lane & " << op.mlane << ") == " << op.vlane << ")";
        if (op.mwarp) pr << " && ((warp & " << op.mwarp << ") == " << op.vwarp << ")";
        if (pout) pr << " && ((gcta & P.out[" << out_idx[o] << "][0]) == P.out[" << out_idx[o] << "][1])";
        const bool sel = plw || (pout && op.code == OPC_XS);  // select-based (no branch)
        const bool is_phase = op.code == OPC_PHASE || op.code == OPC_PHASE_ACC;
        if (!is_phase) flush(touching(1u << op.k));
        if (op.code == OPC_XS && sel && op.mreg == 0) {  // defer (see Flip)
            flips.push_back({op.k, pr.str()});
            continue;
        }
        materialize(op.mreg | (is_phase ? 0u : 1u << op.k));
        if (!pp.uterms[o].empty() || !pp.tterms[o].empty() || !pp.cterms[o].empty()) {  // a factor at the flush
            const uint32_t O = op.mreg & op.vreg, Z = op.mreg & ~op.vreg;
            for (uint32_t T = Z;; T = (T - 1) & Z) {
                live |= 1u << (O | T);
                if (!T) break;
            }
            continue;
        }
        s << " { // op " << o << " code " << op.code << "\n";
        // FP64 ops per thread are counted as expected values: a branch on a
        // CTA-uniform predicate runs in 2^-|mout| of the tiles
        const double w = pout && !sel ? std::ldexp(1.0, -__builtin_popcountll(op.mout)) : 1.0;
        if (plw || pout) s << "  const bool tp = " << pr.str() << ";\n";
        if (pout && !sel) s << "  if (tp) {\n";
        const std::string M = "P.m[" + std::to_string(m_idx[o]) + "]";
        if (op.code == OPC_PHASE_ACC) {
            s << "  const unsigned long long K = " << (sel ? "tp ? " : "") << "(unsigned long long)__double_as_longlong("
              << M << "[" << m_col[o] << "])" << (sel ? " : 0ULL" : "") << ";\n";
            const uint32_t O = op.mreg & op.vreg, Z = op.mreg & ~op.vreg;
            for (uint32_t T = Z;; T = (T - 1) & Z) {
                s << "  mo" << (O | T) << (__builtin_popcount(T) & 1 ? " -= K;\n" : " += K;\n");
                live |= 1u << (O | T);
                if (!T) break;
            }
        } else if (op.code == OPC_PHASE) {
            for (int i = 0; i < kAmpsPerThread; i++) {
                if ((i & op.mreg) != op.vreg) continue;
                const std::string v = A(i);
                const std::string F0 = M + "[" + std::to_string(m_col[o]) + "]",
                                  F1 = M + "[" + std::to_string(m_col[o] + 1) + "]";
                s << "  { const double p1 = -" << F1 << " * " << v << ".y, p2 = " << F1 << " * " << v << ".x; ";
                if (sel)
                    s << "const double nx = fma(" << F0 << ", " << v << ".x, p1), ny = fma(" << F0 << ", " << v
                      << ".y, p2); " << v << ".x = tp ? nx : " << v << ".x; " << v << ".y = tp ? ny : " << v << ".y; }\n";
                else
                    s << v << ".x = fma(" << F0 << ", " << v << ".x, p1); " << v << ".y = fma(" << F0 << ", " << v
                      << ".y, p2); }\n";
                fpc += 4 * w;
            }
        } else if (jit_hadamard(op)) {
            const int k = op.k;
            for (int p = 0; p < kAmpsPerThread / 2; p++) {
                const int i0 = ((p >> k) << (k + 1)) | (p & ((1 << k) - 1)), i1 = i0 | (1 << k);
                const std::string x = A(i0), y = A(i1);
                s << "  { const double2 t = " << x << "; " << x << ".x = t.x + " << y << ".x; " << x << ".y = t.y + "
                  << y << ".y; " << y << ".x = t.x - " << y << ".x; " << y << ".y = t.y - " << y << ".y; }\n";
                fpc += 4;
            }
            s << "  hs *= " << M << "[0];\n";
            fpc += 1;
        } else {
            const int k = op.k;
            for (int p = 0; p < kAmpsPerThread / 2; p++) {
                const int i0 = ((p >> k) << (k + 1)) | (p & ((1 << k) - 1)), i1 = i0 | (1 << k);
                if ((i0 & (int)op.mreg) != (int)op.vreg) continue;
                const std::string x = A(i0), y = A(i1);
                if (op.code == OPC_XS) {
                    if (sel)
                        s << "  { const double2 t = " << x << "; " << x << ".x = tp ? " << y << ".x : " << x << ".x; "
                          << x << ".y = tp ? " << y << ".y : " << x << ".y; " << y << ".x = tp ? t.x : " << y << ".x; "
                          << y << ".y = tp ? t.y : " << y << ".y; }\n";
                    else
                        std::swap(reg[i0], reg[i1]);
                    continue;
                }
                if (op.code == OPC_U2 && fm.u2) {
                    // 3M form (as OPC_U4): s = p + q, k_r = sum_c A_rc s_c,
                    // Re = k_r - sum_c (A+B)_rc q_c, Im = k_r + sum_c (B-A)_rc p_c;
                    // 14 FP64 ops per pair instead of 16.  Parameter row pair:
                    // [0..3] A, [4..7] -(A+B), [8..11] B-A (jit_pack_params).
                    auto G = [&](int idx) {
                        return "P.m[" + std::to_string(m_idx[o] + (idx >> 3)) + "][" + std::to_string(idx & 7) + "]";
                    };
                    s << "  { const double s0 = " << x << ".x + " << x << ".y, s1 = " << y << ".x + " << y << ".y; "
                      << "const double k0 = fma(" << G(1) << ", s1, " << G(0) << " * s0), k1 = fma(" << G(3) << ", s1, "
                      << G(2) << " * s0); "
                      << "const double n0 = fma(" << G(4) << ", " << x << ".y, fma(" << G(5) << ", " << y << ".y, k0)); "
                      << "const double n1 = fma(" << G(8) << ", " << x << ".x, fma(" << G(9) << ", " << y << ".x, k0)); "
                      << "const double n2 = fma(" << G(6) << ", " << x << ".y, fma(" << G(7) << ", " << y << ".y, k1)); "
                      << "const double n3 = fma(" << G(10) << ", " << x << ".x, fma(" << G(11) << ", " << y << ".x, k1)); ";
                    if (sel)
                        s << x << ".x = tp ? n0 : " << x << ".x; " << x << ".y = tp ? n1 : " << x << ".y; " << y
                          << ".x = tp ? n2 : " << y << ".x; " << y << ".y = tp ? n3 : " << y << ".y; }\n";
                    else
                        s << x << ".x = n0; " << x << ".y = n1; " << y << ".x = n2; " << y << ".y = n3; }\n";
                    fpc += 14 * w;
                    continue;
                }
                // OPC_U2R, or OPC_U2 in the direct form
                std::ostringstream pp;
                if (op.code == OPC_U2R) {
                    pp << "const double p1 = " << M << "[2] * " << y << ".x, p2 = " << M << "[2] * " << y << ".y, p3 = "
                       << M << "[4] * " << x << ".x, p4 = " << M << "[4] * " << x << ".y; ";
                } else {
                    pp << "const double p1 = fma(-" << M << "[1], " << x << ".y, fma(" << M << "[2], " << y << ".x, -"
                       << M << "[3] * " << y << ".y)); const double p2 = fma(" << M << "[1], " << x << ".x, fma(" << M
                       << "[2], " << y << ".y, " << M << "[3] * " << y << ".x)); const double p3 = fma(" << M << "[4], "
                       << x << ".x, fma(-" << M << "[5], " << x << ".y, -" << M << "[7] * " << y
                       << ".y)); const double p4 = fma(" << M << "[4], " << x << ".y, fma(" << M << "[5], " << x
                       << ".x, " << M << "[7] * " << y << ".x)); ";
                }
                s << "  { " << pp.str();
                const char *dst[4] = {".x", ".y", ".x", ".y"};
                const std::string xs[4] = {x, x, y, y};
                const char *mm[4] = {"[0]", "[0]", "[6]", "[6]"};
                const char *pv[4] = {"p1", "p2", "p3", "p4"};
                if (sel) {
                    for (int q = 0; q < 4; q++)
                        s << "const double n" << q << " = fma(" << M << mm[q] << ", " << xs[q] << dst[q] << ", " << pv[q]
                          << "); ";
                    for (int q = 0; q < 4; q++)
                        s << xs[q] << dst[q] << " = tp ? n" << q << " : " << xs[q] << dst[q] << "; ";
                } else {
                    for (int q = 0; q < 4; q++)
                        s << xs[q] << dst[q] << " = fma(" << M << mm[q] << ", " << xs[q] << dst[q] << ", " << pv[q]
                          << "); ";
                }
                s << "}\n";
                fpc += (op.code == OPC_U2R ? 8 : 16) * w;
            }
        }
        if (pout && !sel) s << "  }\n";
        s << " }\n";
    }
    flush(live);
    if (n_had) {
        for (int i = 0; i < kAmpsPerThread; i++) s << " " << A(i) << ".x *= hs; " << A(i) << ".y *= hs;\n";
        fpc += 2 * kAmpsPerThread;
    }
    materialize(1);  // register bit 0 lies inside one 256-bit store
    std::ostringstream ro;  // the readout variant's reduction, emitted after the stores
    if (st.jit_readout) {
        // <Q_i> fused into the pass: per tile bit t the sum of |a|^2 over the
        // tile's amplitudes with bit t set, and the tile total (index 12),
        // in a fixed order (deterministic).  Register bit j holds tile bit
        // nib(cur, j), except that a pending flip of bit j (stored with the
        // slot address XORed, see Flip) exchanges its 0 and 1 halves.
        // (emitted after the stores, so that they leave before the reduction's
        // shuffles and barrier; only the pending flips' predicates, which the
        // store consumes, are evaluated here)
        const int NWR = kPassThreads / 32;
        ro << " {\n  __shared__ double rsum[" << NWR * (kTileBits + 1) << "];\n";
        for (int i = 0; i < kAmpsPerThread; i++)
            ro << "  const double rp" << i << " = fma(" << A(i) << ".x, " << A(i) << ".x, " << A(i) << ".y * " << A(i)
              << ".y);\n";
        // fixed-order tree sums over a register subset
        auto tree = [&](std::vector<int> idx) {
            std::vector<std::string> t;
            for (int i : idx) t.push_back("rp" + std::to_string(i));
            while (t.size() > 1) {
                std::vector<std::string> u;
                for (size_t k = 0; k + 1 < t.size(); k += 2) u.push_back("(" + t[k] + " + " + t[k + 1] + ")");
                if (t.size() & 1) u.push_back(t.back());
                t.swap(u);
            }
            return t.empty() ? std::string("0.0") : t[0];
        };
        std::vector<int> all;
        for (int i = 0; i < kAmpsPerThread; i++) all.push_back(i);
        ro << "  const double rtot = " << tree(all) << ";\n";
        std::vector<std::string> val(kTileBits);
        for (int j = 0; j < kRegBits; j++) {
            std::vector<int> one, zero;
            for (int i = 0; i < kAmpsPerThread; i++) ((i >> j) & 1 ? one : zero).push_back(i);
            std::string fp = "false";
            for (const Flip &f : flips)
                if (f.k == j) fp = "(" + fp + ") != (" + f.pred + ")";
            s << " const bool rf" << j << " = " << fp << ";\n";
            ro << "  const double rb" << j << " = rf" << j << " ? " << tree(zero) << " : " << tree(one) << ";\n";
            val[nib(cur, j)] = "rb" + std::to_string(j);
        }
        for (int j = 0; j < 5; j++) val[nib(cur, kLaneNib + j)] = "(((lane >> " + std::to_string(j) + ") & 1) ? rtot : 0.0)";
        for (int j = 0; j < kWarpBits; j++)
            val[nib(cur, kWarpNib + j)] = "(((warp >> " + std::to_string(j) + ") & 1) ? rtot : 0.0)";
        val.push_back("rtot");
        for (int t = 0; t <= kTileBits; t++) {
            ro << "  { double v = " << val[t] << ";";
            for (int d = 16; d > 0; d >>= 1) ro << " v += __shfl_xor_sync(0xffffffffu, v, " << d << ");";
            ro << " if (lane == 0) rsum[warp * " << kTileBits + 1 << " + " << t << "] = v; }\n";
        }
        ro << "  __syncthreads();\n  if (threadIdx.x < " << kTileBits + 1 << ") { double v = rsum[threadIdx.x];";
        ro << " for (int w = 1; w < " << NWR << "; w++) v += rsum[w * " << kTileBits + 1 << " + threadIdx.x];";
        ro << " P.red[(unsigned long long)blockIdx.x * " << kTileBits + 1 << " + threadIdx.x] = v; }\n }\n";
        // |a|^2, the total, both halves per register bit, the warp butterflies
        fpc += 2.0 * kAmpsPerThread + (kAmpsPerThread - 1) + kRegBits * 2 * (kAmpsPerThread / 2 - 1) +
               (kTileBits + 1) * 5;
    }
    s << " {\n  double2 *p = P.st + base + (" << gaddr(cur, "TPO") << ");\n";
    {
        const uint64_t cfs = cur;
        flip_mask("gf", "unsigned long long", [&](int k) { return "TPO[" + std::to_string(nib(cfs, k)) + "]"; });
    }
    for (int j = 0; j < kAmpsPerThread / 2; j++)
        s << "  asm volatile(\"st.global.v4.f64 [%0], {%1,%2,%3,%4};\" :: \"l\"(p + ((" << roff(cur, j, "TPO") << ") ^ gf)), \"d\"("
          << A(2 * j) << ".x), \"d\"(" << A(2 * j) << ".y), \"d\"(" << A(2 * j + 1) << ".x), \"d\"(" << A(2 * j + 1)
          << ".y) : \"memory\");\n";
    s << " }\n";
    s << ro.str();
    s << " }\n";
    // Phase offset between the two CTAs an SM runs.  CTAs of the first wave
    // start together and, running identical code, stay in step: both re-
    // layout (shared-memory bound) at the same time and both compute (FP64
    // bound) at the same time.  The first-wave CTAs of slot 0 (blockIdx <
    // SM count: the SM's slot-1 CTA is blockIdx + SM count) finish late by
    // P.desync ns, so every later CTA on the SM starts out of step with its
    // neighbour.  Branch-free (a branch here changes the kernel's uniform-
    // register allocation); P.desync = SM count << 32 | ns, 0 = off.
    s << " { const unsigned long long d = P.desync; __nanosleep(blockIdx.x < (unsigned)(d >> 32) ? (unsigned)d : 0u); }\n";
    s << "}\n";
    const int NTS = (int)pp.tslot_S.size();
    if (NTS) {
        // companion kernel: the per-thread phase slots, once per launch (not per tile)
        s << "extern \"C\" __global__ void __launch_bounds__(" << kPassThreads
          << ") qsim_pass_tab(const __grid_constant__ JP P)\n{\n"
             " const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;\n";
        for (int k = 0; k < NTS; k++) s << " unsigned long long t" << k << " = 0;\n";
        for (size_t o = 0; o < st.ops.size(); o++) {
            if (pp.tterms[o].empty()) continue;
            const KOp &op = st.ops[o];
            s << " { const unsigned long long K = (true";
            if (op.mlane) s << " && ((lane & " << op.mlane << ") == " << op.vlane << ")";
            if (op.mwarp) s << " && ((warp & " << op.mwarp << ") == " << op.vwarp << ")";
            s << ") ? (unsigned long long)__double_as_longlong(P.m[" << m_idx[o] << "][" << m_col[o] << "]) : 0ULL;";
            for (auto &t : pp.tterms[o]) s << " t" << t.first << (t.second < 0 ? " -= K;" : " += K;");
            s << " }\n";
        }
        // e^{i sum} per slot and thread (2 u64 per entry)
        for (int k = 0; k < NTS; k++)
            s << " reinterpret_cast<double2 *>(P.ttab)[" << k * kPassThreads << " + threadIdx.x] = qexp(t" << k
              << ", P.ptab);\n";
        s << "}\n";
    }
    JitPass jp;
    jp.src = s.str();
    jp.param_bytes = L.bytes;
    jp.n_tslots = NTS;
    jp.fp64_per_thread = fpc;
    return jp;
}

void jit_pack_params(const Step &st, void *state, uint64_t rank_bits, std::vector<uint8_t> &buf)
{
    std::vector<int> out_idx, m_idx, m_col;
    Layout L = layout_of(st, out_idx, m_idx, m_col);
    const Forms fm = forms_of(st);
    buf.assign(L.bytes, 0);
    uint8_t *b = buf.data();
    std::memcpy(b + 0, &state, 8);
    std::memcpy(b + 8, &rank_bits, 8);
    const uint64_t desync = 0;  // jit_set_desync
    std::memcpy(b + 16, &desync, 8);
    const void *tab = jit_phase_table();
    std::memcpy(b + 24, &tab, 8);
    std::memcpy(b + kOffInit, &st.pass.init_phys, 8);
    for (int t = kTileBits; t < kTileBits + kMaxFix; t++) {
        const int32_t none = 62;  // no-op insertion (see qdep)
        std::memcpy(b + kOffTs + 4 * t, &none, 4);
    }
    for (int t = 0; t < kTileBits; t++) {
        const uint64_t m = 1ULL << st.pass.tp[t];
        std::memcpy(b + kOffTpm + 8 * t, &m, 8);
        std::memcpy(b + kOffTs + 4 * t, &st.pass.tile_sorted[t], 4);
        const uint64_t mo = 1ULL << st.pass.tp_out[t];
        std::memcpy(b + kOffTpo + 8 * t, &mo, 8);
    }
    {
        // const phase terms: e^{2 pi i c / 2^64} per (monomial, epoch) slot, c
        // the wrapped sum of the slot's unpredicated angles (phase_plan)
        const PhasePlan pp = phase_plan(st);
        std::vector<uint64_t> acc(pp.cslot_S.size(), 0);
        for (size_t o = 0; o < st.ops.size(); o++)
            for (auto &t : pp.cterms[o]) acc[t.first] += t.second < 0 ? (uint64_t)0 - st.ops[o].cfg : st.ops[o].cfg;
        for (size_t k = 0; k < acc.size(); k++) {
            const long double turns = (long double)(int64_t)acc[k] / 18446744073709551616.0L;  // in [-1/2, 1/2)
            const long double a = 2.0L * 3.141592653589793238462643383279502884L * turns;
            const double f[2] = {(double)cosl(a), (double)sinl(a)};
            std::memcpy(b + L.off_m + 64 * (L.c_row + k / 4) + 16 * (k % 4), f, 16);
        }
    }
    for (size_t o = 0; o < st.ops.size(); o++) {
        const KOp &op = st.ops[o];
        if (out_idx[o] >= 0) {
            std::memcpy(b + L.off_out + 16 * out_idx[o], &op.mout, 8);
            std::memcpy(b + L.off_out + 16 * out_idx[o] + 8, &op.vout, 8);
        }
        if (m_idx[o] >= 0) {
            uint8_t *row = b + L.off_m + 64 * m_idx[o];
            if (op.code == OPC_PHASE_ACC) std::memcpy(row + 8 * m_col[o], &op.cfg, 8);       // angle
            else if (op.code == OPC_PHASE) std::memcpy(row + 8 * m_col[o], op.m, 16);       // f
            else if ((op.code == OPC_U4 && fm.u4) || (op.code == OPC_U2 && fm.u2)) {
                // 3M constants of U = A + iB: A, -(A+B), B-A (row-major entries)
                const int dim = op.code == OPC_U4 ? 4 : 2;
                double c[48];
                for (int r = 0; r < dim; r++)
                    for (int q = 0; q < dim; q++) {
                        const double *m = op.code == OPC_U4 ? st.ops[o + r].m + 2 * q : op.m + 2 * (r * 2 + q);
                        const int e = r * dim + q, D2 = dim * dim;
                        c[e] = m[0];
                        c[D2 + e] = -(m[0] + m[1]);
                        c[2 * D2 + e] = m[1] - m[0];
                    }
                std::memcpy(row, c, 8 * 3 * dim * dim);
            } else std::memcpy(row, op.m, 64);
        }
    }
}

bool jit_set_block(std::vector<uint8_t> &buf, const Step &st, const int *pos, int K, uint64_t fixbits)
{
    if (K > kMaxFix || buf.size() < kOffTpo) return false;
    std::vector<int32_t> ts(st.pass.tile_sorted, st.pass.tile_sorted + kTileBits);
    ts.insert(ts.end(), pos, pos + K);
    std::sort(ts.begin(), ts.end());
    ts.resize(kTileBits + kMaxFix, 62);
    std::memcpy(buf.data() + kOffTs, ts.data(), 4 * ts.size());
    std::memcpy(buf.data() + kOffFix, &fixbits, 8);
    return true;
}

void jit_set_red(std::vector<uint8_t> &buf, double *red)
{
    if (buf.size() >= kOffRed + 8) std::memcpy(buf.data() + kOffRed, &red, 8);
}

void jit_set_desync(std::vector<uint8_t> &buf, uint32_t n_sm, uint32_t ns)
{
    const uint64_t d = ns ? ((uint64_t)n_sm << 32) | ns : 0;
    if (buf.size() >= 24) std::memcpy(buf.data() + 16, &d, 8);
}

void jit_set_ttab(std::vector<uint8_t> &buf, void *ttab)
{
    if (buf.size() >= kOffTtab + 8) std::memcpy(buf.data() + kOffTtab, &ttab, 8);
}

void jit_set_init(std::vector<uint8_t> &buf, uint64_t init_phys)
{
    if (buf.size() >= kOffInit + 8) std::memcpy(buf.data() + kOffInit, &init_phys, 8);
}

// e^{2 pi i k / 256}, k < 256 (device, one per process)
const void *jit_phase_table()
{
    static void *d = []() -> void * {
        double h[512];
        for (int k = 0; k < 256; k++) {
            const long double a = 2.0L * 3.14159265358979323846264338327950288L * k / 256.0L;
            h[2 * k] = (double)cosl(a);
            h[2 * k + 1] = (double)sinl(a);
        }
        void *p = nullptr;
        if (cudaMalloc(&p, sizeof(h)) != cudaSuccess || cudaMemcpy(p, h, sizeof(h), cudaMemcpyHostToDevice) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        return p;
    }();
    return d;
}

// ------------------------------------------------------------- driver API
// resolved at run time through cudart so the library loads on hosts without
// a driver (the CPU test container)
const Drv &drv()
{
    static Drv d = []() {
        Drv x{};
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuModuleLoadData", (void **)&x.moduleLoadData, cudaEnableDefault, &q);
        cudaGetDriverEntryPoint("cuModuleGetFunction", (void **)&x.moduleGetFunction, cudaEnableDefault, &q);
        cudaGetDriverEntryPoint("cuFuncSetAttribute", (void **)&x.funcSetAttribute, cudaEnableDefault, &q);
        cudaGetDriverEntryPoint("cuLaunchKernel", (void **)&x.launchKernel, cudaEnableDefault, &q);
        return x;
    }();
    return d;
}

// ------------------------------------------------------------- compiling
// NVRTC of the CUDA 12.9 toolkit, loaded by absolute path: a process that
// imported PyTorch already holds torch's own libnvrtc.so.12 (an older CUDA
// whose ptxas rejects some sm_100a instructions), so the soname alone is not
// enough to get the compiler this library was built with.
struct Nvrtc {
    nvrtcResult (*create)(nvrtcProgram *, const char *, const char *, int, const char *const *, const char *const *);
    nvrtcResult (*compile)(nvrtcProgram, int, const char *const *);
    nvrtcResult (*logSize)(nvrtcProgram, size_t *);
    nvrtcResult (*log)(nvrtcProgram, char *);
    nvrtcResult (*cubinSize)(nvrtcProgram, size_t *);
    nvrtcResult (*cubin)(nvrtcProgram, char *);
    nvrtcResult (*destroy)(nvrtcProgram *);
    bool ok = false;
};

static const Nvrtc &nvrtc()
{
    static Nvrtc n = []() {
        Nvrtc x{};
        const char *env = getenv("CUDA_HOME");
        std::string dir = env ? env : "/usr/local/cuda";
        const char *names[] = {"/lib64/libnvrtc.so.12.9.86", "/lib64/libnvrtc.so.12", "/lib64/libnvrtc.so"};
        void *h = nullptr;
        for (const char *nm : names)
            if ((h = dlopen((dir + nm).c_str(), RTLD_NOW | RTLD_LOCAL))) break;
        if (!h) return x;
        x.create = (decltype(x.create))dlsym(h, "nvrtcCreateProgram");
        x.compile = (decltype(x.compile))dlsym(h, "nvrtcCompileProgram");
        x.logSize = (decltype(x.logSize))dlsym(h, "nvrtcGetProgramLogSize");
        x.log = (decltype(x.log))dlsym(h, "nvrtcGetProgramLog");
        x.cubinSize = (decltype(x.cubinSize))dlsym(h, "nvrtcGetCUBINSize");
        x.cubin = (decltype(x.cubin))dlsym(h, "nvrtcGetCUBIN");
        x.destroy = (decltype(x.destroy))dlsym(h, "nvrtcDestroyProgram");
        x.ok = x.create && x.compile && x.logSize && x.log && x.cubinSize && x.cubin && x.destroy;
        return x;
    }();
    return n;
}

static bool nvrtc_compile(const std::string &src, std::vector<char> &cubin, std::string &log)
{
    const Nvrtc &N = nvrtc();
    if (!N.ok) {
        log = "CUDA 12.9 NVRTC not found under $CUDA_HOME/lib64";
        return false;
    }
    nvrtcProgram prog;
    if (N.create(&prog, src.c_str(), "qsim_pass.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
        log = "nvrtcCreateProgram failed";
        return false;
    }
    const char *opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-default-device", "-diag-suppress=177"};
    nvrtcResult r = N.compile(prog, 4, opts);
    if (r != NVRTC_SUCCESS) {
        size_t n = 0;
        N.logSize(prog, &n);
        log.resize(n);
        N.log(prog, &log[0]);
        N.destroy(&prog);
        return false;
    }
    size_t n = 0;
    N.cubinSize(prog, &n);
    cubin.resize(n);
    N.cubin(prog, cubin.data());
    N.destroy(&prog);
    return true;
}

// On-disk cubin cache for the pass kernels, so that a new process does not
// recompile the structures an earlier one built: $QSIM_JIT_CACHE_DIR (default
// $XDG_CACHE_HOME/qsim_b200_jit or ~/.cache/qsim_b200_jit; "off" disables).
// An entry stores its full source, compared on load (no trust in the hash).
static const char kJitCacheTag[] = "qsim_b200 jit v1 sm_100a --std=c++17 -default-device\n";

static std::string jit_cache_dir()
{
    static const std::string dir = []() -> std::string {
        const char *e = getenv("QSIM_JIT_CACHE_DIR");
        if (e) return std::string(e) == "off" ? std::string() : std::string(e);
        const char *x = getenv("XDG_CACHE_HOME");
        const char *h = getenv("HOME");
        std::string base = x && *x ? std::string(x) : h && *h ? std::string(h) + "/.cache" : std::string();
        return base.empty() ? base : base + "/qsim_b200_jit";
    }();
    return dir;
}

static std::string jit_cache_path(const std::string &src)
{
    uint64_t h = 1469598103934665603ULL;  // FNV-1a over tag + source
    for (const char *p : {kJitCacheTag, src.c_str()})
        for (; *p; p++) h = (h ^ (unsigned char)*p) * 1099511628211ULL;
    char name[32];
    snprintf(name, sizeof(name), "/%016llx.bin", (unsigned long long)h);
    return jit_cache_dir() + name;
}

static bool disk_load(const std::string &src, std::vector<char> &cubin)
{
    if (jit_cache_dir().empty()) return false;
    FILE *f = fopen(jit_cache_path(src).c_str(), "rb");
    if (!f) return false;
    bool ok = false;
    uint64_t ns = 0, nc = 0;
    if (fread(&ns, 8, 1, f) == 1 && ns == src.size() + sizeof(kJitCacheTag) - 1) {
        std::string stored(ns, '\0');
        if (fread(&stored[0], 1, ns, f) == ns && stored == kJitCacheTag + src && fread(&nc, 8, 1, f) == 1 &&
            nc > 0 && nc < (1ULL << 30)) {
            cubin.resize(nc);
            ok = fread(cubin.data(), 1, nc, f) == nc;
        }
    }
    fclose(f);
    return ok;
}

static void disk_store(const std::string &src, const std::vector<char> &cubin)
{
    const std::string dir = jit_cache_dir();
    if (dir.empty()) return;
    for (size_t i = 1; i <= dir.size(); i++)  // mkdir -p; failures only lose the cache
        if (i == dir.size() || dir[i] == '/') mkdir(dir.substr(0, i).c_str(), 0755);
    const std::string path = jit_cache_path(src), tmp = path + "." + std::to_string(getpid()) + ".tmp";
    FILE *f = fopen(tmp.c_str(), "wb");
    if (!f) return;
    const std::string stored = kJitCacheTag + src;
    const uint64_t ns = stored.size(), nc = cubin.size();
    const bool ok = fwrite(&ns, 8, 1, f) == 1 && fwrite(stored.data(), 1, ns, f) == ns && fwrite(&nc, 8, 1, f) == 1 &&
                    fwrite(cubin.data(), 1, nc, f) == nc;
    if (fclose(f) == 0 && ok) rename(tmp.c_str(), path.c_str());
    else remove(tmp.c_str());
}

std::string jit_key(const Step &st)
{
    std::string k;
    auto put = [&](uint64_t v) { k.append(reinterpret_cast<const char *>(&v), 8); };
    put((uint64_t)env_int("QSIM_JIT_MINB", kPassMinBlocks) |
        ((uint64_t)(st.pass.fresh != 0) << 48) | ((uint64_t)(st.jit_block != 0) << 49) |
        ((uint64_t)(st.jit_readout != 0) << 50) |
        ((uint64_t)env_int("QSIM_JIT_U4IL", 0) << 20) | ((uint64_t)env_int("QSIM_JIT_BAR", kJitBarDefault) << 28));
    put(st.pass.cfg0);
    {
        const Forms fm = forms_of(st);
        put((uint64_t)fm.u2 | ((uint64_t)fm.u4 << 1));
    }
    // the generated source indexes the deduplicated out-of-tile predicates
    // (P.out[out_idx[o]], and n_out sizes the parameter struct): the dedup
    // pattern is part of the structure, not only whether an op has one
    std::vector<int> out_idx, m_idx, m_col;
    layout_of(st, out_idx, m_idx, m_col);
    for (size_t o = 0; o < st.ops.size(); o++) {
        const KOp &op = st.ops[o];
        put((uint64_t)op.code | ((uint64_t)op.k << 8) | ((uint64_t)(op.mout != 0) << 16) |
            ((uint64_t)jit_hadamard(op) << 17) | ((uint64_t)(uint32_t)(out_idx[o] + 1) << 32));
        put((uint64_t)op.mreg | ((uint64_t)op.vreg << 8) | ((uint64_t)op.mlane << 16) | ((uint64_t)op.vlane << 24) |
            ((uint64_t)op.mwarp << 32) | ((uint64_t)op.vwarp << 40));
        if (op.code == OPC_TRANS || op.code == OPC_U4) put(op.cfg);
    }
    return k;
}

bool JitCache::compile(const std::vector<const Step *> &steps, std::string &err)
{
    std::vector<std::string> keys, srcs;
    {
        std::lock_guard<std::mutex> g(mu_);
        for (const Step *st : steps) {
            std::string k = jit_key(*st);
            if (fns_.count(k) || std::find(keys.begin(), keys.end(), k) != keys.end()) continue;
            keys.push_back(k);
        }
    }
    if (keys.empty()) return true;
    std::vector<int> ntab;
    std::vector<double> fps;
    for (const Step *st : steps) {
        std::string k = jit_key(*st);
        auto it = std::find(keys.begin(), keys.end(), k);
        if (it != keys.end() && srcs.size() == (size_t)(it - keys.begin())) {
            JitPass jp = jit_generate(*st);
            srcs.push_back(jp.src);
            ntab.push_back(jp.n_tslots);
            fps.push_back(jp.fp64_per_thread);
        }
    }
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::vector<char>> bins(srcs.size());
    std::vector<std::string> logs(srcs.size());
    std::vector<char> ok(srcs.size(), 0);
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t nthreads = std::min<size_t>(srcs.size(), hw);
    std::vector<std::thread> th;
    std::atomic_size_t next{0};
    for (size_t w = 0; w < nthreads; w++)
        th.emplace_back([&]() {
            for (size_t i; (i = next++) < srcs.size();) {
                if (disk_load(srcs[i], bins[i])) { ok[i] = 1; continue; }
                ok[i] = nvrtc_compile(srcs[i], bins[i], logs[i]);
                if (ok[i]) disk_store(srcs[i], bins[i]);
            }
        });
    for (auto &t : th) t.join();
    for (size_t i = 0; i < srcs.size(); i++) {
        if (!ok[i]) {
            err = "NVRTC: " + logs[i].substr(0, 2000);
            return false;
        }
        CUmodule mod;
        CUfunction fn;
        const Drv &D = drv();
        if (!D.moduleLoadData || !D.moduleGetFunction || !D.launchKernel) {
            err = "CUDA driver entry points unavailable";
            return false;
        }
        if (D.moduleLoadData(&mod, bins[i].data()) != CUDA_SUCCESS ||
            D.moduleGetFunction(&fn, mod, "qsim_pass") != CUDA_SUCCESS) {
            err = "cuModuleLoadData/cuModuleGetFunction failed";
            return false;
        }
        D.funcSetAttribute(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, kTileAmps * 16);
        CUfunction tab = nullptr;
        if (ntab[i] && D.moduleGetFunction(&tab, mod, "qsim_pass_tab") != CUDA_SUCCESS) {
            err = "cuModuleGetFunction(qsim_pass_tab) failed";
            return false;
        }
        std::lock_guard<std::mutex> g(mu_);
        mods_.push_back(mod);
        fns_[keys[i]] = Fn{fn, tab, ntab[i], fps[i]};
        compiled++;
    }
    compile_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return true;
}

static void dump_source(const std::string &src, size_t idx)
{
    const char *d = getenv("QSIM_JIT_DUMP");
    if (!d) return;
    std::string path = std::string(d) + "/qsim_pass_" + std::to_string(idx) + ".cu";
    if (FILE *f = fopen(path.c_str(), "w")) {
        fwrite(src.data(), 1, src.size(), f);
        fclose(f);
    }
}

bool jit_compile_only(const std::vector<const Step *> &steps, std::string &err, int &n, double &ms, bool compile,
                      std::vector<double> *fp64_per_amp)
{
    // process-wide key -> source record: equal keys must mean equal sources
    // (the kernel cache is keyed by jit_key), across every plan checked here
    static std::mutex seen_mu;
    static std::unordered_map<std::string, std::string> seen;
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::string> keys, srcs;
    for (size_t i = 0; i < steps.size(); i++) {
        const Step *st = steps[i];
        std::string k = jit_key(*st);
        JitPass jp = jit_generate(*st);
        std::string src = std::move(jp.src);
        if (fp64_per_amp) fp64_per_amp->push_back(jp.fp64_per_thread / kAmpsPerThread);
        dump_source(src, i);
        {
            std::lock_guard<std::mutex> g(seen_mu);
            auto it = seen.find(k);
            if (it == seen.end()) seen.emplace(k, src);
            else if (it->second != src) {
                err = "jit key collision: pass " + std::to_string(i) + " has the key of a different source";
                return false;
            }
        }
        if (std::find(keys.begin(), keys.end(), k) != keys.end()) continue;
        keys.push_back(k);
        srcs.push_back(std::move(src));
    }
    n = (int)srcs.size();
    if (!compile) {
        ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        return true;
    }
    std::vector<std::vector<char>> bins(srcs.size());
    std::vector<std::string> logs(srcs.size());
    std::vector<char> ok(srcs.size(), 0);
    std::atomic_size_t next{0};
    std::vector<std::thread> th;
    const size_t nt = std::min<size_t>(srcs.size(), std::max(1u, std::thread::hardware_concurrency()));
    for (size_t w = 0; w < nt; w++)
        th.emplace_back([&]() {
            for (size_t i; (i = next++) < srcs.size();) ok[i] = nvrtc_compile(srcs[i], bins[i], logs[i]);
        });
    for (auto &t : th) t.join();
    ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    for (size_t i = 0; i < srcs.size(); i++)
        if (!ok[i]) {
            err = logs[i].substr(0, 4000) + "\n--- source ---\n" + srcs[i].substr(0, 4000);
            return false;
        }
    return true;
}

CUfunction JitCache::find(const std::string &key)
{
    std::lock_guard<std::mutex> g(mu_);
    auto it = fns_.find(key);
    return it == fns_.end() ? nullptr : it->second.pass;
}

CUfunction JitCache::find_tab(const std::string &key, int &n_tslots)
{
    std::lock_guard<std::mutex> g(mu_);
    auto it = fns_.find(key);
    n_tslots = it == fns_.end() ? 0 : it->second.n_tslots;
    return it == fns_.end() ? nullptr : it->second.tab;
}

double JitCache::fp64_per_thread(const std::string &key)
{
    std::lock_guard<std::mutex> g(mu_);
    auto it = fns_.find(key);
    return it == fns_.end() ? -1.0 : it->second.fp64;
}

size_t JitCache::size()
{
    std::lock_guard<std::mutex> g(mu_);
    return fns_.size();
}

}  // namespace qsb
