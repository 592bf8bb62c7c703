// plan.cpp -- gate classification, initial layout, fusion/placement planner.
//
// The planner turns the queued LOGICAL gate list into a sequence of device
// steps in PHYSICAL coordinates:
//   * ST_PASS      one fused tile pass (kernels.cu k_pass) applying many gates
//   * ST_GENERIC / ST_PHASE   one gate per launch (small shards, fusion off)
//   * ST_PERM      one controlled register permutation (k_perm)
//   * ST_PERMRUN   a run of permutations of one register in one pass (k_perm_run)
//   * ST_EXCHANGE  the paper's K-pair local<->nonlocal qubit interchange
//                  (Eqs. onequbitchange / twoqubitchange0-5)
// It keeps sigma (qubit <-> physical bit).  SWAP gates are
// relabels of sigma.  Diagonal gates and controls never force locality
// (the optimisation P:623-628 mentions and leaves out).
//
// Reordering rule: a gate may move ahead of skipped gates only if, on every
// qubit they share, both act diagonally (controls count as diagonal).
#include "plan.h"

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <complex>
#include <cstdio>
#include <limits>
#include <sstream>

namespace qsb {

static inline uint64_t bit(int p) { return 1ULL << p; }

void classify(GateRec &g)
{
    g.qN = g.qD = 0;
    if (g.kind == GK_U2) {
        const double *u = g.u;
        bool diag = u[2] == 0 && u[3] == 0 && u[4] == 0 && u[5] == 0;
        bool xs = u[0] == 0 && u[1] == 0 && u[6] == 0 && u[7] == 0 && u[2] == 1 && u[3] == 0 &&
                  u[4] == 1 && u[5] == 0;
        bool real = u[1] == 0 && u[3] == 0 && u[5] == 0 && u[7] == 0;
        g.cls = diag ? CLS_DIAG : xs ? CLS_XS : real ? CLS_REAL : CLS_GENERAL;
        for (int c : g.controls) g.qD |= bit(c);
        if (diag) g.qD |= bit(g.target);
        else g.qN |= bit(g.target);
    } else if (g.kind == GK_PERM) {
        for (int c : g.controls) g.qD |= bit(c);
        for (int t : g.targets) g.qN |= bit(t);
    } else {  // SWAP, U4
        for (int t : g.targets) g.qN |= bit(t);
    }
}

Planner::Planner(int n_, int G_) : n(n_), G(G_), M(n_ - G_), phys_of(n_), qubit_at(n_)
{
    for (int q = 0; q < n; q++) phys_of[q] = qubit_at[q] = q;
}

void Planner::swap_layout(int pa, int pb)
{
    int qa = qubit_at[pa], qb = qubit_at[pb];
    qubit_at[pa] = qb;
    qubit_at[pb] = qa;
    phys_of[qa] = pb;
    phys_of[qb] = pa;
}

void Planner::choose_initial_layout(const std::vector<GateRec> &gates)
{
    const size_t INF = std::numeric_limits<size_t>::max();
    std::vector<size_t> first_use(n, INF);
    std::vector<int> perm_first;
    for (size_t i = 0; i < gates.size(); i++) {
        const GateRec &g = gates[i];
        for (int q = 0; q < n; q++)
            if ((g.qN >> q) & 1)
                if (first_use[q] == INF) first_use[q] = i;
        if (g.kind == GK_PERM)
            for (int t : g.targets)
                if (std::find(perm_first.begin(), perm_first.end(), t) == perm_first.end())
                    perm_first.push_back(t);
    }
    std::vector<int> order;  // logical qubits, low physical bits first
    std::vector<char> placed(n, 0);
    // global (top G bits): the G qubits first used latest (never-used first)
    std::vector<int> byuse(n);
    for (int q = 0; q < n; q++) byuse[q] = q;
    std::stable_sort(byuse.begin(), byuse.end(), [&](int a, int b) {
        if (first_use[a] != first_use[b]) return first_use[a] > first_use[b];
        return a > b;  // ties (e.g. never used): keep the identity layout
    });
    std::vector<int> glob;
    for (int q : byuse) {
        if ((int)glob.size() == G) break;
        bool is_perm = std::find(perm_first.begin(), perm_first.end(), q) != perm_first.end();
        if (!is_perm || (int)perm_first.size() >= n - G + 1) glob.push_back(q);
    }
    for (int q : glob) placed[q] = 1;
    for (int t : perm_first)
        if (!placed[t] && (int)order.size() < n - G) { order.push_back(t); placed[t] = 1; }
    for (int q = 0; q < n; q++)
        if (!placed[q]) { order.push_back(q); placed[q] = 1; }
    std::sort(glob.begin(), glob.end());
    for (int q : glob) order.push_back(q);
    for (int p = 0; p < n; p++) { qubit_at[p] = order[p]; phys_of[order[p]] = p; }
}

PhaseRunPlan plan_phase_run(const KOp *ops, size_t n)
{
    PhaseRunPlan r;
    for (size_t o = 0; o < n; o++) {
        const uint32_t m = ops[o].mreg, v = ops[o].vreg, O = m & v, Z = m & ~v;
        for (uint32_t i = 0; i < (uint32_t)kAmpsPerThread; i++)
            if ((i & m) == v) r.direct += 4;
        for (uint32_t T = Z;; T = (T - 1) & Z) {  // subsets of Z
            r.used |= 1u << (O | T);
            r.acc += 2;  // one 64-bit add
            if (!T) break;
        }
    }
    const double kExp = 20, kMul = 4;  // e^{i theta} (table x Taylor) and complex multiply
    // mode A: distinct (set of monomials below register i) -> one exp each
    uint32_t keys[kAmpsPerThread];
    int nkeys = 0, nregs = 0;
    for (uint32_t i = 0; i < (uint32_t)kAmpsPerThread; i++) {
        uint32_t key = 0;
        for (uint32_t S = 0; S < (uint32_t)kAmpsPerThread; S++)
            if (((r.used >> S) & 1) && (S & i) == S) key |= 1u << S;
        if (!key) continue;
        nregs++;
        bool seen = false;
        for (int k = 0; k < nkeys; k++) seen |= keys[k] == key;
        if (!seen) keys[nkeys++] = key;
    }
    const double costA = nkeys * kExp + nregs * kMul;
    double costB = 0;
    for (uint32_t S = 0; S < (uint32_t)kAmpsPerThread; S++)
        if ((r.used >> S) & 1) costB += kExp + kMul * (double)(kAmpsPerThread >> __builtin_popcount(S));
    r.mode = costB < costA ? 1 : 0;
    r.acc += std::min(costA, costB);
    return r;
}

// ------------------------------------------------------------------ passes
namespace {
constexpr int OP_BARRIER = -1;  // fusion only: an unfusable gate on the qubits in cm

struct POp {
    int code;      // OPC_U2 / OPC_U2R / OPC_XS / OPC_PHASE / OPC_U4 / OP_BARRIER
    int t;         // physical target (U2-type); U4: physical bit of 4x4 index bit 0
    uint64_t cm, cv;
    double m[8];
    int gid;
    int t2 = -1;   // U4: physical bit of 4x4 index bit 1
    double m4[32]; // U4: row-major complex 4x4 (re, im)
    bool fused = false;  // made by fuse_ops
};

}  // namespace

static void set_u2_code(const GateRec &g, POp &p)
{
    p.code = g.cls == CLS_XS ? OPC_XS : g.cls == CLS_REAL ? OPC_U2R : OPC_U2;
    for (int k = 0; k < 8; k++) p.m[k] = g.u[k];
}

namespace {
// thread-coordinate assignment of the 12 tile-local bits (see engine.h)
struct Cfg {
    int r[kRegBits], l[5], w[kWarpBits];
    uint64_t pack() const
    {
        uint64_t c = 0;
        for (int j = 0; j < kRegBits; j++) c |= (uint64_t)r[j] << (4 * j);
        for (int j = 0; j < 5; j++) c |= (uint64_t)l[j] << (4 * (kLaneNib + j));
        for (int j = 0; j < kWarpBits; j++) c |= (uint64_t)w[j] << (4 * (kWarpNib + j));
        return c;
    }
    // global load/store config: register bit 0 and lanes 0, 1 hold the tile
    // bits that sit at physical bits 0, 1, 2 (sb) -- 256-bit accesses, whole lines
    bool store_ok(const int *sb) const { return r[0] == sb[0] && l[0] == sb[1] && l[1] == sb[2]; }
    int role_of(int t, int &j) const
    {
        for (j = 0; j < kRegBits; j++)
            if (r[j] == t) return ROLE_REG;
        for (j = 0; j < 5; j++)
            if (l[j] == t) return ROLE_LANE;
        for (j = 0; j < kWarpBits; j++)
            if (w[j] == t) return ROLE_WARP;
        j = -1;
        return -1;
    }
};

// Complete a register set into a config.  Lanes must cover tile-bit residues
// {0,1,2} mod 3 for conflict-free transposes (kernels.cu swz).
const int kLoadBits[3] = {0, 1, 2};

Cfg make_cfg(const std::vector<int> &reg_in, bool store, const int *sb = kLoadBits)
{
    Cfg c;
    std::vector<int> reg = reg_in;
    if (store) {
        reg.erase(std::remove(reg.begin(), reg.end(), sb[0]), reg.end());
        reg.insert(reg.begin(), sb[0]);
    }
    bool used[kTileBits] = {false};
    for (int j = 0; j < kRegBits; j++) { c.r[j] = reg[j]; used[reg[j]] = true; }
    std::vector<int> lanes;
    if (store) { lanes = {sb[1], sb[2]}; used[sb[1]] = used[sb[2]] = true; }
    // one lane bit of every missing residue first
    for (int res = 0; res < 3; res++) {
        bool have = false;
        for (int t : lanes) have |= (t % 3) == res;
        if (have) continue;
        for (int t = 0; t < kTileBits; t++)
            if (!used[t] && t % 3 == res) { lanes.push_back(t); used[t] = true; break; }
    }
    for (int t = 0; t < kTileBits && (int)lanes.size() < 5; t++)
        if (!used[t]) { lanes.push_back(t); used[t] = true; }
    for (int j = 0; j < 5; j++) c.l[j] = lanes[j];
    int nw = 0;
    for (int t = 0; t < kTileBits; t++)
        if (!used[t]) c.w[nw++] = t;
    return c;
}

// physical bits an op acts on non-diagonally (a barrier op: none)
uint64_t nondiag(const POp &p)
{
    if (p.code == OPC_PHASE || p.code == OP_BARRIER) return 0;
    return bit(p.t) | (p.t2 >= 0 ? bit(p.t2) : 0);
}

// ------------------------------------------------- two-qubit block fusion
// On a fused random layer the pass is bound by the FP64 pipe (DESIGN.md
// §5.2), not by HBM.  A cluster of gates acting only on two qubits {a, b} --
// e.g. the brickwork's U2 (x) U2, CNOT, U2 (x) U2 -- equals one 4x4 unitary
// (the product of the gates' embeddings, Eqs. NUM2-NUM8 written on the 4-dim
// subspace), which costs 16 FMA-pipe ops per amplitude instead of 8 per
// general U2.  Greedy, in sequence order: every two-qubit gate seeds a block
// that absorbs the neighbouring gates on {a, b} that can move next to it (no
// unabsorbed gate on a shared qubit in between); the block is kept only if it
// is cheaper than its gates.  Runs of one-qubit gates on one qubit merge into
// one U2 the same way.  Used on the logical gate list before passes are
// formed (Planner::plan, so blocks are never cut by a pass boundary) and on
// each pass's op list (for what the first round left).
uint64_t qset(const POp &p) { return nondiag(p) | p.cm; }

// FMA-pipe ops per amplitude of the shard (touched fraction included)
double op_cost(const POp &p)
{
    const double touched = std::ldexp(1.0, -__builtin_popcountll(p.cm));
    switch (p.code) {
    case OPC_U2: return 8 * touched;
    case OPC_U2R: return 4 * touched;
    case OPC_XS: return 0;
    case OPC_PHASE: return 4 * touched;
    case OPC_U4: return 16;
    }
    return 0;
}

typedef std::complex<double> cd;

// 4x4 embedding of op p on the subspace index j = bit(pa) + 2 bit(pb)
void embed4(const POp &p, int pa, int pb, cd E[4][4])
{
    for (int r = 0; r < 4; r++)
        for (int c = 0; c < 4; c++) E[r][c] = 0;
    if (p.code == OPC_U4) {
        const bool flip = p.t != pa;  // p's index bit 0 is pb
        auto pm = [&](int x) { return flip ? ((x & 1) << 1) | (x >> 1) : x; };
        for (int r = 0; r < 4; r++)
            for (int c = 0; c < 4; c++)
                E[r][c] = cd(p.m4[8 * pm(r) + 2 * pm(c)], p.m4[8 * pm(r) + 2 * pm(c) + 1]);
        return;
    }
    auto pred = [&](int j) {
        for (int s = 0; s < 2; s++) {
            const int pos = s ? pb : pa;
            if (((p.cm >> pos) & 1) && (int)((p.cv >> pos) & 1) != ((j >> s) & 1)) return false;
        }
        return true;
    };
    for (int j = 0; j < 4; j++) {
        if (!pred(j)) { E[j][j] = 1; continue; }
        if (p.code == OPC_PHASE) { E[j][j] = cd(p.m[0], p.m[1]); continue; }
        const int s = p.t == pa ? 0 : 1;
        const int bj = (j >> s) & 1, j0 = j & ~(1 << s), j1 = j0 | (1 << s);
        E[j0][j] = cd(p.m[bj ? 2 : 0], p.m[bj ? 3 : 1]);  // U[0][bj]
        E[j1][j] = cd(p.m[bj ? 6 : 4], p.m[bj ? 7 : 5]);  // U[1][bj]
    }
}

// absorb into the cluster seeded at g the ops on `mask` that can move next to it
void cluster(const std::vector<POp> &ops, const std::vector<char> &used, size_t g, uint64_t mask, bool allow_pairs,
             std::vector<size_t> &got)
{
    got.assign(1, g);
    auto ok = [&](size_t h, uint64_t stopped) {
        const POp &p = ops[h];
        const uint64_t S = qset(p);
        if (used[h] || p.code == OP_BARRIER || (S & ~mask) || (S & stopped)) return false;
        if (!allow_pairs) return p.code != OPC_PHASE && p.code != OPC_U4 && !p.cm;
        return true;
    };
    uint64_t stopped = 0;
    for (size_t h = g; h-- > 0 && stopped != mask;) {
        const uint64_t S = qset(ops[h]);
        if (!(S & mask)) continue;
        if (ok(h, stopped)) got.push_back(h);
        else stopped |= S & mask;
    }
    stopped = 0;
    for (size_t h = g + 1; h < ops.size() && stopped != mask; h++) {
        const uint64_t S = qset(ops[h]);
        if (!(S & mask)) continue;
        if (ok(h, stopped)) got.push_back(h);
        else stopped |= S & mask;
    }
    std::sort(got.begin(), got.end());
}

// Fuse `ops` in place.  cost[i] = FMA-pipe ops per amplitude of ops[i];
// pair_ok(c) says whether bit c may be one of a block's two qubits.
template <class PairOk>
void fuse_ops(std::vector<POp> &ops, const std::vector<double> &cost, PairOk pair_ok, double margin = 2)
{
    const size_t n = ops.size();
    std::vector<char> used(n, 0);
    std::vector<int> repl_of(n, -1);  // index into repl
    std::vector<POp> repl;
    std::vector<size_t> got;
    // two-qubit blocks
    for (size_t g = 0; g < n; g++) {
        const POp &s = ops[g];
        if (used[g] || s.code == OPC_PHASE || s.code == OP_BARRIER) continue;
        int pa, pb;
        if (s.code == OPC_U4) {
            pa = std::min(s.t, s.t2);
            pb = std::max(s.t, s.t2);
        } else {
            if (__builtin_popcountll(s.cm) != 1) continue;
            const int c = __builtin_ctzll(s.cm);
            pa = std::min(c, s.t);
            pb = std::max(c, s.t);
        }
        if (!pair_ok(pa) || !pair_ok(pb)) continue;
        const uint64_t mask = bit(pa) | bit(pb);
        cluster(ops, used, g, mask, true, got);
        double before = 0;
        for (size_t h : got) before += cost[h];
        if (got.size() < 2 || before <= 16 + margin) continue;  // a 4x4 costs 16 + register copies
        cd B[4][4], E[4][4], T[4][4];
        for (int r = 0; r < 4; r++)
            for (int q = 0; q < 4; q++) B[r][q] = r == q ? 1 : 0;
        for (size_t h : got) {  // B <- E_h B, in sequence order
            embed4(ops[h], pa, pb, E);
            for (int r = 0; r < 4; r++) {
                for (int q = 0; q < 4; q++) T[r][q] = 0;
                for (int k = 0; k < 4; k++) {
                    const double er = E[r][k].real(), ei = E[r][k].imag();
                    if (er == 0 && ei == 0) continue;  // embeddings are sparse
                    for (int q = 0; q < 4; q++)
                        T[r][q] += cd(er * B[k][q].real() - ei * B[k][q].imag(), er * B[k][q].imag() + ei * B[k][q].real());
                }
            }
            for (int r = 0; r < 4; r++)
                for (int q = 0; q < 4; q++) B[r][q] = T[r][q];
        }
        POp u{};
        u.code = OPC_U4;
        u.fused = true;
        u.t = pa;
        u.t2 = pb;
        u.gid = s.gid;
        for (int r = 0; r < 4; r++)
            for (int q = 0; q < 4; q++) {
                u.m4[8 * r + 2 * q] = B[r][q].real();
                u.m4[8 * r + 2 * q + 1] = B[r][q].imag();
            }
        for (size_t h : got) used[h] = 1;
        repl_of[g] = (int)repl.size();
        repl.push_back(u);
    }
    // runs of one-qubit gates on one qubit
    for (size_t g = 0; g < n; g++) {
        const POp &s = ops[g];
        if (used[g] || s.code == OPC_PHASE || s.code == OPC_U4 || s.code == OP_BARRIER || s.cm) continue;
        cluster(ops, used, g, bit(s.t), false, got);
        if (got.size() < 2) continue;
        cd U[2][2] = {{1, 0}, {0, 1}};
        double before = 0;
        for (size_t h : got) {
            const POp &p = ops[h];
            before += cost[h];
            const cd V[2][2] = {{cd(p.m[0], p.m[1]), cd(p.m[2], p.m[3])}, {cd(p.m[4], p.m[5]), cd(p.m[6], p.m[7])}};
            cd W[2][2];
            for (int r = 0; r < 2; r++)
                for (int q = 0; q < 2; q++) W[r][q] = V[r][0] * U[0][q] + V[r][1] * U[1][q];
            for (int r = 0; r < 2; r++)
                for (int q = 0; q < 2; q++) U[r][q] = W[r][q];
        }
        POp u{};
        u.fused = true;
        u.t = s.t;
        u.gid = s.gid;
        const double m[8] = {U[0][0].real(), U[0][0].imag(), U[0][1].real(), U[0][1].imag(),
                             U[1][0].real(), U[1][0].imag(), U[1][1].real(), U[1][1].imag()};
        for (int k = 0; k < 8; k++) u.m[k] = m[k];
        const bool xs = m[0] == 0 && m[1] == 0 && m[6] == 0 && m[7] == 0 && m[2] == 1 && m[3] == 0 && m[4] == 1 &&
                        m[5] == 0;
        const bool real = m[1] == 0 && m[3] == 0 && m[5] == 0 && m[7] == 0;
        u.code = xs ? OPC_XS : real ? OPC_U2R : OPC_U2;
        if (op_cost(u) >= before) continue;
        for (size_t h : got) used[h] = 1;
        repl_of[g] = (int)repl.size();
        repl.push_back(u);
    }
    if (repl.empty()) return;
    std::vector<POp> out;
    out.reserve(n);
    for (size_t g = 0; g < n; g++) {
        if (repl_of[g] >= 0) out.push_back(repl[repl_of[g]]);
        else if (!used[g]) out.push_back(ops[g]);
    }
    ops.swap(out);
}

void fuse_blocks(std::vector<POp> &ops, const int tl_of[64])
{
    std::vector<double> cost;
    for (const POp &p : ops) cost.push_back(op_cost(p));
    fuse_ops(ops, cost, [&](int c) { return c < 64 && tl_of[c] >= 0; });
}

// the same fusion on the LOGICAL gate list (qubit numbers as bits)
std::vector<GateRec> fuse_gates(const std::vector<GateRec> &gates, uint64_t no_blocks_on, double margin)
{
    std::vector<POp> ops(gates.size());
    std::vector<double> cost(gates.size());
    for (size_t i = 0; i < gates.size(); i++) {
        const GateRec &g = gates[i];
        POp &p = ops[i];
        p = POp{};
        p.gid = (int)i;
        if (g.kind != GK_U2) {
            p.code = OP_BARRIER;
            p.t = -1;
            p.cm = g.qN | g.qD;
            continue;
        }
        p.t = g.target;
        for (int c : g.controls) p.cm |= bit(c);
        p.cv = p.cm;
        for (int k = 0; k < 8; k++) p.m[k] = g.u[k];
        p.code = g.cls == CLS_XS ? OPC_XS : g.cls == CLS_REAL ? OPC_U2R : OPC_U2;
        const double touched = std::ldexp(1.0, -(int)g.controls.size());
        cost[i] = (g.cls == CLS_GENERAL ? 8 : g.cls == CLS_XS ? 0 : 4) * touched;
    }
    fuse_ops(ops, cost, [&](int q) { return !((no_blocks_on >> q) & 1); }, margin);
    std::vector<GateRec> out;
    out.reserve(ops.size());
    for (const POp &p : ops) {
        if (!p.fused) { out.push_back(gates[p.gid]); continue; }
        GateRec r;
        r.id = gates[p.gid].id;
        if (p.code == OPC_U4) {
            r.kind = GK_U4;
            r.targets = {p.t, p.t2};
            for (int k = 0; k < 32; k++) r.u4[k] = p.m4[k];
        } else {
            r.kind = GK_U2;
            r.target = p.t;
            for (int k = 0; k < 8; k++) r.u[k] = p.m[k];
        }
        classify(r);
        out.push_back(std::move(r));
    }
    return out;
}
}  // namespace

// Schedule the pass ops (dependency-respecting list scheduling that prefers
// ops whose target is already in registers), insert OPC_TRANS re-layouts,
// split every predicate over the thread coordinates.
// sb: tile bits stored at physical bits 0, 1, 2 (the next pass's low qubits)
static void lower_pass(const std::vector<POp> &pops, const int tl_of[64], Step &st, uint64_t &cfg0, const int *sb)
{
    const size_t n = pops.size();
    // Dependencies: a and b conflict when one acts non-diagonally on a qubit the
    // other touches (target or control).  Reduced per qubit: an op non-diagonal
    // on q waits for the last op non-diagonal on q and for the diagonal uses of
    // q since; a diagonal use waits for the last non-diagonal op.  Same partial
    // order as every conflicting pair, O(ops x qubits per op).
    std::vector<int> npred(n, 0);
    std::vector<std::vector<int>> succ(n);
    {
        std::vector<int> last_nd(64, -1);
        std::vector<std::vector<int>> diag_since(64);
        std::vector<int> dep;
        for (size_t b = 0; b < n; b++) {
            const uint64_t N = nondiag(pops[b]), D = pops[b].cm & ~N;
            dep.clear();
            for (uint64_t m = N; m; m &= m - 1) {
                const int q = __builtin_ctzll(m);
                if (last_nd[q] >= 0) dep.push_back(last_nd[q]);
                dep.insert(dep.end(), diag_since[q].begin(), diag_since[q].end());
                last_nd[q] = (int)b;
                diag_since[q].clear();
            }
            for (uint64_t m = D; m; m &= m - 1) {
                const int q = __builtin_ctzll(m);
                if (last_nd[q] >= 0) dep.push_back(last_nd[q]);
                diag_since[q].push_back((int)b);
            }
            std::sort(dep.begin(), dep.end());
            dep.erase(std::unique(dep.begin(), dep.end()), dep.end());
            for (int a : dep) succ[a].push_back((int)b);
            npred[b] = (int)dep.size();
        }
    }
    std::vector<char> done(n, 0);
    auto ready = [&](size_t b) { return npred[b] == 0; };
    auto finish = [&](size_t b) {
        done[b] = 1;
        for (int c : succ[b]) npred[c]--;
    };
    auto tl = [&](const POp &p) { return tl_of[p.t]; };
    auto in_regs = [&](const Cfg &c, const POp &p) {
        int j;
        if (c.role_of(tl_of[p.t], j) != ROLE_REG) return false;
        return p.t2 < 0 || c.role_of(tl_of[p.t2], j) == ROLE_REG;
    };
    // upcoming register bits: targets of ready ops first, then of the rest, in order
    auto upcoming = [&](bool store, std::vector<int> &reg, const int *lb = kLoadBits) {
        reg.clear();
        if (store) reg.push_back(lb[0]);
        for (int pass = 0; pass < 2 && reg.size() < (size_t)kRegBits; pass++)
            for (size_t b = 0; b < n && reg.size() < (size_t)kRegBits; b++) {
                if (done[b] || pops[b].code == OPC_PHASE) continue;
                if ((pass == 0) != ready(b)) continue;
                const int need[2] = {tl(pops[b]), pops[b].t2 >= 0 ? tl_of[pops[b].t2] : -1};
                const int nn = need[1] >= 0 ? 2 : 1;
                bool skip = false;
                for (int i = 0; i < nn; i++) skip |= store && (need[i] == lb[1] || need[i] == lb[2]);
                if (skip) continue;
                int add[2], na = 0;
                for (int i = 0; i < nn; i++)
                    if (std::find(reg.begin(), reg.end(), need[i]) == reg.end()) add[na++] = need[i];
                if (reg.size() + na > (size_t)kRegBits) continue;  // a block needs both of its bits at once
                for (int i = 0; i < na; i++) reg.push_back(add[i]);
            }
        for (int t = 3; reg.size() < (size_t)kRegBits && t < kTileBits; t++)
            if (std::find(reg.begin(), reg.end(), t) == reg.end()) reg.push_back(t);
    };
    std::vector<int> reg;
    upcoming(true, reg);
    Cfg cfg = make_cfg(reg, true);
    cfg0 = cfg.pack();
    auto emit_trans = [&](const Cfg &nc) {
        KOp tr{};
        tr.code = OPC_TRANS;
        tr.cfg = nc.pack();
        st.ops.push_back(tr);
        st.op_gate.push_back(-1);
        st.op_t.push_back(-1);
        st.op_t2.push_back(-1);
        st.op_cm.push_back(0);
        st.op_cv.push_back(0);
    };
    size_t left = n;
    while (left) {
        size_t pick = n;
        for (size_t b = 0; b < n; b++) {
            if (done[b] || !ready(b)) continue;
            if (pops[b].code == OPC_PHASE || in_regs(cfg, pops[b])) { pick = b; break; }
        }
        if (pick == n) {
            // If one store-capable config (tile bit 0 in a register, bits 1, 2
            // on lanes) can host every remaining op, use it: the pass then ends
            // without the re-layout back to a store config.
            std::vector<int> need;
            bool store_fits = true;
            for (size_t b = 0; b < n && store_fits; b++) {
                if (done[b] || pops[b].code == OPC_PHASE) continue;
                for (int t : {tl(pops[b]), pops[b].t2 >= 0 ? tl_of[pops[b].t2] : -1}) {
                    if (t < 0) continue;
                    if (t == sb[1] || t == sb[2]) store_fits = false;
                    if (t != sb[0] && std::find(need.begin(), need.end(), t) == need.end()) need.push_back(t);
                }
            }
            if (store_fits && need.size() <= (size_t)kRegBits - 1) {
                std::vector<int> r{sb[0]};
                for (int t : need) r.push_back(t);
                for (int t = 0; r.size() < (size_t)kRegBits && t < kTileBits; t++)
                    if (t != sb[1] && t != sb[2] && std::find(r.begin(), r.end(), t) == r.end()) r.push_back(t);
                cfg = make_cfg(r, true, sb);
            } else {
                upcoming(false, reg);
                cfg = make_cfg(reg, false);
            }
            emit_trans(cfg);
            continue;
        }
        const POp &p = pops[pick];
        KOp op{};
        op.code = p.code;
        int j = 0;
        if (p.code != OPC_PHASE) {
            cfg.role_of(tl(p), j);
            op.k = j;
        }
        for (int k = 0; k < 8; k++) op.m[k] = p.m[k];
        if (p.code == OPC_U4) {
            // register bits k < k2; 4x4 index bit 0 <-> register bit k
            int j2 = 0;
            cfg.role_of(tl_of[p.t2], j2);
            const bool flip = j > j2;
            int pt = p.t, pt2 = p.t2;
            if (flip) { std::swap(j, j2); std::swap(pt, pt2); }
            auto perm = [&](int x) { return flip ? ((x & 1) << 1) | (x >> 1) : x; };
            KOp rows[4];
            for (int r = 0; r < 4; r++) {
                rows[r] = KOp{};
                rows[r].code = r ? OPC_DATA : OPC_U4;
                for (int q = 0; q < 4; q++) {
                    rows[r].m[2 * q] = p.m4[8 * perm(r) + 2 * perm(q)];
                    rows[r].m[2 * q + 1] = p.m4[8 * perm(r) + 2 * perm(q) + 1];
                }
            }
            rows[0].k = j;
            rows[0].cfg = (uint64_t)j2;
            for (int r = 0; r < 4; r++) {
                st.ops.push_back(rows[r]);
                st.op_gate.push_back(r ? -1 : p.gid);
                st.op_t.push_back(r ? -1 : pt);
                st.op_t2.push_back(r ? -1 : pt2);
                st.op_cm.push_back(0);
                st.op_cv.push_back(0);
            }
            finish(pick);
            left--;
            continue;
        }
        for (int b = 0; b < 64; b++) {
            if (!((p.cm >> b) & 1)) continue;
            const uint32_t v = (uint32_t)((p.cv >> b) & 1);
            const int t = tl_of[b];
            int role = t >= 0 ? cfg.role_of(t, j) : -1;
            if (role == ROLE_REG) { op.mreg |= 1u << j; op.vreg |= v << j; }
            else if (role == ROLE_LANE) { op.mlane |= 1u << j; op.vlane |= v << j; }
            else if (role == ROLE_WARP) { op.mwarp |= 1u << j; op.vwarp |= v << j; }
            else { op.mout |= 1ULL << b; op.vout |= (uint64_t)v << b; }
        }
        st.ops.push_back(op);
        st.op_gate.push_back(p.gid);
        st.op_t.push_back(p.code == OPC_PHASE ? -1 : p.t);
        st.op_t2.push_back(-1);
        st.op_cm.push_back(p.cm);
        st.op_cv.push_back(p.cv);
        finish(pick);
        left--;
    }
    // mark runs of consecutive phases for angle accumulation (JIT tier)
    for (size_t a = 0; a < st.ops.size();) {
        size_t b = a;
        while (b < st.ops.size() && st.ops[b].code == OPC_PHASE) b++;
        if (b - a < (size_t)kPhaseRunMin) {
            a = b == a ? a + 1 : b;
            continue;
        }
        const PhaseRunPlan pr = plan_phase_run(st.ops.data() + a, b - a);
        const double direct = pr.direct, acc = pr.acc;
        if (b - a >= (size_t)kPhaseRunMin && acc < 0.8 * direct) {
            for (size_t o = a; o < b; o++) {
                KOp &op = st.ops[o];
                op.code = OPC_PHASE_ACC;
                double t = std::atan2(op.m[1], op.m[0]) / (2.0 * M_PI);  // turns in (-1/2, 1/2]
                if (t < 0) t += 1.0;
                const long double scaled = (long double)t * 18446744073709551616.0L;
                op.cfg = scaled >= 18446744073709551615.0L ? 0 : (uint64_t)(scaled + 0.5L);
            }
            KOp fl{};
            fl.code = OPC_PHASE_FLUSH;
            st.ops.insert(st.ops.begin() + b, fl);
            st.op_gate.insert(st.op_gate.begin() + b, -1);
            st.op_t.insert(st.op_t.begin() + b, -1);
            st.op_t2.insert(st.op_t2.begin() + b, -1);
            st.op_cm.insert(st.op_cm.begin() + b, 0);
            st.op_cv.insert(st.op_cv.begin() + b, 0);
            b++;
        }
        a = b == a ? a + 1 : b;
    }
    if (!cfg.store_ok(sb)) {
        std::vector<int> r2;
        for (int k = 0; k < kRegBits; k++)
            if (cfg.r[k] != sb[1] && cfg.r[k] != sb[2]) r2.push_back(cfg.r[k]);
        for (int t = 0; r2.size() < (size_t)kRegBits && t < kTileBits; t++)
            if (t != sb[1] && t != sb[2] && std::find(r2.begin(), r2.end(), t) == r2.end()) r2.push_back(t);
        if (std::find(r2.begin(), r2.end(), sb[0]) == r2.end()) { r2.insert(r2.begin(), sb[0]); r2.pop_back(); }
        emit_trans(make_cfg(r2, true, sb));
    }
}

// The gate-collection loop of a pass (mutates done[], sigma for absorbed SWAP
// relabels, and fills pops/freeb/in_tile).  pops == nullptr: dry run for the
// low-qubit look-ahead (counts only).  Returns the number of gates taken.
static size_t collect_pass(Planner &P, const std::vector<GateRec> &gates, std::vector<char> &done, size_t first,
                           const PlanOptions &opt, std::vector<POp> *pops, std::vector<int> &freeb, bool in_tile[64],
                           std::vector<std::pair<int, int>> *relabels)
{
    const int n = P.n, M = P.M;
    std::vector<int> &phys_of = P.phys_of;
    const uint64_t all = n >= 64 ? ~0ULL : (bit(n) - 1);
    uint64_t bN = 0, bD = 0;
    int scanned = 0;
    size_t taken = 0, npops = 0, pbytes = 0;
    const size_t max_pops = kMaxPassPops;
    // count an op (a dry run builds no POp)
    auto account = [&](int code, uint64_t cm) {
        npops++;
        // parameter bytes the JIT tier will need for it (upper estimate)
        pbytes += (code == OPC_U4 ? 256 : code == OPC_PHASE ? 16 : 64) + (cm ? 16 : 0);
    };
    for (size_t i = first; i < gates.size() && scanned < opt.max_scan && npops + 2 <= max_pops &&
                           pbytes + 512 <= (size_t)kPassParamBudget;
         i++) {
        if (done[i]) continue;
        scanned++;
        const GateRec &g = gates[i];
        auto block = [&]() { bN |= g.qN; bD |= g.qD; };
        if ((g.qN & (bN | bD)) || (g.qD & bN)) {
            block();
            if ((bN & all) == all) break;
            continue;
        }
        if (g.kind == GK_SWAP) {
            P.swap_layout(phys_of[g.targets[0]], phys_of[g.targets[1]]);
            if (relabels) relabels->push_back({g.targets[0], g.targets[1]});
            done[i] = 1;
            continue;
        }
        if (g.kind == GK_PERM) { block(); continue; }
        if (g.kind == GK_U4) {
            const int t0 = phys_of[g.targets[0]], t1 = phys_of[g.targets[1]];
            if (t0 >= M || t1 >= M) { block(); continue; }
            const int extra = (!in_tile[t0]) + (!in_tile[t1]);
            if ((int)freeb.size() + extra > kTileBits - 3) { block(); continue; }
            for (int t : {t0, t1})
                if (!in_tile[t]) { in_tile[t] = true; freeb.push_back(t); }
            account(OPC_U4, 0);
            if (pops) {
                POp p{};
                p.code = OPC_U4;
                p.t = t0;
                p.t2 = t1;
                for (int k = 0; k < 32; k++) p.m4[k] = g.u4[k];
                p.gid = g.id;
                pops->push_back(p);
            }
            done[i] = 1;
            taken++;
            continue;
        }
        uint64_t cm = 0;
        for (int c : g.controls) cm |= bit(phys_of[c]);
        if (g.cls == CLS_DIAG) {
            uint64_t tb = bit(phys_of[g.target]);
            for (int side = 0; side < 2; side++) {
                const double fr = g.u[side ? 6 : 0], fi = g.u[side ? 7 : 1];
                if (fr == 1 && fi == 0) continue;
                account(OPC_PHASE, cm | tb);
                if (!pops) continue;
                POp p{};
                p.code = OPC_PHASE;
                p.gid = g.id;
                p.t = -1;
                p.cm = cm | tb; p.cv = cm | (side ? tb : 0); p.m[0] = fr; p.m[1] = fi;
                pops->push_back(p);
            }
            done[i] = 1;
            taken++;
            continue;
        }
        int t = phys_of[g.target];
        if (t >= M) { block(); continue; }
        if (!in_tile[t]) {
            if ((int)freeb.size() >= kTileBits - 3) { block(); continue; }
            in_tile[t] = true;
            freeb.push_back(t);
        }
        account(OPC_U2, cm);
        if (pops) {
            POp p{};
            set_u2_code(g, p);
            p.t = t;
            p.cm = p.cv = cm;
            p.gid = g.id;
            pops->push_back(p);
        }
        done[i] = 1;
        taken++;
    }
    return taken;
}

void Planner::build_pass(const std::vector<GateRec> &gates, std::vector<char> &done, size_t first,
                         const PlanOptions &opt, std::vector<Step> &out)
{
    std::vector<POp> pops;
    std::vector<int> freeb;
    bool in_tile[64] = {false};
    in_tile[0] = in_tile[1] = in_tile[2] = true;
    std::vector<std::pair<int, int>> relabels;
    static const int win_env = [] {
        const char *v = getenv("QSIM_PLAN_WINDOWS");
        return v ? atoi(v) : -1;
    }();
    if (win_env == 1 || (win_env < 0 && G > 0)) {
        // Sharded plans: after an exchange the first not-done gates of a
        // nearest-neighbour circuit (a chain's staircase) sit on qubits spread
        // over the register, and the greedy first-use order fills the tile with
        // them, so each pass advances the front only a little (config-5 family
        // at 36 q / 8 ranks: ~20 gates per pass).  Candidate tiles: the greedy
        // one and windows of consecutive logical qubits starting at the first
        // frontier qubits; each is scored by a dry run of the collection and the
        // window is preset when it takes clearly more gates.
        auto dry = [&](const std::vector<int> &preset) {
            Planner Q = *this;
            std::vector<char> d2 = done;
            std::vector<int> fb = preset;
            bool it[64] = {false};
            it[0] = it[1] = it[2] = true;
            for (int b : preset) it[b] = true;
            return collect_pass(Q, gates, d2, first, opt, nullptr, fb, it, nullptr);
        };
        const size_t base_score = dry({});
        std::vector<int> front;  // logical qubits of the first not-done non-diagonal gates, in order
        for (size_t i = first; i < gates.size() && front.size() < 8; i++) {
            if (done[i]) continue;
            for (int q = 0; q < n && front.size() < 8; q++)
                if (((gates[i].qN >> q) & 1) && std::find(front.begin(), front.end(), q) == front.end()) front.push_back(q);
        }
        size_t best = base_score;
        std::vector<int> best_w;
        for (int f : front)
            for (int off : {0, -3, -6}) {
                std::vector<int> w;
                for (int q = std::max(0, f + off); q < n && (int)w.size() < kTileBits - 3; q++) {
                    const int pb = phys_of[q];
                    if (pb >= 3 && pb < M) w.push_back(pb);
                }
                if ((int)w.size() < kTileBits - 3) continue;
                const size_t sc = dry(w);
                if (sc > best) { best = sc; best_w = w; }
            }
        if (!best_w.empty() && best >= base_score + base_score / 4 + 2) {
            freeb = best_w;
            for (int b : best_w) in_tile[b] = true;
        }
    }
    collect_pass(*this, gates, done, first, opt, &pops, freeb, in_tile, &relabels);
    // tile: physical bits 0,1,2 + the free bits (first-use order), filled up to 12
    std::vector<int> order;
    for (const POp &p : pops)
        for (int t : {p.code == OPC_PHASE ? -1 : p.t, p.t2})
            if (t >= 3 && std::find(order.begin(), order.end(), t) == order.end()) order.push_back(t);
    for (int b : freeb)
        if (std::find(order.begin(), order.end(), b) == order.end()) order.push_back(b);
    for (int p = 3; (int)order.size() < kTileBits - 3 && p < M; p++)
        if (!in_tile[p]) { in_tile[p] = true; order.push_back(p); }

    Step st;
    st.type = ST_PASS;
    PassDesc &d = st.pass;
    int tl_of[64];
    for (int b = 0; b < 64; b++) tl_of[b] = -1;
    for (int t = 0; t < 3; t++) { d.tp[t] = t; tl_of[t] = t; }
    for (int j = 0; j < kTileBits - 3; j++) { d.tp[3 + j] = order[j]; tl_of[order[j]] = 3 + j; }
    if (opt.block_fusion) fuse_blocks(pops, tl_of);
    // The next pass's low qubits.  Every tile contains physical bits 0, 1, 2
    // (whole 128-B lines per warp access), so whatever logical qubits sit
    // there occupy three of each tile's twelve bits.  The pass stores the
    // three tile qubits the remaining gates need first at physical bits
    // 0, 1, 2 (a permutation of the tile's own bit positions, free at the
    // store), and sigma follows.  Which three: the triple whose
    // next pass (a dry run of the collection) takes the most gates, among
    // the first remap_lookahead tile qubits the remaining gates need.
    int sb[3] = {0, 1, 2};
    for (int t = 0; t < kTileBits; t++) d.tp_out[t] = d.tp[t];
    // store the tile so that logical qubits q3[k] land at physical bit k
    auto remap_low = [&](Planner &Q, const int q3[3], int *tp_out, int *sbits) {
        int dest[kTileBits];
        for (int t = 0; t < kTileBits; t++) dest[t] = d.tp[t];
        for (int k = 0; k < 3; k++) {
            sbits[k] = tl_of[Q.phys_of[q3[k]]];
            int tk = 0;
            while (dest[tk] != k) tk++;
            std::swap(dest[sbits[k]], dest[tk]);
        }
        int was[kTileBits];
        for (int t = 0; t < kTileBits; t++) was[t] = Q.qubit_at[d.tp[t]];
        for (int t = 0; t < kTileBits; t++) {
            if (tp_out) tp_out[t] = dest[t];
            Q.qubit_at[dest[t]] = was[t];
            Q.phys_of[was[t]] = dest[t];
        }
    };
    if (opt.low_remap) {
        // candidates: tile qubits in the order the remaining gates need them
        // (non-diagonally), then the current low qubits, then the rest
        const size_t K = (size_t)std::max(3, opt.remap_lookahead);
        std::vector<int> cand;
        auto in_tile_q = [&](int q) { return phys_of[q] < M && tl_of[phys_of[q]] >= 0; };
        auto add = [&](int q) {
            if (cand.size() < K && in_tile_q(q) && std::find(cand.begin(), cand.end(), q) == cand.end()) cand.push_back(q);
        };
        for (size_t i = first; i < gates.size() && cand.size() < K; i++) {
            if (done[i]) continue;
            for (int q = 0; q < n; q++)
                if ((gates[i].qN >> q) & 1) add(q);
        }
        for (int t = 0; t < 3; t++) add(qubit_at[t]);
        for (int t = 0; t < kTileBits && cand.size() < 3; t++) add(qubit_at[d.tp[t]]);
        int best[3] = {cand[0], cand[1], cand[2]};
        size_t next_first = first;
        while (next_first < gates.size() && done[next_first]) next_first++;
        if (opt.remap_lookahead > 3 && next_first < gates.size()) {
            // one-pass look-ahead: the triple whose next pass takes the most gates
            size_t best_score = 0;
            bool have = false;
            for (size_t a = 0; a < cand.size(); a++)
                for (size_t b = a + 1; b < cand.size(); b++)
                    for (size_t c = b + 1; c < cand.size(); c++) {
                        Planner Q = *this;
                        const int q3[3] = {cand[a], cand[b], cand[c]};
                        int sbq[3];
                        remap_low(Q, q3, nullptr, sbq);
                        std::vector<char> done2 = done;
                        std::vector<int> fb;
                        bool it[64] = {false};
                        it[0] = it[1] = it[2] = true;
                        const size_t score = collect_pass(Q, gates, done2, next_first, opt, nullptr, fb, it, nullptr);
                        if (!have || score > best_score) {
                            best_score = score;
                            have = true;
                            for (int k = 0; k < 3; k++) best[k] = q3[k];
                        }
                    }
        }
        remap_low(*this, best, d.tp_out, sb);
    }
    uint64_t cfg0 = 0;
    lower_pass(pops, tl_of, st, cfg0, sb);
    d.cfg0 = cfg0;
    d.M = M;
    d.n_inst = 1ULL << (M - kTileBits);
    d.n_ops = (int)st.ops.size();
    d.use_smem = 0;
    for (const KOp &k : st.ops)
        if (k.code == OPC_TRANS) d.use_smem = 1;
    int tiles[kTileBits];
    for (int j = 0; j < kTileBits; j++) tiles[j] = d.tp[j];
    std::sort(tiles, tiles + kTileBits);
    for (int j = 0; j < kTileBits; j++) d.tile_sorted[j] = tiles[j];
    out.push_back(std::move(st));
    for (auto &r : relabels) {
        Step s;
        s.type = ST_RELABEL;
        s.ra = r.first;
        s.rb = r.second;
        out.push_back(s);
    }
}

void Planner::emit_generic(const GateRec &g, std::vector<Step> &out)
{
    uint64_t cm = 0;
    for (int c : g.controls) cm |= bit(phys_of[c]);
    if (g.cls == CLS_DIAG) {
        uint64_t tb = bit(phys_of[g.target]);
        for (int side = 0; side < 2; side++) {
            double fr = g.u[side ? 6 : 0], fi = g.u[side ? 7 : 1];
            if (fr == 1 && fi == 0) continue;
            Step s;
            s.type = ST_PHASE;
            s.cm = cm | tb;
            s.cv = cm | (side ? tb : 0);
            s.m[0] = fr;
            s.m[1] = fi;
            s.gate_id = g.id;
            out.push_back(s);
        }
        return;
    }
    Step s;
    s.type = ST_GENERIC;
    s.code = g.cls == CLS_XS ? OPC_XS : g.cls == CLS_REAL ? OPC_U2R : OPC_U2;
    s.t = phys_of[g.target];
    s.cm = s.cv = cm;
    for (int k = 0; k < 8; k++) s.m[k] = g.u[k];
    s.gate_id = g.id;
    out.push_back(s);
}

void Planner::emit_perm(const GateRec &g, std::vector<Step> &out)
{
    Step s;
    s.type = ST_PERM;
    for (int c : g.controls) s.cm |= bit(phys_of[c]);
    s.cv = s.cm;
    for (int t : g.targets) s.ptargets.push_back(phys_of[t]);
    s.perm = g.perm;
    s.gate_id = g.id;
    out.push_back(std::move(s));
}

// Consecutive permutations of the same register (Shor's modular
// multiplications) become one step: one HBM pass instead of one per gate.
size_t Planner::emit_perm_run(const std::vector<GateRec> &gates, std::vector<char> &done, size_t first,
                              std::vector<Step> &out)
{
    const GateRec &g = gates[first];
    std::vector<size_t> run{first};
    const int t = (int)g.targets.size();
    for (size_t i = first + 1; i < gates.size() && run.size() < (size_t)kMaxPermRun; i++) {
        if (done[i]) continue;
        const GateRec &h = gates[i];
        if (h.kind != GK_PERM || h.targets != g.targets) break;
        if (perm_run_smem_bytes(t, t, (int)run.size() + 1) > kPermRunSmemMax) break;  // tables + tiles fit one CTA
        run.push_back(i);
    }
    if (run.size() < 2 || g.targets.size() > 16) {
        emit_perm(g, out);
        done[first] = 1;
        return 1;
    }
    Step s;
    s.type = ST_PERMRUN;
    for (int t : g.targets) s.ptargets.push_back(phys_of[t]);
    for (size_t i : run) {
        const GateRec &h = gates[i];
        uint64_t cm = 0;
        for (int c : h.controls) cm |= bit(phys_of[c]);
        s.run_cm.push_back(cm);
        s.run_gate.push_back(h.id);
        s.perm.insert(s.perm.end(), h.perm.begin(), h.perm.end());
        done[i] = 1;
    }
    s.gate_id = g.id;
    out.push_back(std::move(s));
    return run.size();
}

void Planner::emit_exchange(const std::vector<GateRec> &gates, const std::vector<char> &done, size_t first,
                            std::vector<Step> &out)
{
    std::vector<int> need;
    size_t window = (size_t)8 * n + 16;
    size_t seen = 0;
    for (size_t i = first; i < gates.size() && seen < window && (int)need.size() < G; i++) {
        if (done[i]) continue;
        seen++;
        for (int q = 0; q < n && (int)need.size() < G; q++)
            if (((gates[i].qN >> q) & 1) && phys_of[q] >= M &&
                std::find(need.begin(), need.end(), q) == need.end())
                need.push_back(q);
    }
    // Belady: evict the local qubits whose next non-diagonal use is furthest
    const size_t INF = std::numeric_limits<size_t>::max();
    std::vector<size_t> next_use(n, INF);
    for (size_t i = gates.size(); i-- > first;) {
        if (done[i]) continue;
        for (int q = 0; q < n; q++)
            if ((gates[i].qN >> q) & 1) next_use[q] = i;
    }
    int lo = M >= kTileBits ? 3 : 0;
    std::vector<int> cand;
    for (int p = lo; p < M; p++) cand.push_back(p);
    std::stable_sort(cand.begin(), cand.end(), [&](int a, int b) {
        size_t ua = next_use[qubit_at[a]], ub = next_use[qubit_at[b]];
        if (ua != ub) return ua > ub;
        return a > b;  // prefer the top bits: contiguous exchange blocks
    });
    int K = std::min<int>((int)need.size(), (int)cand.size());
    // Among the 2K furthest-used candidates, prefer victims that are not tile
    // bits of the pass just emitted: that pass can then run block by block
    // under this exchange (runtime overlap), at the price of evicting a qubit
    // used slightly sooner.
    static const int prefer_off_tile = [] { const char *e = getenv("QSIM_PLAN_VICTIM_TILE"); return e ? atoi(e) : 1; }();
    if (prefer_off_tile && !out.empty() && out.back().type == ST_PASS && K > 0) {
        const Step &prev = out.back();
        auto in_tile = [&](int p) {
            for (int t = 0; t < kTileBits; t++)
                if (prev.pass.tp[t] == p || prev.pass.tp_out[t] == p) return true;
            return false;
        };
        const size_t pool = std::min(cand.size(), (size_t)2 * K);
        std::stable_partition(cand.begin(), cand.begin() + pool, [&](int p) { return !in_tile(p); });
    }
    Step s;
    s.type = ST_EXCHANGE;
    for (int i = 0; i < K; i++) {
        s.lpos.push_back(cand[i]);
        s.gpos.push_back(phys_of[need[i]]);
    }
    for (int i = 0; i < K; i++) swap_layout(s.lpos[i], s.gpos[i]);
    out.push_back(std::move(s));
}

// Auto policy: a remap moves half a shard per direction and makes the qubit
// local for every later gate; a pairwise combine moves a whole shard and keeps
// sigma.  Pairwise pays off only for an isolated gate on a global qubit when
// every local qubit a remap could evict is itself needed within the window
// (the remap would have to be undone right away).
bool Planner::prefer_pairwise(const std::vector<GateRec> &gates, const std::vector<char> &done, size_t first) const
{
    const GateRec &g = gates[first];
    const int q = g.target;
    const size_t window = (size_t)4 * n + 8;
    size_t seen = 0;
    int uses = 0;
    uint64_t needed = 0;  // local qubits used non-diagonally in the window
    for (size_t i = first; i < gates.size() && seen < window; i++) {
        if (done[i]) continue;
        seen++;
        if ((gates[i].qN >> q) & 1) uses++;
        needed |= gates[i].qN;
    }
    if (uses > 1) return false;
    const int lo = M >= kTileBits ? 3 : 0;
    for (int p = lo; p < M; p++)
        if (!((needed >> qubit_at[p]) & 1)) return false;  // a free victim exists
    return true;
}

void Planner::remap(const std::vector<int> &local_q, const std::vector<int> &global_q, std::vector<Step> &out)
{
    Step s;
    s.type = ST_EXCHANGE;
    for (size_t i = 0; i < local_q.size(); i++) {
        s.lpos.push_back(phys_of[local_q[i]]);
        s.gpos.push_back(phys_of[global_q[i]]);
    }
    for (size_t i = 0; i < local_q.size(); i++) swap_layout(s.lpos[i], s.gpos[i]);
    out.push_back(std::move(s));
}

// Modelled device time of a planned step list (seconds): a pass costs
// max(FP64 FMA-slot work / FP64 peak, 32 B/amp / HBM peak), a K-pair exchange
// its (2^K-1)/2^K shard share over the link plus the HBM pack/unpack, other
// steps one HBM round trip.  Peaks from PlanOptions: the runtime measures
// FP64 and HBM on its device (qsim_probe_peaks); the link rate is an option.
double plan_cost(const std::vector<Step> &steps, int M, const PlanOptions &opt)
{
    const double amps = std::ldexp(1.0, M), fp64 = opt.peak_fp64, hbm = opt.peak_hbm, nvl = opt.peak_link;
    double t = 0, t_prev_pass = 0;
    const Step *prev = nullptr;
    for (const Step &s : steps) {
        const Step *before = prev;
        prev = &s;
        switch (s.type) {
        case ST_PASS: {
            double f = 0;
            for (const KOp &op : s.ops) {
                const int pb = __builtin_popcount(op.mreg) + __builtin_popcount(op.mlane) +
                               __builtin_popcount(op.mwarp) + __builtin_popcountll(op.mout);
                const double c = op.code == OPC_U2 ? 8 : op.code == OPC_U4 ? 16
                               : (op.code == OPC_U2R || op.code == OPC_PHASE || op.code == OPC_PHASE_ACC) ? 4 : 0;
                f += c * std::ldexp(1.0, -pb);
            }
            t_prev_pass = std::max(2 * f * amps / fp64, 32 * amps / hbm);
            t += t_prev_pass;
            break;
        }
        case ST_EXCHANGE: {
            const int K = (int)s.lpos.size();
            const double share = 1.0 - std::ldexp(1.0, -K);
            const double tx = share * 16 * amps / nvl + 2 * share * 16 * amps / hbm;
            bool ov = opt.overlap && before && before->type == ST_PASS && K >= 1 && K <= 3;
            for (int i = 0; ov && i < kTileBits; i++)
                for (int l : s.lpos)
                    if (before->pass.tp[i] == l || before->pass.tp_out[i] == l) ov = false;
            // overlapped: the pair costs max(pass, exchange) + one block of the pass
            t += ov ? std::max(0.0, tx - t_prev_pass) + t_prev_pass * std::ldexp(1.0, -K) : tx;
            break;
        }
        case ST_PAIRWISE: t += 16 * amps / nvl + 48 * amps / hbm; break;
        case ST_RELABEL: break;
        default: t += 32 * amps / hbm; break;
        }
    }
    return t;
}

void Planner::plan(const std::vector<GateRec> &user_gates, const PlanOptions &opt, std::vector<Step> &out)
{
    const bool fused = opt.fusion && M >= kTileBits;
    if (!fused || !opt.block_fusion) {
        plan_list(user_gates, opt, out);
        return;
    }
    // two-qubit blocks on the whole gate list first (never cut by a pass).
    // No blocks on the initially global qubits: a control or a diagonal gate
    // there is free (no exchange), and an isolated gate there may go pairwise;
    // inside a 4x4 block it would be a non-diagonal target.
    uint64_t no_blocks_on = 0;
    for (int p = M; p < n; p++) no_blocks_on |= bit(qubit_at[p]);
    // Blocks must save FP64 work (cost > 16 + 2).  When that leaves most
    // general one-qubit gates unfused (chain-like circuits, where a U2, CNOT,
    // U2 cluster costs exactly a block's 16), break-even blocks are tried
    // too: same FP64 work, but a block needs no re-layout between its gates
    // and passes hold more of the circuit (config-5 family: 15 -> 10 passes);
    // on other circuits they can cost passes (a QFT adder: 2 -> 3), so the
    // cost model decides.  On a brickwork the strict rule already absorbs
    // every U2 into two-layer blocks and only it is planned.
    auto general_u2 = [](const std::vector<GateRec> &gs) {
        size_t k = 0;
        for (const GateRec &g : gs) k += g.kind == GK_U2 && g.controls.empty() && g.cls == CLS_GENERAL;
        return k;
    };
    std::vector<std::vector<GateRec>> lists;
    lists.push_back(fuse_gates(user_gates, no_blocks_on, 2.0));
    const size_t u2_before = general_u2(user_gates);
    if (u2_before && general_u2(lists[0]) * 4 > u2_before) lists.push_back(fuse_gates(user_gates, no_blocks_on, -0.5));
    // Sharded: tying gates into blocks can change which of them meet a
    // nonlocal qubit (more exchanges): the unblocked list (build_pass still
    // fuses inside each pass) is a candidate too.
    if (G > 0) lists.push_back(user_gates);
    if (opt.force_list >= 0 && opt.force_list < (int)lists.size()) {
        std::vector<GateRec> keep = lists[opt.force_list];
        lists.assign(1, keep);
    }
    if (lists.size() == 1) {
        plan_list(lists[0], opt, out);  // streams its steps (opt.sink)
        return;
    }
    const Planner start = *this;
    PlanOptions o2 = opt;
    o2.sink = nullptr;  // no list is final until all are costed
    std::vector<Step> best;
    Planner after_best = start;
    double best_cost = 0;
    for (size_t i = 0; i < lists.size(); i++) {
        *this = start;
        std::vector<Step> cand;
        plan_list(lists[i], o2, cand);
        const double cost = plan_cost(cand, M, opt);
        if (opt.cand_report) {
            int np = 0, nx = 0;
            for (const Step &st : cand) { np += st.type == ST_PASS; nx += st.type == ST_EXCHANGE || st.type == ST_PAIRWISE; }
            opt.cand_report->push_back("{\"list\":" + std::to_string(i) + ",\"model_s\":" + std::to_string(cost) +
                                       ",\"passes\":" + std::to_string(np) + ",\"exchanges\":" + std::to_string(nx) + "}");
        }
        if (i == 0 || cost < best_cost) {
            best_cost = cost;
            best.swap(cand);
            after_best = *this;
        }
    }
    *this = after_best;
    for (Step &st : best) out.push_back(std::move(st));
    if (opt.sink) opt.sink(out);
}

void Planner::plan_list(const std::vector<GateRec> &gates, const PlanOptions &opt, std::vector<Step> &out)
{
    const bool fused = opt.fusion && M >= kTileBits;
    std::vector<char> done(gates.size(), 0);
    size_t first = 0;
    while (true) {
        if (opt.sink) opt.sink(out);
        while (first < gates.size() && done[first]) first++;
        if (first >= gates.size()) break;
        const GateRec &g = gates[first];
        if (g.kind == GK_SWAP) {
            swap_layout(phys_of[g.targets[0]], phys_of[g.targets[1]]);
            Step s;
            s.type = ST_RELABEL;
            s.ra = g.targets[0];
            s.rb = g.targets[1];
            out.push_back(s);
            done[first] = 1;
            continue;
        }
        bool global_target = false;
        for (int q = 0; q < n; q++)
            if (((g.qN >> q) & 1) && phys_of[q] >= M) global_target = true;
        if (global_target) {
            const bool pw = g.kind == GK_U2 && (opt.global_policy == GP_PAIRWISE ||
                                                (opt.global_policy == GP_AUTO && prefer_pairwise(gates, done, first)));
            if (pw) {
                Step s;
                s.type = ST_PAIRWISE;
                s.code = g.cls == CLS_XS ? OPC_XS : g.cls == CLS_REAL ? OPC_U2R : OPC_U2;
                s.t = phys_of[g.target];
                for (int c : g.controls) s.cm |= bit(phys_of[c]);
                s.cv = s.cm;
                for (int k = 0; k < 8; k++) s.m[k] = g.u[k];
                s.gate_id = g.id;
                out.push_back(s);
                done[first] = 1;
            } else {
                emit_exchange(gates, done, first, out);
            }
            continue;
        }
        if (g.kind == GK_PERM) {
            emit_perm_run(gates, done, first, out);
            continue;
        }
        if (fused) {
            build_pass(gates, done, first, opt, out);
        } else {
            emit_generic(g, out);
            done[first] = 1;
        }
    }
}

// ------------------------------------------------------------------- JSON
std::string plan_to_json(const Planner &P, const std::vector<Step> &steps)
{
    std::ostringstream o;
    o.precision(17);
    o << "{\"n\":" << P.n << ",\"G\":" << P.G << ",\"M\":" << P.M << ",\"final_phys_of\":[";
    for (int q = 0; q < P.n; q++) o << (q ? "," : "") << P.phys_of[q];
    o << "],\"steps\":[";
    for (size_t s = 0; s < steps.size(); s++) {
        const Step &st = steps[s];
        if (s) o << ",";
        switch (st.type) {
        case ST_PASS: {
            o << "{\"type\":\"pass\",\"tile\":[";
            for (int j = 0; j < kTileBits; j++) o << (j ? "," : "") << st.pass.tile_sorted[j];
            o << "],\"tp\":[";
            for (int j = 0; j < kTileBits; j++) o << (j ? "," : "") << st.pass.tp[j];
            o << "],\"tp_out\":[";
            for (int j = 0; j < kTileBits; j++) o << (j ? "," : "") << st.pass.tp_out[j];
            o << "],\"cfg0\":" << st.pass.cfg0 << ",\"ops\":[";
            for (size_t k = 0; k < st.ops.size(); k++) {
                const KOp &op = st.ops[k];
                o << (k ? "," : "") << "{\"gate\":" << st.op_gate[k] << ",\"t\":" << st.op_t[k]
                  << ",\"t2\":" << (k < st.op_t2.size() ? st.op_t2[k] : -1)
                  << ",\"cm\":" << st.op_cm[k] << ",\"cv\":" << st.op_cv[k] << ",\"code\":" << op.code
                  << ",\"k\":" << op.k << ",\"cfg\":" << op.cfg
                  << ",\"mreg\":" << op.mreg << ",\"vreg\":" << op.vreg << ",\"mlane\":" << op.mlane
                  << ",\"vlane\":" << op.vlane << ",\"mwarp\":" << op.mwarp << ",\"vwarp\":" << op.vwarp
                  << ",\"mout\":" << op.mout << ",\"vout\":" << op.vout << ",\"m\":[";
                const int rows = op.code == OPC_U4 ? 4 : 1;  // U4: rows 1..3 in the next ops
                for (int r = 0; r < rows; r++)
                    for (int j = 0; j < 8; j++) o << (r || j ? "," : "") << st.ops[k + r].m[j];
                o << "]}";
            }
            o << "]}";
            break;
        }
        case ST_GENERIC:
        case ST_PHASE:
            o << "{\"type\":\"" << (st.type == ST_GENERIC ? "generic" : "phase") << "\",\"gate\":" << st.gate_id
              << ",\"code\":" << st.code << ",\"t\":" << st.t << ",\"cm\":" << st.cm << ",\"cv\":" << st.cv
              << ",\"m\":[";
            for (int j = 0; j < 8; j++) o << (j ? "," : "") << st.m[j];
            o << "]}";
            break;
        case ST_PERM:
            o << "{\"type\":\"perm\",\"gate\":" << st.gate_id << ",\"cm\":" << st.cm << ",\"targets\":[";
            for (size_t j = 0; j < st.ptargets.size(); j++) o << (j ? "," : "") << st.ptargets[j];
            o << "]}";
            break;
        case ST_PERMRUN:
            o << "{\"type\":\"permrun\",\"gates\":[";
            for (size_t j = 0; j < st.run_gate.size(); j++) o << (j ? "," : "") << st.run_gate[j];
            o << "],\"cms\":[";
            for (size_t j = 0; j < st.run_cm.size(); j++) o << (j ? "," : "") << st.run_cm[j];
            o << "],\"targets\":[";
            for (size_t j = 0; j < st.ptargets.size(); j++) o << (j ? "," : "") << st.ptargets[j];
            o << "]}";
            break;
        case ST_EXCHANGE:
            o << "{\"type\":\"exchange\",\"lpos\":[";
            for (size_t j = 0; j < st.lpos.size(); j++) o << (j ? "," : "") << st.lpos[j];
            o << "],\"gpos\":[";
            for (size_t j = 0; j < st.gpos.size(); j++) o << (j ? "," : "") << st.gpos[j];
            o << "]}";
            break;
        case ST_RELABEL:
            o << "{\"type\":\"relabel\",\"a\":" << st.ra << ",\"b\":" << st.rb << "}";
            break;
        case ST_PAIRWISE:
            o << "{\"type\":\"pairwise\",\"gate\":" << st.gate_id << ",\"code\":" << st.code << ",\"t\":" << st.t
              << ",\"cm\":" << st.cm << ",\"cv\":" << st.cv << ",\"m\":[";
            for (int j = 0; j < 8; j++) o << (j ? "," : "") << st.m[j];
            o << "]}";
            break;
        }
    }
    o << "]}";
    return o.str();
}

}  // namespace qsb
