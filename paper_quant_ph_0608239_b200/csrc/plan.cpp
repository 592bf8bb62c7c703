// plan.cpp -- gate classification, initial layout, fusion/placement planner.
//
// The planner turns the queued LOGICAL gate list into a sequence of device
// steps in PHYSICAL coordinates:
//   * ST_PASS      one fused tile pass (kernels.cu k_pass) applying many gates
//   * ST_GENERIC / ST_PHASE   one gate per launch (small shards, fusion off)
//   * ST_PERM      one controlled register permutation (k_perm)
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
#include <cmath>
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
    } else {
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

// ------------------------------------------------------------------ passes
namespace {
struct POp {
    int code;      // OPC_U2 / OPC_U2R / OPC_XS / OPC_PHASE
    int t;         // physical target (U2-type)
    uint64_t cm, cv;
    double m[8];
    int gid;
};

struct RoleState {
    int rt[3];  // role -> triple
};
}  // namespace

static void set_u2_code(const GateRec &g, POp &p)
{
    p.code = g.cls == CLS_XS ? OPC_XS : g.cls == CLS_REAL ? OPC_U2R : OPC_U2;
    for (int k = 0; k < 8; k++) p.m[k] = g.u[k];
}

// simulate role assignment + transposes; returns cost, fills ops if emit
static int lower_pass(const std::vector<POp> &pops, const int tri[3][3], const int init_rt[3],
                      bool emit, std::vector<KOp> *kops, std::vector<int> *kgate, Step *st = nullptr)
{
    int where[64];  // physical bit -> triple index (or -1)
    int widx[64];
    for (int p = 0; p < 64; p++) where[p] = -1, widx[p] = 0;
    for (int x = 0; x < 3; x++)
        for (int j = 0; j < 3; j++) { where[tri[x][j]] = x; widx[tri[x][j]] = j; }
    int rt[3] = {init_rt[0], init_rt[1], init_rt[2]};
    auto role_of = [&](int x) {
        for (int r = 0; r < 3; r++)
            if (rt[r] == x) return r;
        return -1;
    };
    int cost = 0;
    for (size_t o = 0; o < pops.size(); o++) {
        const POp &p = pops[o];
        int role = -1, k = 0;
        if (p.code != OPC_PHASE) {
            int t = p.t;
            if (t == 0) { role = ROLE_REG; k = 0; }
            else if (t == 1 || t == 2) { role = ROLE_LANE; k = t - 1; }
            else {
                int x = where[t];
                role = role_of(x);
                if (role == ROLE_WARP) {
                    // evict the role whose triple is needed furthest ahead
                    int best = ROLE_REG;
                    size_t bestd = 0;
                    for (int pr = ROLE_REG; pr <= ROLE_LANE; pr++) {
                        int xx = rt[pr];
                        size_t d = pops.size() + 1;
                        for (size_t q = o + 1; q < pops.size(); q++)
                            if (pops[q].code != OPC_PHASE && where[pops[q].t] == xx) { d = q - o; break; }
                        if (d > bestd || (d == bestd && pr == ROLE_LANE)) { bestd = d; best = pr; }
                    }
                    if (emit) {
                        KOp tr{};
                        tr.code = OPC_TRANS;
                        tr.ta = ROLE_WARP;
                        tr.tb = best;
                        kops->push_back(tr);
                        kgate->push_back(-1);
                        st->op_t.push_back(-1);
                        st->op_cm.push_back(0);
                        st->op_cv.push_back(0);
                    }
                    std::swap(rt[ROLE_WARP], rt[best]);
                    cost += 4;
                    role = best;
                }
                k = (role == ROLE_REG ? 1 : 2) + widx[t];
            }
            if (role == ROLE_LANE) cost += 1;
        }
        if (!emit) continue;
        KOp op{};
        op.code = p.code;
        op.role = role;
        op.k = k;
        for (int j = 0; j < 8; j++) op.m[j] = p.m[j];
        // split the predicate over the roles
        for (int b = 0; b < 64; b++) {
            if (!((p.cm >> b) & 1)) continue;
            uint32_t v = (uint32_t)((p.cv >> b) & 1);
            if (b == 0) { op.mreg |= 1u; op.vreg |= v; }
            else if ((b == 1 || b == 2)) { op.mlane |= 1u << (b - 1); op.vlane |= v << (b - 1); }
            else if (where[b] >= 0) {
                int r = role_of(where[b]), j = widx[b];
                if (r == ROLE_REG) { op.mreg |= 1u << (1 + j); op.vreg |= v << (1 + j); }
                else if (r == ROLE_LANE) { op.mlane |= 1u << (2 + j); op.vlane |= v << (2 + j); }
                else { op.mwarp |= 1u << j; op.vwarp |= v << j; }
            } else {
                op.mout |= 1ULL << b;
                op.vout |= (uint64_t)v << b;
            }
        }
        kops->push_back(op);
        kgate->push_back(p.gid);
        st->op_t.push_back(p.code == OPC_PHASE ? -1 : p.t);
        st->op_cm.push_back(p.cm);
        st->op_cv.push_back(p.cv);
    }
    return cost;
}

void Planner::build_pass(const std::vector<GateRec> &gates, std::vector<char> &done, size_t first,
                         const PlanOptions &opt, std::vector<Step> &out)
{
    std::vector<POp> pops;
    std::vector<int> freeb;
    bool in_tile[64] = {false};
    in_tile[0] = in_tile[1] = in_tile[2] = true;
    const uint64_t all = n >= 64 ? ~0ULL : (bit(n) - 1);
    uint64_t bN = 0, bD = 0;
    int scanned = 0;
    std::vector<std::pair<int, int>> relabels;
    // each op may need a transpose in front of it: keep the lowered pass within kMaxPassOps
    const size_t max_pops = kMaxPassOps / 2;
    for (size_t i = first; i < gates.size() && scanned < opt.max_scan && pops.size() + 2 <= max_pops; i++) {
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
            swap_layout(phys_of[g.targets[0]], phys_of[g.targets[1]]);
            relabels.push_back({g.targets[0], g.targets[1]});
            done[i] = 1;
            continue;
        }
        if (g.kind == GK_PERM) { block(); continue; }
        uint64_t cm = 0;
        for (int c : g.controls) cm |= bit(phys_of[c]);
        if (g.cls == CLS_DIAG) {
            uint64_t tb = bit(phys_of[g.target]);
            POp p{};
            p.code = OPC_PHASE;
            p.gid = g.id;
            p.t = -1;
            if (!(g.u[0] == 1 && g.u[1] == 0)) {
                p.cm = cm | tb; p.cv = cm; p.m[0] = g.u[0]; p.m[1] = g.u[1];
                pops.push_back(p);
            }
            if (!(g.u[6] == 1 && g.u[7] == 0)) {
                p.cm = cm | tb; p.cv = cm | tb; p.m[0] = g.u[6]; p.m[1] = g.u[7];
                pops.push_back(p);
            }
            done[i] = 1;
            continue;
        }
        int t = phys_of[g.target];
        if (t >= M) { block(); continue; }
        if (!in_tile[t]) {
            if ((int)freeb.size() >= 9) { block(); continue; }
            in_tile[t] = true;
            freeb.push_back(t);
        }
        POp p{};
        set_u2_code(g, p);
        p.t = t;
        p.cm = p.cv = cm;
        p.gid = g.id;
        pops.push_back(p);
        done[i] = 1;
    }
    // order free bits by first use, then fill the tile
    std::vector<int> order;
    for (const POp &p : pops)
        if (p.code != OPC_PHASE && p.t >= 3 &&
            std::find(order.begin(), order.end(), p.t) == order.end())
            order.push_back(p.t);
    for (int p = 3; (int)order.size() < 9 && p < M; p++)
        if (!in_tile[p]) { in_tile[p] = true; order.push_back(p); }
    for (int b : freeb)
        if (std::find(order.begin(), order.end(), b) == order.end()) order.push_back(b);

    Step st;
    st.type = ST_PASS;
    int tri[3][3];
    for (int x = 0; x < 3; x++)
        for (int j = 0; j < 3; j++) tri[x][j] = order[3 * x + j];
    // choose the initial role assignment with the lowest simulated cost
    static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    int best = 0, bestc = 1 << 30;
    for (int a = 0; a < 6; a++) {
        int c = lower_pass(pops, tri, perms[a], false, nullptr, nullptr);
        if (c < bestc) { bestc = c; best = a; }
    }
    lower_pass(pops, tri, perms[best], true, &st.ops, &st.op_gate, &st);
    PassDesc &d = st.pass;
    d.M = M;
    d.n_inst = 1ULL << (M - kTileBits);
    d.op_begin = 0;
    d.n_ops = (int)st.ops.size();
    d.use_smem = 0;
    for (const KOp &k : st.ops)
        if (k.code == OPC_TRANS) d.use_smem = 1;
    for (int x = 0; x < 3; x++)
        for (int j = 0; j < 3; j++) d.tri[x][j] = tri[x][j];
    for (int r = 0; r < 3; r++) d.role_tri[r] = perms[best][r];
    int tiles[kTileBits] = {0, 1, 2};
    for (int j = 0; j < 9; j++) tiles[3 + j] = order[j];
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
    Step s;
    s.type = ST_EXCHANGE;
    for (int i = 0; i < K; i++) {
        s.lpos.push_back(cand[i]);
        s.gpos.push_back(phys_of[need[i]]);
    }
    for (int i = 0; i < K; i++) swap_layout(s.lpos[i], s.gpos[i]);
    out.push_back(std::move(s));
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

void Planner::plan(const std::vector<GateRec> &gates, const PlanOptions &opt, std::vector<Step> &out)
{
    std::vector<char> done(gates.size(), 0);
    size_t first = 0;
    const bool fused = opt.fusion && M >= kTileBits;
    while (true) {
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
            emit_exchange(gates, done, first, out);
            continue;
        }
        if (g.kind == GK_PERM) {
            emit_perm(g, out);
            done[first] = 1;
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
            o << "],\"tri\":[";
            for (int x = 0; x < 3; x++)
                for (int j = 0; j < 3; j++) o << (x + j ? "," : "") << st.pass.tri[x][j];
            o << "],\"role_tri\":[" << st.pass.role_tri[0] << "," << st.pass.role_tri[1] << ","
              << st.pass.role_tri[2] << "],\"ops\":[";
            for (size_t k = 0; k < st.ops.size(); k++) {
                const KOp &op = st.ops[k];
                o << (k ? "," : "") << "{\"gate\":" << st.op_gate[k] << ",\"t\":" << st.op_t[k]
                  << ",\"cm\":" << st.op_cm[k] << ",\"cv\":" << st.op_cv[k] << ",\"code\":" << op.code
                  << ",\"role\":" << op.role << ",\"k\":" << op.k << ",\"ta\":" << op.ta << ",\"tb\":" << op.tb
                  << ",\"mreg\":" << op.mreg << ",\"vreg\":" << op.vreg << ",\"mlane\":" << op.mlane
                  << ",\"vlane\":" << op.vlane << ",\"mwarp\":" << op.mwarp << ",\"vwarp\":" << op.vwarp
                  << ",\"mout\":" << op.mout << ",\"vout\":" << op.vout << ",\"m\":[";
                for (int j = 0; j < 8; j++) o << (j ? "," : "") << op.m[j];
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
        }
    }
    o << "]}";
    return o.str();
}

}  // namespace qsb
