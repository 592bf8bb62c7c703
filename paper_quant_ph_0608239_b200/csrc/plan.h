// plan.h -- host-side gate queue classification and the fusion / placement
// planner.  Pure C++, no CUDA.
#pragma once
#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "engine.h"

namespace qsb {

enum GateKind { GK_U2 = 0, GK_PERM = 2, GK_SWAP = 3, GK_U4 = 4 /* planner-made fused block */ };
enum GateClass { CLS_GENERAL = 0, CLS_REAL = 1, CLS_DIAG = 2, CLS_XS = 3 };

// A validated gate in LOGICAL qubits.
struct GateRec {
    int kind = GK_U2;
    int target = -1;                  // U2
    std::vector<int> controls;
    std::vector<int> targets;         // PERM (register order) / SWAP (2) / U4 (index bits 0, 1)
    double u[8] = {1, 0, 0, 0, 0, 0, 1, 0};
    double u4[32] = {0};              // U4: row-major complex 4x4
    int cls = CLS_GENERAL;
    std::vector<uint32_t> perm;
    uint64_t qN = 0;  // logical qubits acted on non-diagonally
    uint64_t qD = 0;  // logical qubits acted on only diagonally (controls, diag target)
    int id = 0;       // position in the user's sequence
};

void classify(GateRec &g);  // sets cls, qN, qD

// Phase runs (engine.h OPC_PHASE_ACC): register predicate (i & m) == v expands
// into monomials x^S = prod_{b in S} i_b over the 4 register bits; an op adds
// its angle to acc[S] (sign (-1)^|T|, S = O | T, T subset of the zero bits).
// The flush applies e^{i theta_i}, theta_i = sum_{S subset of i} acc[S], either
// per distinct register angle (mode A) or per monomial (mode B).
struct PhaseRunPlan {
    uint32_t used = 0;      // monomials S (bit S of the 16-bit set) with an accumulator
    double direct = 0;      // FP64-pipe ops per thread applying the run op by op
    double acc = 0;         // integer adds + flush (cheaper mode)
    int mode = 0;           // 0: per register angle, 1: per monomial
};
PhaseRunPlan plan_phase_run(const KOp *ops, size_t n);

enum StepType { ST_PASS = 0, ST_GENERIC = 1, ST_PHASE = 2, ST_PERM = 3, ST_EXCHANGE = 4, ST_RELABEL = 5, ST_PAIRWISE = 6,
                ST_PERMRUN = 7 };

// global-target policy: remap (K-pair interchange),
// pairwise (partner shards combine, sigma unchanged), or auto
enum GlobalPolicy { GP_REMAP = 0, GP_PAIRWISE = 1, GP_AUTO = 2 };

struct Step {
    int type = ST_PASS;
    // ST_PASS
    PassDesc pass{};              // op_begin relative to this step's ops
    std::vector<KOp> ops;
    std::vector<int> op_gate;     // gate id behind each op (-1 for TRANS)
    std::vector<int> op_t;        // physical target of each op (-1: PHASE/TRANS)
    std::vector<int> op_t2;       // OPC_U4: physical bit of 4x4 index bit 1 (else -1)
    std::vector<uint64_t> op_cm, op_cv;  // full-index predicate of each op (for introspection)
    // ST_GENERIC: one U2 on physical target t, controls (full-index mask/val)
    // ST_PAIRWISE: one U2 on GLOBAL physical target t (partner shards combine)
    // ST_PHASE  : multiply by f where (full & mask) == val
    int code = OPC_U2;
    int t = -1;
    uint64_t cm = 0, cv = 0;
    double m[8] = {0};
    int gate_id = -1;
    // ST_PERM / ST_PERMRUN
    std::vector<int> ptargets;    // physical positions, register order
    std::vector<uint32_t> perm;   // PERMRUN: the R tables back to back
    std::vector<uint64_t> run_cm; // PERMRUN: full-index control mask of each perm (fires on all ones)
    std::vector<int> run_gate;    // PERMRUN: gate id of each perm
    // ST_EXCHANGE: swap local bits lpos[i] with global bits gpos[i]
    std::vector<int> lpos, gpos;
    // ST_RELABEL: swap physical roles of logical qubits a,b (no data)
    int ra = -1, rb = -1;
    // ST_PASS, JIT tier: 1 = the block variant of the kernel (its launches
    // cover the tiles whose fixed local bits equal the launch's fixbits,
    // jit_set_block; the overlapped pass + exchange)
    int jit_block = 0;
    // ST_PASS, JIT tier: 1 = the readout variant (the pass also writes, per
    // tile, the sums of |a|^2 over the amplitudes with each tile bit set and
    // the tile total to P.red[tile * 13 + ...]: <Q_i> fused into the last pass
    // before qsim_expectations)
    int jit_readout = 0;
};

struct PlanOptions {
    bool fusion = true;
    bool block_fusion = true;  // fuse gate clusters on two tile qubits into 4x4 blocks (OPC_U4)
    bool low_remap = true;     // a pass stores the next pass's first-needed qubits at physical bits 0,1,2
    int remap_lookahead = 6;   // candidates searched for those three (<= 3: the first three needed)
    int max_scan = 1 << 30;   // look-ahead window (gates) per pass
    int global_policy = GP_AUTO;
    // device-time model inputs (plan_cost): the FP64-pipe flop/s and HBM
    // bytes/s the fused passes ACHIEVE, link bytes/s per direction.  The
    // runtime fills FP64 and HBM from the probe of its device
    // (qsim_probe_peaks) times the fractions the passes reach (kPassFp64Eff,
    // kPassHbmEff, measured round 2: 0.66-0.68 of the DFMA peak on
    // block-heavy passes, 0.73-0.86 of HBM on streaming ones) and the link
    // from the option "peak_link_gbs"; the defaults are those fractions of
    // the B200 peaks (34.2 TFLOP/s DFMA probe, 6.55 TB/s copy).
    static constexpr double kPassFp64Eff = 0.68, kPassHbmEff = 0.8;
    double peak_fp64 = kPassFp64Eff * 34.2e12, peak_hbm = kPassHbmEff * 6.55e12, peak_link = 0.77e12;
    // introspection (qsim_plan_json): plan only candidate list i (>= 0), and
    // report each candidate's modelled time and step counts
    int force_list = -1;
    // the runtime overlaps a pass with the exchange after it (runtime option
    // overlap on this transport): plan_cost models such a pair as
    // max(pass, exchange) + one block of the pass
    bool overlap = false;
    std::vector<std::string> *cand_report = nullptr;
    // called with the step list each time the planner has appended finished
    // steps (earlier steps never change again): the runtime launches them
    // while planning continues
    std::function<void(std::vector<Step> &)> sink;
};

class Planner {
public:
    Planner(int n, int G);
    int n, G, M;
    std::vector<int> phys_of;   // logical qubit -> physical bit
    std::vector<int> qubit_at;  // physical bit -> logical qubit

    // initial sigma by look-ahead: perm targets on the lowest
    // bits; the G qubits whose first non-diagonal use is latest go global.
    void choose_initial_layout(const std::vector<GateRec> &gates);
    void plan(const std::vector<GateRec> &gates, const PlanOptions &opt, std::vector<Step> &out);
    // explicit paper "SWAP K" command
    void remap(const std::vector<int> &local_q, const std::vector<int> &global_q, std::vector<Step> &out);

private:
    bool prefer_pairwise(const std::vector<GateRec> &gates, const std::vector<char> &done, size_t first) const;
    void emit_exchange(const std::vector<GateRec> &gates, const std::vector<char> &done, size_t first,
                       std::vector<Step> &out);
    void build_pass(const std::vector<GateRec> &gates, std::vector<char> &done, size_t first,
                    const PlanOptions &opt, std::vector<Step> &out);
    void emit_generic(const GateRec &g, std::vector<Step> &out);
    void emit_perm(const GateRec &g, std::vector<Step> &out);
    size_t emit_perm_run(const std::vector<GateRec> &gates, std::vector<char> &done, size_t first,
                         std::vector<Step> &out);

public:
    void swap_layout(int pa, int pb);

private:
    void plan_list(const std::vector<GateRec> &gates, const PlanOptions &opt, std::vector<Step> &out);
};

// modelled device seconds of a step list on 2^M-amplitude shards (planner choices)
double plan_cost(const std::vector<Step> &steps, int M, const PlanOptions &opt = PlanOptions());

std::string plan_to_json(const Planner &final_state, const std::vector<Step> &steps);

}  // namespace qsb
