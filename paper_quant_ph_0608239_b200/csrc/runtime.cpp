// runtime.cpp -- the qsim_* C-ABI (include/qsim.h): context, validation,
// gate queue, flush (planner -> device steps), exchange engine (virtual
// shards / NCCL), reductions, sampling and readout.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/qsim.h"
#include "comm.h"
#include "jit.h"
#include "kernels.h"
#include "plan.h"

using namespace qsb;

namespace {

struct TimedRange {
    cudaEvent_t a, b;
    int cat;  // 0 pass, 1 generic, 2 perm, 3 exchange, 4 reduce
    uint64_t bytes;
};

}  // namespace

// Last flush's plan: resubmitting the same gate list from the same layout
// (e.g. every step of a benchmark or a repeated circuit) skips planning,
// code-generation keys and parameter packing.
struct PlanCache {
    bool valid = false;
    bool with_init = false;
    std::vector<GateRec> queue;
    std::vector<int> phys_before, phys_init, phys_after;
    std::vector<Step> steps;
    std::vector<std::string> jkeys;
    std::vector<std::vector<std::vector<uint8_t>>> params;  // [step][shard]
};

static bool same_gate(const GateRec &a, const GateRec &b)
{
    return a.kind == b.kind && a.target == b.target && a.controls == b.controls && a.targets == b.targets &&
           std::memcmp(a.u, b.u, sizeof(a.u)) == 0 && a.perm == b.perm;
}

struct qsim_ctx_s {
    int n = 0, P = 1, G = 0, M = 0, rank = 0, transport = QSIM_TRANSPORT_LOCAL;
    std::vector<double2 *> shards;
    bool own_shards = false;
    double2 *scratch = nullptr;
    size_t scratch_bytes = 0;
    bool own_scratch = false;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int n_sm = 148;  // SMs of the current device (persistent pass grid)
    Comm *comm = nullptr;  // SPMD transports (NCCL, loopback)
    double comm_timeout_ms = 600e3;
    // exchange pipeline: transfers run on xstream, pack/unpack on stream
    cudaStream_t xstream = nullptr;
    cudaEvent_t x_ready[2] = {nullptr, nullptr}, x_done[2] = {nullptr, nullptr}, x_used[2] = {nullptr, nullptr};
    Planner *planner = nullptr;
    bool initialized = false, init_pending = false;
    uint64_t init_index = 0;
    std::vector<GateRec> queue;
    PlanCache pc;
    bool plan_cache = true;
    // device program buffers (d_ops: interpreter programs longer than its parameter block)
    KOp *d_ops = nullptr;
    unsigned long long *d_ttab = nullptr;  // per-thread phase factors (double2) of the current JIT pass (qsim_pass_tab)
    size_t d_ttab_cap = 0;
    size_t d_ops_cap = 0;
    uint32_t *d_perm = nullptr;
    size_t d_perm_cap = 0;
    KOp *h_ops = nullptr;
    size_t h_ops_cap = 0;
    uint32_t *h_perm = nullptr;
    size_t h_perm_cap = 0;
    cudaEvent_t upload_done = nullptr;
    double2 **d_shard_ptrs = nullptr;
    double *d_red = nullptr;
    // <Q_i> fused into the last pass (option fuse_readout): expectations_impl
    // asks for it (want_readout), flush runs that pass's readout variant
    // (readout_step) writing per-tile partials into d_rdo, and the readout
    // then reduces those (readout_ready) instead of reading the state again
    int fuse_readout = 1;
    bool want_readout = false, readout_ready = false;
    int64_t readout_step = -1;
    double *d_rdo = nullptr;
    size_t d_rdo_cap = 0;
    FusedExpectDesc rdo_desc{};
    size_t d_red_cap = 0;
    // the two-level sampler's own buffers (its rank-order reductions use d_red)
    double *d_samp = nullptr;
    size_t d_samp_cap = 0;
    // options
    bool fusion = true, timing = false, block_fusion = true, low_remap = true;
    int remap_lookahead = PlanOptions().remap_lookahead;
    int max_scan = 1 << 30;
    int jit = 1;           // 1: pass-specialised NVRTC kernels, 0: interpreter k_pass only
    int global_policy = GP_AUTO;
    int pass_variant = 2;  // k_pass min CTAs per SM (1: <=255 regs, 2: <=128 regs)
    int desync_ns = 1500;  // JIT pass: first-wave phase offset of the slot-0 CTAs (option desync_ns; 0 = off)
    int64_t chunk_mb = 1024;
    int64_t sample_batch = 0;  // two-level sampler: high bins per batch cap (option sample_batch; 0 = by memory)
    double peak_link_gbs = 0;  // planner link rate per direction (option peak_link_gbs; 0 = nominal)
    // SPMD: the planner's FP64 / HBM / link rates, measured at creation and
    // reduced to their minimum over the ranks, so that every rank plans with
    // identical inputs (the plans must agree step for step); 0 = not measured
    double plan_fp64 = 0, plan_hbm = 0, plan_link_gbs = 0;
    int overlap = 1;  // pass + exchange overlap: 1 = SPMD transports, 2 = also virtual shards, 0 = off
    cudaEvent_t ov_evs[64] = {};
    int ov_next = 0;
    // stats
    qsim_stats stats{};
    std::vector<TimedRange> ranges;
    std::vector<cudaEvent_t> event_pool;
    bool poisoned = false;
    std::string last_error;
};

#define FAIL(ctx, code, ...)                                            \
    do {                                                                \
        char _b[512];                                                   \
        snprintf(_b, sizeof(_b), __VA_ARGS__);                          \
        if (ctx) (ctx)->last_error = _b;                                \
        return code;                                                    \
    } while (0)

#define CK(ctx, call)                                                                               \
    do {                                                                                            \
        cudaError_t _e = (call);                                                                    \
        if (_e != cudaSuccess) {                                                                    \
            cudaGetLastError();                                                                     \
            (ctx)->poisoned = true;                                                                 \
            FAIL(ctx, QSIM_ERR_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(_e), __FILE__, __LINE__); \
        }                                                                                           \
    } while (0)

// a Comm call (comm.h): nonzero = transport error, message in _err
#define CKC(ctx, call)                                                                            \
    do {                                                                                          \
        std::string _err;                                                                         \
        if ((ctx)->comm->call) {                                                                  \
            (ctx)->poisoned = true;                                                               \
            FAIL(ctx, QSIM_ERR_COMM, "%s", _err.c_str());                                         \
        }                                                                                         \
    } while (0)

static bool spmd(const qsim_ctx_s *c) { return c->comm != nullptr && c->P > 1; }

// Wait for the context's stream.  SPMD: poll the transport's asynchronous
// error state meanwhile and give up after comm_timeout_ms (an SPMD call
// mismatch or a dead peer then returns QSIM_ERR_COMM instead of hanging).
static qsim_status sync_stream(qsim_ctx c)
{
    if (c->comm) {
        std::string err;
        if (c->comm->wait(c->stream, c->comm_timeout_ms, err)) {
            c->poisoned = true;
            FAIL(c, QSIM_ERR_COMM, "%s", err.c_str());
        }
        return QSIM_OK;
    }
    CK(c, cudaStreamSynchronize(c->stream));
    return QSIM_OK;
}

#define LAUNCHED(ctx)                                                                         \
    do {                                                                                      \
        cudaError_t _e = cudaGetLastError();                                                  \
        if (_e != cudaSuccess) {                                                              \
            (ctx)->poisoned = true;                                                           \
            FAIL(ctx, QSIM_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(_e));            \
        }                                                                                     \
        (ctx)->stats.kernel_launches++;                                                       \
    } while (0)

// FP64-pipe instructions the interpreter tier k_pass executes on one pass
// over a 2^M shard: per touched amplitude 8 for a complex 2x2, 4 for a real
// 2x2, 4 for a phase (OPC_PHASE_ACC is applied like OPC_PHASE there), 0 for
// an exact swap, 16 for a fused 4x4 block; the predicate bits (controls)
// halve the touched set.  The JIT tier's count comes from its generator
// (JitPass::fp64_per_thread: 3M blocks, integer phase runs, lazy flushes).
static double pass_fp64_slots(const Step &s, int M)
{
    double tot = 0;
    for (const KOp &op : s.ops) {
        if (op.code == OPC_TRANS || op.code == OPC_XS || op.code == OPC_PHASE_FLUSH || op.code == OPC_DATA) continue;
        if (op.code == OPC_U4) { tot += 16 * std::ldexp(1.0, M); continue; }
        const int pb = __builtin_popcount(op.mreg) + __builtin_popcount(op.mlane) + __builtin_popcount(op.mwarp) +
                       __builtin_popcountll(op.mout);
        const double per = op.code == OPC_U2 ? 8.0 : 4.0;
        tot += per * std::ldexp(1.0, M - pb);
    }
    return tot;
}

static JitCache &jit_cache()
{
    static JitCache *c = new JitCache();  // process-wide, one device per process
    return *c;
}

static int ilog2(int P)
{
    int g = 0;
    while ((1 << g) < P) g++;
    return g;
}

// ------------------------------------------------------------ validation
static bool unitary(const qsim_c128 *u)
{
    // U^dag U - I, entries (i,j) = sum_k conj(U_ki) U_kj
    double r[2][2][2];
    for (int i = 0; i < 2; i++)
        for (int j = 0; j < 2; j++) {
            double re = 0, im = 0;
            for (int k = 0; k < 2; k++) {
                const qsim_c128 a = u[2 * k + i], b = u[2 * k + j];
                re += a.re * b.re + a.im * b.im;
                im += a.re * b.im - a.im * b.re;
            }
            r[i][j][0] = re - (i == j ? 1.0 : 0.0);
            r[i][j][1] = im;
        }
    for (int i = 0; i < 2; i++)
        for (int j = 0; j < 2; j++)
            if (std::fabs(r[i][j][0]) > 1e-12 || std::fabs(r[i][j][1]) > 1e-12 || !std::isfinite(r[i][j][0]))
                return false;
    return true;
}

static qsim_status to_rec(qsim_ctx ctx, int n, const qsim_gate &g, GateRec &r)
{
    auto inr = [&](int q) { return q >= 0 && q < n; };
    r = GateRec();
    if (g.kind == QSIM_G_1Q || g.kind == QSIM_G_CTRL) {
        int nc = g.kind == QSIM_G_1Q ? 0 : g.n_controls;
        if (nc < 0 || nc > QSIM_MAX_CONTROLS) FAIL(ctx, QSIM_ERR_ARG, "n_controls=%d out of [0,%d]", nc, QSIM_MAX_CONTROLS);
        if (!inr(g.target)) FAIL(ctx, QSIM_ERR_QUBIT_RANGE, "target %d outside [0,%d)", g.target, n);
        uint64_t seen = 1ULL << g.target;
        for (int i = 0; i < nc; i++) {
            int c = g.controls[i];
            if (!inr(c)) FAIL(ctx, QSIM_ERR_QUBIT_RANGE, "control %d outside [0,%d)", c, n);
            if ((seen >> c) & 1) FAIL(ctx, QSIM_ERR_DUP_QUBIT, "qubit %d repeated", c);
            seen |= 1ULL << c;
            r.controls.push_back(c);
        }
        if (!unitary(g.u)) FAIL(ctx, QSIM_ERR_NOT_UNITARY, "matrix is not unitary within 1e-12");
        r.kind = GK_U2;
        r.target = g.target;
        for (int k = 0; k < 4; k++) { r.u[2 * k] = g.u[k].re; r.u[2 * k + 1] = g.u[k].im; }
    } else if (g.kind == QSIM_G_PERM) {
        int nt = g.n_targets, nc = g.n_controls;
        if (nt < 1 || nt > QSIM_MAX_PERM_TARGETS) FAIL(ctx, QSIM_ERR_ARG, "n_targets=%d out of [1,%d]", nt, QSIM_MAX_PERM_TARGETS);
        if (nt > n) FAIL(ctx, QSIM_ERR_ARG, "n_targets > n");
        if (nc < 0 || nc > QSIM_MAX_CONTROLS) FAIL(ctx, QSIM_ERR_ARG, "n_controls=%d out of range", nc);
        if (!g.perm) FAIL(ctx, QSIM_ERR_ARG, "perm is NULL");
        uint64_t seen = 0;
        for (int i = 0; i < nt; i++) {
            int t = g.targets[i];
            if (!inr(t)) FAIL(ctx, QSIM_ERR_QUBIT_RANGE, "target %d outside [0,%d)", t, n);
            if ((seen >> t) & 1) FAIL(ctx, QSIM_ERR_DUP_QUBIT, "qubit %d repeated", t);
            seen |= 1ULL << t;
            r.targets.push_back(t);
        }
        for (int i = 0; i < nc; i++) {
            int c = g.controls[i];
            if (!inr(c)) FAIL(ctx, QSIM_ERR_QUBIT_RANGE, "control %d outside [0,%d)", c, n);
            if ((seen >> c) & 1) FAIL(ctx, QSIM_ERR_DUP_QUBIT, "qubit %d repeated", c);
            seen |= 1ULL << c;
            r.controls.push_back(c);
        }
        const uint32_t W = 1u << nt;
        std::vector<char> hit(W, 0);
        r.perm.assign(g.perm, g.perm + W);
        for (uint32_t w = 0; w < W; w++) {
            if (g.perm[w] >= W || hit[g.perm[w]]) FAIL(ctx, QSIM_ERR_NOT_PERMUTATION, "perm is not a bijection of [0,%u)", W);
            hit[g.perm[w]] = 1;
        }
        r.kind = GK_PERM;
    } else if (g.kind == QSIM_G_SWAP) {
        int a = g.targets[0], b = g.targets[1];
        if (!inr(a) || !inr(b)) FAIL(ctx, QSIM_ERR_QUBIT_RANGE, "swap qubit outside [0,%d)", n);
        if (a == b) FAIL(ctx, QSIM_ERR_DUP_QUBIT, "swap of qubit %d with itself", a);
        r.kind = GK_SWAP;
        r.targets = {a, b};
    } else {
        FAIL(ctx, QSIM_ERR_ARG, "unknown gate kind %d", g.kind);
    }
    classify(r);
    return QSIM_OK;
}

// ------------------------------------------------------------ helpers
static cudaEvent_t ev_get(qsim_ctx c)
{
    if (!c->event_pool.empty()) {
        cudaEvent_t e = c->event_pool.back();
        c->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

// NVTX ranges (header-only NVTX3: a no-op unless a tool such as Nsight
// Systems injects itself) name every engine phase on the host timeline.
static const char *const kRangeName[] = {"qsim pass", "qsim generic gate", "qsim permutation",
                                         "qsim exchange", "qsim readout", "qsim overlapped pass+exchange"};
struct RangeGuard {
    qsim_ctx c;
    int cat;
    uint64_t bytes;
    cudaEvent_t a = nullptr;
    RangeGuard(qsim_ctx c_, int cat_, uint64_t bytes_) : c(c_), cat(cat_), bytes(bytes_)
    {
        nvtxRangePushA(kRangeName[cat]);
        if (c->timing) {
            a = ev_get(c);
            cudaEventRecord(a, c->stream);
        }
    }
    ~RangeGuard()
    {
        if (c->timing) {
            cudaEvent_t b = ev_get(c);
            cudaEventRecord(b, c->stream);
            c->ranges.push_back({a, b, cat, bytes});
        }
        nvtxRangePop();
    }
};

static qsim_status collect_timing(qsim_ctx c)
{
    if (c->ranges.empty()) return QSIM_OK;
    { qsim_status _s = sync_stream(c); if (_s != QSIM_OK) return _s; }
    for (auto &r : c->ranges) {
        float ms = 0;
        cudaEventElapsedTime(&ms, r.a, r.b);
        switch (r.cat) {
        case 0: c->stats.pass_ms += ms; c->stats.pass_amp_bytes += r.bytes; break;
        case 1: c->stats.generic_ms += ms; break;
        case 2: c->stats.perm_ms += ms; break;
        case 3: c->stats.exchange_ms += ms; break;
        case 5: c->stats.overlap_ms += ms; break;
        default: c->stats.reduce_ms += ms; break;
        }
        c->event_pool.push_back(r.a);
        c->event_pool.push_back(r.b);
    }
    c->ranges.clear();
    return QSIM_OK;
}

template <class T>
static qsim_status ensure_dev(qsim_ctx c, T *&p, size_t &cap, size_t need)
{
    if (need <= cap) return QSIM_OK;
    size_t nc = std::max(need, cap * 2);
    if (p) {
        { qsim_status _s = sync_stream(c); if (_s != QSIM_OK) return _s; }
        CK(c, cudaFree(p));
        p = nullptr;
    }
    cudaError_t e = cudaMalloc((void **)&p, nc * sizeof(T));
    if (e != cudaSuccess) { cap = 0; FAIL(c, QSIM_ERR_OOM, "cudaMalloc(%zu): %s", nc * sizeof(T), cudaGetErrorString(e)); }
    cap = nc;
    return QSIM_OK;
}

template <class T>
static qsim_status ensure_host(qsim_ctx c, T *&p, size_t &cap, size_t need)
{
    if (need <= cap) return QSIM_OK;
    size_t nc = std::max(need, cap * 2);
    if (c->upload_done) CK(c, cudaEventSynchronize(c->upload_done));
    if (p) CK(c, cudaFreeHost(p));
    p = nullptr;
    CK(c, cudaMallocHost((void **)&p, nc * sizeof(T)));
    cap = nc;
    return QSIM_OK;
}

static inline uint64_t rank_sub(uint64_t r, const std::vector<int> &gpos, int M)
{
    uint64_t v = 0;
    for (size_t i = 0; i < gpos.size(); i++) v |= ((r >> (gpos[i] - M)) & 1) << i;
    return v;
}
static inline uint64_t with_sub(uint64_t r, const std::vector<int> &gpos, int M, uint64_t v)
{
    for (size_t i = 0; i < gpos.size(); i++) {
        uint64_t b = 1ULL << (gpos[i] - M);
        r = ((v >> i) & 1) ? (r | b) : (r & ~b);
    }
    return r;
}

// ------------------------------------------------------------ exchange
// Piece pipeline of the SPMD exchanges (P:759-779 split each send into
// buffers; here the buffers are also pipelined).  Piece k is staged on the
// engine stream (pack into slot k&1), transferred on xstream (one grouped
// send/recv), and finished on the engine stream (unpack / combine).  With two
// slots the transfer of piece k overlaps the finish of piece k-1 and the
// stage of piece k+1; a slot is re-used only after its previous finish.
template <class Stage, class Xfer, class Finish>
static qsim_status pipeline(qsim_ctx c, uint64_t nb, Stage stage, Xfer xfer, Finish finish)
{
    if (!c->xstream) {
        CK(c, cudaStreamCreateWithFlags(&c->xstream, cudaStreamNonBlocking));
        for (int i = 0; i < 2; i++) {
            CK(c, cudaEventCreateWithFlags(&c->x_ready[i], cudaEventDisableTiming));
            CK(c, cudaEventCreateWithFlags(&c->x_done[i], cudaEventDisableTiming));
            CK(c, cudaEventCreateWithFlags(&c->x_used[i], cudaEventDisableTiming));
        }
    }
    qsim_status st;
    auto finish_one = [&](uint64_t j) -> qsim_status {
        const int sl = (int)(j & 1);
        CK(c, cudaStreamWaitEvent(c->stream, c->x_done[sl], 0));
        if ((st = finish(j, sl)) != QSIM_OK) return st;
        CK(c, cudaEventRecord(c->x_used[sl], c->stream));
        return QSIM_OK;
    };
    for (uint64_t k = 0; k < nb; k++) {
        const int sl = (int)(k & 1);
        if ((st = stage(k, sl)) != QSIM_OK) return st;
        CK(c, cudaEventRecord(c->x_ready[sl], c->stream));
        CK(c, cudaStreamWaitEvent(c->xstream, c->x_ready[sl], 0));
        if (k >= 2) CK(c, cudaStreamWaitEvent(c->xstream, c->x_used[sl], 0));
        if ((st = xfer(k, sl)) != QSIM_OK) return st;
        CK(c, cudaEventRecord(c->x_done[sl], c->xstream));
        if (k >= 1 && (st = finish_one(k - 1)) != QSIM_OK) return st;
    }
    return nb ? finish_one(nb - 1) : QSIM_OK;
}

static qsim_status exec_exchange(qsim_ctx c, const Step &s)
{
    const int K = (int)s.lpos.size(), M = c->M;
    if (K == 0) return QSIM_OK;
    const uint64_t chunk = 1ULL << (M - K);
    const uint64_t nval = 1ULL << K;
    RangeGuard rg(c, 3, 0);
    c->stats.exchanges++;
    if (c->transport == QSIM_TRANSPORT_VIRTUAL) {
        for (uint64_t r = 0; r < (uint64_t)c->P; r++) {
            const uint64_t my = rank_sub(r, s.gpos, M);
            for (uint64_t v = 0; v < nval; v++) {
                if (v == my) continue;
                const uint64_t peer = with_sub(r, s.gpos, M, v);
                if (peer < r) continue;
                launch_swap_blocks(c->shards[r], c->shards[peer], M, K, s.lpos.data(), v, my, c->stream);
                LAUNCHED(c);
            }
        }
        c->stats.exchange_bytes += (nval - 1) * chunk * 16;
        return QSIM_OK;
    }
    if (!spmd(c)) FAIL(c, QSIM_ERR_STATE, "exchange without a multi-shard transport");
    // SPMD (NCCL / loopback): every rank trades chunk v with the peer whose
    // global sub-bits are v, in pieces through the pipeline
    const uint64_t my = rank_sub((uint64_t)c->rank, s.gpos, M);
    bool contiguous = true;
    {
        std::vector<int> l = s.lpos;
        std::sort(l.begin(), l.end());
        for (int i = 0; i < K; i++)
            if (l[i] != M - K + i) contiguous = false;
    }
    const uint64_t npeer = nval - 1;
    const uint64_t scratch_amps = c->scratch_bytes / sizeof(double2);
    const uint64_t per_piece = 2 * npeer * (contiguous ? 1 : 2);  // two slots of recv (+ send) buffers
    uint64_t piece = chunk;
    const uint64_t limit_amps = (uint64_t)c->chunk_mb * (1ULL << 20) / sizeof(double2);
    while (piece > 1 && (piece * per_piece > scratch_amps || piece > limit_amps)) piece >>= 1;
    if (piece * per_piece > scratch_amps) FAIL(c, QSIM_ERR_OOM, "scratch too small for exchange");
    const uint64_t slot_amps = piece * npeer * (contiguous ? 1 : 2);
    auto recvb = [&](int slot) { return c->scratch + slot * slot_amps; };
    auto sendb = [&](int slot) { return c->scratch + slot * slot_amps + piece * npeer; };
    std::vector<uint64_t> vals;
    for (uint64_t v = 0; v < nval; v++)
        if (v != my) vals.push_back(v);
    qsim_status st = pipeline(
        c, chunk / piece,
        [&](uint64_t k, int slot) -> qsim_status {  // stage: pack the outgoing blocks
            if (contiguous) return QSIM_OK;
            for (size_t i = 0; i < vals.size(); i++) {
                launch_pack(c->shards[0], sendb(slot) + i * piece, M, K, s.lpos.data(), vals[i], k * piece, piece, 0,
                            c->stream);
                LAUNCHED(c);
            }
            return QSIM_OK;
        },
        [&](uint64_t k, int slot) -> qsim_status {  // transfer (xstream)
            CKC(c, group_start(_err));
            for (size_t i = 0; i < vals.size(); i++) {
                const int peer = (int)with_sub((uint64_t)c->rank, s.gpos, M, vals[i]);
                const double2 *src;
                if (contiguous) {
                    uint64_t base = 0;
                    for (int b = 0; b < K; b++)
                        if ((vals[i] >> b) & 1) base |= 1ULL << s.lpos[b];
                    src = c->shards[0] + base + k * piece;
                } else {
                    src = sendb(slot) + i * piece;
                }
                CKC(c, send(src, piece * sizeof(double2), peer, c->xstream, _err));
                CKC(c, recv(recvb(slot) + i * piece, piece * sizeof(double2), peer, c->xstream, _err));
            }
            CKC(c, group_end(_err));
            return QSIM_OK;
        },
        [&](uint64_t k, int slot) -> qsim_status {  // finish: unpack the incoming blocks in place
            for (size_t i = 0; i < vals.size(); i++) {
                launch_pack(c->shards[0], recvb(slot) + i * piece, M, K, s.lpos.data(), vals[i], k * piece, piece, 1,
                            c->stream);
                LAUNCHED(c);
            }
            return QSIM_OK;
        });
    if (st != QSIM_OK) return st;
    c->stats.exchange_bytes += npeer * chunk * 16;
    return QSIM_OK;
}

// pairwise handling of a gate on a global target: the two ranks
// that differ only in the target bit combine their shards; sigma unchanged
static qsim_status exec_pairwise(qsim_ctx c, const Step &s)
{
    const int M = c->M;
    const uint64_t gbit = 1ULL << (s.t - M);
    const uint64_t lmask = (1ULL << M) - 1;
    const uint64_t mloc = s.cm & lmask, vloc = s.cv & lmask, mhi = s.cm & ~lmask, vhi = s.cv & ~lmask;
    RangeGuard rg(c, 3, 0);
    c->stats.exchanges++;
    if (c->transport == QSIM_TRANSPORT_VIRTUAL) {
        for (uint64_t r = 0; r < (uint64_t)c->P; r++) {
            if (r & gbit) continue;
            if (((r << M) & mhi) != vhi) continue;  // controls on global qubits (never the target)
            launch_pair_gate(c->shards[r], c->shards[r | gbit], M, mloc, vloc, s.code == OPC_XS, s.m, c->stream);
            LAUNCHED(c);
        }
        c->stats.exchange_bytes += (uint64_t)c->P * (16ULL << M);
        return QSIM_OK;
    }
    if (!spmd(c)) FAIL(c, QSIM_ERR_STATE, "pairwise step without a multi-shard transport");
    const uint64_t r = (uint64_t)c->rank;
    if (((r << M) & mhi) != vhi) return QSIM_OK;  // the partner skips too (same control bits)
    const int peer = (int)(r ^ gbit);
    const bool hi = (r & gbit) != 0;
    static const double xs_m[8] = {0, 0, 1, 0, 1, 0, 0, 0};
    const double *m = s.code == OPC_XS ? xs_m : s.m;
    // self_first: bit 0 -> own' = u00 own + u01 other; bit 1 -> own' = u10 other + u11 own
    const double *c0 = hi ? m + 4 : m + 0, *c1 = hi ? m + 6 : m + 2;
    const uint64_t shard = 1ULL << M, scratch_amps = c->scratch_bytes / sizeof(double2);
    uint64_t piece = shard;
    const uint64_t limit_amps = (uint64_t)c->chunk_mb * (1ULL << 20) / sizeof(double2);
    while (piece > 1 && (2 * piece > scratch_amps || piece > limit_amps)) piece >>= 1;
    if (2 * piece > scratch_amps) FAIL(c, QSIM_ERR_OOM, "scratch too small for a pairwise exchange");
    qsim_status st = pipeline(
        c, shard / piece, [&](uint64_t, int) -> qsim_status { return QSIM_OK; },
        [&](uint64_t k, int slot) -> qsim_status {
            CKC(c, group_start(_err));
            CKC(c, send(c->shards[0] + k * piece, piece * sizeof(double2), peer, c->xstream, _err));
            CKC(c, recv(c->scratch + slot * piece, piece * sizeof(double2), peer, c->xstream, _err));
            CKC(c, group_end(_err));
            return QSIM_OK;
        },
        [&](uint64_t k, int slot) -> qsim_status {
            launch_pair_combine(c->shards[0] + k * piece, c->scratch + slot * piece, k * piece, piece, mloc, vloc, c0,
                                c1, !hi, c->stream);
            LAUNCHED(c);
            return QSIM_OK;
        });
    if (st != QSIM_OK) return st;
    c->stats.exchange_bytes += 16ULL << M;
    return QSIM_OK;
}

// ------------------------------------------------------------ flush
static qsim_status upload_program(qsim_ctx c, std::vector<Step> &steps)
{
    // pass programs travel in the kernel parameter block, except interpreter
    // programs longer than kMaxPassOps: those are read from global memory
    size_t nops = 0, nperm = 0;
    for (Step &s : steps) {
        if (s.type == ST_PERM || s.type == ST_PERMRUN) nperm += s.perm.size();
        if (s.type == ST_PASS && s.ops.size() > (size_t)kMaxPassOps) nops += s.ops.size();
    }
    qsim_status st;
    if (nops) {
        if ((st = ensure_host(c, c->h_ops, c->h_ops_cap, nops)) != QSIM_OK) return st;
        if ((st = ensure_dev(c, c->d_ops, c->d_ops_cap, nops)) != QSIM_OK) return st;
        if (c->upload_done) CK(c, cudaEventSynchronize(c->upload_done));  // staging reuse
        size_t q = 0;
        for (Step &s : steps)
            if (s.type == ST_PASS && s.ops.size() > (size_t)kMaxPassOps) {
                std::copy(s.ops.begin(), s.ops.end(), c->h_ops + q);
                s.t = (int)q;  // program offset
                q += s.ops.size();
            }
        CK(c, cudaMemcpyAsync(c->d_ops, c->h_ops, nops * sizeof(KOp), cudaMemcpyHostToDevice, c->stream));
        if (!c->upload_done) CK(c, cudaEventCreateWithFlags(&c->upload_done, cudaEventDisableTiming));
        CK(c, cudaEventRecord(c->upload_done, c->stream));
    }
    if (nperm == 0) return QSIM_OK;
    if ((st = ensure_host(c, c->h_perm, c->h_perm_cap, nperm + 1)) != QSIM_OK) return st;
    if ((st = ensure_dev(c, c->d_perm, c->d_perm_cap, nperm + 1)) != QSIM_OK) return st;
    if (c->upload_done) CK(c, cudaEventSynchronize(c->upload_done));  // staging reuse
    size_t p = 0;
    for (Step &s : steps) {
        if (s.type == ST_PERM || s.type == ST_PERMRUN) {
            // k_perm / k_perm_run gather: out[w] = in[perm^-1(w)]; a run's tables back to back
            const size_t TT = (size_t)1 << s.ptargets.size();
            for (size_t w = 0; w < s.perm.size(); w++) c->h_perm[p + (w / TT) * TT + s.perm[w]] = (uint32_t)(w % TT);
            s.t = (int)p;  // perm offset
            p += s.perm.size();
        }
    }
    if (nperm) CK(c, cudaMemcpyAsync(c->d_perm, c->h_perm, nperm * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
    if (!c->upload_done) CK(c, cudaEventCreateWithFlags(&c->upload_done, cudaEventDisableTiming));
    CK(c, cudaEventRecord(c->upload_done, c->stream));
    return QSIM_OK;
}

static int local_ranks(qsim_ctx c, int i) { return c->transport == QSIM_TRANSPORT_VIRTUAL ? i : c->rank; }
static int n_local(qsim_ctx c) { return c->transport == QSIM_TRANSPORT_VIRTUAL ? c->P : 1; }

// insertion sort of a few tile positions (bounded, no std::sort threshold games)
static void sort_small(int *a, int n)
{
    for (int i = 1; i < n; i++)
        for (int j = i; j > 0 && a[j - 1] > a[j]; j--) std::swap(a[j - 1], a[j]);
}

static qsim_status exec_perm_run(qsim_ctx c, const Step &s)
{
    PermRunDesc d{};
    const int M = c->M, t = (int)s.ptargets.size();
    // smaller tiles than k_perm's: the run's tables share the shared memory,
    // and more resident CTAs hide the load latency of the gather
    static const int run_tb = [] { const char *e = getenv("QSIM_PERMRUN_TILE"); return e ? atoi(e) : 11; }();
    int tb = std::min(std::max(std::min(run_tb, M), t), kPermTileBits);  // t <= 12 = kPermTileBits
    const int R = (int)s.run_cm.size();
    while (tb > t && perm_run_smem_bytes(tb, t, R) > kPermRunSmemMax) tb--;
    d.M = M;
    d.t = t;
    d.tile_bits = tb;
    d.R = R;
    d.tab_offset = s.t;
    bool used[64] = {false};
    for (int i = 0; i < t; i++) { d.tile_pos[i] = s.ptargets[i]; used[s.ptargets[i]] = true; }
    int nb = t;
    for (int p = 0; p < M && nb < tb; p++)
        if (!used[p]) { d.tile_pos[nb++] = p; used[p] = true; }
    int srt[kPermTileBits];
    for (int i = 0; i < tb; i++) srt[i] = d.tile_pos[i];
    sort_small(srt, tb);
    for (int i = 0; i < tb; i++) d.tile_sorted[i] = srt[i];
    d.n_inst = 1ULL << (M - tb);
    d.contiguous = 1;
    for (int i = 0; i < tb; i++)
        if (d.tile_pos[i] != i) d.contiguous = 0;
    for (int j = 0; j < d.R; j++)
        for (int b = 0; b < 64; b++) {
            if (!((s.run_cm[j] >> b) & 1)) continue;
            int tl = -1;
            for (int i = 0; i < tb; i++)
                if (d.tile_pos[i] == b) tl = i;
            if (tl >= 0) { d.m_tile[j] |= 1u << tl; d.v_tile[j] |= 1u << tl; }
            else { d.m_out[j] |= 1ULL << b; d.v_out[j] |= 1ULL << b; }
        }
    // composition head (PermRunDesc): the perms at the top of the gather
    // chain (highest j) without in-tile controls; of those, the ones whose
    // controls sit on instance bits >= 4 (or on rank bits) form the
    // slow head.  QSIM_PERMRUN_COMPOSE=0 disables (A/B), QSIM_PERMRUN_SLOWBIT sets the bit.
    static const int compose = [] { const char *e = getenv("QSIM_PERMRUN_COMPOSE"); return e ? atoi(e) : 1; }();
    static const int slow_bit = [] { const char *e = getenv("QSIM_PERMRUN_SLOWBIT"); return e ? atoi(e) : 4; }();
    if (compose && perm_run_smem_bytes(tb, t, R, true) <= kPermRunSmemMax) {
        for (int j = R - 1; j >= 0 && d.m_tile[j] == 0; j--) d.pre_mask |= 1u << j;
        for (int j = R - 1; j >= 0 && ((d.pre_mask >> j) & 1); j--) {
            bool slow = true;
            for (int b = 0; b < M && slow; b++) {
                if (!((d.m_out[j] >> b) & 1)) continue;
                int below = 0;  // tile positions below b: the instance bit of b is b - below
                for (int i = 0; i < tb; i++) below += d.tile_pos[i] < b;
                slow = b - below >= slow_bit;
            }
            if (!slow) break;
            d.slow_mask |= 1u << j;
        }
    }
    static const int bulk = [] { const char *e = getenv("QSIM_PERMRUN_BULK"); return e ? atoi(e) : 1; }();
    d.bulk = bulk && d.contiguous;
    if (perm_run_smem(d) > kPermRunSmemMax) FAIL(c, QSIM_ERR_ARG, "permutation run too large for shared memory");
    RangeGuard rg(c, 2, 0);
    for (int i = 0; i < n_local(c); i++) {
        d.rank_bits = (uint64_t)local_ranks(c, i) << M;
        launch_perm_run(d, c->shards[i], c->d_perm, c->n_sm, c->stream);
        LAUNCHED(c);
        c->stats.perm_launches++;
    }
    return QSIM_OK;
}

static qsim_status exec_perm(qsim_ctx c, const Step &s)
{
    PermDesc d{};
    const int M = c->M, t = (int)s.ptargets.size();
    int tb = std::min(kPermTileBits, M);
    if (tb < t) tb = t;
    if (tb > kPermTileBits) FAIL(c, QSIM_ERR_ARG, "permutation of %d targets exceeds the %d-bit tile", t, kPermTileBits);
    d.M = M;
    d.t = t;
    d.tile_bits = tb;
    d.perm_offset = s.t;
    bool used[64] = {false};
    for (int i = 0; i < t; i++) { d.tile_pos[i] = s.ptargets[i]; used[s.ptargets[i]] = true; }
    int nb = t;
    for (int p = 0; p < M && nb < tb; p++)
        if (!used[p]) { d.tile_pos[nb++] = p; used[p] = true; }
    int srt[kPermTileBits];
    for (int i = 0; i < tb; i++) srt[i] = d.tile_pos[i];
    sort_small(srt, tb);
    for (int i = 0; i < tb; i++) d.tile_sorted[i] = srt[i];
    d.n_inst = 1ULL << (M - tb);
    d.contiguous = 1;
    for (int i = 0; i < tb; i++)
        if (d.tile_pos[i] != i) d.contiguous = 0;
    for (int b = 0; b < 64; b++) {
        if (!((s.cm >> b) & 1)) continue;
        int tl = -1;
        for (int i = 0; i < tb; i++)
            if (d.tile_pos[i] == b) tl = i;
        if (tl >= 0) { d.m_ctrl_tile |= 1u << tl; d.v_ctrl_tile |= 1u << tl; }
        else { d.m_ctrl_out |= 1ULL << b; d.v_ctrl_out |= 1ULL << b; }
    }
    RangeGuard rg(c, 2, 0);
    for (int i = 0; i < n_local(c); i++) {
        d.rank_bits = (uint64_t)local_ranks(c, i) << M;
        launch_perm(d, c->shards[i], c->d_perm, c->stream);
        LAUNCHED(c);
        c->stats.perm_launches++;
    }
    return QSIM_OK;
}

// One JIT pass launch of `count` tile instances of local shard i on
// `stream` (the companion per-thread phase-table kernel first when
// with_tab).  fn: the kernel (nullptr: the pass's own); K > 0: the block
// variant's launch over the tiles whose local bits fix_pos equal fixbits'.
static qsim_status launch_jit_range(qsim_ctx c, size_t si, int i, uint64_t count, cudaStream_t stream, bool with_tab,
                                    CUfunction fn = nullptr, const int *fix_pos = nullptr, int K = 0,
                                    uint64_t fixbits = 0, double *red = nullptr)
{
    PlanCache &pc = c->pc;
    const Step &s = pc.steps[si];
    if (!fn) fn = jit_cache().find(pc.jkeys[si]);
    int nts = 0;
    CUfunction tabfn = jit_cache().find_tab(pc.jkeys[si], nts);
    if (!fn) FAIL(c, QSIM_ERR_STATE, "jit pass kernel missing");
    qsim_status st;
    if (tabfn && (st = ensure_dev(c, c->d_ttab, c->d_ttab_cap, (size_t)2 * nts * kPassThreads)) != QSIM_OK) return st;
    const uint64_t rb = (uint64_t)local_ranks(c, i) << c->M;
    auto &pp = pc.params[si];
    if (pp.size() != (size_t)n_local(c)) pp.assign(n_local(c), {});
    if (pp[i].empty()) jit_pack_params(s, c->shards[i], rb, pp[i]);
    if (s.pass.fresh) jit_set_init(pp[i], s.pass.init_phys);  // changes between flushes
    if (tabfn) jit_set_ttab(pp[i], c->d_ttab);
    jit_set_desync(pp[i], (uint32_t)c->n_sm, (uint32_t)c->desync_ns);
    jit_set_red(pp[i], red);
    // (the launch copies the parameter block)
    if (!jit_set_block(pp[i], s, fix_pos, K, fixbits)) FAIL(c, QSIM_ERR_STATE, "jit pass: too many fixed bits");
    size_t sz = pp[i].size();
    void *extra[] = {CU_LAUNCH_PARAM_BUFFER_POINTER, pp[i].data(), CU_LAUNCH_PARAM_BUFFER_SIZE, &sz, CU_LAUNCH_PARAM_END};
    if (tabfn && with_tab) {  // the per-thread phase slots (the same for every shard and range)
        CUresult ct = drv().launchKernel(tabfn, 1, 1, 1, kPassThreads, 1, 1, 0, (CUstream)stream, nullptr, extra);
        if (ct != CUDA_SUCCESS) {
            c->poisoned = true;
            FAIL(c, QSIM_ERR_CUDA, "cuLaunchKernel(jit pass table) failed: %d", (int)ct);
        }
        LAUNCHED(c);
    }
    unsigned grid, block, smem;
    jit_launch_dims(s, c->n_sm, grid, block, smem);
    grid = (unsigned)count;
    CUresult cr = drv().launchKernel(fn, grid, 1, 1, block, 1, 1, smem, (CUstream)stream, nullptr, extra);
    if (cr != CUDA_SUCCESS) {
        c->poisoned = true;
        FAIL(c, QSIM_ERR_CUDA, "cuLaunchKernel(jit pass) failed: %d", (int)cr);
    }
    LAUNCHED(c);
    return QSIM_OK;
}

static cudaEvent_t ov_event(qsim_ctx c)
{
    cudaEvent_t &e = c->ov_evs[c->ov_next];
    c->ov_next = (c->ov_next + 1) % 64;
    if (!e) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    return e;
}

// Whether the pass at si and the exchange after it can run overlapped: the
// exchange's local bits are not tile bits of the pass (so the pass's tiles
// split into the exchange's 2^K blocks by those instance bits), K <= 3, JIT
// tier, more than one shard.
static bool overlap_ok(qsim_ctx c, size_t si)
{
    PlanCache &pc = c->pc;
    if (!c->overlap || !c->jit || si + 1 >= pc.steps.size() || c->P < 2) return false;
    // virtual shards share one GPU's HBM: their "transfer" is copy work the
    // pass competes with, so the overlap there only on request (overlap = 2)
    if (c->transport == QSIM_TRANSPORT_VIRTUAL ? c->overlap < 2 : !spmd(c)) return false;
    const Step &p = pc.steps[si], &x = pc.steps[si + 1];
    if (p.type != ST_PASS || x.type != ST_EXCHANGE || !jit_cache().find(pc.jkeys[si])) return false;
    const int K = (int)x.lpos.size(), M = c->M;
    if (K < 1 || K > 3 || M - kTileBits < K) return false;
    for (int t = 0; t < kTileBits; t++)
        for (int l : x.lpos)
            if (p.pass.tp[t] == l || p.pass.tp_out[t] == l) return false;
    return true;
}

// The pass at si and the K-pair exchange at si + 1, overlapped:
// the pass runs block by block (the 2^K blocks of the exchange, as instance
// ranges), each outgoing block's transfer starting on the transfer stream as
// soon as its block is computed while the engine stream computes the next;
// the block that stays is computed last, under the last transfers.  Rounds
// follow the XOR schedule (round j: the peer whose sub-value is mine ^ j), so
// every round pairs the ranks and no transfer waits on a cycle.
static qsim_status exec_pass_exchange(qsim_ctx c, size_t si)
{
    PlanCache &pc = c->pc;
    const Step &p = pc.steps[si], &x = pc.steps[si + 1];
    const int K = (int)x.lpos.size(), M = c->M;
    const uint64_t nval = 1ULL << K, chunk = 1ULL << (M - K);
    const uint64_t n_inst = p.pass.n_inst, per = n_inst >> K;
    // block v: the tiles whose local bits lpos[b] equal bit b of v
    auto fix_of = [&](uint64_t v) {
        uint64_t f = 0;
        for (int b = 0; b < K; b++)
            if ((v >> b) & 1) f |= 1ULL << x.lpos[b];
        return f;
    };
    // the block variant of the pass kernel (compiled here on first use; cached
    // in memory and on disk like every pass kernel)
    Step bv = p;
    bv.jit_block = 1;
    const std::string bkey = jit_key(bv);
    CUfunction bfn = jit_cache().find(bkey);
    if (!bfn) {
        std::string jerr;
        if (!jit_cache().compile({&bv}, jerr)) FAIL(c, QSIM_ERR_CUDA, "jit block variant: %s", jerr.substr(0, 300).c_str());
        bfn = jit_cache().find(bkey);
    }
    auto block = [&](int i, uint64_t v, bool tab) {
        return launch_jit_range(c, si, i, per, c->stream, tab, bfn, x.lpos.data(), K, fix_of(v));
    };
    qsim_status st;
    if (!c->xstream) {  // created by pipeline() otherwise
        CK(c, cudaStreamCreateWithFlags(&c->xstream, cudaStreamNonBlocking));
        for (int i = 0; i < 2; i++) {
            CK(c, cudaEventCreateWithFlags(&c->x_ready[i], cudaEventDisableTiming));
            CK(c, cudaEventCreateWithFlags(&c->x_done[i], cudaEventDisableTiming));
            CK(c, cudaEventCreateWithFlags(&c->x_used[i], cudaEventDisableTiming));
        }
    }
    RangeGuard rg(c, 5, (uint64_t)n_local(c) * (32ULL << M));
    c->stats.passes += n_local(c);
    c->stats.jit_launches += n_local(c);
    c->stats.exchanges++;
    c->stats.overlapped++;  // (its time is overlap_ms, not pass_ms / exchange_ms)
    bool tab_done = false;
    // the transfer stream starts after everything before this step
    cudaEvent_t e0 = ov_event(c);
    CK(c, cudaEventRecord(e0, c->stream));
    CK(c, cudaStreamWaitEvent(c->xstream, e0, 0));
    if (c->transport == QSIM_TRANSPORT_VIRTUAL) {
        // pairs of blocks (shard r, block v) <-> (shard peer, block my_r), by round
        std::vector<char> done_blk((size_t)c->P * nval, 0);
        for (uint64_t j = 1; j < nval; j++)
            for (uint64_t r = 0; r < (uint64_t)c->P; r++) {
                const uint64_t my = rank_sub(r, x.gpos, M), v = my ^ j, peer = with_sub(r, x.gpos, M, v);
                if (peer < r) continue;
                for (auto rb : {std::make_pair(r, v), std::make_pair(peer, my)}) {
                    if (done_blk[rb.first * nval + rb.second]) continue;
                    if ((st = block((int)rb.first, rb.second, !tab_done)) != QSIM_OK) return st;
                    tab_done = true;
                    done_blk[rb.first * nval + rb.second] = 1;
                }
                cudaEvent_t e = ov_event(c);
                CK(c, cudaEventRecord(e, c->stream));
                CK(c, cudaStreamWaitEvent(c->xstream, e, 0));
                launch_swap_blocks(c->shards[r], c->shards[peer], M, K, x.lpos.data(), v, my, c->xstream);
                LAUNCHED(c);
            }
        for (uint64_t r = 0; r < (uint64_t)c->P; r++) {
            const uint64_t my = rank_sub(r, x.gpos, M);
            if ((st = block((int)r, my, !tab_done)) != QSIM_OK) return st;
            tab_done = true;
        }
        c->stats.exchange_bytes += (nval - 1) * chunk * 16;
    } else {
        const uint64_t my = rank_sub((uint64_t)c->rank, x.gpos, M);
        bool contiguous = true;  // the blocks are contiguous when lpos are the top K bits
        {
            std::vector<int> l = x.lpos;
            std::sort(l.begin(), l.end());
            for (int i = 0; i < K; i++)
                if (l[i] != M - K + i) contiguous = false;
        }
        const uint64_t scratch_amps = c->scratch_bytes / sizeof(double2), nbuf = contiguous ? 1 : 2;
        const uint64_t limit_amps = (uint64_t)c->chunk_mb * (1ULL << 20) / sizeof(double2);
        uint64_t piece = chunk;
        while (piece > 1 && (nbuf * piece > scratch_amps || piece > limit_amps)) piece >>= 1;
        if (nbuf * piece > scratch_amps) FAIL(c, QSIM_ERR_OOM, "scratch too small for exchange");
        double2 *rbuf = c->scratch, *sbuf = c->scratch + piece;
        for (uint64_t j = 1; j < nval; j++) {
            const uint64_t v = my ^ j;
            const int peer = (int)with_sub((uint64_t)c->rank, x.gpos, M, v);
            if ((st = block(0, v, !tab_done)) != QSIM_OK) return st;
            tab_done = true;
            cudaEvent_t e = ov_event(c);
            CK(c, cudaEventRecord(e, c->stream));
            CK(c, cudaStreamWaitEvent(c->xstream, e, 0));
            const uint64_t base = fix_of(v);
            // block v goes to the peer, the peer's block `my` lands here, in
            // pieces through the scratch, all on the transfer stream (a piece's
            // send completes before its unpack overwrites it)
            for (uint64_t k = 0; k < chunk / piece; k++) {
                const double2 *src = c->shards[0] + base + k * piece;
                if (!contiguous) {
                    launch_pack(c->shards[0], sbuf, M, K, x.lpos.data(), v, k * piece, piece, 0, c->xstream);
                    LAUNCHED(c);
                    src = sbuf;
                }
                CKC(c, group_start(_err));
                CKC(c, send(src, piece * sizeof(double2), peer, c->xstream, _err));
                CKC(c, recv(rbuf, piece * sizeof(double2), peer, c->xstream, _err));
                CKC(c, group_end(_err));
                launch_pack(c->shards[0], rbuf, M, K, x.lpos.data(), v, k * piece, piece, 1, c->xstream);
                LAUNCHED(c);
            }
        }
        if ((st = block(0, my, !tab_done)) != QSIM_OK) return st;
        c->stats.exchange_bytes += (nval - 1) * chunk * 16;
    }
    cudaEvent_t e1 = ov_event(c);
    CK(c, cudaEventRecord(e1, c->xstream));
    CK(c, cudaStreamWaitEvent(c->stream, e1, 0));
    return QSIM_OK;
}

// Launch step si of the plan (its uploads done, its JIT kernel compiled).
static qsim_status exec_step(qsim_ctx c, size_t si)
{
    PlanCache &pc = c->pc;
    const Step &s = pc.steps[si];
    const int M = c->M;
    qsim_status st;
    switch (s.type) {
    case ST_PASS: {
        RangeGuard rg(c, 0, (uint64_t)n_local(c) * (32ULL << M));
        CUfunction fn = c->jit ? jit_cache().find(pc.jkeys[si]) : nullptr;
        // the readout variant when this is the last data step before qsim_expectations
        CUfunction rfn = nullptr;
        if (fn && (int64_t)si == c->readout_step) {
            Step rv = s;
            rv.jit_readout = 1;
            const std::string rkey = jit_key(rv);
            rfn = jit_cache().find(rkey);
            if (!rfn) {
                std::string jerr;
                if (jit_cache().compile({&rv}, jerr)) rfn = jit_cache().find(rkey);
            }
            const size_t W = kTileBits + 1;
            if (rfn && ensure_dev(c, c->d_rdo, c->d_rdo_cap, (size_t)n_local(c) * s.pass.n_inst * W) != QSIM_OK)
                rfn = nullptr;
        }
        for (int i = 0; i < n_local(c); i++) {
            const uint64_t rb = (uint64_t)local_ranks(c, i) << M;
            if (fn) {
                double *red = rfn ? c->d_rdo + (size_t)i * s.pass.n_inst * (kTileBits + 1) : nullptr;
                if ((st = launch_jit_range(c, si, i, s.pass.n_inst, c->stream, i == 0, rfn, nullptr, 0, 0, red)) !=
                    QSIM_OK)
                    return st;
                c->stats.jit_launches++;
            } else {
                PassDesc d = s.pass;
                d.rank_bits = rb;
                launch_pass(d, s.ops.data(), c->shards[i], c->pass_variant, c->stream,
                            s.ops.size() > (size_t)kMaxPassOps ? c->d_ops + s.t : nullptr);
                LAUNCHED(c);
            }
            c->stats.passes++;
            if (c->timing) {  // executed FP64-pipe instructions, pairs with pass_ms
                const double fpt = fn ? jit_cache().fp64_per_thread(pc.jkeys[si]) : -1.0;
                c->stats.pass_fp64_slots += fpt >= 0 ? fpt * kPassThreads * (double)s.pass.n_inst : pass_fp64_slots(s, M);
            }
        }
        if (rfn) {  // the tile bits' and instance bits' physical positions after the store
            FusedExpectDesc &d = c->rdo_desc;
            d.M = M;
            d.n_inst = s.pass.n_inst;
            for (int b = 0; b < 64; b++) d.tile_of[b] = -1, d.inst_bit[b] = -1;
            for (int t = 0; t < kTileBits; t++) d.tile_of[s.pass.tp_out[t]] = t;
            for (int b = 0, k = 0; b < M; b++)
                if (d.tile_of[b] < 0) d.inst_bit[b] = k++;
            c->readout_ready = true;
            c->stats.fused_readouts++;
        }
        break;
    }
    case ST_GENERIC:
    case ST_PHASE: {
        RangeGuard rg(c, 1, 0);
        for (int i = 0; i < n_local(c); i++) {
            const uint64_t rb = (uint64_t)local_ranks(c, i) << M;
            if (s.type == ST_GENERIC)
                launch_gate_generic(c->shards[i], M, rb, s.t, s.cm, s.cv, s.code, s.m, c->stream);
            else
                launch_phase_generic(c->shards[i], M, rb, s.cm, s.cv, s.m[0], s.m[1], c->stream);
            LAUNCHED(c);
            c->stats.generic_launches++;
        }
        break;
    }
    case ST_PERM:
        if ((st = exec_perm(c, s)) != QSIM_OK) return st;
        break;
    case ST_PERMRUN:
        if ((st = exec_perm_run(c, s)) != QSIM_OK) return st;
        break;
    case ST_EXCHANGE:
        if ((st = exec_exchange(c, s)) != QSIM_OK) return st;
        break;
    case ST_RELABEL:
        c->stats.relabels++;
        break;
    case ST_PAIRWISE:
        if ((st = exec_pairwise(c, s)) != QSIM_OK) return st;
        break;
    }
    return QSIM_OK;
}

// Whether step s can launch with nothing uploaded or compiled first: no
// permutation tables, no interpreter program in global memory, and (JIT
// tier) its kernel already in the cache.  key: the JIT key of a pass.
static bool launchable_now(qsim_ctx c, const Step &s, std::string &key)
{
    if (s.type == ST_PERM || s.type == ST_PERMRUN) return false;
    if (s.type != ST_PASS) return true;
    if (!c->jit) return s.ops.size() <= (size_t)kMaxPassOps;
    key = jit_key(s);
    return jit_cache().find(key) != nullptr;
}

// FP64 and HBM peaks of this process's device, measured once (DFMA probe and
// streaming copy, ~0.1 s) for the planner's device-time model; 0 if the probe fails
static void measured_peaks(double &fp64, double &hbm)
{
    static double f = -1, b = -1;
    static std::mutex mu;
    std::lock_guard<std::mutex> g(mu);
    if (f < 0) {
        if (probe_peaks(&f, &b, 2) != 0) f = b = 0;
    }
    fp64 = f;
    hbm = b;
}

// SPMD creation (collective): measure the link rate to the partner rank
// (rank ^ 1; pieces of up to 64 MiB through the scratch, NCCL send/recv or
// the loopback copy), take the process's FP64 / HBM probe, and reduce all
// three to their minimum over the ranks (all-gather), so that every rank's
// planner sees the same numbers.
static qsim_status probe_spmd_rates(qsim_ctx c)
{
    double f = 0, b = 0;
    measured_peaks(f, b);
    double link = 0;
    const size_t bytes = std::min<size_t>((c->scratch_bytes / 2) / 16 * 16, (size_t)64 << 20);
    if (bytes >= ((size_t)1 << 20)) {
        cudaEvent_t e0 = ev_get(c), e1 = ev_get(c);
        const int peer = c->rank ^ 1;
        float best = 1e30f;
        for (int it = 0; it < 4; it++) {
            CK(c, cudaEventRecord(e0, c->stream));
            CKC(c, group_start(_err));
            CKC(c, send(c->scratch, bytes, peer, c->stream, _err));
            CKC(c, recv((char *)c->scratch + bytes, bytes, peer, c->stream, _err));
            CKC(c, group_end(_err));
            CK(c, cudaEventRecord(e1, c->stream));
            { qsim_status _s = sync_stream(c); if (_s != QSIM_OK) return _s; }
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it) best = std::min(best, ms);
        }
        c->event_pool.push_back(e0);
        c->event_pool.push_back(e1);
        link = best > 0 ? bytes / (best * 1e-3) / 1e9 : 0;
    }
    // min over ranks (a 0 anywhere -> 0: the nominal fallback everywhere)
    const double mine[3] = {f, b, link};
    double *dbuf = nullptr;
    if (cudaMalloc((void **)&dbuf, sizeof(double) * 3 * (c->P + 1)) != cudaSuccess) {
        cudaGetLastError();
        FAIL(c, QSIM_ERR_OOM, "rate probe buffer");
    }
    std::vector<double> all(3 * c->P);
    qsim_status st = QSIM_OK;
    if (cudaMemcpyAsync(dbuf, mine, sizeof(mine), cudaMemcpyHostToDevice, c->stream) != cudaSuccess) st = QSIM_ERR_CUDA;
    std::string err;
    if (st == QSIM_OK && c->comm->all_gather(dbuf, dbuf + 3, 3, c->stream, err)) {
        c->poisoned = true;
        c->last_error = err;
        st = QSIM_ERR_COMM;
    }
    if (st == QSIM_OK && cudaMemcpyAsync(all.data(), dbuf + 3, sizeof(double) * 3 * c->P, cudaMemcpyDeviceToHost,
                                         c->stream) != cudaSuccess)
        st = QSIM_ERR_CUDA;
    if (st == QSIM_OK) st = sync_stream(c);
    cudaFree(dbuf);
    if (st != QSIM_OK) return st;
    double m[3] = {all[0], all[1], all[2]};
    for (int r = 1; r < c->P; r++)
        for (int k = 0; k < 3; k++) m[k] = std::min(m[k], all[3 * r + k]);
    c->plan_fp64 = m[0];
    c->plan_hbm = m[1];
    c->plan_link_gbs = m[2];
    return QSIM_OK;
}

static qsim_status flush_impl(qsim_ctx c);
static qsim_status flush(qsim_ctx c)
{
    nvtxRangePushA("qsim flush (plan + launch)");
    const qsim_status st = flush_impl(c);
    nvtxRangePop();
    return st;
}

static qsim_status flush_impl(qsim_ctx c)
{
    c->readout_ready = false;
    c->readout_step = -1;
    if (c->poisoned) FAIL(c, QSIM_ERR_STATE, "context poisoned: %s", c->last_error.c_str());
    if (!c->init_pending && c->queue.empty()) return QSIM_OK;
    if (!c->init_pending && !c->initialized) FAIL(c, QSIM_ERR_STATE, "gates queued before qsim_init_basis");
    auto t0 = std::chrono::steady_clock::now();
    PlanCache &pc = c->pc;
    bool hit = c->plan_cache && pc.valid && pc.with_init == c->init_pending && pc.queue.size() == c->queue.size() &&
               (c->init_pending || pc.phys_before == c->planner->phys_of);
    for (size_t i = 0; hit && i < c->queue.size(); i++) hit = same_gate(pc.queue[i], c->queue[i]);
    const bool with_init = c->init_pending;
    uint64_t init_phys = 0;
    if (!hit) {
        pc.valid = false;
        pc.phys_before = c->planner->phys_of;
    }
    if (c->init_pending) {
        if (hit) {
            c->planner->phys_of = pc.phys_init;
            for (int q = 0; q < c->n; q++) c->planner->qubit_at[pc.phys_init[q]] = q;
        } else {
            c->planner->choose_initial_layout(c->queue);
            pc.phys_init = c->planner->phys_of;
        }
        init_phys = 0;
        for (int q = 0; q < c->n; q++)
            if ((c->init_index >> q) & 1) init_phys |= 1ULL << c->planner->phys_of[q];
        c->init_pending = false;
        c->initialized = true;
    }
    std::vector<Step> &steps = pc.steps;
    // After qsim_init_basis: a plan that starts (after relabels) with a pass
    // synthesises the basis state in that pass's registers instead of reading
    // the shard, and the zero-fill is skipped; otherwise the init kernel runs
    // before the first data step.
    bool init_left = with_init;
    auto mark_fresh = [&](size_t from) {
        if (!init_left) return;
        for (size_t i = from; i < steps.size(); i++) {
            if (steps[i].type == ST_RELABEL) continue;
            if (steps[i].type == ST_PASS) { steps[i].pass.fresh = 1; steps[i].pass.init_phys = init_phys; }
            return;
        }
    };
    auto launch_init_all = [&]() -> qsim_status {
        init_left = false;
        const uint64_t owner = init_phys >> c->M, li = init_phys & ((1ULL << c->M) - 1);
        for (int k = 0; k < n_local(c); k++) {
            const bool mine = (uint64_t)local_ranks(c, k) == owner;
            launch_init(c->shards[k], 1ULL << c->M, mine ? (int64_t)li : -1, c->stream);
            LAUNCHED(c);
        }
        return QSIM_OK;
    };
    // launch step i (and, for an overlapped pass + exchange, step i + 1 too:
    // *used = steps consumed)
    auto launch_one = [&](size_t i, size_t *used) -> qsim_status {
        *used = 1;
        if (init_left && steps[i].type != ST_RELABEL) {
            if (steps[i].type == ST_PASS && steps[i].pass.fresh) init_left = false;
            else if (qsim_status e = launch_init_all()) return e;
        }
        if (overlap_ok(c, i)) {
            *used = 2;
            return exec_pass_exchange(c, i);
        }
        return exec_step(c, i);
    };
    // a pass whose successor is not planned yet waits for it when the state is
    // sharded (it may be an exchange to overlap with)
    auto wait_successor = [&](const std::vector<Step> &out, size_t i) {
        return ((c->overlap && c->P > 1) || c->want_readout) && c->jit && out[i].type == ST_PASS &&
               i + 1 == out.size();
    };
    size_t next = 0;  // first step not launched yet
    if (hit) {
        c->planner->phys_of = pc.phys_after;
        for (int q = 0; q < c->n; q++) c->planner->qubit_at[pc.phys_after[q]] = q;
        c->queue.clear();
        c->stats.plan_cache_hits++;
        c->stats.plan_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    } else {
        // Plan, launching each step as soon as the planner emits it when it
        // needs nothing uploaded or compiled: the device runs the first
        // passes while the host plans the rest.  The first step that needs an
        // upload or a new JIT kernel ends the streaming; the rest of the plan
        // then goes the batch way below (one upload, parallel NVRTC).
        steps.clear();
        pc.jkeys.clear();
        pc.params.clear();
        bool streaming = true;
        qsim_status err = QSIM_OK;
        double launch_ms = 0;
        PlanOptions opt;
        opt.fusion = c->fusion;
        opt.block_fusion = c->block_fusion;
        opt.low_remap = c->low_remap;
        opt.remap_lookahead = c->remap_lookahead;
        opt.max_scan = c->max_scan;
        opt.global_policy = c->global_policy;
        opt.overlap = c->jit && c->P > 1 &&
                      (c->transport == QSIM_TRANSPORT_VIRTUAL ? c->overlap >= 2 : spmd(c) && c->overlap >= 1);
        if (c->P > 1) {  // the sharded planner weighs alternatives by modelled device time
            double f = c->plan_fp64, b = c->plan_hbm;
            if (!spmd(c)) measured_peaks(f, b);  // one process: the same values for every shard
            if (spmd(c) && c->plan_link_gbs > 0 && c->peak_link_gbs <= 0) opt.peak_link = c->plan_link_gbs * 1e9;
            if (f > 0) opt.peak_fp64 = PlanOptions::kPassFp64Eff * f;
            if (b > 0) opt.peak_hbm = PlanOptions::kPassHbmEff * b;
            if (c->peak_link_gbs > 0) opt.peak_link = c->peak_link_gbs * 1e9;
        }
        opt.sink = [&](std::vector<Step> &out) {
            if (!streaming || err != QSIM_OK) return;
            const auto tl = std::chrono::steady_clock::now();
            while (next < out.size()) {
                mark_fresh(next);
                std::string key;
                if (!launchable_now(c, out[next], key)) { streaming = false; break; }
                if (wait_successor(out, next)) break;  // streaming continues at the next emit
                if (pc.jkeys.size() < out.size()) { pc.jkeys.resize(out.size()); pc.params.resize(out.size()); }
                pc.jkeys[next] = key;
                size_t used = 1;
                if ((err = launch_one(next, &used)) != QSIM_OK) break;
                next += used;
            }
            launch_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tl).count();
        };
        c->planner->plan(c->queue, opt, steps);
        pc.queue.swap(c->queue);
        c->queue.clear();
        pc.with_init = with_init;
        pc.phys_after = c->planner->phys_of;
        c->stats.plan_ms +=
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count() - launch_ms;
        if (err != QSIM_OK) return err;
        pc.jkeys.resize(steps.size());
        pc.params.resize(steps.size());
        pc.valid = true;
        c->stats.streamed_steps += next;
    }
    c->stats.flushes++;
    if (next == steps.size()) {
        return init_left ? launch_init_all() : QSIM_OK;  // no data step (only relabels, or no gates)
    }
    mark_fresh(next);
    qsim_status st = upload_program(c, steps);
    if (st != QSIM_OK) return st;
    if (c->jit && !hit) {
        std::vector<const Step *> ps;
        for (size_t i = next; i < steps.size(); i++)
            if (steps[i].type == ST_PASS) ps.push_back(&steps[i]);
        std::string jerr;
        auto tj = std::chrono::steady_clock::now();
        if (!jit_cache().compile(ps, jerr)) {
            c->jit = 0;  // keep running on the interpreter tier, but say why
            c->last_error = jerr;
        }
        c->stats.plan_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tj).count();
        for (size_t i = next; i < steps.size(); i++)
            if (steps[i].type == ST_PASS) pc.jkeys[i] = jit_key(steps[i]);
    }
    if (c->want_readout && c->jit) {  // the last data step, if a pass not launched yet, fuses the readout
        size_t L = steps.size();
        while (L > 0 && steps[L - 1].type == ST_RELABEL) L--;
        if (L > next && steps[L - 1].type == ST_PASS) c->readout_step = (int64_t)(L - 1);
    }
    for (size_t i = next, used = 1; i < steps.size(); i += used)
        if ((st = launch_one(i, &used)) != QSIM_OK) return st;
    return init_left ? launch_init_all() : QSIM_OK;
}

// ------------------------------------------------------------ ABI
extern "C" {

const char *qsim_status_str(qsim_status s)
{
    switch (s) {
    case QSIM_OK: return "QSIM_OK";
    case QSIM_ERR_ARG: return "QSIM_ERR_ARG";
    case QSIM_ERR_QUBIT_RANGE: return "QSIM_ERR_QUBIT_RANGE";
    case QSIM_ERR_DUP_QUBIT: return "QSIM_ERR_DUP_QUBIT";
    case QSIM_ERR_NOT_UNITARY: return "QSIM_ERR_NOT_UNITARY";
    case QSIM_ERR_NOT_PERMUTATION: return "QSIM_ERR_NOT_PERMUTATION";
    case QSIM_ERR_OOM: return "QSIM_ERR_OOM";
    case QSIM_ERR_CUDA: return "QSIM_ERR_CUDA";
    case QSIM_ERR_COMM: return "QSIM_ERR_COMM";
    case QSIM_ERR_STATE: return "QSIM_ERR_STATE";
    case QSIM_ERR_UNSUPPORTED: return "QSIM_ERR_UNSUPPORTED";
    }
    return "unknown";
}

const char *qsim_last_error(qsim_ctx ctx) { return ctx ? ctx->last_error.c_str() : ""; }

size_t qsim_scratch_bytes(int n_qubits, int n_ranks)
{
    if (n_ranks <= 1 || n_qubits < 2) return 0;
    const int M = n_qubits - ilog2(n_ranks);
    const size_t shard = (size_t)16 << M;
    return std::min<size_t>(shard, (size_t)4 << 30);
}

qsim_status qsim_get_loopback_id(void *out128)
{
    if (!out128) return QSIM_ERR_ARG;
    new_loopback_id(out128);
    return QSIM_OK;
}

qsim_status qsim_get_unique_id(void *out128)
{
    if (!out128) return QSIM_ERR_ARG;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return QSIM_ERR_COMM;
    std::memcpy(out128, &id, sizeof(id));
    return QSIM_OK;
}

qsim_status qsim_create_rank(int n_qubits, int n_gpus, int rank, const void *nccl_unique_id, void *shard,
                             size_t shard_bytes, void *scratch, size_t scratch_bytes, void *cuda_stream,
                             qsim_ctx *out)
{
    if (!out || n_gpus < 1 || (n_gpus & (n_gpus - 1)) || n_gpus > 64) return QSIM_ERR_ARG;
    if (n_gpus > 1 && !nccl_unique_id) return QSIM_ERR_ARG;
    const int G = ilog2(n_gpus);
    if (n_qubits - G < 1 || n_qubits > 62) return QSIM_ERR_ARG;
    if (shard && shard_bytes != ((size_t)16 << (n_qubits - G))) return QSIM_ERR_ARG;
    qsim_config cfg;
    std::memset(&cfg, 0, sizeof(cfg));
    cfg.n_qubits = n_qubits;
    cfg.n_ranks = n_gpus;
    cfg.rank = n_gpus > 1 ? rank : 0;
    cfg.transport = n_gpus > 1 ? QSIM_TRANSPORT_NCCL : QSIM_TRANSPORT_LOCAL;
    cfg.shards[0] = shard;
    cfg.scratch = scratch;
    cfg.scratch_bytes = scratch_bytes;
    cfg.stream = cuda_stream;
    if (n_gpus > 1) std::memcpy(cfg.nccl_id, nccl_unique_id, sizeof(cfg.nccl_id));
    return qsim_create_ext(&cfg, out);
}

qsim_status qsim_create_ext(const qsim_config *cfg, qsim_ctx *out)
{
    if (!cfg || !out) return QSIM_ERR_ARG;
    *out = nullptr;
    const int n = cfg->n_qubits, P = cfg->n_ranks;
    if (n < 1 || n > 62) return QSIM_ERR_QUBIT_RANGE;
    if (P < 1 || P > 64 || (P & (P - 1))) return QSIM_ERR_ARG;
    const int G = ilog2(P);
    if (n - G < 1) return QSIM_ERR_ARG;
    if (cfg->transport == QSIM_TRANSPORT_LOCAL && P != 1) return QSIM_ERR_ARG;
    if (cfg->transport < 0 || cfg->transport > 3) return QSIM_ERR_ARG;
    const bool spmd_tp = cfg->transport == QSIM_TRANSPORT_NCCL || cfg->transport == QSIM_TRANSPORT_LOOPBACK;
    if (spmd_tp && (cfg->rank < 0 || cfg->rank >= P)) return QSIM_ERR_ARG;
    cudaGetLastError();  // do not inherit a stale error of another context
    qsim_ctx c = new qsim_ctx_s();
    c->n = n;
    c->P = P;
    c->G = G;
    c->M = n - G;
    c->rank = spmd_tp ? cfg->rank : 0;
    c->transport = cfg->transport;
    c->planner = new Planner(n, G);
    auto bail = [&](qsim_status s) {
        qsim_destroy(c);
        return s;
    };
    const size_t shard_bytes = (size_t)16 << c->M;
    const int nsh = cfg->transport == QSIM_TRANSPORT_VIRTUAL ? P : 1;
    bool any_null = false;
    for (int i = 0; i < nsh; i++) any_null |= cfg->shards[i] == nullptr;
    c->own_shards = any_null;
    for (int i = 0; i < nsh; i++) {
        double2 *p = (double2 *)cfg->shards[i];
        if (any_null) {
            if (cudaMalloc((void **)&p, shard_bytes) != cudaSuccess) {
                cudaGetLastError();
                c->shards.resize(i);
                return bail(QSIM_ERR_OOM);
            }
        } else if ((uintptr_t)p % 256) {
            return bail(QSIM_ERR_ARG);
        }
        c->shards.push_back(p);
    }
    if (cfg->stream) {
        c->stream = (cudaStream_t)cfg->stream;
    } else {
        if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) return bail(QSIM_ERR_CUDA);
        c->own_stream = true;
    }
    if (spmd_tp) {
        c->scratch = (double2 *)cfg->scratch;
        c->scratch_bytes = cfg->scratch_bytes;
        if (!c->scratch) {
            c->scratch_bytes = qsim_scratch_bytes(n, P);
            if (cudaMalloc((void **)&c->scratch, c->scratch_bytes) != cudaSuccess) {
                cudaGetLastError();
                return bail(QSIM_ERR_OOM);
            }
            c->own_scratch = true;
        }
        if (const char *e = getenv("QSIM_COMM_TIMEOUT_S")) c->comm_timeout_ms = 1e3 * atof(e);
        std::string err;
        c->comm = cfg->transport == QSIM_TRANSPORT_NCCL ? make_nccl_comm(cfg->nccl_id, P, cfg->rank, c->comm_timeout_ms, err)
                                                        : make_loopback_comm(cfg->nccl_id, P, cfg->rank, c->comm_timeout_ms, err);
        if (!c->comm) {
            fprintf(stderr, "qsim_create_ext: %s\n", err.c_str());
            return bail(QSIM_ERR_COMM);
        }
        if (P > 1) {
            qsim_status ps = probe_spmd_rates(c);
            if (ps != QSIM_OK) return bail(ps);
        }
    }
    {
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess)
            cudaDeviceGetAttribute(&c->n_sm, cudaDevAttrMultiProcessorCount, dev);
        cudaGetLastError();
    }
    if (cudaMalloc((void **)&c->d_shard_ptrs, sizeof(double2 *) * nsh) != cudaSuccess) return bail(QSIM_ERR_OOM);
    if (cudaMemcpy(c->d_shard_ptrs, c->shards.data(), sizeof(double2 *) * nsh, cudaMemcpyHostToDevice) != cudaSuccess)
        return bail(QSIM_ERR_CUDA);
    *out = c;
    return QSIM_OK;
}

qsim_status qsim_create(int n_qubits, int n_gpus, qsim_ctx *out)
{
    if (n_gpus != 1) return QSIM_ERR_ARG;
    qsim_config cfg;
    std::memset(&cfg, 0, sizeof(cfg));
    cfg.n_qubits = n_qubits;
    cfg.n_ranks = 1;
    cfg.transport = QSIM_TRANSPORT_LOCAL;
    return qsim_create_ext(&cfg, out);
}

qsim_status qsim_destroy(qsim_ctx c)
{
    if (!c) return QSIM_OK;
    if (c->stream && !c->poisoned) cudaStreamSynchronize(c->stream);
    if (c->xstream && !c->poisoned) cudaStreamSynchronize(c->xstream);
    delete c->comm;
    for (int i = 0; i < 2; i++)
        for (cudaEvent_t e : {c->x_ready[i], c->x_done[i], c->x_used[i]})
            if (e) cudaEventDestroy(e);
    if (c->xstream) cudaStreamDestroy(c->xstream);
    if (c->own_shards)
        for (double2 *p : c->shards) cudaFree(p);
    if (c->own_scratch) cudaFree(c->scratch);
    if (c->d_ops) cudaFree(c->d_ops);
    if (c->d_ttab) cudaFree(c->d_ttab);
    if (c->d_perm) cudaFree(c->d_perm);
    if (c->d_red) cudaFree(c->d_red);
    if (c->d_rdo) cudaFree(c->d_rdo);
    if (c->d_samp) cudaFree(c->d_samp);
    if (c->d_shard_ptrs) cudaFree(c->d_shard_ptrs);
    if (c->h_ops) cudaFreeHost(c->h_ops);
    if (c->h_perm) cudaFreeHost(c->h_perm);
    if (c->upload_done) cudaEventDestroy(c->upload_done);
    for (auto &r : c->ranges) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : c->event_pool) cudaEventDestroy(e);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c->planner;
    delete c;
    return QSIM_OK;
}

#define GUARD(c)                                                                          \
    do {                                                                                  \
        if (!(c)) return QSIM_ERR_ARG;                                                    \
        if ((c)->poisoned) FAIL(c, QSIM_ERR_STATE, "context poisoned: %s", (c)->last_error.c_str()); \
    } while (0)

qsim_status qsim_init_basis(qsim_ctx c, uint64_t index)
{
    GUARD(c);
    if (c->n < 64 && index >> c->n) FAIL(c, QSIM_ERR_ARG, "index %llu >= 2^%d", (unsigned long long)index, c->n);
    // discard queued gates: the state is being re-initialised
    c->queue.clear();
    delete c->planner;
    c->planner = new Planner(c->n, c->G);
    c->init_pending = true;
    c->init_index = index;
    return QSIM_OK;
}

static qsim_status enqueue(qsim_ctx c, const qsim_gate &g)
{
    GateRec r;
    qsim_status s = to_rec(c, c->n, g, r);
    if (s != QSIM_OK) return s;
    if (!c->initialized && !c->init_pending) FAIL(c, QSIM_ERR_STATE, "gate before qsim_init_basis");
    r.id = (int)c->queue.size();
    c->queue.push_back(std::move(r));
    c->stats.gates++;
    return QSIM_OK;
}

qsim_status qsim_apply_1q(qsim_ctx c, int q, const qsim_c128 u[4])
{
    GUARD(c);
    if (!u) return QSIM_ERR_ARG;
    qsim_gate g;
    std::memset(&g, 0, sizeof(g));
    g.kind = QSIM_G_1Q;
    g.target = q;
    for (int k = 0; k < 4; k++) g.u[k] = u[k];
    return enqueue(c, g);
}

qsim_status qsim_apply_controlled(qsim_ctx c, const int *controls, int n_controls, int target, const qsim_c128 u[4])
{
    GUARD(c);
    if (!u || (n_controls > 0 && !controls) || n_controls < 0 || n_controls > QSIM_MAX_CONTROLS) return QSIM_ERR_ARG;
    qsim_gate g;
    std::memset(&g, 0, sizeof(g));
    g.kind = QSIM_G_CTRL;
    g.target = target;
    g.n_controls = n_controls;
    for (int i = 0; i < n_controls; i++) g.controls[i] = controls[i];
    for (int k = 0; k < 4; k++) g.u[k] = u[k];
    return enqueue(c, g);
}

qsim_status qsim_apply_perm(qsim_ctx c, const int *controls, int n_controls, const int *targets, int n_targets,
                            const uint32_t *perm)
{
    GUARD(c);
    if ((n_controls > 0 && !controls) || n_controls < 0 || n_controls > QSIM_MAX_CONTROLS) return QSIM_ERR_ARG;
    if (!targets || n_targets < 1 || n_targets > QSIM_MAX_PERM_TARGETS) return QSIM_ERR_ARG;
    qsim_gate g;
    std::memset(&g, 0, sizeof(g));
    g.kind = QSIM_G_PERM;
    g.n_controls = n_controls;
    g.n_targets = n_targets;
    for (int i = 0; i < n_controls; i++) g.controls[i] = controls[i];
    for (int i = 0; i < n_targets; i++) g.targets[i] = targets[i];
    g.perm = perm;
    return enqueue(c, g);
}

qsim_status qsim_apply_swap(qsim_ctx c, int a, int b)
{
    GUARD(c);
    qsim_gate g;
    std::memset(&g, 0, sizeof(g));
    g.kind = QSIM_G_SWAP;
    g.targets[0] = a;
    g.targets[1] = b;
    return enqueue(c, g);
}

qsim_status qsim_run_circuit(qsim_ctx c, const qsim_gate *gates, size_t n_gates)
{
    GUARD(c);
    if (n_gates && !gates) return QSIM_ERR_ARG;
    if (!c->initialized && !c->init_pending) FAIL(c, QSIM_ERR_STATE, "gate before qsim_init_basis");
    // validated straight into the queue; on an error the queue is cut back
    const size_t q0 = c->queue.size();
    c->queue.resize(q0 + n_gates);
    for (size_t i = 0; i < n_gates; i++) {
        qsim_status s = to_rec(c, c->n, gates[i], c->queue[q0 + i]);
        if (s != QSIM_OK) {
            c->queue.resize(q0);
            std::string e = c->last_error;
            FAIL(c, s, "gate %zu: %s", i, e.c_str());
        }
        c->queue[q0 + i].id = (int)(q0 + i);
    }
    c->stats.gates += n_gates;
    return QSIM_OK;
}

qsim_status qsim_remap(qsim_ctx c, const int *local_qubits, const int *global_qubits, int K)
{
    GUARD(c);
    if (K < 0 || K > c->G || (K && (!local_qubits || !global_qubits))) FAIL(c, QSIM_ERR_ARG, "K=%d out of [0,%d]", K, c->G);
    qsim_status s = flush(c);
    if (s != QSIM_OK) return s;
    uint64_t seen = 0;
    std::vector<int> lq, gq;
    for (int i = 0; i < K; i++) {
        int l = local_qubits[i], g = global_qubits[i];
        if (l < 0 || l >= c->n || g < 0 || g >= c->n) FAIL(c, QSIM_ERR_QUBIT_RANGE, "qubit outside range");
        if (((seen >> l) & 1) || ((seen >> g) & 1) || l == g) FAIL(c, QSIM_ERR_DUP_QUBIT, "qubit repeated");
        seen |= (1ULL << l) | (1ULL << g);
        if (c->planner->phys_of[l] >= c->M) FAIL(c, QSIM_ERR_ARG, "qubit %d is not local", l);
        if (c->planner->phys_of[g] < c->M) FAIL(c, QSIM_ERR_ARG, "qubit %d is not nonlocal", g);
        lq.push_back(l);
        gq.push_back(g);
    }
    std::vector<Step> steps;
    c->planner->remap(lq, gq, steps);
    for (auto &st : steps)
        if ((s = exec_exchange(c, st)) != QSIM_OK) return s;
    return QSIM_OK;
}

qsim_status qsim_sync(qsim_ctx c)
{
    GUARD(c);
    qsim_status s = flush(c);
    if (s != QSIM_OK) return s;
    { qsim_status _s = sync_stream(c); if (_s != QSIM_OK) return _s; }
    return collect_timing(c);
}

qsim_status qsim_get_layout(qsim_ctx c, int *out)
{
    GUARD(c);
    if (!out) return QSIM_ERR_ARG;
    qsim_status s = flush(c);
    if (s != QSIM_OK) return s;
    for (int q = 0; q < c->n; q++) out[q] = c->planner->phys_of[q];
    return QSIM_OK;
}

// cross-shard sum of per-shard host vectors in fixed rank order
static qsim_status sum_over_ranks(qsim_ctx c, std::vector<std::vector<double>> &per, double *out, size_t len)
{
    if (spmd(c)) {
        qsim_status s;
        if ((s = ensure_dev(c, c->d_red, c->d_red_cap, len * (c->P + 1))) != QSIM_OK) return s;
        CK(c, cudaMemcpyAsync(c->d_red, per[0].data(), len * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        CKC(c, all_gather(c->d_red, c->d_red + len, len, c->stream, _err));
        std::vector<double> all(len * c->P);
        CK(c, cudaMemcpyAsync(all.data(), c->d_red + len, len * c->P * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        { qsim_status _s = sync_stream(c); if (_s != QSIM_OK) return _s; }
        for (size_t j = 0; j < len; j++) {
            double a = 0.0;
            for (int r = 0; r < c->P; r++) a += all[r * len + j];
            out[j] = a;
        }
        return QSIM_OK;
    }
    for (size_t j = 0; j < len; j++) {
        double a = 0.0;
        for (size_t r = 0; r < per.size(); r++) a += per[r][j];
        out[j] = a;
    }
    return QSIM_OK;
}

static qsim_status probabilities_impl(qsim_ctx c, const int *qubits, int k, double *out)
{
    if (k < 0 || k > 24 || (k && !qubits) || !out) FAIL(c, QSIM_ERR_ARG, "bad qubit list (k=%d)", k);
    if (!c->initialized && !c->init_pending) FAIL(c, QSIM_ERR_STATE, "readout before qsim_init_basis");
    uint64_t seen = 0;
    for (int j = 0; j < k; j++) {
        if (qubits[j] < 0 || qubits[j] >= c->n) FAIL(c, QSIM_ERR_QUBIT_RANGE, "qubit %d", qubits[j]);
        if ((seen >> qubits[j]) & 1) FAIL(c, QSIM_ERR_DUP_QUBIT, "qubit %d repeated", qubits[j]);
        seen |= 1ULL << qubits[j];
    }
    qsim_status s = flush(c);
    if (s != QSIM_OK) return s;
    const int M = c->M, cb = std::min(12, M);
    ProbsDesc d{};
    d.cb = cb;
    d.M = M;
    d.k = k;
    uint32_t listed_low = 0;
    uint64_t listed_chunk = 0;
    for (int j = 0; j < k; j++) {
        const int p = c->planner->phys_of[qubits[j]];
        d.pos[j] = p;
        if (p < cb) { d.lowpos[d.k_low++] = p; listed_low |= 1u << p; }
        else if (p < M) listed_chunk |= 1ULL << (p - cb);
    }
    d.red_mask = ((1u << cb) - 1) & ~listed_low;
    for (int b = 0; b < M - cb; b++)
        if (!((listed_chunk >> b) & 1)) d.freepos[d.n_free++] = b;
    const uint64_t nch = 1ULL << (M - cb);
    const size_t partial_len = (size_t)nch << d.k_low, B = (size_t)1 << k;
    if (partial_len * 8 > ((size_t)8 << 30)) FAIL(c, QSIM_ERR_UNSUPPORTED, "marginal partial buffer too large");
    if ((s = ensure_dev(c, c->d_red, c->d_red_cap, partial_len + B)) != QSIM_OK) return s;
    std::vector<std::vector<double>> per(n_local(c), std::vector<double>(B));
    RangeGuard rg(c, 4, 0);
    for (int i = 0; i < n_local(c); i++) {
        d.rank = (uint64_t)local_ranks(c, i);
        launch_probs(c->shards[i], d, c->d_red, c->d_red + partial_len, c->stream);
        LAUNCHED(c);
        CK(c, cudaMemcpyAsync(per[i].data(), c->d_red + partial_len, B * sizeof(double), cudaMemcpyDeviceToHost,
                              c->stream));
        { qsim_status _s = sync_stream(c); if (_s != QSIM_OK) return _s; }
    }
    return sum_over_ranks(c, per, out, B);
}

qsim_status qsim_probabilities(qsim_ctx c, const int *qubits, int k, double *out)
{
    GUARD(c);
    return probabilities_impl(c, qubits, k, out);
}

// <Q_i> (Eq. Shor7): per-shard physical-bit sums on the device, rank order
// sum + logical order on the device (k_expect_logical; same additions in the
// same order as a host loop), then one D2H of n doubles into `out`.
static qsim_status expectations_impl(qsim_ctx c, double *out, bool sync)
{
    if (!out) return QSIM_ERR_ARG;
    if (!c->initialized && !c->init_pending) FAIL(c, QSIM_ERR_STATE, "readout before qsim_init_basis");
    c->want_readout = c->fuse_readout != 0;
    qsim_status s = flush(c);
    c->want_readout = false;
    if (s != QSIM_OK) return s;
    const bool fused = c->readout_ready;
    c->readout_ready = false;
    const int M = c->M, cb = std::min(12, M), n = c->n, S = spmd(c) ? c->P : n_local(c);
    const uint64_t nch = 1ULL << (M - cb);
    const size_t plen = std::max<size_t>(nch * (cb + 1), fused ? expect_fused_scratch(c->rdo_desc.n_inst) : 0),
                 vlen = (size_t)M + 1;
    // partial sums | this process's shard vectors | all ranks' vectors (NCCL) | logical result
    const size_t need = plen + (size_t)n_local(c) * vlen + (size_t)S * vlen + n;
    if ((s = ensure_dev(c, c->d_red, c->d_red_cap, need)) != QSIM_OK) return s;
    double *own = c->d_red + plen, *all = own + (size_t)n_local(c) * vlen, *res = all + (size_t)S * vlen;
    RangeGuard rg(c, 4, 0);
    for (int i = 0; i < n_local(c); i++) {
        if (fused)  // from the last pass's per-tile partials: no second read of the state (d_red as scratch)
            launch_expect_fused(c->d_rdo + (size_t)i * c->rdo_desc.n_inst * (kTileBits + 1), c->rdo_desc, c->d_red,
                                own + (size_t)i * vlen, c->stream);
        else
            launch_expect(c->shards[i], M, c->d_red, own + (size_t)i * vlen, c->stream);
        LAUNCHED(c);
    }
    const double *phys = own;
    if (spmd(c)) {
        CKC(c, all_gather(own, all, vlen, c->stream, _err));
        phys = all;
    }
    ExpectMap m{};
    m.n = n;
    m.M = M;
    m.S = S;
    for (int q = 0; q < n; q++) m.phys_of[q] = c->planner->phys_of[q];
    launch_expect_logical(phys, m, res, c->stream);
    LAUNCHED(c);
    CK(c, cudaMemcpyAsync(out, res, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (sync) { qsim_status _s = sync_stream(c); if (_s != QSIM_OK) return _s; }
    return QSIM_OK;
}

qsim_status qsim_expectations(qsim_ctx c, double *out)
{
    GUARD(c);
    return expectations_impl(c, out, true);
}

qsim_status qsim_expectations_async(qsim_ctx c, double *out)
{
    GUARD(c);
    return expectations_impl(c, out, false);
}

// Two-level sampler for k > 24 listed qubits (up to the whole
// register): the same draw u_s and the same outcome min{beta : C(beta) > u_s}
// as the one-level rule (reading R14), with C(beta) = C_hi(beta_hi - 1) +
// C_lo(beta_lo).  Level 1: the marginal of the top kh listed qubits (the
// qsim_probabilities path), its CDF and, per shot, the high bin and the
// residual draw, on the device.  Level 2: for the distinct high bins, the
// conditional marginal of the c low listed qubits (k_bin_marginal, every
// shard's part summed in rank order), its CDF and the low bits by binary
// search, on the device.  Memory: 2^kh + batches of <= 2^24 bin entries.
static qsim_status measure_two_level(qsim_ctx c, const int *qubits, int k, uint64_t seed, uint64_t n_shots,
                                     uint64_t *out)
{
    const int kh = std::max(20, k - 16), cl = k - kh;
    uint64_t seen = 0;
    for (int j = 0; j < k; j++) {
        if (qubits[j] < 0 || qubits[j] >= c->n) FAIL(c, QSIM_ERR_QUBIT_RANGE, "qubit %d", qubits[j]);
        if ((seen >> qubits[j]) & 1) FAIL(c, QSIM_ERR_DUP_QUBIT, "qubit %d repeated", qubits[j]);
        seen |= 1ULL << qubits[j];
    }
    std::vector<double> phi((size_t)1 << kh);
    qsim_status s = probabilities_impl(c, qubits + cl, kh, phi.data());
    if (s != QSIM_OK) return s;
    if (!n_shots) return QSIM_OK;
    const size_t BH = phi.size(), per = (size_t)1 << cl;
    size_t batch_rows = std::max<size_t>(1, ((size_t)1 << 24) / per);
    if (c->sample_batch > 0) batch_rows = std::min(batch_rows, (size_t)c->sample_batch);
    // device: p_hi | CDF | res (n) | rows (batch_rows x per) | bhi, shot_idx, out (n each) | bins | shot_row (u32)
    const size_t need = 2 * BH + n_shots + batch_rows * per + 3 * n_shots + batch_rows + n_shots / 2 + 8;
    if ((s = ensure_dev(c, c->d_samp, c->d_samp_cap, need)) != QSIM_OK) return s;
    double *dp = c->d_samp, *dc = dp + BH, *dres = dc + BH, *drows = dres + n_shots;
    uint64_t *dbhi = (uint64_t *)(drows + batch_rows * per), *didx = dbhi + n_shots, *dout = didx + n_shots,
             *dbins = dout + n_shots;
    uint32_t *drow = (uint32_t *)(dbins + batch_rows);
    RangeGuard rg(c, 4, 0);
    CK(c, cudaMemcpyAsync(dp, phi.data(), BH * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    launch_sample_hi(dp, kh, seed, n_shots, dc, dbhi, dres, c->stream);
    LAUNCHED(c);
    std::vector<uint64_t> bhi(n_shots);
    CK(c, cudaMemcpyAsync(bhi.data(), dbhi, n_shots * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
    { qsim_status _s = sync_stream(c); if (_s != QSIM_OK) return _s; }
    // shots grouped by high bin (host bookkeeping: which rows to build)
    std::vector<uint64_t> order(n_shots);
    for (uint64_t i = 0; i < n_shots; i++) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) { return bhi[a] < bhi[b]; });
    int pos_lo[24], pos_hi[24], pos_un[64], nu = 0;
    for (int j = 0; j < cl; j++) pos_lo[j] = c->planner->phys_of[qubits[j]];
    for (int j = 0; j < kh; j++) pos_hi[j] = c->planner->phys_of[qubits[cl + j]];
    for (int q = 0; q < c->n; q++)
        if (!((seen >> q) & 1)) pos_un[nu++] = c->planner->phys_of[q];
    // rows of one batch: per shard its part, summed in rank order (on the
    // host for SPMD ranks, as the marginals are)
    std::vector<std::vector<double>> per_rank(n_local(c));
    std::vector<double> rows;
    for (uint64_t i0 = 0; i0 < n_shots;) {
        std::vector<uint64_t> bins;
        std::vector<uint32_t> shot_row;
        std::vector<uint64_t> shot_idx;
        uint64_t i = i0;
        while (i < n_shots) {
            const uint64_t b = bhi[order[i]];
            if (bins.empty() || bins.back() != b) {
                if (bins.size() == batch_rows) break;
                bins.push_back(b);
            }
            shot_row.push_back((uint32_t)(bins.size() - 1));
            shot_idx.push_back(order[i]);
            i++;
        }
        const size_t nb = bins.size(), len = nb * per;
        CK(c, cudaMemcpyAsync(dbins, bins.data(), nb * sizeof(uint64_t), cudaMemcpyHostToDevice, c->stream));
        rows.assign(len, 0.0);
        for (int r = 0; r < n_local(c); r++) {
            per_rank[r].assign(len, 0.0);
            launch_bin_marginal(c->shards[r], c->M, (uint64_t)local_ranks(c, r), cl, pos_lo, kh, pos_hi, nu, pos_un,
                                dbins, nb, drows, c->stream);
            LAUNCHED(c);
            CK(c, cudaMemcpyAsync(per_rank[r].data(), drows, len * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
            { qsim_status _s = sync_stream(c); if (_s != QSIM_OK) return _s; }
        }
        if ((s = sum_over_ranks(c, per_rank, rows.data(), len)) != QSIM_OK) return s;
        CK(c, cudaMemcpyAsync(drows, rows.data(), len * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        CK(c, cudaMemcpyAsync(drow, shot_row.data(), shot_row.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
        CK(c, cudaMemcpyAsync(didx, shot_idx.data(), shot_idx.size() * sizeof(uint64_t), cudaMemcpyHostToDevice, c->stream));
        launch_sample_lo(drows, nb, cl, drow, didx, shot_idx.size(), dbhi, dres, dout, c->stream);
        LAUNCHED(c);
        { qsim_status _s = sync_stream(c); if (_s != QSIM_OK) return _s; }
        i0 = i;
    }
    CK(c, cudaMemcpyAsync(out, dout, n_shots * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
    { qsim_status _s = sync_stream(c); if (_s != QSIM_OK) return _s; }
    return QSIM_OK;
}

qsim_status qsim_measure(qsim_ctx c, const int *qubits, int k, uint64_t seed, uint64_t n_shots, uint64_t *out)
{
    GUARD(c);
    if (n_shots && !out) return QSIM_ERR_ARG;
    if (k > 24) {
        if (k > 40 || k > c->n || !qubits) FAIL(c, QSIM_ERR_ARG, "measure: k=%d (at most min(n, 40) listed qubits)", k);
        return measure_two_level(c, qubits, k, seed, n_shots, out);
    }
    const size_t B = (size_t)1 << (k < 0 ? 0 : k);
    std::vector<double> p(B);
    qsim_status s = probabilities_impl(c, qubits, k, p.data());
    if (s != QSIM_OK) return s;
    const size_t need = 2 * B + n_shots + 1;  // p, CDF (doubles) + outcomes (uint64)
    if ((s = ensure_dev(c, c->d_red, c->d_red_cap, need)) != QSIM_OK) return s;
    double *dp = c->d_red, *dc = c->d_red + B;
    uint64_t *dout = (uint64_t *)(c->d_red + 2 * B);
    CK(c, cudaMemcpyAsync(dp, p.data(), B * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    launch_sample(dp, k, seed, n_shots, dc, dout, c->stream);
    LAUNCHED(c);
    if (n_shots) CK(c, cudaMemcpyAsync(out, dout, n_shots * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
    { qsim_status _s = sync_stream(c); if (_s != QSIM_OK) return _s; }
    return QSIM_OK;
}

qsim_status qsim_get_amplitudes(qsim_ctx c, uint64_t first, uint64_t count, qsim_c128 *host_out)
{
    GUARD(c);
    if (count && !host_out) return QSIM_ERR_ARG;
    if (c->n < 64 && (first > (1ULL << c->n) || count > (1ULL << c->n) - first)) FAIL(c, QSIM_ERR_ARG, "range outside [0,2^n)");
    if (!c->initialized && !c->init_pending) FAIL(c, QSIM_ERR_STATE, "readout before qsim_init_basis");
    qsim_status s = flush(c);
    if (s != QSIM_OK) return s;
    // SPMD: every rank gathers the amplitudes it owns (zeros elsewhere), the
    // pieces are all-gathered and summed in rank order (exactly one rank holds
    // each index, so the sum is a selection)
    const int S = spmd(c) ? c->P : 1;
    const uint64_t piece = std::max<uint64_t>(1, (1ULL << 22) / S);
    if ((s = ensure_dev(c, c->d_red, c->d_red_cap, 2 * piece * (S > 1 ? S + 1 : 1))) != QSIM_OK) return s;
    const int virt = c->transport == QSIM_TRANSPORT_VIRTUAL;
    for (uint64_t off = 0; off < count; off += piece) {
        const uint64_t cnt = std::min(piece, count - off);
        double2 *dout = (double2 *)c->d_red;
        launch_gather(dout, first + off, cnt, c->d_shard_ptrs, virt, c->rank, c->M, c->n, c->planner->phys_of.data(),
                      c->stream);
        LAUNCHED(c);
        if (S > 1) {
            double *all = c->d_red + 2 * piece;
            CKC(c, all_gather((const double *)dout, all, 2 * cnt, c->stream, _err));
            launch_sum_ranks(all, (double *)dout, 2 * cnt, S, c->stream);
            LAUNCHED(c);
        }
        CK(c, cudaMemcpyAsync(host_out + off, dout, cnt * sizeof(double2), cudaMemcpyDeviceToHost, c->stream));
        { qsim_status _s = sync_stream(c); if (_s != QSIM_OK) return _s; }
    }
    return QSIM_OK;
}

qsim_status qsim_set_option(qsim_ctx c, const char *key, int64_t value)
{
    GUARD(c);
    if (!key) return QSIM_ERR_ARG;
    std::string k(key);
    if (k == "fusion") { c->fusion = value != 0; c->pc.valid = false; }
    else if (k == "block_fusion") { c->block_fusion = value != 0; c->pc.valid = false; }
    else if (k == "low_remap") { c->low_remap = value != 0; c->pc.valid = false; }
    else if (k == "remap_lookahead") { c->remap_lookahead = (int)std::max<int64_t>(0, std::min<int64_t>(value, 24)); c->pc.valid = false; }
    else if (k == "timing") c->timing = value != 0;
    else if (k == "max_scan") { c->max_scan = value < 1 ? 1 : (int)std::min<int64_t>(value, 1 << 30); c->pc.valid = false; }
    else if (k == "exchange_chunk_mb") c->chunk_mb = value < 1 ? 1 : value;
    else if (k == "sample_batch") c->sample_batch = std::max<int64_t>(value, 0);
    else if (k == "peak_link_gbs") c->peak_link_gbs = (double)std::max<int64_t>(value, 0);
    else if (k == "overlap") c->overlap = (int)std::min<int64_t>(std::max<int64_t>(value, 0), 2);
    else if (k == "comm_timeout_ms") {
        c->comm_timeout_ms = value < 1 ? 1.0 : (double)value;
        if (c->comm) c->comm->timeout_ms = c->comm_timeout_ms;
    }
    else if (k == "pass_variant") c->pass_variant = value == 1 ? 1 : 2;
    else if (k == "fuse_readout") c->fuse_readout = value ? 1 : 0;
    else if (k == "desync_ns") c->desync_ns = (int)std::min<int64_t>(std::max<int64_t>(value, 0), 1000000);
    else if (k == "jit") { c->jit = value != 0; c->pc.valid = false; }
    else if (k == "plan_cache") { c->plan_cache = value != 0; c->pc.valid = false; }
    else if (k == "global_policy") {
        if (value < 0 || value > 2) FAIL(c, QSIM_ERR_ARG, "global_policy must be 0 (remap), 1 (pairwise) or 2 (auto)");
        c->global_policy = (int)value;
        c->pc.valid = false;
    }
    else FAIL(c, QSIM_ERR_ARG, "unknown option '%s'", key);
    return QSIM_OK;
}

qsim_status qsim_get_stats(qsim_ctx c, qsim_stats *out)
{
    GUARD(c);
    if (!out) return QSIM_ERR_ARG;
    qsim_status s = collect_timing(c);
    if (s != QSIM_OK) return s;
    *out = c->stats;
    out->jit_kernels = jit_cache().size();
    out->jit_compile_ms = jit_cache().compile_ms;
    out->link_gbs = c->plan_link_gbs;
    return QSIM_OK;
}

qsim_status qsim_reset_stats(qsim_ctx c)
{
    GUARD(c);
    qsim_status s = collect_timing(c);
    if (s != QSIM_OK) return s;
    std::memset(&c->stats, 0, sizeof(c->stats));
    return QSIM_OK;
}

qsim_status qsim_probe_peaks(double *fp64_tflops, double *copy_gbs)
{
    if (!fp64_tflops && !copy_gbs) return QSIM_ERR_ARG;
    double f = 0, b = 0;
    if (qsb::probe_peaks(fp64_tflops ? &f : nullptr, copy_gbs ? &b : nullptr, 5) != 0) return QSIM_ERR_CUDA;
    if (fp64_tflops) *fp64_tflops = f / 1e12;
    if (copy_gbs) *copy_gbs = b / 1e9;
    return QSIM_OK;
}

qsim_status qsim_exchange_peers(int n_qubits, int n_ranks, int rank, const int *gpos, int K, int *peers, int *self_v)
{
    if (n_ranks < 1 || (n_ranks & (n_ranks - 1)) || rank < 0 || rank >= n_ranks || K < 0 || K > 6 ||
        (K && (!gpos || !peers)) || !self_v)
        return QSIM_ERR_ARG;
    const int M = n_qubits - ilog2(n_ranks);
    std::vector<int> g(gpos, gpos + K);
    for (int i = 0; i < K; i++)
        if (g[i] < M || g[i] >= n_qubits) return QSIM_ERR_QUBIT_RANGE;
    *self_v = (int)rank_sub((uint64_t)rank, g, M);
    for (uint64_t v = 0; v < (1ULL << K); v++) peers[v] = (int)with_sub((uint64_t)rank, g, M, v);
    return QSIM_OK;
}

qsim_status qsim_plan_json(int n_qubits, int n_ranks, const qsim_gate *gates, size_t n_gates, int fusion, char *buf,
                           size_t buf_bytes)
{
    if (n_qubits < 1 || n_qubits > 62 || n_ranks < 1 || (n_ranks & (n_ranks - 1)) || !buf) return QSIM_ERR_ARG;
    const int G = ilog2(n_ranks);
    if (n_qubits - G < 1) return QSIM_ERR_ARG;
    std::vector<GateRec> recs(n_gates);
    for (size_t i = 0; i < n_gates; i++) {
        qsim_status s = to_rec(nullptr, n_qubits, gates[i], recs[i]);
        if (s != QSIM_OK) return s;
        recs[i].id = (int)i;
    }
    Planner P(n_qubits, G);
    P.choose_initial_layout(recs);
    std::string init = "{\"initial_phys_of\":[";
    for (int q = 0; q < n_qubits; q++) init += (q ? "," : "") + std::to_string(P.phys_of[q]);
    init += "],\"plan\":";
    std::vector<Step> steps;
    PlanOptions opt;
    opt.fusion = (fusion & 3) != 0;
    opt.block_fusion = !(fusion & 0x100);
    opt.low_remap = !(fusion & 0x200);
    if ((fusion >> 12) & 31) opt.remap_lookahead = ((fusion >> 12) & 31) - 1;
    opt.global_policy = (fusion >> 4) & 3 ? ((fusion >> 4) & 3) - 1 : GP_AUTO;
    if ((fusion >> 17) & 7) opt.force_list = ((fusion >> 17) & 7) - 1;
    opt.overlap = (fusion >> 20) & 1;
    std::vector<std::string> cands;
    opt.cand_report = &cands;
    const auto tp0 = std::chrono::steady_clock::now();
    P.plan(recs, opt, steps);
    const double plan_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tp0).count();
    std::string jit_info;
    if ((fusion & 3) == 2 || (fusion & 0x400)) {  // NVRTC-compile (2) or only generate + key-check (bit 10) the pass kernels
        std::vector<const Step *> ps;
        for (const Step &s : steps)
            if (s.type == ST_PASS) ps.push_back(&s);
        std::vector<Step> rvs;  // readout variants (bit 21)
        if ((fusion >> 21) & 1) {
            rvs.reserve(ps.size());
            for (const Step *s : ps) {
                rvs.push_back(*s);
                rvs.back().jit_readout = 1;
            }
            for (const Step &s : rvs) ps.push_back(&s);
        }
        std::string err;
        int nk = 0;
        double ms = 0;
        std::vector<double> fpa;
        bool ok = jit_compile_only(ps, err, nk, ms, (fusion & 3) == 2, &fpa);
        std::string fps;
        for (size_t i = 0; i < fpa.size(); i++) fps += (i ? "," : "") + std::to_string(fpa[i]);
        std::string e;
        for (char ch : err) e += (ch == '"' || ch == '\\') ? ' ' : (ch == '\n' ? ' ' : ch);
        jit_info = ",\"jit\":{\"ok\":" + std::string(ok ? "true" : "false") + ",\"kernels\":" + std::to_string(nk) +
                   ",\"compile_ms\":" + std::to_string(ms) + ",\"fp64_per_amp\":[" + fps + "],\"error\":\"" + e + "\"}";
    }
    std::string cj;
    for (size_t i = 0; i < cands.size(); i++) cj += (i ? "," : "") + cands[i];
    std::string js = init + plan_to_json(P, steps) + jit_info + ",\"plan_ms\":" + std::to_string(plan_ms) +
                     ",\"candidates\":[" + cj + "]}";
    if (js.size() + 1 > buf_bytes) return QSIM_ERR_ARG;
    std::memcpy(buf, js.c_str(), js.size() + 1);
    return QSIM_OK;
}

}  // extern "C"
