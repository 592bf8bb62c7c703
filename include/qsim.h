/*
 * qsim.h -- C-ABI of the B200-native state-vector gate engine
 * (arXiv quant-ph/0608239, De Raedt et al., "Massive Parallel Quantum
 * Computer Simulator").  Library: paper_quant_ph_0608239_b200/libqsim_b200.so
 *
 * Problem statement: the state of an L-qubit machine
 * is a vector of 2^L complex amplitudes a(x_{L-1}..x_0); qubit 0 is the
 * least-significant bit of the index.  Gates update it in place with the
 * rules of Eqs. NUM2-NUM8.  Amplitudes are complex128
 * ("8 bytes for a real number"), stored [re, im] interleaved.
 *
 * Conventions
 *   - controls fire on |1>;
 *   - a 2x2 matrix u[4] is row-major [u00, u01, u10, u11] and maps
 *     (a0, a1) -> (u00 a0 + u01 a1, u10 a0 + u11 a1) for every index pair
 *     differing only in the target bit (Eqs. NUM2-NUM5 generalised);
 *   - every host array passed in is copied before the call returns and is
 *     never retained (caller keeps ownership);
 *   - all functions return qsim_status; no exception crosses the ABI.  On
 *     an argument error the state is untouched.  After QSIM_ERR_CUDA or
 *     QSIM_ERR_COMM the context is poisoned: only qsim_destroy is valid.
 *   - gate calls ENQUEUE (so the planner can fuse); readout calls and
 *     qsim_sync flush the queue.  A context is used by one host thread.
 *
 * Distribution: with P = 2^G shards (GPUs or
 * virtual shards) each holds 2^M amplitudes, M = n - G.  Physical index
 * bits >= M select the shard ("nonlocal"/global qubits); the qubit
 * permutation sigma of P:553-568 maps logical qubits to physical bits and
 * is maintained by the library; readouts always use LOGICAL order.
 */
#ifndef QSIM_H
#define QSIM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct qsim_ctx_s *qsim_ctx;

/* layout-compatible with cuDoubleComplex / std::complex<double> */
typedef struct {
    double re, im;
} qsim_c128;

typedef enum {
    QSIM_OK = 0,
    QSIM_ERR_ARG = 1,              /* bad pointer / size / option */
    QSIM_ERR_QUBIT_RANGE = 2,      /* qubit index outside [0, n) */
    QSIM_ERR_DUP_QUBIT = 3,        /* a qubit repeated among controls/targets */
    QSIM_ERR_NOT_UNITARY = 4,      /* max |U^dag U - I| > 1e-12 */
    QSIM_ERR_NOT_PERMUTATION = 5,  /* perm is not a bijection of [0, 2^t) */
    QSIM_ERR_OOM = 6,              /* device allocation failed */
    QSIM_ERR_CUDA = 7,             /* CUDA runtime error (context poisoned) */
    QSIM_ERR_COMM = 8,             /* NCCL error (context poisoned) */
    QSIM_ERR_STATE = 9,            /* readout before qsim_init_basis */
    QSIM_ERR_UNSUPPORTED = 10      /* valid request outside implemented limits */
} qsim_status;

typedef enum { QSIM_G_1Q = 0, QSIM_G_CTRL = 1, QSIM_G_PERM = 2, QSIM_G_SWAP = 3 } qsim_gate_kind;

#define QSIM_MAX_CONTROLS 8
#define QSIM_MAX_PERM_TARGETS 12

/* One gate of a circuit (qsim_run_circuit).
 *   QSIM_G_1Q  : target, u
 *   QSIM_G_CTRL: controls[0..n_controls), target, u   (CNOT, CP, C-V, Toffoli)
 *   QSIM_G_PERM: controls[0..n_controls), targets[0..n_targets), perm
 *                (register bit b <-> targets[b]; perm has 2^n_targets entries)
 *   QSIM_G_SWAP: targets[0], targets[1] (a qubit SWAP: handled as a relabel
 *                of sigma, no data moves) */
typedef struct {
    int32_t kind;
    int32_t target;
    int32_t n_controls;
    int32_t n_targets;
    int32_t controls[QSIM_MAX_CONTROLS];
    int32_t targets[QSIM_MAX_PERM_TARGETS];
    qsim_c128 u[4];
    const uint32_t *perm;
} qsim_gate;

typedef enum {
    QSIM_TRANSPORT_LOCAL = 0,    /* one shard on the current device (P must be 1) */
    QSIM_TRANSPORT_VIRTUAL = 1,  /* P shards, all on the current device, exchanged by
                                    device copies: a test backend for the sharded path */
    QSIM_TRANSPORT_NCCL = 2,     /* one process per GPU, shard exchanges over NCCL */
    QSIM_TRANSPORT_LOOPBACK = 3  /* SPMD ranks as host threads of ONE process on ONE device:
                                    the NCCL transport's exchange / readout code with each
                                    send-recv pair a device copy (comm id from
                                    qsim_get_loopback_id); tests the SPMD path on one GPU */
} qsim_transport;

/* Creation parameters.  Device buffers and the stream may be supplied by the
 * caller (e.g. PyTorch allocations); NULL means "library allocates/creates".
 * Caller-supplied buffers must outlive the context.
 *   shards[r]   : device buffer of 2^M complex128 for shard r (VIRTUAL: r < P;
 *                 LOCAL/NCCL: only shards[0], this process's shard), 256-B aligned
 *   scratch     : device scratch of scratch_bytes (exchange staging, reductions);
 *                 qsim_scratch_bytes() returns the recommended size
 *   stream      : cudaStream_t to enqueue all work on
 *   nccl_id     : 128-byte ncclUniqueId from qsim_get_unique_id on rank 0,
 *                 broadcast to all ranks by the caller (NCCL transport), or
 *                 the id from qsim_get_loopback_id (LOOPBACK transport)
 * SPMD transports (NCCL, LOOPBACK): every rank makes the same sequence of
 * calls.  A rank that waits longer than the communication timeout (option
 * "comm_timeout_ms", env QSIM_COMM_TIMEOUT_S; default 600 s) for its peers
 * aborts the communicator and returns QSIM_ERR_COMM (context poisoned). */
typedef struct {
    int32_t n_qubits;   /* 1 <= n <= 62 */
    int32_t n_ranks;    /* P in {1,2,4,...,64}, power of two, n - log2 P >= 1 */
    int32_t rank;       /* this process's rank (NCCL), else 0 */
    int32_t transport;  /* qsim_transport */
    void *shards[64];
    void *scratch;
    size_t scratch_bytes;
    void *stream;
    uint8_t nccl_id[128];
} qsim_config;

/* Standalone single-GPU context on the current CUDA device; the library
 * cudaMallocs the 2^n state and creates its stream.  n_gpus must be 1
 * (multi-GPU contexts are created per rank with qsim_create_ext). */
qsim_status qsim_create(int n_qubits, int n_gpus, qsim_ctx *out);
/* General creation; see qsim_config. */
qsim_status qsim_create_ext(const qsim_config *cfg, qsim_ctx *out);
/* SPMD creation of rank `rank` of n_gpus (NCCL transport, one process per
 * GPU): the shorthand of qsim_create_ext for that case.
 * nccl_unique_id: the 128 bytes rank 0 drew with qsim_get_unique_id (every
 * rank passes the same bytes).  shard/scratch/cuda_stream may be NULL (the
 * library allocates/creates); caller-supplied ones must outlive the context
 * and shard_bytes must be 16 * 2^(n - log2 n_gpus).  n_gpus == 1 makes a
 * LOCAL context (nccl_unique_id ignored). */
qsim_status qsim_create_rank(int n_qubits, int n_gpus, int rank, const void *nccl_unique_id, void *shard,
                             size_t shard_bytes, void *scratch, size_t scratch_bytes, void *cuda_stream,
                             qsim_ctx *out);
/* Recommended scratch bytes for (n, P). */
size_t qsim_scratch_bytes(int n_qubits, int n_ranks);
/* ncclUniqueId (128 bytes) for rank 0 to broadcast. */
qsim_status qsim_get_unique_id(void *out128);
/* Id (128 bytes) of a new loopback group: every rank's qsim_config.nccl_id
 * carries it (QSIM_TRANSPORT_LOOPBACK). */
qsim_status qsim_get_loopback_id(void *out128);
qsim_status qsim_destroy(qsim_ctx ctx);

/* |index> (INITIAL STATE).  Lazy: the initial sigma is chosen by
 * look-ahead over the gates queued before the next flush.  index < 2^n. */
qsim_status qsim_init_basis(qsim_ctx ctx, uint64_t index);

/* Single-qubit gate on qubit q (Eqs. NUM2-NUM5; H, X, Y, R(phi)
 * and any unitary U).  u: host, row-major, copied.  Errors (state untouched):
 * QSIM_ERR_QUBIT_RANGE, QSIM_ERR_NOT_UNITARY (max |U^dag U - I| > 1e-12),
 * QSIM_ERR_ARG (NULL u).  Gates queued before any qsim_init_basis make the
 * next flush fail with QSIM_ERR_STATE. */
qsim_status qsim_apply_1q(qsim_ctx ctx, int q, const qsim_c128 u[4]);

/* Controlled gate: U on target where all n_controls control qubits are 1
 * (CNOT Eq. NUM6, controlled phase Eq. COMM5 P:285-295,
 * controlled-V Eq. NUM7, Toffoli Eq. NUM8).
 * n_controls <= QSIM_MAX_CONTROLS.  controls, u: host, copied.  Errors (state
 * untouched): QSIM_ERR_QUBIT_RANGE, QSIM_ERR_DUP_QUBIT (a qubit repeated among
 * controls and target), QSIM_ERR_NOT_UNITARY, QSIM_ERR_ARG. */
qsim_status qsim_apply_controlled(qsim_ctx ctx, const int *controls, int n_controls, int target,
                                  const qsim_c128 u[4]);

/* Controlled classical reversible map of a target register (the
 * "conditional operation" of Shor's step 2):
 * |c, w> -> |c, perm[w]> when all controls are 1.  Register bit b of w is
 * qubit targets[b]; n_targets <= QSIM_MAX_PERM_TARGETS; perm: host array of
 * 2^n_targets entries, copied.  Errors (state untouched): QSIM_ERR_NOT_PERMUTATION
 * (not a bijection of [0, 2^n_targets)), QSIM_ERR_QUBIT_RANGE,
 * QSIM_ERR_DUP_QUBIT, QSIM_ERR_ARG. */
qsim_status qsim_apply_perm(qsim_ctx ctx, const int *controls, int n_controls, const int *targets,
                            int n_targets, const uint32_t *perm);

/* Quantum SWAP of qubits a and b (relabel of sigma; no data movement). */
qsim_status qsim_apply_swap(qsim_ctx ctx, int a, int b);

/* The paper's "SWAP K l_1..l_K g_1..g_K" command (App. A
 * P:1244-1258): exchange data so that the K given qubits that are currently
 * nonlocal become local and the K given local qubits become nonlocal
 * (Eqs. onequbitchange, twoqubitchange0-5).  Optional: the planner inserts
 * such exchanges itself.  Flushes. */
qsim_status qsim_remap(qsim_ctx ctx, const int *local_qubits, const int *global_qubits, int K);

/* Enqueue a whole gate list (see qsim_gate). Validated entirely before any
 * gate is queued. */
qsim_status qsim_run_circuit(qsim_ctx ctx, const qsim_gate *gates, size_t n_gates);

/* Marginal probabilities over the k listed qubits (k <= 24):
 * out[beta] = sum_{x : x_{qubits[b]} = beta_b} |a(x)|^2, host array of 2^k
 * doubles.  k = 0 gives the norm (Eq. STAT1).  Deterministic
 * fixed-order summation.  Non-collapsing. */
qsim_status qsim_probabilities(qsim_ctx ctx, const int *qubits, int k, double *out);

/* <Q_i> = sum_k p_k k_i for every qubit i (Eq. Shor7); host
 * array of n doubles.  Non-collapsing. */
qsim_status qsim_expectations(qsim_ctx ctx, double *out);
/* The same, enqueued: returns once the reduction and the copy into `out`
 * are on the context's stream; `out` holds the result after qsim_sync (or
 * any later synchronising call).  With pinned (page-locked) `out` the host
 * can enqueue the next circuit while this one runs; with pageable memory
 * the copy, and so the call, waits for the device. */
qsim_status qsim_expectations_async(qsim_ctx ctx, double *out);

/* n_shots basis states of the listed qubits drawn with probability
 * |<x|Phi>|^2 by inverse CDF with the counter-based
 * SplitMix64 rule (reading R14): u_s = draw_s x total, outcome =
 * min{beta : C(beta) > u_s}, C the prefix sum over beta in increasing order
 * (beta bit b <-> qubits[b]).  Non-collapsing.  Host out[n_shots].
 * k <= 24: one level (the 2^k marginal, its CDF and a binary search per
 * shot on the device).  24 < k <= min(n, 40), up to the whole register:
 * two levels with the same outcome rule, C(beta) = C_hi(beta_hi - 1) +
 * C_lo(beta_lo): the marginal of the top kh = max(20, k - 16) listed qubits
 * picks the high bits and the residual draw, then the conditional marginal of
 * the low k - kh listed qubits inside the drawn high bins (device kernels;
 * sharded states sum every shard's part in rank order).  QSIM_ERR_ARG for
 * k > 40. */
qsim_status qsim_measure(qsim_ctx ctx, const int *qubits, int k, uint64_t seed, uint64_t n_shots,
                         uint64_t *out);

/* Copy `count` amplitudes starting at LOGICAL index `first` to host memory
 * (sigma undone).  For tests / small states. */
qsim_status qsim_get_amplitudes(qsim_ctx ctx, uint64_t first, uint64_t count, qsim_c128 *host_out);

/* Flush the queue and wait for the device. */
qsim_status qsim_sync(qsim_ctx ctx);

/* Current qubit -> physical-bit map (sigma^-1 of P:558); out[n]. Flushes. */
qsim_status qsim_get_layout(qsim_ctx ctx, int *phys_of_qubit);

/* Options (integers): "fusion" (1 = fused tile passes [default], 0 = one
 * generic kernel per gate), "block_fusion" (1 = inside a pass, gate clusters
 * on two tile qubits become one 4x4 unitary and one-qubit runs one 2x2
 * [default]; 0 = every gate applied as given), "timing" (1 = CUDA-event time
 * every launch), "max_scan" (planner look-ahead window), "exchange_chunk_mb"
 * (exchange piece cap; the pieces are double-buffered between the engine
 * stream and a transfer stream), "comm_timeout_ms", "jit", "plan_cache",
 * "pass_variant", "global_policy", "sample_batch" (two-level sampler: cap on
 * the high bins whose conditional marginals are built per batch; 0 = sized by
 * memory, <= 2^24 entries), "peak_link_gbs" (link GB/s per direction
 * for the sharded planner's device-time model; its FP64 and HBM rates are
 * measured once per process on the device, qsim_probe_peaks), "overlap" (a pass followed by an
 * exchange whose local bits are not tile bits of the pass runs block by block,
 * each block's transfer overlapping the next block's compute: 1 = on the
 * NCCL / loopback transports [default]; 2 = also on virtual shards, where the
 * transfer is device copy work on the same HBM; 0 = in sequence), "desync_ns"
 * (pass kernels: the first-wave CTAs of SM slot 0 finish this many ns late so
 * that the two CTAs an SM runs stay out of step -- one re-layouts through
 * shared memory while the other computes; default 1500, 0 = off),
 * "fuse_readout" (1 = qsim_expectations runs the last pass of its flush as a
 * readout variant that also sums |a|^2 per tile bit, so <Q_i> needs no second
 * read of the state [default]; 0 = separate reduction kernels). */
qsim_status qsim_set_option(qsim_ctx ctx, const char *key, int64_t value);

typedef struct {
    uint64_t gates;            /* user gates enqueued (N_O) */
    uint64_t flushes;
    uint64_t passes;           /* fused tile-pass launches */
    uint64_t generic_launches; /* one-gate kernels */
    uint64_t perm_launches;
    uint64_t exchanges;        /* K-swap remaps */
    uint64_t exchange_bytes;   /* bytes this rank sent */
    uint64_t kernel_launches;  /* all kernels of this library */
    uint64_t relabels;         /* SWAP gates absorbed into sigma */
    double pass_ms;            /* event time of fused passes (timing=1) */
    double generic_ms;
    double perm_ms;
    double exchange_ms;
    double reduce_ms;
    double plan_ms;            /* host planning time */
    uint64_t pass_amp_bytes;   /* algorithmic bytes of the timed passes (32 B/amp/pass) */
    uint64_t jit_launches;     /* passes run by a pass-specialised (NVRTC) kernel */
    uint64_t jit_kernels;      /* specialised kernels in the process cache */
    double jit_compile_ms;     /* total NVRTC + module-load time in this process */
    double pass_fp64_slots;    /* algorithmic FP64 FMA-pipe instructions of the timed passes (timing=1) */
    uint64_t plan_cache_hits;  /* flushes that reused a cached plan */
    uint64_t streamed_steps;   /* plan steps launched while the planner was still running */
    uint64_t overlapped;       /* pass + exchange pairs run overlapped (option "overlap"; counted in
                                  passes and exchanges too) */
    double overlap_ms;         /* event time of the overlapped pairs (timing=1; not in pass_ms/exchange_ms) */
    double link_gbs;           /* SPMD: partner-link rate per direction measured at creation, minimum over
                                  the ranks (the planner's link rate); 0 = not measured */
    uint64_t fused_readouts;   /* qsim_expectations calls served by the readout variant of the last pass
                                  (option "fuse_readout"): no separate read of the state */
} qsim_stats;

qsim_status qsim_get_stats(qsim_ctx ctx, qsim_stats *out);
qsim_status qsim_reset_stats(qsim_ctx ctx);

/* Roofline denominators measured on the current CUDA device (no context
 * needed; takes ~0.1 s): *fp64_tflops = FP64 FMA-pipe throughput of a DFMA
 * probe (8 independent chains per thread, 2 x 256-thread CTAs per SM, the
 * pass kernel's residency), in TFLOP/s (2 flop per FMA); *copy_gbs =
 * streaming copy of 1 GiB (read + write bytes) in GB/s.  Either pointer may
 * be NULL (that probe is skipped).  QSIM_ERR_CUDA if no device. */
qsim_status qsim_probe_peaks(double *fp64_tflops, double *copy_gbs);

const char *qsim_status_str(qsim_status s);
const char *qsim_last_error(qsim_ctx ctx);

/* Host-only planner introspection (no GPU needed): plan `gates` for an
 * n-qubit state over P shards (initial sigma by look-ahead) and write a JSON
 * description of the steps (passes, perms, exchanges, pairwise combines,
 * relabels) into buf.  flags: bits 0-1 = fusion (0 off, 1 on, 2 on + NVRTC-
 * compile the pass kernels as a host-only check); bits 4-5 = global policy
 * + 1 (0 = default auto); bit 8 = no block fusion; bit 9 = no low-qubit
 * remap; bit 10 = generate the pass kernels' sources and check that equal
 * kernel-cache keys mean equal sources (no compile; across every plan checked
 * in this process; reported under "jit"); bits 12-16 = remap look-ahead + 1
 * (0 = default 6); bits 17-19 = candidate gate list + 1 to plan alone
 * (0 = all, costed; each candidate's modelled time is reported under
 * "candidates"); bit 20 = cost the plan for a transport that overlaps a pass
 * with the exchange after it (the runtime's "overlap" on NCCL/loopback); bit 21
 * = with bits 0-1 = 2 or bit 10, also generate / compile every pass's readout
 * variant (option "fuse_readout").  Returns QSIM_ERR_ARG if buf is too small. */
qsim_status qsim_plan_json(int n_qubits, int n_ranks, const qsim_gate *gates, size_t n_gates,
                           int flags, char *buf, size_t buf_bytes);

/* Host-only exchange routing of a K-pair remap ("we first compute
 * the ranks of the other MPI processes with which the MPI process has to
 * communicate"): the remap swaps local bits l_i with nonlocal physical bits
 * gpos[i]; chunk v of `rank` (the amplitudes whose l-bits equal v) goes to
 * peers[v] (2^K entries), and *self_v is the chunk that stays.  Used by the
 * NCCL exchange and by the CPU (gloo) tests of the sharded path. */
qsim_status qsim_exchange_peers(int n_qubits, int n_ranks, int rank, const int *gpos, int K, int *peers,
                                int *self_v);

#ifdef __cplusplus
}
#endif
#endif /* QSIM_H */
