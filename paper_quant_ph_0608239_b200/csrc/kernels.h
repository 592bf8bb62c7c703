// kernels.h -- host launch wrappers of the sm_100a kernels (kernels.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "engine.h"

namespace qsb {

struct ProbsDesc {
    int32_t cb;          // chunk bits (min(12, M))
    int32_t M;
    int32_t k;           // listed qubits
    int32_t k_low;       // listed qubits with physical bit < cb
    int32_t n_free;      // chunk-index bits not fixed by listed qubits
    int32_t rank_glob_ok_mask_unused;
    uint64_t rank;       // this shard's rank
    uint32_t red_mask;   // chunk bits to reduce (unlisted, < cb)
    int32_t lowpos[12];  // physical positions of low listed qubits (partial bin bit j)
    int32_t pos[24];     // physical position of listed qubit j (any class)
    int32_t freepos[64]; // chunk-index bit positions that are free
};

// gops: the program in device memory (programs longer than kMaxPassOps), else nullptr
void launch_pass(const PassDesc &d, const KOp *ops /* host */, double2 *st, int variant, cudaStream_t s,
                 const KOp *gops = nullptr);
void launch_gate_generic(double2 *st, int M, uint64_t rank_bits, int t, uint64_t cm, uint64_t cv, int code,
                         const double *m, cudaStream_t s);
void launch_phase_generic(double2 *st, int M, uint64_t rank_bits, uint64_t cm, uint64_t cv, double fr, double fi,
                          cudaStream_t s);
void launch_perm(const PermDesc &d, double2 *st, const uint32_t *perm_tab, cudaStream_t s);
size_t perm_run_smem(const PermRunDesc &d);
void launch_perm_run(const PermRunDesc &d, double2 *st, const uint32_t *perm_tab, int n_sm, cudaStream_t s);
void launch_init(double2 *st, uint64_t n_amps, int64_t one_at, cudaStream_t s);
void launch_probs(const double2 *st, const ProbsDesc &d, double *partial, double *out, cudaStream_t s);
void launch_expect(const double2 *st, int M, double *partial, double *out /* M+1 */, cudaStream_t s);
struct ExpectMap {
    int n, M, S;          // logical qubits, local bits, shards (rank s = index s)
    int phys_of[64];      // logical qubit -> physical bit
};
// <Q_b> of a shard from the readout variant of its last pass (Step::
// jit_readout): partial[tile * (kTileBits + 1) + t] = sum of |a|^2 over the
// tile's amplitudes with tile bit t set (t < kTileBits), t = kTileBits the
// tile total.
struct FusedExpectDesc {
    int M;
    int tile_of[64];     // physical bit -> tile bit of the pass (-1: an instance bit)
    int inst_bit[64];    // physical bit -> bit of the tile (instance) index, for instance bits
    uint64_t n_inst;
};
// scratch: expect_fused_scratch(n_inst) doubles
size_t expect_fused_scratch(uint64_t n_inst);
void launch_expect_fused(const double *partial, const FusedExpectDesc &d, double *scratch, double *out /* M + 1 */,
                         cudaStream_t s);
void launch_expect_logical(const double *phys /* S x (M+1) */, const ExpectMap &m, double *out /* n */,
                           cudaStream_t s);
void launch_sample(const double *p, int k, uint64_t seed, uint64_t n_shots, double *cdf, uint64_t *out,
                   cudaStream_t s);
void launch_gather(double2 *out, uint64_t first, uint64_t count, double2 *const *shards_dev, int virt, int my_rank,
                   int M, int n, const int *phys_of, cudaStream_t s);
void launch_swap_blocks(double2 *A, double2 *B, int M, int K, const int *lpos, uint64_t cA, uint64_t cB,
                        cudaStream_t s);
void launch_pack(const double2 *shard, double2 *buf, int M, int K, const int *lpos, uint64_t c, uint64_t first,
                 uint64_t count, int unpack, cudaStream_t s);
void launch_pair_gate(double2 *A, double2 *B, int M, uint64_t mloc, uint64_t vloc, int xs, const double *m,
                      cudaStream_t s);
void launch_pair_combine(double2 *own, const double2 *other, uint64_t off, uint64_t count, uint64_t mloc,
                         uint64_t vloc, const double *c0, const double *c1, int self_first, cudaStream_t s);
void launch_sum_ranks(const double *all, double *out, uint64_t count, int S, cudaStream_t s);
// conditional marginals of the c low listed qubits inside bins of the kh high
// listed qubits (two-level sampling of k > 24 qubits); this shard's part
void launch_bin_marginal(const double2 *st, int M, uint64_t rank, int c, const int *pos_lo, int kh,
                         const int *pos_hi, int nu, const int *pos_un, const uint64_t *bins, uint64_t nb, double *out,
                         cudaStream_t s);
// level 1 of the two-level sampler: CDF of the high-qubit marginal (2^kh),
// per shot the high bin and the residual draw
void launch_sample_hi(const double *p, int kh, uint64_t seed, uint64_t n_shots, double *cdf, uint64_t *bhi,
                      double *res, cudaStream_t s);
// level 2: prefix sums of nrows bin rows (2^c each, in place), then per shot
// (shot_idx[t], its row shot_row[t]) the low bits; out[s] = lo | bhi[s] << c
void launch_sample_lo(double *rows, uint64_t nrows, int c, const uint32_t *shot_row, const uint64_t *shot_idx,
                      uint64_t n, const uint64_t *bhi, const double *res, uint64_t *out, cudaStream_t s);
int pass_regs_per_thread();
// measured FP64 FMA-pipe flop/s (DFMA probe) and streaming-copy bytes/s (read + write) of the current device
int probe_peaks(double *fp64_flops, double *copy_bytes_per_s, int reps);

}  // namespace qsb
