// jit.h -- pass-specialised sm_100a kernels (the fast tier of k_pass).
//
// A fused pass's STRUCTURE (op codes, register bits, predicate masks, shared
// memory re-layouts) is generated into CUDA source from our own template and
// compiled with NVRTC for sm_100a; the per-pass DATA (matrices, phases,
// tile bit positions, out-of-tile predicates) travels in the kernel
// parameter block.  Structures repeat across passes/circuits, so compiled
// kernels are cached by structure (and on disk by source text).  General
// gates use the same expression sequence as the interpreter k_pass (bitwise-
// identical states); phase runs (exact integer angle accumulation per
// monomial, lazily flushed, CTA-uniform and per-thread terms summed once per
// tile / launch) and Hadamard-form gates (sum/difference, one scale at the
// store) round differently and agree to 1e-13.  A re-layout's barriers span
// only the warps that exchange data through it (a CTA half when the top warp
// slot keeps its tile bit, the warp alone when all warp slots do).
#pragma once
#include <cuda.h>

#include <cstdint>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "plan.h"

namespace qsb {

struct Drv {
    CUresult (*moduleLoadData)(CUmodule *, const void *);
    CUresult (*moduleGetFunction)(CUfunction *, CUmodule, const char *);
    CUresult (*funcSetAttribute)(CUfunction, CUfunction_attribute, int);
    CUresult (*launchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                             CUstream, void **, void **);
};
const Drv &drv();
// device table of e^{2 pi i k/256} used by the phase-run flush
const void *jit_phase_table();

struct JitPass {
    std::string src;     // generated source (cache key)
    size_t param_bytes;  // size of the parameter block
    int n_tslots = 0;    // per-thread phase slots the companion kernel qsim_pass_tab fills (0: none)
    double fp64_per_thread = 0;  // FP64-pipe instructions one thread executes per tile (expected value)
};

// Generate the specialised kernel source for a pass step.
JitPass jit_generate(const Step &st);
// Pack the parameter block of a pass for one shard.
void jit_pack_params(const Step &st, void *state, uint64_t rank_bits, std::vector<uint8_t> &buf);
// update the basis-state index a fresh pass (PassDesc::fresh) synthesises
void jit_set_init(std::vector<uint8_t> &buf, uint64_t init_phys);
// Block variant (Step::jit_block): restrict a launch to the tiles whose
// physical bits pos[0..K) equal those of fixbits (the instance index then
// enumerates the other non-tile bits; 2^(M - 12 - K) instances); K = 0
// undoes it.  false if K is too large.
bool jit_set_block(std::vector<uint8_t> &buf, const Step &st, const int *pos, int K, uint64_t fixbits);
// readout variant (Step::jit_readout): where the per-tile bit sums go
void jit_set_red(std::vector<uint8_t> &buf, double *red);
// first-wave phase offset of the slot-0 CTAs (see jit_generate), ns; 0 = off
void jit_set_desync(std::vector<uint8_t> &buf, uint32_t n_sm, uint32_t ns);
// device table (n_tslots x kPassThreads uint64) qsim_pass_tab writes and the pass reads
void jit_set_ttab(std::vector<uint8_t> &buf, void *ttab);

// NVRTC-compile the specialised kernels of `steps` without loading them
// (host-only check; n = distinct structures)
// compile=false: generate only.  Either way, fails on a jit_key collision
// (two different sources under one key, across all plans checked in this process).
// fp64_per_amp: FP64-pipe instructions per amplitude of each step's kernel.
bool jit_compile_only(const std::vector<const Step *> &steps, std::string &err, int &n, double &ms,
                      bool compile = true, std::vector<double> *fp64_per_amp = nullptr);

// Launch shape: one non-persistent CTA per 2^12-amplitude tile, loads to registers.
void jit_launch_dims(const Step &st, int n_sm, unsigned &grid, unsigned &block, unsigned &smem);

// structural key of a pass (what the generated source depends on)
std::string jit_key(const Step &st);

class JitCache {
public:
    // generate + compile every pass structure not yet cached (NVRTC in
    // parallel host threads); false + err on failure
    bool compile(const std::vector<const Step *> &steps, std::string &err);
    CUfunction find(const std::string &key);
    // the companion per-thread phase-table kernel of a pass (nullptr: none)
    CUfunction find_tab(const std::string &key, int &n_tslots);
    // FP64-pipe instructions per thread and tile of a cached kernel (-1: not cached)
    double fp64_per_thread(const std::string &key);
    size_t size();
    double compile_ms = 0;
    int compiled = 0;

private:
    std::mutex mu_;
    struct Fn {
        CUfunction pass = nullptr, tab = nullptr;
        int n_tslots = 0;
        double fp64 = 0;  // JitPass::fp64_per_thread
    };
    std::unordered_map<std::string, Fn> fns_;
    std::vector<CUmodule> mods_;
};

}  // namespace qsb
