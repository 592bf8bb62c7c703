// engine.h -- structures shared by the host planner (plan.cpp) and the
// sm_100a kernels (kernels.cu).  No CUDA types here so the planner builds
// with a plain C++ compiler.
//
// Fused tile pass.  A pass loads a tile of 2^12 amplitudes
// spanned by 12 physical index bits -- tile-local bits 0,1,2 are physical
// bits 0,1,2 (so every warp access is made of whole 128-B lines), bits 3..11
// are 9 free local bits -- applies a list of gates to it, and stores it back:
// one HBM read + write (32 B/amplitude) for many gates.
//
// A "config" assigns the 12 tile-local bits to thread coordinates:
//   i    (kRegBits bits, in-thread register index) <-> r[0..kRegBits-1]
//   lane (5 bits)                                  <-> l[0..4]
//   warp (the rest)                                <-> w[0..kWarpBits-1]
// (kRegBits = 4: 16 amplitudes per thread, 256 threads per 12-bit tile;
//  kRegBits = 5: 32 amplitudes per thread, 128 threads.)
// Gates are applied to register bits only (k = position in r); OPC_TRANS
// moves the tile to another config through XOR-swizzled shared memory.
// Load/store configs have r[0] = 0, l[0] = 1, l[1] = 2 (256-bit accesses of
// amplitude pairs, whole 128-B lines per 4 lanes).
// A config is packed in nibbles: r0 .. r(kRegBits-1) l0 .. l4 w0 .. w(kWarpBits-1).
#pragma once
#include <cstddef>
#include <cstdint>

namespace qsb {

#ifndef QSB_TILE_BITS
#define QSB_TILE_BITS 12
#endif
#ifndef QSB_REG_BITS
#define QSB_REG_BITS 4
#endif
constexpr int kTileBits = QSB_TILE_BITS;      // tile = 3 fixed low bits + 9 free bits
constexpr int kTileAmps = 1 << kTileBits;
constexpr int kRegBits = QSB_REG_BITS;        // in-thread register bits
constexpr int kAmpsPerThread = 1 << kRegBits;
constexpr int kWarpBits = kTileBits - kRegBits - 5;  // register bits + 5 lane bits + warp bits
constexpr int kPassThreads = 32 << kWarpBits;
constexpr int kLaneNib = kRegBits, kWarpNib = kRegBits + 5;  // nibble offsets in a packed config
// fused-pass CTAs per SM the register file holds (<= 128 registers per thread
// for 16 amplitudes, <= 168 for 32)
constexpr int kPassMinBlocks = kRegBits == 4 ? 8192 / kTileAmps : 3;
constexpr int kPermTileBits = 12;
constexpr int kPhaseRunMin = 4;             // k_perm tile (targets + low bits)
constexpr int kPermTileAmps = 1 << kPermTileBits;
// ops of one pass travel in the interpreter's kernel parameter block (<= 32 KB
// on sm_100) up to kMaxPassOps; longer programs are read from global memory.
constexpr int kMaxPassOps = 240;
// planner limits per pass: gates (ops before re-layouts) and an estimate of the
// JIT tier's parameter bytes (matrices, phase angles, out-of-tile predicates)
constexpr int kMaxPassPops = 480;
constexpr int kPassParamBudget = 28 * 1024;

enum OpCode : int32_t {
    OPC_U2 = 0,     // general complex 2x2 on register bit k
    OPC_U2R = 1,    // real 2x2 (imaginary parts zero), e.g. Hadamard
    OPC_XS = 2,     // exact [[0,1],[1,0]]: conditional swap (CNOT/Toffoli target)
    OPC_PHASE = 3,  // multiply by f = m[0] + i m[1] where the predicate holds
    OPC_TRANS = 4,  // re-layout the tile to config `cfg` through shared memory
    // A run of >= kPhaseRunMin consecutive phases: OPC_PHASE_ACC ops add their
    // angle (cfg = round(phi / 2pi * 2^64), exact mod 2pi) to per-register
    // integer accumulators; OPC_PHASE_FLUSH multiplies each amplitude once by
    // e^{i theta} (JIT tier).  The interpreter applies OPC_PHASE_ACC like
    // OPC_PHASE (same m[0], m[1]) and ignores OPC_PHASE_FLUSH.
    OPC_PHASE_ACC = 5,
    OPC_PHASE_FLUSH = 6,
    // Fused two-qubit block (plan.cpp fuse_blocks): a general complex 4x4 on
    // register bits k < k2 (k2 in `cfg`), 4x4 index j = bit_k + 2 bit_k2.
    // m[] holds row 0; the next three ops (OPC_DATA) hold rows 1..3.  Never
    // predicated.  16 FMA-pipe ops per amplitude, replacing >= 3 gates that
    // would cost more (a brickwork U2 (x) U2, CNOT, U2 (x) U2 block: 32).
    OPC_U4 = 7,
    OPC_DATA = 8
};

enum Role : int32_t { ROLE_REG = 0, ROLE_LANE = 1, ROLE_WARP = 2, ROLE_OUT = 3 };

// One kernel op (128 B).  Predicate: (i & mreg) == vreg && (lane & mlane) == vlane
// && (warp & mwarp) == vwarp && (full_index & mout) == vout, where full_index =
// (rank << M) | local index, restricted to bits outside the tile.
struct alignas(16) KOp {
    int32_t code;
    int32_t k;  // register bit (0..kRegBits-1) of the target
    uint32_t mreg, vreg;
    uint32_t mlane, vlane;
    uint32_t mwarp, vwarp;
    uint64_t mout, vout;
    uint64_t cfg;  // OPC_TRANS: the new config; OPC_PHASE_ACC: angle; OPC_U4: k2
    uint64_t pad;
    double m[8];  // u00r u00i u01r u01i u10r u10i u11r u11i ; PHASE: f = (m[0], m[1])
};
static_assert(sizeof(KOp) == 128, "KOp layout");

struct PassDesc {
    uint64_t rank_bits;  // rank << M
    uint64_t n_inst;     // 2^(M-12) tile instances
    uint64_t cfg0;       // load config
    uint64_t init_phys;  // fresh: the physical index of the basis state qsim_init_basis set
    int32_t M;
    int32_t n_ops;
    int32_t use_smem;
    int32_t fresh;       // first data step after qsim_init_basis: synthesize the tile, no HBM read,
                         // and the zero-fill pass is skipped
    int32_t tp[kTileBits];           // physical position of tile-local bit t (load)
    int32_t tile_sorted[kTileBits];  // tp sorted ascending (instance deposit)
    int32_t tp_out[kTileBits];       // physical position tile-local bit t is stored at (a
                                     // permutation of tp: the next pass's low qubits)
};

#ifdef __CUDACC__
#define QSB_HD __host__ __device__ __forceinline__
#else
#define QSB_HD inline
#endif
QSB_HD int cfg_nib(uint64_t c, int j) { return (int)((c >> (4 * j)) & 15); }

// Controlled permutation of a target register (one launch per perm gate).
struct PermDesc {
    uint64_t rank_bits;
    uint64_t n_inst;
    uint64_t m_ctrl_out, v_ctrl_out;  // control predicate on bits outside the tile
    uint32_t m_ctrl_tile, v_ctrl_tile;  // control predicate on tile-local bits
    int32_t M;
    int32_t t;           // target bits = tile-local bits 0..t-1 (register order)
    int32_t tile_bits;   // total tile bits (t + extras)
    int32_t perm_offset; // into the device perm-table array (uint32 entries)
    int32_t contiguous;  // tile_pos[b] == b for all b (offset == tile index)
    int32_t tile_pos[kPermTileBits];    // physical position of tile-local bit b
    int32_t tile_sorted[kPermTileBits]; // same positions sorted ascending
};

// A run of controlled permutations of ONE target register (consecutive perm
// gates with identical targets, e.g. Shor's modular multiplications by
// y^(2^j) mod G) applied in one pass (k_perm_run): each element
// gathers through the inverse tables of the perms whose controls it satisfies.
constexpr int kMaxPermRun = 32;
// shared memory of one k_perm_run CTA: two staged tiles (16 B per element),
// one control mask per extra-bit pattern, R tables of 2^t uint16
constexpr size_t kPermRunSmemMax = 226 * 1024;  // 227 KB per block less room for the kernel's static smem
QSB_HD size_t perm_run_smem_bytes(int tile_bits, int t, int R, bool compose = false)
{
    // 2 tile buffers | in-tile control masks | R inverse tables [+ the slow-head
    // table + 2 composed tables] (uint16)
    return ((size_t)32 << tile_bits) + ((size_t)4 << (tile_bits - t)) + (size_t)(R + (compose ? 3 : 0)) * ((size_t)2 << t);
}
struct PermRunDesc {
    uint64_t rank_bits;
    uint64_t n_inst;
    int32_t M;
    int32_t t;           // target bits = tile-local bits 0..t-1 (register order)
    int32_t tile_bits;
    int32_t R;           // perms in the run (<= kMaxPermRun)
    int32_t contiguous;
    int32_t tab_offset;  // first inverse table (R tables of 2^t uint32) in the perm-table array
    int32_t tile_pos[kPermTileBits];
    int32_t tile_sorted[kPermTileBits];
    uint32_t m_tile[kMaxPermRun], v_tile[kMaxPermRun];  // controls on tile-local bits
    uint64_t m_out[kMaxPermRun], v_out[kMaxPermRun];    // controls outside the tile (incl. rank bits)
    // Composition (k_perm_run): pre_mask = the perms at the head of the gather
    // chain (highest j first) with no in-tile control: for a tile their active
    // subset is CTA-uniform, so they are composed into one table per tile.
    // slow_mask (a head of pre_mask) = those whose controls change at most
    // every 2^b tiles of a CTA's contiguous instance range: composed once per
    // change into the slow table the per-tile composition starts from.
    // (pre_mask != 0: instances in one contiguous range per CTA; else grid-stride)
    uint32_t pre_mask, slow_mask;
    int32_t bulk;  // contiguous tiles staged by one bulk copy each (k_perm_run)
};

}  // namespace qsb
