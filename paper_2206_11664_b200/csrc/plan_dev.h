// Device-visible plan structures (POD). Shared by the host lowering
// (csrc/plan/lower.cpp), the compiled interpreter kernel (cuda/pass_kernel.cu)
// and the run-time specialised kernels (cuda/jit.cpp compiles them with
// NVRTC, which sees this header as an embedded string) -- so it includes
// nothing but <cstdint> outside NVRTC.
#pragma once

#ifdef __CUDACC_RTC__
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
typedef unsigned short uint16_t;
#else
#include <cstdint>
#endif

namespace sdb {

// ------------------------------------------------------- device-side plan
// A tile pass: persistent CTAs (two per SM) walk tiles of 2^k amplitudes
// whose index bits outside the pass's local set are fixed (the tile's
// "outer" bits). Each thread holds 2^R amplitudes in registers (a "register
// config": R local coordinates vary across a thread's registers, the other
// k-R across threads) and runs the pass's host-compiled micro-program:
//   LOAD  - read the tile from HBM straight into registers (config `arg`);
//   CFG   - shared-memory transpose into a new register config; an optional
//           affine GF(2) index map (pending CNOT runs) is applied on the
//           write side for free;
//   BFLY  - unnormalised Hadamard butterflies on register coordinates;
//   POINT - pointwise S/CZ quarter-turns and exp(-i dt Lambda) (PointDev);
//   STORE - write the registers back to HBM.
// One pass = one full-state HBM read + write. Loads/stores are coalesced
// when a config's threads cover local coordinates 0..2 in lanes 0..2 (8
// lanes x 16 B = one 128-byte line); the lowering arranges that for the
// LOAD and STORE configs.
//
// Shared-memory slot of local index l (16-byte amplitudes): swz(l) XORs the
// low 3 bits with bits 3-5, 6-8 and 9-11, so coordinate c lands in slot bit
// (c mod 3); lanes 0..2 of every config get coordinates with distinct
// residues, which makes each quarter-warp of a 128-bit access conflict-free.
// swz is GF(2)-linear, which the kernel and the lowering both exploit.

// kOpSwap: register slot (mask & 15) <-> lane bit (mask >> 4) by warp shuffles,
// then the op's config (like kOpCfg, without shared memory).
// Literal CZ-pair entries a specialised kernel carries per POINT (entries are
// grouped by outer bit, so a shard of <= 24 outer bits always fits).
constexpr int kMaxLitPairs = 24;

// kOpLaneBfly: Hadamard butterfly on the coordinate at lane bit `mask` (3 or 4)
// by warp shuffles, config unchanged (a lane swap plus a register butterfly
// for a coordinate no later stage of the pass needs in a register).
enum MicroKind : int { kOpLoad = 0, kOpCfg = 1, kOpBfly = 2, kOpPoint = 3, kOpStore = 4, kOpSwap = 5, kOpLaneBfly = 6 };

// Register coordinates per thread: R <= kMaxR (2^R amplitudes per thread).
// The interpreter kernel runs R = 4; specialised kernels may run R = 5
// (32 amplitudes per thread, half the threads, fewer transposes per pass).
constexpr int kMaxR = 5;

struct MicroOpDev {
    int kind;
    uint32_t mask;  // LOAD/CFG: register coordinates (R bits among k); BFLY: register slots (bits 0..R-1);
                    // POINT: bit 0 = apply the pass scale here (folded into the phase factor);
                    // STORE: bit 1 = apply the pass scale, bit 2 = block barrier first
                    // (in-place store through a CNOT map with no transpose since the load);
                    // SWAP: register slot (bits 0..3) | lane bit << 4; LANEBFLY: lane bit
    int perm;       // CFG: PermDev index applied on the write side, or -1
    int arg;        // LOAD/CFG: index of this config among the pass's configs; POINT: PointDev index
    uint32_t pad;   // POINT: bit s = QT(r_s) for the register combination s of the current config
    uint32_t pad2;
    uint64_t cidx;  // LOAD/CFG: local coordinate index of register coordinate j in byte j
    uint16_t swc[8];     // LOAD/CFG: swizzled slot offset of register coordinate j;
                         // POINT: compact angle-table index of register coordinate j
    uint16_t fo[3][8];   // POINT (factor mode): swizzled compact slot offset of register
                         // coordinate j in factor table f
    uint64_t c_off[6];   // LOAD/CFG: physical offsets of the register coordinates;
                         // STORE with a store permutation: sigma-mapped offsets
};
static_assert(sizeof(MicroOpDev) % 16 == 0, "micro-ops are staged as int4 words");

// Per-thread constant of one register config (host-computed): the local
// index of the thread's register-0 amplitude (low 16 bits) and its swizzled
// shared-memory slot (high 16 bits).
using CfgThreadDev = uint32_t;

// Affine map on local coordinates: l' = lo[l & 63] ^ hi[l >> 6] ^ b(h),
// b(h) = XOR of flip[j] over the outer control bits set in the tile index.
// lo/hi hold swizzled slots (the swizzle is GF(2)-linear, so it commutes
// with the XOR composition); flip[] holds swizzled slots too.
struct PermDev {
    uint16_t lo[64];
    uint16_t hi[64];
    int n_ctrl;
    int pad;
    int ctrl_phys[32];
    uint32_t flip[32];
};

// Pointwise factor on the full physical index i = outer(h) | local(l):
//   q(i)   = popc(i & s1) + 2 popc(i & s2) + 2 [QT(l) ^ parity(l & M(h)) ^ C(h)]   (mod 4)
//            s1/s2 split into local-coordinate masks (s1L, s2L) and outer
//            physical masks (s1H, s2H); QT: local-local CZ pairs as a
//            2^k-bit table; M(h): local ends of local-outer pairs whose outer
//            end is set; C(h): parity of outer-outer pairs
//   phi(i) = -dt * sum_t c_t (-1)^{popc(i & zmask_t)}
//   a     <- a * i^q * exp(i*phi)
// Direct mode (n_seg == 0, few terms): per amplitude, sum over the terms
// with the outer sign folded per tile. Table mode groups the terms by their
// local part u (compacted onto the table coordinates `table_mask`); per tile
// A[u] = sum c_t (-1)^{popc(h & zh_t)}, and a Walsh-Hadamard transform over
// the table_bits compact coordinates in shared memory gives phi/(-dt) for
// every amplitude of the tile (SURVEY section 7 "Diagonal").
struct PointDev {
    uint64_t s1H;
    uint64_t s2H;
    uint32_t s1L;
    uint32_t s2L;
    int n_lo;      // local-outer CZ pairs, packed (coord << 8) | phys
    int lo_off;
    int n_oo;      // outer-outer CZ pairs (2-bit physical masks)
    int oo_off;
    int qt_word;   // word offset of the 2^k-bit QT table inside the pass's staged QT region, -1 if none
    int n_terms;
    int term_off;  // into term_hmask / term_lmask / term_coeffs
    int n_seg;
    int seg_off;   // into SegDev
    uint32_t table_mask;  // full mode: local coordinates spanned by the angle table
    int table_bits;       // popcount(table_mask)
    // Factor mode (n_fac > 0): the terms' local parts split into n_fac
    // disjoint coordinate sets (no term spans two), so
    //   exp(-i dt theta(l)) = prod_f E_f[pext(l, fac_mask[f])]
    // with per-tile complex tables E_f of 2^fac_bits[f] entries (2^b sincos
    // per tile instead of one per amplitude).
    int n_fac;
    uint32_t fac_mask[3];
    int fac_bits[3];
    int fac_sbeg[3];  // factor f: its segments are [fac_sbeg, fac_send) relative to seg_off
    int fac_send[3];
    int fac_coff[3];  // complex table of factor f: double offset (even) in the table region
    int c0_seg;       // factor mode: segment of the tile-constant terms (u = 0), -1 if none (PlanDev::tile_phase)
};

struct SegDev {
    uint32_t u;  // compact table index of the terms' local part
    int begin;   // terms [begin, end) relative to PointDev::term_off
    int end;
    int fac;     // factor table the segment belongs to (factor mode)
};

struct PassDev {
    int k;        // local qubit count (tile = 2^k amplitudes)
    int n_outer;  // outer bit count (= n_local - k)
    int n_ops;
    int op_off;
    int lpos[16];  // physical bit position of local coordinate j
    int opos[64];  // physical bit position of outer coordinate j
    double scale;  // exact power of two (applied once, see MicroOpDev)
    int flags;     // kPassNeedsTable
    int table_point;  // PointDev whose angle table is built at tile start, -1 if none
    int n_cfg;        // register configs in the program
    int cfg_off;      // offset of config 0's per-thread table in PlanDev::cfg_tb
    int rbits;        // R: register coordinates per config
    int qt_off;       // first QT word of this pass in PlanDev::qt_words
    int n_qt_words;   // QT words staged into shared memory
    int tab_words;    // 8-byte words of the per-tile table region (even; 0 if none)
    int pat_shift;    // tile-index bits >= pat_shift select the table's sign pattern (rebuild on change)
    int blocked;      // 1: each CTA walks a contiguous block of tiles (table reuse), 0: grid-strided
    int tphase_off;   // >= 0: per-tile phase of the table point's tile-constant terms at PlanDev::tile_phase + off
    double table_scale;  // factor mode: exact scale folded into E_0 (1 if applied elsewhere)
    int store_perm;      // 1: store out of place through a local bit permutation sigma
    int st_lpos[16];     // sigma(lpos[j])
    int st_opos[64];     // sigma(opos[j])
    // Fused qubit-remap exchange (store_perm passes in front of an exchange):
    // with a destination table (kernel argument xdst) the store writes each
    // amplitude straight into the receiving rank's buffer over peer memory:
    // chunk c = sigma-index >> x_t0 goes to xdst[c] at its low bits | own << x_t0,
    // own = this rank's bits at the swapped global positions x_gpos.
    int x_bits;          // swapped bits g' (0: no exchange follows)
    int x_t0;            // n_local - g'
    int x_gpos[8];       // global (physical) bit of swap i
};
constexpr int kPassNeedsTable = 1;


struct PlanDev {
    const PassDev* passes;
    const MicroOpDev* ops;
    const PermDev* perms;
    const PointDev* points;
    const SegDev* segs;
    const uint32_t* lo_pairs;
    const uint64_t* oo_pairs;
    const uint64_t* qt_words;
    const CfgThreadDev* cfg_tb; // per-config per-thread bases (MicroOpDev::arg)
    const uint64_t* term_hmask; // outer (physical) part of each term's z-mask
    const uint32_t* term_lmask; // local-coordinate part (direct mode)
    const double* term_coeffs;  // c_t * dt_scale; the kernel multiplies by -dt
    const double2* tile_phase;  // per-tile exp(-i dt theta_0) of passes with tphase_off >= 0
};

}  // namespace sdb
