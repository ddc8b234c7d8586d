// qc_internal.h -- internal types of libqc (host planner <-> CUDA kernels).
//
// Vocabulary:
//   * physical bit p  : bit p of the amplitude index in device memory.  Logical
//     qubit q (Definition 1) lives at physical bit layout[q]; the
//     canonical layout is layout[q] = n-1-q.
//   * PGate           : one gate lowered to physical bits and a kernel class
//     (generic / diagonal / permutation, controls as a mask) -- SURVEY 8(b)
//     "op class drives kernel choice".
//   * tile            : 2^k amplitudes sharing the values of all bits outside
//     the tile bit set T; rows of 2^rb contiguous amplitudes (T includes
//     physical bits 0..rb-1) are moved HBM<->smem by TMA bulk copies.
//   * sub-stage       : a run of consecutive gates of one fused pass whose
//     non-diagonal targets lie in a 4-bit "slot group" G subset of T; each
//     thread task holds the 16 amplitudes that differ only in G in registers.
#pragma once
#include <complex>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/qc.h"

namespace qc {

using cd = std::complex<double>;

constexpr int kMaxQubits = 40;
constexpr int kSlotBits = 4;          // R: 16 amplitudes per thread task
constexpr int kSlots = 1 << kSlotBits;
constexpr int kComputeWarps = 8;      // fused kernel: 8 compute warps ...
constexpr int kComputeThreads = kComputeWarps * 32;
constexpr int kFusedThreads = kComputeThreads + 32;  // ... + 1 TMA producer warp
constexpr int kPadBytes = 16;         // smem padding per row (bank-conflict relief)

// ---------------------------------------------------------------- gates
enum class GK : int32_t { DENSE1 = 0, PERM1 = 1, DIAG1 = 2, DENSE2 = 3, SWAP2 = 4 };

struct PGate {
  GK kind;
  int t0 = -1, t1 = -1;      // physical target bits; DENSE2: t0 = MSB of the 4x4 index
  uint64_t cmask = 0, cval = 0;  // control bits (physical) and required values
  cd m[16];                   // DENSE1: 2x2 row-major; DIAG1: d0=m[0], d1=m[1]; DENSE2: 4x4
  bool d0_is_one = false;     // DIAG1 with d0 == 1 exactly: only the |1> half changes
  int src_op = -1;            // index in the caller's op list (diagnostics)
};

// ------------------------------------------------------- fused encoding
enum FKind : int32_t { F_DENSE1 = 0, F_PERM1 = 1, F_DIAG1 = 2, F_DENSE2 = 3, F_SWAP2 = 4 };
enum FDsrc : int32_t { D_SLOT = 0, D_LOCAL = 1, D_OUTER = 2 };

template <typename T>
struct alignas(16) FOpT {
  int32_t kind;           // FKind
  int32_t sb0, sb1;       // slot bits (0..3) of the targets; DENSE2: sb0 = MSB
  int32_t dsrc, dbit;     // DIAG1 index bit: slot bit / tile-local bit / physical outer bit
  int32_t d0_is_one;
  uint32_t smask, sval;   // control predicate on slot bits
  uint32_t lmask, lval;   // control predicate on tile-local (non-group) bits
  uint32_t pad0, pad1;
  uint64_t omask, oval;   // control predicate on physical outer bits (per tile)
  T m[32];                // complex entries, interleaved re,im
};

struct SubStageDesc {
  int32_t op_begin, op_end;
  int32_t g[kSlotBits];   // tile-local positions of slot bits 0..3 (ascending)
};

struct PassDesc {
  int32_t k, rb;          // tile bits, row bits (T contains physical 0..rb-1)
  int32_t n_hi;           // k - rb
  int32_t n_outer;
  int32_t hi_pos[16];     // physical bit of tile-local bit rb+j
  int32_t outer_pos[64];  // physical bit of outer bit j (tile index bit j)
  uint64_t n_tiles;
  int32_t sub_begin, sub_end;
};

struct FusedPassPlan {
  PassDesc desc;
  std::vector<int> gate_ids;  // gates (indices into the lowered list) in this pass
};

struct FusedPlan {
  bool ok = true;
  std::vector<FusedPassPlan> passes;
  std::vector<SubStageDesc> subs;
  std::vector<FOpT<double>> ops;  // converted to float for complex64 at upload
};

// Planner (plan.cpp).  k = tile bits (<= n), returns passes covering all gates.
FusedPlan plan_fused(int n, int k, int rb, const std::vector<PGate>& gates);

// ------------------------------------------------------- per-gate kernel args
template <typename T>
struct GateArgs {
  uint64_t count;         // work items
  int32_t nins;           // zero-bit insertions (ascending positions)
  int32_t ins[4];
  uint64_t setmask;       // OR'ed after insertion (control values)
  int32_t t0, t1;
  int32_t d0_is_one;
  int32_t pad;
  T m[32];
};

// Launchers (kernels_*.cu).  All enqueue on `stream`; return cudaError_t as int.
int launch_gate(void* state, int n, bool dbl, const PGate& g, void* stream);
int launch_fused_pass(void* state, bool dbl, const PassDesc& pd, const void* d_subs,
                      const void* d_ops, int ctas, void* stream);
size_t fused_smem_bytes(bool dbl, int k, int rb);
int fused_configure(bool dbl, size_t smem);  // opt-in to >48 KiB smem
int launch_init_random(void* state, int n, bool dbl, uint64_t seed, void* stream);
int launch_init_basis(void* state, int n, bool dbl, uint64_t k, void* stream);
// gather canonical [first, first+count) from a permuted layout into dst (device)
int launch_gather(const void* state, void* dst, int n, bool dbl, const int* layout,
                  uint64_t first, uint64_t count, bool scatter, void* stream);
int launch_norm2(const void* state, int n, bool dbl, double* d_partial, int nblocks,
                 void* stream);
int sm_count();

}  // namespace qc
