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
//   * sub-stage       : a run of consecutive ops of one fused pass whose
//     non-diagonal targets lie in a 4-bit "slot group" G subset of T; each
//     thread task holds the 16 amplitudes that differ only in G in registers.
#pragma once
#include <complex>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../../include/qc.h"
#include "fused_types.h"

namespace qc {

using cd = std::complex<double>;

constexpr int kMaxQubits = 40;
constexpr size_t kBlobMax = 40 * 1024;  // op blob of one pass (staged in smem)

// ---------------------------------------------------------------- gates
enum class GK : int32_t {
  DENSE1 = 0, PERM1 = 1, DIAG1 = 2, DENSE2 = 3, SWAP2 = 4,
  SPARSE2 = 5,  // 4x4, <= 2 non-zeros per row: out[r] = m[2r] x[col[2r]] + m[2r+1] x[col[2r+1]]
  PERM2 = 6,    // 4x4 permutation: out[r] = x[col[r]]
  DIAG2 = 7,    // diag(m[0..3])
  DENSEK = 8    // generic gate (qc_mgate): 2^nt x 2^nt dense on targets tk[0..nt) (tk[0] = MSB), nt = 3..4
};

struct PGate {
  GK kind = GK::DENSE1;
  int t0 = -1, t1 = -1;          // physical target bits; 2-bit kinds: index = 2*bit(t0)+bit(t1)
  uint64_t cmask = 0, cval = 0;  // control bits (physical) and required values
  cd m[16];                      // DENSE1: 2x2 row-major; DIAG1: d0=m[0], d1=m[1]; DENSE2: 4x4
  int8_t col[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  bool d0_is_one = false;        // DIAG1 with d0 == 1 exactly: only the |1> half changes
  int src_op = -1;
  int nt = 0;                    // DENSEK: target count and physical target bits (MSB first)
  int tk[4] = {-1, -1, -1, -1};
  std::shared_ptr<const std::vector<cd>> mk;  // DENSEK: row-major 2^nt x 2^nt
};

uint64_t pgate_targets(const PGate& g);         // physical target bits
void pgate_swap_bits(PGate& g, int a, int b);  // relabel physical bits a <-> b

bool pgate_is_two(const PGate& g);
uint64_t pgate_bits(const PGate& g);            // targets | controls
void pgate_dense4(const PGate& g, cd out[16]);  // 2-bit kinds as a dense 4x4

// Host block fusion (fuse.cpp): merge gates on <= 2 bits, classify exactly.
// local_mask: bits a merged block may act on (rank bits of a sharded state
// stay out of blocks; gates touching them pass through unchanged).
std::vector<PGate> fuse_blocks(const std::vector<PGate>& in, uint64_t local_mask);

// ------------------------------------------------------- fused encoding
// FHdr, FTermT, SubStageDesc, PassDesc, op kinds / patterns: fused_types.h

// Precision-independent IR of one fused op.
struct FOpIR {
  FHdr h{};
  std::vector<cd> coefs;     // M1/M2: non-zero entries, row-major; DSCALE: d0, d1
  struct Term { uint8_t src, bit, val; cd d0, d1; };
  std::vector<Term> terms;   // PRUN, ordered local, outer, none
  // PRUN: terms whose control is a slot bit (bit = slot index).  Their gates
  // also follow the run as ordinary ops marked `folded`: the interpreter runs
  // those, the JIT multiplies the slot terms into the run's per-slot factors.
  std::vector<Term> sterms;
  bool folded = false;
  cd dense[16];              // M1/M2: the exact matrix (row-major), for code generation
  std::vector<cd> mk;        // F_MK: 2^k x 2^k over the op's slot bits in canonical order
                             // (matrix index bit j = the j-th lowest of its slot bits)
};

struct FusedPassPlan {
  PassDesc desc;
  std::vector<SubStageDesc> subs;
  std::vector<FOpIR> ops;
};

struct FusedPlan {
  bool ok = true;
  std::vector<FusedPassPlan> passes;
  // remap: the data of physical bit p ends at physical bit perm[p]
  std::vector<int> perm;
  int64_t remap_swaps = 0;
  int64_t restore_passes = 0;  // swap-only passes that restore the input layout
};

// Planner (plan.cpp).  k = tile bits (<= n), returns passes covering all gates.
// remap: passes may end with swaps of row bits and tile bits (plan.perm).
// flops_budget > 0: a pass stops taking gates once their algorithmic flops per
// amplitude (gate_flops) would exceed it (the HBM/ALU ridge of a pass).
// seeds: tile-choice starting points (choose_tile): 0 the in-order greedy
// tile, 1 also the best window of consecutive bits, 2 every such window (each
// hill-climbed); -1: QC_PLAN_SEEDS (default 0).
FusedPlan plan_fused(int n, int k, int rb, const std::vector<PGate>& gates, bool remap = false,
                     double flops_budget = 0, int seeds = -1);
// Algorithmic flops per amplitude of the fused plan (ALU roofline numerator).
double plan_flops_per_amp(const FusedPlan& plan);
double pass_flops_per_amp(const FusedPassPlan& pp);
// Pack the plan into one device blob for precision T (fills desc.blob_*).
std::vector<uint8_t> pack_plan(FusedPlan& plan, bool dbl);

// ------------------------------------------------------- per-gate kernel args
template <typename T>
struct GateArgs {
  uint64_t count;         // work items
  int32_t nins;           // zero-bit insertions (ascending positions): targets + controls
  int32_t ins[QC_MGATE_MAX_QUBITS];
  uint64_t setmask;       // OR'ed after insertion (control values)
  int32_t t0, t1;
  int32_t d0_is_one;
  int32_t pad;
  T m[32];
};

// Per-gate kernel of a generic gate on k = 3..4 targets (qc_mgate): the
// matrix travels in the kernel's parameter space (__grid_constant__).
template <typename T>
struct GateArgsK {
  uint64_t count;         // groups of 2^k amplitudes
  int32_t nins;
  int32_t ins[QC_MGATE_MAX_QUBITS];
  uint64_t setmask;       // control values
  int32_t k;
  int32_t tpos[4];        // physical target bits, tpos[0] = matrix MSB
  T m[2 * 256];           // row-major 2^k x 2^k, interleaved re,im
};

// NVRTC-specialised fused passes (jit.cu).
struct JitKernel {
  void* f = nullptr;  // CUfunction
  size_t smem = 0;
  int nbuf = 3;
  int threads = kFusedThreads;  // compute warps * 32 + the TMA producer warp
};
bool jit_available(std::string* why);
bool jit_build(const FusedPlan& plan, bool dbl, std::vector<JitKernel>& out, std::string& err);
int jit_launch(const JitKernel& k, void* state, const PassDesc& pd, const QcTmapSet& tms, int ctas,
               void* stream);
bool jit_compile_only(const FusedPlan& plan, bool dbl, int& compiled, std::string& err);
std::string jit_source_for_test(const FusedPlan& plan, bool dbl, size_t pass);

// Launchers (kernels_*.cu).  All enqueue on `stream`; return cudaError_t as int.
int launch_gate(void* state, int n, bool dbl, const PGate& g, void* stream);
int launch_fused_pass(void* state, bool dbl, const PassDesc& pd, const void* d_blob, const QcTmapSet& tms,
                      int ctas, void* stream);
bool make_row_tmap(void* base, int n, int rb, bool dbl, QcTmap* out);
bool make_box_tmap(void* base, int nbits, bool dbl, uint64_t tile_bits_set, QcTmap* out, PassDesc* d);
int fused_configure(bool dbl);
int launch_init_random(void* state, int n, bool dbl, uint64_t seed, void* stream, uint64_t first = 0,
                       uint64_t count = 0);
int launch_swap_regions(void* a, void* b, uint64_t bytes, void* stream);
int launch_init_basis(void* state, int n, bool dbl, uint64_t k, void* stream);
// gather canonical [first, first+count) from a permuted layout into dst (device)
int launch_gather(const void* state, void* dst, int n, bool dbl, const int* layout,
                  uint64_t first, uint64_t count, bool scatter, void* stream);
int launch_norm2(const void* state, int n, bool dbl, double* d_partial, int nblocks,
                 void* stream);
int sm_count();
int fma_peak(bool dbl, double* tflops);  // measurement utility (qc_debug_fma_peak)

}  // namespace qc
