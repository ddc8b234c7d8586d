// fused_types.h -- plain data shared by the host planner, the AOT fused
// kernel and the NVRTC-compiled (JIT) fused kernels.  Must compile as host
// C++, CUDA C++ and NVRTC (no standard headers under NVRTC).
#pragma once
#ifdef __CUDACC_RTC__
typedef unsigned char uint8_t;
typedef unsigned short uint16_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
#else
#include <cstdint>
#endif

namespace qc {

constexpr int kSlotBits = 4;          // 16 amplitudes per thread task
constexpr int kSlots = 1 << kSlotBits;
#ifndef QC_COMPUTE_WARPS
#define QC_COMPUTE_WARPS 8
#endif
constexpr int kComputeWarps = QC_COMPUTE_WARPS;  // fused kernel: compute warps ...
constexpr int kComputeThreads = kComputeWarps * 32;
constexpr int kFusedThreads = kComputeThreads + 32;  // ... + 1 TMA producer warp
// Compute warps form kGroups groups that take alternate tiles.  With NBUF not
// a multiple of kGroups a buffer's consecutive tiles go to different groups,
// and a group running ahead could wait for phase p+1 of a buffer whose phase
// p is still pending -- a parity wait would then match phase p-1.  The
// producer therefore publishes a per-buffer tile tag, and consumers wait for
// their tile's tag before the parity wait (qc_fused_pipeline).
#ifndef QC_GROUPS
#define QC_GROUPS 2
#endif
constexpr int kGroups = QC_GROUPS;    // compute warps form groups working on alternate tiles
constexpr int kGroupThreads = kComputeThreads / kGroups;
constexpr int kWSlots = 4;            // phase-run factor sets: tile index mod 4
constexpr int kPadBytes = 16;         // smem padding per row (bank-conflict relief)
constexpr int kMaxPrun = 64;          // phase runs with a per-tile factor, per pass

// Fused op kinds, bit sources and exact matrix patterns.
// F_MK: dense 2^k x 2^k (k = 3, 4) on k slot bits in canonical order; sb1 = k,
// sb0 = the slot bit NOT in the op when k = 3.
enum FKind : uint8_t { F_M1 = 0, F_M2 = 1, F_DSCALE = 2, F_PRUN = 3, F_MK = 4 };
enum FSrc : uint8_t { S_SLOT = 0, S_LOCAL = 1, S_OUTER = 2, S_NONE = 3 };
enum FPat : uint8_t { P_DENSE = 0, P_DIAG = 1, P_ANTI = 2, P_MOVE = 3, P_PAIRS1 = 4, P_PAIRS2 = 5,
                      P_PAIRS3 = 6 };

struct alignas(16) FHdr {
  uint8_t kind, sb0, sb1, dsrc;      // dsrc: DSCALE / PRUN base-bit source; M ops: FPat
  uint8_t dbit, smask, sval, flags;  // flags bit0: d0 is one (DSCALE) / any d0 != 1 (PRUN)
  uint8_t nz[4];                     // M2 P_MOVE: source column of each row
  uint8_t identmask;                 // M1/M2 DIAG/PAIRS: rows that are exactly identity rows
  uint8_t nt_local, nt_outer, nt_none;  // PRUN term counts (stored local, outer, none)
  uint16_t wslot, pad0;              // PRUN: per-tile factor slot
  uint32_t coef;                     // offset of coefficients (complex) / terms
  uint32_t lmask, lval;              // predicate on tile-local bits (per task)
  uint64_t omask, oval;              // predicate on physical outer bits (per tile)
};
static_assert(sizeof(FHdr) == 48, "FHdr layout");

template <typename T>
struct alignas(8) FTermT {
  uint8_t src, bit, val, d0one;
  uint32_t pad;
  T d0r, d0i, d1r, d1i;
};

struct SubStageDesc {
  int32_t op_begin, op_end;  // indices into the pass's header array
  int32_t g[kSlotBits];      // tile-local positions of slot bits 0..3 (ascending)
};

// Opaque 128-byte TMA tensor map (CUtensorMap), passed as a __grid_constant__.
struct alignas(64) QcTmap {
  uint64_t opaque[16];
};
// The tensor maps of one launch: m[0] for a tile in one buffer, m[h] for
// sub-tile h of a tile spanning shards (PassDesc::grp).
struct alignas(64) QcTmapSet {
  QcTmap m[8];
};

struct PassDesc {
  int32_t k, rb;          // tile bits, row bits (T contains physical 0..rb-1)
  int32_t pshift;         // smem: one 16-byte pad every 2^pshift amplitudes
  int32_t g4;             // tile transport: 0 one cp.async.bulk per row; 1 TMA tile::gather4 /
                          // scatter4 (4 rows per request); 2 one TMA box per tile (bx_*)
  int32_t n_hi;           // k - rb
  int32_t n_outer;
  int32_t hi_pos[16];     // physical bit of tile-local bit rb+j
  int32_t outer_pos[64];  // physical bit of outer bit j (tile index bit j)
  uint64_t n_tiles;
  uint64_t blob_off;      // byte offset of this pass's blob in the plan blob
  uint32_t blob_bytes;    // [subs][hdrs][coefs][terms], 16-byte aligned sections
  uint32_t n_sub, n_ops, n_prun;
  uint32_t off_hdr, off_coef, off_term;  // section offsets inside the pass blob
  uint32_t pad_;
  int32_t bx_dims;        // g4 == 2: dims of the pass's 5-D tensor map; dim d spans physical
  int32_t bx_start[6];    // bits [bx_start[d], bx_start[d+1]): its tile bits (the box) below,
                          // outer bits (the coordinate) above
  uint32_t bx_xmask;      // tile bits beyond the 5th run, relative to bx_start[4]: one box per
  int32_t bx_sub;         // combination of them; each box holds 2^bx_sub amplitudes
  uint64_t rank_bits;     // sharded state: this rank's global bits (rank << n_loc), OR-ed
                          // into every tile's base for predicates / diagonal bits only
  uint64_t addr_bits;     // OR-ed into amplitude addresses (loopback: shards share one buffer)
  // Tiles spanning shards (dist.cu: pair segments, QC_OPT_EXCHANGE 2, and
  // group plans, 3): the plan's index includes rank bits; a tile may hold j
  // of them (`grp`), always its top j local bits, and then its 2^j sub-tiles
  // (indexed by those bits' value h) live in 2^j ranks' buffers.
  uint64_t tile0;         // first tile index of this launch (n_tiles = tiles of this launch)
  uint64_t addr_strip;    // plan bits cleared from tile bases / row offsets before addressing
  int32_t grp;            // j (<= 3): sub-tile h moves via tmaps.m[h], sub_state[h], sub_addr[h]
  int32_t pad1_;
  uint64_t sub_addr[8];   // grp > 0: addr_bits of sub-tile h (OR-ed into its addresses)
  uint64_t sub_state[8];  // grp > 0: buffer of sub-tile h (per-row copy transport)
};

}  // namespace qc
