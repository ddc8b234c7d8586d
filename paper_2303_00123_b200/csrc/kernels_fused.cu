// kernels_fused.cu -- the AOT fused tile-pass kernel (north-star "gate-fusion
// pass"), interpreting the planner's op blob.
//
// One launch applies every op of a planner pass (plan.cpp) in ONE HBM round
// trip.  The pass fixes a set T of k physical bits (always including bits
// 0..rb-1, so each tile is 2^{k-rb} rows of 2^rb contiguous amplitudes).  A
// tile is the 2^k amplitudes sharing one value of the n-k outer bits; every
// op of the pass acts inside a tile because its non-diagonal targets are in
// T, while controls / diagonal bits outside T are per-tile constants.  That is
// the paper's per-gate loop (Alg. alg:1q / alg:ctrl-1q / alg:2q)
// regrouped: the 2^{n-1} pair updates of a gate are partitioned by tile, and
// consecutive gates are applied to a tile while it sits in shared memory.
//
// This kernel is generic: the pass's ops are decoded at run time from a blob
// staged in smem.  Repeated circuits are served by the NVRTC-specialised
// kernels of jit.cpp instead (same pipeline, ops compiled in), which avoid the
// decode and the register shuffling an interpreter pays.
#include <cuda.h>
#include <cuda_runtime.h>

#include <bit>
#include <cstdlib>
#include <cstring>

#include "fused_common.cuh"
#include "qc_internal.h"

namespace qc {
namespace {

template <typename T>
struct InterpBody {
  using C = typename CT<T>::type;
  const uint8_t* gblob;
  const PassDesc* pd;
  const SubStageDesc* subs;
  const FHdr* hdr;
  const C* coef;
  const FTermT<T>* term;
  C* W;  // [kWSlots][kMaxPrun][2] per-tile phase-run factors (tile index mod kWSlots)

  static __device__ __forceinline__ size_t smem_bytes(const PassDesc& p) {
    return (size_t)p.blob_bytes + (size_t)kWSlots * kMaxPrun * 2 * sizeof(C);
  }
  __device__ __forceinline__ void setup(unsigned char* extra, const PassDesc& p) {
    const uint4* src = reinterpret_cast<const uint4*>(gblob + p.blob_off);
    uint4* dst = reinterpret_cast<uint4*>(extra);
    for (uint32_t i = threadIdx.x; i < p.blob_bytes / 16; i += blockDim.x) dst[i] = src[i];
    subs = reinterpret_cast<const SubStageDesc*>(extra);
    hdr = reinterpret_cast<const FHdr*>(extra + p.off_hdr);
    coef = reinterpret_cast<const C*>(extra + p.off_coef);
    term = reinterpret_cast<const FTermT<T>*>(extra + p.off_term);
    W = reinterpret_cast<C*>(extra + p.blob_bytes);
    pd = &p;
  }

  __device__ __forceinline__ void prologue(uint64_t tbase, int par) {
    if (!pd->n_prun) return;
    // per-tile factors of the phase runs: terms on outer bits + unconditional
    for (uint32_t o = qc_gtid(); o < pd->n_ops; o += kGroupThreads) {
      const FHdr h = hdr[o];
      if (h.kind != F_PRUN) continue;
      C w0 = qc_one<C>(), w1 = qc_one<C>();
      const FTermT<T>* t = term + h.coef + h.nt_local;
      for (int x = 0; x < h.nt_outer + h.nt_none; ++x) {
        const FTermT<T> tt = t[x];
        if (x < h.nt_outer && (int)((tbase >> tt.bit) & 1ull) != tt.val) continue;
        C d1;
        d1.x = tt.d1r;
        d1.y = tt.d1i;
        w1 = qc_cmul(d1, w1);
        if (!tt.d0one) {
          C d0;
          d0.x = tt.d0r;
          d0.y = tt.d0i;
          w0 = qc_cmul(d0, w0);
        }
      }
      W[(par * kMaxPrun + h.wslot) * 2 + 0] = w0;
      W[(par * kMaxPrun + h.wslot) * 2 + 1] = w1;
    }
    qc_compute_bar();
  }

  __device__ __forceinline__ void apply(const FHdr& h, C (&v)[kSlots], uint32_t lb, uint64_t tbase,
                                        int par) {
    if ((tbase & h.omask) != h.oval) return;
    if ((lb & h.lmask) != h.lval) return;
    const C* cp = coef + h.coef;
    const uint32_t sm = h.smask, sv = h.sval;
    switch (h.kind) {
      case F_M1: {
#define QC_M1_CASE(B)                                              \
  case B:                                                          \
    switch (h.dsrc) {                                              \
      case P_DENSE: qc_m1_dense<B>(v, cp, sm, sv); break;          \
      case P_ANTI: qc_m1_anti<B>(v, cp, sm, sv); break;            \
      case P_MOVE: qc_m1_move<B>(v, sm, sv); break;                \
      default: qc_m1_diag<B>(v, cp, h.identmask, sm, sv); break;   \
    }                                                              \
    break;
        switch (h.sb0) {
          QC_M1_CASE(0)
          QC_M1_CASE(1)
          QC_M1_CASE(2)
          QC_M1_CASE(3)
        }
#undef QC_M1_CASE
        break;
      }
      case F_M2: {
        uint32_t cols;
        memcpy(&cols, h.nz, 4);
#define QC_M2_CASE(B0, B1)                                                        \
  case B0 * 4 + B1:                                                               \
    switch (h.dsrc) {                                                             \
      case P_PAIRS1: qc_m2_pairs<B0, B1, 1>(v, cp, h.identmask, sm, sv); break;   \
      case P_PAIRS2: qc_m2_pairs<B0, B1, 2>(v, cp, h.identmask, sm, sv); break;   \
      case P_PAIRS3: qc_m2_pairs<B0, B1, 3>(v, cp, h.identmask, sm, sv); break;   \
      case P_DIAG: qc_m2_diag<B0, B1>(v, cp, h.identmask, sm, sv); break;         \
      case P_MOVE: qc_m2_move<B0, B1>(v, cols, sm, sv); break;                    \
      default: qc_m2_dense<B0, B1>(v, cp, sm, sv); break;                         \
    }                                                                             \
    break;
        switch (h.sb0 * 4 + h.sb1) {
          QC_M2_CASE(0, 1)
          QC_M2_CASE(0, 2)
          QC_M2_CASE(0, 3)
          QC_M2_CASE(1, 0)
          QC_M2_CASE(1, 2)
          QC_M2_CASE(1, 3)
          QC_M2_CASE(2, 0)
          QC_M2_CASE(2, 1)
          QC_M2_CASE(2, 3)
          QC_M2_CASE(3, 0)
          QC_M2_CASE(3, 1)
          QC_M2_CASE(3, 2)
        }
#undef QC_M2_CASE
        break;
      }
      case F_MK: {
        const int miss = h.sb1 == 4 ? 4 : h.sb0;
        switch (miss) {
          case 0: qc_mk_dense<0>(v, cp, sm, sv); break;
          case 1: qc_mk_dense<1>(v, cp, sm, sv); break;
          case 2: qc_mk_dense<2>(v, cp, sm, sv); break;
          case 3: qc_mk_dense<3>(v, cp, sm, sv); break;
          default: qc_mk_dense<4>(v, cp, sm, sv); break;
        }
        break;
      }
      case F_DSCALE: {
        const int bit = (h.dsrc == S_LOCAL) ? (int)((lb >> h.dbit) & 1u) : (int)((tbase >> h.dbit) & 1ull);
        if (bit == 0 && (h.flags & 1)) break;
        qc_scale_slots(v, cp[bit], sm, sv);
        break;
      }
      default: {  // F_PRUN
        C w0 = W[(par * kMaxPrun + h.wslot) * 2 + 0];
        C w1 = W[(par * kMaxPrun + h.wslot) * 2 + 1];
        const FTermT<T>* t = term + h.coef;
        for (int x = 0; x < h.nt_local; ++x) {
          const FTermT<T> tt = t[x];
          if ((int)((lb >> tt.bit) & 1u) != tt.val) continue;
          C d1;
          d1.x = tt.d1r;
          d1.y = tt.d1i;
          w1 = qc_cmul(d1, w1);
          if (!tt.d0one) {
            C d0;
            d0.x = tt.d0r;
            d0.y = tt.d0i;
            w0 = qc_cmul(d0, w0);
          }
        }
        const bool any0 = h.flags & 1;
        if (h.dsrc == S_SLOT) {
          switch (h.sb0) {
            case 0: qc_prun_slot<0>(v, w0, w1, any0); break;
            case 1: qc_prun_slot<1>(v, w0, w1, any0); break;
            case 2: qc_prun_slot<2>(v, w0, w1, any0); break;
            default: qc_prun_slot<3>(v, w0, w1, any0); break;
          }
        } else {
          const int bit = (h.dsrc == S_LOCAL) ? (int)((lb >> h.dbit) & 1u) : (int)((tbase >> h.dbit) & 1ull);
          if (bit || any0) qc_scale_slots(v, bit ? w1 : w0, 0u, 0u);
        }
        break;
      }
    }
  }

  __device__ __forceinline__ void tile(C* buf, uint64_t tbase, int par) {
    const int ps = pd->pshift;
    const uint32_t PAD = kPadBytes / sizeof(C);
    const uint32_t ntasks = 1u << (pd->k - kSlotBits);
    for (uint32_t si = 0; si < pd->n_sub; ++si) {
      if (si != 0) qc_compute_bar();
      const SubStageDesc sd = subs[si];
      uint32_t poff[kSlots];
#pragma unroll
      for (int s = 0; s < kSlots; ++s) {
        uint32_t off = 0;
#pragma unroll
        for (int j = 0; j < kSlotBits; ++j)
          if (s & (1 << j)) off |= 1u << sd.g[j];
        poff[s] = off + (off >> ps) * PAD;
      }
      for (uint32_t task = qc_gtid(); task < ntasks; task += kGroupThreads) {
        uint32_t lb = task;
#pragma unroll
        for (int j = 0; j < kSlotBits; ++j) lb = qc_ins0(lb, sd.g[j]);
        const uint32_t pb = lb + (lb >> ps) * PAD;
        C v[kSlots];
#pragma unroll
        for (int s = 0; s < kSlots; ++s) v[s] = buf[pb + poff[s]];
        for (int oi = sd.op_begin; oi < sd.op_end; ++oi) {
          const FHdr h = hdr[oi];
          apply(h, v, lb, tbase, par);
        }
#pragma unroll
        for (int s = 0; s < kSlots; ++s) buf[pb + poff[s]] = v[s];
      }
    }
  }
};

template <typename T, int NBUF>
__global__ void __launch_bounds__(kFusedThreads, 1)
    fused_pass_kernel(typename CT<T>::type* __restrict__ state, const PassDesc pd,
                      const uint8_t* __restrict__ gblob, const __grid_constant__ QcTmapSet tmaps) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  InterpBody<T> body;
  body.gblob = gblob;
  qc_fused_pipeline<typename CT<T>::type, NBUF>(state, pd, &tmaps, smem_raw, body);
}

constexpr size_t kMaxSmem = 227 * 1024;

template <typename T>
size_t smem_for(const PassDesc& pd, int nbuf) {
  using C = typename CT<T>::type;
  return qc_pipeline_smem<C>(pd.k, pd.rb, pd.pshift, nbuf) + pd.blob_bytes + (size_t)kWSlots * kMaxPrun * 2 * sizeof(C);
}

template <typename T>
int pick_nbuf(const PassDesc& pd) {
  for (int nb = 4; nb >= kGroups; --nb)
    if (smem_for<T>(pd, nb) <= kMaxSmem) return nb;
  return 0;
}

template <typename T>
int configure_t() {
  cudaError_t e;
  e = cudaFuncSetAttribute(fused_pass_kernel<T, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)kMaxSmem);
  if (e != cudaSuccess) return (int)e;
  e = cudaFuncSetAttribute(fused_pass_kernel<T, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)kMaxSmem);
  if (e != cudaSuccess) return (int)e;
  e = cudaFuncSetAttribute(fused_pass_kernel<T, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)kMaxSmem);
  if (e != cudaSuccess) return (int)e;
  e = cudaFuncSetAttribute(fused_pass_kernel<T, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)kMaxSmem);
  return (int)e;
}

template <typename T>
int launch_t(void* state, const PassDesc& pd, const void* d_blob, const QcTmapSet& tms, int ctas,
             cudaStream_t st) {
  using C = typename CT<T>::type;
  const int nb = pick_nbuf<T>(pd);
  if (nb == 0) return (int)cudaErrorInvalidValue;
  const size_t smem = smem_for<T>(pd, nb);
  uint64_t grid = pd.n_tiles;
  if (grid > (uint64_t)ctas) grid = (uint64_t)ctas;
  C* s = reinterpret_cast<C*>(state);
  auto blob = reinterpret_cast<const uint8_t*>(d_blob);
  switch (nb) {
    case 4: fused_pass_kernel<T, 4><<<(unsigned)grid, kFusedThreads, smem, st>>>(s, pd, blob, tms); break;
    case 3: fused_pass_kernel<T, 3><<<(unsigned)grid, kFusedThreads, smem, st>>>(s, pd, blob, tms); break;
    case 2: fused_pass_kernel<T, 2><<<(unsigned)grid, kFusedThreads, smem, st>>>(s, pd, blob, tms); break;
    default: fused_pass_kernel<T, 1><<<(unsigned)grid, kFusedThreads, smem, st>>>(s, pd, blob, tms); break;
  }
  return (int)cudaGetLastError();
}

}  // namespace

int fused_configure(bool dbl) { return dbl ? configure_t<double>() : configure_t<float>(); }

int launch_fused_pass(void* state, bool dbl, const PassDesc& pd, const void* d_blob, const QcTmapSet& tms,
                      int ctas, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  return dbl ? launch_t<double>(state, pd, d_blob, tms, ctas, st)
             : launch_t<float>(state, pd, d_blob, tms, ctas, st);
}

namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encoder() {
  static EncodeFn enc = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      enc = reinterpret_cast<EncodeFn>(fn);
  }
  return enc;
}
}  // namespace

// L2 promotion of the box tensor maps (QC_TMAP_PROMO 0 none, 1 64 B, 2 128 B,
// 3 256 B = default; experiment knob).
CUtensorMapL2promotion box_promotion() {
  static const int v = getenv("QC_TMAP_PROMO") ? atoi(getenv("QC_TMAP_PROMO")) : 3;
  return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                : v == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                         : v == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}

// 5-D tensor map that moves one whole tile per TMA request (PassDesc g4 == 2).
// The tile's bit set T (physical bits of an nbits-bit index) splits into runs
// of consecutive bits; dim d starts at run d and extends up to the next run,
// so its box covers the run and its coordinate selects the outer bits above
// it.  Runs longer than a box dimension allows (256 elements) are split.
// Tile bits beyond the 5th run stay in dim 4's coordinate: one box per
// combination of them (they are the tile's top bits, so each box is a
// contiguous slice of the tile in smem).
// base == nullptr: layout only (host planning; no driver call).
bool make_box_tmap(void* base, int nbits, bool dbl, uint64_t T, QcTmap* out, PassDesc* d) {
  EncodeFn enc = base ? encoder() : nullptr;
  if ((base && !enc) || !(T & 1ull)) return false;
  const int epa = dbl ? 2 : 1;                // f64 elements per amplitude
  const int max0 = dbl ? 7 : 8, maxd = 8;    // box dim <= 256 elements
  int start[64], len[64], nr = 0;             // tile runs
  for (int p = 0; p < nbits; ++p) {
    if (!((T >> p) & 1ull)) continue;
    if (nr && start[nr - 1] + len[nr - 1] == p && len[nr - 1] < (nr == 1 ? max0 : maxd)) {
      ++len[nr - 1];
    } else {
      start[nr] = p;
      len[nr] = 1;
      ++nr;
    }
  }
  const int nd = nr < 5 ? nr : 5;
  uint32_t xmask = 0;
  int sub = 0;
  for (int i = 0; i < nr; ++i) {
    if (i < nd) {
      sub += len[i];
      continue;
    }
    for (int b = 0; b < len[i]; ++b) xmask |= 1u << (start[i] + b - start[4]);
  }
  if (std::popcount(xmask) > 4) return false;  // > 16 boxes per tile: keep the gather4 rows
  cuuint64_t gdim[5], gstride[4];
  cuuint32_t box[5], estr[5] = {1, 1, 1, 1, 1};
  for (int i = 0; i < nd; ++i) {
    const int end = i + 1 < nd ? start[i + 1] : nbits;
    if (end - start[i] + (i == 0 && dbl ? 1 : 0) > 32) return false;  // tensor-map dims are <= 2^32
  }
  for (int i = 0; i < 5; ++i) {
    if (i < nd) {
      const int end = i + 1 < nd ? start[i + 1] : nbits;
      gdim[i] = ((cuuint64_t)1 << (end - start[i])) * (i == 0 ? epa : 1);
      box[i] = (cuuint32_t)((1u << len[i]) * (i == 0 ? epa : 1));
      if (i) gstride[i - 1] = ((cuuint64_t)8 * epa) << start[i];
      d->bx_start[i] = start[i];
    } else {
      gdim[i] = 1;
      box[i] = 1;
      gstride[i - 1] = 16;
    }
  }
  d->bx_dims = nd;
  d->bx_start[nd] = nbits;
  d->bx_xmask = xmask;
  d->bx_sub = sub;
  if (!base) return true;
  CUtensorMap tm;
  const CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, base, gdim, gstride, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         box_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  memcpy(out, &tm, sizeof tm);
  return true;
}

// 2D tensor map over the state: rows of 2^rb amplitudes (as f64 elements) x
// 2^(n-rb) rows, box = one row; used with tile::gather4 / scatter4.
bool make_row_tmap(void* base, int n, int rb, bool dbl, QcTmap* out) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode enc = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      enc = reinterpret_cast<Encode>(fn);
  }
  if (!enc) return false;
  const uint64_t elems = (uint64_t)(dbl ? 2 : 1) << rb;
  // Rows above 1 KiB (8 KiB per gather4 request) deadlocked intermittently
  // under load on B200 in round 1, before the per-buffer tile tags of the
  // ring (fused_types.h).  Round 2 re-tested 2 KiB rows with the cap lifted
  // (QC_GATHER4_MAX_ROW=2048: 288 stress runs, c128 + c64, no hang, parity
  // green -- profiles/round2_stress_gather4_2k.log): the hang was the
  // parity aliasing the tags fixed.  The cap stays because the default box
  // transport never wants gather4 rows that wide.
  static const uint64_t max_row = getenv("QC_GATHER4_MAX_ROW") ? strtoull(getenv("QC_GATHER4_MAX_ROW"), nullptr, 10)
                                                                  : 1024;
  if (elems * 8 > max_row || elems > 256 || n - rb > 31 || n - rb < 2) return false;
  cuuint64_t gdim[2] = {elems, (cuuint64_t)1 << (n - rb)};
  cuuint64_t gstride[1] = {elems * 8};
  cuuint32_t box[2] = {(cuuint32_t)elems, 1};
  cuuint32_t estr[2] = {1, 1};
  static_assert(sizeof(QcTmap) == sizeof(CUtensorMap), "tensor map size");
  CUtensorMap tm;
  const CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, gdim, gstride, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  memcpy(out, &tm, sizeof tm);
  return true;
}

}  // namespace qc
