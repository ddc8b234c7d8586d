// fused_common.cuh -- device code shared by the AOT (interpreting) fused
// kernel and the NVRTC-specialised fused kernels: PTX wrappers for TMA bulk
// copies / mbarriers, complex arithmetic, the register-level gate bodies, and
// the warp-specialised tile pipeline.  Compiles under nvcc and NVRTC.
//
// Tile pipeline (persistent grid, 1 CTA per SM, kFusedThreads threads):
//   warp 8      TMA producer: cp.async.bulk global->smem for each row of the
//               next tile (mbarrier complete_tx), cp.async.bulk smem->global
//               of finished tiles (bulk_group), NBUF-deep ring.
//   warps 0..7  compute, in 2 groups of 4 warps taking alternate tiles:
//               Body::tile() applies the pass's ops to the tile in smem
//               (sub-stages of 16-amplitude register tasks, group-local named
//               barriers), then fence.proxy.async + mbarrier arrive.
// Rows are padded by 16 B in smem so slot strides of 1..16 amplitudes hit
// distinct bank quads (complex128).
#pragma once
#include "fused_types.h"

namespace qc {

template <typename T> struct CT;
template <> struct CT<double> { typedef double2 type; };
template <> struct CT<float> { typedef float2 type; };

// ------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t qc_saddr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void qc_mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(qc_saddr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void qc_fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void qc_mbar_arrive_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(qc_saddr(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void qc_mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(qc_saddr(b)) : "memory");
}
// Watchdog: a wait that has not completed after ~2^35 cycles (~15 s) traps,
// turning a pipeline bug into a launch error instead of a hung GPU.
__device__ __forceinline__ void qc_mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  const uint32_t a = qc_saddr(b);
  uint32_t spins = 0;
  long long t0 = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (!done && ((++spins & 1023u) == 0)) {
      const long long t = clock64();
      if (t0 == 0) t0 = t;
      else if (t - t0 > (1ll << 35)) asm volatile("trap;");
    }
  } while (!done);
}
__device__ __forceinline__ void qc_bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          qc_saddr(dst)),
      "l"(src), "r"(bytes), "r"(qc_saddr(bar))
      : "memory");
}
__device__ __forceinline__ void qc_bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(qc_saddr(src)), "r"(bytes)
               : "memory");
}
// 4 rows of a 2D tensor map (rows x row-elements) per request (sm_100a).
__device__ __forceinline__ void qc_gather4(void* dst, const QcTmap* tm, int32_t r0, int32_t r1, int32_t r2,
                                           int32_t r3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(qc_saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(qc_saddr(bar))
      : "memory");
}
__device__ __forceinline__ void qc_scatter4(const QcTmap* tm, int32_t r0, int32_t r1, int32_t r2, int32_t r3,
                                            const void* src) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.tile::scatter4.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
          reinterpret_cast<uint64_t>(tm)),
      "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(qc_saddr(src))
      : "memory");
}
// One 5-D TMA box (the whole tile) per request: dims in ascending physical
// bit order, so the box lands in smem in tile-local index order.
// L2 cache hints of the box transport (experiment knob, JIT passes only:
// QC_L2_HINT 1 = evict_first on tile loads and stores -- the state streams
// through L2 once per pass).
#ifndef QC_L2_HINT
#define QC_L2_HINT 0
#endif
__device__ __forceinline__ uint64_t qc_l2_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void qc_box_load(void* dst, const QcTmap* tm, const int32_t (&c)[5], uint64_t* bar) {
#if QC_L2_HINT
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(qc_saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(qc_saddr(bar)),
      "l"(qc_l2_policy())
      : "memory");
#else
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(qc_saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(qc_saddr(bar))
      : "memory");
#endif
}
__device__ __forceinline__ void qc_box_store(const QcTmap* tm, const int32_t (&c)[5], const void* src) {
#if QC_L2_HINT
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%1, %2, %3, %4, %5}], [%6], %7;"
               ::"l"(reinterpret_cast<uint64_t>(tm)),
               "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(qc_saddr(src)), "l"(qc_l2_policy())
               : "memory");
#else
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
                   reinterpret_cast<uint64_t>(tm)),
               "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(qc_saddr(src))
               : "memory");
#endif
}
// Box coordinates of a tile: per dim, the outer bits above its tile run
// (dim 0 in f64 elements: 2 per complex128 amplitude, 1 per complex64).
template <typename C>
__device__ __forceinline__ void qc_box_coords(const PassDesc& pd, uint64_t base, int32_t (&c)[5]) {
#pragma unroll
  for (int d = 0; d < 5; ++d) {
    c[d] = 0;
    if (d < pd.bx_dims) {
      const int lo = pd.bx_start[d], w = pd.bx_start[d + 1] - lo;
      const uint64_t v = (base >> lo) & ((1ull << w) - 1ull);
      c[d] = (int32_t)(d == 0 ? v * (sizeof(C) / 8) : v);
    }
  }
}
__device__ __forceinline__ void qc_bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void qc_bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void qc_bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void qc_fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// Named barrier of the calling thread's compute group (ids 1..kGroups).  The
// non-.aligned form: callers may arrive from divergent code (e.g. the
// single-thread phase-run prologue); reconverge the warp first anyway.
__device__ __forceinline__ void qc_compute_bar() {
  __syncwarp();
  asm volatile("barrier.sync %0, %1;" ::"r"(1 + (int)threadIdx.x / kGroupThreads), "n"(kGroupThreads)
               : "memory");
}
// Programmatic dependent launch (no-ops when the launch did not opt in): the
// next pass's CTAs are launched while this one drains and do their setup; only
// the producer warp touches global memory, and it waits for the previous grid
// (complete + flushed) before its first load.
__device__ __forceinline__ void qc_grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void qc_grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ uint32_t qc_gtid() { return threadIdx.x % kGroupThreads; }
__device__ __forceinline__ uint32_t qc_ins0(uint32_t x, int p) {
  return ((x >> p) << (p + 1)) | (x & ((1u << p) - 1u));
}
__device__ __forceinline__ uint64_t qc_tile_base(const PassDesc& pd, uint64_t t) {
  uint64_t g = 0;
  for (int j = 0; j < pd.n_outer; ++j) g |= ((t >> j) & 1ull) << pd.outer_pos[j];
  return g;
}

// ------------------------------------------------------ complex helpers
template <typename C>
__device__ __forceinline__ void qc_cmac(C& acc, const C m, const C a) {
  acc.x = fma(m.x, a.x, acc.x);
  acc.y = fma(m.x, a.y, acc.y);
  acc.x = fma(-m.y, a.y, acc.x);
  acc.y = fma(m.y, a.x, acc.y);
}
template <typename C>
__device__ __forceinline__ C qc_cmul(const C m, const C a) {
  C o;
  o.x = m.x * a.x - m.y * a.y;
  o.y = m.x * a.y + m.y * a.x;
  return o;
}
template <typename C>
__device__ __forceinline__ C qc_one() {
  C z;
  z.x = 1;
  z.y = 0;
  return z;
}

// ------------------------------------------- register ops on 16 slots
// M1: 2x2 on slot bit B; M2: 4x4 on slot bits (B0 = MSB of the 4x4 index,
// B1 = LSB).  The planner picks the exact structure of the matrix (zeros are
// exact): DENSE, PAIRS<X> (row r has non-zeros only in columns r and r^X),
// DIAG (identity rows skipped), ANTI (off-diagonal only) or MOVE (exact
// permutation: pure register moves, bit-exact).  Pairs / quads are processed
// one at a time; slot predicates (controls on slot bits) are per pair/quad.
template <int B>
__device__ __forceinline__ constexpr int qc_pair_base(int p) {
  return ((p >> B) << (B + 1)) | (p & ((1 << B) - 1));
}
template <int B0, int B1>
__device__ __forceinline__ constexpr int qc_quad_base(int q) {
  constexpr int LO = B0 < B1 ? B0 : B1, HI = B0 < B1 ? B1 : B0;
  int s = ((q >> LO) << (LO + 1)) | (q & ((1 << LO) - 1));
  return ((s >> HI) << (HI + 1)) | (s & ((1 << HI) - 1));
}
template <int B0, int B1>
__device__ __forceinline__ constexpr int qc_quad_el(int s, int r) {
  return s | (((r >> 1) & 1) << B0) | ((r & 1) << B1);
}

template <int B, typename C>
__device__ __forceinline__ void qc_m1_dense(C (&v)[kSlots], const C* __restrict__ cp, uint32_t sm,
                                            uint32_t sv) {
  const C m00 = cp[0], m01 = cp[1], m10 = cp[2], m11 = cp[3];
#pragma unroll
  for (int p = 0; p < kSlots / 2; ++p) {
    const int s0 = qc_pair_base<B>(p), s1 = s0 | (1 << B);
    if ((s0 & sm) != sv) continue;
    const C a = v[s0], b = v[s1];
    C o0 = qc_cmul(m00, a), o1 = qc_cmul(m10, a);
    qc_cmac(o0, m01, b);
    qc_cmac(o1, m11, b);
    v[s0] = o0;
    v[s1] = o1;
  }
}
template <int B, typename C>
__device__ __forceinline__ void qc_m1_anti(C (&v)[kSlots], const C* __restrict__ cp, uint32_t sm,
                                           uint32_t sv) {
  const C m01 = cp[0], m10 = cp[1];
#pragma unroll
  for (int p = 0; p < kSlots / 2; ++p) {
    const int s0 = qc_pair_base<B>(p), s1 = s0 | (1 << B);
    if ((s0 & sm) != sv) continue;
    const C a = v[s0], b = v[s1];
    v[s0] = qc_cmul(m01, b);
    v[s1] = qc_cmul(m10, a);
  }
}
template <int B, typename C>
__device__ __forceinline__ void qc_m1_move(C (&v)[kSlots], uint32_t sm, uint32_t sv) {
#pragma unroll
  for (int p = 0; p < kSlots / 2; ++p) {
    const int s0 = qc_pair_base<B>(p), s1 = s0 | (1 << B);
    if ((s0 & sm) != sv) continue;
    const C a = v[s0];
    v[s0] = v[s1];
    v[s1] = a;
  }
}
// DIAG: cp holds the entries of the non-identity rows only (row 0 first).
template <int B, typename C>
__device__ __forceinline__ void qc_m1_diag(C (&v)[kSlots], const C* __restrict__ cp, uint32_t ident,
                                           uint32_t sm, uint32_t sv) {
  const bool i0 = ident & 1u, i1 = ident & 2u;
  const C d0 = cp[0], d1 = cp[i0 ? 0 : 1];
#pragma unroll
  for (int p = 0; p < kSlots / 2; ++p) {
    const int s0 = qc_pair_base<B>(p), s1 = s0 | (1 << B);
    if ((s0 & sm) != sv) continue;
    if (!i0) v[s0] = qc_cmul(d0, v[s0]);
    if (!i1) v[s1] = qc_cmul(d1, v[s1]);
  }
}

template <int B0, int B1, int X, typename C>
__device__ __forceinline__ void qc_m2_pairs(C (&v)[kSlots], const C* __restrict__ cp, uint32_t ident,
                                            uint32_t sm, uint32_t sv) {
#pragma unroll
  for (int q = 0; q < kSlots / 4; ++q) {
    const int s = qc_quad_base<B0, B1>(q);
    if ((s & sm) != sv) continue;
    C a[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) a[c] = v[qc_quad_el<B0, B1>(s, c)];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (ident & (1u << r)) continue;
      C o = qc_cmul(cp[2 * r], a[r]);
      qc_cmac(o, cp[2 * r + 1], a[r ^ X]);
      v[qc_quad_el<B0, B1>(s, r)] = o;
    }
  }
}
template <int B0, int B1, typename C>
__device__ __forceinline__ void qc_m2_diag(C (&v)[kSlots], const C* __restrict__ cp, uint32_t ident,
                                           uint32_t sm, uint32_t sv) {
#pragma unroll
  for (int q = 0; q < kSlots / 4; ++q) {
    const int s = qc_quad_base<B0, B1>(q);
    if ((s & sm) != sv) continue;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (ident & (1u << r)) continue;
      const int e = qc_quad_el<B0, B1>(s, r);
      v[e] = qc_cmul(cp[r], v[e]);
    }
  }
}
template <int B0, int B1, typename C>
__device__ __forceinline__ void qc_m2_move(C (&v)[kSlots], uint32_t cols, uint32_t sm, uint32_t sv) {
#pragma unroll
  for (int q = 0; q < kSlots / 4; ++q) {
    const int s = qc_quad_base<B0, B1>(q);
    if ((s & sm) != sv) continue;
    C a[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) a[c] = v[qc_quad_el<B0, B1>(s, c)];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint32_t c = (cols >> (8 * r)) & 0xffu;
      v[qc_quad_el<B0, B1>(s, r)] = c == 0 ? a[0] : c == 1 ? a[1] : c == 2 ? a[2] : a[3];
    }
  }
}
template <int B0, int B1, typename C>
__device__ __forceinline__ void qc_m2_dense(C (&v)[kSlots], const C* __restrict__ cp, uint32_t sm,
                                            uint32_t sv) {
#pragma unroll
  for (int q = 0; q < kSlots / 4; ++q) {
    const int s = qc_quad_base<B0, B1>(q);
    if ((s & sm) != sv) continue;
    C a[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) a[c] = v[qc_quad_el<B0, B1>(s, c)];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      C o = qc_cmul(cp[4 * r], a[0]);
#pragma unroll
      for (int c = 1; c < 4; ++c) qc_cmac(o, cp[4 * r + c], a[c]);
      v[qc_quad_el<B0, B1>(s, r)] = o;
    }
  }
}

// F_MK (generic 3- / 4-target gate) in canonical slot order: MISS = the slot
// bit not in the op (k = 3) or 4 (k = 4: every slot bit, index = slot).  A
// slot-bit predicate can only be on MISS.
template <int MISS>
__device__ __forceinline__ constexpr int qc_mk_expand(int c) {
  return MISS >= 4 ? c : (((c >> MISS) << (MISS + 1)) | (c & ((1 << MISS) - 1)));
}
template <int MISS, typename C>
__device__ __forceinline__ void qc_mk_dense(C (&v)[kSlots], const C* __restrict__ cp, uint32_t sm, uint32_t sv) {
  constexpr int K = MISS < 4 ? 3 : 4, D = 1 << K, NB = MISS < 4 ? 2 : 1;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int s0 = MISS < 4 ? (b << MISS) : 0;
    if ((s0 & sm) != sv) continue;
    C a[D];
#pragma unroll
    for (int c = 0; c < D; ++c) a[c] = v[s0 | qc_mk_expand<MISS>(c)];
#pragma unroll
    for (int r = 0; r < D; ++r) {
      C o = qc_cmul(cp[D * r], a[0]);
#pragma unroll
      for (int c = 1; c < D; ++c) qc_cmac(o, cp[D * r + c], a[c]);
      v[s0 | qc_mk_expand<MISS>(r)] = o;
    }
  }
}

template <typename C>
__device__ __forceinline__ void qc_scale_slots(C (&v)[kSlots], const C w, uint32_t sm, uint32_t sv) {
#pragma unroll
  for (int s = 0; s < kSlots; ++s)
    if ((s & sm) == sv) v[s] = qc_cmul(w, v[s]);
}
// Phase run with its base bit on slot bit B: |1> slots x w1, |0> slots x w0.
template <typename C>
__device__ __forceinline__ void qc_swap(C& a, C& b) {
  const C t = a;
  a = b;
  b = t;
}

// Lane-dependent swap as selects (no divergent branch: both paths would need
// their own copies of the 16 registers and a reconvergence point).
template <typename C>
__device__ __forceinline__ void qc_cswap(bool p, C& a, C& b) {
  const C x = a, y = b;
  a.x = p ? y.x : x.x;
  a.y = p ? y.y : x.y;
  b.x = p ? x.x : y.x;
  b.y = p ? x.y : y.y;
}

template <int B, typename C>
__device__ __forceinline__ void qc_prun_slot(C (&v)[kSlots], const C w0, const C w1, bool any0) {
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    if (s & (1 << B))
      v[s] = qc_cmul(w1, v[s]);
    else if (any0)
      v[s] = qc_cmul(w0, v[s]);
  }
}

// ------------------------------------------------------- tile pipeline
// QC_WARP_SYNC 1: consumers poll the buffer tag and arrive on the `empty`
// barrier once per warp (after __syncwarp) instead of once per thread.
#ifndef QC_WARP_SYNC
#define QC_WARP_SYNC 0
#endif
// Body must provide:
//   static size_t smem_bytes(const PassDesc&)          extra smem it needs
//   void setup(unsigned char* extra, const PassDesc&)   all threads, before sync
//   void prologue(uint64_t tbase, int par)             compute threads, per tile
//   void tile(C* buf, uint64_t tbase, int par)          compute threads, per tile
// Tile transport of a tile spanning shards (pd.grp = j > 0): its top j
// tile-local bits are rank bits, so its 2^j sub-tiles (2^(k-j) amplitudes
// each, contiguous in smem) are moved separately, each from / to its own
// buffer (tmaps->m[h], sub_state[h], sub_addr[h]); other passes: one sub-tile
// (tmaps->m[0], state, addr_bits).
template <typename C, int NBUF, class Body>
__device__ __forceinline__ void qc_fused_pipeline(C* __restrict__ state, const PassDesc& pd,
                                                  const QcTmapSet* tmaps, unsigned char* smem_raw, Body& body) {
  const int rb = pd.rb, k = pd.k, ps = pd.pshift;
  const uint32_t PAD = kPadBytes / sizeof(C);
  const uint32_t row_amps = 1u << rb;
  const uint32_t nrows = 1u << (k - rb);
  const uint32_t buf_amps = (1u << k) + ((1u << k) >> ps) * PAD;
  // smem offset (in amplitudes) of tile-local row r: padded every 2^ps amps
  auto row_at = [&](uint32_t r) { const uint32_t l = r << rb; return l + (l >> ps) * PAD; };
  C* bufs = reinterpret_cast<C*>(smem_raw);
  unsigned char* p = smem_raw + (size_t)NBUF * buf_amps * sizeof(C);
  uint64_t* row_off = reinterpret_cast<uint64_t*>(p);
  p += (size_t)nrows * 8;
  unsigned char* extra = p;
  p += Body::smem_bytes(pd);
  uint64_t* full = reinterpret_cast<uint64_t*>(p);
  uint64_t* empty = full + NBUF;
  volatile uint32_t* buf_tile = reinterpret_cast<volatile uint32_t*>(empty + NBUF);  // tile tag per buffer
  const int tid = threadIdx.x;

  body.setup(extra, pd);
  for (uint32_t r = tid; r < nrows; r += blockDim.x) {
    uint64_t g = 0;
    for (int j = 0; j < pd.n_hi; ++j) g |= (uint64_t)((r >> j) & 1u) << pd.hi_pos[j];
    row_off[r] = g & ~pd.addr_strip;
  }
  if (tid == 0) {
    for (int b = 0; b < NBUF; ++b) {
      qc_mbar_init(&full[b], 1);
      qc_mbar_init(&empty[b], QC_WARP_SYNC ? kGroupThreads / 32 : kGroupThreads);
      buf_tile[b] = 0xffffffffu;
    }
    qc_fence_mbar_init();
  }
  __syncthreads();
  // every CTA of this grid is resident (grid <= SMs): the next pass may launch
  qc_grid_dep_launch();

  const uint64_t n_tiles = pd.n_tiles;
  const uint64_t my_n =
      (blockIdx.x < n_tiles) ? (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  if (tid >= kComputeThreads) {
    // ============================ TMA producer warp ============================
    const int lane = tid & 31;
    const uint32_t row_bytes = row_amps * (uint32_t)sizeof(C);
    const uint32_t tile_bytes = nrows * row_bytes;
    qc_grid_dep_wait();
    for (uint64_t i = 0; i < my_n + NBUF; ++i) {
      const int b = (int)(i % NBUF);
      C* buf = bufs + (size_t)b * buf_amps;
      if (i >= NBUF) {  // buffer b holds finished tile i-NBUF: write it back
        const uint64_t ip = i - NBUF;
        qc_mbar_wait(&empty[b], (uint32_t)((ip / NBUF) & 1ull));
        const uint64_t base = qc_tile_base(pd, pd.tile0 + blockIdx.x + ip * gridDim.x) & ~pd.addr_strip;
        if (pd.g4 == 2) {
          if (lane == 0) {
            for (int h = 0; h < (1 << pd.grp); ++h) {
              int32_t c[5];
              qc_box_coords<C>(pd, base | (pd.grp ? pd.sub_addr[h] : pd.addr_bits), c);
              const int32_t c4 = c[4];
              C* hb = buf + ((size_t)h << (k - pd.grp));
              uint32_t v = 0, j = 0;
              do {  // every combination of the extra tile bits (one box if none)
                c[4] = c4 | (int32_t)v;
                qc_box_store(&tmaps->m[h], c, hb + ((size_t)j << pd.bx_sub));
                v = (v - pd.bx_xmask) & pd.bx_xmask;
                ++j;
              } while (v);
            }
          }
        } else if (pd.g4) {
          for (uint32_t r = 4 * lane; r < nrows; r += 128) {
            const int h = (int)(r >> (k - rb - pd.grp));  // sub-tile: the row's top grp bits
            const uint64_t bb = base | (pd.grp ? pd.sub_addr[h] : pd.addr_bits);
            qc_scatter4(&tmaps->m[h], (int32_t)((bb | row_off[r]) >> rb), (int32_t)((bb | row_off[r + 1]) >> rb),
                        (int32_t)((bb | row_off[r + 2]) >> rb), (int32_t)((bb | row_off[r + 3]) >> rb),
                        buf + row_at(r));
          }
        } else {
          for (uint32_t r = lane; r < nrows; r += 32) {
            const int h = (int)(r >> (k - rb - pd.grp));
            C* st = pd.grp ? reinterpret_cast<C*>(pd.sub_state[h]) : state;
            qc_bulk_s2g(st + (base | (pd.grp ? pd.sub_addr[h] : pd.addr_bits) | row_off[r]), buf + row_at(r),
                        row_bytes);
          }
        }
        qc_bulk_commit();
        qc_bulk_wait_read0();  // smem of buffer b may be overwritten after this
        __syncwarp();
      }
      if (i < my_n) {
        const uint64_t base = qc_tile_base(pd, pd.tile0 + blockIdx.x + i * gridDim.x) & ~pd.addr_strip;
        if (lane == 0) {
          // full[b]'s pending phase now belongs to tile i (atomic: the tag is
          // polled by the consumer groups -- an explicit flag, not a data race)
          atomicExch(const_cast<uint32_t*>(&buf_tile[b]), (uint32_t)i);
          qc_mbar_arrive_expect_tx(&full[b], tile_bytes);
        }
        __syncwarp();
        if (pd.g4 == 2) {
          if (lane == 0) {
            for (int h = 0; h < (1 << pd.grp); ++h) {
              int32_t c[5];
              qc_box_coords<C>(pd, base | (pd.grp ? pd.sub_addr[h] : pd.addr_bits), c);
              const int32_t c4 = c[4];
              C* hb = buf + ((size_t)h << (k - pd.grp));
              uint32_t v = 0, j = 0;
              do {
                c[4] = c4 | (int32_t)v;
                qc_box_load(hb + ((size_t)j << pd.bx_sub), &tmaps->m[h], c, &full[b]);
                v = (v - pd.bx_xmask) & pd.bx_xmask;
                ++j;
              } while (v);
            }
          }
        } else if (pd.g4) {
          for (uint32_t r = 4 * lane; r < nrows; r += 128) {
            const int h = (int)(r >> (k - rb - pd.grp));
            const uint64_t bb = base | (pd.grp ? pd.sub_addr[h] : pd.addr_bits);
            qc_gather4(buf + row_at(r), &tmaps->m[h], (int32_t)((bb | row_off[r]) >> rb),
                       (int32_t)((bb | row_off[r + 1]) >> rb), (int32_t)((bb | row_off[r + 2]) >> rb),
                       (int32_t)((bb | row_off[r + 3]) >> rb), &full[b]);
          }
        } else {
          for (uint32_t r = lane; r < nrows; r += 32) {
            const int h = (int)(r >> (k - rb - pd.grp));
            const C* st = pd.grp ? reinterpret_cast<const C*>(pd.sub_state[h]) : state;
            qc_bulk_g2s(buf + row_at(r), st + (base | (pd.grp ? pd.sub_addr[h] : pd.addr_bits) | row_off[r]),
                        row_bytes, &full[b]);
          }
        }
      }
    }
    qc_bulk_wait0();
    return;
  }

  // =============================== compute warps ===============================
  // Two groups of compute warps take alternate tiles, so one group's smem
  // round trips and barriers overlap the other group's arithmetic.
  for (uint64_t i = (uint64_t)(tid / kGroupThreads); i < my_n; i += kGroups) {
    const int b = (int)(i % NBUF);
    const int par = (int)(i % kWSlots);
    // global index of the tile's first amplitude (rank bits included): used
    // for control predicates and diagonal bits; memory addresses stay local
    const uint64_t tbase = qc_tile_base(pd, pd.tile0 + blockIdx.x + i * gridDim.x) | pd.rank_bits;
    body.prologue(tbase, par);
    if (kGroups > 1 && NBUF % kGroups) {
      // wait until the producer has claimed buffer b for this tile (see fused_types.h)
#if QC_WARP_SYNC
      // one poller per warp (32x fewer atomics on the tag word)
      if ((threadIdx.x & 31) == 0)
        while (atomicOr(const_cast<uint32_t*>(&buf_tile[b]), 0u) != (uint32_t)i) __nanosleep(64);
      __syncwarp();
#else
      while (atomicOr(const_cast<uint32_t*>(&buf_tile[b]), 0u) != (uint32_t)i) __nanosleep(64);
#endif
    }
    qc_mbar_wait(&full[b], (uint32_t)((i / NBUF) & 1ull));
    body.tile(bufs + (size_t)b * buf_amps, tbase, par);
    qc_fence_proxy_async();  // generic-proxy smem writes -> visible to the TMA store
#if QC_WARP_SYNC
    __syncwarp();            // the warp's fenced writes precede lane 0's (release) arrive
    if ((threadIdx.x & 31) == 0) qc_mbar_arrive(&empty[b]);
#else
    qc_mbar_arrive(&empty[b]);
#endif
  }
}

// Bytes of smem the pipeline itself needs (buffers + row offsets + barriers).
template <typename C>
__host__ __device__ inline size_t qc_pipeline_smem(int k, int rb, int pshift, int nbuf) {
  const size_t PAD = kPadBytes / sizeof(C);
  const size_t nrows = (size_t)1 << (k - rb);
  const size_t buf_amps = ((size_t)1 << k) + (((size_t)1 << k) >> pshift) * PAD;
  return (size_t)nbuf * buf_amps * sizeof(C) + nrows * 8 + 2 * (size_t)nbuf * 8 + (size_t)nbuf * 4;
}

}  // namespace qc
