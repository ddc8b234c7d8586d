// kernels_fused.cu -- the fused tile pass (north-star "gate-fusion pass").
//
// One launch applies every gate of a planner pass (plan.cpp) in ONE HBM round
// trip.  The pass fixes a set T of k physical bits (always including bits
// 0..rb-1, so each tile is 2^{k-rb} rows of 2^rb contiguous amplitudes).  A
// tile is the 2^k amplitudes sharing one value of the n-k outer bits; every
// gate of the pass acts inside a tile because its non-diagonal targets are in
// T, while controls / diagonal bits outside T are per-tile constants.  That is
// the paper's per-gate loop (Alg. alg:1q / alg:ctrl-1q / alg:2q)
// regrouped: the 2^{n-1} pair updates of a gate are partitioned by tile, and
// consecutive gates are applied to a tile while it sits in shared memory.
//
// Structure (persistent grid, 1 CTA per SM, 288 threads):
//   warp 8      TMA producer: cp.async.bulk global->smem for each row of the
//               next tile (mbarrier complete_tx), cp.async.bulk smem->global
//               of finished tiles (bulk_group), NBUF-deep ring.
//   warps 0..7  compute: per sub-stage, each thread task loads the 16
//               amplitudes differing in the 4 slot bits into registers,
//               applies the sub-stage's gates there (2x2 / 4x4 matvecs, moves,
//               diagonal scalings), writes them back; named barrier between
//               sub-stages; fence.proxy.async + mbarrier arrive when done.
// Rows are padded by 16 B in smem so that slot strides of 1..16 amplitudes
// hit distinct bank quads (complex128).
#include <cuda_runtime.h>

#include "qc_internal.h"

namespace qc {
namespace {

template <typename T> struct CT;
template <> struct CT<double> { using type = double2; };
template <> struct CT<float> { using type = float2; };

// ------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t saddr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  const uint32_t a = saddr(b);
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(saddr(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void compute_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kComputeThreads) : "memory");
}

__device__ __forceinline__ uint32_t insert0_32(uint32_t x, int p) {
  return ((x >> p) << (p + 1)) | (x & ((1u << p) - 1u));
}

__device__ __forceinline__ uint64_t tile_base(const PassDesc& pd, uint64_t t) {
  uint64_t g = 0;
  for (int j = 0; j < pd.n_outer; ++j) g |= ((t >> j) & 1ull) << pd.outer_pos[j];
  return g;
}

// ----------------------------------------------------- register gate bodies
template <typename C, typename T>
__device__ __forceinline__ void cmad2(C& o, const C a, const C b, T m0r, T m0i, T m1r, T m1i) {
  o.x = m0r * a.x - m0i * a.y + m1r * b.x - m1i * b.y;
  o.y = m0r * a.y + m0i * a.x + m1r * b.y + m1i * b.x;
}

template <int B, typename C, typename T>
__device__ __forceinline__ void r_dense1(C (&v)[kSlots], const T* __restrict__ m, uint32_t smask,
                                         uint32_t sval) {
  const T m0r = m[0], m0i = m[1], m1r = m[2], m1i = m[3];
  const T m2r = m[4], m2i = m[5], m3r = m[6], m3i = m[7];
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    if (s & (1 << B)) continue;
    if ((s & smask) != sval) continue;
    const int s1 = s | (1 << B);
    const C a = v[s], b = v[s1];
    cmad2(v[s], a, b, m0r, m0i, m1r, m1i);
    cmad2(v[s1], a, b, m2r, m2i, m3r, m3i);
  }
}

template <int B, typename C>
__device__ __forceinline__ void r_perm1(C (&v)[kSlots], uint32_t smask, uint32_t sval) {
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    if (s & (1 << B)) continue;
    if ((s & smask) != sval) continue;
    const int s1 = s | (1 << B);
    const C a = v[s];
    v[s] = v[s1];
    v[s1] = a;
  }
}

template <typename C, typename T>
__device__ __forceinline__ void cscale(C& x, T dr, T di) {
  const C a = x;
  x.x = dr * a.x - di * a.y;
  x.y = dr * a.y + di * a.x;
}

template <int B, typename C, typename T>
__device__ __forceinline__ void r_diag1_slot(C (&v)[kSlots], const T* __restrict__ m, int d0_is_one,
                                             uint32_t smask, uint32_t sval) {
  const T d0r = m[0], d0i = m[1], d1r = m[2], d1i = m[3];
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    if ((s & smask) != sval) continue;
    if (s & (1 << B)) {
      cscale(v[s], d1r, d1i);
    } else if (!d0_is_one) {
      cscale(v[s], d0r, d0i);
    }
  }
}

template <typename C, typename T>
__device__ __forceinline__ void r_scale_all(C (&v)[kSlots], T dr, T di, uint32_t smask, uint32_t sval) {
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    if ((s & smask) != sval) continue;
    cscale(v[s], dr, di);
  }
}

template <int B0, int B1, typename C, typename T>
__device__ __forceinline__ void r_dense2(C (&v)[kSlots], const T* __restrict__ m, uint32_t smask,
                                         uint32_t sval) {
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    if (s & ((1 << B0) | (1 << B1))) continue;
    if ((s & smask) != sval) continue;
    int id[4];
    C a[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      id[r] = s | (((r >> 1) & 1) << B0) | ((r & 1) << B1);
      a[r] = v[id[r]];
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      T ore = 0, oim = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const T mr = m[2 * (4 * r + c)], mi = m[2 * (4 * r + c) + 1];
        ore += mr * a[c].x - mi * a[c].y;
        oim += mr * a[c].y + mi * a[c].x;
      }
      v[id[r]].x = ore;
      v[id[r]].y = oim;
    }
  }
}

template <int B0, int B1, typename C>
__device__ __forceinline__ void r_swap2(C (&v)[kSlots], uint32_t smask, uint32_t sval) {
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    if (s & ((1 << B0) | (1 << B1))) continue;
    if ((s & smask) != sval) continue;
    const int i0 = s | (1 << B0), i1 = s | (1 << B1);
    const C a = v[i0];
    v[i0] = v[i1];
    v[i1] = a;
  }
}

template <typename C, typename T>
__device__ __forceinline__ void apply_op(const FOpT<T>& op, C (&v)[kSlots], uint32_t lb,
                                         uint64_t tbase) {
  if ((tbase & op.omask) != op.oval) return;
  if ((lb & op.lmask) != op.lval) return;
  const uint32_t sm = op.smask, sv = op.sval;
  switch (op.kind) {
    case F_DENSE1:
      switch (op.sb0) {
        case 0: r_dense1<0>(v, op.m, sm, sv); break;
        case 1: r_dense1<1>(v, op.m, sm, sv); break;
        case 2: r_dense1<2>(v, op.m, sm, sv); break;
        default: r_dense1<3>(v, op.m, sm, sv); break;
      }
      break;
    case F_PERM1:
      switch (op.sb0) {
        case 0: r_perm1<0>(v, sm, sv); break;
        case 1: r_perm1<1>(v, sm, sv); break;
        case 2: r_perm1<2>(v, sm, sv); break;
        default: r_perm1<3>(v, sm, sv); break;
      }
      break;
    case F_DIAG1:
      if (op.dsrc == D_SLOT) {
        switch (op.sb0) {
          case 0: r_diag1_slot<0>(v, op.m, op.d0_is_one, sm, sv); break;
          case 1: r_diag1_slot<1>(v, op.m, op.d0_is_one, sm, sv); break;
          case 2: r_diag1_slot<2>(v, op.m, op.d0_is_one, sm, sv); break;
          default: r_diag1_slot<3>(v, op.m, op.d0_is_one, sm, sv); break;
        }
      } else {
        const int bit = (op.dsrc == D_LOCAL) ? (int)((lb >> op.dbit) & 1u)
                                             : (int)((tbase >> op.dbit) & 1ull);
        if (bit == 0 && op.d0_is_one) break;
        r_scale_all(v, op.m[2 * bit], op.m[2 * bit + 1], sm, sv);
      }
      break;
    case F_DENSE2:
      switch (op.sb0 * 4 + op.sb1) {
        case 1: r_dense2<0, 1>(v, op.m, sm, sv); break;
        case 2: r_dense2<0, 2>(v, op.m, sm, sv); break;
        case 3: r_dense2<0, 3>(v, op.m, sm, sv); break;
        case 4: r_dense2<1, 0>(v, op.m, sm, sv); break;
        case 6: r_dense2<1, 2>(v, op.m, sm, sv); break;
        case 7: r_dense2<1, 3>(v, op.m, sm, sv); break;
        case 8: r_dense2<2, 0>(v, op.m, sm, sv); break;
        case 9: r_dense2<2, 1>(v, op.m, sm, sv); break;
        case 11: r_dense2<2, 3>(v, op.m, sm, sv); break;
        case 12: r_dense2<3, 0>(v, op.m, sm, sv); break;
        case 13: r_dense2<3, 1>(v, op.m, sm, sv); break;
        default: r_dense2<3, 2>(v, op.m, sm, sv); break;
      }
      break;
    default: {  // F_SWAP2 (symmetric: planner passes sb0 < sb1)
      switch (op.sb0 * 4 + op.sb1) {
        case 1: r_swap2<0, 1>(v, sm, sv); break;
        case 2: r_swap2<0, 2>(v, sm, sv); break;
        case 3: r_swap2<0, 3>(v, sm, sv); break;
        case 6: r_swap2<1, 2>(v, sm, sv); break;
        case 7: r_swap2<1, 3>(v, sm, sv); break;
        default: r_swap2<2, 3>(v, sm, sv); break;
      }
      break;
    }
  }
}

// ------------------------------------------------------------------ kernel
template <typename T, int NBUF>
__global__ void __launch_bounds__(kFusedThreads, 1)
    fused_pass_kernel(typename CT<T>::type* __restrict__ state, const PassDesc pd,
                      const SubStageDesc* __restrict__ subs, const FOpT<T>* __restrict__ ops) {
  using C = typename CT<T>::type;
  constexpr uint32_t PAD = kPadBytes / sizeof(C);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int rb = pd.rb, k = pd.k;
  const uint32_t row_amps = 1u << rb;
  const uint32_t row_stride = row_amps + PAD;
  const uint32_t nrows = 1u << (k - rb);
  const uint32_t buf_amps = nrows * row_stride;
  C* bufs = reinterpret_cast<C*>(smem_raw);
  uint64_t* row_off = reinterpret_cast<uint64_t*>(smem_raw + (size_t)NBUF * buf_amps * sizeof(C));
  uint64_t* full = row_off + nrows;
  uint64_t* empty = full + NBUF;
  const int tid = threadIdx.x;

  // global offset of every tile-local row (hi bits deposited at hi_pos)
  for (uint32_t r = tid; r < nrows; r += blockDim.x) {
    uint64_t g = 0;
    for (int j = 0; j < pd.n_hi; ++j) g |= (uint64_t)((r >> j) & 1u) << pd.hi_pos[j];
    row_off[r] = g;
  }
  if (tid == 0) {
    for (int b = 0; b < NBUF; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], kComputeThreads);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const uint64_t n_tiles = pd.n_tiles;
  const uint64_t my_n =
      (blockIdx.x < n_tiles) ? (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  if (tid >= kComputeThreads) {
    // ============================ TMA producer warp ============================
    const int lane = tid & 31;
    const uint32_t row_bytes = row_amps * (uint32_t)sizeof(C);
    const uint32_t tile_bytes = nrows * row_bytes;
    for (uint64_t i = 0; i < my_n + NBUF; ++i) {
      const int b = (int)(i % NBUF);
      C* buf = bufs + (size_t)b * buf_amps;
      if (i >= NBUF) {  // buffer b holds finished tile i-NBUF: write it back
        const uint64_t ip = i - NBUF;
        mbar_wait(&empty[b], (uint32_t)((ip / NBUF) & 1ull));
        const uint64_t base = tile_base(pd, blockIdx.x + ip * gridDim.x);
        for (uint32_t r = lane; r < nrows; r += 32)
          bulk_s2g(state + (base | row_off[r]), buf + (size_t)r * row_stride, row_bytes);
        bulk_commit();
        bulk_wait_read0();  // smem of buffer b may be overwritten after this
        __syncwarp();
      }
      if (i < my_n) {
        const uint64_t base = tile_base(pd, blockIdx.x + i * gridDim.x);
        if (lane == 0) mbar_arrive_expect_tx(&full[b], tile_bytes);
        __syncwarp();
        for (uint32_t r = lane; r < nrows; r += 32)
          bulk_g2s(buf + (size_t)r * row_stride, state + (base | row_off[r]), row_bytes, &full[b]);
      }
    }
    bulk_wait0();
    return;
  }

  // =============================== compute warps ===============================
  const uint32_t ntasks = 1u << (k - kSlotBits);
  for (uint64_t i = 0; i < my_n; ++i) {
    const int b = (int)(i % NBUF);
    mbar_wait(&full[b], (uint32_t)((i / NBUF) & 1ull));
    C* buf = bufs + (size_t)b * buf_amps;
    const uint64_t tbase = tile_base(pd, blockIdx.x + i * gridDim.x);
    for (int si = pd.sub_begin; si < pd.sub_end; ++si) {
      if (si != pd.sub_begin) compute_bar();
      const SubStageDesc sd = subs[si];
      uint32_t poff[kSlots];
#pragma unroll
      for (int s = 0; s < kSlots; ++s) {
        uint32_t off = 0;
#pragma unroll
        for (int j = 0; j < kSlotBits; ++j)
          if (s & (1 << j)) off |= 1u << sd.g[j];
        poff[s] = off + (off >> rb) * PAD;
      }
      for (uint32_t task = tid; task < ntasks; task += kComputeThreads) {
        uint32_t lb = task;
#pragma unroll
        for (int j = 0; j < kSlotBits; ++j) lb = insert0_32(lb, sd.g[j]);
        const uint32_t pb = lb + (lb >> rb) * PAD;
        C v[kSlots];
#pragma unroll
        for (int s = 0; s < kSlots; ++s) v[s] = buf[pb + poff[s]];
        for (int oi = sd.op_begin; oi < sd.op_end; ++oi) apply_op(ops[oi], v, lb, tbase);
#pragma unroll
        for (int s = 0; s < kSlots; ++s) buf[pb + poff[s]] = v[s];
      }
    }
    fence_proxy_async();  // generic-proxy smem writes -> visible to the TMA store
    mbar_arrive(&empty[b]);
  }
}

template <typename T>
size_t smem_for(int k, int rb, int nbuf) {
  using C = typename CT<T>::type;
  const size_t PAD = kPadBytes / sizeof(C);
  const size_t nrows = (size_t)1 << (k - rb);
  const size_t buf_amps = nrows * (((size_t)1 << rb) + PAD);
  return (size_t)nbuf * buf_amps * sizeof(C) + nrows * 8 + 2 * (size_t)nbuf * 8;
}

constexpr size_t kMaxSmem = 227 * 1024;

template <typename T>
int pick_nbuf(int k, int rb) {
  for (int nb = 3; nb >= 1; --nb)
    if (smem_for<T>(k, rb, nb) <= kMaxSmem) return nb;
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
  return (int)e;
}

template <typename T>
int launch_t(void* state, const PassDesc& pd, const void* d_subs, const void* d_ops, int ctas,
             cudaStream_t st) {
  using C = typename CT<T>::type;
  const int nb = pick_nbuf<T>(pd.k, pd.rb);
  if (nb == 0) return (int)cudaErrorInvalidValue;
  const size_t smem = smem_for<T>(pd.k, pd.rb, nb);
  uint64_t grid = pd.n_tiles;
  if (grid > (uint64_t)ctas) grid = (uint64_t)ctas;
  C* s = reinterpret_cast<C*>(state);
  auto subs = reinterpret_cast<const SubStageDesc*>(d_subs);
  auto ops = reinterpret_cast<const FOpT<T>*>(d_ops);
  switch (nb) {
    case 3: fused_pass_kernel<T, 3><<<(unsigned)grid, kFusedThreads, smem, st>>>(s, pd, subs, ops); break;
    case 2: fused_pass_kernel<T, 2><<<(unsigned)grid, kFusedThreads, smem, st>>>(s, pd, subs, ops); break;
    default: fused_pass_kernel<T, 1><<<(unsigned)grid, kFusedThreads, smem, st>>>(s, pd, subs, ops); break;
  }
  return (int)cudaGetLastError();
}

}  // namespace

size_t fused_smem_bytes(bool dbl, int k, int rb) {
  if (dbl) {
    const int nb = pick_nbuf<double>(k, rb);
    return nb ? smem_for<double>(k, rb, nb) : 0;
  }
  const int nb = pick_nbuf<float>(k, rb);
  return nb ? smem_for<float>(k, rb, nb) : 0;
}

int fused_configure(bool dbl, size_t) { return dbl ? configure_t<double>() : configure_t<float>(); }

int launch_fused_pass(void* state, bool dbl, const PassDesc& pd, const void* d_subs,
                      const void* d_ops, int ctas, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  return dbl ? launch_t<double>(state, pd, d_subs, d_ops, ctas, st)
             : launch_t<float>(state, pd, d_subs, d_ops, ctas, st);
}

}  // namespace qc
