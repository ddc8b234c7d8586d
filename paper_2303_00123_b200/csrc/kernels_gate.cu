// kernels_gate.cu -- one kernel launch per gate (the unfused path).
//
// Each launch is the paper's single `for j` loop (Alg. alg:1q P:633-651,
// alg:ctrl-1q P:856-880, alg:2q P:883-919) written for sm_100a: a grid-stride
// loop over the 2^{n-1-c} pairs (2^{n-2-c} quads) with 64-bit indices
// (DESIGN R3).  Index generation inserts zero bits at the sorted target and
// control positions -- the paper's m_L/m_C/m_R mask form generalised to any
// number of inserted bits -- and ORs in the control values
// ("a_j = a_j + 2^{n-q_c-1}").  Classes:
//   DENSE1  2x2 matvec on (a_j, b_j)
//   PERM1   swap phi[a_j] <-> phi[b_j] (X, CNOT, CCX)
//   DIAG1   d0 == 1: scale only b_j (Z, P, CZ, CP)
//           else  : scale every amplitude by d[bit] (RZ)
//   DENSE2  4x4 matvec on quads (a,b,c,d) indexed by the LISTED order (R1)
//   SWAP2   psi[b] = phi[c], psi[c] = phi[b]
#include <cuda_runtime.h>

#include "qc_internal.h"

namespace qc {
namespace {

template <typename T> struct CT;
template <> struct CT<double> { using type = double2; };
template <> struct CT<float> { using type = float2; };

__device__ __forceinline__ uint64_t insert0(uint64_t x, int p) {
  const uint64_t lo = x & ((1ull << p) - 1);
  return ((x >> p) << (p + 1)) | lo;
}

// One work item (pair / quad / amplitude) of a gate: load phase then store
// phase, so a thread can issue the loads of several items before any store.
template <typename T, int KIND>
struct Item {
  using C = typename CT<T>::type;
  uint64_t id[4];
  C v[4];
  __device__ __forceinline__ void load(const C* __restrict__ s, const GateArgs<T>& a, uint64_t j) {
    uint64_t x = j;
#pragma unroll 4
    for (int i = 0; i < 4; ++i)
      if (i < a.nins) x = insert0(x, a.ins[i]);
    for (int i = 4; i < a.nins; ++i) x = insert0(x, a.ins[i]);  // many controls (qc_mgate)
    x |= a.setmask;
    if (KIND == (int)GK::DENSE1 || KIND == (int)GK::PERM1) {
      id[0] = x;
      id[1] = x | (1ull << a.t0);
      v[0] = s[id[0]];
      v[1] = s[id[1]];
    } else if (KIND == (int)GK::DIAG1) {
      id[0] = x;
      v[0] = s[x];
    } else if (KIND == (int)GK::DENSE2) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        id[r] = x | ((uint64_t)((r >> 1) & 1) << a.t0) | ((uint64_t)(r & 1) << a.t1);
        v[r] = s[id[r]];
      }
    } else {  // SWAP2
      id[0] = x | (1ull << a.t0);
      id[1] = x | (1ull << a.t1);
      v[0] = s[id[0]];
      v[1] = s[id[1]];
    }
  }
  __device__ __forceinline__ void store(C* __restrict__ s, const GateArgs<T>& a) const {
    if (KIND == (int)GK::DENSE1) {
      const C u = v[0], w = v[1];
      C o0, o1;
      o0.x = a.m[0] * u.x - a.m[1] * u.y + a.m[2] * w.x - a.m[3] * w.y;
      o0.y = a.m[0] * u.y + a.m[1] * u.x + a.m[2] * w.y + a.m[3] * w.x;
      o1.x = a.m[4] * u.x - a.m[5] * u.y + a.m[6] * w.x - a.m[7] * w.y;
      o1.y = a.m[4] * u.y + a.m[5] * u.x + a.m[6] * w.y + a.m[7] * w.x;
      s[id[0]] = o0;
      s[id[1]] = o1;
    } else if (KIND == (int)GK::PERM1 || KIND == (int)GK::SWAP2) {  // pure moves (bit-exact)
      s[id[0]] = v[1];
      s[id[1]] = v[0];
    } else if (KIND == (int)GK::DIAG1) {
      // d0 == 1: x already has the target bit set (inserted + setmask).
      const int bit = (int)((id[0] >> a.t0) & 1ull);
      const T dr = a.m[2 * bit], di = a.m[2 * bit + 1];
      C o;
      o.x = dr * v[0].x - di * v[0].y;
      o.y = dr * v[0].y + di * v[0].x;
      s[id[0]] = o;
    } else {  // DENSE2
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        T ore = 0, oim = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const T mr = a.m[2 * (4 * r + c)], mi = a.m[2 * (4 * r + c) + 1];
          ore += mr * v[c].x - mi * v[c].y;
          oim += mr * v[c].y + mi * v[c].x;
        }
        C o;
        o.x = ore;
        o.y = oim;
        s[id[r]] = o;
      }
    }
  }
};

// Grid-stride loop, U items per thread per iteration (items j + u*stride:
// consecutive lanes stay on consecutive indices), all U items' loads issued
// before their stores -- U x the bytes in flight per thread.
template <typename T, int KIND>
__global__ void __launch_bounds__(256) gate_kernel(typename CT<T>::type* __restrict__ s,
                                                   const GateArgs<T> a) {
  constexpr int U = KIND == (int)GK::DENSE2 ? 2 : 4;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; j + (U - 1) * stride < a.count; j += U * stride) {
    Item<T, KIND> it[U];
#pragma unroll
    for (int u = 0; u < U; ++u) it[u].load(s, a, j + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) it[u].store(s, a);
  }
  for (; j < a.count; j += stride) {  // tail
    Item<T, KIND> it;
    it.load(s, a, j);
    it.store(s, a);
  }
}

// Generic gate on K = 3..4 targets: one thread per group of 2^K amplitudes
// (zero bits inserted at the sorted target + control positions, control
// values OR-ed in), 2^K x 2^K complex matvec with the matrix read
// from parameter space (uniform operands), loads of a group before its stores.
template <typename T, int K>
__global__ void __launch_bounds__(128) gate_kernel_k(typename CT<T>::type* __restrict__ s,
                                                     const __grid_constant__ GateArgsK<T> a) {
  using C = typename CT<T>::type;
  constexpr int D = 1 << K;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < a.count; j += stride) {
    uint64_t x = j;
    for (int i = 0; i < a.nins; ++i) x = insert0(x, a.ins[i]);
    x |= a.setmask;
    uint64_t id[D];
    C v[D];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      uint64_t y = x;
#pragma unroll
      for (int t = 0; t < K; ++t)
        if ((c >> (K - 1 - t)) & 1) y |= 1ull << a.tpos[t];
      id[c] = y;
      v[c] = s[y];
    }
#pragma unroll
    for (int r = 0; r < D; ++r) {
      T ore = 0, oim = 0;
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const T mr = a.m[2 * (D * r + c)], mi = a.m[2 * (D * r + c) + 1];
        ore = fma(mr, v[c].x, ore);
        ore = fma(-mi, v[c].y, ore);
        oim = fma(mr, v[c].y, oim);
        oim = fma(mi, v[c].x, oim);
      }
      C o;
      o.x = ore;
      o.y = oim;
      s[id[r]] = o;
    }
  }
}

template <typename T>
int launch_gate_k(void* state, int n, const PGate& g, cudaStream_t st) {
  GateArgsK<T> a{};
  const uint64_t ins = g.cmask | pgate_targets(g);
  a.nins = 0;
  for (int p = 0; p < n; ++p)
    if (ins & (1ull << p)) a.ins[a.nins++] = p;
  a.count = 1ull << (n - a.nins);
  a.setmask = g.cval;
  a.k = g.nt;
  for (int t = 0; t < g.nt; ++t) a.tpos[t] = g.tk[t];
  const size_t d2 = (size_t)1 << (2 * g.nt);
  for (size_t i = 0; i < d2; ++i) {
    a.m[2 * i] = (T)(*g.mk)[i].real();
    a.m[2 * i + 1] = (T)(*g.mk)[i].imag();
  }
  using C = typename CT<T>::type;
  C* s = reinterpret_cast<C*>(state);
  const int threads = 128;
  uint64_t blocks = (a.count + threads - 1) / threads;
  const uint64_t cap = (uint64_t)sm_count() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  if (g.nt == 3) gate_kernel_k<T, 3><<<(unsigned)blocks, threads, 0, st>>>(s, a);
  else gate_kernel_k<T, 4><<<(unsigned)blocks, threads, 0, st>>>(s, a);
  return (int)cudaGetLastError();
}

template <typename T>
int launch_gate_t(void* state, int n, const PGate& g, cudaStream_t st) {
  if (g.kind == GK::DENSEK) return launch_gate_k<T>(state, n, g, st);
  GateArgs<T> a{};
  uint64_t ins = g.cmask;
  int nt = 0;
  if (g.kind == GK::DENSE2 || g.kind == GK::SWAP2) {
    ins |= (1ull << g.t0) | (1ull << g.t1);
    nt = 2;
  } else if (g.kind == GK::DIAG1 && !g.d0_is_one) {
    nt = 0;  // every amplitude (with matching controls) is scaled
  } else {
    ins |= 1ull << g.t0;
    nt = 1;
  }
  a.nins = 0;
  for (int p = 0; p < n; ++p)
    if (ins & (1ull << p)) a.ins[a.nins++] = p;
  const int nbits_fixed = a.nins;
  (void)nt;
  a.count = 1ull << (n - nbits_fixed);
  a.setmask = g.cval;
  if (g.kind == GK::DIAG1 && g.d0_is_one) a.setmask |= 1ull << g.t0;
  a.t0 = g.t0;
  a.t1 = g.t1;
  a.d0_is_one = g.d0_is_one ? 1 : 0;
  const int nm = (g.kind == GK::DENSE2) ? 16 : 4;
  for (int i = 0; i < nm; ++i) {
    a.m[2 * i] = (T)g.m[i].real();
    a.m[2 * i + 1] = (T)g.m[i].imag();
  }
  using C = typename CT<T>::type;
  C* s = reinterpret_cast<C*>(state);
  const int threads = 256;
  uint64_t blocks = (a.count + threads - 1) / threads;
  const uint64_t cap = (uint64_t)sm_count() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  switch (g.kind) {
    case GK::DENSE1: gate_kernel<T, 0><<<(unsigned)blocks, threads, 0, st>>>(s, a); break;
    case GK::PERM1: gate_kernel<T, 1><<<(unsigned)blocks, threads, 0, st>>>(s, a); break;
    case GK::DIAG1: gate_kernel<T, 2><<<(unsigned)blocks, threads, 0, st>>>(s, a); break;
    case GK::DENSE2: gate_kernel<T, 3><<<(unsigned)blocks, threads, 0, st>>>(s, a); break;
    case GK::SWAP2: gate_kernel<T, 4><<<(unsigned)blocks, threads, 0, st>>>(s, a); break;
  }
  return (int)cudaGetLastError();
}

}  // namespace

int sm_count() {
  static int cached = 0;
  if (!cached) {
    int dev = 0;
    cudaGetDevice(&dev);
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    cached = v;
  }
  return cached;
}

int launch_gate(void* state, int n, bool dbl, const PGate& g, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  return dbl ? launch_gate_t<double>(state, n, g, st) : launch_gate_t<float>(state, n, g, st);
}

}  // namespace qc
