// kernels_util.cu -- state initialisation, canonical-order gather/scatter,
// norm reduction.  Not on the timed circuit path.
#include <cuda_runtime.h>

#include <cmath>

#include "qc_internal.h"

namespace qc {
namespace {

struct Layout {
  int8_t pos[64];  // pos[q] = physical bit of logical qubit q
};

__device__ __forceinline__ uint64_t splitmix64(uint64_t seed, uint64_t ctr) {
  // Counter-based splitmix64 (DESIGN input recipe; same stream as qcgen).
  uint64_t z = seed + (ctr + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double u_pm1(uint64_t x) {
  // (x>>11) * 2^-52 - 1: both steps exact.
  return __dsub_rn(__dmul_rn((double)(x >> 11), 0x1p-52), 1.0);
}

// Amplitude j of the buffer is global amplitude first + j.
template <typename C>
__global__ void init_random_kernel(C* s, uint64_t N, uint64_t first, uint64_t seed, double scale);

template <>
__global__ void init_random_kernel<double2>(double2* s, uint64_t N, uint64_t first, uint64_t seed,
                                            double scale) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += stride) {
    const uint64_t i = first + j;
    double2 v;
    v.x = __dmul_rn(u_pm1(splitmix64(seed, 2 * i)), scale);
    v.y = __dmul_rn(u_pm1(splitmix64(seed, 2 * i + 1)), scale);
    s[j] = v;
  }
}

template <>
__global__ void init_random_kernel<float2>(float2* s, uint64_t N, uint64_t first, uint64_t seed,
                                           double scale) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += stride) {
    const uint64_t i = first + j;
    float2 v;
    v.x = __double2float_rn(__dmul_rn(u_pm1(splitmix64(seed, 2 * i)), scale));
    v.y = __double2float_rn(__dmul_rn(u_pm1(splitmix64(seed, 2 * i + 1)), scale));
    s[j] = v;
  }
}

// Swap two equal, disjoint device ranges (loopback exchange), 16-byte units.
// Swap two equal regions (16-B words).  4 words of each region per thread in
// flight (all 8 loads before the stores): the exchange's peer region is read
// and written over NVLink, whose latency needs the extra bytes in flight.
__global__ void swap_regions_kernel(uint4* __restrict__ a, uint4* __restrict__ b, uint64_t n16) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; j + 3 * stride < n16; j += 4 * stride) {
    uint4 x[4], y[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x[u] = a[j + u * stride];
      y[u] = b[j + u * stride];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[j + u * stride] = y[u];
      b[j + u * stride] = x[u];
    }
  }
  for (; j < n16; j += stride) {
    const uint4 x = a[j], y = b[j];
    a[j] = y;
    b[j] = x;
  }
}

template <typename C>
__global__ void set_one_kernel(C* s, uint64_t k) {
  C v;
  v.x = 1;
  v.y = 0;
  s[k] = v;
}

__device__ __forceinline__ uint64_t canon_to_phys(uint64_t i, int n, const Layout& L) {
  uint64_t p = 0;
  for (int q = 0; q < n; ++q) p |= ((i >> (n - 1 - q)) & 1ull) << L.pos[q];
  return p;
}

template <typename C>
__global__ void gather_kernel(const C* __restrict__ s, C* __restrict__ dst, int n, Layout L,
                              uint64_t first, uint64_t count, int scatter) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += stride) {
    const uint64_t p = canon_to_phys(first + j, n, L);
    if (scatter)
      const_cast<C*>(s)[p] = dst[j];
    else
      dst[j] = s[p];
  }
}

template <typename C>
__global__ void norm2_kernel(const C* __restrict__ s, uint64_t N, double* partial) {
  double acc = 0.0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride) {
    const C v = s[i];
    acc += (double)v.x * (double)v.x + (double)v.y * (double)v.y;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    partial[blockIdx.x] = t;
  }
}

unsigned blocks_for(uint64_t count, int threads) {
  uint64_t b = (count + threads - 1) / threads;
  const uint64_t cap = (uint64_t)sm_count() * 8;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}

}  // namespace

int launch_init_random(void* state, int n, bool dbl, uint64_t seed, void* stream, uint64_t first,
                       uint64_t count) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const uint64_t N = count ? count : (1ull << n);
  const double scale = std::sqrt(1.5 / (double)(1ull << n));  // normalisation of the global state
  if (dbl)
    init_random_kernel<double2><<<blocks_for(N, 256), 256, 0, st>>>((double2*)state, N, first, seed, scale);
  else
    init_random_kernel<float2><<<blocks_for(N, 256), 256, 0, st>>>((float2*)state, N, first, seed, scale);
  return (int)cudaGetLastError();
}

int launch_swap_regions(void* a, void* b, uint64_t bytes, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const uint64_t n16 = bytes / 16;
  const uint64_t cap = (uint64_t)sm_count() * 8;  // 8 x 256 threads per SM, grid-stride
  uint64_t blocks = blocks_for((n16 + 3) / 4, 256);
  if (blocks > cap) blocks = cap;
  swap_regions_kernel<<<(unsigned)blocks, 256, 0, st>>>((uint4*)a, (uint4*)b, n16);
  return (int)cudaGetLastError();
}

int launch_init_basis(void* state, int n, bool dbl, uint64_t k, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t bytes = (size_t)(dbl ? 16 : 8) << n;
  cudaError_t e = cudaMemsetAsync(state, 0, bytes, st);
  if (e != cudaSuccess) return (int)e;
  if (dbl)
    set_one_kernel<double2><<<1, 1, 0, st>>>((double2*)state, k);
  else
    set_one_kernel<float2><<<1, 1, 0, st>>>((float2*)state, k);
  return (int)cudaGetLastError();
}

int launch_gather(const void* state, void* dst, int n, bool dbl, const int* layout,
                  uint64_t first, uint64_t count, bool scatter, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Layout L{};
  for (int q = 0; q < n; ++q) L.pos[q] = (int8_t)layout[q];
  if (dbl)
    gather_kernel<double2><<<blocks_for(count, 256), 256, 0, st>>>(
        (const double2*)state, (double2*)dst, n, L, first, count, scatter ? 1 : 0);
  else
    gather_kernel<float2><<<blocks_for(count, 256), 256, 0, st>>>(
        (const float2*)state, (float2*)dst, n, L, first, count, scatter ? 1 : 0);
  return (int)cudaGetLastError();
}

int launch_norm2(const void* state, int n, bool dbl, double* d_partial, int nblocks,
                 void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const uint64_t N = 1ull << n;
  if (dbl)
    norm2_kernel<double2><<<nblocks, 256, 0, st>>>((const double2*)state, N, d_partial);
  else
    norm2_kernel<float2><<<nblocks, 256, 0, st>>>((const float2*)state, N, d_partial);
  return (int)cudaGetLastError();
}

}  // namespace qc

// ---------------------------------------------------------------- FMA peak
// Measurement utility (qc_debug_fma_peak): 8 independent FMA chains per
// thread, so the FP64 / FP32 pipe -- not latency -- bounds the loop.
namespace qc {
template <typename T>
__global__ void fma_peak_kernel(T* out, int iters, T a, T b) {
  T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  const T s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == (T)-1.2345) out[0] = s;  // keep the chains live
}

int fma_peak(bool dbl, double* tflops) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  void* out = nullptr;
  cudaError_t e = cudaMalloc(&out, 64);
  if (e != cudaSuccess) return (int)e;
  const int blocks = sms * 4, threads = 512, iters = dbl ? 1024 : 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(a);
    if (dbl)
      fma_peak_kernel<double><<<blocks, threads>>>((double*)out, iters, 0.999999, 1e-7);
    else
      fma_peak_kernel<float><<<blocks, threads>>>((float*)out, iters, 0.999f, 1e-3f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (rep > 0 && ms < best) best = ms;
  }
  e = cudaGetLastError();
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  const double flops = 2.0 * 64.0 * (double)iters * threads * blocks;
  *tflops = flops / (best * 1e-3) / 1e12;
  return (int)e;
}
}  // namespace qc
