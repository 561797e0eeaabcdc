// Experiment build (not the product): instrumented / dynamically scheduled
// variants of the 3DES kernel to study per-warp progress on long launches.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../paper_2007_10752_b200/csrc/gen/tdes_gen.cuh"

namespace {
constexpr int kThreads = 256;
constexpr int kTile = 1024;

struct RM {
  uint32_t s[48][48];
  uint32_t k[48][48];
};

__device__ __forceinline__ void transpose32(uint32_t (&a)[32]) {
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const uint32_t lo = a[k], hi = a[k + 16];
    a[k] = __byte_perm(lo, hi, 0x5410);
    a[k + 16] = __byte_perm(lo, hi, 0x7632);
  }
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    if (k & 8) continue;
    const uint32_t lo = a[k], hi = a[k + 8];
    a[k] = __byte_perm(lo, hi, 0x6240);
    a[k + 8] = __byte_perm(lo, hi, 0x7351);
  }
#pragma unroll
  for (int s = 4; s >= 1; s >>= 1) {
    const uint32_t m = s == 4 ? 0x0F0F0F0Fu : s == 2 ? 0x33333333u : 0x55555555u;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (k & s) continue;
      const uint32_t lo = a[k], hi = a[k + s];
      a[k] = tdes_gen::lop3<0xCA>(m, lo, hi << s);
      a[k + s] = tdes_gen::lop3<0xCA>(m, lo >> s, hi);
    }
  }
}

template <bool START_A>
__device__ __forceinline__ void stage(uint32_t (&P)[64], const RM& mk, int r0) {
#pragma unroll 1
  for (int r = r0; r < r0 + 16; r += 2) {
    if (START_A) {
      tdes_gen::round_A<false>(P, mk.s[r], mk.k[r], 0u);
      tdes_gen::round_B<false>(P, mk.s[r + 1], mk.k[r + 1], 0u);
    } else {
      tdes_gen::round_B<false>(P, mk.s[r], mk.k[r], 0u);
      tdes_gen::round_A<false>(P, mk.s[r + 1], mk.k[r + 1], 0u);
    }
  }
}

__device__ __forceinline__ void do_tile(const uint4* in4, uint4* out4, unsigned lane, const RM& mk) {
  uint32_t X[32], Y[32];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint4 v = __ldcs(in4 + 32 * i + lane);
    X[2 * i] = v.x; Y[2 * i] = v.y; X[2 * i + 1] = v.z; Y[2 * i + 1] = v.w;
  }
  transpose32(X);
  transpose32(Y);
  uint32_t P[64];
#pragma unroll
  for (int j = 0; j < 32; ++j) { P[j] = X[j]; P[32 + j] = Y[j]; }
  stage<true>(P, mk, 0);
  stage<false>(P, mk, 16);
  stage<true>(P, mk, 32);
  uint32_t Q[64];
  tdes_gen::output_planes(P, Q);
#pragma unroll
  for (int j = 0; j < 32; ++j) { X[j] = Q[j]; Y[j] = Q[32 + j]; }
  transpose32(X);
  transpose32(Y);
#pragma unroll
  for (int i = 0; i < 16; ++i)
    __stcs(out4 + 32 * i + lane, make_uint4(X[2 * i], Y[2 * i], X[2 * i + 1], Y[2 * i + 1]));
}

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// mode 0: static grid-stride; mode 1: dynamic (atomic counter, per warp);
// mode 2: static contiguous range per CTA, warps claim tiles from a shared-memory counter
template <int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB)
exp_kernel(const uint2* in, uint2* out, size_t ntiles, const __grid_constant__ RM mk, int mode,
           unsigned long long* counter, unsigned long long* trace) {
  const unsigned lane = threadIdx.x & 31u;
  const size_t gw = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  const uint64_t t0 = gtime();
  const long long c0 = clock64();
  unsigned count = 0;
  __shared__ unsigned long long sctr;
  if (mode == 2) {
    if (threadIdx.x == 0) sctr = 0;
    __syncthreads();
    const size_t lo = ntiles * blockIdx.x / gridDim.x, hi = ntiles * (blockIdx.x + 1) / gridDim.x;
    for (;;) {
      unsigned long long t = 0;
      if (lane == 0) t = atomicAdd(&sctr, 1ull);
      t = __shfl_sync(0xffffffffu, t, 0) + lo;
      if (t >= hi) break;
      do_tile(reinterpret_cast<const uint4*>(in + t * kTile), reinterpret_cast<uint4*>(out + t * kTile), lane, mk);
      ++count;
    }
  } else if (mode == 0) {
    for (size_t tile = gw; tile < ntiles; tile += nwarps, ++count)
      do_tile(reinterpret_cast<const uint4*>(in + tile * kTile), reinterpret_cast<uint4*>(out + tile * kTile), lane, mk);
  } else {
    for (;;) {
      unsigned long long t = 0;
      if (lane == 0) t = atomicAdd(counter, 1ull);
      t = __shfl_sync(0xffffffffu, t, 0);
      if (t >= ntiles) break;
      do_tile(reinterpret_cast<const uint4*>(in + t * kTile), reinterpret_cast<uint4*>(out + t * kTile), lane, mk);
      ++count;
    }
  }
  const uint64_t t1 = gtime();
  const long long c1 = clock64();
  if (lane == 0 && trace) {
    trace[4 * gw + 0] = t0;
    trace[4 * gw + 1] = t1;
    trace[4 * gw + 2] = (unsigned long long)(c1 - c0);
    trace[4 * gw + 3] = ((unsigned long long)smid << 32) | count | ((unsigned long long)(threadIdx.x >> 5) << 48);
  }
}
}  // namespace

extern "C" int exp_launch(const uint32_t* masks /*48*48*/, const void* in, void* out, size_t ntiles,
                          int grid, int mode, unsigned long long* counter,
                          unsigned long long* trace, void* stream) {
  static RM mk;
  for (int r = 0; r < 48; ++r)
    for (int b = 0; b < 48; ++b) {
      const uint32_t m = masks[48 * r + b] ? 0xFFFFFFFFu : 0u;
      mk.k[r][b] = m;
      mk.s[r][b] = m | 1u;
    }
  if (mode >= 2)
    exp_kernel<512, 1><<<grid, 512, 0, (cudaStream_t)stream>>>((const uint2*)in, (uint2*)out, ntiles, mk,
                                                              mode - 1, counter, trace);
  else
    exp_kernel<256, 2><<<grid, 256, 0, (cudaStream_t)stream>>>((const uint2*)in, (uint2*)out, ntiles, mk,
                                                              mode, counter, trace);
  return (int)cudaGetLastError();
}
