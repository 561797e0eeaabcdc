// Measurement / synthetic-input helpers (include/tdes_bench.h).  No cipher
// arithmetic lives here.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/tdes_bench.h"
#include "tdes_error.h"

namespace {

int fail(cudaError_t e) { return tdes_internal::cuda_fail(e); }

int grid_for(size_t n, int threads) {
  size_t g = (n + threads - 1) / threads;
  const size_t cap = 148u * 32u;
  return (int)(g < cap ? (g ? g : 1) : cap);
}

__global__ void splitmix_kernel(uint64_t* out, size_t n, uint64_t first, uint64_t seed) {
  for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (size_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + (first + j + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    out[j] = z ^ (z >> 31);
  }
}

__global__ void sum64_kernel(const uint64_t* in, size_t n, unsigned long long* res) {
  unsigned long long acc = 0;
  for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (size_t)gridDim.x * blockDim.x)
    acc += in[j];
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(res, acc);
}

__global__ void mismatch_kernel(const uint64_t* a, const uint64_t* b, size_t n,
                                unsigned long long* res) {
  unsigned long long acc = 0;
  for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (size_t)gridDim.x * blockDim.x)
    acc += a[j] != b[j];
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(res, acc);
}

template <unsigned LUT>
__device__ __forceinline__ uint32_t lop3v(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm volatile("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
  return d;
}

// 16 independent LOP3 chains per thread; each iteration issues exactly 16
// LOP3 whose inputs are the previous iteration's results (volatile asm, so
// ptxas cannot fuse or drop them).
__global__ void __launch_bounds__(256) lop3_peak_kernel(uint32_t* sink, int iters) {
  uint32_t x[16];
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = t * (2 * k + 1) + 0x9E3779B9u * k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = lop3v<0x96>(x[k], x[(k + 1) & 15], x[(k + 5) & 15]);
  }
  uint32_t r = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) r ^= x[k];
  sink[t] = r;
}

}  // namespace

extern "C" int tdes_fill_splitmix64(void* dev_out, size_t nblocks, uint64_t first_index,
                                    uint64_t seed, tdes_stream_t stream) {
  if (nblocks == 0) return TDES_OK;
  if (!dev_out) return TDES_ERR_INVALID_ARG;
  if ((uintptr_t)dev_out & 7u) return TDES_ERR_MISALIGNED;
  splitmix_kernel<<<grid_for(nblocks, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<uint64_t*>(dev_out), nblocks, first_index, seed);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TDES_OK : fail(e);
}

extern "C" int tdes_sum64(const void* dev_in, size_t nblocks, uint64_t* dev_result,
                          tdes_stream_t stream) {
  if (!dev_result) return TDES_ERR_INVALID_ARG;
  if (nblocks == 0) return TDES_OK;
  if (!dev_in) return TDES_ERR_INVALID_ARG;
  if ((uintptr_t)dev_in & 7u) return TDES_ERR_MISALIGNED;
  sum64_kernel<<<grid_for(nblocks, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint64_t*>(dev_in), nblocks,
      reinterpret_cast<unsigned long long*>(dev_result));
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TDES_OK : fail(e);
}

extern "C" int tdes_count_mismatch(const void* a, const void* b, size_t nblocks, uint64_t* dev_count,
                                   tdes_stream_t stream) {
  if (!dev_count) return TDES_ERR_INVALID_ARG;
  if (nblocks == 0) return TDES_OK;
  if (!a || !b) return TDES_ERR_INVALID_ARG;
  if (((uintptr_t)a | (uintptr_t)b) & 7u) return TDES_ERR_MISALIGNED;
  mismatch_kernel<<<grid_for(nblocks, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint64_t*>(a), static_cast<const uint64_t*>(b), nblocks,
      reinterpret_cast<unsigned long long*>(dev_count));
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TDES_OK : fail(e);
}

extern "C" int tdes_lop3_peak(uint32_t* dev_sink, int grid, int cta, int iters, uint64_t* ops_out,
                              tdes_stream_t stream) {
  if (!dev_sink || grid <= 0 || cta <= 0 || cta > 256 || iters <= 0) return TDES_ERR_INVALID_ARG;
  lop3_peak_kernel<<<grid, cta, 0, reinterpret_cast<cudaStream_t>(stream)>>>(dev_sink, iters);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(e);
  if (ops_out) *ops_out = (uint64_t)grid * (uint64_t)cta * (uint64_t)iters * 16u;
  return TDES_OK;
}
