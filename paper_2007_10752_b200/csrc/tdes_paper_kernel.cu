// The paper's own GPU design (§IV) on sm_100a -- SURVEY
// NEXT-3: a like-for-like baseline that quantifies the bitsliced kernel
// against the paper's bit-per-thread decomposition on the same B200.  Not the
// product path; exposed as tdes_paper_ecb() for comparison and tested for
// parity like everything else.
//
//   key kernel   3 CTAs x 56 threads, one thread per permuted key bit:
//                PC-1 in parallel, 16 serial rounds of {2 threads rotate the
//                halves, 48 threads apply PC-2}.
//   crypt kernel one 64-thread CTA per 64-bit block, one thread per bit, one
//                char per bit in shared memory:
//                IP in parallel; per round 48 threads E + key XOR, 8 groups x
//                4 threads S-boxes (one reads the table, four write bits),
//                32 threads P, 32 threads XOR, swap; FP in parallel.
//   3DES         three launches E(K1), D(K2), E(K3); D reverses the key
//                order.
// Tables live in the read-only path (__ldg of __device__ arrays); the
// shift table in __constant__ memory (uniform access).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/tdes_paper.h"
#include "tdes_error.h"

namespace {

// Tables for the device, from the generated product tables (tools/des_tables.py);
// c_shifts is statically initialised at module load, so calls never write shared state.
#include "gen/tdes_paper_tables.cuh"


__global__ void __launch_bounds__(64) paper_keygen_kernel(const uint8_t* keys /*3x8*/,
                                                          uint8_t* subkeys /*3x16x48*/) {
  __shared__ uint8_t key[64], cd[56], tmp[56];
  const int k = blockIdx.x, t = threadIdx.x;
  if (t < 64) key[t] = (keys[8 * k + t / 8] >> (7 - t % 8)) & 1;  // char per bit
  __syncthreads();
  if (t < 56) cd[t] = key[__ldg(&d_pc1[t]) - 1];                 // PC-1, one thread per bit
  __syncthreads();
  for (int r = 0; r < 16; ++r) {                                  // serial over rounds
    const int s = c_shifts[r];
    if (t < 2) {                                                  // two threads rotate the halves
      for (int i = 0; i < 28; ++i) tmp[28 * t + i] = cd[28 * t + (i + s) % 28];
      for (int i = 0; i < 28; ++i) cd[28 * t + i] = tmp[28 * t + i];
    }
    __syncthreads();
    if (t < 48) subkeys[(k * 16 + r) * 48 + t] = cd[__ldg(&d_pc2[t]) - 1];  // PC-2
    __syncthreads();
  }
}

__global__ void __launch_bounds__(64) paper_crypt_kernel(const uint8_t* in, uint8_t* out,
                                                         const uint8_t* ks /*16x48*/, int decrypt) {
  __shared__ uint8_t blk[64], v[64], L[32], R[32], e[48], sb[32], f[32], nr[32];
  const int t = threadIdx.x;
  const size_t b = blockIdx.x;
  blk[t] = (in[8 * b + t / 8] >> (7 - t % 8)) & 1;                // block -> chars in smem
  __syncthreads();
  v[t] = blk[__ldg(&d_ip[t]) - 1];                                // IP in parallel
  __syncthreads();
  if (t < 32) L[t] = v[t];
  else R[t - 32] = v[t];                                          // split
  __syncthreads();
  for (int r = 0; r < 16; ++r) {
    const uint8_t* k = ks + 48 * (decrypt ? 15 - r : r);          // reversed for decryption
    if (t < 48) e[t] = R[__ldg(&d_e[t]) - 1] ^ __ldg(&k[t]);     // E + key XOR
    __syncthreads();
    if (t < 32) {                                                 // 8 groups x 4 threads
      const int g = t >> 2, j = t & 3;
      const uint8_t* x = e + 6 * g;
      const int row = 2 * x[0] + x[5], col = 8 * x[1] + 4 * x[2] + 2 * x[3] + x[4];
      const int val = __ldg(&d_sbox[g * 64 + row * 16 + col]);
      sb[4 * g + j] = (val >> (3 - j)) & 1;
    }
    __syncthreads();
    if (t < 32) f[t] = sb[__ldg(&d_p[t]) - 1];                    // P
    __syncthreads();
    if (t < 32) nr[t] = L[t] ^ f[t];                              // XOR with left
    __syncthreads();
    if (t < 32) {                                                 // swap
      L[t] = R[t];
      R[t] = nr[t];
    }
    __syncthreads();
  }
  v[t] = t < 32 ? R[t] : L[t - 32];                               // combine R16||L16
  __syncthreads();
  blk[t] = v[__ldg(&d_fp[t]) - 1];                                // FP
  __syncthreads();
  if (t < 8) {
    uint8_t byte = 0;
    for (int i = 0; i < 8; ++i) byte = (uint8_t)((byte << 1) | blk[8 * t + i]);
    out[8 * b + t] = byte;
  }
}

int fail(cudaError_t e) { return tdes_internal::cuda_fail(e); }

}  // namespace

extern "C" int tdes_paper_ecb(const uint8_t* dev_keys, const void* in, void* out, size_t nblocks,
                              int decrypt, void* workspace, size_t workspace_bytes,
                              tdes_stream_t stream) {
  if (!dev_keys || (decrypt != 0 && decrypt != 1)) return TDES_ERR_INVALID_ARG;
  if (!workspace || workspace_bytes < 3 * 16 * 48) return TDES_ERR_WORKSPACE;
  if (nblocks == 0) return TDES_OK;
  if (!in || !out) return TDES_ERR_INVALID_ARG;
  if (nblocks > 0x7FFFFFFFu) return TDES_ERR_INVALID_ARG;  // one CTA per block (grid.x limit)
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* sk = static_cast<uint8_t*>(workspace);
  paper_keygen_kernel<<<3, 64, 0, st>>>(dev_keys, sk);
  const uint8_t* K[3] = {sk, sk + 16 * 48, sk + 2 * 16 * 48};
  const unsigned grid = (unsigned)nblocks;
  // E_K1 D_K2 E_K3 or D_K3 E_K2 D_K1: three launches
  const int order_enc[3] = {0, 1, 2}, order_dec[3] = {2, 1, 0};
  const int* order = decrypt ? order_dec : order_enc;
  for (int s = 0; s < 3; ++s) {
    const int dir = (s == 1) ^ decrypt;
    paper_crypt_kernel<<<grid, 64, 0, st>>>(s == 0 ? static_cast<const uint8_t*>(in)
                                                   : static_cast<const uint8_t*>(out),
                                            static_cast<uint8_t*>(out), K[order[s]], dir);
  }
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TDES_OK : fail(e);
}
