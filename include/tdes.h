/*
 * tdes.h -- C ABI of the B200 (sm_100a) bitsliced 3DES-EDE ECB library.
 *
 * The boundary follows the paper's statement of the problem (arXiv 2007.10752,
 * /root/reference/PAPER.md, cited as P:<line>):
 *   - key generation takes the 3 base keys and outputs 3x16 round keys of 48
 *     bits (§IV.A; algorithm §III.A);
 *   - the encrypt/decrypt step takes "the plaintext, subkeys, and mode" (P:109,
 *     §IV.B) and computes C = E_K3(D_K2(E_K1(P))) or P = D_K1(E_K2(D_K3(C)))
 *     (§III.B) on every 64-bit block independently -- ECB.
 * The schedule is an explicit, caller-owned argument (no hidden global state);
 * the mode is the choice of entry point.
 *
 * Conventions
 *   - A block is 8 bytes; FIPS bit 1 is the most significant bit of byte 0
 *     (reading Q1).  Block i occupies bytes 8i..8i+7.  Keys are 8 raw
 *     bytes in the same order; parity bits (FIPS bits 8,16,...,64) are ignored
 *     (PC-1 never reads them).
 *   - Whole blocks only: there is no padding ("consisting of 64-bit
 *     blocks").  Lengths are counts of blocks (size_t, 64-bit indexing).
 *   - Return values: 0 = TDES_OK, otherwise a negative TDES_ERR_* code.  No C++
 *     exception crosses this boundary.  All functions are thread-safe and
 *     re-entrant; the library keeps no shared mutable state apart from a
 *     per-device launch-geometry cache (written once per device, atomically),
 *     and each host thread caches the launch operands of the last two key
 *     schedules it used (thread-local, keyed by the schedule's contents, so a
 *     caller may reuse or modify a tdes_schedule freely).
 */
#ifndef TDES_H_
#define TDES_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Opaque CUDA stream handle (cudaStream_t / CUstream); NULL = legacy default stream. */
typedef struct CUstream_st *tdes_stream_t;

#define TDES_OK 0
#define TDES_ERR_INVALID_ARG (-1) /* NULL schedule/key/pointer with nblocks > 0, bad enum,
                                     nblocks > SIZE_MAX/16; TDES_DEBUG builds also: in/out
                                     not device memory of the current device            */
#define TDES_ERR_MISALIGNED (-2)  /* in or out not 8-byte aligned                        */
#define TDES_ERR_OVERLAP (-3)     /* in and out partially overlap (in == out is allowed)  */
#define TDES_ERR_CUDA (-4)        /* a CUDA call failed; see tdes_last_cuda_error()       */
#define TDES_ERR_WORKSPACE (-5)   /* host-pipeline workspace too small                   */

/*
 * Key schedule of one 3DES key triple (§III.A, run once per base key).
 *
 *   subkey[k][r]  48-bit round key r+1 of base key k+1, FIPS order: subkey bit 1
 *                 is bit 47 of the integer.
 *   mask[d][s][b] the same subkeys expanded to all-ones / all-zeros lane masks
 *                 (0xFFFFFFFF if the bit is 1) in the order the fused 48-round
 *                 kernel consumes them, d = 0 encrypt, 1 decrypt:
 *                   encrypt: K1 r1..16, K2 r16..1, K3 r1..16  (E_K1, D_K2, E_K3)
 *                   decrypt: K3 r16..1, K2 r1..16, K1 r16..1  (D_K3, E_K2, D_K1)
 *                 "D" is the same rounds with the round-key order reversed.
 *                 b is the position in the 48-bit E-expanded half (subkey bit b+1).
 * The struct is plain data in caller (host) memory; the library never retains a
 * pointer to it.
 */
typedef struct tdes_schedule {
  uint64_t subkey[3][16];
  uint32_t mask[2][48][48];
} tdes_schedule;

/* k1, k2, k3: 8 bytes each (host).  Writes *out.  Weak keys and the 2-key
 * (K1 = K3) / 1-key (K1 = K2 = K3) keying options are accepted silently.
 * Errors: TDES_ERR_INVALID_ARG on a NULL pointer. */
int tdes_key_schedule(const uint8_t k1[8], const uint8_t k2[8], const uint8_t k3[8],
                      tdes_schedule *out);

/*
 * 3DES-EDE ECB encrypt / decrypt of nblocks blocks, device to
 * device, enqueued on `stream` (asynchronous; kernel faults surface at the
 * caller's next synchronize).
 *   s       host pointer to a schedule from tdes_key_schedule; what the kernel
 *           needs of it is copied into the launch parameters (the 48 packed
 *           subkeys, which each CTA expands into its key operands on the device,
 *           plus the uniform-path s operands), so *s may be freed or changed as
 *           soon as the call returns.
 * Kernel choice (automatic, by launch size in 1024-block tiles): <= 384 tiles the
 * S-box-split latency kernel, above that the throughput kernel (tdes_ecb_crypt_mode
 * in tdes_bench.h forces one).  All produce identical output.
 *   in,out  device pointers (current device), 8-byte aligned; in == out (in
 *           place) is allowed, any other overlap is TDES_ERR_OVERLAP.  16-byte
 *           alignment of both selects 128-bit loads/stores.
 *   nblocks number of 8-byte blocks; 0 returns TDES_OK without a launch.
 * The library allocates nothing and never synchronizes.
 * Errors (checked in this order, nothing is launched on an error):
 *   TDES_ERR_INVALID_ARG  s, in or out NULL (nblocks > 0), nblocks > SIZE_MAX/16;
 *                         in a TDES_DEBUG build (libtdes_b200_debug.so) also in or
 *                         out not device (or managed) memory of the current device
 *                         per cudaPointerGetAttributes -- release builds do not
 *                         make that driver call and a host pointer faults in the
 *                         kernel instead (reported at the next synchronize);
 *   TDES_ERR_MISALIGNED   in or out not 8-byte aligned;
 *   TDES_ERR_OVERLAP      in != out and the ranges overlap;
 *   TDES_ERR_CUDA         cudaGetDevice or the launch failed (tdes_last_cuda_error). 
 */
int tdes_ecb_encrypt(const tdes_schedule *s, const void *in, void *out, size_t nblocks,
                     tdes_stream_t stream);
int tdes_ecb_decrypt(const tdes_schedule *s, const void *in, void *out, size_t nblocks,
                     tdes_stream_t stream);

/*
 * Single DES (the K1 = K2 = K3 degenerate case, run as 16 rounds instead
 * of 48).  A separate entry point so that its 3x throughput is never reported
 * as 3DES.  des_schedule holds the 16 masks of one key in encrypt order
 * (mask[0]) and decrypt order (mask[1]).
 */
typedef struct des_schedule {
  uint64_t subkey[16];
  uint32_t mask[2][16][48];
} des_schedule;

int des_key_schedule(const uint8_t k[8], des_schedule *out);
int des_ecb_encrypt(const des_schedule *s, const void *in, void *out, size_t nblocks,
                    tdes_stream_t stream);
int des_ecb_decrypt(const des_schedule *s, const void *in, void *out, size_t nblocks,
                    tdes_stream_t stream);

/*
 * End-to-end host -> device -> host 3DES ECB (the paper's flow: "CPU sends the
 * plaintext ... to the global memory of the GPU").  Splits the input
 * into chunks of chunk_blocks, and round-robins them over nstreams caller
 * streams: per chunk, H2D copy, kernel, D2H copy on one stream, so copies of
 * one chunk overlap the kernel of another.  Blocks until the result is in
 * host_out (it synchronizes the given streams).
 *   host_in/host_out  host buffers (pinned for copy/compute overlap); may alias.
 *   workspace         device buffer of >= nstreams * chunk_blocks * 8 bytes,
 *                     16-byte aligned (the chunks then take the 128-bit path).
 *   chunk_blocks      blocks per chunk, even (> 0).
 *   decrypt           0 = encrypt, 1 = decrypt.
 * Errors: TDES_ERR_INVALID_ARG, TDES_ERR_MISALIGNED (workspace not 16-byte
 * aligned or chunk_blocks odd), TDES_ERR_WORKSPACE, TDES_ERR_CUDA.
 */
int tdes_ecb_crypt_host(const tdes_schedule *s, int decrypt, const void *host_in, void *host_out,
                        size_t nblocks, void *workspace, size_t workspace_bytes,
                        size_t chunk_blocks, const tdes_stream_t *streams, int nstreams);

/* Static description of the compiled kernel (for roofline accounting).
 *   sbox_lop3_total  T = LOP3 gates over the 8 S-box circuits (one round)
 *   threads_per_cta, blocks_per_thread, min_ctas_per_sm: launch shape. */
typedef struct tdes_kernel_info {
  int sbox_lop3_total;
  int sbox_lop3[8];
  int threads_per_cta;
  int blocks_per_thread;
  int min_ctas_per_sm;
} tdes_kernel_info;
int tdes_get_kernel_info(tdes_kernel_info *out);

/* Human-readable text of a TDES_ERR_* code (static storage). */
const char *tdes_strerror(int code);

/* cudaError_t of the last TDES_ERR_CUDA returned on this host thread by any
 * entry point of the library (tdes.h, tdes_bench.h, tdes_paper.h); 0 if none. */
int tdes_last_cuda_error(void);

#ifdef __cplusplus
}
#endif
#endif /* TDES_H_ */
