/*
 * tdes_bench.h -- measurement and synthetic-input helpers of the B200 3DES
 * library.  None of these perform cipher arithmetic; they exist so that large
 * workloads are generated and checked on the device (no PCIe in the timed
 * path) and so that the roofline denominator is measured on the same GPU.
 * Same error conventions as tdes.h.
 */
#ifndef TDES_BENCH_H_
#define TDES_BENCH_H_

#include <stddef.h>
#include <stdint.h>

#include "tdes.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Fill dev_out (8-byte aligned device buffer of nblocks blocks) with the
 * synthetic plaintext of DESIGN.md "Input recipe": block j is the 8
 * little-endian bytes of splitmix64 counter (first_index + j + 1) under seed,
 *   z = seed + (i+1)*0x9E3779B97F4A7C15; z = (z^z>>30)*0xBF58476D1CE4E5B9;
 *   z = (z^z>>27)*0x94D049BB133111EB; block = z^z>>31   (all mod 2^64).
 * Same generator as synthetic/__init__.py, so shards of any world size see
 * the same global data. */
int tdes_fill_splitmix64(void *dev_out, size_t nblocks, uint64_t first_index, uint64_t seed,
                         tdes_stream_t stream);

/* *dev_result (device uint64) += sum over blocks of the little-endian uint64
 * value of each block, mod 2^64 (a mergeable digest).  Caller zeroes it. */
int tdes_sum64(const void *dev_in, size_t nblocks, uint64_t *dev_result, tdes_stream_t stream);

/* *dev_count (device uint64) += number of blocks where a and b differ. */
int tdes_count_mismatch(const void *dev_a, const void *dev_b, size_t nblocks,
                        uint64_t *dev_count, tdes_stream_t stream);

/*
 * LOP3 peak microbenchmark: grid x cta threads, each running `iters`
 * iterations of `chains` independent lop3.b32 chains (16 LOP3 per iteration
 * per thread).  Writes a data-dependent word per thread to dev_sink (grid*cta
 * uint32) so nothing is dead.  *ops_out = total LOP3 thread-instructions the
 * launch executes (for ops/s = ops / elapsed).
 */
int tdes_lop3_peak(uint32_t *dev_sink, int grid, int cta, int iters, uint64_t *ops_out,
                   tdes_stream_t stream);

/* 3DES ECB with an explicit kernel choice (for measurement and tests):
 *   mode 0  automatic (what tdes_ecb_encrypt/decrypt do: the S-box-split latency
 *           kernel for small launches, the throughput kernel otherwise)
 *   mode 1  throughput kernel (32 blocks per thread, one warp per 1024-block tile;
 *           s operands in the launch parameters, k/d expanded on the device)
 *   mode 2  S-box-split latency kernel (a team of warps per 1024-block tile: 8
 *           warps with one S-box each below 149 tiles, 4 warps with two adjacent
 *           S-boxes each from 149 tiles on)
 *   mode 3  throughput kernel with all key operands expanded on the device: the
 *           launch carries only the 48 packed 48-bit subkeys (384 B); every CTA
 *           expands them into every folded key operand, s included, in shared
 *           memory at start (NEXT-4's pure device path; slower on long launches)
 * Same arguments and errors as tdes_ecb_encrypt; decrypt 0/1. */
int tdes_ecb_crypt_mode(const tdes_schedule *s, int decrypt, const void *in, void *out,
                        size_t nblocks, int mode, tdes_stream_t stream);

/* Number of SMs of the current device and max resident CTAs/SM of the 3DES
 * kernel (its occupancy), for grid accounting. */
int tdes_device_geometry(int *num_sms, int *ctas_per_sm);

/* Host only (no GPU needed; for the CPU emulator test): the key operands the 3DES
 * throughput kernel receives for schedule s and direction decrypt (0/1), with the
 * planes' pending masks folded in (DESIGN.md §6 "mask folding").  Writes up to
 * out_words uint32 words to out, in this order:
 *   s[48][stride], k[48][stride]   combined operands of the E-positions that need
 *                                  a key IMAD (slots 0..slots-1 per round; the
 *                                  slot -> E-position map is the generator's plan)
 *   d[48][dstride]                 masks folded by the unfused outputs
 *   fix_s[3][dstride], fix_k[3][dstride]  priming of round A's free positions before
 *                                  round 0 and after the swaps at rounds 16 and 32
 *   fin_s[64], fin_k[64]           final unmasking per plane
 * and stores the total word count in *words (also when out is NULL or too small:
 * then nothing is written and TDES_ERR_WORKSPACE is returned).  *geom (if not NULL)
 * receives {slots, stride, nfree, dstride}. */
int tdes_fold_operands(const tdes_schedule *s, int decrypt, uint32_t *out, size_t out_words,
                       size_t *words, int *geom);

#ifdef __cplusplus
}
#endif
#endif /* TDES_BENCH_H_ */
