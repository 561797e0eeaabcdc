/*
 * tdes_paper.h -- the paper's own GPU design (arXiv 2007.10752 §IV)
 * compiled for sm_100a, kept as a like-for-like COMPARISON baseline for the
 * bitsliced product kernel.  Not the product path.
 */
#ifndef TDES_PAPER_H_
#define TDES_PAPER_H_

#include <stddef.h>
#include <stdint.h>

#include "tdes.h"

#ifdef __cplusplus
extern "C" {
#endif

/*
 * 3DES-EDE ECB with the paper's kernels: a key-generation kernel (3 CTAs x 56
 * threads) and three launches (E_K1, D_K2, E_K3 or the reverse,
 * P:122) of a crypt kernel with one 64-thread CTA per block and one char per
 * bit in shared memory.
 *   dev_keys   device pointer to 24 bytes: K1 || K2 || K3 (FIPS byte order)
 *   in, out    device buffers of nblocks 8-byte blocks (in == out allowed)
 *   decrypt    0 = encrypt, 1 = decrypt
 *   workspace  device buffer >= 2304 bytes (3 x 16 x 48 subkey chars)
 * Asynchronous on `stream`.  nblocks <= 2^31 - 1 (one CTA per block).
 * Errors: TDES_ERR_INVALID_ARG, TDES_ERR_WORKSPACE, TDES_ERR_CUDA.
 */
int tdes_paper_ecb(const uint8_t *dev_keys, const void *in, void *out, size_t nblocks,
                   int decrypt, void *workspace, size_t workspace_bytes, tdes_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* TDES_PAPER_H_ */
