/*
 * The C ABI used from plain C (no Python, no torch): a user of include/tdes.h
 * links libtdes_b200.so and the CUDA runtime, builds a key schedule, and runs
 * 3DES-EDE ECB on device buffers.  Checks the NIST SP 800-67 example block
 * (keys 0123456789ABCDEF 23456789ABCDEF01 456789ABCDEF0123, plaintext
 * "The quic" = 5468652071756663 -> A826FD8CE53B855F; tests/golden/des_kat.txt), the
 * round trip on a ragged multi-tile buffer, in place, and the error codes of a
 * misaligned and an overlapping call.  Exit 0 = pass.
 *
 *   gcc -std=c11 -Iinclude -I/usr/local/cuda/include tests/c/abi_kat.c \
 *       -Lpaper_2007_10752_b200 -ltdes_b200 -L/usr/local/cuda/lib64 -lcudart -o abi_kat
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "tdes.h"

static int fail(const char *what, int rc) {
  fprintf(stderr, "FAIL %s: rc=%d (%s), cudaError=%d\n", what, rc, tdes_strerror(rc), tdes_last_cuda_error());
  return 1;
}

static void hex8(const char *h, uint8_t out[8]) {
  for (int i = 0; i < 8; ++i) {
    unsigned v;
    sscanf(h + 2 * i, "%2x", &v);
    out[i] = (uint8_t)v;
  }
}

int main(void) {
  uint8_t k1[8], k2[8], k3[8], pt[8], ct_exp[8];
  hex8("0123456789ABCDEF", k1);
  hex8("23456789ABCDEF01", k2);
  hex8("456789ABCDEF0123", k3);
  hex8("5468652071756663", pt);
  hex8("A826FD8CE53B855F", ct_exp);
  tdes_schedule *s = (tdes_schedule *)malloc(sizeof *s);
  int rc = tdes_key_schedule(k1, k2, k3, s);
  if (rc) return fail("tdes_key_schedule", rc);

  const size_t n = 3 * 1024 + 77;  /* several tiles and a ragged tail */
  uint8_t *h = (uint8_t *)malloc(8 * n), *g = (uint8_t *)malloc(8 * n);
  for (size_t i = 0; i < 8 * n; ++i) h[i] = (uint8_t)(i * 131u + 7u);
  memcpy(h, pt, 8);  /* block 0 = the SP 800-67 example */
  void *d_in, *d_out;
  if (cudaMalloc(&d_in, 8 * n + 16) != cudaSuccess || cudaMalloc(&d_out, 8 * n) != cudaSuccess) {
    fprintf(stderr, "FAIL cudaMalloc\n");
    return 1;
  }
  cudaMemcpy(d_in, h, 8 * n, cudaMemcpyHostToDevice);
  if ((rc = tdes_ecb_encrypt(s, d_in, d_out, n, NULL))) return fail("tdes_ecb_encrypt", rc);
  cudaMemcpy(g, d_out, 8 * n, cudaMemcpyDeviceToHost);
  if (memcmp(g, ct_exp, 8) != 0) {
    fprintf(stderr, "FAIL: SP 800-67 example block %02X%02X%02X%02X%02X%02X%02X%02X\n", g[0], g[1], g[2], g[3], g[4],
            g[5], g[6], g[7]);
    return 1;
  }
  if ((rc = tdes_ecb_decrypt(s, d_out, d_out, n, NULL))) return fail("tdes_ecb_decrypt (in place)", rc);
  cudaMemcpy(g, d_out, 8 * n, cudaMemcpyDeviceToHost);
  if (memcmp(g, h, 8 * n) != 0) {
    fprintf(stderr, "FAIL: decrypt(encrypt(x)) != x\n");
    return 1;
  }
  if (tdes_ecb_encrypt(s, (uint8_t *)d_in + 4, d_out, 1, NULL) != TDES_ERR_MISALIGNED) {
    fprintf(stderr, "FAIL: misaligned input accepted\n");
    return 1;
  }
  if (tdes_ecb_encrypt(s, d_in, (uint8_t *)d_in + 8, 4, NULL) != TDES_ERR_OVERLAP) {
    fprintf(stderr, "FAIL: overlapping buffers accepted\n");
    return 1;
  }
  if (cudaDeviceSynchronize() != cudaSuccess) {
    fprintf(stderr, "FAIL: cudaDeviceSynchronize\n");
    return 1;
  }
  cudaFree(d_in);
  cudaFree(d_out);
  free(h);
  free(g);
  free(s);
  printf("ABI_KAT_OK\n");
  return 0;
}
