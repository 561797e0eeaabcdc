/*
 * tdes_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of 3DES-EDE in ECB mode,
 * written literally from arXiv 2007.10752 ("Bit-level Parallelization of 3DES
 * Encryption on GPU", /root/reference/PAPER.md, cited below as P:<line>).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * leg may load this library.  The product path (paper_2007_10752_b200/) never
 * imports, links or executes anything under oracle/, and this file shares no
 * code, headers, tables or helpers with it.
 *
 * Representation: one `unsigned char` per bit, exactly as the paper's own data
 * representation ("the smallest available data type (char) is used to
 * represent bits").  Bit 1 is the most significant bit of byte 0 (reading Q1 in
 * DESIGN.md).  Every table below is copied verbatim from the paper's Appendix A
 * (P:208-353), 1-based as printed; the S-box table is read as the 512 integers
 * in printed order (reading Q7).
 *
 * Parallelism: an OpenMP `parallel for` over blocks, mirroring the paper's CPU
 * baseline ("the omp parallel for pragma was used on the for loop that
 * iterates over each block of plaintext").
 *
 * Parity status: pinned (tests/test_oracle.py) by published known-answer
 * vectors, algebraic invariants, table structure and an independent library.
 */
#include <stddef.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned char BYTE;

/* ---- Appendix A: constant arrays, verbatim ---------------- */

/* P:211-222 "Permuted choice table" */
static const BYTE pc_1[56] = {
    57, 49, 41, 33, 25, 17, 9,
    1, 58, 50, 42, 34, 26, 18,
    10, 2, 59, 51, 43, 35, 27,
    19, 11, 3, 60, 52, 44, 36,
    63, 55, 47, 39, 31, 23, 15,
    7, 62, 54, 46, 38, 30, 22,
    14, 6, 61, 53, 45, 37, 29,
    21, 13, 5, 28, 20, 12, 4};

/* P:226-232 */
static const int shift_keys[16] = {
    1, 1, 2, 2,
    2, 2, 2, 2,
    1, 2, 2, 2,
    2, 2, 2, 1};

/* P:234-245 "Key-Compression Table" */
static const BYTE pc_2[48] = {
    14, 17, 11, 24, 1, 5,
    3, 28, 15, 6, 21, 10,
    23, 19, 12, 4, 26, 8,
    16, 7, 27, 20, 13, 2,
    41, 52, 31, 37, 47, 55,
    30, 40, 51, 45, 33, 48,
    44, 49, 39, 56, 34, 53,
    46, 42, 50, 36, 29, 32};

/* P:247-258 "Initial Permutation" */
static const BYTE initial_perm[64] = {
    58, 50, 42, 34, 26, 18, 10, 2,
    60, 52, 44, 36, 28, 20, 12, 4,
    62, 54, 46, 38, 30, 22, 14, 6,
    64, 56, 48, 40, 32, 24, 16, 8,
    57, 49, 41, 33, 25, 17, 9, 1,
    59, 51, 43, 35, 27, 19, 11, 3,
    61, 53, 45, 37, 29, 21, 13, 5,
    63, 55, 47, 39, 31, 23, 15, 7};

/* P:260-269 "Expansion D-box Table" */
static const BYTE exp_d[48] = {
    32, 1, 2, 3, 4, 5, 4, 5,
    6, 7, 8, 9, 8, 9, 10, 11,
    12, 13, 12, 13, 14, 15, 16, 17,
    16, 17, 18, 19, 20, 21, 20, 21,
    22, 23, 24, 25, 24, 25, 26, 27,
    28, 29, 28, 29, 30, 31, 32, 1};

/* P:271-327 "S-box Table, total 8 s-boxes" (boxes 0..4 at P:274-303, boxes
 * 5..7 at P:310-327 after the extraction break; reading Q7). */
static const BYTE s[8][4][16] = {
    {{14, 4, 13, 1, 2, 15, 11, 8, 3, 10, 6, 12, 5, 9, 0, 7},
     {0, 15, 7, 4, 14, 2, 13, 1, 10, 6, 12, 11, 9, 5, 3, 8},
     {4, 1, 14, 8, 13, 6, 2, 11, 15, 12, 9, 7, 3, 10, 5, 0},
     {15, 12, 8, 2, 4, 9, 1, 7, 5, 11, 3, 14, 10, 0, 6, 13}},
    {{15, 1, 8, 14, 6, 11, 3, 4, 9, 7, 2, 13, 12, 0, 5, 10},
     {3, 13, 4, 7, 15, 2, 8, 14, 12, 0, 1, 10, 6, 9, 11, 5},
     {0, 14, 7, 11, 10, 4, 13, 1, 5, 8, 12, 6, 9, 3, 2, 15},
     {13, 8, 10, 1, 3, 15, 4, 2, 11, 6, 7, 12, 0, 5, 14, 9}},
    {{10, 0, 9, 14, 6, 3, 15, 5, 1, 13, 12, 7, 11, 4, 2, 8},
     {13, 7, 0, 9, 3, 4, 6, 10, 2, 8, 5, 14, 12, 11, 15, 1},
     {13, 6, 4, 9, 8, 15, 3, 0, 11, 1, 2, 12, 5, 10, 14, 7},
     {1, 10, 13, 0, 6, 9, 8, 7, 4, 15, 14, 3, 11, 5, 2, 12}},
    {{7, 13, 14, 3, 0, 6, 9, 10, 1, 2, 8, 5, 11, 12, 4, 15},
     {13, 8, 11, 5, 6, 15, 0, 3, 4, 7, 2, 12, 1, 10, 14, 9},
     {10, 6, 9, 0, 12, 11, 7, 13, 15, 1, 3, 14, 5, 2, 8, 4},
     {3, 15, 0, 6, 10, 1, 13, 8, 9, 4, 5, 11, 12, 7, 2, 14}},
    {{2, 12, 4, 1, 7, 10, 11, 6, 8, 5, 3, 15, 13, 0, 14, 9},
     {14, 11, 2, 12, 4, 7, 13, 1, 5, 0, 15, 10, 3, 9, 8, 6},
     {4, 2, 1, 11, 10, 13, 7, 8, 15, 9, 12, 5, 6, 3, 0, 14},
     {11, 8, 12, 7, 1, 14, 2, 13, 6, 15, 0, 9, 10, 4, 5, 3}},
    {{12, 1, 10, 15, 9, 2, 6, 8, 0, 13, 3, 4, 14, 7, 5, 11},
     {10, 15, 4, 2, 7, 12, 9, 5, 6, 1, 13, 14, 0, 11, 3, 8},
     {9, 14, 15, 5, 2, 8, 12, 3, 7, 0, 4, 10, 1, 13, 11, 6},
     {4, 3, 2, 12, 9, 5, 15, 10, 11, 14, 1, 7, 6, 0, 8, 13}},
    {{4, 11, 2, 14, 15, 0, 8, 13, 3, 12, 9, 7, 5, 10, 6, 1},
     {13, 0, 11, 7, 4, 9, 1, 10, 14, 3, 5, 12, 2, 15, 8, 6},
     {1, 4, 11, 13, 12, 3, 7, 14, 10, 15, 6, 8, 0, 5, 9, 2},
     {6, 11, 13, 8, 1, 4, 10, 7, 9, 5, 0, 15, 14, 2, 3, 12}},
    {{13, 2, 8, 4, 6, 15, 11, 1, 10, 9, 3, 14, 5, 0, 12, 7},
     {1, 15, 13, 8, 10, 3, 7, 4, 12, 5, 6, 11, 0, 14, 9, 2},
     {7, 11, 4, 1, 9, 12, 14, 2, 0, 6, 10, 13, 15, 3, 5, 8},
     {2, 1, 14, 7, 4, 10, 8, 13, 15, 12, 9, 0, 3, 5, 6, 11}}};

/* P:329-340 "Straight Permutation Table" */
static const BYTE per[32] = {
    16, 7, 20, 21,
    29, 12, 28, 17,
    1, 15, 23, 26,
    5, 18, 31, 10,
    2, 8, 24, 14,
    32, 27, 3, 9,
    19, 13, 30, 6,
    22, 11, 4, 25};

/* P:342-353 "Final Permutation Table" */
static const BYTE final_perm[64] = {
    40, 8, 48, 16, 56, 24, 64, 32,
    39, 7, 47, 15, 55, 23, 63, 31,
    38, 6, 46, 14, 54, 22, 62, 30,
    37, 5, 45, 13, 53, 21, 61, 29,
    36, 4, 44, 12, 52, 20, 60, 28,
    35, 3, 43, 11, 51, 19, 59, 27,
    34, 2, 42, 10, 50, 18, 58, 26,
    33, 1, 41, 9, 49, 17, 57, 25};

/* ---- Bit plumbing (reading Q1: bit 1 = MSB of byte 0) ----------------- */

/* 8 octets -> 64 chars; out[0] is FIPS bit 1. */
static void bytes_to_bits(const uint8_t in[8], BYTE out[64]) {
  for (int i = 0; i < 64; i++) out[i] = (BYTE)((in[i / 8] >> (7 - (i % 8))) & 1);
}

static void bits_to_bytes(const BYTE in[64], uint8_t out[8]) {
  for (int b = 0; b < 8; b++) {
    uint8_t v = 0;
    for (int i = 0; i < 8; i++) v = (uint8_t)((v << 1) | (in[8 * b + i] & 1));
    out[b] = v;
  }
}

/* "57th bit of the original key will be the 1st bit of the permuted key and so
 * on. The same logic applies for every permutation function":
 * out[i] = in[table[i]] with the table 1-based as printed. */
static void permute(const BYTE *in, BYTE *out, const BYTE *table, int n) {
  for (int i = 0; i < n; i++) out[i] = in[table[i] - 1];
}

/* ---- §III.A key generation ---------------------------------- */

/* subkeys[r][0..47], r = 0..15 for rounds 1..16. */
static void key_schedule(const uint8_t key[8], BYTE subkeys[16][48]) {
  BYTE k[64], cd[56], C[28], D[28], tmp[28], CD[56];
  bytes_to_bits(key, k);
  permute(k, cd, pc_1, 56);                 /* "64-bit key is permuted to 56 bits using the pc_1 array" */
  memcpy(C, cd, 28);                        /* "divided into two 28-bit arrays" (reading Q14) */
  memcpy(D, cd + 28, 28);
  for (int r = 0; r < 16; r++) {            /* "repeated 16 times" */
    int sh = shift_keys[r];                 /* "circularly left-shifted using the shift_keys array" (reading Q13) */
    for (int i = 0; i < 28; i++) tmp[i] = C[(i + sh) % 28];
    memcpy(C, tmp, 28);
    for (int i = 0; i < 28; i++) tmp[i] = D[(i + sh) % 28];
    memcpy(D, tmp, 28);
    memcpy(CD, C, 28);                      /* "A combination of the two arrays" */
    memcpy(CD + 28, D, 28);
    permute(CD, subkeys[r], pc_2, 48);      /* "permuted to 48-bit ... using the pc_2 array" */
  }
}

/* ---- §III.B the Feistel function and one DES ---------------- */

/* Six bits b1..b6 -> 4 bits through box g (0-based):
 * "Middle 4 bits ... column", outer bits -> row (reading Q2:
 * row = 2*b1 + b6, col = 8*b2 + 4*b3 + 2*b4 + b5). Output MSB first. */
static void sbox(int g, const BYTE six[6], BYTE four[4]) {
  int row = 2 * six[0] + six[5];
  int col = 8 * six[1] + 4 * six[2] + 2 * six[3] + six[4];
  int v = s[g][row][col];
  for (int i = 0; i < 4; i++) four[i] = (BYTE)((v >> (3 - i)) & 1);
}

static void feistel_f(const BYTE R[32], const BYTE k[48], BYTE f[32]) {
  BYTE e[48], sb[32];
  permute(R, e, exp_d, 48);                         /* "permuted to 48 bits with an exp_d array" */
  for (int i = 0; i < 48; i++) e[i] ^= k[i];        /* "XORed with the round key" */
  for (int g = 0; g < 8; g++) sbox(g, e + 6 * g, sb + 4 * g); /* S-boxes */
  permute(sb, f, per, 32);                          /* "permuted again to 32 bits with a per array" */
}

/* One DES on 64 chars.  decrypt != 0 uses the reversed round-key order. */
static void des_bits(const BYTE in[64], BYTE subkeys[16][48], int decrypt, BYTE out[64]) {
  BYTE v[64], L[32], R[32], f[32], newR[32], RL[64];
  permute(in, v, initial_perm, 64);
  memcpy(L, v, 32);
  memcpy(R, v + 32, 32);
  for (int r = 0; r < 16; r++) {
    const BYTE *k = subkeys[decrypt ? 15 - r : r];
    feistel_f(R, k, f);
    for (int i = 0; i < 32; i++) newR[i] = L[i] ^ f[i]; /* P:71 (reading Q3: current left half) */
    memcpy(L, R, 32);                                   /* P:72 swap */
    memcpy(R, newR, 32);
  }
  memcpy(RL, R, 32);                        /* P:74 "combined" (reading Q4: R16 || L16) */
  memcpy(RL + 32, L, 32);
  permute(RL, out, final_perm, 64);
}

/* ---- §III.B 3DES composition -------------------------------- */

typedef struct {
  BYTE ks[3][16][48];
} oracle_triple;

static void triple_schedule(const uint8_t k1[8], const uint8_t k2[8], const uint8_t k3[8],
                            oracle_triple *t) {
  key_schedule(k1, t->ks[0]);               /* "run three times for each base key" */
  key_schedule(k2, t->ks[1]);
  key_schedule(k3, t->ks[2]);
}

static void tdes_block(const oracle_triple *t, int decrypt, const uint8_t in[8], uint8_t out[8]) {
  BYTE a[64], b[64];
  bytes_to_bits(in, a);
  if (!decrypt) {
    /* ciphertext = E_K3(D_K2(E_K1(plaintext))) */
    des_bits(a, (BYTE(*)[48])t->ks[0], 0, b);
    des_bits(b, (BYTE(*)[48])t->ks[1], 1, a);
    des_bits(a, (BYTE(*)[48])t->ks[2], 0, b);
  } else {
    /* plaintext = D_K1(E_K2(D_K3(ciphertext))) */
    des_bits(a, (BYTE(*)[48])t->ks[2], 1, b);
    des_bits(b, (BYTE(*)[48])t->ks[1], 0, a);
    des_bits(a, (BYTE(*)[48])t->ks[0], 1, b);
  }
  bits_to_bytes(b, out);
}

/* ---- Exported entry points -------------------------------------------- */

/* Subkeys of one 8-byte key, each as 48 chars (FIPS order), rounds 1..16. */
void oracle_des_key_schedule(const uint8_t key[8], uint8_t subkeys_out[16 * 48]) {
  BYTE ks[16][48];
  key_schedule(key, ks);
  memcpy(subkeys_out, ks, sizeof ks);
}

/* One single DES of an 8-byte block. */
void oracle_des_block(const uint8_t key[8], int decrypt, const uint8_t in[8], uint8_t out[8]) {
  BYTE ks[16][48], a[64], b[64];
  key_schedule(key, ks);
  bytes_to_bits(in, a);
  des_bits(a, ks, decrypt, b);
  bits_to_bytes(b, out);
}

/* S-box g (0..7) on a 6-bit value whose MSB is b1; returns the 4-bit output. */
int oracle_sbox(int g, int six) {
  BYTE in6[6], out4[4];
  for (int i = 0; i < 6; i++) in6[i] = (BYTE)((six >> (5 - i)) & 1);
  sbox(g, in6, out4);
  return (out4[0] << 3) | (out4[1] << 2) | (out4[2] << 1) | out4[3];
}

/* f(R, k) on packed values: R as 32 bits (bit 1 = MSB), k as 48 bits (bit 1 =
 * bit 47 of the integer); returns 32 bits. */
uint32_t oracle_feistel_f(uint32_t r, uint64_t k) {
  BYTE R[32], K[48], f[32];
  for (int i = 0; i < 32; i++) R[i] = (BYTE)((r >> (31 - i)) & 1);
  for (int i = 0; i < 48; i++) K[i] = (BYTE)((k >> (47 - i)) & 1);
  feistel_f(R, K, f);
  uint32_t v = 0;
  for (int i = 0; i < 32; i++) v = (v << 1) | f[i];
  return v;
}

/* Expose a table for structural tests: which = 0 pc_1, 1 pc_2, 2 initial_perm,
 * 3 exp_d, 4 per, 5 final_perm, 6 shift_keys, 7 s (flattened 512).  Returns the
 * entry count and copies the entries (as ints) into out (capacity >= 512). */
int oracle_table(int which, int *out) {
  const BYTE *t = 0;
  int n = 0;
  switch (which) {
    case 0: t = pc_1; n = 56; break;
    case 1: t = pc_2; n = 48; break;
    case 2: t = initial_perm; n = 64; break;
    case 3: t = exp_d; n = 48; break;
    case 4: t = per; n = 32; break;
    case 5: t = final_perm; n = 64; break;
    case 6: for (int i = 0; i < 16; i++) out[i] = shift_keys[i]; return 16;
    case 7: t = &s[0][0][0]; n = 512; break;
    default: return -1;
  }
  for (int i = 0; i < n; i++) out[i] = t[i];
  return n;
}

/* 3DES-EDE ECB over n independent 8-byte blocks ("each block is
 * encrypted independently"), OpenMP over blocks.  threads <= 0 means
 * the OpenMP default.  Returns the thread count actually used. */
int oracle_tdes_ecb(const uint8_t k1[8], const uint8_t k2[8], const uint8_t k3[8],
                    const uint8_t *in, uint8_t *out, size_t n, int decrypt, int threads) {
  oracle_triple t;
  triple_schedule(k1, k2, k3, &t);
  int used = 1;
#ifdef _OPENMP
  if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel for num_threads(threads) schedule(static)
  for (long long i = 0; i < (long long)n; i++) {
    if (i == 0) used = omp_get_num_threads();
    tdes_block(&t, decrypt, in + 8 * i, out + 8 * i);
  }
#else
  (void)threads;
  for (size_t i = 0; i < n; i++) tdes_block(&t, decrypt, in + 8 * i, out + 8 * i);
#endif
  return used;
}
