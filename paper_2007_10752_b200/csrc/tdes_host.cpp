// Host side of the C ABI: key schedule + lane-mask packing.
//
// The DES key schedule (§III.A) is microseconds of work per
// key triple, so it runs here on packed 64-bit integers instead of in a GPU
// kernel (the paper's Fig. 2 kernel).  Tables come from the
// generated tdes_host_tables.h (tools/gen_tdes.py), independent of oracle/.
#include <stdint.h>
#include <string.h>

#include "../../include/tdes.h"
#include "gen/tdes_host_tables.h"

namespace {

uint64_t load_be64(const uint8_t k[8]) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v = (v << 8) | k[i];
  return v;  // FIPS bit n is bit (64 - n)
}

// 16 subkeys of 48 bits; subkey bit 1 (FIPS) = integer bit 47.
void des_subkeys(const uint8_t key[8], uint64_t sk[16]) {
  const uint64_t K = load_be64(key);
  uint64_t cd = 0;
  for (int i = 0; i < 56; ++i) cd = (cd << 1) | ((K >> (64 - kPC1[i])) & 1u);  // PC-1
  uint32_t C = (uint32_t)(cd >> 28) & 0x0FFFFFFFu;                              // halves
  uint32_t D = (uint32_t)cd & 0x0FFFFFFFu;
  for (int r = 0; r < 16; ++r) {
    const int s = kShifts[r];                                                   // rotations
    C = ((C << s) | (C >> (28 - s))) & 0x0FFFFFFFu;
    D = ((D << s) | (D >> (28 - s))) & 0x0FFFFFFFu;
    const uint64_t CD = ((uint64_t)C << 28) | D;
    uint64_t k = 0;
    for (int i = 0; i < 48; ++i) k = (k << 1) | ((CD >> (56 - kPC2[i])) & 1u);  // PC-2
    sk[r] = k;
  }
}

void expand(uint64_t sk, uint32_t m[48]) {
  for (int b = 0; b < 48; ++b) m[b] = ((sk >> (47 - b)) & 1u) ? 0xFFFFFFFFu : 0u;
}

}  // namespace

extern "C" int tdes_key_schedule(const uint8_t k1[8], const uint8_t k2[8], const uint8_t k3[8],
                                 tdes_schedule *out) {
  if (!k1 || !k2 || !k3 || !out) return TDES_ERR_INVALID_ARG;
  memset(out, 0, sizeof *out);
  des_subkeys(k1, out->subkey[0]);
  des_subkeys(k2, out->subkey[1]);
  des_subkeys(k3, out->subkey[2]);
  for (int r = 0; r < 16; ++r) {
    // encrypt: E_K1 (r1..16), D_K2 (r16..1), E_K3 (r1..16)
    expand(out->subkey[0][r], out->mask[0][r]);
    expand(out->subkey[1][15 - r], out->mask[0][16 + r]);
    expand(out->subkey[2][r], out->mask[0][32 + r]);
    // decrypt: D_K3 (r16..1), E_K2 (r1..16), D_K1 (r16..1)
    expand(out->subkey[2][15 - r], out->mask[1][r]);
    expand(out->subkey[1][r], out->mask[1][16 + r]);
    expand(out->subkey[0][15 - r], out->mask[1][32 + r]);
  }
  return TDES_OK;
}

extern "C" int des_key_schedule(const uint8_t k[8], des_schedule *out) {
  if (!k || !out) return TDES_ERR_INVALID_ARG;
  memset(out, 0, sizeof *out);
  des_subkeys(k, out->subkey);
  for (int r = 0; r < 16; ++r) {
    expand(out->subkey[r], out->mask[0][r]);       // encrypt order
    expand(out->subkey[15 - r], out->mask[1][r]);  // decrypt: reversed
  }
  return TDES_OK;
}

extern "C" const char *tdes_strerror(int code) {
  switch (code) {
    case TDES_OK: return "ok";
    case TDES_ERR_INVALID_ARG: return "invalid argument";
    case TDES_ERR_MISALIGNED: return "buffer not 8-byte aligned";
    case TDES_ERR_OVERLAP: return "input and output partially overlap";
    case TDES_ERR_CUDA: return "CUDA error (see tdes_last_cuda_error)";
    case TDES_ERR_WORKSPACE: return "workspace too small";
    default: return "unknown error";
  }
}
