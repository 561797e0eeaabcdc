// Bitsliced 3DES-EDE ECB for B200 (sm_100a) -- the hot path of arXiv 2007.10752.
//
// What it computes (§III): for every independent 64-bit
// block (ECB) C = E_K3(D_K2(E_K1(P))) or the inverse.
// How: instead of the paper's one-CTA-per-block,
// one-thread-per-bit design, every thread owns 32 blocks and holds
// them as 64 bit-planes (plane j = FIPS-renamed bit j of all 32 blocks):
//
//   S1 load      a warp's 8 KiB tile (32 blocks per lane): one TMA bulk copy into
//                shared memory, prefetched during the previous tile, then LDS.128
//   S2 transpose two 32x32 bit transposes (PRMT for the 16/8 stages)
//   S3 IP        register renaming (free)
//   S4 48 rounds key XOR (one IMAD each, FMA pipe; operands from LDCU + a shared-
//                memory key table), 8 LOP3 S-box circuits, XOR into the
//                other half; E and P are operand/destination renaming (free);
//                the three DES stages are fused, IP/FP between them cancel
//   S6 FP        register renaming (free)
//   S7 store     inverse transpose + coalesced stores (in place allowed)
//
// All arithmetic is bitwise (LOP3/PRMT/SHF on the integer ALU pipe); nothing
// is a contraction, so there are no tensor cores here.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <atomic>
#include <type_traits>

#include "../../include/tdes.h"
#include "../../include/tdes_bench.h"
#include "gen/tdes_gen.cuh"
#include "tdes_error.h"

namespace {

// 16 warps per CTA, one CTA per SM; ptxas keeps the round in 125 registers
// without spills (<= 128 for 512 threads).  Warps per CTA measured on B200 with
// the current kernel (tools/exp/ab_warps.py, us per launch, 12 -> 16 warps):
// 2^21 blocks 69 -> 61, 2^22 121 -> 111, 2^24 373 -> 370, 2^27 2873 -> 2849;
// 8-11 warps slower everywhere above 2^21.  (Before the TMA staging cut the
// register count from 156, 12 warps were best.)
#ifndef TDES_THREADS
#define TDES_THREADS 512
#endif
#ifndef TDES_WORDS
#define TDES_WORDS 1
#endif
constexpr int kThreads = TDES_THREADS;
constexpr int kMinCtasPerSm = 1;
// Words per bit-plane: a thread holds kWords independent 32-block groups, so
// each loaded key value and each instruction-issue decision serves kWords words.
constexpr int kWords = TDES_WORDS;
constexpr int kGroupBlocks = 32 * 32;  // one 32-block group per lane: 1024 blocks = 8 KiB per warp
constexpr int kBlocksPerThread = 32 * kWords;
constexpr int kTileBlocks = kGroupBlocks * kWords;  // per warp
// Two-round bodies per loop iteration of the 3DES round loop (single DES: 1).
// Measured on B200, 1 GiB, current kernel: 1 -> 2 (a 21 KB body) 374 -> 377 GB/s;
// 3 (33 KB) 363, 4 (40 KB) 352: beyond the 32 KB L1.5 instruction cache.  (Before the TMA staging / 16-warp CTA, 2 was 2-3%
// slower: the body then had to share the instruction cache with more warps'
// divergent positions.)
#ifndef TDES_ROUND_UNROLL
#define TDES_ROUND_UNROLL 2
#endif
constexpr int kRoundUnroll3 = TDES_ROUND_UNROLL;
// Two-round bodies per loop iteration of the single-DES round loop.
#ifndef TDES_ROUND_UNROLL1
#define TDES_ROUND_UNROLL1 1
#endif
constexpr int kRoundUnroll1 = TDES_ROUND_UNROLL1;
// TMA-staged loads: each warp's next 8 KiB tile is fetched into a per-warp
// shared-memory buffer by one cp.async.bulk (completion on a per-warp mbarrier)
// while the warp computes the current tile, hiding the HBM latency at tile start.
// Measured on B200, 1 GiB: single DES 946 -> 966 GB/s, 3DES unchanged (371 GB/s);
// claiming the next tile later (two thirds into the rounds) was 1-3% slower.
#ifndef TDES_TMA
#define TDES_TMA 1
#endif
constexpr bool kTma = TDES_TMA && kWords == 1;
constexpr int kWarps = kThreads / 32;
constexpr unsigned kTileBytes = kTileBlocks * 8u;

// mulhi.s32(0x7FFFFFFF, s) = (s - 1) / 2 for s = +-1 (tdes_gen::kxor with
// MULHI, and the split kernel's k).  Passed as a kernel argument so it lives in a
// register instead of being folded into an immediate (which would force s out of
// the uniform datapath).
constexpr uint32_t kMulhiC = 0x7FFFFFFFu;

// Key material, consumption order (round, E-bit): s = k | 1 (+1 or -1) where k
// is the subkey bit's all-ones / all-zeros lane mask; x ^ k = x * s + k is one
// IMAD (tdes_gen::kxor).
//
// Mask folding: the planes carry pending uniform masks, so s/k are
// the combined "pending mask ^ key bit" operands of the E-positions that still
// need a key IMAD (tdes_gen::kKeySlots of 48), d are the masks the unfused
// outputs fold into their planes, fix the operands that prime round A's free
// positions before round 0 and after each stage-boundary swap, fin the final
// unmasking of all 64 planes.  RoundMasks is the whole set as the host computes
// it (build_masks; tdes_fold_operands returns it).
template <int NROUNDS>
struct alignas(16) RoundMasks {
  uint32_t s[NROUNDS][tdes_gen::kKeyStride];
  uint32_t k[NROUNDS][tdes_gen::kKeyStride];
  uint32_t d[NROUNDS][tdes_gen::kDeltaStride];
  uint32_t fix_s[3][tdes_gen::kDeltaStride], fix_k[3][tdes_gen::kDeltaStride];
  uint32_t fin_s[64], fin_k[64];
};

// The subkeys bit-packed, one 48-bit word per round (384 B for 3DES): the launch
// parameter of the split kernel and of the device-key throughput kernel, which
// expand every operand they need from it on the device.
template <int NROUNDS>
struct RoundKeys {
  uint64_t k[NROUNDS];  // bit 47 - b = subkey bit b (E position b), consumption order
};

// The throughput kernel's launch parameters (SKeys): only the s operands, which
// the round reads as uniform operands -- and the uniform datapath loads only from
// the constant bank, i.e. from the launch parameters -- plus the packed subkeys,
// from which each CTA expands k, d, the fix-ups and the unmask into shared memory
// (expand_keys).  7.9 KB for 3DES instead of the 18 KB RoundMasks of round 1,
// whose k/d copy from the constant bank cost each CTA ~4 us at start
// (tools/exp/trace_prologue.py).
template <int NROUNDS>
struct alignas(16) SKeys {
  uint32_t s[NROUNDS][tdes_gen::kKeyStride];
  uint32_t fix_s[3][tdes_gen::kDeltaStride], fix_k[3][tdes_gen::kDeltaStride];
  uint32_t fin_s[64], fin_k[64];
  uint64_t k[NROUNDS];
};

// Mask folding, symbolically.  The planes' pending masks M are
// tracked through the fused rounds exactly as the kernel applies them (fix-ups,
// rounds, swaps): round r is round_A for even r, round_B for odd r, and a free
// E-position of round r reads its plane as is, which is correct because the
// previous round's unfused output (or a fix-up) set that plane's mask to the key
// bit of exactly that position.  Every M is 0 or one key bit key(r, pos), and
// which one depends only on the generator's plan, not on the key -- so every
// operand word is key(a) ^ key(b) for a static pair of key-bit references
// (index r * 48 + pos, kNoRef = none).  OpRefs holds those pairs; it is a
// compile-time constant used by the host (build_masks) and, on the device, by
// the throughput kernel's prologue, which expands the 384-byte packed subkeys
// into its operand tables (NEXT-4, the paper's key-expansion step).
constexpr uint16_t kNoRef = 0xFFFF;

template <int NSTAGES>
struct OpRefs {
  static constexpr int NR = 16 * NSTAGES;
  uint16_t sk[NR][tdes_gen::kKeyStride][2];   // s = v | 1, k = v
  uint16_t d[NR][tdes_gen::kDeltaStride][2];  // folded-output masks
  uint16_t fix[3][tdes_gen::kDeltaStride][2]; // fix_s = v | 1, fix_k = v
  uint16_t fin[64];                           // fin_s = v | 1, fin_k = v (one reference)
};

template <int NSTAGES>
constexpr OpRefs<NSTAGES> build_refs() {
  using namespace tdes_gen;
  constexpr int NR = 16 * NSTAGES;
  OpRefs<NSTAGES> o{};
  for (int r = 0; r < NR; ++r) {
    for (int q = 0; q < kKeyStride; ++q) o.sk[r][q][0] = o.sk[r][q][1] = kNoRef;
    for (int u = 0; u < kDeltaStride; ++u) o.d[r][u][0] = o.d[r][u][1] = kNoRef;
  }
  for (int b = 0; b < 3; ++b)
    for (int t = 0; t < kDeltaStride; ++t) o.fix[b][t][0] = o.fix[b][t][1] = kNoRef;
  uint16_t M[64] = {};
  for (int j = 0; j < 64; ++j) M[j] = kNoRef;
  auto key = [](int r, int pos) { return (uint16_t)(r * 48 + pos); };
  auto boundary = [](int r) { return NSTAGES == 3 && (r == 16 || r == 32); };
  auto fixup = [&](int b, int r) {  // prime round_A's free positions for round r
    for (int t = 0; t < kFoldFree; ++t) {
      const int pos = kFoldFreePos[0][t], j = kFoldSrc[0][pos];
      o.fix[b][t][0] = M[j];
      o.fix[b][t][1] = key(r, pos);
      M[j] = key(r, pos);
    }
  };
  fixup(0, 0);
  for (int r = 0; r < NR; ++r) {
    const int x = r & 1;
    if (boundary(r)) {
      for (int t = 0; t < 32; ++t) {
        const uint16_t tmp = M[kHalfA[t]];
        M[kHalfA[t]] = M[kHalfB[t]];
        M[kHalfB[t]] = tmp;
      }
      fixup(r >> 4, r);
    }
    for (int q = 0; q < kKeySlots; ++q) {
      const int pos = kFoldKeyPos[x][q];
      o.sk[r][q][0] = M[kFoldSrc[x][pos]];
      o.sk[r][q][1] = key(r, pos);
    }
    for (int u = 0; u < kFoldFree; ++u) {
      const int j = kFoldUDst[x][u];
      if (r + 1 < NR && !boundary(r + 1)) {
        o.d[r][u][0] = M[j];
        o.d[r][u][1] = key(r + 1, kFoldUNext[x][u]);
        M[j] = key(r + 1, kFoldUNext[x][u]);
      }  // else the mask stays: d = 0
    }
  }
  for (int j = 0; j < 64; ++j) o.fin[j] = M[j];
  return o;
}

constexpr OpRefs<3> kRefs3 = build_refs<3>();
constexpr OpRefs<1> kRefs1 = build_refs<1>();
template <int NSTAGES>
constexpr const OpRefs<NSTAGES>& refs_host() {
  if constexpr (NSTAGES == 3) return kRefs3; else return kRefs1;
}
// Device copies (read once per CTA by the prologue; 10 KB for 3DES).
__device__ const OpRefs<3> kDevRefs3 = build_refs<3>();
__device__ const OpRefs<1> kDevRefs1 = build_refs<1>();
template <int NSTAGES>
__device__ __forceinline__ const OpRefs<NSTAGES>& refs_dev() {
  if constexpr (NSTAGES == 3) return kDevRefs3; else return kDevRefs1;
}


// x >> s as the high word of x * 2^(32-s): IMAD.HI on the FMA pipe instead of
// SHF on the integer ALU pipe (the kernel's bound).  Left shifts already
// compile to IMAD.SHL.
#ifndef TDES_SHR_FMA
#define TDES_SHR_FMA 1
#endif
template <int S>
__device__ __forceinline__ uint32_t shr_fma(uint32_t x) {
#if TDES_SHR_FMA
  uint32_t d;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(x), "n"(1u << (32 - S)));
  return d;
#else
  return x >> S;
#endif
}

// One bit-level transpose stage: swap bit S of the row and column index.
template <int S>
__device__ __forceinline__ void bitstage(uint32_t (&a)[32], uint32_t m) {
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    if (k & S) continue;
    const uint32_t lo = a[k], hi = a[k + S];
    a[k] = tdes_gen::lop3<0xCA>(m, lo, hi << S);            // m ? lo : (hi << S)
    a[k + S] = tdes_gen::lop3<0xCA>(m, shr_fma<S>(lo), hi);  // m ? (lo >> S) : hi
  }
}

// In-register 32x32 bit-matrix transpose: a[i] bit j <-> a[j] bit i.
// Stage s swaps bit s of the row and column index; s = 16 and 8 are whole
// half-words / bytes and run as one PRMT per output word.
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
  bitstage<4>(a, 0x0F0F0F0Fu);
  bitstage<2>(a, 0x33333333u);
  bitstage<1>(a, 0x55555555u);
}

// Plane type: one word (uint32_t) or kWords words (tdes_gen::Vec).
template <int W>
struct PlaneOf {
  using type = tdes_gen::Vec<W>;
};
template <>
struct PlaneOf<1> {
  using type = uint32_t;
};
__device__ __forceinline__ uint32_t& word(uint32_t& v, int) { return v; }
template <int W>
__device__ __forceinline__ uint32_t& word(tdes_gen::Vec<W>& v, int i) {
  return v.w[i];
}

// ---- TMA (bulk async copy) helpers ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
// Arm `bar` for `bytes` and start one bulk copy global -> shared (one thread).
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of dst
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!done);
}

// A staged (TMA-loaded) full group from shared memory, same lane layout as the
// VEC4 global path: lane l reads 16 bytes at 512 i + 16 l (conflict free).
__device__ __forceinline__ void load_group_smem(const uint4* buf, unsigned lane, uint32_t (&X)[32],
                                                uint32_t (&Y)[32]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint4 v = buf[32 * i + lane];
    X[2 * i] = v.x;
    Y[2 * i] = v.y;
    X[2 * i + 1] = v.z;
    Y[2 * i + 1] = v.w;
  }
  transpose32(X);
  transpose32(Y);
}

// One 1024-block group (32 lanes x 32 blocks) from `base` into bit-planes X (low
// words) and Y (high words).  VEC4: in 16-byte aligned -> 128-bit loads.
template <bool VEC4>
__device__ __forceinline__ void load_group(const uint2* in, size_t base, size_t nblocks, unsigned lane,
                                           uint32_t (&X)[32], uint32_t (&Y)[32]) {
  const bool full = base + kGroupBlocks <= nblocks;
  // ---- S1: load.  Plane bit i <-> the i-th block this lane loads. ----
  if (VEC4) {
    const uint4* in4 = reinterpret_cast<const uint4*>(in + base);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const size_t b = base + 64 * i + 2 * lane;
      uint4 v;
      if (full || b + 1 < nblocks) {
        v = __ldcs(in4 + 32 * i + lane);
      } else {
        v = make_uint4(0u, 0u, 0u, 0u);
        if (b < nblocks) {
          const uint2 h = __ldcs(in + b);
          v.x = h.x;
          v.y = h.y;
        }
      }
      X[2 * i] = v.x;
      Y[2 * i] = v.y;
      X[2 * i + 1] = v.z;
      Y[2 * i + 1] = v.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const size_t b = base + 32 * i + lane;
      uint2 v = make_uint2(0u, 0u);
      if (full || b < nblocks) v = __ldcs(in + b);
      X[i] = v.x;
      Y[i] = v.y;
    }
  }
  transpose32(X);
  transpose32(Y);
}

// Inverse of load_group: planes X, Y back to blocks, stored from `base`.
template <bool VEC4>
__device__ __forceinline__ void store_group(uint2* out, size_t base, size_t nblocks, unsigned lane,
                                            uint32_t (&X)[32], uint32_t (&Y)[32]) {
  const bool full = base + kGroupBlocks <= nblocks;
  transpose32(X);
  transpose32(Y);
  if (VEC4) {
    uint4* out4 = reinterpret_cast<uint4*>(out + base);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const size_t b = base + 64 * i + 2 * lane;
      const uint4 v = make_uint4(X[2 * i], Y[2 * i], X[2 * i + 1], Y[2 * i + 1]);
      if (full || b + 1 < nblocks) {
        __stcs(out4 + 32 * i + lane, v);
      } else if (b < nblocks) {
        __stcs(out + b, make_uint2(v.x, v.y));
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const size_t b = base + 32 * i + lane;
      if (full || b < nblocks) __stcs(out + b, make_uint2(X[i], Y[i]));
    }
  }
}

// One warp tile: kWords groups of 1024 consecutive blocks from `base`; word w
// of every plane holds group w.
// TMA staging (kTma): `staged` = this tile sits in `buf` (wait on `bar` with
// `phase`); `prefetch` claims the warp's next tile and starts its copy into `buf`
// once the current one has been read out of it.
// KV = ParamKeys (host-folded operands in the launch parameters) or DevKeys
// (operands expanded on the device into shared memory); see below.
template <int NSTAGES, bool VEC4, class KV, class Prefetch>
__device__ __forceinline__ void crypt_tile(const uint2* in, uint2* out, size_t base, size_t nblocks,
                                           unsigned lane, const KV& kv, uint32_t c, uint4* buf, uint64_t* bar,
                                           bool staged, uint32_t phase, Prefetch&& prefetch) {
  using V = typename PlaneOf<kWords>::type;
  V P[64];
  // ---- S1 load + S2 transpose to bit-planes ----
  if (kTma && staged) {
    mbar_wait(bar, phase);
    uint32_t X[32], Y[32];
    load_group_smem(buf, lane, X, Y);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      word(P[j], 0) = X[j];
      word(P[32 + j], 0) = Y[j];
    }
  } else {
#pragma unroll
    for (int w = 0; w < kWords; ++w) {
      uint32_t X[32], Y[32];
      load_group<VEC4>(in, base + (size_t)w * kGroupBlocks, nblocks, lane, X, Y);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        word(P[j], w) = X[j];
        word(P[32 + j], w) = Y[j];
      }
    }
  }
  if (kTma) {
    __syncwarp();  // every lane has consumed buf
    prefetch();
  }
  // ---- S3..S6: IP (renaming), 16*NSTAGES rounds, FP (renaming) ----
  // One two-round loop body for all stages keeps all warps of the SM inside
  // the instruction cache.  The middle stage starts on the half the first one
  // updated last, so at each stage boundary the halves swap
  // register roles and the same A-then-B body continues.
  constexpr int kUnroll = NSTAGES == 3 ? kRoundUnroll3 : kRoundUnroll1;
  kv.fixup(P, 0, c);
#pragma unroll kUnroll
  for (int r = 0; r < 16 * NSTAGES; r += 2) {
    if (NSTAGES == 3 && (r == 16 || r == 32)) {
      tdes_gen::swap_halves(P);
      kv.fixup(P, r >> 4, c);
    }
    kv.two_rounds(P, r, c);
  }
  kv.unmask(P, c);
  V Q[64];
  tdes_gen::output_planes(P, Q);
  // ---- S7: back to blocks, store ----
#pragma unroll
  for (int w = 0; w < kWords; ++w) {
    uint32_t X[32], Y[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      X[j] = word(Q[j], w);
      Y[j] = word(Q[32 + j], w);
    }
    store_group<VEC4>(out, base + (size_t)w * kGroupBlocks, nblocks, lane, X, Y);
  }
}

// ---- key operand sources of the throughput kernel ----
// Both variants expand the packed subkeys on the device, at CTA start, into the
// operands the rounds read from shared memory (expand_keys).  They differ in s:
//   ParamKeys (WITH_S = false; the launch parameters are SKeys): s is read in the
//     round as a uniform operand (LDCU) straight from the launch parameters, k and
//     d from the shared-memory table with broadcast LDS.128 (4 values each);
//   DevKeys (WITH_S = true, NEXT-4; the launch parameters are the 384-byte
//     RoundKeys): s comes from the shared-memory table as well, into vector
//     registers (IMAD x * s + k with every operand a vector register) -- 6.5%
//     slower on long launches, faster to start.
// Table layout per round: [s (kKv uint4, DevKeys only) | k (kKv) | d (kDv)], then
// the fix-up and unmask words ff = fix_s[3][kDeltaStride] fix_k[3][kDeltaStride]
// fin_s[64] fin_k[64].
template <int NSTAGES, bool WITH_S>
struct KeyTable {
  static constexpr int kKv = tdes_gen::kKeyStride / 4, kDv = tdes_gen::kDeltaStride / 4;
  static constexpr int kSt = (WITH_S ? 2 : 1) * kKv + kDv;  // uint4 per round
  static constexpr int kS = 0, kK = WITH_S ? kKv : 0, kD = kK + kKv;  // offsets in a round
  static constexpr int kTabVecs = kSt * 16 * NSTAGES;
  static constexpr int kFixFinWords = 2 * 3 * tdes_gen::kDeltaStride + 2 * 64;
  static constexpr int kVecs = kTabVecs + kFixFinWords / 4;
  const uint4* tab;
  const uint32_t* ff;
  template <class V>
  __device__ __forceinline__ void fixup(V (&P)[64], int b, uint32_t c) const {
    tdes_gen::fold_fixup_A<false>(P, ff + tdes_gen::kDeltaStride * b, ff + tdes_gen::kDeltaStride * (3 + b), c);
  }
  template <class V>
  __device__ __forceinline__ void unmask(V (&P)[64], uint32_t c) const {
    tdes_gen::fold_unmask<false>(P, ff + 6 * tdes_gen::kDeltaStride, ff + 6 * tdes_gen::kDeltaStride + 64, c);
  }
};

template <int NSTAGES>
struct ParamKeys {
  using T = KeyTable<NSTAGES, false>;
  const SKeys<16 * NSTAGES>& kp;
  T t;
  template <class V>
  __device__ __forceinline__ void fixup(V (&P)[64], int b, uint32_t c) const {
    tdes_gen::fold_fixup_A<false>(P, kp.fix_s[b], kp.fix_k[b], c);
  }
  template <class V>
  __device__ __forceinline__ void unmask(V (&P)[64], uint32_t c) const {
    tdes_gen::fold_unmask<false>(P, kp.fin_s, kp.fin_k, c);
  }
  template <class V>
  __device__ __forceinline__ void two_rounds(V (&P)[64], int r, uint32_t c) const {
    const uint4* t0 = t.tab + T::kSt * r;
    const uint4* t1 = t.tab + T::kSt * (r + 1);
    // s as uint2 pairs: every uniform load is 64-bit, also for an odd slot count
    const uint2* s0 = reinterpret_cast<const uint2*>(kp.s[r]);
    const uint2* s1 = reinterpret_cast<const uint2*>(kp.s[r + 1]);
    tdes_gen::round_A<false>(P, s0, t0 + T::kK, t0 + T::kD, c);
    tdes_gen::round_B<false>(P, s1, t1 + T::kK, t1 + T::kD, c);
  }
};

template <int NSTAGES>
struct DevKeys : KeyTable<NSTAGES, true> {
  using T = KeyTable<NSTAGES, true>;
  __device__ DevKeys(const uint4* tab, const uint32_t* ff) : T{tab, ff} {}
  template <class V>
  __device__ __forceinline__ void two_rounds(V (&P)[64], int r, uint32_t c) const {
    const uint4* t0 = this->tab + T::kSt * r;
    const uint4* t1 = this->tab + T::kSt * (r + 1);
    tdes_gen::round_A<false>(P, t0 + T::kS, t0 + T::kK, t0 + T::kD, c);
    tdes_gen::round_B<false>(P, t1 + T::kS, t1 + T::kK, t1 + T::kD, c);
  }
};

// Launch parameters of the key material (DEVKEYS: the packed subkeys only).
template <int NSTAGES, bool DEVKEYS>
using KeyParam = std::conditional_t<DEVKEYS, RoundKeys<16 * NSTAGES>, SKeys<16 * NSTAGES>>;

// The prologue's expansion: every operand word = key(a) ^ key(b) over OpRefs, the
// key bits taken from the packed subkeys (bit 47 - pos of round r = E-position pos).
// Two phases, so the reference-pair loads (global memory, L2) overlap the copy of
// the packed subkeys into shared memory: load_refs issues every load this thread
// needs at once (compile-time trip counts over kThreads threads), expand_keys
// combines them with the key bits once those are in shared memory.
template <int NSTAGES>
struct RefRegs {
  static constexpr int NR = 16 * NSTAGES;
  static constexpr int kSk = (NR * tdes_gen::kKeyStride + kThreads - 1) / kThreads;
  static constexpr int kD = (NR * tdes_gen::kDeltaStride + kThreads - 1) / kThreads;
  static constexpr int kFix = (3 * tdes_gen::kDeltaStride + kThreads - 1) / kThreads;
  static constexpr int kFin = (64 + kThreads - 1) / kThreads;
  uint32_t sk[kSk], d[kD], fix[kFix];  // two 16-bit references each
  uint16_t fin[kFin];
};

template <int NSTAGES>
__device__ __forceinline__ void load_refs(RefRegs<NSTAGES>& rr) {
  using namespace tdes_gen;
  using RR = RefRegs<NSTAGES>;
  const OpRefs<NSTAGES>& o = refs_dev<NSTAGES>();
  const uint32_t* sk = reinterpret_cast<const uint32_t*>(&o.sk[0][0][0]);
  const uint32_t* d = reinterpret_cast<const uint32_t*>(&o.d[0][0][0]);
  const uint32_t* fix = reinterpret_cast<const uint32_t*>(&o.fix[0][0][0]);
  const int t = threadIdx.x;
#pragma unroll
  for (int j = 0; j < RR::kSk; ++j) {
    const int i = t + j * kThreads;
    rr.sk[j] = i < RR::NR * kKeyStride ? sk[i] : 0xFFFFFFFFu;
  }
#pragma unroll
  for (int j = 0; j < RR::kD; ++j) {
    const int i = t + j * kThreads;
    rr.d[j] = i < RR::NR * kDeltaStride ? d[i] : 0xFFFFFFFFu;
  }
#pragma unroll
  for (int j = 0; j < RR::kFix; ++j) {
    const int i = t + j * kThreads;
    rr.fix[j] = i < 3 * kDeltaStride ? fix[i] : 0xFFFFFFFFu;
  }
#pragma unroll
  for (int j = 0; j < RR::kFin; ++j) {
    const int i = t + j * kThreads;
    rr.fin[j] = i < 64 ? o.fin[i] : kNoRef;
  }
}

template <int NSTAGES, bool WITH_S>
__device__ __forceinline__ void expand_keys(const RefRegs<NSTAGES>& rr, const uint64_t* kbits, uint4* smem) {
  using KT = KeyTable<NSTAGES, WITH_S>;
  using RR = RefRegs<NSTAGES>;
  using namespace tdes_gen;
  auto bit = [&](uint32_t ref) -> uint32_t {
    return ref == kNoRef ? 0u : 0u - (uint32_t)((kbits[ref / 48] >> (47 - ref % 48)) & 1u);
  };
  auto pair = [&](uint32_t two) { return bit(two & 0xFFFFu) ^ bit(two >> 16); };  // little endian: [0] low
  uint32_t* t32 = reinterpret_cast<uint32_t*>(smem);
  const int t = threadIdx.x;
#pragma unroll
  for (int j = 0; j < RR::kSk; ++j) {
    const int i = t + j * kThreads;
    if (i < RR::NR * kKeyStride) {
      const int r = i / kKeyStride, q = i % kKeyStride;
      const uint32_t v = pair(rr.sk[j]);
      if (WITH_S) t32[4 * (r * KT::kSt + KT::kS) + q] = v | 1u;  // s
      t32[4 * (r * KT::kSt + KT::kK) + q] = v;                   // k
    }
  }
#pragma unroll
  for (int j = 0; j < RR::kD; ++j) {
    const int i = t + j * kThreads;
    if (i < RR::NR * kDeltaStride) {
      const int r = i / kDeltaStride, u = i % kDeltaStride;
      t32[4 * (r * KT::kSt + KT::kD) + u] = pair(rr.d[j]);
    }
  }
  uint32_t* ff = t32 + 4 * KT::kTabVecs;
#pragma unroll
  for (int j = 0; j < RR::kFix; ++j) {
    const int i = t + j * kThreads;
    if (i < 3 * kDeltaStride) {
      const uint32_t v = pair(rr.fix[j]);
      ff[i] = v | 1u;
      ff[3 * kDeltaStride + i] = v;
    }
  }
#pragma unroll
  for (int j = 0; j < RR::kFin; ++j) {
    const int i = t + j * kThreads;
    if (i < 64) {
      const uint32_t v = bit(rr.fin[j]);
      ff[6 * kDeltaStride + i] = v | 1u;
      ff[6 * kDeltaStride + 64 + i] = v;
    }
  }
}

// NSTAGES = 3: fused 3DES (48 rounds); NSTAGES = 1: single DES (16 rounds).
// DEVKEYS: s from the shared-memory table too (DevKeys) instead of the launch
// parameters (ParamKeys).
// Work distribution: CTA c owns the contiguous tile range
// [ntiles*c/grid, ntiles*(c+1)/grid); its warps claim tiles one at a time
// from a shared-memory counter.  Warps of one SM progress at very different
// rates under the hardware's warp arbitration, so a static per-warp split
// leaves the SM waiting on its slowest warp (measured: 1.6-2x slower).
template <int NSTAGES, bool VEC4, bool DEVKEYS>
__global__ void __launch_bounds__(kThreads, kMinCtasPerSm)
tdes_ecb_kernel(const uint2* in, uint2* out, size_t nblocks,
                const __grid_constant__ KeyParam<NSTAGES, DEVKEYS> kp, uint32_t c) {
  using KT = KeyTable<NSTAGES, DEVKEYS>;
  __shared__ unsigned int next_tile;
  __shared__ uint64_t kbits[16 * NSTAGES];
  __shared__ uint4 ksm[KT::kVecs];  // the key table (9.9 KiB for 3DES; 17.4 KiB with s)
  const unsigned lane = threadIdx.x & 31u;
  const unsigned warp = threadIdx.x >> 5;
  const size_t ntiles = (nblocks + kTileBlocks - 1) / kTileBlocks;
  const size_t lo = ntiles * blockIdx.x / gridDim.x;
  const size_t hi = ntiles * (blockIdx.x + 1) / gridDim.x;
  extern __shared__ uint4 tma_buf[];  // kTma: [kWarps][kTileBytes / 16], dynamic
  __shared__ uint64_t tma_bar[kWarps];
  uint4* buf = tma_buf + warp * (kTileBytes / 16);
  // a tile is staged by TMA when it is full (16-byte aligned, VEC4 path)
  auto stageable = [&](size_t t) { return kTma && VEC4 && t < hi && (t + 1) * kTileBlocks <= nblocks; };
  // First tiles are assigned statically (warp w: lo + w) and their TMA copies are
  // issued before the key expansion, so the HBM latency of the first load overlaps
  // the prologue; later tiles come from the shared counter (starting at kWarps).
  if (threadIdx.x == 0) next_tile = kWarps;
  size_t tile = lo + warp;
  bool staged = stageable(tile);
  // key operands: reference pairs (global) in flight while the packed subkeys go
  // to shared memory (warp-uniform parameter loads); then expand
  // (Issuing these loads before the first-tile TMA copies shortens the prologue at
  // >= 2^24 blocks from ~5 to ~2.2 us -- they no longer queue behind 128 KiB of HBM
  // reads per SM -- but made whole launches 5-10 us slower (tools/exp/trace_drain.py,
  // ab_sizes.py), so the TMA copies go first.)
  RefRegs<NSTAGES> rr;
  if (kTma && lane == 0) {
    mbar_init(&tma_bar[warp]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (staged) tma_load(buf, in + tile * kTileBlocks, kTileBytes, &tma_bar[warp]);
  }
  load_refs<NSTAGES>(rr);
  for (int r = (int)warp; r < 16 * NSTAGES; r += kWarps) {
    const uint64_t v = kp.k[r];
    if (lane == 0) kbits[r] = v;
  }
  __syncthreads();
  expand_keys<NSTAGES, DEVKEYS>(rr, kbits, ksm);
  __syncthreads();
  auto claim = [&]() -> size_t {
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(&next_tile, 1u);
    return lo + __shfl_sync(0xffffffffu, t, 0);
  };
  using KV = std::conditional_t<DEVKEYS, DevKeys<NSTAGES>, ParamKeys<NSTAGES>>;
  const KV kv = [&]() {
    const uint32_t* ff = reinterpret_cast<const uint32_t*>(ksm + KT::kTabVecs);
    if constexpr (DEVKEYS)
      return KV(ksm, ff);
    else
      return KV{kp, KeyTable<NSTAGES, false>{ksm, ff}};
  }();
  uint32_t phase = 0;
  while (tile < hi) {
    size_t next = hi;
    bool next_staged = false;
    auto prefetch = [&]() {
      next = claim();
      next_staged = stageable(next);
      if (lane == 0 && next_staged) tma_load(buf, in + next * kTileBlocks, kTileBytes, &tma_bar[warp]);
    };
    crypt_tile<NSTAGES, VEC4>(in, out, tile * kTileBlocks, nblocks, lane, kv, c, buf, &tma_bar[warp], staged,
                              phase, prefetch);
    if (staged) phase ^= 1u;
    if (kTma) {
      tile = next;
      staged = next_staged;
    } else {
      tile = claim();
    }
  }
}

// ------------------------------------------------ small-N latency mode -----
// SURVEY NEXT-5.  With few tiles the main kernel runs each 1024-block tile on
// one warp, so a launch lasts as long as one warp's 48 serial rounds.  Here a
// team of 8 warps shares one tile: warp g evaluates S-box g (warp-uniform, no
// divergence) for all 32 block-groups of the tile (lane l = group l), i.e. the
// paper's idea of spreading one block's round over many threads,
// applied at S-box granularity.  The 64 planes x 32 groups of state live in
// shared memory (row stride 33 words: both the [group] and the [plane] access
// patterns are bank-conflict free); every thread keeps the 4 planes of each
// half that its S-box writes (P is a permutation, so these partition each
// half) in registers and publishes them after each update; one barrier per
// round.  Transposes are lane-parallel (5 shuffle butterfly stages).  From 149
// tiles on (more than one team per SM) teams of 4 warps run two adjacent S-boxes
// per warp (SPW = 2): two independent S-box chains per warp, one warp per SMSP.
// WPT = warps per team: 8 = one S-box per warp; 4 = two adjacent S-boxes per warp
// (two independent S-box chains per warp); 16 = half an S-box per warp (outputs
// 0-1 or 2-3: the compiler drops the gates only the other pair needs).  The
// launcher picks by size.
template <int WPT>
constexpr int kSplitThreads = 32 * WPT;  // one team
template <int WPT>
constexpr int kBoxesPerWarp = WPT >= 8 ? 1 : 8 / WPT;
template <int WPT>
constexpr int kOutsPerBox = WPT == 16 ? 2 : 4;
constexpr int kStride = 33;

// 32x32 bit transpose across a warp: lane i holds row i on entry; on exit lane
// j holds column j (bit i = entry lane i's bit j).  Stage s swaps bit s of the
// lane index with bit s of the bit index.
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, unsigned lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const uint32_t m0 = s == 16  ? 0x0000FFFFu
                        : s == 8 ? 0x00FF00FFu
                        : s == 4 ? 0x0F0F0F0Fu
                        : s == 2 ? 0x33333333u
                                 : 0x55555555u;  // bits whose index has bit s clear
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, s);
    const bool hi = (lane & s) != 0;
    const uint32_t t = __funnelshift_l(y, y, hi ? 32 - s : s);  // rotl: lanes with bit s move bits down
    const uint32_t keep = hi ? ~m0 : m0;
    x = (x & keep) | (t & ~keep);
  }
  return x;
}

// Team barrier.  bar.sync counts arriving threads per barrier id, so the warps
// may reach it from the different S-box cases of the specialised kernel.
template <int WPT>
__device__ __forceinline__ void team_sync() {
  asm volatile("bar.sync 0, %0;" ::"n"(kSplitThreads<WPT>) : "memory");
}

// Per-warp key material for the split kernel: s = k | 1 (+1 / -1) and k (0 / ~0)
// of the 6 key bits of each of this warp's S-boxes for every round (48 bytes per
// S-box and round: LDS.128s and no arithmetic between the load and the round's
// IMADs, so the loads issued before a barrier complete while the team waits).
// Measured against loading s only and rebuilding k = mulhi(c, s) before the
// barrier: see DESIGN.md §6.
template <int NB>
struct alignas(16) SplitRoundKeys {
  uint32_t s[6 * NB], k[6 * NB];
};
template <int WPT, int NROUNDS>
struct SplitKeys {
  SplitRoundKeys<kBoxesPerWarp<WPT>> r[WPT][NROUNDS];
};

// S-box j of warp G, and the first of its outputs the warp owns.
template <int WPT>
__device__ __forceinline__ int split_box(int G, int j) {
  return WPT == 16 ? G >> 1 : kBoxesPerWarp<WPT> * G + j;
}
template <int WPT>
__device__ __forceinline__ int split_out0(int G) {
  return WPT == 16 ? 2 * (G & 1) : 0;
}

// One round of the split kernel for warp G: read the E-windows of half IN from
// shared memory, key XOR (s, k prefetched a round earlier), the S-box(es), publish
// the planes of the other half this warp owns.
template <int WPT, int IN>
__device__ __forceinline__ void split_round(int G, uint32_t* st, const int (&win)[2][6 * kBoxesPerWarp<WPT>],
                                            const int (&own)[2][kBoxesPerWarp<WPT> * kOutsPerBox<WPT>],
                                            uint32_t (&H)[2][kBoxesPerWarp<WPT> * kOutsPerBox<WPT>],
                                            const uint32_t (&S)[6 * kBoxesPerWarp<WPT>],
                                            const uint32_t (&K)[6 * kBoxesPerWarp<WPT>]) {
  constexpr int OUT = 1 - IN, NB = kBoxesPerWarp<WPT>, NO = kOutsPerBox<WPT>;
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    uint32_t x[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) x[i] = tdes_gen::kxor<false>(st[win[IN][6 * j + i]], S[6 * j + i], K[6 * j + i], 0u);
    if constexpr (NO == 4) {
      tdes_gen::sbox_by_index(split_box<WPT>(G, j), x[0], x[1], x[2], x[3], x[4], x[5], H[OUT][4 * j],
                              H[OUT][4 * j + 1], H[OUT][4 * j + 2], H[OUT][4 * j + 3]);
    } else {  // half an S-box: the unused pair's results (and gates only they need) are dropped
      uint32_t u0 = 0u, u1 = 0u;
      if (split_out0<WPT>(G) == 0)
        tdes_gen::sbox_by_index(split_box<WPT>(G, j), x[0], x[1], x[2], x[3], x[4], x[5], H[OUT][0], H[OUT][1], u0,
                                u1);
      else
        tdes_gen::sbox_by_index(split_box<WPT>(G, j), x[0], x[1], x[2], x[3], x[4], x[5], u0, u1, H[OUT][0],
                                H[OUT][1]);
    }
  }
#pragma unroll
  for (int o = 0; o < NB * NO; ++o) st[own[OUT][o]] = H[OUT][o];
}

// Load round r's key operands of this warp (off the critical path: issued before
// the barrier that ends round r - 1).
template <int NB, int NROUNDS>
__device__ __forceinline__ void split_keys(const SplitRoundKeys<NB> (&ks)[NROUNDS], int r, uint32_t,
                                           uint32_t (&S)[6 * NB], uint32_t (&K)[6 * NB]) {
  const uint4* v = reinterpret_cast<const uint4*>(&ks[r]);
  uint32_t w[12 * NB];
#pragma unroll
  for (int q = 0; q < 3 * NB; ++q) {
    const uint4 a = v[q];
    w[4 * q] = a.x; w[4 * q + 1] = a.y; w[4 * q + 2] = a.z; w[4 * q + 3] = a.w;
  }
#pragma unroll
  for (int i = 0; i < 6 * NB; ++i) {
    S[i] = w[i];
    K[i] = w[6 * NB + i];
  }
}

// The 48 rounds of one tile for warp G (warp-uniform; GC >= 0: G = GC known at
// compile time, the S-box-specialised variant).  The rounds run in (A, B) / (B, A)
// pairs, so no per-round branch picks the half; the key operands of the next round
// are loaded before each barrier.  Measured (B200, back-to-back 3DES launches):
// 16.5 -> 14.4 us for 1-16 tiles, 16.5 -> 14.5 us at 2^17 blocks, 20.5 -> 18.5 us at
// 2^18.
template <int WPT, int NSTAGES, int GC>
__device__ __forceinline__ void split_rounds(int G_, uint32_t* st,
                                             const SplitRoundKeys<kBoxesPerWarp<WPT>> (&ks)[16 * NSTAGES],
                                             unsigned lane, uint32_t c) {
  constexpr int NB = kBoxesPerWarp<WPT>, NO = kOutsPerBox<WPT>;
  const int G = GC >= 0 ? GC : G_;
  int win[2][6 * NB], own[2][NB * NO];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int g = split_box<WPT>(G, j);
#pragma unroll
      for (int i = 0; i < 6; ++i) win[h][6 * j + i] = tdes_gen::kWin[h][g][i] * kStride + lane;
#pragma unroll
      for (int o = 0; o < NO; ++o) own[h][NO * j + o] = tdes_gen::kOwn[h][g][split_out0<WPT>(G) + o] * kStride + lane;
    }
  }
  uint32_t S[6 * NB], K[6 * NB];
  split_keys(ks, 0, c, S, K);
  team_sync<WPT>();
  uint32_t H[2][NB * NO];  // the planes of half A (0) and B (1) this warp writes
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int o = 0; o < NB * NO; ++o) H[h][o] = st[own[h][o]];
  // stage s round rr updates A iff (rr + s) is even: stages 0 and 2
  // run (A, B) pairs, stage 1 (B, A) pairs.  Updating A reads half B (IN = 1).
#pragma unroll
  for (int stage = 0; stage < NSTAGES; ++stage) {
#pragma unroll 1
    for (int rr = 0; rr < 16; rr += 2) {
      const int r = 16 * stage + rr;
      if (stage & 1) split_round<WPT, 0>(G, st, win, own, H, S, K);
      else split_round<WPT, 1>(G, st, win, own, H, S, K);
      split_keys(ks, r + 1, c, S, K);
      team_sync<WPT>();
      if (stage & 1) split_round<WPT, 1>(G, st, win, own, H, S, K);
      else split_round<WPT, 0>(G, st, win, own, H, S, K);
      if (r + 2 < 16 * NSTAGES) split_keys(ks, r + 2, c, S, K);
      team_sync<WPT>();
    }
  }
}

// The specialised rounds: a constant warp index per case (split_rounds is inlined
// and specialised), cases 0 .. WPT-1.
template <int WPT, int NSTAGES, int C0>
__device__ __forceinline__ void split_rounds_spec(int G, uint32_t* st,
                                                  const SplitRoundKeys<kBoxesPerWarp<WPT>> (&ks)[16 * NSTAGES],
                                                  unsigned lane, uint32_t c) {
  if constexpr (C0 < WPT) {
    if (G == C0) split_rounds<WPT, NSTAGES, C0>(G, st, ks, lane, c);
    else split_rounds_spec<WPT, NSTAGES, C0 + 1>(G, st, ks, lane, c);
  }
}

// The tile loop of warp G: load (lane-parallel transposes into the shared round
// state), the rounds, store.  SPEC: the rounds run in a copy specialised for the
// warp's S-box(es) (no per-round dispatch).  Only the rounds are specialised: the
// load and store stay outside the per-warp dispatch, where the compiler knows the
// warp is converged (inside it, every warp shuffle got a divergence fallback and
// the specialised kernel grew to 220 KB of code, slower than the dispatching one
// from 2^17 blocks on).
template <int WPT, int NSTAGES, bool SPEC>
__device__ __forceinline__ void split_body(int G, const uint2* in, uint2* out, size_t nblocks, uint32_t* st,
                                           const SplitRoundKeys<kBoxesPerWarp<WPT>> (&ks)[16 * NSTAGES],
                                           unsigned lane, uint32_t c) {
  constexpr int QW = 32 / WPT;  // 32-block groups per warp in the load and store
  const size_t ntiles = (nblocks + kGroupBlocks - 1) / kGroupBlocks;
  for (size_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const size_t base = tile * kGroupBlocks;
    // load: warp G takes groups QW*G .. QW*G + QW - 1 (32 consecutive blocks each)
#pragma unroll
    for (int qq = 0; qq < QW; ++qq) {
      const int q = QW * G + qq;
      const size_t b = base + 32 * q + lane;
      const uint2 v = b < nblocks ? __ldcs(in + b) : make_uint2(0u, 0u);
      st[lane * kStride + q] = warp_transpose32(v.x, lane);  // plane `lane` of group q
      st[(32 + lane) * kStride + q] = warp_transpose32(v.y, lane);
    }
    if (SPEC) {
      split_rounds_spec<WPT, NSTAGES, 0>(G, st, ks, lane, c);
      __syncwarp();  // converged again (keeps the store's shuffles free of divergence fallbacks)
    } else {
      split_rounds<WPT, NSTAGES, -1>(G, st, ks, lane, c);
    }
    // FP (renaming) + store: warp G writes the groups it loaded
#pragma unroll
    for (int qq = 0; qq < QW; ++qq) {
      const int q = QW * G + qq;
      const uint32_t wx = warp_transpose32(st[tdes_gen::kOutSrc[lane] * kStride + q], lane);
      const uint32_t wy = warp_transpose32(st[tdes_gen::kOutSrc[32 + lane] * kStride + q], lane);
      const size_t b = base + 32 * q + lane;
      if (b < nblocks) __stcs(out + b, make_uint2(wx, wy));
    }
    team_sync<WPT>();
  }
}

// SPEC: every warp runs the rounds in a copy specialised for its S-box (no per-round
// dispatch).  With the load and store outside the per-S-box switch (split_body) the
// kernel is 3.2 K instructions (51 KB) instead of 13.8 K, and it is faster at every
// split size: 128 tiles (C1) 14.2 -> 12.3 us back to back, 27.8 -> 23.4 us single
// (profiles/r02/split_spec_ab.txt), so auto mode always uses it; the dispatching
// variant stays as a -DTDES_SPLIT_SPEC_MAX=<tiles> experiment switch.
template <int NSTAGES, int WPT, bool SPEC>
__global__ void __launch_bounds__(kSplitThreads<WPT>)
tdes_split_kernel(const uint2* in, uint2* out, size_t nblocks,
                  const __grid_constant__ RoundKeys<16 * NSTAGES> mk, uint32_t c) {
  constexpr int NB = kBoxesPerWarp<WPT>;
  __shared__ uint32_t st[64 * kStride];
  __shared__ SplitKeys<WPT, 16 * NSTAGES> ks;
  const unsigned lane = threadIdx.x & 31u;
  const int g = threadIdx.x >> 5;  // this warp
  // the 6 subkey bits of each of this warp's S-boxes per round (bit 47 - b of the
  // packed subkey = E position b)
  for (int r = lane; r < 16 * NSTAGES; r += 32) {
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const uint32_t kb = (uint32_t)(mk.k[r] >> (42 - 6 * split_box<WPT>(g, j))) & 63u;
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        const uint32_t k = 0u - ((kb >> (5 - i)) & 1u);
        ks.r[g][r].s[6 * j + i] = k | 1u;
        ks.r[g][r].k[6 * j + i] = k;
      }
    }
  }
  __syncwarp();
  split_body<WPT, NSTAGES, SPEC>(g, in, out, nblocks, st, ks.r[g], lane, c);
}

// ------------------------------------------------------------ launching ---

constexpr int kMaxDevices = 64;
std::atomic<int> g_sms[kMaxDevices];
std::atomic<int> g_occ[kMaxDevices][2][2][2];  // [dev][stages==3][vec4][devkeys]

template <bool VEC4>
constexpr size_t kDynSmem = kTma && VEC4 ? (size_t)kWarps * kTileBytes : 0;

// Also raises the kernel's dynamic shared-memory limit (TMA buffers) once per device.
template <int NSTAGES, bool VEC4, bool DEVKEYS>
int occupancy(int dev) {
  int v = g_occ[dev][NSTAGES == 3][VEC4][DEVKEYS].load(std::memory_order_relaxed);
  if (v > 0) return v;
  int occ = 0;
  if (kDynSmem<VEC4> > 0)
    cudaFuncSetAttribute(tdes_ecb_kernel<NSTAGES, VEC4, DEVKEYS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kDynSmem<VEC4>);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tdes_ecb_kernel<NSTAGES, VEC4, DEVKEYS>, kThreads,
                                                    kDynSmem<VEC4>) != cudaSuccess ||
      occ <= 0)
    occ = kMinCtasPerSm;
  g_occ[dev][NSTAGES == 3][VEC4][DEVKEYS].store(occ, std::memory_order_relaxed);
  return occ;
}

int num_sms(int dev) {
  int v = g_sms[dev].load(std::memory_order_relaxed);
  if (v > 0) return v;
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
    sms = 148;
  g_sms[dev].store(sms, std::memory_order_relaxed);
  return sms;
}

using tdes_internal::cuda_fail;

// Caller guarantees nblocks <= SIZE_MAX >> 4 (so nblocks * 8 cannot wrap).
int check_buffers(const void* in, const void* out, size_t nblocks) {
  if (!in || !out) return TDES_ERR_INVALID_ARG;
  if (((uintptr_t)in | (uintptr_t)out) & 7u) return TDES_ERR_MISALIGNED;
  const uintptr_t a = (uintptr_t)in, b = (uintptr_t)out, len = (uintptr_t)nblocks * 8u;
  if (a != b && a < b + len && b < a + len) return TDES_ERR_OVERLAP;
  int rc = tdes_internal::check_device_pointer(in);
  if (rc == TDES_OK) rc = tdes_internal::check_device_pointer(out);
  return rc;
}

// Auto mode: the split (latency) kernel for launches of at most this many
// 1024-block tiles, the throughput kernel above (measured crossover).
constexpr size_t kSplitMaxTiles = 384;
#ifndef TDES_SPLIT_SPEC_MAX
#define TDES_SPLIT_SPEC_MAX 384
#endif
constexpr size_t kSplitSpecMaxTiles = TDES_SPLIT_SPEC_MAX;  // the S-box-specialised split kernel (tdes_split_kernel<., ., true>)
// Teams of 4 warps with two S-boxes each (SPW = 2) from this many tiles on, teams of
// 8 with one below: measured (B200, back to back) <= 16 tiles 10.3 vs 11.2-13.6 us,
// 128 tiles 12.3 both, 256 tiles 16.4 vs 14.7 us (profiles/r02/split_spw_ab.txt).
#ifndef TDES_SPLIT_SPW2_MIN
#define TDES_SPLIT_SPW2_MIN 149
#endif
constexpr size_t kSplitSpw2MinTiles = TDES_SPLIT_SPW2_MIN;
// Team size below kSplitSpw2MinTiles (experiment switch: 8 or 16 warps).
#ifndef TDES_SPLIT_SMALL_WPT
#define TDES_SPLIT_SMALL_WPT 8
#endif
constexpr int kSplitSmallWpt = TDES_SPLIT_SMALL_WPT;
// Auto mode uses the throughput kernel whose s operands stay in the launch
// parameters (mode 1) above kSplitMaxTiles.  (Until its prologue expanded k and d
// on the device and issued the first tile's TMA copy before that expansion, the
// all-device-keys variant, mode 3, started ~2 us sooner and was used up to 768
// tiles; now mode 1 is as fast or faster at every size: tools/exp/size_timing.py,
// profiles/sizes_r02.txt.)

// Host: the operand words for key masks `masks` (consumption order, 0 / ~0).
template <int NSTAGES>
void build_masks(const uint32_t (*masks)[48], RoundMasks<16 * NSTAGES>& mk) {
  using namespace tdes_gen;
  constexpr int NR = 16 * NSTAGES;
  const OpRefs<NSTAGES>& o = refs_host<NSTAGES>();
  auto bit = [&](uint16_t ref) -> uint32_t { return ref == kNoRef ? 0u : (masks[ref / 48][ref % 48] ? ~0u : 0u); };
  memset(&mk, 0, sizeof mk);
  for (int r = 0; r < NR; ++r) {
    for (int q = 0; q < kKeySlots; ++q) {
      const uint32_t v = bit(o.sk[r][q][0]) ^ bit(o.sk[r][q][1]);
      mk.s[r][q] = v | 1u;  // s = k | 1
      mk.k[r][q] = v;
    }
    for (int u = 0; u < kFoldFree; ++u) mk.d[r][u] = bit(o.d[r][u][0]) ^ bit(o.d[r][u][1]);
  }
  for (int b = 0; b < 3; ++b)
    for (int t = 0; t < kFoldFree; ++t) {
      const uint32_t v = bit(o.fix[b][t][0]) ^ bit(o.fix[b][t][1]);
      mk.fix_s[b][t] = v | 1u;
      mk.fix_k[b][t] = v;
    }
  for (int j = 0; j < 64; ++j) {
    mk.fin_s[j] = bit(o.fin[j]) | 1u;
    mk.fin_k[j] = bit(o.fin[j]);
  }
}

// The consumption-order key masks packed one 48-bit word per round (bit 47 - b =
// E-position b): the 384-byte launch parameter of the split kernel and of the
// device-key throughput kernel.
template <int NSTAGES>
RoundKeys<16 * NSTAGES> pack_keys(const uint32_t (*masks)[48]) {
  RoundKeys<16 * NSTAGES> ms;
  for (int r = 0; r < 16 * NSTAGES; ++r) {
    uint64_t w = 0;
    for (int b = 0; b < 48; ++b) w = (w << 1) | (masks[r][b] ? 1u : 0u);
    ms.k[r] = w;
  }
  return ms;
}

// build_masks costs ~10 us of host time per call; launches with the same key
// material (the common case: one key, many launches) reuse the result.  Two
// entries per thread and variant, so alternating encrypt/decrypt also hits.
template <int NSTAGES>
const SKeys<16 * NSTAGES>& cached_skeys(const uint32_t (*masks)[48]) {
  struct Entry {
    uint32_t key[16 * NSTAGES][48];
    SKeys<16 * NSTAGES> sk;
    bool valid = false;
  };
  thread_local Entry cache[2];
  thread_local int next = 0;
  for (Entry& e : cache)
    if (e.valid && memcmp(e.key, masks, sizeof e.key) == 0) return e.sk;
  Entry& e = cache[next];
  next ^= 1;
  memcpy(e.key, masks, sizeof e.key);
  RoundMasks<16 * NSTAGES> mk;
  build_masks<NSTAGES>(masks, mk);
  memcpy(e.sk.s, mk.s, sizeof e.sk.s);
  memcpy(e.sk.fix_s, mk.fix_s, sizeof e.sk.fix_s);
  memcpy(e.sk.fix_k, mk.fix_k, sizeof e.sk.fix_k);
  memcpy(e.sk.fin_s, mk.fin_s, sizeof e.sk.fin_s);
  memcpy(e.sk.fin_k, mk.fin_k, sizeof e.sk.fin_k);
  const RoundKeys<16 * NSTAGES> pk = pack_keys<NSTAGES>(masks);
  memcpy(e.sk.k, pk.k, sizeof e.sk.k);
  e.valid = true;
  return e.sk;
}

// The packed subkeys (the split kernel's and mode 3's launch parameter), cached the
// same way: packing costs ~2 us of host time per call, a hit one 9 KB memcmp.
template <int NSTAGES>
const RoundKeys<16 * NSTAGES>& cached_rkeys(const uint32_t (*masks)[48]) {
  struct Entry {
    uint32_t key[16 * NSTAGES][48];
    RoundKeys<16 * NSTAGES> rk;
    bool valid = false;
  };
  thread_local Entry cache[2];
  thread_local int next = 0;
  for (Entry& e : cache)
    if (e.valid && memcmp(e.key, masks, sizeof e.key) == 0) return e.rk;
  Entry& e = cache[next];
  next ^= 1;
  memcpy(e.key, masks, sizeof e.key);
  e.rk = pack_keys<NSTAGES>(masks);
  e.valid = true;
  return e.rk;
}

template <int NSTAGES, bool DEVKEYS>
cudaError_t launch_throughput(const KeyParam<NSTAGES, DEVKEYS>& kp, const uint2* pin, uint2* pout, size_t nblocks,
                              bool vec4, int dev, cudaStream_t stream) {
  // one resident CTA per SM; with fewer tiles than SMs, one tile per CTA
  const size_t ntiles = (nblocks + kTileBlocks - 1) / kTileBlocks;
  const int occ = vec4 ? occupancy<NSTAGES, true, DEVKEYS>(dev) : occupancy<NSTAGES, false, DEVKEYS>(dev);
  const size_t resident = (size_t)num_sms(dev) * (size_t)occ;
  const unsigned grid = (unsigned)(ntiles < resident ? ntiles : resident);
  if (vec4)
    tdes_ecb_kernel<NSTAGES, true, DEVKEYS><<<grid, kThreads, kDynSmem<true>, stream>>>(pin, pout, nblocks, kp,
                                                                                         kMulhiC);
  else
    tdes_ecb_kernel<NSTAGES, false, DEVKEYS><<<grid, kThreads, kDynSmem<false>, stream>>>(pin, pout, nblocks, kp,
                                                                                           kMulhiC);
  return cudaGetLastError();
}

// mode: 0 auto, 1 throughput kernel (host-folded key operands), 2 split
// (latency) kernel, 3 throughput kernel with device-expanded key operands.
template <int NSTAGES>
int launch(const uint32_t (*masks)[48], const void* in, void* out, size_t nblocks,
           cudaStream_t stream, int mode = 0) {
  if (nblocks == 0) return TDES_OK;
  if (nblocks > (SIZE_MAX >> 4)) return TDES_ERR_INVALID_ARG;
  const int rc = check_buffers(in, out, nblocks);
  if (rc) return rc;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e);
  if (dev < 0 || dev >= kMaxDevices) return TDES_ERR_INVALID_ARG;
  const bool vec4 = (((uintptr_t)in | (uintptr_t)out) & 15u) == 0;
  const size_t ngroups = (nblocks + kGroupBlocks - 1) / kGroupBlocks;
  if (mode == 2 || (mode == 0 && ngroups <= kSplitMaxTiles)) {
    const size_t cap = (size_t)num_sms(dev) * 8u;  // up to 8 teams per SM
    const unsigned sgrid = (unsigned)(ngroups < cap ? ngroups : cap);
    const RoundKeys<16 * NSTAGES>& ms = cached_rkeys<NSTAGES>(masks);
    const uint2* pin = static_cast<const uint2*>(in);
    uint2* pout = static_cast<uint2*>(out);
    const bool spec = ngroups <= kSplitSpecMaxTiles;
    if (ngroups < kSplitSpw2MinTiles) {
      if (spec)
        tdes_split_kernel<NSTAGES, kSplitSmallWpt, true><<<sgrid, kSplitThreads<kSplitSmallWpt>, 0, stream>>>(
            pin, pout, nblocks, ms, kMulhiC);
      else
        tdes_split_kernel<NSTAGES, kSplitSmallWpt, false><<<sgrid, kSplitThreads<kSplitSmallWpt>, 0, stream>>>(
            pin, pout, nblocks, ms, kMulhiC);
    } else {
      if (spec)
        tdes_split_kernel<NSTAGES, 4, true><<<sgrid, kSplitThreads<4>, 0, stream>>>(pin, pout, nblocks, ms, kMulhiC);
      else
        tdes_split_kernel<NSTAGES, 4, false><<<sgrid, kSplitThreads<4>, 0, stream>>>(pin, pout, nblocks, ms, kMulhiC);
    }
    e = cudaGetLastError();
    return e == cudaSuccess ? TDES_OK : cuda_fail(e);
  }
  const uint2* pin = static_cast<const uint2*>(in);
  uint2* pout = static_cast<uint2*>(out);
  if (mode == 3)
    e = launch_throughput<NSTAGES, true>(cached_rkeys<NSTAGES>(masks), pin, pout, nblocks, vec4, dev, stream);
  else
    e = launch_throughput<NSTAGES, false>(cached_skeys<NSTAGES>(masks), pin, pout, nblocks, vec4, dev, stream);
  if (e != cudaSuccess) return cuda_fail(e);
  return TDES_OK;
}

}  // namespace

extern "C" int tdes_ecb_encrypt(const tdes_schedule* s, const void* in, void* out, size_t nblocks,
                                tdes_stream_t stream) {
  if (!s) return TDES_ERR_INVALID_ARG;
  return launch<3>(s->mask[0], in, out, nblocks, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int tdes_ecb_decrypt(const tdes_schedule* s, const void* in, void* out, size_t nblocks,
                                tdes_stream_t stream) {
  if (!s) return TDES_ERR_INVALID_ARG;
  return launch<3>(s->mask[1], in, out, nblocks, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int tdes_ecb_crypt_mode(const tdes_schedule* s, int decrypt, const void* in, void* out,
                                   size_t nblocks, int mode, tdes_stream_t stream) {
  if (!s || (decrypt != 0 && decrypt != 1) || mode < 0 || mode > 3) return TDES_ERR_INVALID_ARG;
  return launch<3>(s->mask[decrypt], in, out, nblocks, reinterpret_cast<cudaStream_t>(stream), mode);
}

extern "C" int des_ecb_encrypt(const des_schedule* s, const void* in, void* out, size_t nblocks,
                               tdes_stream_t stream) {
  if (!s) return TDES_ERR_INVALID_ARG;
  return launch<1>(s->mask[0], in, out, nblocks, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int des_ecb_decrypt(const des_schedule* s, const void* in, void* out, size_t nblocks,
                               tdes_stream_t stream) {
  if (!s) return TDES_ERR_INVALID_ARG;
  return launch<1>(s->mask[1], in, out, nblocks, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int tdes_ecb_crypt_host(const tdes_schedule* s, int decrypt, const void* host_in,
                                   void* host_out, size_t nblocks, void* workspace,
                                   size_t workspace_bytes, size_t chunk_blocks,
                                   const tdes_stream_t* streams, int nstreams) {
  if (!s || (decrypt != 0 && decrypt != 1) || nstreams <= 0 || !streams || chunk_blocks == 0)
    return TDES_ERR_INVALID_ARG;
  if (nblocks == 0) return TDES_OK;
  if (!host_in || !host_out || !workspace) return TDES_ERR_INVALID_ARG;
  if (((uintptr_t)workspace & 15u) || (chunk_blocks & 1u)) return TDES_ERR_MISALIGNED;
  if (workspace_bytes / 8u / (size_t)nstreams < chunk_blocks) return TDES_ERR_WORKSPACE;
  if (nblocks > (SIZE_MAX >> 4)) return TDES_ERR_INVALID_ARG;
  const uint8_t* src = static_cast<const uint8_t*>(host_in);
  uint8_t* dst = static_cast<uint8_t*>(host_out);
  const size_t chunk_bytes = chunk_blocks * 8u;
  // On a failure part-way through, copies already queued on the other streams
  // still read host_in / write host_out and the workspace: wait for all of them
  // before returning, so the caller may free or reuse the buffers at once.
  auto drain = [&](int rc) {
    for (int i = 0; i < nstreams; ++i) (void)cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(streams[i]));
    return rc;
  };
  size_t c = 0;
  for (size_t off = 0; off < nblocks; off += chunk_blocks, ++c) {
    const size_t nb = nblocks - off < chunk_blocks ? nblocks - off : chunk_blocks;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(streams[c % (size_t)nstreams]);
    uint8_t* dev = static_cast<uint8_t*>(workspace) + (c % (size_t)nstreams) * chunk_bytes;
    cudaError_t e = cudaMemcpyAsync(dev, src + off * 8u, nb * 8u, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return drain(cuda_fail(e));
    const int rc = launch<3>(s->mask[decrypt], dev, dev, nb, st);
    if (rc) return drain(rc);
    e = cudaMemcpyAsync(dst + off * 8u, dev, nb * 8u, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return drain(cuda_fail(e));
  }
  for (int i = 0; i < nstreams; ++i) {
    const cudaError_t e = cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(streams[i]));
    if (e != cudaSuccess) return cuda_fail(e);
  }
  return TDES_OK;
}

extern "C" int tdes_get_kernel_info(tdes_kernel_info* out) {
  if (!out) return TDES_ERR_INVALID_ARG;
  out->sbox_lop3_total = tdes_gen::kSboxLop3Total;
  for (int g = 0; g < 8; ++g) out->sbox_lop3[g] = tdes_gen::kSboxLop3[g];
  out->threads_per_cta = kThreads;
  out->blocks_per_thread = kBlocksPerThread;
  out->min_ctas_per_sm = kMinCtasPerSm;
  return TDES_OK;
}

namespace tdes_internal {
namespace {
thread_local int g_last_cuda_error = 0;
}
int cuda_fail(cudaError_t e) {
  g_last_cuda_error = (int)e;
  return TDES_ERR_CUDA;
}
int check_device_pointer(const void* p) {
#ifdef TDES_DEBUG
  cudaPointerAttributes a;
  const cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();  // not sticky: clear it
    return TDES_ERR_INVALID_ARG;
  }
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) return TDES_ERR_INVALID_ARG;
  if ((a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) || a.device != dev)
    return TDES_ERR_INVALID_ARG;
#else
  (void)p;
#endif
  return TDES_OK;
}
}  // namespace tdes_internal

extern "C" int tdes_last_cuda_error(void) { return tdes_internal::g_last_cuda_error; }

extern "C" int tdes_fold_operands(const tdes_schedule* s, int decrypt, uint32_t* out, size_t out_words,
                                  size_t* words, int* geom) {
  if (!s || !words || (decrypt != 0 && decrypt != 1)) return TDES_ERR_INVALID_ARG;
  static_assert(sizeof(RoundMasks<48>) % sizeof(uint32_t) == 0, "word-sized layout");
  *words = sizeof(RoundMasks<48>) / sizeof(uint32_t);
  if (geom) {
    geom[0] = tdes_gen::kKeySlots;
    geom[1] = tdes_gen::kKeyStride;
    geom[2] = tdes_gen::kFoldFree;
    geom[3] = tdes_gen::kDeltaStride;
  }
  if (!out || out_words < *words) return TDES_ERR_WORKSPACE;
  RoundMasks<48> mk;
  build_masks<3>(s->mask[decrypt], mk);
  memcpy(out, &mk, sizeof mk);
  return TDES_OK;
}

extern "C" int tdes_device_geometry(int* sms, int* ctas_per_sm) {
  if (!sms || !ctas_per_sm) return TDES_ERR_INVALID_ARG;
  int dev = 0;
  const cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e);
  if (dev < 0 || dev >= kMaxDevices) return TDES_ERR_INVALID_ARG;
  *sms = num_sms(dev);
  *ctas_per_sm = occupancy<3, true, false>(dev);
  return TDES_OK;
}
