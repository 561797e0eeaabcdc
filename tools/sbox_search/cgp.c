/*
 * cgp.c -- gate-count reduction of finished 3-input-LUT (LOP3) circuits for one
 * DES S-box by Cartesian Genetic Programming with neutral drift.
 *
 * The greedy decomposition search (sbox_search.c) stalls at a local optimum; CGP
 * explores the space of *correct* circuits around it: a (1 + lambda) evolution
 * strategy mutates a few genes (a gate's LUT byte, one of its three inputs, or an
 * output's source) and accepts the child when it is still exact on all 64 inputs
 * of all four outputs and uses no more active gates than the parent.  Equal-cost
 * moves drift through the neutral network; a move that disconnects a gate lowers
 * the cost.  The cost model is the kernel's (tools/gen_tdes.py circuit_cost):
 * active gates only -- every output costs one LOP3 into its destination plane
 * whether it is a plain signal (XOR or XNOR) or fused as a 2-input join
 * h(u, v) of two signals (one LOP3(P, u, v), no gate).
 *
 * Input (stdin): one line  "<t0> <t1> <t2> <t3>"  (64-bit truth tables, hex),
 *   one line "<ngates>", ngates lines "<lut> <a> <b> <c>", then four output lines
 *   "p <sig> <neg>" or "f <u> <v> <h>".
 * Usage: cgp <seconds> <seed> <slack> [lambda] [depth_mode]
 *   slack = extra (initially inactive) gate slots available to the search.
 *   depth_mode = 2: budget mode -- fitness = wrong output bits + W x (active gates
 *   above the best count - 1), W = argv[6] (default 16); a child is accepted if its
 *   fitness is no worse, so the search may give up exactness to drop a gate and
 *   then drift back to an exact circuit one gate smaller (printed when found).
 *   depth_mode = 5: fold credit -- neutral drift on exact circuits minimising
 *   gates - foldable outputs (a fold saves the round a key IMAD and its loads,
 *   measured worth about one gate: profiles/r02/circuits_ab.txt), never above the
 *   starting gate count, depth within 2 of the start; prints every improvement.
 *   depth_mode = 4: sample -- neutral drift among exact circuits of at most the
 *   starting gate count, printing the current circuit every 2^L generations
 *   (L = argv[6], default 22; smaller L = variants closer to the start)
 *   (structurally different equal-cost alternatives, for measured selection);
 *   argv[7] (default 0) lets the drift use that many gates more than the start
 *   (tools/run_resub.py then resubstitutes each sample).
 *   depth_mode = 3: polish -- minimise (gates, -foldable outputs, depth) (a folded
 *   output saves the round one key IMAD; measured worth about half a gate).
 *   depth_mode = 1: minimise (gates, depth) lexicographically -- a child is accepted
 *   only if it is no worse in either order, and every strictly better circuit is
 *   printed (used to bring a reduced circuit's depth back down: a deeper S-box
 *   lengthens the round's critical path).
 * Output (stdout): every strictly better circuit found, as one JSON line
 *   {"gates": [[lut, a, b, c], ...], "outputs": [...], "neg": [...], "fuse": [...]}
 * with inactive gates removed and signals renumbered.  Exact verification is
 * repeated by the caller (tools/run_cgp.py) and by tools/gen_tdes.py.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define MAXN 64
typedef uint64_t tt_t;

typedef struct {
  uint8_t lut[MAXN];
  uint8_t in[MAXN][3];
  int otype[4];  /* 0 plain, 1 fused */
  int osig[4], oneg[4];
  int ou[4], ov[4], oh[4];
} G;

static int N;  /* gate slots */
static tt_t VARS[6], TGT[4];

static inline uint64_t rnd(uint64_t *s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* PTX lop3 semantics: bit of result = lut[(a << 2) | (b << 1) | c]. */
static inline tt_t lut3(unsigned lut, tt_t a, tt_t b, tt_t c) {
  const tt_t m7 = -(tt_t)((lut >> 7) & 1), m6 = -(tt_t)((lut >> 6) & 1), m5 = -(tt_t)((lut >> 5) & 1),
             m4 = -(tt_t)((lut >> 4) & 1), m3 = -(tt_t)((lut >> 3) & 1), m2 = -(tt_t)((lut >> 2) & 1),
             m1 = -(tt_t)((lut >> 1) & 1), m0 = -(tt_t)(lut & 1);
  const tt_t hi = (c & m7) | (~c & m6), lo_a1 = (c & m5) | (~c & m4);  /* a=1: b=1 / b=0 */
  const tt_t b1a0 = (c & m3) | (~c & m2), b0a0 = (c & m1) | (~c & m0);
  const tt_t a1 = (b & hi) | (~b & lo_a1), a0 = (b & b1a0) | (~b & b0a0);
  return (a & a1) | (~a & a0);
}

static inline tt_t h2(unsigned h, tt_t u, tt_t v) {  /* h index = (u << 1) | v */
  tt_t r = 0;
  if (h & 1) r |= ~u & ~v;
  if (h & 2) r |= ~u & v;
  if (h & 4) r |= u & ~v;
  if (h & 8) r |= u & v;
  return r;
}

/* Marks active gates; returns their number. */
static int active(const G *g, uint8_t *act) {
  memset(act, 0, N);
  int stack[4 * MAXN], sp = 0, cnt = 0;
  for (int o = 0; o < 4; o++) {
    if (g->otype[o] == 0) stack[sp++] = g->osig[o];
    else { stack[sp++] = g->ou[o]; stack[sp++] = g->ov[o]; }
  }
  while (sp) {
    const int s = stack[--sp];
    if (s < 6) continue;
    const int k = s - 6;
    if (act[k]) continue;
    act[k] = 1;
    cnt++;
    for (int j = 0; j < 3; j++) stack[sp++] = g->in[k][j];
  }
  return cnt;
}

/* Number of wrong output bits (0 = exact). */
static int errors(const G *g, const uint8_t *act) {
  tt_t sig[6 + MAXN];
  for (int i = 0; i < 6; i++) sig[i] = VARS[i];
  for (int k = 0; k < N; k++)
    if (act[k]) sig[6 + k] = lut3(g->lut[k], sig[g->in[k][0]], sig[g->in[k][1]], sig[g->in[k][2]]);
  int e = 0;
  for (int o = 0; o < 4; o++) {
    tt_t v = g->otype[o] == 0 ? sig[g->osig[o]] ^ (g->oneg[o] ? ~0ull : 0ull)
                              : h2(g->oh[o], sig[g->ou[o]], sig[g->ov[o]]);
    e += __builtin_popcountll(v ^ TGT[o]);
  }
  return e;
}

static int depth(const G *g, const uint8_t *act) {
  int d[6 + MAXN] = {0}, best = 0;
  for (int k = 0; k < N; k++) {
    if (!act[k]) continue;
    int m = 0;
    for (int j = 0; j < 3; j++) if (d[g->in[k][j]] > m) m = d[g->in[k][j]];
    d[6 + k] = m + 1;
  }
  for (int o = 0; o < 4; o++) {
    int v = g->otype[o] == 0 ? d[g->osig[o]] : (d[g->ou[o]] > d[g->ov[o]] ? d[g->ou[o]] : d[g->ov[o]]);
    if (v > best) best = v;
  }
  return best;
}

/* Outputs whose Feistel XOR can also fold a key mask (tools/gen_tdes.py
 * fold_producers): an unfused output, or a fused XOR/XNOR join one of whose
 * operands is a gate with at most two distinct inputs and no other consumer. */
static int foldable(const G *g, const uint8_t *act) {
  int uses[6 + MAXN] = {0};
  for (int k = 0; k < N; k++) {
    if (!act[k]) continue;
    const int a = g->in[k][0], b = g->in[k][1], c = g->in[k][2];
    uses[a]++;
    if (b != a) uses[b]++;
    if (c != a && c != b) uses[c]++;
  }
  for (int o = 0; o < 4; o++)
    if (g->otype[o]) {
      uses[g->ou[o]]++;
      if (g->ov[o] != g->ou[o]) uses[g->ov[o]]++;
    }
  int n = 0;
  for (int o = 0; o < 4; o++) {
    if (g->otype[o] == 0) { n++; continue; }
    if (g->oh[o] != 6 && g->oh[o] != 9) continue;
    const int sg[2] = {g->ou[o], g->ov[o]};
    for (int j = 0; j < 2; j++) {
      const int x = sg[j];
      if (x < 6) continue;
      const int k = x - 6, a = g->in[k][0], b = g->in[k][1], c = g->in[k][2];
      const int distinct = 1 + (b != a) + (c != a && c != b);
      if (distinct <= 2 && uses[x] == 1) { n++; break; }
    }
  }
  return n;
}

static void mutate(G *g, uint64_t *rs) {
  const int nm = 1 + (int)(rnd(rs) % 3);
  for (int t = 0; t < nm; t++) {
    const uint64_t r = rnd(rs);
    const int pick = (int)(r % (4 * N + 8));
    if (pick < 4 * N) {
      const int k = pick / 4, f = pick % 4;
      if (f == 3) g->lut[k] = (uint8_t)(rnd(rs) & 0xFF);
      else g->in[k][f] = (uint8_t)(rnd(rs) % (uint64_t)(6 + k));
    } else {
      const int o = (pick - 4 * N) % 4;
      const int ns = 6 + N;
      if (((r >> 32) & 7) == 0) g->otype[o] ^= 1;
      if (g->otype[o] == 0) {
        g->osig[o] = (int)(rnd(rs) % (uint64_t)ns);
        g->oneg[o] = (int)(rnd(rs) & 1);
      } else {
        const uint64_t q = rnd(rs);
        if (q & 1) g->ou[o] = (int)(rnd(rs) % (uint64_t)ns);
        if (q & 2) g->ov[o] = (int)(rnd(rs) % (uint64_t)ns);
        if ((q & 12) || !(q & 3)) g->oh[o] = (int)(rnd(rs) & 15);
      }
    }
  }
}

static void print_json(const G *g) {
  uint8_t act[MAXN];
  active(g, act);
  int map[6 + MAXN];
  for (int i = 0; i < 6; i++) map[i] = i;
  int n = 0;
  for (int k = 0; k < N; k++) map[6 + k] = act[k] ? 6 + n++ : -1;
  printf("{\"gates\": [");
  int first = 1;
  for (int k = 0; k < N; k++) {
    if (!act[k]) continue;
    printf("%s[%d, %d, %d, %d]", first ? "" : ", ", g->lut[k], map[g->in[k][0]], map[g->in[k][1]], map[g->in[k][2]]);
    first = 0;
  }
  printf("], \"outputs\": [");
  for (int o = 0; o < 4; o++) printf("%s%d", o ? ", " : "", g->otype[o] == 0 ? map[g->osig[o]] : -1);
  printf("], \"neg\": [");
  for (int o = 0; o < 4; o++) printf("%s%d", o ? ", " : "", g->otype[o] == 0 ? g->oneg[o] : 0);
  printf("], \"fuse\": [");
  for (int o = 0; o < 4; o++) {
    if (g->otype[o] == 0) printf("%snull", o ? ", " : "");
    else printf("%s[%d, %d, %d]", o ? ", " : "", map[g->ou[o]], map[g->ov[o]], g->oh[o]);
  }
  printf("], \"depth\": %d}\n", depth(g, act));
  fflush(stdout);
}

int main(int argc, char **argv) {
  if (argc < 4) {
    fprintf(stderr, "usage: cgp <seconds> <seed> <slack> [lambda]\n");
    return 2;
  }
  const double secs = atof(argv[1]);
  uint64_t rs = strtoull(argv[2], 0, 10) * 0x9E3779B97F4A7C15ull + 1;
  const int slack = atoi(argv[3]);
  const int lambda = argc > 4 ? atoi(argv[4]) : 4;
  const int depth_mode = argc > 5 ? atoi(argv[5]) : 0;
  const int weight = argc > 6 ? atoi(argv[6]) : 16;
  for (int i = 0; i < 6; i++) {
    VARS[i] = 0;
    for (int v = 0; v < 64; v++) if ((v >> (5 - i)) & 1) VARS[i] |= 1ull << v;
  }
  if (scanf("%lx %lx %lx %lx", &TGT[0], &TGT[1], &TGT[2], &TGT[3]) != 4) return 2;
  int n0;
  if (scanf("%d", &n0) != 1 || n0 + slack > MAXN) return 2;
  G p;
  memset(&p, 0, sizeof p);
  /* the given gates keep their order; `slack` inactive random slots are spread
     between them so that any gate can later be rewired through one */
  N = n0 + slack;
  int pos[6 + MAXN];
  for (int i = 0; i < 6; i++) pos[i] = i;
  for (int k = 0; k < n0; k++) pos[6 + k] = 6 + k + (int)(((long)(k + 1) * slack) / (n0 + 1));
  uint8_t used[MAXN] = {0};
  for (int k = 0; k < n0; k++) used[pos[6 + k] - 6] = 1;
  for (int k = 0; k < N; k++)
    if (!used[k]) {
      p.lut[k] = (uint8_t)(rnd(&rs) & 0xFF);
      for (int j = 0; j < 3; j++) p.in[k][j] = (uint8_t)(rnd(&rs) % (uint64_t)(6 + k));
    }
  for (int k = 0; k < n0; k++) {
    int lut, a, b, c;
    if (scanf("%d %d %d %d", &lut, &a, &b, &c) != 4) return 2;
    const int s[3] = {a, b, c}, slot = pos[6 + k] - 6;
    p.lut[slot] = (uint8_t)lut;
    for (int j = 0; j < 3; j++) p.in[slot][j] = (uint8_t)pos[s[j]];
  }
  for (int o = 0; o < 4; o++) {
    char t[4];
    int x, y, z;
    if (scanf("%3s %d %d", t, &x, &y) != 3) return 2;
    if (t[0] == 'p') {
      p.otype[o] = 0;
      p.osig[o] = pos[x];
      p.oneg[o] = y;
    } else {
      if (scanf("%d", &z) != 1) return 2;
      p.otype[o] = 1;
      p.ou[o] = pos[x];
      p.ov[o] = pos[y];
      p.oh[o] = z;
    }
  }
  uint8_t act[MAXN];
  int pc = active(&p, act);
  if (errors(&p, act) != 0) {
    fprintf(stderr, "initial circuit is not exact\n");
    return 3;
  }
  int pd = depth(&p, act), best = pc, bestd = pd;
  const int d0 = pd;
  fprintf(stderr, "start: %d gates, depth %d\n", pc, pd);
  const clock_t t0 = clock();
  long gen = 0;
  if (depth_mode == 5) {
    const int g0 = pc;
    int pcost = pc - foldable(&p, act), bcost = pcost;
    fprintf(stderr, "fold-credit start: %d gates, cost %d, depth %d\n", pc, pcost, pd);
    for (;;) {
      if ((++gen & 0xFFFF) == 0 && (double)(clock() - t0) / CLOCKS_PER_SEC > secs) break;
      for (int l = 0; l < lambda; l++) {
        G c = p;
        mutate(&c, &rs);
        uint8_t ca[MAXN];
        const int cc = active(&c, ca);
        if (cc > g0 || errors(&c, ca) != 0) continue;
        const int ccost = cc - foldable(&c, ca), cd = depth(&c, ca);
        if (ccost > pcost || cd > d0 + 2) continue;
        p = c;
        pcost = ccost;
        if (ccost < bcost) {
          bcost = ccost;
          fprintf(stderr, "gen %ld: %d gates, cost %d, depth %d\n", gen, cc, ccost, cd);
          print_json(&p);
        }
        break;
      }
    }
    fprintf(stderr, "done: %ld generations, best cost %d\n", gen, bcost);
    return 0;
  }
  if (depth_mode == 4) {
    const int cap = pc + (argc > 7 ? atoi(argv[7]) : 0);  /* argv[7]: drift up to this many gates more */
    const long every = (1L << (argc > 6 ? atoi(argv[6]) : 22)) - 1;
    for (;;) {
      if ((++gen & 0xFFFF) == 0 && (double)(clock() - t0) / CLOCKS_PER_SEC > secs) break;
      if ((gen & every) == 0) print_json(&p);
      G c = p;
      mutate(&c, &rs);
      uint8_t ca[MAXN];
      const int cc = active(&c, ca);
      if (cc > cap || errors(&c, ca) != 0) continue;
      p = c;
    }
    return 0;
  }
  if (depth_mode == 3) {
    int pfo = foldable(&p, act), bfo = pfo, bd3 = pd, bc3 = pc;
    fprintf(stderr, "polish start: %d gates, %d foldable, depth %d\n", pc, pfo, pd);
    for (;;) {
      if ((++gen & 0xFFFF) == 0 && (double)(clock() - t0) / CLOCKS_PER_SEC > secs) break;
      for (int l = 0; l < lambda; l++) {
        G c = p;
        mutate(&c, &rs);
        uint8_t ca[MAXN];
        const int cc = active(&c, ca);
        if (cc > pc) continue;
        if (errors(&c, ca) != 0) continue;
        const int cfo = foldable(&c, ca), cd = depth(&c, ca);
        if (cc < pc || cfo > pfo || (cfo == pfo && cd <= pd)) {
          p = c, pc = cc, pfo = cfo, pd = cd;
          if (cc < bc3 || (cc == bc3 && (cfo > bfo || (cfo == bfo && cd < bd3)))) {
            bc3 = cc, bfo = cfo, bd3 = cd;
            fprintf(stderr, "gen %ld: %d gates, %d foldable, depth %d\n", gen, cc, cfo, cd);
            print_json(&p);
          }
          break;
        }
      }
    }
    fprintf(stderr, "done: %ld generations\n", gen);
    return 0;
  }
  if (depth_mode == 2) {
    int budget = pc - 1;
    int pf = weight;  /* parent fitness: exact, one gate over budget */
    for (;;) {
      if ((++gen & 0xFFFF) == 0 && (double)(clock() - t0) / CLOCKS_PER_SEC > secs) break;
      for (int l = 0; l < lambda; l++) {
        G c = p;
        mutate(&c, &rs);
        uint8_t ca[MAXN];
        const int cc = active(&c, ca);
        const int ce = errors(&c, ca);
        const int cf = ce + weight * (cc > budget ? cc - budget : 0);
        if (cf <= pf) {
          p = c;
          pf = cf;
          if (ce == 0 && cc <= budget) {
            fprintf(stderr, "gen %ld: %d gates, depth %d\n", gen, cc, depth(&c, ca));
            print_json(&p);
            budget = cc - 1;
            pf = weight;
          }
          break;
        }
      }
    }
    fprintf(stderr, "done: %ld generations, budget %d\n", gen, budget);
    return 0;
  }
  for (;;) {
    if ((++gen & 0xFFFF) == 0 && (double)(clock() - t0) / CLOCKS_PER_SEC > secs) break;
    G bestc;
    int bc = 1 << 30, bd = 1 << 30, have = 0;
    for (int l = 0; l < lambda; l++) {
      G c = p;
      mutate(&c, &rs);
      uint8_t ca[MAXN];
      const int cc = active(&c, ca);
      if (cc > pc) continue;
      if (errors(&c, ca) != 0) continue;
      const int cd = depth(&c, ca);
      if (!have || cc < bc || (cc == bc && cd < bd)) {
        bestc = c, bc = cc, bd = cd, have = 1;
      }
    }
    if (!have) continue;
    if (depth_mode) {
      if (bc < pc || (bc == pc && bd <= pd)) {
        p = bestc;
        pc = bc;
        pd = bd;
        if (bc < best || (bc == best && bd < bestd)) {
          best = bc;
          bestd = bd;
          fprintf(stderr, "gen %ld: %d gates, depth %d\n", gen, bc, bd);
          print_json(&p);
        }
      }
      continue;
    }
    /* neutral drift: accept equal cost as long as the depth stays within 2 of the start */
    if (bc < pc || bd <= d0 + 2) {
      p = bestc;
      if (bc < best) {
        best = bc;
        fprintf(stderr, "gen %ld: %d gates, depth %d\n", gen, bc, bd);
        print_json(&p);
      }
      pc = bc;
      pd = bd;
    }
  }
  fprintf(stderr, "done: %ld generations, best %d\n", gen, best);
  return 0;
}
