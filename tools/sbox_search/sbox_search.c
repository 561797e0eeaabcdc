/*
 * sbox_search.c -- search for small 3-input-LUT (LOP3) circuits computing the
 * four output bits of one DES S-box (6 inputs -> 4 outputs).
 *
 * Method: recursive Shannon-style decomposition in the spirit of Kwan,
 * "Reducing the Gate Count of Bitslice DES" (2000), adapted to arbitrary
 * 3-input gates:
 *   create(target, mask):
 *     1. an existing signal equals target (or its complement) on mask -> reuse;
 *     2. one new LUT over any three existing signals fits target on mask;
 *     3. otherwise pick a selector input x_i not yet used on this path, build
 *        f0 for the x_i = 0 half, then f1 for the x_i = 1 half either as the
 *        plain target (mux form) or as target ^ f0 (xor form), and join them
 *        with one LUT(x_i, f0, f1).  Every selector/form is tried on a copy of
 *        the circuit at the top `full_levels` levels and the smallest wins;
 *        deeper levels pick one at random.
 *   Outputs are built one after another so later ones reuse earlier gates.
 * Complements are free: a LUT consumer absorbs them, and the kernel XORs each
 * output into the other Feistel half with XOR or XNOR (one LOP3 either way).
 *
 * Many randomized trials (output order, selector order, triple scan order)
 * run in parallel (OpenMP); the smallest circuit is printed as one JSON line:
 *   {"gates": [[lut, a, b, c], ...], "outputs": [s0..s3], "neg": [0/1 x4]}
 * Signals 0..5 are inputs x0..x5 (x0 = S-box input bit b1 = MSB of the 6-bit
 * value, truth-table bit v has x_i = bit (5-i) of v); signal 6+k is gate k.
 *
 * Usage: sbox_search <trials> <seed> <levels> <t0> <t1> <t2> <t3>
 *        levels = full_levels + 10 * all_forms + 100 * fuse + 1000 * double_levels
 *        (all_forms: try AND/OR join forms too; fuse: fold the Feistel XOR into
 *        2-input output joins, minimizing gates + unfused outputs)
 *        (t_o = 64-bit truth table of output bit o, hex)
 * The result is verified exhaustively by the caller (tools/run_sbox_search.py)
 * and again by tools/gen_tdes.py before any code is emitted.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MAXG 160
typedef uint64_t tt_t;

typedef struct {
  tt_t tt[MAXG];
  uint8_t lut[MAXG];
  uint8_t in[MAXG][3];
  int n;
} St;

static tt_t VARS[6];

static inline uint64_t rnd(uint64_t *s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline tt_t lut_eval(int lut, tt_t a, tt_t b, tt_t c) {
  tt_t r = 0;
  for (int k = 0; k < 8; k++)
    if ((lut >> k) & 1) r |= ((k & 4) ? a : ~a) & ((k & 2) ? b : ~b) & ((k & 1) ? c : ~c);
  return r;
}

/* LUT over (A,B,C) equal to T on M, or -1. Unconstrained entries are 0. */
static inline int fit3(tt_t A, tt_t B, tt_t C, tt_t T, tt_t M) {
  int lut = 0;
  const tt_t nA = ~A, nB = ~B, nC = ~C;
  const tt_t ab[4] = {M & nA & nB, M & nA & B, M & A & nB, M & A & B};
  for (int q = 0; q < 4; q++) {
    const tt_t r0 = ab[q] & nC, r1 = ab[q] & C;
    const tt_t t0 = T & r0, t1 = T & r1;
    if (t0 && t0 != r0) return -1;
    if (t1 && t1 != r1) return -1;
    if (t0) lut |= 1 << (2 * q);
    if (t1) lut |= 1 << (2 * q + 1);
  }
  return lut;
}

static int add_gate(St *s, int lut, int a, int b, int c) {
  if (s->n >= MAXG) return -1;
  const int k = s->n++;
  s->lut[k] = (uint8_t)lut;
  s->in[k][0] = (uint8_t)a;
  s->in[k][1] = (uint8_t)b;
  s->in[k][2] = (uint8_t)c;
  s->tt[k] = lut_eval(lut, s->tt[a], s->tt[b], s->tt[c]);
  return k;
}

static int find_existing(const St *s, tt_t T, tt_t M, int *neg) {
  for (int g = s->n - 1; g >= 0; g--) {
    const tt_t d = (s->tt[g] ^ T) & M;
    if (!d) { *neg = 0; return g; }
    if (d == M) { *neg = 1; return g; }
  }
  return -1;
}

/* one new gate over three existing signals (each unordered triple once, keyed
 * by its smallest index; the outer scan starts at a random index) */
static int find_single(St *s, tt_t T, tt_t M, uint64_t *rng) {
  const int n = s->n;
  const int off = n ? (int)(rnd(rng) % (uint64_t)n) : 0;
  for (int ia = 0; ia < n; ia++) {
    const int a = (ia + off) % n;
    const tt_t A = s->tt[a];
    for (int b = a + 1; b < n; b++) {
      const tt_t B = s->tt[b];
      for (int c = b + 1; c < n; c++) {
        const int lut = fit3(A, B, s->tt[c], T, M);
        if (lut >= 0) return add_gate(s, lut, a, b, c);
      }
    }
  }
  return -1;
}

/* two new gates: T = LUT(a, b, g), g = LUT(c, d, e), a..e existing.  For each
 * pair (a, b) the regions where T is not constant fix g up to a per-region
 * polarity; a triple scan then looks for g.  Expensive (O(n^5) worst case):
 * used only at the top recursion levels (Cfg.double_levels). */
static int find_double(St *s, tt_t T, tt_t M, uint64_t *rng) {
  const int n = s->n;
  if (n + 2 > MAXG) return -1;
  const int off = n ? (int)(rnd(rng) % (uint64_t)n) : 0;
  for (int ia = 0; ia < n; ia++) {
    const int a = (ia + off) % n;
    const tt_t A = s->tt[a];
    for (int b = 0; b < n; b++) {
      if (b == a) continue;
      const tt_t B = s->tt[b];
      const tt_t R[4] = {M & ~A & ~B, M & ~A & B, M & A & ~B, M & A & B};
      int mixed[4], k = 0;
      tt_t U = 0;
      for (int q = 0; q < 4; q++) {
        const tt_t t = T & R[q];
        if (t && t != R[q]) mixed[k++] = q, U |= R[q];
      }
      if (k == 0) continue;
      for (int pol = 0; pol < (1 << (k - 1)); pol++) {
        tt_t flip = 0;
        for (int j = 1; j < k; j++)
          if ((pol >> (j - 1)) & 1) flip |= R[mixed[j]];
        const tt_t Tg = T ^ flip;
        for (int c = 0; c < n; c++) {
          const tt_t C = s->tt[c];
          for (int d = c + 1; d < n; d++) {
            const tt_t D = s->tt[d];
            for (int e = d + 1; e < n; e++) {
              const int lut = fit3(C, D, s->tt[e], Tg, U);
              if (lut < 0) continue;
              const int g = add_gate(s, lut, c, d, e);
              const int out = fit3(A, B, s->tt[g], T, M);
              if (out >= 0) return add_gate(s, out, a, b, g);
              s->n--; /* cannot happen; undo */
            }
          }
        }
      }
    }
  }
  return -1;
}

typedef struct {
  int full_levels;
  int all_forms;
  int fuse;
  int double_levels;
} Cfg;

static int create(St *s, tt_t T, tt_t M, int selused, int level, const Cfg *cfg, uint64_t *rng,
                  int *neg);

/* Build T on M with selector input i.  The half x_i = `first` is built first
 * (f0), then the other half (f1) with the join form `form`:
 *   0 mux      f1 = T
 *   1 xor      f1 = T ^ f0
 *   2 and      T = f0 & f1 on the other half (needs T => f0 there): f1 free where f0 = 0
 *   3 andn     T = ~f0 & f1 (needs T => ~f0): f1 free where f0 = 1
 *   4 or       T = f0 | f1 (needs f0 => T): f1 free where f0 = 1
 *   5 orn      T = ~f0 | f1 (needs ~f0 => T): f1 free where f0 = 0
 * and one LUT(x_i, f0, f1) joins them (fit3 finds it for every polarity).
 * Returns the signal or -1 (also when the form's precondition fails). */
#define NFORMS 6
static int try_sel(St *s, tt_t T, tt_t M, int selused, int level, int i, int first, int form,
                   const Cfg *cfg, uint64_t *rng, int *neg) {
  const tt_t X = first ? VARS[i] : ~VARS[i];   /* region built first */
  const tt_t M0 = M & X, M1 = M & ~X;
  int n0, n1;
  const int f0 = create(s, T, M0, selused | (1 << i), level + 1, cfg, rng, &n0);
  if (f0 < 0) return -1;
  const tt_t F = s->tt[f0];
  tt_t T1 = T, K1 = M1;
  switch (form) {
    case 0: break;
    case 1: T1 = T ^ F; break;
    case 2: if (T & ~F & M1) return -1; K1 = M1 & F; break;
    case 3: if (T & F & M1) return -1; K1 = M1 & ~F; break;
    case 4: if (~T & F & M1) return -1; K1 = M1 & ~F; break;
    case 5: if (~T & ~F & M1) return -1; K1 = M1 & F; break;
  }
  int f1 = -1;
  if (K1) {
    f1 = create(s, T1, K1, selused | (1 << i), level + 1, cfg, rng, &n1);
    if (f1 < 0) return -1;
  }
  int ex = find_existing(s, T, M, neg);
  if (ex >= 0) return ex;
  const int g1 = f1 >= 0 ? f1 : f0;
  const int lut = fit3(VARS[i], F, s->tt[g1], T, M);
  if (lut < 0) return -1;
  *neg = 0;
  return add_gate(s, lut, i, f0, g1);
}

static int create(St *s, tt_t T, tt_t M, int selused, int level, const Cfg *cfg, uint64_t *rng,
                  int *neg) {
  int g = find_existing(s, T, M, neg);
  if (g >= 0) return g;
  g = find_single(s, T, M, rng);
  if (g >= 0) {
    *neg = 0;
    return g;
  }
  if (level < cfg->double_levels) {
    g = find_double(s, T, M, rng);
    if (g >= 0) {
      *neg = 0;
      return g;
    }
  }
  int cand[6], nc = 0;
  for (int i = 0; i < 6; i++)
    if (!(selused & (1 << i))) cand[nc++] = i;
  if (!nc) return -1;
  for (int k = nc - 1; k > 0; k--) { /* shuffle */
    const int j = (int)(rnd(rng) % (uint64_t)(k + 1));
    const int t = cand[k];
    cand[k] = cand[j];
    cand[j] = t;
  }
  if (level >= cfg->full_levels) {
    /* greedy below the fully explored levels: random selector, first feasible form */
    const int first = (int)(rnd(rng) & 1);
    const int f0form = (int)(rnd(rng) % NFORMS);
    St *tmp = (St *)malloc(sizeof(St));
    int r = -1;
    for (int q = 0; q < NFORMS && r < 0; q++) {
      memcpy(tmp, s, sizeof(St));
      r = try_sel(tmp, T, M, selused, level, cand[0], first, (f0form + q) % NFORMS, cfg, rng, neg);
      if (r >= 0) memcpy(s, tmp, sizeof(St));
    }
    free(tmp);
    return r;
  }
  St *best = NULL, *tmp = (St *)malloc(sizeof(St));
  int bestg = -1, bestneg = 0;
  for (int k = 0; k < nc; k++) {
    for (int fw = 0; fw < 2 * NFORMS; fw++) {
      const int first = fw / NFORMS, form = fw % NFORMS;
      if (!cfg->all_forms && form > 1) continue;
      memcpy(tmp, s, sizeof(St));
      int ng;
      const int r = try_sel(tmp, T, M, selused, level, cand[k], first, form, cfg, rng, &ng);
      if (r < 0) continue;
      if (!best || tmp->n < best->n) {
        if (!best) best = (St *)malloc(sizeof(St));
        memcpy(best, tmp, sizeof(St));
        bestg = r;
        bestneg = ng;
      }
    }
  }
  free(tmp);
  if (!best) return -1;
  memcpy(s, best, sizeof(St));
  free(best);
  *neg = bestneg;
  return bestg;
}

/* Per output: either a plain signal (out, neg; the kernel XORs it into the
 * other half with one LOP3), or -- fused mode -- a 2-input function fh(fu, fv)
 * (4-bit table, index (u<<1)|v) folded into that same LOP3: P ^= fh(u, v) is
 * LOP3(P, u, v).  Either way each output costs exactly one LOP3 into P, so the
 * cost of a circuit is its gate count (ALU ops per S-box per round = gates + 4);
 * fusion pays off when an output's final join is 2-input and needs no gate. */
typedef struct {
  St s;
  int out[4], neg[4];
  int fu[4], fv[4], fh[4];
  int cost;
} Result;

/* 2-input table h with h(U, V) = T on M, or -1 */
static inline int fit2(tt_t U, tt_t V, tt_t T, tt_t M) {
  int h = 0;
  const tt_t r[4] = {M & ~U & ~V, M & ~U & V, M & U & ~V, M & U & V};
  for (int q = 0; q < 4; q++) {
    const tt_t t = T & r[q];
    if (t && t != r[q]) return -1;
    if (t) h |= 1 << q;
  }
  return h;
}

typedef struct {
  int plain, g, neg, u, v, h, cost;
} OutChoice;

/* Try to realize T on the full space as a fused 2-input join h(f0, f1):
 * f0 = T on the x_i = first half, then f1 from the form:
 *   0 XOR  f1 = T ^ f0 everywhere
 *   1 OR   f1 = T where f0 = 0 (needs f0 => T); free where f0 = 1 (or T = 1 on the first half)
 *   2 AND  f1 = T where f0 = 1 (needs T => f0); free where f0 = 0 */
static int try_fused(St *s, tt_t T, int i, int first, int form, const Cfg *cfg, uint64_t *rng,
                     OutChoice *oc) {
  const tt_t X = first ? VARS[i] : ~VARS[i];
  const int n_before = s->n;
  int n0, n1;
  const int f0 = create(s, T, X, 1 << i, 1, cfg, rng, &n0);
  if (f0 < 0) return -1;
  const tt_t F = s->tt[f0] ^ (n0 ? ~0ull : 0ull); /* == T on X */
  tt_t T1 = T, K1 = ~0ull;
  switch (form) {
    case 0: T1 = T ^ F; break;
    case 1: if (F & ~T & ~X) return -1; K1 = (X & ~T) | (~X & ~F); break;
    case 2: if (T & ~F & ~X) return -1; K1 = (X & T) | (~X & F); break;
  }
  int f1;
  if (!K1) f1 = f0, n1 = 0;
  else f1 = create(s, T1, K1, 0, 1, cfg, rng, &n1);
  if (f1 < 0) return -1;
  const int h = fit2(s->tt[f0], s->tt[f1], T, ~0ull);
  if (h < 0) return -1;
  oc->plain = 0;
  oc->u = f0;
  oc->v = f1;
  oc->h = h;
  oc->cost = s->n - n_before;
  return 0;
}

/* Build output target T choosing the cheapest of: an existing signal (+1 XOR),
 * a 2-input function of two existing signals (fused, +0), fused Shannon joins,
 * or a plain build (+1 XOR).  Leaves the chosen construction in *s. */
static int create_output(St *s, tt_t T, const Cfg *cfg, uint64_t *rng, OutChoice *best) {
  int neg;
  best->cost = 1 << 20;
  /* existing pair -> fused, free */
  const int n = s->n;
  for (int u = 0; u < n; u++)
    for (int v = u + 1; v < n; v++) {
      const int h = fit2(s->tt[u], s->tt[v], T, ~0ull);
      if (h >= 0) {
        best->plain = 0, best->u = u, best->v = v, best->h = h, best->cost = 0;
        return 0;
      }
    }
  int g = find_existing(s, T, ~0ull, &neg);
  if (g >= 0) {
    best->plain = 1, best->g = g, best->neg = neg, best->cost = 1;
    return 0;
  }
  St *bestst = (St *)malloc(sizeof(St)), *tmp = (St *)malloc(sizeof(St));
  int have = 0;
  /* plain build */
  memcpy(tmp, s, sizeof(St));
  g = create(tmp, T, ~0ull, 0, 0, cfg, rng, &neg);
  if (g >= 0) {
    best->plain = 1, best->g = g, best->neg = neg, best->cost = tmp->n - s->n;
    memcpy(bestst, tmp, sizeof(St));
    have = 1;
  }
  /* fused Shannon joins */
  for (int i = 0; i < 6; i++)
    for (int first = 0; first < 2; first++)
      for (int form = 0; form < 3; form++) {
        OutChoice oc;
        memcpy(tmp, s, sizeof(St));
        if (try_fused(tmp, T, i, first, form, cfg, rng, &oc) < 0) continue;
        if (oc.cost < best->cost || (oc.cost == best->cost && (rnd(rng) & 1))) {
          *best = oc;
          memcpy(bestst, tmp, sizeof(St));
          have = 1;
        }
      }
  if (have) memcpy(s, bestst, sizeof(St));
  free(bestst);
  free(tmp);
  return have ? 0 : -1;
}

static void run_trial(const tt_t targets[4], const Cfg *cfg, uint64_t seed, Result *res) {
  uint64_t rng = seed;
  St *s = &res->s;
  memset(s, 0, sizeof *s);
  for (int i = 0; i < 6; i++) s->tt[i] = VARS[i];
  s->n = 6;
  int order[4] = {0, 1, 2, 3};
  for (int k = 3; k > 0; k--) {
    const int j = (int)(rnd(&rng) % (uint64_t)(k + 1));
    const int t = order[k];
    order[k] = order[j];
    order[j] = t;
  }
  int unfused = 0;
  for (int q = 0; q < 4; q++) {
    const int o = order[q];
    res->fh[o] = -1;
    if (cfg->fuse) {
      OutChoice oc;
      if (create_output(s, targets[o], cfg, &rng, &oc) < 0) {
        s->n = MAXG + 1;
        return;
      }
      if (oc.plain) {
        res->out[o] = oc.g, res->neg[o] = oc.neg, unfused++;
      } else {
        res->out[o] = -1, res->neg[o] = 0;
        res->fu[o] = oc.u, res->fv[o] = oc.v, res->fh[o] = oc.h;
      }
      continue;
    }
    int ng = 0;
    const int g = create(s, targets[o], ~0ull, 0, 0, cfg, &rng, &ng);
    if (g < 0) {
      s->n = MAXG + 1;
      return;
    }
    res->out[o] = g;
    res->neg[o] = ng;
    unfused++;
  }
  (void)unfused;
  res->cost = s->n - 6;
}

/* remove gates not reachable from the outputs, renumber */
static void prune(Result *r) {
  St *s = &r->s;
  int live[MAXG] = {0};
  for (int o = 0; o < 4; o++) {
    if (r->fh[o] >= 0) live[r->fu[o]] = live[r->fv[o]] = 1;
    else live[r->out[o]] = 1;
  }
  for (int g = s->n - 1; g >= 6; g--)
    if (live[g])
      for (int j = 0; j < 3; j++) live[s->in[g][j]] = 1;
  int map[MAXG];
  St t;
  memset(&t, 0, sizeof t);
  for (int i = 0; i < 6; i++) {
    t.tt[i] = s->tt[i];
    map[i] = i;
  }
  t.n = 6;
  for (int g = 6; g < s->n; g++) {
    if (!live[g]) continue;
    map[g] = add_gate(&t, s->lut[g], map[s->in[g][0]], map[s->in[g][1]], map[s->in[g][2]]);
  }
  int unfused = 0;
  for (int o = 0; o < 4; o++) {
    if (r->fh[o] >= 0) {
      r->fu[o] = map[r->fu[o]], r->fv[o] = map[r->fv[o]];
    } else {
      r->out[o] = map[r->out[o]];
      unfused++;
    }
  }
  memcpy(s, &t, sizeof t);
  (void)unfused;
  r->cost = s->n - 6;
}

/* Local search step: drop the gates used only by 1-2 randomly chosen outputs
 * and rebuild those outputs against everything that remains (1-3 outputs). */
static void improve_trial(const Result *start, const tt_t targets[4], const Cfg *cfg,
                          uint64_t seed, Result *res) {
  uint64_t rng = seed;
  memcpy(res, start, sizeof(Result));
  int order[4] = {0, 1, 2, 3};
  for (int k = 3; k > 0; k--) {
    const int j = (int)(rnd(&rng) % (uint64_t)(k + 1));
    const int t = order[k];
    order[k] = order[j];
    order[j] = t;
  }
  const int nsel = 1 + (int)(rnd(&rng) % 3); /* rebuild 1-3 of the 4 outputs */
  for (int q = 0; q < nsel; q++) {
    res->fh[order[q]] = -1;
    res->out[order[q]] = 0; /* placeholder: input x0 keeps nothing alive */
  }
  prune(res);
  St *s = &res->s;
  for (int q = 0; q < nsel; q++) {
    const int o = order[q];
    if (cfg->fuse) {
      OutChoice oc;
      if (create_output(s, targets[o], cfg, &rng, &oc) < 0) {
        res->cost = 1 << 20;
        return;
      }
      if (oc.plain) res->out[o] = oc.g, res->neg[o] = oc.neg, res->fh[o] = -1;
      else res->fu[o] = oc.u, res->fv[o] = oc.v, res->fh[o] = oc.h, res->out[o] = -1;
    } else {
      int ng = 0;
      const int g = create(s, targets[o], ~0ull, 0, 0, cfg, &rng, &ng);
      if (g < 0) {
        res->cost = 1 << 20;
        return;
      }
      res->out[o] = g, res->neg[o] = ng, res->fh[o] = -1;
    }
  }
  prune(res);
}

static int read_circuit(Result *r) {
  St *s = &r->s;
  memset(r, 0, sizeof *r);
  for (int i = 0; i < 6; i++) s->tt[i] = VARS[i];
  s->n = 6;
  int n;
  if (scanf("%d", &n) != 1) return -1;
  for (int k = 0; k < n; k++) {
    int lut, a, b, c;
    if (scanf("%d %d %d %d", &lut, &a, &b, &c) != 4) return -1;
    add_gate(s, lut, a, b, c);
  }
  for (int o = 0; o < 4; o++) {
    int fused, a, b, c;
    if (scanf("%d %d %d %d", &fused, &a, &b, &c) != 4) return -1;
    if (fused) r->fu[o] = a, r->fv[o] = b, r->fh[o] = c, r->out[o] = -1;
    else r->out[o] = a, r->neg[o] = b, r->fh[o] = -1;
  }
  prune(r);
  return 0;
}

static void print_result(const Result *b) {
  printf("{\"gates\": [");
  for (int g = 6; g < b->s.n; g++)
    printf("%s[%d, %d, %d, %d]", g > 6 ? ", " : "", b->s.lut[g], b->s.in[g][0], b->s.in[g][1],
           b->s.in[g][2]);
  printf("], \"outputs\": [%d, %d, %d, %d], \"neg\": [%d, %d, %d, %d], \"fuse\": [", b->out[0],
         b->out[1], b->out[2], b->out[3], b->neg[0], b->neg[1], b->neg[2], b->neg[3]);
  for (int o = 0; o < 4; o++) {
    if (b->fh[o] >= 0) printf("%s[%d, %d, %d]", o ? ", " : "", b->fu[o], b->fv[o], b->fh[o]);
    else printf("%snull", o ? ", " : "");
  }
  printf("], \"cost\": %d}\n", b->cost);
}

/* improve mode: hill climbing with parallel restarts from the best circuit so
 * far; equal-cost moves are accepted so the walk can cross plateaus. */
static int improve_main(int argc, char **argv) {
  if (argc != 10) {
    fprintf(stderr, "usage: %s improve rounds trials seed levels t0 t1 t2 t3 < circuit\n", argv[0]);
    return 2;
  }
  const int rounds = atoi(argv[2]);
  const long trials = atol(argv[3]);
  const uint64_t seed = strtoull(argv[4], 0, 10);
  const int lv = atoi(argv[5]);
  Cfg cfg = {lv % 10, (lv / 10) % 10 >= 1, (lv / 100) % 10 >= 1, lv / 1000};
  tt_t targets[4];
  for (int o = 0; o < 4; o++) targets[o] = strtoull(argv[6 + o], 0, 16);
  Result cur;
  if (read_circuit(&cur) < 0) {
    fprintf(stderr, "bad circuit on stdin\n");
    return 2;
  }
  Result best = cur;
  for (int it = 0; it < rounds; it++) {
    Result rb;
    rb.cost = 1 << 20;
#pragma omp parallel
    {
      Result *r = (Result *)malloc(sizeof(Result));
#pragma omp for schedule(dynamic, 1)
      for (long t = 0; t < trials; t++) {
        improve_trial(&cur, targets, &cfg, seed * 7777777ull + (uint64_t)it * 1000003ull + (uint64_t)t, r);
#pragma omp critical
        {
          if (r->cost < rb.cost) memcpy(&rb, r, sizeof(Result));
        }
      }
      free(r);
    }
    if (rb.cost <= cur.cost) cur = rb;
    if (cur.cost < best.cost) {
      best = cur;
      fprintf(stderr, "round %d: cost %d\n", it, best.cost);
    }
  }
  print_result(&best);
  return 0;
}

int main(int argc, char **argv) {
  if (argc > 1 && strcmp(argv[1], "improve") == 0) {
    for (int i = 0; i < 6; i++) {
      VARS[i] = 0;
      for (int v = 0; v < 64; v++)
        if ((v >> (5 - i)) & 1) VARS[i] |= 1ull << v;
    }
    return improve_main(argc, argv);
  }
  if (argc != 8) {
    fprintf(stderr, "usage: %s trials seed full_levels t0 t1 t2 t3\n", argv[0]);
    return 2;
  }
  const long trials = atol(argv[1]);
  const uint64_t seed = strtoull(argv[2], 0, 10);
  const int lv = atoi(argv[3]);
  Cfg cfg = {lv % 10, (lv / 10) % 10 >= 1, (lv / 100) % 10 >= 1, lv / 1000};
  tt_t targets[4];
  for (int o = 0; o < 4; o++) targets[o] = strtoull(argv[4 + o], 0, 16);
  for (int i = 0; i < 6; i++) {
    VARS[i] = 0;
    for (int v = 0; v < 64; v++)
      if ((v >> (5 - i)) & 1) VARS[i] |= 1ull << v;
  }
  Result best;
  best.s.n = MAXG + 1;
  best.cost = 1 << 20;
#pragma omp parallel
  {
    Result *r = (Result *)malloc(sizeof(Result));
#pragma omp for schedule(dynamic, 1)
    for (long t = 0; t < trials; t++) {
      run_trial(targets, &cfg, seed * 1000003ull + (uint64_t)t * 7919ull + 1, r);
      if (r->s.n > MAXG) continue;
      prune(r);
#pragma omp critical
      {
        if (r->cost < best.cost) memcpy(&best, r, sizeof(Result));
      }
    }
    free(r);
  }
  if (best.s.n > MAXG) {
    printf("{\"error\": \"no circuit\"}\n");
    return 1;
  }
  printf("{\"gates\": [");
  for (int g = 6; g < best.s.n; g++)
    printf("%s[%d, %d, %d, %d]", g > 6 ? ", " : "", best.s.lut[g], best.s.in[g][0], best.s.in[g][1],
           best.s.in[g][2]);
  printf("], \"outputs\": [%d, %d, %d, %d], \"neg\": [%d, %d, %d, %d], \"fuse\": [", best.out[0],
         best.out[1], best.out[2], best.out[3], best.neg[0], best.neg[1], best.neg[2], best.neg[3]);
  for (int o = 0; o < 4; o++) {
    if (best.fh[o] >= 0) printf("%s[%d, %d, %d]", o ? ", " : "", best.fu[o], best.fv[o], best.fh[o]);
    else printf("%snull", o ? ", " : "");
  }
  printf("], \"cost\": %d}\n", best.cost);
  return 0;
}
