/*
 * resub.c -- gate-count reduction of a finished 3-input-LUT (LOP3) circuit for one
 * DES S-box by resubstitution with observability don't-cares.
 *
 * CGP (cgp.c) changes 1-3 genes per child, so rewiring a gate to three new inputs
 * with a new LUT byte (four genes at once, each of them right) is rare there.  This
 * pass does exactly that, exhaustively, for every gate g of the circuit:
 *
 *   MFFC(g)  = g plus the gates only g's cone uses (they die when g is rebuilt);
 *   care(g)  = the inputs on which complementing g changes an output (the rest are
 *              observability don't-cares);
 *   S        = signals outside g's transitive fanout and outside MFFC(g);
 *   0-resub  : g = s or ~s on care(g) for some s in S          (gain |MFFC|)
 *   1-resub  : g = LUT(a, b, c) on care(g), a, b, c in S        (gain |MFFC| - 1)
 *   2-resub  : g = LUT(x, y, LUT(a, b, c)), all from S          (gain |MFFC| - 2)
 *
 * and the same for the outputs: an output is a plain signal (one LOP3 XOR/XNOR into
 * its plane) or a fused join h(u, v) absorbed into that LOP3 (tools/gen_tdes.py),
 * so an output may be re-expressed as h(u', v') of existing signals (freeing the
 * old sources' cones) or as h(LUT(a, b, c), v') (one new gate).
 *
 * Complemented replacements are absorbed by the consumers (LUT bytes, output neg,
 * join tables).  Every applied change is followed by an exact check of all four
 * outputs on all 64 inputs (reverted if not exact -- a guard, never expected); the
 * caller (tools/run_resub.py) verifies again with tools/gen_tdes.py.
 *
 * Input (stdin): the cgp.c format ("<t0> <t1> <t2> <t3>", "<ngates>", gate lines
 *   "<lut> <a> <b> <c>", four output lines "p <sig> <neg>" or "f <u> <v> <h>").
 * Usage: resub <seed> [max improvements]
 * Output: one JSON line (cgp.c format) if the gate count went down, else nothing;
 *   progress on stderr.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define MAXS 96
typedef uint64_t tt_t;

static tt_t VARS[6], TGT[4];

typedef struct {
  int n;                 /* gates; signal 6 + k = gate k (topological order) */
  uint8_t lut[MAXS];
  int in[MAXS][3];
  int otype[4], osig[4], oneg[4], ou[4], ov[4], oh[4];
} C;

static uint64_t rs_state;
static inline uint64_t rnd(void) {
  uint64_t z = (rs_state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline tt_t lut3(unsigned lut, tt_t a, tt_t b, tt_t c) {
  tt_t r = 0;
  for (int k = 0; k < 8; k++)
    if ((lut >> k) & 1) r |= ((k & 4) ? a : ~a) & ((k & 2) ? b : ~b) & ((k & 1) ? c : ~c);
  return r;
}
static inline tt_t h2(unsigned h, tt_t u, tt_t v) {
  tt_t r = 0;
  if (h & 1) r |= ~u & ~v;
  if (h & 2) r |= ~u & v;
  if (h & 4) r |= u & ~v;
  if (h & 8) r |= u & v;
  return r;
}

static void sim(const C *c, tt_t *tt) {
  for (int i = 0; i < 6; i++) tt[i] = VARS[i];
  for (int k = 0; k < c->n; k++) tt[6 + k] = lut3(c->lut[k], tt[c->in[k][0]], tt[c->in[k][1]], tt[c->in[k][2]]);
}
static tt_t out_tt(const C *c, const tt_t *tt, int o) {
  return c->otype[o] == 0 ? tt[c->osig[o]] ^ (c->oneg[o] ? ~0ull : 0ull) : h2(c->oh[o], tt[c->ou[o]], tt[c->ov[o]]);
}
static int exact(const C *c) {
  tt_t tt[6 + MAXS];
  sim(c, tt);
  for (int o = 0; o < 4; o++) if (out_tt(c, tt, o) != TGT[o]) return 0;
  return 1;
}

/* reference counts of every signal (gate inputs, counted once per distinct input, + outputs) */
static void refs(const C *c, int *rc) {
  memset(rc, 0, sizeof(int) * (6 + MAXS));
  for (int k = 0; k < c->n; k++) {
    const int a = c->in[k][0], b = c->in[k][1], d = c->in[k][2];
    rc[a]++;
    if (b != a) rc[b]++;
    if (d != a && d != b) rc[d]++;
  }
  for (int o = 0; o < 4; o++) {
    if (c->otype[o] == 0) rc[c->osig[o]]++;
    else { rc[c->ou[o]]++; if (c->ov[o] != c->ou[o]) rc[c->ov[o]]++; }
  }
}

/* dereference signal s (its reference just dropped to zero): mark it and every gate
   that only it kept alive; returns the number of gates marked. */
static int deref(const C *c, int s, int *rc, uint8_t *dead) {
  if (s < 6 || dead[s]) return 0;
  dead[s] = 1;
  int n = 1;
  const int k = s - 6, a = c->in[k][0], b = c->in[k][1], d = c->in[k][2];
  const int f[3] = {a, b, d};
  for (int j = 0; j < 3; j++) {
    if ((j == 1 && b == a) || (j == 2 && (d == a || d == b))) continue;
    if (--rc[f[j]] == 0) n += deref(c, f[j], rc, dead);
  }
  return n;
}

/* transitive fanout of signal s (s included) */
static void tfo(const C *c, int s, uint8_t *in_tfo) {
  memset(in_tfo, 0, 6 + MAXS);
  in_tfo[s] = 1;
  for (int k = 0; k < c->n; k++)
    if (in_tfo[c->in[k][0]] || in_tfo[c->in[k][1]] || in_tfo[c->in[k][2]]) in_tfo[6 + k] = 1;
}

/* inputs on which complementing signal s changes some output */
static tt_t care_of(const C *c, int s) {
  tt_t tt[6 + MAXS], tf[6 + MAXS];
  sim(c, tt);
  memcpy(tf, tt, sizeof tt);
  tf[s] = ~tt[s];
  for (int k = s - 6 + 1; k < c->n; k++)
    if (k >= 0) tf[6 + k] = lut3(c->lut[k], tf[c->in[k][0]], tf[c->in[k][1]], tf[c->in[k][2]]);
  tt_t care = 0;
  for (int o = 0; o < 4; o++) care |= out_tt(c, tt, o) ^ out_tt(c, tf, o);
  return care;
}

/* Is (on `care`) the function `f` a LUT of (a, b, d)?  Returns the LUT byte or -1. */
static inline int fit3(tt_t f, tt_t care, tt_t a, tt_t b, tt_t d) {
  int lut = 0;
  for (int k = 0; k < 8; k++) {
    const tt_t cell = ((k & 4) ? a : ~a) & ((k & 2) ? b : ~b) & ((k & 1) ? d : ~d) & care;
    const tt_t on = cell & f, off = cell & ~f;
    if (on && off) return -1;
    if (on) lut |= 1 << k;
  }
  return lut;
}

/* Remove dead gates and renumber (keeps topological order). */
static void compact(C *c) {
  int rc[6 + MAXS];
  uint8_t live[6 + MAXS] = {0};
  for (int o = 0; o < 4; o++) {
    if (c->otype[o] == 0) live[c->osig[o]] = 1;
    else live[c->ou[o]] = live[c->ov[o]] = 1;
  }
  for (int k = c->n - 1; k >= 0; k--)
    if (live[6 + k]) for (int j = 0; j < 3; j++) live[c->in[k][j]] = 1;
  (void)rc;
  int map[6 + MAXS];
  for (int i = 0; i < 6; i++) map[i] = i;
  int n = 0;
  C d = *c;
  for (int k = 0; k < c->n; k++) {
    if (!live[6 + k]) { map[6 + k] = -1; continue; }
    map[6 + k] = 6 + n;
    d.lut[n] = c->lut[k];
    for (int j = 0; j < 3; j++) d.in[n][j] = map[c->in[k][j]];
    n++;
  }
  d.n = n;
  for (int o = 0; o < 4; o++) {
    if (c->otype[o] == 0) d.osig[o] = map[c->osig[o]];
    else { d.ou[o] = map[c->ou[o]]; d.ov[o] = map[c->ov[o]]; }
  }
  *c = d;
}

/* Replace every use of signal s by r (complemented if neg); consumers absorb the
   complement.  Only gates/outputs outside `skip` (s's own replacement) are changed. */
static void redirect(C *c, int s, int r, int neg) {
  for (int k = 0; k < c->n; k++)
    for (int j = 0; j < 3; j++)
      if (c->in[k][j] == s) {
        c->in[k][j] = r;
        if (neg) {
          const int bit = 2 - j;  /* input j is bit (2 - j) of the LUT index */
          unsigned L = c->lut[k], M = 0;
          for (int i = 0; i < 8; i++) if ((L >> i) & 1) M |= 1u << (i ^ (1 << bit));
          c->lut[k] = (uint8_t)M;
        }
      }
  for (int o = 0; o < 4; o++) {
    if (c->otype[o] == 0) {
      if (c->osig[o] == s) { c->osig[o] = r; c->oneg[o] ^= neg; }
    } else {
      unsigned h = c->oh[o];
      if (c->ou[o] == s) {
        c->ou[o] = r;
        if (neg) { unsigned m = 0; for (int i = 0; i < 4; i++) if ((h >> i) & 1) m |= 1u << (i ^ 2); h = m; }
      }
      if (c->ov[o] == s) {
        c->ov[o] = r;
        if (neg) { unsigned m = 0; for (int i = 0; i < 4; i++) if ((h >> i) & 1) m |= 1u << (i ^ 1); h = m; }
      }
      c->oh[o] = (int)h;
    }
  }
}

/* Insert a new gate right before gate index pos (signal 6 + pos); signals >= 6 + pos shift by one. */
static int insert_gate(C *c, int pos, int lut, int a, int b, int d) {
  for (int k = c->n; k > pos; k--) {
    c->lut[k] = c->lut[k - 1];
    for (int j = 0; j < 3; j++) c->in[k][j] = c->in[k - 1][j];
  }
  c->n++;
  for (int k = 0; k < c->n; k++) {
    if (k == pos) continue;
    for (int j = 0; j < 3; j++) if (c->in[k][j] >= 6 + pos) c->in[k][j]++;
  }
  for (int o = 0; o < 4; o++) {
    if (c->osig[o] >= 6 + pos) c->osig[o]++;
    if (c->ou[o] >= 6 + pos) c->ou[o]++;
    if (c->ov[o] >= 6 + pos) c->ov[o]++;
  }
  c->lut[pos] = (uint8_t)lut;
  c->in[pos][0] = a >= 6 + pos ? a + 1 : a;
  c->in[pos][1] = b >= 6 + pos ? b + 1 : b;
  c->in[pos][2] = d >= 6 + pos ? d + 1 : d;
  return 6 + pos;
}

/* topological re-sort (new gates may sit after their consumers' other inputs) */
static int topo(C *c) {
  int order[MAXS], state[MAXS] = {0}, no = 0;
  int stack[4 * MAXS], sp;
  for (int k0 = 0; k0 < c->n; k0++) {
    if (state[k0]) continue;
    sp = 0;
    stack[sp++] = k0;
    while (sp) {
      const int k = stack[sp - 1];
      if (state[k] == 0) {
        state[k] = 1;
        for (int j = 0; j < 3; j++) {
          const int s = c->in[k][j];
          if (s >= 6 && state[s - 6] == 0) stack[sp++] = s - 6;
          else if (s >= 6 && state[s - 6] == 1) return 0;  /* cycle */
        }
      } else {
        sp--;
        if (state[k] == 1) { state[k] = 2; order[no++] = k; }
      }
    }
  }
  int map[6 + MAXS];
  for (int i = 0; i < 6; i++) map[i] = i;
  for (int i = 0; i < no; i++) map[6 + order[i]] = 6 + i;
  C d = *c;
  for (int i = 0; i < no; i++) {
    const int k = order[i];
    d.lut[i] = c->lut[k];
    for (int j = 0; j < 3; j++) d.in[i][j] = map[c->in[k][j]];
  }
  for (int o = 0; o < 4; o++) {
    d.osig[o] = c->otype[o] == 0 ? map[c->osig[o]] : 0;
    if (c->otype[o]) { d.ou[o] = map[c->ou[o]]; d.ov[o] = map[c->ov[o]]; }
  }
  *c = d;
  return 1;
}

static int cand_set(const C *c, int s, const uint8_t *dead, int *S) {
  uint8_t in_tfo[6 + MAXS];
  tfo(c, s, in_tfo);
  int ns = 0;
  for (int i = 0; i < 6 + c->n; i++) if (!in_tfo[i] && !dead[i]) S[ns++] = i;
  return ns;
}

/* try to rebuild gate signal s cheaper; applies the change and returns the gain */
static int try_gate(C *c, int s) {
  int rc[6 + MAXS];
  uint8_t dead[6 + MAXS] = {0};
  refs(c, rc);
  rc[s] = 0;
  const int m = deref(c, s, rc, dead);
  int S[6 + MAXS];
  const int ns = cand_set(c, s, dead, S);
  tt_t tt[6 + MAXS];
  sim(c, tt);
  const tt_t care = care_of(c, s), f = tt[s];
  /* 0-resub */
  for (int i = 0; i < ns; i++) {
    const tt_t x = tt[S[i]];
    if (((x ^ f) & care) == 0 || ((~x ^ f) & care) == 0) {
      C d = *c;
      redirect(&d, s, S[i], ((x ^ f) & care) != 0);
      if (!topo(&d)) continue;
      compact(&d);
      if (exact(&d)) { *c = d; return m; }
    }
  }
  if (m < 2) return 0;
  /* 1-resub */
  for (int i = 0; i < ns; i++)
    for (int j = i; j < ns; j++)
      for (int l = j; l < ns; l++) {
        const int lut = fit3(f, care, tt[S[i]], tt[S[j]], tt[S[l]]);
        if (lut < 0) continue;
        C d = *c;
        const int k = s - 6;
        d.lut[k] = (uint8_t)lut;
        d.in[k][0] = S[i]; d.in[k][1] = S[j]; d.in[k][2] = S[l];
        if (!topo(&d)) continue;
        compact(&d);
        if (d.n < c->n && exact(&d)) { const int g = c->n - d.n; *c = d; return g; }
      }
  if (m < 3) return 0;
  /* 2-resub: g = LUT2(x, y, n1), n1 = LUT1(a, b, e).  For a pair (x, y), n1 must
     equal f or ~f (on care) inside each (x, y) cell where f is not constant. */
  for (int i = 0; i < ns; i++)
    for (int j = i + 1; j < ns; j++) {
      const tt_t X = tt[S[i]], Y = tt[S[j]];
      tt_t cells[4];
      int nc = 0, cidx[4];
      for (int q = 0; q < 4; q++) {
        const tt_t cell = ((q & 2) ? X : ~X) & ((q & 1) ? Y : ~Y) & care;
        if ((cell & f) && (cell & ~f)) { cells[nc] = cell; cidx[nc] = q; nc++; }
      }
      if (nc == 0) continue;  /* then f is a function of (x, y) alone: 1-resub covers it */
      for (int pol = 0; pol < (1 << (nc - 1)); pol++) {  /* n1's polarity per cell (first fixed) */
        tt_t want = 0, wcare = 0;
        for (int q = 0; q < nc; q++) {
          wcare |= cells[q];
          want |= cells[q] & (((pol >> q) & 1) ? ~f : f);
        }
        for (int a = 0; a < ns; a++)
          for (int b = a; b < ns; b++)
            for (int e = b; e < ns; e++) {
              const int l1 = fit3(want, wcare, tt[S[a]], tt[S[b]], tt[S[e]]);
              if (l1 < 0) continue;
              const tt_t n1 = lut3((unsigned)l1, tt[S[a]], tt[S[b]], tt[S[e]]);
              const int l2 = fit3(f, care, X, Y, n1);
              if (l2 < 0) continue;
              (void)cidx;
              C d = *c;
              const int k = s - 6;
              const int ns1 = insert_gate(&d, k, l1, S[a], S[b], S[e]);  /* gate s moves to s + 1 */
              d.lut[k + 1] = (uint8_t)l2;
              d.in[k + 1][0] = S[i] >= 6 + k ? S[i] + 1 : S[i];
              d.in[k + 1][1] = S[j] >= 6 + k ? S[j] + 1 : S[j];
              d.in[k + 1][2] = ns1;
              if (!topo(&d)) continue;
              compact(&d);
              if (d.n < c->n && exact(&d)) { const int g = c->n - d.n; *c = d; return g; }
            }
      }
    }
  return 0;
}

/* try to re-express output o cheaper (fused joins of existing signals, or of one new gate) */
static int try_output(C *c, int o) {
  int rc[6 + MAXS];
  uint8_t dead[6 + MAXS] = {0};
  refs(c, rc);
  int m = 0;
  if (c->otype[o] == 0) {
    if (--rc[c->osig[o]] == 0) m += deref(c, c->osig[o], rc, dead);
  } else {
    if (--rc[c->ou[o]] == 0) m += deref(c, c->ou[o], rc, dead);
    if (c->ov[o] != c->ou[o] && --rc[c->ov[o]] == 0) m += deref(c, c->ov[o], rc, dead);
  }
  if (m == 0) return 0;
  tt_t tt[6 + MAXS];
  sim(c, tt);
  int S[6 + MAXS], ns = 0;
  for (int i = 0; i < 6 + c->n; i++) if (!dead[i]) S[ns++] = i;
  const tt_t f = TGT[o];
  /* existing pair */
  for (int i = 0; i < ns; i++)
    for (int j = i; j < ns; j++)
      for (int h = 0; h < 16; h++) {
        if (h2(h, tt[S[i]], tt[S[j]]) != f) continue;
        C d = *c;
        d.otype[o] = 1; d.ou[o] = S[i]; d.ov[o] = S[j]; d.oh[o] = h;
        compact(&d);
        if (d.n < c->n && exact(&d)) { const int g = c->n - d.n; *c = d; return g; }
      }
  if (m < 2) return 0;
  /* h(n1, v): on the v-cells where h(., vv) is the identity or complement, n1 = f or ~f;
     where h(., vv) is constant, f must equal it */
  for (int j = 0; j < ns; j++) {
    const tt_t V = tt[S[j]];
    for (int h = 0; h < 16; h++) {
      tt_t want = 0, wcare = 0;
      int ok = 1;
      for (int vv = 0; vv < 2 && ok; vv++) {
        const tt_t cell = vv ? V : ~V;
        const int h0 = (h >> (0 + vv)) & 1, h1 = (h >> (2 + vv)) & 1;  /* h(u=0,vv), h(u=1,vv) */
        if (h0 == h1) { if ((cell & (h0 ? ~f : f)) != 0) ok = 0; }
        else { wcare |= cell; want |= cell & (h1 ? f : ~f); }
      }
      if (!ok || wcare == 0) continue;
      for (int a = 0; a < ns; a++)
        for (int b = a; b < ns; b++)
          for (int e = b; e < ns; e++) {
            const int l1 = fit3(want, wcare, tt[S[a]], tt[S[b]], tt[S[e]]);
            if (l1 < 0) continue;
            C d = *c;
            const int nsig = insert_gate(&d, d.n, l1, S[a], S[b], S[e]);
            d.otype[o] = 1; d.ou[o] = nsig; d.ov[o] = S[j]; d.oh[o] = h;
            compact(&d);
            if (d.n < c->n && exact(&d)) { const int g = c->n - d.n; *c = d; return g; }
          }
    }
  }
  return 0;
}

static void print_json(const C *c) {
  printf("{\"gates\": [");
  for (int k = 0; k < c->n; k++)
    printf("%s[%d, %d, %d, %d]", k ? ", " : "", c->lut[k], c->in[k][0], c->in[k][1], c->in[k][2]);
  printf("], \"outputs\": [");
  for (int o = 0; o < 4; o++) printf("%s%d", o ? ", " : "", c->otype[o] == 0 ? c->osig[o] : -1);
  printf("], \"neg\": [");
  for (int o = 0; o < 4; o++) printf("%s%d", o ? ", " : "", c->otype[o] == 0 ? c->oneg[o] : 0);
  printf("], \"fuse\": [");
  for (int o = 0; o < 4; o++) {
    if (c->otype[o] == 0) printf("%snull", o ? ", " : "");
    else printf("%s[%d, %d, %d]", o ? ", " : "", c->ou[o], c->ov[o], c->oh[o]);
  }
  printf("]}\n");
  fflush(stdout);
}

int main(int argc, char **argv) {
  rs_state = (argc > 1 ? strtoull(argv[1], 0, 10) : 1) * 0x9E3779B97F4A7C15ull + 7;
  const int passes = argc > 2 ? atoi(argv[2]) : 64;
  for (int i = 0; i < 6; i++) {
    VARS[i] = 0;
    for (int v = 0; v < 64; v++) if ((v >> (5 - i)) & 1) VARS[i] |= 1ull << v;
  }
  if (scanf("%lx %lx %lx %lx", &TGT[0], &TGT[1], &TGT[2], &TGT[3]) != 4) return 2;
  C c;
  memset(&c, 0, sizeof c);
  if (scanf("%d", &c.n) != 1 || c.n > MAXS - 8) return 2;
  for (int k = 0; k < c.n; k++) {
    int l;
    if (scanf("%d %d %d %d", &l, &c.in[k][0], &c.in[k][1], &c.in[k][2]) != 4) return 2;
    c.lut[k] = (uint8_t)l;
  }
  for (int o = 0; o < 4; o++) {
    char t[4];
    int x, y, z;
    if (scanf("%3s %d %d", t, &x, &y) != 3) return 2;
    if (t[0] == 'p') { c.otype[o] = 0; c.osig[o] = x; c.oneg[o] = y; }
    else { if (scanf("%d", &z) != 1) return 2; c.otype[o] = 1; c.ou[o] = x; c.ov[o] = y; c.oh[o] = z; }
  }
  if (!exact(&c)) { fprintf(stderr, "initial circuit is not exact\n"); return 3; }
  compact(&c);
  const int n0 = c.n;
  for (int p = 0; p < passes; p++) {
    /* one improvement per pass (signal numbers change), random order over gates and outputs */
    int order[MAXS + 4], no = 0, improved = 0;
    for (int k = 0; k < c.n; k++) order[no++] = 6 + k;
    for (int o = 0; o < 4; o++) order[no++] = -1 - o;
    for (int i = no - 1; i > 0; i--) { const int j = (int)(rnd() % (uint64_t)(i + 1)); const int t = order[i]; order[i] = order[j]; order[j] = t; }
    for (int i = 0; i < no && !improved; i++) {
      const int before = c.n;
      const int g = order[i] < 0 ? try_output(&c, -1 - order[i]) : try_gate(&c, order[i]);
      if (g > 0) {
        fprintf(stderr, "pass %d: %s %d -> %d gates\n", p, order[i] < 0 ? "output" : "gate", before, c.n);
        improved = 1;
      }
    }
    if (!improved) break;
  }
  if (c.n < n0) print_json(&c);
  fprintf(stderr, "done: %d -> %d gates\n", n0, c.n);
  return 0;
}
