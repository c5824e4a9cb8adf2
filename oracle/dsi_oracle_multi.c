/*
 * dsi_oracle_multi.c -- CPU oracle of multi-drafter DSI (m > 2 models,
 * SURVEY 8(f) N4): Algorithm 1 of arXiv 2405.14105 as stated,
 * lookahead 1 ("set to 1 for simplicity"), no bound on threads.
 *
 * TEST INFRASTRUCTURE ONLY (see dsi_oracle.h).  Shares no code with the
 * product path.  Two forms:
 *   - oracle_multi_tree: a literal event simulation of the whole thread tree
 *     (lines 2-17: every finished thread spawns m children; the current
 *     verifier terminates mismatching siblings and those after j*, relabels,
 *     goes back when the new verifier already finished; the verifier at level
 *     N returns).  Exponential in N: pins only.
 *   - oracle_multi_chain: the same schedule along the verified prefix only
 *     (App. C: "we continue this process until the output ... is
 *     obtained from the last verifier thread").  Linear in N.
 * Readings: dsi_oracle.h and DESIGN.md R25.
 *
 * Citations: P:n = /root/reference/PAPER.md line n.
 */
#include <stdlib.h>
#include <string.h>

#include "dsi_oracle.h"

static int multi_valid(const oracle_multi_config *c) {
  int32_t j, m;
  if (!c) return 0;
  if (c->n_drafters < 1 || c->n_drafters > ORACLE_MAX_MODELS - 1) return 0;
  if (c->n_tokens < 1 || c->t_target < 1) return 0;
  m = c->n_drafters + 1;
  for (j = 1; j < m; j++) {
    const int64_t t = c->t_drafter[j - 1];
    if (t < 1 || t > c->t_target) return 0;                 /* Assumption 2 */
    if (j > 1 && t < c->t_drafter[j - 2]) return 0;         /* ordered by latency (R25) */
    if (!(c->accept_rate[j - 1] >= 0.0 && c->accept_rate[j - 1] <= 1.0)) return 0;
  }
  if (c->rng_halves != 0 && c->rng_halves != 1) return 0;
  return 1;
}

/* 16-bit half j8 of a Philox output (the halves layout, R26): the high half of word
 * j8 for j8 < 4, the low half of word j8 - 4 otherwise. */
static uint32_t multi_half16(const uint32_t out[4], int j8) {
  uint32_t word = out[j8 & 3];
  if (j8 < 4) return word >> 16;
  return word & 0xFFFFu;
}

/* A_{j,p}: does drafter j's token at position p (on the verified prefix) equal the
 * target's?  Philox at counter (q, j-1, trial, stream_id), word (p-1) & 3; with rng_halves,
 * the 16-bit half (p-1) & 7 of counter (q = (p-1) >> 3, 2(j-1), trial, stream_id) against the
 * threshold's high half T, a tie (v == T) decided by the same half of counter word 2(j-1)+1
 * against its low half R:  A = [v 2^16 + w < floor(a_j 2^32)]. */
int oracle_multi_indicator(const oracle_multi_config *cfg, uint64_t seed, uint64_t trial,
                           int pattern, int32_t j, int32_t p) {
  const int32_t m = cfg ? cfg->n_drafters + 1 : 0;
  uint32_t ctr[4], key[2], out[4];
  if (!multi_valid(cfg) || j < 1 || j >= m || p < 1 || p > cfg->n_tokens - 1) return -1;
  if (pattern) {
    /* digit p-1 of the trial index in base m is j*(p) - 1; A_{j,p} = [j >= j*(p)] */
    uint64_t x = trial;
    int32_t i;
    for (i = 1; i < p; i++) x /= (uint64_t)m;
    return (int32_t)(x % (uint64_t)m) + 1 <= j;
  }
  key[0] = (uint32_t)seed;
  key[1] = (uint32_t)(seed >> 32);
  ctr[2] = (uint32_t)trial;
  ctr[3] = cfg->stream_id;
  if (cfg->rng_halves) {
    const uint64_t thr = oracle_threshold(cfg->accept_rate[j - 1]);
    const uint64_t T = thr >> 16, R = thr & 0xFFFFu;
    const int j8 = (int)((p - 1) & 7);
    uint32_t v, w;
    ctr[0] = (uint32_t)((p - 1) >> 3);
    ctr[1] = (uint32_t)(2 * (j - 1));
    oracle_philox4x32_10(ctr, key, out);
    v = multi_half16(out, j8);
    if (v < T) return 1;
    if (v > T) return 0;
    ctr[1] = (uint32_t)(2 * (j - 1) + 1); /* the tie-break draw */
    oracle_philox4x32_10(ctr, key, out);
    w = multi_half16(out, j8);
    return w < R;
  }
  ctr[0] = (uint32_t)((p - 1) >> 2);
  ctr[1] = (uint32_t)(j - 1);
  oracle_philox4x32_10(ctr, key, out);
  return (uint64_t)out[(p - 1) & 3] < oracle_threshold(cfg->accept_rate[j - 1]);
}

/* ---------------------------------------------------------------------- */
/* The thread tree.                                                        */
/* ---------------------------------------------------------------------- */
typedef struct {
  int64_t start, finish;
  int64_t first_child; /* index of the first of its m children, -1 until spawned */
  int64_t parent;      /* -1 for the threads of line 2                            */
  int32_t model;       /* j in 1..m                                               */
  int32_t level;       /* position of the token it generates, |J| + 1             */
  unsigned char alive, done;
} tnode;

typedef struct {
  tnode *v;
  int64_t n, cap;
} tpool;

typedef struct {
  int64_t *v;
  int64_t n, cap;
} theap; /* min-heap of node indices */

/* Event order: finish tick, then drafters before the target (a drafter as slow as
 * the target has sampled its token when the verifier compares, "all threads
 * ... have already finished"), then lower levels, then creation order. */
static int node_before(const tpool *P, int64_t a, int64_t b) {
  const tnode *x = &P->v[a], *y = &P->v[b];
  if (x->finish != y->finish) return x->finish < y->finish;
  if (x->model != y->model) return x->model < y->model;
  if (x->level != y->level) return x->level < y->level;
  return a < b;
}

static int heap_add(theap *h, const tpool *P, int64_t x) {
  int64_t i;
  if (h->n == h->cap) {
    int64_t nc = h->cap ? 2 * h->cap : 1024;
    int64_t *nv = (int64_t *)realloc(h->v, (size_t)nc * sizeof(int64_t));
    if (!nv) return -1;
    h->v = nv;
    h->cap = nc;
  }
  i = h->n++;
  h->v[i] = x;
  while (i > 0) {
    int64_t up = (i - 1) / 2;
    if (!node_before(P, h->v[i], h->v[up])) break;
    { int64_t t = h->v[i]; h->v[i] = h->v[up]; h->v[up] = t; }
    i = up;
  }
  return 0;
}

static int64_t heap_take(theap *h, const tpool *P) {
  int64_t top = h->v[0], i = 0;
  h->v[0] = h->v[--h->n];
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, s = i;
    if (l < h->n && node_before(P, h->v[l], h->v[s])) s = l;
    if (r < h->n && node_before(P, h->v[r], h->v[s])) s = r;
    if (s == i) break;
    { int64_t t = h->v[i]; h->v[i] = h->v[s]; h->v[s] = t; }
    i = s;
  }
  return top;
}

/* Initiate m threads C_{J + (j)}, j = 1..m, on the prefix ending at `parent` (line 2
 * with parent = -1, line 6 otherwise), all starting at time t. */
static int spawn(tpool *P, theap *h, int64_t parent, int32_t level, int64_t t,
                 const oracle_multi_config *c, int64_t max_threads) {
  const int32_t m = c->n_drafters + 1;
  int32_t j;
  if (P->n + m > max_threads) return -2;
  if (P->n + m > P->cap) {
    int64_t nc = P->cap ? 2 * P->cap : 1024;
    tnode *nv;
    while (nc < P->n + m) nc *= 2;
    nv = (tnode *)realloc(P->v, (size_t)nc * sizeof(tnode));
    if (!nv) return -1;
    P->v = nv;
    P->cap = nc;
  }
  if (parent >= 0) P->v[parent].first_child = P->n;
  for (j = 1; j <= m; j++) {
    tnode *x = &P->v[P->n];
    x->start = t;
    x->finish = t + (j == m ? c->t_target : c->t_drafter[j - 1]);
    x->first_child = -1;
    x->parent = parent;
    x->model = j;
    x->level = level;
    x->alive = 1;
    x->done = 0;
    if (heap_add(h, P, P->n)) return -1;
    P->n++;
  }
  return 0;
}

/* Terminate a thread and all its descendants (lines 8 and 10). */
static int kill_subtree(tpool *P, int64_t x, int32_t m) {
  int64_t *stack = NULL, n = 0, cap = 0;
  int rc = 0;
  stack = (int64_t *)malloc(64 * sizeof(int64_t));
  if (!stack) return -1;
  cap = 64;
  stack[n++] = x;
  while (n > 0) {
    const int64_t y = stack[--n];
    int32_t j;
    P->v[y].alive = 0;
    if (P->v[y].first_child < 0) continue;
    for (j = 0; j < m; j++) {
      if (n == cap) {
        int64_t *ns = (int64_t *)realloc(stack, (size_t)(2 * cap) * sizeof(int64_t));
        if (!ns) { rc = -1; goto out; }
        stack = ns;
        cap *= 2;
      }
      stack[n++] = P->v[y].first_child + j;
    }
  }
out:
  free(stack);
  return rc;
}

int oracle_multi_tree(const oracle_multi_config *cfg, uint64_t seed, uint64_t trial, int pattern,
                      int64_t max_threads, oracle_multi_out *out) {
  tpool P = {0};
  theap H = {0};
  int32_t m, N, v = 1;
  int64_t verifier, first_group = 0;
  int rc = -1;
  if (!multi_valid(cfg) || !out) return -1;
  m = cfg->n_drafters + 1;
  N = cfg->n_tokens;
  if (pattern) {
    /* m^(N-1) patterns must fit the 64-bit trial index */
    double cnt = 1.0;
    int32_t i;
    for (i = 1; i < N; i++) cnt *= (double)m;
    if (cnt > 18446744073709551615.0) return -1;
  }
  memset(out, 0, sizeof(*out));
  out->nonsi = (int64_t)N * cfg->t_target;

  /* line 2: m threads on the prompt; line 3: C_(m) is the current verifier */
  if ((rc = spawn(&P, &H, -1, 1, 0, cfg, max_threads)) != 0) goto done;
  verifier = first_group + (m - 1);
  rc = -1;

  while (H.n > 0) {
    int64_t x = heap_take(&H, &P);
    tnode *cx = &P.v[x];
    if (!cx->alive) continue; /* terminated threads never report (lines 8, 10) */
    cx->done = 1;
    if (cx->level < N) {
      /* line 6: initiate m threads on the prefix ending with x's token */
      int s = spawn(&P, &H, x, cx->level + 1, cx->finish, cfg, max_threads);
      if (s) { rc = s; goto done; }
      cx = &P.v[x];
    } else if (cx->model == m) {
      /* line 17: RETURN -- taken by the current verifier only (R25) */
      if (x == verifier) {
        out->dsi = cx->finish;
        rc = 0;
        goto done;
      }
      continue;
    } else {
      continue;
    }
    /* line 7: is x the current verifier?  The go-back of lines 13-14 re-enters here. */
    while (x == verifier && P.v[x].level < N) {
      const int32_t p = P.v[x].level;
      const int64_t sib0 = (P.v[x].parent >= 0) ? P.v[P.v[x].parent].first_child : first_group;
      int32_t j, jstar = m;
      /* line 9: j* = smallest j' whose token equals the verifier's (the target's) */
      for (j = 1; j < m; j++) {
        int a;
        if (!P.v[sib0 + j - 1].done) goto done; /* must have finished */
        a = oracle_multi_indicator(cfg, seed, trial, pattern, j, p);
        if (a < 0) goto done;
        if (a && P.v[sib0 + j - 1].alive) { jstar = j; break; }
      }
      /* line 8: terminate siblings with a different token; line 10: those after j* */
      for (j = 1; j <= m; j++) {
        int same = (j == m) || oracle_multi_indicator(cfg, seed, trial, pattern, j, p) == 1;
        if (!same || j > jstar)
          if (kill_subtree(&P, sib0 + j - 1, m)) goto done;
      }
      out->settled[jstar - 1] += 1;
      /* line 11: label C_{J + (j*, m)} as the current verifier; line 12: v = v + 1 */
      {
        const tnode *keep = &P.v[sib0 + jstar - 1];
        if (keep->first_child < 0) goto done; /* finished before x, so it has children */
        verifier = keep->first_child + (m - 1);
      }
      v += 1;
      if (v != p + 1) goto done;
      /* lines 13-14: if the new verifier already finished, go back to line 7 with it */
      if (!P.v[verifier].done) break;
      x = verifier;
      if (P.v[x].level == N) { /* an already finished last verifier returns (line 17) */
        out->dsi = P.v[x].finish;
        rc = 0;
        goto done;
      }
    }
  }
  rc = -1; /* the verifier chain never reached level N */
done:
  if (rc == 0) out->threads = P.n;
  free(P.v);
  free(H.v);
  return rc;
}

int oracle_multi_chain(const oracle_multi_config *cfg, uint64_t seed, uint64_t trial, int pattern,
                       oracle_multi_out *out) {
  int32_t m, N, p;
  int64_t s; /* start time of the threads of the current level (the verified prefix's end) */
  if (!multi_valid(cfg) || !out) return -1;
  m = cfg->n_drafters + 1;
  N = cfg->n_tokens;
  memset(out, 0, sizeof(*out));
  out->nonsi = (int64_t)N * cfg->t_target;
  s = 0; /* line 2: level 1 starts at 0 */
  for (p = 1; p < N; p++) {
    /* level p: m siblings start at s; the target sibling (the verifier) finishes at
       s + t_m, every drafter sibling has finished by then (Assumption 2); the kept one
       is j*, whose children (level p+1, incl. the next verifier) start when it ends */
    int32_t j, jstar = m;
    for (j = 1; j < m; j++) {
      const int a = oracle_multi_indicator(cfg, seed, trial, pattern, j, p);
      if (a < 0) return -1;
      if (a) { jstar = j; break; }
    }
    out->settled[jstar - 1] += 1;
    s += (jstar == m) ? cfg->t_target : cfg->t_drafter[jstar - 1];
  }
  /* level N: the last verifier starts at s and returns at s + t_m (line 17) */
  out->dsi = s + cfg->t_target;
  return 0;
}

int oracle_multi_run(const oracle_multi_config *cfg, uint64_t seed, uint64_t first, uint64_t count,
                     int pattern, oracle_multi_sums *sums, int64_t *dsi, int32_t *settled) {
  uint64_t i;
  int32_t j, m;
  if (!sums || !multi_valid(cfg)) return -1;
  m = cfg->n_drafters + 1;
  for (i = 0; i < count; i++) {
    oracle_multi_out o;
    if (oracle_multi_chain(cfg, seed, first + i, pattern, &o)) return -1;
    if (dsi) dsi[i] = o.dsi;
    if (settled)
      for (j = 0; j < m; j++) settled[i * (uint64_t)m + (uint64_t)j] = o.settled[j];
    sums->trials += 1;
    sums->sum_dsi += o.dsi;
    sums->sumsq_dsi += (uint64_t)o.dsi * (uint64_t)o.dsi;
    for (j = 0; j < m; j++) sums->sum_settled[j] += o.settled[j];
    sums->n_dsi_gt_nonsi += o.dsi > o.nonsi;
  }
  return 0;
}
