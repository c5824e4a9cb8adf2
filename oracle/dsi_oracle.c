/*
 * dsi_oracle.c -- plain, slow, single-threaded CPU oracle of the DSI Monte
 * Carlo latency simulator (arXiv 2405.14105).
 *
 * TEST INFRASTRUCTURE ONLY (see dsi_oracle.h).  Shares no code with the
 * product path.  It is deliberately literal: the SI latency comes from the
 * paper's pseudocode loop and the DSI latency from an event simulation of
 * Algorithm 1; neither uses the per-segment closed form the GPU evaluates.
 *
 * Citations: P:n = /root/reference/PAPER.md line n.
 */
#include "dsi_oracle.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11).  One round maps        */
/* (c0,c1,c2,c3) with key (k0,k1) to                                         */
/*   (hi(M1*c2) ^ c1 ^ k0, lo(M1*c2), hi(M0*c0) ^ c3 ^ k1, lo(M0*c0)),      */
/* M0 = 0xD2511F53, M1 = 0xCD9E8D57; the key is bumped by the Weyl constants */
/* W0 = 0x9E3779B9, W1 = 0xBB67AE85 between rounds.  Pinned by the Random123 */
/* known-answer vectors in tests/golden/philox4x32_10_kat.txt.               */
/* ------------------------------------------------------------------------ */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  int round;
  for (round = 0; round < 10; round++) {
    uint64_t p0, p1;
    uint32_t n0, n1, n2, n3;
    if (round > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    n1 = (uint32_t)p1;
    n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* A_p = [u < floor(a * 2^32)]: a = 0 never accepts, a = 1 always accepts.  */
/* a * 2^32 is an exact scaling of a double, so the floor is exact.          */
uint64_t oracle_threshold(double a) {
  double x = a * 4294967296.0;
  uint64_t t;
  if (!(a >= 0.0) || a > 1.0) return 0;
  t = (uint64_t)x; /* truncation == floor for x >= 0 */
  return t;
}

/* The indicator stream of one trial.                                        */
/*   key = (seed_lo, seed_hi); counter = (q_lo, q_hi, trial, stream_id);     */
/*   position p >= 1 uses q = (p-1) >> 2 and output word (p-1) & 3.          */
typedef struct {
  uint32_t key[2];
  uint32_t trial_lo;
  uint32_t stream_id;
  uint64_t thr;
  int pattern;
  uint64_t pattern_bits;
  int halves;
} indicator_stream;

/* The "halves" layout (R26; an alternative RNG contract, not the paper's -- the paper */
/* leaves the generator unspecified).  Position p >= 1 has call q = (p-1) >> 3 and     */
/* offset j = (p-1) & 7; its 16-bit draw v is the high half of output word j (j < 4) or the low   */
/* half of word j-4 of Philox at counter (q, 0, trial, stream_id).  With thr = T * 2^16 + R:      */
/*   v < T  -> accepted;   v > T -> rejected;                                                    */
/*   v == T -> accepted iff w < R, w the same half of the same word of counter (q, 1, trial,     */
/*             stream_id).                                                                       */
/* thr = 2^32 (a = 1) has T = 2^16 > v: always accepted; thr = 0 never.                          */
static uint32_t half16(const uint32_t out[4], int j) {
  uint32_t word = out[j & 3];
  if (j < 4) return word >> 16;
  return word & 0xFFFFu;
}

static int indicator_halves(const indicator_stream *s, int64_t p) {
  uint32_t ctr[4], out[4];
  uint64_t q = (uint64_t)(p - 1) >> 3;
  int j = (int)((p - 1) & 7);
  uint64_t T = s->thr >> 16, R = s->thr & 0xFFFFu;
  uint32_t v, w;
  ctr[0] = (uint32_t)q;
  ctr[1] = 0;
  ctr[2] = s->trial_lo;
  ctr[3] = s->stream_id;
  oracle_philox4x32_10(ctr, s->key, out);
  v = half16(out, j);
  if (v < T) return 1;
  if (v > T) return 0;
  ctr[1] = 1; /* the tie-break draw */
  oracle_philox4x32_10(ctr, s->key, out);
  w = half16(out, j);
  return w < R;
}

static int indicator(const indicator_stream *s, int64_t p) {
  uint32_t ctr[4], out[4];
  uint64_t q;
  if (s->pattern) {
    /* enumeration mode: A_p = bit (p-1) of the trial index */
    if (p - 1 >= 64) return 0;
    return (int)((s->pattern_bits >> (p - 1)) & 1u);
  }
  if (s->halves) return indicator_halves(s, p);
  q = (uint64_t)(p - 1) >> 2;
  ctr[0] = (uint32_t)q;
  ctr[1] = (uint32_t)(q >> 32);
  ctr[2] = s->trial_lo;
  ctr[3] = s->stream_id;
  oracle_philox4x32_10(ctr, s->key, out);
  return (uint64_t)out[(p - 1) & 3] < s->thr;
}

/* ------------------------------------------------------------------------ */
/* SI: the pseudocode of App. F.4, literally.                     */
/*   while total_toks < N: n = get_num_accepted(); total_toks += n + 1;      */
/*                         total_cost += k * t_d + t_t                        */
/* get_num_accepted() = number of leading accepted drafts among the next k   */
/* (n = min{i | A_i = 0} - 1, capped at k).  Indicators beyond    */
/* position N-1 may be read; the result does not depend on them (any read    */
/* of A(p), p >= N, ends the loop whatever its value).                       */
/* ------------------------------------------------------------------------ */
/* TTFT variant: the first iteration's first draft costs t_d1 and its target   */
/* forward t_t1 (each model's first forward).                          */
static void si_literal(const indicator_stream *s, int32_t N, int32_t k, int64_t t_t, int64_t t_d,
                       int64_t t_t1, int64_t t_d1, int32_t *iters_out, int64_t *cost_out,
                       int64_t *si_hist) {
  int64_t total_toks = 0;
  int64_t total_cost = 0;
  int32_t iters = 0;
  while (total_toks < N) {
    int32_t n = 0;
    int64_t start = total_toks;
    while (n < k && indicator(s, total_toks + n + 1) == 1) n += 1;
    total_toks += n + 1;
    if (iters == 0)
      total_cost += t_d1 + (int64_t)(k - 1) * t_d + t_t1;
    else
      total_cost += (int64_t)k * t_d + t_t;
    iters += 1;
    /* unbiased accepted-drafts histogram: only iterations whose whole k-draft
       window lies in positions 1..N-1 (north_star's SI pin) */
    if (si_hist && start + k + 1 <= N) si_hist[n] += 1;
  }
  *iters_out = iters;
  *cost_out = total_cost;
}

/* ------------------------------------------------------------------------ */
/* DSI: event simulation of Algorithm 1 + App. D lookahead       */
/* on SP identical FIFO target servers.                           */
/*                                                                            */
/* Reading (R1-R4, R7-R10): within a segment that starts at time T  */
/* with c tokens committed                                                    */
/*  - thread 0, a target forward on the committed prefix, is requested at T  */
/*    (Alg.1 line 2 at t=0; line 6's child C_{J+(m,m)} after a rejection);   */
/*  - the single drafter never blocks: draft of position c+j is done at      */
/*    T + j*t_d (Assumption 3);                                        */
/*  - verification task b >= 1 is requested when its k drafts are done, at   */
/*    T + b*k*t_d, while its first draft position c+(b-1)k+1 <= N-1;         */
/*  - a target forward on the prefix ending at e yields the target's tokens  */
/*    up to position e+1; thread 0 has e = c, thread b has e = c + b*k;      */
/*  - positions are settled in order; a mismatch (A_p = 0) commits the        */
/*    target's token p and terminates every other thread, queued task and    */
/*    draft (Alg.1 lines 8 and 10), restarting at the completion time;       */
/*  - the run ends when position N is settled (Alg.1 line 17 returns only    */
/*    from a target thread).                                       */
/* Events at equal times: server release (TARGET_DONE) before claims         */
/* (REQUEST); R8.                                                   */
/* ------------------------------------------------------------------------ */
/* Fresh-verifier variant only: EV_FRESH_DONE completes a fresh forward (a     */
/* completion, like EV_TARGET_DONE) and EV_CHECK -- the decision whether to   */
/* start one -- runs after every other event of its time stamp.               */
enum { EV_TARGET_DONE = 0, EV_FRESH_DONE = 1, EV_REQUEST = 2, EV_CHECK = 3 };

typedef struct {
  int64_t time;
  int32_t cls;
  int64_t b;      /* thread index within the segment */
  int64_t epoch;  /* segment the event belongs to (stale => cancelled) */
} event;

typedef struct {
  event *v;
  size_t n, cap;
} heap;

static int ev_less(const event *x, const event *y) {
  if (x->time != y->time) return x->time < y->time;
  if (x->cls != y->cls) return x->cls < y->cls;
  return x->b < y->b;
}

static int heap_push(heap *h, event e) {
  size_t i;
  if (h->n == h->cap) {
    size_t nc = h->cap ? 2 * h->cap : 64;
    event *nv = (event *)realloc(h->v, nc * sizeof(event));
    if (!nv) return -1;
    h->v = nv;
    h->cap = nc;
  }
  i = h->n++;
  h->v[i] = e;
  while (i > 0) {
    size_t parent = (i - 1) / 2;
    if (!ev_less(&h->v[i], &h->v[parent])) break;
    {
      event t = h->v[i];
      h->v[i] = h->v[parent];
      h->v[parent] = t;
    }
    i = parent;
  }
  return 0;
}

static event heap_pop(heap *h) {
  event top = h->v[0];
  size_t i = 0;
  h->v[0] = h->v[--h->n];
  for (;;) {
    size_t l = 2 * i + 1, r = l + 1, s = i;
    if (l < h->n && ev_less(&h->v[l], &h->v[s])) s = l;
    if (r < h->n && ev_less(&h->v[r], &h->v[s])) s = r;
    if (s == i) break;
    {
      event t = h->v[i];
      h->v[i] = h->v[s];
      h->v[s] = t;
    }
    i = s;
  }
  return top;
}

typedef struct {
  int64_t *v;
  size_t head, tail, cap;
} fifo;

static int fifo_push(fifo *q, int64_t b) {
  if (q->tail == q->cap) {
    size_t nc = q->cap ? 2 * q->cap : 64;
    int64_t *nv = (int64_t *)realloc(q->v, nc * sizeof(int64_t));
    if (!nv) return -1;
    q->v = nv;
    q->cap = nc;
  }
  q->v[q->tail++] = b;
  return 0;
}

/* TTFT variant: in the first segment the drafter's first draft takes t_d1  */
/* (draft c+j is done at t_d1 + (j-1) t_d) and thread 0 -- the target pool's */
/* first-ever forward -- takes t_t1; everything later costs the TPOTs.       */
typedef struct {
  unsigned char *v;
  size_t cap;
} flagset;

static int flags_set(flagset *f, int64_t i) { /* 0 on success */
  if ((size_t)i >= f->cap) {
    size_t nc = f->cap ? 2 * f->cap : 64;
    unsigned char *nv;
    while (nc <= (size_t)i) nc *= 2;
    nv = (unsigned char *)realloc(f->v, nc);
    if (!nv) return -1;
    memset(nv + f->cap, 0, nc - f->cap);
    f->v = nv;
    f->cap = nc;
  }
  f->v[i] = 1;
  return 0;
}

static int flag_get(const flagset *f, int64_t i) { return (size_t)i < f->cap && f->v[i]; }

/* Fresh-verifier variant: completion time of each started thread of the segment */
/* (0 = not started).                                                           */
typedef struct {
  int64_t *v;
  size_t cap;
} timeset;

static int time_set(timeset *f, int64_t i, int64_t t) { /* 0 on success */
  if ((size_t)i >= f->cap) {
    size_t nc = f->cap ? 2 * f->cap : 64;
    int64_t *nv;
    while (nc <= (size_t)i) nc *= 2;
    nv = (int64_t *)realloc(f->v, nc * sizeof(int64_t));
    if (!nv) return -1;
    memset(nv + f->cap, 0, (nc - f->cap) * sizeof(int64_t));
    f->v = nv;
    f->cap = nc;
  }
  f->v[i] = t;
  return 0;
}

static int64_t time_get(const timeset *f, int64_t i) { return (size_t)i < f->cap ? f->v[i] : 0; }

/* Fresh-verifier variant (R24).  Thm 2's proof     */
/* (P:445): when the verifier accepts and commits x_{k+1}, "DSI either invokes */
/* a new current verifier thread or labels an existing thread as the current  */
/* verifier".  Read as: each time the committed prefix grows to position p at */
/* time tau (after every other event at tau), unless a started target thread */
/* covering p+1 completes by tau + t_t, a fresh target forward starts at tau  */
/* on one extra server (outside the SP pool): its prefix is the committed     */
/* tokens plus the drafts done by tau, at most k of them (the lookahead,      */
/* P:143), so it yields the target's tokens for p+1 .. min(d, p+k)+1 (d = the */
/* last draft done by tau) at tau + t_t.  A newer fresh forward supersedes an */
/* older one (which no longer covers p+1); a rejection cancels it like every  */
/* other thread.                                                              */
/* Optional event trace (oracle_trace_trial; SPEC S:177-180 TraceEvent, SURVEY 8(c).2 "optional
   debug outputs"): one JSON object per line appended to a caller buffer, in processing order
   (the caller sorts by time).  NULL outside oracle_trace_trial. */
typedef struct {
  char *buf;
  size_t cap, len;
  int overflow;
} trace_sink;
static trace_sink *g_trace = NULL;

static void trace_ev(const char *kind, int64_t t, int64_t pos, int64_t thread, int64_t seg) {
  int n;
  if (!g_trace) return;
  n = snprintf(g_trace->buf + g_trace->len, g_trace->cap - g_trace->len,
               "{\"kind\": \"%s\", \"time\": %lld, \"position\": %lld, \"thread\": %lld, \"segment\": %lld}\n",
               kind, (long long)t, (long long)pos, (long long)thread, (long long)seg);
  if (n < 0 || (size_t)n >= g_trace->cap - g_trace->len) {
    g_trace->overflow = 1;
    return;
  }
  g_trace->len += (size_t)n;
}

static int dsi_event_sim(const indicator_stream *s, int32_t N, int32_t k, int32_t SP, int64_t t_t,
                         int64_t t_d, int64_t t_t1, int64_t t_d1, int fresh, oracle_trial_out *out) {
  heap h = {0, 0, 0};
  fifo q = {0, 0, 0, 0};
  flagset fin = {0, 0}; /* threads of the current segment that have finished */
  timeset ends = {0, 0}; /* fresh variant: completion time of started threads */
  int64_t T = 0;   /* segment start time */
  int64_t c = 0;   /* committed tokens */
  int64_t epoch = 0;
  int64_t fresh_id = 0;
  int32_t segments = 0, peak_busy = 0, max_queue = 0, forwards = 0;
  int rc = -1;
  const int ttft = t_t1 != t_t || t_d1 != t_d;

  for (;;) { /* one iteration per segment */
    int64_t r = c + 1;          /* next unresolved position */
    int64_t next_done = 0;      /* the next thread whose tokens are settled (the verifier) */
    int32_t busy = 0;
    int64_t b;
    int64_t n_fin = 0;          /* threads of this segment finished so far */
    int restarted = 0;
    /* fresh variant: the live fresh forward covers [f_lo, f_hi], completes at f_end */
    int f_live = 0, f_done = 0;
    int64_t f_lo = 0, f_hi = 0, f_end = 0;
    epoch += 1;
    segments += 1;
    /* time at which the draft of position c+j is done: T + lag + j*t_d */
    const int64_t lag = segments == 1 ? t_d1 - t_d : 0;
    q.head = q.tail = 0;        /* cancelled tasks leave the queue */
    if (fin.v) memset(fin.v, 0, fin.cap);
    if (ends.v) memset(ends.v, 0, ends.cap * sizeof(int64_t));

    h.n = 0; /* cancellation: every pending thread, task and draft is dropped */
    trace_ev("SegmentStart", T, c + 1, -1, segments);
    if (heap_push(&h, (event){T, EV_REQUEST, 0, epoch})) goto done;

    while (!restarted) {
      event e;
      int64_t r_before;
      if (h.n == 0) goto done; /* cannot happen: position N is always settled */
      e = heap_pop(&h);
      if (e.epoch != epoch) continue; /* cancelled thread / task */
      r_before = r;
      if (e.cls == EV_REQUEST) {
        /* the drafter keeps drafting: task b+1 is requested once its k drafts
           are done, while its first draft position c+b*k+1 is <= N-1 */
        b = e.b + 1;
        if (c + (b - 1) * (int64_t)k + 1 <= (int64_t)N - 1)
          if (heap_push(&h, (event){T + lag + b * (int64_t)k * t_d, EV_REQUEST, b, epoch})) goto done;
        if (busy < SP) {
          busy += 1;
          forwards += 1;
          if (busy > peak_busy) peak_busy = busy;
          trace_ev("VerifyDispatch", e.time, e.b == 0 ? c + 1 : c + e.b * (int64_t)k + 1, e.b, segments);
          const int64_t service = (segments == 1 && e.b == 0) ? t_t1 : t_t;
          if (heap_push(&h, (event){e.time + service, EV_TARGET_DONE, e.b, epoch})) goto done;
          if (fresh && time_set(&ends, e.b, e.time + service)) goto done;
        } else {
          trace_ev("VerifyQueued", e.time, c + e.b * (int64_t)k + 1, e.b, segments);
          if (fifo_push(&q, e.b)) goto done;
          if ((int32_t)(q.tail - q.head) > max_queue) max_queue = (int32_t)(q.tail - q.head);
        }
        continue;
      }
      if (e.cls == EV_CHECK) { /* fresh variant: start a fresh forward for position r? */
        int64_t j = r - c, bb, d;
        if (e.b != r) continue; /* the prefix has grown since: a later check decides */
        bb = (j == 1) ? 0 : (j - 1 + k - 1) / k; /* the regular thread covering r */
        if (time_get(&ends, bb) && time_get(&ends, bb) <= e.time + t_t) continue;
        if (f_live && !f_done && f_lo <= r && r <= f_hi && f_end <= e.time + t_t) continue;
        d = c + (e.time - T) / t_d; /* the last draft done by now */
        trace_ev("FreshDispatch", e.time, r, -1, segments);
        f_live = 1;
        f_done = 0;
        f_lo = r;
        f_hi = (d < r - 1 + k ? d : r - 1 + k) + 1;
        f_end = e.time + t_t;
        fresh_id += 1;
        forwards += 1;
        if (heap_push(&h, (event){f_end, EV_FRESH_DONE, fresh_id, epoch})) goto done;
        continue;
      }
      if (e.cls == EV_FRESH_DONE) {
        if (e.b != fresh_id) continue; /* superseded */
        f_done = 1;
      } else { /* EV_TARGET_DONE */
        /* Threads complete in index order: start times strictly increase and every
           service takes t_t (SURVEY 8(c).2 asks the oracle to assert it).  Only the
           TTFT variant's slower first forward can break it, in the first segment only. */
        if (!(ttft && segments == 1) && e.b != n_fin) goto done;
        n_fin += 1;
        busy -= 1;
        trace_ev("VerifyDone", e.time, e.b == 0 ? c + 1 : c + e.b * (int64_t)k + 1, e.b, segments);
        trace_ev("ServerFreed", e.time, -1, e.b, segments);
        if (q.head < q.tail) { /* FIFO: the head of the queue starts now */
          int64_t nb = q.v[q.head++];
          trace_ev("VerifyDispatch", e.time, c + nb * (int64_t)k + 1, nb, segments);
          busy += 1;
          forwards += 1;
          if (busy > peak_busy) peak_busy = busy;
          if (heap_push(&h, (event){e.time + t_t, EV_TARGET_DONE, nb, epoch})) goto done;
          if (fresh && time_set(&ends, nb, e.time + t_t)) goto done;
        }
        if (flags_set(&fin, e.b)) goto done;
      }
      if (!fresh) {
        int64_t hi, p;
        /* Positions are settled in order.  A thread that finishes before an
           earlier one (possible only when the first forward is slower, TTFT)
           waits: its tokens are read when the verifier reaches it (Alg. 1
           lines 133-134, "if C has already finished, go back"). */
        while (!restarted && flag_get(&fin, next_done)) {
          const int64_t bb = next_done++;
          hi = (bb == 0) ? c + 1 : c + bb * (int64_t)k + 1;
          for (p = r; p <= hi; p++) {
            if (p == N) { /* the N-th token is committed: L_DSI */
              trace_ev("TokenEmitted", e.time, p, bb, segments);
              out->dsi = e.time;
              rc = 0;
              goto done;
            }
            /* assertion: the draft of position p exists by now (t_d <= t_t, t_d1 <= t_t1) */
            if (T + lag + (p - c) * t_d > e.time) goto done;
            trace_ev("DraftDone", T + lag + (p - c) * t_d, p, -1, segments);
            if (indicator(s, p) == 0) { /* rejection: restart from the target's token */
              trace_ev("Reject", e.time, p, bb, segments);
              trace_ev("TokenEmitted", e.time, p, bb, segments);
              T = e.time;
              c = p;
              restarted = 1;
              break;
            }
            trace_ev("Accept", e.time, p, bb, segments);
            trace_ev("TokenEmitted", e.time, p, bb, segments);
          }
          if (!restarted) r = hi + 1;
        }
      } else {
        /* fresh variant: position r is settled once a finished thread covers it
           (regular thread 0 covers c+1, thread b >= 1 covers c+(b-1)k+2 ..
           c+bk+1, the fresh forward [f_lo, f_hi]); in order, as above */
        for (;;) {
          const int64_t j = r - c;
          const int64_t bb = (j == 1) ? 0 : (j - 1 + k - 1) / k;
          if (!flag_get(&fin, bb) && !(f_live && f_done && f_lo <= r && r <= f_hi)) break;
          if (r == N) {
            trace_ev("TokenEmitted", e.time, r, bb, segments);
            out->dsi = e.time;
            rc = 0;
            goto done;
          }
          if (T + (r - c) * t_d > e.time) goto done; /* the draft exists (t_d <= t_t) */
          trace_ev("DraftDone", T + (r - c) * t_d, r, -1, segments);
          if (indicator(s, r) == 0) {
            trace_ev("Reject", e.time, r, bb, segments);
            trace_ev("TokenEmitted", e.time, r, bb, segments);
            T = e.time;
            c = r;
            restarted = 1;
            break;
          }
          trace_ev("Accept", e.time, r, bb, segments);
          trace_ev("TokenEmitted", e.time, r, bb, segments);
          r += 1;
        }
        if (!restarted && r != r_before)
          if (heap_push(&h, (event){e.time, EV_CHECK, r, epoch})) goto done;
      }
    }
  }
done:
  out->dsi_segments = segments;
  out->dsi_peak_busy = peak_busy;
  out->dsi_max_queue = max_queue;
  out->dsi_forwards = forwards;
  free(h.v);
  free(q.v);
  free(fin.v);
  free(ends.v);
  return rc;
}

static int valid(const oracle_config *cfg) {
  if (!cfg) return 0;
  if (cfg->n_tokens < 1 || cfg->lookahead < 1 || cfg->sp_degree < 1) return 0;
  if (cfg->t_drafter < 1 || cfg->t_target < cfg->t_drafter) return 0; /* Assumption 2 */
  if (cfg->t_target_first < 0 || cfg->t_drafter_first < 0) return 0;
  {
    const int64_t tt1 = cfg->t_target_first ? cfg->t_target_first : cfg->t_target;
    const int64_t td1 = cfg->t_drafter_first ? cfg->t_drafter_first : cfg->t_drafter;
    if (td1 > tt1) return 0; /* Assumption 2 for the first forwards */
    if (cfg->fresh_verifier && (tt1 != cfg->t_target || td1 != cfg->t_drafter)) return 0;
  }
  if (!(cfg->accept_rate >= 0.0 && cfg->accept_rate <= 1.0)) return 0;
  if (cfg->rng_halves != 0 && cfg->rng_halves != 1) return 0;
  return 1;
}

int oracle_trial(const oracle_config *cfg, uint64_t seed, uint64_t trial, int pattern,
                 oracle_trial_out *out, int64_t *si_hist, int64_t *seg_hist) {
  indicator_stream s;
  int32_t N, p, last_zero = 0;
  if (!valid(cfg) || !out) return -1;
  if (pattern && cfg->n_tokens > 33) return -1;
  N = cfg->n_tokens;
  memset(out, 0, sizeof(*out));
  s.key[0] = (uint32_t)seed;
  s.key[1] = (uint32_t)(seed >> 32);
  s.trial_lo = (uint32_t)trial;
  s.stream_id = cfg->stream_id;
  s.thr = oracle_threshold(cfg->accept_rate);
  s.pattern = pattern;
  s.pattern_bits = trial;
  s.halves = cfg->rng_halves;

  /* per-trial counts over positions 1..N-1 (position N has no indicator) */
  out->m = 1;
  for (p = 1; p <= N - 1; p++) {
    if (indicator(&s, p)) {
      out->acc += 1;
    } else {
      out->m += 1;
      if (seg_hist) seg_hist[(p - last_zero) < 63 ? (p - last_zero) : 63] += 1;
      last_zero = p;
    }
  }
  if (seg_hist) seg_hist[(N - last_zero) < 63 ? (N - last_zero) : 63] += 1;

  {
    const int64_t tt1 = cfg->t_target_first ? cfg->t_target_first : cfg->t_target;
    const int64_t td1 = cfg->t_drafter_first ? cfg->t_drafter_first : cfg->t_drafter;
    out->nonsi = tt1 + (int64_t)(N - 1) * cfg->t_target; /* P:537; TTFT first */
    si_literal(&s, N, cfg->lookahead, cfg->t_target, cfg->t_drafter, tt1, td1, &out->iters, &out->si,
               si_hist);
    if (dsi_event_sim(&s, N, cfg->lookahead, cfg->sp_degree, cfg->t_target, cfg->t_drafter, tt1, td1,
                      cfg->fresh_verifier != 0, out))
      return -1;
  }
  if (out->dsi_segments != out->m) return -1;
  return 0;
}

/* One trial with its DSI event trace written to buf (JSON lines, NUL-terminated); *len = bytes
   written.  Returns oracle_trial's code, or -2 if buf is too small. */
int oracle_trace_trial(const oracle_config *cfg, uint64_t seed, uint64_t trial, int pattern,
                       oracle_trial_out *out, char *buf, size_t cap, size_t *len) {
  trace_sink t = {buf, cap, 0, 0};
  int rc;
  if (!buf || cap == 0 || !len) return -1;
  buf[0] = 0;
  g_trace = &t;
  rc = oracle_trial(cfg, seed, trial, pattern, out, NULL, NULL);
  g_trace = NULL;
  *len = t.len;
  return t.overflow ? -2 : rc;
}

int oracle_run(const oracle_config *cfg, uint64_t seed, uint64_t first, uint64_t count,
               int pattern, oracle_sums *sums,
               int32_t *acc, int32_t *m, int32_t *iters, int64_t *si, int64_t *dsi,
               int64_t *si_hist, int64_t *seg_hist) {
  uint64_t i;
  if (!sums) return -1;
  for (i = 0; i < count; i++) {
    oracle_trial_out o;
    if (oracle_trial(cfg, seed, first + i, pattern, &o, si_hist, seg_hist)) return -1;
    if (acc) acc[i] = o.acc;
    if (m) m[i] = o.m;
    if (iters) iters[i] = o.iters;
    if (si) si[i] = o.si;
    if (dsi) dsi[i] = o.dsi;
    sums->trials += 1;
    sums->sum_acc += o.acc;
    sums->sum_m += o.m;
    sums->sum_iters += o.iters;
    sums->sum_si += o.si;
    sums->sum_dsi += o.dsi;
    sums->sumsq_si += (uint64_t)o.si * (uint64_t)o.si;
    sums->sumsq_dsi += (uint64_t)o.dsi * (uint64_t)o.dsi;
    sums->n_dsi_gt_nonsi += o.dsi > o.nonsi;
    sums->n_dsi_gt_si += o.dsi > o.si;
  }
  return 0;
}
