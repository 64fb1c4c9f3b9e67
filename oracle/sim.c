/*
 * ORACLE (test infrastructure only) -- plain fp64/int64 CPU reference of the GDP
 * step-time cost model.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code
 * with paper_1910_01578_b200/ (the product).
 *
 * What it computes: SPEC.md:275-284 `simulate` (the cost model named by the north
 * star), as made precise by SURVEY.md §8(c) O11 and the readings R19/R20 listed in
 * DESIGN.md §"Readings".  This file follows O11's formulation literally: per-op
 * ready times rdy[], a per-device min-heap keyed (ready_time, id), a pending list
 * of copy-arrival allocations, and instants visited in increasing time order with
 * the per-instant rounds
 *   (1) apply copy allocations due now,
 *   (2) finish ops ending now in ascending id (frees, then out-edge relaxation in
 *       ascending consumer id; cross-device transfers serialised FIFO on the
 *       directed channel (D u -> D w), arrival = max(t, ch_free)+ceil(bytes/bw)+lat),
 *   (3) each idle device (ascending) starts its heap minimum if ready_time <= t,
 *   (4) sample per-device peaks,
 *   (5) repeat (2)-(4) while some op started now with zero duration.
 * Reward (§4.1 P:177 "negative square root of the run time", "-10" for
 * invalid placements): r = valid ? -sqrt(makespan / 1e6) : -10.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { int64_t key; int32_t id; int32_t dst; } item_t;   /* heap entry */

typedef struct { item_t *a; int n, cap; } heap_t;

static int item_less(const item_t *x, const item_t *y) {
  return x->key < y->key || (x->key == y->key && x->id < y->id);
}
static void heap_push(heap_t *h, item_t it) {
  if (h->n == h->cap) { h->cap = h->cap ? 2 * h->cap : 64; h->a = (item_t *)realloc(h->a, sizeof(item_t) * h->cap); }
  int i = h->n++;
  h->a[i] = it;
  while (i > 0) {
    int p = (i - 1) / 2;
    if (!item_less(&h->a[i], &h->a[p])) break;
    item_t t = h->a[p]; h->a[p] = h->a[i]; h->a[i] = t; i = p;
  }
}
static item_t heap_pop(heap_t *h) {
  item_t top = h->a[0];
  h->a[0] = h->a[--h->n];
  int i = 0;
  for (;;) {
    int l = 2 * i + 1, r = l + 1, m = i;
    if (l < h->n && item_less(&h->a[l], &h->a[m])) m = l;
    if (r < h->n && item_less(&h->a[r], &h->a[m])) m = r;
    if (m == i) break;
    item_t t = h->a[m]; h->a[m] = h->a[i]; h->a[i] = t; i = m;
  }
  return top;
}

typedef struct {
  int32_t N; int64_t E;
  const int64_t *cost, *out, *mem;
  const int32_t *coloc;
  /* CSR built once */
  int64_t *optr; int32_t *oidx;   /* out-edges, consumers ascending */
  int64_t *iptr; int32_t *iidx;   /* in-edges, producers ascending */
  int32_t d;
  const int64_t *cap; const int32_t *speed; const int64_t *bpt; const int32_t *lat;
} ctx_t;

static void build_csr(ctx_t *c, const int32_t *edges) {
  int32_t N = c->N; int64_t E = c->E;
  c->optr = (int64_t *)calloc(N + 1, sizeof(int64_t));
  c->iptr = (int64_t *)calloc(N + 1, sizeof(int64_t));
  c->oidx = (int32_t *)malloc(sizeof(int32_t) * (E ? E : 1));
  c->iidx = (int32_t *)malloc(sizeof(int32_t) * (E ? E : 1));
  for (int64_t e = 0; e < E; e++) { c->optr[edges[2 * e] + 1]++; c->iptr[edges[2 * e + 1] + 1]++; }
  for (int32_t v = 0; v < N; v++) { c->optr[v + 1] += c->optr[v]; c->iptr[v + 1] += c->iptr[v]; }
  int64_t *fo = (int64_t *)malloc(sizeof(int64_t) * (N + 1));
  int64_t *fi = (int64_t *)malloc(sizeof(int64_t) * (N + 1));
  memcpy(fo, c->optr, sizeof(int64_t) * (N + 1));
  memcpy(fi, c->iptr, sizeof(int64_t) * (N + 1));
  /* edges are given sorted by (producer, consumer): fills are ascending per row
     for out-edges; in-edges get ascending producers because producers ascend. */
  for (int64_t e = 0; e < E; e++) {
    int32_t u = edges[2 * e], w = edges[2 * e + 1];
    c->oidx[fo[u]++] = w;
    c->iidx[fi[w]++] = u;
  }
  free(fo); free(fi);
}

static void free_csr(ctx_t *c) { free(c->optr); free(c->iptr); free(c->oidx); free(c->iidx); }

static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

/* one placement; outputs: rep[0]=makespan, rep[1]=cross_bytes, rep[2]=valid, rep[3]=violation */
static void simulate_one(const ctx_t *c, const uint8_t *D, int64_t *rep, int64_t *peak, int64_t *busy,
                         int64_t *start_out, double *reward) {
  const int32_t N = c->N, d = c->d;
  for (int k = 0; k < d; k++) { peak[k] = 0; busy[k] = 0; }
  rep[0] = rep[1] = 0; rep[2] = 0; rep[3] = 0;
  for (int32_t v = 0; v < N; v++)
    if (D[v] >= d) { rep[3] = 3; *reward = -10.0; if (start_out) for (int32_t u = 0; u < N; u++) start_out[u] = -1; return; }
  int violation = 0;
  if (c->coloc) {
    /* every group must map to one device: compare with the first member seen */
    int32_t maxg = -1;
    for (int32_t v = 0; v < N; v++) if (c->coloc[v] > maxg) maxg = c->coloc[v];
    if (maxg >= 0) {
      int32_t *gdev = (int32_t *)malloc(sizeof(int32_t) * (maxg + 1));
      for (int32_t g = 0; g <= maxg; g++) gdev[g] = -1;
      for (int32_t v = 0; v < N; v++) {
        int32_t g = c->coloc[v];
        if (g < 0) continue;
        if (gdev[g] < 0) gdev[g] = D[v]; else if (gdev[g] != D[v]) violation = 1;
      }
      free(gdev);
    }
  }
  int64_t *rdy = (int64_t *)calloc(N, sizeof(int64_t));
  int32_t *rem_in = (int32_t *)malloc(sizeof(int32_t) * N);
  int32_t *rem_cons = (int32_t *)malloc(sizeof(int32_t) * N);
  int64_t mem[8], chfree[64];
  int32_t run_op[8]; int64_t run_fin[8];
  heap_t heaps[8]; heap_t pending = {0, 0, 0};
  memset(heaps, 0, sizeof(heaps));
  for (int k = 0; k < d; k++) { mem[k] = 0; run_op[k] = -1; run_fin[k] = 0; }
  for (int k = 0; k < d * d; k++) chfree[k] = 0;
  int64_t cross = 0;
  for (int32_t v = 0; v < N; v++) {
    rem_in[v] = (int32_t)(c->iptr[v + 1] - c->iptr[v]);
    rem_cons[v] = (int32_t)(c->optr[v + 1] - c->optr[v]);
    mem[D[v]] += c->mem[v];                         /* static bytes resident all step */
    busy[D[v]] += c->cost[v] * (int64_t)c->speed[D[v]];
    for (int64_t e = c->optr[v]; e < c->optr[v + 1]; e++)
      if (D[c->oidx[e]] != D[v]) cross += c->out[v];
    if (start_out) start_out[v] = -1;
  }
  for (int k = 0; k < d; k++) peak[k] = mem[k];
  for (int32_t v = 0; v < N; v++)
    if (rem_in[v] == 0) { item_t it = {0, v, 0}; heap_push(&heaps[D[v]], it); }
  int64_t t = 0, makespan = 0;
  int32_t fin[8];
  for (;;) {
    int changed;
    do {
      changed = 0;
      /* (1) copy allocations due now */
      while (pending.n > 0 && pending.a[0].key <= t) { item_t it = heap_pop(&pending); mem[it.dst] += c->out[it.id]; }
      /* (2) finishes at t, ascending id */
      int nf = 0;
      for (int k = 0; k < d; k++) if (run_op[k] >= 0 && run_fin[k] == t) fin[nf++] = run_op[k];
      qsort(fin, nf, sizeof(int32_t), cmp_i32);
      for (int i = 0; i < nf; i++) {
        int32_t v = fin[i]; int k = D[v];
        run_op[k] = -1;
        for (int64_t e = c->iptr[v]; e < c->iptr[v + 1]; e++) {
          int32_t u = c->iidx[e];
          if (D[u] != k) mem[k] -= c->out[u];                 /* copy held by consumer v */
          if (--rem_cons[u] == 0) mem[D[u]] -= c->out[u];     /* producer output dead */
        }
        if (c->optr[v + 1] == c->optr[v]) mem[k] -= c->out[v]; /* sink output */
        for (int64_t e = c->optr[v]; e < c->optr[v + 1]; e++) {
          int32_t w = c->oidx[e]; int tk = D[w];
          int64_t arr;
          if (tk == k) arr = t;
          else {
            int64_t bw = c->bpt[k * d + tk];
            int64_t xfer = (c->out[v] + bw - 1) / bw + c->lat[k * d + tk];
            int64_t st = t > chfree[k * d + tk] ? t : chfree[k * d + tk];
            arr = st + xfer;
            chfree[k * d + tk] = arr;
            if (arr <= t) mem[tk] += c->out[v];
            else { item_t it = {arr, v, tk}; heap_push(&pending, it); }
          }
          if (arr > rdy[w]) rdy[w] = arr;
          if (--rem_in[w] == 0) { item_t it = {rdy[w], w, 0}; heap_push(&heaps[tk], it); }
        }
      }
      /* (3) dispatch */
      for (int k = 0; k < d; k++) {
        if (run_op[k] >= 0 || heaps[k].n == 0 || heaps[k].a[0].key > t) continue;
        item_t it = heap_pop(&heaps[k]);
        int64_t dur = c->cost[it.id] * (int64_t)c->speed[k];
        run_op[k] = it.id; run_fin[k] = t + dur;
        if (start_out) start_out[it.id] = t;
        mem[k] += c->out[it.id];
        if (run_fin[k] > makespan) makespan = run_fin[k];
        if (dur == 0) changed = 1;
      }
      /* (4) peaks */
      for (int k = 0; k < d; k++) if (mem[k] > peak[k]) peak[k] = mem[k];
    } while (changed);
    /* next instant */
    int64_t nt = INT64_MAX;
    for (int k = 0; k < d; k++) {
      if (run_op[k] >= 0) { if (run_fin[k] < nt) nt = run_fin[k]; }
      else if (heaps[k].n > 0 && heaps[k].a[0].key < nt) nt = heaps[k].a[0].key;
    }
    if (pending.n > 0 && pending.a[0].key < nt) nt = pending.a[0].key;
    if (nt == INT64_MAX) break;
    t = nt;
  }
  int oom = 0;
  for (int k = 0; k < d; k++) if (peak[k] > c->cap[k]) oom = 1;
  rep[0] = makespan; rep[1] = cross;
  rep[3] = violation ? 1 : (oom ? 2 : 0);
  rep[2] = rep[3] == 0;
  *reward = rep[2] ? -sqrt((double)makespan / 1e6) : -10.0;
  for (int k = 0; k < d; k++) free(heaps[k].a);
  free(pending.a); free(rdy); free(rem_in); free(rem_cons);
}

typedef struct {
  const ctx_t *c; const uint8_t *D; int64_t B, b0, b1;
  int64_t *rep, *peak, *busy; double *reward;
} job_t;

static void *run_job(void *p) {
  job_t *j = (job_t *)p;
  for (int64_t b = j->b0; b < j->b1; b++)
    simulate_one(j->c, j->D + b * j->c->N, j->rep + 4 * b, j->peak + b * j->c->d, j->busy + b * j->c->d,
                 NULL, j->reward + b);
  return NULL;
}

/* Batch entry: B placements (B x N bytes, placement-major).  threads <= 1 runs on
   the calling thread.  rep is B x 4 int64 (makespan, cross_bytes, valid, violation). */
int oracle_simulate_batch(int32_t N, int64_t E, const int32_t *edges, const int64_t *cost,
                          const int64_t *out, const int64_t *mem, const int32_t *coloc, int32_t d,
                          const int64_t *cap, const int32_t *speed, const int64_t *bpt,
                          const int32_t *lat, const uint8_t *D, int64_t B, int32_t threads,
                          int64_t *rep, int64_t *peak, int64_t *busy, double *reward,
                          int64_t *start_first /* nullable: start times of placement 0 */) {
  if (N <= 0 || d < 1 || d > 8) return 1;
  ctx_t c = {0};
  c.N = N; c.E = E; c.cost = cost; c.out = out; c.mem = mem; c.coloc = coloc;
  c.d = d; c.cap = cap; c.speed = speed; c.bpt = bpt; c.lat = lat;
  build_csr(&c, edges);
  if (start_first && B > 0) {
    double r;
    simulate_one(&c, D, rep, peak, busy, start_first, &r);
  }
  if (threads <= 1) {
    for (int64_t b = 0; b < B; b++) simulate_one(&c, D + b * N, rep + 4 * b, peak + b * d, busy + b * d, NULL, reward + b);
  } else {
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * threads);
    job_t *jobs = (job_t *)malloc(sizeof(job_t) * threads);
    for (int i = 0; i < threads; i++) {
      jobs[i].c = &c; jobs[i].D = D; jobs[i].B = B;
      jobs[i].b0 = B * i / threads; jobs[i].b1 = B * (i + 1) / threads;
      jobs[i].rep = rep; jobs[i].peak = peak; jobs[i].busy = busy; jobs[i].reward = reward;
      pthread_create(&th[i], NULL, run_job, &jobs[i]);
    }
    for (int i = 0; i < threads; i++) pthread_join(th[i], NULL);
    free(th); free(jobs);
  }
  free_csr(&c);
  return 0;
}
