// Step-time cost model (SPEC.md:275-284 `simulate`, semantics in DESIGN.md §"Cost model")
// and the reward / advantage of PAPER.md §4.1.
//
// One CTA (one warp) per sampled placement.  The discrete-event list schedule is
// reformulated so that no per-op ready time and no priority queue is needed:
//   * every op keeps a counter of inputs that have not ARRIVED yet; it becomes available
//     at the instant the counter reaches 0, so its ready time is that instant;
//   * ops that become available at the same instant are sorted by id (warp bitonic sort)
//     and appended to their device's FIFO, which is therefore sorted by (ready, id) --
//     dispatch pops the FIFO head (= SPEC's "smallest (ready_time, node id)");
//   * cross-device transfers are appended to their directed channel's FIFO; arrivals on a
//     channel are monotone, so the next arrival is the channel head, and arrival instants
//     (which allocate the receiver's copy) come from at most 64 heads;
//   * at most one op per device finishes per round, so the channels written in a round
//     are disjoint and the finishing ops' out-edges are processed lane-parallel, with the
//     FIFO serialisation of a channel done by a segmented warp prefix sum of transfer times.
// Lanes 0..d-1 own the devices (running op, finish time).  Device time is int32 (the host
// rejects graphs whose total duration + transfer could reach 2^31 ticks).
#include <climits>
#include <cstdlib>

#include "common.cuh"
#include "cost2.cuh"

namespace gdp {
namespace {

struct CostGraph {
  int N;
  long long E;
  const int *out_ptr, *out_idx, *out_src, *in_ptr, *in_idx, *cost, *leader;
  const long long *out_bytes, *mem_bytes;
  int has_coloc;
};

__device__ __forceinline__ int warp_min_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ void smem_add_ll(long long *p, long long v) {
  atomicAdd(reinterpret_cast<unsigned long long *>(p), static_cast<unsigned long long>(v));
}

__global__ void __launch_bounds__(32) k_cost(CostGraph G, TopoArgs T, const uint8_t *__restrict__ Dall, int B,
                                             int *rem_all, int *rcons_all, int2 *fifo_all, int *new_all,
                                             int4 *chq_all, gdp_sim_report *rep, long long *peak_out,
                                             long long *busy_out, double *reward) {
  const int b = blockIdx.x, lane = threadIdx.x;
  const unsigned lt = (1u << lane) - 1u;
  const int N = G.N, d = T.d;
  const uint8_t *D = Dall + (size_t)b * N;
  int *rem = rem_all + (size_t)b * N;
  int *rcons = rcons_all + (size_t)b * N;
  int2 *fifo = fifo_all + (size_t)b * N;
  int *nl = new_all + (size_t)b * 2 * N;      // [0, N): unsorted new list, [N, 2N): sorted
  int4 *chq = chq_all + (size_t)b * (G.E > 0 ? G.E : 1);

  __shared__ long long s_mem[8], s_peak[8];
  __shared__ int s_dhead[8], s_dtail[8];
  __shared__ int s_ccnt[64], s_chead[64], s_ctail[64], s_cfree[64], s_charr[64];
  __shared__ int s_nnew, s_flag;

  if (lane == 0) { s_nnew = 0; s_flag = 0; }
  s_ccnt[lane] = 0;
  s_ccnt[lane + 32] = 0;
  __syncwarp();

  // ---- node pass: validity, static memory, busy, device op counts, counters
  long long lmem[8], lbusy[8];
  int lcnt[8];
#pragma unroll
  for (int k = 0; k < 8; k++) { lmem[k] = 0; lbusy[k] = 0; lcnt[k] = 0; }
  int flag = 0;
  for (int v = lane; v < N; v += 32) {
    int k = D[v];
    if (k >= d) { flag |= 2; continue; }
    if (G.has_coloc && D[G.leader[v]] != k) flag |= 1;
    long long mb = G.mem_bytes[v];
    long long du = (long long)G.cost[v] * T.speed[k];
#pragma unroll
    for (int t = 0; t < 8; t++)
      if (t == k) { lmem[t] += mb; lbusy[t] += du; lcnt[t] += 1; }
    rem[v] = G.in_ptr[v + 1] - G.in_ptr[v];
    rcons[v] = G.out_ptr[v + 1] - G.out_ptr[v];
  }
  flag = __reduce_or_sync(0xffffffffu, flag);
  long long mymem = 0, mybusy = 0;
  int mycnt = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) {
    long long a = warp_sum_ll(lmem[k]), c = warp_sum_ll(lbusy[k]);
    int n = __reduce_add_sync(0xffffffffu, lcnt[k]);
    if (lane == k) { mymem = a; mybusy = c; mycnt = n; }
  }
  gdp_sim_report R;
  R.makespan = 0; R.cross_bytes = 0; R.valid = 0; R.violation = 0;
  for (int i = 0; i < 6; i++) R.pad[i] = 0;
  if (flag & 2) {   // malformed: an entry >= d
    if (lane == 0) {
      R.violation = 3;
      rep[b] = R;
      reward[b] = -10.0;
    }
    if (lane < d) {
      if (peak_out) peak_out[(size_t)b * d + lane] = 0;
      if (busy_out) busy_out[(size_t)b * d + lane] = 0;
    }
    return;
  }
  if (lane < d) {
    s_mem[lane] = mymem;
    s_peak[lane] = mymem;
  }
  // ---- edge pass: channel counts, cross bytes
  long long lcross = 0;
  for (long long e = lane; e < G.E; e += 32) {
    int u = G.out_src[e], w = G.out_idx[e];
    int su = D[u], tw = D[w];
    if (su != tw) {
      atomicAdd(&s_ccnt[su * 8 + tw], 1);
      lcross += G.out_bytes[u];
    }
  }
  long long cross = warp_sum_ll(lcross);
  __syncwarp();
  // device FIFO regions from op counts (exclusive prefix across lanes 0..7)
  {
    int c = lane < d ? mycnt : 0;
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane < 8) { s_dhead[lane] = inc - c; s_dtail[lane] = inc - c; }
  }
  // channel FIFO regions (64 channels, 2 per lane, exclusive prefix in channel order)
  {
    int c0 = s_ccnt[2 * lane], c1 = s_ccnt[2 * lane + 1];
    int pair = c0 + c1, inc = pair;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    int base = inc - pair;
    s_chead[2 * lane] = s_ctail[2 * lane] = base;
    s_chead[2 * lane + 1] = s_ctail[2 * lane + 1] = base + c0;
    s_cfree[2 * lane] = s_cfree[2 * lane + 1] = 0;
    s_charr[2 * lane] = s_charr[2 * lane + 1] = INT_MAX;
  }
  __syncwarp();
  // ---- sources (in-degree 0) are available at t = 0, appended in ascending id
  for (int base = 0; base < N; base += 32) {
    int v = base + lane;
    bool src = v < N && G.in_ptr[v + 1] == G.in_ptr[v];
    int k = src ? D[v] : 0;
    int off = 0, cnt = 0;
    for (int dev = 0; dev < d; dev++) {
      unsigned m = __ballot_sync(0xffffffffu, src && k == dev);
      if (src && k == dev) off = __popc(m & lt);
      if (lane == dev) cnt = __popc(m);
    }
    if (src) fifo[s_dtail[k] + off] = make_int2(v, 0);
    __syncwarp();
    if (lane < d) s_dtail[lane] += cnt;
    __syncwarp();
  }

  // ---- event loop
  int run_op = -1, fin = 0;
  int mk = 0;
  int t = 0;
  bool first = true;
  int dispatched = 0;
  for (;;) {
    if (!first) {
      int cand = INT_MAX;
      if (lane < d && run_op >= 0) cand = fin;
      cand = min(cand, min(s_charr[lane], s_charr[lane + 32]));
      t = warp_min_i(cand);
      if (t == INT_MAX) break;
    }
    first = false;
    for (int round = 0;; round++) {
      if (lane == 0) s_nnew = 0;
      __syncwarp();
      // (1) copy arrivals due now (only the first round can have any)
      if (round == 0) {
#pragma unroll
        for (int h = 0; h < 2; h++) {
          int c = lane + 32 * h;
          int head = s_chead[c], tail = s_ctail[c];
          int arr = s_charr[c];
          while (head < tail && arr <= t) {
            int4 q = chq[head];
            int dst = c & 7;
            smem_add_ll(&s_mem[dst], G.out_bytes[q.z]);
            if (atomicSub(&rem[q.y], 1) == 1) nl[atomicAdd(&s_nnew, 1)] = q.y;
            head++;
            arr = head < tail ? chq[head].x : INT_MAX;
          }
          s_chead[c] = head;
          s_charr[c] = arr;
        }
      }
      __syncwarp();
      // (2) ops finishing now: one per device at most; channels are disjoint per source device
      unsigned fm = __ballot_sync(0xffffffffu, lane < d && run_op >= 0 && fin == t);
      while (fm) {
        const int k = __ffs(fm) - 1;
        fm &= fm - 1;
        const int v = __shfl_sync(0xffffffffu, run_op, k);
        if (lane == k) run_op = -1;
        // frees: the copies this op held, producers whose last consumer this was, sink output
        const int ib = G.in_ptr[v], ie = G.in_ptr[v + 1];
        for (int e = ib + lane; e < ie; e += 32) {
          int u = G.in_idx[e];
          int du = D[u];
          long long ob = G.out_bytes[u];
          if (du != k) smem_add_ll(&s_mem[k], -ob);
          if (atomicSub(&rcons[u], 1) == 1) smem_add_ll(&s_mem[du], -ob);
        }
        const int ob0 = G.out_ptr[v], oe = G.out_ptr[v + 1];
        const long long obv = G.out_bytes[v];
        if (ob0 == oe && lane == 0) smem_add_ll(&s_mem[k], -obv);
        for (int base = ob0; base < oe; base += 32) {
          const int e = base + lane;
          const bool valid = e < oe;
          const int w = valid ? G.out_idx[e] : 0;
          const int tw = valid ? (int)D[w] : 0;
          const bool cross = valid && tw != k;
          int xfer = 0;
          if (cross) {
            long long bw = T.bpt[k * 8 + tw];
            xfer = (int)((obv + bw - 1) / bw) + T.lat[k * 8 + tw];
          }
          const int c = k * 8 + tw;
          const int base_t = cross ? max(t, s_cfree[c]) : t;
          int pre = 0, mytot = 0;
          for (int dst = 0; dst < d; dst++) {
            int val = (cross && tw == dst) ? xfer : 0;
            int inc = val;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              int y = __shfl_up_sync(0xffffffffu, inc, o);
              if (lane >= o) inc += y;
            }
            if (cross && tw == dst) pre = inc;
            int tot = __shfl_sync(0xffffffffu, inc, 31);
            if (lane == dst) mytot = tot;
          }
          const int arr = cross ? base_t + pre : t;
          const bool enq = cross && arr > t;
          int rank = 0, ecnt = 0;
          for (int dst = 0; dst < d; dst++) {
            unsigned m = __ballot_sync(0xffffffffu, enq && tw == dst);
            if (enq && tw == dst) rank = __popc(m & lt);
            if (lane == dst) ecnt = __popc(m);
          }
          __syncwarp();
          if (valid) {
            if (!enq) {
              if (cross) smem_add_ll(&s_mem[tw], obv);
              if (atomicSub(&rem[w], 1) == 1) nl[atomicAdd(&s_nnew, 1)] = w;
            } else {
              const int pos = s_ctail[c] + rank;
              chq[pos] = make_int4(arr, w, v, 0);
              if (rank == 0 && s_chead[c] == s_ctail[c]) s_charr[c] = arr;
            }
          }
          __syncwarp();
          if (lane < d) {
            const int cc = k * 8 + lane;
            if (mytot > 0) s_cfree[cc] = max(t, s_cfree[cc]) + mytot;
            s_ctail[cc] += ecnt;
          }
          __syncwarp();
        }
      }
      __syncwarp();
      // (3) ops that became available now (ready = t): sort by id, append to device FIFOs
      const int n = s_nnew;
      if (n > 0) {
        const int *sorted;
        if (n <= 32) {
          int x = lane < n ? nl[lane] : INT_MAX;
#pragma unroll
          for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
            for (int j = kk >> 1; j > 0; j >>= 1) {
              int o = __shfl_xor_sync(0xffffffffu, x, j);
              bool up = (lane & kk) == 0, lower = (lane & j) == 0;
              x = (lower == up) ? min(x, o) : max(x, o);
            }
          }
          if (lane < n) nl[N + lane] = x;
        } else {
          for (int i = lane; i < n; i += 32) {
            int x = nl[i], r = 0;
            for (int j = 0; j < n; j++) r += nl[j] < x;
            nl[N + r] = x;
          }
        }
        __syncwarp();
        sorted = nl + N;
        int gotcnt = 0;
        for (int base = 0; base < n; base += 32) {
          const int i = base + lane;
          const bool valid = i < n;
          const int v = valid ? sorted[i] : 0;
          const int k = valid ? (int)D[v] : 0;
          int off = 0, cnt = 0;
          for (int dev = 0; dev < d; dev++) {
            unsigned m = __ballot_sync(0xffffffffu, valid && k == dev);
            if (valid && k == dev) off = __popc(m & lt);
            if (lane == dev) cnt = __popc(m);
          }
          if (valid) fifo[s_dtail[k] + off] = make_int2(v, t);
          __syncwarp();
          if (lane < d) { s_dtail[lane] += cnt; gotcnt += cnt; }
          __syncwarp();
        }
        // zero-duration corner case: entries appended in an earlier round of this same
        // instant share ready time t; keep the FIFO sorted by (ready, id)
        if (round > 0 && lane < d && gotcnt > 0) {
          int head = s_dhead[lane], tail = s_dtail[lane];
          int s0 = tail;
          while (s0 > head && fifo[s0 - 1].y == t) s0--;
          for (int i = s0 + 1; i < tail; i++) {
            int2 key = fifo[i];
            int j = i - 1;
            while (j >= s0 && fifo[j].x > key.x) { fifo[j + 1] = fifo[j]; j--; }
            fifo[j + 1] = key;
          }
        }
        __syncwarp();
      }
      // (4) dispatch: each idle device starts its FIFO head
      bool zero = false;
      if (lane < d && run_op < 0) {
        int head = s_dhead[lane];
        if (head < s_dtail[lane]) {
          int v = fifo[head].x;
          s_dhead[lane] = head + 1;
          int dur = G.cost[v] * T.speed[lane];
          run_op = v;
          fin = t + dur;
          mk = max(mk, fin);
          smem_add_ll(&s_mem[lane], G.out_bytes[v]);
          zero = dur == 0;
          dispatched++;
        }
      }
      __syncwarp();
      // (5) peak after all changes of this round
      if (lane < d) s_peak[lane] = max(s_peak[lane], s_mem[lane]);
      if (!__any_sync(0xffffffffu, zero)) break;
    }
  }
  mk = -warp_min_i(-mk);
  dispatched = __reduce_add_sync(0xffffffffu, dispatched);
  __syncwarp();
  int oom = 0;
  if (lane < d) {
    oom = s_peak[lane] > T.cap[lane];
    if (peak_out) peak_out[(size_t)b * d + lane] = s_peak[lane];
    if (busy_out) busy_out[(size_t)b * d + lane] = mybusy;
  }
  oom = __reduce_or_sync(0xffffffffu, oom);
  if (lane == 0) {
    R.makespan = mk;
    R.cross_bytes = cross;
    R.violation = (flag & 1) ? 1 : (oom ? 2 : 0);
    if (dispatched != N) R.violation = 3;   // cannot happen for a validated DAG
    R.valid = R.violation == 0;
    rep[b] = R;
    reward[b] = R.valid ? -__dsqrt_rn(__ddiv_rn((double)mk, 1e6)) : -10.0;
  }
}

// A_b = r_b - (running sum before b) / (running count before b), the running state in the global
// trial order (reading R22).  The running sum is one sequential chain of fp64 additions
// (the oracle's order, bit-exact); only the chain runs on lane 0 -- the rewards are staged into
// shared memory by the whole warp and the divisions run lane-parallel -- in chunks of AC.
constexpr int AC = 2048;
__global__ void __launch_bounds__(32) k_advantage(const double *__restrict__ r, int B, double *sum, long long *cnt,
                                                  double *__restrict__ adv) {
  __shared__ double sr[AC], sp[AC];
  const int lane = threadIdx.x;
  double s = *sum;
  const long long c0 = *cnt;
  for (int b0 = 0; b0 < B; b0 += AC) {
    const int n = min(AC, B - b0);
    for (int i = lane; i < n; i += 32) sr[i] = r[b0 + i];
    __syncwarp();
    if (lane == 0) {
      for (int i = 0; i < n; i++) {
        sp[i] = s;
        s = __dadd_rn(s, sr[i]);
      }
    }
    s = __shfl_sync(0xffffffffu, s, 0);
    __syncwarp();
    for (int i = lane; i < n; i += 32) {
      const long long c = c0 + b0 + i;
      adv[b0 + i] = (c == 0) ? 0.0 : __dsub_rn(sr[i], __ddiv_rn(sp[i], (double)c));
    }
    __syncwarp();
  }
  if (lane == 0) {
    *sum = s;
    *cnt = c0 + B;
  }
}

}  // namespace

static TopoArgs topo_args(const gdp_topo_s *t) {
  TopoArgs T;
  T.d = t->d;
  for (int i = 0; i < 8; i++) { T.cap[i] = t->cap[i]; T.speed[i] = t->speed[i]; }
  for (int i = 0; i < 64; i++) {
    T.bpt[i] = t->bpt[i];
    T.lat[i] = t->lat[i];
    T.inv_bpt[i] = t->bpt[i] > 0 ? 1.0 / (double)t->bpt[i] : 0.0;
  }
  return T;
}

static Cost5Graph cost5_graph(const gdp_graph_s *g) {
  Cost5Graph C;
  C.N = g->N; C.E = g->E; C.ok = g->c5_ok ? 1 : 0;
  C.slots = static_cast<const Slot5 *>(g->slots5); C.srcq = static_cast<const Slot5 *>(g->srcq5);
  C.ebytes = static_cast<const long long *>(g->ebytes5);
  C.irec = static_cast<const IRec *>(g->irec);
  C.in_ptr = g->in_ptr;
  C.out_idx = g->out_idx; C.out_src = g->out_src; C.cost = g->cost; C.leader = g->leader;
  C.outdeg = g->outdeg5; C.gbig0 = g->gbig5; C.bigb0 = g->bigb5;
  C.out_bytes = g->out_bytes; C.mem_bytes = g->mem_bytes;
  C.nsrc = g->nsrc5; C.nbigb = g->nbigb5; C.ngbig = g->ngbig5; C.nflagw = g->nflagw5;
  C.bytes32 = g->bytes32_5;
  C.has_coloc = g->has_coloc ? 1 : 0;
  return C;
}

// 5: k_cost5 (cost5.cu) whenever every duration and every transfer takes >= 1 tick and its
// state fits in shared memory; 3: k_cost3 (cost2.cu, zero-duration ops / zero-tick transfers);
// 1: k_cost below (per-placement state larger than shared memory)
int cost_kernel_choice(const gdp_graph_s *g, const gdp_topo_s *t, int force) {
  const TopoArgs T = topo_args(t);
  const bool ok5 = cost5_eligible(T, cost5_graph(g), g->min_cost, g->min_edge_bytes);
  const bool ok3 = cost2_smem_bytes(g->N) <= 227 * 1024;
  if (force == 5 && ok5) return 5;
  if (force == 3 && ok3) return 3;
  if (force == 1) return 1;
  return ok5 ? 5 : (ok3 ? 3 : 1);
}

int cost_wave(const gdp_graph_s *g, const gdp_topo_s *t) {
  return cost_kernel_choice(g, t, 0) == 5 ? cost5_wave(cost5_graph(g)) : 0;
}

gdp_status launch_cost(const gdp_graph_s *g, const gdp_topo_s *t, const uint8_t *D, int B, gdp_sim_report *rep,
                       long long *peak, long long *busy, double *reward, const WS &w, int force, cudaStream_t s) {
  const TopoArgs T = topo_args(t);
  const int k = cost_kernel_choice(g, t, force);
  if (k == 5 && launch_cost5(cost5_graph(g), T, g->min_cost, g->min_edge_bytes, D, B, w.c_scratch, w.c_per_place, rep,
                             peak, busy, reward, s)) {
    GDP_LAUNCH_CHECK("k_cost5");
    return GDP_OK;
  }
  if (k == 3) {
    Cost2Graph C;
    C.N = g->N; C.E = g->E;
    C.nrec = static_cast<const NRec *>(g->nrec); C.erec = static_cast<const NRec *>(g->erec);
    C.irec = static_cast<const IRec *>(g->irec);
    C.cnt0 = g->cnt0; C.bigid = g->bigid; C.big_in = g->big_in; C.big_out = g->big_out; C.nbig = g->nbig;
    C.out_idx = g->out_idx; C.out_src = g->out_src; C.in_ptr = g->in_ptr; C.cost = g->cost; C.leader = g->leader;
    C.out_bytes = g->out_bytes; C.mem_bytes = g->mem_bytes; C.has_coloc = g->has_coloc ? 1 : 0;
    if (launch_cost2(C, T, D, B, w.c_scratch, w.c_per_place, rep, peak, busy, reward, s)) {
      GDP_LAUNCH_CHECK("k_cost3");
      return GDP_OK;
    }
  }
  CostGraph G;
  G.N = g->N;
  G.E = g->E;
  G.out_ptr = g->out_ptr; G.out_idx = g->out_idx; G.out_src = g->out_src;
  G.in_ptr = g->in_ptr; G.in_idx = g->in_idx;
  G.cost = g->cost; G.leader = g->leader;
  G.out_bytes = g->out_bytes; G.mem_bytes = g->mem_bytes;
  G.has_coloc = g->has_coloc ? 1 : 0;
  note_launch("k_cost", s);
  k_cost<<<B, 32, 0, s>>>(G, T, D, B, w.c_rem, w.c_rcons, w.c_fifo, w.c_new, w.c_chq, rep, peak, busy, reward);
  GDP_LAUNCH_CHECK("k_cost");
  return GDP_OK;
}

void launch_advantage(const double *r, int B, double *sum, long long *cnt, double *adv, cudaStream_t s) {
  note_launch("k_advantage", s);
  k_advantage<<<1, 32, 0, s>>>(r, B, sum, cnt, adv);
}

}  // namespace gdp
