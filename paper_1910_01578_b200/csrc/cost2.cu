// Cost model, k_cost3: the warp-cooperative instant-by-instant kernel that gdp_cost runs when
// k_cost5 (cost5.cu) does not apply -- zero-duration ops or zero-tick transfers, which need
// same-instant rounds (cost.cu's k_cost takes graphs whose state does not fit in shared
// memory).  Same event semantics as the oracle (DESIGN.md §7 "Cost model"):
//
//  * lane k < d OWNS device k: its running op and finish time (registers), its FIFO of
//    available ops, and its outgoing channels (k -> t): channel state is only ever touched by
//    lane k, so enqueue (at lane k's finishes) and dequeue (arrivals) need no atomics and no
//    warp-wide coordination;
//  * an op keeps a counter of inputs not yet ARRIVED; it becomes available at the instant the
//    counter reaches 0 (its ready time), so no per-op ready time and no priority queue exist:
//    ops made available at one instant are sorted by id and appended to their device FIFO,
//    which is thus sorted by (ready, id) -- dispatch pops its head (SPEC.md:278 (c));
//  * per op one byte of counters in smem (low nibble: inputs not yet arrived, high nibble:
//    consumers not yet finished; degree >= 15 -> global counters), 4-bit device ids in smem;
//  * FIFOs and channel queues keep their first K entries (full records) in smem; the rest
//    overflow to global and are pulled back with cp.async as the head advances;
//  * the successor / producer records an op's finish needs are staged into smem by
//    cp.async while the op waits at its FIFO head (double-buffered per device).
// One CTA (one warp) per placement.
#include <climits>
#include <cstdlib>

#include "common.cuh"
#include "cost2.cuh"
#include "cost_util.cuh"

namespace gdp {
namespace {
using namespace cu;

constexpr int SO = 8;     // staged out-edge records per slot
constexpr int SI = 8;     // staged in-edge records per slot
constexpr int KF = 4;     // FIFO entries kept in smem per device
constexpr int KC = 4;     // channel entries kept in smem per channel
constexpr int NINC = 32;  // per-device list of ops made available this round (overflow -> global)

struct Smem {
  NRec st_out[8][2][SO];
  IRec st_in[8][2][SI];
  Ent fc[8][KF];
  Ent cc[8][8][KC];
  NRec inc[8][NINC];
  NRec sreq[8];
  NRec run[8];                    // k_cost3: record of the op running on each device
  int run_slot[8];                // k_cost3: its staging slot
  unsigned mw[3][8];              // k_cost3: resident bytes per device, 16 + 16 + 32 bits
  unsigned memlo[8], memhi[8];   // per-device resident bytes as two 32-bit words (native atomics)
  long long peak[8];
  int ch_head[8][8], ch_tail[8][8], ch_free[8][8], ch_arr[8][8], ch_off[8][8];
  int ccnt[64];
  int inc_n[8], doff[8], sreq_slot[8];
};

// an op became available now: append to device dev's incoming list for this round
__device__ __forceinline__ void push_inc(Smem &S, NRec *ov, int dev, const NRec &r) {
  const int i = atomicAdd(&S.inc_n[dev], 1);
  if (i < NINC) copy_rec(&S.inc[dev][i], &r);
  else copy_rec(ov + S.doff[dev] + i, &r);
}

__device__ __forceinline__ gdp_sim_report empty_report() {
  gdp_sim_report R;
  R.makespan = 0; R.cross_bytes = 0; R.valid = 0; R.violation = 0;
  for (int i = 0; i < 6; i++) R.pad[i] = 0;
  return R;
}

// per-placement views of shared and global scratch
struct Ctx {
  int N, d, b, lane, cwords, dwords;
  unsigned lt;
  unsigned *cnt, *Dn;
  const uint8_t *D;
  Ent *fifo, *chq;
  NRec *ov;
  int *bigc;
};
__device__ __forceinline__ Ctx make_ctx(const Cost2Graph &G, const TopoArgs &T, const uint8_t *Dall,
                                        unsigned char *scratch, size_t per_place, unsigned char *smem_raw) {
  Ctx C;
  C.N = G.N; C.d = T.d; C.b = blockIdx.x; C.lane = threadIdx.x;
  C.lt = (1u << C.lane) - 1u;
  C.cnt = reinterpret_cast<unsigned *>(smem_raw + sizeof(Smem));
  C.cwords = (C.N + 3) >> 2;
  C.Dn = C.cnt + C.cwords;
  C.dwords = (C.N + 7) >> 3;
  C.D = Dall + (size_t)C.b * C.N;
  unsigned char *base = scratch + (size_t)C.b * per_place;
  C.fifo = reinterpret_cast<Ent *>(base);
  C.chq = C.fifo + C.N;
  C.ov = reinterpret_cast<NRec *>(C.chq + (G.E > 0 ? G.E : 1));
  C.bigc = reinterpret_cast<int *>(C.ov + C.N);
  return C;
}

// Warp-wide prologue shared by both kernels: counters and packed device ids into shared
// memory, static memory / busy / op counts per device, cross bytes, co-location check,
// per-device and per-channel overflow regions, sources appended to their FIFO at t = 0.
// Returns false (outputs written) when the placement holds an entry >= d.
__device__ __forceinline__ bool prologue(const Cost2Graph &G, const TopoArgs &T, Smem &S, const Ctx &C,
                                         gdp_sim_report *rep, long long *peak_out, long long *busy_out,
                                         double *reward, int &flag, long long &mymem, long long &mybusy,
                                         long long &cross, int &ftail) {
  const int N = C.N, d = C.d, b = C.b, lane = C.lane, cwords = C.cwords, dwords = C.dwords;
  const unsigned lt = C.lt;
  unsigned *cnt = C.cnt, *Dn = C.Dn;
  const uint8_t *D = C.D;
  Ent *fifo = C.fifo;
  int *bigc = C.bigc;
  // ---------------------------------------------------------------- prologue (warp-wide)
  for (int i = lane; i < cwords; i += 32) cnt[i] = G.cnt0[i];
  long long lmem[8], lbusy[8];
  int lcnt[8];
  flag = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) { lmem[k] = 0; lbusy[k] = 0; lcnt[k] = 0; }
  for (int p = lane; p < dwords; p += 32) {
    unsigned packed = 0;
    for (int j = 0; j < 8; j++) {
      const int v = 8 * p + j;
      if (v >= N) break;
      int k = D[v];
      if (k >= d) { flag |= 2; k = 0; }
      packed |= (unsigned)k << (4 * j);
      const long long mb = G.mem_bytes[v];
      const long long du = (long long)G.cost[v] * T.speed[k];
#pragma unroll
      for (int q = 0; q < 8; q++)
        if (q == k) { lmem[q] += mb; lbusy[q] += du; lcnt[q] += 1; }
      if (G.has_coloc && D[G.leader[v]] != D[v]) flag |= 1;
    }
    Dn[p] = packed;
  }
  for (int j = lane; j < G.nbig; j += 32) { bigc[j] = G.big_in[j]; bigc[G.nbig + j] = G.big_out[j]; }
  S.ccnt[lane] = 0;
  S.ccnt[lane + 32] = 0;
  if (lane < 8) S.inc_n[lane] = 0;
  flag = __reduce_or_sync(0xffffffffu, flag);
  mymem = 0; mybusy = 0;
  int mycnt = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) {
    long long a = warp_sum_ll(lmem[k]), c = warp_sum_ll(lbusy[k]);
    int n = __reduce_add_sync(0xffffffffu, lcnt[k]);
    if (lane == k) { mymem = a; mybusy = c; mycnt = n; }
  }
  if (flag & 2) {   // malformed: an entry >= d
    if (lane == 0) {
      gdp_sim_report R = empty_report();
      R.violation = 3;
      rep[b] = R;
      reward[b] = -10.0;
    }
    if (lane < d) {
      if (peak_out) peak_out[(size_t)b * d + lane] = 0;
      if (busy_out) busy_out[(size_t)b * d + lane] = 0;
    }
    return false;
  }
  if (lane < 8) {
    S.memlo[lane] = (unsigned)((unsigned long long)mymem & 0xffffffffull);
    S.memhi[lane] = (unsigned)((unsigned long long)mymem >> 32);
    S.peak[lane] = mymem;
  }
  __syncwarp();
  long long lcross = 0;
  for (long long e = lane; e < G.E; e += 32) {
    const int u = G.out_src[e], w = G.out_idx[e];
    const int su = dev_of(Dn, u), tw = dev_of(Dn, w);
    if (su != tw) {
      atomicAdd(&S.ccnt[su * 8 + tw], 1);
      lcross += G.out_bytes[u];
    }
  }
  cross = warp_sum_ll(lcross);
  __syncwarp();
  {  // device regions (FIFO overflow, incoming overflow) from op counts
    int c = lane < d ? mycnt : 0, inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane < 8) S.doff[lane] = inc - c;
  }
  {  // channel regions, channels 2*lane and 2*lane+1 in (source, target) order
    const int c0 = S.ccnt[2 * lane], c1 = S.ccnt[2 * lane + 1];
    const int pair = c0 + c1;
    int inc = pair;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    const int c = 2 * lane;
    S.ch_off[c >> 3][c & 7] = inc - pair;
    S.ch_off[(c + 1) >> 3][(c + 1) & 7] = inc - pair + c0;
  }
  if (lane < 8) {
#pragma unroll
    for (int q = 0; q < 8; q++) {
      S.ch_head[lane][q] = 0; S.ch_tail[lane][q] = 0; S.ch_free[lane][q] = 0; S.ch_arr[lane][q] = INF;
    }
  }
  __syncwarp();
  // sources are available at t = 0: appended to their FIFO in ascending id
  ftail = 0;   // lane k: FIFO tail (relative to the device region)
  for (int v0 = 0; v0 < N; v0 += 32) {
    const int v = v0 + lane;
    const bool src = v < N && G.in_ptr[v + 1] == G.in_ptr[v];
    if (!__any_sync(0xffffffffu, src)) continue;
    const int k = src ? dev_of(Dn, v) : 0;
    int off = 0, cntk = 0;
    for (int dev = 0; dev < d; dev++) {
      const unsigned m = __ballot_sync(0xffffffffu, src && k == dev);
      if (src && k == dev) off = __popc(m & lt);
      if (lane == dev) cntk = __popc(m);
    }
    const int tail_k = __shfl_sync(0xffffffffu, ftail, k & 7);
    if (src) {
      NRec r;
      load_rec(r, G.nrec + v);
      const int pos = tail_k + off;
      if (pos < KF) store_ent(&S.fc[k][pos], r, 0, 0);
      else store_ent(fifo + S.doff[k] + pos, r, 0, 0);
    }
    ftail += cntk;
    __syncwarp();
  }

  return true;
}

// ------------------------------------------------------------------------------------------
// k_cost3: the work of one instant spread over the whole warp:
//  * channel (k -> q) is owned by lane (8k + q) / 2, which caches its head arrival in a
//    register and pops its arrivals (all owners in parallel);
//  * a finishing op's in-edges and out-edges are handled one per lane; out-edges into the
//    same channel are ranked with __match_any_sync, so their FIFO arrival times
//    max(t, free) + (rank + 1) * xfer are computed in parallel (every transfer of one op on
//    one channel has the same size, so the serial recurrence has this closed form);
//  * per-device resident bytes are three 32-bit words (bits 0-15, 16-31, 32-63) updated with
//    fire-and-forget shared reductions; the owner lane carries and samples them once per round;
//  * lane q < d still owns device q: FIFO append, dispatch, staging of its records, peak.
constexpr int MEM_NORM = 1024;   // adds per lane between carries (32 lanes x 1024 x 2^16 < 2^32)

__device__ __forceinline__ void mem_carry_all(Smem &S) {   // atomic-safe carry of every device
#pragma unroll
  for (int q = 0; q < 8; q++) {
    const unsigned o0 = atomicAnd(&S.mw[0][q], 0xffffu);
    atomicAdd(&S.mw[1][q], o0 >> 16);
    const unsigned o1 = atomicAnd(&S.mw[1][q], 0xffffu);
    atomicAdd(&S.mw[2][q], o1 >> 16);
  }
}
__device__ __forceinline__ void add_mem3(Smem &S, int dev, long long v, int &nadd) {
  atomicAdd(&S.mw[0][dev], (unsigned)(v & 0xffff));
  atomicAdd(&S.mw[1][dev], (unsigned)((v >> 16) & 0xffff));
  atomicAdd(&S.mw[2][dev], (unsigned)(int)(v >> 32));
  if (++nadd >= MEM_NORM) { mem_carry_all(S); nadd = 0; }
}
// owner of device q, no concurrent adders: value, normalised in place
__device__ __forceinline__ long long mem_sample(Smem &S, int q) {
  const unsigned w0 = S.mw[0][q], w1 = S.mw[1][q], w2 = S.mw[2][q];
  const long long v = ((long long)(int)w2 << 32) + ((long long)w1 << 16) + (long long)w0;
  S.mw[0][q] = (unsigned)(v & 0xffff);
  S.mw[1][q] = (unsigned)((v >> 16) & 0xffff);
  S.mw[2][q] = (unsigned)(int)(v >> 32);
  return v;
}
// input counter of the op a record describes (cost bit 31 = global counters)
__device__ __forceinline__ bool dec_in(unsigned *cnt, const NRec &r, int *bigc, const int *bigid) {
  if (r.cost < 0) return atomicSub(&bigc[bigid[r.id]], 1) == 1;
  const int sh = (r.id & 3) * 8;
  return ((atomicSub(&cnt[r.id >> 2], 1u << sh) >> sh) & 15u) == 1u;
}
// consumer counter of an in-edge's producer (IRec.pad = its global counter index, or -1)
__device__ __forceinline__ bool dec_out(unsigned *cnt, const IRec &ir, int *bigc, int nbig) {
  if (ir.pad >= 0) return atomicSub(&bigc[ir.pad + nbig], 1) == 1;
  const int sh = (ir.u & 3) * 8 + 4;
  return ((atomicSub(&cnt[ir.u >> 2], 1u << sh) >> sh) & 15u) == 1u;
}
// a device lane stages the out-/in-edge records of op r into its slot sl
__device__ __forceinline__ void stage_records(Smem &S, const Cost2Graph &G, int k, int sl, const NRec &r) {
  const int no = min(r.oe - r.ob, SO), ni = min(r.ie - r.ib, SI);
  const int4 *eo = reinterpret_cast<const int4 *>(G.erec + r.ob);
  int4 *so = reinterpret_cast<int4 *>(&S.st_out[k][sl][0]);
  for (int j = 0; j < 2 * no; j++) cp16(so + j, eo + j);
  for (int j = 0; j < ni; j++) cp16(&S.st_in[k][sl][j], G.irec + r.ib + j);
}

__device__ __forceinline__ int pop_channel3(Smem &S, const Ctx &C, const Cost2Graph &G, int c, int a, int t,
                                            int &head, int off, int &nadd) {
  const int q = c & 7;
  Ent *ring = &S.cc[0][0][0] + c * KC;
  const int tail = (&S.ch_tail[0][0])[c];
  int popped = 0;
  while (a <= t) {
    if (popped) { cp_commit(); cp_wait0(); }   // the refill issued by the previous pop
    Ent &e = ring[head % KC];
    add_mem3(S, q, e.bytes, nadd);
    if (dec_in(C.cnt, e.r, C.bigc, G.bigid)) push_inc(S, C.ov, q, e.r);
    if (head + KC < tail) cp_ent(&e, C.chq + off + head + KC);
    head++;
    popped = 1;
    a = head < tail ? ring[head % KC].t : INF;
  }
  (&S.ch_head[0][0])[c] = head;
  (&S.ch_arr[0][0])[c] = a;
  return a;
}

__device__ __forceinline__ void finish_op3(Smem &S, const Ctx &C, const Cost2Graph &G, const TopoArgs &T,
                                           int k, int t, int &nadd) {
  const int lane = C.lane;
  NRec r;
  load_rec(r, &S.run[k]);
  const int sl = S.run_slot[k];
  const int nin = r.ie - r.ib, nout = r.oe - r.ob;
  // frees: copies this op held, producers whose last consumer it was, sink output
  for (int j = lane; j < nin; j += 32) {
    IRec ir;
    if (j < SI) ir = S.st_in[k][sl][j];
    else ir = G.irec[r.ib + j];
    const int du = dev_of(C.Dn, ir.u);
    if (du != k) add_mem3(S, k, -ir.bytes, nadd);
    if (dec_out(C.cnt, ir, C.bigc, G.nbig)) add_mem3(S, du, -ir.bytes, nadd);
  }
  if (nout == 0 && lane == 0) add_mem3(S, k, -r.bytes, nadd);
  int *chf = &S.ch_free[0][0], *cht = &S.ch_tail[0][0], *chh = &S.ch_head[0][0], *cha = &S.ch_arr[0][0];
  const int *cho = &S.ch_off[0][0];
  for (int j0 = 0; j0 < nout; j0 += 32) {
    const int j = j0 + lane;
    const bool v = j < nout;
    NRec wr;
    int tw = -1;
    if (v) {
      if (j < SO) wr = S.st_out[k][sl][j];
      else load_rec(wr, G.erec + r.ob + j);
      tw = dev_of(C.Dn, wr.id);
    }
    const bool cross = v && tw != k;
    if (v && !cross && dec_in(C.cnt, wr, C.bigc, G.bigid)) push_inc(S, C.ov, k, wr);
    if (__any_sync(0xffffffffu, cross)) {
      const unsigned grp = __match_any_sync(0xffffffffu, cross ? tw : -1);
      if (cross) {
        const int rank = __popc(grp & C.lt), n = __popc(grp);
        const int c = k * 8 + tw;
        const int f = chf[c];
        const int x = xfer_time3(r.bytes, c, T);
        const int base = max(t, f);
        const int arr = base + (rank + 1) * x;
        if (arr == t) {   // zero-time transfers (x = 0, channel free): the copies land now
          add_mem3(S, tw, r.bytes, nadd);
          if (dec_in(C.cnt, wr, C.bigc, G.bigid)) push_inc(S, C.ov, tw, wr);
          if (rank == 0) chf[c] = t;
        } else {
          const int head = chh[c], tail = cht[c], pos = tail + rank;
          __syncwarp(grp);   // every rank has read the channel state before rank 0 moves it
          if (pos < head + KC) store_ent(&S.cc[0][0][0] + c * KC + pos % KC, wr, arr, r.bytes);
          else store_ent(C.chq + cho[c] + pos, wr, arr, r.bytes);
          if (rank == 0) {
            chf[c] = base + n * x;
            cht[c] = tail + n;
            if (tail == head) cha[c] = base + x;
          }
        }
      }
      if (j0 + 32 < nout) __syncwarp();   // channel state of this chunk before the next one
    }
  }
}

__global__ void __launch_bounds__(32) k_cost3(Cost2Graph G, TopoArgs T, const uint8_t *__restrict__ Dall,
                                              unsigned char *scratch, size_t per_place, gdp_sim_report *rep,
                                              long long *peak_out, long long *busy_out, double *reward, int dbg) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem &S = *reinterpret_cast<Smem *>(smem_raw);
  const Ctx C = make_ctx(G, T, Dall, scratch, per_place, smem_raw);
  const int N = C.N, d = C.d, b = C.b, lane = C.lane;
  Ent *fifo = C.fifo;
  NRec *ov = C.ov;
  int flag, ftail;
  long long mymem, mybusy, cross;
  if (!prologue(G, T, S, C, rep, peak_out, busy_out, reward, flag, mymem, mybusy, cross, ftail)) return;
  if (dbg == 1) return;
  if (lane < 8) {
    S.mw[0][lane] = (unsigned)(mymem & 0xffff);
    S.mw[1][lane] = (unsigned)((mymem >> 16) & 0xffff);
    S.mw[2][lane] = (unsigned)(int)(mymem >> 32);
  }
  __syncwarp();
  int fhead = 0;
  const bool dl = lane < d;
  const int c0 = 2 * lane, c1 = 2 * lane + 1;   // my channels (k = c / 8 -> q = c % 8)
  int ca0 = INF, ca1 = INF;                       // their head arrivals (channels start empty)
  int hd0 = 0, hd1 = 0;                           // their heads
  const int of0 = (&S.ch_off[0][0])[c0], of1 = (&S.ch_off[0][0])[c1];
  int fin = 0, running = 0, mk = 0, dispatched = 0, nadd = 0;
  int cur = 0, cur_inst = -2, nxt_id = -1, nxt_inst = -2;
  long long pk = mymem;
  int t = 0, n_inst = 0, n_round = 0, n_need = 0;
  long long tacc[6] = {0, 0, 0, 0, 0, 0}, tp = clock64();   // dbg == 3: cycles per phase
#define PH(i) if (dbg == 3) { const long long tn = clock64(); tacc[i] += tn - tp; tp = tn; }
  for (int inst = 0;; inst++) {
    if (inst > 0) {
      const int cand = min(dl && running ? fin : INF, min(ca0, ca1));
      t = __reduce_min_sync(0xffffffffu, cand);
      if (t == INF) break;
    }
    PH(0)
    {  // records staged at the previous instant may still be in flight
      const bool need = dl && running && fin == t && cur_inst == inst - 1;
      if (__any_sync(0xffffffffu, need)) { cp_wait0(); n_need++; } else cp_wait1();
    }
    n_inst++;
    for (int round = 0;; round++) {
      n_round++;
      if (round > 0) cp_wait0();
      __syncwarp();
      PH(1)
      // (1) copy arrivals due now, every channel owner in parallel (first round only)
      if (round == 0) {
        if (ca0 <= t) ca0 = pop_channel3(S, C, G, c0, ca0, t, hd0, of0, nadd);
        if (ca1 <= t) ca1 = pop_channel3(S, C, G, c1, ca1, t, hd1, of1, nadd);
        __syncwarp();
      }
      PH(2)
      // (2) ops finishing now, each handled by the whole warp
      const bool fmine = dl && running && fin == t;
      unsigned fm = __ballot_sync(0xffffffffu, fmine);
      if (fmine) running = 0;
      while (fm) {
        const int k = __ffs(fm) - 1;
        fm &= fm - 1;
        finish_op3(S, C, G, T, k, t, nadd);
      }
      __syncwarp();
      PH(3)
      ca0 = (&S.ch_arr[0][0])[c0];
      ca1 = (&S.ch_arr[0][0])[c1];
      bool zero = false;
      if (dl) {
        // (3) ops made available now (ready = t) join my FIFO in id order
        const int n = S.inc_n[lane];
        if (n > 0) {
          NRec *L = &S.inc[lane][0];
          NRec *O = ov + S.doff[lane];
          for (int i = 1; i < n; i++) {   // insertion sort by id (n is small except after wide fan-outs)
            NRec key;
            load_rec(key, i < NINC ? &L[i] : &O[i]);
            int j = i - 1;
            while (j >= 0) {
              NRec *pj = j < NINC ? &L[j] : &O[j];
              if (pj->id <= key.id) break;
              copy_rec(j + 1 < NINC ? &L[j + 1] : &O[j + 1], pj);
              j--;
            }
            copy_rec(j + 1 < NINC ? &L[j + 1] : &O[j + 1], &key);
          }
          Ent *F = fifo + S.doff[lane];
          if (round > 0) {
            // zero-duration corner case: entries appended earlier in this instant share ready
            // time t and must stay merged by id with the new ones (rare path, done in global)
            for (int i = fhead; i < min(ftail, fhead + KF); i++) F[i] = S.fc[lane][i % KF];
            int tail = ftail;
            for (int i = 0; i < n; i++) store_ent(&F[tail++], i < NINC ? L[i] : O[i], t, 0);
            int s0 = ftail;
            while (s0 > fhead && F[s0 - 1].t == t) s0--;
            for (int i = s0 + 1; i < tail; i++) {
              Ent key = F[i];
              int j = i - 1;
              while (j >= s0 && F[j].r.id > key.r.id) { F[j + 1] = F[j]; j--; }
              F[j + 1] = key;
            }
            for (int i = fhead; i < min(tail, fhead + KF); i++) S.fc[lane][i % KF] = F[i];
            ftail = tail;
            nxt_id = -1;
          } else {
            for (int i = 0; i < n; i++) {
              const NRec &r = i < NINC ? L[i] : O[i];
              if (ftail < fhead + KF) store_ent(&S.fc[lane][ftail % KF], r, t, 0);
              else store_ent(F + ftail, r, t, 0);
              ftail++;
            }
          }
          S.inc_n[lane] = 0;
        }
        // (4) dispatch my FIFO head if idle
        bool staged_now = false;
        if (!running && fhead < ftail) {
          Ent &e = S.fc[lane][fhead % KF];
          NRec run;
          load_rec(run, &e.r);
          const int dur = (run.cost & 0x7fffffff) * T.speed[lane];
          running = 1;
          fin = t + dur;
          mk = max(mk, fin);
          add_mem3(S, lane, run.bytes, nadd);
          zero = dur == 0;
          dispatched++;
          cur ^= 1;
          copy_rec(&S.run[lane], &run);
          S.run_slot[lane] = cur;
          if (run.id == nxt_id) {   // its records were staged while it waited
            cur_inst = nxt_inst;
          } else {                  // stage now
            cur_inst = inst;
            stage_records(S, G, lane, cur, run);
            staged_now = true;
          }
          nxt_id = -1;
          if (fhead + KF < ftail) cp_ent(&e, fifo + S.doff[lane] + fhead + KF);
          fhead++;
        }
        // (5) stage the records of the op now waiting at my FIFO head
        if (running && nxt_id < 0 && fhead < ftail && !staged_now) {
          NRec r;
          load_rec(r, &S.fc[lane][fhead % KF].r);
          stage_records(S, G, lane, cur ^ 1, r);
          nxt_id = r.id;
          nxt_inst = inst;
        }
      }
      cp_commit();
      PH(4)
      __syncwarp();
      // (6) peak after all changes of this round
      if (dl) pk = max(pk, mem_sample(S, lane));
      if (!__any_sync(0xffffffffu, zero)) break;
    }
    PH(5)
  }
#undef PH
  cp_wait0();
  mk = __reduce_max_sync(0xffffffffu, mk);
  dispatched = __reduce_add_sync(0xffffffffu, dispatched);
  int oom = 0;
  if (dl) {
    oom = pk > T.cap[lane];
    if (peak_out) peak_out[(size_t)b * d + lane] = pk;
    if (busy_out) busy_out[(size_t)b * d + lane] = mybusy;
  }
  if (dbg == 2 && busy_out && lane == 0) {   // diagnostics: instants / rounds
    busy_out[(size_t)b * d] = n_inst;
    if (d > 1) busy_out[(size_t)b * d + 1] = n_round;
  }
  if (dbg == 3 && busy_out && lane == 0)     // diagnostics: cycles per phase (d >= 6)
    for (int i = 0; i < 6 && i < d; i++) busy_out[(size_t)b * d + i] = tacc[i];
  if (dbg == 3 && busy_out && lane == 0 && d >= 8) {
    busy_out[(size_t)b * d + 6] = n_need;
    busy_out[(size_t)b * d + 7] = n_inst;
  }
  oom = __reduce_or_sync(0xffffffffu, oom);
  if (lane == 0) {
    gdp_sim_report R = empty_report();
    R.makespan = mk;
    R.cross_bytes = cross;
    R.violation = (flag & 1) ? 1 : (oom ? 2 : 0);
    if (dispatched != N) R.violation = 3;   // cannot happen for a validated DAG
    R.valid = R.violation == 0;
    rep[b] = R;
    reward[b] = R.valid ? -__dsqrt_rn(__ddiv_rn((double)mk, 1e6)) : -10.0;
  }
}

}  // namespace

size_t cost2_smem_bytes(int N) { return sizeof(Smem) + 4 * (size_t)((N + 3) / 4) + 4 * (size_t)((N + 7) / 8); }

size_t cost2_scratch_per_placement(int N, long long E, int nbig) {
  size_t b = sizeof(Ent) * ((size_t)N + (size_t)(E > 0 ? E : 1)) + sizeof(NRec) * (size_t)N +
             sizeof(int) * 2 * (size_t)(nbig > 0 ? nbig : 1);
  return (b + 255) & ~(size_t)255;
}

bool launch_cost2(const Cost2Graph &G, const TopoArgs &T, const uint8_t *D, int B, unsigned char *scratch,
                  size_t per_place, gdp_sim_report *rep, long long *peak, long long *busy, double *reward,
                  cudaStream_t s) {
  const size_t smem = cost2_smem_bytes(G.N);
  if (smem > 227 * 1024) return false;
  static_assert(2 * SO + SI <= 32, "one staging request fits one warp pass");
  static size_t configured = 0;
  if (smem > 40 * 1024 && smem > configured) {
    cudaFuncSetAttribute(k_cost3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = smem;
  }
  note_launch("k_cost3", s);
  k_cost3<<<B, 32, smem, s>>>(G, T, D, scratch, per_place, rep, peak, busy, reward, 0);
  return true;
}

}  // namespace gdp
