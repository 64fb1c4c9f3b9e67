// Cost model, windowed multi-warp kernel (the default when its preconditions hold; k_cost3 in
// cost2.cu otherwise).  Same event semantics as the oracle (SPEC.md:275-284 `simulate`, O11 and
// the readings R19/R20 in DESIGN.md); this formulation runs the devices of one placement in
// parallel, one warp per device, in windows of simulated time:
//
//  * every cross-device transfer takes at least L ticks (L = min over device pairs of latency +
//    ceil(smallest edge's bytes / bandwidth), >= 1, capped at WMAX), so an op finishing
//    at tick tau in the window [T, T + W) (W <= L) can only affect another device at tick
//    >= T + W.  Inside a window the devices are therefore independent: warp q processes the
//    events of device q in time order (arrivals on its incoming channels, its finish,
//    its dispatch) without hearing from the others; the warps meet at a named barrier at the
//    end of the window and jump to the next window start (the earliest pending event);
//  * the schedule never depends on memory, so memory is accounted for off the critical path:
//    device warps add their per-tick deltas into window buckets, and a separate memory warp
//    applies producer deaths (a producer's output dies at the LAST finish tick among its
//    consumers: each consumer finish does an atomic max on the producer's death tick, and the
//    consumer that brings the counter to zero queues the producer) and sweeps the buckets in
//    tick order for the per-device peak, up to R4 windows behind the device warps.
// Requires: every op duration >= 1 (no zero-duration rounds) and L >= 1 (host checks).
#include <climits>
#include <cstdlib>

#include "common.cuh"
#include "cost2.cuh"
#include "cost_util.cuh"

namespace gdp {
namespace {
using namespace cu;

#ifndef COST4_SLEEP_NS
#define COST4_SLEEP_NS 3200   // memory warp back-off when no window is pending (A/B: 200 -> 3200 ns, 96.4 -> 95.85 ms)
#endif
#ifndef COST4_WMAX
#define COST4_WMAX 8
#endif
constexpr int WMAX = COST4_WMAX;   // window length cap (ticks) = buckets per window
#ifndef COST4_R4
#define COST4_R4 8
#endif
constexpr int R4 = COST4_R4;   // windows the memory warp may lag behind
constexpr int SO4 = 8;     // staged out-edge records per slot
constexpr int SI4 = 8;     // staged in-edge records per slot (2 * SO4 + SI4 = 24 staging lanes)
#ifndef COST4_KF
#define COST4_KF 4
#endif
#ifndef COST4_KC
#define COST4_KC 4
#endif
#ifndef COST4_NINC
#define COST4_NINC 8
#endif
constexpr int KF4 = COST4_KF;       // FIFO entries kept in smem per device
constexpr int KC4 = COST4_KC;       // prefetched channel entries per channel
constexpr int NINC4 = COST4_NINC;   // ops made available at one local instant (overflow -> global)

struct Smem4 {
  NRec st_out[8][2][SO4];
  IRec st_in[8][2][SI4];
  Ent fc[8][KF4];
  Ent cc[64][KC4];                 // consumer-side prefetch ring of channel c = 8k + q
  NRec inc[8][NINC4];
  NRec run[8];                     // record of the op running on each device
  int run_slot[8];
  unsigned long long smb[8][2];    // mbarrier of each staging slot (bulk copies complete_tx)
  unsigned lb[R4][8][WMAX][3];     // device-warp memory deltas per window set / device / tick
  long long db[R4][8][WMAX];       // producer deaths (memory warp only)
  int cfree[64], ctail[64], cstamp[64];                        // producer side (warp k)
  int pfirst[2][64], ptail[2][64];   // published per window parity: first push's arrival, tail
  int tn[3];                       // next window start, atomic min over devices' next events and first pushes
  int phs[2][64];                  // consumer head at the start of window w (parity w & 1)
  int coff[64], ccnt[64];
  int doff[8], ftail0[8], opcnt[8];
  long long stat[8], busyv[8];
  int Tw[R4], dq_end[R4];
  int dq_tail, flag, oom, mk, disp, nwin;
  int win_done, mem_done, dev_done;
  unsigned long long cross;
#ifdef COST4_PROF
  unsigned prof[8][10];
#endif
};

struct Scratch4 {   // per-placement global scratch (same prefix as k_cost2 / k_cost3)
  size_t fifo, chq, ov, bigc, dtick, dq, total;
};
__host__ __device__ inline Scratch4 scratch4_layout(int N, long long E, int nbig) {
  Scratch4 s;
  s.fifo = 0;
  s.chq = s.fifo + sizeof(Ent) * (size_t)N;
  s.ov = s.chq + sizeof(Ent) * (size_t)(E > 0 ? E : 1);
  s.bigc = s.ov + sizeof(NRec) * (size_t)N;
  s.dtick = s.bigc + sizeof(int) * 2 * (size_t)(nbig > 0 ? nbig : 1);
  s.dq = (s.dtick + sizeof(int) * (size_t)N + 15) & ~(size_t)15;
  s.total = (s.dq + sizeof(int4) * (size_t)N + 255) & ~(size_t)255;
  return s;
}

#ifdef COST4_PROF   // per-phase cycle totals of each device warp (lane 0), printed by block 0
#define PROF_MARK(k)                                           \
  do {                                                         \
    __syncwarp();                                              \
    const unsigned now_ = (unsigned)clock();                   \
    if (lane == 0) S.prof[q][k] += now_ - plast;               \
    plast = now_;                                              \
  } while (0)
#else
#define PROF_MARK(k) \
  do {               \
  } while (0)
#endif
__device__ __forceinline__ int ld_acq(const int *p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(int *p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
__device__ __forceinline__ void bar_devices(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}
// 64-bit delta as 16 + 16 + 32-bit fire-and-forget shared reductions (few adds per bucket)
__device__ __forceinline__ void add3(unsigned *w, long long v) {
  atomicAdd(&w[0], (unsigned)(v & 0xffff));
  atomicAdd(&w[1], (unsigned)((v >> 16) & 0xffff));
  atomicAdd(&w[2], (unsigned)(int)(v >> 32));
}
__device__ __forceinline__ long long read3(const unsigned *w) {
  return ((long long)(int)w[2] << 32) + ((long long)w[1] << 16) + (long long)w[0];
}
__device__ __forceinline__ bool dec_in4(unsigned *cnt, const NRec &r, int *bigc, const int *bigid) {
  if (r.cost < 0) return atomicSub(&bigc[bigid[r.id]], 1) == 1;
  const int sh = (r.id & 3) * 8;
  return ((atomicSub(&cnt[r.id >> 2], 1u << sh) >> sh) & 15u) == 1u;
}
__device__ __forceinline__ bool dec_out4(unsigned *cnt, const IRec &ir, int *bigc, int nbig) {
  if (ir.pad >= 0) return atomicSub(&bigc[ir.pad + nbig], 1) == 1;
  const int sh = (ir.u & 3) * 8 + 4;
  return ((atomicSub(&cnt[ir.u >> 2], 1u << sh) >> sh) & 15u) == 1u;
}
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(unsigned long long *mbar, unsigned parity) {
  unsigned done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                 "selp.b32 %0, 1, 0, P1;\n\t}\n"
                 : "=r"(done)
                 : "r"(smem_u32(mbar)), "r"(parity)
                 : "memory");
}
// the device lane stages the out-/in-edge records of op r into its slot sl: two bulk copies
// (contiguous record ranges) completing on the slot's mbarrier
__device__ __forceinline__ void stage_records4(Smem4 &S, const Cost2Graph &G, int q, int sl, const NRec &r) {
  const unsigned no = (unsigned)min(r.oe - r.ob, SO4), ni = (unsigned)min(r.ie - r.ib, SI4);
  unsigned long long *mb = &S.smb[q][sl];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // earlier generic reads of the slot
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)),
               "r"(no * (unsigned)sizeof(NRec) + ni * (unsigned)sizeof(IRec))
               : "memory");
  if (no)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(&S.st_out[q][sl][0])), "l"(G.erec + r.ob), "r"(no * (unsigned)sizeof(NRec)),
                 "r"(smem_u32(mb))
                 : "memory");
  if (ni)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(&S.st_in[q][sl][0])), "l"(G.irec + r.ib), "r"(ni * (unsigned)sizeof(IRec)),
                 "r"(smem_u32(mb))
                 : "memory");
}
__device__ __forceinline__ void put_inc(Smem4 &S, NRec *ovq, int q, int pos, const NRec &r) {
  if (pos < NINC4) copy_rec(&S.inc[q][pos], &r);
  else copy_rec(ovq + pos, &r);
}

// 2 CTAs per SM cap the registers at 96; more registers (one CTA per SM) run a placement ~8 %
// faster but need two waves for B = 256 (A/B: 99.5 ms vs 182.5 ms at 112 registers)
// MINB = resident CTAs per SM the register allocation is sized for: 2 (96 registers) or 3 (72
// registers, a few spills; chosen when shared memory admits a third CTA and the batch is larger
// than one wave of two per SM — profiles/r1_ab_s6/cost4_sleep.md)
template <int MINB>
__global__ void __launch_bounds__(288, MINB) k_cost4(Cost2Graph G, TopoArgs T, const uint8_t *__restrict__ Dall,
                                                  unsigned char *scratch, size_t per_place, gdp_sim_report *rep,
                                                  long long *peak_out, long long *busy_out, double *reward, int Wl,
                                                  int dbg) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem4 &S = *reinterpret_cast<Smem4 *>(smem_raw);
  const int N = G.N, d = T.d, b = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nthr = blockDim.x;
  const unsigned FULL = 0xffffffffu, lt = (1u << lane) - 1u;
  unsigned *cnt = reinterpret_cast<unsigned *>(smem_raw + sizeof(Smem4));
  const int cwords = (N + 3) >> 2;
  unsigned *Dn = cnt + cwords;
  const int dwords = (N + 7) >> 3;
  const uint8_t *D = Dall + (size_t)b * N;
  const Scratch4 L4 = scratch4_layout(N, G.E, G.nbig);
  unsigned char *base = scratch + (size_t)b * per_place;
  Ent *fifo = reinterpret_cast<Ent *>(base + L4.fifo);
  Ent *chq = reinterpret_cast<Ent *>(base + L4.chq);
  NRec *ov = reinterpret_cast<NRec *>(base + L4.ov);
  int *bigc = reinterpret_cast<int *>(base + L4.bigc);
  int *dtick = reinterpret_cast<int *>(base + L4.dtick);
  int4 *dq = reinterpret_cast<int4 *>(base + L4.dq);

  // ------------------------------------------------------------ prologue (whole block)
  for (int i = tid; i < cwords; i += nthr) cnt[i] = G.cnt0[i];
  for (int j = tid; j < G.nbig; j += nthr) { bigc[j] = G.big_in[j]; bigc[G.nbig + j] = G.big_out[j]; }
  for (int v = tid; v < N; v += nthr) dtick[v] = -1;
  if (tid < 64) { S.ccnt[tid] = 0; S.cstamp[tid] = -1; S.cfree[tid] = 0; S.ctail[tid] = 0; S.phs[0][tid] = 0; }
  if (tid < 8) { S.stat[tid] = 0; S.busyv[tid] = 0; S.opcnt[tid] = 0; }
  if (tid == 0) {
    S.flag = 0; S.oom = 0; S.cross = 0; S.dq_tail = 0; S.mk = 0; S.disp = 0; S.nwin = 0;
    S.win_done = -1; S.mem_done = -1; S.dev_done = 0;
    S.tn[0] = INF; S.tn[1] = INF; S.tn[2] = INF;
  }
  if (tid < 16) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&S.smb[tid >> 1][tid & 1])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < R4 * 8 * WMAX * 3; i += nthr) (&S.lb[0][0][0][0])[i] = 0u;
  for (int i = tid; i < R4 * 8 * WMAX; i += nthr) (&S.db[0][0][0])[i] = 0;
  __syncthreads();
  {
    long long lmem[8], lbusy[8];
    int lcnt[8], flag = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) { lmem[k] = 0; lbusy[k] = 0; lcnt[k] = 0; }
    for (int p = tid; p < dwords; p += nthr) {
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
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const long long a = warp_sum_ll(lmem[k]), c = warp_sum_ll(lbusy[k]);
      const int n = __reduce_add_sync(FULL, lcnt[k]);
      if (lane == 0 && n) {
        atomicAdd(reinterpret_cast<unsigned long long *>(&S.stat[k]), (unsigned long long)a);
        atomicAdd(reinterpret_cast<unsigned long long *>(&S.busyv[k]), (unsigned long long)c);
        atomicAdd(&S.opcnt[k], n);
      }
    }
    flag = __reduce_or_sync(FULL, flag);
    if (lane == 0 && flag) atomicOr(&S.flag, flag);
  }
  __syncthreads();
  if (S.flag & 2) {   // malformed: an entry >= d
    if (tid == 0) {
      gdp_sim_report R;
      R.makespan = 0; R.cross_bytes = 0; R.valid = 0; R.violation = 3;
      for (int i = 0; i < 6; i++) R.pad[i] = 0;
      rep[b] = R;
      reward[b] = -10.0;
    }
    if (tid < d) {
      if (peak_out) peak_out[(size_t)b * d + tid] = 0;
      if (busy_out) busy_out[(size_t)b * d + tid] = 0;
    }
    return;
  }
  {
    long long lcross = 0;
    for (long long e = tid; e < G.E; e += nthr) {
      const int u = G.out_src[e], w = G.out_idx[e];
      const int su = dev_of(Dn, u), tw = dev_of(Dn, w);
      if (su != tw) {
        atomicAdd(&S.ccnt[su * 8 + tw], 1);
        lcross += G.out_bytes[u];
      }
    }
    lcross = warp_sum_ll(lcross);
    if (lane == 0 && lcross) atomicAdd(&S.cross, (unsigned long long)lcross);
  }
  __syncthreads();
  if (warp == 0) {
    {  // device regions (FIFO overflow, incoming overflow) from op counts
      const int c = lane < d ? S.opcnt[lane] : 0;
      int inc = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += y;
      }
      if (lane < 8) S.doff[lane] = inc - c;
    }
    {  // channel regions, channels 2*lane and 2*lane+1
      const int c0 = S.ccnt[2 * lane], c1 = S.ccnt[2 * lane + 1];
      const int pair = c0 + c1;
      int inc = pair;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += y;
      }
      S.coff[2 * lane] = inc - pair;
      S.coff[2 * lane + 1] = inc - pair + c0;
    }
    __syncwarp();
    // sources are available at t = 0: appended to their FIFO in ascending id
    int ftail = 0;   // lane k: tail of device k
    for (int v0 = 0; v0 < N; v0 += 32) {
      const int v = v0 + lane;
      const bool src = v < N && G.in_ptr[v + 1] == G.in_ptr[v];
      if (!__any_sync(FULL, src)) continue;
      const int k = src ? dev_of(Dn, v) : 0;
      int off = 0, cntk = 0;
      for (int dev = 0; dev < d; dev++) {
        const unsigned m = __ballot_sync(FULL, src && k == dev);
        if (src && k == dev) off = __popc(m & lt);
        if (lane == dev) cntk = __popc(m);
      }
      const int tail_k = __shfl_sync(FULL, ftail, k & 7);
      if (src) {
        NRec r;
        load_rec(r, G.nrec + v);
        const int pos = tail_k + off;
        if (pos < KF4) store_ent(&S.fc[k][pos], r, 0, 0);
        else store_ent(fifo + S.doff[k] + pos, r, 0, 0);
      }
      ftail += cntk;
      __syncwarp();
    }
    if (lane < 8) S.ftail0[lane] = ftail;
  }
  __syncthreads();
  if (dbg == 1) return;

  if (warp < d) {
    // ---------------------------------------------------------------- device warp q
    const int q = warp;
    const bool devl = lane == q;                 // FIFO / dispatch / staging of device q
    const bool own = lane < d && lane != q;      // consumer of channel (lane -> q)
    const int cin = 8 * lane + q;
    const int offc = own ? S.coff[cin] : 0;
    Ent *ring = &S.cc[own ? cin : 0][0];
    int head = 0, tknown = 0, filled = 0, ha = INF, hs = 0;
    unsigned pend = 0;                           // ring slots with a prefetch in flight
    NRec *ovq = ov + S.doff[q];
    Ent *fq_g = fifo + S.doff[q];
    const int spd = T.speed[q];
    int fhead = 0, ftail = S.ftail0[q], running = 0, fin = 0, mk = 0, disp = 0;
    int cur = 0, nxt_id = -1;
    unsigned nst0 = 0, nst1 = 0;                 // bulk stagings issued per slot (mbarrier phases)
    int li = 0, T0 = 0, w = 0, memd = -1;
#ifdef COST4_PROF
    if (lane < 10) S.prof[q][lane] = 0;
    unsigned plast = (unsigned)clock(), ninst = 0;
#endif
    for (;; w++) {
      const int set = w % R4;
      if (w - R4 > memd) {   // the memory warp must have released this window set
        if (lane == 0)
          while ((memd = ld_acq(&S.mem_done)) < w - R4) { }
        memd = __shfl_sync(FULL, memd, 0);
      }
      if (q == 0 && lane == 0) {
        S.Tw[set] = T0;
        S.tn[(w + 1) % 3] = INF;   // read last after barrier w - 2, written from window w + 1 on
      }
      // (pfirst[w & 1][c] needs no reset: it is read after window w only if channel c was pushed
      // to in window w, and the first of those pushes wrote it)
      const int Tend = T0 + Wl;
      PROF_MARK(0);
      for (;;) {
        // key 2 tau (+1 unless my op finishes at tau); an idle device with a non-empty FIFO
        // dispatches at once (only the sources at t = 0)
        const unsigned NK = 0xffffffffu;
        const unsigned dc = running ? 2u * (unsigned)fin : (fhead < ftail ? 2u * (unsigned)T0 + 1u : NK);
        const unsigned cand = min(devl ? dc : NK, own && ha != INF ? 2u * (unsigned)ha + 1u : NK);
        const unsigned key = __reduce_min_sync(FULL, cand);
        const int tau = (int)(key >> 1);
        if (key == NK || tau >= Tend) {   // my next event opens a later window
          if (lane == 0 && key != NK) atomicMin(&S.tn[w % 3], tau);
          PROF_MARK(1);
          break;
        }
        PROF_MARK(1);
#ifdef COST4_PROF
        ninst++;
#endif
        const bool fnow = (key & 1) == 0;
        if (devl) {
          cp_wait1();   // FIFO refills older than the last instant
          if (fnow) mbar_wait(&S.smb[q][cur], ((cur ? nst1 : nst0) - 1u) & 1u);   // staged records
        }
        __syncwarp();
        PROF_MARK(2);
        long long delta = 0;
        int navail = 0;
        // (1) the copy arriving now on my incoming channel (at most one per channel per tick)
        {
          bool av = false;
          NRec ar;
          if (own && ha == tau) {
            int s = head % KC4;
            if (pend & (1u << s)) { cp_wait0(); pend = 0; }
            load_rec(ar, &ring[s].r);
            delta += ring[s].bytes;
            av = dec_in4(cnt, ar, bigc, G.bigid);
            head++;
            if (head < tknown) {
              s = head % KC4;
              if (pend & (1u << s)) { cp_wait0(); pend = 0; }
              ha = ring[s].t;
            } else {
              ha = INF;
            }
            if (filled < tknown) {   // keep KC4 entries ahead
              cp_ent(&ring[filled % KC4], chq + offc + filled);
              cp_commit();
              pend |= 1u << (filled % KC4);
              filled++;
            }
          }
          const unsigned m = __ballot_sync(FULL, av);
          if (av) put_inc(S, ovq, q, __popc(m & lt), ar);
          navail = __popc(m);
        }
        PROF_MARK(3);
        // (2) my op finishes now: its edges one per lane
        if (fnow) {
          if (devl) running = 0;
          NRec r;
          load_rec(r, &S.run[q]);
          const int sl = S.run_slot[q];
          const int nin = r.ie - r.ib, nout = r.oe - r.ob;
          // frees: copies this op held (local), producers whose last consumer it is (queued)
          for (int j = lane; j < nin; j += 32) {
            IRec ir;
            if (j < SI4) ir = S.st_in[q][sl][j];
            else ir = G.irec[r.ib + j];
            if (dev_of(Dn, ir.u) != q) delta -= ir.bytes;
            atomicMax(&dtick[ir.u], tau);
            if (dec_out4(cnt, ir, bigc, G.nbig)) {
              const int i = atomicAdd(&S.dq_tail, 1);
              dq[i] = make_int4(ir.u, 0, (int)(ir.bytes & 0xffffffffLL), (int)(ir.bytes >> 32));
            }
          }
          if (nout == 0 && lane == 0) delta -= r.bytes;
          PROF_MARK(4);
          for (int j0 = 0; j0 < nout; j0 += 32) {
            const int j = j0 + lane;
            const bool v = j < nout;
            NRec wr;
            int tw = -1;
            if (v) {
              if (j < SO4) wr = S.st_out[q][sl][j];
              else load_rec(wr, G.erec + r.ob + j);
              tw = dev_of(Dn, wr.id);
            }
            const bool cross = v && tw != q;
            const bool avs = v && !cross && dec_in4(cnt, wr, bigc, G.bigid);
            const unsigned m = __ballot_sync(FULL, avs);
            if (avs) put_inc(S, ovq, q, navail + __popc(m & lt), wr);
            navail += __popc(m);
            const unsigned cm = __ballot_sync(FULL, cross);
            if (cm) {
              const unsigned grp = (cm & (cm - 1)) ? __match_any_sync(FULL, cross ? tw : -1) : cm;
              if (cross) {
                const int rank = __popc(grp & lt), n = __popc(grp);
                const int c = 8 * q + tw;
                const int f = S.cfree[c];
                const int x = xfer_time3(r.bytes, c, T);
                const int bs = max(tau, f);
                const int tail = S.ctail[c];
                const int chs = S.phs[w & 1][c];
                __syncwarp(grp);   // every rank has read the channel state before rank 0 moves it
                const int pos = tail + rank, arr = bs + (rank + 1) * x;
                // the consumer consumed position pos - KC4 before this window: its ring slot is
                // free, so the entry goes straight there; otherwise to global for a later prefetch
                if (pos < chs + KC4) store_ent(&S.cc[c][pos % KC4], wr, arr, r.bytes);
                else store_ent(chq + S.coff[c] + pos, wr, arr, r.bytes);
                if (rank == 0) {
                  S.cfree[c] = bs + n * x;
                  S.ctail[c] = tail + n;
                  if (S.cstamp[c] != w) {   // first push of this window: the consumer may not know it yet
                    S.cstamp[c] = w;
                    S.pfirst[w & 1][c] = bs + x;
                    atomicMin(&S.tn[w % 3], bs + x);
                  }
                }
              }
              __syncwarp();
            }
          }
        }
        __syncwarp();
        PROF_MARK(5);
        // (3) device lane: ops made available now join the FIFO in id order; dispatch; stage
        if (devl) {
          const int n = navail;
          NRec *Li = &S.inc[q][0];
          NRec run;
          bool go = false;
          if (n == 1 && !running && fhead == ftail) {   // common case: straight to dispatch
            load_rec(run, Li);
            ftail++;
            fhead++;
            go = true;
          } else {
            if (n > 0) {
              for (int i = 1; i < n; i++) {   // insertion sort by id (n is small except after wide fan-outs)
                NRec key;
                load_rec(key, i < NINC4 ? &Li[i] : &ovq[i]);
                int j = i - 1;
                while (j >= 0) {
                  NRec *pj = j < NINC4 ? &Li[j] : &ovq[j];
                  if (pj->id <= key.id) break;
                  copy_rec(j + 1 < NINC4 ? &Li[j + 1] : &ovq[j + 1], pj);
                  j--;
                }
                copy_rec(j + 1 < NINC4 ? &Li[j + 1] : &ovq[j + 1], &key);
              }
              for (int i = 0; i < n; i++) {
                const NRec &rr = i < NINC4 ? Li[i] : ovq[i];
                if (ftail < fhead + KF4) store_ent(&S.fc[q][ftail % KF4], rr, tau, 0);
                else store_ent(fq_g + ftail, rr, tau, 0);
                ftail++;
              }
            }
            if (!running && fhead < ftail) {
              Ent &e = S.fc[q][fhead % KF4];
              load_rec(run, &e.r);
              if (fhead + KF4 < ftail) cp_ent(&e, fq_g + fhead + KF4);
              fhead++;
              go = true;
            }
          }
          bool staged = false;
          if (go) {
            running = 1;
            fin = tau + (run.cost & 0x7fffffff) * spd;
            mk = max(mk, fin);
            delta += run.bytes;
            disp++;
            cur ^= 1;
            copy_rec(&S.run[q], &run);
            S.run_slot[q] = cur;
            if (run.id != nxt_id) {   // not staged while it waited: stage now
              stage_records4(S, G, q, cur, run);
              if (cur) nst1++; else nst0++;
              staged = true;
            }
            nxt_id = -1;
          }
          if (!staged && running && nxt_id < 0 && fhead < ftail) {   // stage the op waiting at the head
            NRec sr;
            load_rec(sr, &S.fc[q][fhead % KF4].r);
            stage_records4(S, G, q, cur ^ 1, sr);
            if (cur) nst0++; else nst1++;
            nxt_id = sr.id;
          }
          cp_commit();
        }
        // (4) my memory delta at tau
        if (delta != 0) add3(&S.lb[set][q][tau - T0][0], delta);
        PROF_MARK(6);
        li++;
      }
      // publish the end-of-window state, meet, and find the next window start
      if (own) S.phs[(w + 1) & 1][cin] = head;
      if (lane < d) S.ptail[w & 1][8 * q + lane] = S.ctail[8 * q + lane];
      PROF_MARK(7);
      bar_devices(32 * d);   // bar.sync orders the window's shared and global writes for all device warps
      PROF_MARK(8);
      // the next window start and my channel's state first (independent loads in flight together;
      // pfirst is meaningful only if the channel was pushed to in window w), then the memory-warp
      // release (its memory clobber would otherwise order these loads behind it)
      const int Tn = S.tn[w % 3];
      const int tn_c = own ? S.ptail[w & 1][cin] : 0;
      const int pf_c = own ? S.pfirst[w & 1][cin] : INF;
      if (q == 0 && lane == 31) {   // a lane that rarely has global writes in flight (release fence)
        S.dq_end[set] = S.dq_tail;
        st_rel(&S.win_done, w);
      }
      if (own) {   // my channel: entries pushed in this window
        const int tn = tn_c;
        if (ha == INF && tn > tknown) ha = pf_c;
        const int lim = min(tn, head + KC4);
        for (; filled < lim; filled++) {
          if (filled >= tknown && filled < hs + KC4) continue;   // the producer wrote it into the ring
          cp_ent(&ring[filled % KC4], chq + offc + filled);
          cp_commit();
          pend |= 1u << (filled % KC4);
        }
        tknown = tn;
        hs = head;
      }
      if (Tn == INF) break;
      T0 = Tn;
    }
    cp_wait0();
#ifdef COST4_PROF
    if (b == 0 && lane == 0)
      printf("PROF q=%d win=%d inst=%u pre=%u key=%u wait=%u arr=%u finin=%u finout=%u disp=%u post=%u bar=%u\n", q,
             w + 1, ninst, S.prof[q][0], S.prof[q][1], S.prof[q][2], S.prof[q][3], S.prof[q][4], S.prof[q][5],
             S.prof[q][6], S.prof[q][7], S.prof[q][8]);
#endif
    if (devl) {
      atomicMax(&S.mk, mk);
      atomicAdd(&S.disp, disp);
    }
    if (q == 0 && lane == 0) {
      S.nwin = w + 1;
      st_rel(&S.dev_done, 1);
    }
  } else {
    // ---------------------------------------------------------------- memory warp
    long long mem = lane < d ? S.stat[lane] : 0, pk = mem;
    int done_w = -1, dq_start = 0;
    for (;;) {
      int wd = 0, fin_all = 0;
      if (lane == 0) {
        wd = ld_acq(&S.win_done);
        fin_all = ld_acq(&S.dev_done);
      }
      wd = __shfl_sync(FULL, wd, 0);
      fin_all = __shfl_sync(FULL, fin_all, 0);
      if (wd > done_w) {
        // producer deaths queued in windows done_w+1 .. wd
        const int dq_stop = S.dq_end[wd % R4];
        for (int i = dq_start + lane; i < dq_stop; i += 32) {
          const int4 en = __ldcg(dq + i);
          const int u = en.x;
          const long long bytes = ((long long)(unsigned)en.z) | ((long long)en.w << 32);
          const int tk = __ldcg(dtick + u);
          const int du = dev_of(Dn, u);
          int ww = done_w + 1;
          while (ww < wd && tk >= S.Tw[ww % R4] + Wl) ww++;
          atomicAdd(reinterpret_cast<unsigned long long *>(&S.db[ww % R4][du][tk - S.Tw[ww % R4]]),
                    (unsigned long long)(-bytes));
        }
        dq_start = dq_stop;
        __syncwarp();
        for (int ww = done_w + 1; ww <= wd; ww++) {   // tick-ordered sweep of each window
          const int s = ww % R4;
          if (lane < d) {
            for (int o = 0; o < Wl; o++) {
              unsigned *wv = &S.lb[s][lane][o][0];
              mem += read3(wv) + S.db[s][lane][o];
              pk = max(pk, mem);
              wv[0] = 0u; wv[1] = 0u; wv[2] = 0u;
              S.db[s][lane][o] = 0;
            }
          }
          __syncwarp();
          if (lane == 0) st_rel(&S.mem_done, ww);
        }
        done_w = wd;
      } else if (fin_all && done_w == S.nwin - 1) {
        break;
      } else {
        if (COST4_SLEEP_NS > 0) __nanosleep(COST4_SLEEP_NS);
      }
    }
    if (lane < d) {
      if (pk > T.cap[lane]) atomicOr(&S.oom, 1);
      if (peak_out) peak_out[(size_t)b * d + lane] = pk;
      if (busy_out) busy_out[(size_t)b * d + lane] = S.busyv[lane];
    }
    if (dbg == 2 && busy_out && lane == 0) busy_out[(size_t)b * d] = S.nwin;
  }
  __syncthreads();
  if (tid == 0) {
    gdp_sim_report R;
    R.makespan = S.mk; R.cross_bytes = (long long)S.cross; R.valid = 0; R.violation = 0;
    for (int i = 0; i < 6; i++) R.pad[i] = 0;
    R.violation = (S.flag & 1) ? 1 : (S.oom ? 2 : 0);
    if (S.disp != N) R.violation = 3;   // cannot happen for a validated DAG
    R.valid = R.violation == 0;
    rep[b] = R;
    reward[b] = R.valid ? -__dsqrt_rn(__ddiv_rn((double)S.mk, 1e6)) : -10.0;
  }
}

}  // namespace

size_t cost4_smem_bytes(int N) { return sizeof(Smem4) + 4 * (size_t)((N + 3) / 4) + 4 * (size_t)((N + 7) / 8); }
size_t cost4_scratch_per_placement(int N, long long E, int nbig) { return scratch4_layout(N, E, nbig).total; }

// Wl = the shortest possible transfer: min over device pairs of latency + ceil(smallest edge's
// bytes / bandwidth), capped at WMAX
int cost4_window(const TopoArgs &T, int min_cost, int N, long long min_edge_bytes) {
  static const bool off = getenv("GDP_COST_V3") != nullptr || getenv("GDP_COST_V2") != nullptr;
  if (off) return 0;
  const int d = T.d;
  if (d < 1 || d > 8 || min_cost < 1) return 0;   // zero-duration ops need same-instant rounds
  int L = WMAX;
  for (int k = 0; k < d; k++) {
    if (T.speed[k] < 1) return 0;
    for (int q = 0; q < d; q++)
      if (k != q) {
        long long x = T.lat[k * 8 + q];
        if (min_edge_bytes > 0 && T.bpt[k * 8 + q] > 0) x += (min_edge_bytes - 1) / T.bpt[k * 8 + q] + 1;
        L = L < x ? L : (int)x;
      }
  }
  if (L < 1) return 0;                           // a transfer could land in its own window
  if (cost4_smem_bytes(N) > 227 * 1024) return 0;
  return L;
}

bool launch_cost4(const Cost2Graph &G, const TopoArgs &T, int min_cost, long long min_edge_bytes, const uint8_t *D, int B,
                  unsigned char *scratch, size_t per_place, gdp_sim_report *rep, long long *peak, long long *busy,
                  double *reward, cudaStream_t s) {
  const int L = cost4_window(T, min_cost, G.N, min_edge_bytes);
  if (L < 1) return false;
  if (per_place < cost4_scratch_per_placement(G.N, G.E, G.nbig)) return false;
  const int d = T.d, nthr = 32 * (d + 1);
  const size_t smem = cost4_smem_bytes(G.N);
  static size_t configured2 = 0, configured3 = 0;
  if (smem > 40 * 1024 && smem > configured2) {
    cudaFuncSetAttribute(k_cost4<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured2 = smem;
  }
  if (smem > 40 * 1024 && smem > configured3) {
    cudaFuncSetAttribute(k_cost4<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured3 = smem;
  }
  static_assert(2 * SO4 + SI4 == 24, "24 staging lanes");
  static const int dbg = getenv("GDP_COST_DBG") ? atoi(getenv("GDP_COST_DBG")) : 0;
  // GDP_COST4_MINB = 2 | 3 forces a variant (A/B); otherwise the 72-register one runs when it
  // keeps more CTAs resident per SM and the batch does not fit one wave of the 96-register one
  static const int force = getenv("GDP_COST4_MINB") ? atoi(getenv("GDP_COST4_MINB")) : 0;
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  int occ2 = 0, occ3 = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_cost4<2>, nthr, smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ3, k_cost4<3>, nthr, smem);
  const bool use3 = force ? force == 3 : (occ3 > occ2 && (long long)B > (long long)occ2 * nsm);
  note_launch("k_cost4", s);
  if (use3)
    k_cost4<3><<<B, nthr, smem, s>>>(G, T, D, scratch, per_place, rep, peak, busy, reward, L, dbg);
  else
    k_cost4<2><<<B, nthr, smem, s>>>(G, T, D, scratch, per_place, rep, peak, busy, reward, L, dbg);
  return true;
}

}  // namespace gdp
