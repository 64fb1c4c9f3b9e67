// Cost model (a12), the default kernel: one SIMULATION warp and one MEMORY warp per placement.
//
// Same event semantics as the oracle (SPEC.md:275-284 `simulate`, SURVEY O11 with the readings
// R19/R20 in DESIGN.md §2), in the arrival-event formulation: an op keeps a count of inputs not
// yet ARRIVED and becomes available at the instant the count reaches zero (= its ready time), so
// device FIFOs are appended in time order and stay sorted by (ready, id) without a priority
// queue; the events of an instant are the copy arrivals due now (one per directed channel at
// most, because every transfer takes >= 1 tick) and the finishes due now (ascending op id).
//
//  * Simulation warp (the critical path).  Lane q < d owns device q: its running op (record in
//    registers), its FIFO and the staging slots of its out-edge records.  Lane L owns the
//    directed channels 2L and 2L+1 (c = 8 * src + dst): the head arrival time of each in a
//    register.  An instant is: t = min over the lanes' candidates (one REDUX), arrivals popped by
//    their owners in parallel, each finishing op's out-edges one per lane (same device -> input
//    arrived now; other device -> FIFO push on the directed channel, ranked with match_any so
//    that max(t, free) + (rank + 1) * xfer is computed in parallel), the ops made available now
//    appended to their device FIFO in id order, idle devices dispatch their FIFO head.  Nothing
//    of the memory accounting is on this path: the warp only appends 8-byte items (instant,
//    kind, device, index) to a ring in shared memory.
//  * Memory warp (off the critical path, lagging).  Consumes the item ring 32 items at a time:
//    allocations (an op's output from its start, a copy from its arrival), the frees of a finish
//    (the copies the op held; producers whose LAST consumer this is -- a per-placement counter in
//    global memory, one atomic per producer and batch; the op's own output if it is a sink), and
//    samples each device's resident bytes whenever the instant changes (= after every change of
//    an instant, the oracle's step (4)).
//  * Per-op state in shared memory is only the input counters: ops with one input need none,
//    ops with exactly two inputs one "first input arrived" bit (a compact bitmap), ops with
//    3..15 inputs a 4-bit counter, more a global counter (C4: 6.9 KB).  Device ids are not in
//    shared memory: a finishing op's consumers' devices -- and each cross edge's transfer time,
//    so no division is on the critical path -- come with its staged out-edge records (a
//    per-placement word per out-edge slot that k_cost5_pre writes), the memory warp reads the
//    placement row from L2.  Static memory, busy time, channel sizes and the co-location check
//    also come from k_cost5_pre (one CTA per placement, fully parallel).  With 18.1 KB of shared
//    memory per placement (compact channel rings, heads fetched by bulk copies), twelve CTAs
//    (placements) share an SM at C4.
// Requires (host-checked): every duration >= 1 and every transfer >= 1 tick (no same-instant
// rounds), N and E < 2^25, degrees < 2^16.  Otherwise gdp_cost runs k_cost3 / k_cost (cost2.cu,
// cost.cu).
#include <algorithm>
#include <climits>
#include <vector>

#include "common.cuh"
#include "cost2.cuh"
#include "cost_util.cuh"

namespace gdp {
namespace {
using namespace cu;

constexpr int KC5 = 4;      // channel entries kept in shared memory per channel (power of 2)
#ifndef COST5_KF
#define COST5_KF 2
#endif
#ifndef COST5_SO
#define COST5_SO 5
#endif
#ifndef COST5_NINC
#define COST5_NINC 1
#endif
constexpr int KF5 = COST5_KF;       // FIFO entries kept in shared memory per device (power of 2)
constexpr int SO5 = COST5_SO;       // staged out-edge records per slot (more: read from global at the finish)
constexpr int NINC5 = COST5_NINC;   // ops made available at one instant kept in shared memory per device
#ifndef COST5_RI
#define COST5_RI 64
#endif
#ifndef COST5_MB
#define COST5_MB 32
#endif
#ifndef COST5_MBAR
#define COST5_MBAR 0   // 1: the memory warp sleeps on an mbarrier the simulation warp arrives on per 32 items
                       // (measured 162.8 ms vs 142.3 ms polling at C4 B = 1776: kept off)
#endif
#ifndef COST5_TRI
#define COST5_TRI 1   // three-input ops count in 2-bit fields (4-bit fields for 4..15 inputs)
#endif
#ifndef COST5_SLEEP
#define COST5_SLEEP 4500
#endif
#ifndef COST5_SPIN
#define COST5_SPIN 8
#endif
constexpr int RI5 = COST5_RI;       // memory item ring (power of 2)
constexpr int MB5 = COST5_MB;       // the memory warp waits for this many items (or the end) before a batch

#ifdef COST5_PROF   // per-phase cycle totals of the simulation warp (lane 0), printed by block 0
#define P5(i)                                              \
  do {                                                     \
    const long long now_ = clock64();                      \
    prof[i] += now_ - plast;                               \
    plast = now_;                                          \
  } while (0)
#define P5C(i) (prof[i]++)
#else
#define P5(i) \
  do {        \
  } while (0)
#define P5C(i) \
  do {         \
  } while (0)
#endif

// IT_FIN: an op with inputs finished (idx = its id); the memory warp expands it into its in-edges
enum { IT_ALLOC_OP = 0, IT_ALLOC_COPY = 1, IT_INEDGE = 2, IT_SINK = 3, IT_END = 4, IT_FIN = 5 };


struct Pre5 {   // per-placement results of k_cost5_pre
  long long stat[8], busy[8];
  long long cross;
  int opcnt[8];
  int chcnt[64];
  int flag;      // bit 0 co-location violation, bit 1 malformed (an entry >= d)
  int pad[3];
};

constexpr int NCH = 56;     // directed channels src != dst, compact index 7 src + dst - (dst > src)
__host__ __device__ __forceinline__ int cidx(int src, int dst) { return 7 * src + dst - (dst > src ? 1 : 0); }
__device__ __forceinline__ int cdst(int ci) {
  const int s = ci / 7, r = ci - 7 * s;
  return r + (r >= s ? 1 : 0);
}

struct Smem5 {
  int4 chd[NCH];                    // each channel's head entry: the consumer's packed record (Slot5;
                                    // fetched by a bulk copy of its out-edge slot when it becomes the head)
  int2 cq[NCH][KC5];                // channel rings, compact: (out-edge slot, arrival tick)
  unsigned long long hbar[NCH];     // mbarrier of each channel's head fetch
  int4 stage[8][2][SO5];            // out-edge slots (packed Slot5) of the running / next op of each device
  unsigned sdev[8][2][SO5];         // each staged slot's word from k_cost5_pre: consumer device | transfer time << 3
  int4 fc[8][KF5];                  // FIFO rings: id, cost, ob, nn (the queue fields a dispatch reads)
  int4 inc[8][NINC5];               // ops made available at this instant (same fields)
  unsigned long long items[RI5];    // memory items: t | code << 32
  unsigned long long ibar;          // mbarrier: one phase per 32 items appended (and one at the end)
  int4 drun[8];                     // the op running on each device: id, ob, nn -- what its finish
                                    // reads (one 16-byte load / store instead of a 32-byte Q5: -1.7 %)
  int4 ch[NCH];                     // per channel: tail, free (transfer end), head, overflow offset
  int ca[NCH];                      // arrival tick of each channel's head entry (INF: empty; contiguous: the
                                    // next-event REDUX reads two per lane without bank conflicts)
  int4 dv[8];                       // per device: finish of the running op (INF: idle), FIFO head, tail, #available now
  int4 dv2[8];                      // per device: staging slot of the running op, op staged in the other, speed
  int doff[8];
  int mhead;                        // items consumed by the memory warp
  int mk, disp, oom;
  int simw;                         // which of the two warps simulates (the other does the memory accounting)
};

struct Scratch5 {
  size_t pre, sdev, outcnt, gbig, fifo, ov, chq, total;
};
__host__ __device__ inline Scratch5 scratch5_layout(int N, long long E, int ngbig) {
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  Scratch5 s;
  s.pre = 0;
  s.sdev = al(sizeof(Pre5));
  s.outcnt = s.sdev + al(4 * (size_t)(E > 0 ? E : 1) + 16);
  s.gbig = s.outcnt + al(4 * (size_t)N);
  s.fifo = s.gbig + al(4 * (size_t)(ngbig > 0 ? ngbig : 1));
  s.ov = s.fifo + al(sizeof(Q5) * (size_t)N);
  s.chq = s.ov + al(sizeof(Q5) * (size_t)N);
  s.total = s.chq + al(sizeof(int2) * (size_t)(E > 0 ? E : 1));
  return s;
}

// fields of a packed record (Slot5 layout, held as int4)
constexpr int M25 = (1 << 25) - 1;
__device__ __forceinline__ int rec_id(const int4 &r) { return r.x & M25; }
__device__ __forceinline__ int rec_ob(const int4 &r) { return r.z & M25; }
__device__ __forceinline__ int rec_cinfo(const int4 &r) {
  const unsigned ix = ((unsigned)r.w >> 16) | ((((unsigned)r.z >> 27) & 3u) << 16) | (((unsigned)r.x >> 25) << 18);
  return (int)((((unsigned)r.z >> 25) & 3u) | (ix << 2));
}
__device__ __forceinline__ void cp_4(void *s, const void *g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g)
               : "memory");
}
// a channel's new head: its out-edge slot (16 bytes) copied by the bulk-copy engine, completing
// on the channel's mbarrier (independent of the cp.async groups of the staging copies)
__device__ __forceinline__ void head_fetch(int4 *dst, const Slot5 *src, unsigned long long *mb) {
  const unsigned m = (unsigned)__cvta_generic_to_shared(mb);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16;" ::"r"(m) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(m)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive5(unsigned long long *mb) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(mb)) : "memory");
}
// sleep (suspended in hardware, not polling) until the phase of parity ph completes or ~20 us
// pass; the caller re-reads the ring either way (if the simulation warp ran an even number of
// batches ahead the parity alone cannot tell, so the time limit is what keeps that case live)
__device__ __forceinline__ void mbar_sleep5(unsigned long long *mb, unsigned ph) {
  unsigned done;
  const unsigned m = (unsigned)__cvta_generic_to_shared(mb);
  asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, 20000;\n\t"
               "selp.b32 %0, 1, 0, P1;\n\t}\n"
               : "=r"(done)
               : "r"(m), "r"(ph)
               : "memory");
  (void)done;
}
__device__ __forceinline__ void head_wait(unsigned long long *mb, unsigned ph) {
  unsigned done = 0;
  const unsigned m = (unsigned)__cvta_generic_to_shared(mb);
  while (!done)
    asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                 "selp.b32 %0, 1, 0, P1;\n\t}\n"
                 : "=r"(done)
                 : "r"(m), "r"(ph)
                 : "memory");
}
// shared-memory words addressed by their 32-bit shared-window address (computed once per kernel)
__device__ __forceinline__ unsigned atoms_xor(unsigned a, unsigned x) {
  unsigned v;
  asm volatile("atom.shared.xor.b32 %0, [%1], %2;" : "=r"(v) : "r"(a), "r"(x) : "memory");
  return v;
}
__device__ __forceinline__ unsigned atoms_add(unsigned a, unsigned x) {
  unsigned v;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(v) : "r"(a), "r"(x) : "memory");
  return v;
}
// an input of op (cinfo) arrived now: true iff it was the last one (the op becomes available now)
__device__ __forceinline__ bool arrive5(unsigned flag_s, unsigned bigb_s, int *gbig, int cinfo) {
#if COST5_TRI
  if (cinfo == 0) return true;
  const int kind = cinfo & 3;
  const int ix = cinfo >> 2;
  if (kind == 0) {   // three inputs: a 2-bit count (from 3) at field ix - 1 of the counter words
    const int p = ix - 1, sh = (p & 15) * 2;
    return ((atoms_add(bigb_s + 4u * (unsigned)(p >> 4), 0u - (1u << sh)) >> sh) & 3u) == 1u;
  }
#else
  const int kind = cinfo & 3;
  if (kind == 0) return true;
  const int ix = cinfo >> 2;
#endif
  if (kind == 1) {
    const unsigned bit = 1u << (ix & 31);
    return (atoms_xor(flag_s + 4u * (unsigned)(ix >> 5), bit) & bit) != 0u;
  }
  if (kind == 2) {
    const int sh = (ix & 7) * 4;
    return ((atoms_add(bigb_s + 4u * (unsigned)(ix >> 3), 0u - (1u << sh)) >> sh) & 15u) == 1u;
  }
  return atomicSub(&gbig[ix], 1) == 1;
}

__device__ __forceinline__ unsigned long long item5(int t, int kind, int dev, int idx, unsigned pos) {
  const unsigned code = ((pos / RI5) & 1u) | ((unsigned)kind << 1) | ((unsigned)dev << 4) | ((unsigned)idx << 7);
  return (unsigned long long)(unsigned)t | ((unsigned long long)code << 32);
}

// ------------------------------------------------------------------------ pre-pass
// One CTA per placement: static memory / busy time / op count per device, co-location and
// malformed flags, per out-edge slot the consumer's device and the transfer time (one word per slot, out-CSR
// order), cross bytes and per-channel transfer counts (the sizes of the global overflow
// regions), consumer counters of the memory warp, global input counters.  The placement row
// (N bytes) is staged in shared memory with 16-byte loads when it fits (dynamic shared memory
// = N rounded to 16; 0 = read from global), so the random D[u] / D[w] reads of the edge pass hit
// shared memory; the edge pass takes 4 consecutive slots per thread (16-byte loads of the
// producer / consumer ids, one 32-bit store of their 4 device bytes).
__global__ void __launch_bounds__(512) k_cost5_pre(Cost5Graph G, TopoArgs T, const uint8_t *__restrict__ Dall,
                                                   unsigned char *scratch, size_t per_place, int dsm) {
  extern __shared__ __align__(16) uint8_t sD[];
  __shared__ unsigned long long s_stat[8], s_busy[8], s_cross;
  __shared__ int s_cnt[8], s_ch[64], s_flag;
  __shared__ int s_chw[16][64];   // per-warp channel counts (no contention on 64 addresses)
  __shared__ long long s_bpt[64];
  __shared__ double s_ibpt[64];
  __shared__ int s_lat[64];
  const int N = G.N, d = T.d, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  const unsigned FULL = 0xffffffffu;
  const uint8_t *Dg = Dall + (size_t)b * N;
  const Scratch5 L = scratch5_layout(N, G.E, G.ngbig);
  unsigned char *base = scratch + (size_t)b * per_place;
  Pre5 *pre = reinterpret_cast<Pre5 *>(base + L.pre);
  unsigned *sdev = reinterpret_cast<unsigned *>(base + L.sdev);
  int *outcnt = reinterpret_cast<int *>(base + L.outcnt);
  int *gbig = reinterpret_cast<int *>(base + L.gbig);
  if (tid < 8) { s_stat[tid] = 0; s_busy[tid] = 0; s_cnt[tid] = 0; }
  if (tid < 64) {
    s_ch[tid] = 0;
    s_bpt[tid] = T.bpt[tid];   // the channel tables in shared memory: the edge pass indexes them per lane
    s_ibpt[tid] = T.inv_bpt[tid];
    s_lat[tid] = T.lat[tid];
  }
  for (int i = tid; i < 16 * 64; i += blockDim.x) (&s_chw[0][0])[i] = 0;
  if (tid == 0) { s_cross = 0; s_flag = 0; }
  if (dsm) {   // the row into shared memory (B x N rows are 16-byte aligned when N % 16 == 0)
    if ((reinterpret_cast<uintptr_t>(Dg) & 15) == 0) {
      const int n16 = N / 16;
      for (int i = tid; i < n16; i += blockDim.x) reinterpret_cast<uint4 *>(sD)[i] = __ldg(reinterpret_cast<const uint4 *>(Dg) + i);
      for (int v = 16 * n16 + tid; v < N; v += blockDim.x) sD[v] = Dg[v];
    } else {
      for (int v = tid; v < N; v += blockDim.x) sD[v] = Dg[v];
    }
  }
  __syncthreads();
  const uint8_t *D = dsm ? sD : Dg;
  {
    long long lm[8], lb[8];
    int lc[8], flag = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) { lm[k] = 0; lb[k] = 0; lc[k] = 0; }
    for (int v = tid; v < N; v += blockDim.x) {
      int k = D[v];
      if (k >= d) { flag |= 2; k = 0; }
      const long long mb = G.mem_bytes[v];
      const long long du = (long long)G.cost[v] * T.speed[k];
#pragma unroll
      for (int q = 0; q < 8; q++)
        if (q == k) { lm[q] += mb; lb[q] += du; lc[q] += 1; }
      if (G.has_coloc && D[G.leader[v]] != D[v]) flag |= 1;
    }
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const long long a = warp_sum_ll(lm[k]), c = warp_sum_ll(lb[k]);
      const int n = __reduce_add_sync(FULL, lc[k]);
      if (lane == 0 && n) {
        atomicAdd(&s_stat[k], (unsigned long long)a);
        atomicAdd(&s_busy[k], (unsigned long long)c);
        atomicAdd(&s_cnt[k], n);
      }
    }
    flag = __reduce_or_sync(FULL, flag);
    if (lane == 0 && flag) atomicOr(&s_flag, flag);
  }
  {
    long long lcross = 0;
    int *chw = s_chw[(tid >> 5) & 15];
    // per slot: the consumer's device (3 bits) and, for a cross edge, its transfer time (the
    // simulation warp stages the word with the slot: no division on its critical path)
    auto edge = [&](long long e, int u, int w) -> unsigned {
      const int su = D[u], tw = D[w];
      unsigned x = 0;
      if (su != tw && su < d && tw < d) {
        atomicAdd(&chw[su * 8 + tw], 1);
        const long long by = __ldg(G.ebytes + e);
        lcross += by;
        {   // = xfer_time3(by, 8 su + tw, T) on the shared-memory tables
          const int c = 8 * su + tw;
          const long long bw = s_bpt[c];
          long long qq = (long long)((double)by * s_ibpt[c]);
          long long rr = by - qq * bw;
          while (rr < 0) { qq--; rr += bw; }
          while (rr >= bw) { qq++; rr -= bw; }
          x = (unsigned)((int)(qq + (rr > 0)) + s_lat[c]);
        }
      }
      return (x << 3) | ((unsigned)tw & 7u);
    };
    const long long E4 = G.E / 4;
    const int4 *src4 = reinterpret_cast<const int4 *>(G.out_src), *idx4 = reinterpret_cast<const int4 *>(G.out_idx);
    for (long long q = tid; q < E4; q += blockDim.x) {   // 4 slots per thread
      const int4 u = __ldg(src4 + q), w = __ldg(idx4 + q);
      const long long e = 4 * q;
      const unsigned b0 = edge(e, u.x, w.x), b1 = edge(e + 1, u.y, w.y), b2 = edge(e + 2, u.z, w.z),
                     b3 = edge(e + 3, u.w, w.w);
      reinterpret_cast<uint4 *>(sdev)[q] = make_uint4(b0, b1, b2, b3);
    }
    for (long long e = 4 * E4 + tid; e < G.E; e += blockDim.x) sdev[e] = edge(e, G.out_src[e], G.out_idx[e]);
    lcross = warp_sum_ll(lcross);
    if (lane == 0 && lcross) atomicAdd(&s_cross, (unsigned long long)lcross);
  }
  {  // consumer counters of the memory warp: a 16-byte vector copy of the out-degrees
    const int n4 = N / 4;
    const int4 *src = reinterpret_cast<const int4 *>(G.outdeg);
    int4 *dst = reinterpret_cast<int4 *>(outcnt);
    for (int i = tid; i < n4; i += blockDim.x) dst[i] = __ldg(src + i);
    for (int v = 4 * n4 + tid; v < N; v += blockDim.x) outcnt[v] = G.outdeg[v];
  }
  for (int i = tid; i < G.ngbig; i += blockDim.x) gbig[i] = G.gbig0[i];
  __syncthreads();
  if (tid < 64) {
    int c = 0;
    for (int w = 0; w < 16; w++) c += s_chw[w][tid];
    s_ch[tid] = c;
  }
  __syncthreads();
  if (tid < 8) {
    pre->stat[tid] = (long long)s_stat[tid];
    pre->busy[tid] = (long long)s_busy[tid];
    pre->opcnt[tid] = s_cnt[tid];
  }
  if (tid < 64) pre->chcnt[tid] = s_ch[tid];
  if (tid == 0) { pre->cross = (long long)s_cross; pre->flag = s_flag; }
}

// ------------------------------------------------------------------------ main kernel
// The two warps of a 64-thread CTA occupy warp slots 2i, 2i + 1 of their SM, i.e. sub-partitions
// (0, 1) or (2, 3) (slot mod 4; measured, tools/lat/smsp.cu).  With warp 0 always simulating, every
// simulation warp would share sub-partitions 0 and 2 while 1 and 3 hold the mostly sleeping memory
// warps; so successive CTAs on the same (SM, sub-partition pair) alternate the simulating warp.
__device__ unsigned g_c5_pair[2 * 1024];
#ifndef COST5_MINB
#define COST5_MINB 16
#endif
// B32: every output < 2^31 bytes (Cost5Graph::bytes32), so the memory warp broadcasts 32-bit
// deltas; a template parameter rather than a branch, which costs registers in the shared budget
template <bool B32>
__global__ void __launch_bounds__(64, COST5_MINB) k_cost5(Cost5Graph G, TopoArgs T, const uint8_t *__restrict__ Dall,
                                              unsigned char *scratch, size_t per_place, gdp_sim_report *rep,
                                              long long *peak_out, long long *busy_out, double *reward) {
  __shared__ Smem5 S;                                       // fixed state (static: direct addressing)
  extern __shared__ __align__(16) unsigned char smem_raw[];   // input counters: flag bits, byte counters
  const int N = G.N, d = T.d, b = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const unsigned FULL = 0xffffffffu, lt = (1u << lane) - 1u;
#ifdef COST5_TIMING   // per-placement wall time (us) and SM in the report's padding (tools/cost5_spread.py)
  unsigned long long t_beg;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_beg));
#endif
  unsigned *flags = reinterpret_cast<unsigned *>(smem_raw);
  unsigned *bigb = flags + G.nflagw;
  const unsigned flag_s = (unsigned)__cvta_generic_to_shared(flags), bigb_s = flag_s + 4u * (unsigned)G.nflagw;
  const uint8_t *D = Dall + (size_t)b * N;
  const Scratch5 L = scratch5_layout(N, G.E, G.ngbig);
  unsigned char *base = scratch + (size_t)b * per_place;
  const Pre5 *pre = reinterpret_cast<const Pre5 *>(base + L.pre);
  const unsigned *sdev_g = reinterpret_cast<const unsigned *>(base + L.sdev);
  int *outcnt = reinterpret_cast<int *>(base + L.outcnt);
  int *gbig = reinterpret_cast<int *>(base + L.gbig);
  int4 *fifo_g = reinterpret_cast<int4 *>(base + L.fifo);
  int4 *ov_g = reinterpret_cast<int4 *>(base + L.ov);
  int2 *chq_g = reinterpret_cast<int2 *>(base + L.chq);

  // ------------------------------------------------------------ prologue (both warps)
  {
    for (int i = tid; i < G.nflagw; i += 64) flags[i] = 0u;
    for (int i = tid; i < G.nbigb; i += 64) bigb[i] = G.bigb0[i];
    for (int i = tid; i < RI5; i += 64) S.items[i] = 1ull << 32;   // lap parity 1: empty for lap 0
    if (tid < NCH) {
      S.ca[tid] = INF;
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&S.hbar[tid])));
    }
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&S.ibar)));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < 8) { S.dv[tid] = make_int4(INF, 0, 0, 0); S.dv2[tid] = make_int4(0, -1, T.speed[tid], 0); }
    if (tid == 0) {
      S.mhead = 0; S.mk = 0; S.disp = 0; S.oom = 0;
      unsigned wid, sm;
      asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      S.simw = (int)(atomicAdd(&g_c5_pair[(2 * sm + ((wid >> 1) & 1u)) & 2047u], 1u) & 1u);
    }
    if (tid == 32) {
      int o = 0;
      for (int k = 0; k < 8; k++) { S.doff[k] = o; o += pre->opcnt[k]; }
      o = 0;
      for (int a = 0; a < 8; a++)
        for (int b2 = 0; b2 < 8; b2++)
          if (a != b2) { S.ch[cidx(a, b2)] = make_int4(0, 0, 0, o); o += pre->chcnt[8 * a + b2]; }
    }
  }
  const int pflag = pre->flag;
  __syncthreads();
  if (pflag & 2) {   // malformed: an entry >= d
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

  if (warp == S.simw) {
    // ============================================================ simulation warp
    // Warp-uniform serial event processing: every lane executes the same code on the same
    // values (so a lane reads back its own stores of the shared state and no lane diverges);
    // lane parallelism only where it pays -- the next-event minimum (one REDUX over the 64
    // channel heads and 8 running finishes), the out-edges of a finish, the in-edge items and
    // the staging copies (those sections end with __syncwarp).
    int t = 0;   // the instant; after the loop the last one = the makespan (the last event is a finish)
    unsigned spend = 0;                 // this lane's staging copies in flight (bit 2k + slot)
    unsigned itail = 0, mcache = 0;     // items appended; memory-warp head as last read
    unsigned incm = 0;                  // devices with ops made available at this instant
    unsigned long long hpn = 0, hph = 0;  // channels with a head fetch in flight; their mbarrier phases
#ifdef COST5_PROF
    long long prof[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, plast = clock64();
#endif
    auto ensure = [&](unsigned n) {
      while (itail + n - mcache > (unsigned)RI5) {
        P5C(8);
        mcache = (unsigned)*reinterpret_cast<volatile int *>(&S.mhead);
        if (itail + n - mcache > (unsigned)RI5) __nanosleep(64);
      }
    };
    auto item = [&](int kind, int dev, int idx) {   // uniform: every lane stores the same item
      ensure(1);
      S.items[itail & (RI5 - 1)] = item5(t, kind, dev, idx, itail);
      itail++;
#if COST5_MBAR
      if ((itail & 31u) == 0u && lane == 0) mbar_arrive5(&S.ibar);   // a batch of 32 is complete
#endif
    };
    auto to_inc = [&](int q, const int4 &x) {     // uniform; x: the op's packed record
      const int n = S.dv[q].w;
      if (n < NINC5) S.inc[q][n] = x;
      else ov_g[S.doff[q] + n] = x;
      S.dv[q].w = n + 1;
      incm |= 1u << q;
    };
    // uniform input arrival (no other lane touches the counters concurrently)
    auto arrive_u = [&](int cinfo) -> bool {
#if COST5_TRI
      if (cinfo == 0) return true;
      const int kind = cinfo & 3;
      const int ix = cinfo >> 2;
      if (kind == 0) {
        const int p = ix - 1, sh = (p & 15) * 2;
        const unsigned w = bigb[p >> 4];
        bigb[p >> 4] = w - (1u << sh);
        return ((w >> sh) & 3u) == 1u;
      }
#else
      const int kind = cinfo & 3;
      if (kind == 0) return true;
      const int ix = cinfo >> 2;
#endif
      if (kind == 1) {
        const unsigned bit = 1u << (ix & 31), w = flags[ix >> 5];
        flags[ix >> 5] = w ^ bit;
        return (w & bit) != 0u;
      }
      if (kind == 2) {
        const int sh = (ix & 7) * 4;
        const unsigned w = bigb[ix >> 3];
        bigb[ix >> 3] = w - (1u << sh);
        return ((w >> sh) & 15u) == 1u;
      }
      const int o = gbig[ix];
      gbig[ix] = o - 1;
      return o == 1;
    };
    auto stage = [&](int k, int sl, const int4 &r) {   // lane j copies out-edge slot j and its device byte
      const int no = min(r.w & 0xffff, SO5);
      if (lane < no) {
        const int e = rec_ob(r) + lane;
        cp16(&S.stage[k][sl][lane], G.slots + e);
        cp_4(&S.sdev[k][sl][lane], sdev_g + e);
        spend |= 1u << (2 * k + sl);
      }
      cp_commit();
    };

    __syncwarp();
    // sources are available at t = 0: appended to their FIFO in ascending id (uniform)
    for (int i = 0; i < G.nsrc; i++) {
      const int4 r = reinterpret_cast<const int4 *>(G.srcq)[i];   // packed record
      const int q = D[rec_id(r)];
      const int f = S.dv[q].z;
      if (f < KF5) S.fc[q][f] = r;
      else fifo_g[S.doff[q] + f] = r;
      S.dv[q].z = f + 1;
    }
    unsigned att = (1u << d) - 1u;   // devices to dispatch at t = 0
    int cmin = INF, dmin = INF, dfr = INF;   // next-event operands (see "next instant")
    unsigned ce0 = 0, ce1 = 0;
    for (bool first = true;; first = false) {
      if (!first) {
        // ---------------------------------------------------------- next instant
        // both minima (and the channels at the heads' minimum) were taken before the previous
        // dispatch, which never touches the channel heads and only lowers the running finishes'
        // minimum; the running finishes are lane-held registers (lane k: device k)
        {
          const int tn = min(cmin, dmin);
          if (tn == INF) break;
          t = tn;
        }
        const unsigned e0 = cmin == t ? ce0 : 0u, e1 = cmin == t ? ce1 : 0u;
        unsigned ef = __ballot_sync(FULL, dfr == t);
        P5C(9);
        P5(0);
        // ---------------------------------------------------------- (1) copies arriving now
        for (unsigned m0 = e0, m1 = e1; m0 | m1;) {
          int c;
          if (m0) { c = 2 * (__ffs(m0) - 1); m0 &= m0 - 1; }
          else { c = 2 * (__ffs(m1) - 1) + 1; m1 &= m1 - 1; }
          const int4 cs = S.ch[c];
          const int h = cs.z, tail = cs.x, s = h & (KC5 - 1), q = cdst(c);
          const unsigned long long cb = 1ull << c;
          if (hpn & cb) {   // the head's record was fetched when it became the head (>= 1 instant ago)
            head_wait(&S.hbar[c], (unsigned)((hph >> c) & 1ull));
            hph ^= cb;
            hpn &= ~cb;
          }
          const int4 r = S.chd[c];   // the consumer's packed record
          const int e = S.cq[c][s].x;
          S.ch[c].z = h + 1;
          if (h + KC5 < tail) S.cq[c][s] = chq_g[cs.w + h + KC5];   // from the global overflow (rare)
          if (h + 1 < tail) {   // a new head: its arrival, and its record from the out-edge slot
            const int2 nx = S.cq[c][(h + 1) & (KC5 - 1)];
            S.ca[c] = nx.y;
            __syncwarp();   // every lane has read chd[c] before the copy overwrites it
            if (lane == 0) head_fetch(&S.chd[c], G.slots + nx.x, &S.hbar[c]);
            hpn |= cb;
          } else {
            S.ca[c] = INF;
          }
          item(IT_ALLOC_COPY, q, e);   // the memory warp reads the copy's bytes from slot e
          if (arrive_u(rec_cinfo(r))) to_inc(q, r);
        }
        P5(1);
        // ---------------------------------------------------------- (2) ops finishing now, ascending id
        att = ef;
        if (ef) P5C(10);
        while (ef) {
          int k = __ffs(ef) - 1;
          if (ef & (ef - 1)) {
            int best = S.drun[k].x;
            for (unsigned m = ef & (ef - 1); m; m &= m - 1) {
              const int k2 = __ffs(m) - 1, id2 = S.drun[k2].x;
              if (id2 < best) { best = id2; k = k2; }
            }
          }
          ef &= ~(1u << k);
          Q5 r;   // id, ob, nn (unpacked at the dispatch)
          {
            const int4 rr = S.drun[k];
            r.id = rr.x; r.ob = rr.y; r.nn = rr.z;
          }
          const int sl = S.dv2[k].x;
          S.dv[k].x = INF;
          if (lane == k) dfr = INF;
          const int nout = r.nn & 0xffff;
          // its frees, one item: the memory warp expands it into the in-edges (the copies this op
          // held, producers it was the last consumer of) and, for a sink, its own output
          item(IT_FIN, k, r.id);
          for (int j0 = 0; j0 < nout; j0 += 32) {   // out-edges, one per lane
            const int j = j0 + lane;
            const bool valid = j < nout;
            int4 e = make_int4(0, 0, 0, 0);   // the consumer's packed record
            int tw = k;
            unsigned sw = 0;
            if (valid) {
              if (j < SO5) {
                if (spend & (1u << (2 * k + sl))) { cp_wait0(); spend = 0; }
                e = S.stage[k][sl][j];
                sw = S.sdev[k][sl][j];
              } else {
                e = reinterpret_cast<const int4 *>(G.slots)[r.ob + j];
                sw = sdev_g[r.ob + j];
              }
              tw = (int)(sw & 7u);
            }
            const bool same = valid && tw == k, cross = valid && tw != k;
            const bool av = same && arrive5(flag_s, bigb_s, gbig, rec_cinfo(e));
            const unsigned am = __ballot_sync(FULL, av);
            const unsigned cm = __ballot_sync(FULL, cross);
            if (am) {   // ops made available now on device k, in lane (= id) order
              const int n0 = S.dv[k].w;
              if (av) {
                const int pos = n0 + __popc(am & lt);
                if (pos < NINC5) S.inc[k][pos] = e;
                else ov_g[S.doff[k] + pos] = e;
              }
              __syncwarp();
              S.dv[k].w = n0 + __popc(am);
              incm |= 1u << k;
            }
            if (cm) {   // FIFO pushes on the directed channels k -> tw, ranked within each channel
              const unsigned grp = (cm & (cm - 1)) ? __match_any_sync(FULL, cross ? tw : -1) : cm;
              if (cross) {
                const int rank = __popc(grp & lt), n = __popc(grp);
                const int c = cidx(k, tw);
                const int4 cs = S.ch[c];
                const int tail = cs.x, f = cs.y, hd = cs.z;
                const int x = (int)(sw >> 3);   // the transfer time k_cost5_pre computed
                const int bt = max(t, f);
                const int pos = tail + rank, arr = bt + (rank + 1) * x;
                const int2 ce = make_int2(r.ob + j, arr);
                if (pos < hd + KC5) S.cq[c][pos & (KC5 - 1)] = ce;
                else chq_g[cs.w + pos] = ce;
                if (pos == hd) S.chd[c] = e;   // an empty channel's new head
                if (rank == 0) {
                  *reinterpret_cast<int2 *>(&S.ch[c]) = make_int2(tail + n, bt + n * x);   // tail, free
                  if (tail == hd) S.ca[c] = bt + x;   // the channel was empty: a new head
                }
              }
            }
            __syncwarp();
          }
        }
        P5(2);
      }
      // the channel heads are final for the next instant: their minimum now, its latency hidden
      // behind the dispatch below
      {
        const int ca0 = lane < NCH / 2 ? S.ca[2 * lane] : INF, ca1 = lane < NCH / 2 ? S.ca[2 * lane + 1] : INF;
        cmin = (int)__reduce_min_sync(FULL, (unsigned)min(ca0, ca1));
        ce0 = __ballot_sync(FULL, ca0 == cmin);   // the channels whose head arrives at cmin
        ce1 = __ballot_sync(FULL, ca1 == cmin);
      }
      // the running finishes' minimum likewise; the dispatch below lowers it with each new finish
      // (recomputed every instant: skipping it on instants without a finish, where it cannot have
      // risen, measured 1 % slower -- the branch costs more than the REDUX)
      dmin = (int)__reduce_min_sync(FULL, (unsigned)dfr);
      // ---------------------------------------------------------- (3) FIFO append + dispatch
      for (att |= incm, incm = 0; att; att &= att - 1) {
        P5(3);
        P5C(11);
        const int k = __ffs(att) - 1;
        const int4 dvk = S.dv[k], dv2k = S.dv2[k];
        const int n = dvk.w;
        bool running = dvk.x != INF, go = false;
        int fh = dvk.y, ft = dvk.z;
        int4 run;   // packed record
        if (n > 0) {
          S.dv[k].w = 0;
          int4 *Li = &S.inc[k][0];
          int4 *Lo = ov_g + S.doff[k];
          if (n == 1 && !running && fh == ft) {   // common case: straight to dispatch
            run = Li[0];
            go = true;
          } else {
            for (int i = 1; i < n; i++) {   // insertion sort by id (n is small except after wide fan-outs)
              const int4 key = i < NINC5 ? Li[i] : Lo[i];
              int j = i - 1;
              while (j >= 0) {
                const int4 pj = j < NINC5 ? Li[j] : Lo[j];
                if ((pj.x & M25) <= (key.x & M25)) break;
                (j + 1 < NINC5 ? Li[j + 1] : Lo[j + 1]) = pj;
                j--;
              }
              (j + 1 < NINC5 ? Li[j + 1] : Lo[j + 1]) = key;
            }
            for (int i = 0; i < n; i++, ft++) {
              const int4 x = i < NINC5 ? Li[i] : Lo[i];
              if (ft < fh + KF5) S.fc[k][ft & (KF5 - 1)] = x;
              else fifo_g[S.doff[k] + ft] = x;
            }
            S.dv[k].z = ft;
          }
        }
        if (!go && !running && fh < ft) {   // pop the FIFO head
          const int s = fh & (KF5 - 1);
          run = S.fc[k][s];
          if (fh + KF5 < ft) S.fc[k][s] = fifo_g[S.doff[k] + fh + KF5];   // position fh + KF5 from the overflow (rare)
          S.dv[k].y = ++fh;
          go = true;
        }
        P5(4);
        int cur = dv2k.x, nxt = dv2k.y;
        if (go) {
          P5C(7);
          const int fin = t + run.y * dv2k.z;
          S.dv[k].x = fin;
          if (lane == k) dfr = fin;
          dmin = min(dmin, fin);
          S.drun[k] = make_int4(rec_id(run), rec_ob(run), run.w, 0);
          item(IT_ALLOC_OP, k, rec_id(run));
          cur ^= 1;   // the slot the head was staged into, or the one it is staged into now
          if (run.x != nxt && (run.w & 0xffff)) stage(k, cur, run);
          nxt = -1;
          running = true;
        }
        P5(5);
        if (running && fh < ft && nxt < 0) {   // stage the op now waiting at the head
          const int4 hr = S.fc[k][fh & (KF5 - 1)];
          nxt = hr.x;   // packed: compared with run.x
          if (hr.w & 0xffff) stage(k, cur ^ 1, hr);
        }
        *reinterpret_cast<int2 *>(&S.dv2[k]) = make_int2(cur, nxt);
        P5(6);
      }
      __syncwarp();
      P5(3);
    }
#ifdef COST5_PROF
    if (b == 0 && lane == 0)
      printf("C5PROF inst=%lld fin_inst=%lld ensure_waits=%lld next=%lld arr=%lld fin=%lld disp=%lld\n", prof[9],
             prof[10], prof[8], prof[0], prof[1], prof[2], prof[3]);
    if (b == 0 && lane == 0)
      printf("C5DISP iters=%lld go=%lld top+redux=%lld decide=%lld goblk=%lld look=%lld\n", prof[11], prof[7], prof[3],
             prof[4], prof[5], prof[6]);
#endif
    // ---------------------------------------------------------- end of the simulation
    item(IT_END, 0, 0);
#if COST5_MBAR
    if (lane == 0) mbar_arrive5(&S.ibar);   // the last (partial) batch
#endif
    cp_wait0();
    if (lane == 0) S.mk = t;
  } else {
    // ============================================================ memory warp
    const bool dl = lane < d;
    long long mem = dl ? pre->stat[lane] : 0, pk = mem;
    int last_t = -1, ndisp = 0;
    unsigned mh = 0;
    int nwait = 0;
    bool done = false;
    auto kind_end = [](unsigned long long x) { return ((unsigned)(x >> 33) & 7u) == (unsigned)IT_END; };
#ifdef COST5_PROF
    long long nidle = 0, nbatch = 0, nitems = 0, m0 = clock64();
#endif
    while (!done) {
      const unsigned pos = mh + lane;
      const unsigned long long it = *reinterpret_cast<volatile unsigned long long *>(&S.items[pos & (RI5 - 1)]);
      const unsigned code = (unsigned)(it >> 32);
      const bool valid = (code & 1u) == ((pos / RI5) & 1u);
      const unsigned vm = __ballot_sync(FULL, valid);
      const int n = vm == FULL ? 32 : __ffs(~vm) - 1;
#if COST5_MBAR
      if (n < 32 && !__any_sync(FULL, valid && kind_end(it))) {
        // sleep until the simulation warp completes the batch starting at mh (mh is a multiple
        // of 32 until the end): no polling instructions on the simulation warps' issue slots
        mbar_sleep5(&S.ibar, (mh >> 5) & 1u);
        continue;
      }
#endif
      if (n < MB5 && !__any_sync(FULL, valid && kind_end(it))) {
        // wait for a batch of MB5 items unless the simulation has ended: few, large batches
        // leave the issue slots to the simulation warps
        if (n == 0 || ++nwait < COST5_SPIN) {
#ifdef COST5_PROF
          nidle++;
#endif
          __nanosleep(COST5_SLEEP);
          continue;
        }
      }
      nwait = 0;
#ifdef COST5_NOMEM   // experiment: consume the items without the accounting (peaks wrong)
      done = __any_sync(FULL, lane < n && kind_end(it));
      mh += n;
      __syncwarp();
      if (lane == 0) asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&S.mhead)), "r"(mh) : "memory");
      continue;
#endif
#ifdef COST5_PROF
      nbatch++;
      nitems += n;
#endif
      const bool mine = lane < n;
      const int ti0 = (int)(unsigned)(it & 0xffffffffull);
      const int kind0 = (int)((code >> 1) & 7u), dev0 = (int)((code >> 4) & 7u), idx0 = (int)(code >> 7);
      ndisp += __popc(__ballot_sync(FULL, mine && kind0 == IT_ALLOC_OP));   // one item per dispatch
      // the batch expanded in order: an IT_FIN item becomes its op's in-edges (in-CSR order), every
      // other item stays one; processed 32 expanded items at a time
      int ib0 = 0, cnt = 0, sink = 0;
      if (mine) {
        if (kind0 == IT_FIN) {
          ib0 = G.in_ptr[idx0];
          sink = G.outdeg[idx0] == 0;
          cnt = G.in_ptr[idx0 + 1] - ib0 + sink;   // its in-edges, then (a sink) its output
        } else {
          cnt = 1;
        }
      }
      int iend = cnt;   // inclusive prefix sum: item i covers expanded positions [iend - cnt, iend)
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, iend, o);
        if (lane >= o) iend += y;
      }
      const int total = __shfl_sync(FULL, iend, 31);
      // per item, what an expanded position needs: kind | device << 3 | sink << 6, and for a
      // finish the in-edge index of position 0 (in-edge slot = base + position)
      const int code0 = kind0 | (dev0 << 3) | (sink << 6), base0 = ib0 - (iend - cnt);
      for (int w0 = 0; w0 < total; w0 += 32) {
        const int w = w0 + lane;
        int src = 0;   // the item covering position w: the number of items whose range ends at or before w
#pragma unroll
        for (int step = 16; step; step >>= 1) {
          const int e = __shfl_sync(FULL, iend, src + step - 1);
          if (e <= w) src += step;
        }
        const bool vmine = w < total;
        const int ti = __shfl_sync(FULL, ti0, src), code = __shfl_sync(FULL, code0, src);
        const int base = __shfl_sync(FULL, base0, src), idx_s = __shfl_sync(FULL, idx0, src);
        const int send = __shfl_sync(FULL, iend, src);
        const int kind_s = code & 7, dev = (code >> 3) & 7;
        const bool fsink = kind_s == IT_FIN && (code >> 6) && w == send - 1;   // the last position of a sink's FIN
        const int kind = kind_s == IT_FIN ? (fsink ? IT_SINK : IT_INEDGE) : kind_s;
        const int idx = kind_s == IT_FIN ? (fsink ? idx_s : base + w) : idx_s;
        int dA = -1, dB = -1, u = -1;
        long long xA = 0, xB = 0, bu = 0;
        int du = 0;
        if (vmine) {
          if (kind == IT_ALLOC_OP) { dA = dev; xA = G.out_bytes[idx]; }
          else if (kind == IT_ALLOC_COPY) { dA = dev; xA = G.ebytes[idx]; }   // idx = the copy's out-edge slot
          else if (kind == IT_SINK) { dA = dev; xA = -G.out_bytes[idx]; }
          else if (kind == IT_INEDGE) {
            const IRec ir = G.irec[idx];
            u = ir.u;
            bu = ir.bytes;
            du = D[u];
            if (du != dev) { dA = dev; xA = -bu; }   // the copy this op held
          } else {
            done = true;
          }
        }
        done = __any_sync(FULL, done);
        {  // producers whose last consumer finishes: one counter update per producer and round
          const unsigned grp = __match_any_sync(FULL, u);
          const int leader = __ffs(grp) - 1, last = 31 - __clz(grp), cnt2 = __popc(grp);
          int old = 0;
          if (u >= 0 && lane == leader) old = atomicSub(&outcnt[u], cnt2);
          old = __shfl_sync(FULL, old, leader);
          if (u >= 0 && lane == last && old == cnt2) { dB = du; xB = -bu; }
        }
        // apply in item order; sample the peak whenever the instant changes.  Each device lane
        // walks only its own contributions of the round, in item order, and samples its peak when
        // the instant changes between them: exact, since a device's bytes only change at its own
        // contributions (an instant boundary between two of them sees the value the earlier
        // sample already took).  Walking all 32 items on every lane instead (7 shuffles each)
        // measured 3.6 % slower on the whole kernel: the memory warps' issue slots and shuffles
        // compete with the simulation warps at sixteen placements per SM.
        // device masks from four ballots each (valid + the device's three bits)
        unsigned myA, myB;
        {
          const unsigned va = __ballot_sync(FULL, dA >= 0), a0 = __ballot_sync(FULL, dA & 1),
                         a1 = __ballot_sync(FULL, (dA >> 1) & 1), a2 = __ballot_sync(FULL, (dA >> 2) & 1);
          const unsigned vb = __ballot_sync(FULL, dB >= 0), b0 = __ballot_sync(FULL, dB & 1),
                         b1 = __ballot_sync(FULL, (dB >> 1) & 1), b2 = __ballot_sync(FULL, (dB >> 2) & 1);
          const unsigned s0 = (lane & 1) ? 0u : ~0u, s1 = (lane & 2) ? 0u : ~0u, s2 = (lane & 4) ? 0u : ~0u;
          myA = lane < 8 ? va & (a0 ^ s0) & (a1 ^ s1) & (a2 ^ s2) : 0u;
          myB = lane < 8 ? vb & (b0 ^ s0) & (b1 ^ s1) & (b2 ^ s2) : 0u;
        }
        unsigned my = myA | myB;
        const int iters = (int)__reduce_max_sync(FULL, (unsigned)__popc(my));
        for (int r2 = 0; r2 < iters; r2++) {
          const int i = my ? __ffs(my) - 1 : 0;
          const int tI = __shfl_sync(FULL, ti, i);
          if (B32) {   // every delta is one output's bytes, < 2^31: one 32-bit broadcast each
            const int aX = __shfl_sync(FULL, (int)xA, i), bX = __shfl_sync(FULL, (int)xB, i);
            if (my) {
              if (tI != last_t) { pk = max(pk, mem); last_t = tI; }
              mem += ((myA >> i) & 1u) ? aX : bX;   // an item's two deltas go to different devices
              my &= my - 1;
            }
          } else {
            const long long aX = __shfl_sync(FULL, xA, i), bX = __shfl_sync(FULL, xB, i);
            if (my) {
              if (tI != last_t) { pk = max(pk, mem); last_t = tI; }
              mem += (((myA >> i) & 1u) ? aX : 0ll) + (((myB >> i) & 1u) ? bX : 0ll);
              my &= my - 1;
            }
          }
        }
      }
      mh += n;
      __syncwarp();
      if (lane == 0) {
        asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&S.mhead)),
                     "r"(mh)
                     : "memory");
      }
    }
    pk = max(pk, mem);
    if (lane == 0) S.disp = ndisp;
#ifdef COST5_PROF
    if (b == 0 && lane == 0)
      printf("C5MEM batches=%lld items=%lld idle_polls=%lld cycles=%lld\n", nbatch, nitems, nidle, clock64() - m0);
#endif
    if (dl) {
      if (pk > T.cap[lane]) atomicOr(&S.oom, 1);
      if (peak_out) peak_out[(size_t)b * d + lane] = pk;
      if (busy_out) busy_out[(size_t)b * d + lane] = pre->busy[lane];
    }
  }
  __syncthreads();
  if (tid == 0) {
    gdp_sim_report R;
    R.makespan = S.mk; R.cross_bytes = pre->cross;
    for (int i = 0; i < 6; i++) R.pad[i] = 0;
#ifdef COST5_TIMING
    {
      unsigned long long t_end;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
      const unsigned us = (unsigned)((t_end - t_beg) / 1000ull);
      unsigned sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      R.pad[0] = us & 255u; R.pad[1] = (us >> 8) & 255u; R.pad[2] = (us >> 16) & 255u; R.pad[3] = us >> 24;
      R.pad[4] = (uint8_t)sm; R.pad[5] = (uint8_t)S.simw;
    }
#endif
    R.violation = (pflag & 1) ? 1 : (S.oom ? 2 : 0);
    if (S.disp != N) R.violation = 3;   // cannot happen for a validated DAG
    R.valid = R.violation == 0;
    rep[b] = R;
    reward[b] = R.valid ? -__dsqrt_rn(__ddiv_rn((double)S.mk, 1e6)) : -10.0;
  }
}

}  // namespace

size_t cost5_smem_bytes(int nflagw, int nbigb) { return 4 * (size_t)nflagw + 4 * (size_t)nbigb; }   // dynamic part
size_t cost5_scratch_per_placement(int N, long long E, int ngbig) { return scratch5_layout(N, E, ngbig).total; }

// every transfer takes >= 1 tick and every duration >= 1 (no same-instant rounds)
bool cost5_eligible(const TopoArgs &T, const Cost5Graph &G, int min_cost, long long min_edge_bytes) {
  const int d = T.d;
  if (!G.ok || d < 1 || d > 8 || min_cost < 1) return false;
  for (int k = 0; k < d; k++) {
    if (T.speed[k] < 1) return false;
    for (int q = 0; q < d; q++)
      if (k != q) {
        long long x = T.lat[k * 8 + q];
        if (min_edge_bytes > 0 && min_edge_bytes != LLONG_MAX && T.bpt[k * 8 + q] > 0)
          x += (min_edge_bytes - 1) / T.bpt[k * 8 + q] + 1;
        if (x < 1) return false;
      }
  }
  return sizeof(Smem5) + cost5_smem_bytes(G.nflagw, G.nbigb) <= 227 * 1024;
}

// placements that run at once: resident k_cost5 CTAs per SM x SMs (0 if not eligible)
int cost5_wave(const Cost5Graph &G) {
  const size_t smem = cost5_smem_bytes(G.nflagw, G.nbigb);
  if (sizeof(Smem5) + smem > 227 * 1024) return 0;
  const void *fn = G.bytes32 ? (const void *)k_cost5<true> : (const void *)k_cost5<false>;
  cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);   // all of it shared
  if (smem + sizeof(Smem5) > 48 * 1024)
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0, dev = 0, nsm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 64, smem) != cudaSuccess) return 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return occ * nsm;
}

bool launch_cost5(const Cost5Graph &G, const TopoArgs &T, int min_cost, long long min_edge_bytes, const uint8_t *D,
                  int B, unsigned char *scratch, size_t per_place, gdp_sim_report *rep, long long *peak,
                  long long *busy, double *reward, cudaStream_t s) {
  if (!cost5_eligible(T, G, min_cost, min_edge_bytes)) return false;
  if (per_place < cost5_scratch_per_placement(G.N, G.E, G.ngbig)) return false;
  const size_t smem = cost5_smem_bytes(G.nflagw, G.nbigb);
  static size_t configured[2] = {0, 0};
  static bool carve[2] = {false, false};
  const int b32 = G.bytes32 ? 1 : 0;
  const void *fn = b32 ? (const void *)k_cost5<true> : (const void *)k_cost5<false>;
  if (!carve[b32]) {
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);   // all of it shared
    carve[b32] = true;
  }
  if (smem + sizeof(Smem5) > 48 * 1024 && smem > configured[b32]) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured[b32] = smem;
  }
  // the pre-pass stages the placement row in shared memory when it fits (up to 160 KB)
  const int dsm = G.N <= 160 * 1024 ? (G.N + 15) / 16 * 16 : 0;
  static int pre_configured = 0;
  if (dsm > 48 * 1024 && dsm > pre_configured) {
    cudaFuncSetAttribute(k_cost5_pre, cudaFuncAttributeMaxDynamicSharedMemorySize, dsm);
    pre_configured = dsm;
  }
  note_launch("k_cost5_pre", s);
  k_cost5_pre<<<B, 512, dsm, s>>>(G, T, D, scratch, per_place, dsm);
  note_launch("k_cost5", s);
  if (b32) k_cost5<true><<<B, 64, smem, s>>>(G, T, D, scratch, per_place, rep, peak, busy, reward);
  else k_cost5<false><<<B, 64, smem, s>>>(G, T, D, scratch, per_place, rep, peak, busy, reward);
  return true;
}

// ------------------------------------------------------------------------ graph records (host)
gdp_status cost5_build(int N, long long E, const int *optr, const int *oidx, const int *iptr, const int *cost,
                       const long long *out_bytes, Cost5Host *h) {
  h->ok = N < (1 << 25) && E < (1LL << 25);
  h->slots.assign((size_t)std::max<long long>(E, 1), Slot5{});
  h->ebytes.assign((size_t)std::max<long long>(E, 1), 0);
  h->srcq.clear();
  h->bigb.clear();
  h->gbig.clear();
  h->outdeg.assign(N, 0);
  std::vector<Q5> q(N);
  int nb = 0, nf = 0;
  std::vector<unsigned char> nibs;
  std::vector<int> tri;   // three-input ops (COST5_TRI): 2-bit counts after the 4-bit ones
  for (int v = 0; v < N; v++) {
    const int din = iptr[v + 1] - iptr[v], dout = optr[v + 1] - optr[v];
    if (din >= 65536 || dout >= 65536) h->ok = false;
    Q5 &r = q[v];
    r.id = v; r.cost = cost[v]; r.ob = optr[v]; r.ib = iptr[v]; r.arr = 0; r.u = 0;
    r.nn = (dout & 0xffff) | ((din & 0xffff) << 16);
    if (din <= 1) r.cinfo = 0;
    else if (din == 2) r.cinfo = 1 | (nf++ << 2);
    else if (COST5_TRI && din == 3) { r.cinfo = 0; tri.push_back(v); }   // encoded below
    else if (din <= 15) { r.cinfo = 2 | (nb << 2); nibs.push_back((unsigned char)din); nb++; }
    else { r.cinfo = 3 | ((int)h->gbig.size() << 2); h->gbig.push_back(din); }
    if (din == 0) h->srcq.push_back(pack_slot5(r.id, r.cost, r.ob, dout, r.cinfo));
    h->outdeg[v] = dout;
  }
  while (nibs.size() % 32) nibs.push_back(0);
  const int nibw = (int)(nibs.size() / 8);
  for (size_t i = 0; i < tri.size(); i++)   // kind 0 with index 1 + (2-bit field position in the counter words)
    q[tri[i]].cinfo = (int)((1 + (size_t)nibw * 16 + i) << 2);
  for (int v = 0; v < N; v++)
    for (int e = optr[v]; e < optr[v + 1]; e++) {
      const Q5 &w = q[oidx[e]];
      h->slots[(size_t)e] = pack_slot5(w.id, w.cost, w.ob, w.nn & 0xffff, w.cinfo);
      h->ebytes[(size_t)e] = out_bytes[v];   // the producer's output: the size of the copy on this edge
    }
  h->nflagw = (nf + 31) / 32;
  h->bytes32 = true;
  for (int v = 0; v < N; v++)
    if (out_bytes[v] >= (1LL << 31)) h->bytes32 = false;
  h->bigb.assign((size_t)nibw + (tri.size() + 15) / 16, 0xffffffffu);   // 2-bit fields start at 3
  for (int i = 0; i < nibw; i++) h->bigb[(size_t)i] = 0u;
  for (size_t i = 0; i < nibs.size(); i++) h->bigb[i / 8] |= (unsigned)nibs[i] << (4 * (i % 8));
  return GDP_OK;
}

}  // namespace gdp
