// Records and launchers of the shared-memory cost kernels (k_cost5 in cost5.cu, k_cost3 in cost2.cu).
#pragma once
#include <vector>

#include "common.cuh"

namespace gdp {

struct __align__(16) NRec {   // one op: what dispatch / finish need, 32 bytes
  int id, cost, ob, oe;       // id, compute cost, out-CSR range [ob, oe)
  int ib, ie;                 // in-CSR range [ib, ie)
  long long bytes;            // output bytes
};
struct __align__(16) IRec {   // one in-edge: producer and its output bytes
  int u, pad;
  long long bytes;
};

struct Cost2Graph {
  int N;
  long long E;
  const NRec *nrec;            // N, graph-static
  const NRec *erec;            // E, out-CSR order: erec[e] = nrec[out_idx[e]]
  const IRec *irec;            // E, in-CSR order
  const unsigned *cnt0;        // ceil(N/4) words: per op byte = min(indeg,15) | min(outdeg,15) << 4
  const int *bigid;            // N: index into big_in / big_out for degree >= 15, else -1
  const int *big_in, *big_out;
  int nbig;
  const int *out_idx, *out_src, *in_ptr, *cost, *leader;
  const long long *out_bytes, *mem_bytes;
  int has_coloc;
};

// ---- k_cost5 (cost5.cu): graph-static records of the simulation warp
struct __align__(16) Q5 {     // an op in a queue (channel ring, FIFO, available list), 32 bytes
  int id, cost, ob, nn;       // id, compute cost, first out-edge slot, out-degree | in-degree << 16
  int cinfo;                  // input counter: kind (bits 0-1: 0 = at most one input, 1 = two inputs
                              // (flag bit), 2 = 4-bit counter (3..15 inputs), 3 = global counter) | index << 2
  int ib;                     // first in-edge slot
  int arr, u;                 // channel entries: arrival tick and producer id
};
// The 16-byte queue record of an op (the consumer w of an out-edge slot e = (v -> w), out-CSR
// order; a source; a FIFO / available / channel-head entry): its id, compute cost, first out-edge
// slot, out-degree and input-counter info (kind + index, 27 bits) packed into the spare high bits
// (N, E < 2^25, degrees < 2^16):
//   x = id | ix[18:25) << 25      y = cost
//   z = ob | kind << 25 | ix[16:18) << 27      w = out-degree | ix[0:16) << 16
// where cinfo = kind | ix << 2 (kind 0: at most one input, 1: two inputs (flag bit), 2: 4-bit
// counter (3..15 inputs), 3: global counter).  The copy's bytes are in ebytes (per slot).
struct __align__(16) Slot5 {
  int x, cost, z, w;
};
__host__ __device__ __forceinline__ Slot5 pack_slot5(int id, int cost, int ob, int nout, int cinfo) {
  const unsigned kind = (unsigned)cinfo & 3u, ix = (unsigned)cinfo >> 2;
  Slot5 s;
  s.x = (int)((unsigned)id | ((ix >> 18) << 25));
  s.cost = cost;
  s.z = (int)((unsigned)ob | (kind << 25) | (((ix >> 16) & 3u) << 27));
  s.w = (int)(((unsigned)nout & 0xffffu) | ((ix & 0xffffu) << 16));
  return s;
}
struct Cost5Host {            // host images built at graph creation (cost5_build)
  bool ok = false;
  bool bytes32 = false;        // every output < 2^31 bytes: the memory warp applies 32-bit deltas
  std::vector<Slot5> slots;
  std::vector<long long> ebytes;   // per out-edge slot: the producer's output bytes (k_cost5_pre, contiguous)
  std::vector<Slot5> srcq;     // the sources, ascending id
  std::vector<int> gbig, outdeg;
  std::vector<unsigned> bigb;  // 4-bit counters (in-degree 3..15), 8 per word, 16-byte padded
  int nflagw = 0;              // words of the two-input flag bitmap
};
struct Cost5Graph {
  int N;
  long long E;
  int ok;
  const Slot5 *slots;
  const long long *ebytes;
  const Slot5 *srcq;
  const IRec *irec;
  const int *out_idx, *out_src, *cost, *leader, *outdeg, *gbig0;
  const int *in_ptr;   // N + 1: in-CSR offsets (the memory warp expands a finish into its in-edges)
  const unsigned *bigb0;
  const long long *out_bytes, *mem_bytes;
  int nsrc, nbigb, ngbig, nflagw, has_coloc;
  int bytes32;                 // Cost5Host::bytes32
};
gdp_status cost5_build(int N, long long E, const int *optr, const int *oidx, const int *iptr, const int *cost,
                       const long long *out_bytes, Cost5Host *h);
size_t cost5_smem_bytes(int nflagw, int nbigb);
size_t cost5_scratch_per_placement(int N, long long E, int ngbig);
int cost5_wave(const Cost5Graph &G);
bool cost5_eligible(const TopoArgs &T, const Cost5Graph &G, int min_cost, long long min_edge_bytes);
bool launch_cost5(const Cost5Graph &G, const TopoArgs &T, int min_cost, long long min_edge_bytes, const uint8_t *D,
                  int B, unsigned char *scratch, size_t per_place, gdp_sim_report *rep, long long *peak,
                  long long *busy, double *reward, cudaStream_t s);

size_t cost2_smem_bytes(int N);
size_t cost2_scratch_per_placement(int N, long long E, int nbig);
bool launch_cost2(const Cost2Graph &G, const TopoArgs &T, const uint8_t *D, int B, unsigned char *scratch,
                  size_t per_place, gdp_sim_report *rep, long long *peak, long long *busy, double *reward,
                  cudaStream_t s);

}  // namespace gdp
