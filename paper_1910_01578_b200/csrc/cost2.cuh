// Records and launcher of the shared-memory cost model (cost2.cu).
#pragma once
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

size_t cost2_smem_bytes(int N);
size_t cost2_scratch_per_placement(int N, long long E, int nbig);
size_t cost4_smem_bytes(int N);
int cost4_window(const TopoArgs &T, int min_cost, int N, long long min_edge_bytes);   // window length, 0 = not eligible
size_t cost4_scratch_per_placement(int N, long long E, int nbig);
bool launch_cost4(const Cost2Graph &G, const TopoArgs &T, int min_cost, long long min_edge_bytes, const uint8_t *D, int B,
                  unsigned char *scratch, size_t per_place, gdp_sim_report *rep, long long *peak, long long *busy,
                  double *reward, cudaStream_t s);
bool launch_cost2(const Cost2Graph &G, const TopoArgs &T, const uint8_t *D, int B, unsigned char *scratch,
                  size_t per_place, gdp_sim_report *rep, long long *peak, long long *busy, double *reward,
                  cudaStream_t s);

}  // namespace gdp
