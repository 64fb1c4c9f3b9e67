// Device helpers shared by the shared-memory cost kernels (cost2.cu, cost5.cu).
#pragma once
#include <climits>

#include "common.cuh"
#include "cost2.cuh"

namespace gdp {
namespace cu {

constexpr int INF = INT_MAX;

struct __align__(16) Ent {   // FIFO entry (t = ready) / channel entry (t = arrival, bytes = copy size)
  NRec r;
  int t, pad;
  long long bytes;
};

__device__ __forceinline__ void cp16(void *s, const void *g) {
  unsigned a = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(a), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_ent(Ent *s, const Ent *g) {
  cp16(reinterpret_cast<int4 *>(s), g);
  cp16(reinterpret_cast<int4 *>(s) + 1, reinterpret_cast<const int4 *>(g) + 1);
  cp16(reinterpret_cast<int4 *>(s) + 2, reinterpret_cast<const int4 *>(g) + 2);
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

__device__ __forceinline__ void copy_rec(NRec *dst, const NRec *src) {
  const int4 *s = reinterpret_cast<const int4 *>(src);
  int4 *d = reinterpret_cast<int4 *>(dst);
  d[0] = s[0];
  d[1] = s[1];
}
__device__ __forceinline__ void store_ent(Ent *dst, const NRec &r, int t, long long bytes) {
  int4 *d = reinterpret_cast<int4 *>(dst);
  const int4 *s = reinterpret_cast<const int4 *>(&r);
  d[0] = s[0];
  d[1] = s[1];
  d[2] = make_int4(t, 0, (int)(bytes & 0xffffffffLL), (int)(bytes >> 32));
}
__device__ __forceinline__ void load_rec(NRec &r, const NRec *src) {
  const int4 *s = reinterpret_cast<const int4 *>(src);
  int4 a = s[0], b = s[1];
  r.id = a.x; r.cost = a.y; r.ob = a.z; r.oe = a.w; r.ib = b.x; r.ie = b.y;
  r.bytes = ((long long)(unsigned)b.z) | ((long long)b.w << 32);
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ int dev_of(const unsigned *Dn, int v) { return (Dn[v >> 3] >> ((v & 7) * 4)) & 15; }

// ceil(bytes / bw) + lat with one fp64 multiply by the reciprocal and an exact integer fix-up
__device__ __forceinline__ int xfer_time3(long long bytes, int c, const TopoArgs &T) {
  const long long bw = T.bpt[c];
  long long q = (long long)((double)bytes * T.inv_bpt[c]);
  long long r = bytes - q * bw;
  while (r < 0) { q--; r += bw; }
  while (r >= bw) { q++; r -= bw; }
  return (int)(q + (r > 0)) + T.lat[c];
}
}  // namespace cu
}  // namespace gdp
