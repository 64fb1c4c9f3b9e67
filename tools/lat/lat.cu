// latency microbenchmark of warp-level primitives on sm_100a (one warp)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(long long *out, int *g, int seed) {
  __shared__ unsigned s[1024];
  const int lane = threadIdx.x;
  for (int i = lane; i < 1024; i += 32) s[i] = i * seed;
  __syncwarp();
  unsigned v = lane + seed, acc = 0;
  const int R = 256;
  long long t0, t1;
#define MEASURE(idx, body) \
  t0 = clock64(); for (int r = 0; r < R; r++) { body; } t1 = clock64(); if (lane == 0) out[idx] = (t1 - t0) / R;
  MEASURE(0, v = s[v & 1023])                                   // dependent LDS
  MEASURE(1, v = atomicAdd(&s[v & 1023], 1u) & 1023)            // dependent ATOMS with return
  MEASURE(2, v = __reduce_min_sync(0xffffffffu, v) + lane)      // REDUX
  MEASURE(3, v = __shfl_sync(0xffffffffu, v, (v + 1) & 31))     // SHFL dependent
  MEASURE(4, v = __match_any_sync(0xffffffffu, v & 7) + v)      // MATCH.ANY
  MEASURE(5, v = __ballot_sync(0xffffffffu, v & 1) + v)         // VOTE ballot
  MEASURE(6, v = (unsigned)__any_sync(0xffffffffu, v & 1) + v + 1)  // VOTE any
  MEASURE(7, __syncwarp(); v = v * 3 + 1)                      // syncwarp + IMAD
  MEASURE(8, v = v * 3 + 1)                                     // dependent IMAD
  MEASURE(9, atomicAdd(&s[(v + r) & 1023], 1u); v = v * 3 + 1)  // RED (no return) + IMAD
  MEASURE(10, v = (unsigned)(long long)((double)v * 1.0000001))   // fp64 mul chain w/ conversions
  MEASURE(11, { long long q = (long long)ceil(__ddiv_rn((double)(v + 1000), 37.0)); v = (unsigned)q; })
  MEASURE(12, v = g[v & 1023])                                  // dependent global load (L1/L2)
  MEASURE(13, if (v & 1) { v = v * 5 + 3; } else { v = v * 7 + 1; })  // branchy
  if (lane == 0) out[14] = v + acc;
}
int main() {
  long long *o; int *g;
  cudaMalloc(&o, 16 * 8); cudaMalloc(&g, 4096 * 4); cudaMemset(g, 0, 4096 * 4);
  k<<<1, 32>>>(o, g, 3);
  long long h[16];
  cudaMemcpy(h, o, 16 * 8, cudaMemcpyDeviceToHost);
  const char *names[] = {"LDS dep", "ATOMS ret dep", "REDUX min", "SHFL dep", "MATCH.ANY", "ballot", "any",
                         "syncwarp+IMAD", "IMAD dep", "RED+IMAD", "fp64 mul+cvt", "ddiv ceil", "LDG dep", "branchy"};
  for (int i = 0; i < 14; i++) printf("%-16s %lld cycles\n", names[i], h[i]);
  return 0;
}
