// Which SM sub-partition (warp slot % 4) do the warps of small CTAs land on?
// nvcc -gencode arch=compute_100a,code=sm_100a -o smsp smsp.cu && ./smsp
#include <cstdio>
#include <vector>
__global__ void k(int *out, int threads) {
  unsigned w, sm;
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(w));
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  long long t0 = clock64();
  while (clock64() - t0 < 20000000) {}
  if ((threadIdx.x & 31) == 0) {
    int i = blockIdx.x * (threads / 32) + threadIdx.x / 32;
    out[2 * i] = w;
    out[2 * i + 1] = sm;
  }
}
int main() {
  for (int threads : {64, 128, 256}) {
    for (int per_sm : {2, 4, 8, 9}) {
      int B = 148 * per_sm * 64 / threads, nw = B * threads / 32;
      int *d;
      cudaMalloc(&d, nw * 2 * sizeof(int));
      k<<<B, threads>>>(d, threads);
      std::vector<int> h(nw * 2);
      cudaMemcpy(h.data(), d, nw * 2 * sizeof(int), cudaMemcpyDeviceToHost);
      int cnt[8][4] = {};
      for (int i = 0; i < nw; i++) cnt[i % (threads / 32) < 8 ? i % (threads / 32) : 7][h[2 * i] % 4]++;
      printf("threads=%d CTAs/SM(64-thread equiv)=%d: ", threads, per_sm);
      for (int j = 0; j < threads / 32 && j < 8; j++) printf("warp%d->[%d %d %d %d] ", j, cnt[j][0], cnt[j][1], cnt[j][2], cnt[j][3]);
      printf("\n");
      cudaFree(d);
    }
  }
}
