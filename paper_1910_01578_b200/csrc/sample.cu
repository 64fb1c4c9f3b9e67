// D ~ pi_theta(G) (§3) and the policy-gradient seed
// dL/dlogits (P:93 PPO, Eq. 1).
//  * k_node_prep: per node, the fp32 softmax CDF and log-probabilities of its d logits.
//  * k_sample:    one CTA per placement; each thread draws 4 nodes from one Philox4x32-10
//                 call (counter (v>>2, gidx, step, gidx>>32), key = seed) by inverse CDF,
//                 log pi_b summed over co-location leaders in fp64 (fixed-order block reduce).
//  * k_logit_grad: thread per node: dL/dz_vk = -s sum_b w_b ([D_bv = k] - p_vk) [v leader]
//                 + (beta/N) p_vk (log p_vk + H_v), with w_b = A_b rho_b [unclipped].
#include "common.cuh"

namespace gdp {
namespace {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; r++) {
    unsigned hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    unsigned hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

// logits rows have stride ld >= d: a head padded to ld devices of which the first d are active
// (mixed device counts); cdf / logp are stored with stride d
__global__ void k_node_prep(const float *logits, int ld, int N, int d, float *cdf, float *logp, int *lastpos) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= N) return;
  const float *z = logits + (size_t)v * ld;
  float mx = z[0];
  for (int k = 1; k < d; k++) mx = fmaxf(mx, z[k]);
  float e[kMaxD], s = 0.f;
  for (int k = 0; k < d; k++) {
    e[k] = expf(z[k] - mx);
    s += e[k];
  }
  float ls = logf(s), c = 0.f;
  int last = 0;
  for (int k = 0; k < d; k++) {
    float p = e[k] / s;
    c += p;
    cdf[(size_t)v * d + k] = c;
    logp[(size_t)v * d + k] = (z[k] - mx) - ls;
    if (p > 0.f) last = k;
  }
  lastpos[v] = last;
}

constexpr int ST = 256;
__global__ void __launch_bounds__(ST) k_sample(const float *__restrict__ cdf, const float *__restrict__ logp,
                                               const int *__restrict__ lastpos, const int *__restrict__ leader,
                                               int N, int d, uint64_t seed, uint64_t offset, uint64_t step_val,
                                               const uint64_t *step_ptr, uint8_t *D, float *logprob) {
  const uint64_t step = step_ptr ? *step_ptr : step_val;   // device counter: graph replays advance it
  __shared__ double red[ST / 32];
  const int b = blockIdx.x;
  const uint64_t gidx = offset + (uint64_t)b;
  const uint2 key = make_uint2((unsigned)(seed & 0xffffffffu), (unsigned)(seed >> 32));
  double acc = 0.0;
  const int nq = (N + 3) >> 2;
  uint8_t *Db = D + (size_t)b * N;
  for (int q = threadIdx.x; q < nq; q += ST) {
    uint4 w = philox4x32_10(make_uint4((unsigned)q, (unsigned)(gidx & 0xffffffffu), (unsigned)(step & 0xffffffffu),
                                       (unsigned)(gidx >> 32)),
                            key);
    unsigned ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int j = 0; j < 4; j++) {
      int v = 4 * q + j;
      if (v >= N) break;
      float u = (float)(ws[j] >> 8) * 5.9604644775390625e-08f;  // 2^-24
      const float *cv = cdf + (size_t)v * d;
      int k = -1;
      for (int t = 0; t < d; t++)
        if (u < cv[t]) { k = t; break; }
      if (k < 0) k = lastpos[v];
      Db[v] = (uint8_t)k;
      if (leader[v] == v) acc += (double)logp[(size_t)v * d + k];
    }
  }
  // fixed-order block reduction
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < ST / 32; i++) s += red[i];
    logprob[b] = (float)s;
  }
}

__global__ void k_colocate(const int *leader, int N, int B, uint8_t *D) {
  size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)N * B) return;
  int v = (int)(e % N);
  size_t b = e / N;
  int l = leader[v];
  if (l != v) D[b * N + v] = D[b * N + l];
}

// w_b = A_b rho_b if the min() of the clipped surrogate picks the unclipped branch, else 0
__global__ void k_weights(const double *adv, const float *logprob, const float *old_logprob, float eps, int B,
                          double *wb) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  double A = adv[b];
  double rho = old_logprob ? exp((double)logprob[b] - (double)old_logprob[b]) : 1.0;
  double lo = 1.0 - (double)eps, hi = 1.0 + (double)eps;
  double cl = rho < lo ? lo : (rho > hi ? hi : rho);
  wb[b] = (rho * A <= cl * A) ? rho * A : 0.0;
}

__global__ void k_logit_grad(const float *__restrict__ logits, int ld, const uint8_t *__restrict__ D,
                             const int *__restrict__ leader, const double *__restrict__ wb, float beta, float scale,
                             int N, int d, int B, float *dlog) {
  extern __shared__ double swb[];
  for (int b = threadIdx.x; b < B; b += blockDim.x) swb[b] = wb[b];
  __syncthreads();
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= N) return;
  const float *z = logits + (size_t)v * ld;
  float mx = z[0];
  for (int k = 1; k < d; k++) mx = fmaxf(mx, z[k]);
  float e[kMaxD], s = 0.f;
  for (int k = 0; k < d; k++) {
    e[k] = expf(z[k] - mx);
    s += e[k];
  }
  float ls = logf(s);
  double acc[kMaxD];
  for (int k = 0; k < kMaxD; k++) acc[k] = 0.0;
  double sw = 0.0;
  const bool lead = leader[v] == v;
  if (lead) {
    for (int b = 0; b < B; b++) {
      int k = D[(size_t)b * N + v];
      double w = swb[b];
      sw += w;
#pragma unroll
      for (int t = 0; t < kMaxD; t++)
        if (t == k) acc[t] += w;
    }
  }
  float p[kMaxD], lp[kMaxD], Hv = 0.f;
  for (int k = 0; k < d; k++) {
    p[k] = e[k] / s;
    lp[k] = (z[k] - mx) - ls;
    Hv -= p[k] * lp[k];
  }
  const float bn = beta / (float)N;
  for (int k = 0; k < d; k++) {
    float g = (float)(-(double)scale * (acc[k] - (double)p[k] * sw));
    g += bn * p[k] * (lp[k] + Hv);
    dlog[(size_t)v * ld + k] = g;
  }
  for (int k = d; k < ld; k++) dlog[(size_t)v * ld + k] = 0.f;   // masked head columns
}

}  // namespace

void launch_sample(const float *logits, int ld, const int *leader, bool has_coloc, int N, int d, int B, uint64_t seed,
                   uint64_t offset, uint64_t step, const uint64_t *step_ptr, float *cdf, float *logp, int *lastpos,
                   uint8_t *D, float *logprob, cudaStream_t s) {
  note_launch("k_node_prep", s);
  k_node_prep<<<(N + 255) / 256, 256, 0, s>>>(logits, ld, N, d, cdf, logp, lastpos);
  note_launch("k_sample", s, (double)B * N + 4.0 * (double)N * (2 * d + 1));
  k_sample<<<B, ST, 0, s>>>(cdf, logp, lastpos, leader, N, d, seed, offset, step, step_ptr, D, logprob);
  if (has_coloc) {
    size_t n = (size_t)N * B;
    note_launch("k_colocate", s);
    k_colocate<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(leader, N, B, D);
  }
}

void launch_node_prep(const float *logits, int ld, int N, int d, float *cdf, float *logp, int *lastpos,
                      cudaStream_t s) {
  note_launch("k_node_prep", s);
  k_node_prep<<<(N + 255) / 256, 256, 0, s>>>(logits, ld, N, d, cdf, logp, lastpos);
}

void launch_logit_grad(const float *logits, int ld, const uint8_t *D, const int *leader, const double *adv,
                       const float *logprob, const float *old_logprob, float eps, float beta, float scale,
                       int N, int d, int B, double *wb, float *dlog, cudaStream_t s) {
  note_launch("k_weights", s);
  k_weights<<<(B + 255) / 256, 256, 0, s>>>(adv, logprob, old_logprob, eps, B, wb);
  size_t smem = (size_t)B * sizeof(double);
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_logit_grad, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  note_launch("k_logit_grad", s, (double)B * N + 4.0 * 2 * (double)N * d);
  k_logit_grad<<<(N + 127) / 128, 128, smem, s>>>(logits, ld, D, leader, wb, beta, scale, N, d, B, dlog);
}

}  // namespace gdp
