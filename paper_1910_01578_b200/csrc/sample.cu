// D ~ pi_theta(G) (§3) and the policy-gradient seed
// dL/dlogits (P:93 PPO, Eq. 1).
//  * k_node_prep: per node, the fp32 softmax CDF and log-probabilities of its d logits.
//  * k_sample:    one CTA per placement; each thread draws 4 nodes from one Philox4x32-10
//                 call (counter (v>>2, gidx, step, gidx>>32), key = seed) by inverse CDF,
//                 log pi_b summed over co-location leaders in fp64 (fixed-order block reduce).
//  * k_logit_grad: thread per node: dL/dz_vk = -s sum_b w_b ([D_bv = k] - p_vk) [v leader]
//                 + (beta/N) p_vk (log p_vk + H_v), with w_b = A_b rho_b [unclipped].
#include "common.cuh"
#include "philox.cuh"

namespace gdp {
namespace {

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
  float ls = logf(s), is = 1.f / s, c = 0.f;   // p = e / s as e * (1 / s), like the AR decode (ar.cu)
  int last = 0;
  for (int k = 0; k < d; k++) {
    float p = e[k] * is;
    c += p;
    cdf[(size_t)v * d + k] = c;
    logp[(size_t)v * d + k] = (z[k] - mx) - ls;
    if (p > 0.f) last = k;
  }
  lastpos[v] = last;
}

// a11.  Grid = (node chunks of 4 x 256 nodes, groups of SBG placements): a thread owns 4
// consecutive nodes, keeps their CDF, log-probabilities and fallbacks in registers (read once, not
// once per placement), and for each placement of its group draws its 4 uniforms from one
// Philox4x32-10 call (counter (v>>2, gidx, step, gidx>>32), key = seed).  The inverse CDF is the
// count of CDF entries <= u (the CDF is non-decreasing, so that count is the first k with
// u < c_k; d -> the last k with p_k > 0).  The 4 device bytes leave as one 32-bit store (rows
// 4-byte aligned) or 4 byte stores.  log pi_b: a fixed-order warp reduction per 128 nodes into
// part[b][warp chunk], then k_sample_lp sums the warp chunks in order (deterministic).
constexpr int ST = 256;
constexpr int SBG = 16;
__global__ void __launch_bounds__(ST) k_sample(const float *__restrict__ cdf, const float *__restrict__ logp,
                                               const int *__restrict__ lastpos, const int *__restrict__ leader,
                                               int has_coloc, int N, int d, int B, uint64_t seed, uint64_t offset,
                                               uint64_t step_val, const uint64_t *step_ptr, uint8_t *D,
                                               double *part, int nwc) {
  const uint64_t step = step_ptr ? *step_ptr : step_val;   // device counter: graph replays advance it
  const uint2 key = make_uint2((unsigned)(seed & 0xffffffffu), (unsigned)(seed >> 32));
  const int q = blockIdx.x * ST + threadIdx.x, lane = threadIdx.x & 31;
  const int wc = q >> 5;                                   // warp chunk (128 nodes)
  float c[4][kMaxD], lp[4][kMaxD];
  int last[4];
  bool lead[4];
#pragma unroll
  for (int j = 0; j < 4; j++) {
    const int v = 4 * q + j;
    const bool ok = v < N;
#pragma unroll
    for (int t = 0; t < kMaxD; t++) {
      c[j][t] = (ok && t < d) ? __ldg(cdf + (size_t)v * d + t) : __int_as_float(0x7f800000);
      lp[j][t] = (ok && t < d) ? __ldg(logp + (size_t)v * d + t) : 0.f;
    }
    last[j] = ok ? __ldg(lastpos + v) : 0;
    lead[j] = ok && (!has_coloc || __ldg(leader + v) == v);
  }
  const bool any = 4 * q < N;
  const bool aligned = ((N & 3) == 0) && 4 * q + 3 < N;
  const int b1 = min(B, (int)(blockIdx.y + 1) * SBG);
  for (int b = blockIdx.y * SBG; b < b1; b++) {
    const uint64_t gidx = offset + (uint64_t)b;
    double acc = 0.0;
    if (any) {
      const uint4 w = philox4x32_10(make_uint4((unsigned)q, (unsigned)(gidx & 0xffffffffu),
                                               (unsigned)(step & 0xffffffffu), (unsigned)(gidx >> 32)),
                                    key);
      const unsigned ws[4] = {w.x, w.y, w.z, w.w};
      unsigned packed = 0;
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const float u = (float)(ws[j] >> 8) * 5.9604644775390625e-08f;  // 2^-24
        int k = 0;
#pragma unroll
        for (int t = 0; t < kMaxD; t++) k += (c[j][t] <= u);
        if (k >= d) k = last[j];
        float l = 0.f;
#pragma unroll
        for (int t = 0; t < kMaxD; t++) l = (t == k) ? lp[j][t] : l;
        if (lead[j]) acc += (double)l;
        packed |= (unsigned)k << (8 * j);
      }
      uint8_t *Db = D + (size_t)b * N;
      if (aligned) *reinterpret_cast<unsigned *>(Db + 4 * q) = packed;
      else
        for (int j = 0; j < 4 && 4 * q + j < N; j++) Db[4 * q + j] = (uint8_t)(packed >> (8 * j));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0 && wc < nwc) part[(size_t)b * nwc + wc] = acc;
  }
}

// log pi_b = sum of the warp chunks' partial sums in chunk order
__global__ void k_sample_lp(const double *__restrict__ part, int nwc, int B, float *logprob) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  double s = 0.0;
  for (int i = 0; i < nwc; i++) s += part[(size_t)b * nwc + i];
  logprob[b] = (float)s;
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

// a14, part 1: per (node, device) the fp64 sum over one chunk of placements of w_b [D_bv = k];
// a thread covers 4 consecutive nodes (one 32-bit load of their device bytes per placement when
// the rows are 4-byte aligned); chunk c of the placements -> part[c][v][k] (fixed order later)
constexpr int LG_T = 128;
__global__ void __launch_bounds__(LG_T) k_logit_acc(const uint8_t *__restrict__ D, const double *__restrict__ wb,
                                                     int N, int d, int B, int b_per, double *part) {
  const int q = blockIdx.x * LG_T + threadIdx.x;
  const int v0 = 4 * q;
  const int c = blockIdx.y, b0 = c * b_per, b1 = min(B, b0 + b_per);
  double acc[4][kMaxD];
#pragma unroll
  for (int j = 0; j < 4; j++)
#pragma unroll
    for (int k = 0; k < kMaxD; k++) acc[j][k] = 0.0;
  if (v0 < N) {
    const bool aligned = ((N & 3) == 0) && v0 + 3 < N;
    for (int b = b0; b < b1; b++) {
      const double w = __ldg(wb + b);
      unsigned x;
      if (aligned) x = __ldg(reinterpret_cast<const unsigned *>(D + (size_t)b * N + v0));
      else {
        x = 0;
        for (int j = 0; j < 4 && v0 + j < N; j++) x |= (unsigned)D[(size_t)b * N + v0 + j] << (8 * j);
      }
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const unsigned k = (x >> (8 * j)) & 0xffu;
#pragma unroll
        for (int t = 0; t < kMaxD; t++) acc[j][t] += (t == (int)k) ? w : 0.0;
      }
    }
  }
  for (int j = 0; j < 4; j++) {
    const int v = v0 + j;
    if (v >= N) break;
#pragma unroll
    for (int t = 0; t < kMaxD; t++)
      if (t < d) part[((size_t)c * N + v) * d + t] = acc[j][t];
  }
}

// a14, part 2: dL/dz_vk = -s (sum_b w_b [D_bv = k] - p_vk sum_b w_b) [v leader] + (beta/N) p_vk
// (log p_vk + H_v); the chunk partials summed in chunk order (deterministic)
__global__ void k_logit_fin(const float *__restrict__ logits, int ld, const int *__restrict__ leader,
                            const double *__restrict__ wb, const double *__restrict__ part, int nchunks, float beta,
                            float scale, int N, int d, int B, float *dlog) {
  __shared__ double s_sw;
  if (threadIdx.x == 0) {
    double sw = 0.0;
    for (int b = 0; b < B; b++) sw += wb[b];
    s_sw = sw;
  }
  __syncthreads();
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= N) return;
  const float *z = logits + (size_t)v * ld;
  float mx = z[0];
  for (int k = 1; k < d; k++) mx = fmaxf(mx, z[k]);
  float e[kMaxD], s = 0.f;
  for (int k = 0; k < d; k++) {
    e[k] = expf(z[k] - mx);
    s += e[k];
  }
  const float ls = logf(s);
  const bool lead = leader[v] == v;
  const double sw = lead ? s_sw : 0.0;
  float p[kMaxD], lp[kMaxD], Hv = 0.f;
  for (int k = 0; k < d; k++) {
    p[k] = e[k] / s;
    lp[k] = (z[k] - mx) - ls;
    Hv -= p[k] * lp[k];
  }
  const float bn = beta / (float)N;
  for (int k = 0; k < d; k++) {
    double acc = 0.0;
    if (lead)
      for (int c = 0; c < nchunks; c++) acc += part[((size_t)c * N + v) * d + k];
    float g = (float)(-(double)scale * (acc - (double)p[k] * sw));
    g += bn * p[k] * (lp[k] + Hv);
    dlog[(size_t)v * ld + k] = g;
  }
  for (int k = d; k < ld; k++) dlog[(size_t)v * ld + k] = 0.f;   // masked head columns
}

}  // namespace

void launch_sample(const float *logits, int ld, const int *leader, bool has_coloc, int N, int d, int B, uint64_t seed,
                   uint64_t offset, uint64_t step, const uint64_t *step_ptr, float *cdf, float *logp, int *lastpos,
                   double *spart, uint8_t *D, float *logprob, cudaStream_t s) {
  note_launch("k_node_prep", s);
  k_node_prep<<<(N + 255) / 256, 256, 0, s>>>(logits, ld, N, d, cdf, logp, lastpos);
  const int nq = (N + 3) / 4, nchunk = (nq + ST - 1) / ST, nwc = nchunk * (ST / 32);
  note_launch("k_sample", s, (double)B * N + 4.0 * (double)N * (2 * d + 2) + 8.0 * B * nwc);
  k_sample<<<dim3(nchunk, (B + SBG - 1) / SBG), ST, 0, s>>>(cdf, logp, lastpos, leader, has_coloc ? 1 : 0, N, d, B,
                                                            seed, offset, step, step_ptr, D, spart, nwc);
  note_launch("k_sample_lp", s, 8.0 * B * nwc + 4.0 * B);
  k_sample_lp<<<(B + 127) / 128, 128, 0, s>>>(spart, nwc, B, logprob);
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
                       int N, int d, int B, double *wb, double *part, float *dlog, cudaStream_t s) {
  note_launch("k_weights", s);
  k_weights<<<(B + 255) / 256, 256, 0, s>>>(adv, logprob, old_logprob, eps, B, wb);
  // placements split into chunks so that ~4 waves of threads stream the B x N bytes
  const int nq = (N + 3) / 4, nblk = (nq + LG_T - 1) / LG_T;
  int nch = (148 * 8 + nblk - 1) / nblk;   // ~8 CTAs of 128 threads per SM
  nch = nch < 1 ? 1 : (nch > kLogitChunks ? kLogitChunks : nch);
  if (nch > B) nch = B;
  const int b_per = (B + nch - 1) / nch;
  nch = (B + b_per - 1) / b_per;
  note_launch("k_logit_acc", s, (double)B * N + 8.0 * d * (double)N * nch);
  k_logit_acc<<<dim3(nblk, nch), LG_T, 0, s>>>(D, wb, N, d, B, b_per, part);
  note_launch("k_logit_grad", s, 8.0 * d * (double)N * nch + 4.0 * 2 * (double)N * d);
  k_logit_fin<<<(N + 127) / 128, 128, 0, s>>>(logits, ld, leader, wb, part, nch, beta, scale, N, d, B, dlog);
}

}  // namespace gdp

namespace gdp {
void launch_sum_parts(const double *part, int nparts, int B, float *logprob, cudaStream_t s) {
  note_launch("k_sample_lp", s, 8.0 * B * nparts + 4.0 * B);
  k_sample_lp<<<(B + 127) / 128, 128, 0, s>>>(part, nparts, B, logprob);
}
void launch_colocate(const int *leader, int N, int B, uint8_t *D, cudaStream_t s) {
  const size_t n = (size_t)N * B;
  note_launch("k_colocate", s);
  k_colocate<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(leader, N, B, D);
}
}  // namespace gdp
