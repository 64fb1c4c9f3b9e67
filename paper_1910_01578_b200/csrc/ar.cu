// Autoregressive-within-segment placer (SPEC.md:562 leaves open whether the paper's
// placer is autoregressive inside a segment; reading R35).  Nodes in Kahn order, segments
// of S positions.  For placement b and leader i of a segment,
//     z_{b,i} = base_i + (1/c_i) sum_{j < i, j leader, same segment} EW[D_bj],   EW = E Wh'
// (Wh' = gamma_h (.) W_h the folded head weight, E = GDP_P_AR_E), c_i the number of such j
// (z = base when c_i = 0).  Segments are independent, so the decode runs one warp per group of
// consecutive segments x 32 placements (one per lane); a lane walks its segments position by
// position with its running sum acc (d fp32 registers) -- the only sequential dependence.
//  * k_ar_table:  EW (d x d) in fp32, written behind the N x d base logits by gdp_place.
//  * k_ar_decode: sample (the R17 Philox uniform of the leader, inverse fp32 CDF exactly as
//                 k_node_prep / k_sample compute it), score (teacher placements: gdp_logprob) or
//                 greedy (argmax, ties -> lowest id); log pi partials per (placement, group) in
//                 fp64, summed in group order by k_sample_lp; non-leaders copy their leader.
//  * k_ar_grad:   the same walk over the sampled placements, per position
//                 dz_{b,i} = -s w_b ([k = D_bi] - p_{b,i}) [i leader] + beta/(B N) p (log p + H)
//                 (w_b: k_weights, the PPO branch); dL/dbase_i = sum_b dz (fp32 butterfly over the
//                 32 lanes, fp64 across b-blocks in order), dL/dEW[k] = sum_{b,i} (n_{b,i,k}/c_i) dz
//                 with n the per-device counts of the earlier leaders (64 fp32 registers per
//                 lane, butterfly, then k_ar_dew_fin sums the warps in order): deterministic.
//  * k_ar_head_bwd: dWh' += E^T dEW, grad[E] += dEW Wh'^T (the gate and W_h gradients then follow
//                 from dWh' exactly as for the head logits).
#include "common.cuh"
#include "philox.cuh"

namespace gdp {
namespace {

constexpr int AW = 4;   // warps per CTA

__global__ void k_ar_table(const float *__restrict__ E, const float *__restrict__ Wh, int d, float *EW) {
  const int t = threadIdx.x;
  if (t >= d * d) return;
  const int k = t / d, m = t % d;
  float s = 0.f;
  for (int c = 0; c < kH; c++) s = fmaf(E[k * kH + c], Wh[c * d + m], s);
  EW[t] = s;
}

// z = base + acc / c (c = 0: base), padded with -inf beyond d; fp32 softmax as in k_node_prep
struct Soft {
  float z[kMaxD], p[kMaxD], lp[kMaxD];
};
__device__ __forceinline__ void soft(const float *base, const float *acc, float rc, int d, Soft &o) {
#pragma unroll
  for (int t = 0; t < kMaxD; t++) o.z[t] = t < d ? fmaf(acc[t], rc, base[t]) : -__int_as_float(0x7f800000);
  float mx = o.z[0];
#pragma unroll
  for (int t = 1; t < kMaxD; t++)
    if (t < d) mx = fmaxf(mx, o.z[t]);
  float e[kMaxD], s = 0.f;
#pragma unroll
  for (int t = 0; t < kMaxD; t++) {
    e[t] = t < d ? expf(o.z[t] - mx) : 0.f;
    s += e[t];
  }
  const float ls = logf(s), is = 1.f / s;
#pragma unroll
  for (int t = 0; t < kMaxD; t++) {
    o.p[t] = e[t] * is;
    o.lp[t] = t < d ? (o.z[t] - mx) - ls : 0.f;
  }
}

// Sum of x[0..8) over the 32 lanes by a reduce-scatter butterfly (9 shuffles instead of 40):
// afterwards lane 4t holds the total of x[t].  Fixed pattern: deterministic.
__device__ __forceinline__ float warp_sum8(const float *x, int lane) {
  float y[4], z[2];
  const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const float r = __shfl_xor_sync(0xffffffffu, u16 ? x[i] : x[i + 4], 16);
    y[i] = (u16 ? x[i + 4] : x[i]) + r;
  }
#pragma unroll
  for (int i = 0; i < 2; i++) {
    const float r = __shfl_xor_sync(0xffffffffu, u8 ? y[i] : y[i + 2], 8);
    z[i] = (u8 ? y[i + 2] : y[i]) + r;
  }
  float w = (u4 ? z[1] : z[0]) + __shfl_xor_sync(0xffffffffu, u4 ? z[0] : z[1], 4);
  w += __shfl_xor_sync(0xffffffffu, w, 2);
  w += __shfl_xor_sync(0xffffffffu, w, 1);
  return w;
}
static_assert(kMaxD == 8, "warp_sum8 covers kMaxD = 8 devices");

// Per-warp staging of 32 segment positions: node id (~v for a co-location non-leader) and its
// base-logit row, so that the position walk reads shared memory instead of three dependent
// global loads (perm -> leader -> logits row) per position.
constexpr int TP = 32;
struct Tile {
  int v[TP];
  float b[TP][kMaxD + 1];
};
__device__ __forceinline__ int stage(Tile &t, const float *__restrict__ base, const int *__restrict__ perm,
                                     const int *__restrict__ leader, int p0, int p1, int d, int lane,
                                     bool leaders_only) {
  const int np = min(TP, p1 - p0);
  __syncwarp();
  if (lane < np) {
    const int v = __ldg(perm + p0 + lane);
    const bool lead = __ldg(leader + v) == v;
    t.v[lane] = lead ? v : ~v;
    if (lead || !leaders_only)
#pragma unroll
      for (int k = 0; k < kMaxD; k++)
        if (k < d) t.b[lane][k] = __ldg(base + (size_t)v * d + k);
  }
  __syncwarp();
  return np;
}

template <int MODE>
__global__ void __launch_bounds__(32 * AW)
    k_ar_decode(const float *__restrict__ base, const float *__restrict__ EWg, const int *__restrict__ perm,
                const int *__restrict__ leader, int N, int d, int S, int nseg, int spg, int G, int B, uint64_t seed,
                uint64_t offset, uint64_t step_val, const uint64_t *step_ptr, uint8_t *D, double *part) {
  __shared__ float EW[kMaxD * kMaxD];
  __shared__ Tile tiles[AW];
  for (int i = threadIdx.x; i < d * d; i += blockDim.x) EW[i] = EWg[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = blockIdx.x * AW + w;
  if (g >= G) return;
  Tile &T = tiles[w];
  const uint64_t step = step_ptr ? *step_ptr : step_val;
  const int b = blockIdx.y * 32 + lane;
  const bool active = b < B;
  const uint64_t gidx = offset + (uint64_t)b;
  uint8_t *Db = D + (size_t)(active ? b : 0) * N;
  double lpacc = 0.0;
  const int s1 = min(nseg, (g + 1) * spg);
  for (int sg = g * spg; sg < s1; sg++) {
    float acc[kMaxD];
#pragma unroll
    for (int t = 0; t < kMaxD; t++) acc[t] = 0.f;
    float rc = 0.f;   // 1 / (leaders decided so far in this segment), 0 before the first
    int c = 0;
    const int p1 = min(N, (sg + 1) * S);
    for (int p0 = sg * S; p0 < p1; p0 += TP) {
      const int np = stage(T, base, perm, leader, p0, p1, d, lane, true);
      for (int q = 0; q < np; q++) {
        const int v = T.v[q];
        if (v < 0) continue;   // non-leader (warp-uniform): copies its leader afterwards
        Soft o;
        soft(T.b[q], acc, rc, d, o);
        int k = 0;
        if (MODE == kArDecodeSample) {
          const float u = philox_uniform(seed, gidx, step, v);
          float cum = 0.f;
          int last = 0;
#pragma unroll
          for (int t = 0; t < kMaxD; t++) {
            if (t < d) {
              cum += o.p[t];
              k += (cum <= u);
              if (o.p[t] > 0.f) last = t;
            }
          }
          if (k >= d) k = last;
        } else if (MODE == kArDecodeScore) {
          k = active ? min((int)Db[v], d - 1) : 0;
        } else {
          float bz = o.z[0];
#pragma unroll
          for (int t = 1; t < kMaxD; t++)
            if (t < d && o.z[t] > bz) { bz = o.z[t]; k = t; }
        }
        float l = 0.f;
#pragma unroll
        for (int t = 0; t < kMaxD; t++) l = (t == k) ? o.lp[t] : l;
        if (active) {
          lpacc += (double)l;
          if (MODE != kArDecodeScore) Db[v] = (uint8_t)k;
        }
#pragma unroll
        for (int t = 0; t < kMaxD; t++)
          if (t < d) acc[t] += EW[k * d + t];
        rc = 1.f / (float)(++c);
      }
    }
  }
  if (active) part[(size_t)b * G + g] = lpacc;
}

// one warp per (segment group, placement chunk); lanes = 32 placements of one b-block, the
// chunk's b-blocks in order
#ifndef AR_GRAD_MINB
#define AR_GRAD_MINB 4   // 128 registers: 16 warps per SM (1.85 -> 1.65 ms at C4, B = 1332; 44 B of spills)
#endif
__global__ void __launch_bounds__(32 * AW, AR_GRAD_MINB)
    k_ar_grad(const float *__restrict__ base, const float *__restrict__ EWg, const int *__restrict__ perm,
              const int *__restrict__ leader, int N, int d, int S, int nseg, int spg, int G, int B, int bb_per,
              const uint8_t *__restrict__ D, const double *__restrict__ wb, float bn, float scale,
              double *lpart, float *dewpart) {
  __shared__ float EW[kMaxD * kMaxD];
  __shared__ Tile tiles[AW];
  for (int i = threadIdx.x; i < d * d; i += blockDim.x) EW[i] = EWg[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = blockIdx.x * AW + w, chunk = blockIdx.y;
  if (g >= G) return;
  Tile &T = tiles[w];
  const int nbb = (B + 31) / 32, bb0 = chunk * bb_per, bb1 = min(nbb, bb0 + bb_per);
  float dew[kMaxD][kMaxD];
#pragma unroll
  for (int k = 0; k < kMaxD; k++)
#pragma unroll
    for (int t = 0; t < kMaxD; t++) dew[k][t] = 0.f;
  const int s1 = min(nseg, (g + 1) * spg);
  double *lp_rows = lpart + (size_t)chunk * N * d;
  for (int bb = bb0; bb < bb1; bb++) {
    const int b = bb * 32 + lane;
    const bool active = b < B;
    const float wgt = active ? (float)(-(double)scale * wb[b]) : 0.f;   // dL / dlog pi_b
    const uint8_t *Db = D + (size_t)(active ? b : 0) * N;
    for (int sg = g * spg; sg < s1; sg++) {
      float acc[kMaxD], cnt[kMaxD];
#pragma unroll
      for (int t = 0; t < kMaxD; t++) acc[t] = cnt[t] = 0.f;
      float rc = 0.f;
      int c = 0;
      const int p1 = min(N, (sg + 1) * S);
      for (int p0 = sg * S; p0 < p1; p0 += TP) {
        const int np = stage(T, base, perm, leader, p0, p1, d, lane, false);
        for (int q = 0; q < np; q++) {
          const int p = p0 + q;
          // the running chunk partial of this position, fetched before the math hides its latency
          double prev = 0.0;
          if ((lane & 3) == 0 && (lane >> 2) < d && bb != bb0) prev = lp_rows[(size_t)p * d + (lane >> 2)];
          const int vv = T.v[q];
          const bool lead = vv >= 0;   // warp-uniform
          Soft o;
          soft(T.b[q], acc, rc, d, o);
          float H = 0.f;
#pragma unroll
          for (int t = 0; t < kMaxD; t++) H -= o.p[t] * o.lp[t];
          const int kD = (lead && active) ? min((int)Db[vv], d - 1) : 0;
          float dz[kMaxD];
#pragma unroll
          for (int t = 0; t < kMaxD; t++) {
            float x = bn * o.p[t] * (o.lp[t] + H);
            if (lead) x += wgt * ((t == kD ? 1.f : 0.f) - o.p[t]);
            dz[t] = (active && t < d) ? x : 0.f;
          }
          if (c) {
#pragma unroll
            for (int k = 0; k < kMaxD; k++) {
              const float f = cnt[k] * rc;
#pragma unroll
              for (int t = 0; t < kMaxD; t++) dew[k][t] = fmaf(f, dz[t], dew[k][t]);
            }
          }
          const float val = warp_sum8(dz, lane);
          if ((lane & 3) == 0 && (lane >> 2) < d) lp_rows[(size_t)p * d + (lane >> 2)] = prev + (double)val;
          if (lead) {
#pragma unroll
            for (int t = 0; t < kMaxD; t++) {
              if (t < d) acc[t] += EW[kD * d + t];
              cnt[t] += (t == kD) ? 1.f : 0.f;
            }
            rc = 1.f / (float)(++c);
          }
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kMaxD; k++)
#pragma unroll
    for (int t = 0; t < kMaxD; t++) {
      float x = dew[k][t];
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o2);
      dew[k][t] = x;
    }
  if (lane == 0) {
    float *o = dewpart + ((size_t)chunk * G + g) * d * d;
#pragma unroll
    for (int k = 0; k < kMaxD; k++)
#pragma unroll
      for (int t = 0; t < kMaxD; t++)
        if (k < d && t < d) o[k * d + t] = dew[k][t];
  }
}

// dL/dbase in topological rows: the chunk partials in chunk order
__global__ void k_ar_dlog_fin(const double *__restrict__ lpart, int nch, int N, int d, float *dlt) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)N * d) return;
  double s = 0.0;
  for (int c = 0; c < nch; c++) s += lpart[(size_t)c * N * d + e];
  dlt[e] = (float)s;
}

// dL/dEW: one CTA per entry; thread t sums the warp partials t, t + 256, ... in order, then a
// fixed-order tree over the threads (deterministic)
__global__ void __launch_bounds__(256) k_ar_dew_fin(const float *__restrict__ dewpart, int nparts, int d, float *dEW) {
  __shared__ double red[256];
  const int e = blockIdx.x, t = threadIdx.x;
  double s = 0.0;
  for (int i = t; i < nparts; i += 256) s += (double)dewpart[(size_t)i * d * d + e];
  red[t] = s;
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if (t < h) red[t] += red[t + h];
    __syncthreads();
  }
  if (t == 0) dEW[e] = (float)red[0];
}

__global__ void k_ar_head_bwd(const float *__restrict__ E, const float *__restrict__ Wh,
                              const float *__restrict__ dEW, int d, float *dWh, float *gE) {
  const int t = threadIdx.x;
  if (t >= kH * d) return;
  {  // dWh'[c][m] += sum_k E[k][c] dEW[k][m]
    const int c = t / d, m = t % d;
    float s = 0.f;
    for (int k = 0; k < d; k++) s = fmaf(E[k * kH + c], dEW[k * d + m], s);
    dWh[c * d + m] += s;
  }
  {  // grad E[k][c] += sum_m dEW[k][m] Wh'[c][m]
    const int k = t / kH, c = t % kH;
    float s = 0.f;
    for (int m = 0; m < d; m++) s = fmaf(dEW[k * d + m], Wh[c * d + m], s);
    gE[k * kH + c] += s;
  }
}

__global__ void k_ar_weights(const double *adv, const float *logprob, const float *old_logprob, float eps, int B,
                             double *wb) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  double A = adv[b];
  double rho = old_logprob ? exp((double)logprob[b] - (double)old_logprob[b]) : 1.0;
  double lo = 1.0 - (double)eps, hi = 1.0 + (double)eps;
  double cl = rho < lo ? lo : (rho > hi ? hi : rho);
  wb[b] = (rho * A <= cl * A) ? rho * A : 0.0;
}

}  // namespace

int ar_groups(int N, int S) {
  const int nseg = (N + S - 1) / S;
  const int nq = (N + 3) / 4, nwc = (nq + 255) / 256 * 8;   // k_sample's chunk count (ws.spart)
  return nseg < nwc ? nseg : nwc;
}

void launch_ar_table(const float *E, const float *Wh, int d, float *EW, cudaStream_t s) {
  note_launch("k_ar_table", s);
  k_ar_table<<<1, kMaxD * kMaxD, 0, s>>>(E, Wh, d, EW);
}

void launch_ar_decode(int mode, const float *logits, const int *perm, const int *leader, bool has_coloc, int N,
                      int d, int S, int B, uint64_t seed, uint64_t offset, uint64_t step, const uint64_t *step_ptr,
                      uint8_t *D, double *part, float *logprob, cudaStream_t s) {
  const int nseg = (N + S - 1) / S, G = ar_groups(N, S), spg = (nseg + G - 1) / G;
  const float *EW = logits + (size_t)N * d;
  dim3 grid((G + AW - 1) / AW, (B + 31) / 32);
  const double bytes = 4.0 * N * d + 8.0 * N + (double)B * N + 8.0 * B * G;
  if (mode == kArDecodeSample) {
    note_launch("k_ar_decode", s, bytes);
    k_ar_decode<kArDecodeSample><<<grid, 32 * AW, 0, s>>>(logits, EW, perm, leader, N, d, S, nseg, spg, G, B, seed,
                                                          offset, step, step_ptr, D, part);
  } else if (mode == kArDecodeScore) {
    note_launch("k_ar_score", s, bytes);
    k_ar_decode<kArDecodeScore><<<grid, 32 * AW, 0, s>>>(logits, EW, perm, leader, N, d, S, nseg, spg, G, B, 0, 0,
                                                         0, nullptr, D, part);
  } else {
    note_launch("k_ar_greedy", s, bytes);
    k_ar_decode<kArDecodeGreedy><<<grid, 32 * AW, 0, s>>>(logits, EW, perm, leader, N, d, S, nseg, spg, G, B, 0, 0,
                                                          0, nullptr, D, part);
  }
  if (logprob) launch_sum_parts(part, G, B, logprob, s);
  if (mode != kArDecodeScore && has_coloc) launch_colocate(leader, N, B, D, s);
}

void launch_ar_grad(const float *logits, const int *perm, const int *leader, int N, int d, int S, int B,
                    const uint8_t *D, const double *adv, const float *logprob, const float *old_logprob, float eps,
                    float beta, float scale, double *wb, double *lpart, float *dewpart, size_t dewpart_floats,
                    float *dlt, float *dEW, cudaStream_t s) {
  note_launch("k_weights", s);
  k_ar_weights<<<(B + 255) / 256, 256, 0, s>>>(adv, logprob, old_logprob, eps, B, wb);
  const int nseg = (N + S - 1) / S, G = ar_groups(N, S), spg = (nseg + G - 1) / G;
  const int nbb = (B + 31) / 32;
  int nch = nbb < kLogitChunks ? nbb : kLogitChunks;
  while (nch > 1 && (size_t)nch * G * d * d > dewpart_floats) nch--;
  const int bb_per = (nbb + nch - 1) / nch;
  nch = (nbb + bb_per - 1) / bb_per;
  const float bn = beta / ((float)B * (float)N);
  note_launch("k_ar_grad", s, 4.0 * N * d + 8.0 * N + (double)B * N + 8.0 * B + 8.0 * nch * N * d);
  k_ar_grad<<<dim3((G + AW - 1) / AW, nch), 32 * AW, 0, s>>>(logits, logits + (size_t)N * d, perm, leader, N, d, S,
                                                              nseg, spg, G, B, bb_per, D, wb, bn, scale, lpart,
                                                              dewpart);
  note_launch("k_ar_dlog_fin", s, 8.0 * nch * N * d + 4.0 * N * d);
  k_ar_dlog_fin<<<(unsigned)(((size_t)N * d + 255) / 256), 256, 0, s>>>(lpart, nch, N, d, dlt);
  note_launch("k_ar_dew_fin", s);
  k_ar_dew_fin<<<d * d, 256, 0, s>>>(dewpart, nch * G, d, dEW);
}

void launch_ar_head_bwd(const float *E, const float *Wh, const float *dEW, int d, float *dWh, float *gE,
                        cudaStream_t s) {
  note_launch("k_ar_head_bwd", s);
  k_ar_head_bwd<<<1, kH * kMaxD, 0, s>>>(E, Wh, dEW, d, dWh, gE);
}

}  // namespace gdp
