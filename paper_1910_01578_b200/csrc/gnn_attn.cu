// Graph aggregation (§3.1 Eq. 2) and segment-recurrent attention
// (§3.2).
//
//  * k_gather_max:      warp per node, lanes own 2 of the 64 channels; neighbour rows
//                       (256 B, coalesced) are streamed in ascending id, strict '>' keeps
//                       the first (lowest-id) maximiser.  Empty N(v) -> 0.
//  * k_gather_max_bwd:  the max-pool backward as a GATHER over the symmetric CSR:
//                       dZ_u[c] = sum_{v in N(u), argmax_v[c] = u} dA_v[c] (no atomics,
//                       fixed order), fused with the sigmoid derivative Z(1-Z).
//  * attention:         one CTA per (segment, head); queries of segment tau attend to
//                       keys [max(0, tau S - M), min((tau+1) S, N)) with an online softmax;
//                       the backward splits dK/dV into the own-segment part (flows into x)
//                       and the memory part (stop-gradient: parameters only).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace gdp {
namespace {

// Neighbour ids are fetched 32 at a time (one coalesced load, shuffled out) and the rows of GU
// neighbours are requested before any is compared (comparisons stay in ascending-id order).
// Nodes with more than kHeavyDeg neighbours (the heavy tail of the GNMT graphs: attention
// memories read by every decoder step, degree up to 361) would set the kernel's duration with
// one warp each; they get one CTA each instead (blocks after the warp-per-node range): its 8
// warps scan 8 contiguous, ascending ranges of the neighbour list and the partial results are
// combined in range order, so the first maximiser still wins (and backward sums stay in a
// fixed order).
constexpr int GU = 4;
constexpr int GW = 8;   // warps per CTA

__device__ __forceinline__ void gmax_range(const float2 *Z2, const int *__restrict__ idx, int b, int e, int lane,
                                           float2 &m, int &a0, int &a1) {
  for (int j0 = b; j0 < e; j0 += 32) {
    const int n = min(32, e - j0);
    const int mine = lane < n ? __ldg(idx + j0 + lane) : 0;
    for (int k0 = 0; k0 < n; k0 += GU) {
      int u[GU];
      float2 z[GU];
#pragma unroll
      for (int t = 0; t < GU; t++) {
        u[t] = __shfl_sync(0xffffffffu, mine, (k0 + t) & 31);
        if (k0 + t < n) z[t] = __ldg(Z2 + (size_t)u[t] * (kH / 2) + lane);
      }
#pragma unroll
      for (int t = 0; t < GU; t++) {
        if (k0 + t >= n) break;
        if (a0 < 0 || z[t].x > m.x) { m.x = z[t].x; a0 = u[t]; }   // strict '>': first maximiser wins
        if (a1 < 0 || z[t].y > m.y) { m.y = z[t].y; a1 = u[t]; }
      }
    }
  }
}

__global__ void __launch_bounds__(32 * GW) k_gather_max(const float *__restrict__ Z, const int *__restrict__ ptr,
                                                        const int *__restrict__ idx, const int *__restrict__ heavy,
                                                        int nb_main, float *A, int *ARG, int N) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float2 *Z2 = reinterpret_cast<const float2 *>(Z);   // lane owns channels 2 lane, 2 lane + 1
  float2 m = make_float2(0.f, 0.f);
  int a0 = -1, a1 = -1;
  if ((int)blockIdx.x < nb_main) {   // warp per node
    const int v = blockIdx.x * GW + warp;
    if (v >= N) return;
    const int b = ptr[v], e = ptr[v + 1];
    if (e - b > kHeavyDeg) return;
    gmax_range(Z2, idx, b, e, lane, m, a0, a1);
    reinterpret_cast<float2 *>(A)[(size_t)v * (kH / 2) + lane] = m;
    reinterpret_cast<int2 *>(ARG)[(size_t)v * (kH / 2) + lane] = make_int2(a0, a1);
    return;
  }
  __shared__ float2 sm[GW][32];
  __shared__ int2 sa[GW][32];
  const int v = heavy[blockIdx.x - nb_main];
  const int b = ptr[v], e = ptr[v + 1], len = (e - b + GW - 1) / GW;
  const int rb = b + warp * len, re = min(e, rb + len);
  if (rb < re) gmax_range(Z2, idx, rb, re, lane, m, a0, a1);
  sm[warp][lane] = m;
  sa[warp][lane] = make_int2(a0, a1);
  __syncthreads();
  if (warp != 0) return;
  for (int w = 1; w < GW; w++) {   // ascending ranges: a later range wins only if strictly greater
    const float2 mw = sm[w][lane];
    const int2 aw = sa[w][lane];
    if (aw.x >= 0 && (a0 < 0 || mw.x > m.x)) { m.x = mw.x; a0 = aw.x; }
    if (aw.y >= 0 && (a1 < 0 || mw.y > m.y)) { m.y = mw.y; a1 = aw.y; }
  }
  reinterpret_cast<float2 *>(A)[(size_t)v * (kH / 2) + lane] = m;
  reinterpret_cast<int2 *>(ARG)[(size_t)v * (kH / 2) + lane] = make_int2(a0, a1);
}

__device__ __forceinline__ void gmax_bwd_range(const float2 *dA2, const int2 *ARG2, const int *__restrict__ idx, int b,
                                               int e, int lane, int u, float &s0, float &s1) {
  for (int j0 = b; j0 < e; j0 += 32) {
    const int n = min(32, e - j0);
    const int mine = lane < n ? __ldg(idx + j0 + lane) : 0;
    for (int k0 = 0; k0 < n; k0 += GU) {
      int2 ag[GU];
      float2 g[GU];
#pragma unroll
      for (int t = 0; t < GU; t++) {
        const int v = __shfl_sync(0xffffffffu, mine, (k0 + t) & 31);
        if (k0 + t < n) {
          ag[t] = __ldg(ARG2 + (size_t)v * (kH / 2) + lane);
          g[t] = __ldg(dA2 + (size_t)v * (kH / 2) + lane);
        }
      }
#pragma unroll
      for (int t = 0; t < GU; t++) {   // ascending neighbour order, as the oracle sums
        if (k0 + t >= n) break;
        if (ag[t].x == u) s0 += g[t].x;
        if (ag[t].y == u) s1 += g[t].y;
      }
    }
  }
}

__global__ void __launch_bounds__(32 * GW) k_gather_max_bwd(const float *__restrict__ dA, const int *__restrict__ ARG,
                                                            const float *__restrict__ Z, const int *__restrict__ ptr,
                                                            const int *__restrict__ idx, const int *__restrict__ heavy,
                                                            int nb_main, float *dPre, int N) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float2 *dA2 = reinterpret_cast<const float2 *>(dA);
  const int2 *ARG2 = reinterpret_cast<const int2 *>(ARG);
  float s0 = 0.f, s1 = 0.f;
  int u;
  if ((int)blockIdx.x < nb_main) {
    u = blockIdx.x * GW + warp;
    if (u >= N) return;
    const int b = ptr[u], e = ptr[u + 1];
    if (e - b > kHeavyDeg) return;
    gmax_bwd_range(dA2, ARG2, idx, b, e, lane, u, s0, s1);
  } else {
    __shared__ float2 ss[GW][32];
    u = heavy[blockIdx.x - nb_main];
    const int b = ptr[u], e = ptr[u + 1], len = (e - b + GW - 1) / GW;
    const int rb = b + warp * len, re = min(e, rb + len);
    if (rb < re) gmax_bwd_range(dA2, ARG2, idx, rb, re, lane, u, s0, s1);
    ss[warp][lane] = make_float2(s0, s1);
    __syncthreads();
    if (warp != 0) return;
    s0 = 0.f; s1 = 0.f;
    for (int w = 0; w < GW; w++) {   // fixed (range) order
      s0 += ss[w][lane].x;
      s1 += ss[w][lane].y;
    }
  }
  const float2 z = reinterpret_cast<const float2 *>(Z)[(size_t)u * (kH / 2) + lane];
  reinterpret_cast<float2 *>(dPre)[(size_t)u * (kH / 2) + lane] = make_float2(s0 * z.x * (1.f - z.x), s1 * z.y * (1.f - z.y));
}

constexpr int AQ = 128;  // queries (or keys) per thread block pass
constexpr int AK = 64;   // keys (or queries) per shared-memory tile
constexpr float kScale = 0.25f;   // 1 / sqrt(16)

// a 16-float tile row into registers with four 16-byte shared loads (the rows are broadcast to
// the whole warp, so one LDS.128 replaces four scalar LDS: the kernels were LDS-issue bound)
__device__ __forceinline__ void row16(const float *r, float *x) {
  const float4 *r4 = reinterpret_cast<const float4 *>(r);
#pragma unroll
  for (int t = 0; t < 4; t++) {
    const float4 v = r4[t];
    x[4 * t] = v.x; x[4 * t + 1] = v.y; x[4 * t + 2] = v.z; x[4 * t + 3] = v.w;
  }
}

__device__ __forceinline__ void key_range(int tau, int N, int S, int M, int *lo, int *hi) {
  long long q0 = (long long)tau * S;
  *lo = (M < 0) ? 0 : (int)max(0LL, q0 - M);
  *hi = (int)min((long long)N, q0 + S);
}

// qkv: N x 192 [Q | K | V], head h uses columns h*16 .. h*16+15 of each block.
__global__ void __launch_bounds__(AQ) k_attn_fwd(const float *__restrict__ qkv, float *o, float *lse, int N,
                                                 int S, int M) {
  __shared__ __align__(16) float Ks[AK][kDH], Vs[AK][kDH];
  const int tau = blockIdx.x, hd = blockIdx.y;
  int lo, hi;
  key_range(tau, N, S, M, &lo, &hi);
  const int q0 = tau * S, q1 = min(N, q0 + S);
  for (int qb = q0; qb < q1; qb += AQ) {
    const int i = qb + threadIdx.x;
    const bool valid = i < q1;
    float q[kDH], acc[kDH];
    float mx = -INFINITY, l = 0.f;
#pragma unroll
    for (int c = 0; c < kDH; c++) {
      q[c] = valid ? qkv[(size_t)i * 192 + hd * kDH + c] : 0.f;
      acc[c] = 0.f;
    }
    for (int kb = lo; kb < hi; kb += AK) {
      __syncthreads();
      for (int e = threadIdx.x; e < AK * kDH; e += AQ) {
        int j = e / kDH, c = e % kDH;
        int r = kb + j;
        Ks[j][c] = r < hi ? qkv[(size_t)r * 192 + 64 + hd * kDH + c] : 0.f;
        Vs[j][c] = r < hi ? qkv[(size_t)r * 192 + 128 + hd * kDH + c] : 0.f;
      }
      __syncthreads();
      const int nk = min(AK, hi - kb);
      for (int j = 0; j < nk; j++) {
        float kr[kDH], vr[kDH];
        row16(Ks[j], kr);
        row16(Vs[j], vr);
        float s = 0.f;
#pragma unroll
        for (int c = 0; c < kDH; c++) s = fmaf(q[c], kr[c], s);
        s *= kScale;
        if (s > mx) {
          float f = expf(mx - s);
          l *= f;
#pragma unroll
          for (int c = 0; c < kDH; c++) acc[c] *= f;
          mx = s;
        }
        float p = expf(s - mx);
        l += p;
#pragma unroll
        for (int c = 0; c < kDH; c++) acc[c] = fmaf(p, vr[c], acc[c]);
      }
    }
    if (valid) {
      float inv = 1.f / l;
#pragma unroll
      for (int c = 0; c < kDH; c++) o[(size_t)i * kH + hd * kDH + c] = acc[c] * inv;
      lse[(size_t)i * kHeads + hd] = mx + logf(l);
    }
  }
}

// Dd[i][h] = sum_c dO[i][h*16+c] * O[i][h*16+c]
__global__ void k_attn_bwd_prep(const float *o, const float *dout, float *Dd, int N) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N * kHeads) return;
  int i = e / kHeads, h = e % kHeads;
  float s = 0.f;
  for (int c = 0; c < kDH; c++) s = fmaf(dout[(size_t)i * kH + h * kDH + c], o[(size_t)i * kH + h * kDH + c], s);
  Dd[e] = s;
}

// dQ (query-major): dqkv[:, 0:64]
__global__ void __launch_bounds__(AQ) k_attn_bwd_dq(const float *__restrict__ qkv, const float *__restrict__ lse,
                                                    const float *__restrict__ dout, const float *__restrict__ Dd,
                                                    float *dqkv, int N, int S, int M) {
  __shared__ __align__(16) float Ks[AK][kDH], Vs[AK][kDH];
  const int tau = blockIdx.x, hd = blockIdx.y;
  int lo, hi;
  key_range(tau, N, S, M, &lo, &hi);
  const int q0 = tau * S, q1 = min(N, q0 + S);
  for (int qb = q0; qb < q1; qb += AQ) {
    const int i = qb + threadIdx.x;
    const bool valid = i < q1;
    float q[kDH], dq[kDH], dob[kDH];
    float L = valid ? lse[(size_t)i * kHeads + hd] : 0.f;
    float D = valid ? Dd[(size_t)i * kHeads + hd] : 0.f;
#pragma unroll
    for (int c = 0; c < kDH; c++) {
      q[c] = valid ? qkv[(size_t)i * 192 + hd * kDH + c] : 0.f;
      dob[c] = valid ? dout[(size_t)i * kH + hd * kDH + c] : 0.f;
      dq[c] = 0.f;
    }
    for (int kb = lo; kb < hi; kb += AK) {
      __syncthreads();
      for (int e = threadIdx.x; e < AK * kDH; e += AQ) {
        int j = e / kDH, c = e % kDH;
        int r = kb + j;
        Ks[j][c] = r < hi ? qkv[(size_t)r * 192 + 64 + hd * kDH + c] : 0.f;
        Vs[j][c] = r < hi ? qkv[(size_t)r * 192 + 128 + hd * kDH + c] : 0.f;
      }
      __syncthreads();
      const int nk = min(AK, hi - kb);
      for (int j = 0; j < nk; j++) {
        float kr[kDH], vr[kDH];
        row16(Ks[j], kr);
        row16(Vs[j], vr);
        float s = 0.f, dp = 0.f;
#pragma unroll
        for (int c = 0; c < kDH; c++) {
          s = fmaf(q[c], kr[c], s);
          dp = fmaf(dob[c], vr[c], dp);
        }
        float p = expf(s * kScale - L);
        float ds = p * (dp - D) * kScale;
#pragma unroll
        for (int c = 0; c < kDH; c++) dq[c] = fmaf(ds, kr[c], dq[c]);
      }
    }
    if (valid) {
#pragma unroll
      for (int c = 0; c < kDH; c++) dqkv[(size_t)i * 192 + hd * kDH + c] = dq[c];
    }
  }
}

__device__ __forceinline__ void dkv_accum(int ni, const float (*Qs)[kDH], const float (*dOs)[kDH],
                                          const float *Ls, const float *Ds, const float *k, const float *v,
                                          float *DK, float *DV) {
  for (int r = 0; r < ni; r++) {
    float qr[kDH], gr[kDH];
    row16(Qs[r], qr);
    row16(dOs[r], gr);
    float s = 0.f, dp = 0.f;
#pragma unroll
    for (int c = 0; c < kDH; c++) {
      s = fmaf(qr[c], k[c], s);
      dp = fmaf(gr[c], v[c], dp);
    }
    float p = expf(s * kScale - Ls[r]);
    float ds = p * (dp - Ds[r]) * kScale;
#pragma unroll
    for (int c = 0; c < kDH; c++) {
      DV[c] = fmaf(p, gr[c], DV[c]);
      DK[c] = fmaf(ds, qr[c], DK[c]);
    }
  }
}

// dK, dV (key-major).  Keys of segment sigma are attended by query segments tau >= sigma
// whose range starts at or before them.  tau == sigma -> own part (dqkv[:, 64:192]);
// tau > sigma -> memory part (dkvm[:, 0:128]), which is stop-gradient for x.
__global__ void __launch_bounds__(AQ) k_attn_bwd_dkv(const float *__restrict__ qkv, const float *__restrict__ lse,
                                                     const float *__restrict__ dout, const float *__restrict__ Dd,
                                                     float *dqkv, float *dkvm, int N, int S, int M, int nseg) {
  __shared__ __align__(16) float Qs[AK][kDH], dOs[AK][kDH];
  __shared__ float Ls[AK], Ds[AK];
  const int sig = blockIdx.x, hd = blockIdx.y;
  const int j0 = sig * S, j1 = min(N, j0 + S);
  int tau_hi = nseg - 1;
  if (M >= 0) tau_hi = min(nseg - 1, (int)(((long long)j1 - 1 + M) / S));
  for (int jb = j0; jb < j1; jb += AQ) {
    const int j = jb + threadIdx.x;
    const bool valid = j < j1;
    float k[kDH], v[kDH], dk[kDH], dv[kDH], dkm[kDH], dvm[kDH];
#pragma unroll
    for (int c = 0; c < kDH; c++) {
      k[c] = valid ? qkv[(size_t)j * 192 + 64 + hd * kDH + c] : 0.f;
      v[c] = valid ? qkv[(size_t)j * 192 + 128 + hd * kDH + c] : 0.f;
      dk[c] = dv[c] = dkm[c] = dvm[c] = 0.f;
    }
    for (int tau = sig; tau <= tau_hi; tau++) {
      int lo, hi;
      key_range(tau, N, S, M, &lo, &hi);
      const bool inr = valid && j >= lo;
      const int q0 = tau * S, q1 = min(N, q0 + S);
      for (int ib = q0; ib < q1; ib += AK) {
        __syncthreads();
        for (int e = threadIdx.x; e < AK * kDH; e += AQ) {
          int r = e / kDH, c = e % kDH;
          int i = ib + r;
          Qs[r][c] = i < q1 ? qkv[(size_t)i * 192 + hd * kDH + c] : 0.f;
          dOs[r][c] = i < q1 ? dout[(size_t)i * kH + hd * kDH + c] : 0.f;
        }
        for (int r = threadIdx.x; r < AK; r += AQ) {
          int i = ib + r;
          Ls[r] = i < q1 ? lse[(size_t)i * kHeads + hd] : 0.f;
          Ds[r] = i < q1 ? Dd[(size_t)i * kHeads + hd] : 0.f;
        }
        __syncthreads();
        if (!inr) continue;
        const int ni = min(AK, q1 - ib);
        if (tau == sig) dkv_accum(ni, Qs, dOs, Ls, Ds, k, v, dk, dv);
        else dkv_accum(ni, Qs, dOs, Ls, Ds, k, v, dkm, dvm);
      }
    }
    if (valid) {
#pragma unroll
      for (int c = 0; c < kDH; c++) {
        dqkv[(size_t)j * 192 + 64 + hd * kDH + c] = dk[c];
        dqkv[(size_t)j * 192 + 128 + hd * kDH + c] = dv[c];
        dkvm[(size_t)j * 128 + hd * kDH + c] = dkm[c];
        dkvm[(size_t)j * 128 + 64 + hd * kDH + c] = dvm[c];
      }
    }
  }
}

}  // namespace

// algorithmic (unique) bytes: CSR (N + 1 + nnz) x 4, Z read once N x 64 x 4, A and ARG written
void launch_gather_max(const float *Z, const int *ptr, const int *idx, const int *heavy, int n_heavy, float *A,
                       int *ARG, int N, long long nnz, cudaStream_t s) {
  const int nb_main = (N + GW - 1) / GW;
  const unsigned blocks = (unsigned)(nb_main + n_heavy);
  note_launch("k_gather_max", s, 4.0 * ((double)N + 1 + (double)nnz) + 3.0 * 4 * 64 * (double)N);
  k_gather_max<<<blocks, 32 * GW, 0, s>>>(Z, ptr, idx, heavy, nb_main, A, ARG, N);
}

void launch_gather_max_bwd(const float *dA, const int *ARG, const float *Z, const int *ptr, const int *idx,
                           const int *heavy, int n_heavy, float *dPre, int N, long long nnz, cudaStream_t s) {
  const int nb_main = (N + GW - 1) / GW;
  const unsigned blocks = (unsigned)(nb_main + n_heavy);
  // CSR, dA and ARG of every neighbour read once per node (unique), dPre written
  note_launch("k_gather_max_bwd", s, 4.0 * ((double)N + 1 + (double)nnz) + 3.0 * 4 * 64 * (double)N);
  k_gather_max_bwd<<<blocks, 32 * GW, 0, s>>>(dA, ARG, Z, ptr, idx, heavy, nb_main, dPre, N);
}

// no_attention ablation (NEXT-3, reading R34): o = ReLU(V) per node; backward dV = dO [V > 0],
// dQ = dK = 0 and no memory rows
__global__ void k_relu_v(const float *__restrict__ qkv, float *o, int N) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)N * 64) return;
  const size_t i = e / 64, c = e % 64;
  o[e] = fmaxf(qkv[i * 192 + 128 + c], 0.f);
}
__global__ void k_relu_v_bwd(const float *__restrict__ qkv, const float *__restrict__ dout, float *dqkv, float *dkvm,
                             int N) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)N * 64) return;
  const size_t i = e / 64, c = e % 64;
  dqkv[i * 192 + c] = 0.f;
  dqkv[i * 192 + 64 + c] = 0.f;
  dqkv[i * 192 + 128 + c] = qkv[i * 192 + 128 + c] > 0.f ? dout[e] : 0.f;
  dkvm[i * 128 + c] = 0.f;
  dkvm[i * 128 + 64 + c] = 0.f;
}

void launch_relu_v(const float *qkv, float *o, int N, cudaStream_t s) {
  note_launch("k_relu_v", s);
  k_relu_v<<<(unsigned)(((size_t)N * 64 + 255) / 256), 256, 0, s>>>(qkv, o, N);
}
void launch_relu_v_bwd(const float *qkv, const float *dout, float *dqkv, float *dkvm, int N, cudaStream_t s) {
  note_launch("k_relu_v_bwd", s);
  k_relu_v_bwd<<<(unsigned)(((size_t)N * 64 + 255) / 256), 256, 0, s>>>(qkv, dout, dqkv, dkvm, N);
}

// 4 x 64 flops per (query, key) pair over the key sets K(i) (QK^T and PV), i.e. the forward
static double attn_flops(int N, int S, int M) {
  double pairs = 0.0;
  for (long long t0 = 0; t0 < N; t0 += S) {
    const long long q = std::min<long long>(S, N - t0);
    const long long lo = M < 0 ? 0 : std::max<long long>(0, t0 - M);
    pairs += (double)q * (double)(t0 + q - lo);
  }
  return 4.0 * 64 * pairs;
}


// the tensor-core attention launches put the segments on gridDim.y (<= 65535); more segments
// (e.g. S = 1 with N > 65535) take the SIMT kernels, which put them on gridDim.x
static bool attn_tc_grid_ok(int N, int S) { return (N + S - 1) / S <= 65535; }

void launch_attn_fwd(const float *qkv, float *o, float *lse, int N, int S, int M, cudaStream_t s) {
  int nseg = (N + S - 1) / S;
  if (tensor_core_attention_on() && attn_fwd_tc_eligible(S, M) && attn_tc_grid_ok(N, S)) {   // tensor-core mode: tcgen05 tiles (attn_tc.cu)
    note_launch("k_attn_fwd_tc", s, 4.0 * (double)N * (192 + 64 + kHeads), attn_flops(N, S, M));
    launch_attn_fwd_tc(qkv, o, lse, N, S, M, s);
    return;
  }
  note_launch("k_attn_fwd", s, 4.0 * (double)N * (192 + 64 + kHeads), attn_flops(N, S, M));
  k_attn_fwd<<<dim3(nseg, kHeads), AQ, 0, s>>>(qkv, o, lse, N, S, M);
}

void launch_attn_bwd(const float *qkv, const float *o, const float *lse, const float *dout, float *dqkv,
                     float *dkvm, float *Dd, int N, int S, int M, cudaStream_t s) {
  int nseg = (N + S - 1) / S;
  if (tensor_core_attention_on() && attn_bwd_tc_long_eligible(S, M) && attn_tc_grid_ok(N, S)) {   // tensor-core mode (attn_tc.cu)
    note_launch("k_attn_bwd_dq_tc", s, 4.0 * (double)N * (192 + 64 + 64 + kHeads + 64), attn_flops(N, S, M));
    launch_attn_bwd_dq_tc(qkv, o, lse, dout, dqkv, N, S, M, s);
    note_launch("k_attn_bwd_dkv_tc", s, 4.0 * (double)N * (192 + 64 + 64 + kHeads + 128 + 128), 1.5 * attn_flops(N, S, M));
    launch_attn_bwd_dkv_tc(qkv, o, lse, dout, dqkv, dkvm, N, S, M, s);
    return;
  }
  note_launch("k_attn_bwd_prep", s);
  k_attn_bwd_prep<<<(N * kHeads + 255) / 256, 256, 0, s>>>(o, dout, Dd, N);
  note_launch("k_attn_bwd_dq", s, 4.0 * (double)N * (192 + 64 + 64 + 2 * kHeads), attn_flops(N, S, M));
  k_attn_bwd_dq<<<dim3(nseg, kHeads), AQ, 0, s>>>(qkv, lse, dout, Dd, dqkv, N, S, M);
  note_launch("k_attn_bwd_dkv", s, 4.0 * (double)N * (192 + 64 + 128 + 2 * kHeads), 1.5 * attn_flops(N, S, M));
  k_attn_bwd_dkv<<<dim3(nseg, kHeads), AQ, 0, s>>>(qkv, lse, dout, Dd, dqkv, dkvm, N, S, M, nseg);
}

}  // namespace gdp
