// Dense building blocks of the policy network (fp32 SIMT, deterministic reductions).
//  * k_gemm:   Y = epi(X W + b) (+ R) for the tall-skinny maps of §3.1 Eq. 2-3 and the
//              Transformer-XL projections of §3.2 (M = N nodes, K, Nout <= 257).
//  * k_wgrad:  dW = X^T dY split over row chunks, summed in fixed chunk order.
//  * LayerNorm forward/backward (pre-LN), column sums (mean over nodes).
#include <algorithm>

#include "common.cuh"

namespace gdp {

namespace {
constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

__device__ __forceinline__ float apply_epi(int epi, float v) {
  switch (epi) {
    case EPI_SIGMOID: return 1.0f / (1.0f + expf(-v));
    case EPI_TANH: return tanhf(v);
    case EPI_RELU: return v > 0.f ? v : 0.f;
    default: return v;
  }
}

__global__ void __launch_bounds__(NT) k_gemm(GemmArgs a) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int ty = tid / 16, tx = tid % 16;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j] = 0.f;
  for (int k0 = 0; k0 < a.K; k0 += BK) {
    // A tile: BM rows x BK cols; element (r, kk) -> As[kk][r]
#pragma unroll
    for (int i = 0; i < (BM * BK) / NT; i++) {
      int e = tid + i * NT;
      int r = e / BK, kk = e % BK;
      int m = m0 + r, k = k0 + kk;
      float v = 0.f;
      if (m < a.M && k < a.K) {
        v = (k < a.K1) ? a.X1[(size_t)m * a.ldx1 + k] : a.X2[(size_t)m * a.ldx2 + (k - a.K1)];
      }
      As[kk][r] = v;
    }
#pragma unroll
    for (int i = 0; i < (BK * BN) / NT; i++) {
      int e = tid + i * NT;
      int kk = e / BN, c = e % BN;
      int k = k0 + kk, n = n0 + c;
      Bs[kk][c] = (k < a.K && n < a.Nout) ? a.W[(size_t)k * a.ldw_k + (size_t)n * a.ldw_n] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; kk++) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; i++) av[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; j++) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; i++) {
    int m = m0 + ty * 4 + i;
    if (m >= a.M) continue;
#pragma unroll
    for (int j = 0; j < 4; j++) {
      int n = n0 + tx * 4 + j;
      if (n >= a.Nout) continue;
      float v = acc[i][j];
      if (a.bias) v += a.bias[n];
      if (a.epi == EPI_MASK) v = a.aux[(size_t)m * a.ldaux + n] > 0.f ? v : 0.f;
      else v = apply_epi(a.epi, v);
      if (a.R) v += a.R[(size_t)m * a.ldr + n];
      float *dst;
      if (n < a.split) dst = a.Y + (size_t)m * a.ldy + n;
      else dst = a.Y2 + (size_t)m * a.ldy2 + (n - a.split);
      if (a.accumulate) v += *dst;
      *dst = v;
    }
  }
}

// ---- wgrad: partial[chunk][k][n] = sum_{rows in chunk} Xaug[r][k] dY[r][n]
// The grid covers the K real input columns; the bias row (Xaug's column K of ones) is the
// column sum of dY, accumulated by the ty == 0 threads of the blockIdx.x == 0 blocks, so it
// costs no extra 64-wide K tile.  Rows per chunk (rpc, a multiple of BK) are chosen on the
// host so that the grid holds about 2 blocks per SM; fixed per shape, hence deterministic.
constexpr int WK = 32;   // rows of X / dY per k_wgrad stage
__global__ void __launch_bounds__(NT, 3) k_wgrad(int M, int K, int Kaug, int Nout, const float *X1, int ldx1,
                                                 int K1, const float *X2, int ldx2, const float *dY, int ldy,
                                                 float *part, int rpc) {
  __shared__ float Xs[WK][BM + 4];
  __shared__ float Ys[WK][BN + 4];
  const int tid = threadIdx.x;
  const int k0 = blockIdx.x * BM, n0 = blockIdx.y * BN, chunk = blockIdx.z;
  const int r0 = chunk * rpc, r1 = min(M, r0 + rpc);
  const int ty = tid / 16, tx = tid % 16;
  const bool bias_rows = Kaug > K && blockIdx.x == 0 && ty == 0;
  float acc[4][4], bacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j] = 0.f;
  // the next stage's X and dY values are loaded into registers while this stage is multiplied
  constexpr int PX = (BM * WK) / NT, PY = (BN * WK) / NT;
  float xr[PX], yr[PY];
  auto fetch = [&](int rb) {
#pragma unroll
    for (int i = 0; i < PX; i++) {
      const int e = tid + i * NT, rr = e / BM, kk = e % BM;
      const int r = rb + rr, k = k0 + kk;
      xr[i] = (r < r1 && k < K) ? ((k < K1) ? X1[(size_t)r * ldx1 + k] : X2[(size_t)r * ldx2 + (k - K1)]) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < PY; i++) {
      const int e = tid + i * NT, rr = e / BN, c = e % BN;
      const int r = rb + rr, n = n0 + c;
      yr[i] = (r < r1 && n < Nout) ? dY[(size_t)r * ldy + n] : 0.f;
    }
  };
  if (r0 < r1) fetch(r0);
  for (int rb = r0; rb < r1; rb += WK) {
#pragma unroll
    for (int i = 0; i < PX; i++) {
      const int e = tid + i * NT;
      Xs[e / BM][e % BM] = xr[i];
    }
#pragma unroll
    for (int i = 0; i < PY; i++) {
      const int e = tid + i * NT;
      Ys[e / BN][e % BN] = yr[i];
    }
    __syncthreads();
    if (rb + WK < r1) fetch(rb + WK);
#pragma unroll
    for (int rr = 0; rr < WK; rr++) {
      const float4 xv = *reinterpret_cast<const float4 *>(&Xs[rr][ty * 4]);
      const float4 yv = *reinterpret_cast<const float4 *>(&Ys[rr][tx * 4]);
      const float xa[4] = {xv.x, xv.y, xv.z, xv.w}, ya[4] = {yv.x, yv.y, yv.z, yv.w};
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = fmaf(xa[i], ya[j], acc[i][j]);
      if (bias_rows) {
#pragma unroll
        for (int j = 0; j < 4; j++) bacc[j] += ya[j];
      }
    }
    __syncthreads();
  }
  float *P = part + (size_t)chunk * Kaug * Nout;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    int k = k0 + ty * 4 + i;
    if (k >= K) continue;
#pragma unroll
    for (int j = 0; j < 4; j++) {
      int n = n0 + tx * 4 + j;
      if (n < Nout) P[(size_t)k * Nout + n] = acc[i][j];
    }
  }
  if (bias_rows) {
#pragma unroll
    for (int j = 0; j < 4; j++) {
      int n = n0 + tx * 4 + j;
      if (n < Nout) P[(size_t)K * Nout + n] = bacc[j];
    }
  }
}

// out[e] (+)= sum over chunks of part[c][e]: a block takes 32 consecutive outputs (lanes:
// coalesced 128-byte loads) x 8 warps; warp w sums chunks w, w + 8, ... in order, then the 8
// partial sums are added in warp order (deterministic)
__global__ void __launch_bounds__(256) k_reduce_chunks(const float *part, int chunks, int count, float *out,
                                                       int accumulate) {
  __shared__ float red[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (e < count) {
#pragma unroll 4
    for (int c = w; c < chunks; c += 8) s += part[(size_t)c * count + e];
  }
  red[w][lane] = s;
  __syncthreads();
  if (w == 0 && e < count) {
    float t = red[0][lane];
#pragma unroll
    for (int k = 1; k < 8; k++) t += red[k][lane];
    out[e] = accumulate ? out[e] + t : t;
  }
}

// ---- LayerNorm: one warp per row of 64 (2 values per lane)
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void k_layernorm(const float *x, const float *g, const float *b, float *y, float *mu, float *rs,
                            int N) {
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= N) return;
  const float *xr = x + (size_t)w * kH;
  float v0 = xr[lane], v1 = xr[lane + 32];
  float m = warp_sum(v0 + v1) * (1.0f / kH);
  float d0 = v0 - m, d1 = v1 - m;
  float var = warp_sum(d0 * d0 + d1 * d1) * (1.0f / kH);
  float r = 1.0f / sqrtf(var + kLnEps);
  y[(size_t)w * kH + lane] = d0 * r * g[lane] + b[lane];
  y[(size_t)w * kH + lane + 32] = d1 * r * g[lane + 32] + b[lane + 32];
  if (lane == 0) {
    mu[w] = m;
    rs[w] = r;
  }
}

constexpr int LN_ROWS = 64;   // rows per block (fixed => deterministic partials; ~5 blocks per SM at C4)
__global__ void k_layernorm_bwd(const float *x, const float *mu, const float *rs, const float *g,
                                const float *da, const float *dae, float *dx, int dx_acc, const float *res,
                                float *part, int N) {
  __shared__ float red[8][128];
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int r0 = blockIdx.x * LN_ROWS, r1 = min(N, r0 + LN_ROWS);
  float pg0 = 0.f, pg1 = 0.f, pb0 = 0.f, pb1 = 0.f;
  float g0 = g[lane], g1 = g[lane + 32];
  for (int r = r0 + warp; r < r1; r += 8) {
    size_t o = (size_t)r * kH;
    float m = mu[r], rr = rs[r];
    float xh0 = (x[o + lane] - m) * rr, xh1 = (x[o + lane + 32] - m) * rr;
    float a0 = da[o + lane], a1 = da[o + lane + 32];
    float t0 = a0, t1 = a1;
    if (dae) {
      t0 += dae[o + lane];
      t1 += dae[o + lane + 32];
    }
    pg0 += t0 * xh0;
    pg1 += t1 * xh1;
    pb0 += t0;
    pb1 += t1;
    if (dx) {
      float dh0 = a0 * g0, dh1 = a1 * g1;
      float s1 = warp_sum(dh0 + dh1) * (1.0f / kH);
      float s2 = warp_sum(dh0 * xh0 + dh1 * xh1) * (1.0f / kH);
      float r0v = rr * (dh0 - s1 - xh0 * s2), r1v = rr * (dh1 - s1 - xh1 * s2);
      if (res) {   // the residual branch's gradient (x1 = x + ..., y = x1 + ...)
        r0v += res[o + lane];
        r1v += res[o + lane + 32];
      }
      if (dx_acc) {
        dx[o + lane] += r0v;
        dx[o + lane + 32] += r1v;
      } else {
        dx[o + lane] = r0v;
        dx[o + lane + 32] = r1v;
      }
    }
  }
  red[warp][lane] = pg0;
  red[warp][lane + 32] = pg1;
  red[warp][lane + 64] = pb0;
  red[warp][lane + 96] = pb1;
  __syncthreads();
  if (threadIdx.x < 128) {
    float s = 0.f;
    for (int w = 0; w < 8; w++) s += red[w][threadIdx.x];
    part[(size_t)blockIdx.x * 128 + threadIdx.x] = s;
  }
}

// column sums of an N x C matrix (C <= 256): per-block partials over LN_ROWS rows
__global__ void k_colsum_part(const float *x, int N, int C, float *part) {
  int r0 = blockIdx.x * LN_ROWS, r1 = min(N, r0 + LN_ROWS);
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float s = 0.f;
    for (int r = r0; r < r1; r++) s += x[(size_t)r * C + c];
    part[(size_t)blockIdx.x * C + c] = s;
  }
}

__global__ void k_reduce_scaled(const float *part, int chunks, int count, float scale, float *out) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= count) return;
  float s = 0.f;
  for (int c = 0; c < chunks; c++) s += part[(size_t)c * count + e];
  out[e] = s * scale;
}

__global__ void k_rows_gather(const float *src, const int *perm, float *dst, int N, int C) {
  size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)N * C) return;
  int r = (int)(e / C), c = (int)(e % C);
  dst[e] = src[(size_t)perm[r] * C + c];
}
__global__ void k_rows_scatter(const float *src, const int *perm, float *dst, int N, int C, int acc) {
  size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)N * C) return;
  int r = (int)(e / C), c = (int)(e % C);
  float *p = dst + (size_t)perm[r] * C + c;
  *p = acc ? *p + src[e] : src[e];
}
__global__ void k_tanh_grad(const float *dHn, const float *Hn, float *dP, size_t n) {
  size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  float h = Hn[e];
  dP[e] = dHn[e] * (1.f - h * h);
}
// dkvt = [dQ | dK_own + dK_mem | dV_own + dV_mem] (N x 192) from dqkv (N x 192) and dkvm (N x 128),
// one float4 per thread
__global__ void k_dkvt(const float4 *dqkv, const float4 *dkvm, float4 *dkvt, int N) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)N * 48) return;
  const size_t r = e / 48;
  const int c = (int)(e % 48);
  float4 v = dqkv[e];
  if (c >= 16) {
    const float4 m = dkvm[r * 32 + (c - 16)];
    v.x += m.x; v.y += m.y; v.z += m.z; v.w += m.w;
  }
  dkvt[e] = v;
}
__global__ void k_fill_rows(float *dst, const float *row, float scale, int N, int C) {
  size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)N * C) return;
  dst[e] = row[e % C] * scale;
}

inline unsigned nblk(size_t n, int t) { return (unsigned)((n + t - 1) / t); }
}  // namespace

static thread_local bool t_tc = false, t_tc_attn = false;
void set_tensor_cores(int mode) { t_tc = mode != 0; t_tc_attn = mode == 1; }
bool tensor_cores_on() { return t_tc; }
bool tensor_core_attention_on() { return t_tc_attn; }
static thread_local bool t_noattn = false;
void set_no_attention(bool on) { t_noattn = on; }
bool no_attention() { return t_noattn; }

static int num_sms_dense() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

void launch_gemm(const GemmArgs &a, cudaStream_t s) {
  if (a.M <= 0) return;
  if (t_tc && tc_eligible(a)) {
    launch_gemm_tc(a, s);
    return;
  }
  dim3 grid((a.M + BM - 1) / BM, (a.Nout + BN - 1) / BN);
  note_launch("k_gemm", s, gemm_bytes(a), 2.0 * a.M * a.K * a.Nout);
  k_gemm<<<grid, NT, 0, s>>>(a);
}

void launch_wgrad(int M, int K, int Nout, const float *X1, int ldx1, int K1, const float *X2, int ldx2,
                  const float *dY, int ldy, bool with_bias, float *part, size_t part_floats, float *out,
                  bool accumulate, cudaStream_t s) {
  const int Kaug = K + (with_bias ? 1 : 0);
  if (t_tc && wgrad_tc_eligible(M, K, Nout)) {   // tensor-core mode: tcgen05 split-K (tc_wgrad.cu)
    const int chunks = launch_wgrad_tc(M, K, Nout, X1, ldx1, K1, X2, ldx2, dY, ldy, with_bias, part, part_floats, s);
    if (chunks > 0) {
      const int count = Kaug * Nout;
      note_launch("k_reduce_chunks", s);
      k_reduce_chunks<<<nblk(count, 32), 256, 0, s>>>(part, chunks, count, out, accumulate ? 1 : 0);
      return;
    }
  }
  const int gx = (K + BM - 1) / BM, gy = (Nout + BN - 1) / BN;
  // about 3 blocks per SM (the launch bound), within the partial buffer, at least WK rows per chunk
  long long want = (3LL * num_sms_dense() + gx * gy - 1) / (gx * gy);
  want = std::min<long long>(want, (long long)(part_floats / ((size_t)Kaug * Nout)));
  want = std::max<long long>(1, std::min<long long>(want, (M + WK - 1) / WK));
  const int rpc = (int)(((M + want - 1) / want + WK - 1) / WK * WK);
  const int chunks = (M + rpc - 1) / rpc;
  dim3 grid(gx, gy, chunks);
  note_launch("k_wgrad", s, 4.0 * M * (K + Nout) + 4.0 * chunks * Kaug * Nout, 2.0 * M * Kaug * Nout);
  k_wgrad<<<grid, NT, 0, s>>>(M, K, Kaug, Nout, X1, ldx1, K1, X2, ldx2, dY, ldy, part, rpc);
  int count = Kaug * Nout;
  note_launch("k_reduce_chunks", s);
  k_reduce_chunks<<<nblk(count, 32), 256, 0, s>>>(part, chunks, count, out, accumulate ? 1 : 0);
}

void launch_layernorm(const float *x, const float *g, const float *b, float *y, float *mu, float *rs, int N,
                      cudaStream_t s) {
  note_launch("k_layernorm", s);
  k_layernorm<<<nblk((size_t)N * 32, 256), 256, 0, s>>>(x, g, b, y, mu, rs, N);
}

void launch_layernorm_bwd(const float *x, const float *mu, const float *rs, const float *g, const float *da,
                          const float *da_extra, float *dx, bool dx_accumulate, const float *res, float *dgb,
                          float *part, int N, cudaStream_t s) {
  int chunks = (N + LN_ROWS - 1) / LN_ROWS;
  note_launch("k_layernorm_bwd", s);
  k_layernorm_bwd<<<chunks, 256, 0, s>>>(x, mu, rs, g, da, da_extra, dx, dx_accumulate ? 1 : 0, res, part, N);
  note_launch("k_reduce_chunks", s);
  k_reduce_chunks<<<nblk(128, 32), 256, 0, s>>>(part, chunks, 128, dgb, 1);
}

void launch_colsum(const float *x, int N, int C, float scale, float *out, float *part, cudaStream_t s) {
  int chunks = (N + LN_ROWS - 1) / LN_ROWS;
  note_launch("k_colsum_part", s);
  k_colsum_part<<<chunks, 256, 0, s>>>(x, N, C, part);
  note_launch("k_reduce_scaled", s);
  k_reduce_scaled<<<nblk(C, 256), 256, 0, s>>>(part, chunks, C, scale, out);
}

void launch_rows_gather(const float *src, const int *perm, float *dst, int N, int C, cudaStream_t s) {
  note_launch("k_rows_gather", s);
  k_rows_gather<<<nblk((size_t)N * C, 256), 256, 0, s>>>(src, perm, dst, N, C);
}
void launch_rows_scatter(const float *src, const int *perm, float *dst, int N, int C, bool accumulate,
                         cudaStream_t s) {
  note_launch("k_rows_scatter", s);
  k_rows_scatter<<<nblk((size_t)N * C, 256), 256, 0, s>>>(src, perm, dst, N, C, accumulate ? 1 : 0);
}
void launch_tanh_grad(const float *dHn, const float *Hn, float *dP, int n, cudaStream_t s) {
  note_launch("k_tanh_grad", s);
  k_tanh_grad<<<nblk(n, 256), 256, 0, s>>>(dHn, Hn, dP, (size_t)n);
}
void launch_dkvt(const float *dqkv, const float *dkvm, float *dkvt, int N, cudaStream_t s) {
  note_launch("k_dkvt", s);
  k_dkvt<<<nblk((size_t)N * 48, 256), 256, 0, s>>>(reinterpret_cast<const float4 *>(dqkv),
                                                    reinterpret_cast<const float4 *>(dkvm),
                                                    reinterpret_cast<float4 *>(dkvt), N);
}
void launch_fill_rows(float *dst, const float *row, float scale, int N, int C, cudaStream_t s) {
  note_launch("k_fill_rows", s);
  k_fill_rows<<<nblk((size_t)N * C, 256), 256, 0, s>>>(dst, row, scale, N, C);
}

}  // namespace gdp
