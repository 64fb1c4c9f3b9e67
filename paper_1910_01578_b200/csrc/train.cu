// One GDP-one training update around the policy gradient:
//  * k_logprob:  one CTA per placement, log pi_b = sum over co-location leaders of
//                log p_v[D_b v] (R18), fp64 sum in a fixed order
//                (same per-node log-softmax as k_node_prep);
//  * k_greedy:   argmax decode for zero-shot placement (NEXT-2);
//  * k_sumsq:    ||g||^2 in fp64: 2 CTAs per SM, each a contiguous chunk read with 16-byte
//                loads, fixed-order block reduction -> one partial per CTA (deterministic);
//  * k_adam:     every CTA sums the partials in the same order, clip factor
//                min(1, max_norm / (||g|| + 1e-6)) (R31), then the bias-corrected
//                Adam step elementwise in fp64 on fp32 state.
// HBM-bound: 4 bytes read (k_sumsq) + 16 read + 12 written (k_adam) per parameter.
#include "common.cuh"

namespace gdp {
namespace {

constexpr int LT = 256;
__global__ void __launch_bounds__(LT) k_logprob(const float *__restrict__ logp, const int *__restrict__ leader,
                                                const uint8_t *__restrict__ D, int N, int d, float *logprob) {
  __shared__ double red[LT / 32];
  const int b = blockIdx.x;
  const uint8_t *Db = D + (size_t)b * N;
  double acc = 0.0;
  for (int v = threadIdx.x; v < N; v += LT)
    if (leader[v] == v) acc += (double)logp[(size_t)v * d + Db[v]];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < LT / 32; i++) s += red[i];
    logprob[b] = (float)s;
  }
}

// greedy decode (NEXT-2): per node the argmax of its leader's logits (strict >, so
// ties go to the lowest device id); non-leaders thereby copy their leader
__global__ void k_greedy(const float *__restrict__ logits, int ld, const int *__restrict__ leader, int N, int d,
                         uint8_t *D) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= N) return;
  const float *z = logits + (size_t)leader[v] * ld;
  int best = 0;
  float bz = z[0];
  for (int k = 1; k < d; k++)
    if (z[k] > bz) { bz = z[k]; best = k; }
  D[v] = (uint8_t)best;
}

constexpr int AT = 256;
__global__ void __launch_bounds__(AT) k_sumsq(const float *__restrict__ g, long long n, double *part) {
  __shared__ double red[AT / 32];
  const long long per = (n + gridDim.x - 1) / gridDim.x;
  const long long lo = (long long)blockIdx.x * per, hi = min(n, lo + per);
  double acc = 0.0;
  // 16-byte loads over the aligned interior, scalars at the ends
  long long a = min(hi, (lo + 3) & ~3LL), z = max(a, hi & ~3LL);
  for (long long i = lo + threadIdx.x; i < a; i += AT) acc += (double)g[i] * g[i];
  const float4 *g4 = reinterpret_cast<const float4 *>(g);
  for (long long i = a / 4 + threadIdx.x; i < z / 4; i += AT) {
    const float4 x = g4[i];
    acc += (double)x.x * x.x + (double)x.y * x.y + (double)x.z * x.z + (double)x.w * x.w;
  }
  for (long long i = z + threadIdx.x; i < hi; i += AT) acc += (double)g[i] * g[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < AT / 32; i++) s += red[i];
    part[blockIdx.x] = s;
  }
}

__device__ __forceinline__ void adam1(float &th, float &m, float &v, float g32, double scale, double lr, double b1,
                                      double b2, double eps, double c1, double c2) {
  const double g = (double)g32 * scale;
  const double mm = b1 * (double)m + (1.0 - b1) * g;
  const double vv = b2 * (double)v + (1.0 - b2) * g * g;
  th = (float)((double)th - lr * (mm * c1) / (sqrt(vv * c2) + eps));
  m = (float)mm;
  v = (float)vv;
}

__global__ void __launch_bounds__(AT) k_adam(const float *__restrict__ g, long long n, const double *__restrict__ part,
                                             int nparts, double max_norm, double lr, double b1, double b2, double eps,
                                             double c1, double c2, float *theta, float *m, float *v,
                                             double *norm_out) {
  __shared__ double s_scale;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < nparts; i++) s += part[i];   // same order in every CTA
    const double norm = sqrt(s);
    const double f = max_norm / (norm + 1e-6);
    // a non-finite gradient (NaN, or Inf: Inf * 0 = NaN) leaves theta, m and v untouched; the
    // norm reports it (gdp_grad_check names the parameter)
    s_scale = isfinite(norm) ? (f < 1.0 ? f : 1.0) : -1.0;
    if (blockIdx.x == 0 && norm_out) *norm_out = norm;
  }
  __syncthreads();
  const double scale = s_scale;
  if (scale < 0.0) return;
  const long long n4 = n / 4;
  float4 *t4 = reinterpret_cast<float4 *>(theta), *m4 = reinterpret_cast<float4 *>(m),
         *v4 = reinterpret_cast<float4 *>(v);
  const float4 *g4 = reinterpret_cast<const float4 *>(g);
  for (long long i = (long long)blockIdx.x * AT + threadIdx.x; i < n4; i += (long long)gridDim.x * AT) {
    float4 th = t4[i], mm = m4[i], vv = v4[i];
    const float4 gg = g4[i];
    adam1(th.x, mm.x, vv.x, gg.x, scale, lr, b1, b2, eps, c1, c2);
    adam1(th.y, mm.y, vv.y, gg.y, scale, lr, b1, b2, eps, c1, c2);
    adam1(th.z, mm.z, vv.z, gg.z, scale, lr, b1, b2, eps, c1, c2);
    adam1(th.w, mm.w, vv.w, gg.w, scale, lr, b1, b2, eps, c1, c2);
    t4[i] = th;
    m4[i] = mm;
    v4[i] = vv;
  }
  for (long long i = 4 * n4 + (long long)blockIdx.x * AT + threadIdx.x; i < n; i += (long long)gridDim.x * AT)
    adam1(theta[i], m[i], v[i], g[i], scale, lr, b1, b2, eps, c1, c2);
}

// index of the first non-finite gradient entry (atomicMin; n if none)
__global__ void k_first_nonfinite(const float *__restrict__ g, long long n, unsigned long long *first) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (!isfinite(g[i])) atomicMin(first, (unsigned long long)i);
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace

int adam_parts() { return 2 * sm_count() < kAdamScratch ? 2 * sm_count() : kAdamScratch; }

void launch_greedy(const float *logits, int ld, const int *leader, int N, int d, uint8_t *D, cudaStream_t s) {
  note_launch("k_greedy", s);
  k_greedy<<<(N + 255) / 256, 256, 0, s>>>(logits, ld, leader, N, d, D);
}

void launch_logprob(const float *logp, const int *leader, const uint8_t *D, int N, int d, int B, float *logprob,
                    cudaStream_t s) {
  note_launch("k_logprob", s);
  k_logprob<<<B, LT, 0, s>>>(logp, leader, D, N, d, logprob);
}

long long first_nonfinite(const float *g, long long n, unsigned long long *scratch, cudaStream_t s) {
  unsigned long long h = (unsigned long long)n;
  if (cudaMemcpyAsync(scratch, &h, sizeof(h), cudaMemcpyHostToDevice, s) != cudaSuccess) return -1;
  note_launch("k_first_nonfinite", s);
  k_first_nonfinite<<<2 * sm_count(), 256, 0, s>>>(g, n, scratch);
  if (cudaMemcpyAsync(&h, scratch, sizeof(h), cudaMemcpyDeviceToHost, s) != cudaSuccess) return -1;
  if (cudaStreamSynchronize(s) != cudaSuccess) return -1;
  return (long long)h;
}

// out = sum_i grads[i] in the fixed order i = 0, 1, ... (deterministic), 16-byte vectors
struct GradPtrs {
  const float *p[16];
};
__global__ void k_grad_sum(GradPtrs P, int n, long long len, int first, float *out) {
  const long long n4 = len / 4;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    float4 acc = first ? make_float4(0.f, 0.f, 0.f, 0.f) : reinterpret_cast<const float4 *>(out)[i];
    for (int k = 0; k < n; k++) {
      const float4 x = reinterpret_cast<const float4 *>(P.p[k])[i];
      acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
    }
    reinterpret_cast<float4 *>(out)[i] = acc;
  }
  for (long long i = 4 * n4 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < len;
       i += (long long)gridDim.x * blockDim.x) {
    float acc = first ? 0.f : out[i];
    for (int k = 0; k < n; k++) acc += P.p[k][i];
    out[i] = acc;
  }
}

void launch_grad_sum(const float *const *grads, int n, long long len, float *out, cudaStream_t s) {
  for (int k0 = 0; k0 < n; k0 += 16) {
    GradPtrs P;
    const int m = n - k0 < 16 ? n - k0 : 16;
    for (int k = 0; k < m; k++) P.p[k] = grads[k0 + k];
    note_launch("k_grad_sum", s, 4.0 * (double)len * (m + 1 + (k0 ? 1 : 0)));
    k_grad_sum<<<2 * sm_count(), 256, 0, s>>>(P, m, len, k0 == 0, out);
  }
}

void launch_clip_adam(const float *g, long long n, double max_norm, double lr, double b1, double b2, double eps,
                      double c1, double c2, float *theta, float *m, float *v, double *scratch, double *norm_out,
                      cudaStream_t s) {
  const int parts = adam_parts();
  note_launch("k_sumsq", s);
  k_sumsq<<<parts, AT, 0, s>>>(g, n, scratch);
  note_launch("k_adam", s);
  k_adam<<<parts, AT, 0, s>>>(g, n, scratch, parts, max_norm, lr, b1, b2, eps, c1, c2, theta, m, v, norm_out);
}

}  // namespace gdp
