// The policy network pi_theta of GDP: orchestration of gdp_embed (§3.1), gdp_place
// (§3.2-3.3) and gdp_policy_grad (§3 PPO gradient, hand-derived backward), plus the
// superposition gate kernels (Eq. 4).  Everything runs on `stream`; nothing is
// allocated here (all scratch is carved from the caller's workspace).
#include "common.cuh"

namespace gdp {

// theta offsets (computed by gdp_param_layout in api.cu)
extern void param_offsets(int F, int d, long long *off, bool ar);

namespace {

struct GateMap {            // one gated dense map
  int offP, offq;           // gate projection P (64 x w), q (w)
  int width;                // w = fan-in of the gated weight
  int goff;                 // offset of gamma_j inside the 1216-vector
};
struct GateTable { GateMap m[kGateCount]; };

// one thread per gate entry (kGamTotal of them over the 13 maps): gamma = 2 sigma(q + z P)
__global__ void k_gates(const float *theta, const float *z, GateTable T, float *gam) {
  __shared__ float sz[kH];
  if (threadIdx.x < kH) sz[threadIdx.x] = z[threadIdx.x];
  __syncthreads();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= kGamTotal) return;
  int j = 0;
  while (j + 1 < kGateCount && T.m[j + 1].goff <= t) j++;
  const GateMap g = T.m[j];
  const int i = t - g.goff;
  float s = theta[g.offq + i];
#pragma unroll 16
  for (int k = 0; k < kH; k++) s = fmaf(sz[k], theta[g.offP + k * g.width + i], s);
  gam[t] = 2.f / (1.f + expf(-s));
}

// W' = diag(gamma) W for one Transformer-XL layer (gamma pointers nullable -> 1).
struct FoldArgs {
  const float *theta;
  int oWq, obq, oWk, obk, oWv, obv, oWo, oW1, oW2;
  const float *gq, *gk, *gv, *go, *g1, *g2;
  float *Wqkv, *bqkv, *Wo, *W1, *W2;
};
__global__ void k_fold_layer(FoldArgs a) {
  const int n0 = 64 * 192, n1 = n0 + 192, n2 = n1 + 64 * 64, n3 = n2 + 64 * 256, n4 = n3 + 256 * 64;
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n4) return;
  const float *th = a.theta;
  if (e < n0) {
    int i = e / 192, c = e % 192, blk = c / 64, cc = c % 64;
    int off = blk == 0 ? a.oWq : (blk == 1 ? a.oWk : a.oWv);
    const float *g = blk == 0 ? a.gq : (blk == 1 ? a.gk : a.gv);
    a.Wqkv[e] = th[off + i * 64 + cc] * (g ? g[i] : 1.f);
  } else if (e < n1) {
    int c = e - n0, blk = c / 64, cc = c % 64;
    int off = blk == 0 ? a.obq : (blk == 1 ? a.obk : a.obv);
    a.bqkv[c] = th[off + cc];
  } else if (e < n2) {
    int f = e - n1, i = f / 64;
    a.Wo[f] = th[a.oWo + f] * (a.go ? a.go[i] : 1.f);
  } else if (e < n3) {
    int f = e - n2, i = f / 256;
    a.W1[f] = th[a.oW1 + f] * (a.g1 ? a.g1[i] : 1.f);
  } else {
    int f = e - n3, i = f / 64;
    a.W2[f] = th[a.oW2 + f] * (a.g2 ? a.g2[i] : 1.f);
  }
}
__global__ void k_fold_head(const float *theta, int oW, int d, const float *gh, float *Wh) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= kH * d) return;
  Wh[e] = theta[oW + e] * (gh ? gh[e / d] : 1.f);
}

// Gate backward, step 1: per (map, row i): grad W_j[i,:] += gamma_i dW'_j[i,:];
// dgamma_i = sum_c W_j[i,c] dW'_j[i,c];  dpre_i = dgamma_i gamma_i (1 - gamma_i / 2);
// the augmented bias row of dW' goes to grad b_j.
struct RowMap {
  const float *dW;   // augmented temp, row stride ld, columns [col0, col0 + ncols)
  int ld, col0, ncols, fan_in;
  int offW, offb;
  const float *gam;  // nullable (gamma == 1, no gate gradient)
  float *dpre;       // nullable
};
struct RowTable { RowMap m[16]; int count; };
// one warp per row (lanes over the row's columns, coalesced); dgamma_i summed lane-strided then by
// a fixed xor butterfly (deterministic)
__global__ void k_gate_bwd_rows(const float *theta, RowTable T, float *grad) {
  int j = blockIdx.y;
  if (j >= T.count) return;
  const RowMap r = T.m[j];
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i > r.fan_in) return;
  const float *src = r.dW + (size_t)i * r.ld + r.col0;
  if (i == r.fan_in) {   // bias row
    for (int c = lane; c < r.ncols; c += 32) grad[r.offb + c] += src[c];
    return;
  }
  const float g = r.gam ? r.gam[i] : 1.f;
  float dg = 0.f;
  for (int c = lane; c < r.ncols; c += 32) {
    const float dw = src[c];
    dg = fmaf(theta[r.offW + i * r.ncols + c], dw, dg);
    grad[r.offW + i * r.ncols + c] += g * dw;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dg += __shfl_xor_sync(0xffffffffu, dg, o);
  if (lane == 0 && r.gam && r.dpre) r.dpre[i] = dg * g * (1.f - 0.5f * g);
}

// step 2: grad P_j[k,i] += z_k dpre_j[i], grad q_j[i] += dpre_j[i]
__global__ void k_gate_bwd_P(const float *z, const float *dpre, GateTable T, float *grad) {
  int j = blockIdx.y;
  const GateMap g = T.m[j];
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (kH + 1) * g.width) return;
  int k = e / g.width, i = e % g.width;
  float dp = dpre[g.goff + i];
  if (k < kH) grad[g.offP + k * g.width + i] += z[k] * dp;
  else grad[g.offq + i] += dp;
}

// step 3: dz_k = sum_j sum_i P_j[k,i] dpre_j[i] (fixed order), then scaled by 1/N
// one block per k: threads take gate entries t, t + 256, ... (fixed), then a fixed smem tree
__global__ void k_gate_bwd_z(const float *theta, const float *dpre, GateTable T, float invN, float *dzN) {
  __shared__ float red[256];
  const int k = blockIdx.x;
  float s = 0.f;
  for (int t = threadIdx.x; t < kGamTotal; t += blockDim.x) {
    int j = 0;
    while (j + 1 < kGateCount && T.m[j + 1].goff <= t) j++;
    const GateMap g = T.m[j];
    const int i = t - g.goff;
    s = fmaf(theta[g.offP + k * g.width + i], dpre[t], s);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) dzN[k] = red[0] * invN;
}

inline unsigned nblk(size_t n, int t) { return (unsigned)((n + t - 1) / t); }

GemmArgs gemm(int M, int K, int Nout, const float *X, int ldx, const float *W, int ldw_k, int ldw_n, float *Y,
              int ldy) {
  GemmArgs a{};
  a.M = M; a.K = K; a.Nout = Nout;
  a.X1 = X; a.ldx1 = ldx; a.K1 = K;
  a.X2 = nullptr; a.ldx2 = 0;
  a.W = W; a.ldw_k = ldw_k; a.ldw_n = ldw_n;
  a.bias = nullptr; a.R = nullptr; a.ldr = 0; a.aux = nullptr; a.ldaux = 0;
  a.Y = Y; a.ldy = ldy; a.split = Nout; a.Y2 = nullptr; a.ldy2 = 0;
  a.accumulate = 0; a.epi = EPI_NONE;
  return a;
}

struct Offs {
  long long o[GDP_P_COUNT + 1];
  long long operator[](int i) const { return o[i]; }
};

int layer_base(int l) {   // first param id of XL layer l (0 = cond, 1 = xl0, 2 = xl1)
  return l == 0 ? GDP_P_COND_LN1_G : (l == 1 ? GDP_P_XL0_LN1_G : GDP_P_XL1_LN1_G);
}
enum { LN1G = 0, LN1B, WQ, BQ, WK, BK, WV, BV, WO, BO, LN2G, LN2B, W1, B1, W2, B2 };

GateTable gate_table(const Offs &off) {
  GateTable T;
  int goff = 0;
  for (int l = 0; l < 2; l++) {
    int base = l == 0 ? GDP_P_GATE0_Q_P : GDP_P_GATE1_Q_P;
    for (int j = 0; j < 6; j++) {
      GateMap &g = T.m[l * 6 + j];
      g.offP = (int)off[base + 2 * j];
      g.offq = (int)off[base + 2 * j + 1];
      g.width = j == 5 ? kFFN : kH;
      g.goff = goff;
      goff += g.width;
    }
  }
  T.m[12].offP = (int)off[GDP_P_GATE_HEAD_P];
  T.m[12].offq = (int)off[GDP_P_GATE_HEAD_Q];
  T.m[12].width = kH;
  T.m[12].goff = goff;
  return T;
}

const float *gam_of(const WS &w, const GateTable &T, int layer /*0,1*/, int j) {
  return w.gam + T.m[layer * 6 + j].goff;
}

void fold_layer(const WS &w, const Offs &off, const float *theta, int l, const float *const *g, cudaStream_t s) {
  const Layer &L = w.L[l];
  const int b = layer_base(l);
  FoldArgs a;
  a.theta = theta;
  a.oWq = (int)off[b + WQ]; a.obq = (int)off[b + BQ];
  a.oWk = (int)off[b + WK]; a.obk = (int)off[b + BK];
  a.oWv = (int)off[b + WV]; a.obv = (int)off[b + BV];
  a.oWo = (int)off[b + WO]; a.oW1 = (int)off[b + W1]; a.oW2 = (int)off[b + W2];
  a.gq = g ? g[0] : nullptr; a.gk = g ? g[1] : nullptr; a.gv = g ? g[2] : nullptr;
  a.go = g ? g[3] : nullptr; a.g1 = g ? g[4] : nullptr; a.g2 = g ? g[5] : nullptr;
  a.Wqkv = L.Wqkv; a.bqkv = L.bqkv; a.Wo = L.Wo; a.W1 = L.W1; a.W2 = L.W2;
  const int n = 64 * 192 + 192 + 64 * 64 + 64 * 256 + 256 * 64;
  note_launch("k_fold_layer", s);
  k_fold_layer<<<nblk(n, 256), 256, 0, s>>>(a);
}

// one Transformer-XL layer forward over x (topological order), weights already folded
void layer_fwd(const WS &w, const Offs &off, const float *theta, int l, const float *x, int N, int S, int M,
               cudaStream_t s) {
  Layer L = w.L[l];
  const int b = layer_base(l);
  launch_layernorm(x, theta + off[b + LN1G], theta + off[b + LN1B], L.a, L.mu1, L.rs1, N, s);
  GemmArgs g = gemm(N, kH, 192, L.a, kH, L.Wqkv, 192, 1, L.qkv, 192);
  g.bias = L.bqkv;
  launch_gemm(g, s);
  if (no_attention()) launch_relu_v(L.qkv, L.o, N, s);
  else launch_attn_fwd(L.qkv, L.o, L.lse, N, S, M, s);
  g = gemm(N, kH, kH, L.o, kH, L.Wo, kH, 1, L.x1, kH);
  g.bias = theta + off[b + BO];
  g.R = x; g.ldr = kH;
  launch_gemm(g, s);
  launch_layernorm(L.x1, theta + off[b + LN2G], theta + off[b + LN2B], L.c, L.mu2, L.rs2, N, s);
  g = gemm(N, kH, kFFN, L.c, kH, L.W1, kFFN, 1, L.m, kFFN);
  g.bias = theta + off[b + B1];
  g.epi = EPI_RELU;
  launch_gemm(g, s);
  g = gemm(N, kFFN, kH, L.m, kFFN, L.W2, kH, 1, L.y, kH);
  g.bias = theta + off[b + B2];
  g.R = L.x1; g.ldr = kH;
  launch_gemm(g, s);
}

// one Transformer-XL layer backward: dy -> dx (dx = or += ); weight gradients of the folded
// maps land in L.dW* (augmented with the bias row); LN gradients go straight to grad.
void layer_bwd(const WS &w, const Offs &off, const float *theta, int l, const float *x, const float *dy,
               float *dx, bool dx_acc, float *grad, int N, int S, int M, cudaStream_t s) {
  const Layer L = w.L[l];
  const int b = layer_base(l);
  // FFN: y = x1 + m W2' + b2, m = relu(c W1' + b1)
  GemmArgs g = gemm(N, kH, kFFN, dy, kH, L.W2, 1, kH, w.dm, kFFN);   // dm = dy W2'^T, masked by m > 0
  g.epi = EPI_MASK; g.aux = L.m; g.ldaux = kFFN;
  launch_gemm(g, s);
  launch_wgrad(N, kFFN, kH, L.m, kFFN, kFFN, nullptr, 0, dy, kH, true, w.part, w.part_floats, L.dW2, false, s);
  g = gemm(N, kFFN, kH, w.dm, kFFN, L.W1, 1, kFFN, w.dc, kH);       // dc = dm W1'^T
  launch_gemm(g, s);
  launch_wgrad(N, kH, kFFN, L.c, kH, kH, nullptr, 0, w.dm, kFFN, true, w.part, w.part_floats, L.dW1, false, s);
  // x1 -> LN2 -> c: dx1 = dy + LN2_bwd(dc)
  launch_layernorm_bwd(L.x1, L.mu2, L.rs2, theta + off[b + LN2G], w.dc, nullptr, w.dx1, false, dy,
                       grad + off[b + LN2G], w.part, N, s);
  // x1 = x + o Wo' + bo
  g = gemm(N, kH, kH, w.dx1, kH, L.Wo, 1, kH, w.dout, kH);          // do = dx1 Wo'^T
  launch_gemm(g, s);
  launch_wgrad(N, kH, kH, L.o, kH, kH, nullptr, 0, w.dx1, kH, true, w.part, w.part_floats, L.dWo, false, s);
  // attention backward: dqkv = [dQ | dK_own | dV_own], dkvm = [dK_mem | dV_mem]
  if (no_attention()) launch_relu_v_bwd(L.qkv, w.dout, w.dqkv, w.dkvm, N, s);
  else launch_attn_bwd(L.qkv, L.o, L.lse, w.dout, w.dqkv, w.dkvm, w.dd, N, S, M, s);
  // totals for the parameter gradients: dkvt = [dQ | dK_own + dK_mem | dV_own + dV_mem]
  launch_dkvt(w.dqkv, w.dkvm, w.dkvt, N, s);
  launch_wgrad(N, kH, 192, L.a, kH, kH, nullptr, 0, w.dkvt, 192, true, w.part, w.part_floats, L.dWqkv, false, s);
  // da (own rows, flows into x) and dam (memory rows: parameters only, stop-gradient)
  g = gemm(N, 192, kH, w.dqkv, 192, L.Wqkv, 1, 192, w.da, kH);
  launch_gemm(g, s);
  g = gemm(N, 128, kH, w.dkvm, 128, L.Wqkv + 64, 1, 192, w.dam, kH);
  launch_gemm(g, s);
  launch_layernorm_bwd(x, L.mu1, L.rs1, theta + off[b + LN1G], w.da, w.dam, dx, dx_acc, w.dx1,
                       grad + off[b + LN1G], w.part, N, s);
}

void add_layer_rows(RowTable &T, const WS &w, const Offs &off, int l, const float *const *g, float *dpre_base,
                    const GateTable &GT, int gl) {
  const Layer &L = w.L[l];
  const int b = layer_base(l);
  const int ids[6][2] = {{WQ, BQ}, {WK, BK}, {WV, BV}, {WO, BO}, {W1, B1}, {W2, B2}};
  for (int j = 0; j < 6; j++) {
    RowMap &r = T.m[T.count++];
    r.offW = (int)off[b + ids[j][0]];
    r.offb = (int)off[b + ids[j][1]];
    r.gam = g ? g[j] : nullptr;
    r.dpre = (g && dpre_base) ? dpre_base + GT.m[gl * 6 + j].goff : nullptr;
    if (j < 3) { r.dW = L.dWqkv; r.ld = 192; r.col0 = 64 * j; r.ncols = 64; r.fan_in = 64; }
    else if (j == 3) { r.dW = L.dWo; r.ld = 64; r.col0 = 0; r.ncols = 64; r.fan_in = 64; }
    else if (j == 4) { r.dW = L.dW1; r.ld = 256; r.col0 = 0; r.ncols = 256; r.fan_in = 64; }
    else { r.dW = L.dW2; r.ld = 64; r.col0 = 0; r.ncols = 64; r.fan_in = 256; }
  }
}

void run_rows(const RowTable &T, const float *theta, float *grad, cudaStream_t s) {
  if (T.count == 0) return;
  dim3 grid(nblk(257, 8), T.count);   // 8 rows (warps) per block, fan-in + bias row <= 257
  note_launch("k_gate_bwd_rows", s);
  k_gate_bwd_rows<<<grid, 256, 0, s>>>(theta, T, grad);
}

}  // namespace

// ------------------------------------------------------------------ entry-point bodies
gdp_status run_embed(const gdp_graph_s *g, const float *theta, float *node_emb, const WS &w, int d,
                     cudaStream_t s) {
  Offs off;
  param_offsets(g->F, d, off.o, false);   // the GNN's offsets do not depend on the head
  const int N = g->N;
  // H0 = X W_in + b_in (affine input projection)
  GemmArgs a = gemm(N, g->F, kH, g->X, g->ldX, theta + off[GDP_P_GNN_IN_W], kH, 1, w.H[0], kH);
  a.bias = theta + off[GDP_P_GNN_IN_B];
  launch_gemm(a, s);
  for (int l = 0; l < kGNN; l++) {
    const int pW = GDP_P_GNN_0_W + 4 * l;
    // Z = sigmoid(H W + b), computed once per node (Eq. 2 inner affine + sigma)
    a = gemm(N, kH, kH, w.H[l], kH, theta + off[pW], kH, 1, w.Z[l], kH);
    a.bias = theta + off[pW + 1];
    a.epi = EPI_SIGMOID;
    launch_gemm(a, s);
    launch_gather_max(w.Z[l], g->nbr_ptr, g->nbr_idx, g->heavy, g->n_heavy, w.A[l], w.ARG[l], N, g->E_sym, s);
    // H' = tanh([H | A] W_f + b_f) (Eq. 3)
    float *out = (l == kGNN - 1) ? w.H[3] : w.H[l + 1];
    a = gemm(N, 2 * kH, kH, w.H[l], kH, theta + off[pW + 2], kH, 1, out, kH);
    a.K1 = kH; a.X2 = w.A[l]; a.ldx2 = kH;
    a.bias = theta + off[pW + 3];
    a.epi = EPI_TANH;
    launch_gemm(a, s);
  }
  GDP_CUDA_CHECK(cudaMemcpyAsync(node_emb, w.H[3], (size_t)N * kH * sizeof(float), cudaMemcpyDeviceToDevice, s));
  GDP_LAUNCH_CHECK("gdp_embed");
  return GDP_OK;
}

gdp_status run_place(const gdp_graph_s *g, const gdp_config *c, const float *theta, const float *node_emb,
                     float *logits, const WS &w, cudaStream_t s) {
  Offs off;
  const int d = c->num_devices, N = g->N, S = c->seg_len, M = c->mem_len;
  param_offsets(g->F, d, off.o, c->autoregressive != 0);
  if (g->perm_identity)
    GDP_CUDA_CHECK(cudaMemcpyAsync(w.Etopo, node_emb, (size_t)N * kH * sizeof(float), cudaMemcpyDeviceToDevice, s));
  else
    launch_rows_gather(node_emb, g->perm, w.Etopo, N, kH, s);
  const GateTable GT = gate_table(off);
  const float *g0[6], *g1[6];
  const float *gh = nullptr;
  const bool sup = c->superposition != 0;
  if (sup) {
    // conditioner: one extra Transformer-XL layer, mean over nodes, gates (Eq. 4)
    fold_layer(w, off, theta, 0, nullptr, s);
    layer_fwd(w, off, theta, 0, w.Etopo, N, S, M, s);
    launch_colsum(w.L[0].y, N, kH, 1.0f / (float)N, w.z, w.part, s);
    note_launch("k_gates", s);
    k_gates<<<nblk(kGamTotal, 128), 128, 0, s>>>(theta, w.z, GT, w.gam);
    for (int j = 0; j < 6; j++) { g0[j] = gam_of(w, GT, 0, j); g1[j] = gam_of(w, GT, 1, j); }
    gh = w.gam + GT.m[12].goff;
  }
  fold_layer(w, off, theta, 1, sup ? g0 : nullptr, s);
  fold_layer(w, off, theta, 2, sup ? g1 : nullptr, s);
  note_launch("k_fold_head", s);
  k_fold_head<<<nblk(kH * d, 256), 256, 0, s>>>(theta, (int)off[GDP_P_HEAD_W], d, gh, w.Wh);
  layer_fwd(w, off, theta, 1, w.Etopo, N, S, M, s);
  layer_fwd(w, off, theta, 2, w.L[1].y, N, S, M, s);
  GemmArgs a = gemm(N, kH, d, w.L[2].y, kH, w.Wh, d, 1, g->perm_identity ? logits : w.logits_topo, d);
  a.bias = theta + off[GDP_P_HEAD_B];
  launch_gemm(a, s);
  if (!g->perm_identity) launch_rows_scatter(w.logits_topo, g->perm, logits, N, d, false, s);
  if (c->autoregressive)   // R35: EW = E Wh' behind the base logits
    launch_ar_table(theta + off[GDP_P_AR_E], w.Wh, d, logits + (size_t)N * d, s);
  GDP_LAUNCH_CHECK("gdp_place");
  return GDP_OK;
}

gdp_status run_policy_grad(const gdp_graph_s *g, const gdp_config *c, const float *theta, const float *logits,
                           const uint8_t *D, int B, const double *adv, const float *logprob,
                           const float *old_logprob, float eps, float beta, float scale, float *grad, const WS &w,
                           cudaStream_t s, cudaEvent_t const *bucket_done) {
  // bucket_done (nullable): events recorded as the gradient buckets become final, in the order
  // the backward completes them -- [xl0 .. head] (placement layers, gates, head), the
  // conditioner, the GNN (gdp_grad_buckets) -- so that their all-reduce can start early
  auto mark = [&](int i) {
    if (bucket_done && bucket_done[i]) cudaEventRecord(bucket_done[i], s);
  };
  Offs off;
  const int d = c->num_devices, N = g->N, S = c->seg_len, M = c->mem_len;
  param_offsets(g->F, d, off.o, c->autoregressive != 0);
  const bool sup = c->superposition != 0;
  const GateTable GT = gate_table(off);
  // a14: dL/dlogits (caller order) -> topological order
  const bool ar = c->autoregressive != 0;
  const float *dlt = w.dlog;
  if (ar) {   // R35: dL/dbase straight into topological rows, dL/dEW into w.dEW
    launch_ar_grad(logits, g->perm, g->leader, N, d, S, B, D, adv, logprob, old_logprob, eps, beta, scale, w.wb,
                   w.lpart, w.part, w.part_floats, w.dlog_topo, w.dEW, s);
    dlt = w.dlog_topo;
  } else {
    launch_logit_grad(logits, d, D, g->leader, adv, logprob, old_logprob, eps, beta, scale, N, active_devices(c), B,
                      w.wb, w.lpart, w.dlog, s);
    if (!g->perm_identity) {
      launch_rows_gather(w.dlog, g->perm, w.dlog_topo, N, d, s);
      dlt = w.dlog_topo;
    }
  }
  // head: logits = y2 Wh' + bh
  launch_wgrad(N, kH, d, w.L[2].y, kH, kH, nullptr, 0, dlt, d, true, w.part, w.part_floats, w.dWh, false, s);
  if (ar)   // EW = E Wh': dWh' += E^T dEW, grad[E] += dEW Wh'^T
    launch_ar_head_bwd(theta + off[GDP_P_AR_E], w.Wh, w.dEW, d, w.dWh, grad + off[GDP_P_AR_E], s);
  GemmArgs a = gemm(N, d, kH, dlt, d, w.Wh, 1, d, w.dy, kH);
  launch_gemm(a, s);
  // placement layers (reverse order)
  layer_bwd(w, off, theta, 2, w.L[1].y, w.dy, w.dxa, false, grad, N, S, M, s);
  layer_bwd(w, off, theta, 1, w.Etopo, w.dxa, w.dEt, false, grad, N, S, M, s);
  // folded-weight gradients -> W, b and the gates
  RowTable RT;
  RT.count = 0;
  const float *g0[6], *g1[6];
  for (int j = 0; j < 6; j++) { g0[j] = gam_of(w, GT, 0, j); g1[j] = gam_of(w, GT, 1, j); }
  add_layer_rows(RT, w, off, 1, sup ? g0 : nullptr, w.dgam, GT, 0);
  add_layer_rows(RT, w, off, 2, sup ? g1 : nullptr, w.dgam, GT, 1);
  {
    RowMap &r = RT.m[RT.count++];
    r.dW = w.dWh; r.ld = d; r.col0 = 0; r.ncols = d; r.fan_in = kH;
    r.offW = (int)off[GDP_P_HEAD_W]; r.offb = (int)off[GDP_P_HEAD_B];
    r.gam = sup ? w.gam + GT.m[12].goff : nullptr;
    r.dpre = sup ? w.dgam + GT.m[12].goff : nullptr;
  }
  run_rows(RT, theta, grad, s);
  if (!sup) { mark(0); mark(1); }   // no conditioner: its gradient stays zero
  if (sup) {
    dim3 gp(nblk((kH + 1) * kFFN, 256), kGateCount);
    note_launch("k_gate_bwd_P", s);
    k_gate_bwd_P<<<gp, 256, 0, s>>>(w.z, w.dgam, GT, grad);
    mark(0);
    note_launch("k_gate_bwd_z", s);
    k_gate_bwd_z<<<kH, 256, 0, s>>>(theta, w.dgam, GT, 1.0f / (float)N, w.dz);
    // conditioner: z = mean_v C_v -> dC_v = dz / N for every node
    launch_fill_rows(w.dy, w.dz, 1.0f, N, kH, s);
    layer_bwd(w, off, theta, 0, w.Etopo, w.dy, w.dEt, true, grad, N, S, M, s);
    RowTable RC;
    RC.count = 0;
    add_layer_rows(RC, w, off, 0, nullptr, nullptr, GT, 0);
    run_rows(RC, theta, grad, s);
    mark(1);
  }
  // back to caller order
  const float *dE = w.dEt;
  if (!g->perm_identity) {
    launch_rows_scatter(w.dEt, g->perm, w.dE, N, kH, false, s);
    dE = w.dE;
  }
  // GNN backward (Eq. 3 then Eq. 2), layers in reverse
  const float *dHn = dE;
  float *bufs[2] = {w.dH, w.dHn};
  for (int l = kGNN - 1; l >= 0; l--) {
    const int pW = GDP_P_GNN_0_W + 4 * l;
    const float *Hn = (l == kGNN - 1) ? w.H[3] : w.H[l + 1];
    launch_tanh_grad(dHn, Hn, w.dP, N * kH, s);
    launch_wgrad(N, 2 * kH, kH, w.H[l], kH, kH, w.A[l], kH, w.dP, kH, true, w.part, w.part_floats,
                 grad + off[pW + 2], true, s);
    float *dH = bufs[l & 1];
    a = gemm(N, kH, 2 * kH, w.dP, kH, theta + off[pW + 2], 1, kH, dH, kH);   // [dH | dA] = dP Wf^T
    a.split = kH; a.Y2 = w.dAg; a.ldy2 = kH;
    launch_gemm(a, s);
    launch_gather_max_bwd(w.dAg, w.ARG[l], w.Z[l], g->nbr_ptr, g->nbr_idx, g->heavy, g->n_heavy, w.dP, N, g->E_sym, s);   // dP := dpre
    launch_wgrad(N, kH, kH, w.H[l], kH, kH, nullptr, 0, w.dP, kH, true, w.part, w.part_floats, grad + off[pW],
                 true, s);
    a = gemm(N, kH, kH, w.dP, kH, theta + off[pW], 1, kH, dH, kH);             // dH += dpre W^T
    a.accumulate = 1;
    launch_gemm(a, s);
    dHn = dH;
  }
  launch_wgrad(N, g->F, kH, g->X, g->ldX, g->F, nullptr, 0, dHn, kH, true, w.part, w.part_floats,
               grad + off[GDP_P_GNN_IN_W], true, s);
  mark(2);
  GDP_LAUNCH_CHECK("gdp_policy_grad");
  return GDP_OK;
}

}  // namespace gdp
