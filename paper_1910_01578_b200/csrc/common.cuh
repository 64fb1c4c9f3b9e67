// Internal declarations of libgdp.so (the product).  Shares nothing with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/gdp.h"

namespace gdp {

constexpr int kH = 64;       // hidden size h
constexpr int kHeads = 4;
constexpr int kDH = 16;      // head dim
constexpr int kFFN = 256;
constexpr int kGNN = 3;
constexpr int kMaxD = 8;
constexpr float kLnEps = 1e-5f;

void set_error(const std::string &msg);
// counts kernel launches (gdp_launch_count); while gdp_profile_enable(1) is on it also records
// a CUDA event on s tagged with the kernel name and its algorithmic bytes / flops (0 = not stated)
void note_launch(const char *name, cudaStream_t s, double bytes = 0.0, double flops = 0.0);
gdp_status cuda_status(cudaError_t e, const char *what);

#define GDP_CUDA_CHECK(expr)                                      \
  do {                                                            \
    cudaError_t _e = (expr);                                      \
    if (_e != cudaSuccess) return gdp::cuda_status(_e, #expr);    \
  } while (0)

#define GDP_LAUNCH_CHECK(what)                                    \
  do {                                                            \
    cudaError_t _e = cudaGetLastError();                          \
    if (_e != cudaSuccess) return gdp::cuda_status(_e, what);     \
  } while (0)

}  // namespace gdp

// ------------------------------------------------------------------ graph / topology
struct gdp_graph_s {
  int N = 0, F = 0;
  int ldX = 0;                                      // row stride of X: F rounded up to 4 (16-byte rows for TMA)
  int64_t E = 0, E_sym = 0;
  int device = 0;
  // device arrays (caller node ids)
  float *X = nullptr;                               // N x ldX (columns F..ldX-1 zero)
  int *nbr_ptr = nullptr, *nbr_idx = nullptr;       // symmetric neighbour CSR (N+1, E_sym)
  int *heavy = nullptr;                             // nodes with more than kHeavyDeg neighbours, ascending
  int n_heavy = 0;
  int *out_ptr = nullptr, *out_idx = nullptr, *out_src = nullptr;  // out CSR, consumers ascending
  int *in_ptr = nullptr, *in_idx = nullptr;         // in CSR, producers ascending
  int *cost = nullptr;                              // int32 compute cost
  long long *out_bytes = nullptr, *mem_bytes = nullptr;
  int *perm = nullptr;                              // Kahn order: perm[i] = node at position i
  int *leader = nullptr;                            // co-location leader (self if none)
  bool perm_identity = true, has_coloc = false;
  // host aggregates (overflow check)
  long long sum_cost = 0;
  long long sum_edge_out_bytes = 0;                 // sum over edges of producer output bytes
  long long n_edges_cross_max = 0;
  int max_indeg = 0, max_outdeg = 0;
  int min_cost = 0;   // smallest compute cost (k_cost5 needs every duration >= 1)
  long long min_edge_bytes = 0;   // smallest producer output over edges (k_cost5: shortest transfer); LLONG_MAX: no edges
  // shared-memory cost model records (cost2.cuh)
  void *nrec = nullptr, *erec = nullptr, *irec = nullptr;
  unsigned *cnt0 = nullptr;
  int *bigid = nullptr, *big_in = nullptr, *big_out = nullptr;
  int nbig = 0;
  // k_cost5 records (cost5.cu)
  bool c5_ok = false;
  void *slots5 = nullptr, *srcq5 = nullptr, *ebytes5 = nullptr;
  int *gbig5 = nullptr, *outdeg5 = nullptr;
  unsigned *bigb5 = nullptr;
  int nsrc5 = 0, nbigb5 = 0, ngbig5 = 0, nflagw5 = 0, bytes32_5 = 0;
};

struct gdp_topo_s {
  int d = 0;
  long long cap[8];
  int speed[8];
  long long bpt[64];
  int lat[64];
  double inv_bpt[64];   // 1 / bpt (cost kernels: reciprocal estimate + exact fix-up)
};

// Topology passed by value to kernels
struct TopoArgs {
  int d;
  long long cap[8];
  int speed[8];
  long long bpt[64];
  int lat[64];
  double inv_bpt[64];   // 1 / bpt (cost kernels: reciprocal estimate + exact fix-up)
};

namespace gdp {

// ------------------------------------------------------------------ workspace layout
struct Layer {       // saved activations of one Transformer-XL layer (topological row order)
  float *x, *a, *mu1, *rs1, *qkv, *o, *lse, *x1, *c, *mu2, *rs2, *m, *y;
  // folded (gated) weights
  float *Wqkv, *bqkv, *Wo, *W1, *W2;
  // dW' (augmented with the bias row) for the gate backward
  float *dWqkv, *dWo, *dW1, *dW2;
};

struct WS {
  // embed
  float *H[4], *Z[3], *A[3];
  int *ARG[3];
  // place
  float *Etopo, *zsum, *z, *gam, *Wh, *dWh, *logits_topo;
  Layer L[3];  // 0 = conditioner, 1 = xl0, 2 = xl1
  // grad scratch
  double *wb, *lpart, *spart;
  float *dlog, *dlog_topo, *dy, *dx1, *dm, *dc, *dout, *dqkv, *dkvm, *dkvt, *da, *dam, *dxa, *dEt, *dE;
  float *dH, *dHn, *dAg, *dP, *dd;
  float *dEW;            // autoregressive placer: dL/dEW (d x d)
  float *part;           // wgrad / column-sum partials
  float *dgam, *dz, *dzp;
  size_t part_floats;
  // sample
  float *cdf, *logp;
  int *lastpos;
  // cost scratch: B regions of c_per_place bytes (v2) or the v1 arrays
  unsigned char *c_scratch;
  size_t c_per_place;
  int *c_rem, *c_rcons, *c_new;
  int2 *c_fifo;
  int4 *c_chq;
  size_t bytes;
};

bool ws_layout(const gdp_graph_s *g, int d, int B, char *base, WS *w);

// Gated dense maps per placement layer, in theta order: q, k, v, o, f1, f2; then head.
constexpr int kGateCount = 13;
constexpr int kGamTotal = 2 * (5 * kH + kFFN) + kH;   // 1216

// ------------------------------------------------------------------ kernels (launchers)
enum Epi { EPI_NONE = 0, EPI_SIGMOID = 1, EPI_TANH = 2, EPI_RELU = 3, EPI_MASK = 4 };

struct GemmArgs {
  int M, K, Nout;
  const float *X1; int ldx1; int K1;        // operand columns [0, K1)
  const float *X2; int ldx2;                // operand columns [K1, K) (nullable)
  const float *W; int ldw_k, ldw_n;         // W(k, n) = W[k * ldw_k + n * ldw_n]
  const float *bias;                        // Nout (nullable)
  const float *R; int ldr;                  // residual added after the activation (nullable)
  const float *aux; int ldaux;              // EPI_MASK: multiply by (aux > 0)
  float *Y; int ldy; int split;             // columns < split -> Y
  float *Y2; int ldy2;                      // columns >= split -> Y2 (col - split)
  int accumulate;                           // Y = Y + result
  int epi;
};
void launch_gemm(const GemmArgs &a, cudaStream_t s);
// algorithmic bytes of one GEMM launch: X, W, Y (+ residual, mask, accumulated Y), fp32
inline double gemm_bytes(const GemmArgs &a) {
  const double my = (double)a.M * a.Nout;
  return 4.0 * ((double)a.M * a.K + (double)a.K * a.Nout + my + (a.R ? my : 0.0) + (a.aux ? my : 0.0) +
                (a.accumulate ? my : 0.0));
}
// tcgen05 path (tc_gemm.cu); launch_gemm routes eligible shapes there when the calling
// entry point enabled tensor cores (gdp_config.tensor_cores)
bool tc_eligible(const GemmArgs &a);
void launch_gemm_tc(const GemmArgs &a, cudaStream_t s);
// gdp_config.tensor_cores: 0 SIMT fp32, 1 tcgen05 dense maps + attention, 2 tcgen05 dense maps with
// the SIMT attention (diagnostic: compares the attention tiles inside one tensor-core step)
void set_tensor_cores(int mode);
bool tensor_cores_on();
bool tensor_core_attention_on();
bool attn_fwd_tc_eligible(int S, int M);
void launch_attn_fwd_tc(const float *qkv, float *o, float *lse, int N, int S, int M, cudaStream_t s);
bool attn_bwd_tc_long_eligible(int S, int M);   // any M: query-major dQ + key-major dK / dV
void launch_attn_bwd_dq_tc(const float *qkv, const float *o, const float *lse, const float *dout, float *dqkv, int N,
                           int S, int M, cudaStream_t s);
void launch_attn_bwd_dkv_tc(const float *qkv, const float *o, const float *lse, const float *dout, float *dqkv,
                            float *dkvm, int N, int S, int M, cudaStream_t s);
// ablation variant of the entry point in progress (gdp_config.no_attention)
void set_no_attention(bool on);
bool no_attention();

// dW_aug[(K + with_bias) x Nout] = [X, 1]^T dY over all M rows, deterministic split-K over rows.
// Result: out (+)= sum (accumulate flag).  part must hold chunks * (K+1) * Nout floats.
void launch_wgrad(int M, int K, int Nout, const float *X1, int ldx1, int K1, const float *X2, int ldx2,
                  const float *dY, int ldy, bool with_bias, float *part, size_t part_floats, float *out,
                  bool accumulate, cudaStream_t s);
// tensor-core mode (tc_wgrad.cu): the same partials by tcgen05 (tf32 X and dY, fp32 accumulation;
// the bias row an fp32 column sum); returns the chunk count written to part, 0 if not launched
bool wgrad_tc_eligible(int M, int K, int Nout);
int launch_wgrad_tc(int M, int K, int Nout, const float *X1, int ldx1, int K1, const float *X2, int ldx2,
                    const float *dY, int ldy, bool with_bias, float *part, size_t part_floats, cudaStream_t s);

void launch_layernorm(const float *x, const float *g, const float *b, float *y, float *mu, float *rs, int N,
                      cudaStream_t s);
// dx (+)= LN backward of da (+ res, nullable: the residual branch); param grads from (da + da_extra)
// accumulated into dgb[0..63] (gain) and dgb[64..127] (bias).
void launch_layernorm_bwd(const float *x, const float *mu, const float *rs, const float *g, const float *da,
                          const float *da_extra, float *dx, bool dx_accumulate, const float *res, float *dgb,
                          float *part, int N, cudaStream_t s);
// dkvt = [dQ | dK_own + dK_mem | dV_own + dV_mem] (16-byte aligned rows)
void launch_dkvt(const float *dqkv, const float *dkvm, float *dkvt, int N, cudaStream_t s);
void launch_colsum(const float *x, int N, int C, float scale, float *out, float *part, cudaStream_t s);

// nnz = ptr[N] (symmetric neighbour entries), used only for the algorithmic byte count;
// heavy (n_heavy) = the nodes with more than kHeavyDeg neighbours, one CTA each
constexpr int kHeavyDeg = 64;
void launch_gather_max(const float *Z, const int *ptr, const int *idx, const int *heavy, int n_heavy, float *A,
                       int *ARG, int N, long long nnz, cudaStream_t s);
void launch_gather_max_bwd(const float *dA, const int *ARG, const float *Z, const int *ptr, const int *idx,
                           const int *heavy, int n_heavy, float *dPre, int N, long long nnz, cudaStream_t s);

void launch_attn_fwd(const float *qkv, float *o, float *lse, int N, int S, int M, cudaStream_t s);
void launch_relu_v(const float *qkv, float *o, int N, cudaStream_t s);
void launch_relu_v_bwd(const float *qkv, const float *dout, float *dqkv, float *dkvm, int N, cudaStream_t s);
void launch_attn_bwd(const float *qkv, const float *o, const float *lse, const float *dout, float *dqkv,
                     float *dkvm, float *Dd, int N, int S, int M, cudaStream_t s);

void launch_rows_gather(const float *src, const int *perm, float *dst, int N, int C, cudaStream_t s);
void launch_rows_scatter(const float *src, const int *perm, float *dst, int N, int C, bool accumulate,
                         cudaStream_t s);
void launch_tanh_grad(const float *dHn, const float *Hn, float *dP, int n, cudaStream_t s);
void launch_fill_rows(float *dst, const float *row, float scale, int N, int C, cudaStream_t s);

// sampling / loss
void launch_sample(const float *logits, int ld, const int *leader, bool has_coloc, int N, int d, int B, uint64_t seed,
                   uint64_t offset, uint64_t step, const uint64_t *step_ptr, float *cdf, float *logp, int *lastpos,
                   double *spart, uint8_t *D, float *logprob, cudaStream_t s);
void launch_node_prep(const float *logits, int ld, int N, int d, float *cdf, float *logp, int *lastpos,
                      cudaStream_t s);
// dL/dlogits (a14): part = kLogitChunks x N x kMaxD doubles of scratch (ws.lpart)
constexpr int kLogitChunks = 16;
void launch_logit_grad(const float *logits, int ld, const uint8_t *D, const int *leader, const double *adv,
                       const float *logprob, const float *old_logprob, float eps, float beta, float scale,
                       int N, int d, int B, double *wb, double *part, float *dlog, cudaStream_t s);

// training update (NEXT-1)
constexpr int kAdamScratch = 1024;   // doubles of caller scratch for gdp_clip_adam (GDP_ADAM_SCRATCH)
int adam_parts();
void launch_logprob(const float *logp, const int *leader, const uint8_t *D, int N, int d, int B, float *logprob,
                    cudaStream_t s);
void launch_greedy(const float *logits, int ld, const int *leader, int N, int d, uint8_t *D, cudaStream_t s);
// log pi_b = sum of part[b][0..nparts) in order; non-leaders copy their leader's device
void launch_sum_parts(const double *part, int nparts, int B, float *logprob, cudaStream_t s);
void launch_colocate(const int *leader, int N, int B, uint8_t *D, cudaStream_t s);
// autoregressive-within-segment placer (ar.cu, reading R35).  EW (d x d)
// follows the N x d base logits in the caller's logits buffer.
constexpr int kArDecodeSample = 0, kArDecodeScore = 1, kArDecodeGreedy = 2;
void launch_ar_table(const float *E, const float *Wh, int d, float *EW, cudaStream_t s);
// groups of consecutive segments a decode / gradient warp walks (<= the k_sample chunk count, so
// that ws.spart holds B x groups partial sums)
int ar_groups(int N, int S);
void launch_ar_decode(int mode, const float *logits, const int *perm, const int *leader, bool has_coloc, int N,
                      int d, int S, int B, uint64_t seed, uint64_t offset, uint64_t step, const uint64_t *step_ptr,
                      uint8_t *D, double *part, float *logprob, cudaStream_t s);
// dL/dbase (topological rows, dlt) and dL/dEW (dEW, d x d) of the R35 loss; part / dewpart scratch
void launch_ar_grad(const float *logits, const int *perm, const int *leader, int N, int d, int S, int B,
                    const uint8_t *D, const double *adv, const float *logprob, const float *old_logprob, float eps,
                    float beta, float scale, double *wb, double *lpart, float *dewpart, size_t dewpart_floats,
                    float *dlt, float *dEW, cudaStream_t s);
// dWh' += E^T dEW (rows 0..63 of the augmented head gradient), grad[E] += dEW Wh'^T
void launch_ar_head_bwd(const float *E, const float *Wh, const float *dEW, int d, float *dWh, float *gE,
                        cudaStream_t s);
// devices a call samples / scores over: gdp_config.active_devices, or num_devices when 0
int active_devices(const gdp_config *c);
// synchronous: index of the first non-finite entry of g[0, n) (n if none, -1 on a CUDA error);
// scratch = one device uint64
long long first_nonfinite(const float *g, long long n, unsigned long long *scratch, cudaStream_t s);
void launch_clip_adam(const float *g, long long n, double max_norm, double lr, double b1, double b2, double eps,
                      double c1, double c2, float *theta, float *m, float *v, double *scratch, double *norm_out,
                      cudaStream_t s);

// cost model
// kernel gdp_cost runs (5, 3 or 1); `force` != 0 asks whether that kernel applies (it is
// returned if so, else the automatic choice)
int cost_kernel_choice(const gdp_graph_s *g, const gdp_topo_s *t, int force);
int cost_wave(const gdp_graph_s *g, const gdp_topo_s *t);   // placements per full wave of k_cost5 (0: n/a)
gdp_status launch_cost(const gdp_graph_s *g, const gdp_topo_s *t, const uint8_t *D, int B,
                       gdp_sim_report *rep, long long *peak, long long *busy, double *reward, const WS &w,
                       int force, cudaStream_t s);
void launch_advantage(const double *r, int B, double *sum, long long *cnt, double *adv, cudaStream_t s);

}  // namespace gdp
