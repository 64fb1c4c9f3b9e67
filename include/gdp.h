/*
 * gdp.h -- C ABI of libgdp.so, the B200 (sm_100a) hot path of GDP
 * ("GDP: Generalized Device Placement for Dataflow Graphs", arXiv 1910.01578).
 *
 * One batched policy step (§3, Eq. 1-4; §4.1 reward):
 *   gdp_embed        GraphSAGE max-pool embedding            (§3.1, Eq. 2-3)
 *   gdp_place        segment-recurrent Transformer-XL placer  (§3.2-3.3, Eq. 4)
 *                    with superposition conditioning -> per-node device logits
 *   gdp_sample       B placements D ~ pi_theta(G)             (§3)
 *   gdp_cost         step-time cost model + reward            (§4.1)
 *   gdp_advantage    reward minus mean of all previous trials (§4.1)
 *   gdp_policy_grad  PPO / REINFORCE gradient of theta        (§3, Eq. 1)
 *
 * Conventions (all entry points):
 *   - Plain pointers only.  "dev" pointers are CUDA device memory on the current
 *     device, "host" pointers are host memory.  The caller owns every buffer passed
 *     in; the library owns gdp_graph / gdp_topo objects until their destroy call.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Compute calls are asynchronous on `stream`; argument validation is synchronous
 *     and returns a status.  Device faults surface at the caller's next sync.
 *   - No allocation happens inside the hot-path calls: all scratch comes from the
 *     caller's workspace `ws` (size from gdp_workspace_size).
 *   - Per-node arrays at the boundary are in the CALLER's node-id order.  The
 *     library computes the Kahn order pi (ties by smallest id) and runs
 *     the segment-recurrent placer in pi order internally.
 *   - Same inputs => bit-identical outputs.
 *   - Errors: a status code (never an exception); gdp_last_error() gives a
 *     thread-local message.  An invalid placement is a verdict in the report,
 *     not an error.
 */
#ifndef GDP_H_
#define GDP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GDP_OK = 0,
  GDP_ERR_ARG = 1,        /* bad scalar argument / null pointer / unsupported config */
  GDP_ERR_GRAPH = 2,      /* edge endpoint out of range, self edge, duplicate edge, negative cost/bytes */
  GDP_ERR_CYCLE = 3,      /* the edge list is not a DAG */
  GDP_ERR_SHAPE = 4,      /* sizes disagree (e.g. F or d differs from the graph / config) */
  GDP_ERR_CUDA = 5,       /* a CUDA call failed (message in gdp_last_error) */
  GDP_ERR_OVERFLOW = 6,   /* sum of durations + transfers could reach 2^31 ticks (device time is int32) */
  GDP_ERR_NONFINITE = 7,  /* non-finite gradient (gdp_grad_check; gdp_clip_adam skips such an update) */
  GDP_ERR_WORKSPACE = 8   /* ws_bytes smaller than gdp_workspace_size */
} gdp_status;

typedef struct gdp_graph_s *gdp_graph;
typedef struct gdp_topo_s *gdp_topo;

/* Model configuration.  The network sizes are the SURVEY §8 defaults
 * (h = 64, 4 heads, 3 GNN rounds, 2 placement layers + 1 conditioner layer,
 * FFN 4h); other values return GDP_ERR_ARG. */
typedef struct {
  int32_t hidden;         /* h, must be 64 */
  int32_t heads;          /* must be 4 (head dim 16) */
  int32_t gnn_layers;     /* L, must be 3 */
  int32_t xl_layers;      /* must be 2 */
  int32_t ffn;            /* must be 256 */
  int32_t num_devices;    /* d, 1..8 ("up to eight") */
  int32_t seg_len;        /* S >= 1: Transformer-XL segment length */
  int32_t mem_len;        /* M >= 0 cached positions before each segment, or -1 = every earlier segment */
  int32_t superposition;  /* 1: Eq. 4 gates on every placer dense map and the head; 0: gates == 1 */
  int32_t tensor_cores;   /* 0: every dense map in fp32 (SIMT, the 1e-4 parity mode); 1: dense maps
                             Y = X W (forward and the backward dX = dY W^T) with 16 <= width <= 256,
                             1 <= K <= 256, ceil32(K) * ceil16(width) <= 40960 and >= 128 rows on
                             tcgen05 tensor cores with tf32 operands -- the fp32 bit patterns of X and
                             W truncated to their upper 19 bits (sign, exponent, 10 mantissa bits) --
                             and fp32 accumulation in TMEM; the weight gradients dW = X^T dY of the
                             maps with 16 <= width <= 256, K <= 256 and >= 128 rows likewise (tf32
                             X and dY, fp32 accumulation; the bias row an fp32 column sum); the
                             segment attention on tcgen05 tiles with bf16 Q, K, V and softmax
                             numerators.  2 (diagnostic): as 1 but with the
                             SIMT attention kernels, so that tests compare the attention tiles inside
                             one tensor-core step */
  int32_t no_attention;   /* ablation: 1 replaces every attention
                             sublayer (placer and conditioner) by the per-node map
                             o = ReLU(LN1(x) W_v + b_v) (reading R34); 0: attention */
  int32_t active_devices; /* mixed device counts: the head has num_devices (D_max)
                             outputs, sampling / log pi / greedy / the loss use the first
                             active_devices (the rest masked to -inf, zero gradient); 0 = all */
  int32_t autoregressive; /* SURVEY NEXT-4 / SPEC.md:562, reading R35: 1 = the
                             autoregressive-within-segment placer -- node i's logits add
                             (gamma_h (.) mean of E[D_j] over the leaders j decided before it in
                             its segment) W_h, E = GDP_P_AR_E (d x h); gdp_sample / gdp_logprob /
                             gdp_greedy decode each segment position by position and
                             gdp_policy_grad differentiates through it.  0 = per-node heads (R13).
                             Requires active_devices = 0. */
} gdp_config;

/* One cost-model verdict per placement. */
typedef struct {
  int64_t makespan;       /* ticks (1 tick = 1 us) */
  int64_t cross_bytes;    /* sum of output_bytes over cross-device edges */
  uint8_t valid;          /* 1 iff violation == 0 */
  uint8_t violation;      /* 0 none, 1 co-location, 2 out of memory, 3 malformed (device id >= d) */
  uint8_t pad[6];
} gdp_sim_report;

/* Flat parameter vector theta (fp32), in this order.  Matrices are row-major
 * fan_in x fan_out; every dense map is y = x W + b.  Gate projections P_j (64 x w_j)
 * and q_j (w_j) give gamma_j = 2 sigmoid(z P_j + q_j) for the placer's dense maps
 * (gate0.* for placement layer 0, gate1.* for layer 1, gate.head for the head). */
typedef enum {
  GDP_P_GNN_IN_W = 0,   /* F x 64    input projection */
  GDP_P_GNN_IN_B,       /* 64 */
  GDP_P_GNN_0_W,        /* 64 x 64   Eq. 2 W^(0) */
  GDP_P_GNN_0_B,        /* 64        Eq. 2 b^(0) */
  GDP_P_GNN_0_WF,       /* 128 x 64  Eq. 3 f^(1) on concat(h_v, h_N(v)) */
  GDP_P_GNN_0_BF,       /* 64 */
  GDP_P_GNN_1_W, GDP_P_GNN_1_B, GDP_P_GNN_1_WF, GDP_P_GNN_1_BF,
  GDP_P_GNN_2_W, GDP_P_GNN_2_B, GDP_P_GNN_2_WF, GDP_P_GNN_2_BF,
  /* three Transformer-XL layers, each: ln1.g, ln1.b (64), Wq (64x64), bq, Wk, bk, Wv, bv,
     Wo, bo, ln2.g, ln2.b, W1 (64x256), b1 (256), W2 (256x64), b2 (64) */
  GDP_P_COND_LN1_G, GDP_P_COND_LN1_B, GDP_P_COND_WQ, GDP_P_COND_BQ, GDP_P_COND_WK, GDP_P_COND_BK,
  GDP_P_COND_WV, GDP_P_COND_BV, GDP_P_COND_WO, GDP_P_COND_BO, GDP_P_COND_LN2_G, GDP_P_COND_LN2_B,
  GDP_P_COND_W1, GDP_P_COND_B1, GDP_P_COND_W2, GDP_P_COND_B2,
  GDP_P_XL0_LN1_G, GDP_P_XL0_LN1_B, GDP_P_XL0_WQ, GDP_P_XL0_BQ, GDP_P_XL0_WK, GDP_P_XL0_BK,
  GDP_P_XL0_WV, GDP_P_XL0_BV, GDP_P_XL0_WO, GDP_P_XL0_BO, GDP_P_XL0_LN2_G, GDP_P_XL0_LN2_B,
  GDP_P_XL0_W1, GDP_P_XL0_B1, GDP_P_XL0_W2, GDP_P_XL0_B2,
  GDP_P_XL1_LN1_G, GDP_P_XL1_LN1_B, GDP_P_XL1_WQ, GDP_P_XL1_BQ, GDP_P_XL1_WK, GDP_P_XL1_BK,
  GDP_P_XL1_WV, GDP_P_XL1_BV, GDP_P_XL1_WO, GDP_P_XL1_BO, GDP_P_XL1_LN2_G, GDP_P_XL1_LN2_B,
  GDP_P_XL1_W1, GDP_P_XL1_B1, GDP_P_XL1_W2, GDP_P_XL1_B2,
  /* gates, per placement layer l: q, k, v, o, f1 (P 64x64, q 64), f2 (P 64x256, q 256) */
  GDP_P_GATE0_Q_P, GDP_P_GATE0_Q_Q, GDP_P_GATE0_K_P, GDP_P_GATE0_K_Q, GDP_P_GATE0_V_P, GDP_P_GATE0_V_Q,
  GDP_P_GATE0_O_P, GDP_P_GATE0_O_Q, GDP_P_GATE0_F1_P, GDP_P_GATE0_F1_Q, GDP_P_GATE0_F2_P, GDP_P_GATE0_F2_Q,
  GDP_P_GATE1_Q_P, GDP_P_GATE1_Q_Q, GDP_P_GATE1_K_P, GDP_P_GATE1_K_Q, GDP_P_GATE1_V_P, GDP_P_GATE1_V_Q,
  GDP_P_GATE1_O_P, GDP_P_GATE1_O_Q, GDP_P_GATE1_F1_P, GDP_P_GATE1_F1_Q, GDP_P_GATE1_F2_P, GDP_P_GATE1_F2_Q,
  GDP_P_GATE_HEAD_P,    /* 64 x 64 */
  GDP_P_GATE_HEAD_Q,    /* 64 */
  GDP_P_HEAD_W,         /* 64 x d   per-node device logits (Fig. 1 "d") */
  GDP_P_HEAD_B,         /* d */
  GDP_P_AR_E,           /* d x 64    device embedding of the autoregressive placer (empty unless
                           gdp_config.autoregressive) */
  GDP_P_COUNT           /* = 91 tensors */
} gdp_param_id;

/* ------------------------------------------------------------------ setup (untimed) */

/* Fill *out with the SURVEY §8 defaults for d devices (S = 128, M = 128,
 * superposition on, tensor_cores 0).  Errors: GDP_ERR_ARG if d is not in 1..8 or out is NULL. */
gdp_status gdp_default_config(int32_t d, gdp_config *out);

/* Thread-local message describing the last non-OK status (never NULL). */
const char *gdp_last_error(void);

/* Diagnostic: total number of CUDA kernels this library has launched in this process
 * (all threads, all devices).  bench.py reads it around the timed region. */
uint64_t gdp_launch_count(void);

/* Diagnostic: per-kernel timing for the roofline report (bench.py "kernels"; north_star's
 * "evidenced by" list).  gdp_profile_enable(1) clears earlier records and makes every kernel
 * launch of the library record a CUDA event on its stream just before the launch, tagged with
 * the kernel's name and its algorithmic bytes and flops (0 where not stated);
 * gdp_profile_enable(0) stops recording and keeps the records.  gdp_profile_mark(stream)
 * records a closing event on stream (a void* cudaStream_t).  A launch's time is the gap to the
 * next event on the same stream: exact when the GPU is kept busy (bench.py gates the stream
 * with a spin kernel before enqueuing the step), an upper bound otherwise.
 * gdp_profile_read synchronises the events and writes, for up to max_names distinct kernels in
 * first-launch order, the name (static string owned by the library), the number of timed
 * launches, the summed ms, bytes and flops; it returns the number written, or -1 (see
 * gdp_last_error).  Not for use inside CUDA graph capture.  Errors: GDP_ERR_ARG from
 * gdp_profile_mark when profiling is off. */
gdp_status gdp_profile_enable(int32_t on);
gdp_status gdp_profile_mark(void *stream);
int32_t gdp_profile_read(int32_t max_names, const char **names, int32_t *launches, double *ms, double *bytes,
                         double *flops);

/* Diagnostic: build identification string of this library (never NULL). */
const char *gdp_build_info(void);

/* Host-only graph check: ids in range, no self or duplicate edges,
 * acyclic.  edges: host E x 2 int32 (producer, consumer).  topo_order (host, N,
 * nullable) receives Kahn's order with ties broken by smallest id.
 * Errors: GDP_ERR_ARG (N <= 0, E < 0, edges NULL with E > 0), GDP_ERR_GRAPH, GDP_ERR_CYCLE. */
gdp_status gdp_graph_validate(int32_t N, int64_t E, const int32_t *edges, int32_t *topo_order);

/* Create a graph G(V, E): N ops, F meta features per op, E
 * data-dependency edges.  All inputs are HOST arrays and are copied:
 *   feat          N x F float32 row-major, the initial representations h_v^(0)
 *   edges         E x 2 int32 (producer, consumer)
 *   compute_cost  N int64 ticks (>= 0, <= 2^31-1)
 *   output_bytes  N int64 (>= 0)
 *   memory_bytes  N int64 (>= 0), resident on the op's device for the whole step
 *   coloc_group   N int32 group id or -1, nullable (no co-location constraints)
 * The device copies (features, symmetric neighbour CSR, in/out CSR, Kahn order,
 * group leaders) live on the current CUDA device until gdp_graph_destroy.
 * Synchronous.  Errors: GDP_ERR_ARG, GDP_ERR_GRAPH, GDP_ERR_CYCLE, GDP_ERR_CUDA. */
gdp_status gdp_graph_create(int32_t N, int32_t F, const float *feat, int64_t E, const int32_t *edges,
                            const int64_t *compute_cost, const int64_t *output_bytes,
                            const int64_t *memory_bytes, const int32_t *coloc_group, gdp_graph *out);
gdp_status gdp_graph_destroy(gdp_graph g);

/* Device topology, all HOST arrays, copied:
 *   mem_capacity  d int64 bytes;  speed d int32 (> 0) multiplier on compute_cost;
 *   bytes_per_tick d x d int64 (> 0 off the diagonal, symmetric; diagonal ignored);
 *   latency d x d int32 ticks (>= 0; diagonal ignored).
 * Errors: GDP_ERR_ARG (d not in 1..8, bad entries, asymmetric bandwidth). */
gdp_status gdp_topo_create(int32_t d, const int64_t *mem_capacity, const int32_t *speed,
                           const int64_t *bytes_per_tick, const int32_t *latency, gdp_topo *out);
gdp_status gdp_topo_destroy(gdp_topo t);

/* Flat-theta layout for config c and feature width F: *n_params (nullable) and
 * offsets[GDP_P_COUNT + 1] (nullable; offsets[i] = first element of tensor i,
 * offsets[GDP_P_COUNT] = n_params).  Errors: GDP_ERR_ARG. */
gdp_status gdp_param_layout(const gdp_config *c, int32_t F, int64_t *offsets, int64_t *n_params);

/* Bytes of workspace the hot-path calls need for graph g, config c and up to B
 * placements per gdp_cost / gdp_policy_grad call.  Errors: GDP_ERR_ARG. */
gdp_status gdp_workspace_size(gdp_graph g, const gdp_config *c, int32_t B, size_t *bytes);

/* ------------------------------------------------------------------ hot path */

/* §3.1 graph embedding (Eq. 2-3): H0 = X W_in + b_in; for l < 3:
 * Z = sigmoid(H W_l + b_l); a_v = max_{u in N(v)} Z_u (N(v) = preds U succs, first
 * index on ties, 0 if empty); H = tanh([H | a] W_f,l + b_f,l).
 *   theta     dev fp32 [n_params]
 *   node_emb  dev fp32 N x 64 (out), caller node order
 *   ws        dev workspace; activations saved here are consumed by gdp_policy_grad
 * Errors: GDP_ERR_ARG, GDP_ERR_WORKSPACE, GDP_ERR_CUDA. */
gdp_status gdp_embed(gdp_graph g, const gdp_config *c, const float *theta, float *node_emb,
                     void *ws, size_t ws_bytes, void *stream);

/* §3.2-3.3 placement network on node_emb in Kahn order: conditioner layer ->
 * z = mean over nodes -> gates gamma_j = 2 sigmoid(z P_j + q_j) (Eq. 4) -> two
 * Transformer-XL layers (segments of S nodes attending to themselves and to the
 * stop-gradient cached states of the previous M positions; no positional terms,
 * P:144-148) -> logits = (gamma_head . y) W_head + b_head.
 *   node_emb  dev fp32 N x 64 (in, as written by gdp_embed)
 *   logits    dev fp32 N x d (out), caller node order.  With gdp_config.autoregressive the buffer
 *             holds N + d rows: the N x d base logits, then the d x d table EW = (E . gamma_head) W_head
 *             (row k: the logit shift a decided device k contributes, reading R35); every call that
 *             takes `logits` below reads both parts in that mode.
 * Errors: GDP_ERR_ARG (d mismatch, S < 1, M < -1), GDP_ERR_WORKSPACE, GDP_ERR_CUDA. */
gdp_status gdp_place(gdp_graph g, const gdp_config *c, const float *theta, const float *node_emb,
                     float *logits, void *ws, size_t ws_bytes, void *stream);

/* D ~ pi_theta(G).  For sample b (global index
 * gidx = sample_offset + b) and node v: Philox4x32-10 with key (seed mod 2^32,
 * seed >> 32) and counter (v >> 2, gidx mod 2^32, step mod 2^32, gidx >> 32), word
 * v & 3, u = (word >> 8) 2^-24; D[b][v] = min{k : u < cdf_v[k]} over the fp32 softmax
 * CDF of logits row v (fallback: last k with p > 0).  Co-location non-leaders copy
 * the leader (lowest id in the group).  logprob[b] = sum over leaders of log p_v[D].
 *   logits      dev fp32 N x d (in);  placements dev uint8 B x N (out, placement-major)
 *   logprob     dev fp32 B (out)
 * ws must be sized for at least B placements (gdp_workspace_size); log pi is summed in fp64 in a
 * fixed order (per 128-node chunk, then the chunks in order): bit-identical across runs.
 * Autoregressive mode (R35): each segment (S positions of the Kahn order) is decoded position by
 * position -- leader v of placement b takes z = base_v + mean of EW[D_bj] over the leaders j
 * decided before it in its segment, then the same uniform and fp32 inverse CDF as above; log pi
 * sums per (placement, segment group) in Kahn order, then the groups in order.
 * Errors: GDP_ERR_ARG (B < 1), GDP_ERR_WORKSPACE, GDP_ERR_CUDA. */
gdp_status gdp_sample(gdp_graph g, const gdp_config *c, const float *logits, int32_t B, uint64_t seed,
                      uint64_t sample_offset, uint64_t step, uint8_t *placements, float *logprob,
                      void *ws, size_t ws_bytes, void *stream);

/* gdp_sample with the Philox step read from device memory (*step_dev, uint64) when the kernel
 * runs, so that a captured CUDA graph draws fresh placements on every replay once the caller
 * advances the counter inside the graph.  Same arguments, results and errors as gdp_sample
 * (plus GDP_ERR_ARG for step_dev NULL). */
gdp_status gdp_sample_at(gdp_graph g, const gdp_config *c, const float *logits, int32_t B, uint64_t seed,
                         uint64_t sample_offset, const uint64_t *step_dev, uint8_t *placements, float *logprob,
                         void *ws, size_t ws_bytes, void *stream);

/* Step-time cost model (semantics in DESIGN.md §"Cost model"):
 * per placement, list scheduling in integer ticks -- duration = compute_cost x
 * speed[D v]; one transfer per cross-device edge, FIFO on the directed channel
 * (D u -> D v), ceil(bytes / bytes_per_tick) + latency; each device runs one op at a
 * time, choosing the smallest (ready time, id); liveness memory model; co-location
 * and capacity checks.  One CTA per placement.  reward[b] = valid ? -sqrt(makespan /
 * 1e6) : -10.
 *   placements dev uint8 B x N (in);  rep dev gdp_sim_report B (out)
 *   peak_mem   dev int64 B x d (out, nullable);  busy dev int64 B x d (out, nullable)
 *   reward     dev fp64 B (out)
 * Errors: GDP_ERR_ARG, GDP_ERR_SHAPE (topology d != config d), GDP_ERR_OVERFLOW,
 * GDP_ERR_WORKSPACE, GDP_ERR_CUDA.  Invalid placements are verdicts, not errors. */
gdp_status gdp_cost(gdp_graph g, gdp_topo t, const uint8_t *placements, int32_t B, gdp_sim_report *rep,
                    int64_t *peak_mem, int64_t *busy, double *reward, void *ws, size_t ws_bytes,
                    void *stream);

/* Diagnostic: which cost kernel gdp_cost runs for this graph and topology (host only, no
 * launch): 5 = simulation-warp + memory-warp kernel (every duration >= 1 tick and every
 * transfer >= 1 tick), 3 = warp-cooperative instant-by-instant kernel (zero-duration ops or
 * zero-tick transfers: same-instant rounds), 1 = global-memory kernel (per-placement state
 * larger than shared memory).  All three compute the same integers (DESIGN.md §7 "Cost
 * model").  Returns 0 and sets the error for NULL handles. */
int32_t gdp_cost_kernel(gdp_graph g, gdp_topo t);

/* Diagnostic: placements the default cost kernel (5) runs at once on the current device --
 * resident CTAs per SM (shared memory per placement grows with the ops' input counters) times
 * the SMs.  A batch of that many placements costs about as long as one placement (the launch
 * time is one placement's simulation latency); bench.py sizes its batch with it.  0 if kernel 5
 * does not apply or for NULL handles. */
int32_t gdp_cost_wave(gdp_graph g, gdp_topo t);

/* Diagnostic (tests): the table of intermediates that gdp_embed / gdp_place / gdp_policy_grad
 * save in the workspace, as (name, byte offset from ws, rows, cols, is_int32) -- fp32 unless
 * is_int32.  GNN tensors (H0..H3, Z0..Z2, A0..A2 = max-pooled neighbourhoods, ARG0..ARG2 =
 * first-index argmax, -1 if none) are in caller node order; the placer's (Etopo, L<l>.a / qkv
 * / o / lse / x1 / c / m / y per layer l = 0 conditioner, 1, 2, and the folded weights
 * L<l>.Wqkv / bqkv / Wo / W1 / W2, Wh) in Kahn order; z, gam are the superposition context and
 * gates.  Backward scratch (dlog, dy, dm, dc, dx1, dout, dqkv, dkvm, da, dam, dEt, dH, dHn, dAg,
 * dP) holds the values of the LAST layer gdp_policy_grad processed.  The offsets do not depend
 * on B.  Writes at most max_names entries and returns the number of tensors, -1 on bad
 * arguments.  The parity tests read them to hold every kernel to the oracle on the kernel's
 * own inputs, and to adopt the GPU's decision at max-pool near-ties and ReLU inputs near zero
 * ("tie import"). */
int32_t gdp_debug_tensors(gdp_graph g, const gdp_config *c, int32_t max_names, const char **names,
                          int64_t *offsets, int64_t *rows, int64_t *cols, int32_t *is_int);

/* Gradient buckets, in the order the backward of gdp_policy_grad completes them (SURVEY §8(e):
 * the all-reduce of a bucket can start while the rest of the backward runs):
 *   0: placement layers, gates and head [off(GDP_P_XL0_LN1_G), n_params)
 *   1: the conditioner layer            [off(GDP_P_COND_LN1_G), off(GDP_P_XL0_LN1_G))
 *   2: the GNN                          [0, off(GDP_P_COND_LN1_G))
 * first/last host int64[GDP_GRAD_BUCKETS] (out): element ranges of the flat theta.
 * Errors: GDP_ERR_ARG. */
#define GDP_GRAD_BUCKETS 3
gdp_status gdp_grad_buckets(const gdp_config *c, int32_t F, int64_t *first, int64_t *last);

/* gdp_policy_grad that also records bucket_events[i] (GDP_GRAD_BUCKETS cudaEvent_t passed as
 * void*, created by the caller) on `stream` as soon as bucket i's gradient entries are final, so
 * that a caller can launch the bucket's NCCL all-reduce on a side stream waiting on the event
 * while the backward continues (Eq. 1 average over ranks).  Otherwise identical. */
gdp_status gdp_policy_grad_bucketed(gdp_graph g, const gdp_config *c, const float *theta, const float *logits,
                                    const uint8_t *placements, int32_t B, const double *adv, const float *logprob,
                                    const float *old_logprob, float clip_eps, float entropy_coef, float loss_scale,
                                    float *grad, void *ws, size_t ws_bytes, void *const *bucket_events,
                                    void *stream);

/* Sum of per-graph gradients (Eq. 1 sum over graphs): out = grads[0] + grads[1] + ...
 * in that fixed order (deterministic).  grads host array of n_grads device pointers, each fp32
 * [len]; out dev fp32 [len] (may alias none of them).  Asynchronous on stream.
 * Errors: GDP_ERR_ARG, GDP_ERR_CUDA. */
gdp_status gdp_grad_sum(const float *const *grads, int32_t n_grads, int64_t len, float *out, void *stream);

/* Finite check of a gradient ("a NaN gradient must raise a training error naming the
 * parameter"): SYNCHRONOUS on `stream`.  GDP_OK if every entry of grad[0, n_params) is
 * finite, else GDP_ERR_NONFINITE with gdp_last_error() naming the first offending entry's
 * parameter tensor (gdp_param_id and its name) and element.  grad dev fp32 n_params (layout of
 * (c, F)); scratch dev, >= 8 bytes.  Errors: GDP_ERR_ARG, GDP_ERR_NONFINITE, GDP_ERR_CUDA. */
gdp_status gdp_grad_check(const float *grad, const gdp_config *c, int32_t F, double *scratch, void *stream);

/* Diagnostic / test entry: gdp_cost on an explicitly chosen kernel (5, 3 or 1; 0 = the
 * automatic choice gdp_cost makes).  GDP_ERR_ARG if that kernel does not apply to (g, t)
 * (e.g. 5 with a zero-duration op).  Used by the tests to hold every kernel to the oracle on
 * the same inputs; otherwise identical to gdp_cost. */
gdp_status gdp_cost_with_kernel(gdp_graph g, gdp_topo t, const uint8_t *placements, int32_t B,
                                gdp_sim_report *rep, int64_t *peak_mem, int64_t *busy, double *reward,
                                void *ws, size_t ws_bytes, int32_t kernel, void *stream);

/* Advantage ("average reward of all the previous trials as a bias term"):
 * for b = 0..B-1 in order, adv[b] = (count == 0) ? 0 : reward[b] - sum / count, then
 * sum += reward[b], count += 1.  One state per graph.
 *   reward dev fp64 B;  run_sum dev fp64 [1] (in/out);  run_count dev int64 [1] (in/out)
 *   adv dev fp64 B (out).  Errors: GDP_ERR_ARG, GDP_ERR_CUDA. */
gdp_status gdp_advantage(const double *reward, int32_t B, double *run_sum, int64_t *run_count, double *adv,
                         void *stream);

/* Policy gradient (P:93 PPO; Eq. 1 batch objective):
 *   L = -loss_scale * sum_b min(rho_b A_b, clip(rho_b, 1-eps, 1+eps) A_b)
 *       - entropy_coef * (1/N) sum_v H(p_v),
 * rho_b = exp(logprob_b - old_logprob_b) (rho = 1 with the gradient of log pi when
 * old_logprob is NULL), log pi_b = sum over co-location leaders of log p_v[D_b v].
 * The gradient flows end to end through the placer and the GNN; cached
 * Transformer-XL states are stop-gradient.  grad += dL/dtheta.
 * Must follow gdp_embed and gdp_place of the same theta with the same ws.
 * Autoregressive mode (R35): p_v becomes the per-placement p_{b,v} of the decode, the entropy term
 * the mean over placements and nodes, and the gradient also reaches GDP_P_AR_E through EW.
 *   logits dev fp32 N x d;  placements dev uint8 B x N;  adv dev fp64 B
 *   logprob dev fp32 B (used only when old_logprob != NULL);  old_logprob dev fp32 B or NULL
 *   grad dev fp32 [n_params] (accumulated)
 * Errors: GDP_ERR_ARG, GDP_ERR_WORKSPACE, GDP_ERR_CUDA. */
gdp_status gdp_policy_grad(gdp_graph g, const gdp_config *c, const float *theta, const float *logits,
                           const uint8_t *placements, int32_t B, const double *adv, const float *logprob,
                           const float *old_logprob, float clip_eps, float entropy_coef, float loss_scale,
                           float *grad, void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------ training update */

/* log pi_b of GIVEN placements under the current logits ("pi(D|G)"):
 * sum over co-location leaders of log softmax(logits_v)[D_b v], fp64 sum in a fixed order.
 * The PPO epochs need it to form rho = exp(log pi_new - log pi_old).
 *   logits dev fp32 N x d (in);  placements dev uint8 B x N (in);  logprob dev fp32 B (out)
 * Uses the sampling scratch of ws (sized for B placements in autoregressive mode, where the
 * logits of each leader follow the GIVEN devices of the earlier leaders of its segment).
 * Errors: GDP_ERR_ARG, GDP_ERR_WORKSPACE, GDP_ERR_CUDA. */
gdp_status gdp_logprob(gdp_graph g, const gdp_config *c, const float *logits, const uint8_t *placements, int32_t B,
                       float *logprob, void *ws, size_t ws_bytes, void *stream);

/* Greedy decode for zero-shot placement: per node the
 * argmax of its co-location leader's logits, ties -> lowest device id; optional log pi of it.
 *   logits dev fp32 N x d (in);  placement dev uint8 N (out);  logprob dev fp32 [1] (out, nullable:
 *   then ws may be NULL, except in autoregressive mode, where each segment is decoded greedily
 *   position by position and ws is required).  Errors: GDP_ERR_ARG, GDP_ERR_WORKSPACE, GDP_ERR_CUDA. */
gdp_status gdp_greedy(gdp_graph g, const gdp_config *c, const float *logits, uint8_t *placement, float *logprob,
                      void *ws, size_t ws_bytes, void *stream);

/* Doubles of device scratch gdp_clip_adam needs. */
#define GDP_ADAM_SCRATCH 1024

/* Global-norm gradient clipping then one bias-corrected Adam step (
 * DESIGN.md readings R31, R32):
 *   s = min(1, max_norm / (||grad||_2 + 1e-6));  g = s * grad
 *   m = beta1 m + (1 - beta1) g;  v = beta2 v + (1 - beta2) g^2
 *   theta -= lr * (m / (1 - beta1^t)) / (sqrt(v / (1 - beta2^t)) + eps)
 * ||grad|| is summed in fp64 in a fixed order (deterministic); the update is evaluated in fp64
 * and stored as fp32.  All arrays are device pointers with 16-byte alignment:
 *   grad fp32 [n] (in);  theta, m, v fp32 [n] (in/out);  scratch fp64 [GDP_ADAM_SCRATCH];
 *   norm_out fp64 [1] (out, nullable: the pre-clip norm).  t >= 1 is the step number.
 * A non-finite gradient (NaN or Inf anywhere: ||grad|| is not finite) leaves theta, m and v
 * unchanged and norm_out reports the non-finite norm; gdp_grad_check then names the offending
 * parameter.
 * Errors: GDP_ERR_ARG (NULL, n < 1, t < 1, misaligned, beta outside [0, 1)), GDP_ERR_CUDA. */
gdp_status gdp_clip_adam(const float *grad, int64_t n, double max_norm, double lr, double beta1, double beta2,
                         double eps, int64_t t, float *theta, float *m, float *v, double *scratch, double *norm_out,
                         void *stream);

#ifdef __cplusplus
}
#endif
#endif /* GDP_H_ */
