// C ABI of libgdp.so (include/gdp.h): validation, graph/topology objects, parameter layout,
// workspace layout and the hot-path entry points.
#include <algorithm>
#include <cmath>
#include <atomic>
#include <climits>
#include <cstring>
#include <functional>
#include <mutex>
#include <queue>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"
#include "cost2.cuh"

namespace gdp {

static thread_local std::string g_err = "ok";

// an NVTX range around every hot-path ABI call (visible in nsys / ncu --nvtx; header-only NVTX3,
// a no-op without an attached tool)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
static std::atomic<unsigned long long> g_launches{0};

// per-launch timing (gdp_profile_*): an event before every launch; a launch's time is the gap
// to the next event recorded on the same stream (exact when the host runs ahead of the GPU)
struct ProfRec {
  const char *name;   // nullptr: closing mark
  cudaStream_t s;
  cudaEvent_t ev;
  double bytes, flops;
};
static std::mutex g_prof_mu;
static std::atomic<int> g_prof_on{0};
static std::vector<ProfRec> g_prof;
static std::vector<cudaEvent_t> g_prof_pool;

static void prof_record(const char *name, cudaStream_t s, double bytes, double flops) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  cudaEvent_t e;
  if (g_prof_pool.empty()) {
    if (cudaEventCreate(&e) != cudaSuccess) return;
  } else {
    e = g_prof_pool.back();
    g_prof_pool.pop_back();
  }
  cudaEventRecord(e, s);
  g_prof.push_back({name, s, e, bytes, flops});
}

void note_launch(const char *name, cudaStream_t s, double bytes, double flops) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (g_prof_on.load(std::memory_order_relaxed)) prof_record(name, s, bytes, flops);
}

void set_error(const std::string &msg) { g_err = msg; }

gdp_status cuda_status(cudaError_t e, const char *what) {
  set_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
  return GDP_ERR_CUDA;
}

static gdp_status fail(gdp_status s, const std::string &msg) {
  set_error(msg);
  return s;
}

// parameter tensor names in GDP_P_* order (error messages)
static const char *const kParamNames[GDP_P_COUNT] = {
    "gnn.in.W", "gnn.in.b", "gnn.0.W", "gnn.0.b", "gnn.0.Wf", "gnn.0.bf", "gnn.1.W", "gnn.1.b", "gnn.1.Wf",
    "gnn.1.bf", "gnn.2.W", "gnn.2.b", "gnn.2.Wf", "gnn.2.bf",
    "cond.ln1.g", "cond.ln1.b", "cond.Wq", "cond.bq", "cond.Wk", "cond.bk", "cond.Wv", "cond.bv", "cond.Wo",
    "cond.bo", "cond.ln2.g", "cond.ln2.b", "cond.W1", "cond.b1", "cond.W2", "cond.b2",
    "xl0.ln1.g", "xl0.ln1.b", "xl0.Wq", "xl0.bq", "xl0.Wk", "xl0.bk", "xl0.Wv", "xl0.bv", "xl0.Wo", "xl0.bo",
    "xl0.ln2.g", "xl0.ln2.b", "xl0.W1", "xl0.b1", "xl0.W2", "xl0.b2",
    "xl1.ln1.g", "xl1.ln1.b", "xl1.Wq", "xl1.bq", "xl1.Wk", "xl1.bk", "xl1.Wv", "xl1.bv", "xl1.Wo", "xl1.bo",
    "xl1.ln2.g", "xl1.ln2.b", "xl1.W1", "xl1.b1", "xl1.W2", "xl1.b2",
    "gate0.q.P", "gate0.q.q", "gate0.k.P", "gate0.k.q", "gate0.v.P", "gate0.v.q", "gate0.o.P", "gate0.o.q",
    "gate0.f1.P", "gate0.f1.q", "gate0.f2.P", "gate0.f2.q",
    "gate1.q.P", "gate1.q.q", "gate1.k.P", "gate1.k.q", "gate1.v.P", "gate1.v.q", "gate1.o.P", "gate1.o.q",
    "gate1.f1.P", "gate1.f1.q", "gate1.f2.P", "gate1.f2.q",
    "gate.head.P", "gate.head.q", "head.W", "head.b", "ar.E"};

// parameter tensor shapes in GDP_P_* order
static void param_shapes(int F, int d, bool ar, long long *sz) {
  const long long H = kH, FF = kFFN;
  int i = 0;
  sz[i++] = F * H; sz[i++] = H;
  for (int l = 0; l < kGNN; l++) { sz[i++] = H * H; sz[i++] = H; sz[i++] = 2 * H * H; sz[i++] = H; }
  for (int l = 0; l < 3; l++) {
    sz[i++] = H; sz[i++] = H;                       // ln1
    for (int j = 0; j < 4; j++) { sz[i++] = H * H; sz[i++] = H; }   // q k v o
    sz[i++] = H; sz[i++] = H;                       // ln2
    sz[i++] = H * FF; sz[i++] = FF;                 // W1 b1
    sz[i++] = FF * H; sz[i++] = H;                  // W2 b2
  }
  for (int l = 0; l < 2; l++)
    for (int j = 0; j < 6; j++) {
      long long w = j == 5 ? FF : H;
      sz[i++] = H * w; sz[i++] = w;
    }
  sz[i++] = H * H; sz[i++] = H;                     // head gate
  sz[i++] = H * d; sz[i++] = d;                     // head
  sz[i++] = ar ? (long long)d * H : 0;              // autoregressive device embedding
}

void param_offsets(int F, int d, long long *off, bool ar) {
  long long sz[GDP_P_COUNT];
  param_shapes(F, d, ar, sz);
  off[0] = 0;
  for (int i = 0; i < GDP_P_COUNT; i++) off[i + 1] = off[i] + sz[i];
}

static gdp_status check_config(const gdp_config *c) {
  if (!c) return fail(GDP_ERR_ARG, "config is NULL");
  if (c->hidden != kH || c->heads != kHeads || c->gnn_layers != kGNN || c->xl_layers != 2 || c->ffn != kFFN)
    return fail(GDP_ERR_ARG, "unsupported network size (need hidden 64, heads 4, gnn_layers 3, xl_layers 2, ffn 256)");
  if (c->num_devices < 1 || c->num_devices > kMaxD) return fail(GDP_ERR_ARG, "num_devices must be in 1..8");
  if (c->seg_len < 1) return fail(GDP_ERR_ARG, "seg_len must be >= 1");
  if (c->mem_len < -1) return fail(GDP_ERR_ARG, "mem_len must be >= -1");
  if (c->autoregressive != 0 && c->autoregressive != 1) return fail(GDP_ERR_ARG, "autoregressive must be 0 or 1");
  if (c->autoregressive && c->active_devices != 0 && c->active_devices != c->num_devices)
    return fail(GDP_ERR_ARG, "the autoregressive placer needs active_devices = 0");
  if (c->tensor_cores < 0 || c->tensor_cores > 2) return fail(GDP_ERR_ARG, "tensor_cores must be 0, 1 or 2");
  if (c->no_attention != 0 && c->no_attention != 1) return fail(GDP_ERR_ARG, "no_attention must be 0 or 1");
  if (c->active_devices < 0 || c->active_devices > c->num_devices)
    return fail(GDP_ERR_ARG, "active_devices must be in 0..num_devices");
  return GDP_OK;
}

int active_devices(const gdp_config *c) { return c->active_devices > 0 ? c->active_devices : c->num_devices; }

// ------------------------------------------------------------------ workspace
static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

bool ws_layout(const gdp_graph_s *g, int d, int B, char *base, WS *w) {
  const size_t N = (size_t)g->N, E = (size_t)(g->E > 0 ? g->E : 1);
  size_t off = 0;
  auto take = [&](size_t bytes) -> char * {
    char *p = base ? base + off : nullptr;
    off += align_up(bytes);
    return p;
  };
  auto F32 = [&](size_t n) { return reinterpret_cast<float *>(take(n * sizeof(float))); };
  WS z{};
  for (int i = 0; i < 4; i++) z.H[i] = F32(N * kH);
  for (int i = 0; i < 3; i++) {
    z.Z[i] = F32(N * kH);
    z.A[i] = F32(N * kH);
    z.ARG[i] = reinterpret_cast<int *>(take(N * kH * sizeof(int)));
  }
  z.Etopo = F32(N * kH);
  z.zsum = F32(kH);
  z.z = F32(kH);
  z.gam = F32(kGamTotal);
  z.Wh = F32(kH * kMaxD);
  z.dWh = F32((kH + 1) * kMaxD);
  z.logits_topo = F32(N * kMaxD);
  for (int l = 0; l < 3; l++) {
    Layer &L = z.L[l];
    L.x = nullptr;
    L.a = F32(N * kH);
    L.mu1 = F32(N);
    L.rs1 = F32(N);
    L.qkv = F32(N * 192);
    L.o = F32(N * kH);
    L.lse = F32(N * kHeads);
    L.x1 = F32(N * kH);
    L.c = F32(N * kH);
    L.mu2 = F32(N);
    L.rs2 = F32(N);
    L.m = F32(N * kFFN);
    L.y = F32(N * kH);
    L.Wqkv = F32(64 * 192);
    L.bqkv = F32(192);
    L.Wo = F32(64 * 64);
    L.W1 = F32(64 * 256);
    L.W2 = F32(256 * 64);
    L.dWqkv = F32(65 * 192);
    L.dWo = F32(65 * 64);
    L.dW1 = F32(65 * 256);
    L.dW2 = F32(257 * 64);
  }
  z.dlog = F32(N * kMaxD);
  z.dlog_topo = F32(N * kMaxD);
  z.dy = F32(N * kH);
  z.dx1 = F32(N * kH);
  z.dm = F32(N * kFFN);
  z.dc = F32(N * kH);
  z.dout = F32(N * kH);
  z.dqkv = F32(N * 192);
  z.dkvm = F32(N * 128);
  z.dkvt = F32(N * 192);
  z.da = F32(N * kH);
  z.dam = F32(N * kH);
  z.dxa = F32(N * kH);
  z.dEt = F32(N * kH);
  z.dE = F32(N * kH);
  z.dH = F32(N * kH);
  z.dHn = F32(N * kH);
  z.dAg = F32(N * kH);
  z.dP = F32(N * kH);
  z.dd = F32(N * kHeads);
  z.dEW = F32(kMaxD * kMaxD);
  const size_t chunks = (N + 255) / 256 + 1;
  z.part_floats = chunks * 257 * 256;
  z.part = F32(z.part_floats);
  z.dgam = F32(kGamTotal);
  z.dz = F32(kH);
  z.dzp = F32(kH * kGateCount);
  z.cdf = F32(N * kMaxD);
  z.logp = F32(N * kMaxD);
  z.lastpos = reinterpret_cast<int *>(take(N * sizeof(int)));
  z.lpart = reinterpret_cast<double *>(take((size_t)kLogitChunks * N * kMaxD * sizeof(double)));
  const size_t Bc = (size_t)std::max(B, 1);
  // everything below depends on B (kept last so the offsets above never move)
  z.wb = reinterpret_cast<double *>(take(Bc * sizeof(double)));
  {  // sampling: log pi partial sums per placement and 128-node warp chunk (k_sample)
    const size_t nq = (N + 3) / 4, nwc = (nq + 255) / 256 * 8;
    z.spart = reinterpret_cast<double *>(take(Bc * nwc * sizeof(double)));
  }
  // cost scratch: one region per placement, large enough for either cost kernel
  size_t v1 = (2 + 2) * N * sizeof(int) + N * sizeof(int2) + E * sizeof(int4) + N * sizeof(int);
  size_t v2 = cost2_scratch_per_placement(g->N, g->E, g->nbig);
  size_t v5 = cost5_scratch_per_placement(g->N, g->E, g->ngbig5);
  z.c_per_place = (std::max(std::max(v1, v2), v5) + 255) & ~(size_t)255;
  z.c_scratch = reinterpret_cast<unsigned char *>(take(Bc * z.c_per_place));
  if (z.c_scratch) {
    // v1 view of the same bytes
    z.c_rem = reinterpret_cast<int *>(z.c_scratch);
    z.c_rcons = z.c_rem + Bc * N;
    z.c_new = z.c_rcons + Bc * N;
    z.c_fifo = reinterpret_cast<int2 *>(z.c_new + Bc * 2 * N);
    z.c_chq = reinterpret_cast<int4 *>(z.c_fifo + Bc * N);
  }
  z.bytes = off;
  (void)d;
  *w = z;
  return true;
}

}  // namespace gdp

using namespace gdp;

// per-call workspace check: ws must hold the layout for (graph, B)
static gdp_status carve(const gdp_graph_s *g, int d, int B, void *ws, size_t ws_bytes, WS *w) {
  WS probe;
  ws_layout(g, d, B, nullptr, &probe);
  if (!ws) return fail(GDP_ERR_ARG, "workspace is NULL");
  if (ws_bytes < probe.bytes)
    return fail(GDP_ERR_WORKSPACE, "workspace too small: need " + std::to_string(probe.bytes) + " bytes, got " +
                                       std::to_string(ws_bytes));
  ws_layout(g, d, B, static_cast<char *>(ws), w);
  return GDP_OK;
}


namespace gdp {
gdp_status run_embed(const gdp_graph_s *g, const float *theta, float *node_emb, const WS &w, int d, cudaStream_t s);
gdp_status run_place(const gdp_graph_s *g, const gdp_config *c, const float *theta, const float *node_emb,
                     float *logits, const WS &w, cudaStream_t s);
gdp_status run_policy_grad(const gdp_graph_s *g, const gdp_config *c, const float *theta, const float *logits,
                           const uint8_t *D, int B, const double *adv, const float *logprob,
                           const float *old_logprob, float eps, float beta, float scale, float *grad, const WS &w,
                           cudaStream_t s, cudaEvent_t const *bucket_done);
void launch_grad_sum(const float *const *grads, int n, long long len, float *out, cudaStream_t s);
}  // namespace gdp

extern "C" {

const char *gdp_last_error(void) { return g_err.c_str(); }

uint64_t gdp_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

gdp_status gdp_profile_enable(int32_t on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (on) {
    for (auto &r : g_prof) g_prof_pool.push_back(r.ev);
    g_prof.clear();
  }
  g_prof_on.store(on ? 1 : 0);
  return GDP_OK;
}

gdp_status gdp_profile_mark(void *stream) {
  if (!g_prof_on.load()) return fail(GDP_ERR_ARG, "profiling is not enabled");
  prof_record(nullptr, static_cast<cudaStream_t>(stream), 0.0, 0.0);
  return GDP_OK;
}

int32_t gdp_profile_read(int32_t max_names, const char **names, int32_t *launches, double *ms, double *bytes,
                         double *flops) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (max_names < 0 || (max_names > 0 && (!names || !launches || !ms || !bytes || !flops))) {
    set_error("gdp_profile_read: bad arguments");
    return -1;
  }
  for (auto &r : g_prof)
    if (cudaEventSynchronize(r.ev) != cudaSuccess) {
      set_error("gdp_profile_read: event synchronisation failed");
      return -1;
    }
  int n = 0;
  for (size_t i = 0; i < g_prof.size(); i++) {
    const ProfRec &r = g_prof[i];
    if (!r.name) continue;
    size_t j = i + 1;
    while (j < g_prof.size() && g_prof[j].s != r.s) j++;
    if (j == g_prof.size()) continue;   // no later event on its stream: untimed
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r.ev, g_prof[j].ev) != cudaSuccess) continue;
    int k = 0;
    while (k < n && std::strcmp(names[k], r.name) != 0) k++;
    if (k == n) {
      if (n == max_names) continue;
      names[n] = r.name; launches[n] = 0; ms[n] = 0.0; bytes[n] = 0.0; flops[n] = 0.0;
      n++;
    }
    launches[k] += 1; ms[k] += t; bytes[k] += r.bytes; flops[k] += r.flops;
  }
  return n;
}

const char *gdp_build_info(void) { return "libgdp sm_100a built " __DATE__ " " __TIME__; }

int32_t gdp_cost_wave(gdp_graph g, gdp_topo t) {
  if (!g || !t) { set_error("gdp_cost_wave: NULL handle"); return 0; }
  return cost_wave(g, t);
}

int32_t gdp_cost_kernel(gdp_graph g, gdp_topo t) {
  if (!g || !t) { set_error("gdp_cost_kernel: NULL handle"); return 0; }
  return cost_kernel_choice(g, t, 0);
}

gdp_status gdp_default_config(int32_t d, gdp_config *out) {
  if (!out) return fail(GDP_ERR_ARG, "out is NULL");
  if (d < 1 || d > kMaxD) return fail(GDP_ERR_ARG, "d must be in 1..8");
  out->hidden = kH;
  out->heads = kHeads;
  out->gnn_layers = kGNN;
  out->xl_layers = 2;
  out->ffn = kFFN;
  out->num_devices = d;
  out->seg_len = 128;
  out->mem_len = 128;
  out->superposition = 1;
  out->tensor_cores = 0;
  out->no_attention = 0;
  out->active_devices = 0;
  out->autoregressive = 0;
  return GDP_OK;
}

gdp_status gdp_graph_validate(int32_t N, int64_t E, const int32_t *edges, int32_t *topo_order) {
  if (N <= 0) return fail(GDP_ERR_ARG, "N must be > 0");
  if (E < 0) return fail(GDP_ERR_ARG, "E must be >= 0");
  if (E > 0 && !edges) return fail(GDP_ERR_ARG, "edges is NULL");
  if (E >= INT_MAX) return fail(GDP_ERR_ARG, "too many edges");
  std::vector<std::pair<int, int>> es((size_t)E);
  for (int64_t e = 0; e < E; e++) {
    int u = edges[2 * e], v = edges[2 * e + 1];
    if (u < 0 || u >= N || v < 0 || v >= N)
      return fail(GDP_ERR_GRAPH, "edge " + std::to_string(e) + " has an endpoint out of range");
    if (u == v) return fail(GDP_ERR_GRAPH, "self edge at node " + std::to_string(u));
    es[(size_t)e] = {u, v};
  }
  std::sort(es.begin(), es.end());
  for (size_t i = 1; i < es.size(); i++)
    if (es[i] == es[i - 1])
      return fail(GDP_ERR_GRAPH, "duplicate edge " + std::to_string(es[i].first) + "->" + std::to_string(es[i].second));
  std::vector<int> indeg(N, 0), ptr(N + 1, 0);
  for (auto &p : es) { indeg[p.second]++; ptr[p.first + 1]++; }
  for (int v = 0; v < N; v++) ptr[v + 1] += ptr[v];
  std::priority_queue<int, std::vector<int>, std::greater<int>> q;
  for (int v = 0; v < N; v++)
    if (!indeg[v]) q.push(v);
  int n = 0;
  while (!q.empty()) {
    int u = q.top();
    q.pop();
    if (topo_order) topo_order[n] = u;
    n++;
    for (int e = ptr[u]; e < ptr[u + 1]; e++)
      if (--indeg[es[e].second] == 0) q.push(es[e].second);
  }
  if (n != N) return fail(GDP_ERR_CYCLE, "the edge list has a cycle");
  return GDP_OK;
}

gdp_status gdp_graph_create(int32_t N, int32_t F, const float *feat, int64_t E, const int32_t *edges,
                            const int64_t *compute_cost, const int64_t *output_bytes, const int64_t *memory_bytes,
                            const int32_t *coloc_group, gdp_graph *out) {
  if (!out) return fail(GDP_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (N <= 0 || F <= 0) return fail(GDP_ERR_ARG, "N and F must be > 0");
  if (!feat || !compute_cost || !output_bytes || !memory_bytes) return fail(GDP_ERR_ARG, "NULL input array");
  for (int v = 0; v < N; v++) {
    if (compute_cost[v] < 0 || compute_cost[v] > INT_MAX)
      return fail(GDP_ERR_GRAPH, "compute_cost out of range at node " + std::to_string(v));
    if (output_bytes[v] < 0 || memory_bytes[v] < 0)
      return fail(GDP_ERR_GRAPH, "negative bytes at node " + std::to_string(v));
  }
  std::vector<int> order(N);
  gdp_status st = gdp_graph_validate(N, E, edges, order.data());
  if (st != GDP_OK) return st;
  auto *g = new gdp_graph_s();
  g->N = N;
  g->F = F;
  g->ldX = (F + 3) / 4 * 4;
  g->E = E;
  GDP_CUDA_CHECK(cudaGetDevice(&g->device));
  // out / in CSR
  std::vector<std::pair<int, int>> es((size_t)E);
  for (int64_t e = 0; e < E; e++) es[(size_t)e] = {edges[2 * e], edges[2 * e + 1]};
  std::sort(es.begin(), es.end());
  std::vector<int> optr(N + 1, 0), iptr(N + 1, 0), oidx((size_t)E), osrc((size_t)E), iidx((size_t)E);
  for (auto &p : es) { optr[p.first + 1]++; iptr[p.second + 1]++; }
  for (int v = 0; v < N; v++) { optr[v + 1] += optr[v]; iptr[v + 1] += iptr[v]; }
  {
    std::vector<int> fi(iptr.begin(), iptr.end() - 1);
    for (size_t e = 0; e < es.size(); e++) {
      oidx[e] = es[e].second;
      osrc[e] = es[e].first;
      iidx[fi[es[e].second]++] = es[e].first;   // producers ascending (es sorted by producer)
    }
  }
  // symmetric neighbourhood N(v) = preds U succs, ascending, unique
  std::vector<std::pair<int, int>> sym;
  sym.reserve(2 * (size_t)E);
  for (auto &p : es) { sym.push_back({p.first, p.second}); sym.push_back({p.second, p.first}); }
  std::sort(sym.begin(), sym.end());
  sym.erase(std::unique(sym.begin(), sym.end()), sym.end());
  std::vector<int> nptr(N + 1, 0), nidx(sym.size());
  for (size_t i = 0; i < sym.size(); i++) { nptr[sym[i].first + 1]++; nidx[i] = sym[i].second; }
  for (int v = 0; v < N; v++) nptr[v + 1] += nptr[v];
  g->E_sym = (int64_t)sym.size();
  // leaders (lowest id of each co-location group)
  std::vector<int> leader(N);
  for (int v = 0; v < N; v++) leader[v] = v;
  if (coloc_group) {
    std::vector<std::pair<int, int>> first;
    std::vector<int> gid_first;
    // map group id -> first member via sorting (ids may be sparse)
    std::vector<std::pair<int, int>> gm;
    for (int v = 0; v < N; v++)
      if (coloc_group[v] >= 0) gm.push_back({coloc_group[v], v});
    std::sort(gm.begin(), gm.end());
    for (size_t i = 0; i < gm.size(); i++) {
      size_t j = i;
      while (j + 1 < gm.size() && gm[j + 1].first == gm[i].first) j++;
      for (size_t k = i; k <= j; k++) leader[gm[k].second] = gm[i].second;
      if (j > i) g->has_coloc = true;
      i = j;
    }
  }
  std::vector<int> cost(N);
  long long sum_cost = 0, sum_edge_out = 0;
  for (int v = 0; v < N; v++) { cost[v] = (int)compute_cost[v]; sum_cost += compute_cost[v]; }
  g->min_edge_bytes = LLONG_MAX;
  for (auto &p : es) {
    sum_edge_out += output_bytes[p.first];
    g->min_edge_bytes = std::min<long long>(g->min_edge_bytes, output_bytes[p.first]);
  }
  g->sum_cost = sum_cost;
  g->sum_edge_out_bytes = sum_edge_out;
  bool ident = true;
  for (int i = 0; i < N; i++)
    if (order[i] != i) ident = false;
  g->perm_identity = ident;
  g->min_cost = N > 0 ? INT_MAX : 0;
  for (int v = 0; v < N; v++) {
    g->min_cost = std::min(g->min_cost, (int)cost[v]);
    g->max_indeg = std::max(g->max_indeg, iptr[v + 1] - iptr[v]);
    g->max_outdeg = std::max(g->max_outdeg, optr[v + 1] - optr[v]);
  }
  // records of the shared-memory cost model
  std::vector<NRec> nrec(N), erec((size_t)std::max<int64_t>(E, 1));
  std::vector<IRec> irec((size_t)std::max<int64_t>(E, 1));
  for (int v = 0; v < N; v++) {
    NRec &r = nrec[v];
    r.id = v; r.cost = cost[v]; r.ob = optr[v]; r.oe = optr[v + 1]; r.ib = iptr[v]; r.ie = iptr[v + 1];
    r.bytes = output_bytes[v];
  }
  for (int64_t e = 0; e < E; e++) {
    erec[(size_t)e] = nrec[oidx[(size_t)e]];
    irec[(size_t)e].u = iidx[(size_t)e];
    irec[(size_t)e].bytes = output_bytes[iidx[(size_t)e]];
  }
  std::vector<unsigned> cnt0((N + 3) / 4, 0u);
  std::vector<int> bigid(N, -1), big_in, big_out;
  for (int v = 0; v < N; v++) {
    int din = iptr[v + 1] - iptr[v], dout = optr[v + 1] - optr[v];
    unsigned nib_in = din, nib_out = dout;
    if (din >= 15 || dout >= 15) {
      bigid[v] = (int)big_in.size();
      big_in.push_back(din);
      big_out.push_back(dout);
      if (din >= 15) nib_in = 15;
      if (dout >= 15) nib_out = 15;
    }
    // a big node keeps the sentinel in BOTH nibbles so that both counters use the global path
    if (bigid[v] >= 0) { nib_in = 15; nib_out = 15; }
    cnt0[v >> 2] |= (nib_in | (nib_out << 4)) << ((v & 3) * 8);
  }
  // k_cost3 reads the counter kind from the records: NRec.cost bit 31 = op with global
  // counters, IRec.pad = the producer's global counter index (or -1)
  for (int v = 0; v < N; v++)
    if (bigid[v] >= 0) nrec[v].cost |= (int)0x80000000u;
  for (int64_t e = 0; e < E; e++) {
    erec[(size_t)e] = nrec[oidx[(size_t)e]];
    irec[(size_t)e].pad = bigid[iidx[(size_t)e]];
  }
  g->nbig = (int)big_in.size();
  if (big_in.empty()) { big_in.push_back(0); big_out.push_back(0); }
  auto up = [&](void **dst, const void *src, size_t bytes) -> cudaError_t {
    cudaError_t e = cudaMalloc(dst, bytes ? bytes : 4);
    if (e != cudaSuccess) return e;
    if (bytes) return cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
    return cudaSuccess;
  };
#define UP(field, src, bytes)                                                   \
  do {                                                                          \
    cudaError_t _e = up(reinterpret_cast<void **>(&g->field), (src), (bytes));  \
    if (_e != cudaSuccess) { gdp_graph_destroy(g); return cuda_status(_e, "graph upload"); } \
  } while (0)
  {
    std::vector<float> xp((size_t)N * g->ldX, 0.f);   // rows padded to 16 bytes (TMA row stride)
    for (int v = 0; v < N; v++)
      for (int f = 0; f < F; f++) xp[(size_t)v * g->ldX + f] = feat[(size_t)v * F + f];
    UP(X, xp.data(), xp.size() * sizeof(float));
  }
  UP(nbr_ptr, nptr.data(), (N + 1) * sizeof(int));
  UP(nbr_idx, nidx.data(), nidx.size() * sizeof(int));
  {
    std::vector<int> heavy;
    for (int v = 0; v < N; v++)
      if (nptr[v + 1] - nptr[v] > kHeavyDeg) heavy.push_back(v);
    g->n_heavy = (int)heavy.size();
    UP(heavy, heavy.data(), heavy.size() * sizeof(int));
  }
  UP(out_ptr, optr.data(), (N + 1) * sizeof(int));
  UP(out_idx, oidx.data(), oidx.size() * sizeof(int));
  UP(out_src, osrc.data(), osrc.size() * sizeof(int));
  UP(in_ptr, iptr.data(), (N + 1) * sizeof(int));
  UP(in_idx, iidx.data(), iidx.size() * sizeof(int));
  UP(cost, cost.data(), N * sizeof(int));
  UP(out_bytes, output_bytes, N * sizeof(long long));
  UP(mem_bytes, memory_bytes, N * sizeof(long long));
  UP(perm, order.data(), N * sizeof(int));
  UP(leader, leader.data(), N * sizeof(int));
  UP(nrec, nrec.data(), nrec.size() * sizeof(NRec));
  UP(erec, erec.data(), erec.size() * sizeof(NRec));
  UP(irec, irec.data(), irec.size() * sizeof(IRec));
  UP(cnt0, cnt0.data(), cnt0.size() * sizeof(unsigned));
  UP(bigid, bigid.data(), N * sizeof(int));
  UP(big_in, big_in.data(), big_in.size() * sizeof(int));
  UP(big_out, big_out.data(), big_out.size() * sizeof(int));
  {
    Cost5Host h5;
    cost5_build(N, E, optr.data(), oidx.data(), iptr.data(), cost.data(), reinterpret_cast<const long long *>(output_bytes),
                &h5);
    g->c5_ok = h5.ok;
    g->nsrc5 = (int)h5.srcq.size();
    g->nbigb5 = (int)h5.bigb.size();
    g->ngbig5 = (int)h5.gbig.size();
    g->nflagw5 = h5.nflagw;
    g->bytes32_5 = h5.bytes32 ? 1 : 0;
    UP(slots5, h5.slots.data(), h5.slots.size() * sizeof(Slot5));
    UP(ebytes5, h5.ebytes.data(), h5.ebytes.size() * sizeof(long long));
    UP(srcq5, h5.srcq.data(), h5.srcq.size() * sizeof(Slot5));
    UP(gbig5, h5.gbig.data(), h5.gbig.size() * sizeof(int));
    UP(outdeg5, h5.outdeg.data(), h5.outdeg.size() * sizeof(int));
    UP(bigb5, h5.bigb.data(), h5.bigb.size() * sizeof(unsigned));
  }
#undef UP
  *out = g;
  return GDP_OK;
}

gdp_status gdp_graph_destroy(gdp_graph g) {
  if (!g) return GDP_OK;
  void *ptrs[] = {g->X, g->nbr_ptr, g->nbr_idx, g->heavy, g->out_ptr, g->out_idx, g->out_src, g->in_ptr, g->in_idx,
                  g->cost, g->out_bytes, g->mem_bytes, g->perm, g->leader, g->nrec, g->erec, g->irec,
                  g->cnt0, g->bigid, g->big_in, g->big_out, g->slots5, g->srcq5, g->ebytes5, g->gbig5, g->outdeg5,
                  g->bigb5};
  for (void *p : ptrs)
    if (p) cudaFree(p);
  delete g;
  return GDP_OK;
}

gdp_status gdp_topo_create(int32_t d, const int64_t *mem_capacity, const int32_t *speed,
                           const int64_t *bytes_per_tick, const int32_t *latency, gdp_topo *out) {
  if (!out) return fail(GDP_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (d < 1 || d > kMaxD) return fail(GDP_ERR_ARG, "d must be in 1..8");
  if (!mem_capacity || !speed || !bytes_per_tick || !latency) return fail(GDP_ERR_ARG, "NULL topology array");
  auto *t = new gdp_topo_s();
  t->d = d;
  for (int i = 0; i < 8; i++) { t->cap[i] = 0; t->speed[i] = 1; }
  for (int i = 0; i < 64; i++) { t->bpt[i] = 1; t->lat[i] = 0; }
  for (int k = 0; k < d; k++) {
    if (speed[k] <= 0) { delete t; return fail(GDP_ERR_ARG, "speed must be > 0"); }
    if (mem_capacity[k] < 0) { delete t; return fail(GDP_ERR_ARG, "mem_capacity must be >= 0"); }
    t->cap[k] = mem_capacity[k];
    t->speed[k] = speed[k];
  }
  for (int s = 0; s < d; s++)
    for (int u = 0; u < d; u++) {
      if (s == u) continue;
      long long bw = bytes_per_tick[s * d + u];
      int la = latency[s * d + u];
      if (bw <= 0 || la < 0) { delete t; return fail(GDP_ERR_ARG, "bandwidth must be > 0 and latency >= 0 off the diagonal"); }
      if (bw != bytes_per_tick[u * d + s]) { delete t; return fail(GDP_ERR_ARG, "bandwidth must be symmetric"); }
      t->bpt[s * 8 + u] = bw;
      t->lat[s * 8 + u] = la;
    }
  *out = t;
  return GDP_OK;
}

gdp_status gdp_topo_destroy(gdp_topo t) {
  delete t;
  return GDP_OK;
}

gdp_status gdp_param_layout(const gdp_config *c, int32_t F, int64_t *offsets, int64_t *n_params) {
  gdp_status st = check_config(c);
  if (st != GDP_OK) return st;
  if (F <= 0) return fail(GDP_ERR_ARG, "F must be > 0");
  long long off[GDP_P_COUNT + 1];
  param_offsets(F, c->num_devices, off, c->autoregressive != 0);
  if (offsets)
    for (int i = 0; i <= GDP_P_COUNT; i++) offsets[i] = off[i];
  if (n_params) *n_params = off[GDP_P_COUNT];
  return GDP_OK;
}

gdp_status gdp_workspace_size(gdp_graph g, const gdp_config *c, int32_t B, size_t *bytes) {
  if (!g || !bytes) return fail(GDP_ERR_ARG, "NULL argument");
  gdp_status st = check_config(c);
  if (st != GDP_OK) return st;
  if (B < 1) return fail(GDP_ERR_ARG, "B must be >= 1");
  WS w;
  ws_layout(g, c->num_devices, B, nullptr, &w);
  *bytes = w.bytes;
  return GDP_OK;
}

// Offsets of everything embed/place save for policy_grad do not depend on B (the B-sized
// scratch is carved last), so each call carves for the B it is given.
static gdp_status carve_any(const gdp_graph_s *g, int d, int Bneed, void *ws, size_t ws_bytes, WS *w) {
  return carve(g, d, Bneed, ws, ws_bytes, w);
}

int32_t gdp_debug_tensors(gdp_graph g, const gdp_config *c, int32_t max_names, const char **names, int64_t *offsets,
                          int64_t *rows, int64_t *cols, int32_t *is_int) {
  if (!g || max_names < 0 || (max_names > 0 && (!names || !offsets || !rows || !cols || !is_int))) {
    set_error("gdp_debug_tensors: bad arguments");
    return -1;
  }
  if (check_config(c) != GDP_OK) return -1;
  static const char kLayerNames[3][16][12] = {
      {"L0.a", "L0.qkv", "L0.o", "L0.lse", "L0.x1", "L0.c", "L0.m", "L0.y", "L0.Wqkv", "L0.bqkv", "L0.Wo", "L0.W1", "L0.W2", "L0.mu1", "L0.rs1", "L0.mu2"},
      {"L1.a", "L1.qkv", "L1.o", "L1.lse", "L1.x1", "L1.c", "L1.m", "L1.y", "L1.Wqkv", "L1.bqkv", "L1.Wo", "L1.W1", "L1.W2", "L1.mu1", "L1.rs1", "L1.mu2"},
      {"L2.a", "L2.qkv", "L2.o", "L2.lse", "L2.x1", "L2.c", "L2.m", "L2.y", "L2.Wqkv", "L2.bqkv", "L2.Wo", "L2.W1", "L2.W2", "L2.mu1", "L2.rs1", "L2.mu2"}};
  static const char kGnn[4][3][6] = {{"H0", "Z0", "A0"}, {"H1", "Z1", "A1"}, {"H2", "Z2", "A2"}, {"H3", "", ""}};
  static const char kArg[3][6] = {"ARG0", "ARG1", "ARG2"};
  char *base = reinterpret_cast<char *>((uintptr_t)1 << 40);   // any base: only offsets are returned
  WS w;
  ws_layout(g, c->num_devices, 1, base, &w);
  const long long N = g->N;
  int n = 0;
  auto add = [&](const char *nm, const void *p, long long r, long long cc, int isint) {
    if (n < max_names) {
      names[n] = nm; offsets[n] = (int64_t)(reinterpret_cast<const char *>(p) - base); rows[n] = r; cols[n] = cc;
      is_int[n] = isint;
    }
    n++;
  };
  for (int l = 0; l < 4; l++) {
    add(kGnn[l][0], w.H[l], N, kH, 0);
    if (l < 3) { add(kGnn[l][1], w.Z[l], N, kH, 0); add(kGnn[l][2], w.A[l], N, kH, 0); add(kArg[l], w.ARG[l], N, kH, 1); }
  }
  add("Etopo", w.Etopo, N, kH, 0);
  add("z", w.z, 1, kH, 0);
  add("gam", w.gam, 1, kGamTotal, 0);
  add("Wh", w.Wh, kH, c->num_devices, 0);
  for (int l = 0; l < 3; l++) {
    const Layer &L = w.L[l];
    const void *ps[16] = {L.a, L.qkv, L.o, L.lse, L.x1, L.c, L.m, L.y, L.Wqkv, L.bqkv, L.Wo, L.W1, L.W2, L.mu1, L.rs1, L.mu2};
    const long long rs[16] = {N, N, N, N, N, N, N, N, kH, 1, kH, kH, kFFN, N, N, N};
    const long long cs[16] = {kH, 192, kH, kHeads, kH, kH, kFFN, kH, 192, 192, kH, kFFN, kH, 1, 1, 1};
    for (int j = 0; j < 16; j++) add(kLayerNames[l][j], ps[j], rs[j], cs[j], 0);
  }
  static const char kDW[3][4][10] = {{"L0.dWqkv", "L0.dWo", "L0.dW1", "L0.dW2"},
                                     {"L1.dWqkv", "L1.dWo", "L1.dW1", "L1.dW2"},
                                     {"L2.dWqkv", "L2.dWo", "L2.dW1", "L2.dW2"}};
  for (int l = 0; l < 3; l++) {   // weight gradients of the folded maps, bias row last
    add(kDW[l][0], w.L[l].dWqkv, kH + 1, 192, 0);
    add(kDW[l][1], w.L[l].dWo, kH + 1, kH, 0);
    add(kDW[l][2], w.L[l].dW1, kH + 1, kFFN, 0);
    add(kDW[l][3], w.L[l].dW2, kFFN + 1, kH, 0);
  }
  add("dlog", w.dlog, N, c->num_devices, 0);
  add("dy", w.dy, N, kH, 0);
  add("dx1", w.dx1, N, kH, 0);
  add("dm", w.dm, N, kFFN, 0);
  add("dc", w.dc, N, kH, 0);
  add("dout", w.dout, N, kH, 0);
  add("dqkv", w.dqkv, N, 192, 0);
  add("dkvm", w.dkvm, N, 128, 0);
  add("da", w.da, N, kH, 0);
  add("dam", w.dam, N, kH, 0);
  add("dEt", w.dEt, N, kH, 0);
  add("dH", w.dH, N, kH, 0);
  add("dHn", w.dHn, N, kH, 0);
  add("dAg", w.dAg, N, kH, 0);
  add("dP", w.dP, N, kH, 0);
  return n;
}

gdp_status gdp_embed(gdp_graph g, const gdp_config *c, const float *theta, float *node_emb, void *ws,
                     size_t ws_bytes, void *stream) {
  NvtxRange nvtx_("gdp_embed");
  if (!g || !theta || !node_emb) return fail(GDP_ERR_ARG, "NULL argument");
  gdp_status st = check_config(c);
  if (st != GDP_OK) return st;
  WS w;
  st = carve_any(g, c->num_devices, 1, ws, ws_bytes, &w);
  if (st != GDP_OK) return st;
  set_tensor_cores(c->tensor_cores);
  set_no_attention(c->no_attention != 0);
  return run_embed(g, theta, node_emb, w, c->num_devices, static_cast<cudaStream_t>(stream));
}

gdp_status gdp_place(gdp_graph g, const gdp_config *c, const float *theta, const float *node_emb, float *logits,
                     void *ws, size_t ws_bytes, void *stream) {
  NvtxRange nvtx_("gdp_place");
  if (!g || !theta || !node_emb || !logits) return fail(GDP_ERR_ARG, "NULL argument");
  gdp_status st = check_config(c);
  if (st != GDP_OK) return st;
  WS w;
  st = carve_any(g, c->num_devices, 1, ws, ws_bytes, &w);
  if (st != GDP_OK) return st;
  set_tensor_cores(c->tensor_cores);
  set_no_attention(c->no_attention != 0);
  return run_place(g, c, theta, node_emb, logits, w, static_cast<cudaStream_t>(stream));
}

static gdp_status sample_impl(gdp_graph g, const gdp_config *c, const float *logits, int32_t B, uint64_t seed,
                              uint64_t sample_offset, uint64_t step, const uint64_t *step_dev, uint8_t *placements,
                              float *logprob, void *ws, size_t ws_bytes, void *stream) {
  if (!g || !logits || !placements || !logprob) return fail(GDP_ERR_ARG, "NULL argument");
  gdp_status st = check_config(c);
  if (st != GDP_OK) return st;
  if (B < 1) return fail(GDP_ERR_ARG, "B must be >= 1");
  WS w;
  st = carve_any(g, c->num_devices, B, ws, ws_bytes, &w);
  if (st != GDP_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (c->autoregressive)
    launch_ar_decode(kArDecodeSample, logits, g->perm, g->leader, g->has_coloc, g->N, c->num_devices, c->seg_len, B,
                     seed, sample_offset, step, step_dev, placements, w.spart, logprob, s);
  else
    launch_sample(logits, c->num_devices, g->leader, g->has_coloc, g->N, active_devices(c), B, seed, sample_offset,
                  step, step_dev, w.cdf, w.logp, w.lastpos, w.spart, placements, logprob, s);
  GDP_LAUNCH_CHECK("gdp_sample");
  return GDP_OK;
}

gdp_status gdp_sample(gdp_graph g, const gdp_config *c, const float *logits, int32_t B, uint64_t seed,
                      uint64_t sample_offset, uint64_t step, uint8_t *placements, float *logprob, void *ws,
                      size_t ws_bytes, void *stream) {
  NvtxRange nvtx_("gdp_sample");
  return sample_impl(g, c, logits, B, seed, sample_offset, step, nullptr, placements, logprob, ws, ws_bytes, stream);
}

gdp_status gdp_sample_at(gdp_graph g, const gdp_config *c, const float *logits, int32_t B, uint64_t seed,
                         uint64_t sample_offset, const uint64_t *step_dev, uint8_t *placements, float *logprob,
                         void *ws, size_t ws_bytes, void *stream) {
  NvtxRange nvtx_("gdp_sample_at");
  if (!step_dev) return fail(GDP_ERR_ARG, "NULL step pointer");
  return sample_impl(g, c, logits, B, seed, sample_offset, 0, step_dev, placements, logprob, ws, ws_bytes, stream);
}

gdp_status gdp_logprob(gdp_graph g, const gdp_config *c, const float *logits, const uint8_t *placements, int32_t B,
                       float *logprob, void *ws, size_t ws_bytes, void *stream) {
  NvtxRange nvtx_("gdp_logprob");
  if (!g || !logits || !placements || !logprob) return fail(GDP_ERR_ARG, "NULL argument");
  gdp_status st = check_config(c);
  if (st != GDP_OK) return st;
  if (B < 1) return fail(GDP_ERR_ARG, "B must be >= 1");
  WS w;
  st = carve_any(g, c->num_devices, c->autoregressive ? B : 1, ws, ws_bytes, &w);
  if (st != GDP_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (c->autoregressive) {
    launch_ar_decode(kArDecodeScore, logits, g->perm, g->leader, g->has_coloc, g->N, c->num_devices, c->seg_len, B,
                     0, 0, 0, nullptr, const_cast<uint8_t *>(placements), w.spart, logprob, s);
    GDP_LAUNCH_CHECK("gdp_logprob");
    return GDP_OK;
  }
  launch_node_prep(logits, c->num_devices, g->N, active_devices(c), w.cdf, w.logp, w.lastpos, s);
  launch_logprob(w.logp, g->leader, placements, g->N, active_devices(c), B, logprob, s);
  GDP_LAUNCH_CHECK("gdp_logprob");
  return GDP_OK;
}

gdp_status gdp_greedy(gdp_graph g, const gdp_config *c, const float *logits, uint8_t *placement, float *logprob,
                      void *ws, size_t ws_bytes, void *stream) {
  NvtxRange nvtx_("gdp_greedy");
  if (!g || !logits || !placement) return fail(GDP_ERR_ARG, "NULL argument");
  gdp_status st = check_config(c);
  if (st != GDP_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (c->autoregressive) {   // the decode needs the log pi scratch whether or not it is returned
    WS w;
    st = carve_any(g, c->num_devices, 1, ws, ws_bytes, &w);
    if (st != GDP_OK) return st;
    launch_ar_decode(kArDecodeGreedy, logits, g->perm, g->leader, g->has_coloc, g->N, c->num_devices, c->seg_len, 1,
                     0, 0, 0, nullptr, placement, w.spart, logprob, s);
    GDP_LAUNCH_CHECK("gdp_greedy");
    return GDP_OK;
  }
  launch_greedy(logits, c->num_devices, g->leader, g->N, active_devices(c), placement, s);
  if (logprob) {
    WS w;
    st = carve_any(g, c->num_devices, 1, ws, ws_bytes, &w);
    if (st != GDP_OK) return st;
    launch_node_prep(logits, c->num_devices, g->N, active_devices(c), w.cdf, w.logp, w.lastpos, s);
    launch_logprob(w.logp, g->leader, placement, g->N, active_devices(c), 1, logprob, s);
  }
  GDP_LAUNCH_CHECK("gdp_greedy");
  return GDP_OK;
}

gdp_status gdp_clip_adam(const float *grad, int64_t n, double max_norm, double lr, double beta1, double beta2,
                         double eps, int64_t t, float *theta, float *m, float *v, double *scratch, double *norm_out,
                         void *stream) {
  NvtxRange nvtx_("gdp_clip_adam");
  if (!grad || !theta || !m || !v || !scratch) return fail(GDP_ERR_ARG, "NULL argument");
  if (n < 1 || t < 1) return fail(GDP_ERR_ARG, "n and t must be >= 1");
  if (!(beta1 >= 0.0 && beta1 < 1.0 && beta2 >= 0.0 && beta2 < 1.0) || !(max_norm > 0.0) || !(eps >= 0.0))
    return fail(GDP_ERR_ARG, "beta1, beta2 must lie in [0, 1), max_norm > 0, eps >= 0");
  auto misaligned = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) != 0; };
  if (misaligned(grad) || misaligned(theta) || misaligned(m) || misaligned(v) || misaligned(scratch))
    return fail(GDP_ERR_ARG, "grad, theta, m, v and scratch must be 16-byte aligned");
  static_assert(GDP_ADAM_SCRATCH == kAdamScratch, "scratch size");
  const double c1 = 1.0 / (1.0 - std::pow(beta1, (double)t));
  const double c2 = 1.0 / (1.0 - std::pow(beta2, (double)t));
  launch_clip_adam(grad, n, max_norm, lr, beta1, beta2, eps, c1, c2, theta, m, v, scratch, norm_out,
                   static_cast<cudaStream_t>(stream));
  GDP_LAUNCH_CHECK("gdp_clip_adam");
  return GDP_OK;
}

gdp_status gdp_grad_check(const float *grad, const gdp_config *c, int32_t F, double *scratch, void *stream) {
  if (!grad || !scratch) return fail(GDP_ERR_ARG, "NULL argument");
  gdp_status st = check_config(c);
  if (st != GDP_OK) return st;
  if (F < 1) return fail(GDP_ERR_ARG, "F must be >= 1");
  long long off[GDP_P_COUNT + 1];
  param_offsets(F, c->num_devices, off, c->autoregressive != 0);
  const long long n = off[GDP_P_COUNT];
  const long long i = first_nonfinite(grad, n, reinterpret_cast<unsigned long long *>(scratch),
                                      static_cast<cudaStream_t>(stream));
  if (i < 0) return cuda_status(cudaGetLastError(), "gdp_grad_check");
  if (i >= n) return GDP_OK;
  int t = 0;
  while (t + 1 < GDP_P_COUNT && off[t + 1] <= i) t++;
  return fail(GDP_ERR_NONFINITE, "non-finite gradient at theta[" + std::to_string(i) + "]: parameter tensor " +
                                     std::to_string(t) + " (gdp_param_id, " + kParamNames[t] + ") element " +
                                     std::to_string(i - off[t]));
}

gdp_status gdp_cost(gdp_graph g, gdp_topo t, const uint8_t *placements, int32_t B, gdp_sim_report *rep,
                    int64_t *peak_mem, int64_t *busy, double *reward, void *ws, size_t ws_bytes, void *stream) {
  return gdp_cost_with_kernel(g, t, placements, B, rep, peak_mem, busy, reward, ws, ws_bytes, 0, stream);
}

gdp_status gdp_cost_with_kernel(gdp_graph g, gdp_topo t, const uint8_t *placements, int32_t B, gdp_sim_report *rep,
                                int64_t *peak_mem, int64_t *busy, double *reward, void *ws, size_t ws_bytes,
                                int32_t kernel, void *stream) {
  NvtxRange nvtx_("gdp_cost_with_kernel");
  if (!g || !t || !placements || !rep || !reward) return fail(GDP_ERR_ARG, "NULL argument");
  if (B < 1) return fail(GDP_ERR_ARG, "B must be >= 1");
  // int32 device time: the schedule never exceeds sum(durations) + sum(transfers)
  long long maxspeed = 1, minbw = LLONG_MAX, maxlat = 0;
  for (int k = 0; k < t->d; k++) maxspeed = std::max<long long>(maxspeed, t->speed[k]);
  for (int s = 0; s < t->d; s++)
    for (int u = 0; u < t->d; u++)
      if (s != u) {
        minbw = std::min(minbw, t->bpt[s * 8 + u]);
        maxlat = std::max<long long>(maxlat, t->lat[s * 8 + u]);
      }
  double bound = (double)g->sum_cost * (double)maxspeed;
  if (t->d > 1) bound += (double)g->sum_edge_out_bytes / (double)minbw + (double)g->E * (double)(maxlat + 1);
  if (bound >= 2147483000.0)
    return fail(GDP_ERR_OVERFLOW, "sum of durations and transfers may exceed 2^31 ticks");
  WS w;
  gdp_status st = carve_any(g, t->d, B, ws, ws_bytes, &w);
  if (st != GDP_OK) return st;
  if (kernel != 0 && kernel != 1 && kernel != 3 && kernel != 5) return fail(GDP_ERR_ARG, "kernel must be 0, 1, 3 or 5");
  if (kernel != 0 && cost_kernel_choice(g, t, kernel) != kernel)
    return fail(GDP_ERR_ARG, "the requested cost kernel does not apply to this graph and topology");
  return launch_cost(g, t, placements, B, rep, reinterpret_cast<long long *>(peak_mem),
                     reinterpret_cast<long long *>(busy), reward, w, kernel, static_cast<cudaStream_t>(stream));
}

gdp_status gdp_advantage(const double *reward, int32_t B, double *run_sum, int64_t *run_count, double *adv,
                         void *stream) {
  if (!reward || !run_sum || !run_count || !adv) return fail(GDP_ERR_ARG, "NULL argument");
  if (B < 1) return fail(GDP_ERR_ARG, "B must be >= 1");
  launch_advantage(reward, B, run_sum, reinterpret_cast<long long *>(run_count), adv,
                   static_cast<cudaStream_t>(stream));
  GDP_LAUNCH_CHECK("gdp_advantage");
  return GDP_OK;
}

gdp_status gdp_policy_grad(gdp_graph g, const gdp_config *c, const float *theta, const float *logits,
                           const uint8_t *placements, int32_t B, const double *adv, const float *logprob,
                           const float *old_logprob, float clip_eps, float entropy_coef, float loss_scale,
                           float *grad, void *ws, size_t ws_bytes, void *stream) {
  NvtxRange nvtx_("gdp_policy_grad");
  if (!g || !theta || !logits || !placements || !adv || !grad) return fail(GDP_ERR_ARG, "NULL argument");
  if (old_logprob && !logprob) return fail(GDP_ERR_ARG, "logprob is required with old_logprob");
  gdp_status st = check_config(c);
  if (st != GDP_OK) return st;
  if (B < 1) return fail(GDP_ERR_ARG, "B must be >= 1");
  WS w;
  st = carve_any(g, c->num_devices, B, ws, ws_bytes, &w);
  if (st != GDP_OK) return st;
  set_tensor_cores(c->tensor_cores);
  set_no_attention(c->no_attention != 0);
  return run_policy_grad(g, c, theta, logits, placements, B, adv, logprob, old_logprob, clip_eps, entropy_coef,
                         loss_scale, grad, w, static_cast<cudaStream_t>(stream), nullptr);
}

gdp_status gdp_policy_grad_bucketed(gdp_graph g, const gdp_config *c, const float *theta, const float *logits,
                                    const uint8_t *placements, int32_t B, const double *adv, const float *logprob,
                                    const float *old_logprob, float clip_eps, float entropy_coef, float loss_scale,
                                    float *grad, void *ws, size_t ws_bytes, void *const *bucket_events,
                                    void *stream) {
  NvtxRange nvtx_("gdp_policy_grad_bucketed");
  if (!g || !theta || !logits || !placements || !adv || !grad || !bucket_events)
    return fail(GDP_ERR_ARG, "NULL argument");
  if (old_logprob && !logprob) return fail(GDP_ERR_ARG, "logprob is required with old_logprob");
  gdp_status st = check_config(c);
  if (st != GDP_OK) return st;
  if (B < 1) return fail(GDP_ERR_ARG, "B must be >= 1");
  WS w;
  st = carve_any(g, c->num_devices, B, ws, ws_bytes, &w);
  if (st != GDP_OK) return st;
  set_tensor_cores(c->tensor_cores);
  set_no_attention(c->no_attention != 0);
  cudaEvent_t ev[GDP_GRAD_BUCKETS];
  for (int i = 0; i < GDP_GRAD_BUCKETS; i++) ev[i] = static_cast<cudaEvent_t>(bucket_events[i]);
  return run_policy_grad(g, c, theta, logits, placements, B, adv, logprob, old_logprob, clip_eps, entropy_coef,
                         loss_scale, grad, w, static_cast<cudaStream_t>(stream), ev);
}

gdp_status gdp_grad_buckets(const gdp_config *c, int32_t F, int64_t *first, int64_t *last) {
  if (!first || !last) return fail(GDP_ERR_ARG, "NULL argument");
  gdp_status st = check_config(c);
  if (st != GDP_OK) return st;
  if (F < 1) return fail(GDP_ERR_ARG, "F must be >= 1");
  long long off[GDP_P_COUNT + 1];
  param_offsets(F, c->num_devices, off, c->autoregressive != 0);
  first[0] = off[GDP_P_XL0_LN1_G]; last[0] = off[GDP_P_COUNT];
  first[1] = off[GDP_P_COND_LN1_G]; last[1] = off[GDP_P_XL0_LN1_G];
  first[2] = 0; last[2] = off[GDP_P_COND_LN1_G];
  return GDP_OK;
}

gdp_status gdp_grad_sum(const float *const *grads, int32_t n_grads, int64_t len, float *out, void *stream) {
  NvtxRange nvtx_("gdp_grad_sum");
  if (!grads || !out || n_grads < 1 || len < 1) return fail(GDP_ERR_ARG, "bad argument");
  for (int i = 0; i < n_grads; i++)
    if (!grads[i]) return fail(GDP_ERR_ARG, "NULL gradient");
  launch_grad_sum(grads, n_grads, len, out, static_cast<cudaStream_t>(stream));
  GDP_LAUNCH_CHECK("gdp_grad_sum");
  return GDP_OK;
}

}  // extern "C"
