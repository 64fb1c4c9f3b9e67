// tcgen05 weight gradients of the dense maps (a15, tensor-core mode): dW_aug = [X, 1]^T dY over
// all N node rows, deterministic split-K over row chunks.
//
// The contraction runs over the nodes, so both operands are "MN-major" for the tensor core:
// A = X^T (M = the map's fan-in K, contraction = rows) and B = dY (N = the map's width), each
// read by TMA as 64-row x 32-column fp32 boxes whose 128-byte rows (one node, 32 consecutive
// columns) are exactly the rows of the MN-major SWIZZLE_128B_BASE32B layout (the only MN-major
// layout the tf32 MMA takes: TMA's SWIZZLE_128B_ATOM_32B, 32-byte granules XOR row % 4; LBO = the
// next 32-column box, SBO = the next 4 nodes).  tf32 operands (the fp32 patterns
// truncated, as the dense maps' forward), fp32 accumulation in TMEM: M = 128 per half of the
// fan-in (K <= 256: at most two halves, the unused 32-column blocks of a half stay zero),
// N = width padded to 16.
//
// One CTA per row chunk (<= one per SM): warp 0 streams the chunk's 64-row stages by TMA
// (up to 4 in flight),
// warp 1 issues 8 x (halves) MMAs per stage (K = 8 nodes each), warps 2-5 sum the bias row
// (column sums of dY) from the same shared-memory stages and, at the end, drain TMEM into the
// chunk's partial [K + 1 x width] (the k_wgrad layout); k_reduce_chunks adds the partials in
// chunk order.
#include <string.h>

#include <algorithm>

#include "common.cuh"
#include "tc_util.cuh"

namespace gdp {
namespace {
using namespace tc;

constexpr int WR = 64;            // node rows per stage
constexpr int WBOX = WR * 128;    // one 64-row x 32-column fp32 box (8 KB)
constexpr int NTW = 192;          // warp 0 TMA, warp 1 MMA, warps 2..5 bias sums + epilogue
constexpr int MAXSTW = 4;

struct WgParams {
  int M, K, K1, Nout;
  int kb1, kb;     // X boxes taken from X1 (with a second operand), all X boxes (ceil(K / 32))
  int nb;          // dY boxes (ceil(Nout / 32))
  int nm;          // fan-in halves of 128 (1 or 2)
  int Np;          // width padded to 16 (UMMA N)
  int rpc;         // rows per chunk (a multiple of WR)
  int stages, ncols, with_bias;
};
struct WgMaps { CUtensorMap x1, x2, dy; };

// MN-major SWIZZLE_128B_BASE32B descriptor (layout type 1; the only MN-major layout of the tf32
// MMA): 128-byte rows along M / N (32 tf32), 32-byte granule g of row r at g ^ (r % 4), 4-row K
// groups SBO = 512 bytes apart, 32-element M / N blocks LBO apart
__device__ __forceinline__ uint64_t desc_mn_b32(uint32_t saddr, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;
  return d;
}

__global__ void __launch_bounds__(NTW, 1) k_wgrad_tc(const __grid_constant__ WgMaps mp, WgParams p, float *part) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  __shared__ __align__(8) uint64_t full[MAXSTW], empty[MAXSTW], dfull;
  __shared__ uint32_t tmem_base;
  unsigned char *sm = smraw + ((1024u - (su32(smraw) & 1023u)) & 1023u);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int xslots = 4 * p.nm, sbytes = (xslots + p.nb) * WBOX;
  const int c = blockIdx.x, r0 = c * p.rpc, r1 = min(p.M, r0 + p.rpc);
  const int nst = (r1 - r0 + WR - 1) / WR;   // stages of this chunk (>= 1)
  if (tid == 0) {
    for (int s = 0; s < p.stages; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1 + 4); }
    mbar_init(&dfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // the fan-in blocks no TMA box fills stay zero (the unused rows of an M = 128 half)
  for (int s = 0; s < p.stages; s++)
    for (int b = p.kb; b < xslots; b++)
      for (int i = tid; i < WBOX / 16; i += NTW)
        reinterpret_cast<int4 *>(sm + (size_t)s * sbytes + (size_t)b * WBOX)[i] = make_int4(0, 0, 0, 0);
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)),
                 "r"(p.ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      for (int it = 0; it < nst; it++) {
        const int s = it % p.stages;
        mbar_wait(&empty[s], ((uint32_t)(it / p.stages) & 1u) ^ 1u);
        unsigned char *st = sm + (size_t)s * sbytes;
        const int row = r0 + it * WR;
        mbar_expect_tx(&full[s], (uint32_t)(p.kb + p.nb) * WBOX);
        for (int b = 0; b < p.kb; b++) {
          if (b < p.kb1) tma_load_2d(st + (size_t)b * WBOX, &mp.x1, b * 32, row, &full[s]);
          else tma_load_2d(st + (size_t)b * WBOX, &mp.x2, (b - p.kb1) * 32, row, &full[s]);
        }
        for (int b = 0; b < p.nb; b++) tma_load_2d(st + (size_t)(xslots + b) * WBOX, &mp.dy, b * 32, row, &full[s]);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // kind::tf32, D fp32, A and B tf32 and MN-major (bits 15, 16), N >> 3 at 17, M >> 4 at 24
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) |
                           ((uint32_t)(p.Np >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    if (lane == 0) {
      for (int it = 0; it < nst; it++) {
        const int s = it % p.stages;
        mbar_wait(&full[s], (uint32_t)(it / p.stages) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t st = su32(sm + (size_t)s * sbytes);
        for (int k8 = 0; k8 < WR / 8; k8++) {
          const uint64_t bd = desc_mn_b32(st + (uint32_t)(xslots * WBOX + k8 * 1024), WBOX);
          for (int h = 0; h < p.nm; h++) {
            const uint64_t ad = desc_mn_b32(st + (uint32_t)(h * 4 * WBOX + k8 * 1024), WBOX);
            const uint32_t accum = (it | k8) ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, q;\n\t}\n" ::"r"(tmem + (uint32_t)(h * p.Np)),
                "l"(ad), "l"(bd), "r"(idesc), "r"(accum));
          }
        }
        mma_commit(&empty[s]);
      }
      mma_commit(&dfull);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ bias sums, then the epilogue
    const int t = tid - 64;   // 0..127: columns t and t + 128
    float bs0 = 0.f, bs1 = 0.f;
    for (int it = 0; it < nst; it++) {
      const int s = it % p.stages;
      mbar_wait(&full[s], (uint32_t)(it / p.stages) & 1u);
      if (p.with_bias) {
        const unsigned char *dy = sm + (size_t)s * sbytes + (size_t)xslots * WBOX;
#pragma unroll
        for (int u = 0; u < 2; u++) {
          const int n = t + 128 * u;
          if (n < p.Nout) {
            const unsigned char *bx = dy + (size_t)(n >> 5) * WBOX + (n & 7) * 4;
            const int g = (n & 31) >> 3;   // 32-byte granule
            float sacc = 0.f;
#pragma unroll 8
            for (int i = 0; i < WR; i++) sacc += *reinterpret_cast<const float *>(bx + i * 128 + ((g ^ (i & 3)) << 5));
            if (u == 0) bs0 += sacc; else bs1 += sacc;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    float *P = part + (size_t)c * (p.K + p.with_bias) * p.Nout;
    if (p.with_bias) {
      if (t < p.Nout) P[(size_t)p.K * p.Nout + t] = bs0;
      if (t + 128 < p.Nout) P[(size_t)p.K * p.Nout + t + 128] = bs1;
    }
    mbar_wait(&dfull, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int q = warp & 3;
    for (int h = 0; h < p.nm; h++) {
      const int k = h * 128 + q * 32 + lane;   // TMEM lane = fan-in row of dW
      const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(h * p.Np);
      for (int n0 = 0; n0 < p.Np; n0 += 32) {
        const int nbk = min(4, (p.Np - n0) >> 3);   // warp-uniform
        uint32_t v[32];
#pragma unroll
        for (int u = 0; u < 4; u++)
          if (u < nbk) tmem_ld8(tb + (uint32_t)(n0 + 8 * u), v + 8 * u);
        tmem_wait_ld();
        if (k < p.K) {
          float *dst = P + (size_t)k * p.Nout;
#pragma unroll
          for (int u = 0; u < 32; u++)
            if (u < 8 * nbk && n0 + u < p.Nout) dst[n0 + u] = __uint_as_float(v[u]);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.ncols));
  }
}

bool make_map(CUtensorMap *m, const float *base, int cols, int rows, int ld) {
  return tma_map_f32(m, base, cols, rows, ld, WR, true);
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

bool wgrad_tc_eligible(int M, int K, int Nout) { return Nout >= 16 && Nout <= 256 && K >= 1 && K <= 256 && M >= 128; }

// returns the number of row chunks written to part (0: not launched -- the caller runs k_wgrad)
int launch_wgrad_tc(int M, int K, int Nout, const float *X1, int ldx1, int K1, const float *X2, int ldx2,
                    const float *dY, int ldy, bool with_bias, float *part, size_t part_floats, cudaStream_t s) {
  WgParams p;
  WgMaps mp;
  memset(&p, 0, sizeof(p));
  memset(&mp, 0, sizeof(mp));
  p.M = M; p.K = K; p.Nout = Nout; p.with_bias = with_bias ? 1 : 0;
  const bool two = X2 != nullptr && K1 < K;
  p.K1 = two ? K1 : K;
  p.kb = (K + 31) / 32;
  p.kb1 = two ? K1 / 32 : p.kb;
  p.nb = (Nout + 31) / 32;
  p.nm = (K + 127) / 128;
  p.Np = (Nout + 15) / 16 * 16;
  p.ncols = 32;
  while (p.ncols < p.nm * p.Np) p.ncols <<= 1;
  if ((two && K1 % 32) || !make_map(&mp.x1, X1, p.K1, M, ldx1) || (two && !make_map(&mp.x2, X2, K - K1, M, ldx2)) ||
      !make_map(&mp.dy, dY, Nout, M, ldy))
    return 0;
  const size_t sbytes = (size_t)(4 * p.nm + p.nb) * WBOX;
  const size_t dyn_max = 224 * 1024;
  p.stages = (int)((dyn_max - 1024) / sbytes);
  if (p.stages > MAXSTW) p.stages = MAXSTW;
  if (p.stages < 2) return 0;
  // chunks: about one per SM, whole stages, within the partial buffer
  const int Kaug = K + p.with_bias;
  long long chunks = sm_count();
  chunks = std::min<long long>(chunks, (long long)(part_floats / ((size_t)Kaug * Nout)));
  chunks = std::max<long long>(1, std::min<long long>(chunks, (M + WR - 1) / WR));
  p.rpc = (int)(((M + chunks - 1) / chunks + WR - 1) / WR * WR);
  const int nchunks = (M + p.rpc - 1) / p.rpc;
  const size_t smem = (size_t)p.stages * sbytes + 1024;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_wgrad_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_max);
    configured = true;
  }
  note_launch("k_wgrad_tc", s, 4.0 * M * (K + Nout) + 4.0 * nchunks * Kaug * Nout, 2.0 * M * Kaug * Nout);
  k_wgrad_tc<<<nchunks, NTW, smem, s>>>(mp, p, part);
  return nchunks;
}

}  // namespace gdp
