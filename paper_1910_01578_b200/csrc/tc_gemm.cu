// tcgen05 tensor-core path for the tall-skinny dense maps of the policy network (tf32 operands,
// fp32 accumulation in TMEM): Y = epi(X W + b) (+R), the same contract as k_gemm.
//
// The maps are HBM-bound (K, Nout <= 256: at most 32 flop per byte of fp32 X and Y against a
// ridge of ~250), so the kernel is built to stream X through the SM once at full bandwidth:
//
//  * X stays fp32 in HBM and is consumed as tf32 by `tcgen05.mma.kind::tf32` straight from the
//    shared-memory tile TMA wrote (`cp.async.bulk.tensor.2d`, 128 rows x 32 fp32 = one
//    SWIZZLE_128B row of 128 bytes per node): no thread touches X on its way to the tensor core.
//  * Persistent CTAs (one per SM, 10 warps), warp-specialised:
//      warp 0      TMA producer: a ring of up to 8 16-KB stages (one K chunk of one 128-row tile
//                  each), full / empty mbarriers;
//      warp 1      MMA issuer (one elected lane): per chunk 4 MMAs (K = 8 each, M = 128,
//                  N = Nout padded to 16) into one of TWO TMEM accumulators, `tcgen05.commit`
//                  frees the stage, a second commit hands the finished accumulator over;
//      warps 2-9   epilogue, per 32-row x 32-column block (warp w owns TMEM lanes 32 (w % 4)..,
//                  warps 2-5 / 6-9 alternate the column blocks): `tcgen05.ld.32x32b.x8` x 4 under
//                  one wait, the fused epilogue (bias, sigmoid / tanh / ReLU / ReLU-mask, residual,
//                  split output, accumulate) in registers, the block written to a swizzled 4-KB
//                  shared-memory buffer and stored by TMA (`cp.async.bulk.tensor` store, rows
//                  beyond M / columns beyond Nout clipped); the one input tile an epilogue reads
//                  (residual R, ReLU mask, or Y itself when accumulating) arrives by TMA into the
//                  same buffer one block ahead.  Two buffers per warp; the MMAs of the next tile
//                  fill the other TMEM accumulator meanwhile.
//  * W (<= 64 KB as fp32) is staged once per CTA in the same K-major SWIZZLE_128B layout while
//    the producer already streams X.
//  * Rows whose stride TMA cannot take (not a multiple of 16 bytes, e.g. the d = 2 head's
//    backward) are loaded by the producer warp itself into the same layout, and outputs TMA
//    cannot take are written by the epilogue threads directly -- same kernel, same arithmetic.
// tf32 operand semantics (include/gdp.h, gdp_config.tensor_cores): the tensor core reads the
// fp32 bit patterns of X and W and uses their upper 19 bits (sign, exponent, 10 mantissa bits),
// i.e. truncation toward zero; products and fp32 accumulation in TMEM.
#include <cuda.h>
#include <string.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tc_util.cuh"

namespace gdp {
namespace {
using namespace tc;

constexpr int TM = 128;             // rows per tile (UMMA M)
constexpr int KC = 32;              // fp32 columns per K chunk (128 bytes: one swizzle row)
constexpr int CB = TM * KC * 4;     // bytes per X stage (16 KB)
constexpr int NT = 320;             // warp 0 TMA, warp 1 MMA, warps 2..9 epilogue
constexpr int NEW = 8;              // epilogue warps
constexpr int MAXST = 8;
constexpr int kWMax = 64 * 1024;    // W tile bytes (fp32) the kernel stages
constexpr int EB = 32 * 128;        // epilogue block: 32 rows x 32 fp32 columns, SWIZZLE_128B (4 KB)
constexpr int kDynMax = 224 * 1024; // dynamic shared memory (227 KB per CTA less the static part)

struct TfParams {
  int nch;      // K chunks per tile (Kp / 32)
  int nch1;     // chunks from X1 (K1 / 32 with a second operand, else nch)
  int Np;       // Nout padded to 16 (UMMA N)
  int ncols;    // TMEM columns allocated (2 accumulators of Np)
  int stages;   // X ring depth
  int tma;      // 1: TMA loads of X; 0: the producer warp loads
  int wvec;     // W rows along its contiguous dimension are 16-byte aligned
  int Ns;       // TMEM columns per accumulator (Np rounded up to 32)
  int tstore;   // 1: TMA-store epilogue (maps y1 / y2), 0: direct stores
  int tin;      // TMA-store epilogue input tile: 0 none, 1 R, 2 aux (mask), 3 Y (accumulate)
  int nbusy;    // epilogue warps with work in every tile (the accumulator's release count)
};
struct Maps {   // TMA descriptors (kernel parameters, __grid_constant__)
  CUtensorMap x1, x2;   // X column ranges [0, K1) and [K1, K): box 128 x 32
  CUtensorMap y1, y2;   // Y columns [0, split) and Y2 [split, Nout): box 32 x 32
  CUtensorMap t;        // the epilogue's input tile (R, aux or Y): box 32 x 32
};

// activations of the tensor-core mode's epilogues (fast-math: relative error ~1e-6, far inside
// the mode's 2e-2 parity tolerance)
template <int EPI>
__device__ __forceinline__ float act(float v) {
  if (EPI == EPI_SIGMOID) return __fdividef(1.0f, 1.0f + __expf(-v));   // 1 / inf = 0 for v << 0
  if (EPI == EPI_TANH) {
    const float t = __expf(-2.0f * fabsf(v));
    return copysignf(__fdividef(1.0f - t, 1.0f + t), v);
  }
  if (EPI == EPI_RELU) return v > 0.f ? v : 0.f;
  return v;
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap *map, int x, int y, const void *src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(su32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }


// one 8-column group of row m: bias, activation / mask, residual, store (or accumulate)
template <int EPI>
__device__ __forceinline__ void epilogue8(const GemmArgs &a, int m, int c0, const uint32_t *v, bool vec_epi,
                                          bool vec_out) {
  float x[8];
  if (vec_epi && c0 + 8 <= a.Nout) {   // full group: 16-byte loads of mask and residual
    float mk[8], rr[8];
    if (EPI == EPI_MASK) {
      const float4 *p = reinterpret_cast<const float4 *>(a.aux + (size_t)m * a.ldaux + c0);
      const float4 u0 = p[0], u1 = p[1];
      mk[0] = u0.x; mk[1] = u0.y; mk[2] = u0.z; mk[3] = u0.w; mk[4] = u1.x; mk[5] = u1.y; mk[6] = u1.z; mk[7] = u1.w;
    }
    if (a.R) {
      const float4 *p = reinterpret_cast<const float4 *>(a.R + (size_t)m * a.ldr + c0);
      const float4 u0 = p[0], u1 = p[1];
      rr[0] = u0.x; rr[1] = u0.y; rr[2] = u0.z; rr[3] = u0.w; rr[4] = u1.x; rr[5] = u1.y; rr[6] = u1.z; rr[7] = u1.w;
    }
#pragma unroll
    for (int j = 0; j < 8; j++) {
      float y = __uint_as_float(v[j]);
      if (a.bias) y += a.bias[c0 + j];
      if (EPI == EPI_MASK) y = mk[j] > 0.f ? y : 0.f;
      else y = act<EPI>(y);
      if (a.R) y += rr[j];
      x[j] = y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const int n = c0 + j;
      float y = __uint_as_float(v[j]);
      if (n < a.Nout) {
        if (a.bias) y += a.bias[n];
        if (EPI == EPI_MASK) y = a.aux[(size_t)m * a.ldaux + n] > 0.f ? y : 0.f;
        else y = act<EPI>(y);
        if (a.R) y += a.R[(size_t)m * a.ldr + n];
      }
      x[j] = y;
    }
  }
  if (vec_out && c0 + 8 <= a.Nout && (c0 + 8 <= a.split || c0 >= a.split)) {
    float *dst = (c0 < a.split) ? a.Y + (size_t)m * a.ldy + c0 : a.Y2 + (size_t)m * a.ldy2 + (c0 - a.split);
    float4 *d4 = reinterpret_cast<float4 *>(dst);
    float4 p0 = make_float4(x[0], x[1], x[2], x[3]), p1 = make_float4(x[4], x[5], x[6], x[7]);
    if (a.accumulate) {
      const float4 q0 = d4[0], q1 = d4[1];
      p0.x += q0.x; p0.y += q0.y; p0.z += q0.z; p0.w += q0.w;
      p1.x += q1.x; p1.y += q1.y; p1.z += q1.z; p1.w += q1.w;
    }
    d4[0] = p0;
    d4[1] = p1;
  } else {
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const int n = c0 + j;
      if (n >= a.Nout) break;
      float *dst = (n < a.split) ? a.Y + (size_t)m * a.ldy + n : a.Y2 + (size_t)m * a.ldy2 + (n - a.split);
      *dst = a.accumulate ? *dst + x[j] : x[j];
    }
  }
}

#ifdef GEMM_PROF
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ unsigned long long g_gprof[8];
#endif
template <int EPI>
__global__ void __launch_bounds__(NT, 1) k_gemm_tc(const __grid_constant__ Maps mp, GemmArgs a, TfParams p) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  __shared__ __align__(8) uint64_t full[MAXST], empty[MAXST], tfull[2], tempty[2], tinb[NEW][2];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(16) float sBias[256];
  const CUtensorMap *mx1 = &mp.x1, *mx2 = &mp.x2;
  // SWIZZLE_128B tiles need 1024-byte alignment of the shared-window address
  unsigned char *sm = smraw + ((1024u - (su32(smraw) & 1023u)) & 1023u);
  unsigned char *sW = sm + (size_t)p.stages * CB;   // [chunk][n][128 B]
  unsigned char *sE = sW + (size_t)p.nch * p.Np * 128;   // NEW x 2 epilogue blocks (EB each)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Np = p.Np;
#ifdef GEMM_PROF
  const unsigned long long t_start = gtime();
  __shared__ unsigned long long pt[16];
  if (tid < 16) pt[tid] = 0;
#endif

  if (tid == 0) {
    for (int s = 0; s < p.stages; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int c = 0; c < 2; c++) { mbar_init(&tfull[c], 1); mbar_init(&tempty[c], p.nbusy); }
    for (int w = 0; w < NEW; w++) { mbar_init(&tinb[w][0], 1); mbar_init(&tinb[w][1], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (p.tma) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(mx1)) : "memory");
      if (p.nch1 < p.nch) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(mx2)) : "memory");
    }
  }
  __syncthreads();
  const int ntiles = (a.M + TM - 1) / TM;
  uint32_t tmem = 0;
  if (warp != 0) {
    // the producer warp starts streaming X at once; the other 9 warps allocate TMEM and stage W
    // -> [chunk k / 32][n][granule ((k % 32) / 4) ^ (n % 8)][k % 4] (raw fp32 bits) meanwhile,
    // walking W's contiguous dimension with 16-byte loads where aligned (W is L2-resident)
    if (warp == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)),
                   "r"(p.ncols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
    }
    const int t = tid - 32, nt = NT - 32;
    const int Kp = p.nch * KC;
    for (int n = t; n < 256; n += nt) sBias[n] = (a.bias && n < a.Nout) ? a.bias[n] : 0.f;
    auto wst = [&](int k, int n, float w) {
      const int kk = k & (KC - 1);
      *reinterpret_cast<float *>(sW + (size_t)(k / KC) * Np * 128 + n * 128 + (((kk >> 2) ^ (n & 7)) << 4) +
                                 (kk & 3) * 4) = w;
    };
    // all of a thread's loads (<= 16 of 16 bytes: W <= 64 KB over 288 threads) are issued
    // before any store, so the staging costs one L2 round trip
    constexpr int WPT = (kWMax / 16 + NT - 33) / (NT - 32);
    float4 wr[WPT];
    if (a.ldw_n == 1) {   // W(k, n) = W[k ldw_k + n]: 4 consecutive n per item
      const int nq = Np / 4;
#pragma unroll
      for (int i = 0; i < WPT; i++) {
        const int e = t + i * nt, k = e / nq, n = (e - k * nq) * 4;
        float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
        if (e < Kp * nq && k < a.K) {
          const float *src = a.W + (size_t)k * a.ldw_k + n;
          if (p.wvec && n + 3 < a.Nout) w = __ldg(reinterpret_cast<const float4 *>(src));
          else {
            if (n < a.Nout) w.x = src[0];
            if (n + 1 < a.Nout) w.y = src[1];
            if (n + 2 < a.Nout) w.z = src[2];
            if (n + 3 < a.Nout) w.w = src[3];
          }
        }
        wr[i] = w;
      }
#pragma unroll
      for (int i = 0; i < WPT; i++) {
        const int e = t + i * nt, k = e / nq, n = (e - k * nq) * 4;
        if (e < Kp * nq) { wst(k, n, wr[i].x); wst(k, n + 1, wr[i].y); wst(k, n + 2, wr[i].z); wst(k, n + 3, wr[i].w); }
      }
    } else {              // W(k, n) = W[k ldw_k + n ldw_n]: 4 consecutive k per item (one granule)
      const int kq = Kp / 4;
#pragma unroll
      for (int i = 0; i < WPT; i++) {
        const int e = t + i * nt, n = e / kq, k = (e - n * kq) * 4;
        float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
        if (e < Np * kq && n < a.Nout) {
          const float *src = a.W + (size_t)k * a.ldw_k + (size_t)n * a.ldw_n;
          if (p.wvec && k + 3 < a.K) w = __ldg(reinterpret_cast<const float4 *>(src));
          else {
            if (k < a.K) w.x = src[0];
            if (k + 1 < a.K) w.y = src[a.ldw_k];
            if (k + 2 < a.K) w.z = src[2 * a.ldw_k];
            if (k + 3 < a.K) w.w = src[3 * a.ldw_k];
          }
        }
        wr[i] = w;
      }
#pragma unroll
      for (int i = 0; i < WPT; i++) {
        const int e = t + i * nt, n = e / kq, k = (e - n * kq) * 4;
        const int kk = k & (KC - 1);
        if (e < Np * kq)
          *reinterpret_cast<float4 *>(sW + (size_t)(k / KC) * Np * 128 + n * 128 + (((kk >> 2) ^ (n & 7)) << 4)) = wr[i];
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> async proxy
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    asm volatile("bar.sync 1, %0;" ::"n"(NT - 32) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    tmem = tmem_base;
#ifdef GEMM_PROF
    if (tid == 32) pt[0] = gtime() - t_start;
#endif
  }

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int m0 = tile * TM;
      for (int kc = 0; kc < p.nch; kc++, it++) {
        const int s = it % p.stages;
        const uint32_t ph = (uint32_t)(it / p.stages) & 1u;
        if (lane == 0) mbar_wait(&empty[s], ph ^ 1u);
        __syncwarp();
        unsigned char *dst = sm + (size_t)s * CB;
        if (p.tma) {
          if (lane == 0) {
            mbar_expect_tx(&full[s], CB);
            if (kc < p.nch1) tma_load_2d(dst, mx1, kc * KC, m0, &full[s]);
            else tma_load_2d(dst, mx2, (kc - p.nch1) * KC, m0, &full[s]);
          }
        } else {
          // rows TMA cannot take: lanes fill (row, 16-byte granule) items of the same layout
#pragma unroll 4
          for (int i = lane; i < TM * 8; i += 32) {
            const int r = i >> 3, g = i & 7, m = m0 + r;
            float v[4];
#pragma unroll
            for (int j = 0; j < 4; j++) {
              const int k = kc * KC + g * 4 + j;
              v[j] = 0.f;
              if (m < a.M && k < a.K)
                v[j] = (k < a.K1) ? a.X1[(size_t)m * a.ldx1 + k] : a.X2[(size_t)m * a.ldx2 + (k - a.K1)];
            }
            *reinterpret_cast<float4 *>(dst + r * 128 + ((g ^ (r & 7)) << 4)) = make_float4(v[0], v[1], v[2], v[3]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // kind::tf32, D fp32 (bit 4), A / B tf32 (format 2, bits 7 / 10), both K-major, N >> 3 at bit
    // 17, M >> 4 at bit 24
    const uint32_t idesc =
        (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(Np >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
    int it = 0, j = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, j++) {
      const int acc = j & 1;
      const uint32_t use = (uint32_t)(j >> 1);
      if (lane == 0) {
        mbar_wait(&tempty[acc], (use & 1u) ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + (uint32_t)(acc * p.Ns);
        for (int kc = 0; kc < p.nch; kc++, it++) {
          const int s = it % p.stages;
          mbar_wait(&full[s], (uint32_t)(it / p.stages) & 1u);
#ifdef GEMM_PROF
          if (it < 2) pt[1 + it] = gtime() - t_start;
#endif
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t xa = su32(sm + (size_t)s * CB), wb = su32(sW + (size_t)kc * Np * 128);
#pragma unroll
          for (int k = 0; k < KC / 8; k++) {
            const uint64_t ad = desc_sw128(xa + 32 * k), bd = desc_sw128(wb + 32 * k);
            const uint32_t accum = (kc | k) ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                "l"(ad), "l"(bd), "r"(idesc), "r"(accum));
          }
          mma_commit(&empty[s]);   // the stage is free once these MMAs have read it
        }
        mma_commit(&tfull[acc]);   // the accumulator is complete
#ifdef GEMM_PROF
        if (j < 4) pt[12 + j] = gtime() - t_start;
#endif
      }
      __syncwarp();
    }
  } else if (p.tstore) {
    // ------------------------------------------------------------ epilogue (warps 2..9), TMA stores
    const int ew = warp - 2, q = warp & 3, h = ew >> 2;
    const int nblk = (Np + 31) / 32;
    unsigned char *ebuf = sE + (size_t)ew * 2 * EB;
    const CUtensorMap *mt = &mp.t;
    // the blocks this warp handles, in order: (tile, column block cb = h, h + 2, ...)
    auto first_cb = [&]() { return h; };
    int tile = blockIdx.x, cb = first_cb();
    while (tile < ntiles && cb >= nblk) { tile += gridDim.x; cb = first_cb(); }   // (nblk == 1, h == 1)
    auto advance = [&](int &tl, int &c) {
      c += 2;
      if (c >= nblk) { tl += gridDim.x; c = first_cb(); if (c >= nblk) tl = ntiles; }
    };
    if (p.tin && tile < ntiles && lane == 0) {   // the first block's input tile
      mbar_expect_tx(&tinb[ew][0], EB);
      tma_load_2d(ebuf, mt, cb * 32, tile * TM + 32 * q, &tinb[ew][0]);
    }
    // a warp with a block in one tile has blocks in every tile (the same column blocks), so the
    // distinct tiles it meets are this CTA's consecutive tiles j = 0, 1, ...
    int j = -1, last_tile = -1;
    uint32_t bc = 0;   // blocks processed (buffer bc & 1)
    while (tile < ntiles) {
      if (tile != last_tile) {   // a new tile: wait for its accumulator
        if (last_tile >= 0) {    // release the previous one
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[j & 1]);
#ifdef GEMM_PROF
          if (tid == 64 && j < 4) pt[3 + j] = gtime() - t_start;
#endif
        }
        j++;
        last_tile = tile;
        mbar_wait(&tfull[j & 1], (uint32_t)(j >> 1) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#ifdef GEMM_PROF
        if (tid == 64 && j < 4) pt[8 + j] = gtime() - t_start;
#endif
      }
      const int buf = (int)(bc & 1u);
      unsigned char *eb = ebuf + buf * EB;
      int ntile = tile, ncb = cb;
      advance(ntile, ncb);
      if (lane == 0) {
        if (p.tin) {
          if (ntile < ntiles) {   // prefetch the next block's input tile into the other buffer
            bulk_wait_read<0>();   // its previous store has read it
            mbar_expect_tx(&tinb[ew][buf ^ 1], EB);
            tma_load_2d(ebuf + (buf ^ 1) * EB, mt, ncb * 32, ntile * TM + 32 * q, &tinb[ew][buf ^ 1]);
          }
        } else {
          bulk_wait_read<1>();     // the store that used this buffer two blocks ago has read it
        }
      }
      __syncwarp();
      uint32_t v[32];
      const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)((j & 1) * p.Ns + cb * 32);
#pragma unroll
      for (int u = 0; u < 4; u++) tmem_ld8(tb + 8u * u, v + 8 * u);
      tmem_wait_ld();
      if (p.tin) mbar_wait(&tinb[ew][buf], (bc >> 1) & 1u);
      // row = lane: granule g (columns 4g..4g+3) at (g ^ (lane & 7)) * 16 in the row's 128 bytes
      unsigned char *row = eb + lane * 128;
      const float *bb = sBias + cb * 32;
#pragma unroll
      for (int g = 0; g < 8; g++) {
        float4 *pp = reinterpret_cast<float4 *>(row + ((g ^ (lane & 7)) << 4));
        const float4 b4 = *reinterpret_cast<const float4 *>(bb + 4 * g);
        float y0 = __uint_as_float(v[4 * g]) + b4.x, y1 = __uint_as_float(v[4 * g + 1]) + b4.y;
        float y2 = __uint_as_float(v[4 * g + 2]) + b4.z, y3 = __uint_as_float(v[4 * g + 3]) + b4.w;
        float4 in = make_float4(0.f, 0.f, 0.f, 0.f);
        if (p.tin) in = *pp;
        if (EPI == EPI_MASK) {
          y0 = in.x > 0.f ? y0 : 0.f; y1 = in.y > 0.f ? y1 : 0.f; y2 = in.z > 0.f ? y2 : 0.f; y3 = in.w > 0.f ? y3 : 0.f;
        } else {
          y0 = act<EPI>(y0); y1 = act<EPI>(y1); y2 = act<EPI>(y2); y3 = act<EPI>(y3);
          if (p.tin) { y0 += in.x; y1 += in.y; y2 += in.z; y3 += in.w; }   // residual, or Y += result
        }
        *pp = make_float4(y0, y1, y2, y3);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> TMA store
      __syncwarp();
      if (lane == 0) {
        const int col = cb * 32, r0 = tile * TM + 32 * q;
        if (col < a.split) tma_store_2d(&mp.y1, col, r0, eb);
        else tma_store_2d(&mp.y2, col - a.split, r0, eb);
        bulk_commit();
      }
      bc++;
      tile = ntile;
      cb = ncb;
    }
    if (last_tile >= 0) {
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[j & 1]);
    }
    if (lane == 0) bulk_wait_all();
#ifdef GEMM_PROF
    if (tid == 64 && j < 4) pt[3 + j] = gtime() - t_start;
    if (tid == 64) pt[7] = gtime() - t_start;
#endif
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..9), direct stores
    const int q = warp & 3, h = (warp - 2) >> 2;
    const int half = Np / 2;   // a multiple of 8
    const bool vec_out = (a.ldy % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.Y) & 15) == 0) &&
                         (a.Y2 == nullptr || ((a.ldy2 % 4 == 0) && (reinterpret_cast<uintptr_t>(a.Y2) & 15) == 0)) &&
                         (a.split % 8 == 0 || a.split >= a.Nout);
    const bool vec_epi = (a.aux == nullptr || ((a.ldaux % 4 == 0) && (reinterpret_cast<uintptr_t>(a.aux) & 15) == 0)) &&
                         (a.R == nullptr || ((a.ldr % 4 == 0) && (reinterpret_cast<uintptr_t>(a.R) & 15) == 0));
    int j = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, j++) {
      const int acc = j & 1;
      const uint32_t use = (uint32_t)(j >> 1);
      mbar_wait(&tfull[acc], use & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int m = tile * TM + q * 32 + lane;
      const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * p.Ns);
      for (int c0 = h * half; c0 < (h + 1) * half; c0 += 32) {
        const int nb = min(4, ((h + 1) * half - c0) >> 3);   // warp-uniform
        uint32_t v[32];
#pragma unroll
        for (int u = 0; u < 4; u++)
          if (u < nb) tmem_ld8(tb + (uint32_t)(c0 + 8 * u), v + 8 * u);
        tmem_wait_ld();
        if (m < a.M) {
#pragma unroll
          for (int u = 0; u < 4; u++)
            if (u < nb) epilogue8<EPI>(a, m, c0 + 8 * u, v + 8 * u, vec_epi, vec_out);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);   // the MMA warp may overwrite this accumulator
    }
  }
  __syncthreads();
#ifdef GEMM_PROF
  if (tid == 0 && (blockIdx.x == 0 || blockIdx.x == 100))
    printf("GPROF b%d M=%d K=%d N=%d epi=%d R=%d staged %llu full0 %llu full1 %llu | issued %llu %llu %llu | seen %llu %llu %llu | done %llu %llu %llu | end %llu\n", blockIdx.x, a.M, a.K,
           a.Nout, a.epi, a.R != nullptr, pt[0], pt[1], pt[2], pt[12], pt[13], pt[14], pt[8], pt[9], pt[10], pt[3], pt[4], pt[5], pt[7]);
#endif
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.ncols));
  }
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

bool make_map(CUtensorMap *m, const float *base, int cols, int rows, int ld, int brows) {
  return tc::tma_map_f32(m, base, cols, rows, ld, brows);
}

template <int EPI>
void launch_epi(const Maps &mp, const GemmArgs &a, const TfParams &p, int grid, size_t smem, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_gemm_tc<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynMax);
    configured = true;
  }
  k_gemm_tc<EPI><<<grid, NT, smem, s>>>(mp, a, p);
}

}  // namespace

namespace tc {
namespace {
PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 f = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      f = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return f;
}
}  // namespace

bool tma_map_f32(CUtensorMap *m, const float *base, int cols, int rows, int ld, int brows, bool atom32) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = encoder();
  if (!enc || !base || (reinterpret_cast<uintptr_t>(base) & 15) || (ld % 4) || cols < 1 || rows < 1) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {32u, (cuuint32_t)brows};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE,
             atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace tc

bool tc_eligible(const GemmArgs &a) {
  const int Kp = (a.K + KC - 1) / KC * KC, Np = (a.Nout + 15) / 16 * 16;
  return a.Nout >= 16 && a.Nout <= 256 && a.K >= 1 && a.K <= 256 && a.M >= TM && (size_t)Kp * Np * 4 <= kWMax;
}

void launch_gemm_tc(const GemmArgs &a, cudaStream_t s) {
  TfParams p;
  Maps mp;
  memset(&p, 0, sizeof(p));
  memset(&mp, 0, sizeof(mp));
  const int Kp = (a.K + KC - 1) / KC * KC;
  p.nch = Kp / KC;
  p.Np = (a.Nout + 15) / 16 * 16;
  p.Ns = (p.Np + 31) / 32 * 32;
  p.ncols = 32;
  while (p.ncols < 2 * p.Ns) p.ncols <<= 1;
  // X: TMA when the rows are 16-byte aligned (and a second operand starts on a chunk)
  const bool two = a.X2 != nullptr && a.K1 < a.K;
  p.nch1 = two ? a.K1 / KC : p.nch;
  p.tma = (!two || a.K1 % KC == 0) && make_map(&mp.x1, a.X1, two ? a.K1 : a.K, a.M, a.ldx1, TM) &&
          (!two || make_map(&mp.x2, a.X2, a.K - a.K1, a.M, a.ldx2, TM));
  p.wvec = (reinterpret_cast<uintptr_t>(a.W) & 15) == 0 &&
           (a.ldw_n == 1 ? a.ldw_k % 4 == 0 : (a.ldw_k == 1 && a.ldw_n % 4 == 0));
  // epilogue: TMA stores when the outputs (and the one input tile) are 16-byte aligned rows
  int tin = 0, ldt = 0, extra = 0;
  const float *T = nullptr;
  if (a.R) { tin = 1; T = a.R; ldt = a.ldr; extra++; }
  if (a.epi == EPI_MASK) { tin = 2; T = a.aux; ldt = a.ldaux; extra++; }
  const bool split = a.Y2 != nullptr && a.split < a.Nout;
  if (a.accumulate) { tin = 3; T = a.Y; ldt = a.ldy; extra += split ? 2 : 1; }
  p.tstore = extra <= 1 && (!split || a.split % 32 == 0) &&
             make_map(&mp.y1, a.Y, split ? a.split : a.Nout, a.M, a.ldy, 32) &&
             (!split || make_map(&mp.y2, a.Y2, a.Nout - a.split, a.M, a.ldy2, 32)) &&
             (!tin || make_map(&mp.t, T, a.Nout, a.M, ldt, 32));
  p.tin = p.tstore ? tin : 0;
  p.nbusy = (p.tstore && p.Ns / 32 < 2) ? NEW / 2 : NEW;
  const size_t wbytes = (size_t)Kp * p.Np * 4, ebytes = p.tstore ? (size_t)NEW * 2 * EB : 0;
  const size_t budget = kDynMax - 1024;   // less the alignment pad
  p.stages = (int)((budget - wbytes - ebytes) / CB);
  if (p.stages > MAXST) p.stages = MAXST;
  const size_t smem = (size_t)p.stages * CB + wbytes + ebytes + 1024;
  const int ntiles = (a.M + TM - 1) / TM;
  const int grid = ntiles < num_sms() ? ntiles : num_sms();
  note_launch("k_gemm_tc", s, gemm_bytes(a), 2.0 * a.M * a.K * a.Nout);
  switch (a.epi) {
    case EPI_SIGMOID: launch_epi<EPI_SIGMOID>(mp, a, p, grid, smem, s); break;
    case EPI_TANH: launch_epi<EPI_TANH>(mp, a, p, grid, smem, s); break;
    case EPI_RELU: launch_epi<EPI_RELU>(mp, a, p, grid, smem, s); break;
    case EPI_MASK: launch_epi<EPI_MASK>(mp, a, p, grid, smem, s); break;
    default: launch_epi<EPI_NONE>(mp, a, p, grid, smem, s); break;
  }
}

}  // namespace gdp
