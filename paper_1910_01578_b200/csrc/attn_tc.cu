// tcgen05 tensor-core tiles of the segment attention (a7) for the
// tensor-core mode (bf16 operands, fp32 accumulation in TMEM), segments of S <= 128 queries.
// Forward: any memory length (M = inf included), online softmax over 128-key blocks.
//
// One CTA (4 warps, thread = query row) per (segment tau, head h), 4 CTAs per SM:
//   1. Q (128 x 16), K (keys x 16) and V^T (16 x keys) -> bf16 in shared memory, UMMA canonical
//      K-major SWIZZLE_NONE layout (as in tc_gemm.cu); the next block's K/V rows are loaded into
//      registers one block ahead;
//   2. one `tcgen05.mma.kind::f16` M = 128, N = keys (<= 128), K = 16 gives S = Q K^T in TMEM;
//   3. each warp drains its 32 TMEM lanes (`tcgen05.ld.32x32b.x16`, several under one wait):
//      row max of S, then p = 2^(S log2(e) / 4 - m2), the row sum in fp32, and P as bf16 back
//      to shared memory;
//   4. 8 MMAs (K = 16 keys each) give P V in TMEM columns 0..15 (S is consumed by then);
//   5. O = (P V) / sum and LSE = max + log(sum), the same outputs as k_attn_fwd;
//   with more than 128 keys steps 2-4 repeat per 128-key block with the running max / sum /
//   output rescaled (flash-attention style; O accumulates in fp32 registers).
// Backward: k_attn_bwd_dq_tc (query-major dQ) + k_attn_bwd_dkv_tc (key-major dK / dV), any memory length.
#include <cuda_bf16.h>

#include "common.cuh"
#include "tc_util.cuh"

namespace gdp {
namespace {

constexpr int TQ = 128;    // queries per tile (UMMA M)
constexpr int TKEY = 256;  // keys per tile (UMMA N of Q K^T, K of P V)
constexpr float kScaleTc = 0.25f;   // 1 / sqrt(16)

using tc::su32;
using tc::tmem_wait_ld;
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float *x) {
  uint32_t v[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; j++) x[j] = __uint_as_float(v[j]);
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t *>(&h);
}
// TMEM loads issued back to back with one wait: tmem_ld16_nw, then tmem_wait_ld, then
// reg_fence16 on each destination (an empty volatile asm that the compiler cannot hoist above
// the wait, so no use of the registers is scheduled before the data has landed).
__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, uint32_t *v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void reg_fence16(uint32_t *v) {
  asm volatile(""
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                 "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]));
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {   // sm_100 three-input max
  float y;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(y) : "f"(a), "f"(b), "f"(c));
  return y;
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// B = a row-major [K rows x 16] bf16 tile (canon_off with Kp = 16) read MN-major (N = its 16
// columns, K = its rows): that K-major canonical layout is already the MN-major interleaved layout
// of the transpose (core matrix = 8 rows x 16 bytes), so no transposed copy is staged.
// SWIZZLE_NONE, MN-major: SBO = next 8 columns (128 B), LBO = next 8 rows (256 B); a K step of 16
// rows is 512 B; instruction-descriptor bit 16 = B MN-major.
__device__ __forceinline__ uint64_t desc_bmn(uint32_t saddr) { return tc::desc_none(saddr, 256, 128); }

// Forward key block: 128 keys, so S needs 128 TMEM columns and the tiles 45 KB of shared memory:
// 4 CTAs (16 warps) per SM instead of 2 with 256-key blocks.
constexpr int TKF = 128;
constexpr int KR = TKF / TQ;   // key rows staged per thread
// K / V rows j (+ 128 ...) of one key block (fp32, 16 floats each) into registers
__device__ __forceinline__ void ld_kv(const float *__restrict__ qkv, int kb, int nk, int j0, int hd, float4 (&kk)[KR][4],
                                      float4 (&vv)[KR][4]) {
#pragma unroll
  for (int h2 = 0; h2 < KR; h2++) {
    const int j = j0 + h2 * TQ;
#pragma unroll
    for (int t = 0; t < 4; t++) kk[h2][t] = vv[h2][t] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (j < nk) {
      const float4 *pk = reinterpret_cast<const float4 *>(qkv + (size_t)(kb + j) * 192 + 64 + hd * 16);
      const float4 *pv = reinterpret_cast<const float4 *>(qkv + (size_t)(kb + j) * 192 + 128 + hd * 16);
#pragma unroll
      for (int t = 0; t < 4; t++) { kk[h2][t] = __ldg(pk + t); vv[h2][t] = __ldg(pv + t); }
    }
  }
}

__global__ void __launch_bounds__(TQ, 4) k_attn_fwd_tc(const float *__restrict__ qkv, float *o, float *lse, int N,
                                                      int S, int M) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  unsigned char *sQ = sm;                        // 128 x 16 bf16
  unsigned char *sK = sm + TQ * 16 * 2;          // 256 x 16
  unsigned char *sV = sK + TKF * 16 * 2;        // 128 keys x 16 (MN-major B of P V)
  unsigned char *sP = sV + 16 * TKF * 2;        // 128 x 128
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nseg = gridDim.y;
  // blockIdx.x = head (fastest in dispatch order), so the four heads' longest key ranges go first
  const int tau = nseg - 1 - blockIdx.y, hd = blockIdx.x;
  const int q0 = tau * S, q1 = min(N, q0 + S);
  const int lo = M < 0 ? 0 : max(0, q0 - M), hi = q1;
  // scores in log2 units: s2 = S_ij / 4 * log2(e), p = 2^(s2 - m2)
  const float kC = kScaleTc * 1.4426950408889634f;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)), "r"((uint32_t)TKF));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // Q row tid (16-byte loads; zero rows past the segment)
  {
    const int i = q0 + tid;
    float4 a[4] = {};
    if (i < q1) {
      const float4 *p = reinterpret_cast<const float4 *>(qkv + (size_t)i * 192 + hd * 16);
#pragma unroll
      for (int t = 0; t < 4; t++) a[t] = p[t];
    }
    uint4 lo8 = make_uint4(pack2(a[0].x, a[0].y), pack2(a[0].z, a[0].w), pack2(a[1].x, a[1].y), pack2(a[1].z, a[1].w));
    uint4 hi8 = make_uint4(pack2(a[2].x, a[2].y), pack2(a[2].z, a[2].w), pack2(a[3].x, a[3].y), pack2(a[3].z, a[3].w));
    *reinterpret_cast<uint4 *>(sQ + tc::canon_off(tid, 0, 16)) = lo8;
    *reinterpret_cast<uint4 *>(sQ + tc::canon_off(tid, 8, 16)) = hi8;
  }
  const uint32_t trow_off = (uint32_t)(warp * 32) << 16;
  float m2 = -INFINITY, sum = 0.f, acc[16];
#pragma unroll
  for (int c = 0; c < 16; c++) acc[c] = 0.f;
  uint32_t phase = 0;
  float4 kk[KR][4], vv[KR][4];   // the next key block's rows, loaded one block ahead
  ld_kv(qkv, lo, min(TKF, hi - lo), tid, hd, kk, vv);
  // online softmax over 128-key blocks
  for (int kb = lo; kb < hi; kb += TKF) {
    const int nk = min(TKF, hi - kb), Np = (nk + 15) & ~15;
#pragma unroll
    for (int h2 = 0; h2 < KR; h2++) {   // K / V rows tid and tid + 128 of this block -> bf16 tiles
      const int j = tid + h2 * TQ;
      *reinterpret_cast<uint4 *>(sK + tc::canon_off(j, 0, 16)) =
          make_uint4(pack2(kk[h2][0].x, kk[h2][0].y), pack2(kk[h2][0].z, kk[h2][0].w), pack2(kk[h2][1].x, kk[h2][1].y),
                     pack2(kk[h2][1].z, kk[h2][1].w));
      *reinterpret_cast<uint4 *>(sK + tc::canon_off(j, 8, 16)) =
          make_uint4(pack2(kk[h2][2].x, kk[h2][2].y), pack2(kk[h2][2].z, kk[h2][2].w), pack2(kk[h2][3].x, kk[h2][3].y),
                     pack2(kk[h2][3].z, kk[h2][3].w));
      *reinterpret_cast<uint4 *>(sV + tc::canon_off(j, 0, 16)) =
          make_uint4(pack2(vv[h2][0].x, vv[h2][0].y), pack2(vv[h2][0].z, vv[h2][0].w), pack2(vv[h2][1].x, vv[h2][1].y),
                     pack2(vv[h2][1].z, vv[h2][1].w));
      *reinterpret_cast<uint4 *>(sV + tc::canon_off(j, 8, 16)) =
          make_uint4(pack2(vv[h2][2].x, vv[h2][2].y), pack2(vv[h2][2].z, vv[h2][2].w), pack2(vv[h2][3].x, vv[h2][3].y),
                     pack2(vv[h2][3].z, vv[h2][3].w));
    }
    if (kb + TKF < hi) ld_kv(qkv, kb + TKF, min(TKF, hi - kb - TKF), tid, hd, kk, vv);   // in flight meanwhile
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();   // (also: the previous block's P V has been drained by every warp)
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base;
    const uint32_t trow = tmem + trow_off;
    // S = Q K^T: M = 128, N = Np, K = 16
    if (tid == 0) {
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(Np >> 3) << 17) | ((uint32_t)(TQ >> 4) << 24);
      const uint64_t ad = tc::desc_none(su32(sQ), 128, 256), bd = tc::desc_none(su32(sK), 128, 256);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                   "l"(ad), "l"(bd), "r"(idesc), "r"(0u));
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar))
                   : "memory");
    }
    tc::mbar_wait(&mbar, phase);
    phase ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // row max of this block (64 columns per TMEM wait), then the rescale of the running sum / output
    float bm = -INFINITY;
    if (nk == TKF) {
#pragma unroll 1
      for (int c0 = 0; c0 < TKF; c0 += 64) {
        uint32_t x[4][16];
#pragma unroll
        for (int u = 0; u < 4; u++) tmem_ld16_nw(trow + c0 + 16 * u, x[u]);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 4; u++) {
          reg_fence16(x[u]);
#pragma unroll
          for (int jj = 0; jj < 16; jj += 2) bm = fmax3(bm, __uint_as_float(x[u][jj]), __uint_as_float(x[u][jj + 1]));
        }
      }
    } else {
      for (int c0 = 0; c0 < Np; c0 += 16) {
        float x[16];
        tmem_ld16(trow + c0, x);
#pragma unroll
        for (int jj = 0; jj < 16; jj++)
          if (c0 + jj < nk) bm = fmaxf(bm, x[jj]);
      }
    }
    const float nm2 = fmaxf(m2, bm * kC);   // kC > 0: the max commutes with the scale
    const float alpha = ex2(m2 - nm2);       // 0 on the first block (m2 = -inf)
    sum *= alpha;
#pragma unroll
    for (int c = 0; c < 16; c++) acc[c] *= alpha;
    m2 = nm2;
    // P = 2^(s2 - m2) as bf16 into shared memory, 32 columns per TMEM wait
    if (nk == TKF) {
#pragma unroll 1
      for (int c0 = 0; c0 < TKF; c0 += 32) {
        uint32_t x[2][16];
        tmem_ld16_nw(trow + c0, x[0]);
        tmem_ld16_nw(trow + c0 + 16, x[1]);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 2; u++) {
          reg_fence16(x[u]);
          float p[16];
#pragma unroll
          for (int jj = 0; jj < 16; jj++) {
            p[jj] = ex2(fmaf(__uint_as_float(x[u][jj]), kC, -m2));
            sum += p[jj];
          }
          *reinterpret_cast<uint4 *>(sP + tc::canon_off(tid, c0 + 16 * u, TKF)) =
              make_uint4(pack2(p[0], p[1]), pack2(p[2], p[3]), pack2(p[4], p[5]), pack2(p[6], p[7]));
          *reinterpret_cast<uint4 *>(sP + tc::canon_off(tid, c0 + 16 * u + 8, TKF)) =
              make_uint4(pack2(p[8], p[9]), pack2(p[10], p[11]), pack2(p[12], p[13]), pack2(p[14], p[15]));
        }
      }
    } else {
      for (int c0 = 0; c0 < TKF; c0 += 16) {
        float x[16];
        if (c0 < Np) tmem_ld16(trow + c0, x);
        float p[16];
#pragma unroll
        for (int jj = 0; jj < 16; jj++) {
          p[jj] = (c0 + jj < nk) ? ex2(fmaf(x[jj], kC, -m2)) : 0.f;
          sum += p[jj];
        }
        *reinterpret_cast<uint4 *>(sP + tc::canon_off(tid, c0, TKF)) =
            make_uint4(pack2(p[0], p[1]), pack2(p[2], p[3]), pack2(p[4], p[5]), pack2(p[6], p[7]));
        *reinterpret_cast<uint4 *>(sP + tc::canon_off(tid, c0 + 8, TKF)) =
            make_uint4(pack2(p[8], p[9]), pack2(p[10], p[11]), pack2(p[12], p[13]), pack2(p[14], p[15]));
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();   // every row's S has been read and P written
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // P V: M = 128, N = 16, K = 256 keys (16 steps), into TMEM columns 0..15
    if (tid == 0) {
      const uint32_t idesc =
          (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(TQ >> 4) << 24);
      const uint32_t sbo = (TKF >> 3) * 128;
      for (int ks = 0; ks < Np / 16; ks++) {
        const uint64_t ad = tc::desc_none(su32(sP) + ks * 256, 128, sbo), bd = desc_bmn(su32(sV) + ks * 512);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                     "l"(ad), "l"(bd), "r"(idesc), "r"(ks > 0 ? 1u : 0u));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar))
                   : "memory");
    }
    tc::mbar_wait(&mbar, phase);
    phase ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    {
      float x[16];
      tmem_ld16(trow, x);
#pragma unroll
      for (int c = 0; c < 16; c++) acc[c] += x[c];
    }
  }
  {
    const int i = q0 + tid;
    if (i < q1) {
      const float inv = 1.f / sum;
      float4 *dst = reinterpret_cast<float4 *>(o + (size_t)i * kH + hd * 16);
#pragma unroll
      for (int t = 0; t < 4; t++)
        dst[t] = make_float4(acc[4 * t] * inv, acc[4 * t + 1] * inv, acc[4 * t + 2] * inv, acc[4 * t + 3] * inv);
      lse[(size_t)i * kHeads + hd] = m2 * 0.6931471805599453f + logf(sum);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"((uint32_t)TKF));
}

// ---------------------------------------------------------------- backward, any memory length
// A key of segment sigma receives memory contributions from the later query segments its key range
// reaches (one when M <= S, several when M > S or M = inf),
// so the backward splits into a query-major dQ pass and a key-major dK / dV pass (as the SIMT
// k_attn_bwd_dq / _dkv), each on tcgen05 with 128 x 128 (query x key) tiles:
//   k_attn_bwd_dq_tc  (segment tau, head h), thread = query row, per 128-key block:
//     S = Q K^T and dP = dO V^T into TMEM columns [0, 128) / [128, 256); p = exp(S/4 - LSE),
//     dS = p (dP - D) / 4 as bf16 to shared memory; dQ_block = dS K (M = 128, N = 16,
//     K = keys) into TMEM columns [0, 16), summed over blocks in fp32 registers.
//   k_attn_bwd_dkv_tc (segment sigma, head h), thread = key row, per query segment tau >= sigma
//     whose key range reaches the block: S^T = K Q^T and dP^T = V dO^T (M = 128 keys, N = queries),
//     P^T and dS^T as bf16, dK_tau = dS^T Q and dV_tau = P^T dO (M = 128 keys, N = 16, K = queries)
//     into TMEM columns [0, 32).  tau == sigma is the own contribution (dqkv[:, 64:192]); the
//     later segments' are summed in fp32 registers into the memory rows dkvm[:, 0:128]
//     (stop-gradient for x), zeros where no later segment reaches the key.  Every output row is
//     written exactly once, no atomics.
__device__ __forceinline__ void st_row16(unsigned char *tile, int r, const float *f) {   // K-major row, Kp = 16
  *reinterpret_cast<uint4 *>(tile + tc::canon_off(r, 0, 16)) =
      make_uint4(pack2(f[0], f[1]), pack2(f[2], f[3]), pack2(f[4], f[5]), pack2(f[6], f[7]));
  *reinterpret_cast<uint4 *>(tile + tc::canon_off(r, 8, 16)) =
      make_uint4(pack2(f[8], f[9]), pack2(f[10], f[11]), pack2(f[12], f[13]), pack2(f[14], f[15]));
}
__device__ __forceinline__ void ld16(const float *p, float *f) {
#pragma unroll
  for (int t = 0; t < 4; t++) {
    const float4 a = reinterpret_cast<const float4 *>(p)[t];
    f[4 * t] = a.x; f[4 * t + 1] = a.y; f[4 * t + 2] = a.z; f[4 * t + 3] = a.w;
  }
}
__device__ __forceinline__ void mma_f16(uint32_t tmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t accum) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
               "l"(ad), "l"(bd), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void mma_commit(uint64_t *mb) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(mb))
               : "memory");
}
__device__ __forceinline__ void sync_for_mma() {   // generic-proxy smem writes / TMEM reads -> MMA
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ uint32_t idesc_f16(int n) {   // bf16 x bf16 -> fp32, M = 128, K-major A and B
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(TQ >> 4) << 24);
}
constexpr uint32_t kSbo128 = (TQ >> 3) * 128;   // next 8-row group of a K-major tile with 128 columns
__device__ __forceinline__ uint32_t idesc_f16_bmn(int n) { return idesc_f16(n) | (1u << 16); }

// dQ key block: 64 keys, so S and dP take 128 TMEM columns together: 4 CTAs per SM.  The shared
// tiles keep their 128-key layouts (Kp = 128); only the first 64 rows / K columns are used.
constexpr int TKQ = 64;
__global__ void __launch_bounds__(TQ, 4) k_attn_bwd_dq_tc(const float *__restrict__ qkv, const float *__restrict__ o,
                                                         const float *__restrict__ lse,
                                                         const float *__restrict__ dout, float *dqkv, int N, int S,
                                                         int M) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  unsigned char *sQ = sm;                 // 128 x 16 (A of S)
  unsigned char *sdO = sQ + TQ * 32;      // 128 x 16 (A of dP)
  unsigned char *sK = sdO + TQ * 32;      // 128 keys x 16 (B of S)
  unsigned char *sV = sK + TQ * 32;       // 128 keys x 16 (B of dP)
  unsigned char *sdS = sV + TQ * 32;      // 128 queries x 128 keys (A of dQ; its B is sK read MN-major)
  const int tid = threadIdx.x, warp = tid >> 5;
  // blockIdx.x = head (fastest in dispatch order), so the four heads' longest key ranges go first
  const int tau = gridDim.y - 1 - blockIdx.y, hd = blockIdx.x;
  const int q0 = tau * S, q1 = min(N, q0 + S);
  const int lo = M < 0 ? 0 : max(0, q0 - M), hi = q1;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)), "r"((uint32_t)(2 * TKQ)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int i = q0 + tid;
  const bool qv = i < q1;
  // L2 = LSE in log2 units (+inf on padding rows, so p = 2^(s2 - L2) = 0 there without a branch)
  const float kC = kScaleTc * 1.4426950408889634f;
  float L2 = INFINITY, D = 0.f;
  {
    float qf[16] = {}, gf[16] = {}, of[16] = {};
    if (qv) {
      ld16(qkv + (size_t)i * 192 + hd * 16, qf);
      ld16(dout + (size_t)i * kH + hd * 16, gf);
      ld16(o + (size_t)i * kH + hd * 16, of);
      L2 = lse[(size_t)i * kHeads + hd] * 1.4426950408889634f;
#pragma unroll
      for (int c = 0; c < 16; c++) D = fmaf(gf[c], of[c], D);
    }
    st_row16(sQ, tid, qf);
    st_row16(sdO, tid, gf);
  }
  static_assert(kScaleTc == 0.25f, "the dS scale is folded into the exponent as 2^-2");
  const float L2q = L2 + 2.f;
  const uint32_t trow_off = (uint32_t)(warp * 32) << 16;
  float acc[16];
#pragma unroll
  for (int c = 0; c < 16; c++) acc[c] = 0.f;
  uint32_t phase = 0;
  float kf[16], vf[16];   // the next key block's rows, loaded one block ahead
  auto ld_kv_row = [&](int kb) {
#pragma unroll
    for (int c = 0; c < 16; c++) kf[c] = vf[c] = 0.f;
    if (tid < TKQ && kb + tid < hi) {
      ld16(qkv + (size_t)(kb + tid) * 192 + 64 + hd * 16, kf);
      ld16(qkv + (size_t)(kb + tid) * 192 + 128 + hd * 16, vf);
    }
  };
  ld_kv_row(lo);
  for (int kb = lo; kb < hi; kb += TKQ) {
    const int nk = min(TKQ, hi - kb), Np = (nk + 15) & ~15;
    if (tid < TKQ) {
      st_row16(sK, tid, kf);
      st_row16(sV, tid, vf);
    }
    if (kb + TKQ < hi) ld_kv_row(kb + TKQ);   // in flight during this block
    sync_for_mma();   // (also: the previous block's dQ has been drained by every warp)
    const uint32_t tmem = tmem_base, trow = tmem + trow_off;
    if (tid == 0) {
      mma_f16(tmem, tc::desc_none(su32(sQ), 128, 256), tc::desc_none(su32(sK), 128, 256), idesc_f16(Np), 0u);
      mma_f16(tmem + (uint32_t)TKQ, tc::desc_none(su32(sdO), 128, 256), tc::desc_none(su32(sV), 128, 256), idesc_f16(Np), 0u);
      mma_commit(&mbar);
    }
    tc::mbar_wait(&mbar, phase);
    phase ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const bool full = nk == TKQ;
    for (int c0 = 0; c0 < Np; c0 += 16) {
      uint32_t sx[16], dpx[16];
      float ds[16];
      tmem_ld16_nw(trow + c0, sx);
      tmem_ld16_nw(trow + TKQ + c0, dpx);
      tmem_wait_ld();
      reg_fence16(sx);
      reg_fence16(dpx);
      // dS = p (dP - D) / 4 with the 1/4 folded into the exponent: p / 4 = 2^(s2 - L2 - 2)
      if (full) {
#pragma unroll
        for (int jj = 0; jj < 16; jj++)
          ds[jj] = ex2(fmaf(__uint_as_float(sx[jj]), kC, -L2q)) * (__uint_as_float(dpx[jj]) - D);
      } else {
#pragma unroll
        for (int jj = 0; jj < 16; jj++) {
          const float d = ex2(fmaf(__uint_as_float(sx[jj]), kC, -L2q)) * (__uint_as_float(dpx[jj]) - D);
          ds[jj] = c0 + jj < nk ? d : 0.f;
        }
      }
      *reinterpret_cast<uint4 *>(sdS + tc::canon_off(tid, c0, TQ)) =
          make_uint4(pack2(ds[0], ds[1]), pack2(ds[2], ds[3]), pack2(ds[4], ds[5]), pack2(ds[6], ds[7]));
      *reinterpret_cast<uint4 *>(sdS + tc::canon_off(tid, c0 + 8, TQ)) =
          make_uint4(pack2(ds[8], ds[9]), pack2(ds[10], ds[11]), pack2(ds[12], ds[13]), pack2(ds[14], ds[15]));
    }
    sync_for_mma();   // every row's S / dP read, dS written
    if (tid == 0) {   // dQ_block = dS K: M = 128, N = 16, K = Np keys
      for (int ks = 0; ks < Np / 16; ks++)
        mma_f16(tmem, tc::desc_none(su32(sdS) + ks * 256, 128, kSbo128), desc_bmn(su32(sK) + ks * 512),
                idesc_f16_bmn(16), ks > 0 ? 1u : 0u);
      mma_commit(&mbar);
    }
    tc::mbar_wait(&mbar, phase);
    phase ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    {
      float x[16];
      tmem_ld16(trow, x);
#pragma unroll
      for (int c = 0; c < 16; c++) acc[c] += x[c];
    }
  }
  if (qv) {
    float4 *dst = reinterpret_cast<float4 *>(dqkv + (size_t)i * 192 + hd * 16);
#pragma unroll
    for (int t = 0; t < 4; t++) dst[t] = make_float4(acc[4 * t], acc[4 * t + 1], acc[4 * t + 2], acc[4 * t + 3]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"((uint32_t)(2 * TKQ)));
}

// dK / dV query chunk: 64 queries, so S^T and dP^T take 128 TMEM columns together and P^T / dS^T
// 16 KB each (48 KB of shared memory: Q and dO are read MN-major as the B of dK / dV, no transposed
// copies; 13.95 ms per C4 M = inf step against 15.6 with the copies).  3 CTAs per SM: 4 (128
// registers) spill the next segment's prefetched rows or, loading them at staging time, expose
// their latency (15.5 ms measured).  A query segment is staged whole and processed as up to two
// chunks; the chunks' dK / dV are summed in fp32 registers.
constexpr int TQC = 64;
constexpr uint32_t kSbo64 = (TQC >> 3) * 128;   // next 8-row group of a K-major tile with 64 columns
__global__ void __launch_bounds__(TQ, 3) k_attn_bwd_dkv_tc(const float *__restrict__ qkv, const float *__restrict__ o,
                                                          const float *__restrict__ lse,
                                                          const float *__restrict__ dout, float *dqkv, float *dkvm,
                                                          int N, int S, int M, int nseg) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  __shared__ __align__(16) float sL[TQ], sD[TQ];
  unsigned char *sK = sm;                 // 128 keys x 16 (A of S^T)
  unsigned char *sV = sK + TQ * 32;       // 128 keys x 16 (A of dP^T)
  unsigned char *sQ = sV + TQ * 32;       // 128 queries x 16 (B of S^T, and MN-major B of dK; chunk c from row 64c)
  unsigned char *sdO = sQ + TQ * 32;      // 128 queries x 16 (B of dP^T, and MN-major B of dV)
  unsigned char *sPt = sdO + TQ * 32;     // 128 keys x 64 queries (A of dV)
  unsigned char *sdSt = sPt + TQ * TQC * 2;   // 128 keys x 64 queries (A of dK)
  const int tid = threadIdx.x, warp = tid >> 5;
  // sigma = 0 has the most query segments; blockIdx.x = head, so every head's heaviest CTAs go first
  const int sig = blockIdx.y, hd = blockIdx.x;
  const int k0 = sig * S, k1 = min(N, k0 + S), nk = k1 - k0;
  const int tau_hi = M < 0 ? nseg - 1 : min(nseg - 1, (int)(((long long)k1 - 1 + M) / S));
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)), "r"((uint32_t)(2 * TQC)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int j = k0 + tid;
  const bool kvalid = tid < nk;
  {
    float kf[16] = {}, vf[16] = {};
    if (kvalid) {
      ld16(qkv + (size_t)j * 192 + 64 + hd * 16, kf);
      ld16(qkv + (size_t)j * 192 + 128 + hd * 16, vf);
    }
    st_row16(sK, tid, kf);
    st_row16(sV, tid, vf);
  }
  const uint32_t trow_off = (uint32_t)(warp * 32) << 16;
  // dK / dV of this thread's key summed over chunks: the own segment's are written to dqkv and
  // reset after tau = sigma, the later segments' accumulate into the memory rows dkvm
  float dkm[16], dvm[16];
#pragma unroll
  for (int c = 0; c < 16; c++) dkm[c] = dvm[c] = 0.f;
  uint32_t phase = 0;
  // the next query segment's rows (Q, dO, O, LSE) are loaded one segment ahead
  float qf[16], gf[16], of[16], Lr = 0.f;
  auto ld_q_rows = [&](int tau) {
    const int i = tau * S + tid;
#pragma unroll
    for (int c = 0; c < 16; c++) qf[c] = gf[c] = of[c] = 0.f;
    Lr = INFINITY;
    if (i < min(N, tau * S + S)) {
      ld16(qkv + (size_t)i * 192 + hd * 16, qf);
      ld16(dout + (size_t)i * kH + hd * 16, gf);
      ld16(o + (size_t)i * kH + hd * 16, of);
      Lr = lse[(size_t)i * kHeads + hd];   // scaled to log2 units at its use, so the load stays in flight
    }
  };
  const float kC = kScaleTc * 1.4426950408889634f;
  ld_q_rows(sig);
  for (int tau = sig; tau <= tau_hi; tau++) {
    const int q0 = tau * S, q1 = min(N, q0 + S), nq = q1 - q0;
    const int lo = M < 0 ? 0 : max(0, q0 - M);
    const bool inr = kvalid && j >= lo;
    {
      float D = 0.f;
#pragma unroll
      for (int c = 0; c < 16; c++) D = fmaf(gf[c], of[c], D);
      st_row16(sQ, tid, qf);
      st_row16(sdO, tid, gf);
      sL[tid] = Lr * 1.4426950408889634f;   // LSE in log2 units, +inf past the segment (p = 0 there)
      sD[tid] = D;
    }
    if (tau < tau_hi) ld_q_rows(tau + 1);   // in flight during this segment
    for (int h0 = 0; h0 < nq; h0 += TQC) {
      const int Nqp = (min(TQC, nq - h0) + 15) & ~15;
      // staged rows visible to the MMAs; every warp has drained the previous chunk's dK / dV
      sync_for_mma();
      const uint32_t tmem = tmem_base, trow = tmem + trow_off;
      if (tid == 0) {   // S^T = K Q^T -> cols [0, Nqp); dP^T = V dO^T -> cols [64, 64 + Nqp)
        mma_f16(tmem, tc::desc_none(su32(sK), 128, 256), tc::desc_none(su32(sQ) + (h0 >> 3) * 256, 128, 256), idesc_f16(Nqp), 0u);
        mma_f16(tmem + (uint32_t)TQC, tc::desc_none(su32(sV), 128, 256), tc::desc_none(su32(sdO) + (h0 >> 3) * 256, 128, 256),
                idesc_f16(Nqp), 0u);
        mma_commit(&mbar);
      }
      tc::mbar_wait(&mbar, phase);
      phase ^= 1u;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int c0 = 0; c0 < Nqp; c0 += 16) {
        uint32_t sx[16], dpx[16];
        float p[16], ds[16];
        tmem_ld16_nw(trow + c0, sx);
        tmem_ld16_nw(trow + TQC + c0, dpx);
        tmem_wait_ld();
        reg_fence16(sx);
        reg_fence16(dpx);
        // dS' = p (dP - D); the 1/4 of dS = dS' / 4 is applied to dK once per chunk
        if (inr) {
#pragma unroll
          for (int q4 = 0; q4 < 16; q4 += 4) {
            const float4 l4 = *reinterpret_cast<const float4 *>(sL + h0 + c0 + q4);
            const float4 d4 = *reinterpret_cast<const float4 *>(sD + h0 + c0 + q4);
            const float lq[4] = {l4.x, l4.y, l4.z, l4.w}, dq[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
            for (int u = 0; u < 4; u++) {
              const int qq = q4 + u;
              p[qq] = ex2(fmaf(__uint_as_float(sx[qq]), kC, -lq[u]));   // 0 past the segment (L = +inf)
              ds[qq] = p[qq] * (__uint_as_float(dpx[qq]) - dq[u]);
            }
          }
        } else {
#pragma unroll
          for (int qq = 0; qq < 16; qq++) p[qq] = ds[qq] = 0.f;
        }
        *reinterpret_cast<uint4 *>(sPt + tc::canon_off(tid, c0, TQC)) =
            make_uint4(pack2(p[0], p[1]), pack2(p[2], p[3]), pack2(p[4], p[5]), pack2(p[6], p[7]));
        *reinterpret_cast<uint4 *>(sPt + tc::canon_off(tid, c0 + 8, TQC)) =
            make_uint4(pack2(p[8], p[9]), pack2(p[10], p[11]), pack2(p[12], p[13]), pack2(p[14], p[15]));
        *reinterpret_cast<uint4 *>(sdSt + tc::canon_off(tid, c0, TQC)) =
            make_uint4(pack2(ds[0], ds[1]), pack2(ds[2], ds[3]), pack2(ds[4], ds[5]), pack2(ds[6], ds[7]));
        *reinterpret_cast<uint4 *>(sdSt + tc::canon_off(tid, c0 + 8, TQC)) =
            make_uint4(pack2(ds[8], ds[9]), pack2(ds[10], ds[11]), pack2(ds[12], ds[13]), pack2(ds[14], ds[15]));
      }
      sync_for_mma();   // S^T / dP^T consumed, P^T and dS^T written
      if (tid == 0) {   // dK = dS^T Q -> cols [0, 16); dV = P^T dO -> cols [16, 32); K = this chunk's queries
        const uint32_t qt = (uint32_t)(h0 >> 3) * 256;
        for (int ks = 0; ks < Nqp / 16; ks++) {
          mma_f16(tmem, tc::desc_none(su32(sdSt) + ks * 256, 128, kSbo64), desc_bmn(su32(sQ) + qt + ks * 512),
                  idesc_f16_bmn(16), ks > 0 ? 1u : 0u);
          mma_f16(tmem + 16u, tc::desc_none(su32(sPt) + ks * 256, 128, kSbo64), desc_bmn(su32(sdO) + qt + ks * 512),
                  idesc_f16_bmn(16), ks > 0 ? 1u : 0u);
        }
        mma_commit(&mbar);
      }
      tc::mbar_wait(&mbar, phase);
      phase ^= 1u;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float dk[16], dv[16];
      tmem_ld16(trow, dk);
      tmem_ld16(trow + 16u, dv);
#pragma unroll
      for (int c = 0; c < 16; c++) { dkm[c] = fmaf(dk[c], kScaleTc, dkm[c]); dvm[c] += dv[c]; }
    }
    if (tau == sig) {
      if (kvalid) {
#pragma unroll
        for (int t = 0; t < 4; t++) {
          reinterpret_cast<float4 *>(dqkv + (size_t)j * 192 + 64 + hd * 16)[t] =
              make_float4(dkm[4 * t], dkm[4 * t + 1], dkm[4 * t + 2], dkm[4 * t + 3]);
          reinterpret_cast<float4 *>(dqkv + (size_t)j * 192 + 128 + hd * 16)[t] =
              make_float4(dvm[4 * t], dvm[4 * t + 1], dvm[4 * t + 2], dvm[4 * t + 3]);
        }
      }
#pragma unroll
      for (int c = 0; c < 16; c++) dkm[c] = dvm[c] = 0.f;
    }
  }
  if (kvalid) {
#pragma unroll
    for (int t = 0; t < 4; t++) {
      reinterpret_cast<float4 *>(dkvm + (size_t)j * 128 + hd * 16)[t] =
          make_float4(dkm[4 * t], dkm[4 * t + 1], dkm[4 * t + 2], dkm[4 * t + 3]);
      reinterpret_cast<float4 *>(dkvm + (size_t)j * 128 + 64 + hd * 16)[t] =
          make_float4(dvm[4 * t], dvm[4 * t + 1], dvm[4 * t + 2], dvm[4 * t + 3]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"((uint32_t)(2 * TQC)));
}

}  // namespace

bool attn_fwd_tc_eligible(int S, int M) { return S >= 1 && S <= TQ && M >= -1; }
// backward: the query-major dQ and key-major dK / dV kernels take every memory length (round 2: the
// single-kernel M <= S tile, TMEM-bound to one CTA per SM, measured 0.93 ms per C4 step against
// 0.46 ms for these two)
bool attn_bwd_tc_long_eligible(int S, int M) { return S >= 1 && S <= TQ && M >= -1; }

static const size_t kSmemDq = (size_t)4 * TQ * 32 + (size_t)TQ * TQ * 2;         // 48 KB
static const size_t kSmemDkv = (size_t)4 * TQ * 32 + (size_t)2 * TQ * TQC * 2;   // 48 KB
void launch_attn_bwd_dq_tc(const float *qkv, const float *o, const float *lse, const float *dout, float *dqkv, int N,
                           int S, int M, cudaStream_t s) {
  const int nseg = (N + S - 1) / S;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_attn_bwd_dq_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemDq);
    configured = true;
  }
  k_attn_bwd_dq_tc<<<dim3(kHeads, nseg), TQ, kSmemDq, s>>>(qkv, o, lse, dout, dqkv, N, S, M);
}
void launch_attn_bwd_dkv_tc(const float *qkv, const float *o, const float *lse, const float *dout, float *dqkv,
                            float *dkvm, int N, int S, int M, cudaStream_t s) {
  const int nseg = (N + S - 1) / S;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_attn_bwd_dkv_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemDkv);
    configured = true;
  }
  k_attn_bwd_dkv_tc<<<dim3(kHeads, nseg), TQ, kSmemDkv, s>>>(qkv, o, lse, dout, dqkv, dkvm, N, S, M, nseg);
}


void launch_attn_fwd_tc(const float *qkv, float *o, float *lse, int N, int S, int M, cudaStream_t s) {
  const int nseg = (N + S - 1) / S;
  const size_t smem = (size_t)(TQ * 16 + TKF * 16 + 16 * TKF + TQ * TKF) * 2;   // 45 KB
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_attn_fwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  k_attn_fwd_tc<<<dim3(kHeads, nseg), TQ, smem, s>>>(qkv, o, lse, N, S, M);
}

}  // namespace gdp
