// tcgen05 tensor-core path for the tall-skinny dense maps of the policy network (bf16
// operands, fp32 accumulation in TMEM): Y = epi(X W + b) (+R), the same contract as k_gemm.
//
// Persistent CTAs (8 warps), up to 4 per SM as shared memory and TMEM allow.  The weight operand W (K x Nout, <= 256 x 256) is
// converted to bf16 once per CTA into shared memory in the UMMA canonical K-major layout
// (SWIZZLE_NONE: 8-row x 16-byte core matrices, LBO = next core matrix along K, SBO = next
// 8-row group).  For every 128-row tile of X: the 4 warps convert the fp32 rows to bf16 into
// the same layout, one elected thread issues K/16 `tcgen05.mma.cta_group::1.kind::f16`
// (M = 128, N = Nout padded to 16) accumulating into TMEM, `tcgen05.commit` arrives on an
// mbarrier, and each warp drains its 32 TMEM lanes with `tcgen05.ld.32x32b.x8` straight into
// the fused epilogue (bias, sigmoid / tanh / ReLU / ReLU-mask, residual, split output).
#include <cuda_bf16.h>

#include "common.cuh"

namespace gdp {
namespace {

constexpr int TM = 128;   // rows per tile (UMMA M)
constexpr int TT = 256;   // threads per CTA (2 warpgroups: load together, split the epilogue columns)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // version = 1 (Blackwell); base offset 0, lbo mode 0, SWIZZLE_NONE
  return d;
}

// byte offset of element (row r, col k) in a canonical K-major SWIZZLE_NONE tile with Kp columns
__device__ __forceinline__ uint32_t canon_off(int r, int k, int Kp) {
  return (uint32_t)(((r >> 3) * (Kp >> 3) + (k >> 3)) * 128 + (r & 7) * 16 + (k & 7) * 2);
}

__device__ __forceinline__ float epi_apply(int epi, float v) {
  switch (epi) {
    case EPI_SIGMOID: return 1.0f / (1.0f + expf(-v));
    case EPI_TANH: return tanhf(v);
    case EPI_RELU: return v > 0.f ? v : 0.f;
    default: return v;
  }
}

__global__ void __launch_bounds__(TT, 4) k_gemm_tc(GemmArgs a, int Kp, int Np, int ncols) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  unsigned char *sA = sm;                                // TM x Kp bf16
  unsigned char *sB = sm + (size_t)TM * Kp * 2;          // Np x Kp bf16
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // W -> bf16 canonical [n][k]: element (n, k) = W[k * ldw_k + n * ldw_n]; consecutive threads
  // walk the contiguous dimension of W
  // (unrolled: the loads of several elements are in flight at once; W is L2-resident)
  if (a.ldw_n == 1) {
#pragma unroll 8
    for (int e = tid; e < (Kp / 2) * Np; e += TT) {
      const int kk = e / Np, n = e % Np, k = 2 * kk;
      float w0 = 0.f, w1 = 0.f;
      if (n < a.Nout) {
        if (k < a.K) w0 = a.W[(size_t)k * a.ldw_k + n];
        if (k + 1 < a.K) w1 = a.W[(size_t)(k + 1) * a.ldw_k + n];
      }
      *reinterpret_cast<__nv_bfloat162 *>(sB + canon_off(n, k, Kp)) = __floats2bfloat162_rn(w0, w1);
    }
  } else {
#pragma unroll 8
    for (int e = tid; e < Np * (Kp / 2); e += TT) {
      const int n = e / (Kp / 2), k = (e % (Kp / 2)) * 2;
      float w0 = 0.f, w1 = 0.f;
      if (n < a.Nout) {
        if (k < a.K) w0 = a.W[(size_t)k * a.ldw_k + (size_t)n * a.ldw_n];
        if (k + 1 < a.K) w1 = a.W[(size_t)(k + 1) * a.ldw_k + (size_t)n * a.ldw_n];
      }
      *reinterpret_cast<__nv_bfloat162 *>(sB + canon_off(n, k, Kp)) = __floats2bfloat162_rn(w0, w1);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(Np >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
  const uint32_t sbo = (uint32_t)(Kp >> 3) * 128;
  const uint32_t aBase = smem_u32(sA), bBase = smem_u32(sB);
  uint32_t phase = 0;
  const int ntiles = (a.M + TM - 1) / TM;
  const bool vec4 = (a.K % 4 == 0) && (a.K1 % 4 == 0) && (a.ldx1 % 4 == 0) && (a.X2 == nullptr || a.ldx2 % 4 == 0) &&
                    ((reinterpret_cast<uintptr_t>(a.X1) & 15) == 0) &&
                    (a.X2 == nullptr || (reinterpret_cast<uintptr_t>(a.X2) & 15) == 0);
  const bool vec_out = (a.ldy % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.Y) & 15) == 0) &&
                       (a.Y2 == nullptr || ((a.ldy2 % 4 == 0) && (reinterpret_cast<uintptr_t>(a.Y2) & 15) == 0)) &&
                       (a.split % 8 == 0 || a.split >= a.Nout);
  const bool vec_epi = (a.aux == nullptr || ((a.ldaux % 4 == 0) && (reinterpret_cast<uintptr_t>(a.aux) & 15) == 0)) &&
                       (a.R == nullptr || ((a.ldr % 4 == 0) && (reinterpret_cast<uintptr_t>(a.R) & 15) == 0));
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int m0 = tile * TM;
    // X rows -> bf16 canonical (two-operand concat: columns [0, K1) from X1, [K1, K) from X2)
    if (vec4) {
      // 16-byte loads, 4 columns per item, unrolled for memory-level parallelism
      const int q = Kp / 4;
#pragma unroll 8
      for (int e = tid; e < TM * q; e += TT) {
        const int r = e / q, k = (e % q) * 4;
        const int m = m0 + r;
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (m < a.M && k < a.K)
          x = (k < a.K1) ? *reinterpret_cast<const float4 *>(a.X1 + (size_t)m * a.ldx1 + k)
                         : *reinterpret_cast<const float4 *>(a.X2 + (size_t)m * a.ldx2 + (k - a.K1));
        __nv_bfloat162 lo = __floats2bfloat162_rn(x.x, x.y), hi = __floats2bfloat162_rn(x.z, x.w);
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t *>(&lo);
        pk.y = *reinterpret_cast<uint32_t *>(&hi);
        *reinterpret_cast<uint2 *>(sA + canon_off(r, k, Kp)) = pk;
      }
    } else {
      for (int e = tid; e < TM * (Kp / 2); e += TT) {
        const int r = e / (Kp / 2), k = (e % (Kp / 2)) * 2;
        const int m = m0 + r;
        float x0 = 0.f, x1 = 0.f;
        if (m < a.M) {
          if (k < a.K) x0 = (k < a.K1) ? a.X1[(size_t)m * a.ldx1 + k] : a.X2[(size_t)m * a.ldx2 + (k - a.K1)];
          if (k + 1 < a.K)
            x1 = (k + 1 < a.K1) ? a.X1[(size_t)m * a.ldx1 + k + 1] : a.X2[(size_t)m * a.ldx2 + (k + 1 - a.K1)];
        }
        *reinterpret_cast<__nv_bfloat162 *>(sA + canon_off(r, k, Kp)) = __floats2bfloat162_rn(x0, x1);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> async proxy
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int ks = 0; ks < Kp / 16; ks++) {
        const uint64_t ad = make_desc(aBase + ks * 256, 128, sbo);
        const uint64_t bd = make_desc(bBase + ks * 256, 128, sbo);
        const uint32_t acc = ks > 0 ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&mbar))
                   : "memory");
    }
    // wait for the accumulator
    {
      uint32_t done = 0;
      while (!done) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.b32 %0, 1, 0, P1;\n\t}\n"
            : "=r"(done)
            : "r"(smem_u32(&mbar)), "r"(phase));
      }
      phase ^= 1;
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // epilogue: thread = row; warp w drains TMEM lanes 32 (w % 4) ..; warpgroup w / 4 takes half the columns
    const int quarter = warp & 3, wg = warp >> 2;
    const int m = m0 + quarter * 32 + lane;
    const int half = ((Np / 8 + 1) / 2) * 8;
    for (int c0 = wg * half; c0 < min(Np, (wg + 1) * half); c0 += 8) {
      uint32_t v[8];
      const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (m >= a.M) continue;
      float x[8];
      if (vec_epi && c0 + 8 <= a.Nout) {   // full 8-column chunk: 16-byte loads of mask and residual
        float mk[8], rr[8];
        if (a.epi == EPI_MASK) {
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
          if (a.epi == EPI_MASK) y = mk[j] > 0.f ? y : 0.f;
          else y = epi_apply(a.epi, y);
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
            if (a.epi == EPI_MASK) y = a.aux[(size_t)m * a.ldaux + n] > 0.f ? y : 0.f;
            else y = epi_apply(a.epi, y);
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
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();   // sA and the TMEM accumulator are reused by the next tile
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols));
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

}  // namespace

bool tc_eligible(const GemmArgs &a) {
  return a.Nout >= 16 && a.Nout <= 256 && a.K >= 1 && a.K <= 256 && a.M >= TM;
}

void launch_gemm_tc(const GemmArgs &a, cudaStream_t s) {
  const int Kp = (a.K + 15) / 16 * 16;
  const int Np = (a.Nout + 15) / 16 * 16;
  int ncols = 32;
  while (ncols < Np) ncols <<= 1;
  const size_t smem = (size_t)(TM + Np) * Kp * 2;
  static bool configured = false;   // largest tile: (128 + 256) x 256 bf16 = 192 KB
  if (!configured) {
    cudaFuncSetAttribute(k_gemm_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  // as many resident CTAs per SM as shared memory (and TMEM columns: 512 per SM) allow, up to 4,
  // so that more 128-row tiles have their loads in flight at once
  const int ntiles = (a.M + TM - 1) / TM;
  int per_sm = (int)((227 * 1024) / (smem + 2048));
  per_sm = per_sm < 512 / ncols ? per_sm : 512 / ncols;
  per_sm = per_sm < 4 ? (per_sm < 1 ? 1 : per_sm) : 4;
  const int slots = per_sm * num_sms();
  const int grid = ntiles < slots ? ntiles : slots;
  note_launch("k_gemm_tc", s, gemm_bytes(a), 2.0 * a.M * a.K * a.Nout);
  k_gemm_tc<<<grid, TT, smem, s>>>(a, Kp, Np, ncols);
}

}  // namespace gdp
