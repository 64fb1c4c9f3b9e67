// Shared PTX helpers of the tcgen05 kernels (tc_gemm.cu, attn_tc.cu): shared-window addresses,
// UMMA shared-memory descriptors, mbarriers, TMEM loads.
#pragma once
#include <cuda.h>
#include <stdint.h>

namespace gdp {
namespace tc {

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// UMMA shared-memory descriptor, K-major SWIZZLE_NONE (8-row x 16-byte core matrices; lbo = next
// core matrix along K, sbo = next 8-row group), Blackwell descriptor version 1
__device__ __forceinline__ uint64_t desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// K-major SWIZZLE_128B: rows of 128 bytes, 16-byte granule g of row r stored at g ^ (r & 7),
// 8-row groups 1024 bytes apart (sbo); the tile base is 1024-byte aligned.  A K step inside the
// 128-byte row is a start-address offset.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                 // lbo (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;       // sbo
  d |= (uint64_t)1 << 46;                 // version
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}
// element (row r, col k) of a canonical K-major SWIZZLE_NONE bf16 tile with Kp columns
__device__ __forceinline__ uint32_t canon_off(int r, int k, int Kp) {
  return (uint32_t)(((r >> 3) * (Kp >> 3) + (k >> 3)) * 128 + (r & 7) * 16 + (k & 7) * 2);
}

__device__ __forceinline__ void mbar_init(uint64_t *mb, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(mb)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t *mb, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                 "selp.b32 %0, 1, 0, P1;\n\t}\n"
                 : "=r"(done)
                 : "r"(su32(mb)), "r"(ph)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *mb) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(mb)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *mb, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(mb)), "r"(bytes) : "memory");
}
// tcgen05.commit: the mbarrier completes when every MMA this thread issued before it has
__device__ __forceinline__ void mma_commit(uint64_t *mb) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(mb))
               : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t *v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// TMA: one 2-D box of `map` at (column x, row y) into shared memory, completing on mbarrier mb
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int x, int y, uint64_t *mb) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(su32(mb))
      : "memory");
}

// host: 2-D fp32 tensor map over rows x cols (row stride ld floats), box brows rows x 32 columns
// (128 bytes), SWIZZLE_128B (16-byte granule g of row r at g ^ (r % 8)) or, with atom32,
// SWIZZLE_128B_ATOM_32B (32-byte granule g of row r at g ^ (r % 4): the only MN-major layout the
// tf32 MMA takes); out-of-range rows / columns read as zero and are not written.  False if TMA
// cannot take the tensor (alignment) or the driver entry point is missing.
bool tma_map_f32(CUtensorMap *m, const float *base, int cols, int rows, int ld, int brows, bool atom32 = false);

}  // namespace tc
}  // namespace gdp
