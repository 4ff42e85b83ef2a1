// ptx.cuh — thin inline-PTX wrappers for sm_100a: mbarrier, TMA, tcgen05/TMEM.
// Encodings follow the PTX ISA for sm_100a (field layouts cross-checked against
// the CUTLASS 4.x headers vendored in the image, used as an encoding reference only).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

namespace ctm {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------------- TMA
// Bulk prefetch of `bytes` (multiple of 16, 16-B aligned) from global memory into L2.
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<uint64_t>(p)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
// 2D tile load global -> shared, completion counted on `bar` (bytes).
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* m, uint64_t* bar, int32_t c0,
                                            int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// 3D tile load (coordinates {c0 inner, c1 rows, c2 plane}), pair form: bytes land in this
// CTA's smem, completion counted on the leader's mbarrier (see tma_load_2d_pair).
__device__ __forceinline__ void tma_load_3d_pair(void* smem_dst, const CUtensorMap* m, uint64_t* bar, int32_t c0,
                                                 int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// 3D tile load into this CTA's smem, completion on this CTA's mbarrier.
__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* m, uint64_t* bar, int32_t c0,
                                            int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// ---------------------------------------------------------------- clusters (CTA pairs)
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
// arrive on the mbarrier at the same smem offset in CTA `cta` of the cluster
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
      "r"(cta)
      : "memory");
}
// Pair TMA load: the bytes land in THIS CTA's smem, the completion is counted on the
// mbarrier at the same offset in the pair's leader (rank 0) -- peer bit 24 cleared.
__device__ __forceinline__ void tma_load_2d_pair(void* smem_dst, const CUtensorMap* m, uint64_t* bar, int32_t c0,
                                                 int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1)
      : "memory");
}

// ---------------------------------------------------------------- tcgen05 / TMEM
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_result) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_result)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// Pair variants (cta_group::2): allocation by the same warp in both CTAs; the MMA is
// issued by the leader only, D spans both CTAs' TMEM (M = 256), A and B halves are read
// from both CTAs' smem at the same offsets.
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* smem_result) {  // whole warp, both CTAs
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_result)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr) {  // whole warp, both CTAs
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}
__device__ __forceinline__ void mma_bf16_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D = A * B + D * 2^-11 (tcgen05.mma's scale-input-d, kind::f16): the fp16x3 weight
// gradients' first p0*p0 MMA of a chunk takes the accumulator of the lifted correction
// products (p1 carries 2^11) down to the scale of the main product, so no lifted third
// plane of an activation block is needed
__device__ __forceinline__ void mma_f16_pair_unlift(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p, 11;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(1u)
      : "memory");
}
// One lane of a converged warp (elect.sync): issue single-thread instructions (tcgen05.mma,
// commits) from converged code so their operands stay in uniform registers (no per-MMA
// R2UR waterfall loop of a divergent lane-0 branch).
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
// Arrive on the mbarrier at this offset in both CTAs of the pair once the MMAs complete.
// A from tensor memory ("TS"): A is read from this CTA's TMEM columns at a_tmem (128 lanes
// x K=16 bf16 = 8 columns), B from shared memory as in mma_bf16_pair.
__device__ __forceinline__ void mma_bf16_pair_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                                 uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// shared memory -> tensor memory copy of a 128-row x 32-byte operand slice (both CTAs of
// the pair, each from its own shared memory at the descriptor's offset)
__device__ __forceinline__ void tmem_cp_128x256b_pair(uint32_t taddr, uint64_t s_desc) {
  asm volatile("tcgen05.cp.cta_group::2.128x256b [%0], %1;" ::"r"(taddr), "l"(s_desc) : "memory");
}
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}

// Arrive on `bar` once all previously issued tcgen05.mma of this thread complete.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
// one column (32 lanes x 32 bit); any column offset is legal (scripts/microtests/tmem_align.cu)
__device__ __forceinline__ float tmem_ld1(uint32_t taddr) {
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
  return __uint_as_float(r);
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld2(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(taddr));
}
// 32 lanes x 32 bit, 32 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
// N consecutive columns into v[0..N), composed at compile time from x16/x8/x4/x2/x1
// loads (no column past N is touched). Needs tmem_ld_wait() before v is read.
template <int N>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, float* v) {
  if constexpr (N >= 16) {
    tmem_ld16(taddr, v);
    tmem_ld_cols<N - 16>(taddr + 16u, v + 16);
  } else if constexpr (N >= 8) {
    tmem_ld8(taddr, v);
    tmem_ld_cols<N - 8>(taddr + 8u, v + 8);
  } else if constexpr (N >= 4) {
    tmem_ld4(taddr, v);
    tmem_ld_cols<N - 4>(taddr + 4u, v + 4);
  } else if constexpr (N >= 2) {
    tmem_ld2(taddr, v);
    tmem_ld_cols<N - 2>(taddr + 2u, v + 2);
  } else if constexpr (N == 1) {
    v[0] = tmem_ld1(taddr);
  }
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor (tcgen05 "matrix descriptor"), K-major operand:
//  bits [0,14) start address >> 4; [16,30) leading byte offset >> 4 (unused for
//  swizzled K-major, set to 1); [32,46) stride byte offset >> 4 (distance between
//  8-row core-matrix groups); [46,48) version = 1 (sm_100); [49,52) base offset = 0;
//  [52] lbo mode = 0; [61,64) layout: 0 none, 2 SW128, 4 SW64, 6 SW32.
__device__ __forceinline__ uint64_t smem_desc_kmajor(uint32_t smem_addr, uint32_t sbo_bytes, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)(layout & 0x7u) << 61;
  return d;
}

// MN-major operand (the M or N index contiguous in memory, K strided), SWIZZLE_128B: atoms
// of 64 bf16 (128 bytes, MN) x 8 rows (K); `lbo_bytes` = distance between consecutive
// 64-element MN atoms, `sbo_bytes` = distance between consecutive 8-row K groups (CuTe's
// canonical MN-major SW128 layout ((8,n),(8,k)):((1,LBO),(8,SBO)) in 16-byte units).
__device__ __forceinline__ uint64_t smem_desc_mn(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;  // SWIZZLE_128B
  return d;
}

// Instruction descriptor, kind::f16 with BF16 A/B, fp32 accumulate, both K-major:
//  [4,6) D format (1 = f32); [7,10) A format (1 = bf16); [10,13) B format (1 = bf16);
//  [15] A major (0 = K); [16] B major (0 = K); [17,23) N >> 3; [24,29) M >> 4.
// kind::f16 with fp16 A and B (formats 0), fp32 accumulate: the fp16x3 mode
__host__ __device__ constexpr uint32_t idesc_f16(uint32_t M, uint32_t N) {
  return (1u << 4) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
__host__ __device__ constexpr uint32_t idesc_bf16(uint32_t M, uint32_t N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
// fp16 operands, both MN-major (the fp16x3 weight gradients)
__host__ __device__ constexpr uint32_t idesc_f16_mn(uint32_t M, uint32_t N) {
  return idesc_f16(M, N) | (1u << 15) | (1u << 16);
}
// The same with both operands MN-major (bits 15 and 16).
__host__ __device__ constexpr uint32_t idesc_bf16_mn(uint32_t M, uint32_t N) {
  return idesc_bf16(M, N) | (1u << 15) | (1u << 16);
}

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 inputs, K = 16), one CTA; ONE thread.
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// bf16 plane split of an fp32 value: p0 = rn_bf16(v), p1 = rn_bf16(v - p0),
// p2 = rn_bf16(v - p0 - p1); each difference is exact in fp32. Three planes hold all 24
// bits of v (p0 + p1 + p2 = v up to 2^-27 |v|); the fast mode stores only p0 and p1 (~17 bits).
__device__ __forceinline__ void bf16_split3(float v, uint16_t& p0, uint16_t& p1, uint16_t& p2) {
  const __nv_bfloat16 h = __float2bfloat16_rn(v);
  const float r = v - __bfloat162float(h);
  const __nv_bfloat16 m = __float2bfloat16_rn(r);
  const __nv_bfloat16 l = __float2bfloat16_rn(r - __bfloat162float(m));
  p0 = __bfloat16_as_ushort(h);
  p1 = __bfloat16_as_ushort(m);
  p2 = __bfloat16_as_ushort(l);
}
// The value's first nplanes planes at p, p + pstride (, p + 2 pstride) (the third plane
// is only computed when stored).
__device__ __forceinline__ void store_planes(uint16_t* p, int64_t pstride, int nplanes, float v) {
  const __nv_bfloat16 h = __float2bfloat16_rn(v);
  const float r = v - __bfloat162float(h);
  const __nv_bfloat16 m = __float2bfloat16_rn(r);
  p[0] = __bfloat16_as_ushort(h);
  p[pstride] = __bfloat16_as_ushort(m);
  if (nplanes > 2) p[2 * pstride] = __bfloat16_as_ushort(__float2bfloat16_rn(r - __bfloat162float(m)));
}
// The same with the plane count known at compile time (the layer epilogues: no per-store
// load and test of the count; S=8 / S=32 layers 1.5-2.5% faster)
template <int NPL>
__device__ __forceinline__ void store_planes(uint16_t* p, int64_t pstride, float v) {
  static_assert(NPL == 2 || NPL == 3, "planes");
  const __nv_bfloat16 h = __float2bfloat16_rn(v);
  const float r = v - __bfloat162float(h);
  const __nv_bfloat16 m = __float2bfloat16_rn(r);
  p[0] = __bfloat16_as_ushort(h);
  p[pstride] = __bfloat16_as_ushort(m);
  if (NPL > 2) p[2 * pstride] = __bfloat16_as_ushort(__float2bfloat16_rn(r - __bfloat162float(m)));
}
// The same with the three plane bases of a point precomputed and a 32-bit element offset,
// so each store's address is one wide multiply-add instead of 64-bit pointer arithmetic per
// plane (fewer integer instructions per output; same-box A/B: layer times unchanged within
// noise, the S=8 epilogue is latency- rather than issue-bound).
template <int NPL>
__device__ __forceinline__ void store_planes_off(uint16_t* q0, uint16_t* q1, uint16_t* q2, uint32_t off, float v) {
  static_assert(NPL == 2 || NPL == 3, "planes");
  const __nv_bfloat16 h = __float2bfloat16_rn(v);
  const float r = v - __bfloat162float(h);
  const __nv_bfloat16 m = __float2bfloat16_rn(r);
  q0[off] = __bfloat16_as_ushort(h);
  q1[off] = __bfloat16_as_ushort(m);
  if (NPL > 2) q2[off] = __bfloat16_as_ushort(__float2bfloat16_rn(r - __bfloat162float(m)));
}
// fp16x3 planes: vs = v * scale (a power of two chosen so |vs| <= 2^14),
// p0 = rn_f16(vs), p1 = rn_f16((vs - p0) * 2^11): 22 significant bits (the difference is
// exact in fp32); the residual plane is lifted by 2^11 so it is subnormal only where p0 is,
// which keeps both planes an exact power-of-two multiple of those of v (results do not depend
// on the block's scale, hence not on how a batch is split). q0/q1 are the plane bases, off a
// 32-bit element offset.
constexpr float kF16Lift = 2048.f;
__device__ __forceinline__ void f16_split(float vs, uint16_t& p0, uint16_t& p1) {
  const __half h = __float2half_rn(vs);
  p0 = __half_as_ushort(h);
  p1 = __half_as_ushort(__float2half_rn((vs - __half2float(h)) * kF16Lift));
}
__device__ __forceinline__ void store_f16_off(uint16_t* q0, uint16_t* q1, uint32_t off, float vs) {
  uint16_t a, b;
  f16_split(vs, a, b);
  q0[off] = a;
  q1[off] = b;
}
// Programmatic dependent launch: the next kernel in the stream may start its prologue
// once every CTA of this grid has called launch_dependents (or exited); wait_prior blocks
// until the previous grid has completed and its memory is visible.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait_prior() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ float bf16_val(uint16_t b) { return __bfloat162float(__ushort_as_bfloat16(b)); }
// the value of an fp16x3 element (two planes, the residual lifted by 2^11), still scaled
__device__ __forceinline__ float f16_val(const uint16_t* p, int64_t pstride) {
  return __half2float(__ushort_as_half(p[pstride])) * (1.f / kF16Lift) + __half2float(__ushort_as_half(p[0]));
}
// the fp32 value of a plane-split element (sum of its planes, small first)
__device__ __forceinline__ float planes_val(const uint16_t* p, int64_t pstride, int nplanes) {
  float v = nplanes > 2 ? bf16_val(p[2 * pstride]) : 0.f;
  v += bf16_val(p[pstride]);
  return v + bf16_val(p[0]);
}

}  // namespace ptx
}  // namespace ctm
