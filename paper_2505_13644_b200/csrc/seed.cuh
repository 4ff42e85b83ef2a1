// seed.cuh — layer 1 of the collapsed jet (steps a1 + a2 + a3 of SURVEY §8(a)),
// the per-call direction preparation, and the readout (a5).
//
// FIXED direction sets: layer 1 needs no tensor cores: z0 = W1 x0 + b1 is a D-term dot
// product per feature and the first-order coefficients z_{1,r} = (W1 V)[:, r] are the
// same for every point, precomputed once (U^T [R, ld]). The kernel is bound by the HBM
// write of the layer-1 block.
// RANDOM directions: the per-point directions make layer 1 a real contraction
// [N(S+2), D] x [D, w1]; seed_random_kernel only writes the input block and layer 1
// runs on the tensor cores (jet_layer.cuh).
#pragma once
#include <cstdint>

#include "jet_layer.cuh"  // ActD, F16Rec, f16_scale_for
#include "ptx.cuh"

namespace ctm {

constexpr int kSeedThreads = 256;
constexpr int kSeedChunk = 4096;  // floats of directions staged in smem per pass

// splitmix64 finaliser of seed + (idx+1) * golden gamma
__device__ __forceinline__ uint64_t splitmix64(uint64_t seed, uint64_t idx) {
  uint64_t z = seed + (idx + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct SeedParams {
  const float* X;        // [N, D]
  int D;
  int64_t n_points;
  const float* W1T;      // [D, ld]   (W1 transposed, zero padded columns)
  const float* b1;       // [ld]
  int ld;                // padded width of layer 1 (= output ld)
  int P;                 // slots per sub-point (one direction block)
  // FIXED directions: z1_r = UT[r, m]; csum[b * ld + m] = the sum over the directions r of
  // block b of z1_r^2 (K=2) or w_r z1_r^4 (K=4)
  const float* UT;       // [R, ld]
  const float* csum;     // [blocks, ld]
  int R;                 // K=2: number of directions; K=4: number of jets J
  int blocks;            // direction blocks per point (jet_layer.cuh, LayerParams::blocks)
  int rb;                // directions (K=4: jets) per block; the last block is zero padded
  uint16_t* out;         // [nplanes][N*blocks*P, ld] bf16 planes
  int64_t pstride;       // elements between planes
  int nplanes;
  int act;               // kAct*
  float* z_out;          // K=2, grad mode (one block): pre-activations [N*P, ld] (z0, W1 u_r, 0) or nullptr
};
// fp16x3 mode of seed_fixed_kernel (a parameter of its own: growing SeedParams made ptxas
// spill in seed_layer_kernel<4, 3>): bounds [max |U|, max |csum|] (float bits) of this call's
// direction images, the sups of |s| and its first four derivatives, the layer-1 block's record
struct SeedF16 {
  const unsigned* bounds;
  float s0, s1, s2, s3, s4;
  F16Rec* out;
  int uniform;  // grad mode: one scale for all slot types (the weight gradients contract over rows)
};

// Where a kernel writes its bf16 planes: plane k of element i at base[k * pstride + i].
struct PlaneOut {
  uint16_t* base;
  int64_t pstride;
  int nplanes;
};

// four adjacent features -> one 8-byte store into each of the NP planes (plane by plane,
// so only the four residuals stay live: the seed kernels run at 40-48 registers)
template <int NP>
__device__ __forceinline__ void seed_store4_at(uint16_t* dst, int64_t pstride, float a, float b, float c, float d) {
  float r[4] = {a, b, c, d};
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    // packed round-to-nearest conversions (one F2FP per pair, the same bits as two scalar
    // cvt.rn.bf16.f32) and the residuals exact in fp32
    const __nv_bfloat162 lo = __floats2bfloat162_rn(r[0], r[1]), hi = __floats2bfloat162_rn(r[2], r[3]);
    if (k + 1 < NP) {
      const float2 fl = __bfloat1622float2(lo), fh = __bfloat1622float2(hi);
      r[0] -= fl.x;
      r[1] -= fl.y;
      r[2] -= fh.x;
      r[3] -= fh.y;
    }
    *reinterpret_cast<uint2*>(dst) =
        make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
    dst += pstride;
  }
}
template <int NP>
__device__ __forceinline__ void seed_store4(const PlaneOut& o, size_t idx, float a, float b, float c, float d) {
  seed_store4_at<NP>(o.base + idx, o.pstride, a, b, c, d);
}

// fp16x3 mode (jet_layer.cuh kFlagF16): four adjacent ALREADY SCALED features x = v * sc as
// two fp16 planes, p0 = rn_f16(x), p1 = rn_f16((x - p0) * 2^11) (ptx::f16_split, packed)
__device__ __forceinline__ void seed_store4_f16s(uint16_t* dst, int64_t pstride, float x0, float x1, float x2,
                                                 float x3) {
  const __half2 h01 = __floats2half2_rn(x0, x1), h23 = __floats2half2_rn(x2, x3);
  const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
  const __half2 l01 = __floats2half2_rn((x0 - f01.x) * ptx::kF16Lift, (x1 - f01.y) * ptx::kF16Lift);
  const __half2 l23 = __floats2half2_rn((x2 - f23.x) * ptx::kF16Lift, (x3 - f23.y) * ptx::kF16Lift);
  *reinterpret_cast<uint2*>(dst) =
      make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
  *reinterpret_cast<uint2*>(dst + pstride) =
      make_uint2(*reinterpret_cast<const uint32_t*>(&l01), *reinterpret_cast<const uint32_t*>(&l23));
}
// (unscaled values: scales them first; the per-element products v * sc are exact)
__device__ __forceinline__ void seed_store4_f16(const PlaneOut& o, size_t idx, float a, float b, float c, float d,
                                                float sc) {
  seed_store4_f16s(o.base + idx, o.pstride, a * sc, b * sc, c * sc, d * sc);
}
__device__ __forceinline__ float max4abs(float a, float b, float c, float d) {
  return fmaxf(fmaxf(fabsf(a), fabsf(b)), fmaxf(fabsf(c), fabsf(d)));
}
// max |v| of a warp's values into a block record (float bits; all lanes call)
__device__ __forceinline__ void warp_max_record(float v, unsigned* dst) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0 && v > 0.f) atomicMax(dst, __float_as_uint(v));
}

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

// Fixed direction sets (K=2: e_d or sigma columns; K=4: the biharmonic family).
// grid: one block per (point, 4*blockDim-feature chunk); each thread owns 4 adjacent
// features, so loads are float4 and the bf16-pair stores are 8 bytes wide. Direction
// block b of the point gets its own slot group [h0; its directions; its partial top], with
// zero rows for the padding of the last block.
template <int KORD, int NP, bool F16 = false>
// (min blocks per SM: the register budget of the single-block kernel, which this store-bound
// kernel needs for its occupancy: 40 registers for K=2 / standard, 48 for K=4 / nested)
// F16 (kNest only): the fp16x3 planes of the nested block with ONE scale (every slot type),
// from the bounds U = max|U| = f.bounds[0], C = max|csum| = f.bounds[1] (C = max |g|^2):
// |h0| <= s0, |g| <= s1 U, |H| <= s2 U^2, |L| <= s3 U C, |Q| <= s4 C^2; the block's record
// holds the max |value| over all slots in maxabs[0] (jet_layer.cuh f16_nest_scales)
__global__ void __launch_bounds__(kSeedThreads, (KORD == 2 || KORD == kStd2) ? 6 : 5)
    seed_layer_kernel(const SeedParams p, const SeedF16 f = {}) {
  const PlaneOut o{p.out, p.pstride, p.nplanes};
  static_assert(!F16 || ((KORD == kNest || KORD == kStd2 || KORD == kStd4) && NP == 2),
                "fp16x3 seed_layer_kernel: the nested block and the standard modes");
  // fp16x3, standard modes: per slot type from U = max|U| = f.bounds[0]: primal s0 (type 0),
  // h1 = s' u <= s1 U (1), h2 = s'' u^2 <= s2 U^2 (kStd2: 2, kStd4: 3), h3 <= s3 U^3 (4),
  // h4 <= s4 U^4 (2)
  float sos[kF16Types], smx[kF16Types];
#pragma unroll
  for (int t2 = 0; t2 < kF16Types; ++t2) sos[t2] = 1.f, smx[t2] = 0.f;
  if constexpr (F16 && KORD != kNest) {
    const float U = __uint_as_float(f.bounds[0]);
    sos[0] = f16_scale_for(f.s0);
    sos[1] = f16_scale_for(f.s1 * U);
    if (KORD == kStd2) {
      sos[2] = f16_scale_for(f.s2 * U * U);
    } else {
      sos[3] = f16_scale_for(f.s2 * U * U);
      sos[4] = f16_scale_for(f.s3 * U * U * U);
      sos[2] = f16_scale_for(f.s4 * U * U * U * U);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0)
      for (int t2 = 0; t2 < kF16Types; ++t2) f.out->scale[t2] = sos[t2];
  }
  auto put4t = [&](size_t idx, float a, float b, float c, float d, int type) {
    if constexpr (F16 && KORD != kNest) {
      seed_store4_f16(o, idx, a, b, c, d, sos[type]);
      smx[type] = fmaxf(smx[type], max4abs(a, b, c, d));
    } else {
      seed_store4<NP>(o, idx, a, b, c, d);
    }
  };
  const int feats = 4 * blockDim.x;
  const int mchunks = (p.ld + feats - 1) / feats;
  const int64_t n = blockIdx.x / mchunks;
  const int m = (blockIdx.x % mchunks) * feats + 4 * threadIdx.x;
  if (m >= p.ld) return;  // ld is a multiple of 128: a thread's 4 features are all in or all out
  const float* x = p.X + n * p.D;  // every thread reads the same x_d: a broadcast load
  float4 z0 = ldg4(p.b1 + m);
  for (int d = 0; d < p.D; ++d) {
    const float4 w = ldg4(p.W1T + (size_t)d * p.ld + m);
    const float xd = __ldg(x + d);
    z0.x = fmaf(w.x, xd, z0.x);
    z0.y = fmaf(w.y, xd, z0.y);
    z0.z = fmaf(w.z, xd, z0.z);
    z0.w = fmaf(w.w, xd, z0.w);
  }
  const float zz[4] = {z0.x, z0.y, z0.z, z0.w};
  float t[4], d1[4], d2[4], d3[4], d4[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const ActD A = act_derivs(p.act, zz[i]);  // s, s', s'', s''', s''''
    t[i] = A.d0; d1[i] = A.d1; d2[i] = A.d2; d3[i] = A.d3; d4[i] = A.d4;
  }
  // one loop over the blocks per rule, so each rule keeps only its own derivatives live
  // (the K=2 loop runs at the register count, and occupancy, of a single-block kernel)
#define CTM_BLOCK_BEGIN                                                  \
  for (int b = 0; b < p.blocks; ++b) {                                   \
    const size_t row0 = ((size_t)n * p.blocks + b) * p.P;                \
    const int r0 = b * p.rb;                                             \
    const int r1 = (r0 + p.rb < p.R) ? r0 + p.rb : p.R;                  \
    put4t(row0 * p.ld + m, t[0], t[1], t[2], t[3], 0);
#define CTM_BLOCK_END }
  if (KORD == kStd2) {
    CTM_BLOCK_BEGIN
    // standard mode: per direction (h1_r, h2_r) = (tanh' z1, tanh'' z1^2)   (x2 = 0)
    auto pair = [&](const float4 u, int r) {
      const size_t rr = row0 + 1 + 2 * (r - r0);
      put4t(rr * p.ld + m, d1[0] * u.x, d1[1] * u.y, d1[2] * u.z, d1[3] * u.w, 1);
      put4t((rr + 1) * p.ld + m, d2[0] * u.x * u.x, d2[1] * u.y * u.y, d2[2] * u.z * u.z, d2[3] * u.w * u.w, 2);
    };
    int r = r0;
#ifndef CTM_SEED_BATCHS
#define CTM_SEED_BATCHS 8
#endif
    for (; r + CTM_SEED_BATCHS <= r1; r += CTM_SEED_BATCHS) {  // U^T loads in flight together
      float4 u[CTM_SEED_BATCHS];
#pragma unroll
      for (int i = 0; i < CTM_SEED_BATCHS; ++i) u[i] = ldg4(p.UT + (size_t)(r + i) * p.ld + m);
#pragma unroll
      for (int i = 0; i < CTM_SEED_BATCHS; ++i) pair(u[i], r + i);
    }
    for (; r < r0 + p.rb; ++r)
      pair((r < r1) ? ldg4(p.UT + (size_t)r * p.ld + m) : make_float4(0.f, 0.f, 0.f, 0.f), r);
    CTM_BLOCK_END
  } else if (KORD == kStd4) {
    CTM_BLOCK_BEGIN
    // standard K=4 mode: per jet (h1, h2, h3, h4) = (s' u, s'' u^2, s''' u^3, s'''' u^4)  (x2 = x3 = x4 = 0)
    for (int j = r0; j < r0 + p.rb; ++j) {
      const float4 u = (j < r1) ? ldg4(p.UT + (size_t)j * p.ld + m) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float z[4] = {u.x, u.y, u.z, u.w};
      float h[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float z2 = z[i] * z[i];
        h[0][i] = d1[i] * z[i];
        h[1][i] = d2[i] * z2;
        h[2][i] = d3[i] * z2 * z[i];
        h[3][i] = d4[i] * z2 * z2;
      }
      const size_t r = row0 + 1 + 4 * (j - r0);
      constexpr int kType[4] = {1, 3, 4, 2};  // h1, h2, h3, h4
#pragma unroll
      for (int k = 0; k < 4; ++k) put4t((r + k) * p.ld + m, h[k][0], h[k][1], h[k][2], h[k][3], kType[k]);
    }
    CTM_BLOCK_END
  } else if (KORD == 2) {
    if (p.z_out) {  // grad mode (one block): the layer-1 pre-activations for the backward pass
      const size_t row0 = (size_t)n * p.P;
      *reinterpret_cast<float4*>(p.z_out + row0 * p.ld + m) = z0;
      for (int r = 0; r < p.R; ++r)
        *reinterpret_cast<float4*>(p.z_out + (row0 + 1 + r) * p.ld + m) = ldg4(p.UT + (size_t)r * p.ld + m);
      *reinterpret_cast<float4*>(p.z_out + (row0 + 1 + p.R) * p.ld + m) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    CTM_BLOCK_BEGIN
    int r = r0;
// batches of 8 rows: 8 loads of U^T in flight per thread (the loads, not the stores, bound
// this loop -- ncu: 42% of stall samples at the first use of a U^T value; C1 seed
// 0.60-0.62 -> 0.50-0.54 ms against batches of 4; 16 ran out of registers under the
// launch bound and was slower)
#ifndef CTM_SEED_BATCH
#define CTM_SEED_BATCH 8
#endif
    for (; r + CTM_SEED_BATCH <= r1; r += CTM_SEED_BATCH) {
      float4 u[CTM_SEED_BATCH];
#pragma unroll
      for (int i = 0; i < CTM_SEED_BATCH; ++i) u[i] = ldg4(p.UT + (size_t)(r + i) * p.ld + m);
#pragma unroll
      for (int i = 0; i < CTM_SEED_BATCH; ++i)
        seed_store4<NP>(o, (row0 + 1 + r - r0 + i) * p.ld + m, d1[0] * u[i].x, d1[1] * u[i].y,
                    d1[2] * u[i].z, d1[3] * u[i].w);
    }
    for (; r < r1; ++r) {
      const float4 u = ldg4(p.UT + (size_t)r * p.ld + m);
      seed_store4<NP>(o, (row0 + 1 + r - r0) * p.ld + m, d1[0] * u.x, d1[1] * u.y, d1[2] * u.z,
                  d1[3] * u.w);
    }
    for (; r < r0 + p.rb; ++r) seed_store4<NP>(o, (row0 + 1 + r - r0) * p.ld + m, 0.f, 0.f, 0.f, 0.f);
    // sum h2 = tanh' * 0 + tanh'' * sum_r z1_r^2   (the input top coefficient is 0)
    const float4 cs = ldg4(p.csum + (size_t)b * p.ld + m);
    seed_store4<NP>(o, (row0 + 1 + p.rb) * p.ld + m, d2[0] * cs.x, d2[1] * cs.y, d2[2] * cs.z,
                d2[3] * cs.w);
    CTM_BLOCK_END
  } else if (KORD == kNest) {
    // nested biharmonic, layer 1 (one block): g_a = W1[:, a] = UT[a] and H = L = Q = 0 at
    // the input, so h_a = s' g_a, H'_ab = s'' g_a g_b, L'_a = s''' g_a |g|^2,
    // Q' = s'''' |g|^4 (the epilogue rule of jet_layer.cuh with H = L = Q = 0); |g|^2 = csum.
    float os = 1.f, mx = 0.f;
    if constexpr (F16) {
      const float U = __uint_as_float(f.bounds[0]), C = __uint_as_float(f.bounds[1]);
      os = f16_scale_for(fmaxf(fmaxf(f.s0, f.s1 * U), fmaxf(f.s2 * U * U, fmaxf(f.s3 * U * C, f.s4 * C * C))));
      if (blockIdx.x == 0 && threadIdx.x == 0)
        for (int t2 = 0; t2 < kF16Types; ++t2) f.out->scale[t2] = os;
    }
    auto putn = [&](size_t idx, float a, float b, float c, float d) {
      if constexpr (F16) {
        seed_store4_f16(o, idx, a, b, c, d, os);
        mx = fmaxf(mx, max4abs(a, b, c, d));
      } else {
        seed_store4<NP>(o, idx, a, b, c, d);
      }
    };
    const size_t row0 = (size_t)n * p.P;
    putn(row0 * p.ld + m, t[0], t[1], t[2], t[3]);
    const float4 cs = ldg4(p.csum + m);
    size_t r = row0 + 1;
    for (int a = 0; a < p.R; ++a, ++r) {
      const float4 u = ldg4(p.UT + (size_t)a * p.ld + m);
      putn(r * p.ld + m, d1[0] * u.x, d1[1] * u.y, d1[2] * u.z, d1[3] * u.w);
    }
    for (int a = 0; a < p.R; ++a) {
      const float4 ua = ldg4(p.UT + (size_t)a * p.ld + m);
      for (int c = a; c < p.R; ++c, ++r) {
        const float4 uc = ldg4(p.UT + (size_t)c * p.ld + m);
        putn(r * p.ld + m, d2[0] * ua.x * uc.x, d2[1] * ua.y * uc.y, d2[2] * ua.z * uc.z, d2[3] * ua.w * uc.w);
      }
    }
    for (int a = 0; a < p.R; ++a, ++r) {
      const float4 u = ldg4(p.UT + (size_t)a * p.ld + m);
      putn(r * p.ld + m, d3[0] * u.x * cs.x, d3[1] * u.y * cs.y, d3[2] * u.z * cs.z, d3[3] * u.w * cs.w);
    }
    putn(r * p.ld + m, d4[0] * cs.x * cs.x, d4[1] * cs.y * cs.y, d4[2] * cs.z * cs.z, d4[3] * cs.w * cs.w);
    if constexpr (F16) warp_max_record(mx, &f.out->maxabs[0]);
  } else {
    CTM_BLOCK_BEGIN
    auto jet = [&](const float4 u, int j) {
      const float z[4] = {u.x, u.y, u.z, u.w};
      float h1[4], h2[4], h3[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        h1[i] = d1[i] * z[i];                       // h1
        h2[i] = d2[i] * z[i] * z[i];                // h2 (z2 = 0)
        h3[i] = d3[i] * z[i] * z[i] * z[i];         // h3 (z2 = z3 = 0)
      }
      const size_t r = row0 + 1 + 3 * (j - r0);
      seed_store4<NP>(o, r * p.ld + m, h1[0], h1[1], h1[2], h1[3]);
      seed_store4<NP>(o, (r + 1) * p.ld + m, h2[0], h2[1], h2[2], h2[3]);
      seed_store4<NP>(o, (r + 2) * p.ld + m, h3[0], h3[1], h3[2], h3[3]);
    };
    int j = r0;
#ifndef CTM_SEED_BATCH4
#define CTM_SEED_BATCH4 8
#endif
    // batches of 8 jets: their U^T loads in flight together (as the K=2 loop above;
    // C4 seed 1.07 -> 0.97 ms)
    for (; j + CTM_SEED_BATCH4 <= r1; j += CTM_SEED_BATCH4) {
      float4 u[CTM_SEED_BATCH4];
#pragma unroll
      for (int i = 0; i < CTM_SEED_BATCH4; ++i) u[i] = ldg4(p.UT + (size_t)(j + i) * p.ld + m);
#pragma unroll
      for (int i = 0; i < CTM_SEED_BATCH4; ++i) jet(u[i], j + i);
    }
    for (; j < r0 + p.rb; ++j)
      jet((j < r1) ? ldg4(p.UT + (size_t)j * p.ld + m) : make_float4(0.f, 0.f, 0.f, 0.f), j);
    // sum_w h4 = tanh'''' * sum_j w_j z1_j^4 over the block's jets   (z2 = z3 = z4 = 0)
    const float4 cs = ldg4(p.csum + (size_t)b * p.ld + m);
    seed_store4<NP>(o, (row0 + 1 + 3 * p.rb) * p.ld + m, d4[0] * cs.x, d4[1] * cs.y, d4[2] * cs.z,
                d4[3] * cs.w);
    CTM_BLOCK_END
  }
#undef CTM_BLOCK_BEGIN
#undef CTM_BLOCK_END
  if constexpr (F16 && KORD != kNest) {
#pragma unroll
    for (int t2 = 0; t2 < kF16Types; ++t2) warp_max_record(smx[t2], &f.out->maxabs[t2]);
  }
}

// Fixed direction sets, K=2 (e_d, sigma columns) and K=4 (the biharmonic family), forward
// only: the same layer-1 rule as seed_layer_kernel, laid out as a streaming store. A block
// owns a 128-feature slice of layer 1 for a contiguous range of points and stages that
// slice of W1^T, U^T, csum and b1 in shared memory once; each warp then runs one point at
// a time (lane: 4 adjacent features), reading the tables from shared memory, so the loop
// in front of the stores has no global-load latency (seed_layer_kernel re-reads U^T from
// L2 for every point: ncu put 42% of its stall samples at the first use of a U^T value).
// Writes are 256 contiguous bytes per warp per plane row.
//   K=2: h0 = s(z0); h1_r = s'(z0) u_r; sum h2 = s''(z0) sum_r u_r^2      (x2 = 0)
//   K=4: per jet h1 = s' u, h2 = s'' u^2, h3 = s''' u^3; sum_w h4 = s'''' sum_j w_j u_j^4
// grid (ld / 128 slices, point groups); dynamic smem: seed_fixed_smem() bytes.
constexpr int kSeedFixedFeats = 128;
constexpr int kSeedFixedWarps = 8;
__host__ __device__ inline size_t seed_fixed_smem(int D, int R, int blocks) {
  return ((size_t)(D + R + blocks + 1) * kSeedFixedFeats + (size_t)kSeedFixedWarps * D) * sizeof(float);
}

template <int KORD, int NP, bool F16 = false>
__global__ void __launch_bounds__(kSeedFixedWarps * 32, 4) seed_fixed_kernel(const SeedParams p, int64_t pts_per_group,
                                                                          const SeedF16 f) {
  extern __shared__ float sm[];
  constexpr int F = kSeedFixedFeats;
  float* w1s = sm;                          // [D][F]
  float* us = w1s + (size_t)p.D * F;        // [R][F]
  float* cs = us + (size_t)p.R * F;         // [blocks][F]
  float* bs = cs + (size_t)p.blocks * F;    // [F]
  float* xs = bs + F;                       // [warps][D]
  const int f0 = blockIdx.x * F;
  for (int i = threadIdx.x; i < (p.D + p.R + p.blocks + 1) * (F / 4); i += blockDim.x) {
    const int row = i / (F / 4), c4 = 4 * (i % (F / 4));
    const float* src = row < p.D ? p.W1T + (size_t)row * p.ld
                     : row < p.D + p.R ? p.UT + (size_t)(row - p.D) * p.ld
                     : row < p.D + p.R + p.blocks ? p.csum + (size_t)(row - p.D - p.R) * p.ld
                     : p.b1;
    *reinterpret_cast<float4*>(sm + (size_t)row * F + c4) = ldg4(src + f0 + c4);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = 4 * lane;
  const int m = f0 + c;
  float* xw = xs + warp * p.D;
  const int64_t nb = blockIdx.y * pts_per_group;
  const int64_t ne = (nb + pts_per_group < p.n_points) ? nb + pts_per_group : p.n_points;
  static_assert(!F16 || NP == 2, "fp16x3: two planes");
  // fp16x3: output scales per slot type (jet_layer.cuh F16Rec) from |h0| <= s0 and, with
  // U = max|U| and C = max|csum|: K=2 |s' u| <= s1 U, |s'' csum| <= s2 C; K=4 |s' u| <= s1 U,
  // |s'' u^2| <= s2 U^2, |s''' u^3| <= s3 U^3, |s'''' csum| <= s4 C
  float os[kF16Types], mx[kF16Types];
#pragma unroll
  for (int t = 0; t < kF16Types; ++t) os[t] = 1.f, mx[t] = 0.f;
  if (F16) {
    const float U = __uint_as_float(f.bounds[0]), C = __uint_as_float(f.bounds[1]);
    os[0] = f16_scale_for(f.s0);
    os[1] = f16_scale_for(f.s1 * U);
    os[2] = f16_scale_for((KORD == 4 ? f.s4 : f.s2) * C);
    if (KORD == 4) {
      os[3] = f16_scale_for(f.s2 * U * U);
      os[4] = f16_scale_for(f.s3 * U * U * U);
    }
    if (f.uniform) {
      const float u = fminf(os[0], fminf(os[1], os[2]));
#pragma unroll
      for (int t = 0; t < kF16Types; ++t) os[t] = u;
    }
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
      for (int t = 0; t < kF16Types; ++t) f.out->scale[t] = os[t];
  }
  // one row of 4 adjacent features at dst: fp16x3 takes values ALREADY scaled for their slot
  // type (the per-point derivative factors carry the scale: (s1 sc) u = (s1 u) sc exactly, as
  // sc is a power of two) and tracks the type's max |scaled value|; unscaled at the end
  auto put4 = [&](uint16_t* dst, float a, float b, float c, float d, int type) {
    if constexpr (F16) {
      seed_store4_f16s(dst, p.pstride, a, b, c, d);
      mx[type] = fmaxf(mx[type], max4abs(a, b, c, d));
    } else {
      seed_store4_at<NP>(dst, p.pstride, a, b, c, d);
    }
  };
  const int64_t ld = p.ld;
  for (int64_t n = nb + warp; n < ne; n += kSeedFixedWarps) {
    for (int d = lane; d < p.D; d += 32) xw[d] = __ldg(p.X + n * p.D + d);
    __syncwarp();
    float4 z0 = *reinterpret_cast<const float4*>(bs + c);
    for (int d = 0; d < p.D; ++d) {
      const float4 w = *reinterpret_cast<const float4*>(w1s + (size_t)d * F + c);
      const float xd = xw[d];
      z0.x = fmaf(w.x, xd, z0.x);
      z0.y = fmaf(w.y, xd, z0.y);
      z0.z = fmaf(w.z, xd, z0.z);
      z0.w = fmaf(w.w, xd, z0.w);
    }
    __syncwarp();  // xw is rewritten for the warp's next point
    // (four explicit calls: a loop over a local array was not unrolled and went to local memory)
    const ActD A0 = act_derivs(p.act, z0.x), A1 = act_derivs(p.act, z0.y), A2 = act_derivs(p.act, z0.z),
               A3 = act_derivs(p.act, z0.w);
    // slot-type scales of the rows (all 1 outside fp16x3): h0 (type 0), s1 u (1), the top (2);
    // K=4 also s2 u^2 (3) and s3 u^3 (4)
    const float sc0 = os[0], sc1 = os[1], sc2 = os[2];
    const float sc3 = (KORD == 4) ? os[3] : 1.f, sc4 = (KORD == 4) ? os[4] : 1.f;
    const float d2s = (KORD == 4) ? sc3 : sc2;  // K=2: s'' multiplies the top row
    const float t[4] = {A0.d0 * sc0, A1.d0 * sc0, A2.d0 * sc0, A3.d0 * sc0},
                d1[4] = {A0.d1 * sc1, A1.d1 * sc1, A2.d1 * sc1, A3.d1 * sc1},
                d2[4] = {A0.d2 * d2s, A1.d2 * d2s, A2.d2 * d2s, A3.d2 * d2s},
                d3[4] = {A0.d3 * sc4, A1.d3 * sc4, A2.d3 * sc4, A3.d3 * sc4},
                d4[4] = {A0.d4 * sc2, A1.d4 * sc2, A2.d4 * sc2, A3.d4 * sc2};
    uint16_t* dst = p.out + (size_t)n * p.blocks * p.P * ld + m;  // row (n * blocks + b) * P + slot
    // grad mode (K=2, one block): the pre-activations [z0; u_r; 0] of the point's slots
    float* zd = (KORD == 2 && p.z_out) ? p.z_out + (size_t)n * p.P * ld + m : nullptr;
    auto putz = [&](float4 v) {
      if (zd) {
        *reinterpret_cast<float4*>(zd) = v;
        zd += ld;
      }
    };
    for (int b = 0; b < p.blocks; ++b) {
      const int r0 = b * p.rb;
      const int r1 = (r0 + p.rb < p.R) ? r0 + p.rb : p.R;
      put4(dst, t[0], t[1], t[2], t[3], 0);
      putz(z0);
      dst += ld;
      for (int r = r0; r < r0 + p.rb; ++r) {
        // the padding directions of a last block (r >= r1) are zero rows
        const float4 u = (r < r1) ? *reinterpret_cast<const float4*>(us + (size_t)r * F + c)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
        put4(dst, d1[0] * u.x, d1[1] * u.y, d1[2] * u.z, d1[3] * u.w, 1);
        putz(u);
        dst += ld;
        if (KORD == 4) {
          put4(dst, d2[0] * u.x * u.x, d2[1] * u.y * u.y, d2[2] * u.z * u.z, d2[3] * u.w * u.w, 3);
          dst += ld;
          put4(dst, d3[0] * u.x * u.x * u.x, d3[1] * u.y * u.y * u.y, d3[2] * u.z * u.z * u.z,
               d3[3] * u.w * u.w * u.w, 4);
          dst += ld;
        }
      }
      const float4 q = *reinterpret_cast<const float4*>(cs + (size_t)b * F + c);
      if (KORD == 4)
        put4(dst, d4[0] * q.x, d4[1] * q.y, d4[2] * q.z, d4[3] * q.w, 2);
      else
        put4(dst, d2[0] * q.x, d2[1] * q.y, d2[2] * q.z, d2[3] * q.w, 2);
      putz(make_float4(0.f, 0.f, 0.f, 0.f));  // x2 = 0: the top pre-activation of layer 1
      dst += ld;
    }
  }
  if constexpr (F16) {
#pragma unroll
    for (int t = 0; t < (KORD == 4 ? kF16Types : 3); ++t) warp_max_record(mx[t] / os[t], &f.out->maxabs[t]);
  }
}

// Stochastic biharmonic (Eq. 12 stochastic), layer 1 in fp32 on the CUDA
// cores: per point, S standard normal directions v_s (explicit or generated), and for
// each feature z1_s = W1 v_s; writes h1, h2, h3 per sample (x2 = x3 = 0) and the
// collapsed top sum_s h4_s = tanh'''' sum_s z1_s^4. K = D is tiny for this operator and
// the 4th powers would amplify a bf16-pair rounding of W1 and v 4x.
// grid: one block per (point, 4*blockDim-feature chunk); dynamic smem: S*D floats.
struct SeedStochParams {
  const float* X;        // [N, D]
  int D;
  const float* W1T;      // [D, ld]
  const float* b1;       // [ld]
  int ld;
  int S;
  const float* V;        // [N, S, D] or nullptr => generated standard normal
  const float* w;        // [S] weights of the collapsed sum, or nullptr (all 1)
  uint64_t seed;
  int64_t point_offset;
  int blocks;            // sample blocks per point, `rb` samples each (last one zero padded)
  int rb;
  int standard;          // 1: standard K=4 layout, per sample (h1, h2, h3, h4), 1 + 4 rb rows
  uint16_t* out;         // planes of [N*blocks*(3rb+2), ld] (standard: [N*blocks*(1+4rb), ld])
  int64_t pstride;
  int nplanes;
  int act;
};

__device__ __forceinline__ float gaussian_draw(uint64_t seed, uint64_t idx);

// fp16x3 mode of seed_stoch_biharmonic_kernel (collapsed layout only): ||W1||_inf (g1, from
// the layer-1 weight statistics), the bound of |v| (vmax: max |V| of explicit directions, or
// vgen for the generated normals), the activation sups, the block's record. With
// Z = ||W1||_inf max|v| >= |z1| and Rw = sum_s |w_s|: |h1| <= s1 Z, |h2| <= s2 Z^2,
// |h3| <= s3 Z^3, |top| <= s4 Rw Z^4, |h0| <= s0 (slot types 1, 3, 4, 2, 0).
struct SeedStochF16 {
  const float* g1;
  const unsigned* vmax;
  float vgen;
  float s0, s1, s2, s3, s4;
  F16Rec* out;
};

template <int NP, bool F16 = false>
__global__ void __launch_bounds__(kSeedThreads) seed_stoch_biharmonic_kernel(const SeedStochParams p,
                                                                             const SeedStochF16 f = {}) {
  extern __shared__ float vsh[];  // [S, D]
  const PlaneOut o{p.out, p.pstride, p.nplanes};
  static_assert(!F16 || NP == 2, "fp16x3: two planes");
  float os[kF16Types], mx[kF16Types];
#pragma unroll
  for (int t = 0; t < kF16Types; ++t) os[t] = 1.f, mx[t] = 0.f;
  if constexpr (F16) {
    const float Z = f.g1[1] * (f.vmax ? __uint_as_float(*f.vmax) : f.vgen);
    float rw = 0.f;
    for (int s = 0; s < p.S; ++s) rw += p.w ? fabsf(p.w[s]) : 1.f;
    os[0] = f16_scale_for(f.s0);
    os[1] = f16_scale_for(f.s1 * Z);
    os[3] = f16_scale_for(f.s2 * Z * Z);
    os[4] = f16_scale_for(f.s3 * Z * Z * Z);
    os[2] = f16_scale_for(f.s4 * rw * Z * Z * Z * Z);
    if (blockIdx.x == 0 && threadIdx.x == 0)
      for (int t = 0; t < kF16Types; ++t) f.out->scale[t] = os[t];
  }
  auto put4 = [&](size_t idx, float a, float b, float c, float d, int type) {
    if constexpr (F16) {
      seed_store4_f16(o, idx, a, b, c, d, os[type]);
      mx[type] = fmaxf(mx[type], max4abs(a, b, c, d));
    } else {
      seed_store4<NP>(o, idx, a, b, c, d);
    }
  };
  const int feats = 4 * blockDim.x;
  const int mchunks = (p.ld + feats - 1) / feats;
  const int64_t n = blockIdx.x / mchunks;
  const int m = (blockIdx.x % mchunks) * feats + 4 * threadIdx.x;
  for (int e = threadIdx.x; e < p.S * p.D; e += blockDim.x) {
    if (p.V) {
      vsh[e] = p.V[(size_t)n * p.S * p.D + e];
    } else {
      const uint64_t idx = (uint64_t)(p.point_offset + n) * (uint64_t)p.S * (uint64_t)p.D + (uint64_t)e;
      vsh[e] = gaussian_draw(p.seed, idx);  // e = s * D + d
    }
  }
  __syncthreads();
  if (m < p.ld) {
  const int P = p.standard ? 1 + 4 * p.rb : 3 * p.rb + 2;  // slots per block
  const int st = p.standard ? 4 : 3;                       // rows per sample
  float4 z0 = __ldg(reinterpret_cast<const float4*>(p.b1 + m));
  for (int d = 0; d < p.D; ++d) {
    const float4 w = __ldg(reinterpret_cast<const float4*>(p.W1T + (size_t)d * p.ld + m));
    const float xd = __ldg(p.X + n * p.D + d);
    z0.x = fmaf(w.x, xd, z0.x);
    z0.y = fmaf(w.y, xd, z0.y);
    z0.z = fmaf(w.z, xd, z0.z);
    z0.w = fmaf(w.w, xd, z0.w);
  }
  const float zz[4] = {z0.x, z0.y, z0.z, z0.w};
  float t[4], d1[4], d2[4], d3[4], d4[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const ActD A = act_derivs(p.act, zz[i]);
    t[i] = A.d0; d1[i] = A.d1; d2[i] = A.d2; d3[i] = A.d3; d4[i] = A.d4;
  }
  for (int b = 0; b < p.blocks; ++b) {
    const size_t row0 = ((size_t)n * p.blocks + b) * P;
    put4(row0 * p.ld + m, t[0], t[1], t[2], t[3], 0);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int s = b * p.rb; s < (b + 1) * p.rb; ++s) {
      float z[4] = {0.f, 0.f, 0.f, 0.f};
      if (s < p.S) {
        for (int d = 0; d < p.D; ++d) {
          const float4 w = __ldg(reinterpret_cast<const float4*>(p.W1T + (size_t)d * p.ld + m));
          const float v = vsh[s * p.D + d];
          z[0] = fmaf(w.x, v, z[0]);
          z[1] = fmaf(w.y, v, z[1]);
          z[2] = fmaf(w.z, v, z[2]);
          z[3] = fmaf(w.w, v, z[3]);
        }
      }
      float h1[4], h2[4], h3[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float z2 = z[i] * z[i];
        h1[i] = d1[i] * z[i];
        h2[i] = d2[i] * z2;
        h3[i] = d3[i] * z2 * z[i];
        acc[i] = fmaf((p.w && s < p.S) ? p.w[s] * z2 : z2, z2, acc[i]);
      }
      const size_t r = row0 + 1 + st * (size_t)(s - b * p.rb);
      put4(r * p.ld + m, h1[0], h1[1], h1[2], h1[3], 1);
      put4((r + 1) * p.ld + m, h2[0], h2[1], h2[2], h2[3], 3);
      put4((r + 2) * p.ld + m, h3[0], h3[1], h3[2], h3[3], 4);
      if (p.standard) {  // h4 of this sample = s'''' z1^4   (x2 = x3 = x4 = 0)
        float h4[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) h4[i] = d4[i] * (z[i] * z[i]) * (z[i] * z[i]);
        put4((r + 3) * p.ld + m, h4[0], h4[1], h4[2], h4[3], 2);  // (type 2: the top's bound covers it)
      }
    }
    if (!p.standard)
      put4((row0 + P - 1) * p.ld + m, d4[0] * acc[0], d4[1] * acc[1], d4[2] * acc[2], d4[3] * acc[3], 2);
  }
  }
  if constexpr (F16) {  // every thread of the block reaches here (warp-uniform records)
#pragma unroll
    for (int t = 0; t < kF16Types; ++t) warp_max_record(mx[t], &f.out->maxabs[t]);
  }
}

// Randomized directions: the layer-1 INPUT block of the collapsed jet,
// rows [x0; u_1 .. u_S; 0] per point (Eq. 8/10 stochastic seeds),
// u_s = v_s or sigma v_s, stored as bf16 pairs [N*(S+2), ldk] (ldk = D padded to 32,
// zero padded). Layer 1 then runs on the tensor cores like every other layer.
// grid: one block per point.
struct SeedRandomParams {
  const float* X;        // [N, D]
  int D;
  int ldk;               // padded row length (multiple of 32)
  int S;
  int Rv;
  const float* V;        // [N, S, Rv] (or [N, Rv, S] if v_trans) or nullptr => generated
  int v_trans;           // V stored [N, Rv, S]: sigma(x_n) [D, R] per point
  int v_shared;          // V [S, ldv]: the same directions for every point (grad mode, fixed sets)
  int ldv;
  const float* sigma;    // [D, Rv] or nullptr (then Rv == D)
  uint64_t seed;
  int64_t point_offset;
  int gaussian;          // generated directions: 0 Rademacher, 1 standard normal
  int blocks;            // direction blocks per point, `rb` directions each (last one zero padded)
  int rb;
  int standard;          // 1: standard Taylor mode layout [x0; (u_s, 0) per direction], 1 + 2 rb rows
  uint16_t* out;         // planes of [N*blocks*(rb+2), ldk] (standard: [N*blocks*(1+2rb), ldk])
  int64_t pstride;
  int nplanes;
  // fp16x3 mode (seed_random_kernel<2, true>, no sigma, collapsed layout): bounds [max |x|,
  // max |V|] (float bits) and the generated directions' bound vgen (Rademacher 1, Gaussian 6)
  const unsigned* f16_bounds;
  float vgen;
  F16Rec* f16_out;
  int f16_uniform;       // grad mode (B_0 of fixed sets, fp16x3 training): one scale for all slot types;
                         // with sigma, f16_bounds[2] = max |sigma| and |u| <= Rv max|sigma| max|v|
};

// Standard normal draw for counter idx: Box-Muller on two splitmix64 outputs
// (counters 2 idx and 2 idx + 1), u1 in (0, 1], u2 in [0, 1), 24-bit uniforms.
__device__ __forceinline__ float gaussian_draw(uint64_t seed, uint64_t idx) {
  const uint64_t a = splitmix64(seed, 2ull * idx), b = splitmix64(seed, 2ull * idx + 1ull);
  const float u1 = ((float)(a >> 40) + 0.5f) * 5.9604644775390625e-8f;  // 2^-24
  const float u2 = (float)(b >> 40) * 5.9604644775390625e-8f;
  return sqrtf(-2.f * logf(u1)) * cospif(2.f * u2);
}

template <int NP, bool F16 = false>
__global__ void __launch_bounds__(kSeedThreads) seed_random_kernel(const SeedRandomParams p) {
  __shared__ float vs[kSeedChunk];
  const PlaneOut o{p.out, p.pstride, p.nplanes};
  static_assert(!F16 || NP == 2, "fp16x3: two planes");
  // fp16x3: primal rows x0 scaled by its bound, direction rows by theirs, zero top rows by 1
  float os0 = 1.f, os1 = 1.f, mx0 = 0.f, mx1 = 0.f;
  if (F16) {
    os0 = f16_scale_for(__uint_as_float(p.f16_bounds[0]));
    const float vb = p.V ? __uint_as_float(p.f16_bounds[1]) : p.vgen;
    os1 = f16_scale_for(p.sigma ? (float)p.Rv * __uint_as_float(p.f16_bounds[2]) * vb : vb);
    if (p.f16_uniform) os0 = os1 = fminf(os0, os1);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      p.f16_out->scale[0] = os0;
      p.f16_out->scale[1] = os1;
      for (int t = 2; t < kF16Types; ++t) p.f16_out->scale[t] = p.f16_uniform ? os0 : 1.f;
    }
  }
  auto put4 = [&](size_t idx, float a, float b, float c, float d, int type) {
    if constexpr (F16) {
      seed_store4_f16(o, idx, a, b, c, d, type == 0 ? os0 : type == 1 ? os1 : p.f16_uniform ? os0 : 1.f);
      const float mv = max4abs(a, b, c, d);
      if (type == 0) mx0 = fmaxf(mx0, mv); else if (type == 1) mx1 = fmaxf(mx1, mv);
    } else {
      seed_store4<NP>(o, idx, a, b, c, d);
    }
  };
  const int64_t n = blockIdx.x;
  const int st = p.standard ? 2 : 1;            // rows per direction
  const int P = p.standard ? 1 + 2 * p.rb : p.rb + 2;  // slots per block
  const size_t pt0 = (size_t)n * p.blocks;      // first sub-point of this point
  const int q4 = p.ldk / 4;                     // 4-column groups per row
  // direction s lives in row 1 + st (s % rb) of sub-point s / rb
  auto dir_row = [&](int s) { return (pt0 + s / p.rb) * P + 1 + st * (s % p.rb); };
  // every block's primal row and zero top row (standard: the zero x2 row of every
  // direction), and the zero rows of the last block's padding
  for (int c4 = threadIdx.x; c4 < q4; c4 += blockDim.x) {
    float x[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = (4 * c4 + i < p.D) ? p.X[n * p.D + 4 * c4 + i] : 0.f;
    for (int b = 0; b < p.blocks; ++b) {
      put4((pt0 + b) * P * p.ldk + 4 * c4, x[0], x[1], x[2], x[3], 0);
      if (!p.standard) put4(((pt0 + b) * P + P - 1) * p.ldk + 4 * c4, 0.f, 0.f, 0.f, 0.f, 2);
    }
    if (p.standard)
      for (int s = 0; s < p.blocks * p.rb; ++s)
        seed_store4<NP>(o, (dir_row(s) + 1) * p.ldk + 4 * c4, 0.f, 0.f, 0.f, 0.f);
    for (int s = p.S; s < p.blocks * p.rb; ++s) put4(dir_row(s) * p.ldk + 4 * c4, 0.f, 0.f, 0.f, 0.f, 1);
  }
  const int per_chunk = kSeedChunk / p.Rv;
  for (int s0 = 0; s0 < p.S; s0 += per_chunk) {
    const int ns = (p.S - s0 < per_chunk) ? (p.S - s0) : per_chunk;
    __syncthreads();
    for (int e = threadIdx.x; e < ns * p.Rv; e += blockDim.x) {
      const int s = s0 + e / p.Rv, r = e % p.Rv;
      float v;
      if (p.V) {
        v = p.v_shared ? p.V[(size_t)s * p.ldv + r]
            : p.v_trans ? p.V[((size_t)n * p.Rv + r) * p.S + s]
                        : p.V[((size_t)n * p.S + s) * p.Rv + r];
      } else {
        const uint64_t idx =
            ((uint64_t)(p.point_offset + n) * (uint64_t)p.S + (uint64_t)s) * (uint64_t)p.Rv + (uint64_t)r;
        v = p.gaussian ? gaussian_draw(p.seed, idx) : ((splitmix64(p.seed, idx) >> 63) ? -1.f : 1.f);
      }
      vs[e] = v;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < ns * q4; e += blockDim.x) {
      const int s = e / q4, c4 = e % q4;
      float u[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int d = 4 * c4 + i;
        float val = 0.f;
        if (d < p.D) {
          if (p.sigma) {
            for (int r = 0; r < p.Rv; ++r) val = fmaf(p.sigma[(size_t)d * p.Rv + r], vs[s * p.Rv + r], val);
          } else {
            val = vs[s * p.Rv + d];
          }
        }
        u[i] = val;
      }
      put4(dir_row(s0 + s) * p.ldk + 4 * c4, u[0], u[1], u[2], u[3], 1);
    }
  }
  if constexpr (F16) {
    warp_max_record(mx0, &p.f16_out->maxabs[0]);
    warp_max_record(mx1, &p.f16_out->maxabs[1]);
  }
}

// csum[b * ld + m] = sum over the directions r of block b (r < R) of w_r UT[r, m]^pow
// (pow 2 or 4; w nullptr = all ones): the per-block constants of the fixed direction sets.
__global__ void block_csum_kernel(const float* __restrict__ UT, int R, int ld, const float* __restrict__ w, int pow,
                                  int blocks, int rb, float* __restrict__ csum) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= ld) return;
  for (int b = 0; b < blocks; ++b) {
    float cs = 0.f;
    for (int r = b * rb; r < (b + 1) * rb && r < R; ++r) {
      const float u = UT[(size_t)r * ld + m];
      const float u2 = u * u;
      cs = fmaf(w ? w[r] : 1.f, pow == 2 ? u2 : u2 * u2, cs);
    }
    csum[(size_t)b * ld + m] = cs;
  }
}

// UT[r, m] = sum_d W1T[d, m] dirs[r, d]; csum[m] = sum_r w_r UT[r, m]^pow (pow 2 or 4).
// dirs is [R, D] (device), w is [R] or nullptr (all ones). One thread per feature.
__global__ void prep_directions_kernel(const float* __restrict__ W1T, int D, int ld, const float* __restrict__ dirs,
                                       int R, const float* __restrict__ w, int pow, float* __restrict__ UT,
                                       float* __restrict__ csum) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= ld) return;
  float cs = 0.f;
  for (int r = 0; r < R; ++r) {
    float u = 0.f;
    for (int d = 0; d < D; ++d) u = fmaf(W1T[(size_t)d * ld + m], dirs[(size_t)r * D + d], u);
    UT[(size_t)r * ld + m] = u;
    const float u2 = u * u;
    cs = fmaf(w ? w[r] : 1.f, pow == 2 ? u2 : u2 * u2, cs);
  }
  if (csum) csum[m] = cs;
}

// The Laplacian's fixed directions e_d: UT[d, m] = W1T[d, m] (z1 of e_d is column d of W1)
// and csum[m] = sum_d W1T[d, m]^2. One thread per feature.
__global__ void prep_laplacian_kernel(const float* __restrict__ W1T, int D, int ld, float* __restrict__ UT,
                                      float* __restrict__ csum) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= ld) return;
  float cs = 0.f;
  for (int d = 0; d < D; ++d) {
    const float u = W1T[(size_t)d * ld + m];
    UT[(size_t)d * ld + m] = u;
    cs = fmaf(u, u, cs);
  }
  csum[m] = cs;
}

// AT[r, m] = sum_d W1T[d, m] sigma[d, r]  (sigma [D, R] row-major)
__global__ void prep_sigma_kernel(const float* __restrict__ W1T, int D, int ld, const float* __restrict__ sigma,
                                  int R, float* __restrict__ AT, float* __restrict__ csum) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= ld) return;
  float cs = 0.f;
  for (int r = 0; r < R; ++r) {
    float u = 0.f;
    for (int d = 0; d < D; ++d) u = fmaf(W1T[(size_t)d * ld + m], sigma[(size_t)d * R + r], u);
    AT[(size_t)r * ld + m] = u;
    cs = fmaf(u, u, cs);
  }
  if (csum) csum[m] = cs;
}

// op[n] = scale * sum_b sum_t partial[n*blocks + b, t, 1];  f[n] = b_out + sum_t partial[n*blocks, t, 0]
// (fixed order; every block carries the primal, its first block gives f)
__global__ void finalize_kernel(const float* __restrict__ partial, int m_tiles, int blocks, int64_t N,
                                const float* __restrict__ b_out, float scale, float* __restrict__ op,
                                float* __restrict__ f) {
  ptx::pdl_wait_prior();  // launched as a programmatic dependent of the last layer kernel
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  float s0 = 0.f, s1 = 0.f;
  const float* pp = partial + n * blocks * m_tiles * 2;
  for (int t = 0; t < m_tiles; ++t) s0 += pp[t * 2 + 0];
  for (int i = 0; i < blocks * m_tiles; ++i) s1 += pp[i * 2 + 1];
  op[n] = scale * s1;
  if (f) f[n] = *b_out + s0;
}

// Readout straight from a layer block (nets with a single hidden layer):
// one warp per point, lanes over features; `blocks` sub-points of P slots per point.
// standard == 2: the op is sum_r w_out . h2_r over rows 2, 4, .., P-1 (standard mode);
// standard == 4: sum_j jw[j] w_out . h4_j over rows 4, 8, .., P-1 (standard K=4 mode, jw
// indexed over all blocks of the point)
__global__ void readout_block_kernel(const uint16_t* __restrict__ in, int64_t pstride, int nplanes, int ld, int P,
                                     int blocks, int width, const float* __restrict__ w_out,
                                     const float* __restrict__ b_out, float scale, int64_t N, float* __restrict__ op,
                                     float* __restrict__ f, int standard, const float* __restrict__ jw, int rb,
                                     int J) {
  const int64_t n = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (n >= N) return;
  float s0 = 0.f, s1 = 0.f;
  for (int b = 0; b < blocks; ++b) {
    const size_t sp = (size_t)n * blocks + b;
    const size_t r0 = sp * P * ld, rt = (sp * P + P - 1) * ld;
    for (int m = lane; m < width; m += 32) {
      if (b == 0) s0 = fmaf(w_out[m], ptx::planes_val(in + r0 + m, pstride, nplanes), s0);
      if (!standard) {
        s1 = fmaf(w_out[m], ptx::planes_val(in + rt + m, pstride, nplanes), s1);
      } else {
        for (int r = standard; r < P; r += standard) {
          const size_t ri = (sp * P + r) * ld;
          const int j = b * rb + r / 4 - 1;
          const float c = (standard == 4) ? ((j < J) ? jw[j] : 0.f) : 1.f;
          s1 = fmaf(c * w_out[m], ptx::planes_val(in + ri + m, pstride, nplanes), s1);
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
  }
  if (lane == 0) {
    op[n] = scale * s1;
    if (f) f[n] = *b_out + s0;
  }
}

// Split W [rows, cols] (row-major, device) into three padded bf16 planes [3][Mpad, Kpad]
// (plane stride Mpad * Kpad); bias into [Mpad]. Padding is zero.
__global__ void split_weights_kernel(const float* __restrict__ W, const float* __restrict__ b, int rows, int cols,
                                     int Mpad, int Kpad, uint16_t* __restrict__ Wp, float* __restrict__ bpad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)Mpad * Kpad;
  if (i >= n) return;
  const int r = (int)(i / Kpad), c = (int)(i % Kpad);
  const float v = (r < rows && c < cols) ? W[(size_t)r * cols + c] : 0.f;
  ptx::bf16_split3(v, Wp[i], Wp[n + i], Wp[2 * n + i]);
  if (c == 0) bpad[r] = (r < rows) ? b[r] : 0.f;
}

// fp16x3 weights, derived from the weights' three bf16 planes Wp [3][Mpad, Kpad] (their sum
// rounds to the fp32 weight exactly: p0 + p1 + p2 is within 2^-27 of it), so they can be
// (re)built whenever the handle switches to the mode, without the caller's arrays.
__device__ __forceinline__ float planes3_val(const uint16_t* Wp, int64_t n, int64_t i) {
  return ptx::bf16_val(Wp[i]) + ptx::bf16_val(Wp[n + i]) + ptx::bf16_val(Wp[2 * n + i]);
}
// Statistics of bf16-plane weights [3][rows, cols], grid-parallel, into acc (float bits,
// zeroed by the caller; atomicMax of non-negative floats is order-independent, so the result
// is deterministic): acc[0] = max |W|, acc[1] = ||W||_inf = max_m sum_k |W[m, k]| (one warp per
// row, lanes strided over k, then a shuffle tree), and with do_cols acc[2] = ||W^T||_inf =
// max_k sum_m |W[m, k]| (one thread per column; the adjoint's bound, fp16x3 training).
__global__ void __launch_bounds__(256) f16_weight_norms_kernel(const uint16_t* __restrict__ Wp, int rows, int cols,
                                                               int do_cols, unsigned* __restrict__ acc) {
  const int64_t n = (int64_t)rows * cols;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = gt >> 5, lane = threadIdx.x & 31;
  if (r < rows) {  // warp-uniform
    float a = 0.f, m = 0.f;
    for (int c = lane; c < cols; c += 32) {
      const float v = fabsf(planes3_val(Wp, n, (int64_t)r * cols + c));
      a += v;
      m = fmaxf(m, v);
    }
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    }
    if (lane == 0) {
      atomicMax(acc + 0, __float_as_uint(m));
      atomicMax(acc + 1, __float_as_uint(a));
    }
  }
  if (do_cols && gt < cols) {
    float s = 0.f;
    for (int rr = 0; rr < rows; ++rr) s += fabsf(planes3_val(Wp, n, (int64_t)rr * cols + gt));
    atomicMax(acc + 2, __float_as_uint(s));
  }
}
// out[0] = 2^-(sa + 11) = 1 / (the scale putting max |W| in (2^13, 2^14]), the factor that
// undoes the planes' scales (split_weights_f16_kernel); out[1] = ||W||_inf (the bound of
// jet_layer.cuh f16_out_scales); outT (grad mode): the same factor and ||W^T||_inf
__global__ void f16_weight_stats_kernel(const unsigned* __restrict__ acc, float* __restrict__ out,
                                        float* __restrict__ outT) {
  out[0] = 1.f / f16_scale_for(__uint_as_float(acc[0]));
  out[1] = __uint_as_float(acc[1]);
  if (outT) {
    outT[0] = out[0];
    outT[1] = __uint_as_float(acc[2]);
  }
}
// fp16x3 weight planes [3][Mpad, Kpad] (zero padding stays zero): p0 = rn_f16(W 2^sa),
// p1 = rn_f16((W 2^sa - p0) 2^11) (the corrections' operands: p1 * B0 and p0 * B1 both carry
// 2^(sa + 11 + sb)), and p0 2^11 (exact) for the leading product with B0 in phase 2 (the same
// 2^(sa + 11 + sb)).
__global__ void split_weights_f16_kernel(const uint16_t* __restrict__ Wp, int64_t n, const float* __restrict__ stats,
                                         uint16_t* __restrict__ W16) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // W * 2^sa with 2^sa = 1 / (stats[0] 2^11): exact (powers of two)
  const float v = planes3_val(Wp, n, i) / (stats[0] * ptx::kF16Lift);
  uint16_t p0, p1;
  ptx::f16_split(v, p0, p1);
  W16[i] = p0;
  W16[n + i] = p1;
  W16[2 * n + i] = __half_as_ushort(__float2half_rn(__half2float(__ushort_as_half(p0)) * ptx::kF16Lift));
}
// max |a_i| over n floats into a record (float bits, atomicMax; the record is zeroed by the caller)
__global__ void maxabs_kernel(const float* __restrict__ a, int64_t n, unsigned* __restrict__ out) {
  float m = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(a[i]));
  warp_max_record(m, out);
}

// W1T [D, ld] = W1^T zero padded; b1 [ld]
__global__ void transpose_w1_kernel(const float* __restrict__ W1, const float* __restrict__ b1, int w1, int D, int ld,
                                    float* __restrict__ W1T, float* __restrict__ b1p) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)D * ld) return;
  const int d = (int)(i / ld), m = (int)(i % ld);
  W1T[i] = (m < w1) ? W1[(size_t)m * D + d] : 0.f;
  if (d == 0) b1p[m] = (m < w1) ? b1[m] : 0.f;
}

// out planes [rows_pad, ldp] <- src [rows, cols] (fp32), zero padded (ctm_gemm_probe)
template <int NP>
__global__ void split_rows_kernel(const float* __restrict__ src, int64_t rows, int cols, int64_t rows_pad, int ldp,
                                  uint16_t* __restrict__ out, int64_t pstride) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= rows_pad * ldp) return;
  const int64_t r = k / ldp;
  const int c = (int)(k % ldp);
  float v = (r < rows && c < cols) ? src[r * cols + c] : 0.f;
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    const __nv_bfloat16 b = __float2bfloat16_rn(v);
    out[q * pstride + k] = __bfloat16_as_ushort(b);
    v -= __bfloat162float(b);
  }
}

// ctm_gemm_probe in the fp16x3 mode: the block's record (every slot type: the scale of the
// measured max |B| and that max) from the bound scratch b[0]
__global__ void probe_f16_record_kernel(const unsigned* __restrict__ b, F16Rec* __restrict__ rec) {
  const float m = __uint_as_float(b[0]);
  for (int t = 0; t < kF16Types; ++t) {
    rec->scale[t] = f16_scale_for(m);
    rec->maxabs[t] = b[0];
  }
}
// ... and its fp16 planes of B * scale [2][rows_pad, ldp]
__global__ void split_rows_f16_kernel(const float* __restrict__ src, int64_t rows, int cols, int64_t rows_pad, int ldp,
                                      const F16Rec* __restrict__ rec, uint16_t* __restrict__ out, int64_t pstride) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= rows_pad * ldp) return;
  const int64_t r = k / ldp;
  const int c = (int)(k % ldp);
  const float v = (r < rows && c < cols) ? src[r * cols + c] : 0.f;
  uint16_t p0, p1;
  ptx::f16_split(v * rec->scale[0], p0, p1);
  out[k] = p0;
  out[pstride + k] = p1;
}

__global__ void pad_vector_kernel(const float* __restrict__ src, int n, int npad, float* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < npad) dst[i] = (i < n) ? src[i] : 0.f;
}

}  // namespace ctm
