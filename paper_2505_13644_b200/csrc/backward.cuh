// backward.cuh — the differentiable path: the adjoint of the collapsed
// K=2 forward for PINN training, L = sum_n gop[n] op[n] + gf[n] f[n].
//
//   top_bwd_kernel     readout + last hidden rule, transposed: Z_bar_{L-1} (bf16 pairs),
//                      per-group partials of dW_L (f = w_L . h0 + b_L, op = c w_L . top)
//   colsum_kernel      deterministic two-stage column sums (db_l from the slot-0 rows of
//                      Z_bar_l, dW_L, db_L): group partials, then reduce_groups_kernel
//   crop_kernel        padded fp32 [rows, ld] -> caller's [rows, cols] (= or +=)
//
// The hidden layers' adjoints run in jet_layer_kernel<kBwd2> (jet_layer.cuh) and the
// weight gradients dW_l = Z_bar_l^T B_{l-1} are plain long-K GEMMs (ctm.cu).
#pragma once
#include <cstdint>

#include "jet_layer.cuh"

namespace ctm {

struct TopBwdParams {
  const float* Z;       // [N*P, ldz] pre-activations of the last hidden layer
  int ldz;
  int P;
  int64_t N;
  int width;            // padded width (threads cover [0, width))
  const float* w_out;   // [width]
  float c;              // op scale (1, or 1/S)
  const float* gop;     // [N]
  const float* gf;      // [N] or nullptr
  const float* jw;      // K=2 weights [P-2] or nullptr
  int act;
  uint16_t* out;        // Z_bar planes [N*P, ldo]
  int64_t pstride;
  int nplanes;
  int ldo;
  float* dw_part;       // [G, width] partials of dW_L
  int G;
  // fp16x3 (top_bwd_kernel<true>): Z_bar as two scaled fp16 planes with ONE scale from the
  // bounds zb = {max |z1|, max |z_top|} of Z and bb (f16_bwd_prep_kernel); maxima per slot type
  // into f16_out
  const float* zb;
  const float* bb;
  float s1, s2, s3;     // sups of the activation's first three derivatives
  F16Rec* f16_out;
};

// grid (width / 512, G); a thread owns four features and the points n = g, g + G, ...
// fp16x3 bounds (F16), TB = |c| max|gop| max|w_L|, HB = max|gf| max|w_L|:
//   |ztb| <= s1 TB;  |z1b_r| <= 2 s2 w Z1 TB;  |z0b| <= s1 HB + (s2 Zt + s3 Rw Z1^2) TB
template <bool F16 = false>
__global__ void __launch_bounds__(128) top_bwd_kernel(const TopBwdParams p) {
  // four adjacent features per thread: float4 loads of Z, 8-byte stores into each plane
  // (the per-element arithmetic is the scalar rule's, in the same order)
  const int m = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  const int g = blockIdx.y;
  float os = 1.f, mx0 = 0.f, mx1 = 0.f, mxt = 0.f;
  if constexpr (F16) {
    const float TB = p.bb[0], HB = p.bb[1], Rw = p.bb[2], wm = p.bb[3], Z1 = p.zb[0], Zt = p.zb[1];
    const float b = fmaxf(p.s1 * TB, fmaxf(2.f * p.s2 * wm * Z1 * TB, p.s1 * HB + (p.s2 * Zt + p.s3 * Rw * Z1 * Z1) * TB));
    os = f16_scale_for(b);
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
      for (int t = 0; t < kF16Types; ++t) p.f16_out->scale[t] = os;
  }
  auto put4 = [&](uint16_t* q, const float* v, float& mx) {
    if constexpr (F16) {
      seed_store4_f16s(q, p.pstride, v[0] * os, v[1] * os, v[2] * os, v[3] * os);
      mx = fmaxf(mx, max4abs(v[0], v[1], v[2], v[3]));
    } else if (p.nplanes == 3) {
      seed_store4_at<3>(q, p.pstride, v[0], v[1], v[2], v[3]);
    } else {
      seed_store4_at<2>(q, p.pstride, v[0], v[1], v[2], v[3]);
    }
  };
  if (m < p.width) {
    const float4 wl4 = *reinterpret_cast<const float4*>(p.w_out + m);
    const float wl[4] = {wl4.x, wl4.y, wl4.z, wl4.w};
    const size_t ldz = (size_t)p.ldz, ldo = (size_t)p.ldo;
    float dwp[4] = {0.f, 0.f, 0.f, 0.f};
    for (int64_t n = g; n < p.N; n += p.G) {
      const size_t row = (size_t)n * p.P;
      const float* zr = p.Z + row * ldz + m;
      const float4 z04 = *reinterpret_cast<const float4*>(zr);
      const float4 zt4 = *reinterpret_cast<const float4*>(zr + (size_t)(p.P - 1) * ldz);
      const float z0[4] = {z04.x, z04.y, z04.z, z04.w}, zt[4] = {zt4.x, zt4.y, zt4.z, zt4.w};
      const ActD A[4] = {act_derivs(p.act, z0[0]), act_derivs(p.act, z0[1]), act_derivs(p.act, z0[2]),
                         act_derivs(p.act, z0[3])};
      const float go = p.gop[n], gfn = p.gf ? p.gf[n] : 0.f;
      float tb[4], hb0[4], szz[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        tb[i] = p.c * go * wl[i];  // adjoint of the collapsed top h_top
        hb0[i] = gfn * wl[i];      // adjoint of h0
        szz[i] = 0.f;
      }
      const float* __restrict__ zs = zr + ldz;
      uint16_t* __restrict__ oz = p.out + (row + 1) * ldo + m;
#pragma unroll 4
      for (int r = 0; r < p.P - 2; ++r) {
        const float4 z14 = *reinterpret_cast<const float4*>(zs + (size_t)r * ldz);
        const float z1[4] = {z14.x, z14.y, z14.z, z14.w};
        const float w = p.jw ? p.jw[r] : 1.f;
        float v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          szz[i] = fmaf(w * z1[i], z1[i], szz[i]);
          v[i] = 2.f * A[i].d2 * w * z1[i] * tb[i];
        }
        put4(oz + (size_t)r * ldo, v, mx1);
      }
      float vt[4], v0[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        vt[i] = A[i].d1 * tb[i];
        v0[i] = A[i].d1 * hb0[i] + (A[i].d2 * zt[i] + A[i].d3 * szz[i]) * tb[i];
        const float top = A[i].d1 * zt[i] + A[i].d2 * szz[i];
        dwp[i] += gfn * A[i].d0 + p.c * go * top;
      }
      put4(p.out + (row + p.P - 1) * ldo + m, vt, mxt);
      put4(p.out + row * ldo + m, v0, mx0);
    }
    *reinterpret_cast<float4*>(p.dw_part + (size_t)g * p.width + m) = make_float4(dwp[0], dwp[1], dwp[2], dwp[3]);
  }
  if constexpr (F16) {  // every lane reaches here (the record is per slot type)
    warp_max_record(mx0, &p.f16_out->maxabs[0]);
    warp_max_record(mx1, &p.f16_out->maxabs[1]);
    warp_max_record(mxt, &p.f16_out->maxabs[2]);
  }
}

// part[g, m] = sum over rows r = g, g + G, ... < nrows of src[row0 + r * stride, m]
// (bf16 planes if src != nullptr, else fp32 `srcf`); grid (ceil(ncols / 128), G)
// (rec != nullptr: fp16x3 planes of src, scaled by rec->scale[0] -- uniform in grad mode)
__global__ void __launch_bounds__(128) colsum_kernel(const uint16_t* __restrict__ src, int64_t pstride, int nplanes,
                                                     const float* __restrict__ srcf, int64_t nrows, int64_t stride,
                                                     int ld, int ncols, int G, float* __restrict__ part,
                                                     const F16Rec* __restrict__ rec = nullptr) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  const int g = blockIdx.y;
  if (m >= ncols) return;
  float acc = 0.f;
  const float inv = rec ? 1.f / rec->scale[0] : 1.f;
  for (int64_t r = g; r < nrows; r += G) {
    const size_t i = (size_t)(r * stride) * ld + m;
    acc += srcf ? srcf[i] : rec ? ptx::f16_val(src + i, pstride) * inv : ptx::planes_val(src + i, pstride, nplanes);
  }
  part[(size_t)g * ncols + m] = acc;
}

// fp16x3 backward bounds (one block of 1024 threads):
//   bb = {|c| max|gop| max|w_L|, max|gf| max|w_L|, Rw = sum_r |w_r| (R without weights), max_r |w_r| (1)};
//   zb[2 l], zb[2 l + 1] = bounds of max |z1|, max |z_top| of the saved Z_l, l = 1 .. L-1:
//   l = 1: max |U| (the fixed directions' images, ubound) and 0 (x2 = 0); l >= 2: ||W_l||_inf
//   (G[2 l + 1]) times the recorded maxima of B_{l-1}'s first-order and top slots (rec[l-1]).
__global__ void __launch_bounds__(1024) f16_bwd_prep_kernel(const unsigned* __restrict__ gmax, int has_gf,
                                                           const float* __restrict__ w_out, int wl,
                                                           float c, const float* __restrict__ jw, int R,
                                                           const unsigned* __restrict__ ubound, int random,
                                                           const float* __restrict__ G, const F16Rec* __restrict__ rec,
                                                           int L, float* __restrict__ bb, float* __restrict__ zb) {
  __shared__ float red[5][32];  // (rows 2..4 used)
  // max |gop|, max |gf| come from maxabs_kernel (grid-parallel) in gmax[0], gmax[1]
  const float a = __uint_as_float(gmax[0]), b = has_gf ? __uint_as_float(gmax[1]) : 0.f;
  float w = 0.f, sw = 0.f, mw = 0.f;
  for (int i = threadIdx.x; i < wl; i += blockDim.x) w = fmaxf(w, fabsf(w_out[i]));
  if (jw)
    for (int i = threadIdx.x; i < R; i += blockDim.x) {
      sw += fabsf(jw[i]);
      mw = fmaxf(mw, fabsf(jw[i]));
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    w = fmaxf(w, __shfl_xor_sync(0xffffffffu, w, o));
    sw += __shfl_xor_sync(0xffffffffu, sw, o);
    mw = fmaxf(mw, __shfl_xor_sync(0xffffffffu, mw, o));
  }
  if ((threadIdx.x & 31) == 0) {
    red[2][threadIdx.x >> 5] = w;
    red[3][threadIdx.x >> 5] = sw;
    red[4][threadIdx.x >> 5] = mw;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      w = fmaxf(w, red[2][k]);
      sw += red[3][k];
      mw = fmaxf(mw, red[4][k]);
    }
    bb[0] = fabsf(c) * a * w;
    bb[1] = b * w;
    bb[2] = jw ? sw : (float)R;
    bb[3] = jw ? mw : 1.f;
    // layer 1: fixed sets z1 = U (max |U| in ubound[0]); per-point directions (layer 1 on
    // the tensor cores, random != 0) z1 = W1 u, bounded by ||W1||_inf max |u| (rec[0])
    zb[2] = random ? G[3] * __uint_as_float(rec[0].maxabs[1]) : __uint_as_float(ubound[0]);
    zb[3] = 0.f;
    for (int l = 2; l <= L - 1; ++l) {
      zb[2 * l] = G[2 * l + 1] * __uint_as_float(rec[l - 1].maxabs[1]);
      zb[2 * l + 1] = G[2 * l + 1] * __uint_as_float(rec[l - 1].maxabs[2]);
    }
  }
}

// out[m] (=|+=) sum_g part[g * ld + m] for m < ncols (ld >= ncols: the row stride of part),
// deterministic: block (32, 32) handles 32 columns; thread (x, y) sums groups y, y + 32, ...
// in order, then a fixed smem tree over y
__global__ void __launch_bounds__(1024) reduce_groups_kernel(const float* __restrict__ part, int G, int ld, int ncols,
                                                             float* __restrict__ out, int accumulate) {
  __shared__ float red[32][33];
  const int m = blockIdx.x * 32 + threadIdx.x;
  float s = 0.f;
  if (m < ncols)
    for (int g = threadIdx.y; g < G; g += 32) s += part[(size_t)g * ld + m];
  red[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  for (int o = 16; o > 0; o >>= 1) {
    if ((int)threadIdx.y < o) red[threadIdx.y][threadIdx.x] += red[threadIdx.y + o][threadIdx.x];
    __syncthreads();
  }
  if (threadIdx.y == 0 && m < ncols) out[m] = accumulate ? out[m] + red[0][threadIdx.x] : red[0][threadIdx.x];
}

// out[0] (=|+=) sum_n v[n] (one block, fixed order: strided partials then a tree)
__global__ void __launch_bounds__(256) vector_sum_kernel(const float* __restrict__ v, int64_t N, float* __restrict__ out,
                                                         int accumulate) {
  __shared__ float red[256];
  float s = 0.f;
  for (int64_t i = threadIdx.x; i < N; i += blockDim.x) s += v[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = accumulate ? out[0] + red[0] : red[0];
}

// dst[i, j] (=|+=) src[i * lds + j] for i < rows, j < cols
__global__ void crop_kernel(const float* __restrict__ src, int lds, int rows, int cols, float* __restrict__ dst,
                            int accumulate) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= (int64_t)rows * cols) return;
  const int i = (int)(k / cols), j = (int)(k % cols);
  const float v = src[(size_t)i * lds + j];
  dst[k] = accumulate ? dst[k] + v : v;
}

// bf16 plane transpose: out[k][c, r] = in[k][r, c] for the three [rows, cols] planes
// (plane stride rows * cols; W^T for kBwd2)
__global__ void transpose_planes_kernel(const uint16_t* __restrict__ in, int rows, int cols,
                                        uint16_t* __restrict__ out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)rows * cols;
  if (k >= n) return;
  const int r = (int)(k / cols), c = (int)(k % cols);
#pragma unroll
  for (int q = 0; q < 3; ++q) out[q * n + (size_t)c * rows + r] = in[q * n + k];
}

}  // namespace ctm
