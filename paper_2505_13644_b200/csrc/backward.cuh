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
};

// grid (width / 128, G); a thread owns one feature and the points n = g, g + G, ...
__global__ void __launch_bounds__(128) top_bwd_kernel(const TopBwdParams p) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  const int g = blockIdx.y;
  if (m >= p.width) return;
  const float wl = p.w_out[m];
  const size_t ldz = (size_t)p.ldz, ldo = (size_t)p.ldo;
  float dwp = 0.f;
  for (int64_t n = g; n < p.N; n += p.G) {
    const size_t row = (size_t)n * p.P;
    const float* zr = p.Z + row * ldz + m;
    const float z0 = zr[0], zt = zr[(size_t)(p.P - 1) * ldz];
    const ActD A = act_derivs(p.act, z0);
    const float go = p.gop[n], gfn = p.gf ? p.gf[n] : 0.f;
    const float tb = p.c * go * wl;  // adjoint of the collapsed top h_top
    const float hb0 = gfn * wl;      // adjoint of h0
    float szz = 0.f;
    const float* __restrict__ zs = zr + ldz;
    uint16_t* __restrict__ oz = p.out + (row + 1) * ldo + m;
#pragma unroll 4
    for (int r = 0; r < p.P - 2; ++r) {
      const float z1 = zs[(size_t)r * ldz];
      const float w = p.jw ? p.jw[r] : 1.f;
      szz = fmaf(w * z1, z1, szz);
      ptx::store_planes(oz + (size_t)r * ldo, p.pstride, p.nplanes, 2.f * A.d2 * w * z1 * tb);
    }
    ptx::store_planes(p.out + (row + p.P - 1) * ldo + m, p.pstride, p.nplanes, A.d1 * tb);
    ptx::store_planes(p.out + row * ldo + m, p.pstride, p.nplanes, A.d1 * hb0 + (A.d2 * zt + A.d3 * szz) * tb);
    const float top = A.d1 * zt + A.d2 * szz;
    dwp += gfn * A.d0 + p.c * go * top;
  }
  p.dw_part[(size_t)g * p.width + m] = dwp;
}

// part[g, m] = sum over rows r = g, g + G, ... < nrows of src[row0 + r * stride, m]
// (bf16 planes if src != nullptr, else fp32 `srcf`); grid (ceil(ncols / 128), G)
__global__ void __launch_bounds__(128) colsum_kernel(const uint16_t* __restrict__ src, int64_t pstride, int nplanes,
                                                     const float* __restrict__ srcf, int64_t nrows, int64_t stride,
                                                     int ld, int ncols, int G, float* __restrict__ part) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  const int g = blockIdx.y;
  if (m >= ncols) return;
  float acc = 0.f;
  for (int64_t r = g; r < nrows; r += G) {
    const size_t i = (size_t)(r * stride) * ld + m;
    acc += srcf ? srcf[i] : ptx::planes_val(src + i, pstride, nplanes);
  }
  part[(size_t)g * ncols + m] = acc;
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
