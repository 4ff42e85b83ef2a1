// wgrad.cuh — weight gradients of the differentiable path on tcgen05 (SURVEY NEXT-3,
// PINN training through the collapsed forward):
//
//   dW_l[o, i] = sum over slot rows r of Zbar_l[r, o] * B_{l-1}[r, i]     (r < N*P)
//
// Zbar_l (the adjoint block of layer l) and B_{l-1} (the recorded input block) are stored as
// the forward stores every slot block: row-major [rows, ld], bf16 planes (jet_layer.cuh). For
// this GEMM the contraction runs over the ROWS, so both operands are MN-major: a TMA box
// {64 features, 64 rows} lands as 64 rows of 128 bytes (SWIZZLE_128B), the canonical
// MN-major atom, and tcgen05.mma reads it with a_major = b_major = MN.
//
// Tiling: CTA pairs (cta_group::2), M = 256 output features o (128 per CTA), N = 256 or 128
// input features i (half of the B columns staged by each CTA). The K = N*P rows are long
// (851,968 at C1), so each (o tile, i tile) is split into `splits` fixed K ranges (one work
// unit each, persistent pairs); a unit accumulates in TMEM over chunks of kChunkKB 64-row
// blocks (in the precision mode's plane schedule, jet_layer.cuh for_each_group), and the
// epilogue warps add each finished chunk into fp32 registers, so no accumulator ever sees
// more than kChunkKB * 4 MMA steps of the leading product (the tensor cores' round-toward-zero
// accumulation). A unit writes its [256, N] partial; wgrad_reduce_kernel sums
// the splits of every element in a fixed order into the caller's dW (= or +=). Bitwise
// deterministic run to run.
#pragma once
#include <cstdint>

#include "jet_layer.cuh"

namespace ctm {

constexpr int kWgChunkKB = 16;   // 64-row K blocks per TMEM accumulation chunk (1024 rows)
constexpr int kWgSlots = 6;                     // 6 x 32 KB operand ring (plane slots, as jet_layer.cuh)
constexpr int kWgSlotBytes = 32 * 1024;
constexpr int kWgradSmem = kWgSlots * kWgSlotBytes + 1024 /*align*/ + 256 /*barriers*/;

struct WgradParams {
  int64_t rows;        // K: slot rows
  int k_blocks;        // ceil(rows / 64)
  int m_pairs;         // Mout / 256
  int n_tiles;         // ceil(Kin / N)
  int splits;          // K ranges per (m, n) tile
  int kb_per_split;    // ceil(k_blocks / splits)
  int nplanes;         // 3: fp32 mode, 2: fast mode (jet_layer.cuh)
  float* part;         // [units][256][N], unit = (m_pair * n_tiles + n_tile) * splits + split
};

// F16: the fp16x3 mode (jet_layer.cuh kFlagF16): both operands two fp16 planes (the residual
// lifted by 2^11) with ONE power-of-two scale per block (grad mode records uniform scales);
// per chunk, phase 1 runs p1*p0 + p0*p1 over the chunk's K (carrying 2^11), phase 2 p0*p0,
// its first MMA scaling the accumulator by 2^-11 (ptx::mma_f16_pair_unlift). The partial is
// scale_Z * scale_B times the gradient; wgrad_reduce_kernel undoes it.
template <int N, bool F16 = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(320, 1)
    wgrad_kernel(const __grid_constant__ CUtensorMap tmZ, const __grid_constant__ CUtensorMap tmB,
                 const WgradParams p) {
  static_assert(N == 128 || N == 256, "N tile");
  constexpr int kHalfN = N / 2;                         // B columns staged by each CTA
  constexpr uint32_t kABytes = 128 * 64 * 2;            // 128 o x 64 rows (two 64-o atoms)
  constexpr uint32_t kBBytes = kHalfN * 64 * 2;         // N/2 i x 64 rows
  constexpr uint32_t kSlot = kWgSlotBytes;
  static_assert(kABytes + kBBytes <= (uint32_t)kSlot, "slot size");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kWgSlots * kSlot);
  uint64_t* empty_bar = full_bar + kWgSlots;
  uint64_t* tmem_full_bar = empty_bar + kWgSlots;   // [2]
  uint64_t* tmem_empty_bar = tmem_full_bar + 2;    // [2] (leader)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int npairs = gridDim.x >> 1;
  const int units = p.m_pairs * p.n_tiles * p.splits;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmZ);
    ptx::tma_prefetch_desc(&tmB);
    for (int s = 0; s < kWgSlots; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tmem_full_bar[b], 1);
      ptx::mbar_init(&tmem_empty_bar[b], 16);  // 8 epilogue warps in each CTA of the pair
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc_pair<kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  ptx::pdl_launch_dependents();
  ptx::pdl_wait_prior();

  // unit u: its tile, its K range [kb0, kb1) in 64-row blocks, and its chunk count
  auto unit_range = [&](int u, int& mp, int& nt, int& kb0, int& kb1) {
    const int tile = u / p.splits, split = u % p.splits;
    mp = tile / p.n_tiles;
    nt = tile % p.n_tiles;
    kb0 = split * p.kb_per_split;
    kb1 = min(p.k_blocks, kb0 + p.kb_per_split);
    if (kb1 < kb0) kb1 = kb0;
  };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      uint32_t it = 0;
      for (int u = pair; u < units; u += npairs) {
        int mp, nt, kb0, kb1;
        unit_range(u, mp, nt, kb0, kb1);
        const int o0 = mp * 256 + (int)rank * 128;
        const int i0 = nt * N + (int)rank * kHalfN;
        for (int c0 = kb0; c0 < kb1; c0 += kWgChunkKB) {
          const int nkb = min(kWgChunkKB, kb1 - c0);
          for_each_group(F16 ? 2 : p.nplanes, F16, nkb, [&](int, int kb, int nslots) {
            const int r0 = (c0 + kb) * 64;
            for (int pl = 0; pl < nslots; ++pl, ++it) {
              const uint32_t s = it % kWgSlots;
              ptx::mbar_wait(&empty_bar[s], ((it / kWgSlots) & 1u) ^ 1u);
              uint8_t* st = smem + s * kSlot;
              if (rank == 0) ptx::mbar_arrive_expect_tx(&full_bar[s], 2u * (kABytes + kBBytes));
              ptx::tma_load_3d_pair(st, &tmZ, &full_bar[s], o0, r0, pl);
              ptx::tma_load_3d_pair(st + 8192, &tmZ, &full_bar[s], o0 + 64, r0, pl);
#pragma unroll
              for (int j = 0; j < kHalfN / 64; ++j)
                ptx::tma_load_3d_pair(st + kABytes + j * 8192, &tmB, &full_bar[s], i0 + 64 * j, r0, pl);
            }
          });
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader warp, elected lane)
    if (rank == 0) {
      const uint32_t idesc = F16 ? ptx::idesc_f16_mn(256, (uint32_t)N) : ptx::idesc_bf16_mn(256, (uint32_t)N);
      const uint64_t desc0 = ptx::smem_desc_mn(ptx::smem_u32(smem), 8192, 1024);
      constexpr uint64_t kS = kSlot >> 4, kB = kABytes >> 4;
      uint32_t it = 0, chunk = 0;
      for (int u = pair; u < units; u += npairs) {
        int mp, nt, kb0, kb1;
        unit_range(u, mp, nt, kb0, kb1);
        for (int c0 = kb0; c0 < kb1; c0 += kWgChunkKB, ++chunk) {
          const int nkb = min(kWgChunkKB, kb1 - c0);
          const uint32_t buf = chunk & 1u;
          ptx::mbar_wait(&tmem_empty_bar[buf], ((chunk >> 1) & 1u) ^ 1u);
          ptx::tc_fence_after();
          const uint32_t d_tmem = tmem_base + buf * (uint32_t)N;
          uint32_t acc = 0;
          bool unlift = F16;  // fp16x3: the chunk's first p0*p0 MMA scales the corrections by 2^-11
          for_each_group(F16 ? 2 : p.nplanes, F16, nkb, [&](int, int, int nslots) {
            for (int pl = 0; pl < nslots; ++pl)
              ptx::mbar_wait(&full_bar[(it + pl) % kWgSlots], ((it + pl) / kWgSlots) & 1u);
            ptx::tc_fence_after();
            const uint64_t dA0 = desc0 + (it % kWgSlots) * kS, dA1 = desc0 + ((it + 1) % kWgSlots) * kS,
                           dA2 = desc0 + ((it + 2) % kWgSlots) * kS;
            if (ptx::elect_one()) {
#pragma unroll
              for (int ks = 0; ks < 4; ++ks) {  // 16 rows = 2 K groups of 8 rows = 2048 bytes
                const uint64_t o = 128u * ks;
                if (nslots == 2) {
                  ptx::mma_bf16_pair(d_tmem, dA1 + o, dA0 + kB + o, idesc, acc);
                  ptx::mma_bf16_pair(d_tmem, dA0 + o, dA1 + kB + o, idesc, 1u);
                  if (!F16) ptx::mma_bf16_pair(d_tmem, dA0 + o, dA0 + kB + o, idesc, 1u);
                } else if (F16 && unlift) {
                  ptx::mma_f16_pair_unlift(d_tmem, dA0 + o, dA0 + kB + o, idesc);
                  unlift = false;
                } else if (nslots == 3) {
                  ptx::mma_bf16_pair(d_tmem, dA2 + o, dA0 + kB + o, idesc, acc);
                  ptx::mma_bf16_pair(d_tmem, dA1 + o, dA1 + kB + o, idesc, 1u);
                  ptx::mma_bf16_pair(d_tmem, dA0 + o, dA2 + kB + o, idesc, 1u);
                  ptx::mma_bf16_pair(d_tmem, dA1 + o, dA0 + kB + o, idesc, 1u);
                  ptx::mma_bf16_pair(d_tmem, dA0 + o, dA1 + kB + o, idesc, 1u);
                } else {
                  ptx::mma_bf16_pair(d_tmem, dA0 + o, dA0 + kB + o, idesc, acc);
                }
                acc = 1u;
              }
              for (int pl = 0; pl < nslots; ++pl) ptx::mma_commit_pair(&empty_bar[(it + pl) % kWgSlots]);
            }
            __syncwarp();
            acc = 1u;
            it += nslots;
          });
          if (ptx::elect_one()) ptx::mma_commit_pair(&tmem_full_bar[buf]);
          __syncwarp();
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..9, both CTAs)
    const int q = warp & 3;            // TMEM lane quadrant
    const int h = (warp - 2) >> 2;     // column half
    constexpr int kCols = kHalfN;      // columns per thread
    uint32_t chunk = 0;
    for (int u = pair; u < units; u += npairs) {
      int mp, nt, kb0, kb1;
      unit_range(u, mp, nt, kb0, kb1);
      float sum[kCols];
#pragma unroll
      for (int c = 0; c < kCols; ++c) sum[c] = 0.f;
      for (int c0 = kb0; c0 < kb1; c0 += kWgChunkKB, ++chunk) {
        const uint32_t buf = chunk & 1u;
        ptx::mbar_wait(&tmem_full_bar[buf], (chunk >> 1) & 1u);
        ptx::tc_fence_after();
        const uint32_t taddr = tmem_base + buf * (uint32_t)N + (uint32_t)(h * kCols) + ((uint32_t)(q * 32) << 16);
#pragma unroll
        for (int c = 0; c < kCols; c += 32) {
          float v[32];
          ptx::tmem_ld32(taddr + (uint32_t)c, v);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) sum[c + j] += v[j];
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_remote(&tmem_empty_bar[buf], 0);
      }
      // this thread's row o of the unit's [256, N] partial, columns [h * N/2, (h + 1) * N/2)
      float* dst = p.part + ((size_t)u * 256 + rank * 128 + q * 32 + lane) * N + h * kCols;
#pragma unroll
      for (int c = 0; c < kCols; c += 4)
        *reinterpret_cast<float4*>(dst + c) = make_float4(sum[c], sum[c + 1], sum[c + 2], sum[c + 3]);
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_pair<kTmemCols>(tmem_base);
  }
}

// dW[o, i] (=|+=) sum_s part[unit(o, i, s)][o % 256][i % N] for o < rows_out, i < cols_in
// (the caller's nn.Linear layout [rows_out, cols_in]); splits summed in order s = 0, 1, ...
// (fp16x3: ra / rb are the operands' scale records, the sum is divided by their uniform scales)
__global__ void wgrad_reduce_kernel(const float* __restrict__ part, int N, int n_tiles, int splits, int rows_out,
                                    int cols_in, float* __restrict__ dW, int accumulate,
                                    const F16Rec* __restrict__ ra = nullptr, const F16Rec* __restrict__ rb = nullptr) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= (int64_t)rows_out * cols_in) return;
  const int o = (int)(k / cols_in), i = (int)(k % cols_in);
  const int tile = (o / 256) * n_tiles + i / N;
  const float* pp = part + ((size_t)tile * splits * 256 + (o % 256)) * N + (i % N);
  float s = 0.f;
  for (int sp = 0; sp < splits; ++sp) s += pp[(size_t)sp * 256 * N];
  if (ra) s /= ra->scale[0] * rb->scale[0];  // powers of two: exact
  dW[k] = accumulate ? dW[k] + s : s;
}

}  // namespace ctm
