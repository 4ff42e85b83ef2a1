// Write-bandwidth microtest: which store width / shape reaches the HBM write ceiling
// (cudaMemsetAsync: 7.28 TB/s on this B200). 2.56 GB buffer, CUDA events, best of 10.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int W>  // bytes per store per thread: 8, 16, 32
__global__ void write_k(uint8_t* __restrict__ p, size_t n_bytes) {
  const size_t stride = (size_t)gridDim.x * blockDim.x * W;
  for (size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * W; i < n_bytes; i += stride) {
    if constexpr (W == 8) {
      *reinterpret_cast<uint2*>(p + i) = make_uint2(7u, 7u);
    } else if constexpr (W == 16) {
      *reinterpret_cast<uint4*>(p + i) = make_uint4(7u, 7u, 7u, 7u);
    } else {
      asm volatile("st.global.v8.f32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};" ::"l"(p + i), "f"(1.0f) : "memory");
    }
  }
}

// the seed's pattern: one block per "point", rows of ld bf16 pairs (two planes), 4 features
// per thread (8-byte stores) vs 8 features per thread (16-byte stores)
template <int F>
__global__ void seed_like(uint16_t* __restrict__ hi, uint16_t* __restrict__ lo, int ld, int P) {
  const size_t n = blockIdx.x;
  const int m = F * threadIdx.x;
  if (m >= ld) return;
  for (int r = 0; r < P; ++r) {
    const size_t off = (n * P + r) * (size_t)ld + m;
    if constexpr (F == 4) {
      *reinterpret_cast<uint2*>(hi + off) = make_uint2(r, r);
      *reinterpret_cast<uint2*>(lo + off) = make_uint2(r, r);
    } else {
      *reinterpret_cast<uint4*>(hi + off) = make_uint4(r, r, r, r);
      *reinterpret_cast<uint4*>(lo + off) = make_uint4(r, r, r, r);
    }
  }
}

int main() {
  const size_t n = 2560ull * 1024 * 1024;
  uint8_t* p;
  cudaMalloc(&p, n);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto bench = [&](const char* name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e9f;
    for (int i = 0; i < 10; ++i) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%-34s %.2f TB/s  %.3f ms\n", name, n / best / 1e9, best);
  };
  bench("cudaMemsetAsync", [&] { cudaMemsetAsync(p, 7, n); });
  for (int blocks : {148 * 4, 148 * 8, 148 * 16, 148 * 64}) {
    char s[64];
    snprintf(s, 64, "grid-stride 8B  blocks=%d", blocks);
    bench(s, [&] { write_k<8><<<blocks, 256>>>(p, n); });
    snprintf(s, 64, "grid-stride 16B blocks=%d", blocks);
    bench(s, [&] { write_k<16><<<blocks, 256>>>(p, n); });
    snprintf(s, 64, "grid-stride 32B blocks=%d", blocks);
    bench(s, [&] { write_k<32><<<blocks, 256>>>(p, n); });
  }
  const int ld = 768, P = 52;
  const size_t pts = n / 4 / ((size_t)ld * P);  // two bf16 planes
  uint16_t* hi = reinterpret_cast<uint16_t*>(p);
  uint16_t* lo = hi + pts * P * ld;
  bench("seed-like 4 feats/thread (8B)", [&] { seed_like<4><<<(unsigned)pts, 192>>>(hi, lo, ld, P); });
  bench("seed-like 8 feats/thread (16B)", [&] { seed_like<8><<<(unsigned)pts, 96>>>(hi, lo, ld, P); });
  printf("(seed-like bytes = %.2f GB)\n", 4.0 * pts * P * ld / 1e9);
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
