// Microtest: does tcgen05.ld.32x32b.x{1,2,4,8,16} accept column offsets that are not
// multiples of the load width? Fill TMEM with tcgen05.st (aligned), read back unaligned.
#include <cstdio>
#include <cstdint>
__global__ void k(int* bad, float* sample) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = slot + ((uint32_t)(warp * 32) << 16);
  const int row = warp * 32 + lane;
  for (int c = 0; c < 512; c += 16) {
    uint32_t r[16];
    for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(row * 1000.f + c + i);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(base + c), "r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5]),"r"(r[6]),"r"(r[7]),
                 "r"(r[8]),"r"(r[9]),"r"(r[10]),"r"(r[11]),"r"(r[12]),"r"(r[13]),"r"(r[14]),"r"(r[15]));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  int nbad = 0;
  const int offs[6] = {0, 1, 3, 5, 13, 101};
  for (int t = 0; t < 6; ++t) {
    const int c = offs[t];
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),
                   "=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]) : "r"(base + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 16; ++i) if (__uint_as_float(r[i]) != row * 1000.f + c + i) ++nbad;
    if (row == 5) sample[t] = __uint_as_float(r[0]);
    uint32_t q[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(q[0]),"=r"(q[1]),"=r"(q[2]),"=r"(q[3]) : "r"(base + c + 2));
    uint32_t o;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(o) : "r"(base + c + 7));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 4; ++i) if (__uint_as_float(q[i]) != row * 1000.f + c + 2 + i) ++nbad;
    if (__uint_as_float(o) != row * 1000.f + c + 7) ++nbad;
  }
  atomicAdd(bad, nbad);
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}
int main() {
  int* bad; float* s; cudaMalloc(&bad, 4); cudaMalloc(&s, 64); cudaMemset(bad, 0, 4);
  k<<<1, 128>>>(bad, s);
  cudaError_t e = cudaDeviceSynchronize();
  int h = -1; float hs[6]; cudaMemcpy(&h, bad, 4, cudaMemcpyDeviceToHost); cudaMemcpy(hs, s, 24, cudaMemcpyDeviceToHost);
  printf("err=%s mismatches=%d sample=%g %g %g %g %g %g\n", cudaGetErrorString(e), h, hs[0], hs[1], hs[2], hs[3], hs[4], hs[5]);
  return 0;
}
