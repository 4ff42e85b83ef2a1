// Microtest: does the allocation kind change HBM write cost on B200?
// ncu reports every layer-kernel store (cudaMalloc'd slot blocks) as "L2 Compression Input
// Sectors" with 0% success. Compare a streaming fp16-plane-like write into
//   (a) cudaMalloc memory, (b) cuMemCreate COMP_NONE, (c) cuMemCreate COMP_GENERIC
// by CUDA events (best of 20, 4 GiB each) and report the pointer's compressibility.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 comp_alloc.cu -lcuda -o comp_alloc
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { auto e_ = (x); if (e_ != 0) { printf("error %d at %s:%d\n", (int)e_, __FILE__, __LINE__); return 1; } } while (0)

__global__ void write_kernel(uint4* p, size_t n, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u + seed;  // non-compressible-looking data
    p[i] = make_uint4(h, h ^ 0x9e3779b9u, h * 3u, h + 12345u);
  }
}

static int vmm_alloc(size_t bytes, int comp, void** out, size_t* sz) {
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = 0;
  prop.allocFlags.compressionType = comp ? CU_MEM_ALLOCATION_COMP_GENERIC : CU_MEM_ALLOCATION_COMP_NONE;
  size_t g = 0;
  CK(cuMemGetAllocationGranularity(&g, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  bytes = (bytes + g - 1) / g * g;
  CUmemGenericAllocationHandle h;
  CK(cuMemCreate(&h, bytes, &prop, 0));
  CUdeviceptr ptr;
  CK(cuMemAddressReserve(&ptr, bytes, 0, 0, 0));
  CK(cuMemMap(ptr, bytes, 0, h, 0));
  CUmemAccessDesc acc = {};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(ptr, bytes, &acc, 1));
  CUmemAllocationProp got = {};
  CK(cuMemGetAllocationPropertiesFromHandle(&got, h));
  printf("  vmm comp requested %d -> granted %d\n", comp, (int)got.allocFlags.compressionType);
  *out = (void*)ptr;
  *sz = bytes;
  return 0;
}

int main() {
  CK(cudaSetDevice(0));
  CK(cudaFree(0));
  int gen = 0;
  CK(cuDeviceGetAttribute(&gen, CU_DEVICE_ATTRIBUTE_GENERIC_COMPRESSION_SUPPORTED, 0));
  printf("generic compression supported: %d\n", gen);
  const size_t bytes = (size_t)4 << 30;
  void* bufs[3];
  size_t sz[3] = {bytes, 0, 0};
  CK(cudaMalloc(&bufs[0], bytes));
  if (vmm_alloc(bytes, 0, &bufs[1], &sz[1])) return 1;
  if (vmm_alloc(bytes, 1, &bufs[2], &sz[2])) return 1;
  const char* names[3] = {"cudaMalloc", "cuMemCreate COMP_NONE", "cuMemCreate COMP_GENERIC"};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep)
    for (int k = 0; k < 3; ++k) {
      const size_t n = bytes / 16;
      float best = 1e9f;
      for (int it = 0; it < 20; ++it) {
        cudaEventRecord(a);
        write_kernel<<<148 * 8, 512>>>((uint4*)bufs[k], n, it);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      CK(cudaGetLastError());
      printf("rep %d %-26s write %.3f ms  %.0f GB/s\n", rep, names[k], best, bytes / best / 1e6);
    }
  return 0;
}
