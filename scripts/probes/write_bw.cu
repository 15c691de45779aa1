// Pure-write HBM bandwidth on B200 by store flavour: is the 3.8 TB/s torch fill figure a
// hardware ceiling or an artifact of the store instruction? (context for dispatch's permute)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void stg128(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(0, 0, 0, 0);
}
__global__ void stg128_cs(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(p + i, make_uint4(0, 0, 0, 0));
}
__global__ void stg256(uint4* p, size_t n) {   // v8.b32 (256-bit) stores
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; 2 * i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t z = 0;
    asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" :: "l"(p + 2 * i), "r"(z) : "memory");
  }
}
// each CTA streams 16 KB smem chunks out with cp.async.bulk (TMA 1-D store)
__global__ void bulk_store(uint8_t* p, size_t bytes) {
  extern __shared__ __align__(128) uint8_t sm[];
  for (int i = threadIdx.x; i < 32768 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const size_t chunk = 32768;
    for (size_t off = blockIdx.x * chunk; off < bytes; off += (size_t)gridDim.x * chunk) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(p + off),
                   "r"((uint32_t)__cvta_generic_to_shared(sm)), "r"((uint32_t)chunk) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
__global__ void copy128(const uint4* a, uint4* b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void read128(const uint4* a, size_t n, uint32_t* sink) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(a + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678) *sink = acc;
}

template <class F>
float best_ms(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaDeviceSynchronize();
  float best = 1e9;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  const size_t bytes = 1ull << 31, n16 = bytes / 16;
  uint8_t *a, *b;
  uint32_t* sink;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMalloc(&sink, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(bulk_store, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  auto gbs = [&](float ms, double by) { return by / ms / 1e6; };
  printf("{");
  for (int occ : {4, 8, 16}) {
    const int grid = sms * occ;
    printf("\"stg128_x%d\": %.0f, ", occ, gbs(best_ms([&] { stg128<<<grid, 256>>>((uint4*)a, n16); }), bytes));
    printf("\"stg128_cs_x%d\": %.0f, ", occ, gbs(best_ms([&] { stg128_cs<<<grid, 256>>>((uint4*)a, n16); }), bytes));
    printf("\"stg256_x%d\": %.0f, ", occ, gbs(best_ms([&] { stg256<<<grid, 256>>>((uint4*)a, n16); }), bytes));
    printf("\"copy_x%d\": %.0f, ", occ, gbs(best_ms([&] { copy128<<<grid, 256>>>((uint4*)a, (uint4*)b, n16); }), 2.0 * bytes));
    printf("\"read_x%d\": %.0f, ", occ, gbs(best_ms([&] { read128<<<grid, 256>>>((uint4*)a, n16, sink); }), bytes));
  }
  for (int occ : {1, 2, 4})
    printf("\"bulk_x%d\": %.0f, ", occ,
           gbs(best_ms([&] { bulk_store<<<sms * occ, 128, 32768>>>(a, bytes); }), bytes));
  printf("\"memset\": %.0f}\n", gbs(best_ms([&] { cudaMemsetAsync(a, 0, bytes); }), bytes));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
