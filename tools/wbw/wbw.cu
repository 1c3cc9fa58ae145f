// Write-only HBM bandwidth probes (diagnostic, not product code): 16-byte vector stores and
// TMA bulk stores from shared memory, persistent grids.
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_st16(uint4 *p, long long n16) {
  const uint4 v = make_uint4(1, 2, 3, 4);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n16; i += (long long)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void k_bulk(unsigned char *p, long long nbytes, int chunk) {
  extern __shared__ __align__(128) unsigned char sm[];
  for (int i = threadIdx.x; i < chunk / 16; i += blockDim.x) reinterpret_cast<uint4 *>(sm)[i] = make_uint4(5, 6, 7, 8);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sm);
    long long nch = nbytes / chunk;
    int inflight = 0;
    for (long long c = blockIdx.x; c < nch; c += gridDim.x) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p + c * chunk), "r"(sa), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (++inflight >= 8) { asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory"); inflight = 4; }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
extern "C" float run(int which, void *p, long long nbytes, int blocks, int threads, int chunk) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  if (which == 1) cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, chunk);
  cudaEventRecord(a);
  if (which == 0) k_st16<<<blocks, threads>>>((uint4 *)p, nbytes / 16);
  else k_bulk<<<blocks, threads, chunk>>>((unsigned char *)p, nbytes, chunk);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}
