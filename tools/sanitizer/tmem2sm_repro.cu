// Minimal reproducer for the compute-sanitizer racecheck report on the 2-SM TMEM allocator
// (profiles/r2_sanitizer_*.log): a cluster of 2 CTAs whose ONLY shared-memory traffic is the
// tcgen05.alloc.cta_group::2 write of the TMEM base address and one read of it after
// tcgen05.fence + cluster barrier -- the same sequence as gemm_bf16_tn_kernel<*, *, 2, *>.
// If racecheck reports "Write access at <pc before the kernel> / Read access at the alloc"
// here too, the hazard is the sanitizer's view of the allocator itself, not the GEMM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tmem2sm tools/sanitizer/tmem2sm_repro.cu
//   compute-sanitizer --tool racecheck /tmp/tmem2sm
#include <cstdio>
#include <cstdint>

__global__ void __cluster_dims__(2, 1, 1) k(unsigned* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(&slot);
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(a) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t base = slot;
  if (threadIdx.x == 0) out[blockIdx.x] = base;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(base) : "memory");
  }
}

int main() {
  unsigned* d;
  cudaMalloc(&d, 2 * sizeof(unsigned));
  k<<<2, 128>>>(d);
  unsigned h[2];
  cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("tmem base per CTA: %u %u (%s)\n", h[0], h[1], cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
