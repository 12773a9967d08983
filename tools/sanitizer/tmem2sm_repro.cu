// Minimal reproducer for the compute-sanitizer racecheck report on the 2-SM TMEM allocator
// (profiles/r2_sanitizer_*.log): clusters of 2 CTAs whose ONLY shared-memory traffic is the
// tcgen05.alloc.cta_group::2 write of the TMEM base address and one read of it after
// tcgen05.fence + cluster barrier -- the same sequence as gemm_bf16_tn_kernel<*, *, 2, *>.
//   variant 0: one cluster, static shared slot
//   variant 1: 74 clusters (every SM), the slot at the end of 200 KB of dynamic shared memory
//   variant 2: variant 1 launched 4x back to back with programmatic dependent launch (the
//              GEMM's launch mode: the next grid's alloc overlaps the previous grid's tail)
// If racecheck reports "Write access at <pc before the kernel> / Read access at the alloc"
// here, the hazard is the sanitizer's view of the allocator itself, not the GEMM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tmem2sm tools/sanitizer/tmem2sm_repro.cu
//   compute-sanitizer --tool racecheck /tmp/tmem2sm [0|1|2]
#include <cstdio>
#include <cstdint>
#include <cstdlib>

template <bool DYN>
__global__ void __cluster_dims__(2, 1, 1) k(unsigned* out, int slot_off) {
  __shared__ uint32_t s_slot;
  extern __shared__ uint8_t dyn[];
  uint32_t* slot = DYN ? reinterpret_cast<uint32_t*>(dyn + slot_off) : &s_slot;
  const int warp = threadIdx.x / 32;
  if (warp == 2) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(slot);
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(a) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t base = *slot;
  if (threadIdx.x == 0) out[blockIdx.x] = base;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(base) : "memory");
  }
}

int main(int argc, char** argv) {
  const int variant = argc > 1 ? atoi(argv[1]) : 0;
  unsigned* d;
  cudaMalloc(&d, 148 * sizeof(unsigned));
  const int smem = 200 * 1024;
  if (variant == 0) {
    k<false><<<2, 256>>>(d, 0);
  } else {
    cudaFuncSetAttribute(k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = variant == 2 ? 1 : 0;
    for (int r = 0; r < (variant == 2 ? 4 : 1); ++r)
      cudaLaunchKernelEx(&cfg, k<true>, d, smem - 16);
  }
  unsigned h[2];
  cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("variant %d: tmem base of CTAs 0, 1: %u %u (%s)\n", variant, h[0], h[1], cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
