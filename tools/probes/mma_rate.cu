// Tensor-core issue-rate probe for the attention kernel's MMA shapes (one CTA per SM): SM cycles
// per tcgen05.mma when one warp issues R back-to-back MMAs, with the same shared-memory
// descriptors as attn_tc.cuh, issued (a) from one divergent lane (`if (lane == 0)`, the round-1
// kernels) or (b) by the whole warp with the lane elected inside the asm (umma_*_w).
//   qk   SS  M=128 N=128 K=16  (S = Q K^T)     pv  TS  M=128 N=128 K=16  (O += P V)
//   n256 SS  M=128 N=256 K=16  (the GEMM's shape)   mix 8 qk + 8 pv
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o /tmp/mma_rate tools/probes/mma_rate.cu
#include <cstdio>
#include "../../paper_2602_16603_b200/csrc/common.cuh"

using namespace fp;

constexpr int R = 512;  // MMAs per timed run

template <int MODE, bool WARP>
__global__ void __launch_bounds__(128, 1) probe(unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + 32768;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 98304);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = *slot;
  if (warp == 0 && (WARP || lane == 0)) {
    constexpr uint32_t id128 = make_idesc_bf16(128, 128, false);
    constexpr uint32_t id256 = make_idesc_bf16(128, 256, false);
    constexpr uint32_t idpv = make_idesc_bf16(128, 128, true);
    const uint32_t qa = smem_u32(sA), kb = smem_u32(sB);
    const uint64_t a0 = make_sdesc_sw128(qa, 16, 1024), b0 = make_sdesc_sw128(kb, 16, 1024);
    const uint64_t v0 = make_sdesc_sw128(kb, 16384, 1024);
    for (int rep = 0; rep < 2; ++rep) {  // rep 0 warms up
      const unsigned long long t0 = clock64();
      for (int g = 0; g < R / 8; ++g) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t off = (uint64_t)(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
          const bool qk = MODE == 0 || MODE == 2 || (MODE == 3 && (g & 1) == 0);
          if (qk) {
            const uint32_t id = MODE == 2 ? id256 : id128;
            const uint32_t d = MODE == 3 ? tb + 128 : tb;
            if (WARP) umma_bf16_ss_w(d, a0 + off, b0 + off, id, kk > 0);
            else umma_bf16_ss(d, a0 + off, b0 + off, id, kk > 0);
          } else {
            const uint64_t vo = (uint64_t)((kk * 2048) >> 4);
            if (WARP) umma_bf16_ts_w(tb + 256, tb + kk * 8, v0 + vo, idpv, 1);
            else umma_bf16_ts(tb + 256, tb + kk * 8, v0 + vo, idpv, 1);
          }
        }
      }
      if (WARP) tc_commit_w(bar);
      else tc_commit(bar);
      mbar_wait(bar, rep & 1);
      const unsigned long long t1 = clock64();
      if (rep == 1 && lane == 0) out[blockIdx.x] = t1 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tb);
  }
}

// N sweep: SS M=128 N=NN K=16 back to back into one accumulator; ACC: 0 restart every 8 MMAs,
// 1 always accumulate, 2 alternate between two accumulators every MMA
template <int NN, int ACC>
__global__ void __launch_bounds__(128, 1) probe_n(unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 98304);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = *slot;
  if (warp == 0 && lane == 0) {
    constexpr uint32_t id = make_idesc_bf16(128, NN, false);
    const uint64_t a0 = make_sdesc_sw128(smem_u32(smem), 16, 1024);
    const uint64_t b0 = make_sdesc_sw128(smem_u32(smem + 32768), 16, 1024);
    for (int rep = 0; rep < 2; ++rep) {
      const unsigned long long t0 = clock64();
      for (int g = 0; g < R / 8; ++g) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t off = (uint64_t)(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
          const uint32_t d = ACC == 2 ? tb + (kk & 1) * 256 : tb;
          const uint32_t acc = ACC == 0 ? (kk > 0) : ACC == 1 ? 1u : (kk > 1);
          umma_bf16_ss(d, a0 + off, b0 + off, id, acc);
        }
      }
      tc_commit(bar);
      mbar_wait(bar, rep & 1);
      const unsigned long long t1 = clock64();
      if (rep == 1) out[blockIdx.x] = t1 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tb);
  }
}

template <int NN, int ACC>
void run_n(unsigned long long* d) {
  const int smem = 98304 + 1024 + 64;
  cudaFuncSetAttribute(probe_n<NN, ACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_n<NN, ACC><<<148, 128, smem>>>(d);
  unsigned long long h[148];
  cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148 * (double)R;
  const double floor_ = 128.0 * NN / 256.0;
  printf("SS M=128 N=%3d %-22s %7.1f cycles / MMA (floor %.0f: %3.0f%%) %s\n", NN,
         ACC == 0 ? "restart every 8" : ACC == 1 ? "always accumulate" : "2 accumulators alt.",
         avg, floor_, 100.0 * floor_ / avg, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

template <int MODE, bool WARP>
void run(const char* name, unsigned long long* d) {
  const int smem = 98304 + 1024 + 64;
  cudaFuncSetAttribute(probe<MODE, WARP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<MODE, WARP><<<148, 128, smem>>>(d);
  unsigned long long h[148];
  cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148 * (double)R;
  const double ideal = MODE == 2 ? 128.0 : 64.0;
  printf("%-6s %-13s %7.1f cycles / MMA (floor %.0f: %3.0f%%) %s\n", name,
         WARP ? "warp-elected" : "lane-0 issue", avg, ideal, 100.0 * ideal / avg,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  run<0, false>("qk", d); run<0, true>("qk", d);
  run<1, false>("pv", d); run<1, true>("pv", d);
  run<2, false>("n256", d); run<2, true>("n256", d);
  run<3, false>("mix", d); run<3, true>("mix", d);
  run_n<64, 0>(d); run_n<128, 0>(d); run_n<192, 0>(d); run_n<256, 0>(d);
  run_n<64, 1>(d); run_n<128, 1>(d); run_n<256, 1>(d);
  run_n<64, 2>(d); run_n<128, 2>(d); run_n<256, 2>(d);
  return 0;
}
