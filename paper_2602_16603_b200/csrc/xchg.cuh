// Tensor-parallel exchange of the row-parallel projections (o_proj, down_proj).
//
// Megatron partitioning: qkv_proj / gate_up_proj are column-parallel (heads, ffn sharded) and
// need no communication; o_proj / down_proj are row-parallel, so each rank's GEMM yields a
// partial sum of the full [M, hidden] output. The reference only models this as a duration
// scale `/tp * (1 + tp_comm_overhead)` (prefillsim/cost_model.py:99-100,166).
//
// The exchange GEMM stores its bf16 partial into this rank's double-buffered exchange slot and
// the last CTA publishes `ready = xcount + 1` (tp_publish_partial). This kernel, the second
// kernel of the same timeline entry, waits for every rank's `ready`, then reads all partials
// over peer memory (NVLink P2P loads) and folds them into the residual stream:
//     h[m, :] = bf16( h[m, :] + part_0[m, :] + part_1[m, :] + ... )     (fp32 sum, rank order)
// The summation order is the same on every rank, so the replicated residual streams stay
// bit-identical across ranks. Buffer reuse is safe without a second barrier: a rank overwrites
// slot (x & 1) at exchange x only after its exchange x-1 saw every peer's exchange-(x-1)
// partial, which each peer produced after finishing its exchange x-2 reads of that slot.
#pragma once
#include "common.cuh"
#include "control.cuh"

namespace fp {

struct XchgParams {
  int M, d;
  __nv_bfloat16* h;  // residual stream [M, ldh] (replicated on every rank)
  long long ldh;
  Guard guard;       // guard.tp carries the peer pointers
};

__global__ void __launch_bounds__(256) tp_allreduce_kernel(const XchgParams p) {
  __shared__ int s_xc;
  grid_dep_wait();
  if (!guard_block(p.guard)) return;
  const TpDev* tp = p.guard.tp;
  if (threadIdx.x == 0) {
    const int xc = *(volatile int*)&tp->local->xcount;
    for (int r = 0; r < tp->size; ++r)
      while (ld_acquire_sys_u64(&tp->peer[r]->ready) < (unsigned long long)xc + 1) __nanosleep(64);
    s_xc = xc;
  }
  __syncthreads();
  const int xc = s_xc;
  const int buf = xc & 1;
  const int n = tp->size;
  const long long vpr = p.d / 8;  // 16-byte vectors per row
  const long long total = (long long)p.M * vpr;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long m = i / vpr, c = (i - m * vpr) * 8;
    __nv_bfloat16* hp = p.h + m * p.ldh + c;
    uint4 v[kTpMax];
#pragma unroll
    for (int r = 0; r < kTpMax; ++r)  // all loads in flight before the sum
      if (r < n) v[r] = ld_cg_v4(tp->part[r][buf] + m * p.d + c);
    const uint4 hv = ld_global_v4(hp);
    float acc[8];
    {
      const uint32_t w[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = unpack_bf16x2(w[j]);
        acc[2 * j] = f.x;
        acc[2 * j + 1] = f.y;
      }
    }
#pragma unroll
    for (int r = 0; r < kTpMax; ++r) {
      if (r < n) {
        const uint32_t w[4] = {v[r].x, v[r].y, v[r].z, v[r].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = unpack_bf16x2(w[j]);
          acc[2 * j] += f.x;
          acc[2 * j + 1] += f.y;
        }
      }
    }
    st_global_v4(hp, make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]),
                                pack_bf16x2(acc[4], acc[5]), pack_bf16x2(acc[6], acc[7])));
  }
  // the last CTA advances the exchange counter (read by the next exchange GEMM / all-reduce)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&tp->local->ar_ctr, 1) == (int)gridDim.x - 1) {
      tp->local->ar_ctr = 0;
      tp->local->xcount = xc + 1;
      __threadfence();
    }
  }
}

}  // namespace fp
