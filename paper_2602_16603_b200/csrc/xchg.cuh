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
  float* ssq;        // [M, d/256] segment sums of squares of the new h (fused next RMSNorm)
  Guard guard;       // guard.tp carries the peer pointers
};

// One warp per (row, 256-column segment): 32 lanes x 8 bf16 = the segment, so the fused
// norm's segment sum of squares is one warp reduction.
__global__ void __launch_bounds__(256, 1) tp_allreduce_kernel(const XchgParams p) {
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
  const int lane = threadIdx.x & 31;
  const int nseg = p.d / 256;
  const long long units = (long long)p.M * nseg;
  const long long wstep = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long u = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); u < units;
       u += wstep) {
    const long long m = u / nseg;
    const int sg = (int)(u - m * nseg);
    const long long c = (long long)sg * 256 + lane * 8;
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
    const uint4 o = make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]),
                               pack_bf16x2(acc[4], acc[5]), pack_bf16x2(acc[6], acc[7]));
    st_global_v4(hp, o);
    if (p.ssq) {
      float ss = 0.f;
      const uint32_t w[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = unpack_bf16x2(w[j]);
        ss += f.x * f.x + f.y * f.y;
      }
#pragma unroll
      for (int off = 8; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
      if ((lane & 15) == 0) p.ssq[m * nseg * 2 + sg * 2 + (lane >> 4)] = ss;  // 128-col segments
    }
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

// Per-op all-reduce (fp_op_tp_allreduce): stage a caller partial into this rank's exchange
// slot and publish it exactly like an exchange GEMM's epilogue does (tp_publish_partial).
__global__ void __launch_bounds__(256) tp_stage_partial_kernel(const TpDev* tp,
                                                               const __nv_bfloat16* src,
                                                               long long vecs) {
  grid_dep_wait();
  const int xc = *(volatile int*)&tp->local->xcount;
  uint4* dst = reinterpret_cast<uint4*>(tp->part[tp->rank][xc & 1]);
  const uint4* s = reinterpret_cast<const uint4*>(src);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < vecs;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = ld_nc_v4(s + i);
  __syncthreads();
  if (threadIdx.x == 0) tp_publish_partial(tp);
}

}  // namespace fp
