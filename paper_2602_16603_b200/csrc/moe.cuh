// MoE routing, dispatch and combine kernels (Qwen3-MoE block) around the grouped expert GEMMs.
//
// Realises the reference's MoE operator pair (prefillsim/cost_model.py:46-52): `gate` and
// `experts` replace gate_up_proj / down_proj in every layer of an `arch = "moe"` model, and stay
// one preemption point each. Semantics follow Qwen3MoeSparseMoeBlock (HF transformers):
// probabilities = softmax over all experts of the router logits (fp32), the top-k of them
// (ties to the lower expert index), renormalised to sum 1 when norm_topk_prob, and the block
// output is sum_j w_j * expert_{e_j}(x).
//
// gate entry:    router GEMM (tcgen05, fused post-attention norm, fp32 logits)
//                -> moe_route_kernel   softmax / top-k per token, expert histogram; its last
//                                      block plans: expert row offsets (exclusive scan) + the
//                                      m-tile table of the grouped GEMMs
//                -> moe_scatter_kernel token rows gathered into expert-contiguous order
// experts entry: grouped gate/up + SwiGLU GEMM -> grouped down GEMM (gemm.cuh MODE 2)
//                -> moe_combine_kernel h += sum_j w_j y_j (j order: deterministic), and the
//                                      next norm's segment sums of squares
// A row's position inside its expert's segment depends on atomic order, but every GEMM output
// row depends only on its own input row, so results are bit-identical run to run.
#pragma once
#include "common.cuh"
#include "control.cuh"

namespace fp {

constexpr int kMoeMaxExperts = 256;
constexpr int kMoeMaxTopK = 16;

struct MoeParams {
  int M;             // token rows of the chunk
  int n_experts, top_k, norm_topk;
  int d;             // hidden
  const float* logits;   // [M, 256] router logits (gate entry)
  int ld_logits;
  int* topk_ids;         // [M, top_k]
  float* topk_w;         // [M, top_k]
  int* slot;             // [M, top_k] row of (token, j) in the expert-ordered buffers
  int* counts;           // [E] histogram (zero between gate entries)
  int* cursor;           // [E] scatter cursors (zero between gate entries)
  int* offsets;          // [E + 1] expert row offsets
  int* mtile_count;      // number of 128-row m-tiles of the grouped GEMMs
  int2* mtiles;          // [max_mtiles] (expert, first row)
  int* perm_tok;         // [M * top_k] token of each expert-ordered row
  int* ticket;           // route blocks finished (the last one plans; zero between gate entries)
  const __nv_bfloat16* h;  // residual stream [M, d] (scatter source, combine target)
  __nv_bfloat16* h_out;
  __nv_bfloat16* xperm;  // [M * top_k, d] gathered rows
  const __nv_bfloat16* yperm;  // [M * top_k, d] expert outputs
  float* ssq;            // [M, d / 256] segment sums of squares of the new h
  Guard guard;
};

DEVI void moe_route_token(const MoeParams& p, int t, int lane) {
  constexpr int PER = kMoeMaxExperts / 32;
  float v[PER];
  const float* lg = p.logits + (long long)t * p.ld_logits;
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int e = lane + 32 * i;
    v[i] = e < p.n_experts ? lg[e] : -INFINITY;
    mx = fmaxf(mx, v[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    v[i] = lane + 32 * i < p.n_experts ? expf(v[i] - mx) : 0.f;
    sum += v[i];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float inv = 1.f / sum;
#pragma unroll
  for (int i = 0; i < PER; ++i) v[i] *= inv;  // probabilities; taken ones become -1
  float wsel[kMoeMaxTopK];
  int isel[kMoeMaxTopK];
  float wsum = 0.f;
  for (int j = 0; j < p.top_k; ++j) {
    float bv = -1.f;
    int bi = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < PER; ++i)
      if (v[i] > bv) {  // strict: within a lane the lower index wins ties
        bv = v[i];
        bi = lane + 32 * i;
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if ((bi & 31) == lane) v[bi >> 5] = -1.f;
    wsel[j] = bv;
    isel[j] = bi;
    wsum += bv;
  }
  if (lane == 0) {
    const float norm = p.norm_topk ? 1.f / wsum : 1.f;
    for (int j = 0; j < p.top_k; ++j) {
      p.topk_ids[t * p.top_k + j] = isel[j];
      p.topk_w[t * p.top_k + j] = wsel[j] * norm;
      atomicAdd(&p.counts[isel[j]], 1);
    }
  }
}

// The plan, by one block of kMoeMaxExperts threads: expert offsets (exclusive scan of the
// histogram) and the grouped GEMMs' m-tile table; re-arms the histogram and the scatter cursors.
// Block-wide scan: warp shuffles, then the warp totals.
DEVI void moe_plan_block(const MoeParams& p) {
  __shared__ int s_wa[kMoeMaxExperts / 32], s_wb[kMoeMaxExperts / 32];
  const int e = threadIdx.x, lane = e & 31, warp = e >> 5;
  const int cnt = e < p.n_experts ? __ldcg(p.counts + e) : 0;
  const int nt = (cnt + 127) / 128;
  int a = cnt, b = nt;  // inclusive scans of rows and m-tiles
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int x = __shfl_up_sync(0xffffffffu, a, o), y = __shfl_up_sync(0xffffffffu, b, o);
    if (lane >= o) {
      a += x;
      b += y;
    }
  }
  if (lane == 31) {
    s_wa[warp] = a;
    s_wb[warp] = b;
  }
  __syncthreads();
  int pa = 0, pb = 0;  // totals of the warps before this one
  for (int w = 0; w < warp; ++w) {
    pa += s_wa[w];
    pb += s_wb[w];
  }
  const int off = pa + a - cnt, t0 = pb + b - nt;
  if (e < p.n_experts) {
    p.offsets[e] = off;
    for (int k = 0; k < nt; ++k) p.mtiles[t0 + k] = make_int2(e, off + 128 * k);
    p.counts[e] = 0;
    p.cursor[e] = 0;
  }
  if (e == kMoeMaxExperts - 1) {  // the last thread's inclusive sums are the totals
    p.offsets[p.n_experts] = pa + a;
    *p.mtile_count = pb + b;
  }
}

// One warp per token: softmax over the experts, top-k by repeated warp argmax, expert histogram;
// the last block to finish turns the histogram into the plan (moe_plan_block).
__global__ void __launch_bounds__(256) moe_route_kernel(const MoeParams p) {
  grid_dep_wait();
  if (!guard_block(p.guard)) return;
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t < p.M) moe_route_token(p, t, lane);
  __shared__ int s_last;
  __threadfence();  // this thread's histogram atomics are ordered before the ticket
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(p.ticket, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();  // every block's histogram is visible
  moe_plan_block(p);
  if (threadIdx.x == 0) *p.ticket = 0;
}

// One warp per token: claim a row in each chosen expert's segment and copy the token's h row.
__global__ void __launch_bounds__(256) moe_scatter_kernel(const MoeParams p) {
  grid_dep_wait();
  if (!guard_block(p.guard)) return;
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= p.M) return;
  const uint4* src = reinterpret_cast<const uint4*>(p.h + (long long)t * p.d);
  const int vecs = p.d / 8;
  for (int j = 0; j < p.top_k; ++j) {
    int row = 0;
    if (lane == 0) {
      const int e = p.topk_ids[t * p.top_k + j];
      row = p.offsets[e] + atomicAdd(&p.cursor[e], 1);
      p.slot[t * p.top_k + j] = row;
      p.perm_tok[row] = t;
    }
    row = __shfl_sync(0xffffffffu, row, 0);
    uint4* dst = reinterpret_cast<uint4*>(p.xperm + (long long)row * p.d);
    for (int i = lane; i < vecs; i += 32) dst[i] = ld_nc_v4(src + i);
  }
}

// One warp per (token, 256-column segment): h += sum_j w_j * y[slot_j] (fp32, j order), and
// the segment's sum of squares of the new (bf16-rounded) h for the next fused norm.
__global__ void __launch_bounds__(256) moe_combine_kernel(const MoeParams p) {
  grid_dep_wait();
  if (!guard_block(p.guard)) return;
  const int lane = threadIdx.x & 31;
  const int nseg = p.d / 256;
  const long long u = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (u >= (long long)p.M * nseg) return;
  const int t = (int)(u / nseg), sg = (int)(u - (long long)t * nseg);
  const int c = sg * 256 + lane * 8;
  float acc[8];
  {
    const uint4 hv = ld_global_v4(p.h + (long long)t * p.d + c);
    const uint32_t w4[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = unpack_bf16x2(w4[i]);
      acc[2 * i] = f.x;
      acc[2 * i + 1] = f.y;
    }
  }
  float y[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int j = 0; j < p.top_k; ++j) {
    const float wj = p.topk_w[t * p.top_k + j];
    const uint4 yv = ld_global_v4(p.yperm + (long long)p.slot[t * p.top_k + j] * p.d + c);
    const uint32_t w4[4] = {yv.x, yv.y, yv.z, yv.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = unpack_bf16x2(w4[i]);
      y[2 * i] += wj * f.x;
      y[2 * i + 1] += wj * f.y;
    }
  }
  float ss = 0.f;
  uint32_t o4[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    o4[i] = pack_bf16x2(acc[2 * i] + y[2 * i], acc[2 * i + 1] + y[2 * i + 1]);
    const float2 f = unpack_bf16x2(o4[i]);
    ss += f.x * f.x + f.y * f.y;
  }
  st_global_v4(p.h_out + (long long)t * p.d + c, make_uint4(o4[0], o4[1], o4[2], o4[3]));
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);  // half warps
  if ((lane & 15) == 0 && p.ssq) p.ssq[(long long)t * nseg * 2 + sg * 2 + (lane >> 4)] = ss;
}

}  // namespace fp
