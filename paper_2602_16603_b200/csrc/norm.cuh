// RMSNorm (optionally fused with the embedding gather / a row gather): one CTA per token row,
// d/8 threads, one 128-bit load per thread, warp-shuffle + shared-memory reduction, fp32 math.
// HBM-bound: reads d*2 bytes and writes d*2 bytes per row (+ d*2 for the embedding copy).
// Small CTAs keep many rows (and their loads) in flight per SM.
#pragma once
#include "common.cuh"
#include "control.cuh"

namespace fp {

struct RmsParams {
  int M;              // rows
  int d;              // hidden size (multiple of 256, <= 8192)
  const __nv_bfloat16* src;  // [*, ld_src] residual stream (or embedding table if ids != null)
  long long ld_src;
  const int* ids;     // optional: token ids -> gather rows of src (embedding) and copy into h
  const int* rows;    // optional: gather row indices into src (final norm of last tokens)
  __nv_bfloat16* h_out;  // with ids: the residual stream is initialised with the embedding row
  long long ld_h;
  const __nv_bfloat16* gamma;  // [d]
  __nv_bfloat16* out;  // [M, ld_out]; null: only the embedding copy + segment sums
  long long ld_out;
  float eps;
  int nseg;            // with ssq: d / 128
  float* ssq;          // optional [M, nseg]: sums of squares per 128-column segment (the
                       // fused-norm input of the next GEMM, see GemmParams::ssq_in)
  Guard guard;
};

__global__ void __launch_bounds__(1024) rmsnorm_kernel(const RmsParams p) {
  __shared__ float red[32];
  grid_dep_wait();
  if (!guard_block(p.guard)) return;
  const int row = blockIdx.x;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  long long srow = row;
  if (p.ids) srow = p.ids[row];
  else if (p.rows) srow = p.rows[row];
  const int c = tid * 8;
  const uint4 raw = ld_global_v4(p.src + srow * p.ld_src + c);
  const uint4 gv = ld_global_v4(p.gamma + c);
  const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
  float f[8];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 v = unpack_bf16x2(w[j]);
    f[2 * j] = v.x;
    f[2 * j + 1] = v.y;
    ss += v.x * v.x + v.y * v.y;
  }
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  // a half warp = one 128-column segment
  if (p.ssq && (lane & 15) == 0) p.ssq[(long long)row * p.nseg + warp * 2 + (lane >> 4)] = ss;
  ss += __shfl_xor_sync(0xffffffffu, ss, 16);
  if (lane == 0) red[warp] = ss;
  if (p.ids && p.h_out) st_global_v4(p.h_out + (long long)row * p.ld_h + c, raw);
  if (p.out == nullptr) return;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    float t = lane < nw ? red[lane] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  const float r = rsqrtf(red[0] / (float)p.d + p.eps);
  const uint32_t gw[4] = {gv.x, gv.y, gv.z, gv.w};
  uint32_t o[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 g = unpack_bf16x2(gw[j]);
    o[j] = pack_bf16x2(f[2 * j] * r * g.x, f[2 * j + 1] * r * g.y);
  }
  st_global_v4(p.out + (long long)row * p.ld_out + c, make_uint4(o[0], o[1], o[2], o[3]));
}

}  // namespace fp
