// RMSNorm (optionally fused with the embedding gather / a row gather), warp per token row.
// HBM-bound: reads d*2 bytes and writes d*2 bytes per row (+ d*2 for the embedding copy).
// 128-bit vectorised loads/stores, warp-shuffle reduction, fp32 math.
#pragma once
#include "common.cuh"
#include "control.cuh"

namespace fp {

struct RmsParams {
  int M;              // rows
  int d;              // hidden size (multiple of 256)
  const __nv_bfloat16* src;  // [*, ld_src] residual stream (or embedding table if ids != null)
  long long ld_src;
  const int* ids;     // optional: token ids -> gather rows of src (embedding) and copy into h
  const int* rows;    // optional: gather row indices into src (final norm of last tokens)
  __nv_bfloat16* h_out;  // with ids: the residual stream is initialised with the embedding row
  long long ld_h;
  const __nv_bfloat16* gamma;  // [d]
  __nv_bfloat16* out;  // [M, ld_out]
  long long ld_out;
  float eps;
  int pad;
  Guard guard;
};

constexpr int kRmsRowsPerBlock = 8;

template <int NV>  // d = NV * 256
__global__ void __launch_bounds__(256, 2) rmsnorm_kernel(const RmsParams p) {
  if (!guard_block(p.guard)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * kRmsRowsPerBlock + warp;
  if (row >= p.M) return;
  long long srow = row;
  if (p.ids) srow = p.ids[row];
  else if (p.rows) srow = p.rows[row];
  const __nv_bfloat16* src = p.src + srow * p.ld_src;
  uint4 raw[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) raw[i] = ld_global_v4(src + (i * 32 + lane) * 8);
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const uint32_t w[4] = {raw[i].x, raw[i].y, raw[i].z, raw[i].w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = unpack_bf16x2(w[j]);
      ss += f.x * f.x + f.y * f.y;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float r = rsqrtf(ss / (float)p.d + p.eps);
  if (p.ids && p.h_out) {
#pragma unroll
    for (int i = 0; i < NV; ++i) st_global_v4(p.h_out + row * p.ld_h + (i * 32 + lane) * 8, raw[i]);
  }
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (i * 32 + lane) * 8;
    const uint4 gv = ld_global_v4(p.gamma + c);
    const uint32_t w[4] = {raw[i].x, raw[i].y, raw[i].z, raw[i].w};
    const uint32_t gw[4] = {gv.x, gv.y, gv.z, gv.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = unpack_bf16x2(w[j]);
      const float2 g = unpack_bf16x2(gw[j]);
      o[j] = pack_bf16x2(f.x * r * g.x, f.y * r * g.y);
    }
    st_global_v4(p.out + row * p.ld_out + c, make_uint4(o[0], o[1], o[2], o[3]));
  }
}

}  // namespace fp
