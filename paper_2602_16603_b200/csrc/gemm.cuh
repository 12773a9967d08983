// Persistent, warp-specialised tcgen05 GEMM for the four dense prefill operators.
//
//   C[M, N] = A[M, K] * B[N, K]^T      A, B bf16 K-major (row-major, K contiguous)
//
// Realises the linear part of the reference's qkv_proj / o_proj / gate_up_proj / down_proj
// timeline entries (prefillsim/cost_model.py:38-44, 234-242): the GEMM M dimension is the
// chunk's concatenated token count `new_total` (cost_model.py:225,236).
//
// Layout of one CTA (256 threads, 1 CTA / SM, persistent over tiles):
//   warp 0      TMA producer (A tile 128x64, B tile BNx64 per stage, 128B swizzle)
//   warp 1      MMA issuer (one thread; tcgen05.mma.cta_group::1.kind::f16, M=128, N=BN, K=16)
//   warp 2      TMEM allocator (2 accumulator stages x BN fp32 columns)
//   warps 4..7  epilogue: tcgen05.ld (one token row per thread) -> fused epilogue -> HBM
// The accumulator is double-buffered in TMEM so the epilogue of tile i overlaps the
// main loop of tile i+1.
#pragma once
#include "common.cuh"
#include "control.cuh"

namespace fp {

enum EpiKind : int {
  EPI_STORE_BF16 = 0,  // out = bf16(acc)
  EPI_STORE_F32 = 1,   // out = acc (fp32; lm_head logits)
  EPI_RESID = 2,       // resid += acc (o_proj, down_proj: residual add)
  EPI_SWIGLU = 3,      // out = silu(gate) * up; B rows packed [gate(BN/2) | up(BN/2)] per tile
  EPI_QKV = 4,         // RoPE(q,k); q -> qbuf, k/v -> paged KV cache
};

struct GemmParams {
  int M, N, K;
  int pad0;
  void* out;
  long long ldo;
  __nv_bfloat16* resid;
  long long ldr;
  // EPI_QKV
  const int* pos;       // [M] position of the token inside its own request
  const int* tok_page;  // [M] physical KV page of the token
  __nv_bfloat16* qbuf;  // [M, q_cols]
  long long ldq;
  __nv_bfloat16* kv_layer;  // this layer's base of the paged KV pool
  const float2* rope;       // [max_pos][64] (cos, sin)
  int q_cols, kv_cols, page_size, n_kv_heads;
  const float* bias;        // [N] q/k/v projection bias (Qwen2.5) or null
  const float* q_norm;      // [128] per-head RMSNorm weight of q (Qwen3) or null
  const float* k_norm;      // [128] ... of k
  float norm_eps;
  int pad2;
  // Tail split-K: the first `full_tiles` tiles (whole waves) run unsplit; each remaining tile
  // is cut into `splits` K-slices so the last wave fills the machine. fp32 partials go to
  // `ws` and the last-arriving CTA of a tile reduces them in split order (deterministic) and
  // runs the fused epilogue. `tickets` must be zero on entry (the reducer resets it).
  int splits;
  int full_tiles;
  float* ws;
  int* tickets;     // [2][1024] per split tile slot: arrivals, done
  int xchg;  // tensor parallel o_proj/down_proj (EPI_STORE_BF16): 1 = store the partial sum
             // into this rank's exchange buffer and publish it (tp_publish_partial; a separate
             // tp_allreduce_kernel folds the partials); 2 = FUSED: after each tile's partial
             // store the epilogue flags the tile to the peers and folds the previous tile of
             // every rank into the residual over NVLink, tile by tile (tp_fold_tile)
  // Fused RMSNorm. The norm weight is folded into the weight columns (W' = W diag(gamma)), so
  // rmsnorm(h) W^T = rsqrt(mean(h^2) + eps) * (h W'^T): the GEMM reads the residual stream h
  // directly and the EPI_QKV / EPI_SWIGLU epilogue scales its row by the rsqrt factor, built
  // from `ssq_in` = per-row sums of squares of h in 128-column segments [M, nseg] (summed in
  // segment order: deterministic). EPI_RESID writes those segment sums of the new h into
  // `ssq_out` (tile n-block nb = segment nb) for the next norm.
  int nseg;
  float norm_eps_in;  // eps of the fused input RMSNorm
  const float* ssq_in;
  float* ssq_out;
  unsigned long long* dbg;  // phase stamps (%globaltimer ns) [cta][16] for diagnostics, or null
  // MODE 2 (grouped MoE experts)
  const int* grp_mtiles;  // [m-tiles] int2 (expert, first A row)
  const int* grp_count;   // number of m-tiles
  const int* grp_off;     // [E + 1] expert row offsets (live-row bound)
  const int* grp_perm;    // [rows] token of each row (fused-norm lookup)
  int grp_b_rows;         // B rows per expert
  // MODE 3 (stream-K): full_tiles = whole tiles processed first (round-robin), the rest of the
  // (tile, k-block) space is cut into gridDim.x equal contiguous ranges; sk_flags[cta] =
  // sk_epoch once that CTA's partial tile is in the workspace
  int* sk_flags;
  int sk_epoch;
  int group_m;  // m-blocks per raster group (0: kGemmGroupM); the launcher sets "all" when the
                // whole A operand fits in L2, so every weight tile is read from HBM once
  Guard guard;
};

// Phase stamps are compiled in only for diagnostic builds (-DFP_GEMM_STAMPS): even an idle
// stamp perturbs the register allocation of the epilogue warps.
#ifdef FP_GEMM_STAMPS
#define GEMM_STAMP(k)                                                                 \
  do {                                                                                \
    if (p.dbg) p.dbg[(blockIdx.x + blockIdx.y * gridDim.x) * 16 + (k)] = globaltimer(); \
  } while (0)
#else
#define GEMM_STAMP(k) \
  do {                \
  } while (0)
#endif

constexpr int kGemmBM = 128;
constexpr int kGemmBK = 64;
constexpr int kGemmThreads = 256;
constexpr int kGemmGroupM = 16;  // m-blocks per raster group (L2 reuse of A and B)

// CG = 1: one CTA computes a 128 x BN tile. CG = 2: a CTA pair (cluster of 2) computes a
// 256 x BN tile with tcgen05.mma.cta_group::2 -- each CTA stages its own 128 A rows and BN/2 B
// rows, so per-SM shared-memory traffic per k-block drops from 96 KB to 64 KB (the 1-CTA
// kernel is smem-port bound at ~70% of the MMA rate).
template <int BN, int CG = 1>
struct GemmCfg {
  static constexpr int A_BYTES = kGemmBM * kGemmBK * 2;
  static constexpr int B_BYTES = (BN / CG) * kGemmBK * 2;
  static constexpr int STAGES = (A_BYTES + B_BYTES) <= 32768 ? 6 : 4;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int TILE_M = kGemmBM * CG;
  static constexpr int SMEM_BYTES = 1024 + STAGES * (A_BYTES + B_BYTES) + 256;
  // stream-K: + two 16 KB buffers for the partner partials of a finishing tile
  static constexpr int SK_SMEM_BYTES = SMEM_BYTES + 2 * 16384;
};

DEVI void tile_coords(int t, int num_m, int num_n, int group, int& mb, int& nb) {
  const int per_group = group * num_n;
  const int g = t / per_group;
  const int first_m = g * group;
  int gm = num_m - first_m;
  if (gm > group) gm = group;
  const int local = t - g * per_group;
  mb = first_m + local % gm;
  nb = local / gm;
}

DEVI float silu_f(float x) { return x / (1.0f + __expf(-x)); }

// Store 32 fp32 values as bf16 (64 bytes) to a 16-byte aligned address.
DEVI void store_row32_bf16(__nv_bfloat16* dst, const float* v) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint4 u;
    u.x = pack_bf16x2(v[8 * i + 0], v[8 * i + 1]);
    u.y = pack_bf16x2(v[8 * i + 2], v[8 * i + 3]);
    u.z = pack_bf16x2(v[8 * i + 4], v[8 * i + 5]);
    u.w = pack_bf16x2(v[8 * i + 6], v[8 * i + 7]);
    st_global_v4(dst + 8 * i, u);
  }
}

// Inter-CTA barrier of the K-slice CTAs of one split tile (epilogue warps only): arrive, then
// spin until `n` arrivals (acquire).
DEVI void split_barrier(int* ctr, int n) {
  __threadfence();
  asm volatile("bar.sync 1, 128;" ::: "memory");
  if (threadIdx.x % 128 == 0) {
    atomicAdd(ctr, 1);
    int v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      if (v >= n) break;
      __nanosleep(32);
    }
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");
}

// Split-K tile reduction. A split tile's fp32 K-slice partials sit in the L2 workspace as
// [split][col/4][row] float4. Its epilogue is cut into 8 items per row, each summing 32 partial
// columns -- [colA, colA + 16) and [colB, colB + 16) -- over the K-slices in split order (the
// same bits on every run), with 4 slices' loads in flight.
struct GmemSum {
  const float4* ws_tile;
  int S;
  template <int ILP = 4>
  DEVI void get(int r, int colA, int colB, float* v) const {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = 0.f;
    const float4* sa = ws_tile + (long long)(colA / 4) * kGemmBM + r;
    const float4* sb = ws_tile + (long long)(colB / 4) * kGemmBM + r;
    const long long sstride = 64LL * kGemmBM;  // 256 columns / 4 per K-slice
    for (int s0 = 0; s0 < S; s0 += ILP) {
      float4 f[ILP][8];
#pragma unroll
      for (int j = 0; j < ILP; ++j)
        if (s0 + j < S) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            f[j][i] = __ldcg(sa + (s0 + j) * sstride + i * kGemmBM);
            f[j][4 + i] = __ldcg(sb + (s0 + j) * sstride + i * kGemmBM);
          }
        }
#pragma unroll
      for (int j = 0; j < ILP; ++j)
        if (s0 + j < S) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            v[4 * i] += f[j][i].x;
            v[4 * i + 1] += f[j][i].y;
            v[4 * i + 2] += f[j][i].z;
            v[4 * i + 3] += f[j][i].w;
          }
        }
    }
  }
};

// Sum provider of the split path: GmemSum's reduction, or the same over the K-slice CTAs of a
// cluster (dsm): each CTA's fp32 partial then sits in its own shared memory as [col/4][row]
// float4 (the layout of one GmemSum slice) and is read through distributed shared memory --
// die-local, no L2 round trips (the L2 version's first item stalls ~4 us on partials just
// written by other SMs). Summed in split order from 0 either way: the same bits.
template <bool DSM>
struct SplitSum {
  const float4* ws_tile;  // L2 workspace of the tile (!DSM)
  uint32_t sbase;         // this CTA's partial, shared::cta address (DSM)
  int S;
  template <int ILP = 4>
  DEVI void get(int r, int colA, int colB, float* v) const {
    if constexpr (!DSM) {
      GmemSum{ws_tile, S}.template get<ILP>(r, colA, colB, v);
      return;
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = 0.f;
    const uint32_t oa = (uint32_t)(((colA / 4) * kGemmBM + r) * 16);
    const uint32_t ob = (uint32_t)(((colB / 4) * kGemmBM + r) * 16);
    for (int s0 = 0; s0 < S; s0 += ILP) {
      float4 f[ILP][8];
#pragma unroll
      for (int j = 0; j < ILP; ++j)
        if (s0 + j < S) {
          const uint32_t b = mapa_shared(sbase, (uint32_t)(s0 + j));
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            f[j][i] = ld_dsmem_f4(b + oa + i * kGemmBM * 16);
            f[j][4 + i] = ld_dsmem_f4(b + ob + i * kGemmBM * 16);
          }
        }
#pragma unroll
      for (int j = 0; j < ILP; ++j)
        if (s0 + j < S) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            v[4 * i] += f[j][i].x;
            v[4 * i + 1] += f[j][i].y;
            v[4 * i + 2] += f[j][i].z;
            v[4 * i + 3] += f[j][i].w;
          }
        }
    }
  }
};

DEVI void store16_bf16(__nv_bfloat16* dst, const float* v) {
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    uint4 u;
    u.x = pack_bf16x2(v[8 * i + 0], v[8 * i + 1]);
    u.y = pack_bf16x2(v[8 * i + 2], v[8 * i + 3]);
    u.z = pack_bf16x2(v[8 * i + 4], v[8 * i + 5]);
    u.w = pack_bf16x2(v[8 * i + 6], v[8 * i + 7]);
    st_global_v4(dst + 8 * i, u);
  }
}

// rsqrt(mean(h^2) + eps) of a row from its 128-column segment sums of squares (nseg is a
// multiple of 4: hidden % 512 == 0), summed in segment order with all loads in flight.
DEVI float fused_norm_rsqrt(const float* sp, int nseg, float eps) {
  const float4* s4 = reinterpret_cast<const float4*>(sp);
  float ssum = 0.f;
  int i = 0;
  for (; i + 4 <= nseg / 4; i += 4) {
    float4 a[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) a[j] = __ldg(s4 + i + j);
#pragma unroll
    for (int j = 0; j < 4; ++j) ssum = (((ssum + a[j].x) + a[j].y) + a[j].z) + a[j].w;
  }
  for (; i < nseg / 4; ++i) {
    const float4 a = __ldg(s4 + i);
    ssum = (((ssum + a.x) + a.y) + a.z) + a.w;
  }
  return rsqrtf(ssum / (float)(nseg * 128) + eps);
}

// Fused tensor-parallel exchange (GemmParams::xchg == 2), run by the 4 epilogue warps (one
// tile row each): wait until every rank has flagged its partial of this output tile, then
// h[m, n0:n0+256] = bf16(h + part_0 + part_1 + ...) (fp32, rank order: the same bits as
// tp_allreduce_kernel on every rank) and the next fused norm's segment sum of squares.
DEVI void tp_fold_tile(const GemmParams& p, const TpDev* tp, int slot, unsigned long long want,
                       int fidx, int m_base, int row_end, int n0, int nb) {
  const int row = threadIdx.x - 128;  // epilogue threads 128..255
  if (row == 0) {
    for (int r = 0; r < tp->size; ++r)
      while (ld_acquire_sys_u64(&tp->peer[r]->flags[slot][fidx]) < want) __nanosleep(64);
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");
  const int m = m_base + row;
  if (m >= row_end) return;
  __nv_bfloat16* hrow = p.resid + (long long)m * p.ldr + n0;
  float ss = 0.f;
#pragma unroll 1
  for (int c = 0; c < 8; ++c) {  // 32 columns at a time, every rank's loads in flight
    uint4 v[kTpMax][4];
#pragma unroll
    for (int r = 0; r < kTpMax; ++r)
      if (r < tp->size) {
        const __nv_bfloat16* src = tp->part[r][slot] + (long long)m * p.ldo + n0 + c * 32;
#pragma unroll
        for (int i = 0; i < 4; ++i) v[r][i] = ld_cg_v4(src + 8 * i);
      }
    float acc[32];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint4 h = ld_global_v4(hrow + c * 32 + 8 * i);
      const uint32_t hw[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = unpack_bf16x2(hw[j]);
        acc[8 * i + 2 * j] = f.x;
        acc[8 * i + 2 * j + 1] = f.y;
      }
    }
#pragma unroll
    for (int r = 0; r < kTpMax; ++r)
      if (r < tp->size) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t w4[4] = {v[r][i].x, v[r][i].y, v[r][i].z, v[r][i].w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 f = unpack_bf16x2(w4[j]);
            acc[8 * i + 2 * j] += f.x;
            acc[8 * i + 2 * j + 1] += f.y;
          }
        }
      }
#pragma unroll
    for (int i = 0; i < 32; ++i) {  // the next norm sees the bf16-rounded values
      const float rv = __bfloat162float(__float2bfloat16(acc[i]));
      ss += rv * rv;
    }
    store_row32_bf16(hrow + c * 32, acc);
    if (c == 3 || c == 7) {  // 128-column segment complete
      if (p.ssq_out) p.ssq_out[(long long)m * p.nseg + nb * 2 + (c >> 2)] = ss;
      ss = 0.f;
    }
  }
}

// Epilogue item g (0..7) of tile row r (token row m) of a split tile; n0 / nb = the tile's first
// column / n-block. Called by all 32 lanes of a warp (valid = false lanes only join shuffles);
// the 8 items of a row are 8 consecutive lanes. Items:
//   EPI_RESID / EPI_STORE_*  columns [32g, 32g + 32)
//   EPI_SWIGLU               gate columns [16g, 16g + 16) and the matching up columns (+128)
//   EPI_QKV                  head h = g / 4, quarter q = g % 4: head columns [16q, 16q + 16)
//                            and their RoPE partners [64 + 16q, 64 + 16q + 16)
// EPI_RESID writes the row's sum of squares (8 chunk sums in chunk order) to ssq_out; the Qwen3
// q/k-norm sums a head's 4 items in quarter order.
template <int EPI, class Sum = GmemSum>
__device__ __forceinline__ void split_item_epilogue(const GemmParams& p, const Sum& sum,
                                                 bool valid, int m, int r, int g, int n0,
                                                 int nb) {
  constexpr int BN = 256;
  const int lane = threadIdx.x & 31;
  float rs = 1.f;  // fused input RMSNorm factor of the row
  if ((EPI == EPI_QKV || EPI == EPI_SWIGLU || EPI == EPI_STORE_F32) && p.ssq_in != nullptr &&
      valid) {
    rs = fused_norm_rsqrt(p.ssq_in + (long long)m * p.nseg, p.nseg, p.norm_eps_in);
  }
  float v[32];
  if constexpr (EPI == EPI_RESID) {
    __nv_bfloat16* hrow = p.resid + (long long)m * p.ldr + n0 + g * 32;
    uint4 hv[4];  // residual loads in flight with the partial loads
    float ss = 0.f;
    if (valid) {
      if (threadIdx.x == 128) GEMM_STAMP(12);
#ifdef FP_GEMM_STAMPS
      // diagnostic builds time the two dependencies apart: partials (13), then the residual
      // row (14, forced by a use of every loaded word)
      sum.get(r, g * 32, g * 32 + 16, v);
      if (threadIdx.x == 128) GEMM_STAMP(13);
#pragma unroll
      for (int i = 0; i < 4; ++i) hv[i] = ld_global_v4(hrow + 8 * i);
      if (threadIdx.x == 128) {
        unsigned acc = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) acc ^= hv[i].x ^ hv[i].y ^ hv[i].z ^ hv[i].w;
        if (acc == 0x12345678u) v[0] += 1e-30f;
        GEMM_STAMP(14);
      }
#else
#pragma unroll
      for (int i = 0; i < 4; ++i) hv[i] = ld_global_v4(hrow + 8 * i);
      sum.get(r, g * 32, g * 32 + 16, v);
#endif
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t hw[4] = {hv[i].x, hv[i].y, hv[i].z, hv[i].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = unpack_bf16x2(hw[j]);
          v[8 * i + 2 * j] += f.x;
          v[8 * i + 2 * j + 1] += f.y;
        }
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) {  // the next norm sees the bf16-rounded values
        const float rv = __bfloat162float(__float2bfloat16(v[i]));
        ss += rv * rv;
      }
      store_row32_bf16(hrow, v);
    }
    float tot = 0.f;  // chunks 0-3 and 4-7: the two 128-column segments of the tile
#pragma unroll
    for (int j = 0; j < 4; ++j) tot += __shfl_sync(0xffffffffu, ss, (lane & ~3) + j);
    if (valid && (g & 3) == 0 && p.ssq_out != nullptr)
      p.ssq_out[(long long)m * p.nseg + nb * 2 + (g >> 2)] = tot;
    if (threadIdx.x == 128 && valid) GEMM_STAMP(15);
  } else if constexpr (EPI == EPI_STORE_BF16 || EPI == EPI_STORE_F32) {
    if (!valid) return;
    sum.get(r, g * 32, g * 32 + 16, v);
    if constexpr (EPI == EPI_STORE_F32) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] *= rs;  // fused norm (MoE router logits)
      float* dst = reinterpret_cast<float*>(p.out) + (long long)m * p.ldo + n0 + g * 32;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        st_global_v4(dst + 4 * i,
                     make_uint4(__float_as_uint(v[4 * i]), __float_as_uint(v[4 * i + 1]),
                                __float_as_uint(v[4 * i + 2]), __float_as_uint(v[4 * i + 3])));
    } else {
      void* out = p.out;
      if (p.xchg) {
        const TpDev* tp = p.guard.tp;
        out = tp->part[tp->rank][tp->local->xcount & 1];
      }
      store_row32_bf16(reinterpret_cast<__nv_bfloat16*>(out) + (long long)m * p.ldo + n0 + g * 32,
                       v);
    }
  } else if constexpr (EPI == EPI_SWIGLU) {
    if (!valid) return;
    // tile columns [0, BN/2) are gate rows, [BN/2, BN) the matching up rows
    sum.get(r, g * 16, BN / 2 + g * 16, v);
    float o[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) o[i] = silu_f(v[i] * rs) * (v[16 + i] * rs);
    store16_bf16(reinterpret_cast<__nv_bfloat16*>(p.out) + (long long)m * p.ldo + nb * (BN / 2) +
                     g * 16,
                 o);
  } else {  // EPI_QKV
    const int hh = g >> 2, q = g & 3;
    const int col0 = n0 + hh * 128;  // the head's first column
    const bool live = valid && col0 < p.q_cols + 2 * p.kv_cols;  // not the zero padding
    const bool is_q = col0 < p.q_cols;
    const bool is_v = col0 >= p.q_cols + p.kv_cols;
    const float* bias = p.bias ? p.bias + col0 : nullptr;
    const float* hn = is_v ? nullptr : (is_q ? p.q_norm : p.k_norm);
    float ss = 0.f;
    if (live) {
      sum.template get<2>(r, hh * 128 + q * 16, hh * 128 + 64 + q * 16, v);  // ILP 2: register budget
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] *= rs;
      if (bias) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          v[i] += __ldg(bias + q * 16 + i);
          v[16 + i] += __ldg(bias + 64 + q * 16 + i);
        }
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) ss += v[i] * v[i];
    }
    if (hn != nullptr) {  // per-head RMSNorm (Qwen3): the head's 4 quarter sums, in order
      float tot = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) tot += __shfl_sync(0xffffffffu, ss, (lane & ~3) + j);
      const float nscale = rsqrtf(tot * (1.f / 128.f) + p.norm_eps);
      if (live) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          v[i] *= nscale * __ldg(hn + q * 16 + i);
          v[16 + i] *= nscale * __ldg(hn + 64 + q * 16 + i);
        }
      }
    }
    if (!live) return;
    const int pos = p.pos[m];
    __nv_bfloat16* dst;
    if (is_q) {
      dst = p.qbuf + (long long)m * p.ldq + col0;
    } else {
      const int kv = is_v ? 1 : 0;
      const int h = (col0 - p.q_cols - kv * p.kv_cols) >> 7;
      const int page = p.tok_page[m];
      dst = p.kv_layer +
            ((((long long)page * 2 + kv) * p.n_kv_heads + h) * p.page_size + (pos % p.page_size)) *
                128;
    }
    if (!is_v) {  // rotate-half RoPE: column j pairs with j + 64
      const float4* cs = reinterpret_cast<const float4*>(p.rope + (long long)pos * 64) + q * 8;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 t4 = __ldg(cs + i);  // (cos, sin) of pair columns 2i, 2i + 1
        const float u1 = v[2 * i], u2 = v[16 + 2 * i];
        const float w1 = v[2 * i + 1], w2 = v[16 + 2 * i + 1];
        v[2 * i] = u1 * t4.x - u2 * t4.y;
        v[16 + 2 * i] = u2 * t4.x + u1 * t4.y;
        v[2 * i + 1] = w1 * t4.z - w2 * t4.w;
        v[16 + 2 * i + 1] = w2 * t4.z + w1 * t4.w;
      }
    }
    store16_bf16(dst + q * 16, v);
    store16_bf16(dst + 64 + q * 16, v + 16);
  }
}

// MODE 0: plain tiles. MODE 1: the instantiation that also runs tail split-K tiles (launched only
// when the launcher chose splits > 1; MODE 0 carries no split code and no extra registers).
// MODE 4: MODE 1 for launches whose tiles are ALL split, launched as clusters of the S K-slice
// CTAs of each tile: the partials stay in each CTA's shared memory and are summed through
// distributed shared memory (SplitSum<true>) between two cluster barriers.
// MODE 2: grouped GEMM for MoE experts -- A rows are expert-ordered segments, the m-tile table
// (expert, first row) and its length come from device memory (moe_plan_block), the B rows of
// expert e start at e * grp_b_rows, rows past the expert's segment are masked, and the fused
// norm looks up each row's token through grp_perm. CG = 1 only.
template <int BN, int EPI, int CG, int MODE>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, const GemmParams p) {
  using Cfg = GemmCfg<BN, CG>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * Cfg::B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint64_t* pbar = tempty + 3;  // MODE 3: partner-partial buffers' barriers [2]
  uint8_t* sPart = sB + STAGES * Cfg::B_BYTES + 256;  // MODE 3: 2 x 16 KB

  const int warp = warp_id();
  const int lane = lane_id();
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;  // CTA rank inside the pair
  const bool leader = rank == 0;
  if (threadIdx.x == 0) GEMM_STAMP(0);
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);  // the leader's expect_tx arrival (+ both CTAs' TMA bytes)
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4 * CG);  // one arrival per epilogue warp of every CTA
      if constexpr (MODE == 3) mbar_init(&pbar[a], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (CG == 2) tmem_alloc_2sm<Cfg::TMEM_COLS>(tmem_slot);
    else tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync_all();  // peer barriers initialised before any arrive
  else __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  if (threadIdx.x == 0) GEMM_STAMP(1);
  // Everything above overlaps the previous kernel's tail (programmatic dependent launch);
  // the boundary check and all data accesses come after the dependency resolves.
  grid_dep_wait();
  const bool run = guard_block(p.guard);
  if (threadIdx.x == 0) GEMM_STAMP(2);

  const int num_m = MODE == 2 ? (run ? *p.grp_count : 0) : (p.M + Cfg::TILE_M - 1) / Cfg::TILE_M;
  const int unit0 = blockIdx.x / CG;      // this CTA (pair)'s first work unit
  const int unit_step = gridDim.x / CG;
  const int num_n = p.N / BN;
  const int num_tiles = num_m * num_n;
  const int num_k = p.K / kGemmBK;
  const int tail_splits = p.splits > 1 ? p.splits : 1;
  const int full_tiles = tail_splits > 1 ? min(p.full_tiles, num_tiles) : num_tiles;
  const int num_units = run ? full_tiles + (num_tiles - full_tiles) * tail_splits : 0;
  // unit -> (tile, K-slice index, slice count, k-block range)
  auto unit_info = [&](int u, int& tile, int& split, int& nsplit, int& kb0, int& kb1) {
    if (u < full_tiles) {
      tile = u;
      split = 0;
      nsplit = 1;
      kb0 = 0;
      kb1 = num_k;
    } else {
      const int v = u - full_tiles;
      tile = full_tiles + v / tail_splits;
      split = v % tail_splits;
      nsplit = tail_splits;
      const int per = (num_k + tail_splits - 1) / tail_splits;
      kb0 = split * per;
      kb1 = min(num_k, kb0 + per);
    }
  };
  // MODE 3 (stream-K). This CTA's range [sk_s, sk_e) of the stream-K (tile, k-block) space
  // (tiles after the full_tiles whole ones, k fastest) runs as: first the partial of the tile
  // its range ends inside (if any: published to the workspace at once, so no CTA ever waits on
  // a chain), then every tile that finishes inside the range -- the first of them, if the
  // range starts inside it, takes the partials of the CTAs before it (its "partners").
  const int dp_tiles = MODE == 3 ? min(p.full_tiles, num_tiles) : 0;
  const long long sk_u = MODE == 3 ? (long long)(num_tiles - dp_tiles) * num_k : 0;
  const int sk_g = gridDim.x;
  const int sk_s = MODE == 3 ? (int)((long long)blockIdx.x * sk_u / sk_g) : 0;
  const int sk_e = MODE == 3 ? (int)((long long)(blockIdx.x + 1) * sk_u / sk_g) : 0;
  const int sk_dp_mine = (MODE == 3 && (int)blockIdx.x < dp_tiles)
                             ? (dp_tiles - 1 - (int)blockIdx.x) / sk_g + 1 : 0;
  const int sk_prod = (MODE == 3 && sk_e > sk_s && sk_e % num_k != 0) ? 1 : 0;
  const int sk_t0 = num_k > 0 ? sk_s / num_k : 0;
  const int sk_fin = MODE == 3 ? max(0, (num_k > 0 ? sk_e / num_k : 0) - sk_t0) : 0;
  const int n_work = !run ? 0
                     : MODE == 3 ? sk_dp_mine + sk_prod + sk_fin
                                 : (unit0 < num_units ? (num_units - unit0 + unit_step - 1) / unit_step : 0);
  // work item -> (tile, K-slice, slices, k-blocks, role: 0 whole / finishing without partners,
  // 1 stream-K partial producer, 2 stream-K finisher with partners)
  auto work_info = [&](int w, int& tile, int& split, int& nsplit, int& kb0, int& kb1, int& role) {
    role = 0;
    if constexpr (MODE == 3) {
      split = 0;
      nsplit = 1;
      if (w < sk_dp_mine) {
        tile = (int)blockIdx.x + w * sk_g;
        kb0 = 0;
        kb1 = num_k;
        return;
      }
      w -= sk_dp_mine;
      int t;
      if (w < sk_prod) {
        t = sk_e / num_k;
        kb1 = sk_e - t * num_k;
        role = 1;
      } else {
        t = sk_t0 + (w - sk_prod);
        kb1 = num_k;
      }
      kb0 = max(sk_s - t * num_k, 0);
      if (role == 0 && kb0 > 0) role = 2;
      tile = dp_tiles + t;
    } else {
      unit_info(unit0 + w * unit_step, tile, split, nsplit, kb0, kb1);
    }
  };
  // tile -> (m-block, n-block, first A row, first B row, end of live rows)
  auto tile_geom = [&](int tile, int& mb, int& nb, int& row_a, int& row_b, int& row_end) {
    if constexpr (MODE == 2) {
      int mt;
      tile_coords(tile, num_m, num_n, kGemmGroupM, mt, nb);
      const int2 te = reinterpret_cast<const int2*>(p.grp_mtiles)[mt];
      mb = mt;
      row_a = te.y;
      row_b = te.x * p.grp_b_rows + nb * BN;
      row_end = p.grp_off[te.x + 1];
    } else {
      tile_coords(tile, num_m, num_n, p.group_m > 0 ? p.group_m : kGemmGroupM, mb, nb);
      row_a = mb * Cfg::TILE_M + (int)rank * kGemmBM;
      row_b = nb * BN + (int)rank * (BN / CG);
      row_end = p.M;
    }
  };

  if (warp == 0) {
    const uint64_t pol_b = policy_evict_last();
    int s = 0;
    uint32_t ph = 0;
    for (int w = 0; w < n_work; ++w) {
      int tile, split, nsplit, kb0, kb1, role;
      work_info(w, tile, split, nsplit, kb0, kb1, role);
      int mb, nb, row_a, row_b, row_end;
      tile_geom(tile, mb, nb, row_a, row_b, row_end);
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&empty[s], ph ^ 1);
        if (lane == 0) {
          if constexpr (CG == 1) {
            mbar_arrive_expect_tx(&full[s], Cfg::A_BYTES + Cfg::B_BYTES);
            if (kb == kb0 && w == 0) GEMM_STAMP(3);
            tma_load_2d(sA + s * Cfg::A_BYTES, &tmA, &full[s], kb * kGemmBK, row_a);
#pragma unroll
            for (int h = 0; h < BN / 128; ++h)  // weight maps use 128-row boxes
              tma_load_2d_hint(sB + s * Cfg::B_BYTES + h * 16384, &tmB, &full[s], kb * kGemmBK,
                               row_b + h * 128, pol_b);
          } else {
            // The peer's bytes are counted on the leader's barrier by the 2-SM TMA; it cannot
            // run ahead into this phase before the leader's MMA released the stage (empty).
            if (leader) mbar_arrive_expect_tx(&full[s], 2 * (Cfg::A_BYTES + Cfg::B_BYTES));
            tma_load_2d_2sm(sA + s * Cfg::A_BYTES, &tmA, &full[s], kb * kGemmBK, row_a, pol_b);
            tma_load_2d_2sm(sB + s * Cfg::B_BYTES, &tmB, &full[s], kb * kGemmBK, row_b, pol_b);
          }
        }
        __syncwarp();
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
    }
    if (lane == 0) grid_dep_launch();  // all loads issued: the next kernel may start its prologue
  } else if (warp == 1 && leader) {
    constexpr uint32_t idesc = make_idesc_bf16(Cfg::TILE_M, BN);
    int s = 0;
    uint32_t ph = 0;
    int it = 0;
    for (int w = 0; w < n_work; ++w, ++it) {
      int tile, split, nsplit, kb0, kb1, role;
      work_info(w, tile, split, nsplit, kb0, kb1, role);
      const int acc = it & 1;
      const uint32_t acc_ph = (it >> 1) & 1;
      mbar_wait(&tempty[acc], acc_ph ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tbase + acc * BN;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (lane == 0 && kb == kb0 && w == 0) GEMM_STAMP(4);
        if (lane == 0) {
          const uint64_t a0 = make_sdesc_sw128(smem_u32(sA + s * Cfg::A_BYTES), 16, 1024);
          const uint64_t b0 = make_sdesc_sw128(smem_u32(sB + s * Cfg::B_BYTES), 16, 1024);
#pragma unroll
          for (int k = 0; k < kGemmBK / 16; ++k) {
            // +32 bytes along K inside the 128B swizzle atom (descriptor address is >>4)
            if constexpr (CG == 1)
              umma_bf16_ss(d_tmem, a0 + 2 * k, b0 + 2 * k, idesc, (kb != kb0 || k != 0));
            else
              umma_bf16_ss_2sm(d_tmem, a0 + 2 * k, b0 + 2 * k, idesc, (kb != kb0 || k != 0));
          }
          if constexpr (CG == 1) tc_commit(&empty[s]);
          else tc_commit_2sm_mc(&empty[s], 0x3);
        }
        __syncwarp();
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
      if (lane == 0) {
        if constexpr (CG == 1) tc_commit(&tfull[acc]);
        else tc_commit_2sm_mc(&tfull[acc], 0x3);
        GEMM_STAMP(5);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    // fused TP exchange state (xchg == 2): the previous tile still to be folded
    int prev_fidx = -1, prev_m = 0, prev_end = 0, prev_n0 = 0, prev_nb = 0;
    const int xc_now = (EPI == EPI_STORE_BF16 && p.xchg) ? p.guard.tp->local->xcount : 0;
    const int xslot = xc_now & 1;
    const unsigned long long xwant = (unsigned long long)xc_now + 1;
    const int q = warp & 3;  // TMEM lane quadrant
    const int row = q * 32 + lane;
    int it = 0;
    // release an accumulator stage: one arrival per warp on the leader's barrier
    auto release_acc = [&](int acc) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 1) mbar_arrive(&tempty[acc]);
        else mbar_arrive_cluster(&tempty[acc], 0);
      }
    };
    for (int w = 0; w < n_work; ++w, ++it) {
      int tile, split, splits, kb0, kb1, role;
      work_info(w, tile, split, splits, kb0, kb1, role);
      int mb, nb, row_a, row_b, row_end;
      tile_geom(tile, mb, nb, row_a, row_b, row_end);
      const int acc = it & 1;
      const uint32_t acc_ph = (it >> 1) & 1;
      const int m = row_a + row;
      const bool live = m < row_end;
      const int n0 = nb * BN;
      // Partial tiles are stored thread-major ([split][col/4][row] float4) so every warp
      // access is one contiguous 512-byte segment.
      const int wtile = (tile - full_tiles) * CG + (int)rank;  // workspace / ticket slot
      float4* ws_tile =
          reinterpret_cast<float4*>(p.ws) + (long long)wtile * splits * (BN / 4) * kGemmBM;
      const uint32_t tacc = tbase + acc * BN + ((uint32_t)(q * 32) << 16);
      if constexpr (MODE == 3) {
        if (role == 1) {
          // stream-K partial: TMEM -> this CTA's workspace slot ([col/4][row] float4), publish
          mbar_wait(&tfull[acc], acc_ph);
          tc_fence_after();
          float4* dst = reinterpret_cast<float4*>(p.ws) + (long long)blockIdx.x * (BN / 4) * kGemmBM + row;
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(tacc + c * 32, r);
            tmem_ld_wait();
            if (live) {
#pragma unroll
              for (int i = 0; i < 8; ++i)
                st_global_v4(dst + (c * 8 + i) * kGemmBM,
                             make_uint4(r[4 * i], r[4 * i + 1], r[4 * i + 2], r[4 * i + 3]));
            }
          }
          release_acc(acc);
          __threadfence();
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (row == 0) st_release_gpu(p.sk_flags + blockIdx.x, p.sk_epoch);
          continue;
        }
        if (role == 2) {
          // stream-K finisher: add the partners' partials (k order) into the TMEM accumulator,
          // 16 KB chunks (32 columns of one partner) double-buffered through shared memory by
          // bulk copies, then run the ordinary epilogue below
          mbar_wait(&tfull[acc], acc_ph);
          tc_fence_after();
          const long long t0u = (long long)(tile - dp_tiles) * num_k;
          const int g_lo = (int)(((t0u + 1) * sk_g + sk_u - 1) / sk_u) - 1;
          const int P = (int)blockIdx.x - g_lo;
          if (threadIdx.x == 128) {
            for (int g = g_lo; g < (int)blockIdx.x; ++g)
              while (ld_acquire_gpu(p.sk_flags + g) != p.sk_epoch) __nanosleep(32);
            fence_proxy_async_global();
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
          const float4* wsb = reinterpret_cast<const float4*>(p.ws);
          const int steps = (BN / 32) * P;
          auto issue = [&](int step) {  // step = c * P + j: columns [32c, 32c + 32) of partner j
            const int c = step / P, j = step - c * P;
            mbar_arrive_expect_tx(&pbar[step & 1], 16384);
            bulk_g2s(sPart + (step & 1) * 16384, wsb + ((long long)(g_lo + j) * (BN / 4) + c * 8) * kGemmBM,
                     16384, &pbar[step & 1]);
          };
          if (threadIdx.x == 128) {
            issue(0);
            if (steps > 1) issue(1);
          }
          float v[32];
#pragma unroll 1
          for (int step = 0; step < steps; ++step) {
            const int c = step / P, j = step - c * P;
            if (j == 0) {
              uint32_t r[32];
              tmem_ld32(tacc + c * 32, r);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
            }
            mbar_wait(&pbar[step & 1], (step >> 1) & 1);
            const float4* sp = reinterpret_cast<const float4*>(sPart + (step & 1) * 16384) + row;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 f = sp[i * kGemmBM];
              v[4 * i] += f.x;
              v[4 * i + 1] += f.y;
              v[4 * i + 2] += f.z;
              v[4 * i + 3] += f.w;
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");  // every thread is done with the buffer
            if (threadIdx.x == 128 && step + 2 < steps) issue(step + 2);
            if (j == P - 1) {
              uint32_t r[32];
#pragma unroll
              for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(v[i]);
              tmem_st32(tacc + c * 32, r);
              tmem_st_wait();
            }
          }
        }
      }
      if ((MODE == 1 || MODE == 4) && splits > 1) {
        mbar_wait(&tfull[acc], acc_ph);
        if (threadIdx.x == 128) GEMM_STAMP(6);
        tc_fence_after();
        // 1) this K-slice's partial tile -> workspace, TMEM released immediately (cluster split:
        //    -> this CTA's shared memory; the pipeline stages are free, all of its MMAs are done)
        constexpr bool dsm = MODE == 4;
        float4* dst = dsm ? reinterpret_cast<float4*>(smem) + row
                          : ws_tile + (long long)split * (BN / 4) * kGemmBM + row;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(tacc + c * 32, r);
          tmem_ld_wait();
          if (live) {  // dead rows (m >= M) are neither stored nor reduced
#pragma unroll
            for (int i = 0; i < 8; ++i)  // generic store: global workspace or shared memory
              *reinterpret_cast<uint4*>(dst + (c * 8 + i) * kGemmBM) =
                  make_uint4(r[4 * i], r[4 * i + 1], r[4 * i + 2], r[4 * i + 3]);
          }
        }
        if (threadIdx.x == 128) GEMM_STAMP(7);
        release_acc(acc);
        // 2) wait until all `splits` K-slices of this 128-row tile slot are stored. Safe to
        //    spin: the launcher gives every CTA at most one split unit, as its last unit, and
        //    the grid never exceeds one CTA (pair) per SM, so all siblings are resident.
        int* tk = p.tickets + wtile;  // [0, 1024): arrivals, +1024: done
        if constexpr (dsm) {  // the tile's K-slice CTAs are this cluster (the other warps join)
          cluster_arrive_release();
          cluster_wait_acquire();
        } else {
          split_barrier(tk, splits);
        }
        if (threadIdx.x == 128) GEMM_STAMP(8);
        // 3) this K-slice's share of the tile's (row, column-group) epilogue items, each the
        //    split-order sum of the partials (deterministic) -- the reduction is spread over
        //    all K-slice CTAs instead of one CTA reducing the whole tile
        const int m_base = row_a;
        const int live_rows = min(kGemmBM, p.M - m_base);
        const SplitSum<dsm> gsum{ws_tile, smem_u32(smem), splits};
        // 8 items per row, row-major: a warp covers 4 whole rows. Warp groups of 32 items are
        // dealt to the K-slice CTAs first (group gi -> slice gi % S, warp gi / S % 4), so a
        // short tile's reduction reads spread over all S SMs instead of the first few (the
        // reads are per-SM bandwidth bound: tools/gemm_stamps.py it_start -> it_sum)
        const int items = live_rows * 8;
        for (int gi = q * splits + split; gi * 32 < items; gi += 4 * splits) {
          const int item = gi * 32 + lane;
          const int r = item >> 3;
          split_item_epilogue<EPI>(p, gsum, item < items, m_base + r, r, item & 7, n0, nb);
        }
        if (threadIdx.x == 128) GEMM_STAMP(9);
        // 4) the last K-slice through resets the tickets for the next launch (cluster split: the
        //    peers' partials stay live until every K-slice has read them)
        if constexpr (dsm) {
          cluster_arrive_release();
          cluster_wait_acquire();
          continue;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (row == 0 && atomicAdd(tk + 1024, 1) == splits - 1) {
          tk[0] = 0;
          tk[1024] = 0;
        }
        continue;
      }
      // Unsplit tile: accumulator columns [col, col+32) of this thread's row from TMEM.
      // fused RMSNorm: the row's rsqrt factor (1 for epilogues without a norm in front)
      float rs = 1.f;
      if ((EPI == EPI_QKV || EPI == EPI_SWIGLU || EPI == EPI_STORE_F32) && p.ssq_in != nullptr &&
          live) {
        const int tok = MODE == 2 ? p.grp_perm[m] : m;
        rs = fused_norm_rsqrt(p.ssq_in + (long long)tok * p.nseg, p.nseg, p.norm_eps_in);
      }
      auto load32 = [&](int col, float* v) {
        uint32_t r[32];
        tmem_ld32(tacc + col, r);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * rs;
      };

      if constexpr (EPI == EPI_RESID) {
        // residual row segment prefetched into registers while the MMA runs (MODE 1 loads it
        // per 32-column chunk instead: the split path's registers leave no room for 128 more)
        constexpr bool kPrefetch = MODE != 1 && MODE != 4;
        uint4 hres[kPrefetch ? BN / 8 : 1];
        __nv_bfloat16* hrow = p.resid + (long long)m * p.ldr + n0;
        if (kPrefetch && live) {
#pragma unroll
          for (int i = 0; i < BN / 8; ++i) hres[i] = ld_global_v4(hrow + 8 * i);
        }
        mbar_wait(&tfull[acc], acc_ph);
        if (threadIdx.x == 128) GEMM_STAMP(6);
        tc_fence_after();
        float ss = 0.f;
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {
          float v[32];
          load32(c * 32, v);
          if (live) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint4 h = kPrefetch ? hres[(c * 4 + i) % (kPrefetch ? BN / 8 : 1)]
                                        : ld_global_v4(hrow + c * 32 + 8 * i);
              const uint32_t hw[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float2 f = unpack_bf16x2(hw[j]);
                v[8 * i + 2 * j] += f.x;
                v[8 * i + 2 * j + 1] += f.y;
              }
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) {  // the next norm sees the bf16-rounded values
              const float rv = __bfloat162float(__float2bfloat16(v[i]));
              ss += rv * rv;
            }
            store_row32_bf16(hrow + c * 32, v);
          }
          if ((c & 3) == 3) {  // a 128-column segment of the new h is complete
            if (live && p.ssq_out) p.ssq_out[(long long)m * p.nseg + nb * (BN / 128) + (c >> 2)] = ss;
            ss = 0.f;
          }
        }
      } else if constexpr (EPI == EPI_STORE_BF16 || EPI == EPI_STORE_F32) {
        void* out = p.out;
        if (EPI == EPI_STORE_BF16 && p.xchg) {
          const TpDev* tp = p.guard.tp;
          out = tp->part[tp->rank][tp->local->xcount & 1];
        }
        mbar_wait(&tfull[acc], acc_ph);
        if (threadIdx.x == 128) GEMM_STAMP(6);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          float v[32];
          load32(c * 32, v);
          if (live) {
            if constexpr (EPI == EPI_STORE_F32) {
              float* dst = reinterpret_cast<float*>(out) + (long long)m * p.ldo + n0 + c * 32;
#pragma unroll
              for (int i = 0; i < 8; ++i)
                st_global_v4(dst + 4 * i,
                             make_uint4(__float_as_uint(v[4 * i]), __float_as_uint(v[4 * i + 1]),
                                        __float_as_uint(v[4 * i + 2]),
                                        __float_as_uint(v[4 * i + 3])));
            } else {
              __nv_bfloat16* dst =
                  reinterpret_cast<__nv_bfloat16*>(out) + (long long)m * p.ldo + n0 + c * 32;
              store_row32_bf16(dst, v);
            }
          }
        }
      } else if constexpr (EPI == EPI_SWIGLU) {
        mbar_wait(&tfull[acc], acc_ph);
        if (threadIdx.x == 128) GEMM_STAMP(6);
        tc_fence_after();
        // Tile columns [0, BN/2) are gate rows, [BN/2, BN) the matching up rows.
#pragma unroll 1
        for (int c = 0; c < BN / 64; ++c) {
          float g[32], up[32];
          load32(c * 32, g);
          load32(BN / 2 + c * 32, up);
          if (live) {
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = silu_f(g[i]) * up[i];
            __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.out) + (long long)m * p.ldo +
                                 nb * (BN / 2) + c * 32;
            store_row32_bf16(dst, v);
          }
        }
      } else {  // EPI_QKV: 128-column heads
        const int pos = live ? p.pos[m] : 0;
        const int page = live ? p.tok_page[m] : 0;
        // (cos, sin) of the row's position for the 64 rotation pairs, prefetched during the MMA
        // (MODE 1 reads them per half at use: no room for 128 prefetched registers there)
        constexpr bool kPrefetch = MODE != 1 && MODE != 4;
        float4 cs[kPrefetch ? 32 : 1];
        const bool rot = n0 < p.q_cols + p.kv_cols;  // tile holds q/k heads (v heads unrotated)
        const float4* cs_src = reinterpret_cast<const float4*>(p.rope + (long long)pos * 64);
        if (kPrefetch && live && rot) {
          const float4* src = reinterpret_cast<const float4*>(p.rope + (long long)pos * 64);
#pragma unroll
          for (int i = 0; i < 32; ++i) cs[i] = __ldg(src + i);
        }
        mbar_wait(&tfull[acc], acc_ph);
        if (threadIdx.x == 128) GEMM_STAMP(6);
        tc_fence_after();
#pragma unroll
        for (int hh = 0; hh < BN / 128; ++hh) {
          const int col0 = n0 + hh * 128;
          if (col0 >= p.q_cols + 2 * p.kv_cols) continue;  // zero padding of the qkv width
          const bool is_q = col0 < p.q_cols;
          const bool is_v = col0 >= p.q_cols + p.kv_cols;
          __nv_bfloat16* dst;
          if (is_q) {
            dst = p.qbuf + (long long)m * p.ldq + col0;
          } else {
            const int kv = is_v ? 1 : 0;
            const int h = (col0 - p.q_cols - kv * p.kv_cols) >> 7;
            dst = p.kv_layer +
                  ((((long long)page * 2 + kv) * p.n_kv_heads + h) * p.page_size +
                   (pos % p.page_size)) *
                      128;
          }
          const float* bias = p.bias ? p.bias + col0 : nullptr;
          const float* hn = is_v ? nullptr : (is_q ? p.q_norm : p.k_norm);
          float nscale = 1.f;
          if (hn != nullptr) {  // per-head RMSNorm (Qwen3): sum of squares over the head first
            float ss = 0.f;
#pragma unroll 1
            for (int c4 = 0; c4 < 4; ++c4) {
              float a[32];
              load32(hh * 128 + c4 * 32, a);
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const float x = a[i] + (bias ? __ldg(bias + c4 * 32 + i) : 0.f);
                ss += x * x;
              }
            }
            nscale = rsqrtf(ss * (1.f / 128.f) + p.norm_eps);
          }
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            // chunk pair (half, half+2): columns j and j+64 of the head for j in this chunk
            float a[32], b[32];
            load32(hh * 128 + half * 32, a);
            load32(hh * 128 + half * 32 + 64, b);
            if (live) {
              if (bias) {
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                  a[i] += __ldg(bias + half * 32 + i);
                  b[i] += __ldg(bias + half * 32 + 64 + i);
                }
              }
              if (hn) {
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                  a[i] *= nscale * __ldg(hn + half * 32 + i);
                  b[i] *= nscale * __ldg(hn + half * 32 + 64 + i);
                }
              }
              if (!is_v) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                  // (cos, sin) of columns 2i, 2i+1
                  const float4 t4 = kPrefetch ? cs[(half * 16 + i) % (kPrefetch ? 32 : 1)]
                                              : __ldg(cs_src + half * 16 + i);
                  const float u1 = a[2 * i], u2 = b[2 * i];
                  const float w1 = a[2 * i + 1], w2 = b[2 * i + 1];
                  a[2 * i] = u1 * t4.x - u2 * t4.y;
                  b[2 * i] = u2 * t4.x + u1 * t4.y;
                  a[2 * i + 1] = w1 * t4.z - w2 * t4.w;
                  b[2 * i + 1] = w2 * t4.z + w1 * t4.w;
                }
              }
              store_row32_bf16(dst + half * 32, a);
              store_row32_bf16(dst + half * 32 + 64, b);
            }
          }
        }
      }
      if (threadIdx.x == 128) GEMM_STAMP(7);
      release_acc(acc);
      if constexpr (EPI == EPI_STORE_BF16 && MODE == 0) {
        if (p.xchg == 2) {
          // flag this tile's partial to the peers, then fold the previous tile of all ranks
          // (its peers' partials are due by now) while the tensor core runs the next tile
          const TpDev* tp = p.guard.tp;
          __threadfence_system();
          asm volatile("bar.sync 1, 128;" ::: "memory");
          const int fidx = tile * CG + (int)rank;
          if (row == 0)
            st_release_sys_u64(&tp->peer[tp->rank]->flags[xslot][fidx], xwant);
          if (prev_fidx >= 0)
            tp_fold_tile(p, tp, xslot, xwant, prev_fidx, prev_m, prev_end, prev_n0, prev_nb);
          prev_fidx = fidx;
          prev_m = row_a;
          prev_end = row_end;
          prev_n0 = n0;
          prev_nb = nb;
        }
      }
    }
    if constexpr (EPI == EPI_STORE_BF16 && MODE == 0) {
      if (p.xchg == 2 && prev_fidx >= 0)
        tp_fold_tile(p, p.guard.tp, xslot, xwant, prev_fidx, prev_m, prev_end, prev_n0, prev_nb);
    }
    if (EPI == EPI_STORE_BF16 && p.xchg) __threadfence_system();  // partials visible to peers
  }

  if (MODE == 4 && run && warp < 4) {  // the cluster split's two barriers
    cluster_arrive_release();
    cluster_wait_acquire();
    cluster_arrive_release();
    cluster_wait_acquire();
  }
  if (threadIdx.x == 0) GEMM_STAMP(10);
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync_all();  // the pair's MMAs/arrivals are all done
  else __syncthreads();
  if (EPI == EPI_STORE_BF16 && p.xchg == 1 && run && threadIdx.x == 0) tp_publish_partial(p.guard.tp);
  if (EPI == EPI_STORE_BF16 && p.xchg == 2 && run && threadIdx.x == 0) {
    // the last CTA out completes the exchange (every tile of every rank is folded)
    const TpDev* tp = p.guard.tp;
    __threadfence();
    if (atomicAdd(&tp->local->ar_ctr, 1) == (int)(gridDim.x * gridDim.y * gridDim.z) - 1) {
      tp->local->ar_ctr = 0;
      tp->local->xcount = tp->local->xcount + 1;
      __threadfence();
    }
  }
  if (threadIdx.x == 64) GEMM_STAMP(11);
  if (warp == 2) {
    tc_fence_after();
    if constexpr (CG == 2) tmem_dealloc_2sm<Cfg::TMEM_COLS>(tbase);
    else tmem_dealloc<Cfg::TMEM_COLS>(tbase);
  }
}

}  // namespace fp
