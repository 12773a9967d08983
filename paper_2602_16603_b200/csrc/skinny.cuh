// Swap-AB ("skinny") tcgen05 GEMM for short launches (M <= 256 tokens): the WEIGHT rows are the
// MMA M dimension (128 per MMA) and the tokens the MMA N dimension (any multiple of 16), so a
// 42-token request pays for 48 accumulator columns instead of a 128-row tile, and every SM
// streams its own contiguous share of the weight matrix.
//
//   C[M, N] = A[M, K] * B[N, K]^T  computed as  C^T[N, M] = B[N, K] * A[M, K]^T
//
// Realises the same reference entries as gemm.cuh (prefillsim/cost_model.py:38-44, 234-242:
// qkv_proj / o_proj / gate_up_proj / down_proj of a chunk with few concatenated tokens, plus the
// lm_head at one row per request). Short launches are weight-streaming bound (a Llama-3-8B layer
// streams 435 MB of weights, ~56 us at 7.7 TB/s, for 18 GFLOP at 42 tokens, ~13 us at
// 1.4 PFLOP/s), so the launch is planned for HBM: the (128-row weight slice, 64-wide k-block) space is cut into one equal contiguous range
// per CTA, stream-K fashion, so all SMs pull weights for the whole launch with no wave
// quantisation. Each CTA's range covers a few "segments" (one weight slice, a k-block range);
// each segment's fp32 partial goes to its own workspace slot ([token][128 cols], coalesced
// stores); after one grid-wide arrival every warp of the grid takes a share of the output's
// (256-column block, 4 token rows) groups, sums each block's slots in contributor order --
// deterministic, the same bits on every run -- and runs the fused epilogue of gemm.cuh
// (split_item_epilogue: residual + segment sums of squares, SwiGLU, QKV + RoPE + paged KV
// scatter, fp32 logits).
//
// The auto plan (runtime.cu launch_gemm_skinny) takes it where the B200 A/B shows it ahead of
// the tiled plans: a few rows (M <= 8: lm_head, tiny chunks) and long-K launches up to 128 rows.
//
// Layout of one CTA (256 threads, 1 CTA / SM): warp 0 TMA producer (weight box 128 x 64 with an
// evict-first hint: streamed once; token boxes 32 x 64, evict-last: re-read by every CTA),
// warp 1 MMA issuer (tcgen05.mma.cta_group::1.kind::f16, M = 128, N = round16(M_tokens)),
// warp 2 TMEM allocator (2 accumulator stages), warps 4..7 drain / finish.
#pragma once
#include "gemm.cuh"

namespace fp {

template <int TOKMAX>
struct SkinnyCfg {
  static constexpr int W_BYTES = 128 * kGemmBK * 2;     // weight box: 16 KB
  static constexpr int X_BYTES = TOKMAX * kGemmBK * 2;  // token rows (32-row boxes)
  static constexpr int STAGE = W_BYTES + X_BYTES;
  static constexpr int STAGES = (196608 / STAGE) < 8 ? (196608 / STAGE) : 8;
  static constexpr int TMEM_COLS = 2 * TOKMAX < 32 ? 32 : 2 * TOKMAX;
  static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE + 256;
};
constexpr int kSkinnyMaxM = 256;

// Partition of the (weight slice, k-block) space: U units over G CTAs, CTA g owns
// [g U / G, (g + 1) U / G). owner(u) = the CTA whose range holds unit u.
struct SkinnyPart {
  long long U;
  int G, num_k;
  DEVI long long start(int g) const { return (long long)g * U / G; }
  DEVI int owner(long long u) const { return (int)(((u + 1) * G + U - 1) / U) - 1; }
};

// Sum provider for split_item_epilogue: the workspace slots of the block's two 128-column halves
// ([token][128] fp32 each), contributors summed in CTA order.
struct SkinnySum {
  const float* ws;
  long long slot_elems;  // M * 128
  int first0, first1, count0, count1;  // slot range of columns [0, 128) and [128, 256)
  template <int ILP = 4>
  DEVI void get(int r, int colA, int colB, float* v) const {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = 0.f;
    const int fa = colA < 128 ? first0 : first1, ca = colA < 128 ? count0 : count1;
    const int fb = colB < 128 ? first0 : first1, cb = colB < 128 ? count0 : count1;
    const float4* sa = reinterpret_cast<const float4*>(ws + (long long)fa * slot_elems +
                                                       (long long)r * 128 + (colA & 127));
    const float4* sb = reinterpret_cast<const float4*>(ws + (long long)fb * slot_elems +
                                                       (long long)r * 128 + (colB & 127));
    const long long st4 = slot_elems / 4;
    const int n = max(ca, cb);
    for (int s0 = 0; s0 < n; s0 += ILP) {
      float4 f[ILP][8];
#pragma unroll
      for (int j = 0; j < ILP; ++j) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
          f[j][i] = s0 + j < ca ? __ldcg(sa + (s0 + j) * st4 + i) : z;
          f[j][4 + i] = s0 + j < cb ? __ldcg(sb + (s0 + j) * st4 + i) : z;
        }
      }
#pragma unroll
      for (int j = 0; j < ILP; ++j) {
        if (s0 + j < n) {
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
  }
};

// tmX: token activations [rows >= M, K] with 32-row boxes; tmW: weights [N, K] with 128-row
// boxes (the maps gemm.cuh uses for B). p.ws needs (gridDim.x + N / 128) * M * 128 floats;
// p.tickets[2048..2049] must be zero on entry (the last CTA out resets them). gridDim.x must not
// exceed the number of SMs (one resident CTA per SM).
template <int EPI, int TOKMAX>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_skinny_kernel(const __grid_constant__ CUtensorMap tmX,
                       const __grid_constant__ CUtensorMap tmW, const GemmParams p) {
  using Cfg = SkinnyCfg<TOKMAX>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
  uint8_t* sW = smem;
  uint8_t* sX = smem + STAGES * Cfg::W_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sX + STAGES * Cfg::X_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  if (threadIdx.x == 0) GEMM_STAMP(0);
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmX);
    tma_prefetch(&tmW);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  if (threadIdx.x == 0) GEMM_STAMP(1);
  grid_dep_wait();
  const bool run = guard_block(p.guard);
  if (threadIdx.x == 0) GEMM_STAMP(2);

  const int M = p.M;
  const int ntok = (M + 15) & ~15;   // MMA N
  const int nbox = (M + 31) >> 5;    // 32-row token boxes per stage
  const int num_k = p.K / kGemmBK;
  SkinnyPart part{(long long)(p.N / 128) * num_k, (int)gridDim.x, num_k};
  const long long u0 = part.start(blockIdx.x), u1 = part.start(blockIdx.x + 1);
  const int t_first = (int)(u0 / num_k);
  const int n_seg = !run || u1 <= u0 ? 0 : (int)((u1 - 1) / num_k) - t_first + 1;
  auto seg = [&](int i, int& t, int& kb0, int& kb1) {
    t = t_first + i;
    kb0 = (int)max(u0 - (long long)t * num_k, 0LL);
    kb1 = (int)min(u1 - (long long)t * num_k, (long long)num_k);
  };

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      int s = 0;
      uint32_t ph = 0;
      for (int i = 0; i < n_seg; ++i) {
        int t, kb0, kb1;
        seg(i, t, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], Cfg::W_BYTES + nbox * 4096);
          if (i == 0 && kb == kb0) GEMM_STAMP(3);
          tma_load_2d_hint(sW + s * Cfg::W_BYTES, &tmW, &full[s], kb * kGemmBK, t * 128, pol_w);
          for (int b = 0; b < nbox; ++b)
            tma_load_2d_hint(sX + s * Cfg::X_BYTES + b * 4096, &tmX, &full[s], kb * kGemmBK,
                             b * 32, pol_x);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
      grid_dep_launch();
    }
    __syncwarp();
  } else if (warp == 1) {
    const uint32_t idesc = make_idesc_bf16(128, ntok);
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < n_seg; ++i) {
      int t, kb0, kb1;
      seg(i, t, kb0, kb1);
      const int acc = i & 1;
      mbar_wait(&tempty[acc], ((i >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tbase + acc * TOKMAX;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (lane == 0 && i == 0 && kb == kb0) GEMM_STAMP(4);
        if (lane == 0) {
          const uint64_t a0 = make_sdesc_sw128(smem_u32(sW + s * Cfg::W_BYTES), 16, 1024);
          const uint64_t b0 = make_sdesc_sw128(smem_u32(sX + s * Cfg::X_BYTES), 16, 1024);
#pragma unroll
          for (int k = 0; k < kGemmBK / 16; ++k)
            umma_bf16_ss(d_tmem, a0 + 2 * k, b0 + 2 * k, idesc, (kb != kb0 || k != 0));
          tc_commit(&empty[s]);
        }
        __syncwarp();
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
      if (lane == 0) tc_commit(&tfull[acc]);
      if (lane == 0 && i == n_seg - 1) GEMM_STAMP(5);
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int row = q * 32 + lane;  // weight row inside the 128-row slice
    const long long slot_elems = (long long)M * 128;
    for (int i = 0; i < n_seg; ++i) {
      int t, kb0, kb1;
      seg(i, t, kb0, kb1);
      const int acc = i & 1;
      mbar_wait(&tfull[acc], (i >> 1) & 1);
      tc_fence_after();
      if (row == 0 && i == 0) GEMM_STAMP(6);
      // partial -> slot (CTA g, slice t) = g + t: [token][128] fp32, each warp store is one
      // contiguous 128-byte row segment
      float* dst = p.ws + (long long)(blockIdx.x + t) * slot_elems + row;
      const uint32_t tacc = tbase + acc * TOKMAX + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < ntok; c += 32) {
        uint32_t r[32];
        tmem_ld32(tacc + c, r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (c + j < M) __stcg(dst + (long long)(c + j) * 128, __uint_as_float(r[j]));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
    if (row == 0) GEMM_STAMP(7);
    if (n_seg > 0) {
      // Every partial of the launch is in the workspace once all CTAs arrive (the grid is at
      // most one CTA per SM, all resident: the next kernel launches only after every CTA has
      // issued its loads). Then the reduction + fused epilogue is spread over all warps of the
      // grid -- a single finisher per block is a serial L2-latency chain (~70 us at M = 256).
      int* ctr = p.tickets + 2048;  // [0] arrivals, [1] departures (zero between launches)
      // the CTA barrier orders the 128 drains before row 0's cumulative gpu-scope fence and
      // arrival; its acquiring spin + the second barrier order everyone's loads after it
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (row == 0) {
        __threadfence();
        atomicAdd(ctr, 1);
        while (ld_acquire_gpu(ctr) < (int)gridDim.x) __nanosleep(20);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (row == 0) GEMM_STAMP(8);
      // work group = 4 token rows x 8 items of one 256-column block (one warp; the 8 items of
      // a row are 8 consecutive lanes, as split_item_epilogue's shuffles require)
      const int gpb = (M + 3) >> 2;
      const int total = (p.N / 256) * gpb;
      // groups dealt to the CTAs first (gi -> CTA gi % G, warp gi / G): the reads are per-SM
      // bandwidth bound, so a short launch spreads them over every SM
      for (int gi = q * (int)gridDim.x + (int)blockIdx.x; gi < total; gi += (int)gridDim.x * 4) {
        const int nb = gi / gpb;
        const int item = (gi - nb * gpb) * 32 + lane;
        const int r = item >> 3;
        const long long ua = (long long)(2 * nb) * num_k;
        const int g_lo0 = part.owner(ua), g_hi0 = part.owner(ua + num_k - 1);
        const int g_lo1 = part.owner(ua + num_k), g_hi1 = part.owner(ua + 2 * num_k - 1);
        SkinnySum sum;
        sum.ws = p.ws;
        sum.slot_elems = slot_elems;
        sum.first0 = g_lo0 + 2 * nb;
        sum.count0 = g_hi0 - g_lo0 + 1;
        sum.first1 = g_lo1 + 2 * nb + 1;
        sum.count1 = g_hi1 - g_lo1 + 1;
        split_item_epilogue<EPI>(p, sum, r < M, r, r, item & 7, nb * 256, nb);
      }
      // the last CTA out re-arms the counters (every CTA has passed the arrival spin)
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (row == 0) GEMM_STAMP(9);
      if (row == 0 && atomicAdd(ctr + 1, 1) == (int)gridDim.x - 1) {
        ctr[0] = 0;
        ctr[1] = 0;
        __threadfence();
      }
    }
  }
  if (threadIdx.x == 0) GEMM_STAMP(10);
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<Cfg::TMEM_COLS>(tbase);
  }
}

}  // namespace fp
