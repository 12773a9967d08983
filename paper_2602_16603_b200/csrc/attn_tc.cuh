// Causal varlen flash-attention prefill on tcgen05 / TMEM / TMA (GQA, head_dim 128).
//
// Realises the reference's `attn` timeline entry (prefillsim/cost_model.py:226-233): each
// request's share of the chunk attends causally to its OWN prefix + share, never across the
// batch (pkg/tests/test_cost_model.py:88-109). All K/V -- the prefix written by earlier chunks
// and this chunk's share written moments ago by the qkv_proj epilogue -- are read from the paged
// cache, one 128-token page per KV tile, so tiles sit at ABSOLUTE request positions and a query
// row's result is independent of chunking and batch composition.
//
// CTA = one 128-row query tile x two query heads of the same KV head (GQA pair), so both heads
// share every K/V tile in shared memory. Warp roles (320 threads, 1 CTA/SM):
//   warp 0       TMA producer: Q tiles once, then K_j, V_j into a 3-slot ring (pages via the
//                block table; 128B-swizzled 64-column boxes)
//   warp 1       TMEM allocator + single-thread MMA issuer:
//                  S_h = Q_h K_j^T      (SS, M=128 N=128 K=128, fp32 accumulators in TMEM)
//                  O_h += P_h V_j       (TS: P read from TMEM, V MN-major from smem)
//                issued ping-pong so head 1's MMAs overlap head 0's softmax and vice versa
//   warps 2-5    softmax for head 0, warps 6-9 softmax for head 1: one query row per thread,
//                exp2 online softmax, lazy O rescale (only when the row max grows by > 2^8),
//                P written back to TMEM over S as bf16, final O / l epilogue to HBM.
// TMEM columns: S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512).
#pragma once
#include "common.cuh"
#include "control.cuh"

namespace fp {

struct AttnTile {
  int q_row0;  // first chunk row of this 128-row tile
  int n_rows;  // valid rows
  int q_pos0;  // position (inside its request) of the first row
  int req;     // request index -> block table row
};

struct AttnTcParams {
  const AttnTile* items;
  int n_items;
  int n_heads, n_kv_heads;
  int pairs_per_kv;               // ceil((n_heads / n_kv_heads) / 2)
  __nv_bfloat16* out;             // [M, n_heads*128]
  long long ldo;
  const int* block_table;         // [n_req, bt_stride]
  int bt_stride;
  long long kv_row_layer;         // row of (layer, page 0, k, head 0, slot 0) in the pool map
  int kv_rows_per_page;           // 2 * n_kv_heads * 128 rows per page (one layer)
  float scale_log2;               // log2(e) / sqrt(128)
  Guard guard;
};

namespace tcattn {
constexpr int THREADS = 320;
constexpr int TILE = 128;
constexpr int TILE_BYTES = 128 * 128 * 2;  // 32 KB: two 64-column swizzle atoms of 16 KB
constexpr int ATOM_BYTES = 16384;
constexpr int STAGES = 3;
constexpr int SMEM_BYTES = 1024 + 2 * TILE_BYTES + STAGES * TILE_BYTES + 256;
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units: rescale O only if max grows > 256x
}  // namespace tcattn

__global__ void __launch_bounds__(tcattn::THREADS, 1)
    attn_prefill_tc_kernel(const __grid_constant__ CUtensorMap tmQ,
                           const __grid_constant__ CUtensorMap tmKV, const AttnTcParams p) {
  using namespace tcattn;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
  uint8_t* sQ = smem;                      // [2][TILE_BYTES]
  uint8_t* sKV = smem + 2 * TILE_BYTES;    // [STAGES][TILE_BYTES]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + STAGES * TILE_BYTES);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + STAGES;
  uint64_t* s_full = kv_empty + STAGES;  // [2]
  uint64_t* p_full = s_full + 2;         // [2]
  uint64_t* o_full = p_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 1);


  const int warp = warp_id();
  const int lane = lane_id();
  // prologue (overlaps the previous kernel's tail under programmatic dependent launch)
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmKV);
    mbar_init(q_full, 1);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int h = 0; h < 2; ++h) {
      mbar_init(&s_full[h], 1);
      mbar_init(&p_full[h], 128);
    }
    mbar_init(o_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  grid_dep_wait();
  const bool run = guard_block(p.guard);

  const AttnTile it = p.items[blockIdx.x];
  const int kvh = blockIdx.y / p.pairs_per_kv;
  const int pair = blockIdx.y % p.pairs_per_kv;
  const int group = p.n_heads / p.n_kv_heads;
  const int head0 = kvh * group + 2 * pair;
  const bool has_head1 = 2 * pair + 1 < group;
  const int head1 = has_head1 ? head0 + 1 : head0;
  const int kv_len = it.q_pos0 + it.n_rows;
  const int n_tiles = (kv_len + TILE - 1) / TILE;
  const int* bt = p.block_table + (long long)it.req * p.bt_stride;

  if (!run) {
    // stopped at this boundary: nothing to do
  } else if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_last();  // K/V tiles are re-read by other q tiles
      mbar_arrive_expect_tx(q_full, 2 * TILE_BYTES);
      for (int h = 0; h < 2; ++h) {
        const int col = (h ? head1 : head0) * 128;
        tma_load_2d(sQ + h * TILE_BYTES, &tmQ, q_full, col, it.q_row0);
        tma_load_2d(sQ + h * TILE_BYTES + ATOM_BYTES, &tmQ, q_full, col + 64, it.q_row0);
      }
      int s = 0;
      uint32_t ph = 0;
      for (int j = 0; j < n_tiles; ++j) {
        const long long page = bt[j];  // page_size == TILE
        for (int kv = 0; kv < 2; ++kv) {
          mbar_wait(&kv_empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&kv_full[s], TILE_BYTES);
          const long long row =
              p.kv_row_layer + page * p.kv_rows_per_page + (long long)(kv * p.n_kv_heads + kvh) * TILE;
          tma_load_2d_hint(sKV + s * TILE_BYTES, &tmKV, &kv_full[s], 0, (int)row, pol);
          tma_load_2d_hint(sKV + s * TILE_BYTES + ATOM_BYTES, &tmKV, &kv_full[s], 64, (int)row,
                           pol);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_qk = make_idesc_bf16(128, 128, false);
    constexpr uint32_t idesc_pv = make_idesc_bf16(128, 128, true);  // V is MN-major
    const uint32_t tS[2] = {tbase, tbase + 128};
    const uint32_t tO[2] = {tbase + 256, tbase + 384};
    uint32_t seq = 0;  // ring sequence number of the next tile to consume
    auto slot_of = [&](uint32_t sq) { return (int)(sq % STAGES); };
    auto wait_tile = [&](uint32_t sq) { mbar_wait(&kv_full[slot_of(sq)], (sq / STAGES) & 1); };
    auto issue_qk = [&](int h, uint32_t ksq) {
      const uint32_t kb = smem_u32(sKV + slot_of(ksq) * TILE_BYTES);
      const uint32_t qb = smem_u32(sQ + h * TILE_BYTES);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {  // head_dim 128 = 8 x K16; two 64-wide swizzle atoms
        const uint32_t off = (kk >> 2) * ATOM_BYTES + (kk & 3) * 32;
        umma_bf16_ss(tS[h], make_sdesc_sw128(qb + off, 16, 1024),
                     make_sdesc_sw128(kb + off, 16, 1024), idesc_qk, kk > 0);
      }
    };
    auto issue_pv = [&](int h, uint32_t vsq, bool acc) {
      const uint32_t vb = smem_u32(sKV + slot_of(vsq) * TILE_BYTES);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {  // 128 kv rows = 8 x K16; P: 8 TMEM columns per step
        umma_bf16_ts(tO[h], tS[h] + kk * 8, make_sdesc_sw128(vb + kk * 2048, ATOM_BYTES, 1024),
                     idesc_pv, (acc || kk > 0) ? 1u : 0u);
      }
    };
    mbar_wait(q_full, 0);
    wait_tile(0);
    tc_fence_after();
    if (lane == 0) {
      issue_qk(0, 0);
      tc_commit(&s_full[0]);
      issue_qk(1, 0);
      tc_commit(&s_full[1]);
      tc_commit(&kv_empty[slot_of(0)]);
    }
    __syncwarp();
    seq = 1;
    for (int j = 0; j < n_tiles; ++j) {
      const bool last = j == n_tiles - 1;
      const uint32_t vsq = seq;      // V_j
      const uint32_t ksq = seq + 1;  // K_{j+1}
      wait_tile(vsq);
      mbar_wait(&p_full[0], j & 1);
      tc_fence_after();
      if (lane == 0) issue_pv(0, vsq, j > 0);
      __syncwarp();
      if (!last) {
        wait_tile(ksq);
        tc_fence_after();
        if (lane == 0) {
          issue_qk(0, ksq);
          tc_commit(&s_full[0]);
        }
        __syncwarp();
      }
      mbar_wait(&p_full[1], j & 1);
      tc_fence_after();
      if (lane == 0) {
        issue_pv(1, vsq, j > 0);
        tc_commit(&kv_empty[slot_of(vsq)]);
        if (!last) {
          issue_qk(1, ksq);
          tc_commit(&s_full[1]);
          tc_commit(&kv_empty[slot_of(ksq)]);
        }
      }
      __syncwarp();
      seq += 2;
    }
    if (lane == 0) tc_commit(o_full);
    __syncwarp();
  } else {
    // ------------------------------------------------------------------ softmax + epilogue
    const int h = (warp - 2) >> 2;  // 0: warps 2-5, 1: warps 6-9
    const int quad = warp & 3;      // TMEM lane quadrant accessible to this warp
    const int row = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const uint32_t tS = tbase + h * 128 + lane_off;
    const uint32_t tO = tbase + 256 + h * 128 + lane_off;
    const int qpos = it.q_pos0 + row;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n_tiles; ++j) {
      mbar_wait(&s_full[h], j & 1);
      tc_fence_after();
      uint32_t sr[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tS + c * 32, sr[c]);
      tmem_ld_wait();
      const int kv0 = j * TILE;
      const bool diag = kv0 + TILE - 1 > it.q_pos0;
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          float v = __uint_as_float(sr[c][i]) * p.scale_log2;
          if (diag && kv0 + c * 32 + i > qpos) v = -INFINITY;
          sr[c][i] = __float_as_uint(v);
          mx = fmaxf(mx, v);
        }
      }
      const float m_new = fmaxf(m, mx);
      if (j == 0) {
        m = m_new;
      } else {
        const bool need = m_new > m + RESCALE_THRESHOLD;
        if (__any_sync(0xffffffffu, need)) {
          const float alpha = need ? fast_exp2(m - m_new) : 1.f;
          if (need) {
            l *= alpha;
            m = m_new;
          }
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
            tmem_ld32(tO + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(tO + c * 32, o);
          }
          tmem_st_wait();
        }
      }
      const float msub = (m == -INFINITY) ? 0.f : m;
      float sum = 0.f;
      uint32_t pk[2][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float p0 = fast_exp2(__uint_as_float(sr[c][i]) - msub);
          const float p1 = fast_exp2(__uint_as_float(sr[c][i + 1]) - msub);
          sum += p0 + p1;
          pk[c >> 1][(c & 1) * 16 + (i >> 1)] = pack_bf16x2(p0, p1);
        }
      }
      l += sum;
      tmem_st32(tS, pk[0]);
      tmem_st32(tS + 32, pk[1]);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_full[h]);
    }
    // epilogue: O / l -> bf16 -> HBM
    mbar_wait(o_full, 0);
    tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    const bool live = row < it.n_rows && (h == 0 || has_head1);
    __nv_bfloat16* dst = p.out + (long long)(it.q_row0 + row) * p.ldo + (h ? head1 : head0) * 128;
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      uint32_t o[32];
      tmem_ld32(tO + c * 32, o);
      tmem_ld_wait();
      if (live) {
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(o[i]) * inv;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint4 u;
          u.x = pack_bf16x2(v[8 * i + 0], v[8 * i + 1]);
          u.y = pack_bf16x2(v[8 * i + 2], v[8 * i + 3]);
          u.z = pack_bf16x2(v[8 * i + 4], v[8 * i + 5]);
          u.w = pack_bf16x2(v[8 * i + 6], v[8 * i + 7]);
          st_global_v4(dst + c * 32 + 8 * i, u);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

}  // namespace fp
