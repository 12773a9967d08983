// Causal varlen flash-attention prefill over the paged KV cache (GQA, head_dim 128).
//
// Realises the reference's `attn` timeline entry (prefillsim/cost_model.py:226-233): every
// request in the chunk attends only to its OWN prefix + its share of the chunk, causally
// (no cross-request attention, test_cost_model.py:88-109). K/V of the whole visible range are
// read from the paged cache, which the qkv_proj epilogue has just written for this chunk.
//
// Work item = one 64-row query tile of one request segment x one query head. KV tiles of 64
// positions are aligned to ABSOLUTE request positions, so a query row's result does not depend
// on how the batch was chunked or which tile it landed in.
//
// This is the first (mma.sync m16n8k16) implementation; the tcgen05 path supersedes it
// where available (attn_tc.cuh).
#pragma once
#include "common.cuh"
#include "control.cuh"

namespace fp {

struct AttnItem {
  int q_row0;  // first chunk row of this tile
  int n_rows;  // valid rows in the tile
  int q_pos0;  // position (inside its request) of the first row
  int req;     // request index -> block table row
};

struct AttnParams {
  const AttnItem* items;
  int n_items;
  int n_heads;
  const __nv_bfloat16* q;  // [M, n_heads*128]
  long long ldq;
  __nv_bfloat16* out;  // [M, n_heads*128]
  long long ldo;
  const __nv_bfloat16* kv_layer;  // this layer's base of the paged pool
  const int* block_table;         // [n_req, bt_stride]
  int bt_stride;
  int n_kv_heads;
  int page_size;
  float scale_log2;  // log2(e) / sqrt(128)
  Guard guard;
};

namespace mmaattn {
constexpr int BM = 64, BN = 64, HD = 128, THREADS = 128;
constexpr int TILE_BYTES = 64 * 256;  // 64 rows x 128 bf16

DEVI uint32_t swz(int r, int c) {  // byte offset of 16B chunk c of row r (16 chunks per row)
  return (uint32_t)(r * 256 + ((c ^ (r & 7)) << 4));
}
DEVI void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
DEVI void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
DEVI void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
DEVI void ldsm_x4(uint32_t addr, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "r"(addr));
}
DEVI void ldsm_x4_t(uint32_t addr, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "r"(addr));
}
DEVI void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// 64 rows x 128 cols bf16 tile: rows [0, n_valid) from row pointers, others zero-filled.
template <typename RowPtr>
DEVI void load_tile(uint32_t sbase, RowPtr rowptr, int n_valid) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int idx = tid + i * THREADS;  // 0..1023
    const int r = idx >> 4, c = idx & 15;
    const bool v = r < n_valid;
    const __nv_bfloat16* src = v ? rowptr(r) + c * 8 : rowptr(0);
    cp_async16(sbase + swz(r, c), src, v);
  }
}
}  // namespace mmaattn

__global__ void __launch_bounds__(mmaattn::THREADS)
    attn_prefill_mma_kernel(const AttnParams p) {
  using namespace mmaattn;
  if (!guard_block(p.guard)) return;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sQ = smem_u32(smem);
  const uint32_t sK0 = sQ + TILE_BYTES;  // K[2], V[2]
  const AttnItem it = p.items[blockIdx.x];
  const int head = blockIdx.y;
  const int kvh = head / (p.n_heads / p.n_kv_heads);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kv_len = it.q_pos0 + it.n_rows;
  const int n_kv_tiles = (kv_len + BN - 1) / BN;
  const int* bt = p.block_table + (long long)it.req * p.bt_stride;
  const long long head_stride = (long long)p.page_size * HD;

  auto kv_rows = [&](int tile, int kv) {
    const int pos0 = tile * BN;
    const int page = bt[pos0 / p.page_size];
    const __nv_bfloat16* base =
        p.kv_layer + ((((long long)page * 2 + kv) * p.n_kv_heads + kvh) * head_stride) +
        (long long)(pos0 % p.page_size) * HD;
    return base;
  };
  auto load_kv = [&](int tile, int buf) {
    const __nv_bfloat16* kb = kv_rows(tile, 0);
    const __nv_bfloat16* vb = kv_rows(tile, 1);
    const int nv = min(BN, kv_len - tile * BN);
    load_tile(sK0 + (2 * buf) * TILE_BYTES, [&](int r) { return kb + r * HD; }, nv);
    load_tile(sK0 + (2 * buf + 1) * TILE_BYTES, [&](int r) { return vb + r * HD; }, nv);
  };

  // Q tile + first KV tile
  const __nv_bfloat16* qb = p.q + (long long)it.q_row0 * p.ldq + head * HD;
  load_tile(sQ, [&](int r) { return qb + (long long)r * p.ldq; }, it.n_rows);
  load_kv(0, 0);
  cp_commit();

  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  uint32_t qf[8][4];
  const int g = lane >> 2, tq = lane & 3;
  const int qpos_a = it.q_pos0 + warp * 16 + g;  // rows g and g+8 of this warp
  const int qpos_b = qpos_a + 8;

  for (int t = 0; t < n_kv_tiles; ++t) {
    if (t + 1 < n_kv_tiles) load_kv(t + 1, (t + 1) & 1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    if (t == 0) {
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const int r = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = ks * 2 + (lane >> 4);
        ldsm_x4(sQ + swz(r, c), qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3]);
      }
    }
    const uint32_t sK = sK0 + (2 * (t & 1)) * TILE_BYTES;
    const uint32_t sV = sK + TILE_BYTES;
    // S = Q K^T  (16 x 64 per warp)
    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {  // pairs of n-tiles
        const int r = np * 16 + (lane & 7) + ((lane >> 4) << 3);
        const int c = ks * 2 + ((lane >> 3) & 1);
        uint32_t b0, b1, b2, b3;
        ldsm_x4(sK + swz(r, c), b0, b1, b2, b3);
        mma16816(s[2 * np], qf[ks], b0, b1);
        mma16816(s[2 * np + 1], qf[ks], b2, b3);
      }
    }
    // scale + causal mask (only tiles that reach past the tile's first query need it)
    const int kv0 = t * BN;
    const bool need_mask = kv0 + BN - 1 > it.q_pos0 + warp * 16;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float v = s[i][j] * p.scale_log2;
        if (need_mask) {
          const int kp = kv0 + i * 8 + tq * 2 + (j & 1);
          const int qp = (j < 2) ? qpos_a : qpos_b;
          if (kp > qp) v = -INFINITY;
        }
        s[i][j] = v;
      }
    }
    // online softmax (base 2)
    float mx[2] = {mrow[0], mrow[1]};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      mx[0] = fmaxf(mx[0], fmaxf(s[i][0], s[i][1]));
      mx[1] = fmaxf(mx[1], fmaxf(s[i][2], s[i][3]));
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
    }
    float alpha[2], msub[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      msub[r] = (mx[r] == -INFINITY) ? 0.f : mx[r];
      alpha[r] = exp2f(mrow[r] - msub[r]);
      mrow[r] = mx[r];
    }
    float rs[2] = {0.f, 0.f};
    uint32_t pf[4][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float p0 = exp2f(s[i][0] - msub[0]);
      const float p1 = exp2f(s[i][1] - msub[0]);
      const float p2 = exp2f(s[i][2] - msub[1]);
      const float p3 = exp2f(s[i][3] - msub[1]);
      rs[0] += p0 + p1;
      rs[1] += p2 + p3;
      pf[i >> 1][(i & 1) * 2 + 0] = pack_bf16x2(p0, p1);
      pf[i >> 1][(i & 1) * 2 + 1] = pack_bf16x2(p2, p3);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) lrow[r] = lrow[r] * alpha[r] + rs[r];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      o[i][0] *= alpha[0];
      o[i][1] *= alpha[0];
      o[i][2] *= alpha[1];
      o[i][3] *= alpha[1];
    }
    // O += P V : A fragments from P, B fragments from V via ldmatrix.trans
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {  // 16 kv per step
      const uint32_t a[4] = {pf[ks][0], pf[ks][1], pf[ks][2], pf[ks][3]};
#pragma unroll
      for (int np = 0; np < 8; ++np) {  // pairs of hd n-tiles
        const int r = ks * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = np * 2 + (lane >> 4);
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(sV + swz(r, c), b0, b1, b2, b3);
        mma16816(o[2 * np], a, b0, b1);
        mma16816(o[2 * np + 1], a, b2, b3);
      }
    }
    __syncthreads();
  }
  // finalize: row sums across the 4 threads of a row group
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 1);
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 2);
  }
  const float inv0 = lrow[0] > 0.f ? 1.f / lrow[0] : 0.f;
  const float inv1 = lrow[1] > 0.f ? 1.f / lrow[1] : 0.f;
  const int ra = warp * 16 + g, rb = ra + 8;
  __nv_bfloat16* ob = p.out + (long long)it.q_row0 * p.ldo + head * HD;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int col = i * 8 + tq * 2;
    if (ra < it.n_rows)
      *reinterpret_cast<uint32_t*>(ob + (long long)ra * p.ldo + col) =
          pack_bf16x2(o[i][0] * inv0, o[i][1] * inv0);
    if (rb < it.n_rows)
      *reinterpret_cast<uint32_t*>(ob + (long long)rb * p.ldo + col) =
          pack_bf16x2(o[i][2] * inv1, o[i][3] * inv1);
  }
}

constexpr int kAttnMmaSmem = mmaattn::TILE_BYTES * 5;

}  // namespace fp
