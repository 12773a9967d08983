// Causal varlen flash-attention prefill on tcgen05 / TMEM / TMA (GQA, head_dim 128).
//
// Realises the reference's `attn` timeline entry (prefillsim/cost_model.py:226-233): each
// request's share of the chunk attends causally to its OWN prefix + share, never across the
// batch (pkg/tests/test_cost_model.py:88-109). All K/V -- the prefix written by earlier chunks
// and this chunk's share written moments ago by the qkv_proj epilogue -- are read from the paged
// cache, one 128-token page per KV tile, so tiles sit at ABSOLUTE request positions and a query
// row's result is independent of chunking and batch composition.
//
// Work item = one 128-row query tile x two query heads of the same KV head (GQA pair): both
// heads share every K/V tile in shared memory. The kernel is PERSISTENT: one CTA per SM takes
// work items from a global counter in longest-first order (the host sorts query tiles by KV
// length), so the causal imbalance between tiles is absorbed dynamically, and the next item's Q
// load and first S = QK^T overlap the current item's last P*V and output epilogue.
// Warp roles (320 threads, 1 CTA/SM):
//   warp 0       scheduler + TMA producer: fetches work, Q tiles, then K_j, V_j into a 3-slot
//                ring (pages via the block table; 128B-swizzled 64-column boxes)
//   warp 1       TMEM allocator + single-thread MMA issuer:
//                  S_h = Q_h K_j^T      (SS, M=128 N=128 K=128, fp32 accumulators in TMEM)
//                  O_h += P_h V_j       (TS: P read from TMEM, V MN-major from smem)
//                issued ping-pong so head 1's MMAs overlap head 0's softmax and vice versa
//   warps 2-5    softmax for head 0, warps 6-9 softmax for head 1: one query row per thread,
//                exp2 online softmax with lazy O rescale (only when the row max grows by > 2^8),
//                P written back to TMEM over S as bf16; per-head O-complete barrier, then the
//                O / l epilogue: full query tiles staged in 128B-swizzled shared memory and
//                written by TMA stores (coalesced), a request's partial last tile row by row.
// Softmax arithmetic is budgeted against the tensor pipe: the scale is folded into one packed
// FFMA2 per element pair, the row max is a tree of 8 chains, row sums use packed FADD2 after P
// is released, and 2 of every 8 exponential pairs run as a degree-3 polynomial on the FMA pipe
// (Cody-Waite split, |rel err| < 1.1e-4 -- below the bf16 rounding P gets anyway): MUFU.EX2
// issues one warp instruction per ~8 cycles per SMSP, the exp phase's floor
// (tools/attn_variants.sh: emulating 0 / 2 / 3 / 4 / 5 of 8 pairs).
// The MMA warp builds descriptors once per 8-MMA group (tools/probes/mma_rate.cu: a descriptor
// built per MMA cost more issue time than an N = 128 MMA executes).
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
  const AttnTile* items;          // query tiles, longest KV range first
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
  int* sched;                     // [2] work counter, finished CTAs (zero between launches)
  unsigned long long* dbg;        // -DFP_GEMM_STAMPS builds: clock64 phase stamps (see ATTN_STAMP)
  Guard guard;
};

// Diagnostic builds only (-DFP_GEMM_STAMPS): SM clock64 at the phases of the first work item of
// CTAs 0..15, KV tiles 0..63: [cta][tile][24] = softmax h0 sees S, h0 arrives P, h1 sees S,
// h1 arrives P, MMA issues PV0, MMA issued QK0(j+1), MMA issues PV1, MMA issued QK1(j+1), MMA
// has K(j+1), -, then per head h: S in registers (10 + 4h), row max done (11 + 4h), P
// computed (12 + 4h), row sum done (13 + 4h).
#ifdef FP_GEMM_STAMPS
#define ATTN_STAMP(it, j, k)                                                              \
  do {                                                                                    \
    if (p.dbg && (it) == 0 && blockIdx.x < 16 && (j) < 64)                                 \
      p.dbg[((int)blockIdx.x * 64 + (j)) * 24 + (k)] = (unsigned long long)clock64();       \
  } while (0)
// Per work item (items 0..31 of CTAs 0..15) at [24576 + (cta * 32 + item) * 8 + k]: MMA warp
// got the item (0), issued its first Q*K^T (1); head-0 softmax row 0: first S seen (2), last P
// out (3), O complete seen (4), epilogue done (5); kernel-relative start of the CTA (6, item 0).
#define ATTN_ISTAMP(it, k)                                                                \
  do {                                                                                    \
    if (p.dbg && (it) < 32 && blockIdx.x < 16)                                             \
      p.dbg[24576 + ((int)blockIdx.x * 32 + (it)) * 8 + (k)] = (unsigned long long)clock64(); \
  } while (0)
#else
#define ATTN_STAMP(it, j, k) \
  do {                       \
  } while (0)
#define ATTN_ISTAMP(it, k) \
  do {                     \
  } while (0)
#endif

namespace tcattn {
constexpr int THREADS = 320;
constexpr int TILE = 128;
constexpr int TILE_BYTES = 128 * 128 * 2;  // 32 KB: two 64-column swizzle atoms of 16 KB
constexpr int ATOM_BYTES = 16384;
#ifndef FP_ATTN_EMU
#define FP_ATTN_EMU 2  // exponential pairs (of every 8) computed by the FMA-pipe polynomial
#endif
#ifndef FP_ATTN_STAGES
#define FP_ATTN_STAGES 3
#endif
constexpr int STAGES = FP_ATTN_STAGES;
// Q tiles (2 heads), the K/V ring, barriers, and one 32 KB output staging tile per head (the
// epilogue writes O there in the 128B-swizzled layout and TMA stores it: coalesced)
constexpr int SMEM_BYTES = 1024 + 2 * TILE_BYTES + STAGES * TILE_BYTES + 512 + 2 * TILE_BYTES;
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units: rescale O only if max grows > 256x
constexpr int SOFTMAX_WARPS = 8;
}  // namespace tcattn

// ---- packed fp32 pairs (sm_100 FFMA2 / FADD2) -----------------------------------------------
DEVI float2 ffma2(float2 a, float2 b, float2 c) {
  float2 r;
  asm("{.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}
DEVI float2 fadd2(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
// 2^x for x <= 0 (or -inf) on the FMA pipe: x = j + f, j = rint(x), f in [-1/2, 1/2];
// 2^f ~ 1 + f (c1 + f (c2 + f c3)); 2^j by adding j to the exponent field.
DEVI float2 exp2_poly2(float2 x) {
  constexpr float kMagic = 12582912.f;  // 1.5 * 2^23: x + magic rounds x to an integer
  x.x = fmaxf(x.x, -127.f);
  x.y = fmaxf(x.y, -127.f);
  const float2 t = fadd2(x, make_float2(kMagic, kMagic));
  const float2 j = fadd2(t, make_float2(-kMagic, -kMagic));
  const float2 f = fadd2(x, make_float2(-j.x, -j.y));
  float2 p = ffma2(f, make_float2(0.05500892549753189f, 0.05500892549753189f),
                   make_float2(0.2422109991312027f, 0.2422109991312027f));
  p = ffma2(p, f, make_float2(0.693282961845398f, 0.693282961845398f));
  p = ffma2(p, f, make_float2(1.f, 1.f));
  // low bits of t hold j (two's complement): add j << 23 to the exponent
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

DEVI void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}

// decoded work item
struct AttnWork {
  AttnTile it;
  int head0, head1;
  bool has_head1;
  int kvh;
  int n_tiles;
};

DEVI AttnWork attn_decode(const AttnTcParams& p, int w) {
  const int hp = p.n_kv_heads * p.pairs_per_kv;
  AttnWork a;
  a.it = p.items[w / hp];
  const int y = w % hp;
  a.kvh = y / p.pairs_per_kv;
  const int pair = y % p.pairs_per_kv;
  const int group = p.n_heads / p.n_kv_heads;
  a.head0 = a.kvh * group + 2 * pair;
  a.has_head1 = 2 * pair + 1 < group;
  a.head1 = a.has_head1 ? a.head0 + 1 : a.head0;
  a.n_tiles = (a.it.q_pos0 + a.it.n_rows + tcattn::TILE - 1) / tcattn::TILE;
  return a;
}

// Registers: 10 warps put 3 warps on two of the four SM sub-partitions, whose 16K-register banks
// cap a thread at 168 registers; ptxas stops there and spills 28 B (one loop-carried scalar per
// KV tile, L1-resident). A __maxnreg__(200) build is spill-free at 193 registers but fails to
// launch on the B200 ("too many resources requested", although 200 x 320 < 64K: the per-sub-
// partition bank limit, 3 warps x 32 x regs <= 16384, is what binds).
__global__ void __launch_bounds__(tcattn::THREADS, 1)
    attn_prefill_tc_kernel(const __grid_constant__ CUtensorMap tmQ,
                           const __grid_constant__ CUtensorMap tmKV,
                           const __grid_constant__ CUtensorMap tmO, const AttnTcParams p) {
  using namespace tcattn;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
  uint8_t* sQ = smem;                      // [2][TILE_BYTES]
  uint8_t* sKV = smem + 2 * TILE_BYTES;    // [STAGES][TILE_BYTES]
  // [2 heads][TILE_BYTES] output staging: 1024-byte aligned (the 128B-swizzle atom the TMA reads)
  uint8_t* sOut = sKV + STAGES * TILE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sOut + 2 * TILE_BYTES);
  uint64_t* q_full = bars;
  uint64_t* q_empty = bars + 1;
  uint64_t* kv_full = bars + 2;
  uint64_t* kv_empty = kv_full + STAGES;
  uint64_t* s_full = kv_empty + STAGES;  // [2]
  uint64_t* p_full = s_full + 2;         // [2]
  uint64_t* o_full = p_full + 2;         // [2] per head: the item's last P*V done
  uint64_t* o_empty = o_full + 2;        // [2]
  uint64_t* w_full = o_empty + 2;        // [2] work ring
  uint64_t* w_empty = w_full + 2;        // [2]
  int* w_ring = reinterpret_cast<int*>(w_empty + 2);  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(w_ring + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  // prologue (overlaps the previous kernel's tail under programmatic dependent launch)
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmKV);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int h = 0; h < 2; ++h) {
      mbar_init(&s_full[h], 1);
      mbar_init(&p_full[h], 128);
      mbar_init(&o_empty[h], 128);
      mbar_init(&o_full[h], 1);
      mbar_init(&w_full[h], 1);
      mbar_init(&w_empty[h], 1 + SOFTMAX_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  grid_dep_wait();
  if (threadIdx.x == 0) ATTN_ISTAMP(0, 6);
  const bool run = guard_block(p.guard);
  const int n_work = p.n_items * p.n_kv_heads * p.pairs_per_kv;

  if (!run) {
    // stopped at this boundary: nothing to do
  } else if (warp == 0) {
    // ------------------------------------------------------------ scheduler + TMA producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_last();  // K/V tiles are re-read by other q tiles
      int s = 0, ws = 0, it = 0;
      uint32_t ph = 0, wph = 0;
      for (;;) {
        // first item static (CTA b takes item b); later ones from the global counter, which
        // launches with no more items than CTAs never touch
        int w = it == 0 ? (int)blockIdx.x
                        : (n_work > (int)gridDim.x ? (int)gridDim.x + atomicAdd(&p.sched[0], 1)
                                                   : n_work);
        if (w >= n_work) w = -1;
        mbar_wait(&w_empty[ws], wph ^ 1);
        w_ring[ws] = w;
        mbar_arrive(&w_full[ws]);
        if (++ws == 2) {
          ws = 0;
          wph ^= 1;
        }
        if (w < 0) {
          grid_dep_launch();  // no more work for this CTA: the next kernel may start its prologue
          break;
        }
        const AttnWork a = attn_decode(p, w);
        const int* bt = p.block_table + (long long)a.it.req * p.bt_stride;
        mbar_wait(q_empty, (it & 1) ^ 1);  // the previous item's last QK^T has run
        mbar_arrive_expect_tx(q_full, 2 * TILE_BYTES);
        for (int h = 0; h < 2; ++h) {
          const int col = (h ? a.head1 : a.head0) * 128;
          tma_load_2d(sQ + h * TILE_BYTES, &tmQ, q_full, col, a.it.q_row0);
          tma_load_2d(sQ + h * TILE_BYTES + ATOM_BYTES, &tmQ, q_full, col + 64, a.it.q_row0);
        }
        for (int j = 0; j < a.n_tiles; ++j) {
          const long long page = bt[j];  // page_size == TILE
          for (int kv = 0; kv < 2; ++kv) {
            mbar_wait(&kv_empty[s], ph ^ 1);
            mbar_arrive_expect_tx(&kv_full[s], TILE_BYTES);
            const long long row = p.kv_row_layer + page * p.kv_rows_per_page +
                                  (long long)(kv * p.n_kv_heads + a.kvh) * TILE;
            tma_load_2d_hint(sKV + s * TILE_BYTES, &tmKV, &kv_full[s], 0, (int)row, pol);
            tma_load_2d_hint(sKV + s * TILE_BYTES + ATOM_BYTES, &tmKV, &kv_full[s], 64, (int)row,
                             pol);
            if (++s == STAGES) {
              s = 0;
              ph ^= 1;
            }
          }
        }
        ++it;
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_qk = make_idesc_bf16(128, 128, false);
    constexpr uint32_t idesc_pv = make_idesc_bf16(128, 128, true);  // V is MN-major
    const uint32_t tS[2] = {tbase, tbase + 128};
    const uint32_t tO[2] = {tbase + 256, tbase + 384};
    uint32_t seq = 0;  // ring sequence number of the next K/V tile to consume
    auto slot_of = [&](uint32_t sq) { return (int)(sq % STAGES); };
    auto wait_tile = [&](uint32_t sq) { mbar_wait(&kv_full[slot_of(sq)], (sq / STAGES) & 1); };
    // Descriptors are built once (Q) or once per group of 8 MMAs (K / V slot) and advanced by
    // constant offsets: building one per MMA costs more issue time than an N = 128 MMA takes
    // to execute (tools/probes/mma_rate.cu: 66 vs ~170 cycles per MMA).
    const uint64_t qdesc[2] = {make_sdesc_sw128(smem_u32(sQ), 16, 1024),
                               make_sdesc_sw128(smem_u32(sQ + TILE_BYTES), 16, 1024)};
    auto issue_qk = [&](int h, uint32_t ksq) {
      const uint64_t kd = make_sdesc_sw128(smem_u32(sKV + slot_of(ksq) * TILE_BYTES), 16, 1024);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {  // head_dim 128 = 8 x K16; two 64-wide swizzle atoms
        const uint64_t off = (uint64_t)(((kk >> 2) * ATOM_BYTES + (kk & 3) * 32) >> 4);
        umma_bf16_ss(tS[h], qdesc[h] + off, kd + off, idesc_qk, kk > 0);
      }
    };
    auto issue_pv = [&](int h, uint32_t vsq, bool acc) {
      const uint64_t vd =
          make_sdesc_sw128(smem_u32(sKV + slot_of(vsq) * TILE_BYTES), ATOM_BYTES, 1024);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {  // 128 kv rows = 8 x K16; P: 8 TMEM columns per step
        umma_bf16_ts(tO[h], tS[h] + kk * 8, vd + (uint64_t)((kk * 2048) >> 4), idesc_pv,
                     (acc || kk > 0) ? 1u : 0u);
      }
    };
    int ws = 0, it = 0;
    uint32_t wph = 0, tc = 0;  // tc: tiles consumed before this item (s_full / p_full phases)
    for (;;) {
      mbar_wait(&w_full[ws], wph);
      const int w = w_ring[ws];
      __syncwarp();
      if (lane == 0) mbar_arrive(&w_empty[ws]);
      if (++ws == 2) {
        ws = 0;
        wph ^= 1;
      }
      if (w < 0) break;
      const int n_tiles = attn_decode(p, w).n_tiles;
      if (lane == 0) ATTN_ISTAMP(it, 0);
      mbar_wait(q_full, it & 1);
      wait_tile(seq);
      tc_fence_after();
      if (lane == 0) ATTN_ISTAMP(it, 1);
      if (lane == 0) {
        issue_qk(0, seq);
        tc_commit(&s_full[0]);
        issue_qk(1, seq);
        tc_commit(&s_full[1]);
        tc_commit(&kv_empty[slot_of(seq)]);
        if (n_tiles == 1) tc_commit(q_empty);
      }
      __syncwarp();
      ++seq;
      for (int j = 0; j < n_tiles; ++j) {
        const bool last = j == n_tiles - 1;
        const uint32_t vsq = seq;      // V_j
        const uint32_t ksq = seq + 1;  // K_{j+1}
        const uint32_t tph = (tc + j) & 1;
        wait_tile(vsq);
        if (j == 0) mbar_wait(&o_empty[0], (it & 1) ^ 1);  // previous item's O0 drained
        mbar_wait(&p_full[0], tph);
        tc_fence_after();
        if (lane == 0) ATTN_STAMP(it, j, 4);
        if (lane == 0) {
          issue_pv(0, vsq, j > 0);
          if (last) tc_commit(&o_full[0]);  // head 0's epilogue need not wait for head 1
        }
        __syncwarp();
        if (!last) {
          wait_tile(ksq);
          tc_fence_after();
          if (lane == 0) ATTN_STAMP(it, j, 8);
          if (lane == 0) {
            issue_qk(0, ksq);
            tc_commit(&s_full[0]);
            ATTN_STAMP(it, j, 5);
          }
          __syncwarp();
        }
        if (j == 0) mbar_wait(&o_empty[1], (it & 1) ^ 1);
        mbar_wait(&p_full[1], tph);
        tc_fence_after();
        if (lane == 0) ATTN_STAMP(it, j, 6);
        if (lane == 0) {
          issue_pv(1, vsq, j > 0);
          if (last) tc_commit(&o_full[1]);
          tc_commit(&kv_empty[slot_of(vsq)]);
          if (!last) {
            issue_qk(1, ksq);
            tc_commit(&s_full[1]);
            ATTN_STAMP(it, j, 7);
            tc_commit(&kv_empty[slot_of(ksq)]);
            if (j + 1 == n_tiles - 1) tc_commit(q_empty);  // last QK^T of the item issued
          }
        }
        __syncwarp();
        seq += last ? 1 : 2;  // the last step consumes V only; the next item's K_0 follows
      }
      tc += n_tiles;
      ++it;
    }
  } else {
    // ------------------------------------------------------------------ softmax + epilogue
    const int h = (warp - 2) >> 2;  // 0: warps 2-5, 1: warps 6-9
    const int quad = warp & 3;      // TMEM lane quadrant accessible to this warp
    const int row = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const uint32_t tS = tbase + h * 128 + lane_off;
    const uint32_t tO = tbase + 256 + h * 128 + lane_off;
    const float sc = p.scale_log2;
    int ws = 0, it = 0;
    uint32_t wph = 0, tc = 0;
    for (;;) {
      mbar_wait(&w_full[ws], wph);
      const int w = w_ring[ws];
      __syncwarp();
      if (lane == 0) mbar_arrive(&w_empty[ws]);
      if (++ws == 2) {
        ws = 0;
        wph ^= 1;
      }
      if (w < 0) break;
      const AttnWork a = attn_decode(p, w);
      const int qpos = a.it.q_pos0 + row;
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < a.n_tiles; ++j) {
        mbar_wait(&s_full[h], (tc + j) & 1);
        tc_fence_after();
        if (row == 0) ATTN_STAMP(it, j, 2 * h);
        if (row == 0 && h == 0 && j == 0) ATTN_ISTAMP(it, 2);
        uint32_t su[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(tS + c * 32, su[c]);
        tmem_ld_wait();
        float sr[128];
#pragma unroll
        for (int i = 0; i < 128; ++i) sr[i] = __uint_as_float(su[i >> 5][i & 31]);
        if (row == 0) ATTN_STAMP(it, j, 10 + 4 * h);
        const int kv0 = j * TILE;
        if (kv0 + TILE - 1 > a.it.q_pos0) {  // diagonal tile: causal mask
#pragma unroll
          for (int i = 0; i < 128; ++i)
            if (kv0 + i > qpos) sr[i] = -INFINITY;
        }
#ifndef FP_ATTN_CHAIN_MAX
        // 8 independent 3-input max chains, then a 3-level tree (latency ~ 16 dependent ops)
        float mc[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) mc[k] = fmaxf(sr[k], sr[8 + k]);
#pragma unroll
        for (int i = 16; i < 128; i += 16) {
#pragma unroll
          for (int k = 0; k < 8; ++k) mc[k] = fmaxf(mc[k], fmaxf(sr[i + k], sr[i + 8 + k]));
        }
        const float mx = fmaxf(fmaxf(fmaxf(mc[0], mc[1]), fmaxf(mc[2], mc[3])),
                               fmaxf(fmaxf(mc[4], mc[5]), fmaxf(mc[6], mc[7])));
#else
        float mx = sr[0];
#pragma unroll
        for (int i = 1; i < 128; ++i) mx = fmaxf(mx, sr[i]);
#endif
        const float m_new = fmaxf(m, mx * sc);  // scaled (log2) units
        if (row == 0) ATTN_STAMP(it, j, 11 + 4 * h);
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
        const float nm = (m == -INFINITY) ? 0.f : -m;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const float2 x = ffma2(make_float2(sr[c * 32 + i], sr[c * 32 + i + 1]),
                                   make_float2(sc, sc), make_float2(nm, nm));
            float2 e;
            if (((i & 15) >> 1) < FP_ATTN_EMU) {  // EMU of every 8 pairs on the FMA pipe
              e = exp2_poly2(x);
            } else {
              e.x = fast_exp2(x.x);
              e.y = fast_exp2(x.y);
            }
            sr[c * 32 + i] = e.x;  // kept for the row sum, taken after P is released
            sr[c * 32 + i + 1] = e.y;
            pk[i >> 1] = pack_bf16x2(e.x, e.y);
          }
          tmem_st16(tS + c * 16, pk);  // P (bf16 pairs) over the consumed S columns
        }
        if (row == 0) ATTN_STAMP(it, j, 12 + 4 * h);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&p_full[h]);
        if (row == 0) ATTN_STAMP(it, j, 2 * h + 1);
        if (row == 0 && h == 0 && j == a.n_tiles - 1) ATTN_ISTAMP(it, 3);
        // row sum off the P -> PV critical path (same pairing and order as before)
        float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < 128; i += 2) {
          const float2 e = make_float2(sr[i], sr[i + 1]);
          if (i & 2) acc1 = fadd2(acc1, e);
          else acc0 = fadd2(acc0, e);
        }
        l += (acc0.x + acc0.y) + (acc1.x + acc1.y);
        if (row == 0) ATTN_STAMP(it, j, 13 + 4 * h);
      }
      // epilogue: O / l -> bf16 -> HBM, then release O for the next item's first P*V
      mbar_wait(&o_full[h], it & 1);
      tc_fence_after();
      if (row == 0 && h == 0) ATTN_ISTAMP(it, 4);
      const float inv = l > 0.f ? 1.f / l : 0.f;
      const bool live = row < a.it.n_rows && (h == 0 || a.has_head1);
      __nv_bfloat16* dst =
          p.out + (long long)(a.it.q_row0 + row) * p.ldo + (h ? a.head1 : a.head0) * 128;
      // all of O in registers with one wait (the S registers are dead here), then release O at
      // once -- the next item's first P*V may overwrite it while these rows are stored
      uint32_t o[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tO + c * 32, o[c]);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&o_empty[h]);
      if (a.it.n_rows == TILE) {
        // full tile: rows -> the head's staging tile (two 64-column 128B-swizzled atoms, the
        // layout TMA reads), then one thread stores it with two TMA boxes. Row-per-thread
        // global stores were uncoalesced (16 B into 32 different lines per instruction): ~5200
        // cycles per item (tools/attn_stamps.py).
        uint8_t* stg = sOut + h * TILE_BYTES;
        const uint32_t bar_id = 1 + h;  // named barrier of this head's 128 softmax threads
        if (row == 0) bulk_wait_group_read0();  // the previous item's store has read the tile
        asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
        if (h == 0 || a.has_head1) {
#pragma unroll
          for (int k = 0; k < 16; ++k) {  // 16-byte chunk k of the row: atom k / 8, chunk k % 8
            const int c = k >> 2, i = k & 3;
            uint4 u;
            u.x = pack_bf16x2(__uint_as_float(o[c][8 * i + 0]) * inv, __uint_as_float(o[c][8 * i + 1]) * inv);
            u.y = pack_bf16x2(__uint_as_float(o[c][8 * i + 2]) * inv, __uint_as_float(o[c][8 * i + 3]) * inv);
            u.z = pack_bf16x2(__uint_as_float(o[c][8 * i + 4]) * inv, __uint_as_float(o[c][8 * i + 5]) * inv);
            u.w = pack_bf16x2(__uint_as_float(o[c][8 * i + 6]) * inv, __uint_as_float(o[c][8 * i + 7]) * inv);
            *reinterpret_cast<uint4*>(stg + (k >> 3) * ATOM_BYTES + row * 128 +
                                      (((k & 7) ^ (row & 7)) << 4)) = u;
          }
          fence_proxy_async();  // generic-proxy smem writes -> visible to the TMA (async proxy)
        }
        asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
        if (row == 0 && (h == 0 || a.has_head1)) {
          const int col = (h ? a.head1 : a.head0) * 128;
          tma_store_2d(&tmO, stg, col, a.it.q_row0);
          tma_store_2d(&tmO, stg + ATOM_BYTES, col + 64, a.it.q_row0);
          bulk_commit_group();
        }
      } else if (live) {
        // partial tile (a request's last rows): only the live rows -- the rows after them
        // belong to the next request
#pragma unroll
        for (int c = 0; c < 4; ++c) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            uint4 u;
            u.x = pack_bf16x2(__uint_as_float(o[c][8 * i + 0]) * inv, __uint_as_float(o[c][8 * i + 1]) * inv);
            u.y = pack_bf16x2(__uint_as_float(o[c][8 * i + 2]) * inv, __uint_as_float(o[c][8 * i + 3]) * inv);
            u.z = pack_bf16x2(__uint_as_float(o[c][8 * i + 4]) * inv, __uint_as_float(o[c][8 * i + 5]) * inv);
            u.w = pack_bf16x2(__uint_as_float(o[c][8 * i + 6]) * inv, __uint_as_float(o[c][8 * i + 7]) * inv);
            st_global_v4(dst + c * 32 + 8 * i, u);
          }
        }
      }
      if (row == 0 && h == 0) ATTN_ISTAMP(it, 5);
      tc += a.n_tiles;
      ++it;
    }
    if (row == 0) bulk_wait_group0();  // this head's TMA stores complete before the CTA exits
  }
  tc_fence_before();
  __syncthreads();
  if (run && n_work > (int)gridDim.x && threadIdx.x == 0) {  // last CTA out re-arms the counter
    __threadfence();
    if (atomicAdd(&p.sched[1], 1) == (int)gridDim.x - 1) {
      p.sched[0] = 0;
      p.sched[1] = 0;
      __threadfence();
    }
  }
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

}  // namespace fp
