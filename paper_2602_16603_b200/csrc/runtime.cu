// Native runtime of the preemptible prefill path: context (= execution pool), weights,
// paged KV pool, task plans (= timelines), guarded entry launches, launch worker, C ABI.
#include <atomic>
#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/flowprefill.h"
#include "attn_tc.cuh"
#include "common.cuh"
#include "control.cuh"
#include "gemm.cuh"
#include "moe.cuh"
#include "norm.cuh"
#include "skinny.cuh"
#include "xchg.cuh"

using namespace fp;

// --------------------------------------------------------------------------- errors
static thread_local std::string g_err;
static int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return set_err(FP_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));   \
  } while (0)
#define REQ(cond, msg)                                      \
  do {                                                      \
    if (!(cond)) return set_err(FP_ERR_ARG, (msg));         \
  } while (0)

// --------------------------------------------------------------------------- TMA maps
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                      const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                      const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion,
                                      CUtensorMapFloatOOBfill);
static PFN_encodeTiled_t get_encode() {
  static PFN_encodeTiled_t fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(p);
  }
  return fn;
}
// 2D bf16 row-major [rows, cols], box = [box_rows, 64 cols], 128B swizzle. Weight (B) maps use
// 128-row boxes: a CTA pair stages 128 rows each, a single CTA issues two boxes per stage.
static int make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols,
                    uint32_t box_rows) {
  PFN_encodeTiled_t enc = get_encode();
  if (!enc) return set_err(FP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(FP_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return FP_OK;
}

// --------------------------------------------------------------------------- random init
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__global__ void init_normal_kernel(__nv_bfloat16* w, long long n, uint64_t seed, float mean,
                                   float stdv) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const uint64_t r = splitmix64(seed ^ (uint64_t)(i * 0x2545F4914F6CDD1Dull));
    const float u1 = ((r >> 40) + 1) * (1.0f / 16777217.0f);
    const float u2 = ((r & 0xFFFFFF)) * (1.0f / 16777216.0f);
    const float z = sqrtf(-2.f * logf(u1)) * cospif(2.f * u2);
    w[i] = __float2bfloat16(mean + stdv * z);
  }
}

// RMSNorm weight folding (fused norm, see GemmParams::ssq_in): W[row, k] *= g_new[k] / g_old[k]
// over rows row0 + b * bstride + j (b < nblocks, j < rpb); g_old == null: divide by 1.
__global__ void fold_cols_kernel(__nv_bfloat16* w, long long row0, int nblocks, long long bstride,
                                 int rpb, int d, const __nv_bfloat16* g_new,
                                 const __nv_bfloat16* g_old) {
  const long long n = (long long)nblocks * rpb * d;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / d;
    const int k = (int)(i - r * d);
    const long long row = row0 + (r / rpb) * bstride + r % rpb;
    float f = __bfloat162float(g_new[k]);
    if (g_old) f /= __bfloat162float(g_old[k]);
    __nv_bfloat16* e = w + row * d + k;
    *e = __float2bfloat16(__bfloat162float(*e) * f);
  }
}

// --------------------------------------------------------------------------- structures
struct Layer {
  // wqkv / wgu hold the norm weights folded into their columns; attn_g / ffn_g are the gammas
  // currently folded in (bf16, as loaded; all ones before any load)
  __nv_bfloat16 *wqkv, *wo, *wgu, *wd, *attn_g, *ffn_g;
  float* bqkv = nullptr;                           // [qkv_n] (qkv_bias models)
  float *q_norm = nullptr, *k_norm = nullptr;      // [128]  (qk_norm models)
  CUtensorMap tm_qkv, tm_o, tm_gu, tm_d;
  // MoE: router [256 (padded experts), d] and expert weights, post-attention norm folded into
  // the router and gate/up columns; gate/up interleaved in 128-row blocks per expert
  __nv_bfloat16 *wr = nullptr, *egu = nullptr, *ed = nullptr;
  CUtensorMap tm_r, tm_egu, tm_ed;
};

struct ChunkPlan {
  int M;          // new tokens in the chunk (cost_model.py:225 new_total)
  int tok0;       // first token of the chunk in the task's concatenated stream
  int item0, n_items;
  int last0, n_last, seq0;  // requests completing in this chunk: rows at last_rows[last0..]
  double attn_flops;        // causal QK^T + PV FLOPs of the chunk (per layer)
};

struct Task {
  int id = 0;
  int n_seqs = 0, total = 0, L = 0, n_entries = 0, max_m = 0, granularity = 0;
  std::vector<int> lens;
  std::vector<ChunkPlan> chunks;
  std::vector<int> pages;  // KV pages owned
  int bt_stride = 0;
  long long upload_bytes = 0;
  // device
  char* meta = nullptr;  // one allocation: ids | pos | tok_page | items | bt | last_rows
  int *d_ids, *d_pos, *d_tpage, *d_bt, *d_last;
  AttnTile* d_items;
  __nv_bfloat16 *h, *q, *ao, *act, *xf;
  float* ssq;  // [max_m, hidden/128] segment sums of squares of h (fused RMSNorm input)
  float* logits;
  TaskCtl* ctl;
  unsigned long long* stamps = nullptr;  // inside the ctl allocation
  CUtensorMap tm_h, tm_ao, tm_act, tm_xf, tm_q;
  CUtensorMap tm_h32, tm_ao32, tm_act32, tm_xf32;  // 32-row boxes: swap-AB skinny GEMM tokens
  // MoE routing state of the current chunk (gate -> experts) and expert-ordered buffers
  float* rlog = nullptr;                       // [max_m, 256] router logits
  char* moe_meta = nullptr;                    // one allocation for the index arrays below
  int *m_ids, *m_slot, *m_counts, *m_cursor, *m_off, *m_mtc, *m_perm;
  float* m_w;
  int2* m_mtiles;
  __nv_bfloat16 *xperm = nullptr, *actp = nullptr, *yperm = nullptr;
  CUtensorMap tm_xperm, tm_actp;
  int moe_rows = 0;                            // rows of the current chunk's routing
  cudaEvent_t ready, done, fence;  // fence: after the last launch that touches the task
  // host execution state
  int gen = 0, seg_first = 0, enq = 0, seg_ack0 = 0, done_recorded = 0;
  std::atomic<int> worker_active{0};
  // sticky launch failure of the async worker (fp_task_poll reports it; the task is dead)
  std::atomic<int> err{0};
  std::string err_msg;
};

struct fp_ctx {
  int device = 0, num_sms = 148;
  fp_model_cfg cfg{};
  // this rank's shard (tp_size == 1: the whole model). qkv_n is padded to the 256-wide GEMM
  // tile; the padding rows of Wqkv are zero and the QKV epilogue skips them.
  int hq = 0, hkv = 0, ffn = 0;
  int qdim = 0, kvdim = 0, qkv_n = 0, vocab_pad = 0;
  int tp_rank = 0, tp_size = 1;
  cudaStream_t stream = nullptr, upload = nullptr, readback = nullptr;
  cudaStream_t release = nullptr;  // task frees, each behind its own task's last launch only
  cudaStream_t own_stream = nullptr;  // lock-step TP groups share rank 0's stream
  // tensor parallel exchange (null when tp_size == 1)
  TpDev tp_host{};
  TpDev* d_tp = nullptr;      // device copy of tp_host
  TpLocal* tp_local = nullptr;
  char* tp_block = nullptr;   // own IPC-shareable block: TpShared | part[0] | part[1]
  std::vector<void*> tp_opened;  // peer blocks opened through IPC
  bool tp_connected = false;
  bool tp_lockstep = false;
  bool tp_fused = true;  // FP_TP_FUSED=0: GEMM + tp_allreduce_kernel even with one process per GPU
  std::vector<Layer> layers;
  __nv_bfloat16 *embed = nullptr, *final_g = nullptr, *lm_head = nullptr;
  CUtensorMap tm_lm;
  CUtensorMap tm_kv;  // paged KV pool as [L*P*2*Hkv*PS, 128] rows
  float2* rope = nullptr;
  __nv_bfloat16* kv = nullptr;
  long long page_elems = 0;  // elements of one page in one layer (2*Hkv*PS*hd)
  int page_size = 128;
  long long kv_pages = 0;
  std::vector<int> free_pages;
  std::mutex page_mu;
  HostCtl* hctl = nullptr;   // host view
  HostCtl* dctl = nullptr;   // device alias
  std::mutex launch_mu;
  // worker
  std::thread worker;
  std::mutex wmu;
  std::condition_variable wcv;
  Task* wtask = nullptr;
  bool wquit = false;
  int window = 8;
  // pinned staging arena for task uploads
  std::mutex stage_mu;
  char* stage = nullptr;
  size_t stage_cap = 0;
  cudaEvent_t stage_ev = nullptr;
  // live per-kernel profiling (CUDA events on the prefill stream) and launch counting
  bool prof_on = false;
  std::vector<fp_prof_rec> prof_meta;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_ev;
  std::vector<cudaEvent_t> ev_pool;
  std::atomic<long long> launches{0};
  // split-K workspace (one prefill stream: launches are serialised, one buffer suffices)
  float* ws = nullptr;
  long long ws_floats = 0;  // capacity of ws
  int* tickets = nullptr;
  int* attn_sched = nullptr;  // persistent attention work counter (self-resetting)
  unsigned long long* gemm_dbg = nullptr;  // FP_GEMM_STAMPS=1: phase stamps of fp_op_gemm launches
  bool use_pair_gemm = true;
  bool use_narrow = true;  // FP_NARROW=0: never 128 x 128 tiles (experiments)
  int force_splits = 0;   // FP_FORCE_SPLITS (experiments)
  int force_pair = -1;    // FP_FORCE_PAIR (experiments): 0 single, 1 pair, 2 narrow, 3 stream-K
  // Stream-K where plan_streamk allows it (under-filled long-K launches) and its cost model
  // wins; FP_STREAMK=0 disables. Everywhere else it measured neutral or worse on the
  // power-capped B200 (the idle SMs of a partial wave cost little energy; the partial round
  // trips add traffic). Policy 3 forces it in the parity tests.
  bool use_streamk = true;
  // Batch-invariant numerics (FP_BATCH_INVARIANT=1 / fp_ctx_set_batch_invariant): no split-K
  // and no stream-K, so every output element is ONE in-order TMEM accumulation over K whatever
  // the launch's M -- a request's logits and KV are then bit-identical alone or in any batch
  // (SURVEY.md §7 hard part 7). Costs the short-request speed-up of split-K.
  bool batch_invariant = false;
  int* sk_flags = nullptr;  // stream-K partial flags [num_sms]
  // Swap-AB skinny GEMM (skinny.cuh) for launches of at most skinny_max_m tokens
  // (FP_SKINNY_MAX_M / fp_ctx_set_skinny_max; 0 disables)
  int skinny_max_m = 128;
  // Cluster split-K (gemm.cuh MODE 4): launches whose tiles are all split reduce inside a
  // cluster through distributed shared memory (FP_SPLIT_DSMEM=0 disables). max_clusters[S] =
  // co-resident clusters of S CTAs of the split kernel (occupancy query, cached; -1 unknown).
  bool split_dsmem = true;
  int max_clusters[9] = {-1, -1, -1, -1, -1, -1, -1, -1, -1};
  int sk_epoch = 0;         // per stream-K launch (flags compare against it: no reset)
};

static cudaEvent_t ev_get(fp_ctx* c) {
  if (c->ev_pool.empty()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  cudaEvent_t e = c->ev_pool.back();
  c->ev_pool.pop_back();
  return e;
}
struct ProfScope {
  fp_ctx* c;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  fp_prof_rec rec{};
  ProfScope(fp_ctx* c_, cudaStream_t st_, int kind, int layer, int M, double flops, double bytes)
      : c(c_), st(st_) {
    rec.kind = kind;
    rec.layer = layer;
    rec.M = M;
    rec.flops = flops;
    rec.bytes = bytes;
    if (c->prof_on) {
      a = ev_get(c);
      cudaEventRecord(a, st);
    }
  }
  ~ProfScope() {
    c->launches++;
    if (c->prof_on) {
      cudaEvent_t b = ev_get(c);
      cudaEventRecord(b, st);
      c->prof_meta.push_back(rec);
      c->prof_ev.push_back({a, b});
    }
  }
};

// --------------------------------------------------------------------------- launches
// Kernel attributes (max dynamic shared memory) are per device: a process with contexts on
// several GPUs sets them per (kernel, device). The bit is published only after the attribute
// is set (concurrent first launches both set it, which is harmless).
template <typename F>
static void once_per_device(std::atomic<unsigned long long>& mask, int dev, F&& set) {
  const unsigned long long bit = 1ull << (dev & 63);
  if (mask.load(std::memory_order_acquire) & bit) return;
  set();
  mask.fetch_or(bit, std::memory_order_acq_rel);
}
// Every kernel is launched with programmatic stream serialisation: its prologue (barrier init,
// TMEM alloc, descriptor prefetch) may start while the previous kernel drains; the kernel
// itself waits (griddepcontrol.wait) before its boundary check and any data access.
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Tail split-K plan for a GEMM of `tiles` output tiles and `num_k` 64-wide k-blocks: whole
// waves run unsplit; the remainder tiles (the partial last wave, or all tiles of a small
// prefill chunk) are cut into S K-slices. Cost model in k-block units: waves * (k-blocks per
// slice + fixed) + partial write/reduce traffic per split. Shape-only, so deterministic.
// Split-K of the persistent kernel: the partial last wave (rem tiles; all tiles for short
// requests) is cut into S K-slices, one unit per CTA (pair) of a single extra round, so the S
// K-slice CTAs of a tile are co-resident and reduce it together (gemm.cuh split path). Cost in
// k-block units (one 128 x 256 x 64 MMA step, ~0.34 us): a unit costs its K-slice plus ~4
// k-blocks of pipeline fill; a split adds kSplitOverheadKb for the partial round trip through
// L2, the inter-CTA barrier and the reduction (~8 us measured on B200, tools/split_sweep.py and
// tools/gemm_stamps.py). A split must win by > 15%. tail_ok = false restricts splitting to
// launches whose tiles all split (no full wave in front).
static constexpr double kSplitOverheadKb = 44.0;
static constexpr double kSplitOverheadKbQkv = 60.0;  // RoPE / KV-scatter items cost more
// Tails behind full waves split only for long K (down_proj): the split-capable instantiation
// runs the full-wave tiles with more register pressure (measured slower for QKV / SwiGLU).
static int g_split_tail = 0;  // FP_SPLIT_TAIL=1 (experiments): tail split for every epilogue / K
static bool split_tail_ok(int epi, int K) {
  if (g_split_tail) return epi != EPI_STORE_F32;
  return epi != EPI_QKV && epi != EPI_SWIGLU && epi != EPI_STORE_F32 && K / kGemmBK >= 128;
}
static double g_split_ov_scale = 1.0;  // FP_SPLIT_OV_SCALE (experiments)
static double split_overhead(int epi) {
  return g_split_ov_scale * (epi == EPI_QKV ? kSplitOverheadKbQkv : kSplitOverheadKb);
}
static double choose_splits(int tiles, int num_k, int num_sms, int* full_tiles, int* splits,
                            bool tail_ok = true, double overhead = kSplitOverheadKb) {
  const int rem = tiles % num_sms;
  const double full_cost = (double)(tiles / num_sms) * (num_k + 4.0);
  *full_tiles = tiles;
  *splits = 1;
  const double unsplit = rem ? num_k + 4.0 : 0.0;
  double best_t = unsplit;
  if (rem && (tail_ok || tiles < num_sms)) {
    for (int S = 2; S <= 32 && rem * S <= num_sms && num_k / S >= 4; ++S) {
      const double t = std::ceil((double)num_k / S) + 4.0 + overhead;
      if (t < best_t - 1e-9 && t < 0.85 * unsplit) {
        best_t = t;
        *splits = S;
        *full_tiles = tiles - rem;
      }
    }
  }
  return full_cost + best_t;
}

// Raster group: one group over all m-blocks when the whole A operand fits comfortably in L2
// (then each weight tile is streamed from HBM once instead of once per 16-m-block group; ncu:
// gate_up at M = 4465 read 573 MB for 271 MB of operands), else kGemmGroupM.
static int g_raster_all_mb = 48;  // FP_RASTER_ALL_MB (0 = always kGemmGroupM)
static int raster_group(const fp_ctx*, const GemmParams& p) {
  return (long long)p.M * p.K * 2 <= ((long long)g_raster_all_mb << 20) ? (1 << 20) : 0;
}

template <int EPI, int CG, int BN = 256>
static void launch_gemm_cg(fp_ctx* c, const CUtensorMap& a, const CUtensorMap& b, GemmParams p,
                           cudaStream_t st) {
  using Cfg = GemmCfg<BN, CG>;
  static std::atomic<unsigned long long> attr{0};  // per device (the attribute is per device)
  once_per_device(attr, c->device, [] {
    cudaFuncSetAttribute(gemm_bf16_tn_kernel<BN, EPI, CG, 0>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
    if constexpr (BN == 256) {
      cudaFuncSetAttribute(gemm_bf16_tn_kernel<BN, EPI, CG, 1>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
      if constexpr (CG == 1)
        cudaFuncSetAttribute(gemm_bf16_tn_kernel<BN, EPI, CG, 4>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
    }
  });
  const int tiles = ((p.M + Cfg::TILE_M - 1) / Cfg::TILE_M) * (p.N / BN);
  const int slots = c->num_sms / CG;  // concurrent tiles (CTA pairs)
  p.group_m = raster_group(c, p);
  p.splits = 1;
  p.full_tiles = tiles;
  // fp32 stores (lm_head, MoE router) split only when all their tiles do (no full wave)
  if (c->ws && BN == 256)
    choose_splits(tiles, p.K / kGemmBK, slots, &p.full_tiles, &p.splits, split_tail_ok(EPI, p.K),
                  split_overhead(EPI));
  if (p.xchg) {  // TP exchange GEMMs publish / fold their partials per tile: never split
    p.splits = 1;
    p.full_tiles = tiles;
  }
  if (c->batch_invariant) {
    p.splits = 1;
    p.full_tiles = tiles;
  }
  if (c->force_splits > 0 && !p.xchg && BN == 256) {  // experiments only (FP_FORCE_SPLITS)
    const int rem = tiles % slots;
    p.splits = rem ? c->force_splits : 1;
    p.full_tiles = tiles - rem;
  }
  // K-slices must be non-empty; the split units must fit one round (one per CTA: the K-slice
  // CTAs of a tile wait for each other) and the workspace / ticket slots
  const int num_k = p.K / kGemmBK;
  while (p.splits > 1 && ((p.splits - 1) * ((num_k + p.splits - 1) / p.splits) >= num_k ||
                          (tiles - p.full_tiles) * p.splits > slots ||
                          (long long)(tiles - p.full_tiles) * CG * p.splits > 8LL * c->num_sms))
    --p.splits;
  if (p.splits == 1) p.full_tiles = tiles;
  p.ws = c->ws;
  p.tickets = c->tickets;
  const int units = p.full_tiles + (tiles - p.full_tiles) * p.splits;
  const int grid = std::max(1, std::min(units, slots)) * CG;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  attrs[1].id = cudaLaunchAttributeClusterDimension;
  attrs[1].val.clusterDim.x = CG;
  attrs[1].val.clusterDim.y = 1;
  attrs[1].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  if constexpr (BN == 256) {
    if (p.splits > 1) {
      // every tile split (short launches): the K-slices of a tile as one cluster, reduced in
      // distributed shared memory -- when all the clusters are co-resident (one round)
      if constexpr (CG == 1) {
        if (c->split_dsmem && p.full_tiles == 0 && p.splits <= 8 && grid == units) {
          int& mc = c->max_clusters[p.splits];
          if (mc < 0) {
            cudaLaunchConfig_t q = cfg;
            cudaLaunchAttribute qa[1];
            qa[0].id = cudaLaunchAttributeClusterDimension;
            qa[0].val.clusterDim.x = p.splits;
            qa[0].val.clusterDim.y = 1;
            qa[0].val.clusterDim.z = 1;
            q.attrs = qa;
            q.numAttrs = 1;
            q.gridDim = dim3(p.splits);
            int n = 0;
            if (cudaOccupancyMaxActiveClusters(&n, gemm_bf16_tn_kernel<BN, EPI, CG, 4>, &q) !=
                cudaSuccess) {
              cudaGetLastError();
              n = 0;
            }
            mc = n;
            if (getenv("FP_DEBUG_PLAN"))
              fprintf(stderr, "[fp] cluster split: %d co-resident clusters of %d CTAs\n", n,
                      p.splits);
          }
          if (units / p.splits <= mc) {
            attrs[1].val.clusterDim.x = p.splits;
            cudaLaunchKernelEx(&cfg, gemm_bf16_tn_kernel<BN, EPI, CG, 4>, a, b, p);
            return;
          }
        }
      }
      cudaLaunchKernelEx(&cfg, gemm_bf16_tn_kernel<BN, EPI, CG, 1>, a, b, p);
      return;
    }
  }
  cudaLaunchKernelEx(&cfg, gemm_bf16_tn_kernel<BN, EPI, CG, 0>, a, b, p);
}

// Grouped (MoE expert) GEMM: persistent over the device-side m-tile table (gemm.cuh MODE 2).
template <int EPI>
static void launch_gemm_grouped(fp_ctx* c, const CUtensorMap& a, const CUtensorMap& b,
                                GemmParams p, cudaStream_t st) {
  using Cfg = GemmCfg<256, 1>;
  auto kern = gemm_bf16_tn_kernel<256, EPI, 1, 2>;
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, c->device, [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  });
  p.splits = 1;
  p.full_tiles = 0;
  launch_pdl(kern, dim3(c->num_sms), dim3(kGemmThreads), Cfg::SMEM_BYTES, st, a, b, p);
}

// Pair (2-CTA, 256-row) tiles or single-CTA (128-row) tiles, whichever the cost model
// predicts faster for this shape: pair tiles run the mainloop ~9% faster per SM (measured on
// B200: less shared-memory traffic per k-block) but pad M to 256 rows and halve the number
// of concurrent tiles. Shape-only decision.
static bool pick_pair(const fp_ctx* c, int epi, int M, int N, int K) {
  if (c->force_pair >= 0) return c->force_pair == 1 && M > kGemmBM;
  if (!c->use_pair_gemm || M <= kGemmBM) return false;
  int ft, sp;
  const int nN = N / 256, num_k = K / kGemmBK;
  const bool tail = split_tail_ok(epi, K);
  const double ov = split_overhead(epi);
  const double t1 = choose_splits(((M + 127) / 128) * nN, num_k, c->num_sms, &ft, &sp, tail, ov);
  const double t2 =
      choose_splits(((M + 255) / 256) * nN, num_k, c->num_sms / 2, &ft, &sp, tail, ov) / 1.09;
  return t2 < t1;
}

// Narrow tiles (128 x 128, one CTA, unsplit) for under-filled residual / QKV GEMMs: twice the
// tiles of the 256-wide kernel at the same M, so mid-size requests fill the machine without
// split-K. Cost in k-block units of a 128 x 256 tile: kNarrowKbCost per k-block (a narrow
// k-block is half the MMA work but moves 2/3 of the shared-memory bytes) + 4 of pipeline fill;
// chosen when it beats the best 256-wide plan by 10%.
static constexpr double kNarrowKbCost = 0.8;
static bool pick_narrow(const fp_ctx* c, int epi, int M, int N, int K) {
  if ((epi != EPI_RESID && epi != EPI_QKV) || !c->use_narrow) return false;
  if (c->force_pair == 2) return true;
  if (c->force_pair >= 0 || c->force_splits > 0) return false;
  const int num_k = K / kGemmBK, nN = N / 256;
  int ft, sp;
  const bool tail = split_tail_ok(epi, K);
  const double ov = split_overhead(epi);
  double t256 = choose_splits(((M + 127) / 128) * nN, num_k, c->num_sms, &ft, &sp, tail, ov);
  if (c->use_pair_gemm && M > kGemmBM)
    t256 = std::min(t256, choose_splits(((M + 255) / 256) * nN, num_k, c->num_sms / 2, &ft, &sp,
                                        tail, ov) / 1.09);
  const long long tiles = (long long)((M + 127) / 128) * (N / 128);
  const double waves = std::ceil((double)tiles / c->num_sms);
  const double t128 = waves * (kNarrowKbCost * num_k + 4.0);
  return t128 * 1.1 < t256;
}

// Stream-K (gemm.cuh MODE 3, 128 x 256 single-CTA tiles): whole tiles for all but the last
// one-to-two waves, then the remaining (tile, k-block) space cut into one equal contiguous range
// per CTA -- no wave quantisation, no idle SMs for under-filled launches. Cost in k-block units:
// the range, pipeline fill, the partial store / flag (kSkFixKb) and, per partner partial a
// finishing tile folds in, one 128 KB bulk read (kSkPartnerKb).
static constexpr double kSkFixKb = 6.0;
// One partner partial = 8 serial 16 KB bulk round trips through the 2 shared-memory buffers
// (~1 us each): measured ~20 k-block equivalents. Launches whose tiles do not fill the machine
// (every tile would need several partners) keep split-K / narrow tiles instead.
static constexpr double kSkPartnerKb = 20.0;
static constexpr int kSkMinKb = 8;  // k-blocks per CTA at least (bounds the partners per tile)
static double g_sk_fix_scale = 1.0;  // FP_SK_FIX_SCALE (experiments)
struct SkPlan {
  int dp_tiles = 0, grid = 0;
  double cost = 1e30;
};
static SkPlan plan_streamk(const fp_ctx* c, int M, int N, int K) {
  SkPlan pl;
  const int T = ((M + kGemmBM - 1) / kGemmBM) * (N / 256), nk = K / kGemmBK, G0 = c->num_sms;
  const int waves = T / G0;
  // automatic use only where it measured a win: under-filled long-K launches (down_proj of
  // mid-size requests, -18% at M = 545); elsewhere pair tiles win (tools/gemm_probe.py)
  if (c->force_pair != 3 && (waves >= 1 || nk < 128)) return pl;
  pl.dp_tiles = waves >= 2 ? (waves - 1) * G0 : 0;
  const long long U = (long long)(T - pl.dp_tiles) * nk;
  pl.grid = (int)std::min<long long>(G0, U / kSkMinKb);
  // an under-filled launch gets at most two CTAs per tile (one partner each): a partner costs
  // far more than the k-blocks a third CTA would save
  if (waves < 1 && c->force_pair != 3) pl.grid = std::min(pl.grid, 2 * T);
  if (pl.grid < 2) return pl;
  const double per = std::ceil((double)U / pl.grid);
  const double partners = std::ceil(nk / per);
  pl.cost = (double)(pl.dp_tiles / G0) * (nk + 4.0) + per + 4.0 +
            g_sk_fix_scale * (kSkFixKb + kSkPartnerKb * partners);
  return pl;
}

template <int EPI>
static void launch_gemm_sk(fp_ctx* c, const CUtensorMap& a, const CUtensorMap& b, GemmParams p,
                           cudaStream_t st, const SkPlan& pl) {
  using Cfg = GemmCfg<256, 1>;
  auto kern = gemm_bf16_tn_kernel<256, EPI, 1, 3>;
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, c->device, [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SK_SMEM_BYTES);
  });
  p.splits = 1;
  p.full_tiles = pl.dp_tiles;
  p.group_m = raster_group(c, p);
  p.ws = c->ws;
  p.tickets = c->tickets;
  p.sk_flags = c->sk_flags;
  p.sk_epoch = ++c->sk_epoch;
  launch_pdl(kern, dim3(pl.grid), dim3(kGemmThreads), Cfg::SK_SMEM_BYTES, st, a, b, p);
}

// Cost (k-block units) of the best plan among single-CTA / pair / narrow tiles, as the pickers
// below see it.
static double plan_cost_tiled(const fp_ctx* c, int epi, int M, int N, int K) {
  int ft, sp;
  const int nN = N / 256, num_k = K / kGemmBK;
  const bool tail = split_tail_ok(epi, K);
  const double ov = split_overhead(epi);
  double t = choose_splits(((M + 127) / 128) * nN, num_k, c->num_sms, &ft, &sp, tail, ov);
  if (c->use_pair_gemm && M > kGemmBM)
    t = std::min(t, choose_splits(((M + 255) / 256) * nN, num_k, c->num_sms / 2, &ft, &sp, tail,
                                  ov) / 1.09);
  if ((epi == EPI_RESID || epi == EPI_QKV) && c->use_narrow) {
    const long long tiles = (long long)((M + 127) / 128) * (N / 128);
    t = std::min(t, std::ceil((double)tiles / c->num_sms) * (kNarrowKbCost * num_k + 4.0));
  }
  return t;
}

// Swap-AB skinny plan (skinny.cuh) for short launches: the weights stream once through all
// SMs, one equal contiguous (128-row weight slice, k-block) range per CTA. Needs the token
// operand's 32-row-box map; not for the TP exchange GEMMs (per-tile publish) nor batch-invariant
// mode (its per-CTA K ranges depend on the launch shape like split-K).
static constexpr int kSkinnySmallM = 8;     // skinny for any K up to this many rows
static constexpr int kSkinnyLongK = 8192;   // ... and up to skinny_max_m rows from this K
template <int EPI, int TOKMAX>
static void launch_skinny_t(fp_ctx* c, const CUtensorMap& x32, const CUtensorMap& w,
                            const GemmParams& p, int grid, cudaStream_t st) {
  using Cfg = SkinnyCfg<TOKMAX>;
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, c->device, [] {
    cudaFuncSetAttribute(gemm_skinny_kernel<EPI, TOKMAX>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  });
  launch_pdl(gemm_skinny_kernel<EPI, TOKMAX>, dim3(grid), dim3(kGemmThreads), Cfg::SMEM_BYTES,
             st, x32, w, p);
}
template <int EPI>
static bool launch_gemm_skinny(fp_ctx* c, const CUtensorMap* x32, const CUtensorMap& w,
                               GemmParams p, cudaStream_t st) {
  // (TP lock-step ranks share one device: a grid-wide arrival must not compete with a peer's)
  if (x32 == nullptr || p.xchg || c->batch_invariant || c->ws == nullptr || c->tp_lockstep)
    return false;
  const bool forced = c->force_pair == 4;
  if (!forced && (c->force_pair >= 0 || c->force_splits > 0 || p.M > c->skinny_max_m))
    return false;
  // Auto rule from the B200 A/B (tools/skinny_ab.py, profiles/r2_skinny_ab.log): the skinny
  // plan wins at a few rows (M = 1: qkv 1.5x, gate_up 1.46x, lm_head 1.24x) and on long-K
  // launches up to 128 rows (down_proj 1.05-1.09x); elsewhere the tiled plans' split-K / narrow
  // tiles are as fast or faster (both sit on the same ~10 us per-launch floor).
  if (!forced && p.M > kSkinnySmallM && p.K < kSkinnyLongK) return false;
  if (p.M < 1 || p.M > kSkinnyMaxM || p.N % 256 != 0 || p.K % kGemmBK != 0)
    return false;
  const long long U = (long long)(p.N / 128) * (p.K / kGemmBK);
  const int grid = (int)std::max(1LL, std::min<long long>(c->num_sms, U / 4));  // >= 4 k-blocks
  if ((long long)(grid + p.N / 128) * p.M * 128 > c->ws_floats) return false;  // partial slots
  p.ws = c->ws;
  p.tickets = c->tickets;
  if (p.M <= 64) launch_skinny_t<EPI, 64>(c, *x32, w, p, grid, st);
  else if (p.M <= 128) launch_skinny_t<EPI, 128>(c, *x32, w, p, grid, st);
  else launch_skinny_t<EPI, 256>(c, *x32, w, p, grid, st);
  return true;
}

template <int EPI>
static void launch_gemm(fp_ctx* c, const CUtensorMap& a, const CUtensorMap& b,
                        const GemmParams& p, cudaStream_t st, const CUtensorMap* a32 = nullptr) {
  if (launch_gemm_skinny<EPI>(c, a32, b, p, st)) return;
  if (!p.xchg && !c->batch_invariant &&
      (c->force_pair == 3 || (c->use_streamk && c->force_pair < 0 && c->force_splits == 0))) {
    const SkPlan pl = plan_streamk(c, p.M, p.N, p.K);
    if (pl.grid >= 2 &&
        (c->force_pair == 3 || pl.cost < 0.92 * plan_cost_tiled(c, EPI, p.M, p.N, p.K))) {
      launch_gemm_sk<EPI>(c, a, b, p, st, pl);
      return;
    }
  }
  if constexpr (EPI == EPI_RESID || EPI == EPI_QKV) {
    if (!p.xchg && pick_narrow(c, EPI, p.M, p.N, p.K)) {
      launch_gemm_cg<EPI, 1, 128>(c, a, b, p, st);
      return;
    }
  }
  if (pick_pair(c, EPI, p.M, p.N, p.K)) launch_gemm_cg<EPI, 2>(c, a, b, p, st);
  else launch_gemm_cg<EPI, 1>(c, a, b, p, st);
}

static int launch_rms(const RmsParams& p, cudaStream_t st) {
  if (p.M == 0) return FP_OK;
  if (p.d % 256 != 0 || p.d > 8192)
    return set_err(FP_ERR_UNSUPPORTED, "rmsnorm: hidden size must be a multiple of 256, <= 8192");
  launch_pdl(rmsnorm_kernel, dim3(p.M), dim3(p.d / 8), 0, st, p);
  return FP_OK;
}

static void launch_attn(const fp_ctx* c, const CUtensorMap& tq, const CUtensorMap& tkv,
                        const CUtensorMap& to,
                        const AttnTcParams& p, cudaStream_t st) {
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, c->device, [] {
    cudaFuncSetAttribute(attn_prefill_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         tcattn::SMEM_BYTES);
  });
  // persistent: one CTA per SM (at most one per work item), work taken longest-first
  const int n_work = p.n_items * p.n_kv_heads * p.pairs_per_kv;
  launch_pdl(attn_prefill_tc_kernel, dim3(std::min(n_work, c->num_sms)), dim3(tcattn::THREADS),
             tcattn::SMEM_BYTES, st, tq, tkv, to, p);
}

static bool boundary_eligible(const fp_ctx* c, int gran, int i, int n_entries) {
  // eligibility of the boundary AFTER entry i (engine.py:127-134 with layer_last/chunk_last)
  const int L = c->cfg.num_layers;
  const int op = i % 5;
  const int layer = (i / 5) % L;
  if (gran == FP_GRAN_OPERATOR) return true;
  if (gran == FP_GRAN_LAYER) return op == 4 || i == n_entries - 1;
  if (gran == FP_GRAN_CHUNK) return (op == 4 && layer == L - 1) || i == n_entries - 1;
  return false;
}

// Enqueue the kernels of one timeline entry. Caller holds launch_mu. Tensor parallel
// o_proj/down_proj entries have two phases: the exchange GEMM (phase 1) and the all-reduce plus
// anything after it (phase 2); a lock-step group on one device launches phase 1 of every rank
// before phase 2 of any rank so no all-reduce waits on a kernel queued behind it.
constexpr int kPhasePre = 1, kPhasePost = 2, kPhaseAll = 3;
// Completion of the chunk's requests after the last layer: final norm + lm_head of their last
// tokens (cost_model.py:240-241 charges this to the chunk).
static int launch_final(fp_ctx* c, Task* t, const ChunkPlan& ch, int layer, const Guard& g2,
                        cudaStream_t st) {
  const fp_model_cfg& m = c->cfg;
  if (ch.n_last == 0) return FP_OK;
  RmsParams r{};
  r.M = ch.n_last;
  r.d = m.hidden;
  r.src = t->h;
  r.ld_src = m.hidden;
  r.rows = t->d_last + ch.last0;
  r.gamma = c->final_g;
  r.out = t->xf;
  r.ld_out = m.hidden;
  r.eps = m.rms_eps;
  r.guard = g2;
  {
    ProfScope ps(c, st, FP_K_RMS_FINAL, layer, ch.n_last, 0.0, 2.0 * ch.n_last * m.hidden * 2);
    int rc = launch_rms(r, st);
    if (rc) return rc;
  }
  GemmParams q{};
  q.M = ch.n_last;
  q.N = c->vocab_pad;
  q.K = m.hidden;
  q.out = t->logits + (long long)ch.seq0 * c->vocab_pad;
  q.ldo = c->vocab_pad;
  q.guard = g2;
  ProfScope ps(c, st, FP_K_LM_HEAD, layer, ch.n_last, 2.0 * ch.n_last * q.N * q.K, 0.0);
  launch_gemm<EPI_STORE_F32>(c, t->tm_xf, c->tm_lm, q, st, &t->tm_xf32);
  return FP_OK;
}

// MoE layer, entries `gate` (op 3) and `experts` (op 4): moe.cuh. The post-attention norm is
// fused into the router and the expert gate/up GEMM (folded weights + the row's rsqrt from the
// segment sums of squares the o_proj epilogue wrote), exactly as for the dense gate_up_proj.
static int launch_moe_entry(fp_ctx* c, Task* t, const ChunkPlan& ch, int layer, int op,
                            const Guard& g, const Guard& g2, cudaStream_t st) {
  const fp_model_cfg& m = c->cfg;
  const int M = ch.M, d = m.hidden, E = m.n_experts, K = m.top_k, I = m.moe_ffn;
  Layer& ly = c->layers[layer];
  MoeParams mp{};
  mp.M = M;
  mp.n_experts = E;
  mp.top_k = K;
  mp.norm_topk = m.norm_topk;
  mp.d = d;
  mp.logits = t->rlog;
  mp.ld_logits = 256;
  mp.topk_ids = t->m_ids;
  mp.topk_w = t->m_w;
  mp.slot = t->m_slot;
  mp.counts = t->m_counts;
  mp.cursor = t->m_cursor;
  mp.offsets = t->m_off;
  mp.mtile_count = t->m_mtc;
  mp.mtiles = t->m_mtiles;
  mp.perm_tok = t->m_perm;
  mp.ticket = t->m_perm + (long long)t->max_m * K;  // the first slack int after perm (zeroed)
  mp.h = t->h;
  mp.h_out = t->h;
  mp.xperm = t->xperm;
  mp.yperm = t->yperm;
  mp.ssq = t->ssq;
  mp.guard = g2;
  const int tok_blocks = (M + 7) / 8;
  const double rows = (double)M * K;
  if (op == FP_OP_GATE) {
    GemmParams p{};
    p.M = M;
    p.N = E <= 128 ? 128 : 256;  // router rows are padded to 256; compute only what is real
    p.K = d;
    p.out = t->rlog;
    p.ldo = 256;
    p.nseg = d / 128;
    p.ssq_in = t->ssq;
    p.norm_eps_in = m.rms_eps;
    p.guard = g;
    {
      ProfScope ps(c, st, FP_K_ROUTER, layer, M, 2.0 * M * E * d, 0.0);
      if (p.N == 128) launch_gemm_cg<EPI_STORE_F32, 1, 128>(c, t->tm_h, ly.tm_r, p, st);
      else launch_gemm<EPI_STORE_F32>(c, t->tm_h, ly.tm_r, p, st);
    }
    ProfScope ps(c, st, FP_K_MOE_DISPATCH, layer, M, 0.0, rows * d * 2 * 2);
    launch_pdl(moe_route_kernel, dim3(tok_blocks), dim3(256), 0, st, mp);  // + plan (last block)
    launch_pdl(moe_scatter_kernel, dim3(tok_blocks), dim3(256), 0, st, mp);
    t->moe_rows = M;
    return FP_OK;
  }
  // experts
  GemmParams p{};
  p.M = (int)rows;
  p.K = d;
  p.N = 2 * I;
  p.out = t->actp;
  p.ldo = I;
  p.nseg = d / 128;
  p.ssq_in = t->ssq;
  p.norm_eps_in = m.rms_eps;
  p.grp_mtiles = reinterpret_cast<const int*>(t->m_mtiles);
  p.grp_count = t->m_mtc;
  p.grp_off = t->m_off;
  p.grp_perm = t->m_perm;
  p.grp_b_rows = 2 * I;
  p.guard = g;
  {
    ProfScope ps(c, st, FP_K_EXPERT_GU, layer, (int)rows, 2.0 * rows * 2 * I * d, 0.0);
    launch_gemm_grouped<EPI_SWIGLU>(c, t->tm_xperm, ly.tm_egu, p, st);
  }
  GemmParams q{};
  q.M = (int)rows;
  q.K = I;
  q.N = d;
  q.out = t->yperm;
  q.ldo = d;
  q.grp_mtiles = p.grp_mtiles;
  q.grp_count = p.grp_count;
  q.grp_off = p.grp_off;
  q.grp_perm = p.grp_perm;
  q.grp_b_rows = d;
  q.guard = g2;
  {
    ProfScope ps(c, st, FP_K_EXPERT_DOWN, layer, (int)rows, 2.0 * rows * I * d, 0.0);
    launch_gemm_grouped<EPI_STORE_BF16>(c, t->tm_actp, ly.tm_ed, q, st);
  }
  {
    ProfScope ps(c, st, FP_K_MOE_COMBINE, layer, M, 0.0, (rows + 2.0 * M) * d * 2);
    const long long units = (long long)M * (d / 256);
    launch_pdl(moe_combine_kernel, dim3((int)((units + 7) / 8)), dim3(256), 0, st, mp);
  }
  if (layer == m.num_layers - 1) return launch_final(c, t, ch, layer, g2, st);
  return FP_OK;
}

static int launch_entry(fp_ctx* c, Task* t, int e, int phase = kPhaseAll) {
  const fp_model_cfg& m = c->cfg;
  const int L = m.num_layers;
  const int ci = e / (5 * L);
  const int layer = (e / 5) % L;
  const int op = e % 5;
  const ChunkPlan& ch = t->chunks[ci];
  const int M = ch.M;
  cudaStream_t st = c->stream;
  Layer& ly = c->layers[layer];

  Guard g{};
  g.host = c->dctl;
  g.task = t->ctl;
  g.entry = e;
  g.gen = t->gen;
  g.task_id = t->id;
  g.first = 1;
  g.eligible = (e != t->seg_first) && boundary_eligible(c, t->granularity, e - 1, t->n_entries);
  g.n_entries = t->n_entries;
  g.tp = c->d_tp;
  Guard g2 = g;
  g2.first = 0;

  const int* ids = t->d_ids + ch.tok0;
  const int* pos = t->d_pos + ch.tok0;
  const int* tpage = t->d_tpage + ch.tok0;
  __nv_bfloat16* kv_layer = c->kv + (long long)layer * c->kv_pages * c->page_elems;

  const bool xchg_op = c->tp_size > 1 && (op == FP_OP_O_PROJ || op == FP_OP_DOWN_PROJ);
  if (!xchg_op && !(phase & kPhasePre)) return FP_OK;  // single-phase entries run in phase 1
  const int nseg = m.hidden / 128;  // fused-norm sum-of-squares segments
  if (m.n_experts > 0 && op >= FP_OP_GATE) return launch_moe_entry(c, t, ch, layer, op, g, g2, st);
  if (op == FP_OP_QKV_PROJ || op == FP_OP_GATE_UP_PROJ) {
    // The input RMSNorm is fused: the GEMM reads h with the norm weight folded into its weight
    // columns and scales rows by rsqrt(mean(h^2) + eps) from the segment sums in t->ssq.
    Guard gg = g;
    if (op == FP_OP_QKV_PROJ && layer == 0) {  // chunk start: embedding gather into h (+ sums)
      RmsParams r{};
      r.M = M;
      r.d = m.hidden;
      r.src = c->embed;
      r.ld_src = m.hidden;
      r.ids = ids;
      r.h_out = t->h;
      r.ld_h = m.hidden;
      r.gamma = ly.attn_g;
      r.eps = m.rms_eps;
      r.nseg = nseg;
      r.ssq = t->ssq;
      r.guard = g;
      ProfScope ps(c, st, FP_K_RMS, layer, M, 0.0, 2.0 * M * m.hidden * 2);
      int rc = launch_rms(r, st);
      if (rc) return rc;
      gg = g2;
    }
    GemmParams p{};
    p.M = M;
    p.K = m.hidden;
    p.guard = gg;
    p.nseg = nseg;
    p.ssq_in = t->ssq;
    p.norm_eps_in = m.rms_eps;
    if (op == FP_OP_QKV_PROJ) {
      p.N = c->qkv_n;
      p.pos = pos;
      p.tok_page = tpage;
      p.qbuf = t->q;
      p.ldq = c->qdim;
      p.kv_layer = kv_layer;
      p.rope = c->rope;
      p.q_cols = c->qdim;
      p.kv_cols = c->kvdim;
      p.page_size = c->page_size;
      p.n_kv_heads = c->hkv;
      p.bias = ly.bqkv;
      p.q_norm = ly.q_norm;
      p.k_norm = ly.k_norm;
      p.norm_eps = m.rms_eps;
      ProfScope ps(c, st, FP_K_QKV, layer, M, 2.0 * M * p.N * p.K, 0.0);
      launch_gemm<EPI_QKV>(c, t->tm_h, ly.tm_qkv, p, st, &t->tm_h32);
    } else {
      p.N = 2 * c->ffn;
      p.out = t->act;
      p.ldo = c->ffn;
      ProfScope ps(c, st, FP_K_GATE_UP, layer, M, 2.0 * M * p.N * p.K, 0.0);
      launch_gemm<EPI_SWIGLU>(c, t->tm_h, ly.tm_gu, p, st, &t->tm_h32);
    }
  } else if (op == FP_OP_ATTN) {
    AttnTcParams a{};
    a.items = t->d_items + ch.item0;
    a.n_items = ch.n_items;
    a.n_heads = c->hq;
    a.n_kv_heads = c->hkv;
    a.pairs_per_kv = (c->hq / c->hkv + 1) / 2;
    a.out = t->ao;
    a.ldo = c->qdim;
    a.block_table = t->d_bt;
    a.bt_stride = t->bt_stride;
    a.kv_row_layer = (long long)layer * c->kv_pages * 2 * c->hkv * c->page_size;
    a.kv_rows_per_page = 2 * c->hkv * c->page_size;
    a.scale_log2 = 1.4426950408889634f / sqrtf((float)m.head_dim);
    a.sched = c->attn_sched;
    a.dbg = c->gemm_dbg;
    a.guard = g;
    if (a.n_items > 0) {
      ProfScope ps(c, st, FP_K_ATTN, layer, M, ch.attn_flops, 0.0);
      launch_attn(c, t->tm_q, c->tm_kv, t->tm_ao, a, st);  // out = ao (map: 128-row boxes)
    }
  } else {  // O_PROJ / DOWN_PROJ: residual add (tensor parallel: partial sum + all-reduce)
    GemmParams p{};
    p.M = M;
    p.N = m.hidden;
    p.resid = t->h;
    p.ldr = m.hidden;
    p.guard = g;
    p.nseg = nseg;
    p.ssq_out = t->ssq;  // segment sums of the new h for the next fused norm
    p.K = op == FP_OP_O_PROJ ? c->qdim : c->ffn;
    const CUtensorMap& ta = op == FP_OP_O_PROJ ? t->tm_ao : t->tm_act;
    const CUtensorMap& tb = op == FP_OP_O_PROJ ? ly.tm_o : ly.tm_d;
    const CUtensorMap* ta32 = op == FP_OP_O_PROJ ? &t->tm_ao32 : &t->tm_act32;
    const int kind = op == FP_OP_O_PROJ ? FP_K_O : FP_K_DOWN;
    if (!xchg_op) {
      ProfScope ps(c, st, kind, layer, M, 2.0 * M * p.N * p.K, 0.0);
      launch_gemm<EPI_RESID>(c, ta, tb, p, st, ta32);
    } else {
      // One process per GPU: the exchange is FUSED into the GEMM (each tile's partial is
      // flagged to the peers and folded tile by tile over NVLink inside the same kernel).
      // Ranks in lock step on one device (launched one after another) cannot wait on each
      // other inside a kernel: they use the GEMM + tp_allreduce_kernel pair.
      const bool fused = !c->tp_lockstep && c->tp_fused &&
                         (long long)((M + 127) / 128) * (m.hidden / 256) <= kTpFlagTiles;
      if (phase & kPhasePre) {
        p.xchg = fused ? 2 : 1;
        p.ldo = m.hidden;
        ProfScope ps(c, st, kind, layer, M, 2.0 * M * p.N * p.K, 0.0);
        launch_gemm<EPI_STORE_BF16>(c, ta, tb, p, st);
      }
      if (fused || !(phase & kPhasePost)) {
        if (fused && op == FP_OP_DOWN_PROJ && layer == L - 1)
          return launch_final(c, t, ch, layer, g2, st);
        return FP_OK;
      }
      XchgParams x{};
      x.M = M;
      x.d = m.hidden;
      x.h = t->h;
      x.ldh = m.hidden;
      x.ssq = t->ssq;
      x.guard = g2;
      const long long vecs = (long long)M * m.hidden / 8;
      const int grid = (int)std::max(1LL, std::min<long long>((vecs + 255) / 256, 8LL * c->num_sms));
      ProfScope ps(c, st, FP_K_XCHG, layer, M, 0.0, (double)(c->tp_size + 2) * M * m.hidden * 2);
      launch_pdl(tp_allreduce_kernel, dim3(grid), dim3(256), 0, st, x);
    }
    if (op == FP_OP_DOWN_PROJ && layer == L - 1) return launch_final(c, t, ch, layer, g2, st);
  }
  return FP_OK;
}

// launch_entry plus the launch status: cudaLaunchKernelEx failures (bad config, missing
// attribute, sticky device error) surface here instead of a silently skipped kernel.
static int launch_entry_checked(fp_ctx* c, Task* t, int e, int phase = kPhaseAll) {
  int rc = launch_entry(c, t, e, phase);
  const cudaError_t le = cudaGetLastError();
  if (rc == FP_OK && le != cudaSuccess)
    rc = set_err(FP_ERR_CUDA, std::string("kernel launch of entry ") + std::to_string(e) + ": " +
                                  cudaGetErrorString(le));
  return rc;
}

// --------------------------------------------------------------------------- worker
static void worker_main(fp_ctx* c) {
  cudaSetDevice(c->device);
  for (;;) {
    Task* t = nullptr;
    {
      std::unique_lock<std::mutex> lk(c->wmu);
      c->wcv.wait(lk, [&] { return c->wquit || c->wtask != nullptr; });
      if (c->wquit) return;
      t = c->wtask;
    }
    while (t->enq < t->n_entries) {
      if (c->hctl->ack_seq != t->seg_ack0) break;  // stopped: leave the rest unlaunched
      int prog = t->seg_first - 1;
      if (c->hctl->progress_task == t->id) prog = std::max(prog, (int)c->hctl->progress_entry);
      if (t->enq - prog <= c->window) {
        std::lock_guard<std::mutex> lk(c->launch_mu);
        const int rc = launch_entry_checked(c, t, t->enq);
        if (rc) {  // stop launching; never report this segment done
          t->err_msg = g_err;
          t->err.store(rc);
          break;
        }
        t->enq++;
      } else {
        std::this_thread::yield();
      }
    }
    {
      std::lock_guard<std::mutex> lk(c->launch_mu);
      if (!t->err.load() && t->enq == t->n_entries) {
        cudaEventRecord(t->done, c->stream);
        t->done_recorded = 1;
      }
      cudaEventRecord(t->fence, c->stream);
    }
    {
      std::lock_guard<std::mutex> lk(c->wmu);
      c->wtask = nullptr;
    }
    t->worker_active.store(0);
  }
}

// --------------------------------------------------------------------------- C ABI
extern "C" {

const char* fp_last_error(void) { return g_err.c_str(); }
int fp_version(void) { return 1; }

// Builds the context into *cp (set as soon as it exists: a failure part-way is cleaned up by
// fp_ctx_destroy, which tolerates unset members).
static int ctx_create_impl(int32_t device, const fp_model_cfg* cfg, int32_t tp_rank,
                           int32_t tp_size, void* nccl_comm, int64_t kv_pages, int32_t page_size,
                           fp_ctx** cp) {
  REQ(cfg, "null argument");
  REQ(nccl_comm == nullptr,
      "nccl_comm must be null: the tensor-parallel exchange runs over peer memory "
      "(fp_tp_connect_local / fp_tp_export + fp_tp_import)");
  REQ(tp_size >= 1 && tp_size <= kTpMax && tp_rank >= 0 && tp_rank < tp_size, "bad tp_rank/tp_size");
  REQ(cfg->head_dim == 128, "head_dim must be 128");
  REQ(cfg->n_heads % cfg->n_kv_heads == 0, "n_heads must be a multiple of n_kv_heads");
  REQ(cfg->n_kv_heads % tp_size == 0, "n_kv_heads must be divisible by tp_size");
  REQ(cfg->hidden % 512 == 0 && cfg->ffn % (128 * tp_size) == 0,
      "hidden%512 and ffn%(128*tp_size) required");
  if (cfg->n_experts > 0) {
    REQ(tp_size == 1, "MoE models run as single-GPU instances (no tensor parallelism)");
    REQ(cfg->n_experts <= kMoeMaxExperts && cfg->top_k >= 1 && cfg->top_k <= kMoeMaxTopK &&
            cfg->top_k <= cfg->n_experts,
        "MoE: n_experts <= 256, 1 <= top_k <= min(16, n_experts)");
    REQ(cfg->moe_ffn > 0 && cfg->moe_ffn % 128 == 0, "MoE: moe_ffn must be a multiple of 128");
  } else {
    REQ(cfg->ffn > 0, "dense models need ffn > 0");
  }
  REQ(page_size == 128, "page_size must be 128 (one attention KV tile per page)");
  REQ(kv_pages > 0, "kv_pages must be > 0");
  CK(cudaSetDevice(device));
  int major = 0;
  CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  if (major != 10) return set_err(FP_ERR_UNSUPPORTED, "requires an sm_100 (B200) device");
  fp_ctx* c = new fp_ctx();
  *cp = c;
  c->device = device;
  c->cfg = *cfg;
  c->tp_rank = tp_rank;
  c->tp_size = tp_size;
  c->hq = cfg->n_heads / tp_size;
  c->hkv = cfg->n_kv_heads / tp_size;
  c->ffn = cfg->ffn / tp_size;
  c->qdim = c->hq * 128;
  c->kvdim = c->hkv * 128;
  c->qkv_n = (c->qdim + 2 * c->kvdim + 255) / 256 * 256;
  c->page_size = page_size;
  c->kv_pages = kv_pages;
  c->page_elems = 2LL * c->hkv * page_size * 128;
  CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
  CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  c->own_stream = c->stream;
  CK(cudaStreamCreateWithFlags(&c->upload, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c->readback, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c->release, cudaStreamNonBlocking));
  // let the async mempool keep freed task workspaces
  cudaMemPool_t pool;
  CK(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t thresh = UINT64_MAX;
  CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));

  const int L = cfg->num_layers, d = cfg->hidden;
  c->layers.resize(L);
  for (int l = 0; l < L; ++l) {
    Layer& ly = c->layers[l];
    CK(cudaMalloc(&ly.wqkv, (size_t)c->qkv_n * d * 2));
    CK(cudaMemset(ly.wqkv, 0, (size_t)c->qkv_n * d * 2));  // padding rows stay zero
    CK(cudaMalloc(&ly.wo, (size_t)d * c->qdim * 2));
    CK(cudaMemset(ly.wo, 0, (size_t)d * c->qdim * 2));  // weights start zero: a partial load
    if (cfg->n_experts == 0) {
      CK(cudaMalloc(&ly.wgu, (size_t)2 * c->ffn * d * 2));
      CK(cudaMemset(ly.wgu, 0, (size_t)2 * c->ffn * d * 2));  // (and a norm refold of rows not
      CK(cudaMalloc(&ly.wd, (size_t)d * c->ffn * 2));            // loaded yet) reads defined data
      CK(cudaMemset(ly.wd, 0, (size_t)d * c->ffn * 2));
    } else {
      const size_t E = cfg->n_experts, I = cfg->moe_ffn;
      CK(cudaMalloc(&ly.wr, (size_t)256 * d * 2));
      CK(cudaMemset(ly.wr, 0, (size_t)256 * d * 2));  // padding experts: logits 0, masked
      CK(cudaMalloc(&ly.egu, E * 2 * I * d * 2));
      CK(cudaMemset(ly.egu, 0, E * 2 * I * d * 2));
      CK(cudaMalloc(&ly.ed, E * d * I * 2));
      CK(cudaMemset(ly.ed, 0, E * d * I * 2));
    }
    CK(cudaMalloc(&ly.attn_g, (size_t)d * 2));
    CK(cudaMalloc(&ly.ffn_g, (size_t)d * 2));
    {
      const std::vector<uint16_t> ones(d, 0x3F80);  // bf16 1.0: nothing folded yet
      CK(cudaMemcpy(ly.attn_g, ones.data(), (size_t)d * 2, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(ly.ffn_g, ones.data(), (size_t)d * 2, cudaMemcpyHostToDevice));
    }
    if (cfg->qkv_bias) {
      CK(cudaMalloc(&ly.bqkv, (size_t)c->qkv_n * 4));
      CK(cudaMemset(ly.bqkv, 0, (size_t)c->qkv_n * 4));
    }
    if (cfg->qk_norm) {
      CK(cudaMalloc(&ly.q_norm, 128 * 4));
      CK(cudaMalloc(&ly.k_norm, 128 * 4));
      CK(cudaMemset(ly.q_norm, 0, 128 * 4));
      CK(cudaMemset(ly.k_norm, 0, 128 * 4));
    }
    int rc;
    if ((rc = make_map(&ly.tm_qkv, ly.wqkv, c->qkv_n, d, 128))) return rc;
    if ((rc = make_map(&ly.tm_o, ly.wo, d, c->qdim, 128))) return rc;
    if (cfg->n_experts == 0) {
      if ((rc = make_map(&ly.tm_gu, ly.wgu, 2 * c->ffn, d, 128))) return rc;
      if ((rc = make_map(&ly.tm_d, ly.wd, d, c->ffn, 128))) return rc;
    } else {
      const long long E = cfg->n_experts, I = cfg->moe_ffn;
      if ((rc = make_map(&ly.tm_r, ly.wr, 256, d, 128))) return rc;
      if ((rc = make_map(&ly.tm_egu, ly.egu, E * 2 * I, d, 128))) return rc;
      if ((rc = make_map(&ly.tm_ed, ly.ed, E * d, I, 128))) return rc;
    }
  }
  CK(cudaMalloc(&c->embed, (size_t)cfg->vocab * d * 2));
  CK(cudaMemset(c->embed, 0, (size_t)cfg->vocab * d * 2));
  c->vocab_pad = (cfg->vocab + 255) / 256 * 256;  // lm_head GEMM tiles are 256 wide
  CK(cudaMalloc(&c->lm_head, (size_t)c->vocab_pad * d * 2));
  CK(cudaMemset(c->lm_head, 0, (size_t)c->vocab_pad * d * 2));
  CK(cudaMalloc(&c->final_g, (size_t)d * 2));
  {
    int rc = make_map(&c->tm_lm, c->lm_head, c->vocab_pad, d, 128);
    if (rc) return rc;
  }
  // RoPE table (rotate-half convention), fp64 on the host
  {
    std::vector<float2> tab((size_t)cfg->max_pos * 64);
    for (int p = 0; p < cfg->max_pos; ++p)
      for (int j = 0; j < 64; ++j) {
        const double inv = 1.0 / std::pow((double)cfg->rope_theta, (2.0 * j) / 128.0);
        const double a = (double)p * inv;
        tab[(size_t)p * 64 + j] = make_float2((float)std::cos(a), (float)std::sin(a));
      }
    CK(cudaMalloc(&c->rope, tab.size() * sizeof(float2)));
    CK(cudaMemcpy(c->rope, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice));
  }
  CK(cudaMalloc(&c->kv, (size_t)L * kv_pages * c->page_elems * 2));
  // zero once: slots past a request's length are read (and masked) by attention tiles, so
  // they must hold finite values
  CK(cudaMemset(c->kv, 0, (size_t)L * kv_pages * c->page_elems * 2));
  {
    if (const char* e = getenv("FP_PAIR_GEMM")) c->use_pair_gemm = atoi(e) != 0;
    if (const char* e = getenv("FP_NARROW")) c->use_narrow = atoi(e) != 0;
    if (const char* e = getenv("FP_STREAMK")) c->use_streamk = atoi(e) != 0;
    if (const char* e = getenv("FP_BATCH_INVARIANT")) c->batch_invariant = atoi(e) != 0;
    if (const char* e = getenv("FP_RASTER_ALL_MB")) g_raster_all_mb = atoi(e);
    if (const char* e = getenv("FP_SK_FIX_SCALE")) g_sk_fix_scale = atof(e);
    if (const char* e = getenv("FP_SPLIT_OV_SCALE")) g_split_ov_scale = atof(e);
    if (const char* e = getenv("FP_SPLIT_TAIL")) g_split_tail = atoi(e);
    if (const char* e = getenv("FP_FORCE_SPLITS")) c->force_splits = atoi(e);
    if (const char* e = getenv("FP_FORCE_PAIR")) c->force_pair = atoi(e);
    if (const char* e = getenv("FP_TP_FUSED")) c->tp_fused = atoi(e) != 0;
    if (const char* e = getenv("FP_SKINNY_MAX_M")) c->skinny_max_m = atoi(e);
    if (const char* e = getenv("FP_SPLIT_DSMEM")) c->split_dsmem = atoi(e) != 0;
    if (const char* e = getenv("FP_GEMM_STAMPS"))
      if (atoi(e)) CK(cudaMalloc(&c->gemm_dbg, (size_t)4096 * 16 * sizeof(unsigned long long)));
    const uint64_t rows = (uint64_t)L * kv_pages * 2 * c->hkv * page_size;
    REQ(rows < (1ull << 31), "KV pool too large for 32-bit TMA row coordinates");
    int rc = make_map(&c->tm_kv, c->kv, rows, 128, 128);
    if (rc) return rc;
  }
  c->free_pages.resize(kv_pages);
  for (long long i = 0; i < kv_pages; ++i) c->free_pages[i] = (int)(kv_pages - 1 - i);
  c->ws_floats = 8LL * c->num_sms * kGemmBM * 256;
  CK(cudaMalloc(&c->ws, (size_t)c->ws_floats * sizeof(float)));
  CK(cudaMalloc(&c->attn_sched, 2 * sizeof(int)));
  CK(cudaMemset(c->attn_sched, 0, 2 * sizeof(int)));
  CK(cudaMalloc(&c->tickets, 4096 * sizeof(int)));
  CK(cudaMalloc(&c->sk_flags, (size_t)c->num_sms * sizeof(int)));
  CK(cudaMemset(c->sk_flags, 0, (size_t)c->num_sms * sizeof(int)));
  CK(cudaMemset(c->tickets, 0, 4096 * sizeof(int)));
  CK(cudaHostAlloc(&c->hctl, sizeof(HostCtl), cudaHostAllocMapped));
  memset((void*)c->hctl, 0, sizeof(HostCtl));
  c->hctl->progress_task = -1;
  CK(cudaHostGetDevicePointer((void**)&c->dctl, (void*)c->hctl, 0));
  // Pre-grow the (shared, never-trimmed) async pool that task workspaces come from: growing it
  // maps physical memory inside cudaMallocAsync, which blocks task creation while the GPU runs
  // (measured: up to ~5 ms per task in a serving loop). FP_POOL_RESERVE_MB overrides the
  // default of 8 GB (capped at a quarter of the free memory); 0 disables.
  {
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    size_t reserve = std::min<size_t>((size_t)8 << 30, free_b / 4);
    if (const char* e = getenv("FP_POOL_RESERVE_MB")) reserve = (size_t)atoll(e) << 20;
    if (reserve > 0) {
      void* r = nullptr;
      CK(cudaMallocAsync(&r, reserve, c->upload));
      CK(cudaFreeAsync(r, c->upload));
      CK(cudaStreamSynchronize(c->upload));
    }
  }
  c->worker = std::thread(worker_main, c);
  return FP_OK;
}

int fp_ctx_create(int32_t device, const fp_model_cfg* cfg, int32_t tp_rank, int32_t tp_size,
                  void* nccl_comm, int64_t kv_pages, int32_t page_size, fp_ctx** out) {
  REQ(out, "null argument");
  fp_ctx* c = nullptr;
  const int rc = ctx_create_impl(device, cfg, tp_rank, tp_size, nccl_comm, kv_pages, page_size, &c);
  if (rc != FP_OK) {
    if (c) {
      const std::string msg = fp_last_error();  // keep the first failure's message
      fp_ctx_destroy(c);
      cudaGetLastError();  // a failed allocation must not surface in a later, unrelated check
      set_err(rc, msg);
    }
    return rc;
  }
  *out = c;
  return FP_OK;
}

int fp_ctx_destroy(fp_ctx* c) {
  if (!c) return FP_OK;
  {
    std::lock_guard<std::mutex> lk(c->wmu);
    c->wquit = true;
  }
  c->wcv.notify_all();
  if (c->worker.joinable()) c->worker.join();
  cudaSetDevice(c->device);
  if (c->tp_lockstep) cudaDeviceSynchronize();  // the shared stream may belong to rank 0
  else cudaStreamSynchronize(c->stream);
  for (auto& ly : c->layers) {
    cudaFree(ly.wqkv);
    cudaFree(ly.wo);
    cudaFree(ly.wgu);
    cudaFree(ly.wd);
    cudaFree(ly.wr);
    cudaFree(ly.egu);
    cudaFree(ly.ed);
    cudaFree(ly.attn_g);
    cudaFree(ly.ffn_g);
    cudaFree(ly.bqkv);
    cudaFree(ly.q_norm);
    cudaFree(ly.k_norm);
  }
  cudaFree(c->embed);
  cudaFree(c->lm_head);
  cudaFree(c->final_g);
  cudaFree(c->rope);
  cudaFree(c->kv);
  cudaFree(c->ws);
  cudaFree(c->tickets);
  cudaFree(c->sk_flags);
  cudaFree(c->attn_sched);
  cudaFree(c->gemm_dbg);
  cudaFreeHost((void*)c->hctl);
  for (void* ptr : c->tp_opened) cudaIpcCloseMemHandle(ptr);
  cudaFree(c->tp_block);
  cudaFree(c->tp_local);
  cudaFree(c->d_tp);
  if (c->stage) cudaFreeHost(c->stage);
  if (c->stage_ev) cudaEventDestroy(c->stage_ev);
  for (cudaStream_t st : {c->own_stream, c->upload, c->readback, c->release})
    if (st) cudaStreamDestroy(st);
  delete c;
  return FP_OK;
}

int fp_ctx_stream(fp_ctx* c, void** s) {
  REQ(c && s, "null argument");
  *s = (void*)c->stream;
  return FP_OK;
}
int fp_ctx_free_pages(fp_ctx* c, int64_t* n) {
  REQ(c && n, "null argument");
  std::lock_guard<std::mutex> lk(c->page_mu);
  *n = (int64_t)c->free_pages.size();
  return FP_OK;
}
int fp_ctx_set_window(fp_ctx* c, int32_t w) {
  REQ(c && w >= 1, "window must be >= 1");
  c->window = w;
  return FP_OK;
}
int fp_debug_gemm_stamps(fp_ctx* c, uint64_t* out, int32_t max_ctas) {
  REQ(c && out && max_ctas > 0, "bad arguments");
  REQ(c->gemm_dbg != nullptr, "phase stamps disabled (set FP_GEMM_STAMPS=1 before fp_ctx_create)");
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaMemcpy(out, c->gemm_dbg, (size_t)std::min(max_ctas, 4096) * 16 * sizeof(uint64_t),
                cudaMemcpyDeviceToHost));
  return FP_OK;
}
int fp_ctx_set_gemm_policy(fp_ctx* c, int32_t pair, int32_t splits) {
  REQ(c && pair >= -1 && pair <= 4 && splits >= 0 && splits <= 32, "bad gemm policy");
  c->force_pair = pair;
  c->force_splits = splits;
  return FP_OK;
}
int fp_ctx_set_skinny_max(fp_ctx* c, int32_t max_m) {
  REQ(c && max_m >= 0, "bad skinny threshold");
  c->skinny_max_m = max_m;
  return FP_OK;
}
int fp_ctx_set_batch_invariant(fp_ctx* c, int32_t on) {
  REQ(c, "null ctx");
  c->batch_invariant = on != 0;
  return FP_OK;
}
int fp_sync(fp_ctx* c) {
  REQ(c, "null ctx");
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  return FP_OK;
}

// Weights arrive as the full (unsharded) canonical tensors; a tensor-parallel rank keeps its
// Megatron shard: q/k/v/gate/up rows (column-parallel), o/down columns (row-parallel), biases
// with their rows, everything else replicated.
// bf16 host vector -> fp32 device vector (biases, q/k norm weights live in fp32)
static int load_f32_vec(float* dst, const void* host, int64_t n) {
  std::vector<float> f(n);
  const uint16_t* h = static_cast<const uint16_t*>(host);
  for (int64_t i = 0; i < n; ++i) {
    uint32_t u = (uint32_t)h[i] << 16;
    memcpy(&f[i], &u, 4);
  }
  CK(cudaMemcpy(dst, f.data(), n * 4, cudaMemcpyHostToDevice));
  return FP_OK;
}

static void fold(fp_ctx* c, __nv_bfloat16* w, long long row0, int nblocks, long long bstride,
                 int rpb, const __nv_bfloat16* g_new, const __nv_bfloat16* g_old) {
  const long long n = (long long)nblocks * rpb * c->cfg.hidden;
  const int grid = (int)std::min<long long>((n + 255) / 256, 16LL * c->num_sms);
  fold_cols_kernel<<<grid, 256, 0, c->stream>>>(w, row0, nblocks, bstride, rpb, c->cfg.hidden,
                                                g_new, g_old);
}

int fp_weights_load(fp_ctx* c, int32_t tensor, int32_t layer, const void* host, int64_t n) {
  REQ(c && host, "null argument");
  CK(cudaSetDevice(c->device));
  const fp_model_cfg& m = c->cfg;
  const long long d = m.hidden, r = c->tp_rank;
  const long long Qd = (long long)m.n_heads * 128, KVd = (long long)m.n_kv_heads * 128;
  const long long F = m.ffn;
  const char* src = static_cast<const char*>(host);
  switch (tensor) {  // replicated, model-level
    case FP_W_EMBED:
    case FP_W_LM_HEAD:
      REQ(n == (long long)m.vocab * d, "weight size mismatch");
      CK(cudaMemcpy(tensor == FP_W_EMBED ? c->embed : c->lm_head, host, (size_t)n * 2,
                    cudaMemcpyHostToDevice));
      return FP_OK;
    case FP_W_FINAL_NORM:
      REQ(n == d, "weight size mismatch");
      CK(cudaMemcpy(c->final_g, host, (size_t)n * 2, cudaMemcpyHostToDevice));
      return FP_OK;
    default:
      break;
  }
  REQ(layer >= 0 && layer < m.num_layers, "bad layer");
  Layer& ly = c->layers[layer];
  switch (tensor) {
    case FP_W_Q:
    case FP_W_K:
    case FP_W_V: {  // column-parallel: this rank's head rows
      const bool q = tensor == FP_W_Q;
      REQ(n == (q ? Qd : KVd) * d, "weight size mismatch");
      const long long rows = q ? c->qdim : c->kvdim;
      const long long off = q ? 0 : (tensor == FP_W_K ? c->qdim : c->qdim + c->kvdim);
      CK(cudaMemcpy(ly.wqkv + off * d, src + r * rows * d * 2, (size_t)rows * d * 2,
                    cudaMemcpyHostToDevice));
      fold(c, ly.wqkv, off, 1, 0, (int)rows, ly.attn_g, nullptr);  // fused input norm
      CK(cudaStreamSynchronize(c->stream));
      return FP_OK;
    }
    case FP_W_O:
    case FP_W_DOWN: {  // row-parallel: this rank's input columns
      const bool o = tensor == FP_W_O;
      const long long full = o ? Qd : F, cols = o ? c->qdim : c->ffn;
      REQ(n == d * full, "weight size mismatch");
      CK(cudaMemcpy2D(o ? ly.wo : ly.wd, (size_t)cols * 2, src + r * cols * 2, (size_t)full * 2,
                      (size_t)cols * 2, (size_t)d, cudaMemcpyHostToDevice));
      return FP_OK;
    }
    case FP_W_GATE:
    case FP_W_UP: {
      // this rank's ffn rows, packed gate/up interleaved in blocks of 128 rows:
      // [g(128) | u(128)] per 256-row block, so one 256-wide GEMM tile holds matching gate and
      // up columns (SwiGLU epilogue).
      REQ(n == F * d, "weight size mismatch");
      const int half = tensor == FP_W_UP ? 1 : 0;
      const char* base = src + r * c->ffn * d * 2;
      for (int b = 0; b < c->ffn / 128; ++b)
        CK(cudaMemcpy(ly.wgu + ((size_t)b * 256 + half * 128) * d, base + (size_t)b * 128 * d * 2,
                      (size_t)128 * d * 2, cudaMemcpyHostToDevice));
      fold(c, ly.wgu, half * 128, c->ffn / 128, 256, 128, ly.ffn_g, nullptr);
      CK(cudaStreamSynchronize(c->stream));
      return FP_OK;
    }
    case FP_W_ATTN_NORM:
    case FP_W_FFN_NORM: {
      // re-fold the projection columns from the gamma folded so far to the new one (load
      // norms before projections to fold with a single rounding)
      REQ(n == d, "weight size mismatch");
      const bool attn = tensor == FP_W_ATTN_NORM;
      __nv_bfloat16* g = attn ? ly.attn_g : ly.ffn_g;
      std::vector<uint16_t> old(d);
      CK(cudaMemcpy(old.data(), g, (size_t)d * 2, cudaMemcpyDeviceToHost));
      const uint16_t* nw = static_cast<const uint16_t*>(host);
      for (long long k = 0; k < d; ++k)
        if ((old[k] & 0x7FFF) == 0 && nw[k] != old[k])
          return set_err(FP_ERR_STATE, "a zero norm weight was folded into the projection; "
                                       "reload the projection weights after this norm");
      __nv_bfloat16* gnew = nullptr;
      CK(cudaMalloc(&gnew, (size_t)d * 2));
      CK(cudaMemcpy(gnew, host, (size_t)d * 2, cudaMemcpyHostToDevice));
      if (attn) {
        fold(c, ly.wqkv, 0, 1, 0, c->qdim + 2 * c->kvdim, gnew, g);
      } else if (m.n_experts > 0) {
        fold(c, ly.wr, 0, 1, 0, m.n_experts, gnew, g);
        fold(c, ly.egu, 0, 1, 0, 2 * m.n_experts * m.moe_ffn, gnew, g);
      } else {
        fold(c, ly.wgu, 0, 1, 0, 2 * c->ffn, gnew, g);
      }
      CK(cudaMemcpyAsync(g, gnew, (size_t)d * 2, cudaMemcpyDeviceToDevice, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      cudaFree(gnew);
      return FP_OK;
    }
    case FP_W_Q_BIAS:
    case FP_W_K_BIAS:
    case FP_W_V_BIAS: {
      REQ(ly.bqkv != nullptr, "model has no qkv bias");
      const bool q = tensor == FP_W_Q_BIAS;
      REQ(n == (q ? Qd : KVd), "bias size mismatch");
      const long long rows = q ? c->qdim : c->kvdim;
      const long long off = q ? 0 : (tensor == FP_W_K_BIAS ? c->qdim : c->qdim + c->kvdim);
      return load_f32_vec(ly.bqkv + off, src + r * rows * 2, rows);
    }
    case FP_W_Q_NORM:
    case FP_W_K_NORM:
      REQ(ly.q_norm != nullptr, "model has no q/k norm");
      REQ(n == 128, "q/k norm size must be head_dim");
      return load_f32_vec(tensor == FP_W_Q_NORM ? ly.q_norm : ly.k_norm, host, n);
    case FP_W_ROUTER: {
      REQ(ly.wr != nullptr, "model has no MoE router");
      const long long E = m.n_experts;
      REQ(n == E * d, "weight size mismatch");
      CK(cudaMemcpy(ly.wr, host, (size_t)n * 2, cudaMemcpyHostToDevice));
      fold(c, ly.wr, 0, 1, 0, (int)E, ly.ffn_g, nullptr);  // fused post-attention norm
      CK(cudaStreamSynchronize(c->stream));
      return FP_OK;
    }
    case FP_W_EXPERT_GATE:
    case FP_W_EXPERT_UP: {
      // per expert: [g(128) | u(128)] per 256-row block, like the dense gate/up packing
      REQ(ly.egu != nullptr, "model has no MoE experts");
      const long long E = m.n_experts, I = m.moe_ffn;
      REQ(n == E * I * d, "weight size mismatch");
      const int half = tensor == FP_W_EXPERT_UP ? 1 : 0;
      for (long long e = 0; e < E; ++e)
        CK(cudaMemcpy2D(ly.egu + ((size_t)e * 2 * I + half * 128) * d, (size_t)256 * d * 2,
                        src + (size_t)e * I * d * 2, (size_t)128 * d * 2, (size_t)128 * d * 2,
                        (size_t)(I / 128), cudaMemcpyHostToDevice));
      fold(c, ly.egu, half * 128, (int)(E * I / 128), 256, 128, ly.ffn_g, nullptr);
      CK(cudaStreamSynchronize(c->stream));
      return FP_OK;
    }
    case FP_W_EXPERT_DOWN: {
      REQ(ly.ed != nullptr, "model has no MoE experts");
      REQ(n == (long long)m.n_experts * d * m.moe_ffn, "weight size mismatch");
      CK(cudaMemcpy(ly.ed, host, (size_t)n * 2, cudaMemcpyHostToDevice));
      return FP_OK;
    }
  }
  return set_err(FP_ERR_ARG, "unknown tensor");
}

int fp_weights_init_random(fp_ctx* c, uint64_t seed, float stdv) {
  REQ(c, "null ctx");
  CK(cudaSetDevice(c->device));
  const fp_model_cfg& m = c->cfg;
  const long long d = m.hidden;
  uint64_t s = seed * 1000003ull;
  // replicated tensors draw the same stream on every rank; shards mix in the rank
  const uint64_t shard = (uint64_t)c->tp_rank * 0x9E3779B97F4A7C15ull;
  auto fill = [&](__nv_bfloat16* p, long long n, float mean, float sd, bool sharded = false) {
    init_normal_kernel<<<1184, 256, 0, c->stream>>>(p, n, (s++) ^ (sharded ? shard : 0), mean, sd);
  };
  fill(c->embed, (long long)m.vocab * d, 0.f, stdv);
  fill(c->lm_head, (long long)m.vocab * d, 0.f, stdv);
  fill(c->final_g, d, 1.f, 0.1f);
  for (auto& ly : c->layers) {
    fill(ly.wqkv, (long long)(c->qdim + 2 * c->kvdim) * d, 0.f, stdv, true);
    fill(ly.wo, d * c->qdim, 0.f, stdv, true);
    fill(ly.attn_g, d, 1.f, 0.1f);
    fill(ly.ffn_g, d, 1.f, 0.1f);
    fold(c, ly.wqkv, 0, 1, 0, c->qdim + 2 * c->kvdim, ly.attn_g, nullptr);  // fused norms
    if (m.n_experts == 0) {
      fill(ly.wgu, 2LL * c->ffn * d, 0.f, stdv, true);
      fill(ly.wd, d * c->ffn, 0.f, stdv, true);
      fold(c, ly.wgu, 0, 1, 0, 2 * c->ffn, ly.ffn_g, nullptr);
    } else {
      const long long E = m.n_experts, I = m.moe_ffn;
      fill(ly.wr, E * d, 0.f, stdv);
      fill(ly.egu, E * 2 * I * d, 0.f, stdv);
      fill(ly.ed, E * d * I, 0.f, stdv);
      fold(c, ly.wr, 0, 1, 0, (int)E, ly.ffn_g, nullptr);
      fold(c, ly.egu, 0, 1, 0, (int)(E * 2 * I), ly.ffn_g, nullptr);
    }
    if (ly.bqkv || ly.q_norm) {
      std::vector<float> v(c->qkv_n, 0.f);
      for (int i = 0; i < c->qdim + 2 * c->kvdim; ++i) v[i] = 0.02f * (float)((int)((s * 2654435761ull + i * 40503ull) % 2001) - 1000) / 1000.f;
      if (ly.bqkv) CK(cudaMemcpy(ly.bqkv, v.data(), c->qkv_n * 4, cudaMemcpyHostToDevice));
      for (int i = 0; i < 128; ++i) v[i] = 1.f + 5.f * v[i];
      if (ly.q_norm) CK(cudaMemcpy(ly.q_norm, v.data(), 512, cudaMemcpyHostToDevice));
      if (ly.k_norm) CK(cudaMemcpy(ly.k_norm, v.data(), 512, cudaMemcpyHostToDevice));
      ++s;
    }
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c->stream));
  return FP_OK;
}

// Builds the task into *tp (set as soon as it exists, so the caller can release a partially
// built task when an allocation fails); validation failures delete it and leave *tp null.
static int task_create_impl(fp_ctx* c, const int32_t* ids, const int32_t* lens, int32_t n_seqs,
                            int32_t chunk_tokens, int32_t granularity, int32_t task_id, Task** tp) {
  REQ(c && ids && lens, "null argument");
  REQ(n_seqs >= 1, "per_request_tokens must be non-empty");  // cost_model.py:205-206
  REQ(chunk_tokens >= 0, "chunk_tokens must be >= 0");
  REQ(granularity >= 0 && granularity <= 3, "bad granularity");
  const fp_model_cfg& m = c->cfg;
  CK(cudaSetDevice(c->device));
  Task* t = new Task();
  *tp = t;
  t->id = task_id;
  t->n_seqs = n_seqs;
  t->L = m.num_layers;
  t->granularity = granularity;
  t->lens.assign(lens, lens + n_seqs);
  long long total = 0;
  for (int i = 0; i < n_seqs; ++i) {
    if (lens[i] < 1) {
      delete t;
      *tp = nullptr;
      return set_err(FP_ERR_ARG, "all token counts must be >= 1");  // cost_model.py:207-208
    }
    if (lens[i] > m.max_pos) {
      delete t;
      *tp = nullptr;
      return set_err(FP_ERR_ARG, "request longer than max_pos");
    }
    total += lens[i];
  }
  t->total = (int)total;
  if (c->tp_size > 1) {
    const long long max_chunk = (chunk_tokens == 0 || chunk_tokens >= total) ? total : chunk_tokens;
    const char* why = !c->tp_connected ? "tensor-parallel context is not connected to its peers"
                      : max_chunk > c->tp_host.part_rows
                          ? "chunk exceeds the tensor-parallel exchange capacity (use chunk_tokens)"
                          : nullptr;
    if (why) {
      delete t;
      *tp = nullptr;
      return set_err(FP_ERR_STATE, why);
    }
  }
  for (long long i = 0; i < total; ++i)
    if (ids[i] < 0 || ids[i] >= m.vocab) {
      delete t;
      *tp = nullptr;
      return set_err(FP_ERR_ARG, "token id out of range");
    }
  // pages
  const int PS = c->page_size;
  std::vector<int> npages(n_seqs);
  int need = 0, maxp = 0;
  for (int i = 0; i < n_seqs; ++i) {
    npages[i] = (lens[i] + PS - 1) / PS;
    need += npages[i];
    maxp = std::max(maxp, npages[i]);
  }
  {
    std::lock_guard<std::mutex> lk(c->page_mu);
    if ((int)c->free_pages.size() < need) {
      delete t;
      *tp = nullptr;
      return set_err(FP_ERR_NOMEM, "KV page pool exhausted");
    }
    for (int i = 0; i < need; ++i) {
      t->pages.push_back(c->free_pages.back());
      c->free_pages.pop_back();
    }
  }
  t->bt_stride = maxp;
  std::vector<int> bt((size_t)n_seqs * maxp, 0);
  {
    int k = 0;
    for (int i = 0; i < n_seqs; ++i)
      for (int j = 0; j < npages[i]; ++j) bt[(size_t)i * maxp + j] = t->pages[k++];
  }
  // chunk plan: cost_model.py:212-233 (requests concatenated, chunks over the stream)
  std::vector<long long> starts(n_seqs + 1, 0);
  for (int i = 0; i < n_seqs; ++i) starts[i + 1] = starts[i] + lens[i];
  std::vector<std::pair<long long, long long>> bounds;
  if (chunk_tokens == 0 || chunk_tokens >= total) bounds.push_back({0, total});
  else
    for (long long lo = 0; lo < total; lo += chunk_tokens)
      bounds.push_back({lo, std::min(lo + chunk_tokens, total)});
  std::vector<int> pos(total), tpage(total), last_rows;
  std::vector<AttnTile> items;
  for (int i = 0; i < n_seqs; ++i)
    for (int p = 0; p < lens[i]; ++p) {
      pos[starts[i] + p] = p;
      tpage[starts[i] + p] = bt[(size_t)i * maxp + p / PS];
    }
  for (auto& b : bounds) {
    ChunkPlan ch{};
    const long long s = b.first, e = b.second;
    ch.M = (int)(e - s);
    ch.tok0 = (int)s;
    ch.item0 = (int)items.size();
    ch.last0 = (int)last_rows.size();
    ch.seq0 = -1;
    std::vector<AttnTile> its;
    for (int r = 0; r < n_seqs; ++r) {
      const long long r0 = starts[r], r1 = starts[r + 1];
      const long long share = std::min(e, r1) - std::max(s, r0);
      if (share <= 0) continue;
      const long long prefix = std::min(std::max(s - r0, 0LL), (long long)lens[r]);
      const int row0 = (int)(std::max(s, r0) - s);
      ch.attn_flops += 4.0 * c->qdim * ((double)share * prefix + (double)share * (share + 1) / 2.0);
      for (long long k = 0; k < share; k += 128) {
        AttnTile it;
        it.q_row0 = row0 + (int)k;
        it.n_rows = (int)std::min(128LL, share - k);
        it.q_pos0 = (int)(prefix + k);
        it.req = r;
        its.push_back(it);
      }
      if (r1 - 1 >= s && r1 - 1 < e) {  // request completes in this chunk
        if (ch.seq0 < 0) ch.seq0 = r;
        last_rows.push_back((int)(r1 - 1 - s));
      }
    }
    std::stable_sort(its.begin(), its.end(), [](const AttnTile& a, const AttnTile& b) {
      return a.q_pos0 + a.n_rows > b.q_pos0 + b.n_rows;  // longest KV range first
    });
    items.insert(items.end(), its.begin(), its.end());
    ch.n_items = (int)items.size() - ch.item0;
    ch.n_last = (int)last_rows.size() - ch.last0;
    if (ch.seq0 < 0) ch.seq0 = 0;
    t->max_m = std::max(t->max_m, ch.M);
    t->chunks.push_back(ch);
  }
  t->n_entries = (int)t->chunks.size() * m.num_layers * 5;
  // device metadata, one allocation
  const size_t n_ids = total, n_items = items.size(), n_bt = bt.size(), n_last = last_rows.size();
  const size_t bytes = (3 * n_ids + n_bt + n_last) * 4 + n_items * sizeof(AttnTile) + 64;
  std::vector<char> host(bytes, 0);
  size_t o = 0;
  auto put = [&](const void* src, size_t nb) {
    size_t at = o;
    if (nb) memcpy(host.data() + o, src, nb);
    o += (nb + 15) & ~size_t(15);
    return at;
  };
  host.resize(bytes + 6 * 16);
  const size_t o_ids = put(ids, n_ids * 4), o_pos = put(pos.data(), n_ids * 4),
               o_tp = put(tpage.data(), n_ids * 4), o_it = put(items.data(), n_items * sizeof(AttnTile)),
               o_bt = put(bt.data(), n_bt * 4), o_last = put(last_rows.data(), n_last * 4);
  // Stream-ordered allocation + upload on the upload stream, from a pinned staging arena, so
  // building a task never waits behind the running task's kernels.
  cudaStream_t up = c->upload;
  {
    std::lock_guard<std::mutex> lk(c->stage_mu);
    if (c->stage_ev) CK(cudaEventSynchronize(c->stage_ev));  // previous upload drained
    if (c->stage_cap < o) {
      if (c->stage) cudaFreeHost(c->stage);
      c->stage_cap = std::max<size_t>(o, 1 << 20);
      CK(cudaHostAlloc(&c->stage, c->stage_cap, cudaHostAllocDefault));
    }
    memcpy(c->stage, host.data(), o);
    CK(cudaMallocAsync((void**)&t->meta, o + 16, up));
    CK(cudaMemcpyAsync(t->meta, c->stage, o, cudaMemcpyHostToDevice, up));
    if (!c->stage_ev) CK(cudaEventCreateWithFlags(&c->stage_ev, cudaEventDisableTiming));
    CK(cudaEventRecord(c->stage_ev, up));
  }
  t->upload_bytes = (long long)o;
  t->d_ids = reinterpret_cast<int*>(t->meta + o_ids);
  t->d_pos = reinterpret_cast<int*>(t->meta + o_pos);
  t->d_tpage = reinterpret_cast<int*>(t->meta + o_tp);
  t->d_items = reinterpret_cast<AttnTile*>(t->meta + o_it);
  t->d_bt = reinterpret_cast<int*>(t->meta + o_bt);
  t->d_last = reinterpret_cast<int*>(t->meta + o_last);
  // workspaces (resume state lives here: h + the live intermediate)
  const long long M = t->max_m, d = m.hidden;
  CK(cudaMallocAsync((void**)&t->h, M * d * 2, up));
  CK(cudaMallocAsync((void**)&t->ssq, M * (d / 128) * 4, up));
  CK(cudaMallocAsync((void**)&t->q, M * c->qdim * 2, up));
  CK(cudaMallocAsync((void**)&t->ao, M * c->qdim * 2, up));
  if (m.n_experts == 0) CK(cudaMallocAsync((void**)&t->act, M * (long long)c->ffn * 2, up));
  CK(cudaMallocAsync((void**)&t->xf, (long long)n_seqs * d * 2, up));
  CK(cudaMallocAsync((void**)&t->logits, (long long)n_seqs * c->vocab_pad * 4, up));
  CK(cudaMemsetAsync(t->logits, 0, (long long)n_seqs * c->vocab_pad * 4, up));
  // decision slots, then the per-entry GO timestamps (entry durations for the blocking bound)
  const size_t stamp_off = (sizeof(TaskCtl) + (size_t)t->n_entries * 4 + 15) & ~(size_t)15;
  const size_t ctl_bytes = stamp_off + (size_t)t->n_entries * 16;
  CK(cudaMallocAsync((void**)&t->ctl, ctl_bytes, up));
  CK(cudaMemsetAsync(t->ctl, 0, ctl_bytes, up));
  CK(cudaMemsetAsync(&t->ctl->stopped_gen, 0xFF, 4, up));  // -1
  t->stamps = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(t->ctl) + stamp_off);
  CK(cudaMemcpyAsync(&t->ctl->stamps, &t->stamps, sizeof(t->stamps), cudaMemcpyHostToDevice, up));
  int rc;
  if ((rc = make_map(&t->tm_h, t->h, M, d, 128))) return rc;
  if ((rc = make_map(&t->tm_ao, t->ao, M, c->qdim, 128))) return rc;
  if ((rc = make_map(&t->tm_h32, t->h, M, d, 32))) return rc;
  if ((rc = make_map(&t->tm_ao32, t->ao, M, c->qdim, 32))) return rc;
  if (m.n_experts == 0) {
    if ((rc = make_map(&t->tm_act, t->act, M, c->ffn, 128))) return rc;
    if ((rc = make_map(&t->tm_act32, t->act, M, c->ffn, 32))) return rc;
  } else {
    // MoE: router logits, routing index arrays (one allocation, zeroed: the histogram and the
    // scatter cursors must start at 0), expert-ordered rows
    const long long E = m.n_experts, K = m.top_k, I = m.moe_ffn, R = M * K;
    const long long max_mt = R / 128 + E + 1;
    CK(cudaMallocAsync((void**)&t->rlog, M * 256 * 4, up));
    const size_t n_int = (size_t)(3 * M * K + 2 * E + (E + 1) + 1 + 2 * max_mt + R + 8);
    CK(cudaMallocAsync((void**)&t->moe_meta, n_int * 4, up));
    CK(cudaMemsetAsync(t->moe_meta, 0, n_int * 4, up));
    int* q = reinterpret_cast<int*>(t->moe_meta);
    t->m_ids = q;
    q += M * K;
    t->m_w = reinterpret_cast<float*>(q);
    q += M * K;
    t->m_slot = q;
    q += M * K;
    t->m_counts = q;
    q += E;
    t->m_cursor = q;
    q += E;
    t->m_off = q;
    q += E + 1;
    t->m_mtc = q;
    q += 1;
    q += (reinterpret_cast<uintptr_t>(q) & 7) ? 1 : 0;  // int2 alignment
    t->m_mtiles = reinterpret_cast<int2*>(q);
    q += 2 * max_mt;
    t->m_perm = q;
    CK(cudaMallocAsync((void**)&t->xperm, R * d * 2, up));
    CK(cudaMallocAsync((void**)&t->actp, R * I * 2, up));
    CK(cudaMallocAsync((void**)&t->yperm, R * d * 2, up));
    if ((rc = make_map(&t->tm_xperm, t->xperm, R, d, 128))) return rc;
    if ((rc = make_map(&t->tm_actp, t->actp, R, I, 128))) return rc;
  }
  if ((rc = make_map(&t->tm_xf, t->xf, n_seqs, d, 128))) return rc;
  if ((rc = make_map(&t->tm_xf32, t->xf, n_seqs, d, 32))) return rc;
  if ((rc = make_map(&t->tm_q, t->q, M, c->qdim, 128))) return rc;
  CK(cudaEventCreateWithFlags(&t->ready, cudaEventDisableTiming));
  CK(cudaEventRecord(t->ready, up));
  CK(cudaEventCreateWithFlags(&t->done, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&t->fence, cudaEventDisableTiming));
  CK(cudaEventRecord(t->fence, up));
  return FP_OK;
}

// A task whose creation failed part-way: nothing of it was launched; drain its uploads, free
// what was allocated and return its KV pages (no leak when the device runs out of memory).
static void task_release_partial(fp_ctx* c, Task* t) {
  cudaStreamSynchronize(c->upload);
  void* bufs[] = {t->meta, t->h, t->ssq, t->q, t->ao, t->act, t->rlog, t->moe_meta,
                  t->xperm, t->actp, t->yperm, t->xf, t->logits, t->ctl};
  for (void* b : bufs)
    if (b) cudaFreeAsync(b, c->upload);
  cudaStreamSynchronize(c->upload);
  for (cudaEvent_t e : {t->ready, t->done, t->fence})
    if (e) cudaEventDestroy(e);
  {
    std::lock_guard<std::mutex> lk(c->page_mu);
    for (int p : t->pages) c->free_pages.push_back(p);
  }
  delete t;
}

int fp_task_create(fp_ctx* c, const int32_t* ids, const int32_t* lens, int32_t n_seqs,
                   int32_t chunk_tokens, int32_t granularity, int32_t task_id, fp_task** out) {
  REQ(out, "null argument");
  Task* t = nullptr;
  const int rc = task_create_impl(c, ids, lens, n_seqs, chunk_tokens, granularity, task_id, &t);
  if (rc != FP_OK) {
    if (t) task_release_partial(c, t);
    cudaGetLastError();  // a failed allocation must not surface in a later, unrelated check
    return rc;
  }
  *out = reinterpret_cast<fp_task*>(t);
  return FP_OK;
}

int fp_task_info(const fp_task* task, fp_task_info_t* info) {
  const Task* t = reinterpret_cast<const Task*>(task);
  REQ(t && info, "null argument");
  info->n_entries = t->n_entries;
  info->n_chunks = (int)t->chunks.size();
  info->n_seqs = t->n_seqs;
  info->total_tokens = t->total;
  info->max_chunk_tokens = t->max_m;
  info->n_pages = (int)t->pages.size();
  info->upload_bytes = t->upload_bytes;
  return FP_OK;
}

int fp_task_num_entries(const fp_task* task) {
  return reinterpret_cast<const Task*>(task)->n_entries;
}

int fp_task_entry_info(const fp_task* task, int32_t e, int32_t* chunk, int32_t* layer,
                       int32_t* op, int32_t* new_tokens) {
  const Task* t = reinterpret_cast<const Task*>(task);
  REQ(t && e >= 0 && e < t->n_entries, "entry out of range");
  const int ci = e / (5 * t->L);
  if (chunk) *chunk = ci;
  if (layer) *layer = (e / 5) % t->L;
  if (op) *op = e % 5;
  if (new_tokens) *new_tokens = t->chunks[ci].M;
  return FP_OK;
}

int fp_task_entry_stamps(fp_ctx* c, fp_task* task, uint64_t* host_out) {
  Task* t = reinterpret_cast<Task*>(task);
  REQ(c && t && host_out, "null argument");
  CK(cudaSetDevice(c->device));
  // a snapshot: entries still running publish their stamps later
  CK(cudaMemcpyAsync(host_out, t->stamps, (size_t)t->n_entries * 16, cudaMemcpyDeviceToHost,
                     c->readback));
  CK(cudaStreamSynchronize(c->readback));
  return FP_OK;
}

int fp_task_destroy(fp_ctx* c, fp_task* task) {
  Task* t = reinterpret_cast<Task*>(task);
  if (!t) return FP_OK;
  REQ(c, "null ctx");
  CK(cudaSetDevice(c->device));
  while (t->worker_active.load()) std::this_thread::yield();
  // Stream-ordered frees behind this task's last launch (t->fence: queued no-op launches of a
  // stopped segment included), on a stream of their own: freed on the prefill stream they
  // would wait for every task enqueued after this one, and the pool would make the next task's
  // allocations (upload stream) wait for those too.
  cudaStream_t st = c->release;
  {
    std::lock_guard<std::mutex> lk(c->launch_mu);
    cudaStreamWaitEvent(st, t->ready, 0);
    cudaStreamWaitEvent(st, t->fence, 0);
    cudaFreeAsync(t->meta, st);
    cudaFreeAsync(t->h, st);
    cudaFreeAsync(t->ssq, st);
    cudaFreeAsync(t->q, st);
    cudaFreeAsync(t->ao, st);
    cudaFreeAsync(t->act, st);
    cudaFreeAsync(t->rlog, st);
    cudaFreeAsync(t->moe_meta, st);
    cudaFreeAsync(t->xperm, st);
    cudaFreeAsync(t->actp, st);
    cudaFreeAsync(t->yperm, st);
    cudaFreeAsync(t->xf, st);
    cudaFreeAsync(t->logits, st);
    cudaFreeAsync(t->ctl, st);
  }
  cudaEventDestroy(t->ready);
  cudaEventDestroy(t->done);
  cudaEventDestroy(t->fence);
  {
    std::lock_guard<std::mutex> lk(c->page_mu);
    for (int p : t->pages) c->free_pages.push_back(p);
  }
  delete t;
  return FP_OK;
}

int fp_task_begin_segment(fp_ctx* c, fp_task* task, int32_t first) {
  Task* t = reinterpret_cast<Task*>(task);
  REQ(c && t, "null argument");
  REQ(first >= 0 && first < t->n_entries, "segment start out of range");
  // a stopped segment's launch worker exits on its own once it observes the ACK
  for (int spin = 0; t->worker_active.load(); ++spin) {
    if (spin > 20000000) return set_err(FP_ERR_STATE, "task is already running");
    std::this_thread::yield();
  }
  std::lock_guard<std::mutex> lk(c->launch_mu);
  t->gen += 1;
  t->seg_first = first;
  t->enq = first;
  t->done_recorded = 0;
  t->seg_ack0 = c->hctl->ack_seq;
  CK(cudaStreamWaitEvent(c->stream, t->ready, 0));
  CK(cudaMemsetAsync(&t->ctl->dec[first], 0, (size_t)(t->n_entries - first) * 4, c->stream));
  CK(cudaEventRecord(t->fence, c->stream));
  return FP_OK;
}

int fp_task_enqueue(fp_ctx* c, fp_task* task, int32_t first, int32_t last) {
  Task* t = reinterpret_cast<Task*>(task);
  REQ(c && t, "null argument");
  REQ(first >= t->seg_first && first <= last && last <= t->n_entries, "bad entry range");
  CK(cudaSetDevice(c->device));
  std::lock_guard<std::mutex> lk(c->launch_mu);
  for (int e = first; e < last; ++e) {
    int rc = launch_entry_checked(c, t, e);
    if (rc) return rc;
  }
  t->enq = std::max(t->enq, (int)last);
  if (last == t->n_entries) {
    CK(cudaEventRecord(t->done, c->stream));
    t->done_recorded = 1;
  }
  CK(cudaEventRecord(t->fence, c->stream));
  CK(cudaGetLastError());
  return FP_OK;
}

int fp_task_start(fp_ctx* c, fp_task* task, int32_t first) {
  Task* t = reinterpret_cast<Task*>(task);
  REQ(c && !c->tp_lockstep, "lock-step tensor-parallel groups launch through fp_tp_enqueue_lockstep");
  int rc = fp_task_begin_segment(c, task, first);
  if (rc) return rc;
  for (int spin = 0;; ++spin) {  // a stopped segment's worker is still winding down
    std::lock_guard<std::mutex> lk(c->wmu);
    if (c->wtask == nullptr) {
      t->worker_active.store(1);
      c->wtask = t;
      break;
    }
    if (spin > 20000000) return set_err(FP_ERR_STATE, "pool occupied");
  }
  c->wcv.notify_all();
  return FP_OK;
}

int fp_task_poll(fp_ctx* c, fp_task* task, fp_task_status* st) {
  Task* t = reinterpret_cast<Task*>(task);
  REQ(c && t && st, "null argument");
  if (int e = t->err.load()) return set_err(e, "async launch failed: " + t->err_msg);
  st->generation = t->gen;
  st->enqueued = t->enq;
  const int ack_seq = c->hctl->ack_seq;
  const bool stopped = ack_seq != t->seg_ack0 && c->hctl->ack_task == t->id;
  if (stopped) {
    st->state = FP_TASK_STOPPED;
    st->cursor = c->hctl->ack_entry;
    return FP_OK;
  }
  if (t->done_recorded && !t->worker_active.load()) {
    cudaError_t q = cudaEventQuery(t->done);
    if (q == cudaSuccess) {
      // re-check the ACK after the event: a stop in the last launched entries wins
      if (c->hctl->ack_seq != t->seg_ack0 && c->hctl->ack_task == t->id) {
        st->state = FP_TASK_STOPPED;
        st->cursor = c->hctl->ack_entry;
      } else {
        st->state = FP_TASK_DONE;
        st->cursor = t->n_entries;
      }
      return FP_OK;
    }
    if (q != cudaErrorNotReady) CK(q);
  }
  st->state = FP_TASK_RUNNING;
  st->cursor = (c->hctl->progress_task == t->id) ? (int)c->hctl->progress_entry : t->seg_first;
  return FP_OK;
}

int fp_signal(fp_ctx* c) {
  REQ(c, "null ctx");
  c->hctl->signal = 1;
  return FP_OK;
}
int fp_clear(fp_ctx* c) {
  REQ(c, "null ctx");
  c->hctl->signal = 0;
  return FP_OK;
}
int fp_poll(fp_ctx* c, fp_status* s) {
  REQ(c && s, "null argument");
  s->ack_seq = c->hctl->ack_seq;
  s->ack_task = c->hctl->ack_task;
  s->ack_entry = c->hctl->ack_entry;
  s->progress_task = c->hctl->progress_task;
  s->progress_entry = c->hctl->progress_entry;
  s->signal = c->hctl->signal;
  s->ack_ns = c->hctl->ack_ns;
  return FP_OK;
}

int fp_task_logits(fp_ctx* c, fp_task* task, float* host_out) {
  Task* t = reinterpret_cast<Task*>(task);
  REQ(c && t && host_out, "null argument");
  CK(cudaSetDevice(c->device));
  // wait for THIS task only (its completion event), so a serving loop reads finished requests
  // while later tasks still run on the prefill stream
  if (t->done_recorded) CK(cudaEventSynchronize(t->done));
  else CK(cudaStreamSynchronize(c->stream));
  CK(cudaMemcpy2DAsync(host_out, (size_t)c->cfg.vocab * 4, t->logits, (size_t)c->vocab_pad * 4,
                       (size_t)c->cfg.vocab * 4, t->n_seqs, cudaMemcpyDeviceToHost, c->readback));
  CK(cudaStreamSynchronize(c->readback));
  return FP_OK;
}

int fp_task_read_routing(fp_ctx* c, fp_task* task, int32_t* ids, float* w, int32_t max_rows) {
  Task* t = reinterpret_cast<Task*>(task);
  REQ(c && t && ids && w, "null argument");
  REQ(c->cfg.n_experts > 0, "not a MoE model");
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  const int rows = std::min(t->moe_rows, (int)max_rows);
  const size_t n = (size_t)rows * c->cfg.top_k;
  CK(cudaMemcpy(ids, t->m_ids, n * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(w, t->m_w, n * 4, cudaMemcpyDeviceToHost));
  return rows;
}

int fp_task_read_kv(fp_ctx* c, fp_task* task, int32_t seq, int32_t layer, void* hk, void* hv) {
  Task* t = reinterpret_cast<Task*>(task);
  REQ(c && t && hk && hv, "null argument");
  REQ(seq >= 0 && seq < t->n_seqs && layer >= 0 && layer < c->cfg.num_layers, "bad seq/layer");
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  const int PS = c->page_size, H = c->hkv, n = t->lens[seq];
  int page_base = 0;
  for (int i = 0; i < seq; ++i) page_base += (t->lens[i] + PS - 1) / PS;
  std::vector<__nv_bfloat16> page((size_t)c->page_elems);
  __nv_bfloat16* ok = static_cast<__nv_bfloat16*>(hk);
  __nv_bfloat16* ov = static_cast<__nv_bfloat16*>(hv);
  const __nv_bfloat16* kvl = c->kv + (long long)layer * c->kv_pages * c->page_elems;
  for (int j = 0; j * PS < n; ++j) {
    const int pg = t->pages[page_base + j];
    CK(cudaMemcpy(page.data(), kvl + (long long)pg * c->page_elems, c->page_elems * 2,
                  cudaMemcpyDeviceToHost));
    for (int s = 0; s < PS && j * PS + s < n; ++s)
      for (int h = 0; h < H; ++h)
        for (int kv = 0; kv < 2; ++kv) {
          const __nv_bfloat16* src = page.data() + ((size_t)(kv * H + h) * PS + s) * 128;
          __nv_bfloat16* dst = (kv ? ov : ok) + ((size_t)(j * PS + s) * H + h) * 128;
          memcpy(dst, src, 256);
        }
  }
  return FP_OK;
}

int fp_prof_enable(fp_ctx* c, int32_t on) {
  REQ(c, "null ctx");
  std::lock_guard<std::mutex> lk(c->launch_mu);
  c->prof_on = on != 0;
  return FP_OK;
}

int fp_prof_collect(fp_ctx* c, fp_prof_rec* out, int32_t max, int32_t* n) {
  REQ(c && n, "null argument");
  CK(cudaSetDevice(c->device));
  std::lock_guard<std::mutex> lk(c->launch_mu);
  CK(cudaStreamSynchronize(c->stream));
  const int cnt = (int)c->prof_meta.size();
  *n = cnt;
  for (int i = 0; i < cnt; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->prof_ev[i].first, c->prof_ev[i].second);
    if (out && i < max) {
      out[i] = c->prof_meta[i];
      out[i].ms = ms;
    }
    c->ev_pool.push_back(c->prof_ev[i].first);
    c->ev_pool.push_back(c->prof_ev[i].second);
  }
  c->prof_meta.clear();
  c->prof_ev.clear();
  return FP_OK;
}

int fp_ctx_launch_count(fp_ctx* c, int64_t* n) {
  REQ(c && n, "null argument");
  *n = c->launches.load();
  return FP_OK;
}

int fp_op_gemm(fp_ctx* c, int32_t epi, const void* A, const void* B, void* C, int32_t M,
               int32_t N, int32_t K) {
  REQ(c && A && B && C, "null argument");
  REQ(M >= 1 && N % 256 == 0 && K % 64 == 0, "gemm: N%256 and K%64 required");
  CK(cudaSetDevice(c->device));
  CUtensorMap ta, tb;
  int rc;
  CUtensorMap ta32;
  if ((rc = make_map(&ta, A, M, K, 128))) return rc;
  if ((rc = make_map(&ta32, A, M, K, 32))) return rc;
  if ((rc = make_map(&tb, B, N, K, 128))) return rc;
  GemmParams p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.out = C;
  p.ldo = N;
  p.resid = static_cast<__nv_bfloat16*>(C);
  p.ldr = N;
  std::lock_guard<std::mutex> lk(c->launch_mu);
  if (c->gemm_dbg) {
    CK(cudaMemsetAsync(c->gemm_dbg, 0, (size_t)4096 * 16 * sizeof(unsigned long long), c->stream));
    p.dbg = c->gemm_dbg;
  }
  if (epi == 0) launch_gemm<EPI_STORE_BF16>(c, ta, tb, p, c->stream, &ta32);
  else if (epi == 1) launch_gemm<EPI_STORE_F32>(c, ta, tb, p, c->stream, &ta32);
  else if (epi == 2) launch_gemm<EPI_RESID>(c, ta, tb, p, c->stream, &ta32);
  else if (epi == 3) {  // SwiGLU over B already packed [gate(128) | up(128)] per 256 rows
    p.ldo = N / 2;
    launch_gemm<EPI_SWIGLU>(c, ta, tb, p, c->stream, &ta32);
  } else return set_err(FP_ERR_ARG, "bad epilogue");
  CK(cudaGetLastError());
  return FP_OK;
}

int fp_op_gate_up_swiglu(fp_ctx* c, const void* x, const void* w_gate, const void* w_up,
                         void* out, int32_t M, int32_t F, int32_t K) {
  REQ(c && x && w_gate && w_up && out, "null argument");
  REQ(M >= 1 && F % 128 == 0 && K % 64 == 0, "gate_up: F%128 and K%64 required");
  CK(cudaSetDevice(c->device));
  std::lock_guard<std::mutex> lk(c->launch_mu);
  // pack [g(128) | u(128)] per 256-row block, the layout of the model's gate/up weights
  __nv_bfloat16* w = nullptr;
  CK(cudaMallocAsync((void**)&w, (size_t)2 * F * K * 2, c->stream));
  for (int half = 0; half < 2; ++half)
    CK(cudaMemcpy2DAsync(w + (size_t)half * 128 * K, (size_t)256 * K * 2, half ? w_up : w_gate,
                         (size_t)128 * K * 2, (size_t)128 * K * 2, (size_t)(F / 128),
                         cudaMemcpyDeviceToDevice, c->stream));
  CUtensorMap ta, tb;
  int rc;
  CUtensorMap ta32;
  if ((rc = make_map(&ta, x, M, K, 128)) || (rc = make_map(&ta32, x, M, K, 32)) ||
      (rc = make_map(&tb, w, 2 * F, K, 128))) {
    cudaFreeAsync(w, c->stream);
    return rc;
  }
  GemmParams p{};
  p.M = M;
  p.N = 2 * F;
  p.K = K;
  p.out = out;
  p.ldo = F;
  launch_gemm<EPI_SWIGLU>(c, ta, tb, p, c->stream, &ta32);
  CK(cudaGetLastError());
  CK(cudaFreeAsync(w, c->stream));
  return FP_OK;
}

int fp_op_qkv_rope_kv(fp_ctx* c, const void* x, const void* w_qkv, void* q_out, void* kv_pages,
                      const int32_t* positions, const int32_t* tok_page, int32_t M, int32_t q_cols,
                      int32_t kv_cols, int32_t K) {
  REQ(c && x && w_qkv && q_out && kv_pages && positions && tok_page, "null argument");
  REQ(M >= 1 && K % 64 == 0 && q_cols % 128 == 0 && kv_cols % 128 == 0 && kv_cols > 0,
      "qkv op: K%64, q_cols%128 and kv_cols%128 required");
  CK(cudaSetDevice(c->device));
  std::lock_guard<std::mutex> lk(c->launch_mu);
  // weight rows padded to a multiple of 256 with zeros (the model's qkv layout)
  const int n = q_cols + 2 * kv_cols, N = (n + 255) / 256 * 256;
  __nv_bfloat16* w = nullptr;
  CK(cudaMallocAsync((void**)&w, (size_t)N * K * 2, c->stream));
  CK(cudaMemsetAsync(w, 0, (size_t)N * K * 2, c->stream));
  CK(cudaMemcpyAsync(w, w_qkv, (size_t)n * K * 2, cudaMemcpyDeviceToDevice, c->stream));
  CUtensorMap ta, tb;
  int rc;
  CUtensorMap ta32;
  if ((rc = make_map(&ta, x, M, K, 128)) || (rc = make_map(&ta32, x, M, K, 32)) ||
      (rc = make_map(&tb, w, N, K, 128))) {
    cudaFreeAsync(w, c->stream);
    return rc;
  }
  GemmParams p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.pos = positions;
  p.tok_page = tok_page;
  p.qbuf = static_cast<__nv_bfloat16*>(q_out);
  p.ldq = q_cols;
  p.kv_layer = static_cast<__nv_bfloat16*>(kv_pages);
  p.rope = c->rope;
  p.q_cols = q_cols;
  p.kv_cols = kv_cols;
  p.page_size = c->page_size;
  p.n_kv_heads = kv_cols / 128;
  p.norm_eps = c->cfg.rms_eps;
  launch_gemm<EPI_QKV>(c, ta, tb, p, c->stream, &ta32);
  CK(cudaGetLastError());
  CK(cudaFreeAsync(w, c->stream));
  return FP_OK;
}

int fp_op_attn_prefill(fp_ctx* c, const void* q, const void* k, const void* v, void* out,
                       int32_t n_q, int32_t kv_len) {
  REQ(c && q && k && v && out, "null argument");
  REQ(n_q >= 1 && kv_len >= n_q, "attn: need 1 <= n_q <= kv_len");
  REQ(c->tp_size == 1, "attn op: single-rank contexts only");
  CK(cudaSetDevice(c->device));
  const int PS = c->page_size, H = c->hkv, npages = (kv_len + PS - 1) / PS;
  std::vector<int> pages;
  {
    std::lock_guard<std::mutex> lk(c->page_mu);
    REQ((int)c->free_pages.size() >= npages, "KV page pool exhausted");
    for (int i = 0; i < npages; ++i) {
      pages.push_back(c->free_pages.back());
      c->free_pages.pop_back();
    }
  }
  std::lock_guard<std::mutex> lk(c->launch_mu);
  cudaStream_t st = c->stream;
  // K / V rows [kv_len, H * 128] into layer 0's pages: [page][k|v][head][slot][128]
  for (int pg = 0; pg < npages; ++pg) {
    const int rows = std::min(PS, kv_len - pg * PS);
    for (int kv = 0; kv < 2; ++kv)
      for (int h = 0; h < H; ++h) {
        __nv_bfloat16* dst = c->kv + (((long long)pages[pg] * 2 + kv) * H + h) * PS * 128;
        const char* src = static_cast<const char*>(kv ? v : k) +
                          ((long long)pg * PS * H * 128 + (long long)h * 128) * 2;
        CK(cudaMemcpy2DAsync(dst, 256, src, (size_t)H * 256, 256, rows, cudaMemcpyDeviceToDevice,
                             st));
      }
  }
  // the query rows are the request's last n_q tokens (prefix = kv_len - n_q)
  std::vector<AttnTile> items;
  for (int r0 = 0; r0 < n_q; r0 += 128)
    items.push_back({r0, std::min(128, n_q - r0), kv_len - n_q + r0, 0});
  std::stable_sort(items.begin(), items.end(), [](const AttnTile& a, const AttnTile& b) {
    return a.q_pos0 + a.n_rows > b.q_pos0 + b.n_rows;
  });
  const size_t bytes = items.size() * sizeof(AttnTile) + pages.size() * 4;
  char* meta = nullptr;
  CK(cudaMallocAsync((void**)&meta, bytes, st));
  CK(cudaMemcpyAsync(meta, items.data(), items.size() * sizeof(AttnTile), cudaMemcpyHostToDevice,
                     st));
  CK(cudaMemcpyAsync(meta + items.size() * sizeof(AttnTile), pages.data(), pages.size() * 4,
                     cudaMemcpyHostToDevice, st));
  CUtensorMap tq, to;
  int rc = make_map(&tq, q, n_q, c->qdim, 128);
  if (rc == FP_OK) rc = make_map(&to, out, n_q, c->qdim, 128);
  if (rc == FP_OK) {
    AttnTcParams a{};
    a.items = reinterpret_cast<const AttnTile*>(meta);
    a.n_items = (int)items.size();
    a.n_heads = c->hq;
    a.n_kv_heads = c->hkv;
    a.pairs_per_kv = (c->hq / c->hkv + 1) / 2;
    a.out = static_cast<__nv_bfloat16*>(out);
    a.ldo = c->qdim;
    a.block_table = reinterpret_cast<const int*>(meta + items.size() * sizeof(AttnTile));
    a.bt_stride = npages;
    a.kv_row_layer = 0;
    a.kv_rows_per_page = 2 * H * PS;
    a.scale_log2 = 1.4426950408889634f / sqrtf(128.f);
    a.sched = c->attn_sched;
    a.dbg = c->gemm_dbg;
    launch_attn(c, tq, c->tm_kv, to, a, st);
  }
  CK(cudaFreeAsync(meta, st));
  CK(cudaStreamSynchronize(st));
  {
    std::lock_guard<std::mutex> lk2(c->page_mu);
    for (int pg : pages) c->free_pages.push_back(pg);
  }
  CK(cudaGetLastError());
  return rc;
}

int fp_op_rmsnorm(fp_ctx* c, const void* x, const void* gamma, void* out, int32_t M, int32_t d,
                  float eps) {
  REQ(c && x && gamma && out, "null argument");
  CK(cudaSetDevice(c->device));
  RmsParams r{};
  r.M = M;
  r.d = d;
  r.src = static_cast<const __nv_bfloat16*>(x);
  r.ld_src = d;
  r.gamma = static_cast<const __nv_bfloat16*>(gamma);
  r.out = static_cast<__nv_bfloat16*>(out);
  r.ld_out = d;
  r.eps = eps;
  std::lock_guard<std::mutex> lk(c->launch_mu);
  int rc = launch_rms(r, c->stream);
  if (rc) return rc;
  CK(cudaGetLastError());
  return FP_OK;
}

// ---- tensor parallelism -----------------------------------------------------------------
static size_t tp_header_bytes() { return (sizeof(TpShared) + 4095) / 4096 * 4096; }

static int tp_alloc_block(fp_ctx* c, int64_t max_tokens) {
  if (c->tp_block) {
    REQ(c->tp_host.part_rows == max_tokens, "exchange already allocated with another capacity");
    return FP_OK;
  }
  const size_t part = (size_t)max_tokens * c->cfg.hidden * 2;
  CK(cudaSetDevice(c->device));
  CK(cudaMalloc(&c->tp_block, tp_header_bytes() + 2 * part));
  CK(cudaMemset(c->tp_block, 0, tp_header_bytes()));
  CK(cudaMalloc(&c->tp_local, sizeof(TpLocal)));
  CK(cudaMemset(c->tp_local, 0, sizeof(TpLocal)));
  c->tp_host.part_rows = max_tokens;
  return FP_OK;
}

// bases[r] = rank r's exchange block as addressable from this context's device
static int tp_finish(fp_ctx* c, char* const* bases) {
  TpDev& d = c->tp_host;
  d.rank = c->tp_rank;
  d.size = c->tp_size;
  d.local = c->tp_local;
  const size_t part = (size_t)d.part_rows * c->cfg.hidden * 2;
  for (int r = 0; r < c->tp_size; ++r) {
    d.peer[r] = reinterpret_cast<TpShared*>(bases[r]);
    for (int b = 0; b < 2; ++b)
      d.part[r][b] = reinterpret_cast<__nv_bfloat16*>(bases[r] + tp_header_bytes() + b * part);
  }
  CK(cudaSetDevice(c->device));
  if (!c->d_tp) CK(cudaMalloc(&c->d_tp, sizeof(TpDev)));
  CK(cudaMemcpy(c->d_tp, &d, sizeof(TpDev), cudaMemcpyHostToDevice));
  c->tp_connected = true;
  return FP_OK;
}

int fp_tp_export(fp_ctx* c, int64_t max_tokens, fp_tp_handle* out) {
  REQ(c && out, "null argument");
  REQ(c->tp_size > 1, "context is not tensor parallel");
  REQ(max_tokens >= 1, "max_tokens must be >= 1");
  int rc = tp_alloc_block(c, max_tokens);
  if (rc) return rc;
  static_assert(sizeof(cudaIpcMemHandle_t) <= sizeof(out->ipc), "ipc handle size");
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, c->tp_block));
  memset(out, 0, sizeof(*out));
  memcpy(out->ipc, &h, sizeof(h));
  out->part_rows = max_tokens;
  out->rank = c->tp_rank;
  out->device = c->device;
  return FP_OK;
}

int fp_tp_import(fp_ctx* c, const fp_tp_handle* all) {
  REQ(c && all, "null argument");
  REQ(c->tp_block, "call fp_tp_export first");
  REQ(!c->tp_connected, "already connected");
  CK(cudaSetDevice(c->device));
  std::vector<char*> bases(c->tp_size);
  for (int r = 0; r < c->tp_size; ++r) {
    REQ(all[r].rank == r, "handles must be ordered by rank");
    REQ(all[r].part_rows == c->tp_host.part_rows, "ranks disagree on the exchange capacity");
    if (r == c->tp_rank) {
      bases[r] = c->tp_block;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, all[r].ipc, sizeof(h));
    void* ptr = nullptr;
    CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    c->tp_opened.push_back(ptr);
    bases[r] = static_cast<char*>(ptr);
  }
  return tp_finish(c, bases.data());
}

int fp_tp_connect_local(fp_ctx** ctxs, int32_t n, int64_t max_tokens) {
  REQ(ctxs && n >= 2 && n <= kTpMax, "need 2..8 contexts");
  REQ(max_tokens >= 1, "max_tokens must be >= 1");
  bool same_device = true;
  for (int r = 0; r < n; ++r) {
    REQ(ctxs[r] && ctxs[r]->tp_size == n && ctxs[r]->tp_rank == r,
        "contexts must be ranks 0..n-1 of a tp_size == n group, in order");
    REQ(!ctxs[r]->tp_connected, "already connected");
    same_device = same_device && ctxs[r]->device == ctxs[0]->device;
  }
  std::vector<char*> bases(n);
  for (int r = 0; r < n; ++r) {
    int rc = tp_alloc_block(ctxs[r], max_tokens);
    if (rc) return rc;
    bases[r] = ctxs[r]->tp_block;
  }
  if (!same_device) {
    for (int a = 0; a < n; ++a) {
      CK(cudaSetDevice(ctxs[a]->device));
      for (int b = 0; b < n; ++b) {
        if (ctxs[b]->device == ctxs[a]->device) continue;
        int ok = 0;
        CK(cudaDeviceCanAccessPeer(&ok, ctxs[a]->device, ctxs[b]->device));
        REQ(ok, "devices without peer access");
        cudaError_t e = cudaDeviceEnablePeerAccess(ctxs[b]->device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else CK(e);
      }
    }
  }
  for (int r = 0; r < n; ++r) {
    int rc = tp_finish(ctxs[r], bases.data());
    if (rc) return rc;
    if (same_device) {  // one device: every rank's kernels go to rank 0's stream, in lock step
      ctxs[r]->stream = ctxs[0]->own_stream;
      ctxs[r]->tp_lockstep = true;
    }
  }
  return FP_OK;
}

int fp_op_tp_allreduce(fp_ctx** ctxs, int32_t n, void* const* h, const void* const* parts,
                       int32_t M) {
  REQ(ctxs && h && parts && n >= 1 && M >= 1, "null argument");
  for (int i = 0; i < n; ++i) {
    REQ(ctxs[i] && ctxs[i]->tp_connected && ctxs[i]->d_tp, "context is not a connected TP rank");
    REQ(M <= ctxs[i]->tp_host.part_rows, "M exceeds the exchange capacity");
    REQ(h[i] && parts[i], "null buffer");
  }
  CK(cudaSetDevice(ctxs[0]->device));
  const int d = ctxs[0]->cfg.hidden;
  const long long vecs = (long long)M * d / 8;
  const int grid = (int)std::max(1LL, std::min<long long>((vecs + 255) / 256, 4LL * ctxs[0]->num_sms));
  std::vector<float*> ssq(n, nullptr);
  // every caller-driven rank publishes before any of them waits (lock-step ranks share a stream)
  for (int i = 0; i < n; ++i) {
    fp_ctx* c = ctxs[i];
    std::lock_guard<std::mutex> lk(c->launch_mu);
    CK(cudaMallocAsync((void**)&ssq[i], (size_t)M * (d / 128) * 4, c->stream));
    tp_stage_partial_kernel<<<grid, 256, 0, c->stream>>>(
        c->d_tp, static_cast<const __nv_bfloat16*>(parts[i]), vecs);
  }
  for (int i = 0; i < n; ++i) {
    fp_ctx* c = ctxs[i];
    std::lock_guard<std::mutex> lk(c->launch_mu);
    XchgParams x{};
    x.M = M;
    x.d = d;
    x.h = static_cast<__nv_bfloat16*>(h[i]);
    x.ldh = d;
    x.ssq = ssq[i];
    x.guard.tp = c->d_tp;  // unguarded (no task): the boundary check passes
    const int g2 = (int)std::max(1LL, std::min<long long>((vecs + 255) / 256, 8LL * c->num_sms));
    tp_allreduce_kernel<<<g2, 256, 0, c->stream>>>(x);
    CK(cudaFreeAsync(ssq[i], c->stream));
  }
  CK(cudaGetLastError());
  return FP_OK;
}

int fp_tp_enqueue_lockstep(fp_ctx** ctxs, fp_task** tasks, int32_t n, int32_t first,
                           int32_t last) {
  REQ(ctxs && tasks && n >= 2, "null argument");
  std::vector<Task*> ts(n);
  for (int r = 0; r < n; ++r) {
    REQ(ctxs[r] && ctxs[r]->tp_lockstep && ctxs[r]->tp_rank == r && ctxs[r]->tp_size == n,
        "contexts must form a lock-step group (fp_tp_connect_local on one device)");
    ts[r] = reinterpret_cast<Task*>(tasks[r]);
    REQ(ts[r] && ts[r]->n_entries == ts[0]->n_entries, "tasks must have identical timelines");
    REQ(first >= ts[r]->seg_first && first <= last && last <= ts[r]->n_entries, "bad entry range");
  }
  CK(cudaSetDevice(ctxs[0]->device));
  std::vector<std::unique_lock<std::mutex>> locks;
  for (int r = 0; r < n; ++r) locks.emplace_back(ctxs[r]->launch_mu);
  for (int e = first; e < last; ++e)
    for (int phase : {kPhasePre, kPhasePost})
      for (int r = 0; r < n; ++r) {  // rank 0 first: its boundary decision precedes the others'
        int rc = launch_entry_checked(ctxs[r], ts[r], e, phase);
        if (rc) return rc;
      }
  for (int r = 0; r < n; ++r) {
    ts[r]->enq = std::max(ts[r]->enq, (int)last);
    if (last == ts[r]->n_entries) {
      CK(cudaEventRecord(ts[r]->done, ctxs[r]->stream));
      ts[r]->done_recorded = 1;
    }
    CK(cudaEventRecord(ts[r]->fence, ctxs[r]->stream));
  }
  CK(cudaGetLastError());
  return FP_OK;
}

int fp_ctx_tp_counters(fp_ctx* c, int32_t* out4) {
  REQ(c && out4, "null argument");
  if (!c->tp_local) {
    memset(out4, 0, 16);
    return FP_OK;
  }
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  TpLocal l;
  CK(cudaMemcpy(&l, c->tp_local, sizeof(l), cudaMemcpyDeviceToHost));
  out4[0] = l.xcount;
  out4[1] = l.bcount;
  out4[2] = l.gemm_ctr;
  out4[3] = l.ar_ctr;
  return FP_OK;
}

}  // extern "C"
