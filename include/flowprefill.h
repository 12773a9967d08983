/* flowprefill.h -- C ABI of the B200-native preemptible prefill forward pass.
 *
 * The reference (FlowPrefill's prefillsim, /root/reference/pkg/src/prefillsim) has no native
 * code: its "forward pass" is the cost model + discrete-event execution pool. Each entry point
 * below replaces one piece of that Python surface; the citation names the reference symbol
 * whose behaviour the call realises on the GPU.
 *
 * Conventions
 *   - every call returns 0 on success or a negative FP_ERR_* code; fp_last_error() returns a
 *     thread-local message. No C++ exception crosses this boundary.
 *   - device memory (weights, paged KV pool, task workspaces) is library-owned. Host arrays are
 *     caller-owned and only borrowed for the duration of a call.
 *   - one context per device (= one execution pool, prefillsim/engine.py:137-144). All calls come
 *     from the owning thread except fp_signal(), which is a single store to pinned memory.
 */
#ifndef FLOWPREFILL_H
#define FLOWPREFILL_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define FP_OK 0
#define FP_ERR_ARG -1
#define FP_ERR_CUDA -2
#define FP_ERR_NOMEM -3
#define FP_ERR_STATE -4
#define FP_ERR_UNSUPPORTED -5

/* Preemption granularity: prefillsim/engine.py:43-47 (PreemptionGranularity). */
#define FP_GRAN_OPERATOR 0
#define FP_GRAN_LAYER 1
#define FP_GRAN_CHUNK 2
#define FP_GRAN_NONE 3

/* Operator kinds of one dense layer, in timeline order: prefillsim/cost_model.py:38-44. */
#define FP_OP_QKV_PROJ 0
#define FP_OP_ATTN 1
#define FP_OP_O_PROJ 2
#define FP_OP_GATE_UP_PROJ 3
#define FP_OP_DOWN_PROJ 4
/* MoE layers (n_experts > 0) replace the last two: prefillsim/cost_model.py:46-52. */
#define FP_OP_GATE 3    /* router: fused post-attention norm, logits GEMM, softmax top-k, dispatch */
#define FP_OP_EXPERTS 4 /* grouped expert gate/up + SwiGLU, grouped down, weighted combine */

/* Weight tensor ids for fp_weights_load (canonical, unpacked Llama layout, bf16 row-major). */
#define FP_W_EMBED 0      /* [vocab, hidden] */
#define FP_W_Q 1          /* [n_heads*head_dim, hidden] */
#define FP_W_K 2          /* [n_kv_heads*head_dim, hidden] */
#define FP_W_V 3          /* [n_kv_heads*head_dim, hidden] */
#define FP_W_O 4          /* [hidden, n_heads*head_dim] */
#define FP_W_GATE 5       /* [ffn, hidden] */
#define FP_W_UP 6         /* [ffn, hidden] */
#define FP_W_DOWN 7       /* [hidden, ffn] */
#define FP_W_ATTN_NORM 8  /* [hidden] */
#define FP_W_FFN_NORM 9   /* [hidden] */
#define FP_W_FINAL_NORM 10 /* [hidden] */
#define FP_W_LM_HEAD 11   /* [vocab, hidden] */
#define FP_W_Q_BIAS 12    /* [n_heads*head_dim]      (Qwen2.5: qkv_bias) */
#define FP_W_K_BIAS 13    /* [n_kv_heads*head_dim] */
#define FP_W_V_BIAS 14    /* [n_kv_heads*head_dim] */
#define FP_W_Q_NORM 15    /* [head_dim]              (Qwen3: qk_norm) */
#define FP_W_K_NORM 16    /* [head_dim] */
#define FP_W_ROUTER 17       /* [n_experts, hidden]                    (MoE) */
#define FP_W_EXPERT_GATE 18  /* [n_experts, moe_ffn, hidden] */
#define FP_W_EXPERT_UP 19    /* [n_experts, moe_ffn, hidden] */
#define FP_W_EXPERT_DOWN 20  /* [n_experts, hidden, moe_ffn] */

typedef struct fp_model_cfg {
  int32_t num_layers; /* CostParams.num_layers, cost_model.py:92 */
  int32_t hidden;
  int32_t n_heads;
  int32_t n_kv_heads;
  int32_t head_dim; /* must be 128 */
  int32_t ffn;
  int32_t vocab;   /* any size; padded internally to a multiple of 256 */
  int32_t max_pos; /* RoPE table length */
  float rope_theta;
  float rms_eps;
  int32_t qkv_bias; /* 1: q/k/v projections carry a bias (Qwen2.5) */
  int32_t qk_norm;  /* 1: per-head RMSNorm of q and k before RoPE (Qwen3) */
  /* MoE (Qwen3-MoE block, every layer sparse; n_experts = 0: dense). ffn is unused then. */
  int32_t n_experts;  /* <= 256 */
  int32_t top_k;      /* <= 16 */
  int32_t moe_ffn;    /* expert intermediate size, multiple of 128 */
  int32_t norm_topk;  /* 1: renormalise the top-k router probabilities to sum 1 */
} fp_model_cfg;

typedef struct fp_ctx fp_ctx;
typedef struct fp_task fp_task;

/* Control-block snapshot (the ACK half of the handshake, engine.py:240-291). */
typedef struct fp_status {
  int32_t ack_seq;        /* bumped once per acknowledged preemption */
  int32_t ack_task;       /* task that stopped */
  int32_t ack_entry;      /* new cursor of that task (first entry not executed) */
  int32_t progress_task;  /* task whose entry most recently passed its boundary check */
  int32_t progress_entry;
  int32_t signal;         /* pending preemption signal (1) or none (0) */
  uint64_t ack_ns;        /* device %globaltimer at the stop decision */
} fp_status;

/* Task execution state (TaskState, engine.py:36-40). */
#define FP_TASK_IDLE 0
#define FP_TASK_RUNNING 1
#define FP_TASK_STOPPED 2
#define FP_TASK_DONE 3
typedef struct fp_task_status {
  int32_t state;
  int32_t cursor;     /* entries [0, cursor) are complete */
  int32_t generation; /* bumped per submit/resume segment (engine.py:286) */
  int32_t enqueued;   /* entries handed to the GPU so far in this segment */
} fp_task_status;

const char* fp_last_error(void);
int fp_version(void);

/* ---- context (one execution pool per device) ---------------------------------------- */
/* Replaces Engine.__init__ (engine.py:161-179). With tp_size > 1 the context is one rank of a
 * Megatron tensor-parallel group (the reference models TP only as a duration scale,
 * cost_model.py:99-100,166, and a lane-equality gate, tp_sync_check, engine.py:50-57): it holds
 * heads n_heads/tp_size (q) and n_kv_heads/tp_size (k/v), ffn/tp_size, and all-reduces the
 * o_proj / down_proj partial sums over peer memory. Connect the group with
 * fp_tp_connect_local (one process) or fp_tp_export + fp_tp_import (one process per GPU)
 * before creating tasks. nccl_comm must be null (the exchange does not go through NCCL). */
int fp_ctx_create(int32_t device, const fp_model_cfg* cfg, int32_t tp_rank, int32_t tp_size,
                  void* nccl_comm, int64_t kv_pages, int32_t page_size, fp_ctx** out);
int fp_ctx_destroy(fp_ctx* ctx);
int fp_ctx_stream(fp_ctx* ctx, void** stream_out); /* cudaStream_t of the prefill stream */
int fp_ctx_free_pages(fp_ctx* ctx, int64_t* free_pages);
int fp_ctx_set_window(fp_ctx* ctx, int32_t entries); /* async look-ahead bound */
int fp_sync(fp_ctx* ctx);

/* ---- weights ------------------------------------------------------------------------ */
int fp_weights_init_random(fp_ctx* ctx, uint64_t seed, float std);
int fp_weights_load(fp_ctx* ctx, int32_t tensor, int32_t layer, const void* host_bf16,
                    int64_t n_elems);

/* ---- task lifecycle ------------------------------------------------------------------ */
/* Replaces build_timeline + ExecutionTask.__init__ (cost_model.py:191-244, engine.py:84-115):
 * requests are concatenated, cut into chunks of chunk_tokens (0 = unchunked), and expanded
 * into n_chunks * num_layers * 5 guarded entries in chunk -> layer -> operator order. */
int fp_task_create(fp_ctx* ctx, const int32_t* token_ids, const int32_t* seq_lens,
                   int32_t n_seqs, int32_t chunk_tokens, int32_t granularity, int32_t task_id,
                   fp_task** out);
int fp_task_num_entries(const fp_task* task);
typedef struct fp_task_info {
  int32_t n_entries, n_chunks, n_seqs, total_tokens, max_chunk_tokens, n_pages;
  int64_t upload_bytes; /* host->device bytes copied by fp_task_create (ids + plan) */
} fp_task_info_t;
int fp_task_info(const fp_task* task, fp_task_info_t* info);
int fp_task_entry_info(const fp_task* task, int32_t entry, int32_t* chunk, int32_t* layer,
                       int32_t* op, int32_t* new_tokens);
/* %globaltimer (ns) at each entry's boundary decision: host_out[e] = GO (0: not executed yet),
 * host_out[n_entries + e] = STOP (0: never stopped there). Entry e-1 ends at entry e's STOP if
 * there was one, else at its GO: the wall-clock form of OperatorTimeline.max_entry_duration
 * (cost_model.py:185-188), the bound on signal -> ACK blocking (test_properties.py:90-94). */
int fp_task_entry_stamps(fp_ctx* ctx, fp_task* task, uint64_t* host_out); /* [2, n_entries] */
int fp_task_destroy(fp_ctx* ctx, fp_task* task);

/* Start a new execution segment from `first` (Engine.submit / Engine.resume,
 * engine.py:207-238): bumps the generation and re-arms the boundary checks of [first, end). */
int fp_task_begin_segment(fp_ctx* ctx, fp_task* task, int32_t first);
/* Enqueue entries [first, last) of the current segment on the prefill stream (synchronous
 * launch, asynchronous execution). Used by the virtual-clock parity driver and the bench. */
int fp_task_enqueue(fp_ctx* ctx, fp_task* task, int32_t first, int32_t last);
/* Asynchronous segment: begin_segment(first) + the context's launch worker keeps at most
 * `window` entries queued ahead of the GPU until the end or a stop. */
int fp_task_start(fp_ctx* ctx, fp_task* task, int32_t first);
int fp_task_poll(fp_ctx* ctx, fp_task* task, fp_task_status* out);

/* ---- preemption handshake (Engine.signal_preempt / _finalize_ack, engine.py:240-291) ---- */
int fp_signal(fp_ctx* ctx);
int fp_clear(fp_ctx* ctx);
int fp_poll(fp_ctx* ctx, fp_status* out);

/* ---- parity taps ----------------------------------------------------------------------- */
int fp_task_logits(fp_ctx* ctx, fp_task* task, float* host_out); /* [n_seqs, vocab] */
/* MoE parity tap: routing of the most recent gate entry (its chunk's rows): expert ids and
 * weights [chunk_tokens, top_k], descending probability. */
int fp_task_read_routing(fp_ctx* ctx, fp_task* task, int32_t* host_ids, float* host_w,
                         int32_t max_rows);
int fp_task_read_kv(fp_ctx* ctx, fp_task* task, int32_t seq, int32_t layer, void* host_k,
                    void* host_v); /* each [seq_len, n_kv_heads, head_dim] bf16 */

/* ---- live kernel profiling (CUDA events around every kernel on the prefill stream) ---- */
#define FP_K_RMS 0
#define FP_K_QKV 1
#define FP_K_ATTN 2
#define FP_K_O 3
#define FP_K_GATE_UP 4
#define FP_K_DOWN 5
#define FP_K_LM_HEAD 6
#define FP_K_RMS_FINAL 7
#define FP_K_XCHG 8 /* tensor-parallel all-reduce of o_proj / down_proj partials */
#define FP_K_ROUTER 9        /* MoE router logits GEMM */
#define FP_K_MOE_DISPATCH 10 /* top-k routing, expert offsets, row gather */
#define FP_K_EXPERT_GU 11    /* grouped expert gate/up + SwiGLU GEMM */
#define FP_K_EXPERT_DOWN 12  /* grouped expert down GEMM */
#define FP_K_MOE_COMBINE 13  /* weighted combine into the residual */
typedef struct fp_prof_rec {
  int32_t kind;  /* FP_K_* */
  int32_t layer;
  int32_t M;     /* token rows of the launch */
  int32_t pad;
  double flops;  /* algorithmic FLOPs of the launch (0 for HBM-bound kernels) */
  double bytes;  /* algorithmic HBM bytes of the launch (0 for tensor-bound kernels) */
  double ms;     /* event-measured duration */
} fp_prof_rec;
int fp_prof_enable(fp_ctx* ctx, int32_t on);
/* Synchronises, returns up to max records (n = total recorded) and clears the log. */
int fp_prof_collect(fp_ctx* ctx, fp_prof_rec* out, int32_t max, int32_t* n);
/* Number of kernels this context has launched (guarded no-ops included). */
int fp_ctx_launch_count(fp_ctx* ctx, int64_t* n);

/* ---- tensor parallelism (config 4: TP = 2/4/8, synchronized operator-boundary preemption) ----
 * Every rank executes the identical entry list; rank 0 alone evaluates each boundary check and
 * publishes the decision in a ring the followers read over peer memory, so all ranks stop at the
 * same entry index (replaces tp_sync_check, engine.py:50-57, used at :254-255).
 * Only rank 0's fp_signal() is observed by the device. */
typedef struct fp_tp_handle {
  char ipc[64];      /* cudaIpcMemHandle_t of the rank's exchange block */
  int64_t part_rows; /* exchange capacity in token rows (max chunk tokens) */
  int32_t rank;
  int32_t device;
} fp_tp_handle;
/* One process per GPU: allocate this rank's exchange block (capacity max_tokens rows) and
 * export it; gather every rank's handle (e.g. torch.distributed.all_gather_object) and pass
 * them, ordered by rank, to fp_tp_import. */
int fp_tp_export(fp_ctx* ctx, int64_t max_tokens, fp_tp_handle* out);
int fp_tp_import(fp_ctx* ctx, const fp_tp_handle* all);
/* One process: connect ranks 0..n-1. On a single device the ranks share rank 0's stream and
 * must be driven in lock step through fp_tp_enqueue_lockstep (phase 1 of an entry -- up to the
 * exchange GEMM -- on every rank before phase 2 on any rank). Destroy followers before rank 0. */
int fp_tp_connect_local(fp_ctx** ctxs, int32_t n, int64_t max_tokens);
int fp_tp_enqueue_lockstep(fp_ctx** ctxs, fp_task** tasks, int32_t n, int32_t first,
                           int32_t last);
/* Synchronises and reads the rank's device counters: [exchanges, boundaries decided,
 * gemm ticket, all-reduce ticket] (tickets are 0 between kernels). */
int fp_ctx_tp_counters(fp_ctx* ctx, int32_t* out4);
/* The row-parallel exchange as a per-op entry point: for every rank i driven by this caller
 * (all ranks of a lock-step group, or this process's rank of a multi-process group),
 * h_i[M, hidden] = bf16(h_i + part_0 + ... + part_{tp-1}) (fp32 sum in rank order; the
 * partials of ranks not in `ctxs` come from their own callers). Device pointers; M <= the
 * exchange capacity. The reference models this step only as `/tp * (1 + tp_comm_overhead)`
 * (prefillsim/cost_model.py:99-100,166). */
int fp_op_tp_allreduce(fp_ctx** ctxs, int32_t n, void* const* h, const void* const* parts,
                       int32_t M);

/* ---- per-operator entry points (device pointers; unit tests and microbenchmarks) -------- */
/* C[M,N] = A[M,K] B[N,K]^T; epi: 0 bf16 store, 1 fp32 store, 2 residual add into C (bf16),
 * 3 SwiGLU: B packed [gate(128) | up(128)] per 256 rows, C[M, N/2] = silu(gate) * up. */
int fp_op_gemm(fp_ctx* ctx, int32_t epi, const void* A, const void* B, void* C, int32_t M,
               int32_t N, int32_t K);
int fp_op_rmsnorm(fp_ctx* ctx, const void* x, const void* gamma, void* out, int32_t M,
                  int32_t d, float eps);
/* out[M, F] = silu(x W_gate^T) * (x W_up^T): the gate_up_proj GEMM with its SwiGLU epilogue. */
int fp_op_gate_up_swiglu(fp_ctx* ctx, const void* x, const void* w_gate, const void* w_up,
                         void* out, int32_t M, int32_t F, int32_t K);
/* qkv_proj with its fused epilogue (fp_task's entry 0 of a layer minus the input norm):
 * [q | k | v] = x W_qkv^T (W_qkv [q_cols + 2 kv_cols, K], q heads, then k heads, then v heads,
 * 128 columns each), RoPE (rotate-half, the context's rope_theta, positions[m] < max_pos) on q
 * and k, q -> q_out [M, q_cols], k and v -> the paged layout kv_pages[page][k|v][kv head]
 * [positions[m] % page_size][128] of the page tok_page[m] (the forward pass's KV write). All
 * pointers are device memory. Replaces the reference's per-kind cost of `qkv_proj`
 * (prefillsim/cost_model.py:151-166) with the computation. */
int fp_op_qkv_rope_kv(fp_ctx* ctx, const void* x, const void* w_qkv, void* q_out, void* kv_pages,
                      const int32_t* positions, const int32_t* tok_page, int32_t M, int32_t q_cols,
                      int32_t kv_cols, int32_t K);
/* Causal prefill attention of one request's last n_q tokens over kv_len keys (prefix =
 * kv_len - n_q): q/out [n_q, n_heads*128], k/v [kv_len, n_kv_heads*128] (bf16, device); K/V go
 * through the paged pool like the forward pass (borrowed free pages). */
int fp_op_attn_prefill(fp_ctx* ctx, const void* q, const void* k, const void* v, void* out,
                       int32_t n_q, int32_t kv_len);
/* GEMM tiling override for experiments and split-K parity tests: pair = -1 auto, 0 single-CTA
 * tiles, 1 CTA-pair tiles, 2 narrow 128 x 128 tiles (residual / QKV epilogues), 3 stream-K
 * (whole tiles, then equal (tile, k-block) ranges per CTA), 4 swap-AB skinny (M <= 256: weight
 * rows as the MMA M dimension, equal weight ranges per CTA); splits = 0
 * auto, S >= 1 forces S K-slices on the partial-wave tiles (clamped so the split units fit one
 * round of the persistent grid). */
int fp_ctx_set_gemm_policy(fp_ctx* ctx, int32_t pair, int32_t splits);
/* Largest launch M (tokens) planned with the swap-AB skinny GEMM under the auto policy
 * (default 128, also FP_SKINNY_MAX_M at fp_ctx_create; 0 disables it). Below it the auto policy
 * takes the skinny plan for M <= 8, and for K >= 8192 (down_proj) up to this M. */
int fp_ctx_set_skinny_max(fp_ctx* ctx, int32_t max_m);
/* Batch-invariant numerics (also FP_BATCH_INVARIANT=1 at fp_ctx_create): no split-K and no
 * stream-K, so each output element is one in-order accumulation over K whatever the launch's
 * M, and a request's logits / KV are bit-identical alone or in any batch (SURVEY.md §7 hard
 * part 7). Off by default: split-K is what makes short requests fast. */
int fp_ctx_set_batch_invariant(fp_ctx* ctx, int32_t on);
/* Diagnostics: with FP_GEMM_STAMPS=1 in the environment at fp_ctx_create, every fp_op_gemm
 * launch records per-CTA phase stamps (%globaltimer ns, 16 slots per CTA: entry, prologue done,
 * boundary check done, first TMA, first MMA, last accumulator commit, epilogue start, partial
 * stored, split barrier passed, split items done, exit, teardown). Copies max_ctas x 16. */
int fp_debug_gemm_stamps(fp_ctx* ctx, uint64_t* out, int32_t max_ctas);

#ifdef __cplusplus
}
#endif
#endif
