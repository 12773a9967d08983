// Cooperative preemption control: the per-boundary device-side check.
//
// The reference models the check as "after the current operator completes, look at the
// preemption signal; if set, unset it, ACK, and suspend" (simulated in
// prefillsim/engine.py:240-291). Here every timeline entry's FIRST kernel evaluates the check
// in its prologue. All CTAs of that kernel agree through one atomicCAS on the entry's decision
// slot, so a kernel either runs completely or not at all; later kernels of the same entry and
// every queued entry of a stopped generation become no-ops.
#pragma once
#include "common.cuh"

namespace fp {

// Pinned, device-mapped host memory: one per context (one execution pool).
struct HostCtl {
  volatile int signal;          // host -> device: 1 = preemption requested
  volatile int ack_seq;         // device -> host: bumped once per acknowledged stop
  volatile int ack_task;        // task id that stopped
  volatile int ack_entry;       // first entry NOT executed (= new cursor)
  volatile int progress_task;   // task whose entry most recently passed its check
  volatile int progress_entry;  // that entry's index
  volatile unsigned long long ack_ns;  // device %globaltimer at the stop decision
  int pad[24];
};

// Device memory: one per task. dec[] holds one decision per timeline entry.
struct TaskCtl {
  int stopped_gen;  // generation that has been stopped (-1: none)
  int pad0;
  unsigned long long* stamps;  // [2][n_entries] %globaltimer at each entry's GO / STOP decision
  int pad[28];
  int dec[1];       // [n_entries]: 0 undecided, 1 go, 2 stop
};

// ---- tensor parallelism: cross-rank state -------------------------------------------------
// The reference keeps TP as one logical lane whose boundary is "synchronised" by a lane-counter
// equality check (tp_sync_check, prefillsim/engine.py:50-57, used at :254-255; the paper's
// synchronized iteration counter). Here every rank runs the identical entry list
// and rank 0 alone decides each boundary; followers adopt rank 0's decision from its ring, so
// all ranks stop at the same entry by construction.
constexpr int kTpMax = 8;
constexpr int kTpRing = 64;

// Per-rank block in peer-visible (IPC-shareable) device memory.
constexpr int kTpFlagTiles = 8192;      // per-tile readiness flags per exchange slot

struct TpShared {
  unsigned long long ready;             // exchange GEMMs whose partial sum is complete
  unsigned long long pad0[15];
  unsigned long long ring[kTpRing];     // rank 0 only: ((boundary + 1) << 2) | decision
  // fused exchange GEMM: flags[slot][tile slot] = exchange + 1 once this rank's partial of that
  // output tile is in part[rank][slot] (monotonic: never reset)
  unsigned long long flags[2][kTpFlagTiles];
};

// Per-rank device-local counters (identical sequences on every rank: only entries that
// actually execute advance them, and all ranks execute the same entries).
struct TpLocal {
  int xcount;    // exchanges (o_proj / down_proj all-reduces) completed
  int gemm_ctr;  // CTA completion ticket of the current exchange GEMM
  int ar_ctr;    // CTA completion ticket of the current all-reduce
  int bcount;    // boundaries decided
  int pad[28];
};

struct TpDev {
  int rank, size;
  long long part_rows;                  // capacity (token rows) of each partial buffer
  TpLocal* local;
  TpShared* peer[kTpMax];               // every rank's shared block (peer[rank] = own)
  __nv_bfloat16* part[kTpMax][2];       // every rank's double-buffered partial [rows, hidden]
};

struct Guard {
  HostCtl* host;  // device alias of the mapped control block (may be null: unguarded)
  TaskCtl* task;  // null: unguarded launch (per-op unit entry points)
  int entry;
  int gen;
  int task_id;
  int first;     // 1 for the first kernel of the entry: evaluates the check
  int eligible;  // the boundary in front of this entry is preemption-eligible
  int n_entries;
  const TpDev* tp;  // null unless tensor parallel
};

constexpr int kDecGo = 1;
constexpr int kDecStop = 2;

// Thread-0-only. Returns true when the kernel must execute.
DEVI bool guard_pass(const Guard& g) {
  if (g.task == nullptr) return true;
  volatile int* sg = &g.task->stopped_gen;
  if (*sg == g.gen) return false;
  if (!g.first) return true;
  volatile int* slot = &g.task->dec[g.entry];
  int d = *slot;  // most CTAs find the decision already made
  if (d) return d == kDecGo;
  // One decider per boundary: CTA 0 reads the pinned host flag (one PCIe read) and publishes
  // the decision; the other CTAs wait for it in L2 instead of all hitting PCIe. A waiter that
  // sees no decision for a long time takes the decider path itself (atomicCAS keeps it
  // consistent), so progress never depends on CTA scheduling order.
  bool decider = blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0;
  if (!decider) {
    for (int spin = 0; spin < 200000; ++spin) {
      d = *slot;
      if (d) return d == kDecGo;
      __nanosleep(32);
    }
    decider = true;
  }
  int want = kDecGo;
  const TpDev* tp = g.tp;
  const int b = tp ? *(volatile int*)&tp->local->bcount : 0;
  if (tp && tp->rank != 0) {
    // follower: adopt rank 0's decision for this boundary (same boundary count on every rank)
    const unsigned long long* ring = &tp->peer[0]->ring[b % kTpRing];
    for (;;) {
      if ((d = *slot)) return d == kDecGo;  // another CTA of this kernel already decided
      const unsigned long long v = ld_acquire_sys_u64(ring);
      if ((long long)(v >> 2) == b + 1) {  // tags are boundary + 1 (0 = never written)
        want = (int)(v & 3);
        break;
      }
      __nanosleep(64);
    }
  } else if (g.eligible && g.host != nullptr && ld_volatile_sys(&g.host->signal)) {
    want = kDecStop;
  }
  const int old = atomicCAS(&g.task->dec[g.entry], 0, want);
  d = old ? old : want;
  if (old == 0 && tp) {
    if (tp->rank == 0)
      st_release_sys_u64(&tp->peer[0]->ring[b % kTpRing], ((unsigned long long)(b + 1) << 2) | d);
    tp->local->bcount = b + 1;
  }
  if (old == 0 && d == kDecStop) {  // later launches of this generation become no-ops
    *sg = g.gen;                    // (they start only after this kernel has exited)
    __threadfence();
  }
  if (old == 0 && g.host != nullptr) {  // the winning CTA publishes the decision
    if (d == kDecStop) {
      g.host->signal = 0;
      g.host->ack_task = g.task_id;
      g.host->ack_entry = g.entry;
      g.host->ack_ns = globaltimer();
      if (g.task->stamps) g.task->stamps[g.n_entries + g.entry] = g.host->ack_ns;
      __threadfence_system();
      g.host->ack_seq = g.host->ack_seq + 1;
      __threadfence_system();
    } else {
      if (g.task->stamps) g.task->stamps[g.entry] = globaltimer();
      g.host->progress_task = g.task_id;
      g.host->progress_entry = g.entry;
      __threadfence_system();
    }
  }
  return d == kDecGo;
}

// Thread 0 of every CTA of an exchange GEMM, after the CTA's partial-sum stores: the last CTA
// to finish publishes "partial of exchange xcount complete" to the peers.
DEVI void tp_publish_partial(const TpDev* tp) {
  __threadfence_system();
  const int xc = *(volatile int*)&tp->local->xcount;
  const int old = atomicAdd(&tp->local->gemm_ctr, 1);
  if (old == (int)(gridDim.x * gridDim.y * gridDim.z) - 1) {
    tp->local->gemm_ctr = 0;
    __threadfence_system();
    st_release_sys_u64(&tp->peer[tp->rank]->ready, (unsigned long long)xc + 1);
  }
}

// Block-wide wrapper; every thread calls it.
DEVI bool guard_block(const Guard& g) {
  __shared__ int s_go;
  if (threadIdx.x == 0) s_go = guard_pass(g) ? 1 : 0;
  __syncthreads();
  return s_go != 0;
}

}  // namespace fp
