"""Pythonic handles over the C ABI: a prefill context (one execution pool per GPU) and tasks.

``PrefillContext`` owns the device: weights, the paged KV pool, the pinned preemption control
block and the launch worker. ``PrefillTask`` is one batched prefill expanded into its guarded
timeline entries (chunk -> layer -> operator, prefillsim/cost_model.py:224-242).
"""

from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .config import ModelShape

GRANULARITY = _lib.FP_GRAN


def _bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit patterns (round to nearest even); uint16 passes through."""
    x = np.asarray(x)
    if x.dtype == np.uint16:
        return np.ascontiguousarray(x)
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


# Norm weights first: the library folds them into the projection columns (fused RMSNorm), and
# a norm loaded after its projection costs a second bf16 rounding of the folded weights.
_WEIGHT_IDS = {
    "attn_norm": _lib.W_ATTN_NORM,
    "ffn_norm": _lib.W_FFN_NORM,
    "wq": _lib.W_Q,
    "wk": _lib.W_K,
    "wv": _lib.W_V,
    "wo": _lib.W_O,
    "w_gate": _lib.W_GATE,
    "w_up": _lib.W_UP,
    "w_down": _lib.W_DOWN,
    "bq": _lib.W_Q_BIAS,
    "bk": _lib.W_K_BIAS,
    "bv": _lib.W_V_BIAS,
    "q_norm": _lib.W_Q_NORM,
    "k_norm": _lib.W_K_NORM,
    "w_router": _lib.W_ROUTER,
    "e_gate": _lib.W_EXPERT_GATE,
    "e_up": _lib.W_EXPERT_UP,
    "e_down": _lib.W_EXPERT_DOWN,
}


class PrefillContext:
    """One execution pool on one GPU (prefillsim/engine.py:137-144, 154-179)."""

    def __init__(
        self,
        shape: ModelShape,
        device: int = 0,
        kv_pages: int = 256,
        page_size: int = 128,
        max_pos: int = 65536,
        window: int = 8,
        tp_rank: int = 0,
        tp_size: int = 1,
    ):
        self.lib = _lib.load()
        self.shape = shape
        self.page_size = page_size
        self.tp_rank, self.tp_size = tp_rank, tp_size
        cfg = _lib.ModelCfg(
            shape.num_layers,
            shape.hidden,
            shape.n_heads,
            shape.n_kv_heads,
            shape.head_dim,
            shape.ffn,
            shape.vocab,
            max_pos,
            shape.rope_theta,
            shape.rms_eps,
            int(shape.qkv_bias),
            int(shape.qk_norm),
            int(shape.n_experts),
            int(shape.top_k),
            int(shape.moe_ffn),
            int(shape.norm_topk),
        )
        h = C.c_void_p()
        _lib.check(
            self.lib.fp_ctx_create(device, C.byref(cfg), tp_rank, tp_size, None, kv_pages,
                                   page_size, C.byref(h)),
            "fp_ctx_create",
        )
        self.h = h
        _lib.check(self.lib.fp_ctx_set_window(h, window), "fp_ctx_set_window")
        s = C.c_void_p()
        _lib.check(self.lib.fp_ctx_stream(h, C.byref(s)), "fp_ctx_stream")
        self.stream_ptr = s.value

    # -- weights ---------------------------------------------------------------------
    def init_random(self, seed: int, std: float = 0.02) -> None:
        _lib.check(self.lib.fp_weights_init_random(self.h, seed, std), "fp_weights_init_random")

    def load_weights(self, w: dict) -> None:
        """Canonical names as in oracle.forward.make_weights ("embed", "{l}.wq", ...)."""

        def put(tid: int, layer: int, arr) -> None:
            bits = _bf16_bits(arr)
            _lib.check(
                self.lib.fp_weights_load(self.h, tid, layer, bits.ctypes.data, bits.size),
                f"fp_weights_load({tid},{layer})",
            )

        put(_lib.W_EMBED, -1, w["embed"])
        put(_lib.W_LM_HEAD, -1, w["lm_head"])
        put(_lib.W_FINAL_NORM, -1, w["final_norm"])
        for l in range(self.shape.num_layers):
            for name, tid in _WEIGHT_IDS.items():
                if f"{l}.{name}" in w:
                    put(tid, l, w[f"{l}.{name}"])

    # -- tasks -----------------------------------------------------------------------
    def create_task(
        self,
        tokens: Sequence[np.ndarray],
        chunk_tokens: Optional[int] = None,
        granularity: str = "operator",
        task_id: int = 0,
    ) -> "PrefillTask":
        return PrefillTask(self, tokens, chunk_tokens, granularity, task_id)

    # -- preemption handshake -------------------------------------------------------
    def signal(self) -> None:
        _lib.check(self.lib.fp_signal(self.h), "fp_signal")

    def clear(self) -> None:
        _lib.check(self.lib.fp_clear(self.h), "fp_clear")

    def poll(self) -> _lib.Status:
        st = _lib.Status()
        _lib.check(self.lib.fp_poll(self.h, C.byref(st)), "fp_poll")
        return st

    def sync(self) -> None:
        _lib.check(self.lib.fp_sync(self.h), "fp_sync")

    def free_pages(self) -> int:
        n = C.c_int64()
        _lib.check(self.lib.fp_ctx_free_pages(self.h, C.byref(n)), "fp_ctx_free_pages")
        return n.value

    def set_window(self, entries: int) -> None:
        _lib.check(self.lib.fp_ctx_set_window(self.h, entries), "fp_ctx_set_window")

    def set_batch_invariant(self, on: bool) -> None:
        """No split-K / stream-K: a request's results are bit-identical in any batch."""
        _lib.check(self.lib.fp_ctx_set_batch_invariant(self.h, 1 if on else 0),
                   "fp_ctx_set_batch_invariant")

    # -- live profiling -------------------------------------------------------------
    def profile(self, on: bool) -> None:
        _lib.check(self.lib.fp_prof_enable(self.h, 1 if on else 0), "fp_prof_enable")

    def drain_profile(self, max_records: int = 1 << 20) -> list[dict]:
        """Synchronise and return every kernel record since the last drain."""
        buf = (_lib.ProfRec * max_records)()
        n = C.c_int32()
        _lib.check(self.lib.fp_prof_collect(self.h, buf, max_records, C.byref(n)),
                   "fp_prof_collect")
        out = []
        for i in range(min(n.value, max_records)):
            r = buf[i]
            out.append({"kind": _lib.KERNEL_KINDS[r.kind], "layer": r.layer, "M": r.M,
                        "flops": r.flops, "bytes": r.bytes, "ms": r.ms})
        return out

    # -- tensor parallelism (one process per GPU) ---------------------------------------
    def tp_export(self, max_tokens: int) -> bytes:
        """This rank's exchange block handle (gather it from every rank, then tp_import)."""
        hd = _lib.TpHandle()
        _lib.check(self.lib.fp_tp_export(self.h, max_tokens, C.byref(hd)), "fp_tp_export")
        return bytes(memoryview(hd))

    def tp_import(self, handles: Sequence[bytes]) -> None:
        arr = (_lib.TpHandle * len(handles))()
        for i, b in enumerate(handles):
            C.memmove(C.byref(arr[i]), b, C.sizeof(_lib.TpHandle))
        _lib.check(self.lib.fp_tp_import(self.h, arr), "fp_tp_import")

    def tp_counters(self) -> dict:
        out = (C.c_int32 * 4)()
        _lib.check(self.lib.fp_ctx_tp_counters(self.h, out), "fp_ctx_tp_counters")
        return {"exchanges": out[0], "boundaries": out[1], "gemm_ticket": out[2],
                "allreduce_ticket": out[3]}

    def launch_count(self) -> int:
        n = C.c_int64()
        _lib.check(self.lib.fp_ctx_launch_count(self.h, C.byref(n)), "fp_ctx_launch_count")
        return n.value

    def close(self) -> None:
        if self.h is not None:
            self.lib.fp_ctx_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


class PrefillTask:
    """One batched (optionally chunked) prefill: a cursor over guarded entries."""

    def __init__(self, ctx: PrefillContext, tokens, chunk_tokens, granularity, task_id):
        self.ctx = ctx
        self.lib = ctx.lib
        self.lens = [int(len(t)) for t in tokens]
        ids = np.ascontiguousarray(np.concatenate(tokens).astype(np.int32))
        lens = np.asarray(self.lens, dtype=np.int32)
        self.task_id = task_id
        h = C.c_void_p()
        _lib.check(
            self.lib.fp_task_create(
                ctx.h,
                ids.ctypes.data,
                lens.ctypes.data,
                len(self.lens),
                int(chunk_tokens or 0),
                GRANULARITY[granularity],
                task_id,
                C.byref(h),
            ),
            "fp_task_create",
        )
        self.h = h
        self.n_entries = self.lib.fp_task_num_entries(h)

    def info(self) -> dict:
        inf = _lib.TaskInfo()
        _lib.check(self.lib.fp_task_info(self.h, C.byref(inf)), "fp_task_info")
        return {k: getattr(inf, k) for k, _ in _lib.TaskInfo._fields_}

    def entry_info(self, i: int) -> tuple[int, int, int, int]:
        c, l, o, n = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        _lib.check(
            self.lib.fp_task_entry_info(self.h, i, C.byref(c), C.byref(l), C.byref(o), C.byref(n)),
            "fp_task_entry_info",
        )
        return c.value, l.value, o.value, n.value

    def begin_segment(self, first: int) -> None:
        _lib.check(self.lib.fp_task_begin_segment(self.ctx.h, self.h, first), "begin_segment")

    def enqueue(self, first: int, last: int) -> None:
        _lib.check(self.lib.fp_task_enqueue(self.ctx.h, self.h, first, last), "fp_task_enqueue")

    def start(self, first: int) -> None:
        _lib.check(self.lib.fp_task_start(self.ctx.h, self.h, first), "fp_task_start")

    def poll(self) -> _lib.TaskStatus:
        st = _lib.TaskStatus()
        _lib.check(self.lib.fp_task_poll(self.ctx.h, self.h, C.byref(st)), "fp_task_poll")
        return st

    def logits(self) -> np.ndarray:
        out = np.empty((len(self.lens), self.ctx.shape.vocab), np.float32)
        _lib.check(self.lib.fp_task_logits(self.ctx.h, self.h, out.ctypes.data), "fp_task_logits")
        return out

    def entry_stamps(self) -> np.ndarray:
        """Device %globaltimer (ns) per entry: row 0 = GO decision (0: not executed), row 1 =
        STOP decision at that boundary (0: never stopped there)."""
        out = np.zeros((2, self.n_entries), np.uint64)
        _lib.check(self.lib.fp_task_entry_stamps(self.ctx.h, self.h, out.ctypes.data),
                   "fp_task_entry_stamps")
        return out

    def entry_durations_s(self) -> np.ndarray:
        """Executed duration of entries 0 .. n-2 in seconds (NaN where unknown): entry e-1
        ends at the STOP decision of boundary e if the task was stopped there, else at entry
        e's GO decision. The last entry has no successor boundary and is not covered."""
        go, stop = self.entry_stamps().astype(np.int64)
        end = np.where(stop[1:] > 0, stop[1:], go[1:])
        d = (end - go[:-1]).astype(np.float64) * 1e-9
        d[(go[:-1] == 0) | (end == 0)] = np.nan
        return d

    def max_entry_s(self) -> float:
        """Longest executed entry of this task (the wall-clock max_entry_duration,
        cost_model.py:185-188)."""
        d = self.entry_durations_s()
        return float(np.nanmax(d)) if np.isfinite(d).any() else 0.0

    def routing(self) -> tuple[np.ndarray, np.ndarray]:
        """MoE tap: (expert ids, weights) [rows, top_k] of the most recent gate entry."""
        sh = self.ctx.shape
        rows = max(self.lens) if len(self.lens) == 1 else sum(self.lens)
        ids = np.empty((rows, sh.top_k), np.int32)
        w = np.empty((rows, sh.top_k), np.float32)
        n = self.lib.fp_task_read_routing(self.ctx.h, self.h, ids.ctypes.data, w.ctypes.data,
                                          rows)
        if n < 0:
            _lib.check(n, "fp_task_read_routing")
        return ids[:n], w[:n]

    def read_kv(self, seq: int, layer: int) -> tuple[np.ndarray, np.ndarray]:
        sh = self.ctx.shape
        n = self.lens[seq]
        k = np.empty((n, sh.n_kv_heads // self.ctx.tp_size, sh.head_dim), np.uint16)
        v = np.empty_like(k)
        _lib.check(
            self.lib.fp_task_read_kv(self.ctx.h, self.h, seq, layer, k.ctypes.data, v.ctypes.data),
            "fp_task_read_kv",
        )
        return bf16_to_f32(k), bf16_to_f32(v)

    def destroy(self) -> None:
        if self.h is not None:
            _lib.check(self.lib.fp_task_destroy(self.ctx.h, self.h), "fp_task_destroy")
            self.h = None


def connect_tp_dist(ctx: PrefillContext, max_tokens: int, group=None) -> None:
    """One process per GPU: exchange the ranks' block handles over torch.distributed (any
    backend; the handles are 88-byte host objects) and map every peer's block."""
    import torch.distributed as dist

    mine = ctx.tp_export(max_tokens)
    handles: list = [None] * ctx.tp_size
    dist.all_gather_object(handles, mine, group=group)
    ctx.tp_import(handles)


class TPGroup:
    """A tensor-parallel group driven from one process.

    Each rank is a ``PrefillContext`` holding its Megatron shard. On one device the ranks share
    rank 0's stream and run in lock step (``fp_tp_enqueue_lockstep``); the device code -- the
    exchange GEMM, the peer-memory all-reduce, the rank-0 boundary decision ring -- is the same
    code a one-process-per-GPU deployment runs (``connect_tp_dist``). The group exposes the
    ``PrefillContext`` surface the engines use, so ``GpuEngine`` drives it unchanged.
    """

    def __init__(self, shape: ModelShape, tp: int, device=0, kv_pages: int = 256,
                 page_size: int = 128, max_pos: int = 65536, max_tokens: int = 8192):
        devices = list(device) if isinstance(device, (list, tuple)) else [device] * tp
        self.shape = shape
        self.tp_size = tp
        self.page_size = page_size
        self.max_tokens = max_tokens
        self.ranks = [PrefillContext(shape, devices[r], kv_pages, page_size, max_pos,
                                     tp_rank=r, tp_size=tp) for r in range(tp)]
        self.lib = self.ranks[0].lib
        arr = (C.c_void_p * tp)(*[c.h.value for c in self.ranks])
        _lib.check(self.lib.fp_tp_connect_local(arr, tp, max_tokens), "fp_tp_connect_local")
        self.stream_ptr = self.ranks[0].stream_ptr

    def init_random(self, seed: int, std: float = 0.02) -> None:
        for c in self.ranks:
            c.init_random(seed, std)

    def load_weights(self, w: dict) -> None:
        for c in self.ranks:  # full tensors; every rank keeps its shard
            c.load_weights(w)

    def create_task(self, tokens, chunk_tokens=None, granularity="operator",
                    task_id: int = 0) -> "TPTask":
        return TPTask(self, tokens, chunk_tokens, granularity, task_id)

    def signal(self) -> None:
        self.ranks[0].signal()  # only rank 0's device reads the flag

    def clear(self) -> None:
        for c in self.ranks:
            c.clear()

    def poll(self) -> _lib.Status:
        return self.ranks[0].poll()

    def sync(self) -> None:
        for c in self.ranks:
            c.sync()

    def free_pages(self) -> int:
        return min(c.free_pages() for c in self.ranks)

    def profile(self, on: bool) -> None:
        for c in self.ranks:
            c.profile(on)

    def drain_profile(self, max_records: int = 1 << 20) -> list[dict]:
        out = []
        for r, c in enumerate(self.ranks):
            for rec in c.drain_profile(max_records):
                rec["rank"] = r
                out.append(rec)
        return out

    def launch_count(self) -> int:
        return sum(c.launch_count() for c in self.ranks)

    def tp_counters(self) -> list[dict]:
        return [c.tp_counters() for c in self.ranks]

    def close(self) -> None:
        for c in reversed(self.ranks):  # followers first: they use rank 0's stream
            c.close()


class TPTask:
    """One prefill task replicated over the ranks of a ``TPGroup`` (identical entry lists)."""

    def __init__(self, group: TPGroup, tokens, chunk_tokens, granularity, task_id):
        self.group = group
        self.ctx = group
        self.lib = group.lib
        self.task_id = task_id
        self.parts = [c.create_task(tokens, chunk_tokens, granularity, task_id)
                      for c in group.ranks]
        self.lens = self.parts[0].lens
        self.n_entries = self.parts[0].n_entries

    def info(self) -> dict:
        return self.parts[0].info()

    def entry_info(self, i: int):
        return self.parts[0].entry_info(i)

    def begin_segment(self, first: int) -> None:
        for t in self.parts:
            t.begin_segment(first)

    def start(self, first: int) -> None:
        """The asynchronous launch worker (``fp_task_start``) drives ONE context. Ranks driven
        in lock step from one process cannot each run a worker (a rank's exchange kernel would
        wait for peers whose launches are queued behind it on the shared stream), so a
        ``TPGroup`` runs the virtual-clock parity driver (``engine.run_on_gpu``) only; the
        wall-clock driver runs tensor parallelism as one process per GPU, each rank a
        ``PrefillContext`` with its own worker (``connect_tp_dist``)."""
        raise NotImplementedError(
            "TPGroup tasks run under the virtual-clock driver only; for the wall-clock driver "
            "run one process per GPU (PrefillContext(tp_rank=..., tp_size=...) + connect_tp_dist)")

    def enqueue(self, first: int, last: int) -> None:
        n = self.group.tp_size
        ctxs = (C.c_void_p * n)(*[c.h.value for c in self.group.ranks])
        tasks = (C.c_void_p * n)(*[t.h.value for t in self.parts])
        _lib.check(self.lib.fp_tp_enqueue_lockstep(ctxs, tasks, n, first, last),
                   "fp_tp_enqueue_lockstep")

    def poll_all(self) -> list:
        return [t.poll() for t in self.parts]

    def poll(self) -> _lib.TaskStatus:
        sts = self.poll_all()
        if len({(s.state, s.cursor) for s in sts}) != 1:
            raise _lib.NativeError(
                "tensor-parallel ranks diverged: "
                + ", ".join(f"rank {r}: state {s.state} cursor {s.cursor}" for r, s in enumerate(sts)))
        return sts[0]

    def logits(self) -> np.ndarray:
        return self.parts[0].logits()  # lm_head is replicated; every rank holds the same logits

    def rank_logits(self) -> list:
        return [t.logits() for t in self.parts]

    def read_kv(self, seq: int, layer: int) -> tuple[np.ndarray, np.ndarray]:
        ks, vs = zip(*(t.read_kv(seq, layer) for t in self.parts))
        return np.concatenate(ks, axis=1), np.concatenate(vs, axis=1)  # heads are rank-major

    def destroy(self) -> None:
        for t in reversed(self.parts):
            t.destroy()
