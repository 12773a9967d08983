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


_WEIGHT_IDS = {
    "wq": _lib.W_Q,
    "wk": _lib.W_K,
    "wv": _lib.W_V,
    "wo": _lib.W_O,
    "w_gate": _lib.W_GATE,
    "w_up": _lib.W_UP,
    "w_down": _lib.W_DOWN,
    "attn_norm": _lib.W_ATTN_NORM,
    "ffn_norm": _lib.W_FFN_NORM,
    "bq": _lib.W_Q_BIAS,
    "bk": _lib.W_K_BIAS,
    "bv": _lib.W_V_BIAS,
    "q_norm": _lib.W_Q_NORM,
    "k_norm": _lib.W_K_NORM,
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
    ):
        self.lib = _lib.load()
        self.shape = shape
        self.page_size = page_size
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
        )
        h = C.c_void_p()
        _lib.check(
            self.lib.fp_ctx_create(device, C.byref(cfg), 0, 1, None, kv_pages, page_size,
                                   C.byref(h)),
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

    def read_kv(self, seq: int, layer: int) -> tuple[np.ndarray, np.ndarray]:
        sh = self.ctx.shape
        n = self.lens[seq]
        k = np.empty((n, sh.n_kv_heads, sh.head_dim), np.uint16)
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
