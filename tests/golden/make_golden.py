"""Generate the committed golden fixtures (run in the build container, not on the GPU box).

1. ``tiny_hf_logits.npz``: last-token logits of the tiny Llama (config 1 shape) computed by
   Hugging Face ``transformers.LlamaForCausalLM`` (fp32, eager attention) on seeded weights and
   tokens. This pins ``oracle/forward.py`` against an independent Llama implementation (the
   reference itself computes no tensors).
2. ``two_request_events.jsonl`` and ``config1_events.jsonl``: event logs produced by running the
   UNMODIFIED reference ``prefillsim.engine.run`` (imported from /root/reference/pkg/src or
   baseline/_ref). These are the scheduling goldens the GPU engine must reproduce bit-exactly.

Usage:  python tests/golden/make_golden.py
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import forward as F  # noqa: E402

TINY_SEED = 1234
TINY_LENS = [37, 130, 64, 201]


def hf_logits(shape: F.Shape, w: dict, tokens: list) -> np.ndarray:
    import torch
    from transformers import LlamaConfig, LlamaForCausalLM

    cfg = LlamaConfig(
        vocab_size=shape.vocab,
        hidden_size=shape.hidden,
        intermediate_size=shape.ffn,
        num_hidden_layers=shape.num_layers,
        num_attention_heads=shape.n_heads,
        num_key_value_heads=shape.n_kv_heads,
        head_dim=shape.head_dim,
        rope_theta=shape.rope_theta,
        rms_norm_eps=shape.rms_eps,
        tie_word_embeddings=False,
        max_position_embeddings=65536,
        attn_implementation="eager",
    )
    model = LlamaForCausalLM(cfg).float().eval()
    sd = {"model.embed_tokens.weight": w["embed"], "lm_head.weight": w["lm_head"],
          "model.norm.weight": w["final_norm"]}
    for l in range(shape.num_layers):
        p = f"model.layers.{l}."
        sd[p + "self_attn.q_proj.weight"] = w[f"{l}.wq"]
        sd[p + "self_attn.k_proj.weight"] = w[f"{l}.wk"]
        sd[p + "self_attn.v_proj.weight"] = w[f"{l}.wv"]
        sd[p + "self_attn.o_proj.weight"] = w[f"{l}.wo"]
        sd[p + "mlp.gate_proj.weight"] = w[f"{l}.w_gate"]
        sd[p + "mlp.up_proj.weight"] = w[f"{l}.w_up"]
        sd[p + "mlp.down_proj.weight"] = w[f"{l}.w_down"]
        sd[p + "input_layernorm.weight"] = w[f"{l}.attn_norm"]
        sd[p + "post_attention_layernorm.weight"] = w[f"{l}.ffn_norm"]
    model.load_state_dict({k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in sd.items()},
                          strict=True)
    out = []
    with torch.no_grad():
        for t in tokens:
            ids = torch.from_numpy(t.astype(np.int64))[None]
            out.append(model(input_ids=ids).logits[0, -1].numpy())
    return np.stack(out).astype(np.float32)


def hf_qwen_logits(shape: F.Shape, w: dict, tokens: list) -> np.ndarray:
    import torch

    if shape.qk_norm:
        from transformers import Qwen3Config as Cfg, Qwen3ForCausalLM as Model
    else:
        from transformers import Qwen2Config as Cfg, Qwen2ForCausalLM as Model
    kw = dict(vocab_size=shape.vocab, hidden_size=shape.hidden, intermediate_size=shape.ffn,
              num_hidden_layers=shape.num_layers, num_attention_heads=shape.n_heads,
              num_key_value_heads=shape.n_kv_heads, rope_theta=shape.rope_theta,
              rms_norm_eps=shape.rms_eps, tie_word_embeddings=False,
              max_position_embeddings=65536, attn_implementation="eager")
    if shape.qk_norm:
        kw["head_dim"] = shape.head_dim
    model = Model(Cfg(**kw)).float().eval()
    sd = {"model.embed_tokens.weight": w["embed"], "lm_head.weight": w["lm_head"],
          "model.norm.weight": w["final_norm"]}
    for l in range(shape.num_layers):
        p = f"model.layers.{l}."
        for hf, ours in (("self_attn.q_proj.weight", "wq"), ("self_attn.k_proj.weight", "wk"),
                         ("self_attn.v_proj.weight", "wv"), ("self_attn.o_proj.weight", "wo"),
                         ("mlp.gate_proj.weight", "w_gate"), ("mlp.up_proj.weight", "w_up"),
                         ("mlp.down_proj.weight", "w_down"),
                         ("input_layernorm.weight", "attn_norm"),
                         ("post_attention_layernorm.weight", "ffn_norm")):
            sd[p + hf] = w[f"{l}.{ours}"]
        if shape.qkv_bias:
            sd[p + "self_attn.q_proj.bias"] = w[f"{l}.bq"]
            sd[p + "self_attn.k_proj.bias"] = w[f"{l}.bk"]
            sd[p + "self_attn.v_proj.bias"] = w[f"{l}.bv"]
        if shape.qk_norm:
            sd[p + "self_attn.q_norm.weight"] = w[f"{l}.q_norm"]
            sd[p + "self_attn.k_norm.weight"] = w[f"{l}.k_norm"]
    missing = set(model.state_dict()) - set(sd)
    missing = {m for m in missing if "rotary" not in m}
    assert not missing, missing
    model.load_state_dict({k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in sd.items()},
                          strict=False)
    out = []
    with torch.no_grad():
        for t in tokens:
            ids = torch.from_numpy(t.astype(np.int64))[None]
            out.append(model(input_ids=ids).logits[0, -1].numpy())
    return np.stack(out).astype(np.float32)


def hf_qwen3_moe_logits(shape: F.Shape, w: dict, tokens: list) -> np.ndarray:
    """Last-token logits of HF ``Qwen3MoeForCausalLM`` (every layer sparse) in fp32."""
    import torch
    from transformers import Qwen3MoeConfig, Qwen3MoeForCausalLM

    cfg = Qwen3MoeConfig(vocab_size=shape.vocab, hidden_size=shape.hidden,
                         num_hidden_layers=shape.num_layers, num_attention_heads=shape.n_heads,
                         num_key_value_heads=shape.n_kv_heads, head_dim=shape.head_dim,
                         rope_theta=shape.rope_theta, rms_norm_eps=shape.rms_eps,
                         num_experts=shape.n_experts, num_experts_per_tok=shape.top_k,
                         moe_intermediate_size=shape.moe_ffn, norm_topk_prob=shape.norm_topk,
                         decoder_sparse_step=1, mlp_only_layers=[], tie_word_embeddings=False,
                         max_position_embeddings=65536, attn_implementation="eager")
    model = Qwen3MoeForCausalLM(cfg).float().eval()
    sd = {"model.embed_tokens.weight": w["embed"], "lm_head.weight": w["lm_head"],
          "model.norm.weight": w["final_norm"]}
    for l in range(shape.num_layers):
        p = f"model.layers.{l}."
        for hf, ours in (("self_attn.q_proj.weight", "wq"), ("self_attn.k_proj.weight", "wk"),
                         ("self_attn.v_proj.weight", "wv"), ("self_attn.o_proj.weight", "wo"),
                         ("self_attn.q_norm.weight", "q_norm"),
                         ("self_attn.k_norm.weight", "k_norm"),
                         ("input_layernorm.weight", "attn_norm"),
                         ("post_attention_layernorm.weight", "ffn_norm"),
                         ("mlp.gate.weight", "w_router"), ("mlp.experts.down_proj", "e_down")):
            sd[p + hf] = w[f"{l}.{ours}"]
        sd[p + "mlp.experts.gate_up_proj"] = np.concatenate([w[f"{l}.e_gate"], w[f"{l}.e_up"]],
                                                            axis=1)
    missing = {m for m in set(model.state_dict()) - set(sd) if "rotary" not in m}
    assert not missing, missing
    model.load_state_dict({k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in sd.items()},
                          strict=False)
    out = []
    with torch.no_grad():
        for t in tokens:
            ids = torch.from_numpy(t.astype(np.int64))[None]
            out.append(model(input_ids=ids).logits[0, -1].numpy())
    return np.stack(out).astype(np.float32)


def moe_golden() -> None:
    sh = F.SHAPES["tiny-moe"]
    w = F.make_weights(sh, TINY_SEED)
    toks = F.make_tokens(TINY_LENS, sh.vocab, TINY_SEED)
    ref = hf_qwen3_moe_logits(sh, w, toks)
    ours = F.forward_logits(sh, w, toks)
    err = np.abs(ours - ref).max()
    print("oracle vs HF tiny-moe: max abs err", err, "max |logit|", np.abs(ref).max())
    assert err < 1e-3, err
    np.savez_compressed(os.path.join(HERE, "tiny-moe_hf_logits.npz"), seed=TINY_SEED,
                        lens=np.array(TINY_LENS), logits=ref)


def reference_events() -> None:
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "prefillsim")):
            sys.path.insert(0, p)
            break
    from prefillsim import engine, workload
    from prefillsim.cost_model import CostParams
    from prefillsim.scheduler import PolicyConfig

    trace = workload.Trace((workload.Request(0, "file", 0.0, 8192, 6.0),
                            workload.Request(1, "text", 0.05, 256, 0.25)))
    res = engine.run(trace, PolicyConfig(), CostParams(), 0, record_events=True)
    res.write_event_log(os.path.join(HERE, "two_request_events.jsonl"))

    # config 1: 2-class trace, tiny 4-layer model, S-EDF operator preemption
    classes = [workload.TaskClass("file", 6833.0, 5186.0, 22390.0, 0.45, 6.0),
               workload.TaskClass("text", 590.0, 652.0, 3040.0, 0.55, 0.25)]
    tr = workload.generate_trace(classes, 2.5, 20.0, seed=1234)
    res = engine.run(tr, PolicyConfig(), CostParams(num_layers=4), 0, record_events=True)
    res.write_event_log(os.path.join(HERE, "config1_events.jsonl"))
    workload.save_trace(tr, os.path.join(HERE, "config1_trace.jsonl"))
    print("config1:", len(tr), "requests", res.commands)
    config2_step_trace()


def config2_step_trace() -> None:
    """bench.py's step workload: the first 128 requests (16 per GPU x 8 GPUs) of the config-2
    3-class trace (text 0.76 @0.25 s, search 0.20 @4.0 s, file 0.04 @6.0 s), made by
    the reference generate_trace (workload.py:162-198, rate 8, 300 s, seed 7). Committed so the
    bench's timed legs never import the reference."""
    from prefillsim import workload

    classes = [workload.TaskClass("text", 590.0, 652.0, 3040.0, 0.76, 0.25),
               workload.TaskClass("search", 5976.0, 3456.0, 16635.0, 0.20, 4.0),
               workload.TaskClass("file", 6833.0, 5186.0, 22390.0, 0.04, 6.0)]
    tr = workload.generate_trace(classes, 8.0, 300.0, seed=7)
    head = workload.Trace(tuple(tr.requests[:128]))
    workload.save_trace(head, os.path.join(HERE, "config2_step_trace.jsonl"))
    print("config2 step trace:", [r.num_tokens for r in head.requests[:16]])


def main() -> None:
    shape = F.SHAPES["tiny"]
    w = F.make_weights(shape, TINY_SEED)
    tokens = F.make_tokens(TINY_LENS, shape.vocab, TINY_SEED)
    ref = hf_logits(shape, w, tokens)
    ours = F.forward_logits(shape, w, tokens)
    err = np.abs(ours - ref).max()
    print("oracle vs HF max abs err:", err, "max |logit|", np.abs(ref).max())
    assert err < 1e-3, err
    np.savez_compressed(os.path.join(HERE, "tiny_hf_logits.npz"), seed=TINY_SEED,
                        lens=np.array(TINY_LENS), logits=ref)
    for name in ("tiny-qwen3", "tiny-qwen2"):
        sh = F.SHAPES[name]
        wq = F.make_weights(sh, TINY_SEED)
        toks = F.make_tokens(TINY_LENS, sh.vocab, TINY_SEED)
        ref = hf_qwen_logits(sh, wq, toks)
        ours = F.forward_logits(sh, wq, toks)
        err = np.abs(ours - ref).max()
        print(f"oracle vs HF {name}: max abs err", err, "max |logit|", np.abs(ref).max())
        assert err < 1e-3, err
        np.savez_compressed(os.path.join(HERE, f"{name}_hf_logits.npz"), seed=TINY_SEED,
                            lens=np.array(TINY_LENS), logits=ref)
    reference_events()


if __name__ == "__main__":
    if "--moe" in sys.argv:
        moe_golden()
    elif "--config2" in sys.argv:
        for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
            if os.path.isdir(os.path.join(p, "prefillsim")):
                sys.path.insert(0, p)
                break
        config2_step_trace()
    else:
        main()
        moe_golden()
