"""Layer-spec builders for the benchmark/parity configurations (BASELINE.json
configs 2-3). Pure host data: (name, kind, param_count) lists in flat
parameter order, fed to make_shards (reference hook.cpp:30-61).
"""
from __future__ import annotations

from typing import List

from .api import LayerSpec


def gpt2_specs(layers: int = 12, d_model: int = 768, ffn_mult: int = 4, vocab: int = 50257,
               ctx: int = 1024, untied_head: bool = False) -> List[LayerSpec]:
    """GPT-2 tensors in the reference's order (model.cpp:39-64, plan_tensors).
    The defaults give GPT-2 small with a tied head: 124,439,808 parameters."""
    d, mu = d_model, ffn_mult
    out = [LayerSpec("wte", "embedding", vocab * d), LayerSpec("wpe", "positional_embedding", ctx * d)]
    for l in range(layers):
        p = f"h{l}."
        out += [
            LayerSpec(p + "ln1.g", "norm", d),
            LayerSpec(p + "ln1.b", "norm", d),
            LayerSpec(p + "attn.qkv.w", "attention_qkv", d * 3 * d),
            LayerSpec(p + "attn.qkv.b", "bias", 3 * d),
            LayerSpec(p + "attn.proj.w", "attention_out_proj", d * d),
            LayerSpec(p + "attn.proj.b", "bias", d),
            LayerSpec(p + "ln2.g", "norm", d),
            LayerSpec(p + "ln2.b", "norm", d),
            LayerSpec(p + "mlp.fc.w", "feed_forward", d * mu * d),
            LayerSpec(p + "mlp.fc.b", "bias", mu * d),
            LayerSpec(p + "mlp.proj.w", "feed_forward", mu * d * d),
            LayerSpec(p + "mlp.proj.b", "bias", d),
        ]
    out += [LayerSpec("ln_f.g", "norm", d), LayerSpec("ln_f.b", "norm", d)]
    if untied_head:
        out.append(LayerSpec("lm_head", "lm_head", d * vocab))
    return out


def llama3_8b_specs(layers: int = 32, d_model: int = 4096, kv_dim: int = 1024, ffn: int = 14336,
                    vocab: int = 128256) -> List[LayerSpec]:
    """Llama-3-8B parameter tensors in HF named_parameters order, mapped onto
    the reference's layer kinds: 8,030,261,248 parameters."""
    d = d_model
    out = [LayerSpec("embed_tokens", "embedding", vocab * d)]
    for l in range(layers):
        p = f"layers.{l}."
        out += [
            LayerSpec(p + "self_attn.q_proj", "attention_qkv", d * d),
            LayerSpec(p + "self_attn.k_proj", "attention_qkv", d * kv_dim),
            LayerSpec(p + "self_attn.v_proj", "attention_qkv", d * kv_dim),
            LayerSpec(p + "self_attn.o_proj", "attention_out_proj", d * d),
            LayerSpec(p + "mlp.gate_proj", "feed_forward", d * ffn),
            LayerSpec(p + "mlp.up_proj", "feed_forward", d * ffn),
            LayerSpec(p + "mlp.down_proj", "feed_forward", ffn * d),
            LayerSpec(p + "input_layernorm", "norm", d),
            LayerSpec(p + "post_attention_layernorm", "norm", d),
        ]
    out += [LayerSpec("norm", "norm", d), LayerSpec("lm_head", "lm_head", d * vocab)]
    return out
