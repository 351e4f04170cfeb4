"""Tensor inventories used by tests, fixtures and bench.

Registration order follows ``model.named_parameters()`` of the HF Llama /
Qwen2 modules (self_attn q,k,v,o, mlp gate,up,down, then the two norms),
which is the order the reference manifest packs in (manifest.cpp:179-202).
"""
from __future__ import annotations

import numpy as np


def llama_shapes(hidden=4096, layers=32, kv=1024, ffn=14336, vocab=128256, qkv_bias=False):
    out = [("model.embed_tokens.weight", (vocab, hidden))]
    for i in range(layers):
        p = f"model.layers.{i}."
        out += [(p + "self_attn.q_proj.weight", (hidden, hidden))]
        if qkv_bias:
            out += [(p + "self_attn.q_proj.bias", (hidden,))]
        out += [(p + "self_attn.k_proj.weight", (kv, hidden))]
        if qkv_bias:
            out += [(p + "self_attn.k_proj.bias", (kv,))]
        out += [(p + "self_attn.v_proj.weight", (kv, hidden))]
        if qkv_bias:
            out += [(p + "self_attn.v_proj.bias", (kv,))]
        out += [(p + "self_attn.o_proj.weight", (hidden, hidden)),
                (p + "mlp.gate_proj.weight", (ffn, hidden)),
                (p + "mlp.up_proj.weight", (ffn, hidden)),
                (p + "mlp.down_proj.weight", (hidden, ffn)),
                (p + "input_layernorm.weight", (hidden,)),
                (p + "post_attention_layernorm.weight", (hidden,))]
    out += [("model.norm.weight", (hidden,)), ("lm_head.weight", (vocab, hidden))]
    return out


def llama3_8b_shapes():
    return llama_shapes()


def qwen25_32b_shapes():
    return llama_shapes(hidden=5120, layers=64, kv=1024, ffn=27648, vocab=152064, qkv_bias=True)


def llama3_70b_shapes():
    return llama_shapes(hidden=8192, layers=80, kv=1024, ffn=28672, vocab=128256)


def nbytes(shape, elem=2):
    n = 1
    for d in shape:
        n *= d
    return n * elem


def llama3_8b():
    shapes = llama3_8b_shapes()
    return [n for n, _ in shapes], [nbytes(s) for _, s in shapes]


def config1():
    """BASELINE config 1: 16 tensors w{0..15} of [8192, 4096] bf16 (1 GiB)."""
    return [(f"w{i}", (8192, 4096)) for i in range(16)]


TINY_SET = [("big", 3 << 20, 11), ("t1", 1000, 12), ("t2", 2000, 13), ("odd", 12345, 14),
            ("w", 200000, 15), ("u", 777, 16), ("mid", 1 << 20, 17)]


def tiny_set():
    """A small mixed set with real bytes (fill_pattern of the reference
    ClusterFix, test_client_core.cpp:76-81)."""
    names, arrays = [], []
    for name, n, salt in TINY_SET:
        names.append(name)
        arrays.append(((salt * 1315423911 + np.arange(n, dtype=np.uint64) * 131) & 0xFF).astype(np.uint8))
    return names, arrays
