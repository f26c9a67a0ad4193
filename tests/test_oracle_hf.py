"""Pins the numeric oracle (oracle/llama_ref.c) to an independent, published
implementation of the same architecture: HuggingFace transformers'
LlamaForCausalLM (the installed transformers 5.5), run in fp32 on the CPU
with the oracle's own synthetic weights loaded.

The reference (espsim) has no numeric path, and LWM-7B is the
Llama-2-7B architecture, so this is what "same accuracy as the
original implementations" can be anchored on: the oracle that
every GPU parity test compares against must reproduce the stock Llama forward
(RMSNorm with unit gains, rotate-half RoPE with theta 10000, SiLU-gated MLP,
causal softmax attention, untied LM head) to fp32 round-off — on the tiny
config 1 model and on one layer of the LWM-7B geometry (hidden 4096, 32 x 128
heads, FFN 11008). Also checks the numpy restatement of the synthetic weight
definition (synthetic.h) bit-exactly against the oracle's.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import llama_ref
from paper_2404_09526_b200.abi import TINY, ModelShape

torch = pytest.importorskip("torch")
transformers = pytest.importorskip("transformers")


def _synthetic_np(seed, tensor, layer, rows, cols, cols_total):
    """synthetic.h restated with numpy uint64 wrap-around, then bf16 RNE."""
    with np.errstate(over="ignore"):
        idx = (rows.astype(np.uint64) * np.uint64(cols_total) + cols.astype(np.uint64))
        key = (np.uint64(tensor) << np.uint64(56)) ^ (np.uint64(layer) << np.uint64(48)) ^ idx
        h = _splitmix64_np(np.uint64(seed) ^ _splitmix64_np(key))
    s = ((h & np.uint64(0xFFFF)).astype(np.int64) + ((h >> np.uint64(16)) & np.uint64(0xFFFF)).astype(np.int64)
         + ((h >> np.uint64(32)) & np.uint64(0xFFFF)).astype(np.int64) + (h >> np.uint64(48)).astype(np.int64))
    x = (s - 131070).astype(np.float32) * np.float32(5.2857997e-07)
    b = x.view(np.uint32)
    b = ((b + np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000))
    return b.view(np.float32)


def _splitmix64_np(x):
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def test_synthetic_weights_numpy_restatement():
    rng = np.random.default_rng(0)
    for tensor, layer, rows, cols in [(2, 0, 512, 512), (6, 1, 1536, 512), (1, 0, 32000, 512),
                                      (8, 31, 4096, 11008)]:
        r = rng.integers(0, rows, 64)
        c = rng.integers(0, cols, 64)
        want = np.array([llama_ref.weight(1234, tensor, layer, int(a), int(b), cols)
                         for a, b in zip(r, c)], np.float32)
        got = _synthetic_np(1234, tensor, layer, r, c, cols)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    w = llama_ref.weights(TINY, "q", 1, 8, 512)
    got = _synthetic_np(1234, 2, 1, np.repeat(np.arange(8), 512), np.tile(np.arange(512), 8), 512)
    assert np.array_equal(w.reshape(-1).view(np.uint32), got.view(np.uint32))


def _hf_model(shape):
    cfg = transformers.LlamaConfig(
        vocab_size=shape.vocab, hidden_size=shape.hidden, intermediate_size=shape.ffn,
        num_hidden_layers=shape.layers, num_attention_heads=shape.heads,
        num_key_value_heads=shape.heads, head_dim=shape.head_dim, rms_norm_eps=shape.rms_eps,
        rope_theta=shape.rope_theta, max_position_embeddings=4096, tie_word_embeddings=False,
        attention_bias=False, mlp_bias=False, hidden_act="silu")
    cfg._attn_implementation = "eager"
    model = transformers.LlamaForCausalLM(cfg).float().eval()
    H, F, V = shape.hidden, shape.ffn, shape.vocab

    def t(name, layer, rows, cols):
        return torch.from_numpy(llama_ref.weights(shape, name, layer, rows, cols))

    with torch.no_grad():
        model.model.embed_tokens.weight.copy_(t("embed", 0, V, H))
        model.lm_head.weight.copy_(t("lm_head", 0, V, H))
        model.model.norm.weight.fill_(1.0)
        for layer_idx, blk in enumerate(model.model.layers):
            blk.self_attn.q_proj.weight.copy_(t("q", layer_idx, H, H))
            blk.self_attn.k_proj.weight.copy_(t("k", layer_idx, H, H))
            blk.self_attn.v_proj.weight.copy_(t("v", layer_idx, H, H))
            blk.self_attn.o_proj.weight.copy_(t("o", layer_idx, H, H))
            blk.mlp.gate_proj.weight.copy_(t("gate", layer_idx, F, H))
            blk.mlp.up_proj.weight.copy_(t("up", layer_idx, F, H))
            blk.mlp.down_proj.weight.copy_(t("down", layer_idx, H, F))
            blk.input_layernorm.weight.fill_(1.0)
            blk.post_attention_layernorm.weight.fill_(1.0)
    return model


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("shape,S,steps", [
    (TINY, 96, 4),
    (ModelShape(layers=1, hidden=4096, heads=32, head_dim=128, ffn=11008, vocab=512), 40, 2),
], ids=["tiny_config1", "lwm7b_layer"])
def test_oracle_matches_hf_llama_fp32(shape, S, steps):
    """Prefill logits and teacher-forced decode-step logits of the fp32 oracle
    (dense prefill + KV-cached decode) against HF LlamaForCausalLM over the
    full sequence, on the same synthetic weights: rel-L2 <= 1e-4 per position
    (fp32 round-off of different summation orders), same greedy tokens."""
    torch.set_num_threads(max(1, min(16, torch.get_num_threads())))
    prompt = np.random.default_rng(5).integers(0, shape.vocab, S).astype(np.int32)
    toks, lg = llama_ref.generate(shape, prompt, steps, emulate_bf16=False)
    model = _hf_model(shape)
    seq = np.concatenate([prompt, toks[:steps]]).astype(np.int64)
    with torch.no_grad():
        out = model(torch.from_numpy(seq)[None]).logits[0].numpy()
    for s in range(steps + 1):
        ref = out[S - 1 + s]
        assert _rel(lg[s], ref) <= 1e-4, (s, _rel(lg[s], ref))
        assert int(np.argmax(ref)) == int(toks[s]), s
