"""The CPU numeric oracle's own consistency (no GPU): the capture / partial-
last-layer prefill and the decode-over-a-given-cache entry points used by the
BASELINE-size parity tests (tests/test_parity_baseline_gpu.py) must
reproduce the plain dense generate() path they shortcut."""
import numpy as np

from oracle import llama_ref
from paper_2404_09526_b200 import abi


def _bf16_bits(a):
    return (np.asarray(a, np.float32).view(np.uint32) >> 16).astype(np.uint16)


def test_prefill_probe_matches_generate():
    shape = abi.TINY
    S = 600
    prompt = np.random.default_rng(3).integers(0, shape.vocab, S).astype(np.int32)
    tok, lg = llama_ref.generate(shape, prompt, 0, emulate_bf16=True)
    pos = [0, 7, 300, S - 1]
    for last_only in (True, False):
        t, l, att, k, v = llama_ref.prefill_probe(shape, prompt, attn_pos=pos, kv_pos=pos,
                                                 last_only=last_only)
        assert t == tok[0]
        assert np.array_equal(l, lg[0])
        assert att.shape == (shape.layers, len(pos), shape.hidden)
        assert np.isfinite(att).all() and np.abs(att).max() > 0
    # the partial last layer captures the same rows as the full one
    _, _, a1, k1, v1 = llama_ref.prefill_probe(shape, prompt, attn_pos=pos, kv_pos=pos)
    _, _, a2, k2, v2 = llama_ref.prefill_probe(shape, prompt, attn_pos=pos, kv_pos=pos,
                                               last_only=False)
    assert np.array_equal(a1, a2) and np.array_equal(k1, k2) and np.array_equal(v1, v2)


def test_decode_cached_matches_generate():
    """A decode step over the oracle's own (bf16-exact) cache == generate's step."""
    shape = abi.TINY
    S = 500
    prompt = np.random.default_rng(4).integers(0, shape.vocab, S).astype(np.int32)
    tok, lg = llama_ref.generate(shape, prompt, 1, emulate_bf16=True)
    _, _, _, K, V = llama_ref.prefill_probe(shape, prompt, kv_pos=list(range(S)))
    t, l, kn, vn, att = llama_ref.decode_cached(shape, _bf16_bits(K), _bf16_bits(V), tok[0])
    assert t == tok[1]
    assert np.array_equal(l, lg[1])
    # the step's own K/V row equals what a prefill of prompt + token caches
    # (up to summation order: the many-row prefill GEMM blocks differently,
    # and bf16 rounding of K/V may flip a last bit)
    full = np.concatenate([prompt, [tok[0]]]).astype(np.int32)
    _, _, _, K2, V2 = llama_ref.prefill_probe(shape, full, kv_pos=[S])
    for a, b in ((kn, K2[:, 0]), (vn, V2[:, 0])):
        assert np.linalg.norm(a - b) / np.linalg.norm(b) < 5e-3


def test_fp32_mode_is_the_unrounded_forward():
    """emulate_bf16=0 (the fp32 check mode) differs from the bf16-emulation
    mode by bf16 rounding only (rel-L2 of logits ~1e-3, not 0 and not O(1))."""
    shape = abi.TINY
    prompt = np.random.default_rng(5).integers(0, shape.vocab, 300).astype(np.int32)
    _, l32 = llama_ref.generate(shape, prompt, 0, emulate_bf16=False)
    _, l16 = llama_ref.generate(shape, prompt, 0, emulate_bf16=True)
    r = np.linalg.norm(l32 - l16) / np.linalg.norm(l32)
    assert 1e-5 < r < 3e-2, r
