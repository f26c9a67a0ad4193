"""Tensor-parallel instances (paper TP = 2 x ESP = 4,
PAPER.md:450): every instance spans tp planes (here all on GPU 0, one stream
each), plane r holding heads [r H/tp, (r+1) H/tp) of the KV and the Megatron
weight shards; the O / down partials are all-reduced across the planes.
ESP ring prefill with proactive scale-down and multi-master decode run on
top, unchanged. Checked against the dense CPU oracle with the measured-floor
rule of tests/test_e2e_gpu.py (the oracle is itself pinned to HF Llama,
tests/test_oracle_hf.py)."""
import os

import numpy as np
import pytest

from paper_2404_09526_b200 import abi
from tests import replay
from tests.test_e2e_gpu import GOLD, Recorder, check_against_oracle

pytestmark = pytest.mark.gpu
LWM7B_2L = abi.ModelShape(layers=2, hidden=4096, heads=32, head_dim=128, ffn=11008, vocab=32000)


@pytest.mark.parametrize("shape,tp,d,S,steps", [
    (abi.TINY, 2, 2, 1500, 4),
    (abi.TINY, 4, 1, 700, 3),
    (LWM7B_2L, 2, 2, 2048, 2),
    # (LWM-7B's FFN 11008 = 172 blocks of 64 splits over tp = 2 or 4, not 8)
    (abi.ModelShape(layers=1, hidden=4096, heads=32, head_dim=128, ffn=11008, vocab=512), 4, 2,
     1024, 2),
], ids=["tiny_tp2_esp2", "tiny_tp4_esp1", "lwm7b_2layers_tp2_esp2", "lwm7b_layer_tp4_esp2"])
def test_tp_prefill_decode_vs_oracle(shape, tp, d, S, steps):
    prompt = np.random.default_rng(tp * 10 + d).integers(0, shape.vocab, S).astype(np.int32)
    rt = abi.Runtime(shape, max(d, 2), kv_capacity=2 * S + 64, tp_planes=[0] * tp)
    try:
        ring = list(range(d))
        # retention onto 2 survivors when the ring has them (scale-down d -> 2)
        retain = [[(d - 1, S // 3), (0, S - S // 3)]] if d > 1 else [[(0, S)]]
        first, lg0, _ = rt.prefill([7], [S], ring, retain, tokens=prompt, want_logits=True)
        assert rt.placement(7) == {i: t for i, t in retain[0]}
        toks, logits = [int(first[0])], [lg0[0]]
        members = sorted({i for i, _ in retain[0]})
        for _ in range(steps):
            out, lg, _ = rt.decode_step(members, [0], [7], want_logits=True)
            toks.append(int(out[0]))
            logits.append(lg[0])
        rt.check_conservation()
    finally:
        rt.close()
    check_against_oracle(shape, prompt, toks, logits)


@pytest.mark.parametrize("tp,lens", [(2, (1027, 333)), (4, (1031,))], ids=["tp2_ragged", "tp4_ragged"])
def test_tp_reduce_scatter_bit_identical_to_all_reduce(tp, lens, monkeypatch):
    """Prefill (rows >= 128 per plane) runs the all-reduces as a reduce-scatter
    fused into the O / down GEMM epilogues (row block q stored into plane q's
    buffer) + a reduction that stores x / xn to the planes; decode rows take
    the all-reduce. Both sum the partials in plane order, so the logits are
    bit-identical to forcing the all-reduce everywhere — here on row counts
    tp does not divide, two requests in one prefill."""
    shape = abi.TINY
    rng = np.random.default_rng(29)
    prompts = [rng.integers(0, shape.vocab, n).astype(np.int32) for n in lens]
    outs = []
    for force in (False, True):
        if force:
            monkeypatch.setenv("ESP_TP_ALLREDUCE", "1")
        rt = abi.Runtime(shape, 2, kv_capacity=8192, tp_planes=[0] * tp)
        try:
            ids = list(range(len(lens)))
            first, lg, _ = rt.prefill(ids, list(lens), [0, 1], [[(0, n)] for n in lens],
                                      tokens=np.concatenate(prompts), want_logits=True)
            dec = rt.decode_step([0], [0], ids, want_logits=True)
            outs.append((np.asarray(first).copy(), np.asarray(lg).copy(), np.asarray(dec[1]).copy()))
        finally:
            rt.close()
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)


def test_tp_multi_request_two_masters():
    """Two requests decoded together by two masters (requests dealt by
    assign_masters), KV of each on both instances, tp = 2: each request's
    logits against the oracle."""
    shape, tp = abi.TINY, 2
    rt = abi.Runtime(shape, 2, kv_capacity=8192, tp_planes=[0] * tp)
    rng = np.random.default_rng(5)
    prompts = {r: rng.integers(0, shape.vocab, n).astype(np.int32) for r, n in ((0, 900), (1, 1300))}
    toks = {r: [] for r in prompts}
    logits = {r: [] for r in prompts}
    try:
        for r, p in prompts.items():
            S = len(p)
            first, lg, _ = rt.prefill([r], [S], [0, 1], [[(0, S // 2), (1, S - S // 2)]], tokens=p,
                                      want_logits=True)
            toks[r].append(int(first[0]))
            logits[r].append(lg[0])
        for _ in range(3):
            out, lg, _ = rt.decode_step([0, 1], [0, 1], [0, 1], want_logits=True)
            for i, r in enumerate((0, 1)):
                toks[r].append(int(out[i]))
                logits[r].append(lg[i])
        rt.check_conservation()
    finally:
        rt.close()
    for r, p in prompts.items():
        check_against_oracle(shape, p, toks[r], logits[r])


@pytest.mark.parametrize("scenario", ["config1_tiny", "tiny_multi", "tiny_preempt"])
def test_tp_replays_reference_scenarios(scenario):
    """The reference engine's recorded decisions (tests/golden/scenario_*.jsonl:
    config 1; 8 requests with varlen ring prefills, multi-master decode and
    scale-up/down; a trace whose engine displaces paused KV onto group mates)
    executed on a tp = 2 runtime: page tables equal the engine's at every
    schedule() (tests/replay.py), KV moves copy every plane's shard, and every
    request's logits match the oracle."""
    path = os.path.join(GOLD, f"scenario_{scenario}.jsonl")
    head, _, _ = replay.load(path)
    rt = abi.Runtime(abi.TINY, head["instances"], kv_capacity=head["kv_capacity"],
                     tp_planes=[0, 0])
    rec = Recorder(rt)
    try:
        replay.replay(rt, path, on_prefill=rec.prefill, on_decode=rec.decode, conservation=True)
    finally:
        rt.close()
    for r, lgs in rec.logits.items():
        toks = [int(np.argmax(l)) for l in lgs]
        check_against_oracle(abi.TINY, rec.prompts[r], toks, lgs)


@pytest.mark.parametrize("tp", [2, 4])
def test_tp_chunked_prefill_replay(tp):
    """The reference's "chunked:512" decisions (scenario_tiny_chunked.jsonl,
    policies.cpp:297-405) on tp planes: prompt chunks ride on decode steps
    (engine.cpp:432-462), each chunk's rows attend per plane over its head
    shard of the gathered earlier KV + the chunk (one causal segment offset
    by the chunk start); tokens and logits against the dense oracle."""
    path = os.path.join(GOLD, "scenario_tiny_chunked.jsonl")
    head, _, _ = replay.load(path)
    rt = abi.Runtime(abi.TINY, head["instances"], kv_capacity=head["kv_capacity"],
                     tp_planes=[0] * tp)
    prompts = {r["id"]: replay.prompt_tokens(r["id"], r["input_len"]) for r in head["requests"]}
    toks = {r: [] for r in prompts}
    logits = {r: [] for r in prompts}

    def on_decode(d, members):
        ch = replay.chunk_of(d, prompts.get(d["chunk_request"]))
        out, lg, _ = rt.decode_step(members, d["masters"], d["batch"], want_logits=True, chunk=ch)
        for i, r in enumerate(d["batch"]):
            toks[r].append(int(out[i]))
            logits[r].append(lg[i])
        if ch is not None and ch["final"]:
            toks[ch["request"]].append(ch["first_token"])
            logits[ch["request"]].append(ch["logits"])

    try:
        replay.replay(rt, path, on_decode=on_decode, conservation=True)
    finally:
        rt.close()
    for r, p in prompts.items():
        assert toks[r], r
        check_against_oracle(abi.TINY, p, toks[r], logits[r])


def test_tp_read_kv_assembles_plane_shards():
    """read_kv on tp planes: plane p's slab holds columns [p H/tp, (p+1) H/tp)
    of every slot; the readback assembles them per token position and agrees
    with tp = 1's to bf16 rounding (layer 0: the same QKV dot products on a
    smaller GEMM shape, a few ulp apart; a misplaced shard would be O(1) off).
    A KV move (every plane's shard copied) leaves the readback unchanged."""
    shape = abi.TINY
    S = 700
    p = np.random.default_rng(4).integers(0, shape.vocab, S).astype(np.int32)
    reads = {}
    for tp in (1, 2):
        kw = {"tp_planes": [0] * tp} if tp > 1 else {"devices": [0, 0]}
        rt = abi.Runtime(shape, 2, kv_capacity=4096, **kw)
        try:
            rt.prefill([1], [S], [0, 1], [[(1, 300), (0, S - 300)]], tokens=p)
            reads[tp] = [rt.read_kv(1, l) for l in range(shape.layers)]
            if tp > 1:
                rt.move_kv(1, 1, 0, 300)
                assert rt.placement(1) == {0: S}
                moved = [rt.read_kv(1, l) for l in range(shape.layers)]
                for (k0, v0), (k1, v1) in zip(reads[tp], moved):
                    assert np.array_equal(k0, k1) and np.array_equal(v0, v1)
        finally:
            rt.close()
    for l in range(shape.layers):
        for a, b in zip(reads[1][l], reads[2][l]):
            assert a.shape == b.shape == (S, shape.hidden)
            fa, fb = abi.bf16_to_f32(a), abi.bf16_to_f32(b)
            tol = 5e-3 if l == 0 else 2e-2
            assert np.linalg.norm(fa - fb) <= tol * np.linalg.norm(fa), l


def test_tp_attention_capture_assembles_plane_shards():
    """Attention capture on tp planes: each plane copies its head columns of
    the captured stripe rows after K1; the capture assembles them per
    position and agrees with tp = 1's to bf16 rounding (a misplaced shard or
    stripe row would be O(1) off)."""
    shape, S, d = abi.TINY, 900, 2
    p = np.random.default_rng(8).integers(0, shape.vocab, S).astype(np.int32)
    pos = [0, 1, 7, 450, 451, S - 1]
    caps = {}
    for tp in (1, 2):
        kw = {"tp_planes": [0] * tp} if tp > 1 else {"devices": [0] * d}
        rt = abi.Runtime(shape, d, kv_capacity=4096, **kw)
        try:
            rt.capture_attention(pos)
            rt.prefill([1], [S], list(range(d)), [[(0, S)]], tokens=p)
            caps[tp] = abi.bf16_to_f32(rt.captured_attention())
        finally:
            rt.close()
    assert caps[1].shape == caps[2].shape == (shape.layers, len(pos), shape.hidden)
    for l in range(shape.layers):
        a, b = caps[1][l], caps[2][l]
        tol = 1e-2 if l == 0 else 3e-2
        assert np.linalg.norm(a - b) <= tol * np.linalg.norm(a), l


@pytest.mark.parametrize("tp", [1, 2])
def test_chunk_only_steps_contiguous_slots(tp):
    """A prompt prefilled only by chunks (chunk-only decode steps, no decode
    batch) on a fresh instance: its slots form one ascending run, so the
    chunk attention reads K/V straight from the slab rows instead of
    gathering them (the fast path of the chunked-prefill baseline); then two
    decode steps. First token + logits against the dense oracle."""
    shape, S, C = abi.TINY, 1300, 512
    prompt = np.random.default_rng(31).integers(0, shape.vocab, S).astype(np.int32)
    kw = {"tp_planes": [0] * tp} if tp > 1 else {"devices": [0]}
    rt = abi.Runtime(shape, 1, kv_capacity=4096, **kw)
    toks, logits = [], []
    try:
        for p0 in range(0, S, C):
            n = min(C, S - p0)
            ch = {"request": 5, "placement": [(0, n)], "tokens": prompt[p0:p0 + n],
                  "final": p0 + n == S}
            rt.decode_step([0], [], [], want_logits=True, chunk=ch)
            if ch["final"]:
                toks.append(int(ch["first_token"]))
                logits.append(np.asarray(ch["logits"]).reshape(-1))
        for _ in range(2):
            out, lg, _ = rt.decode_step([0], [0], [5], want_logits=True)
            toks.append(int(out[0]))
            logits.append(lg[0])
        rt.check_conservation()
    finally:
        rt.close()
    check_against_oracle(shape, prompt, toks, logits)
