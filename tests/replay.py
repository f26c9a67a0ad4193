"""Replays a reference scenario (tests/golden/scenario_*.jsonl, recorded by
oracle/golden_driver.cpp around the UNMODIFIED reference engine) through the
B200 runtime's C-ABI, exactly as the TapPolicy of INTEGRATION.md does:

  at every schedule() call
    1. reconcile engine-internal changes that happened since the last call,
       using ONLY the engine's own events: finish / evict -> esp_free_request;
       "displaced" (engine.cpp:587-648) and "handoff" (engine.cpp:194-244)
       migrations -> esp_move_kv;
    2. require the runtime's page tables == the engine's Request.placement and
       ElasticInstance.kv_used (bit-exact);
    3. execute the ScheduleDecision in apply_decision order (engine.cpp:246-490):
       migrations -> esp_move_kv, prefills -> esp_prefill, decode steps ->
       esp_decode_step (with any chunked-prefill chunk riding on the step).
"""
import json

import numpy as np


def load(path):
    with open(path) as f:
        lines = [json.loads(l) for l in f if l.strip()]
    head = lines[0]
    steps = [l for l in lines if l["kind"] == "step"]
    final = [l for l in lines if l["kind"] == "final"][0]
    return head, steps, final


def prompt_tokens(request_id, n, vocab=32000, seed=7):
    """Synthetic prompt of a request: uniform token ids, seeded per request."""
    rng = np.random.default_rng([seed, request_id])
    return rng.integers(0, vocab, n, dtype=np.int64).astype(np.int32)


def placement_of(state):
    return {int(r): {int(i): int(t) for i, t in pl} for r, pl in state["placement"].items()}


def reconcile(rt, events, expected):
    displaced = set()
    for e in events:
        if e["kind"] in ("finish", "evict"):
            rt.free_request(e["request"])
        elif e["kind"] == "migration" and e["detail"] in ("displaced", "handoff"):
            # engine-internal KV moves: resolve_foreign_kv (engine.cpp:587-648)
            # and the disaggregation handoff (engine.cpp:194-244)
            displaced.add(e["request"])
    exp = placement_of(expected)
    for r in sorted(displaced):
        have = rt.placement(r)
        want = exp.get(r, {})
        surplus = [(i, have.get(i, 0) - want.get(i, 0)) for i in sorted(have)
                   if have.get(i, 0) > want.get(i, 0)]
        deficit = [(i, want.get(i, 0) - have.get(i, 0)) for i in sorted(want)
                   if want.get(i, 0) > have.get(i, 0)]
        si = di = 0
        while si < len(surplus) and di < len(deficit):
            (a, na), (b, nb) = surplus[si], deficit[di]
            mv = min(na, nb)
            rt.move_kv(r, a, b, mv)
            surplus[si] = (a, na - mv)
            deficit[di] = (b, nb - mv)
            if surplus[si][1] == 0:
                si += 1
            if deficit[di][1] == 0:
                di += 1


def assert_state(rt, expected, known_requests, where=""):
    exp = placement_of(expected)
    for r in known_requests:
        got = rt.placement(r)
        assert got == exp.get(r, {}), f"{where}: request {r}: runtime {got} != engine {exp.get(r)}"
    assert rt.kv_used() == expected["kv_used"], f"{where}: kv_used {rt.kv_used()} != {expected['kv_used']}"


def execute(rt, decision, head, on_prefill=None, on_decode=None):
    for m in decision["migrations"]:
        for (req, src, dst, tok) in m["moves"]:
            rt.move_kv(req, src, dst, tok)
    for p in decision["prefills"]:
        reqs = p["requests"]
        retain = [[tuple(x) for x in p["placement"][str(r)]] for r in reqs]
        if on_prefill is not None:
            on_prefill(p, retain)
        else:
            rt.prefill(reqs, p["input_lens"], p["instances"], retain)
    for d in decision["decode_steps"]:
        members = sorted(d["members"] + d["add_instances"])
        if on_decode is not None:
            on_decode(d, members)
        else:
            rt.decode_step(members, d["masters"], d["batch"], chunk=chunk_of(d))


def chunk_of(d, tokens=None):
    """The chunked-prefill chunk riding on a recorded decode step (None if
    none): placement in KvPlacement order, final iff it completes the prompt
    (engine.cpp:570-579); tokens = the full prompt of the request (sliced)."""
    if d.get("chunk_request", -1) < 0 or d.get("chunk_tokens", 0) <= 0:
        return None
    p0, n = d["chunk_prefilled"], d["chunk_tokens"]
    return {"request": d["chunk_request"],
            "placement": [tuple(x) for x in d["chunk_placement"]],
            "final": p0 + n == d["chunk_input_len"],
            "tokens": None if tokens is None else tokens[p0:p0 + n]}


def replay(rt, path, on_prefill=None, on_decode=None, conservation=False):
    head, steps, final = load(path)
    known = [r["id"] for r in head["requests"]]
    for st in steps:
        reconcile(rt, st["events"], st["before"])
        assert_state(rt, st["before"], known, where=f"step k={st['k']}")
        if conservation:
            rt.check_conservation()
        execute(rt, st["decision"], head, on_prefill, on_decode)
    reconcile(rt, final["events"], final["state"])
    assert_state(rt, final["state"], known, where="final")
    return head, steps, final
