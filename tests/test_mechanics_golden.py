"""The hot-path placement mechanics — both the product's host C++ mirror
(through the C-ABI) and the oracle's Python restatement — against
(a) seeded random cases whose expected outputs were produced by running the
reference library itself (tests/golden/mechanics_random.jsonl) and
(b) the known-answer vectors of the reference's own unit tests."""
import json
import os

import pytest

from oracle import placement as P
from paper_2404_09526_b200 import abi

GOLD = os.path.join(os.path.dirname(__file__), "golden", "mechanics_random.jsonl")
with open(GOLD) as f:
    CASES = [json.loads(l) for l in f if l.strip()]

SIB_PATH_ROWS = [  # /root/reference/proj/configs/default_sib.jsonl:1-8
    dict(dop=d, tp=1, alpha_p=4.0 + d, beta_p=0.08 / d, gamma_p=4.8e-08 / d,
         alpha_d=4.0 + 0.8 * d, beta_d=0.06, gamma_d=2e-05,
         compute_bound_batch_threshold=64, tipping_ms=60000.0 / d) for d in range(1, 9)]


def by_fn(name):
    return [c for c in CASES if c["fn"] == name]


@pytest.mark.parametrize("impl", ["abi", "oracle"])
def test_plan_prefill_scale_down(impl):
    cases = by_fn("plan_prefill_scale_down")
    assert len(cases) >= 300
    for c in cases:
        free = c["free_override"] if c["free_override"] else c["free"]
        lens = [c["input_lens"][r] for r in c["requests"]]
        fn = abi.plan_prefill_scale_down if impl == "abi" else P.plan_prefill_scale_down
        if not c["ok"]:
            with pytest.raises((abi.InfeasiblePlanError, P.InfeasiblePlanError)):
                fn(c["instances"], free, lens)
            continue
        dec, fills, rv = fn(c["instances"], free, lens)
        assert dec == c["decode_instances"]
        assert rv == c["ring_volume"]
        for r, fill in zip(c["requests"], fills):
            want = {i: t for i, t in c["placement"][str(r)]}
            assert P.fill_to_map(fill) == want


@pytest.mark.parametrize("impl", ["abi", "oracle"])
def test_plan_decode_step(impl):
    for c in by_fn("plan_decode_step_core"):
        free = {int(k): v for k, v in c["free"].items()}
        if impl == "abi":
            got = abi.plan_decode_step(c["members"], c["batch_size"], free, c["idle"],
                                       SIB_PATH_ROWS, 1, c["enable_scale_up"])
        else:
            got = P.plan_decode_step(c["members"], c["batch_size"], free, c["idle"],
                                     list(range(1, 9)), 64, c["enable_scale_up"])
        feas, masters, add, idle_after = got
        assert feas == c["feasible"], c
        assert masters == c["masters"], c
        assert add == c["add_instances"], c
        assert idle_after == c["idle_after"], c


@pytest.mark.parametrize("impl", ["abi", "oracle"])
def test_assign_masters_and_comm(impl):
    for c in by_fn("assign_masters+decode_step_comm"):
        want = {int(k): v for k, v in c["assignment"].items()}
        if impl == "abi":
            of = abi.assign_masters(c["batch"], c["masters"])
            got = {m: [] for m in sorted(c["masters"])}
            for r, m in sorted(zip(c["batch"], of)):
                got[m].append(r)
            ms = sorted(got)
            q, o, full = abi.decode_step_comm(len(c["group"]), ms, [len(got[m]) for m in ms],
                                              [c["free"][m] for m in ms])
            ok = full is None
        else:
            got = P.assign_masters(c["batch"], c["masters"])
            free = {i: f for i, f in enumerate(c["free"])}
            ok, full, q, o, app = P.decode_step_comm(len(c["group"]), got, free)
            if ok:
                assert {str(k): v for k, v in app.items()} == c["append_at"]
            full = None if ok else full
        assert got == want
        assert ok == c["ok"]
        if ok:
            assert (q, o) == (c["query_volume"], c["overlappable_volume"])
        else:
            assert full == c["full_master"]


@pytest.mark.parametrize("impl", ["abi", "oracle"])
def test_ring_and_proactive_scale_down(impl):
    for c in by_fn("ring+proactive_scale_down"):
        if impl == "abi":
            rounds, total = abi.build_ring_schedule(c["group"], c["segments"])
        else:
            rounds, total, cov = P.build_ring_schedule(c["group"], c["segments"])
            assert cov == c["coverage"]
        assert [[list(t) for t in rd] for rd in rounds] == c["rounds"][: len(rounds)]
        assert all(len(rd) == 0 for rd in c["rounds"][len(rounds):])
        assert total == c["total_comm_volume"]
        free = {i: f for i, f in enumerate(c["free"])}
        tp = [tuple(x) for x in c["target_placement"]]
        try:
            if impl == "abi":
                ex, buf = abi.proactive_scale_down(c["group"], c["segments"], c["group"],
                                                   c["targets"], tp, free)
            else:
                ex, buf = P.proactive_scale_down(c["group"], c["segments"], c["group"],
                                                 c["targets"], dict(tp), free)
            ok = True
        except (abi.InfeasiblePlanError, P.InfeasiblePlanError):
            ok = False
        assert ok == c["ok"], c
        if ok:
            assert (ex, buf) == (c["extra_migration_volume"], c["transient_buffer_tokens"])


@pytest.mark.parametrize("impl", ["abi", "oracle"])
def test_reactive_migrate(impl):
    for c in by_fn("reactive_migrate"):
        free = {i: f for i, f in enumerate(c["free"])}
        fn = abi.reactive_migrate if impl == "abi" else P.reactive_migrate
        r = fn(c["sources"], c["targets"], c["total"], free) if impl == "abi" else \
            fn(free, c["sources"], c["targets"], c["total"])
        assert r["feasible"] == c["feasible"]
        assert r["per_source_headroom"] == c["per_source_headroom"]
        if c["feasible"]:
            assert [list(x) for x in r["final_placement"]] == c["final_placement"]
            assert r["migration_volume"] == c["migration_volume"]
        else:
            assert r["blocked_instance"] == c["blocked_instance"]


def test_sib_and_footprint():
    for c in by_fn("sib"):
        rec = SIB_PATH_ROWS[c["dop"] - 1]
        s = sum(c["lengths"])
        sq = sum(x * x for x in c["lengths"])
        assert abi.sib_prefill_time(SIB_PATH_ROWS, c["dop"], 1, s, sq) == pytest.approx(c["prefill_ms"], rel=1e-12)
        assert P.sib_prefill_time(rec, s, sq) == pytest.approx(c["prefill_ms"], rel=1e-12)
        assert abi.sib_decode_time(SIB_PATH_ROWS, c["dop"], 1, c["batch"], c["resident"],
                                   c["masters"]) == pytest.approx(c["decode_ms"], rel=1e-12)
        assert P.sib_decode_time(rec, c["batch"], c["resident"], c["masters"]) == pytest.approx(c["decode_ms"], rel=1e-12)
    fp = by_fn("kv_bytes_per_token")[0]
    assert abi.kv_bytes_per_token(2, 512, 8, 2) == fp["tiny"] == 4096
    assert abi.kv_bytes_per_token(32, 4096, 32, 2) == fp["lwm7b"] == 524288
    assert P.kv_bytes_per_token(32, 4096, 32, 2) == 524288
    with pytest.raises(abi.ConfigError):
        abi.kv_bytes_per_token(0, 4096, 32, 2)


# ---- known answers from the reference's own unit tests ------------------------

def test_kat_scale_down_free_432():
    # test_scheduler.cpp:369-399: free {4,3,2}, 6 tokens -> survivors {0,1}, {0:4,1:2}, vol 12
    for fn in (abi.plan_prefill_scale_down, P.plan_prefill_scale_down):
        dec, fills, rv = fn([0, 1, 2], [4, 3, 2], [6])
        assert dec == [0, 1] and P.fill_to_map(fills[0]) == {0: 4, 1: 2} and rv == 12
        dec, _, _ = fn([0, 1, 2], [10, 10, 10], [6])
        assert len(dec) == 1


def test_kat_fig6_and_ring():
    # test_esp_mechanics.cpp:51-73: blocks {3,2,1} -> {4,2}, extra 0, buffer 2
    free = {0: 10, 1: 10, 2: 10}
    assert abi.proactive_scale_down([0, 1, 2], [3, 2, 1], [0, 1, 2], [0, 1], [(0, 4), (1, 2)], free) == (0, 2)
    with pytest.raises(abi.InfeasiblePlanError):
        abi.proactive_scale_down([0, 1, 2], [3, 2, 1], [0, 1, 2], [0, 1], [(0, 4), (1, 2)],
                                 {0: 10, 1: 1, 2: 10})
    # test_esp_mechanics.cpp:26-49: coverage all-ones, volume (d-1)*total
    for d in range(1, 17):
        seg = [100 + 37 * i for i in range(d)]
        rounds, total = abi.build_ring_schedule(list(range(d)), seg)
        assert total == (d - 1) * sum(seg)
        _, _, cov = P.build_ring_schedule(list(range(d)), seg)
        assert all(v == 1 for row in cov for v in row)


def test_kat_reactive():
    # test_esp_mechanics.cpp:116-155
    r = abi.reactive_migrate([0, 1, 2], [2], 600000, {0: 100000, 1: 200000, 2: 400000})
    assert not r["feasible"] and r["blocked_instance"] == 0 and r["per_source_headroom"] == 200000
    assert abi.proactive_scale_down([0, 1, 2], [100000, 200000, 300000], [0, 1, 2], [0, 1, 2],
                                    [(0, 100000), (1, 200000), (2, 300000)],
                                    {0: 100000, 1: 200000, 2: 300000})[0] == 0
    r = abi.reactive_migrate([0, 1, 2, 3], [2, 3], 400, {0: 1000, 1: 1000, 2: 500, 3: 1000})
    assert r["feasible"] and r["migration_volume"] == 200
    assert dict(r["final_placement"]) == {3: 300, 2: 100}


def test_kat_masters():
    # test_esp_mechanics.cpp:157-198
    of = abi.assign_masters([10, 11, 12, 13, 14], [0, 1])
    assert of == [0, 1, 0, 1, 0]
    assert abi.decode_step_comm(4, [0, 1], [4, 4], [1000, 1000])[:2] == (24, 8)
    assert abi.decode_step_comm(2, [0, 1], [2, 1], [0, 10])[2] == 0
    # test_scheduler.cpp:433-481: 65 requests -> 2 masters, 64 -> 1; full group grows
    big = dict(dop=2)
    feas, ms, add, _ = abi.plan_decode_step([0, 1], 65, {0: 200000, 1: 200000}, [], SIB_PATH_ROWS)
    assert feas and len(ms) == 2
    feas, ms, add, _ = abi.plan_decode_step([0, 1], 64, {0: 200000, 1: 200000}, [], SIB_PATH_ROWS)
    assert feas and len(ms) == 1
    feas, ms, add, _ = abi.plan_decode_step([0], 1, {0: 0, 1: 1000}, [1], SIB_PATH_ROWS[:2])
    assert feas and add == [1] and ms == [1]
    feas, _, _, _ = abi.plan_decode_step([0], 1, {0: 0, 1: 1000}, [1], SIB_PATH_ROWS[:2], 1, False)
    assert not feas
    del big
