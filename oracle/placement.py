"""Placement oracle — TEST INFRASTRUCTURE ONLY.

Pure-Python restatement of the reference's hot-path placement mechanics
(/root/reference/proj/src, read-only), each function citing the lines it
follows. Pinned by tests/test_placement_oracle.py against
tests/golden/mechanics_random.jsonl, which oracle/golden_driver.cpp generated
by running the reference library itself (oracle/Makefile builds it into
oracle/_ref/). Used by tests to derive expected page-table contents; the
product path (paper_2404_09526_b200) never imports it.
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple


class InfeasiblePlanError(Exception):
    pass


class InternalError(Exception):
    pass


def kv_bytes_per_token(layers: int, hidden_dim: int, kv_heads: int, bpe: int) -> int:
    # cluster.cpp:23-34
    if min(layers, hidden_dim, kv_heads, bpe) <= 0:
        raise ValueError("model config fields must be positive")
    return 2 * layers * hidden_dim * bpe


def plan_prefill_scale_down(instances: Sequence[int], free: Sequence[int],
                            input_lens: Sequence[int]):
    """scheduler.cpp:663-713. Returns (decode_instances, fills, ring_volume);
    fills[r] is the request's (instance, tokens) list in fill order."""
    total = sum(input_lens)
    fr = dict(zip(instances, free))                              # :668-673
    order = sorted(instances, key=lambda i: (-fr[i], i))         # :674-678
    covered, surv = 0, 0
    while surv < len(order) and covered < total:                 # :680-685
        covered += fr[order[surv]]
        surv += 1
    if covered < total:                                          # :686-688
        raise InfeasiblePlanError("batch KV exceeds its instance interval")
    surv = max(surv, 1)                                          # :689
    decode = sorted(order[:surv])                                # :690-691
    room = [fr[order[i]] for i in range(surv)]                   # :694-696
    cursor, fills = 0, []
    for n in input_lens:                                         # :697-710
        rem, fill = n, []
        while rem > 0:
            while cursor < surv and room[cursor] == 0:
                cursor += 1
            if cursor >= surv:
                raise InternalError("scale-down fill overflow")
            take = min(rem, room[cursor])
            fill.append((order[cursor], take))
            room[cursor] -= take
            rem -= take
        fills.append(fill)
    return decode, fills, (len(instances) - 1) * total          # :711-712


def fill_to_map(fill: Sequence[Tuple[int, int]]) -> Dict[int, int]:
    """A fill order as the reference's KvPlacement map (cluster.hpp:44)."""
    out: Dict[int, int] = {}
    for i, t in fill:
        out[i] = out.get(i, 0) + t
    return out


def plan_decode_step(members: List[int], b: int, free: Dict[int, int], idle: List[int],
                     sib_dops: Sequence[int], threshold: int = 64,
                     enable_scale_up: bool = True):
    """scheduler.cpp:726-804 (sib rows exist for widths in sib_dops, all with
    the same compute_bound_batch_threshold). Returns
    (feasible, masters, add_instances, idle_after)."""
    members = list(members)
    idle = list(idle)
    add: List[int] = []
    if b == 0:                                                   # :735
        return False, [], [], idle
    thr = threshold if len(members) in sib_dops else 0           # :737-740

    def take_idle() -> Optional[int]:                            # :745-753
        if not enable_scale_up or not idle or (len(members) + 1) not in sib_dops:
            return None
        return idle.pop(0)

    if thr > 0 and b > thr:                                      # :757-765
        wanted = (b + thr - 1) // thr
        while len(members) < wanted:
            a = take_idle()
            if a is None:
                break
            members.append(a)
            add.append(a)

    def feasible(k: int) -> Optional[List[int]]:                 # :767-784
        order = sorted(members, key=lambda i: (-free[i], i))
        if k > len(order):
            return None
        chosen = sorted(order[:k])
        base, extra = divmod(b, k)
        for i, m in enumerate(chosen):
            if free[m] < base + (1 if i < extra else 0):
                return None
        return chosen

    while True:                                                  # :786-802
        k_start = 1
        if thr > 0 and b > thr:
            k_start = min((b + thr - 1) // thr, len(members))
        for k in range(k_start, len(members) + 1):
            ch = feasible(k)
            if ch is not None:
                return True, ch, add, idle
        a = take_idle()
        if a is None:
            break
        members.append(a)
        add.append(a)
    return False, [], add, idle


def assign_masters(batch: Sequence[int], masters: Sequence[int]) -> Dict[int, List[int]]:
    """esp_mechanics.cpp:220-238."""
    if not masters:
        raise InfeasiblePlanError("no master instances")
    ms = sorted(masters)
    out: Dict[int, List[int]] = {m: [] for m in ms}
    for r in sorted(batch):
        best = ms[0]
        for m in ms:
            if len(out[m]) < len(out[best]):
                best = m
        out[best].append(r)
    return out


def decode_step_comm(d: int, assignment: Dict[int, List[int]], free: Dict[int, int]):
    """esp_mechanics.cpp:240-264 -> (ok, full_master, query_vol, overlap_vol, append_at)."""
    b = sum(len(v) for v in assignment.values())
    qv = b * (d - 1)
    ov = b * (len(assignment) - 1 if assignment else 0)
    append_at = {}
    for m in sorted(assignment):
        reqs = assignment[m]
        if not reqs:
            continue
        if free[m] < len(reqs):
            return False, m, qv, ov, {}
        for r in reqs:
            append_at[r] = m
    return True, -1, qv, ov, append_at


def build_ring_schedule(group: Sequence[int], segments: Sequence[int]):
    """esp_mechanics.cpp:45-70 -> rounds[r] = [(from, to, volume)]; plus
    total volume (:24-30) and coverage (:32-43)."""
    if not group:
        raise InfeasiblePlanError("ring over an empty group")
    if len(group) != len(segments):
        raise InfeasiblePlanError("one segment size per ring instance required")
    if any(s < 0 for s in segments):
        raise InfeasiblePlanError("negative ring segment")
    d = len(group)
    rounds = []
    for r in range(d - 1):
        rounds.append([(group[i], group[(i + 1) % d], segments[(i - r) % d]) for i in range(d)])
    total = sum(v for rd in rounds for (_, _, v) in rd)
    cov = [[0] * d for _ in range(d)]
    for r in range(d):
        for i in range(d):
            cov[i][(i - r) % d] += 1
    return rounds, total, cov


def proactive_scale_down(ring: Sequence[int], segments: Sequence[int], sources, targets,
                         target_placement: Dict[int, int], free: Dict[int, int]):
    """esp_mechanics.cpp:78-136 -> (extra_migration_volume, transient_buffer)."""
    src = set(ring)
    if len(sources) != len(src) or any(s not in src for s in sources):
        raise InfeasiblePlanError("plan sources disagree with the ring group")
    if not targets:
        raise InfeasiblePlanError("plan keeps no target instance")
    if len(targets) > len(src):
        raise InfeasiblePlanError("plan targets exceed the prefill group")
    tg = set(targets)
    if any(t not in src for t in tg):
        raise InfeasiblePlanError("target outside the prefill group")
    circulated = sum(segments)
    if sum(target_placement.values()) != circulated:
        raise InfeasiblePlanError("plan retains a different token count than prefilled")
    per: Dict[int, int] = {}
    for inst, tok in target_placement.items():
        if tok < 0:
            raise InfeasiblePlanError("negative target share")
        if tok > 0 and inst not in tg:
            raise InfeasiblePlanError("placement lands outside target instances")
        per[inst] = per.get(inst, 0) + tok
    for inst, tok in per.items():
        if tok > free.get(inst, 0):
            raise InfeasiblePlanError("target lacks free slots")
    d = len(ring)
    return 0, (circulated + d - 1) // d


def reactive_migrate(free: Dict[int, int], sources, targets, total: int):
    """esp_mechanics.cpp:138-218."""
    if not sources:
        raise InfeasiblePlanError("no source instances")
    if total < 0:
        raise InfeasiblePlanError("negative token total")
    for t in targets:
        if t not in sources:
            raise InfeasiblePlanError("reactive targets must survive from the sources")
    d = len(sources)
    share = (total + d - 1) // d
    res = dict(feasible=False, blocked_instance=-1, per_source_headroom=share,
               final_placement=[], migration_volume=0)
    for s in sources:
        if free[s] < share:
            res["blocked_instance"] = s
            return res
    held, rem = {}, total
    for s in sources:
        held[s] = min(share, rem)
        rem -= held[s]
    if not targets:
        raise InfeasiblePlanError("reactive migration keeps no target instance")
    order = sorted(targets, key=lambda i: (-(free[i] - held[i]), i))
    moving = sum(held[s] for s in sources if s not in set(targets))
    res["migration_volume"] = moving
    final = {t: held[t] for t in targets}
    for t in order:
        if moving == 0:
            break
        take = min(free[t] - final[t], moving)
        if take > 0:
            final[t] += take
            moving -= take
    if moving > 0:
        res["blocked_instance"] = order[-1]
        return res
    res["feasible"] = True
    res["final_placement"] = [(i, t) for i, t in sorted(final.items()) if t > 0]
    return res


def sib_prefill_time(rec: dict, sum_len: float, sum_sq: float) -> float:
    # cost_model.cpp:169-173
    return rec["alpha_p"] + rec["beta_p"] * sum_len + rec["gamma_p"] * sum_sq


def sib_decode_time(rec: dict, b: int, resident: int, k: int) -> float:
    # cost_model.cpp:175-187
    beta = rec["beta_d"] * b
    if b > rec.get("compute_bound_batch_threshold", 64):
        beta /= k
    return rec["alpha_d"] + beta + rec["gamma_d"] * resident / rec["dop"]
