"""Edge cases of the ESP data path on a B200, checked against the dense CPU
oracle (same tolerances as tests/test_e2e_gpu.py): one-token prompts on rings
wider than the prompt (empty stripes), ragged multi-request ring batches,
split-KV chunk boundaries, and the capacity / MasterFull error paths of the
reference taxonomy (cluster.hpp:95-98, esp_mechanics.hpp:104-110)."""
import numpy as np
import pytest

from paper_2404_09526_b200 import abi
from tests.devices import devices
from tests.test_e2e_gpu import check_against_oracle

pytestmark = pytest.mark.gpu


def prompt(n, seed):
    return np.random.default_rng(seed).integers(0, abi.TINY.vocab, n).astype(np.int32)


@pytest.mark.parametrize("d", [1, 4])
def test_one_token_prompt(d):
    """S = 1: at d = 4 three ring positions hold no stripe of the request."""
    p = prompt(1, 3)
    rt = abi.Runtime(abi.TINY, d, devices=devices(d), kv_capacity=64)
    first, lg, _ = rt.prefill([0], [1], list(range(d)), [[(d - 1, 1)]], tokens=p, want_logits=True)
    assert rt.placement(0) == {d - 1: 1}
    toks, lgs = [int(first[0])], [lg[0]]
    for _ in range(3):
        out, lg, _ = rt.decode_step([d - 1], [d - 1], [0], want_logits=True)
        toks.append(int(out[0]))
        lgs.append(lg[0])
    rt.check_conservation()
    check_against_oracle(abi.TINY, p, toks, lgs)


def test_ragged_ring_batch_multi_master():
    """Five requests of 1..1030 tokens in ONE ring prefill at d = 4 (stripes
    of 0..258 rows, several empty), retained over two survivors with one
    cursor shared across the batch (scheduler.cpp:694-709), then multi-master
    decode steps over the survivors."""
    lens = [1030, 257, 130, 3, 1]
    ids = [10, 11, 12, 13, 14]
    prompts = {r: prompt(n, 100 + r) for r, n in zip(ids, lens)}
    rt = abi.Runtime(abi.TINY, 4, devices=[0] * 4, kv_capacity=1100)
    # fill survivors 3 (1000 of its 1100 slots) then 1 in request order, one
    # cursor across the batch; both keep room for the decode appends
    retain, room, cur = [], {3: 1000, 1: 1000}, [3, 1]
    ci = 0
    for n in lens:
        parts, left = [], n
        while left:
            take = min(left, room[cur[ci]])
            if take:
                parts.append((cur[ci], take))
                room[cur[ci]] -= take
                left -= take
            if room[cur[ci]] == 0:
                ci += 1
        retain.append(parts)
    toks = np.concatenate([prompts[r] for r in ids])
    first, lg, _ = rt.prefill(ids, lens, [0, 1, 2, 3], retain, tokens=toks, want_logits=True)
    for r, parts in zip(ids, retain):
        want = {}
        for i, t in parts:
            want[i] = want.get(i, 0) + t
        assert rt.placement(r) == want
    seq = {r: ([int(first[i])], [lg[i]]) for i, r in enumerate(ids)}
    for _ in range(2):
        out, lg2, _ = rt.decode_step([1, 3], [1, 3], ids, want_logits=True)
        for i, r in enumerate(ids):
            seq[r][0].append(int(out[i]))
            seq[r][1].append(lg2[i])
    rt.check_conservation()
    for r, n in zip(ids, lens):
        check_against_oracle(abi.TINY, prompts[r], seq[r][0], seq[r][1])


@pytest.mark.parametrize("n", [511, 512, 513, 1024])
def test_split_kv_chunk_boundaries(n):
    """A request's KV of n tokens split 2:1 over two instances, n around the
    512-slot split-KV chunk: chunk partials are LSE-combined at the master."""
    p = prompt(n, n)
    a = (2 * n) // 3
    rt = abi.Runtime(abi.TINY, 2, devices=devices(2), kv_capacity=2048)
    first, lg, _ = rt.prefill([1], [n], [0, 1], [[(0, a), (1, n - a)]], tokens=p, want_logits=True)
    out, lg2, _ = rt.decode_step([0, 1], [1], [1], want_logits=True)
    check_against_oracle(abi.TINY, p, [int(first[0]), int(out[0])], [lg[0], lg2[0]])


def test_capacity_and_master_full_errors():
    """A placement past an instance's slots is refused before any kernel runs
    (CapacityError, AllocResult{ok=false}); a decode step whose master has no
    free slot for the appended token raises MasterFull
    (DecodeCommResult{ok=false}); the page tables are left untouched."""
    rt = abi.Runtime(abi.TINY, 2, devices=devices(2), kv_capacity=100)
    with pytest.raises(abi.CapacityError):
        rt.prefill([0], [101], [0, 1], [[(0, 101)]], tokens=prompt(101, 1))
    assert rt.kv_used() == [0, 0]
    rt.prefill([1], [100], [0, 1], [[(0, 100)]], tokens=prompt(100, 2))
    with pytest.raises(abi.MasterFullError):
        rt.decode_step([0], [0], [1])
    assert rt.placement(1) == {0: 100}
    rt.check_conservation()
    out, _, _ = rt.decode_step([0, 1], [1], [1])  # master with room: the append goes to 1
    assert rt.placement(1) == {0: 100, 1: 1}


def test_kv_slabs_mapped_for_every_runtime_gpu():
    """The VMM-backed KV slabs grant read/write to every GPU of the runtime
    (cuMemGetAccess on every mapped chunk), so a cross-GPU push into a
    survivor's slab, a chunk gather or a KV move never faults. On a one-GPU
    box: the owner; with >= 2 GPUs: instance 0's slab from GPU 1 as well,
    after a ring prefill whose K/V rest on instance 0."""
    import torch

    n_gpu = torch.cuda.device_count()
    devs = [0, 1] if n_gpu >= 2 else [0, 0]
    p = prompt(700, 9)
    rt = abi.Runtime(abi.TINY, 2, devices=devs, kv_capacity=1024)
    rt.prefill([0], [700], [0, 1], [[(0, 700)]], tokens=p)
    for dev in sorted(set(devs)):
        assert rt.slab_access(0, dev), dev
    st = rt.last_prefill_stats()
    assert st["ring_volume_tokens"] == 700 and st["extra_migration_tokens"] == 0
    rt.close()
