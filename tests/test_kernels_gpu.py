"""Kernel-level parity of the sm_100a kernels against plain PyTorch fp32
references of the same ops (floating-point kernels; tolerances stated)."""
import math

import pytest
import torch

from paper_2404_09526_b200 import abi

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return (a.float() - b.float()).norm().item() / max(b.float().norm().item(), 1e-12)


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 128), (1000, 1536, 512),
                                   (4096, 4096, 4096), (16, 12288, 4096), (3, 32000, 512),
                                   (300, 384, 192)])
def test_gemm_store(M, N, K):
    torch.manual_seed(0)
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    d = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    abi.k_gemm(a.data_ptr(), b.data_ptr(), d.data_ptr(), M, N, K, 0)
    torch.cuda.synchronize()
    ref = a.float() @ b.float().t()
    assert _rel(d, ref) < 1e-2  # bf16 output rounding


def test_gemm_f32_and_residual():
    torch.manual_seed(1)
    M, N, K = 257, 512, 256
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    d = torch.empty(M, N, device="cuda", dtype=torch.float32)
    abi.k_gemm(a.data_ptr(), b.data_ptr(), d.data_ptr(), M, N, K, 2)
    torch.cuda.synchronize()
    ref = a.float() @ b.float().t()
    assert _rel(d, ref) < 1e-5  # fp32 accumulate, fp32 output
    r = torch.randn(M, N, device="cuda", dtype=torch.bfloat16)
    d2 = r.clone()
    abi.k_gemm(a.data_ptr(), b.data_ptr(), d2.data_ptr(), M, N, K, 1)
    torch.cuda.synchronize()
    assert _rel(d2, r.float() + ref) < 1e-2


@pytest.mark.parametrize("M,N,K", [(16, 4096, 4096), (16, 4096, 11008), (1, 512, 1536),
                                   (32, 1024, 640)])
def test_gemm_skinny_splitk_residual(M, N, K):
    """Decode-shaped residual GEMMs take the skinny stream-K path (fp32
    reduction in a workspace, then the residual add in the finalize)."""
    torch.manual_seed(M + N + K)
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    r = torch.randn(M, N, device="cuda", dtype=torch.bfloat16)
    d = r.clone()
    for _ in range(2):  # second call checks the workspace was re-zeroed
        d = r.clone()
        abi.k_gemm(a.data_ptr(), b.data_ptr(), d.data_ptr(), M, N, K, 1)
    torch.cuda.synchronize()
    assert _rel(d, r.float() + a.float() @ b.float().t()) < 1e-2


@pytest.mark.parametrize("M", [1, 16, 32])
@pytest.mark.parametrize("epi", [0, 1, 2, 3])
@pytest.mark.parametrize("mode", ["streamk", "tiles", "auto"])
def test_gemm_skinny_epilogues(M, epi, mode, monkeypatch):
    """Decode-shaped GEMMs, all skinny schedules: stream-K (per-segment fp32
    partial slots, the CTA completing a tile sums them and applies the fused
    epilogue), whole tiles, and the production dispatch ("auto": the 172-tile
    gate_up shape runs as persistent CTA pairs splitting each tile's K, the
    partner's partial added over DSMEM); store, residual, fp32, SiLU(gate)*up."""
    torch.manual_seed(M * 10 + epi)
    N, K = 22016 if epi == 3 else 12288, 4096
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) * 0.05
    ncols = N // 2 if epi == 3 else N
    r = torch.randn(M, ncols, device="cuda", dtype=torch.bfloat16)
    for _ in range(2):  # second call checks the tile counters were reset
        d = r.clone() if epi == 1 else torch.empty(
            M, ncols, device="cuda", dtype=torch.float32 if epi == 2 else torch.bfloat16)
        abi.k_gemm(a.data_ptr(), b.data_ptr(), d.data_ptr(), M, N, K, epi, path=mode)
    torch.cuda.synchronize()
    ref = a.float() @ b.float().t()
    if epi == 1:
        ref = r.float() + ref
    if epi == 3:
        g = ref.view(M, -1, 2, 64)
        ref = (torch.nn.functional.silu(g[:, :, 0]) * g[:, :, 1]).reshape(M, ncols)
    assert _rel(d, ref) < (1e-5 if epi == 2 else 1e-2)


def test_gemm_silu_mul():
    torch.manual_seed(2)
    M, F, K = 200, 384, 256
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    g = torch.randn(F, K, device="cuda", dtype=torch.bfloat16) * 0.1
    u = torch.randn(F, K, device="cuda", dtype=torch.bfloat16) * 0.1
    # physical layout: 128-row blocks of 64 gate rows then 64 up rows
    w = torch.cat([torch.cat([g[i:i + 64], u[i:i + 64]]) for i in range(0, F, 64)])
    d = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)
    abi.k_gemm(a.data_ptr(), w.data_ptr(), d.data_ptr(), M, 2 * F, K, 3)
    torch.cuda.synchronize()
    gg = a.float() @ g.float().t()
    uu = a.float() @ u.float().t()
    ref = torch.nn.functional.silu(gg) * uu
    assert _rel(d, ref) < 1e-2


@pytest.mark.parametrize("M,N,K,epi", [(4096, 4096, 512, 0), (4000, 4096, 320, 1),
                                       (9000, 2560, 256, 2), (4097, 4608, 192, 3)])
def test_gemm_cta_pair_matches_single_cta(M, N, K, epi, monkeypatch):
    """Large GEMMs run on CTA pairs (tcgen05.mma.cta_group::2, 256 x 256
    tiles). Same K order as the 1-CTA kernel, so outputs are bit-identical;
    both also match the fp32 reference."""
    torch.manual_seed(M + N)
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) * 0.1
    odt = torch.float32 if epi == 2 else torch.bfloat16
    ncols = N // 2 if epi == 3 else N
    r = torch.randn(M, ncols, device="cuda", dtype=torch.bfloat16)
    outs = []
    for path in ("auto", "no_pair"):
        d = r.clone() if epi == 1 else torch.empty(M, ncols, device="cuda", dtype=odt)
        abi.k_gemm(a.data_ptr(), b.data_ptr(), d.data_ptr(), M, N, K, epi, path=path)
        torch.cuda.synchronize()
        outs.append(d)
    assert torch.equal(outs[0], outs[1])
    ref = a.float() @ b.float().t()
    if epi == 1:
        ref = r.float() + ref
    elif epi == 3:
        g = ref.view(M, -1, 2, 64)
        ref = (torch.nn.functional.silu(g[:, :, 0]) * g[:, :, 1]).reshape(M, ncols)
    assert _rel(outs[0], ref) < (1e-5 if epi == 2 else 1e-2)


def _ref_striped(q, ks, vs, pos_i, d, origins, heads, hd):
    """fp32 reference: query stripe a (position a*d+pos_i) vs key stripe b of
    origin o (position b*d+o): visible iff b*d+o <= a*d+pos_i."""
    L = q.shape[0]
    qf = q.float().view(L, heads, hd)
    kk, vv, kp = [], [], []
    for k, v, o in zip(ks, vs, origins):
        n = k.shape[0]
        kk.append(k.float().view(n, heads, hd))
        vv.append(v.float().view(n, heads, hd))
        kp.append(torch.arange(n, device=q.device) * d + o)
    K = torch.cat(kk)
    V = torch.cat(vv)
    KP = torch.cat(kp)
    QP = torch.arange(L, device=q.device) * d + pos_i
    s = torch.einsum("qhd,khd->hqk", qf, K) / math.sqrt(hd)
    mask = KP[None, :] <= QP[:, None]
    s = s.masked_fill(~mask[None], float("-inf"))
    p = torch.softmax(s, dim=-1)
    return torch.einsum("hqk,khd->qhd", p, V).reshape(L, heads * hd)


@pytest.mark.parametrize("S,d,pos_i,heads,hd", [(128, 1, 0, 2, 128), (1000, 1, 0, 4, 128),
                                                (4096, 1, 0, 8, 64), (2000, 2, 0, 4, 128),
                                                (2001, 2, 1, 4, 128), (3000, 4, 2, 2, 64),
                                                (5000, 8, 5, 2, 128), (700, 8, 0, 3, 128),
                                                (77, 4, 3, 2, 64), (1500, 3, 2, 2, 128)])
def test_ring_attention_striped(S, d, pos_i, heads, hd):
    torch.manual_seed(S + d + pos_i)
    H = heads * hd
    lens = [len(range(o, S, d)) for o in range(d)]
    blocks = [(torch.randn(lens[o], H, device="cuda", dtype=torch.bfloat16),
               torch.randn(lens[o], H, device="cuda", dtype=torch.bfloat16)) for o in range(d)]
    q = torch.randn(lens[pos_i], H, device="cuda", dtype=torch.bfloat16)
    origins = [((pos_i - r) % d) for r in range(d)]  # ring round order
    out = torch.empty_like(q)
    abi.k_ring_attention(q.data_ptr(), lens[pos_i], pos_i,
                         [blocks[o][0].data_ptr() for o in origins],
                         [blocks[o][1].data_ptr() for o in origins],
                         [lens[o] for o in origins], origins, out.data_ptr(), heads, hd)
    torch.cuda.synchronize()
    ref = _ref_striped(q, [blocks[o][0] for o in origins], [blocks[o][1] for o in origins],
                       pos_i, d, origins, heads, hd)
    err = (out.float() - ref).abs().max().item()
    assert _rel(out, ref) < 1e-2, err


@pytest.mark.parametrize("hd", [64, 128])
def test_decode_attention_paged(hd):
    torch.manual_seed(hd)
    heads, cap = 4, 5000
    H = heads * hd
    ks = [torch.randn(cap, H, device="cuda", dtype=torch.bfloat16) for _ in range(2)]
    vs = [torch.randn(cap, H, device="cuda", dtype=torch.bfloat16) for _ in range(2)]
    b = 3
    q = torch.randn(b, H, device="cuda", dtype=torch.bfloat16)
    g = torch.Generator().manual_seed(0)
    chunks = []
    for r in range(b):
        for inst in range(2):
            n = [700, 1, 256][r] if inst == 0 else [33, 1000, 0][r]
            if n == 0:
                continue
            slots = torch.randperm(cap, generator=g)[:n].to(torch.int32).cuda()
            chunks.append((r, inst, slots))
    out = torch.empty(b, H, device="cuda", dtype=torch.bfloat16)
    abi.k_decode_attention(q.data_ptr(), b, [ks[c[1]].data_ptr() for c in chunks],
                           [vs[c[1]].data_ptr() for c in chunks],
                           [c[2].data_ptr() for c in chunks], [c[2].numel() for c in chunks],
                           [c[0] for c in chunks], out.data_ptr(), heads, hd)
    torch.cuda.synchronize()
    for r in range(b):
        K = torch.cat([ks[c[1]][c[2].long()] for c in chunks if c[0] == r]).float()
        V = torch.cat([vs[c[1]][c[2].long()] for c in chunks if c[0] == r]).float()
        qq = q[r].float().view(heads, hd)
        s = torch.einsum("hd,khd->hk", qq, K.view(-1, heads, hd)) / math.sqrt(hd)
        p = torch.softmax(s, -1)
        ref = torch.einsum("hk,khd->hd", p, V.view(-1, heads, hd)).reshape(H)
        assert _rel(out[r], ref) < 1e-2
