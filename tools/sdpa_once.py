"""cuDNN SDPA (causal, 32 x 128, bf16, S=32768) launched a few times — for an
ncu capture of the library's Blackwell attention kernel beside K1's."""
import torch
from torch.nn.attention import SDPBackend, sdpa_kernel

S, HEADS, HD = 32768, 32, 128
q = torch.randn(1, HEADS, S, HD, device="cuda", dtype=torch.bfloat16)
k = torch.randn_like(q)
v = torch.randn_like(q)
with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
    for _ in range(3):
        torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
torch.cuda.synchronize()
print("ok")
