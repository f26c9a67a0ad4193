# Speculative-offset softmax (ESP_ATTN_SPEC) A/B: kernel tests, then timing.
for sp in 0 1; do
  echo "== SPEC=$sp tests"; ESP_ATTN_SPEC=$sp timeout 300 python -m pytest tests/test_kernels_gpu.py -q -k "ring" 2>&1 | tail -2
done
for r in 1 2; do for sp in 0 1; do for p in 2 3; do
  echo "== SPEC=$sp POLY=$p"; ESP_ATTN_SPEC=$sp ESP_ATTN_POLY=$p timeout 300 python tools/attn_prof.py 2>&1 | grep -E "attn-time|clock" | head -3
done; done; done
for sp in 0 1; do echo "== SPEC=$sp PROF"; ESP_ATTN_SPEC=$sp ESP_ATTN_PROF=1 timeout 300 python tools/attn_prof.py 2>&1 | grep -E "attn-prof" ; done
