# In-step A/B of the exp split (ESP_ATTN_POLY) under the power cap
for r in 1 2; do for p in 1 2 3; do
  ESP_ATTN_POLY=$p timeout 600 python bench.py --skip-cpu --skip-decode --skip-esp-sweep --skip-config3 --skip-scale-down --steps 4 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('POLY=$p', round(d['value']), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])"
done; done
