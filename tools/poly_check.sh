# In-step A/B of the exp split (ESP_ATTN_POLY) under the power cap
for r in 1 2; do for p in 0 1 2; do
  ESP_ATTN_POLY=$p timeout 600 python bench.py --skip-cpu --skip-decode --skip-esp-sweep --skip-config3 --skip-scale-down --steps 4 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('POLY=$p', round(d['value']), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])"
done; done
for p in 0 1 2; do echo "alone POLY=$p $(ESP_ATTN_POLY=$p timeout 300 python tools/attn_prof.py 2>&1 | grep attn-time)"; done
ESP_ATTN_PROF=1 timeout 300 python tools/attn_prof.py 2>&1 | grep -E "attn-prof"
