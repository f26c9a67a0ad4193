# K1 schedule check: tests, timing, DRAM traffic of one launch
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_e2e_gpu.py -q -x -k "ring or config1 or esp_degree or multi or chunked or lwm7b" 2>&1 | tail -2
for r in 1 2; do timeout 300 python tools/attn_prof.py 2>&1 | grep -E "attn-time"; done
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:ring_attention -c 2 python tools/attn_prof.py 2>&1 | grep -E "dram__|gpu__time|hit_rate" 
