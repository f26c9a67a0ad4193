# Decode-path ncu evidence: launch list of one bench decode step (serialised,
# cold-cache per-launch times) and full captures of the decode kernels.
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --skip-esp-sweep --skip-cpu --skip-config3 --skip-scale-down --seq 4096"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/decode_launches.csv $B > gpurun_out/prof_decode_l.log 2>&1
for k in decode_attention_kernel decode_combine_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 40 -c 1 \
    -o gpurun_out/prof_$k -f $B > gpurun_out/prof_$k.log 2>&1
done
