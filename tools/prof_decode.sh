# Decode-path ncu evidence: launch list of the decode probe (serialised,
# cold-cache per-launch times) and full captures of the decode kernels.
mkdir -p gpurun_out
STEPS=2 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/decode_launches.csv python tools/decode_probe.py > gpurun_out/prof_decode_l.log 2>&1
for k in decode_attention_kernel gemm_skinny_swap decode_combine_kernel; do
  STEPS=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 40 -c 1 \
    -o gpurun_out/prof_$k -f python tools/decode_probe.py > gpurun_out/prof_$k.log 2>&1
done
# the cluster split-K GEMM (O projection: grid 128)
STEPS=2 timeout 900 ncu --set full --clock-control none -k regex:gemm_skinny_swap --launch-skip 200 -c 8 \
  -o gpurun_out/prof_swap_many -f python tools/decode_probe.py > gpurun_out/prof_swap_many.log 2>&1
ls -la gpurun_out
