# bench.py on every BASELINE workload that fits one B200 (N=1)
set -x
for w in cfg4b cfg5_q32_n2_c2 cfg5_q32_n2_c4 cfg5_q32_n4_c4; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/wl_$w.json 2> gpurun_out/wl_$w.err
  echo "$w rc=$?" >> gpurun_out/wl_summary.txt
done
timeout 600 python bench.py --workload cfg5_q32_n2_c4 --impl reference --steps 2 --warmup 1 > gpurun_out/wl_ref_cfg5_q32_n2_c4.json 2>&1
cat gpurun_out/wl_summary.txt
