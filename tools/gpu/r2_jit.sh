set -x
python -m pytest tests/test_gpu_jit.py tests/test_gpu_bench_path.py -m gpu -x -q 2>&1 | tail -8 > gpurun_out/r2_jit_tests.log
python tools/sub_stage_launches.py --steps 5 > gpurun_out/r2_sub_stage.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 12 --launch-count 24 --csv --log-file gpurun_out/r2_sub_launches.csv python tools/sub_stage_launches.py --steps 2 > /dev/null 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err
echo "bench rc=$?" >> gpurun_out/r2_bench2.err
cat gpurun_out/r2_jit_tests.log gpurun_out/r2_sub_stage.txt
