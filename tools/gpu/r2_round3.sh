set -x
T="timeout 900"
$T python -m pytest tests/test_gpu_jit.py tests/test_gpu_ozaki.py tests/test_gpu_edges.py tests/test_reference_suite.py tests/test_gpu_bench_path.py -m gpu -q 2>&1 | tail -25 > gpurun_out/r3_tests.log
$T python tools/ozaki_digits.py > gpurun_out/r3_ozaki_digits.txt 2>&1
$T python tools/sub_stage_launches.py --steps 5 > gpurun_out/r3_sub_stage.txt 2>&1
$T ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 12 --launch-count 24 --csv --log-file gpurun_out/r3_sub_launches.csv python tools/sub_stage_launches.py --steps 2 > /dev/null 2>&1
$T python tools/api_path_profile.py > gpurun_out/r3_api_profile.txt 2>&1
$T python bench.py --steps 10 --warmup 3 > gpurun_out/r3_bench.json 2> gpurun_out/r3_bench.err
echo "bench rc=$?" >> gpurun_out/r3_bench.err
cat gpurun_out/r3_tests.log gpurun_out/r3_ozaki_digits.txt gpurun_out/r3_sub_stage.txt
