set -x
T="timeout 900"
$T python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_edges.py tests/test_reference_suite.py tests/test_gpu_bench_path.py tests/test_gpu_jit.py tests/test_cli_harness.py -m gpu -q -x 2>&1 | tail -25 > gpurun_out/r4_tests.log
$T python tools/ozaki_digits.py > gpurun_out/r4_ozaki_digits.txt 2>&1
$T python tools/sub_stage_launches.py --steps 5 > gpurun_out/r4_sub_stage.txt 2>&1
$T ncu --set full --clock-control none --import-source on -k regex:ozaki_merge_kernel -s 1 -c 1 -o gpurun_out/r4_oz16_b256 python tools/ozaki_one.py 16 8 > gpurun_out/r4_ncu1.log 2>&1
$T ncu --set full --clock-control none --import-source on -k regex:ozaki_merge_kernel -s 1 -c 1 -o gpurun_out/r4_oz16_b128 python tools/ozaki_one.py 16 7 > gpurun_out/r4_ncu2.log 2>&1
$T python bench.py --steps 10 --warmup 3 > gpurun_out/r4_bench.json 2> gpurun_out/r4_bench.err
echo "bench rc=$?" >> gpurun_out/r4_bench.err
cat gpurun_out/r4_tests.log gpurun_out/r4_ozaki_digits.txt gpurun_out/r4_sub_stage.txt
