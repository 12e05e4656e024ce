set -x
T="timeout 900"
$T python -m pytest tests/test_gpu_jit.py -m gpu -q -x 2>&1 | tail -30 > gpurun_out/r5_jit_tests.log
$T python tools/sub_stage_launches.py --steps 5 > gpurun_out/r5_sub_stage.txt 2>&1
$T python -m pytest tests/test_gpu_edges.py tests/test_reference_suite.py tests/test_gpu_bench_path.py tests/test_gpu_ozaki.py -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r5_tests.log
cat gpurun_out/r5_jit_tests.log gpurun_out/r5_sub_stage.txt gpurun_out/r5_tests.log
