set -x
timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_reference_suite.py tests/test_gpu_edges.py tests/test_gpu_ozaki.py -m gpu -q -x --timeout 300 2>&1 | tail -15 > gpurun_out/r8_tests.log
timeout 300 python tools/cluster_sizes.py > gpurun_out/r8_cluster_sizes.txt 2>&1
timeout 300 python tools/cluster_sizes.py cfg5_q32_n2_c2 >> gpurun_out/r8_cluster_sizes.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 3 --launch-count 6 --csv --log-file gpurun_out/r8_sub_launches.csv python tools/sub_stage_launches.py --steps 2 > /dev/null 2>&1
timeout 300 python tools/ozaki_digits.py > gpurun_out/r8_ozaki_digits.txt 2>&1
cat gpurun_out/r8_tests.log gpurun_out/r8_cluster_sizes.txt gpurun_out/r8_ozaki_digits.txt
