set -x
timeout 600 python tools/api_path_profile.py 24 4 10 > gpurun_out/r13_api_profile.txt 2>&1
timeout 900 python -m paper_2603_01443_b200 sweep --family brickwall --q 24 --c 1:6 --d 10 --seeds 0 --reps 3 --jit 2 --cut-path api --out gpurun_out/r13_sweep_api_d10.csv > gpurun_out/r13_sweep.log 2>&1
timeout 600 python -m pytest tests/test_gpu_edges.py tests/test_gpu_jit.py tests/test_cli_harness.py tests/test_gpu_sweeps.py tests/test_reference_suite.py -m gpu -q -x --timeout 300 2>&1 | tail -5 > gpurun_out/r13_tests.log
head -40 gpurun_out/r13_api_profile.txt; cat gpurun_out/r13_tests.log
