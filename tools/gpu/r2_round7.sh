set -x
timeout 600 python -m pytest tests/test_gpu_jit.py -m gpu -v -x --timeout 120 -k "cluster or tiered or structure" 2>&1 | tail -80 > gpurun_out/r7_jit.log
cat gpurun_out/r7_jit.log
