set -x
timeout 600 python -m pytest tests/test_gpu_ozaki.py -m gpu -q -x --timeout 300 2>&1 | tail -5 > gpurun_out/r12_tests.log
timeout 300 python tools/ozaki_digits.py > gpurun_out/r12_ozaki_digits.txt 2>&1
cat gpurun_out/r12_tests.log gpurun_out/r12_ozaki_digits.txt
