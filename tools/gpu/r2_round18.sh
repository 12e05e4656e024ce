timeout 600 python -m pytest tests/test_gpu_ozaki.py -m gpu -q -x --timeout 300 2>&1 | tail -2 > gpurun_out/r18.txt
timeout 300 python tools/ozaki_digits.py >> gpurun_out/r18.txt 2>&1
cat gpurun_out/r18.txt
