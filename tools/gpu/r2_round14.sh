timeout 300 python tools/d2h_streams.py > gpurun_out/r14_d2h.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_jit.py -m gpu -q -x --timeout 300 -k "cluster" 2>&1 | tail -3 >> gpurun_out/r14_d2h.txt
cat gpurun_out/r14_d2h.txt
