set -x
timeout 600 python -m pytest tests/test_gpu_ozaki.py -m gpu -q -x --timeout 300 2>&1 | tail -5 > gpurun_out/r11_tests.log
timeout 300 python tools/ozaki_digits.py > gpurun_out/r11_ozaki_digits.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ozaki_merge_kernel -s 1 -c 1 -o gpurun_out/r11_oz16 python tools/ozaki_one.py 16 7 > /dev/null 2>&1
cat gpurun_out/r11_tests.log gpurun_out/r11_ozaki_digits.txt
