# round-2 (session b) evidence pass: smoke, GPU tests, bench (+ reference arm), launch list
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/b_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/b_smoke.log 2>&1
timeout 2000 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider 2>&1 | tail -40 > gpurun_out/b_gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/b_bench.json 2> gpurun_out/b_bench.err
echo "bench rc=$?" >> gpurun_out/b_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/b_bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/b_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-uncut --no-cold > /dev/null 2>&1
tail -3 gpurun_out/b_gpu_tests.log; cat gpurun_out/b_smoke.log | tail -2; cat gpurun_out/b_bench.json
