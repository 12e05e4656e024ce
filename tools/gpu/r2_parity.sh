# round 2: new GPU tests + the rewritten bench
set -x
python -m pytest tests/test_gpu_bench_path.py tests/test_gpu_sharded.py tests/test_gpu_ozaki.py tests/test_cli_harness.py -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2_parity_tests.log
python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
echo "bench rc=$?" >> gpurun_out/r2_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_ref.json 2>&1
tail -c 4000 gpurun_out/r2_bench.json
cat gpurun_out/r2_parity_tests.log
