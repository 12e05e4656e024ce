# session-b evidence pass 3 (int8 base-256 / unit CTAs default): GPU tests, smoke, bench cfg4a + cfg5 q32 c4, small-q merges, cfg3 sweeps
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/d_smoke.log 2>&1
timeout 2000 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/d_gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/d_bench.json 2> gpurun_out/d_bench.err
echo "bench rc=$?" >> gpurun_out/d_bench.err
timeout 600 python bench.py --workload cfg5_q32_n2_c4 --steps 10 --warmup 3 > gpurun_out/d_bench_q32c4.json 2> gpurun_out/d_bench_q32c4.err
timeout 300 python tools/merge_small_q.py > gpurun_out/d_merge_small_q.txt 2>&1
timeout 900 python -m paper_2603_01443_b200 sweep --family brickwall --q 24 --c 1:6 --d 10 --seeds 0 --reps 3 --jit 2 --cut-path api --out gpurun_out/d_sweep_api_d10.csv > gpurun_out/d_sweep.log 2>&1
timeout 900 python -m paper_2603_01443_b200 sweep --family brickwall --q 24 --c 1:6 --d 10 --seeds 0 --reps 3 --jit 2 --cut-path native --out gpurun_out/d_sweep_native_d10.csv >> gpurun_out/d_sweep.log 2>&1
tail -3 gpurun_out/d_gpu_tests.log; tail -1 gpurun_out/d_smoke.log; tail -2 gpurun_out/d_bench.err
