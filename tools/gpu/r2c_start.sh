# session-c start: re-check of the restored tree (smoke, GPU tests, bench, reference arm, launch list)
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/c_smoke.log 2>&1
timeout 2000 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/c_gpu_tests.log
timeout 600 python bench.py > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err
echo "bench rc=$?" >> gpurun_out/c_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/c_bench_ref.json 2>&1
timeout 600 python bench.py --workload cfg5_q32_n2_c4 > gpurun_out/c_bench_q32c4.json 2> gpurun_out/c_bench_q32c4.err
timeout 600 python bench.py --workload cfg4b > gpurun_out/c_bench_cfg4b.json 2> gpurun_out/c_bench_cfg4b.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-uncut --no-cold > /dev/null 2>&1
tail -3 gpurun_out/c_gpu_tests.log; tail -1 gpurun_out/c_smoke.log; tail -2 gpurun_out/c_bench.err
