# evidence pass: smoke, GPU tests, bench (default + cfg5 q32 c4 + cfg4b), reference arm, launch list -> gpurun_out/e_*
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/e_smoke.log 2>&1
timeout 2000 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/e_gpu_tests.log
timeout 600 python bench.py > gpurun_out/e_bench.json 2> gpurun_out/e_bench.err
echo "bench rc=$?" >> gpurun_out/e_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/e_bench_ref.json 2>&1
timeout 600 python bench.py --workload cfg5_q32_n2_c4 > gpurun_out/e_bench_q32c4.json 2> gpurun_out/e_bench_q32c4.err
timeout 600 python bench.py --workload cfg4b > gpurun_out/e_bench_cfg4b.json 2> gpurun_out/e_bench_cfg4b.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/e_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-uncut --no-cold > /dev/null 2>&1
tail -3 gpurun_out/e_gpu_tests.log; tail -1 gpurun_out/e_smoke.log; tail -2 gpurun_out/e_bench.err
