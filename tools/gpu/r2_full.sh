# full evidence pass: GPU tests, bench (+ reference arm), launch list, sanitizers, API-vs-native sweep
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -25 > gpurun_out/full_gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/full_bench.json 2> gpurun_out/full_bench.err
echo "bench rc=$?" >> gpurun_out/full_bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/full_bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/full_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-uncut --no-cold > /dev/null 2>&1
timeout 900 python -m paper_2603_01443_b200 sweep --family brickwall --q 24 --c 1:6 --d 10 --seeds 0 --reps 3 --jit 2 --cut-path api --out gpurun_out/full_sweep_api_d10.csv > gpurun_out/full_sweep.log 2>&1
timeout 900 python -m paper_2603_01443_b200 sweep --family brickwall --q 24 --c 1:6 --d 10 --seeds 0 --reps 3 --jit 2 --cut-path native --out gpurun_out/full_sweep_native_d10.csv >> gpurun_out/full_sweep.log 2>&1
bash tools/gpu/sanitize.sh
cat gpurun_out/full_gpu_tests.log
