set -x
free -g; nproc; cat /proc/cpuinfo | grep "model name" | head -1; nvidia-smi --query-gpu=name,memory.total --format=csv
cat /sys/fs/cgroup/memory.max 2>/dev/null
python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r2_first_tests.log
python bench.py --steps 10 --warmup 3 > gpurun_out/r2_first_bench.json 2> gpurun_out/r2_first_bench.err
tail -c 3000 gpurun_out/r2_first_bench.json
