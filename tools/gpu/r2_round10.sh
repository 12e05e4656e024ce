set -x
timeout 300 python tools/cluster_sizes.py cfg4a > gpurun_out/r10_cluster_sizes.txt 2>&1
timeout 300 python tools/cluster_sizes.py cfg4a 2 >> gpurun_out/r10_cluster_sizes.txt 2>&1
timeout 300 python tools/cluster_sizes.py cfg4a 4 >> gpurun_out/r10_cluster_sizes.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:cs_jit_k --launch-skip 2 -c 1 -o gpurun_out/r10_cluster_rb2 python tools/cluster_sizes.py cfg4a 2 > /dev/null 2>&1
cat gpurun_out/r10_cluster_sizes.txt
