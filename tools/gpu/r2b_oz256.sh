# ncu --set full of the default int8 merge (base 256) at q=30 K=16 and q=32 K=16
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ozaki_merge_kernel -s 1 -c 1 -o gpurun_out/b_oz256_k16 python tools/ozaki_one.py 16 8 > gpurun_out/b_oz256.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:ozaki_merge_kernel -s 1 -c 1 -o gpurun_out/b_oz256_k64 python tools/ozaki_one.py 64 8 >> gpurun_out/b_oz256.log 2>&1
echo done
