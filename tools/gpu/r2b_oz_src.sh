mkdir -p gpurun_out
./tools/tmem_ld_bw > gpurun_out/tmem_bw.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ozaki_merge_kernel -s 1 -c 1 -o gpurun_out/b_oz16 python tools/ozaki_one.py 16 7 > gpurun_out/b_oz16.log 2>&1
echo done
