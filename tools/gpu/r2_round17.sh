timeout 600 ncu --set full --clock-control none --import-source on -k regex:ozaki_merge_kernel -s 1 -c 1 -o gpurun_out/r17_oz16 python tools/ozaki_one.py 16 7 > /dev/null 2>&1
echo done
