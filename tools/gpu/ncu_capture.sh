# ncu --set full captures of the round's final code (run AFTER evidence_pass.sh exited 0 without ncu):
#   the cfg4a merge launch and one variant-stage cluster kernel inside bench.py, the int8 K=16 merge at q=30.
# Bring gpurun_out/n_*.ncu-rep back and summarise here with
#   python profiles/summarize_ncu.py r02 gpurun_out/n_merge.ncu-rep gpurun_out/n_variant.ncu-rep
#   python profiles/summarize_ncu.py r02_ozaki_k16 gpurun_out/n_oz16.ncu-rep
set -x
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-uncut --no-cold"
timeout 300 $B > gpurun_out/n_plain.json 2> gpurun_out/n_plain.err || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:merge_kernel --launch-skip 4 -c 1 \
  -f -o gpurun_out/n_merge $B > gpurun_out/n_merge.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cs_jit --launch-skip 2 -c 2 \
  -f -o gpurun_out/n_variant $B > gpurun_out/n_variant.log 2>&1
timeout 300 python tools/ozaki_one.py 16 8 > gpurun_out/n_oz16_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ozaki_merge -c 1 --launch-skip 1 \
  -f -o gpurun_out/n_oz16 python tools/ozaki_one.py 16 8 > gpurun_out/n_oz16.log 2>&1
ls -la gpurun_out/n_*
