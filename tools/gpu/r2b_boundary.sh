# threshold boundary through the one-call pipeline with the current kernels (int8 base 256, combined prep)
mkdir -p gpurun_out
for d in 5 10 20; do
  timeout 1500 python -m paper_2603_01443_b200 sweep --family brickwall --q 12:30:2 --c 1:10 --d $d --seeds 0 --reps 2 --jit 2 --cut-path native --out gpurun_out/b_boundary_native_d$d.csv --fit gpurun_out/b_boundary_native_d${d}_fit.json > gpurun_out/b_boundary_d$d.log 2>&1
  echo "d=$d rc=$?"
done
python tools/boundary_table.py gpurun_out/b_boundary_native_d5.csv gpurun_out/b_boundary_native_d10.csv gpurun_out/b_boundary_native_d20.csv
