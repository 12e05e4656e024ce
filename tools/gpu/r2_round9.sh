set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cs_jit_k --launch-skip 2 -c 1 -o gpurun_out/r9_cluster_cfg4a python tools/sub_stage_launches.py --steps 1 > gpurun_out/r9_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cs_jit_k --launch-skip 2 -c 1 -o gpurun_out/r9_cluster_cfg5 python tools/sub_stage_launches.py --steps 1 --workload cfg5_q32_n2_c2 > gpurun_out/r9_ncu2.log 2>&1
python - <<'PY' > gpurun_out/r9_occupancy.txt 2>&1
import ctypes, torch
torch.cuda.init()
print(torch.cuda.get_device_properties(0))
PY
tail -3 gpurun_out/r9_ncu1.log gpurun_out/r9_ncu2.log
