# one GPU computes single ranks' shares of the sharded workloads through bench.py's N>1 code path
# (cs_cut_shard_plan, cs_cut_run_sharded with out_range, per-shard parity and e2e) -> gpurun_out/s_*.json
set -x
mkdir -p gpurun_out
run() { timeout 900 python bench.py --workload $1 --emulate-shard $2 $3 > gpurun_out/s_$1_$(echo $2 | tr / of).json 2> gpurun_out/s_$1_$(echo $2 | tr / of).err; echo "rc=$?" >> gpurun_out/s_$1_$(echo $2 | tr / of).err; }
run cfg4a 0/2
run cfg4a 1/2
run cfg4a 0/8
run cfg4a 5/8
run cfg4b 3/8
run cfg5_q32_n2_c2 0/8
run cfg5_q32_n2_c4 7/8
run cfg5_q32_n4_c4 5/8
run cfg5_q34_n2_c2 7/8 --no-e2e
tail -n 2 gpurun_out/s_*.err
