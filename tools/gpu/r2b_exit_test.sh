for i in 1 2 3 4 5 6; do CUTSIM_SEGV_TRACE=1 timeout 120 python tools/api_sub_host.py 24 4 10 3 > gpurun_out/exit_$i.log 2>&1; echo "run $i rc=$?"; done
