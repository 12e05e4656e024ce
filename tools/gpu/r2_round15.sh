timeout 600 python tools/e2e_chunks.py > gpurun_out/r15_e2e_chunks.txt 2>&1
cat gpurun_out/r15_e2e_chunks.txt
