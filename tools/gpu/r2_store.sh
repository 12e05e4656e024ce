timeout 600 ./tools/store_patterns > gpurun_out/r19_store_patterns.txt 2>&1
cat gpurun_out/r19_store_patterns.txt
