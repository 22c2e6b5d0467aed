mkdir -p gpurun_out
timeout 300 ./tools/microbench_dsmem_stream > gpurun_out/dsmem_stream.txt 2>&1
