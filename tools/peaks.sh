nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/peaks tools/micro/peaks.cu && timeout 300 /tmp/peaks > gpurun_out/r02_micro_peaks.json; echo peaks rc=$?
