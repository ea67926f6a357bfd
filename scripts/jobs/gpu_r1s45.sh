mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipe_probe scripts/probes/pipe_probe.cu
timeout 120 /tmp/pipe_probe > gpurun_out/r1s45_pipe_probe.txt 2>&1
cat gpurun_out/r1s45_pipe_probe.txt
