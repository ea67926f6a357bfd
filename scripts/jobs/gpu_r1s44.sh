mkdir -p gpurun_out
cd scripts/probes && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --use_fast_math -I../../include -I../../paper_2505_03780_b200/csrc -o /tmp/softmax_probe softmax_probe.cu > /dev/null 2>&1; cd ../..
timeout 120 /tmp/softmax_probe > gpurun_out/r1s44_softmax_probe.txt 2>&1
cat gpurun_out/r1s44_softmax_probe.txt
