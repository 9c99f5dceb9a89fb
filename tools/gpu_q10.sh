mkdir -p gpurun_out
nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a tools/xu_rate2.cu -o /tmp/xu_rate2 && /tmp/xu_rate2 > gpurun_out/xu_rate2.log 2>&1
for b in 4 8; do BITS=$b T=440 BS=16 timeout 300 python tools/small_stage_graph.py; done > gpurun_out/small_stages.log 2>&1
cat gpurun_out/xu_rate2.log gpurun_out/small_stages.log
