mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "gemm" > gpurun_out/q15_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/q15_tests.log
for b in 4 8; do BITS=$b T=440 BS=16 timeout 300 python tools/small_stage_graph.py; done 2>&1
for b in 8 4; do NO_BUILD=1 SHAPE=440,2304,768 BITS=$b timeout 120 python tools/trace_small.py; done 2>&1 | grep -E "shape|cta   [0-1]:|entry"
