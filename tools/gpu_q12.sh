mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -m gpu -x -q > gpurun_out/q12_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/q12_tests.log
for b in 4 8; do BITS=$b T=440 BS=16 timeout 300 python tools/small_stage_graph.py; done 2>&1 | tee gpurun_out/q12_small_stages.log
BUILD_ONLY=1 python tools/trace_small.py >/dev/null 2>&1
for sh in 440,2304,768 440,768,768; do for b in 4 8; do
  NO_BUILD=1 SHAPE=$sh BITS=$b timeout 120 python tools/trace_small.py; done; done > gpurun_out/q12_trace.log 2>&1
grep -E "shape|cta   0|entry" gpurun_out/q12_trace.log
