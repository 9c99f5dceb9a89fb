timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_gemm_ln.py -m gpu -x -q -k "gemm" 2>&1 | tail -2
for b in 4 8; do BITS=$b T=440 BS=16 timeout 300 python tools/small_stage_graph.py 2>&1 | tail -1; done
for sh in 440,2304,768 440,768,3072; do NO_BUILD=1 SHAPE=$sh BITS=4 timeout 120 python tools/trace_small.py; done 2>&1 | grep -E "shape|cta   [0-1]:|entry"
