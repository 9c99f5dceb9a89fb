timeout 900 python -m pytest tests/test_gpu_gemm_ln.py tests/test_gpu_layer.py -m gpu -x -q 2>&1 | tail -2
timeout 600 python tools/time_lnc.py
BITS=4 T=440 BS=16 timeout 300 python tools/small_stage_graph.py 2>&1 | tail -1
for sh in 440,768,768; do FUSED_LN=1 NO_BUILD=1 SHAPE=$sh BITS=4 timeout 120 python tools/trace_small.py; done 2>&1 | grep -E "shape|cta   [0-1]:|entry"
