timeout 900 python -m pytest tests/test_gpu_gemm_ln.py tests/test_gpu_layer.py -m gpu -x -q 2>&1 | tail -2
timeout 600 python tools/time_lnc.py 2>&1 | grep "N=768"
BITS=4 T=440 BS=16 timeout 300 python tools/small_stage_graph.py 2>&1 | tail -1
