timeout 900 python -m pytest tests/test_gpu_gemm_ln.py -m gpu -x -q 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_layer.py -m gpu -x -q 2>&1 | tail -3
for b in 4 8; do BITS=$b T=440 BS=16 timeout 300 python tools/small_stage_graph.py; done 2>&1
