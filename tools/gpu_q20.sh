timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "requant or gemm" 2>&1 | tail -2
for pr in -1 0; do for b in 4 8; do MKQ_LUT128_PAIRS=$pr BITS=$b T=440 BS=16 timeout 300 python tools/small_stage_graph.py; done; done 2>&1
for pr in -1 0; do MKQ_LUT128_PAIRS=$pr BITS=4 T=681 BS=16 timeout 300 python tools/small_stage_graph.py; done 2>&1
