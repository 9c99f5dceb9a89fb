timeout 900 python -m pytest tests/test_gpu_gemm_ln.py tests/test_gpu_layer.py -m gpu -x -q 2>&1 | tail -1
for i in 1 2; do timeout 300 python tools/stage_times.py --only gemm_o_ln1,gemm_ffn2_ln2; done
BITS=4 T=440 BS=16 timeout 300 python tools/small_stage_graph.py 2>&1 | tail -1
