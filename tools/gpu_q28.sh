timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -m gpu -x -q 2>&1 | tail -2
for b in 4 8; do BITS=$b T=440 BS=16 timeout 300 python tools/small_stage_graph.py; done 2>&1
timeout 900 python bench.py > gpurun_out/q28_bench.json 2> gpurun_out/q28_bench.err; echo bench=$?
